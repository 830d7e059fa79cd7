"""Generate the golden fixtures from the UNMODIFIED reference library.

Runs oracle/_ref/libskridge_ref.so (built from /root/reference/proj/src by
oracle/Makefile) — never the restatement — and stores inputs and outputs:

  tests/golden/small.npz   small known-answer cases (streams, eigensolver,
                           block_lanczos incl. rank drop, preconditioned
                           components, SVRG trace + index stream, L*, kappa~)
  tests/golden/configs.json  BASELINE configs c1, c2 (c3, c4, c5 row-subsampled to n = 16384; c5 at
                           lambda 1e-6 and 1e-8, and unpreconditioned at 1e-6)
                           composed as SURVEY §0 fact 6 prescribes: sigma~,
                           beta_hat, alpha, eta, per-epoch objectives, L(w^), L*,
                           kappa~ (d <= 2000), index-stream head; inputs come
                           from paper_1602_02350_b200.configs.host_instance.

Usage:  python tests/golden/make_golden.py [small] [c1] [c2] [c3] [c4] [c5]
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1602_02350_b200 import configs  # noqa: E402


def idx_hash(idx: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(idx, dtype=np.int64).tobytes()).hexdigest()


def small():
    R = oracle.ref()
    out = {}
    out["uniforms_0"] = R.uniforms(0, 700)
    out["uniforms_5"] = R.uniforms(5, 700)
    out["uniforms_big"] = R.uniforms(2 ** 40 + 3, 700)
    out["gauss_37x5_42"] = R.gaussian_matrix(37, 5, 42)
    rng = np.random.default_rng(1)
    A = rng.standard_normal((12, 12))
    A = A + A.T
    out["eig_in"] = A
    out["eig_vals"], out["eig_vecs"] = R.sym_eigs(A)

    # block_lanczos cases
    X = rng.standard_normal((400, 30)) * (1.0 / np.arange(1, 31))
    out["bl_X"] = X
    sk = R.block_lanczos(X, 5, q=3, seed=4)
    out["bl_U"], out["bl_sigma"], out["bl_V"] = sk.U, sk.sigma, sk.V
    sk2 = R.block_lanczos(X[:60, :14], 3, q=0, seed=1, scale=1.0)
    out["bl2_sigma"], out["bl2_q"] = sk2.sigma, np.array(sk2.q)
    # rank-3 data: width collapses, rank_reduced
    U3, _ = np.linalg.qr(rng.standard_normal((45, 3)))
    V3, _ = np.linalg.qr(rng.standard_normal((30, 3)))
    X3 = np.ascontiguousarray((U3 * np.array([3.0, 1.5, 0.75])) @ V3.T)
    out["rr_X"] = X3
    sk3 = R.block_lanczos(X3, 5, q=1, seed=4, scale=1.0)
    out["rr_k"], out["rr_reduced"], out["rr_sigma"] = np.array(sk3.k), np.array(sk3.rank_reduced), sk3.sigma

    # preconditioned components on bl_X
    y = rng.standard_normal(400)
    lam = 1e-3
    out["pc_y"], out["pc_lam"] = y, np.array(lam)
    prob = R.problem(X, y, lam, sk.U, sk.sigma, 0)
    out["pc_betas"] = prob.betas()
    a, b, _ = prob.scalars()
    out["pc_alpha"], out["pc_beta_hat"] = np.array(a), np.array(b)
    w = rng.standard_normal(30)
    out["pc_w"] = w
    out["pc_obj"] = np.array(prob.objective(w))
    out["pc_grad"] = prob.full_gradient(w)
    out["pc_cg"] = np.stack([prob.component_gradient(i, w) for i in [0, 7, 400, 429]])
    out["pc_aisq"] = R.apply_inv_sqrt(sk.U, sk.sigma, lam, w)
    # SVRG: 4 epochs, m = 2n, BASELINE step-size rule
    P = oracle.port()  # max row norm of X~ (the reference does not expose X~); checked below
    Pp = P.problem(X, y, lam, sk.U, sk.sigma)
    eta = configs.step_size(Pp.scalars()[2])
    out["sv_eta"] = np.array(eta)
    sv = prob.svrg(4, 800, eta, 13)
    out["sv_trace"], out["sv_iter"] = sv.trace, sv.iterate
    out["sv_idx"] = R.index_stream(prob.betas(), 13, 2000)
    out["cum"] = R.cumulative_weights(prob.betas())
    wmin, lmin = R.reference_minimum(X, y, lam)
    out["refmin_w"], out["refmin_L"] = wmin, np.array(lmin)
    out["kappa"] = np.array(R.conditioned_cond(X, lam, sk.U, sk.sigma))
    out["obj_orig"] = np.array(R.objective(X, y, lam, w))
    # identity preconditioner components
    p0 = R.problem(X, y, lam, None, None, 0)
    out["id_betas"], out["id_grad"] = p0.betas(), p0.full_gradient(w)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    print("small.npz written", len(out), "arrays")


def config_case(name: str, n_override: int | None = None, epochs: int | None = None, kappa: bool = True,
                lam: float | None = None, sketched: bool = True):
    R = oracle.ref()
    cfg = configs.CONFIGS[name]
    if n_override:
        cfg = cfg.scaled(n_override)
    if lam is not None:
        cfg = configs.Config(**{**cfg.__dict__, "lam": lam})
    t0 = time.time()
    X, y = configs.host_instance(cfg)
    Xd = X.astype(np.float64)
    yd = y.astype(np.float64)
    n, d = Xd.shape
    digest = hashlib.sha256(np.ascontiguousarray(X).tobytes()).hexdigest()
    sk = R.block_lanczos(Xd, cfg.k, q=cfg.q, seed=cfg.seed, want_right=False)
    t_l = time.time() - t0
    # unsketched baseline (Preconditioner::identity == RidgeFiniteSum, test_ridge.cpp:109-127)
    prob = R.problem(Xd, yd, cfg.lam, sk.U, sk.sigma, 0) if sketched else R.problem(Xd, yd, cfg.lam, None, None, 0)
    betas = prob.betas()
    alpha, beta_hat, _ = prob.scalars()
    # eta = 1/(4 max_i ||x~_i||^2): ||x~_i||^2 = beta_i n/(n+d) (ridge.cpp:124-127)
    max_row_sq = float(np.max(betas[:n]) * n / (n + d))
    eta = configs.eta_for(cfg, max_row_sq, beta_hat)
    ep = epochs or cfg.epochs
    wmin, Lstar = R.reference_minimum(Xd, yd, cfg.lam)
    sv = prob.svrg(ep, 2 * n, eta, cfg.seed, reference=Lstar)
    w_hat = R.apply_inv_sqrt(sk.U, sk.sigma, cfg.lam, sv.iterate) if sketched else sv.iterate
    L = R.objective(Xd, yd, cfg.lam, w_hat)
    idx = R.index_stream(betas, cfg.seed, 100000)
    rec = {
        "config": name, "n": n, "d": d, "dtype": cfg.dtype, "k": cfg.k if sketched else 0, "q": cfg.q, "lambda": cfg.lam,
        "seed": cfg.seed, "epochs": ep, "m": 2 * n, "x_sha256": digest,
        "sigma": sk.sigma.tolist(), "k_used": sk.k, "alpha": alpha, "beta_hat": beta_hat,
        "max_row_sq": max_row_sq, "eta": eta, "trace": sv.trace.tolist(), "L_hat": L, "L_star": Lstar,
        "w_hat_head": w_hat[:8].tolist(), "idx_head": idx[:64].tolist(), "idx_sha256_100k": idx_hash(idx),
        "seconds": {"lanczos": t_l, "total": time.time() - t0},
        "source": "oracle/_ref (unmodified reference library)",
    }
    if kappa and d <= 2000 and sketched:
        rec["kappa"] = R.conditioned_cond(Xd, cfg.lam, sk.U, sk.sigma)
    print(name, "done in", round(time.time() - t0, 1), "s", flush=True)
    return rec


def main():
    which = sys.argv[1:] or ["small", "c1"]
    path = os.path.join(HERE, "configs.json")
    db = json.load(open(path)) if os.path.exists(path) else {}
    if "small" in which:
        small()
    if "c1" in which:
        db["c1"] = config_case("c1")
    if "c2" in which:
        db["c2"] = config_case("c2")
    if "c3" in which:
        db["c3_n16384"] = config_case("c3", n_override=16384, epochs=4, kappa=False)
    if "c4" in which:
        db["c4_n16384"] = config_case("c4", n_override=16384, epochs=12, kappa=False)
    if "c5" in which:
        for lam, tag in ((1e-6, "l6"), (1e-8, "l8")):
            db[f"c5_n16384_{tag}"] = config_case("c5", n_override=16384, epochs=6, lam=lam)
        db["c5_n16384_l6_svrg"] = config_case("c5", n_override=16384, epochs=6, lam=1e-6, sketched=False)
    with open(path, "w") as f:
        json.dump(db, f, indent=1)
    print("configs.json:", list(db))


if __name__ == "__main__":
    main()
