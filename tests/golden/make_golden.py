"""Generate the golden fixtures from the UNMODIFIED reference library.

Runs oracle/_ref/libskridge_ref.so (built from /root/reference/proj/src by
oracle/Makefile) — never the restatement — and stores inputs and outputs:

  tests/golden/small.npz   small known-answer cases (streams, eigensolver,
                           block_lanczos incl. rank drop, preconditioned
                           components, SVRG trace + index stream, L*, kappa~)
  tests/golden/configs.json  BASELINE configs composed as SURVEY §0 fact 6
                           prescribes (sigma~, beta_hat, alpha, eta, per-epoch
                           objectives, L(w^), L*, kappa~, index-stream sha256,
                           X sha256 and row-block sums): c1, c2 and c3 at FULL
                           size; c4 at n/16 (262,144 rows) and c5 at n/16
                           (1,048,576 rows; lambda 1e-4/1e-6/1e-8, preconditioned
                           and unpreconditioned); quick row-subsampled cases at
                           n = 16384.  Inputs are oracle.synth_instance — the
                           host restatement of the device generator — so a
                           row-subsampled instance is the first n rows of the
                           full one and the GPU tests regenerate it on device.

Usage:  python tests/golden/make_golden.py [small] [c1] [c2] [c3s] [c3] [c4] [c5]
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


def config_case(name: str, n_override: int | None = None, epochs: int | None = None, kappa: str = "auto",
                lam: float | None = None, sketched: bool = True):
    """One BASELINE config through the reference's composed pipeline (oracle.pipeline
    -> ref_pipeline: ONE DataMatrix, block_lanczos with q_override, build_sketched,
    preconditioned_components(Auto), reference_minimum, svrg_solve(m = 2n),
    apply_inv_sqrt, objective on the original X).  The instance is the first
    n rows of the config's DEVICE instance (oracle.synth_instance restates the
    device generator), so the GPU tests regenerate it on the device."""
    cfg = configs.CONFIGS[name]
    if n_override:
        cfg = cfg.scaled(n_override)
    if lam is not None:
        cfg = configs.Config(**{**cfg.__dict__, "lam": lam})
    t0 = time.time()
    X, y = oracle.synth_instance(cfg)
    t_gen = time.time() - t0
    n, d = X.shape
    digest = hashlib.sha256(np.ascontiguousarray(X).tobytes()).hexdigest()
    # per-row-block checksums (fp64 sums of 4096-row blocks) for a device-side check
    # that tolerates the rare fp32 rounding ties between the host and device generators
    blk = 4096
    row_sums = [float(np.sum(X[r:r + blk], dtype=np.float64)) for r in range(0, n, blk)]
    ep = epochs or cfg.epochs
    rule = 0 if name in ("c1", "c2") else 1
    out = oracle.pipeline(X, y.astype(np.float64), cfg.lam, cfg.k if sketched else 0, cfg.q, cfg.seed, ep, 2 * n,
                          eta_rule=rule, idx_count=100000, want_U=True)
    rec = {
        "config": name, "n": n, "d": d, "dtype": cfg.dtype, "k": cfg.k if sketched else 0, "q": cfg.q,
        "lambda": cfg.lam, "seed": cfg.seed, "epochs": ep, "m": 2 * n, "x_sha256": digest,
        "x_block_rows": blk, "x_block_sums": row_sums, "y_head": [float(v) for v in y[:8]],
        "sigma": out.sigma.tolist(), "k_used": out.k_used, "alpha": out.alpha, "beta_hat": out.beta_hat,
        "max_row_sq": out.max_row_sq, "eta": out.eta, "trace": out.trace.tolist(), "L_hat": out.L_hat,
        "L_star": out.L_star, "w_hat_head": out.w_hat[:8].tolist(), "idx_head": out.idx[:64].tolist(),
        "idx_sha256_100k": idx_hash(out.idx), "mode": out.mode,
        "seconds": {"generate": t_gen, "sketch": out.sketch_ms / 1e3, "precompute": out.precompute_ms / 1e3,
                    "reference_minimum": out.refmin_ms / 1e3, "solve": out.solve_ms / 1e3,
                    "full_gradient": out.full_gradient_ms / 1e3, "total": time.time() - t0},
        "threads": os.cpu_count(),
        "source": "oracle/_ref (unmodified reference library) on oracle.synth_instance",
    }
    if sketched and kappa != "none":
        if kappa == "auto" and d <= 2000:
            rec["kappa"] = oracle.ref().conditioned_cond(X.astype(np.float64), cfg.lam, out.U, out.sigma)
            rec["kappa_source"] = "conditioned_condition_number"
        else:
            M = oracle.conditioned_matrix(X, cfg.lam, out.U, out.sigma)
            ev = np.linalg.eigvalsh(M)
            rec["kappa"] = float(np.trace(M) / ev[0])
            rec["kappa_source"] = "reference conditioned_matrix (unguarded) + numpy eigvalsh (d > 2000 guard)"
            del M
    print(name, n, "done in", round(time.time() - t0, 1), "s", flush=True)
    return rec


def save(db, path):
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        json.dump(db, f, indent=1)
    os.replace(tmp, path)


def main():
    which = sys.argv[1:] or ["small", "c1"]
    path = os.path.join(HERE, "configs.json")
    db = json.load(open(path)) if os.path.exists(path) else {}

    def put(key, rec):
        db[key] = rec
        save(db, path)

    if "small" in which:
        small()
    if "c1" in which:
        put("c1", config_case("c1"))
    if "c2" in which:
        put("c2", config_case("c2"))
    if "c3s" in which:  # row-subsampled quick cases (first 16384 rows of the instance)
        put("c3_n16384", config_case("c3", n_override=16384, epochs=4, kappa="none"))
        put("c4_n16384", config_case("c4", n_override=16384, epochs=12, kappa="none"))
        for lam, tag in ((1e-6, "l6"), (1e-8, "l8")):
            put(f"c5_n16384_{tag}", config_case("c5", n_override=16384, epochs=6, lam=lam))
        put("c5_n16384_l6_svrg", config_case("c5", n_override=16384, epochs=6, lam=1e-6, sketched=False))
    if "c3" in which:  # full size
        put("c3", config_case("c3", kappa="eigvalsh"))
    if "c4" in which:  # n/16
        put("c4_n262144", config_case("c4", n_override=1 << 18, epochs=8, kappa="eigvalsh"))
    if "c5" in which:  # n/16, the lambda sweep, preconditioned and not
        for lam, tag in ((1e-4, "l4"), (1e-6, "l6"), (1e-8, "l8")):
            put(f"c5_n1048576_{tag}", config_case("c5", n_override=1 << 20, epochs=4, lam=lam))
            put(f"c5_n1048576_{tag}_svrg", config_case("c5", n_override=1 << 20, epochs=4, lam=lam, sketched=False))
    print("configs.json:", list(db))


if __name__ == "__main__":
    main()
