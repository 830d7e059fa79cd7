"""CPU: the oracle restatement (oracle/skr_oracle.c) pinned against golden
vectors produced by the UNMODIFIED reference library (tests/golden/, made by
tests/golden/make_golden.py from oracle/_ref), and against the live reference
library when it is built here.  Bitwise where the restatement follows the
reference's loop order; otherwise the tolerance is stated."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_1602_02350_b200 import configs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLD, "small.npz"))


@pytest.fixture(scope="module")
def O():
    return oracle.port()


def test_streams_bitwise(g, O):
    assert np.array_equal(O.uniforms(0, 700), g["uniforms_0"])
    assert np.array_equal(O.uniforms(5, 700), g["uniforms_5"])
    assert np.array_equal(O.uniforms(2 ** 40 + 3, 700), g["uniforms_big"])
    assert np.array_equal(O.gaussian_matrix(37, 5, 42), g["gauss_37x5_42"])


def test_sym_eigs_bitwise(g, O):
    vals, vecs = O.sym_eigs(g["eig_in"])
    assert np.array_equal(vals, g["eig_vals"]) and np.array_equal(vecs, g["eig_vecs"])


def test_block_lanczos_bitwise(g, O):
    X = g["bl_X"]
    sk = O.block_lanczos(X, 5, q=3, seed=4)
    assert np.array_equal(sk.sigma, g["bl_sigma"])
    assert np.array_equal(sk.U, g["bl_U"]) and np.array_equal(sk.V, g["bl_V"])
    sk2 = O.block_lanczos(X[:60, :14], 3, q=0, seed=1, scale=1.0)
    assert sk2.q == int(g["bl2_q"]) and np.array_equal(sk2.sigma, g["bl2_sigma"])
    sk3 = O.block_lanczos(g["rr_X"], 5, q=1, seed=4, scale=1.0)
    assert sk3.k == int(g["rr_k"]) == 3 and sk3.rank_reduced == bool(g["rr_reduced"])
    assert np.array_equal(sk3.sigma, g["rr_sigma"])


def test_components_bitwise(g, O):
    X, y, lam = g["bl_X"], g["pc_y"], float(g["pc_lam"])
    sk = O.block_lanczos(X, 5, q=3, seed=4)
    p = O.problem(X, y, lam, sk.U, sk.sigma)
    assert np.array_equal(p.betas(), g["pc_betas"])
    a, b, _ = p.scalars()
    assert a == float(g["pc_alpha"]) and b == float(g["pc_beta_hat"])
    w = g["pc_w"]
    assert p.objective(w) == float(g["pc_obj"])
    assert np.array_equal(p.full_gradient(w), g["pc_grad"])
    cg = np.stack([p.component_gradient(i, w) for i in [0, 7, 400, 429]])
    assert np.array_equal(cg, g["pc_cg"])
    assert np.array_equal(O.apply_inv_sqrt(sk.U, sk.sigma, lam, w), g["pc_aisq"])
    assert O.objective(X, y, lam, w) == float(g["obj_orig"])
    p0 = O.problem(X, y, lam)
    assert np.array_equal(p0.betas(), g["id_betas"]) and np.array_equal(p0.full_gradient(w), g["id_grad"])


def test_svrg_and_sampling_bitwise(g, O):
    X, y, lam = g["bl_X"], g["pc_y"], float(g["pc_lam"])
    sk = O.block_lanczos(X, 5, q=3, seed=4)
    p = O.problem(X, y, lam, sk.U, sk.sigma)
    eta = float(g["sv_eta"])
    assert eta == configs.step_size(p.scalars()[2])
    out = p.svrg(4, 800, eta, 13)
    assert np.array_equal(out.trace, g["sv_trace"]) and np.array_equal(out.iterate, g["sv_iter"])
    assert np.array_equal(O.index_stream(p.betas(), 13, 2000), g["sv_idx"])
    assert np.array_equal(O.cumulative_weights(p.betas()), g["cum"])


def test_diagnostics_bitwise(g, O):
    X, y, lam = g["bl_X"], g["pc_y"], float(g["pc_lam"])
    w, L = O.reference_minimum(X, y, lam)
    assert np.array_equal(w, g["refmin_w"]) and L == float(g["refmin_L"])
    sk = O.block_lanczos(X, 5, q=3, seed=4)
    assert O.conditioned_cond(X, lam, sk.U, sk.sigma) == float(g["kappa"])


def test_error_behaviour(O):
    X = np.random.default_rng(0).standard_normal((10, 14))
    with pytest.raises(oracle.OracleError) as e:
        O.block_lanczos(X, 11, q=2, seed=0)
    assert e.value.kind == "ParameterError"
    with pytest.raises(oracle.OracleError) as e:
        O.block_lanczos(X, 2, q=2, seed=0, eps_prime=1.0)
    assert e.value.kind == "ParameterError"
    with pytest.raises(oracle.OracleError) as e:
        O.conditioned_cond(np.zeros((3, 2001)), 1.0, None, None)
    assert e.value.kind == "ScaleGuardError"


def test_c1_against_reference_golden(O):
    """BASELINE c1 composed by hand vs the reference's run."""
    gold = json.load(open(os.path.join(GOLD, "configs.json")))["c1"]
    cfg = configs.CONFIGS["c1"]
    X, y = oracle.synth_instance(cfg)
    n, d = X.shape
    sk = O.block_lanczos(X, cfg.k, q=cfg.q, seed=cfg.seed, want_right=False)
    # data generation (numpy QR) may differ in the last bits across CPUs -> 1e-12
    assert np.max(np.abs(sk.sigma - gold["sigma"]) / np.asarray(gold["sigma"])) < 1e-12
    p = O.problem(X, y, cfg.lam, sk.U, sk.sigma)
    eta = configs.step_size(p.scalars()[2])
    assert abs(eta - gold["eta"]) <= 1e-12 * gold["eta"]
    out = p.svrg(cfg.epochs, 2 * n, eta, cfg.seed)
    assert np.max(np.abs(out.trace - gold["trace"]) / np.abs(gold["trace"])) < 1e-10
    w_hat = O.apply_inv_sqrt(sk.U, sk.sigma, cfg.lam, out.iterate)
    assert abs(O.objective(X, y, cfg.lam, w_hat) - gold["L_hat"]) <= 1e-10 * gold["L_hat"]
    assert O.index_stream(p.betas(), cfg.seed, 64).tolist() == gold["idx_head"]


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built here")
@pytest.mark.parametrize("n,d,k,q,seed", [(333, 17, 4, 2, 3), (128, 64, 8, 3, 9), (50, 20, 20, 2, 1)])
def test_port_equals_reference_live(n, d, k, q, seed):
    P, R = oracle.port(), oracle.ref()
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)) / np.sqrt(np.arange(1, d + 1))
    y = rng.standard_normal(n)
    a, b = P.block_lanczos(X, k, q=q, seed=seed), R.block_lanczos(X, k, q=q, seed=seed)
    assert np.array_equal(a.sigma, b.sigma) and np.array_equal(a.U, b.U)
    pa, pb = P.problem(X, y, 1e-2, a.U, a.sigma), R.problem(X, y, 1e-2, b.U, b.sigma, 0)
    assert np.array_equal(pa.betas(), pb.betas())
    w = rng.standard_normal(d)
    assert np.array_equal(pa.full_gradient(w), pb.full_gradient(w))
    m = 2 * n
    eta = configs.step_size(pa.scalars()[2])
    assert np.array_equal(pa.svrg(3, m, eta, seed).trace, pb.svrg(3, m, eta, seed).trace)
