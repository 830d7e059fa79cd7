"""Known-answer checks of the reference's own test suite, restated on
this implementation: host value-type checks run on CPU, the rest on the GPU
through the C-ABI."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_1602_02350_b200 import skridge as sk


def _sketch(U, sigma):
    d, k = U.shape
    return sk.SketchedSvd(U, np.asarray(sigma, dtype=np.float64), None, k, 3)


def test_build_sketched_coefficients_known_answer():
    """test_precond.cpp:61-68: sigma~ = (2, 1), lambda = 1 -> 1/sqrt(5), 1/sqrt(2)."""
    U = np.eye(3)[:, :2]
    P = sk.build_sketched(_sketch(U, [2.0, 1.0]), 1.0)
    D = P.inv_sqrt_diag()
    assert abs(D[0] - 1.0 / math.sqrt(5.0)) <= 1e-15
    assert abs(D[1] - 1.0 / math.sqrt(2.0)) <= 1e-15
    assert P.tail_coeff() == D[1]


def test_apply_sqrt_inverts_apply_inv_sqrt():
    """test_precond.cpp:133-150: apply_sqrt(apply_inv_sqrt(v)) = v (1e-10), and the
    structured map equals the densified operator (test_precond.cpp:112-123)."""
    rng = np.random.default_rng(5)
    d, k = 30, 6
    U, _ = np.linalg.qr(rng.standard_normal((d, k)))
    sig = np.sort(rng.uniform(0.1, 3.0, k))[::-1]
    lam = 1e-2
    P = sk.build_sketched(_sketch(U, sig), lam)
    v = rng.standard_normal(d)
    back = P.apply_sqrt(P.apply_inv_sqrt(v))
    assert np.max(np.abs(back - v)) <= 1e-10 * np.max(np.abs(v))
    D, c = P.inv_sqrt_diag(), P.tail_coeff()
    dense = c * np.eye(d) + U @ np.diag(D - c) @ U.T
    assert np.max(np.abs(dense @ v - P.apply_inv_sqrt(v))) <= 1e-13
    proj = U.T @ v
    assert abs(P.inv_sqrt_sq_norm(float(v @ v), proj) - float(np.sum((dense @ v) ** 2))) <= 1e-12 * float(v @ v)
    with pytest.raises(sk.DimensionError):
        P.apply_inv_sqrt(np.zeros(d + 1))


def _problem(n=400, d=30, k=5, lam=1e-3, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)) * (1.0 / np.arange(1, d + 1))
    y = rng.standard_normal(n)
    p = sk.RidgeProblem(sk.DataMatrix(X), y, lam)
    sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(k, 0.5, 7, 3))
    return X, y, p, sv


@pytest.mark.gpu
def test_block_lanczos_is_deterministic():
    """test_sketch.cpp:168-184: repeated runs are bitwise identical."""
    X, y, p, sv = _problem()
    sv2 = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(5, 0.5, 7, 3))
    assert np.array_equal(sv.singular_values, sv2.singular_values)
    assert np.array_equal(sv.left, sv2.left) and np.array_equal(sv.right, sv2.right)


@pytest.mark.gpu
def test_coordinate_change_and_mean_beta_trace_identity():
    """test_ridge.cpp:129-138: L~(w~) = L(P^{-1/2} w~) (1e-10);
    test_ridge.cpp:229-237: beta^ = tr(P^{-1/2}(C + lambda I)P^{-1/2}) (1e-8);
    the device map equals the host value type's."""
    X, y, p, sv = _problem()
    n, d = X.shape
    lam = p.lam
    P = sk.build_sketched(sv, lam)
    pg = sk.preconditioned_components(p, P)
    rng = np.random.default_rng(2)
    wt = rng.standard_normal(d)
    w = pg.apply_inv_sqrt(wt)
    assert np.max(np.abs(w - P.apply_inv_sqrt(wt))) <= 1e-13 * np.max(np.abs(w))
    lt = pg.objective(wt)
    assert abs(lt - sk.objective(p, w)) <= 1e-10 * abs(lt)
    D, c = P.inv_sqrt_diag(), P.tail_coeff()
    Pm = c * np.eye(d) + sv.left @ np.diag(D - c) @ sv.left.T
    M = Pm @ (X.T @ X / n + lam * np.eye(d)) @ Pm
    assert abs(pg.mean_beta() - np.trace(M)) <= 1e-8 * np.trace(M)
