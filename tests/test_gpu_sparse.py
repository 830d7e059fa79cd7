"""Sparse data (the reference's SparseMatrix / DataMatrix(SparseMatrix), SURVEY
§8(f) rank 3) through the B200 path, against the unmodified reference on the
same CSR (= its CSC over points) arrays."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_1602_02350_b200 import skridge as sk

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def sparse_instance(n=600, d=80, density=0.08, seed=0):
    """Random CSR with a decaying column scale, canonical (sorted, no zeros)."""
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    rp = [0]
    for i in range(n):
        nnz = max(1, rng.binomial(d, density))
        c = np.sort(rng.choice(d, size=nnz, replace=False))
        v = rng.standard_normal(nnz) / (1.0 + c) ** 0.7
        v[v == 0.0] = 1e-3
        cols.append(c)
        vals.append(v)
        rp.append(rp[-1] + nnz)
    ci = np.concatenate(cols).astype(np.int32)
    va = np.concatenate(vals)
    y = rng.standard_normal(n)
    return (np.asarray(rp, dtype=np.int64), ci, va, d), y


def dense_of(csr, n):
    rp, ci, va, d = csr
    X = np.zeros((n, d))
    for i in range(n):
        X[i, ci[rp[i]:rp[i + 1]]] = va[rp[i]:rp[i + 1]]
    return X


@pytest.fixture(scope="module")
def R():
    if not oracle.ref_available():
        pytest.skip("reference library not built")
    return oracle.ref()


def test_sparse_data_validation():
    (rp, ci, va, d), _ = sparse_instance(n=10, d=6)
    a = sk.DataMatrix.from_csr(rp, ci, va, d)
    assert a.sparse and a.n_local == 10 and a.d == 6
    with pytest.raises(sk.InputError):
        sk.DataMatrix.from_csr(rp, ci, np.where(np.arange(len(va)) == 0, 0.0, va), d)  # explicit zero
    with pytest.raises(sk.InputError):
        sk.DataMatrix.from_csr(rp, np.where(np.arange(len(ci)) == 0, d, ci).astype(np.int32), va, d)  # out of range


def test_sparse_block_lanczos_matches_reference(R):
    csr, _ = sparse_instance()
    n = len(csr[0]) - 1
    a = sk.DataMatrix.from_csr(*csr)
    for k, q, seed in [(6, 3, 4), (10, 2, 1)]:
        got = sk.block_lanczos(a.scaled(1.0 / np.sqrt(n)), sk.LanczosConfig(k, 0.5, seed, q))
        want = R.block_lanczos_csr(csr, k, q=q, seed=seed)
        assert rel(got.singular_values, want.sigma) < 1e-10
        assert np.max(np.abs(got.left @ got.left.T - want.U @ want.U.T)) < 1e-8
        assert got.k == want.k and got.q == want.q
        # the dense path on the densified matrix agrees too
        dense = sk.block_lanczos(sk.DataMatrix(dense_of(csr, n)).scaled(1.0 / np.sqrt(n)),
                                 sk.LanczosConfig(k, 0.5, seed, q))
        assert rel(got.singular_values, dense.singular_values) < 1e-12


def test_sparse_objective_and_reference_minimum(R):
    csr, y = sparse_instance(seed=3)
    n, d = len(csr[0]) - 1, csr[3]
    p = sk.RidgeProblem(sk.DataMatrix.from_csr(*csr), y, 1e-3)
    w = np.random.default_rng(1).standard_normal(d)
    assert abs(sk.objective(p, w) - R.objective_csr(csr, y, 1e-3, w)) <= 1e-12 * R.objective_csr(csr, y, 1e-3, w)
    wm, lm = R.reference_minimum_csr(csr, y, 1e-3)
    r = sk.reference_minimum(p)
    assert rel(r.minimizer, wm) < 1e-9
    assert abs(r.minimum - lm) <= 1e-12 * lm
    spec = sk.dataset_spectrum(p)
    assert rel(spec.eigenvalues, np.sort(np.linalg.eigvalsh(dense_of(csr, n).T @ dense_of(csr, n) / n))[::-1]) < 1e-10
