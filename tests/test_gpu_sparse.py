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


def _lazy_pair(R, seed=0, k=5, lam=1e-3):
    csr, y = sparse_instance(seed=seed)
    n, d = len(csr[0]) - 1, csr[3]
    a = sk.DataMatrix.from_csr(*csr)
    p = sk.RidgeProblem(a, y, lam)
    sv = R.block_lanczos_csr(csr, k, q=3, seed=5)
    pg = sk.preconditioned_components(p, sk.build_sketched(sk.SketchedSvd(sv.U, sv.sigma, None, k, 3), lam))
    po = R.problem_csr(csr, y, lam, sv.U, sv.sigma, mode=1)  # the reference's Lazy mode
    return csr, y, p, pg, po


def test_lazy_components_match_reference(R):
    csr, y, p, pg, po = _lazy_pair(R)
    n, d = len(csr[0]) - 1, csr[3]
    assert pg.mode() == sk.ApplyMode.Lazy
    assert rel(pg.betas(), po.betas()) < 1e-12
    a_o, b_o = po.scalars()[:2]
    assert abs(pg.strong_convexity() - a_o) <= 1e-15 * a_o
    assert abs(pg.mean_beta() - b_o) <= 1e-12 * b_o
    rng = np.random.default_rng(4)
    for _ in range(3):
        w = rng.standard_normal(d)
        assert abs(pg.objective(w) - po.objective(w)) <= 1e-12 * abs(po.objective(w))
        assert rel(pg.full_gradient(w), po.full_gradient(w)) < 1e-11
        for i in (0, 7, n - 1, n, n + d - 1):
            assert rel(pg.component_gradient(i, w), po.component_gradient(i, w)) < 1e-11
    # X~ on demand equals c X + (X U o (D - c)) U^T built on the host
    P = pg.preconditioner()
    U, D, c = P.basis(), P.inv_sqrt_diag(), P.tail_coeff()
    X = dense_of(csr, n)
    assert rel(pg.transformed(), c * X + ((X @ U) * (D - c)) @ U.T) < 1e-12


def test_lazy_svrg_matches_reference_lazy_and_dense(R):
    """svrg_solve over sparse rows (LazyEpochState, ridge.cpp:283-400) against the
    reference's Lazy mode on the same CSR, and the reference's Dense mode on the
    densified matrix (the reference pins dense = lazy traces at 1e-8,
    test_ridge.cpp:272-291)."""
    from paper_1602_02350_b200 import configs
    csr, y, p, pg, po = _lazy_pair(R, seed=2)
    n, d = len(csr[0]) - 1, csr[3]
    eta = configs.step_size(pg.max_row_sq())
    want = po.svrg(5, 2 * n, eta, 11)
    got = sk.svrg_solve(pg, sk.SvrgConfig(5, 2 * n, eta, 11), np.zeros(d))
    tr = np.array([r.objective for r in got.trace])
    assert rel(tr, want.trace) < 1e-10
    assert rel(got.iterate, want.iterate) < 1e-8
    assert np.array_equal(pg.index_stream(11, 4 * n), R.index_stream(po.betas(), 11, 4 * n))
    sv = R.block_lanczos_csr(csr, 5, q=3, seed=5)
    pd = R.problem(dense_of(csr, n), y, p.lam, sv.U, sv.sigma, 0)
    dense = pd.svrg(5, 2 * n, eta, 11)
    assert rel(tr, dense.trace) < 1e-8


def test_lazy_sketched_pipeline_and_unpreconditioned(R):
    """The whole pipeline on sparse data (block_lanczos -> build_sketched ->
    Lazy components -> svrg -> map back) and the identity preconditioner."""
    from paper_1602_02350_b200 import configs
    csr, y = sparse_instance(n=900, d=120, seed=7)
    n, d = len(csr[0]) - 1, csr[3]
    lam = 1e-4
    p = sk.RidgeProblem(sk.DataMatrix.from_csr(*csr), y, lam)
    sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(8, 0.5, 3, 3))
    pg = sk.preconditioned_components(p, sk.build_sketched(sv, lam))
    eta = configs.step_size(pg.max_row_sq())
    ref = sk.reference_minimum(p)
    res = sk.svrg_solve(pg, sk.SvrgConfig(12, 2 * n, eta, 3), np.zeros(d), ref.minimum)
    L = sk.objective(p, pg.apply_inv_sqrt(res.iterate))
    po = R.problem_csr(csr, y, lam, sv.left, sv.singular_values, mode=1)
    want = po.svrg(12, 2 * n, eta, 3)
    assert rel([r.objective for r in res.trace], want.trace) < 1e-9
    assert L - ref.minimum < res.trace[0].objective - ref.minimum  # made progress
    plain = sk.preconditioned_components(p, sk.Preconditioner.identity(d, lam))
    assert plain.mode() == sk.ApplyMode.Lazy
    eta0 = configs.step_size(plain.max_row_sq())
    got0 = sk.svrg_solve(plain, sk.SvrgConfig(3, 2 * n, eta0, 1), np.zeros(d))
    want0 = R.problem_csr(csr, y, lam, None, None, mode=1).svrg(3, 2 * n, eta0, 1)
    assert rel([r.objective for r in got0.trace], want0.trace) < 1e-10


def test_corpus_file_end_to_end(R, tmp_path):
    """read_sparse_corpus -> average_norm_normalize -> sketched Lazy SVRG on the
    device, against the reference reading the same file."""
    from paper_1602_02350_b200 import configs
    csr, y = sparse_instance(n=500, d=60, seed=9)
    path = str(tmp_path / "corpus.txt")
    sk.write_sparse_corpus(csr[0], csr[1], csr[2], y, path)
    ds = sk.read_sparse_corpus(path)
    (rp, ci, va, d), yr = R.read_sparse_corpus(path)
    assert ds.data.sparse and ds.data.d == d and np.array_equal(ds.labels, yr)
    norm = sk.average_norm_normalize(ds, rp, va)
    mean = np.mean([np.linalg.norm(va[rp[i]:rp[i + 1]]) for i in range(len(rp) - 1)])
    assert abs(norm.data.scale() - 1.0 / mean) <= 1e-15 / mean
    lam = 1e-3
    p = sk.RidgeProblem(ds.data, ds.labels, lam)
    sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(6, 0.5, 2, 3))
    want_sv = R.block_lanczos_csr((rp, ci, va, d), 6, q=3, seed=2)
    assert rel(sv.singular_values, want_sv.sigma) < 1e-10
    pg = sk.preconditioned_components(p, sk.build_sketched(sv, lam))
    eta = configs.step_size(pg.max_row_sq())
    got = sk.svrg_solve(pg, sk.SvrgConfig(4, 2 * len(yr), eta, 2), np.zeros(d))
    want = R.problem_csr((rp, ci, va, d), yr, lam, want_sv.U, want_sv.sigma, mode=1).svrg(4, 2 * len(yr), eta, 2)
    assert rel([r.objective for r in got.trace], want.trace) < 1e-9
