"""CPU: host-side logic of the mirror API and the configs (no device calls)."""
import math

import numpy as np
import pytest

import oracle  # noqa: E402  (checker: the host restatement of the device generator)
from paper_1602_02350_b200 import configs, skridge as sk_mod
from paper_1602_02350_b200 import skridge as sk


def test_lanczos_iterations_matches_reference_formula():
    # sketch.cpp:13-16: max(2, ceil(ln n / sqrt(eps')))
    assert sk.lanczos_iterations(8192, 0.5) == 13
    assert sk.lanczos_iterations(3, 0.9) == 2
    assert sk.lanczos_iterations(60, 0.5) == math.ceil(math.log(60) / math.sqrt(0.5))


def test_build_sketched_coefficients_and_errors():
    # test_precond.cpp:61-68: sigma = (2, 1), lambda = 1 -> 1/sqrt(5), 1/sqrt(2)
    sv = sk.SketchedSvd(np.eye(6)[:, :2], np.array([2.0, 1.0]), None, 2, 3)
    p = sk.build_sketched(sv, 1.0)
    assert abs(p.inv_sqrt_diag()[0] - 1 / math.sqrt(5)) < 1e-15
    assert abs(p.inv_sqrt_diag()[1] - 1 / math.sqrt(2)) < 1e-15
    assert p.tail_coeff() == p.inv_sqrt_diag()[-1]
    assert abs(p.min_inv_eigenvalue() - 0.2) < 1e-15
    with pytest.raises(sk.ParameterError):
        sk.build_sketched(sv, 0.0)
    with pytest.raises(sk.ParameterError):
        sk.build_sketched(sv, -1.0)
    with pytest.raises(sk.ParameterError):
        sk.build_sketched(sk.SketchedSvd(np.zeros((6, 0)), np.zeros(0), None, 0, 3), 1.0)
    with pytest.raises(sk.InputError):  # increasing sigma -> decreasing coefficients
        sk.build_sketched(sk.SketchedSvd(np.eye(6)[:, :2], np.array([1.0, 2.0]), None, 2, 3), 1.0)


def test_identity_preconditioner():
    p = sk.Preconditioner.identity(7, 0.5)
    assert p.rank() == 0 and p.tail_coeff() == 1.0 and p.min_inv_eigenvalue() == 1.0
    with pytest.raises(sk.ParameterError):
        sk.Preconditioner.identity(7, 0.0)


def test_configs_match_baseline():
    c = configs.CONFIGS
    assert (c["c1"].n, c["c1"].d, c["c1"].k, c["c1"].q, c["c1"].lam, c["c1"].epochs) == (8192, 256, 16, 3, 1e-3, 20)
    assert (c["c2"].n, c["c2"].d, c["c2"].k, c["c2"].q, c["c2"].lam, c["c2"].epochs) == (65536, 1024, 64, 4, 1e-5, 30)
    assert (c["c3"].n, c["c3"].d, c["c3"].dtype) == (1 << 20, 2048, "f32")
    assert (c["c4"].n, c["c4"].d, c["c4"].k, c["c4"].t_scale) == (1 << 22, 4096, 256, True)
    assert (c["c5"].n, c["c5"].d, c["c5"].k, c["c5"].q) == (1 << 24, 1024, 64, 2)
    s1 = c["c1"].sigma()
    assert s1[0] == 1.0 and abs(s1[9] - 0.1) < 1e-16
    assert abs(c["c2"].sigma()[2] - 0.97 ** 3) < 1e-16
    assert abs(c["c3"].sigma()[3] - 4 ** -1.5) < 1e-16
    s4 = c["c4"].sigma()
    assert abs(s4[49] - 1 / 50) < 1e-16 and abs(s4[50] - 0.02 / 51) < 1e-18


def test_host_instance_shapes_and_dtypes():
    X, y = oracle.synth_instance(configs.CONFIGS["c3"].scaled(64))
    assert X.shape == (64, 2048) and X.dtype == np.float32 and y.dtype == np.float32
    X1, y1 = oracle.synth_instance(configs.CONFIGS["c1"].scaled(100))
    X2, _ = oracle.synth_instance(configs.CONFIGS["c1"].scaled(100))
    assert X1.dtype == np.float64 and np.array_equal(X1, X2)  # seeded
    # the spectrum is imposed: singular values of X / sqrt(n) ~ sigma (G/sqrt(n) ~ orthonormal)
    X, _ = oracle.synth_instance(configs.CONFIGS["c1"].scaled(20000))
    s = np.linalg.svd(X / math.sqrt(20000), compute_uv=False)
    assert abs(s[0] - 1.0) < 0.05 and abs(s[9] - 0.1) < 0.01


def test_step_size_rule():
    assert configs.step_size(2.0) == 1 / 8


@pytest.mark.parametrize("n,world", [(10, 3), (65536, 8), (5, 8), (1 << 20, 2)])
def test_shard_rows_partition(n, world):
    """The library's host shard arithmetic (skr_shard_rows / skr_shard_layout, the
    layout capi.cu uses for skr_data_generate and skr_data_create)."""
    rows = [sk_mod.shard_rows(n, world, r) for r in range(world)]
    assert sum(c for _, c in rows) == n
    for r in range(world - 1):
        assert rows[r][0] + rows[r][1] == rows[r + 1][0]
    assert max(c for _, c in rows) - min(c for _, c in rows) <= 1
    counts = [c for _, c in rows]
    for r in range(world):
        assert sk_mod.shard_layout(counts, r) == (n, rows[r][0])
    with pytest.raises(sk_mod.ParameterError):
        sk_mod.shard_rows(n, world, world)


def test_ratio_host_functions_match_reference():
    """theoretical_ratio / avg_condition_number / run_ratio_curve / SpectrumSummary
    validation (precond.cpp:23-32,165-172,208-219; bench.cpp:195-203) are host
    arithmetic: checked here against the unmodified reference on given spectra."""
    import numpy as np
    import pytest
    import oracle
    from paper_1602_02350_b200 import skridge as sk
    if not oracle.ref_available():
        pytest.skip("reference library not built")
    R = oracle.ref()
    rng = np.random.default_rng(3)
    e = np.sort(rng.exponential(size=50))[::-1] * 3.0
    e[-5:] = 0.0
    lam = 1e-4
    spec = sk.SpectrumSummary(e, lam)
    for k in (1, 2, 17, 45):
        assert sk.theoretical_ratio(spec, k) == R.theoretical_ratio(e, lam, k)
    assert sk.avg_condition_number(spec) == R.avg_condition_number(e, lam)
    assert [r.ratio for r in sk.run_ratio_curve(spec, 45)] == [R.theoretical_ratio(e, lam, k) for k in range(1, 46)]
    bad = e.copy()
    bad[3] = bad[2] * 2
    with pytest.raises(sk.InputError):
        sk.SpectrumSummary(bad, lam)
    neg = e.copy()
    neg[-1] = -1e-3
    with pytest.raises(sk.InputError):
        sk.SpectrumSummary(neg, lam)
    tiny = e.copy()
    tiny[-1] = -1e-14
    assert sk.SpectrumSummary(tiny, lam).eigenvalues[-1] == 0.0
    with pytest.raises(sk.ParameterError):
        sk.theoretical_ratio(spec, 0)
    with pytest.raises(sk.DegenerateSpectrumError):
        sk.theoretical_ratio(sk.SpectrumSummary(np.zeros(4), lam), 2)
