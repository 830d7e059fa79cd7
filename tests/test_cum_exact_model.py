"""CPU model of cumulative_exact_kernel's arithmetic (svrg.cuh): inside one binade the
sequential fp64 running sum is an integer prefix sum.  The model follows the kernel tile by
tile (same tile size, same fall-back rules) and is compared bit for bit with the sequential
loop (np.add.accumulate = svrg.cpp:95-104); the CUDA kernel itself is compared with both in
tests/test_gpu_parity.py::test_cumulative_weights_block_scan_is_bitwise_sequential."""
import numpy as np
import pytest

TILE = 4096
TWO53 = float(2 ** 53)


def model_running_sum(x, tile=TILE):
    """Running sum of x in index order; returns (prefix sums, tiles on the integer path, tiles)."""
    out = np.empty_like(x)
    S = 0.0
    fast = tiles = 0
    for i0 in range(0, x.size, tile):
        xt = x[i0:i0 + tile]
        tiles += 1
        ok = S > 0.0 and np.isfinite(S)
        if ok:
            e = int(np.frexp(S)[1]) - 1              # S in [2^e, 2^(e+1))
            ok = -900 <= e <= 900
        if ok:
            scale, u = np.ldexp(1.0, 52 - e), np.ldexp(1.0, e - 52)
            xs = xt * scale                          # exact: a power of two
            ok = bool(np.all(xs >= 0.0) and np.all(xs < TWO53))
        if ok:
            fl = np.floor(xs)
            fr = xs - fl                             # exact
            ok = not np.any(fr == 0.5)               # a tie rounds by the parity of the sum: in order
        if ok:
            K = int(S * scale)
            pre = np.cumsum(fl.astype(np.int64) + (fr > 0.5))
            ok = K + int(pre[-1]) < 2 ** 53          # the binade is not left
        if ok:
            out[i0:i0 + xt.size] = (K + pre).astype(np.float64) * u
            S = float(out[i0 + xt.size - 1])
            fast += 1
        else:                                        # thread 0, index order
            acc = np.add.accumulate(np.concatenate(([S], xt)))[1:]
            out[i0:i0 + xt.size] = acc
            S = float(acc[-1])
    return out, fast, tiles


def _cases():
    rng = np.random.default_rng(11)
    yield "uniform", rng.uniform(0.5, 1.5, 600_001), 0.9
    yield "lognormal", np.exp(rng.normal(0.0, 4.0, 300_003)), 0.5
    few = rng.integers(1, 8, 131_075).astype(np.float64) * 2.0 ** rng.integers(-30, 3, 131_075)
    yield "ties", few, 0.0
    z = rng.uniform(0.0, 1.0, 70_001)
    z[:5000] = 0.0
    z[rng.integers(0, z.size, 20_000)] = 0.0
    yield "zeros", z, 0.5
    wide = rng.uniform(0.0, 1.0, 50_000)
    wide[::997] *= 2.0 ** 40
    yield "wide", wide, 0.0
    yield "tiny", rng.uniform(0.1, 1.0, 7), 0.0


@pytest.mark.parametrize("name,beta,min_fast", list(_cases()), ids=[c[0] for c in _cases()])
def test_integer_prefix_model_is_bitwise_sequential(name, beta, min_fast):
    total_seq = np.add.accumulate(beta)[-1]
    tot, _, _ = model_running_sum(beta)
    assert tot[-1] == total_seq                      # svrg.cpp:92-94
    x = beta / total_seq
    got, fast, tiles = model_running_sum(x)
    assert np.array_equal(got, np.add.accumulate(x))  # svrg.cpp:95-104
    assert fast >= min_fast * tiles, (fast, tiles)   # the integer path carries the table
