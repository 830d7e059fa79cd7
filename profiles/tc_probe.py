import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_1602_02350_b200 import skridge as sk, _lib
ctx = sk.default_context()
for (M, N, K, sp) in [(128, 64, 32, 1), (300, 64, 1000, 1), (1024, 128, 4096, 4)]:
    rng = np.random.default_rng(1)
    A = rng.standard_normal((M, K)).astype(np.float32); B = rng.standard_normal((N, K)).astype(np.float32)
    C = np.empty(M * N)
    rc = _lib.load().skr_tc_gemm_test(ctx.h, A.ctypes.data, B.ctypes.data, M, N, K, sp, C)
    want = A.astype(np.float64) @ B.astype(np.float64).T
    print(M, N, K, rc, _lib.last_error() if rc else "", np.max(np.abs(C.reshape(M, N) - want)) / np.max(np.abs(want)), flush=True)
