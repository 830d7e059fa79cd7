"""cuBLAS DGEMM throughput on this B200: square 4096/8192 (the FP64 tensor peak the
fp64 Lanczos GEMMs are judged against) and the c2 Lanczos product shapes (what a
library call would reach on the same tall-skinny problems).  Prints JSON."""
import json
import torch


def bench(m, n, k, reps=10):
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return round(2 * m * n * k / ms / 1e9, 2)


out = {"dgemm_4096_tflops": bench(4096, 4096, 4096), "dgemm_8192_tflops": bench(8192, 8192, 8192),
       "c2_T_65536x64x1024_tflops": bench(65536, 64, 1024), "c2_V_64x1024x65536_tflops": bench(64, 1024, 65536),
       "c2_Z_65536x256x1024_tflops": bench(65536, 256, 1024), "c2_G_256x256x65536_tflops": bench(256, 256, 65536)}
print(json.dumps(out))
