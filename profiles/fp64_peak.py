"""cuBLAS DGEMM throughput on this B200 (the FP64 tensor peak the fp64 Lanczos
GEMMs are judged against).  Prints JSON."""
import json
import torch

out = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out[f"dgemm_{n}_tflops"] = round(2 * n ** 3 / ms / 1e9, 2)
print(json.dumps(out))
