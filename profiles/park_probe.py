"""Park / out-of-memory retry probe: what cudaMemGetInfo says around a request that
only fits once the parked buffers are released.   python profiles/park_probe.py [hold_gib]"""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1602_02350_b200 import skridge as sk
hold = int(sys.argv[1]) if len(sys.argv) > 1 else 0
keep = torch.empty(hold << 30, dtype=torch.uint8, device="cuda") if hold else None
ctx = sk.Context(0)
gib = lambda b: round(b / 2**30, 2)
row, parked = 2048 * 4, 8 << 30
print("free at start", gib(torch.cuda.mem_get_info(0)[0]))
data = sk.DataMatrix.generate(sk.SynthSpec(parked // row, 2048, "f32", 1, 0, 0.0, False, 0.1), ctx)
print("free with 8 GiB data", gib(torch.cuda.mem_get_info(0)[0]))
del data
ctx.synchronize()
free_now = torch.cuda.mem_get_info(0)[0]
print("free with the data parked", gib(free_now))
want = free_now + parked // 2
big = sk.DataMatrix.generate(sk.SynthSpec(want // row, 2048, "f32", 2, 0, 0.0, False, 0.1), ctx)
print("big rows", big.n_local, "want GiB", gib(want), "free now", gib(torch.cuda.mem_get_info(0)[0]))
del big
ctx.synchronize()
print("free after del big", gib(torch.cuda.mem_get_info(0)[0]))
print("trim ->", gib(ctx.trim()), "free", gib(torch.cuda.mem_get_info(0)[0]))
