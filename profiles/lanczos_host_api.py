"""Host-side CUDA runtime/driver API time per block_lanczos call (CUPTI via
torch.profiler): which API calls make the wall time of some calls exceed the
device time.    python profiles/lanczos_host_api.py c3"""
import sys, time, json
sys.path.insert(0, '.')
import torch
from torch.profiler import profile, ProfilerActivity
from paper_1602_02350_b200 import configs, skridge as sk
name = sys.argv[1]
cfg = configs.CONFIGS[name]
ctx = sk.default_context()
data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param, cfg.t_scale, cfg.tau))
y = data.labels()
a = sk.scaled_design(sk.RidgeProblem(data, y, cfg.lam))
sk.block_lanczos(a, sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
for i in range(6):
    ctx.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        sv = sk.block_lanczos(a, sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
        ctx.synchronize()
        w = time.perf_counter() - t0
    agg = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CPU:
            t, c, mx = agg.get(e.name, (0.0, 0, 0.0))
            agg[e.name] = (t + e.cpu_time_total, c + 1, max(mx, e.cpu_time_total))
    rows = sorted(agg.items(), key=lambda kv: -kv[1][0])[:6]
    print(json.dumps({"call": i, "wall_s": round(w, 4),
                      "host_api_ms": [(k[:40], round(t / 1e3, 2), c, round(mx / 1e3, 2)) for k, (t, c, mx) in rows]}), flush=True)
