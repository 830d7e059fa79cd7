"""Per-kernel device-time breakdown of one warm block_lanczos (CUPTI via torch.profiler)."""
import json, sys, time
sys.path.insert(0, '.')
import torch
from torch.profiler import profile, ProfilerActivity
from paper_1602_02350_b200 import configs, skridge as sk
for name in (sys.argv[1].split(',') if len(sys.argv) > 1 else ['c3', 'c5']):
    cfg = configs.CONFIGS[name]
    data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param, cfg.t_scale, cfg.tau))
    a = data.scaled(1 / cfg.n ** 0.5)
    lc = sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q)
    t0 = time.perf_counter()
    sk.block_lanczos(a, lc, want_right=False)
    sk.default_context().synchronize()
    cold_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    sk.block_lanczos(a, lc, want_right=False)
    sk.default_context().synchronize()
    warm_s = time.perf_counter() - t0
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        sk.block_lanczos(a, lc, want_right=False)
        sk.default_context().synchronize()
    agg = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            k = e.name[:90]
            t, c = agg.get(k, (0.0, 0))
            agg[k] = (t + e.device_time_total, c + 1)
    tot = sum(t for t, _ in agg.values())
    rows = sorted(agg.items(), key=lambda kv: -kv[1][0])
    print(json.dumps({"config": name, "device_ms_total": round(tot / 1e3, 3),
                      "wall_cold_s": round(cold_s, 4), "wall_warm_s": round(warm_s, 4),
                      "kernels": [{"name": k, "ms": round(t / 1e3, 3), "launches": c} for k, (t, c) in rows[:25]]}), flush=True)
    del a, data
