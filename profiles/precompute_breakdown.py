"""Per-kernel device time of one warm preconditioned_components call (torch profiler,
CUDA activities) at a config: python profiles/precompute_breakdown.py c5"""
import json, sys, time
sys.path.insert(0, '.')
import torch
from paper_1602_02350_b200 import configs, skridge as sk
name = sys.argv[1] if len(sys.argv) > 1 else 'c5'
cfg = configs.CONFIGS[name]
data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param,
                                           cfg.t_scale, cfg.tau))
p = sk.RidgeProblem(data, data.labels(), cfg.lam)
sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
pc = sk.build_sketched(sv, cfg.lam)
pg = sk.preconditioned_components(p, pc)
del pg
sk.default_context().synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    pg = sk.preconditioned_components(p, pc)
    sk.default_context().synchronize()
    wall = time.perf_counter() - t0
rows = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        r = rows.setdefault(e.name[:90], [0.0, 0])
        r[0] += e.device_time_total / 1e3
        r[1] += 1
ks = sorted(rows.items(), key=lambda x: -x[1][0])
print(json.dumps({"config": name, "wall_s": round(wall, 4), "device_ms_total": round(sum(v[0] for _, v in ks), 3),
                  "kernels": [{"name": k, "ms": round(v[0], 3), "launches": v[1]} for k, v in ks[:14]]}))
