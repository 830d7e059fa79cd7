"""Per-kernel device time of the K10 kernels while they run concurrently (torch profiler / CUPTI):
one SVRG epoch at a config.  python profiles/k10_kernel_times.py c3"""
import json, sys
import numpy as np
sys.path.insert(0, '.')
import torch
from torch.profiler import profile, ProfilerActivity
from paper_1602_02350_b200 import configs, skridge as sk
for name in sys.argv[1].split(','):
    cfg = configs.CONFIGS[name]
    data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param, cfg.t_scale, cfg.tau))
    p = sk.RidgeProblem(data, data.labels(), cfg.lam)
    sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
    prob = sk.preconditioned_components(p, sk.build_sketched(sv, cfg.lam))
    eta = configs.eta_for(cfg, prob.max_row_sq(), prob.mean_beta())
    m = min(2 * cfg.n, 1 << 21)
    sk.svrg_solve(prob, sk.SvrgConfig(1, m, eta, cfg.seed), np.zeros(cfg.d))
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        sk.svrg_solve(prob, sk.SvrgConfig(1, m, eta, cfg.seed), np.zeros(cfg.d))
        sk.default_context().synchronize()
    agg = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA and 'sstep' in e.name:
            k = e.name.split('(')[0][-40:]
            t, c = agg.get(k, (0.0, 0))
            agg[k] = (t + e.device_time_total, c + 1)
    print(json.dumps({"config": name, "m": m, "kernels": {k: {"avg_us": round(t / c, 1), "n": c} for k, (t, c) in agg.items()}}), flush=True)
    del prob, p, data
