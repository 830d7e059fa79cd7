import json, sys
import numpy as np
sys.path.insert(0, '.')
from paper_1602_02350_b200 import configs, skridge as sk
name = sys.argv[1]
cfg = configs.CONFIGS[name]
data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param, cfg.t_scale, cfg.tau))
p = sk.RidgeProblem(data, data.labels(), cfg.lam)
sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
prob = sk.preconditioned_components(p, sk.build_sketched(sv, cfg.lam))
eta = configs.eta_for(cfg, prob.max_row_sq(), prob.mean_beta())
ctx = sk.default_context()
for cap in [0, 120, 100, 80, 64, 48]:
    ctx.set_prep_cap(cap)
    for rep in range(2):
        ctx.profile(True)
        res = sk.svrg_solve(prob, sk.SvrgConfig(1, 2 * cfg.n, eta, cfg.seed), np.zeros(cfg.d))
        ms, n = ctx.profile_read("svrg_epoch")
        ctx.profile(False)
    print(json.dumps({"config": name, "cap": cap, "ns_per_step": round(ms / max(n, 1) * 1e6 / (2 * cfg.n), 2)}), flush=True)
