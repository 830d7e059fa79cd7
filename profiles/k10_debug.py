import sys, numpy as np
sys.path.insert(0, '.')
from paper_1602_02350_b200 import configs, skridge as sk
cfg = configs.CONFIGS['c2']
data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param, cfg.t_scale, cfg.tau))
p = sk.RidgeProblem(data, data.labels(), cfg.lam)
sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
prob = sk.preconditioned_components(p, sk.build_sketched(sv, cfg.lam))
eta = configs.step_size(prob.max_row_sq())
res = sk.svrg_solve(prob, sk.SvrgConfig(2, 2 * cfg.n, eta, cfg.seed))
print([r.elapsed_ms for r in res.trace])
