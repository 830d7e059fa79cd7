"""Generate one config's X~ and run K9 (full gradient) a few times (for ncu captures)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_1602_02350_b200 import configs, skridge as sk
cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else 'c5']
data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param, cfg.t_scale, cfg.tau))
p = sk.RidgeProblem(data, data.labels(), cfg.lam)
prob = sk.preconditioned_components(p, sk.Preconditioner.identity(cfg.d, cfg.lam))
w = np.random.default_rng(0).standard_normal(cfg.d) * 1e-2
for _ in range(4):
    mu, obj = prob.full_gradient(w, with_objective=True)
print("ok", obj)
