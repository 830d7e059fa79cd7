"""Chain-kernel cycle breakdown (SKR_DEBUG_CHAIN=1) for one config: python profiles/k10_debug.py c2"""
import sys
sys.path.insert(0, '.')
from paper_1602_02350_b200 import configs, skridge as sk
cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else 'c2']
data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param, cfg.t_scale, cfg.tau))
p = sk.RidgeProblem(data, data.labels(), cfg.lam)
sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
prob = sk.preconditioned_components(p, sk.build_sketched(sv, cfg.lam))
eta = configs.eta_for(cfg, prob.max_row_sq(), prob.mean_beta())
res = sk.svrg_solve(prob, sk.SvrgConfig(2, 2 * cfg.n, eta, cfg.seed))
print(cfg.name, [r.elapsed_ms for r in res.trace])
