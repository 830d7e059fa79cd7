import sys, numpy as np
sys.path.insert(0, '.')
from paper_1602_02350_b200 import configs, skridge as sk
cfg = configs.CONFIGS['c3'].scaled(16384)
X, y = oracle.synth_instance(cfg)
p = sk.RidgeProblem(sk.DataMatrix(X), y, cfg.lam)
sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
pg = sk.preconditioned_components(p, sk.build_sketched(sv, cfg.lam))
eta = configs.eta_for(cfg, pg.max_row_sq(), pg.mean_beta())
res = sk.svrg_solve(pg, sk.SvrgConfig(1, 4096, eta, cfg.seed), np.zeros(cfg.d))
print("ok", [r.objective for r in res.trace])
