"""Bitwise run-to-run determinism of the SVRG chain (same problem, same seed, 3 solves)."""
import sys, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_1602_02350_b200 import configs, skridge as sk
import dataclasses
for name in (sys.argv[1].split(',') if len(sys.argv) > 1 else ['c2', 'c3']):
    base, _, dt = name.partition(':')  # e.g. c3:f64 forces the storage dtype
    cfg = configs.CONFIGS[base].scaled(16384) if base != 'c1' else configs.CONFIGS[base]
    if dt:
        cfg = dataclasses.replace(cfg, dtype=dt)
    X, y = oracle.synth_instance(cfg)
    p = sk.RidgeProblem(sk.DataMatrix(X), y, cfg.lam)
    sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
    pg = sk.preconditioned_components(p, sk.build_sketched(sv, cfg.lam))
    eta = configs.eta_for(cfg, pg.max_row_sq(), pg.mean_beta())
    outs = []
    for rep in range(3):
        res = sk.svrg_solve(pg, sk.SvrgConfig(3, 2 * cfg.n, eta, cfg.seed), np.zeros(cfg.d))
        outs.append((np.array([r.objective for r in res.trace]), np.array(res.iterate)))
    same = all(np.array_equal(outs[0][1], o[1]) for o in outs[1:])
    print(name, "bitwise identical iterates:", same, "max |dw|:", max(float(np.max(np.abs(outs[0][1] - o[1]))) for o in outs[1:]),
          "traces:", [o[0].tolist() for o in outs], flush=True)
