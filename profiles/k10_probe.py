"""K10 probe: per config, 2 SVRG epochs on the device instance -> inner-loop ns
per step (device events around the epochs), bitwise determinism of two solves,
and (SKR_DEBUG_CHAIN=1) the chain's cycle breakdown on stderr.
    python profiles/k10_probe.py c2,c3,c5"""
import json
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_1602_02350_b200 import configs, skridge as sk  # noqa: E402

for name in (sys.argv[1] if len(sys.argv) > 1 else "c2,c3,c5").split(","):
    cfg = configs.CONFIGS[name]
    data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param,
                                               cfg.t_scale, cfg.tau))
    p = sk.RidgeProblem(data, data.labels(), cfg.lam)
    sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
    prob = sk.preconditioned_components(p, sk.build_sketched(sv, cfg.lam))
    eta = configs.eta_for(cfg, prob.max_row_sq(), prob.mean_beta())
    ctx = sk.default_context()
    outs = []
    for rep in range(2):
        ctx.profile(True)
        res = sk.svrg_solve(prob, sk.SvrgConfig(2, 2 * cfg.n, eta, cfg.seed), np.zeros(cfg.d))
        k10_ms, k10_n = ctx.profile_read("svrg_epoch")
        ctx.profile(False)
        outs.append((res, k10_ms / max(k10_n, 1)))
    same = np.array_equal(outs[0][0].iterate, outs[1][0].iterate)
    print(json.dumps({"config": name, "first_call_epoch_ms": round(outs[0][1], 3), "epoch_ms": round(outs[1][1], 3),
                      "ns_per_step": round(outs[1][1] * 1e6 / (2 * cfg.n), 2), "bitwise_repeat": bool(same),
                      "trace": [r.objective for r in outs[1][0].trace]}), flush=True)
    del prob, p, data
