"""Why is the first (and only) epoch of `bench.py --solve c3` slower than the
same epoch in `bench.py` / k10_probe?  Runs the solve path's variants on one
problem and prints the inner-loop time of each.
    python profiles/k10_solve_probe.py c3"""
import json
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_1602_02350_b200 import configs, skridge as sk  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = configs.CONFIGS[name]
ctx = sk.default_context()
data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param,
                                           cfg.t_scale, cfg.tau))
p = sk.RidgeProblem(data, data.labels(), cfg.lam)
sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
ref = sk.reference_minimum(p)


def run(tag, prob, epochs, w0, lstar, stop):
    eta = configs.eta_for(cfg, prob.max_row_sq(), prob.mean_beta())
    ctx.profile(True)
    res = sk.svrg_solve(prob, sk.SvrgConfig(epochs, 2 * cfg.n, eta, cfg.seed), w0, lstar, stop_suboptimality=stop)
    ms, n = ctx.profile_read("svrg_epoch")
    ctx.profile(False)
    print(json.dumps({"variant": tag, "epochs_run": len(res.trace), "inner_ms_per_epoch": round(ms / max(n, 1), 3),
                      "elapsed_ms": [round(r.elapsed_ms, 2) for r in res.trace]}), flush=True)


prob = sk.preconditioned_components(p, sk.build_sketched(sv, cfg.lam))
ctx.synchronize()
run("A first solve on a fresh problem: until eps (w0 None)", prob, cfg.epochs, None, ref.minimum, 1e-6)
run("B same problem again: until eps", prob, cfg.epochs, None, ref.minimum, 1e-6)
run("C same problem: 2 plain epochs (w0 zeros)", prob, 2, np.zeros(cfg.d), None, None)
prob = None
prob = sk.preconditioned_components(p, sk.build_sketched(sv, cfg.lam))
run("D rebuilt problem, no synchronize before the solve: until eps", prob, cfg.epochs, None, ref.minimum, 1e-6)
run("E again", prob, cfg.epochs, None, ref.minimum, 1e-6)
