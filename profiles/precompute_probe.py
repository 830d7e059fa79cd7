"""Time preconditioned_components (the precompute phase) per config, twice (second
reported); prints JSON.  python profiles/precompute_probe.py c2,c3"""
import json, sys, time
sys.path.insert(0, '.')
from paper_1602_02350_b200 import configs, skridge as sk
for name in (sys.argv[1].split(',') if len(sys.argv) > 1 else ['c2']):
    cfg = configs.CONFIGS[name]
    data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param,
                                               cfg.t_scale, cfg.tau))
    p = sk.RidgeProblem(data, data.labels(), cfg.lam)
    sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
    for rep in range(3):
        sk.default_context().synchronize()
        t0 = time.perf_counter()
        pg = sk.preconditioned_components(p, sk.build_sketched(sv, cfg.lam))
        sk.default_context().synchronize()
        dt = time.perf_counter() - t0
        del pg
    print(json.dumps({"config": name, "precompute_s": round(dt, 5)}), flush=True)
