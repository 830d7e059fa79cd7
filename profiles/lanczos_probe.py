"""Time block_lanczos (device-generated BASELINE data) per config; prints JSON lines."""
import json, sys, time
sys.path.insert(0, '.')
from paper_1602_02350_b200 import configs, skridge as sk
import bench
for name in (sys.argv[1].split(',') if len(sys.argv) > 1 else ['c1', 'c2', 'c3', 'c5']):
    cfg = configs.CONFIGS[name]
    data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param, cfg.t_scale, cfg.tau))
    a = data.scaled(1 / cfg.n ** 0.5)
    for rep in range(2):
        sk.default_context().synchronize()
        t0 = time.perf_counter()
        sv = sk.block_lanczos(a, sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
        dt = time.perf_counter() - t0
    fl = bench.lanczos_flops(cfg, cfg.n)
    print(json.dumps({"config": name, "seconds": round(dt, 4), "tflops": round(fl / dt / 1e12, 3),
                      "sigma0": sv.singular_values[0], "sigma_k": sv.singular_values[-1]}), flush=True)
    del a, data
