"""Wall time of block_lanczos called the way bench.py --solve calls it vs the way
lanczos_breakdown.py does (same data), to locate host-side overheads."""
import sys, time, json
sys.path.insert(0, '.')
from paper_1602_02350_b200 import configs, skridge as sk
name = sys.argv[1] if len(sys.argv) > 1 else 'c4'
cfg = configs.CONFIGS[name]
ctx = sk.default_context()
data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param, cfg.t_scale, cfg.tau))
y = data.labels()
lc = sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q)
out = {}
for tag in ("scaled", "ridge", "scaled", "ridge"):
    ctx.synchronize(); t0 = time.perf_counter()
    a = data.scaled(1 / cfg.n ** 0.5) if tag == "scaled" else sk.scaled_design(sk.RidgeProblem(data, y, cfg.lam))
    t1 = time.perf_counter()
    sk.block_lanczos(a, lc, want_right=False)
    ctx.synchronize(); t2 = time.perf_counter()
    out.setdefault(tag, []).append([round(t1 - t0, 4), round(t2 - t1, 4)])
print(json.dumps({"config": name, "handle_s_and_sketch_s": out}))
