import sys, time, json
sys.path.insert(0, '.')
from paper_1602_02350_b200 import configs, skridge as sk
name = sys.argv[1]
cfg = configs.CONFIGS[name]
ctx = sk.default_context()
data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param, cfg.t_scale, cfg.tau))
y = data.labels()
out = []
for i in range(8):
    ctx.synchronize()
    ctx.profile(True)
    t0 = time.perf_counter()
    sv = sk.block_lanczos(sk.scaled_design(sk.RidgeProblem(data, y, cfg.lam)), sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
    ctx.synchronize()
    w = time.perf_counter() - t0
    g = ctx.profile_read("lanczos_gemm")[0]; gt = ctx.profile_read("lanczos_gemm_tc")[0]
    ctx.profile(False)
    out.append((round(w, 4), round(g, 1), round(gt, 1)))
print(name, out)
