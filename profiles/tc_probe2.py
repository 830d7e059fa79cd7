"""One warm block_lanczos at a config (for ncu captures of the tcgen05 products)."""
import sys
sys.path.insert(0, '.')
from paper_1602_02350_b200 import configs, skridge as sk
cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else 'c5']
data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param, cfg.t_scale, cfg.tau))
a = data.scaled(1 / cfg.n ** 0.5)
sv = sk.block_lanczos(a, sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
sk.default_context().synchronize()
print("ok", sv.singular_values[0])
