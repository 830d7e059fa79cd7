"""bench.cpp run_convergence protocol on the GPU: eta grid (7 points) x seeds x
{svrg, sketched-svrg}, with the grid run as concurrent chains (lanes=7) vs one
after another (lanes=1).  python profiles/convergence_probe.py [config] [epochs] [prep_cap|default]"""
import json, sys, time
sys.path.insert(0, '.')
from paper_1602_02350_b200 import configs, skridge as sk
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cap = None if len(sys.argv) <= 3 or sys.argv[3] == "default" else int(sys.argv[3])
cfg = configs.CONFIGS[name]
data = sk.DataMatrix.generate(sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param,
                                           cfg.t_scale, cfg.tau))
p = sk.RidgeProblem(data, data.labels(), cfg.lam)
bc = sk.BenchConfig(lam=cfg.lam, k=cfg.k, epochs=epochs, seeds=[0, 1])
sk.run_convergence(p, sk.BenchConfig(lam=cfg.lam, k=cfg.k, epochs=1, seeds=[0]), lanes=7)  # warm
out = {"config": name, "epochs": epochs, "seeds": bc.seeds, "grid": 7, "prep_cap": cap if cap is not None else "default"}
for lanes in (1, 7):
    t0 = time.perf_counter()
    rows = sk.run_convergence(p, bc, lanes=lanes, prep_cap=cap)
    out[f"seconds_lanes{lanes}"] = round(time.perf_counter() - t0, 3)
    out[f"final_lanes{lanes}"] = {f"{r.method}/{r.seed}": r.suboptimality for r in rows if r.epoch == epochs}
out["speedup"] = round(out["seconds_lanes1"] / out["seconds_lanes7"], 2)
print(json.dumps(out))
