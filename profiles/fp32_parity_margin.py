"""Margins of the fp32 subsampled-config parity gates (sigma 1e-3, eta 1e-3, L(w^) 1e-5)."""
import sys, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import test_gpu_parity as t
from paper_1602_02350_b200 import configs
for name, nn in (("c3", 16384), ("c4", 16384), ("c5", 16384)):
    try:
        gold = t._golden(f"{name}_n{nn}")
    except Exception as e:
        print(name, "no golden", e); continue
    cfg = configs.CONFIGS[name].scaled(nn)
    X, y = oracle.synth_instance(cfg)
    p, sv, pg, eta, res, L = t._pipeline(cfg, X, y, gold["epochs"])
    print(name, "sigma", t.rel(sv.singular_values, gold["sigma"]), "eta", abs(eta - gold["eta"]) / gold["eta"], "L", abs(L - gold["L_hat"]) / gold["L_hat"], "epochs", gold["epochs"], [r.objective for r in res.trace][-3:], flush=True)
