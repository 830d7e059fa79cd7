"""Sparse (Lazy) path timings on a synthetic RCV1-shaped instance: n points, d
features, ~nnz_per_row nonzeros per point (random columns, power-law column
scale), next to the reference's CPU path (oracle/_ref, OpenMP) on the same CSR.
python profiles/sparse_probe.py [n] [d] [nnz_per_row]"""
import json, os, sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_1602_02350_b200 import configs, skridge as sk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
z = int(sys.argv[3]) if len(sys.argv) > 3 else 80
rng = np.random.default_rng(0)
cnt = np.maximum(1, rng.poisson(z, n))
rp = np.zeros(n + 1, dtype=np.int64)
rp[1:] = np.cumsum(cnt)
p_col = 1.0 / np.arange(1, d + 1) ** 0.8
p_col /= p_col.sum()
ci = np.empty(rp[-1], dtype=np.int32)
for i in range(n):
    ci[rp[i]:rp[i + 1]] = np.sort(rng.choice(d, size=cnt[i], replace=False, p=p_col))
va = rng.standard_normal(rp[-1]) / np.sqrt(z)
va[va == 0] = 1e-3
y = rng.standard_normal(n)
lam, k, q = 1e-5, 30, 3
out = {"n": n, "d": d, "nnz": int(rp[-1]), "k": k, "q": q, "lambda": lam}

ctx = sk.default_context()
t0 = time.perf_counter()
a = sk.DataMatrix.from_csr(rp, ci, va, d)
out["upload_s"] = round(time.perf_counter() - t0, 3)
p = sk.RidgeProblem(a, y, lam)
for rep in range(2):
    ctx.synchronize(); t0 = time.perf_counter()
    sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(k, 0.5, 1, q), want_right=False)
    ctx.synchronize(); out["lanczos_s"] = round(time.perf_counter() - t0, 4)
t0 = time.perf_counter()
pg = sk.preconditioned_components(p, sk.build_sketched(sv, lam))
ctx.synchronize(); out["precompute_s"] = round(time.perf_counter() - t0, 4)
w = rng.standard_normal(d) * 1e-2
pg.full_gradient(w)
ctx.profile(True)
for _ in range(20):
    pg.full_gradient(w)
ms, cnt_ = ctx.profile_read("fullgrad")
out["full_gradient_ms"] = round(ms / max(cnt_, 1), 4)
eta = configs.step_size(pg.max_row_sq())
m = 2 * n
res = sk.svrg_solve(pg, sk.SvrgConfig(2, m, eta, 1), np.zeros(d))
k10, kn = ctx.profile_read("svrg_epoch")
ctx.profile(False)
out["lazy_epoch_ms"] = round(k10 / max(kn, 1), 3)
out["lazy_ns_per_step"] = round(k10 / max(kn, 1) * 1e6 / m, 1)
out["trace"] = [r.objective for r in res.trace]

try:
    import oracle
    if oracle.ref_available():
        R = oracle.ref()
        sub = min(n, 50000)  # bounded CPU sample: the first `sub` points
        csr = (rp[: sub + 1], ci[: rp[sub]], va[: rp[sub]], d)
        po = R.problem_csr(csr, y[:sub], lam, sv.left, sv.singular_values, mode=1)
        po.full_gradient(w)
        t0 = time.perf_counter()
        for _ in range(3):
            po.full_gradient(w)
        out["ref_full_gradient_ms_scaled_to_n"] = round((time.perf_counter() - t0) / 3 * 1e3 * n / sub, 2)
        ms_ = min(20000, 2 * sub)
        t0 = time.perf_counter()
        po.svrg(1, ms_, eta, 1)
        out["ref_lazy_us_per_step"] = round((time.perf_counter() - t0) / ms_ * 1e6, 2)
        out["ref_threads"] = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
except Exception as e:  # noqa: BLE001
    out["ref_error"] = str(e)[:200]
print(json.dumps(out))
