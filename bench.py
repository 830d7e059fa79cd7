#!/usr/bin/env python
"""Benchmark of the B200 hot path.

A step is ONE full-gradient pass (the fused K9 pass of
PreconditionedRidge::full_gradient + objective, ridge.cpp:174-236) over the
preconditioned rows X~ of the headline workload: c3 (BASELINE configs[2], the
largest single-GPU config: fp32 storage with fp64 accumulation, n = 2^20 rows
per GPU, d = 2048, k = 128, q = 3).  `value` is the whole-job HBM throughput of
that pass in algorithmic GB/s (n*d*4 bytes of X~ per pass per GPU, all GPUs);
`e2e` is the same metric through the reference-facing C-ABI call with host
buffers (skr_full_gradient: w uploaded, mu and the objective read back every
step).  `--config c2` etc. select another BASELINE config.

Multi-GPU (torchrun): rows are sharded, each rank owns a c3-sized shard (weak
scaling) and the pass ends in one NCCL allreduce of d+1 doubles.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref: the unmodified skridge library, OpenMP on all host cores) on the
same metric, on a bounded row sample of the same instance (see
reference_full_gradient_sample); under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SVRG full-gradient pass throughput (HBM GB/s)"
CLOCK_QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
               "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
               "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the workload runs."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={CLOCK_QUERY}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                self.rows.append(f)

    def summary(self):
        rows = getattr(self, "rows", [])
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        load = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---------------------------------------------------------------------------
REF_SAMPLE_ROWS = 1 << 17   # rows of the instance the CPU reference streams per timed pass (c3: 1/8)
REF_SKETCH_ROWS = 1 << 14   # rows the reference's block_lanczos sees to build U (values do not affect the timing)


def reference_full_gradient_sample(cfg, max_passes: int, budget_s: float, X=None, y=None):
    """The reference's PreconditionedRidge::full_gradient + objective (oracle/_ref: the
    unmodified skridge library, OpenMP on every host core) on a bounded sample of the
    cfg instance: its first min(n, REF_SAMPLE_ROWS) rows, preconditioned with the
    rank-k sketch the reference's own block_lanczos builds from the first
    REF_SKETCH_ROWS rows, apply mode Auto (the reference's stock choice: Lazy when
    n*d > 2e8, ridge.cpp:104-113).  Timed passes stop at max_passes or once budget_s
    is spent.  Returns (seconds per pass, passes, threads, backend, rows, mode, setup_s).
    X, y: the sample rows if the caller already has them (else the host restatement
    of the device generator makes them)."""
    import oracle
    R = oracle.ref() if oracle.ref_available() else oracle.port()
    rows = min(cfg.n, REF_SAMPLE_ROWS)
    t0 = time.perf_counter()
    if X is None:
        X, y = oracle.synth_instance(cfg, rows=rows)
    X = np.ascontiguousarray(X[:rows], dtype=np.float64)
    y = np.ascontiguousarray(y[:rows], dtype=np.float64)
    ks = min(rows, REF_SKETCH_ROWS)
    sv = R.block_lanczos(X[:ks], cfg.k, q=cfg.q, seed=cfg.seed, want_right=False)
    mode = 2 if R.name == "reference" else 0  # ApplyMode::Auto (the port has Dense only)
    prob = R.problem(X, y, cfg.lam, sv.U, sv.sigma, mode)
    setup_s = time.perf_counter() - t0
    w = np.random.default_rng(1).standard_normal(X.shape[1]) * 1e-2
    prob.full_gradient(w)  # warm-up
    prob.objective(w)
    t0 = time.perf_counter()
    k = 0
    while k < max_passes and (k == 0 or time.perf_counter() - t0 < budget_s):
        prob.full_gradient(w)
        prob.objective(w)  # the GPU step also yields the objective
        k += 1
    dt = (time.perf_counter() - t0) / k
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    mode_name = ("lazy" if rows * cfg.d > 200_000_000 else "dense") if mode == 2 else "dense"
    return dt, k, threads, R.name, rows, mode_name, setup_s


def host_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            model = next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")), "")
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def run_reference(args, cfg):
    """--impl reference: the reference CPU path on the same workload (rank 0 only)."""
    import oracle
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libskridge_ref.so not built"}))
        return
    s_bytes = 4 if cfg.dtype == "f32" else 8
    dt, k, threads, kind, rows, mode, setup_s = reference_full_gradient_sample(cfg, max_passes=args.steps,
                                                                               budget_s=90.0)
    val = rows * cfg.d * s_bytes / dt / 1e9
    sample = (f"{k} full_gradient+objective calls of skridge::PreconditionedRidge ({mode} mode, ApplyMode::Auto) "
              f"over the first {rows} of the {cfg.n} rows of the {cfg.name} instance (host restatement of the device "
              f"generator); U from the reference's block_lanczos on the first {min(rows, REF_SKETCH_ROWS)} rows; "
              f"GB/s = rows*d*{s_bytes} algorithmic bytes (the GPU arm's definition) per pass")
    print(json.dumps({
        "metric": METRIC, "value": round(val, 3), "unit": "GB/s", "n_gpus": args.gpus, "steps": k,
        "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype_label(cfg),
        "data": "synthetic (oracle.synth_instance: host restatement of the device Philox generator, same instance)",
        "impl": "reference",
        "config": workload_config(cfg, 1),
        "cpu_baseline": {"value": round(val, 3), "unit": "GB/s", "cores": threads, "kind": kind, "sample": sample,
                         "setup_s": round(setup_s, 2), **host_info()},
        "e2e": {"value": round(val, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def dtype_label(cfg) -> str:
    return "fp32 storage / fp64 accumulate" if cfg.dtype == "f32" else "f64"


def workload_config(cfg, world: int) -> dict:
    s_bytes = 4 if cfg.dtype == "f32" else 8
    return {"workload": f"{cfg.name}: fused full-gradient + objective pass over X~ "
                        f"(n={cfg.n} rows/GPU, d={cfg.d}, {dtype_label(cfg)}, k={cfg.k}, q={cfg.q}, "
                        f"lambda={cfg.lam})",
            "n_per_gpu": cfg.n, "n_total": cfg.n * world, "d": cfg.d, "k": cfg.k, "q": cfg.q, "lambda": cfg.lam,
            "parallelism": f"rows sharded dp{world}",
            "l2": f"inputs larger than L2 (X~ {cfg.n * cfg.d * s_bytes / 1e6:.0f} MB/GPU vs 126 MB L2)"}


# ---------------------------------------------------------------------------
def run_ours(args, cfg):
    import torch
    from paper_1602_02350_b200 import configs, skridge as sk

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    # SKR_BENCH_DIST=1 runs the sharded (NCCL) path even at world 1 (a launch check)
    if world > 1 or os.environ.get("SKR_BENCH_DIST") == "1":
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        nid = [sk.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        ctx = sk.Context(local, rank, world, nid[0])
    else:
        ctx = sk.Context(local)
    sk._default_ctx = ctx
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- workload: c2-shaped shard per GPU, generated on the device
    n_total = cfg.n * world
    spec = sk.SynthSpec(n_total, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param, cfg.t_scale, cfg.tau)
    data = sk.DataMatrix.generate(spec, ctx)
    y = data.labels()
    p = sk.RidgeProblem(data, y, cfg.lam)
    n_loc, d = data.n_local, data.d
    s_bytes = 4 if cfg.dtype == "f32" else 8
    ld = (d + 15) // 16 * 16

    warm_library(sk, configs, ctx)
    walls, gemms, gemms_tc = [], [], []
    for rep in range(4):  # the first call also grows the memory pool; best of the 3 warm calls is reported
        torch.cuda.synchronize()
        barrier()
        ctx.profile(rep >= 1)
        t0 = time.perf_counter()
        sv = sk.block_lanczos(sk.scaled_design(p), sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
        ctx.synchronize()
        wall = max_over_ranks(time.perf_counter() - t0)
        if rep >= 1:
            walls.append(wall)
            gemms.append(max_over_ranks(ctx.profile_read("lanczos_gemm")[0]))
            gemms_tc.append(max_over_ranks(ctx.profile_read("lanczos_gemm_tc")[0]))
        ctx.profile(False)
    lanczos_s, lz_gemm_ms, lz_tc_ms = min(walls), min(gemms), min(gemms_tc)
    for _ in range(2):  # as for the sketch: the second (steady-state) build is reported
        prob = None
        barrier()
        t0 = time.perf_counter()
        pc = sk.build_sketched(sv, cfg.lam)
        prob = sk.preconditioned_components(p, pc)
        ctx.synchronize()
        precompute_s = max_over_ranks(time.perf_counter() - t0)

    # ---- device-resident timed loop: K9 through skr_full_gradient_device
    lib = sk._lib.load()
    w = torch.zeros(ld, dtype=torch.float64, device="cuda")
    w[:d] = torch.randn(d, dtype=torch.float64, device="cuda") * 1e-2
    mu = torch.zeros(ld, dtype=torch.float64, device="cuda")
    obj = torch.zeros(1, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()

    def step():
        rc = lib.skr_full_gradient_device(prob.h, w.data_ptr(), mu.data_ptr(), obj.data_ptr())
        if rc:
            raise RuntimeError(sk._lib.last_error())

    for _ in range(max(3, args.warmup)):
        step()
    ctx.synchronize()
    ctx.profile(True)
    launches0 = ctx.kernel_launches
    barrier()
    torch.cuda.synchronize()
    ctx.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ctx.synchronize()
        launches = ctx.kernel_launches - launches0
        # the dominant kernel's launches inside the timed region only (the soak
        # below runs into the box's power cap and would skew the average)
        k9_ms, k9_n = ctx.profile_read("fullgrad")
        ctx.profile(False)
        # ---- e2e: the reference-facing call with host buffers (w in, mu + objective out),
        # timed right after the device-resident loop (same power state; the soak below runs
        # into the box's power cap)
        wh = w[:d].double().cpu().numpy().copy()
        for _ in range(3):
            prob.full_gradient(wh, with_objective=True)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            prob.full_gradient(wh, with_objective=True)
        e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
        # keep the same loop running ~0.4 s more so the clock sampler sees load
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < 0.4:
            for _ in range(20):
                step()
            ctx.synchronize()
    ms = ev0.elapsed_time(ev1)
    barrier()
    ms = max_over_ranks(ms)
    ms_step = ms / args.steps
    bytes_per_gpu = n_loc * d * s_bytes
    value = world * bytes_per_gpu / (ms_step * 1e-3) / 1e9
    # the dominant kernel: K9's streaming pass (average over the timed launches)
    k9_avg = k9_ms / max(k9_n, 1)
    hbm, bf16, src = peaks()
    achieved = bytes_per_gpu / (k9_avg * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "k9_traffic.json")) as f:
            tj = json.load(f).get(cfg.name)
            traffic = tj.get("traffic_bytes") if tj else None
    except Exception:
        pass

    e2e_value = world * bytes_per_gpu / e2e_s / 1e9

    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": round(ms_step, 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": dtype_label(cfg),
        "data": "synthetic (device Philox4x32-10 generator, BASELINE spectrum)",
        "config": workload_config(cfg, world),
        "passes_per_s": round(1e3 / ms_step, 2),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic,
                     "kernel": k9_kernel_name(cfg), "kernel_ms": round(k9_avg, 5), "peak_source": src,
                     "bytes_per_launch": bytes_per_gpu, "frac_of_8000_spec": round(achieved / 8000.0, 4),
                     "peak_note": "peak = MEASURED_PEAKS hbm_gbs, a read+write copy; a read-only stream "
                                  "(K9 reads X~ once, writes ~0) can exceed it — ncu puts the same launch at "
                                  "81 % of its DRAM peak (profiles/r02_k9_tma_c3_ncu_details.txt)"},
        "e2e": {"value": round(e2e_value, 2), "unit": "GB/s", "h2d_bytes_per_step": d * 8,
                "d2h_bytes_per_step": d * 8 + 8, "ms_per_step": round(e2e_s * 1e3, 4)},
        "gpu_launches": int(launches),
        "gpu_launches_per_step": round(launches / max(1, args.steps), 2),
        "clocks": clk.summary(),
        "lanczos": lanczos_fields(cfg, n_total, n_loc, world, lanczos_s, lz_gemm_ms, lz_tc_ms),
        "precompute_s": round(precompute_s, 4),
    }

    if not args.no_extras:
        try:
            out.update(solve_extras(args, cfg, sk, p, prob, sv, lanczos_s, precompute_s, ctx))
        except Exception as e:  # the headline line must still print
            out["svrg"] = {"error": repr(e)[:300]}
        if world == 1:
            out["lanczos_tf32"] = lanczos_tf32_extra(sk, ctx)
    if world == 1 and not args.no_cpu_baseline and rank == 0:
        rows = min(cfg.n, REF_SAMPLE_ROWS)
        Xs = data.download()[:rows]
        dt, kk, thr, kind, rows, mode, _ = reference_full_gradient_sample(cfg, max_passes=max(3, args.steps),
                                                                          budget_s=15.0, X=Xs, y=y[:rows])
        out["cpu_baseline"] = {"value": round(rows * d * s_bytes / dt / 1e9, 3), "unit": "GB/s", "cores": thr,
                               "kind": kind,
                               "sample": f"{kk} PreconditionedRidge::full_gradient+objective calls (reference, "
                                         f"{mode} mode = ApplyMode::Auto, OpenMP) over the first {rows} rows of "
                                         f"the same {cfg.name} device instance; GB/s = rows*d*{s_bytes} per pass",
                               **host_info()}
    if rank == 0:
        print(json.dumps(out))
    if dist is not None:
        dist.destroy_process_group()


def k9_kernel_name(cfg) -> str:
    """The K9 variant the library dispatches for this shape (capi.cu k9_path)."""
    ld = (cfg.d + 15) // 16 * 16
    row_bytes = ld * (8 if cfg.dtype == "f64" else 4)
    if ld > 1024 or (cfg.dtype == "f32" and row_bytes > 2048):
        return "fullgrad_tma_kernel (K9 v3: bulk-copy tile ring)"
    if cfg.dtype == "f64" and row_bytes > 4096:
        return "fullgrad_rowring_kernel (K9 v5: warp per row, bulk-copy row ring)"
    return "fullgrad_rowwarp_kernel (K9 v4: warp per row)"


FP64_DMMA_TFLOPS = 35.5  # cuBLAS DGEMM 8192^3 measured on this pool's B200 (profiles/fp64_peak.py)


def lanczos_gemm_flops(cfg, n, fp64_path=None):
    """The products skr_lanczos executes (no rank drop).  3xTF32 path: Pi^T X,
    (q-1) x [X prev^T, T^T X], Z = X Q^T for the last block and the Gram Z^T Z
    (fp32-equivalent flops).  fp64 (DMMA) path: Pi^T X, q x [X Q_j^T, T^T X] (the
    last pair gives V_q) and G = Q [V_1..V_q]^T (W x W x d)."""
    d, k, q = cfg.d, cfg.k, cfg.q
    W = q * k
    if fp64_path is None:
        fp64_path = cfg.dtype == "f64"
    if fp64_path:
        return 2 * n * d * k + 4 * n * d * k * q + 2 * W * W * d
    return 2 * n * d * k + 4 * n * d * k * (q - 1) + 2 * n * d * k + 2 * n * W * W


def lanczos_flops(cfg, n):
    """2ndk + 4ndk(q-1) + 2nd*qk + n(qk)^2 algorithmic flops."""
    d, k, q = cfg.d, cfg.k, cfg.q
    return 2 * n * d * k + 4 * n * d * k * (q - 1) + 2 * n * d * q * k + n * (q * k) ** 2


TF32_DENSE_TFLOPS = 1100.0  # B200 dense TF32 tensor peak (B200_PROFILING.md table; not measured on this pool)


def lanczos_fields(cfg, n_total, n_loc, world, wall_s, gemm_ms, tc_ms):
    """The sketch's path and throughput.  fp64 data: DMMA products.  fp32 storage:
    3xTF32 tcgen05 products, redone on the fp64 DMMA path when the Rayleigh-Ritz
    spectrum is too ill-conditioned for fp32 accumulation (capi.cu rr_needs_fp64;
    c3: lambda_1 / lambda_128 = 2e6)."""
    if cfg.dtype == "f64":
        path = "fp64 DMMA (mma.sync m8n8k4)"
    elif gemm_ms > 0.0:
        path = "3xTF32 tcgen05 attempt, redone on fp64 DMMA (ill-conditioned Ritz spectrum)"
    else:
        path = "3xTF32 tcgen05"
    final_ms = gemm_ms if gemm_ms > 0.0 else tc_ms
    dmma = gemm_ms > 0.0
    tf = lanczos_gemm_flops(cfg, n_loc, fp64_path=dmma) / (max(final_ms, 1e-6) * 1e-3) / 1e12
    out = {"seconds": round(wall_s, 4), "path": path,
           "tflops": round(lanczos_flops(cfg, n_total) / wall_s / 1e12 / world, 4),
           "note": "whole block_lanczos call incl. Pi stream, ortho, RR, eigensolve (and a discarded tc attempt)",
           "gemm_ms": round(final_ms, 4), "gemm_tflops_per_gpu": round(tf if dmma else 3 * tf, 3),
           "gemm_peak_tflops": FP64_DMMA_TFLOPS if dmma else TF32_DENSE_TFLOPS,
           "gemm_frac": round((tf if dmma else 3 * tf) / (FP64_DMMA_TFLOPS if dmma else TF32_DENSE_TFLOPS), 3),
           "gemm_note": "Krylov + Rayleigh-Ritz products only (device events); fp64 peak = measured cuBLAS DGEMM "
                        "8192^3 on this B200 (profiles/fp64_peak.py); TF32 = raw 3xTF32 throughput vs the dense TF32 "
                        "nominal"}
    if tc_ms > 0.0 and dmma:
        out["tc_attempt_ms"] = round(tc_ms, 4)
    return out


def lanczos_tf32_extra(sk, ctx):
    """The tensor-core sketch where it is the one used: c5 (configs[4]: fp32 storage,
    n = 2^24, d = 1024, k = 64, q = 2, well-conditioned 0.99^j spectrum): warm
    block_lanczos wall time and the Krylov + Rayleigh-Ritz products' device time (CUDA
    events), as raw TF32 tensor throughput (3 MMAs per 3xTF32 product) against the
    dense TF32 peak."""
    from paper_1602_02350_b200 import configs
    c5 = configs.CONFIGS["c5"]
    data = sk.DataMatrix.generate(sk.SynthSpec(c5.n, c5.d, c5.dtype, c5.seed, c5.spectrum, c5.spectrum_param,
                                               c5.t_scale, c5.tau), ctx)
    a = data.scaled(1 / math.sqrt(c5.n))
    lc = sk.LanczosConfig(c5.k, 0.5, c5.seed, c5.q)
    sk.block_lanczos(a, lc, want_right=False)  # cold call: workspaces
    ctx.synchronize()
    walls, gemms = [], []
    for _ in range(3):  # best of three warm calls (the box's power state moves tensor-heavy phases)
        ctx.profile(True)
        t0 = time.perf_counter()
        sk.block_lanczos(a, lc, want_right=False)
        ctx.synchronize()
        walls.append(time.perf_counter() - t0)
        gemms.append(ctx.profile_read("lanczos_gemm_tc")[0])
        ctx.profile(False)
    wall, gemm_ms = min(walls), min(gemms)
    tf = lanczos_gemm_flops(c5, c5.n, fp64_path=False) / (max(gemm_ms, 1e-6) * 1e-3) / 1e12
    del a, data
    return {"config": "c5 (fp32 storage, n=16777216, d=1024, k=64, q=2)", "path": "3xTF32 tcgen05",
            "seconds": round(wall, 4), "gemm_ms": round(gemm_ms, 3), "gemm_tflops_fp32_equiv": round(tf, 1),
            "tf32_raw_tflops": round(3 * tf, 1), "tf32_peak_tflops": TF32_DENSE_TFLOPS,
            "tf32_frac": round(3 * tf / TF32_DENSE_TFLOPS, 3),
            "note": "3xTF32 tcgen05 products (hi.hi + hi.lo + lo.hi); peak = dense TF32 nominal from "
                    "B200_PROFILING.md (the measured bf16 burst is 0.74x its nominal)"}


def solve_extras(args, cfg, sk, p, prob, sv, lanczos_s, precompute_s, ctx):
    """Epoch time and time-to-eps (eps = 1e-6 absolute suboptimality) of the full solve."""
    from paper_1602_02350_b200 import configs
    ref = sk.reference_minimum(p)
    eta = configs.eta_for(cfg, prob.max_row_sq(), prob.mean_beta())
    m = 2 * p.count()
    ctx.profile(True)
    res = sk.svrg_solve(prob, sk.SvrgConfig(cfg.epochs, m, eta, cfg.seed), None, ref.minimum)
    k10_ms, k10_n = ctx.profile_read("svrg_epoch")
    ctx.profile(False)
    eps = 1e-6
    hit = next((r for r in res.trace if r.suboptimality is not None and r.suboptimality <= eps), None)
    w_hat = prob.apply_inv_sqrt(res.iterate)
    L = sk.objective(p, w_hat)
    return {"svrg": {
        "epochs": len(res.trace), "m": m, "eta": eta, "L_star": ref.minimum, "L_final": L,
        "suboptimality_final": L - ref.minimum,
        "epoch_ms": round(res.trace[-1].elapsed_ms / len(res.trace), 3),
        "inner_loop_ms_per_epoch": round(k10_ms / max(k10_n, 1), 3),
        "inner_loop_ns_per_step": round(k10_ms / max(k10_n, 1) * 1e6 / m, 2),
        "time_to_eps_s": None if hit is None else round(lanczos_s + precompute_s + hit.elapsed_ms / 1e3, 4),
        "epochs_to_eps": None if hit is None else hit.epoch,
        "trace": [r.objective for r in res.trace][:10]}}


def warm_library(sk, configs, ctx):
    """One-time library initialisation (solver handles, kernel attributes, the
    mt19937_64 jump tables, memory-pool growth) on a small instance, outside
    every timed phase — the CPU reference has no such cost to amortise."""
    wd = sk.DataMatrix.generate(sk.SynthSpec(1 << 19, 64, "f64", 9, 0, 0.0, False, 0.1), ctx)
    wp = sk.RidgeProblem(wd, wd.labels(), 1e-3)
    wsv = sk.block_lanczos(sk.scaled_design(wp), sk.LanczosConfig(8, 0.5, 1, 2))
    wprob = sk.preconditioned_components(wp, sk.build_sketched(wsv, 1e-3))
    sk.svrg_solve(wprob, sk.SvrgConfig(2, 1 << 20, configs.step_size(wprob.max_row_sq()), 1), None,
                  sk.reference_minimum(wp).minimum)
    # every inner-loop geometry (chain slice widths 32 / 64 / 128 / 256, both storage types): the
    # first launch of a kernel instantiation loads its code (CUDA lazy loading, tens of ms)
    for d in (1024, 2048, 4096):
        for dt in ("f64", "f32"):
            gd = sk.DataMatrix.generate(sk.SynthSpec(4096, d, dt, 9, 0, 0.0, False, 0.1), ctx)
            gp = sk.RidgeProblem(gd, gd.labels(), 1e-3)
            gsv = sk.block_lanczos(sk.scaled_design(gp), sk.LanczosConfig(8, 0.5, 1, 2))
            gprob = sk.preconditioned_components(gp, sk.build_sketched(gsv, 1e-3))
            sk.svrg_solve(gprob, sk.SvrgConfig(1, 8192, configs.step_size(gprob.max_row_sq()), 1), np.zeros(d))
    ctx.synchronize()


class DistEnv:
    """One process per GPU (torchrun): NCCL process group for the timing plumbing,
    the library's own distributed context for the data path."""

    def __init__(self, sk, force: bool = False):
        import torch
        self.torch = torch
        self.rank, self.world, self.local = dist_env()
        torch.cuda.set_device(self.local)
        self.dist = None
        if self.world > 1 or force:
            import torch.distributed as dist
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            nid = [sk.Context.nccl_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(nid, src=0)
            self.ctx = sk.Context(self.local, self.rank, self.world, nid[0])
            self.dist = dist
        else:
            self.ctx = sk.Context(self.local)
        sk._default_ctx = self.ctx

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.dist is None:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist is not None:
            self.dist.destroy_process_group()


def run_solve(args):
    """End-to-end time-to-eps (eps = 1e-6 absolute suboptimality) per config on N
    GPUs (torchrun, one process per GPU; N = 1 without it): the config's instance
    (fixed size: strong scaling) is row-sharded across the ranks; sketch
    (block_lanczos: NCCL allreduce of the Krylov partials) + precompute
    (preconditioned_components: sharded X~, grouped in-place broadcast of the
    replica) + SVRG epochs (the sequential chain replicated on every rank, the
    full gradient row-sharded) until the first epoch with L(w_s) - L* <= eps (cap:
    cfg.epochs), as SketchedSolveDiagnostics and bench.cpp:182-189 time it; every
    phase is the max over ranks.  c5 adds the BASELINE lambda sweep, preconditioned
    vs unpreconditioned, with one sketch reused across lambdas.  With --cpu-ref,
    rank 0 then times the reference's own pipeline (oracle/_ref, OpenMP on every
    host core) on the first n/--cpu-ref-frac rows of the same instance."""
    from paper_1602_02350_b200 import configs, skridge as sk
    E = DistEnv(sk, force=os.environ.get("SKR_BENCH_DIST") == "1")
    ctx = E.ctx
    eps = 1e-6
    warm_library(sk, configs, ctx)
    for name in args.solve.split(","):
        cfg = configs.CONFIGS[name]
        spec = sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param, cfg.t_scale, cfg.tau)
        data = sk.DataMatrix.generate(spec, ctx)
        y = data.labels()
        # the sketch twice: the first call also grows the device memory pool to
        # this size; the second (reported) is the steady-state cost
        for _ in range(2):
            ctx.synchronize()
            E.barrier()
            t0 = time.perf_counter()
            sv = sk.block_lanczos(sk.scaled_design(sk.RidgeProblem(data, y, cfg.lam)),
                                  sk.LanczosConfig(cfg.k, 0.5, cfg.seed, cfg.q), want_right=False)
            ctx.synchronize()
            sketch_s = E.max(time.perf_counter() - t0)
        lams = [1e-4, 1e-6, 1e-8] if name == "c5" else [cfg.lam]
        if args.lambdas:
            lams = [float(x) for x in args.lambdas.split(",")]
        for lam in lams:
            p = sk.RidgeProblem(data, y, lam)
            E.barrier()
            t0 = time.perf_counter()
            ref = sk.reference_minimum(p)
            refmin_s = E.max(time.perf_counter() - t0)
            for method in (["sketched-svrg", "svrg"] if name == "c5" else ["sketched-svrg"]):
                prob = None
                for _ in range(2):  # as for the sketch: the first build also grows the memory pool
                    prob = None
                    E.barrier()
                    t0 = time.perf_counter()
                    pc = (sk.build_sketched(sv, lam) if method == "sketched-svrg"
                          else sk.Preconditioner.identity(cfg.d, lam))
                    prob = sk.preconditioned_components(p, pc)
                    ctx.synchronize()
                    pre_s = E.max(time.perf_counter() - t0)
                eta = configs.eta_for(cfg, prob.max_row_sq(), prob.mean_beta())
                m = 2 * cfg.n
                row = {"solve": name, "method": method, "lambda": lam, "n": cfg.n, "d": cfg.d, "dtype": cfg.dtype,
                       "n_gpus": E.world, "scaling": "strong (rows of one instance sharded)",
                       "k": cfg.k if method == "sketched-svrg" else 0, "q": cfg.q, "m": m, "eta": eta,
                       "beta_hat": prob.mean_beta(), "alpha": prob.strong_convexity(),
                       "sketch_s": round(sketch_s, 4) if method == "sketched-svrg" else 0.0,
                       "precompute_s": round(pre_s, 4), "reference_minimum_s": round(refmin_s, 4),
                       "L_star": ref.minimum}
                try:
                    ctx.profile(True)
                    E.barrier()
                    res = sk.svrg_solve(prob, sk.SvrgConfig(cfg.epochs, m, eta, cfg.seed), None, ref.minimum,
                                        stop_suboptimality=eps)
                    k10_ms, k10_n = ctx.profile_read("svrg_epoch")
                    tab_ms, _ = ctx.profile_read("tables")
                    ind_ms, ind_n = ctx.profile_read("indices")
                    k9_ms, k9_n = ctx.profile_read("fullgrad")
                    ctx.profile(False)
                    row.update({"tables_ms": round(tab_ms, 3), "indices_ms_per_epoch": round(ind_ms / max(ind_n, 1), 3),
                                "fullgrad_ms": round(k9_ms / max(k9_n, 1), 3),
                                "inner_loop_ms_per_epoch": round(k10_ms / max(k10_n, 1), 3)})
                    hit = next((r for r in res.trace if r.suboptimality is not None and r.suboptimality <= eps), None)
                    setup = row["sketch_s"] + pre_s
                    solve_s = E.max((hit.elapsed_ms if hit else res.trace[-1].elapsed_ms) / 1e3)
                    row.update({
                        "epochs_run": len(res.trace), "epochs_to_eps": hit.epoch if hit else None,
                        "time_to_eps_s": round(setup + solve_s, 4) if hit else None,
                        "epoch_ms": round(res.trace[-1].elapsed_ms / len(res.trace), 3),
                        "inner_loop_ns_per_step": round(k10_ms / max(k10_n, 1) * 1e6 / m, 2),
                        "suboptimality": [r.suboptimality for r in res.trace]})
                except sk.DivergenceError as e:
                    ctx.profile(False)
                    row.update({"diverged": str(e), "suboptimality": [r.suboptimality for r in e.trace]})
                if E.rank == 0:
                    print(json.dumps(row), flush=True)
                del prob
        del data
    if args.cpu_ref and E.rank == 0:
        for name in args.solve.split(","):
            for row in reference_solve_rows(configs.CONFIGS[name], args.cpu_ref_frac, eps, args.lambdas):
                print(json.dumps(row), flush=True)
    E.close()


def reference_solve_rows(cfg, frac: int, eps: float, lambdas: str = ""):
    """The reference's own time-to-eps protocol (ridge.cpp:413-454 + bench.cpp:182-189:
    block_lanczos (q_override) -> build_sketched -> preconditioned_components(Auto)
    -> reference_minimum -> svrg_solve until suboptimality <= eps) with
    SketchedSolveDiagnostics-style phase timings, on the first n / frac rows of the
    cfg instance (host restatement of the device generator), OpenMP on every host
    core.  Sketch and precompute scale ~linearly in n, epochs cost ~2n steps, so the
    full-size figure is extrapolated linearly in n and labelled so."""
    import oracle
    if not oracle.ref_available():
        return [{"solve": cfg.name, "impl": "reference", "unavailable": "oracle/_ref not built"}]
    from paper_1602_02350_b200 import configs
    rows = max(1, cfg.n // frac)
    sub = cfg.scaled(rows)
    X, y = oracle.synth_instance(sub)
    lams = [1e-4, 1e-6, 1e-8] if cfg.name == "c5" else [cfg.lam]
    if lambdas:
        lams = [float(x) for x in lambdas.split(",")]
    out = []
    for lam in lams:
        for method in (["sketched-svrg", "svrg"] if cfg.name == "c5" else ["sketched-svrg"]):
            t0 = time.perf_counter()
            epochs = min(cfg.epochs, 6 if cfg.name == "c5" else 12)  # the solve runs whole; the trace is cut at eps
            po = oracle.pipeline(X, y.astype(np.float64), lam, cfg.k if method == "sketched-svrg" else 0, cfg.q,
                                 cfg.seed, epochs, 2 * rows, eta_rule=0 if cfg.name in ("c1", "c2") else 1,
                                 stop=eps)
            wall = time.perf_counter() - t0
            hit = next((i for i, v in enumerate(po.trace) if v - po.L_star <= eps), None)
            t_eps = None if hit is None else (po.sketch_ms + po.precompute_ms + float(po.trace_ms[hit])) / 1e3
            out.append({"solve": cfg.name, "impl": "reference", "method": method, "lambda": lam,
                        "rows": rows, "n": cfg.n, "sample": f"first n/{frac} rows of the {cfg.name} instance",
                        "threads": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)), **host_info(),
                        "mode": po.mode, "sketch_s": round(po.sketch_ms / 1e3, 3),
                        "precompute_s": round(po.precompute_ms / 1e3, 3),
                        "reference_minimum_s": round(po.refmin_ms / 1e3, 3), "solve_s": round(po.solve_ms / 1e3, 3),
                        "epochs_to_eps": None if hit is None else hit + 1,
                        "time_to_eps_s_at_sample": None if t_eps is None else round(t_eps, 3),
                        "time_to_eps_s_full_extrapolated": None if t_eps is None else round(t_eps * frac, 2),
                        "extrapolation": f"linear in n (x{frac}); measured at n/{frac}",
                        "wall_s": round(wall, 2)})
    return out


def run_sweep(args):
    """K9 alone at every BASELINE shape (identity preconditioner: X~ = X, no copy)."""
    import torch
    from paper_1602_02350_b200 import configs, skridge as sk
    ctx = sk.Context(0)
    sk._default_ctx = ctx
    hbm, _, src = peaks()
    rows = []
    for name in args.sweep.split(","):
        cfg = configs.CONFIGS[name]
        spec = sk.SynthSpec(cfg.n, cfg.d, cfg.dtype, cfg.seed, cfg.spectrum, cfg.spectrum_param, cfg.t_scale, cfg.tau)
        t0 = time.perf_counter()
        data = sk.DataMatrix.generate(spec, ctx)
        gen_s = time.perf_counter() - t0
        p = sk.RidgeProblem(data, data.labels(), cfg.lam)
        prob = sk.preconditioned_components(p, sk.Preconditioner.identity(cfg.d, cfg.lam))
        ld = (cfg.d + 15) // 16 * 16
        w = torch.zeros(ld, dtype=torch.float64, device="cuda")
        w[: cfg.d] = 1e-2
        mu = torch.zeros(ld, dtype=torch.float64, device="cuda")
        obj = torch.zeros(1, dtype=torch.float64, device="cuda")
        lib = sk._lib.load()
        for _ in range(3):
            lib.skr_full_gradient_device(prob.h, w.data_ptr(), mu.data_ptr(), obj.data_ptr())
        ctx.profile(True)
        stream = torch.cuda.ExternalStream(ctx.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(3, min(50, int(2e10 // (cfg.n * cfg.d * (4 if cfg.dtype == "f32" else 8)))))
        e0.record(stream)
        for _ in range(reps):
            lib.skr_full_gradient_device(prob.h, w.data_ptr(), mu.data_ptr(), obj.data_ptr())
        e1.record(stream)
        ctx.synchronize()
        k_ms, k_n = ctx.profile_read("fullgrad")
        ctx.profile(False)
        byts = cfg.n * cfg.d * (4 if cfg.dtype == "f32" else 8)
        step_ms = e0.elapsed_time(e1) / reps
        kern_ms = k_ms / max(k_n, 1)
        rows.append({"config": name, "bytes": byts, "kernel_ms": round(kern_ms, 4), "step_ms": round(step_ms, 4),
                     "kernel_GBps": round(byts / kern_ms / 1e6, 1), "step_GBps": round(byts / step_ms / 1e6, 1),
                     "frac": round(byts / kern_ms / 1e6 / hbm, 4), "gen_s": round(gen_s, 2)})
        print(json.dumps(rows[-1]), flush=True)
        del prob, p, data
    print(json.dumps({"k9_sweep": rows, "peak_GBps": hbm, "peak_source": src}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweep", default="", help="comma list of configs: K9 alone at each shape")
    ap.add_argument("--solve", default="", help="comma list of configs: end-to-end time-to-eps per config")
    ap.add_argument("--lambdas", default="", help="--solve: override the lambda list")
    ap.add_argument("--cpu-ref", action="store_true", help="--solve: also time the reference pipeline (rank 0)")
    ap.add_argument("--cpu-ref-frac", type=int, default=16, help="--solve --cpu-ref: rows sample n / frac")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    from paper_1602_02350_b200 import configs
    cfg = configs.CONFIGS[args.config]
    if args.sweep:
        run_sweep(args)
        return
    if args.solve:
        run_solve(args)
        return
    if args.impl == "reference":
        rank, world, _ = dist_env()
        if rank != 0:
            return
        run_reference(args, cfg)
        return
    run_ours(args, cfg)


if __name__ == "__main__":
    main()
