"""CPU, world_size 2 over gloo: the row-sharded decomposition the multi-GPU path
uses reproduces the single-process oracle.  The shard layout comes from the
library itself (skr_shard_rows / skr_shard_layout, host-only entry points of
libskr_b200.so); each rank holds an uneven row shard and every collective is the
one capi.cu issues over NCCL: allgather of the local counts, allreduce-sum of the
Krylov / Gram / gradient partials, allreduce-max of the row norms, and grouped
per-rank broadcasts straight into place for the replicated beta table and X~
(Ctx::gather_in_place)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(a, op=dist.ReduceOp.SUM):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    dist.all_reduce(t, op=op)
    return t.numpy()


def _gather_in_place(buf, counts, tail=0):
    """Ctx::gather_in_place: rank r broadcasts rows [off_r, off_r + counts[r]) of buf
    (rooted at r) into the same place on every rank; `tail` trailing rows are rank 0's."""
    off = 0
    for r, c in enumerate(counts):
        if c:
            t = torch.from_numpy(np.ascontiguousarray(buf[off:off + c]))
            dist.broadcast(t, src=r)
            buf[off:off + c] = t.numpy()
        off += c
    if tail:
        t = torch.from_numpy(np.ascontiguousarray(buf[off:off + tail]))
        dist.broadcast(t, src=0)
        buf[off:off + tail] = t.numpy()


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_1602_02350_b200 import configs, skridge as skm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O = oracle.port()
        n, d, k, lam, seed = 203, 17, 3, 1e-3, 11
        rng = np.random.default_rng(5)
        X = rng.standard_normal((n, d)) / np.arange(1, d + 1)
        y = rng.standard_normal(n)
        row0, nl = skm.shard_rows(n, world, rank)
        Xl = X[row0:row0 + nl]
        # shard layout from the allgather of local counts (skr_data_create)
        counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(counts, torch.tensor([nl]))
        ng, r0 = skm.shard_layout([int(c) for c in counts], rank)
        assert (ng, r0) == (n, row0)
        # Pi rows of this shard straight from the reference stream (box_muller_kernel)
        flat = O.gaussian_matrix(n * k, 1, seed)[:, 0]  # the same stream, one column
        Pi = O.gaussian_matrix(n, k, seed)
        # Pi(row0 + i, j) is normal number j * n + row0 + i of gaussian_matrix(n, k, seed)
        # (column-major fill, random.cpp:28-41; box_muller_kernel's indexing)
        Pl = np.array([[flat[j * n + row0 + i] for j in range(k)] for i in range(nl)])
        assert np.array_equal(Pl, Pi[row0:row0 + nl])
        # Krylov products: Pi^T X and T^T X with T = X prev
        assert np.allclose(_allreduce(Pl.T @ Xl), Pi.T @ X, rtol=1e-13, atol=1e-13)
        prev = np.linalg.qr(rng.standard_normal((d, k)))[0]
        assert np.allclose(_allreduce((Xl @ prev).T @ Xl), (X @ prev).T @ X, rtol=1e-12, atol=1e-13)
        # Rayleigh-Ritz Gram
        Q = np.linalg.qr(rng.standard_normal((d, 2 * k)))[0]
        assert np.allclose(_allreduce((Xl @ Q).T @ (Xl @ Q)), (X @ Q).T @ (X @ Q), rtol=1e-12, atol=1e-13)
        # preconditioned components: beta table, row-norm max, full gradient + objective
        sk = O.block_lanczos(X, k, q=3, seed=seed)
        full = O.problem(X, y, lam, sk.U, sk.sigma)
        beta_full = full.betas()
        # (the device computes the local data betas; here they come from the oracle rows)
        all_counts = [skm.shard_rows(n, world, r)[1] for r in range(world)]
        b = np.zeros(n + d)
        b[row0:row0 + nl] = beta_full[row0:row0 + nl]
        if rank == 0:
            b[n:] = beta_full[n:]
        _gather_in_place(b, all_counts, tail=d)
        assert np.array_equal(b, beta_full)
        Xt = full.transformed()
        # the X~ replica for the sequential inner loop: every rank's rows broadcast in place
        rep = np.zeros_like(Xt)
        rep[row0:row0 + nl] = Xt[row0:row0 + nl]
        _gather_in_place(rep, all_counts)
        assert np.array_equal(rep, Xt)
        rows = (Xt[row0:row0 + nl] ** 2).sum(1)
        mx = _allreduce(np.array([rows.max() if nl else 0.0]), dist.ReduceOp.MAX)[0]
        assert mx == pytest.approx(full.scalars()[2], rel=1e-14)
        w = rng.standard_normal(d)
        r = Xt[row0:row0 + nl] @ w - y[row0:row0 + nl]
        sums = _allreduce(np.concatenate([Xt[row0:row0 + nl].T @ r, [r @ r]]))
        D, c = oracle.build_sketched(sk.sigma, lam)
        uw = sk.U.T @ w
        pinv = c * c * w + sk.U @ ((D * D - c * c) * uw)
        mu = sums[:d] / n + lam * pinv
        obj = sums[d] / (2 * n) + 0.5 * lam * (c * c * (w @ w) + ((D * D - c * c) * uw * uw).sum())
        assert np.allclose(mu, full.full_gradient(w), rtol=1e-11, atol=1e-14)
        assert obj == pytest.approx(full.objective(w), rel=1e-12)
        # eta from the global max row norm is identical on every rank
        eta = configs.step_size(mx)
        etas = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(etas, torch.tensor([eta], dtype=torch.float64))
        assert len({float(e) for e in etas}) == 1
        q.put((rank, "ok"))
    except Exception as e:  # surface assertion text to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_row_sharded_decomposition_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
