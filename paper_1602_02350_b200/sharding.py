"""Row sharding used by the distributed path (one process per GPU).

Mirrors the C-ABI's layout exactly: skr_data_generate splits n rows as
n_local = n // world + (rank < n % world), row0 = rank * (n // world) +
min(rank, n % world); skr_data_create takes caller shards in rank order and
derives n_global / row0 by an allgather of the local counts.  The collectives
of the row-sharded stages are all sums over disjoint row blocks:

  * Krylov products  Pi^T X, T^T X     -> allreduce(sum) of k x d partials
  * Rayleigh-Ritz Gram (X Q)^T (X Q)    -> allreduce(sum) of qk x qk
  * beta table                          -> each rank writes its rows at row0,
                                           rank 0 the d regulariser entries,
                                           allreduce(sum) over the zeros
  * full gradient / objective           -> allreduce(sum) of d+1 doubles
  * max_i ||x~_i||^2                    -> allreduce(max)
"""
from __future__ import annotations


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """(row0, n_local) of `rank` for n rows over `world` ranks."""
    base, extra = divmod(n, world)
    n_local = base + (1 if rank < extra else 0)
    row0 = rank * base + min(rank, extra)
    return row0, n_local


def layout_from_counts(counts: list[int], rank: int) -> tuple[int, int]:
    """(n_global, row0) from every rank's local row count (skr_data_create)."""
    return sum(counts), sum(counts[:rank])


def pi_normal_index(j: int, i_local: int, row0: int, n_global: int) -> int:
    """Stream position of Pi(row0 + i_local, j) in gaussian_matrix(n, k, seed)
    (column-major fill, random.cpp:28-41)."""
    return j * n_global + row0 + i_local
