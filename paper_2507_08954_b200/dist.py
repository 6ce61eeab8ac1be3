"""Multi-GPU plumbing for sweeps: one process per GPU, no data-path exchange.

Simulations are independent, so a sweep is sharded across
ranks as disjoint blocks of simulations (here: disjoint seed blocks, see
``sweep.build``).  The only collective is the final reduction of the per-GPU
outputs: the log-binned latency histograms (sum) and the per-simulation
summary rows (gather), over NCCL on the GPU box or gloo in the CPU tests.
"""

from __future__ import annotations

import math

import numpy as np


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n items for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def partition(costs, world: int) -> list[list[int]]:
    """Strong-scaling split of ONE fixed sweep over ``world`` ranks: greedy
    LPT on the a-priori costs (sweep.sim_costs), longest first onto the least
    loaded rank that still has room, every rank getting ceil/floor(n/world)
    simulations (equal row blocks for the summary all-gather).  Each rank's
    list is in ascending sim order.  Every rank computes the same split from
    the same inputs, so no exchange is needed before the simulations run."""
    if world < 1:
        raise ValueError("bad world")
    n = len(costs)
    room = [shard_bounds(n, r, world)[1] - shard_bounds(n, r, world)[0] for r in range(world)]
    order = sorted(range(n), key=lambda i: (-costs[i], i))
    load = [0.0] * world
    parts: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        r = min((k for k in range(world) if len(parts[k]) < room[k]), key=lambda k: (load[k], k))
        parts[r].append(i)
        load[r] += costs[i]
    return [sorted(p) for p in parts]


def hist_bin(x, lo: float, hi: float, bins: int):
    """The reducer's latency binning (gfq_engine.cu k_reduce):
    floor((log x - log lo) * bins / (log hi - log lo)), clamped; x <= 0 -> 0."""
    x = np.asarray(x, dtype=np.float64)
    l0 = math.log(lo)
    scale = bins / (math.log(hi) - l0)
    with np.errstate(divide="ignore", invalid="ignore"):
        b = np.floor((np.log(np.where(x > 0, x, 1.0)) - l0) * scale)
    b = np.where(x > 0, b, 0)
    return np.clip(b, 0, bins - 1).astype(np.int64)


def all_reduce_hist(t, group=None):
    """Sum a histogram tensor over all ranks in place (NCCL / gloo)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def gather_rows(t, group=None):
    """All-gather equally shaped per-rank row blocks -> concatenated rows."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return t
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t, group=group)
    return torch.cat(parts, dim=0)
