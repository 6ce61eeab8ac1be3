"""World-size-2 gloo run of the multi-GPU sweep plumbing on CPU: each rank
takes its part of a small fixed sweep (dist.partition, the strong split
bench.py --split strong uses), simulates it with the CPU oracle (as the
stand-in for its GPU; tests/test_gpu_dist.py runs the same with libgfq),
bins latencies into the sweep histogram and the ranks all-reduce; the
result must equal the single-process histogram of the whole sweep, and the
gathered summary rows must cover every simulation."""

from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_hist(rank, world):
    from oracle import oracle as orc
    from paper_2507_08954_b200 import _abi, sweep
    from paper_2507_08954_b200.dist import hist_bin, partition
    w = sweep.c3(n_seeds=1, duration=40.0)
    part = partition(sweep.sim_costs(w), world)[rank]
    hist = np.zeros((w.groups, w.hist_rows, sweep.HIST_BINS), dtype=np.int64)
    rows = []
    for i in part:
        s = w.sims[i]
        tr, tab = w.traces[s.trace], w.tabs[s.flowtab]
        r = orc.run_packed(_abi.Sim.from_buffer_copy(s), tr.arrival, tr.flow, tr.n_flows,
                           {"warm": tab.warm, "cold": tab.cold, "mem": tab.mem,
                            "share": tab.share, "weight": tab.weight},
                           [_abi.device_cfg_from(w.dcfgs[s.device_cfg])], want_audit=False,
                           want_dispatch=False)
        inv = r["rec_inv"]
        lat = r["rec_complete"] - tr.arrival[inv]
        b = hist_bin(lat, sweep.HIST_LO_S, sweep.HIST_HI_S, sweep.HIST_BINS)
        np.add.at(hist, (s.group, tab.hist_row[tr.flow[inv]], b), 1)
        rows.append([i, r["weighted_avg_latency"], len(inv)])
    return hist, np.array(rows, dtype=np.float64).reshape(-1, 3)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_08954_b200.dist import all_reduce_hist, gather_rows
    hist, rows = _shard_hist(rank, world)
    t = all_reduce_hist(torch.from_numpy(hist))
    pad = torch.full((256, 3), -1.0, dtype=torch.float64)
    pad[: rows.shape[0]] = torch.from_numpy(rows)
    g = gather_rows(pad)
    if rank == 0:
        out.put((t.numpy().copy(), g.numpy().copy()))
    dist.destroy_process_group()


def test_two_rank_histogram_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    hist, rows = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref, ref_rows = _shard_hist(0, 1)
    assert np.array_equal(hist, ref)
    got = rows[rows[:, 0] >= 0]
    got = got[np.argsort(got[:, 0])]
    assert np.array_equal(got, ref_rows)


def test_partition_is_a_balanced_cover():
    from paper_2507_08954_b200 import sweep
    from paper_2507_08954_b200.dist import partition
    w = sweep.c5(n_traces=3, duration=60.0)
    costs = sweep.sim_costs(w)
    for world in (1, 2, 3, 8):
        parts = partition(costs, world)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(costs)))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1
        loads = [sum(costs[i] for i in p) for p in parts]
        assert max(loads) <= sum(costs) / world + max(costs)      # LPT bound
