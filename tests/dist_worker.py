"""Rank worker for tests/test_gpu_dist.py (launched by torch.distributed.run):
every rank runs libgfq on its part of ONE fixed sweep (dist.partition, the
strong split), then the histograms are all-reduced and the summary rows
all-gathered over gloo (two ranks sharing the one GPU); rank 0 re-runs the
whole sweep in one process and writes the comparison to argv[1]."""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_08954_b200 import _abi, sweep  # noqa: E402
from paper_2507_08954_b200.dist import all_reduce_hist, gather_rows, partition  # noqa: E402
from paper_2507_08954_b200.engine import Engine  # noqa: E402


def run(eng, w):
    w.upload(eng)
    eng.run(w.sims_array(), outputs=_abi.WANT_STATS | _abi.WANT_HIST, early_exit=True,
            hist_groups=w.groups, hist_rows=w.hist_rows, hist_bins=sweep.HIST_BINS,
            hist_lo_s=sweep.HIST_LO_S, hist_hi_s=sweep.HIST_HI_S)
    assert (eng.output(_abi.OUT_STATUS) == 0).all()
    return (eng.output(_abi.OUT_HIST).astype(np.int64),
            eng.output(_abi.OUT_SUMMARY).reshape(-1, 3),
            eng.output(_abi.OUT_COUNTERS).reshape(-1, _abi.NCOUNTERS)[:, 2].copy())


def main(out):
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    eng = Engine(0)
    w_full = sweep.c3(n_seeds=2, duration=120.0, engine=eng)
    part = partition(sweep.sim_costs(w_full), world)[rank]
    hist, summ, disp = run(eng, sweep.restrict(w_full, part))
    h = all_reduce_hist(torch.from_numpy(hist))
    rows = gather_rows(torch.from_numpy(np.column_stack([summ, disp.astype(np.float64)])))
    ids = gather_rows(torch.tensor(part, dtype=torch.int64))
    if rank == 0:
        ref_hist, ref_summ, ref_disp = run(eng, w_full)
        got = np.zeros((len(w_full.sims), 4))
        got[ids.numpy()] = rows.numpy()
        res = {"world": world, "sims": len(w_full.sims), "parts": [len(p) for p in
                                                                    partition(sweep.sim_costs(w_full), world)],
               "hist_equal": bool(np.array_equal(h.numpy(), ref_hist)),
               "hist_total": int(ref_hist.sum()), "arrivals": int(w_full.arrivals),
               "summary_equal": bool(np.array_equal(got[:, :3], ref_summ)),
               "dispatches_equal": bool(np.array_equal(got[:, 3], ref_disp.astype(np.float64))),
               "ids_cover": sorted(ids.tolist()) == list(range(len(w_full.sims)))}
        with open(out, "w") as fh:
            json.dump(res, fh)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
