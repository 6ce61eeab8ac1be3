"""Per-phase cycle breakdown of the event loop (needs a -DGFQ_PROF=1 build,
e.g. GFQ_LIB=paper_2507_08954_b200/var_prof.so): each simulation's lane 0
accumulates clock64() cycles per phase of WarpSim::run (sim_warp.cuh):
pool minimum, keep-alive refresh scan (inside the drain), drain, tick runs,
arrivals, completions, expiries + swap-outs.  Prints the totals, the share
of each phase and cycles per unit.

    GFQ_LIB=... python tools/prof_phases.py [workload] [--seeds N] [--flags cta|warp]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_08954_b200 import _abi, sweep  # noqa: E402
from paper_2507_08954_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="c3")
ap.add_argument("--seeds", type=int, default=None)
ap.add_argument("--flags", default="")
a = ap.parse_args()
kw = {"n_seeds": a.seeds} if a.seeds else {}
eng = Engine(0)
w = sweep.build(a.workload, 0, engine=eng, **kw)
w.upload(eng)
flags = {"": 0, "cta": _abi.FLAG_CTA, "warp": _abi.FLAG_WARP}[a.flags]
for rep in range(2):
    eng.run(w.sims_array(), outputs=_abi.WANT_STATS, early_exit=True, flags=flags)
c = eng.output(_abi.OUT_COUNTERS).reshape(-1, _abi.NCOUNTERS).astype(np.float64)
ev, calls, disp, ticks = c[:, 0].sum(), c[:, 1].sum(), c[:, 2].sum(), c[:, 3].sum()
names = ["pool_min", "refresh_scan", "drain(+refresh)", "tick_runs", "arrivals", "completions",
         "expiry+swap"]
tot = c[:, 5:12].sum(axis=0)
loop = tot[[0, 2, 3, 4, 5, 6]].sum()
print(f"{a.workload}: {len(c)} sims, events {ev:.0f}, dispatch calls {calls:.0f}, "
      f"dispatches {disp:.0f}, ticks {ticks:.0f}")
print(f"measured phases total {loop / 1e9:.3f} G cycles = {loop / ev:.0f} cycles/event "
      f"(per sim: mean {loop / len(c) / 1e6:.2f} M cycles)")
units = {"pool_min": ev, "refresh_scan": ev, "drain(+refresh)": disp, "tick_runs": ticks,
         "arrivals": disp, "completions": disp, "expiry+swap": ev}
for n, v in zip(names, tot):
    print(f"  {n:16s} {v / 1e9:8.3f} G cyc  {100 * v / loop:5.1f}%  {v / units[n]:8.0f} per "
          f"{'dispatch' if units[n] is disp else 'tick' if units[n] is ticks else 'event'}")
per_sim = c[:, 5:12][:, [0, 2, 3, 4, 5, 6]].sum(axis=1)
print(f"per-sim cycles: min {per_sim.min() / 1e6:.2f}M median {np.median(per_sim) / 1e6:.2f}M "
      f"max {per_sim.max() / 1e6:.2f}M")
