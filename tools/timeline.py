"""Per-simulation schedule of one k_sim launch (needs a -DGFQ_TIMELINE=1
build, e.g. GFQ_LIB=paper_2507_08954_b200/var_tl.so): start/end/SM of every
simulation -> slot occupancy, tail and per-SM busy time.

    GFQ_LIB=... python tools/timeline.py [workload]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_08954_b200 import _abi, sweep  # noqa: E402
from paper_2507_08954_b200.engine import Engine  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = sweep.build(wl, 0)
eng = Engine(0)
w.upload(eng)
for rep in range(3):
    eng.run(w.sims_array(), outputs=_abi.WANT_STATS, early_exit=True)
c = eng.output(_abi.OUT_COUNTERS).reshape(-1, _abi.NCOUNTERS)
t0, t1, sm = c[:, 5].astype(np.float64), c[:, 6].astype(np.float64), c[:, 7]
base = t0.min()
t0 = (t0 - base) / 1e6
t1 = (t1 - base) / 1e6
dur = t1 - t0
ev = c[:, 0]
end = t1.max()
print(f"{wl}: {len(dur)} sims, kernel span {end:.2f} ms")
print(f"sim duration ms: min {dur.min():.2f} median {np.median(dur):.2f} max {dur.max():.2f}")
print(f"ns per event: median {np.median(dur * 1e6 / np.maximum(ev, 1)):.0f}")
order = np.argsort(t0)
print("start-time quantiles (ms):", np.quantile(t0, [0, .25, .5, .58, .6, .75, .9, 1]).round(2))
print("end-time quantiles (ms):", np.quantile(t1, [0, .1, .5, .9, .99, 1]).round(2))
busy = np.zeros(int(sm.max()) + 1)
for s, d in zip(sm, dur):
    busy[s] += d
print(f"per-SM busy (sum of sim durations) ms: min {busy.min():.1f} mean {busy.mean():.1f} max {busy.max():.1f}")
# concurrency over time
ts = np.linspace(0, end, 30)
conc = [int(((t0 <= t) & (t1 > t)).sum()) for t in ts]
print("concurrent sims over time:", conc)
last = np.argsort(-t1)[:5]
for i in last:
    print(f"  late sim {i}: start {t0[i]:.2f} end {t1[i]:.2f} dur {dur[i]:.2f} events {ev[i]} sm {sm[i]}")

# Makespan the measured durations would give under LPT with perfect knowledge
# (same slot count, each slot running its simulations back to back).
import heapq
slots = int(max(((t0 <= t) & (t1 > t)).sum() for t in np.linspace(0, end, 200)))
heap = [0.0] * slots
for d_ in sorted(dur.tolist(), reverse=True):
    heapq.heapreplace(heap, heap[0] + d_)
print(f"slots {slots}: perfect-knowledge LPT makespan {max(heap):.2f} ms vs measured {end:.2f} ms")

out = os.environ.get("TIMELINE_OUT")
if out:
    np.savez(out, t0=t0, t1=t1, sm=sm, ev=ev,
             T=np.array([s.t_overrun for s in w.sims]), alpha=np.array([s.alpha for s in w.sims]),
             dcfg=np.array([s.device_cfg for s in w.sims]), trace=np.array([s.trace for s in w.sims]),
             n=np.array([w.traces[s.trace].n for s in w.sims]), order_cost=np.zeros(len(w.sims)))
