"""Throughput of the C3 sweep against resident simulation warps per SM: the
persistent grid is capped at 148 x k blocks (4 simulation warps each), so
k = 1..4 gives 4..16 warps per SM.  Tells how much latency hiding a larger
occupancy would buy.

    python tools/occ_curve.py [workload]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_08954_b200 import _abi, sweep  # noqa: E402
from paper_2507_08954_b200.engine import Engine  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
eng = Engine(0)
w = sweep.build(wl, 0, engine=eng)
w.upload(eng)
arr = w.sims_array()
for k in (1, 2, 3, 4):
    ms = []
    for rep in range(4):
        eng.run(arr, outputs=_abi.WANT_STATS, early_exit=True, blocks=148 * k)
        ms.append(eng.kernel_ms())
    c = eng.output(_abi.OUT_COUNTERS).reshape(-1, _abi.NCOUNTERS)
    disp = int(c[:, 2].sum())
    t = min(ms[1:])
    print(f"blocks {148 * k:4d} ({4 * k:2d} warps/SM): {t:8.2f} ms  {disp / t / 1e3:8.1f} M disp/s")
torch.cuda.synchronize()
