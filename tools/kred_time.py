import sys; sys.path.insert(0,'.')
import numpy as np
from paper_2507_08954_b200 import _abi, sweep
from paper_2507_08954_b200.engine import Engine
eng = Engine(0)
w = sweep.build(sys.argv[1] if len(sys.argv) > 1 else 'c3', 0, engine=eng)
w.upload(eng)
for outs, name in ((_abi.WANT_STATS | _abi.WANT_HIST, 'stats+hist'), (_abi.WANT_STATS, 'stats')):
    kw = dict(hist_groups=w.groups, hist_rows=w.hist_rows, hist_bins=sweep.HIST_BINS, hist_lo_s=sweep.HIST_LO_S, hist_hi_s=sweep.HIST_HI_S) if outs & _abi.WANT_HIST else {}
    eng.prepare(w.sims_array(), outputs=outs, early_exit=True, **kw)
    for _ in range(3): eng.launch()
    eng.synchronize(); eng.kernel_times()
    for _ in range(5): eng.launch()
    eng.synchronize()
    a, b = eng.kernel_times()
    print(name, 'k_sim %.3f k_reduce %.3f' % (a.mean(), b.mean()))
