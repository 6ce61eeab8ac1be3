"""Measurement of the fairness-audit reducer (`k_fairness`):
metrics.service_gap_report (reference metrics.py:106-187) for every
simulation of the C3 sweep (4096 MQFQ-Sticky simulations, 30 s windows), on
the GPU, against the UNMODIFIED reference's service_gap_report (baseline/_ref)
on the host over a random sample of the same simulations, fed the same
records and audit (the engine's, reference-shaped).  Also checks that the
sampled reference windows equal the GPU's.

    python tools/fair_bench.py [--sample N] [--reps K] [--out file.json]
"""
import argparse
import json
import os
import random
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_08954_b200 import _abi, sweep  # noqa: E402
from paper_2507_08954_b200.engine import BatchResult, Engine, to_sim_result  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sample", type=int, default=128)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--out", default="")
a = ap.parse_args()

eng = Engine(0)
w = sweep.build("c3", 0, engine=eng)
w.upload(eng)
arr = w.sims_array()
cap = 1 << 15
eng.run(arr, outputs=_abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_AUDIT, early_exit=True,
        audit_util_cap=cap, audit_backlog_cap=cap)
res = BatchResult(eng)
assert (res.status == 0).all(), "audit buffers overflowed"
rw = np.ones(sum(t.n_flows for t in w.traces), dtype=np.float64)
dmax = np.array([2] * len(w.sims), dtype=np.int32)           # SchedulerConfig().d_max
# GPU: k_fairness over the whole batch (the call synchronizes), best of reps
ms = []
for _ in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fr = eng.fairness(dmax, rw, 30.0)
    ms.append((time.perf_counter() - t0) * 1e3)
counts = fr.count
n_win = int(counts[:, 0].sum())
gpu_ms = min(ms)

# reference: service_gap_report on a random sample, same inputs
ref = os.path.join(ROOT, "baseline", "_ref")
sys.path.insert(0, ref)
from gpufairq.metrics import service_gap_report  # noqa: E402
from gpufairq.mqfq import SchedulerConfig  # noqa: E402

random.seed(1)
idx = random.sample(range(len(w.sims)), min(a.sample, len(w.sims)))
inputs = []
for i in idx:
    s = w.sims[i]
    sr = to_sim_result(res, i, w.traces[s.trace])
    inputs.append((i, sr, SchedulerConfig(t_overrun=s.t_overrun, alpha=s.alpha)))
t0 = time.perf_counter()
ref_rows = [(i, service_gap_report(sr.records, sr.audit, cfg, 30.0)) for i, sr, cfg in inputs]
cpu_s = time.perf_counter() - t0
n_win_ref = sum(len(r) for _, r in ref_rows)
# parity on the sample: per window (w0, comparable, max gap, bound, violated)
bad = 0
for i, rows in ref_rows:
    wr, wm = fr.windows(i)
    names = w.traces[w.sims[i].trace].names
    if len(rows) != len(wr):
        bad += 1
        continue
    for r, g, m in zip(rows, wr.tolist(), wm.tolist()):
        if (r.window_start_s != g[0] or r.max_gap != g[2] or r.bound != g[3] or
                bool(r.violated) != bool(m[5])):
            bad += 1
            break
line = {"metric": "service_gap_report windows/s", "sims": len(w.sims), "windows": n_win,
        "gpu_ms": gpu_ms, "gpu_windows_per_s": n_win / gpu_ms * 1e3,
        "cpu_reference": {"sims": len(idx), "windows": n_win_ref, "seconds": cpu_s,
                          "windows_per_s": n_win_ref / cpu_s, "cores": 1,
                          "kind": "unmodified reference (baseline/_ref) metrics.service_gap_report"},
        "speedup_vs_one_core": (n_win / gpu_ms * 1e3) / (n_win_ref / cpu_s),
        "sample_mismatches": bad}
print(json.dumps(line))
if a.out:
    open(a.out, "w").write(json.dumps(line) + "\n")
