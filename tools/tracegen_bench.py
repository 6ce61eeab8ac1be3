"""Measurement of the GPU trace generator (`gfq_generate_traces`):
C5's 1563 Azure-shaped traces (100 functions, Zipf 1.5, 600 s, four loads) and
4096 C3 traces, generated on the GPU and made resident, against the
UNMODIFIED reference's `gen_zipf` (baseline/_ref, workload.py:82-111) on one
host core over a sample of the same specs; the sampled traces must be
identical.

    python tools/tracegen_bench.py [--sample N] [--out file.json]
"""
import argparse
import json
import os
import random
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_08954_b200 import sweep  # noqa: E402
from paper_2507_08954_b200.engine import Engine  # noqa: E402
from paper_2507_08954_b200.workload import default_profiles  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sample", type=int, default=24)
ap.add_argument("--out", default="")
a = ap.parse_args()

eng = Engine(0)
names100 = list(default_profiles(100))
shares = [(k + 1) ** -1.5 for k in range(100)]
tot = sum(shares)
mean_exec = sum(sh / tot * p.warm_exec_s for sh, p in zip(shares, default_profiles(100).values()))
workloads = {
    "c5_1563": [(100, 1.5, sweep.C5_RHO[j % 4] * 1.8 / mean_exec, 600.0, 1 + j, names100)
                for j in range(1563)],
    "c3_4096": [(100, 1.5, sweep.C3_RATE, 600.0, 1 + j, names100) for j in range(4096)],
}
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
from gpufairq.workload import gen_zipf  # noqa: E402

out = {"metric": "traces/s and arrivals/s generated (gen_zipf)"}
random.seed(3)
for name, specs in workloads.items():
    eng.generate_traces(specs[:8])                       # warm-up
    best = None
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pts = eng.generate_traces(specs)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    n_arr = sum(p.n for p in pts)
    idx = random.sample(range(len(specs)), min(a.sample, len(specs)))
    t0 = time.perf_counter()
    ref = [gen_zipf(*specs[i][:5], names=specs[i][5]) for i in idx]
    cpu = time.perf_counter() - t0
    n_ref = sum(len(r.entries) for r in ref)
    same = all([(float(t), pts[i].names[f]) for t, f in zip(pts[i].arrival.tolist(),
                                                             pts[i].flow.tolist())]
               == [(t, nm) for t, nm in r.entries] for i, r in zip(idx, ref))
    out[name] = {"traces": len(specs), "arrivals": n_arr, "gpu_s": best,
                 "gpu_traces_per_s": len(specs) / best, "gpu_arrivals_per_s": n_arr / best,
                 "cpu_reference": {"traces": len(idx), "arrivals": n_ref, "seconds": cpu,
                                   "arrivals_per_s": n_ref / cpu, "cores": 1,
                                   "kind": "unmodified reference gen_zipf (baseline/_ref)"},
                 "speedup_vs_one_core": (n_arr / best) / (n_ref / cpu),
                 "sample_identical": bool(same)}
print(json.dumps(out))
if a.out:
    open(a.out, "w").write(json.dumps(out) + "\n")
