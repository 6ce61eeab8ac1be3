"""Reference fingerprints of metrics.service_gap_report (metrics.py:106-187)
for every non-scripted golden case, from the UNMODIFIED reference imported
read-only from /root/reference/pkg/src.  Build container only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_fairness_golden.py

Row per 30 s window: (w0, comparable, n_qualified, qual_hash, hi, lo,
service_sum, max_gap, bound, bound_conservative, violated), where qual_hash
is an order-free hash of the qualified functions' sorted-name ranks,
service_sum the naive sum of their service in name order, and hi / lo the
pair the reference's bound uses (max / min of (normalised service, name)).
"""

from __future__ import annotations

import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from cases import all_cases  # noqa: E402
from fingerprint import fp  # noqa: E402
from make_golden import _ref_imports, ref_inputs  # noqa: E402


def qual_hash(ranks):
    return sum((r * 2654435761 + 1) & 0xFFFFFFFF for r in ranks) & 0xFFFFFFFF


def window_rows(reports, names, cfg):
    rank = {nm: i for i, nm in enumerate(names)}
    rows = []
    for w in reports:
        q = list(w.qualified)
        s = 0.0
        for fn in q:
            s += w.service[fn]
        hi = lo = ""
        if q:
            norm = {fn: w.service[fn] / cfg.weights.get(fn, 1.0) for fn in q}
            hi = max(q, key=lambda fn: (norm[fn], fn))
            lo = min(q, key=lambda fn: (norm[fn], fn))
        rows.append((float(w.window_start_s), bool(w.comparable), len(q),
                     qual_hash(rank[fn] for fn in q), hi, lo, s, float(w.max_gap),
                     float(w.bound), float(w.bound_conservative), bool(w.violated)))
    return rows


def run(case):
    _ref_imports()
    from gpufairq.device import DeviceSet
    from gpufairq.engine import run_simulation
    from gpufairq.metrics import service_gap_report
    from gpufairq.mqfq import SchedulerConfig
    from gpufairq.policies import make_policy
    trace, profiles, devices = ref_inputs(case)
    cfg = SchedulerConfig(**case.get("sched", {}))
    pol = make_policy(case.get("policy", "mqfq"), profiles, cfg)
    res = run_simulation(trace, profiles, pol, DeviceSet(devices),
                         tau_includes_overheads=bool(case.get("tau_inc", False)))
    names = sorted({nm for _, nm in trace.entries})
    rows = window_rows(service_gap_report(res.records, res.audit, cfg), names, cfg)
    return {"name": case["name"], "fp": fp(rows), "windows": len(rows),
            "comparable": sum(r[1] for r in rows), "violated": sum(r[10] for r in rows)}


def main():
    cases = [c for c in all_cases() if not c.get("scripted")]
    t0 = time.time()
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        out = list(ex.map(run, cases, chunksize=2))
    path = os.path.join(HERE, "fairness_golden.json")
    with open(path, "w") as fh:
        json.dump({"generator": "tests/golden/make_fairness_golden.py",
                   "reference": "gpufairq 0.1.0 metrics.service_gap_report (window_s=30)",
                   "cases": out}, fh, separators=(",", ":"))
    print(f"{len(out)} cases in {time.time() - t0:.0f}s -> {path}")


if __name__ == "__main__":
    main()
