"""Generate tests/golden/reference_golden.json by running the UNMODIFIED
reference (gpufairq, imported read-only from /root/reference/pkg/src) on
every case of cases.all_cases().  Run in the build container only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The fixture stores, per case, sha256 fingerprints of the reference's
dispatch trace, records, exec/util/backlog audit, event stream and eviction
log, plus per-run summary values as float.hex.  Nothing here is needed at
test time on the GPU box; the JSON travels with the repo.
"""

from __future__ import annotations

import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, HERE)

from cases import all_cases, extra_cases  # noqa: E402
from fingerprint import fp, hexf, per_function_rows  # noqa: E402


def _ref_imports():
    if REF not in sys.path:
        sys.path.insert(0, REF)
        sys.path.insert(0, REF_TESTS)
    import gpufairq  # noqa: F401
    return gpufairq


def ref_inputs(case):
    _ref_imports()
    from gpufairq.core import FunctionProfile
    from gpufairq.device import DeviceConfig
    from gpufairq.workload import Trace, default_profiles, gen_zipf
    prof = case.get("profiles", {"default": [8]})
    if "default" in prof:
        profiles = default_profiles(*prof["default"])
    elif "c4" in prof:        # cases.c4x_case: sweep.c4's heterogeneous-memory table
        from cases import C4_MEM_MB
        base = default_profiles(*prof["c4"])
        profiles = {nm: FunctionProfile(nm, p.warm_exec_s, p.cold_exec_s, C4_MEM_MB[i % 5],
                                        0.38, 1.0) for i, (nm, p) in enumerate(base.items())}
    else:
        profiles = {r[0]: FunctionProfile(*r) for r in prof["explicit"]}
    tr = case["trace"]
    if "gen" in tr:
        n, s, rate, dur, seed = tr["gen"][:5]
        names = tr.get("names") or list(profiles)[:n]
        trace = gen_zipf(n, s, rate, dur, seed, names=names)
    else:
        ents = [(float(t), nm) for t, nm in tr["entries"]]
        trace = Trace(entries=ents, duration_s=ents[-1][0] if ents else 0.0)
    devices = [DeviceConfig(**d) for d in case.get("devices", [{}])]
    return trace, profiles, devices


def run_reference(case):
    _ref_imports()
    from gpufairq.device import DeviceSet
    from gpufairq.engine import ARRIVAL, COMPLETION, MONITOR_TICK, Simulation
    from gpufairq.metrics import (cold_hit_rate, mean_util, per_function_summary,
                                  weighted_avg_latency)
    from gpufairq.mqfq import SchedulerConfig
    from gpufairq.policies import make_policy

    if case.get("scripted"):
        from oracles import RealSchedulerAdapter, ScriptedDevices, drive
        from gpufairq.core import FunctionProfile
        sc = case["scripted"]
        names = sc["names"]
        profiles = {nm: FunctionProfile(nm, 1.0, 2.0, 100.0, 0.4, 1.0) for nm in names}
        cfg = SchedulerConfig(**case.get("sched", {}))
        arrivals = [tuple(a) for a in sc["arrivals"]]
        tr = drive(RealSchedulerAdapter(profiles, cfg), ScriptedDevices(sc["d"], sc["deny"]),
                   arrivals, sc["execs"], with_unstall=True)
        return {"name": case["name"], "fp": {"transcript": fp(tr)}, "n": len(tr)}

    trace, profiles, devices = ref_inputs(case)
    sched = SchedulerConfig(**case.get("sched", {}))
    policy = make_policy(case.get("policy", "mqfq"), profiles, sched)
    dset = DeviceSet(devices)
    sim = Simulation(trace, profiles, policy, dset,
                     tau_includes_overheads=bool(case.get("tau_inc", False)))
    pos = {}
    for t, seq, kind, payload in sim._heap:
        if kind == ARRIVAL:
            pos[payload.uid] = seq
    events = []
    while True:
        ev = sim.step()
        if ev is None:
            break
        t, kind, payload = ev
        if kind == ARRIVAL:
            pay = pos[payload.uid]
        elif kind == COMPLETION:
            pay = pos[payload]
        elif kind == MONITOR_TICK:
            pay = None
        else:
            pay = payload
        events.append((t, kind, pay))
    result = sim.run()
    recs = result.records
    disp = [(a.now, a.function, a.vt_before, a.global_vt, a.queue_len, a.in_flight,
             a.device, a.start_state) for a in policy.dispatch_log]
    rec_rows = [(r.function, r.arrival_s, r.dispatch_s, r.complete_s, r.start_state, r.device)
                for r in recs]
    util = [(float(t), d, float(u), float(a), e) for t, d, u, a, e in result.audit.util]
    backlog = [(float(t), fn, bool(on)) for t, fn, on in result.audit.backlog]
    exe = [(fn, float(d), float(c), float(p)) for fn, d, c, p in result.audit.exec]
    evict = []
    for dev in dset:
        for t, fn in dev.eviction_log:
            evict.append((float(t), dev.index, fn))
    pf = per_function_summary(recs)
    summary = {
        "weighted_avg_latency_s": weighted_avg_latency(recs) if recs else 0.0,
        "cold_hit_pct": 100.0 * cold_hit_rate(recs),
        "mean_util": float(mean_util(result.audit)),
    }
    return {
        "name": case["name"],
        "fp": {
            "trace": fp([(t, nm) for t, nm in trace.entries]),
            "dispatch": fp(disp), "records": fp(rec_rows), "util": fp(util),
            "backlog": fp(backlog), "exec": fp(exe), "events": fp(events),
            "evictions": fp(evict),   # per device, each in log order
            "per_function": fp(per_function_rows(pf)),
        },
        "summary": {k: hexf(v) for k, v in summary.items()},
        "per_function": {fn: [hexf(v["mean_latency_s"]), hexf(v["var_latency_s"]),
                              v["count"], hexf(v["cold_hit_pct"])] for fn, v in pf.items()},
        "counts": {"arrivals": len(trace.entries), "dispatches": len(disp),
                   "events": len(events), "util_rows": len(util),
                   "dispatch_calls": None},
        "final_time": hexf(events[-1][0]) if events else hexf(0.0),
    }


def main():
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    # the GPU reducers replay CPython >= 3.12's compensated sum(); on 3.10 /
    # 3.11 sum() is plain left-to-right addition and the stats would differ
    assert sys.version_info >= (3, 12), "goldens need CPython >= 3.12 (Neumaier sum())"
    extra = "--extra" in sys.argv
    cases = extra_cases() if extra else all_cases()
    t0 = time.time()
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        # longest first (the 4096-flow c4x cases dominate)
        order = sorted(range(len(cases)), key=lambda i: -len(str(cases[i])))
        res = list(ex.map(run_reference, [cases[i] for i in order], chunksize=1 if extra else 4))
        results = [None] * len(cases)
        for i, r in zip(order, res):
            results[i] = r
    out = {"generator": "tests/golden/make_golden.py",
           "reference": "gpufairq 0.1.0 (/root/reference/pkg/src, unmodified)",
           "python": sys.version.split()[0],
           "cases": results}
    path = os.path.join(HERE, "reference_golden_extra.json" if extra else "reference_golden.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(f"{len(results)} cases in {time.time() - t0:.0f}s -> {path}")


if __name__ == "__main__":
    main()
