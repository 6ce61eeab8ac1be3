"""TEST INFRASTRUCTURE ONLY — ctypes binding of the C oracle (gfq_oracle.c).

The oracle is the parity checker for the GPU engine and the CPU baseline
timed by bench.py.  Only tests/, __graft_entry__.smoke() and bench.py may
import this module; the product package never does.

``run_case(case)`` takes the JSON case description used by the golden
fixtures (tests/golden/cases.py) and returns the reference-shaped outputs
(dispatch rows, records, audit rows, event stream, summary) in the same
normalised form tests/golden/make_golden.py extracts from the reference.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

from paper_2507_08954_b200 import _abi
from paper_2507_08954_b200.core import FunctionProfile
from paper_2507_08954_b200.device import DeviceConfig
from paper_2507_08954_b200.workload import default_profiles, gen_zipf

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgfq_oracle.so")
STATE_NAMES = ("gpu_warm", "host_warm", "cold")
POLICY_CODES = {"mqfq": 0, "fcfs": 1, "batch": 2, "sjf": 3, "fcfs_naive": 4}

_lib = None
_lock = threading.Lock()


class OracleOut(C.Structure):
    P = C.POINTER
    _fields_ = [
        ("cap_records", C.c_int64), ("n_records", C.c_int64),
        ("rec_inv", P(C.c_int64)), ("rec_dispatch", P(C.c_double)),
        ("rec_complete", P(C.c_double)), ("rec_pure", P(C.c_double)),
        ("rec_state", P(C.c_int8)), ("rec_device", P(C.c_int8)),
        ("cap_dispatch", C.c_int64), ("n_dispatch", C.c_int64),
        ("d_inv", P(C.c_int64)), ("d_flow", P(C.c_int32)), ("d_now", P(C.c_double)),
        ("d_vt_before", P(C.c_double)), ("d_gvt", P(C.c_double)),
        ("d_qlen", P(C.c_int64)), ("d_inflight", P(C.c_int64)),
        ("d_device", P(C.c_int8)), ("d_state", P(C.c_int8)),
        ("cap_util", C.c_int64), ("n_util", C.c_int64),
        ("u_time", P(C.c_double)), ("u_inst", P(C.c_double)), ("u_avg", P(C.c_double)),
        ("u_dev", P(C.c_int32)), ("u_effd", P(C.c_int32)),
        ("cap_backlog", C.c_int64), ("n_backlog", C.c_int64),
        ("b_time", P(C.c_double)), ("b_flow", P(C.c_int32)), ("b_on", P(C.c_int8)),
        ("cap_events", C.c_int64), ("n_events_logged", C.c_int64),
        ("ev_time", P(C.c_double)), ("ev_kind", P(C.c_int8)), ("ev_payload", P(C.c_int64)),
        ("cap_evictions", C.c_int64), ("n_evictions", C.c_int64),
        ("x_time", P(C.c_double)), ("x_dev", P(C.c_int32)), ("x_flow", P(C.c_int32)),
        ("f_count", P(C.c_int64)), ("f_mean", P(C.c_double)), ("f_var", P(C.c_double)),
        ("f_cold_pct", P(C.c_double)),
        ("weighted_avg_latency", C.c_double), ("cold_hit_pct", C.c_double),
        ("mean_util", C.c_double), ("final_time", C.c_double),
        ("n_events", C.c_int64), ("n_dispatch_calls", C.c_int64),
        ("status", C.c_int32), ("early_exit", C.c_int32),
    ]


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc)."""
    if force or not os.path.exists(LIB_PATH) or \
            os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "gfq_oracle.c")):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                build()
            L = C.CDLL(LIB_PATH)
            L.gfq_oracle_run.restype = C.c_int
            L.gfq_oracle_run.argtypes = [
                C.POINTER(_abi.Sim), C.POINTER(C.c_double), C.POINTER(C.c_int32),
                C.c_int64, C.c_int32] + [C.POINTER(C.c_double)] * 5 + [
                C.POINTER(_abi.DeviceCfg), C.POINTER(C.c_double), C.POINTER(OracleOut)]
            _lib = L
    return _lib


def _ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


# ---------------------------------------------------------------------------
# case description -> reference-like inputs

def case_inputs(case: dict):
    """Build (entries, profiles dict, device configs) for a case."""
    prof = case.get("profiles", {"default": [8]})
    if "default" in prof:
        args = prof["default"]
        profiles = default_profiles(*args)
    elif "c4" in prof:        # tests/golden/cases.c4x_case: sweep.c4's memory table
        mems = [256.0, 512.0, 1024.0, 1500.0, 3000.0]
        base = default_profiles(*prof["c4"])
        profiles = {nm: FunctionProfile(nm, p.warm_exec_s, p.cold_exec_s, mems[i % 5], 0.38, 1.0)
                    for i, (nm, p) in enumerate(base.items())}
    else:
        profiles = {row[0]: FunctionProfile(*row) for row in prof["explicit"]}
    tr = case["trace"]
    if "gen" in tr:
        n, s, rate, dur, seed = tr["gen"][:5]
        names = tr.get("names") or list(profiles)[:n]
        entries = gen_zipf(n, s, rate, dur, seed, names=names).entries
    else:
        entries = [(float(t), nm) for t, nm in tr["entries"]]
    devices = [DeviceConfig(**d) for d in case.get("devices", [{}])]
    return entries, profiles, devices


def pack(entries, profiles, weights=None):
    names = sorted({nm for _, nm in entries})
    rank = {nm: i for i, nm in enumerate(names)}
    arrival = np.array([t for t, _ in entries], dtype=np.float64)
    flow = np.array([rank[nm] for _, nm in entries], dtype=np.int32)
    weights = weights or {}
    tab = {
        "warm": np.array([profiles[nm].warm_exec_s for nm in names], dtype=np.float64),
        "cold": np.array([profiles[nm].cold_exec_s for nm in names], dtype=np.float64),
        "mem": np.array([profiles[nm].mem_mb for nm in names], dtype=np.float64),
        "share": np.array([profiles[nm].compute_share for nm in names], dtype=np.float64),
        "weight": np.array([weights.get(nm, profiles[nm].weight) for nm in names],
                           dtype=np.float64),
    }
    return names, arrival, flow, tab


def run_packed(sim: _abi.Sim, arrival, flow, n_flows, tab, devcfgs, execs=None,
               want_events=False, want_audit=True, want_dispatch=True,
               want_records=True, want_stats=True, caps=None, early_exit=False):
    """Run one simulation through the oracle on packed inputs; returns the
    raw numpy outputs (trace positions, flow ids, state codes).  Audit and
    event buffers grow and the run repeats when a first guess was short."""
    caps = caps or {"u": 16 * 1024, "x": 4 * 1024, "ev": 64 * 1024}
    while True:
        r = _run_packed_once(sim, arrival, flow, n_flows, tab, devcfgs, execs, want_events,
                             want_audit, want_dispatch, want_records, want_stats, caps,
                             early_exit)
        need = r.pop("_need")
        short = {k: v for k, v in need.items() if v > caps[k]}
        if not short:
            return r
        caps = dict(caps, **{k: v + 16 for k, v in short.items()})


def _run_packed_once(sim, arrival, flow, n_flows, tab, devcfgs, execs, want_events,
                     want_audit, want_dispatch, want_records, want_stats, caps, early_exit=False):
    n = int(arrival.shape[0])
    o = OracleOut()
    o.early_exit = int(bool(early_exit))
    keep = []

    def arr(dtype, size):
        a = np.zeros(max(int(size), 1), dtype=dtype)
        keep.append(a)
        return a

    ct = {np.float64: C.c_double, np.int64: C.c_int64, np.int32: C.c_int32, np.int8: C.c_int8}
    bufs = {}

    def bind(names_types, cap_field, cap):
        setattr(o, cap_field, cap)
        for nm, dt in names_types:
            a = arr(dt, cap)
            bufs[nm] = a
            setattr(o, nm, _ptr(a, ct[dt]))

    if want_records or want_stats:
        bind([("rec_inv", np.int64), ("rec_dispatch", np.float64), ("rec_complete", np.float64),
              ("rec_pure", np.float64), ("rec_state", np.int8), ("rec_device", np.int8)],
             "cap_records", n)
    if want_dispatch:
        bind([("d_inv", np.int64), ("d_flow", np.int32), ("d_now", np.float64),
              ("d_vt_before", np.float64), ("d_gvt", np.float64), ("d_qlen", np.int64),
              ("d_inflight", np.int64), ("d_device", np.int8), ("d_state", np.int8)],
             "cap_dispatch", n)
    if want_audit:
        bind([("u_time", np.float64), ("u_inst", np.float64), ("u_avg", np.float64),
              ("u_dev", np.int32), ("u_effd", np.int32)], "cap_util", caps["u"])
        bind([("b_time", np.float64), ("b_flow", np.int32), ("b_on", np.int8)],
             "cap_backlog", 2 * n + 2)
        bind([("x_time", np.float64), ("x_dev", np.int32), ("x_flow", np.int32)],
             "cap_evictions", caps["x"])
    if want_events:
        bind([("ev_time", np.float64), ("ev_kind", np.int8), ("ev_payload", np.int64)],
             "cap_events", caps["ev"])
    if want_stats:
        for nm, dt in (("f_count", np.int64), ("f_mean", np.float64), ("f_var", np.float64),
                       ("f_cold_pct", np.float64)):
            a = arr(dt, n_flows)
            bufs[nm] = a
            setattr(o, nm, _ptr(a, ct[dt]))
    dc = (_abi.DeviceCfg * max(len(devcfgs), 1))(*devcfgs)
    ex = np.ascontiguousarray(execs if execs is not None else np.zeros(1), dtype=np.float64)
    arrival = np.ascontiguousarray(arrival, dtype=np.float64)
    flow = np.ascontiguousarray(flow, dtype=np.int32)
    rc = lib().gfq_oracle_run(
        C.byref(sim), _ptr(arrival, C.c_double), _ptr(flow, C.c_int32), n, int(n_flows),
        _ptr(tab["warm"], C.c_double), _ptr(tab["cold"], C.c_double),
        _ptr(tab["mem"], C.c_double), _ptr(tab["share"], C.c_double),
        _ptr(tab["weight"], C.c_double), dc, _ptr(ex, C.c_double), C.byref(o))
    res = {"rc": rc, "status": o.status, "n_events": o.n_events,
           "n_dispatch_calls": o.n_dispatch_calls, "final_time": o.final_time,
           "weighted_avg_latency": o.weighted_avg_latency, "cold_hit_pct": o.cold_hit_pct,
           "mean_util": o.mean_util}
    counts = {"rec": o.n_records, "d": o.n_dispatch, "u": o.n_util, "b": o.n_backlog,
              "ev": o.n_events_logged, "x": o.n_evictions}
    res["_need"] = {"u": o.n_util if want_audit else 0, "x": o.n_evictions if want_audit else 0,
                    "ev": o.n_events_logged if want_events else 0}
    for nm, a in bufs.items():
        pre = nm.split("_")[0]
        key = {"rec": "rec", "d": "d", "u": "u", "b": "b", "ev": "ev", "x": "x"}.get(pre)
        res[nm] = a[:counts[key]] if key else a[:n_flows]
    return res


def make_sim(case: dict, n_devices: int) -> _abi.Sim:
    sched = case.get("sched", {})
    sim = _abi.Sim()
    sim.policy = POLICY_CODES[case.get("policy", "mqfq")]
    sim.device_model = _abi.DEVMODEL_SCRIPTED if case.get("scripted") else _abi.DEVMODEL_DEVICESET
    sim.n_devices = n_devices
    sim.tau_includes_overheads = int(bool(case.get("tau_inc", False)))
    sim.group = -1
    sim.t_overrun = float(sched.get("t_overrun", 10.0))
    sim.alpha = float(sched.get("alpha", 2.0))
    sim.default_ttl_s = float(sched.get("default_ttl_s", 2.0))
    return sim


def run_case(case: dict, want_events: bool = False) -> dict:
    """Run a golden case through the oracle; returns reference-shaped rows."""
    if case.get("scripted"):
        return run_scripted_case(case)
    entries, profiles, devices = case_inputs(case)
    sched = case.get("sched", {})
    names, arrival, flow, tab = pack(entries, profiles, sched.get("weights"))
    sim = make_sim(case, len(devices))
    devcfgs = [_abi.device_cfg_from(d) for d in devices]
    r = run_packed(sim, arrival, flow, len(names), tab, devcfgs, want_events=want_events)
    if r["status"] != 0:
        raise RuntimeError(f"oracle status {r['status']}: {_abi.SIM_STATUS.get(r['status'])}")
    return normalise(r, names, arrival, flow)


def normalise(r: dict, names, arrival, flow) -> dict:
    out = {}
    out["dispatch"] = [
        (float(r["d_now"][k]), names[int(r["d_flow"][k])], float(r["d_vt_before"][k]),
         float(r["d_gvt"][k]), int(r["d_qlen"][k]), int(r["d_inflight"][k]),
         int(r["d_device"][k]), STATE_NAMES[int(r["d_state"][k])])
        for k in range(len(r["d_now"]))]
    out["records"] = [
        (names[int(flow[i])], float(arrival[i]), float(r["rec_dispatch"][k]),
         float(r["rec_complete"][k]), STATE_NAMES[int(r["rec_state"][k])],
         int(r["rec_device"][k]))
        for k, i in enumerate(r["rec_inv"].tolist())]
    out["exec"] = [
        (names[int(flow[i])], float(r["rec_dispatch"][k]), float(r["rec_complete"][k]),
         float(r["rec_pure"][k]))
        for k, i in enumerate(r["rec_inv"].tolist())]
    if "u_time" in r:
        out["util"] = [(float(r["u_time"][k]), int(r["u_dev"][k]), float(r["u_inst"][k]),
                        float(r["u_avg"][k]), int(r["u_effd"][k]))
                       for k in range(len(r["u_time"]))]
        out["backlog"] = [(float(r["b_time"][k]), names[int(r["b_flow"][k])], bool(r["b_on"][k]))
                          for k in range(len(r["b_time"]))]
        ev = [(float(r["x_time"][k]), int(r["x_dev"][k]), names[int(r["x_flow"][k])])
              for k in range(len(r["x_time"]))]
        # Device.eviction_log is per device: group stably by device index
        out["evictions"] = sorted(ev, key=lambda row: row[1])
    if "ev_time" in r:
        evs = []
        for k in range(len(r["ev_time"])):
            kind = int(r["ev_kind"][k])
            p = int(r["ev_payload"][k])
            pay = names[p] if kind == _abi.EV_QUEUE_EXPIRY else (None if kind == 2 else p)
            evs.append((float(r["ev_time"][k]), kind, pay))
        out["events"] = evs
    out["summary"] = {
        "weighted_avg_latency_s": r["weighted_avg_latency"],
        "cold_hit_pct": r["cold_hit_pct"],
        "mean_util": r["mean_util"],
    }
    pf = {}
    for f, nm in enumerate(names):
        c = int(r["f_count"][f])
        if c:
            pf[nm] = {"mean_latency_s": float(r["f_mean"][f]),
                      "var_latency_s": float(r["f_var"][f]), "count": c,
                      "cold_hit_pct": float(r["f_cold_pct"][f])}
    out["per_function"] = pf
    out["n_events"] = r["n_events"]
    out["n_dispatch_calls"] = r["n_dispatch_calls"]
    return out


def run_scripted_case(case: dict) -> dict:
    """drive(RealSchedulerAdapter, ScriptedDevices(d, deny), arrivals, execs,
    with_unstall=True) (tests/oracles.py:199-238) -> transcript of
    (round(now, 9), function) pairs."""
    sc = case["scripted"]
    entries = [(float(t), nm) for t, nm in sc["arrivals"]]
    names = sorted({nm for _, nm in entries}) or ["_"]
    rank = {nm: i for i, nm in enumerate(names)}
    arrival = np.array([t for t, _ in entries], dtype=np.float64)
    flow = np.array([rank[nm] for _, nm in entries], dtype=np.int32)
    ones = np.ones(len(names), dtype=np.float64)
    weights = case.get("sched", {}).get("weights", {})
    tab = {"warm": ones, "cold": ones * 2, "mem": ones * 100.0, "share": ones * 0.4,
           "weight": np.array([weights.get(nm, 1.0) for nm in names], dtype=np.float64)}
    sim = make_sim(case, 0)
    sim.scripted_d = int(sc["d"])
    sim.scripted_deny_every = int(sc.get("deny", 0))
    execs = np.array(sc["execs"], dtype=np.float64)
    sim.exec_off = 0
    sim.exec_len = len(execs)
    r = run_packed(sim, arrival, flow, len(names), tab, [], execs=execs,
                   want_audit=False, want_stats=False, want_records=False)
    if r["status"] != 0:
        raise RuntimeError(f"oracle status {r['status']}")
    return {"transcript": [(round(float(r["d_now"][k]), 9), names[int(r["d_flow"][k])])
                           for k in range(len(r["d_now"]))]}
