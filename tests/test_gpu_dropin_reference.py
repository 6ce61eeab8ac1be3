"""The drop-in, driven with the REFERENCE's own objects.

The reference (unmodified, baseline/_ref or /root/reference) builds its own
Trace (gen_zipf), FunctionProfile dict, make_policy(...) policy and
DeviceSet; the same objects (fresh copies) go to the reference's
run_simulation / Simulation and to this repo's, whose results must agree
exactly: InvocationRecords in completion order, audit.dispatches (==
policy.dispatch_log, the same list), audit.backlog / util / exec, each
device's eviction_log, and the Simulation.step() event stream
(engine.py:99-119,214-218; device.py:92,172,177,275).
"""

from __future__ import annotations

import sys

import pytest

from refsuite import locate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    loc = locate()
    if loc is None:
        pytest.skip("reference not installed (tools/install_ref.sh)")
    if loc[0] not in sys.path:
        sys.path.insert(0, loc[0])
    import gpufairq
    return gpufairq


CASES = {
    # configs/default.cfg (BASELINE C1), its 10-function variant, medium.cfg
    "default": dict(n=24, s=1.5, rate=2.69, dur=600.0, seed=1, policy="mqfq",
                    sched=dict(t_overrun=10.0, alpha=2.0), devs=[dict(d_max=2)]),
    "c1_f10": dict(n=10, s=1.5, rate=3.197988, dur=600.0, seed=1, policy="mqfq",
                   sched=dict(t_overrun=10.0, alpha=2.0), devs=[dict(d_max=2)]),
    "two_devices": dict(n=12, s=1.2, rate=3.5, dur=200.0, seed=4, policy="mqfq",
                        sched=dict(t_overrun=5.0, alpha=1.0),
                        devs=[dict(d_max=3), dict(d_max=2, mem_capacity_mb=6000.0)]),
    # memory pressure: LRU admission victims and keep-alive swap-outs
    "evicting": dict(n=16, s=0.8, rate=3.0, dur=300.0, seed=9, policy="mqfq", mem=3000.0,
                     sched=dict(t_overrun=2.0, alpha=0.5),
                     devs=[dict(d_max=3, mem_capacity_mb=7000.0, pool_max_containers=6)]),
    "fcfs": dict(n=12, s=1.5, rate=3.0, dur=300.0, seed=2, policy="fcfs", mem=2500.0,
                 sched={}, devs=[dict(d_max=2, mem_capacity_mb=8000.0)]),
    "batch": dict(n=12, s=1.5, rate=3.0, dur=300.0, seed=3, policy="batch", sched={},
                  devs=[dict(d_max=2)]),
    "sjf": dict(n=12, s=1.5, rate=3.0, dur=300.0, seed=5, policy="sjf", sched={},
                devs=[dict(d_max=2, dynamic_d=True, util_threshold=0.7)]),
    "fcfs_naive": dict(n=8, s=1.5, rate=1.0, dur=200.0, seed=6, policy="fcfs_naive", sched={},
                       devs=[dict(d_max=2, pool_enabled=False)]),
}


def _inputs(ref, c):
    from gpufairq.core import FunctionProfile
    from gpufairq.device import DeviceConfig, DeviceSet
    from gpufairq.mqfq import SchedulerConfig
    from gpufairq.policies import make_policy
    from gpufairq.workload import default_profiles, gen_zipf
    profiles = default_profiles(c["n"])
    if "mem" in c:
        profiles = {k: FunctionProfile(k, p.warm_exec_s, p.cold_exec_s, c["mem"],
                                       p.compute_share, p.weight) for k, p in profiles.items()}
    trace = gen_zipf(c["n"], c["s"], c["rate"], c["dur"], c["seed"], names=list(profiles))
    policy = make_policy(c["policy"], profiles, SchedulerConfig(**c["sched"]))
    devices = DeviceSet([DeviceConfig(**d) for d in c["devs"]])
    return trace, profiles, policy, devices


def _rows(res, policy, devices):
    recs = [(r.function, r.arrival_s, r.dispatch_s, r.complete_s, r.start_state, r.device)
            for r in res.records]
    disp = [(a.now, a.function, a.vt_before, a.global_vt, a.queue_len, a.in_flight, a.device,
             a.start_state) for a in res.audit.dispatches]
    return {"records": recs, "dispatches": disp,
            "backlog": [tuple(x) for x in res.audit.backlog],
            "util": [tuple(x) for x in res.audit.util],
            "exec": [tuple(x) for x in res.audit.exec],
            "evictions": [list(d.eviction_log) for d in devices],
            "shared_log": res.audit.dispatches is policy.dispatch_log}


@pytest.mark.parametrize("name", list(CASES))
def test_run_simulation_with_reference_objects(ref, name):
    from gpufairq.engine import run_simulation as ref_run
    from paper_2507_08954_b200.engine import run_simulation as gpu_run
    c = CASES[name]
    t, p, pol, dev = _inputs(ref, c)
    want = _rows(ref_run(t, p, pol, dev), pol, dev)
    t, p, pol, dev = _inputs(ref, c)
    got = _rows(gpu_run(t, p, pol, dev), pol, dev)
    for k in want:
        assert got[k] == want[k], (name, k)
    assert want["records"]
    if name == "evicting":
        assert sum(len(e) for e in want["evictions"]) > 0


@pytest.mark.parametrize("name", ["default", "two_devices", "evicting"])
def test_simulation_step_with_reference_objects(ref, name):
    """Simulation(...).step() yields the reference's (time, kind, payload)
    sequence; run() then returns the same records and audit."""
    from gpufairq.engine import Simulation as RefSim
    from paper_2507_08954_b200.engine import Simulation as GpuSim

    def stream(sim):
        out = []
        while (ev := sim.step()) is not None:
            t, kind, pay = ev
            if kind == 0:
                pay = (pay.function, pay.arrival_s)
            elif kind == 1:
                pay = None                           # uids come from different counters
            out.append((t, kind, pay, sim.now, len(sim.records)))
        return out

    c = CASES[name]
    t, p, pol, dev = _inputs(ref, c)
    rs = RefSim(t, p, pol, dev)
    want_ev = stream(rs)
    want = _rows(rs.run(), pol, dev)
    t, p, pol, dev = _inputs(ref, c)
    gs = GpuSim(t, p, pol, dev)
    got_ev = stream(gs)
    got = _rows(gs.run(), pol, dev)
    assert got_ev == want_ev
    for k in want:
        assert got[k] == want[k], (name, k)


def test_reference_validation_errors(ref):
    """Unknown functions and decreasing arrival times raise ValueError, as in
    the reference (engine.py:51-53,66-68)."""
    from gpufairq.device import DeviceConfig, DeviceSet
    from gpufairq.mqfq import SchedulerConfig
    from gpufairq.policies import make_policy
    from gpufairq.workload import Trace, default_profiles
    from paper_2507_08954_b200.engine import Simulation, run_simulation
    prof = default_profiles(4)
    pol = make_policy("mqfq", prof, SchedulerConfig())
    with pytest.raises(ValueError, match="unknown"):
        Simulation(Trace(entries=[(0.0, "nope")], duration_s=0.0), prof, pol,
                   DeviceSet([DeviceConfig()]))
    with pytest.raises(ValueError, match="non-decreasing"):
        run_simulation(Trace(entries=[(1.0, "fft"), (0.5, "fft")], duration_s=1.0), prof, pol,
                       DeviceSet([DeviceConfig()]))


@pytest.mark.parametrize("name", ["default", "two_devices", "evicting", "fcfs", "sjf"])
def test_simulation_state_between_steps(ref, name):
    """After EVERY step() the replayed observable state equals the reference's:
    now, records, policy.dispatch_log, audit.backlog / util / exec, each
    device's eviction_log, and the arrival Invocations' start_tag (at their
    arrival step) and dispatch_s / complete_s / start_state (as they happen)."""
    from gpufairq.engine import Simulation as RefSim
    from paper_2507_08954_b200.engine import Simulation as GpuSim

    def last(xs):
        return tuple(xs[-1]) if xs else None

    def snap(sim, pol, dev):
        log = pol.dispatch_log
        d = log[-1] if log else None
        r = sim.records[-1] if sim.records else None
        return (sim.now, len(sim.records),
                None if r is None else (r.function, r.arrival_s, r.dispatch_s, r.complete_s,
                                        r.start_state, r.device),
                len(log), None if d is None else (d.now, d.function, d.vt_before, d.global_vt,
                                                  d.queue_len, d.in_flight, d.device,
                                                  d.start_state),
                len(sim.audit.backlog), last(sim.audit.backlog),
                len(sim.audit.util), last(sim.audit.util),
                len(sim.audit.exec), last(sim.audit.exec),
                tuple(len(x.eviction_log) for x in dev), tuple(last(x.eviction_log) for x in dev))

    def inv_state(invs):
        return [(i.function, i.arrival_s, i.start_tag, i.dispatch_s, i.complete_s,
                 None if i.start_state is None else i.start_state.value) for i in invs]

    c = CASES[name]
    tr, p, rpol, rdev = _inputs(ref, c)
    rs = RefSim(tr, p, rpol, rdev)
    tr, p, gpol, gdev = _inputs(ref, c)
    gs = GpuSim(tr, p, gpol, gdev)
    rinv, ginv = [], []
    k = 0
    while True:
        a, b = rs.step(), gs.step()
        assert (a is None) == (b is None), k
        if a is None:
            break
        assert (a[0], a[1]) == (b[0], b[1]), k
        if a[1] == 0:
            rinv.append(a[2])
            ginv.append(b[2])
            assert a[2].start_tag == b[2].start_tag, (k, a[2], b[2])
        assert snap(rs, rpol, rdev) == snap(gs, gpol, gdev), k
        if k % 97 == 0:
            assert inv_state(rinv) == inv_state(ginv), k
        k += 1
    assert inv_state(rinv) == inv_state(ginv)
    want, got = rs.run(), gs.run()
    assert want.audit.dispatches is rpol.dispatch_log and got.audit.dispatches is gpol.dispatch_log
    assert k > 1000
