"""The Simulation drop-in (engine.py:46-119 shape): the reference's own
test_engine.py scenarios, run through the GPU engine, plus the processed-event
stream against the reference fingerprints of the engine golden cases."""

from __future__ import annotations

import pytest

from cases import engine_cases
from fingerprint import fp
from golden_check import golden

from paper_2507_08954_b200.core import FunctionProfile
from paper_2507_08954_b200.device import DeviceConfig, DeviceSet
from paper_2507_08954_b200.engine import ARRIVAL, MONITOR_TICK, Simulation
from paper_2507_08954_b200.mqfq import SchedulerConfig
from paper_2507_08954_b200.policies import make_policy
from paper_2507_08954_b200.workload import Trace, default_profiles, gen_zipf

pytestmark = pytest.mark.gpu


def sim_for(entries, profiles=None, policy="mqfq", devices=None, **sched_kwargs):
    profiles = profiles or default_profiles(4)
    trace = Trace(entries=list(entries), duration_s=entries[-1][0] if entries else 0.0)
    devices = devices or DeviceSet([DeviceConfig()])
    pol = make_policy(policy, profiles, SchedulerConfig(**sched_kwargs))
    return Simulation(trace, profiles, pol, devices)


def test_empty_trace():
    assert sim_for([]).run().records == []


def test_single_invocation_cold_timing():
    profiles = {"f": FunctionProfile("f", 1.0, 4.0, 100.0, 0.4, 1.0)}
    r = sim_for([(2.0, "f")], profiles=profiles).run().records[0]
    assert r.dispatch_s == 2.0 and r.complete_s == pytest.approx(6.0) and r.start_state == "cold"


def test_validation_at_construction():
    with pytest.raises(ValueError, match="unknown"):
        sim_for([(0.0, "nope")])
    with pytest.raises(ValueError, match="non-decreasing"):
        sim_for([(1.0, "fft"), (0.5, "fft")])


def test_same_time_events_in_insertion_order():
    sim = sim_for([(1.0, "fft"), (1.0, "roberta")])
    arrivals = []
    while (ev := sim.step()) is not None:
        if ev[1] == ARRIVAL:
            arrivals.append(ev)
    assert [a[2].function for a in arrivals] == ["fft", "roberta"]
    assert arrivals[0][0] == arrivals[1][0] == 1.0


def test_monitor_stops_when_idle_and_clock_moves_forward():
    sim = sim_for([(0.0, "fft")])
    last, ticks = -1.0, []
    while (ev := sim.step()) is not None:
        assert ev[0] >= last
        last = ev[0]
        if ev[1] == MONITOR_TICK:
            ticks.append(ev[0])
    assert ticks and len(sim.records) == 1
    assert ticks[-1] >= sim.records[0].complete_s        # one tick after the work is done


def test_conservation_and_determinism():
    trace = gen_zipf(4, 1.5, 1.0, 60.0, seed=3)
    profiles = default_profiles(4)
    a = sim_for(trace.entries, profiles=profiles).run()
    b = sim_for(trace.entries, profiles=profiles).run()
    assert len(a.records) == len(trace.entries)
    assert [(r.function, r.complete_s) for r in a.records] == \
        [(r.function, r.complete_s) for r in b.records]


@pytest.mark.parametrize("case", engine_cases(), ids=lambda c: c["name"])
def test_event_stream_matches_reference(case):
    """Simulation.step() replays the reference's processed-event stream."""
    from oracle import oracle as orc
    entries, profiles, devices = orc.case_inputs(case)
    trace = Trace(entries=entries, duration_s=entries[-1][0] if entries else 0.0)
    pol = make_policy(case.get("policy", "mqfq"), profiles,
                      SchedulerConfig(**case.get("sched", {})))
    sim = Simulation(trace, profiles, pol, DeviceSet(devices),
                     tau_includes_overheads=bool(case.get("tau_inc", False)))
    pos = {inv.uid: i for i, inv in enumerate(sim._inv)}
    evs = []
    while (ev := sim.step()) is not None:
        t, kind, pay = ev
        if kind == ARRIVAL:
            pay = pos[pay.uid]
        elif kind == 1:
            pay = pos[pay]
        evs.append((t, kind, pay))
    gold = golden()[case["name"]]["fp"]
    assert fp(evs) == gold["events"]
    res_records = [(r.function, r.arrival_s, r.dispatch_s, r.complete_s, r.start_state, r.device)
                   for r in sim.records]
    assert fp(res_records) == gold["records"]
