"""GPU tests of the public API: the run_simulation drop-in against the
oracle, reference-shaped results, error mapping, watchdog and overflow
statuses, stream launches and the histogram / stats outputs."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2507_08954_b200 import _abi
from paper_2507_08954_b200.device import DeviceConfig, DeviceSet
from paper_2507_08954_b200.engine import Engine, run_simulation, sim_params
from paper_2507_08954_b200.mqfq import SchedulerConfig
from paper_2507_08954_b200.pack import flow_table, pack_trace
from paper_2507_08954_b200.policies import make_policy
from paper_2507_08954_b200.workload import default_profiles, gen_zipf

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("policy", ["mqfq", "fcfs", "batch", "sjf"])
def test_run_simulation_dropin_matches_oracle(policy):
    profiles = default_profiles(12)
    trace = gen_zipf(12, 1.5, 3.0, 120.0, 5)
    cfg = SchedulerConfig(t_overrun=5.0, alpha=2.0)
    pol = make_policy(policy, profiles, cfg)
    devs = DeviceSet([DeviceConfig(d_max=3), DeviceConfig(d_max=2, mem_capacity_mb=8000.0)])
    res = run_simulation(trace, profiles, pol, devs)
    case = {"trace": {"entries": [[t, nm] for t, nm in trace.entries]},
            "profiles": {"explicit": [[p.name, p.warm_exec_s, p.cold_exec_s, p.mem_mb,
                                       p.compute_share, p.weight] for p in profiles.values()]},
            "policy": policy, "sched": {"t_overrun": 5.0, "alpha": 2.0},
            "devices": [{"d_max": 3}, {"d_max": 2, "mem_capacity_mb": 8000.0}]}
    ref = orc.run_case(case)
    got = [(r.function, r.arrival_s, r.dispatch_s, r.complete_s, r.start_state, r.device)
           for r in res.records]
    assert got == ref["records"]
    assert len(pol.dispatch_log) == len(ref["dispatch"])
    d = pol.dispatch_log[5]
    assert (d.now, d.function, d.vt_before, d.global_vt, d.queue_len, d.in_flight, d.device,
            d.start_state) == ref["dispatch"][5]
    assert res.audit.util == ref["util"] and res.audit.backlog == ref["backlog"]


def _small_engine():
    eng = Engine(0)
    profiles = default_profiles(6)
    pt = pack_trace(gen_zipf(6, 1.5, 2.0, 60.0, 1).entries, profiles)
    eng.upload_traces([pt])
    eng.upload_flowtabs([flow_table(pt.names, profiles)])
    eng.upload_device_cfgs([DeviceConfig()])
    return eng, pt


def test_value_errors_map_to_valueerror():
    eng, _ = _small_engine()
    with pytest.raises(ValueError, match="trace id"):
        s = sim_params("mqfq", SchedulerConfig(), 1, trace=3)
        eng.run([s])
    with pytest.raises(ValueError, match="d_max"):
        eng.upload_device_cfgs([_abi.DeviceCfg(16384.0, 0.9, 12000.0, 0.1, 0.2, 1.0, 0.0, 0, 32, 1, 0)])
    with pytest.raises(ValueError, match="non-decreasing"):
        from paper_2507_08954_b200.pack import PackedTrace
        eng.upload_traces([PackedTrace(["a"], np.array([1.0, 0.5]), np.array([0, 0], np.int32))])
    eng.close()


def test_unadmittable_function_is_rejected():
    """mem_mb > mem_capacity_mb makes the reference spin forever:
    the engine refuses the batch with a ValueError instead."""
    eng, _ = _small_engine()
    eng.upload_device_cfgs([DeviceConfig(mem_capacity_mb=1000.0)])
    with pytest.raises(ValueError, match="mem_capacity"):
        eng.run([sim_params("mqfq", SchedulerConfig(), 1)])
    eng.close()


def test_watchdog_status():
    from paper_2507_08954_b200._lib import EngineError
    eng, _ = _small_engine()
    s = sim_params("mqfq", SchedulerConfig(), 1)
    s.max_events = 50
    with pytest.raises(EngineError, match="watchdog"):
        eng.run([s])
    eng.close()


def test_event_pool_overflow_is_reported_not_truncated():
    from paper_2507_08954_b200._lib import EngineError
    eng, _ = _small_engine()
    with pytest.raises(EngineError, match="event pool"):
        eng.run([sim_params("mqfq", SchedulerConfig(alpha=8.0), 1)], event_capacity=2)
    eng.close()


def test_stream_launch_and_histograms():
    import torch
    eng, pt = _small_engine()
    sims = [sim_params("mqfq", SchedulerConfig(t_overrun=t), 1, group=g)
            for g, t in enumerate((0.0, 10.0))]
    eng.prepare(sims, outputs=_abi.WANT_STATS | _abi.WANT_HIST | _abi.WANT_RECORDS,
                hist_groups=2, hist_rows=len(pt.names), hist_bins=32, hist_lo_s=1e-2,
                hist_hi_s=1e4)
    st = torch.cuda.Stream()
    eng.launch(st)
    st.synchronize()
    eng.synchronize()
    hist = eng.output(_abi.OUT_HIST).reshape(2, len(pt.names), 32)
    cnt = eng.output(_abi.OUT_FLOW_COUNT).reshape(2, -1)
    assert np.array_equal(hist.sum(axis=2), cnt)           # every completion binned once
    from paper_2507_08954_b200.dist import hist_bin
    from paper_2507_08954_b200.engine import BatchResult
    res = BatchResult(eng)
    rec = res.records(0)
    lat = rec["complete"] - pt.arrival
    ref = np.zeros((len(pt.names), 32), np.int64)
    np.add.at(ref, (pt.flow, hist_bin(lat, 1e-2, 1e4, 32)), 1)
    assert np.array_equal(hist[0], ref)
    eng.close()


def test_fast_and_generic_builds_agree_on_stats():
    """The same MQFQ sims through the fast build (stats only) and the
    generic build (audit logs requested) give identical outputs."""
    eng, pt = _small_engine()
    sims = [sim_params("mqfq", SchedulerConfig(t_overrun=t, alpha=a), 1)
            for t in (0.0, 2.0, 10.0) for a in (0.0, 1.0, 4.0)]
    fast = eng.run(sims, outputs=_abi.WANT_STATS)
    a = (fast.summary.copy(), fast.get(_abi.OUT_FLOW_MEAN).copy(), fast.counters[:, :4].copy())
    gen = eng.run(sims, outputs=_abi.WANT_STATS | _abi.WANT_AUDIT)
    assert np.array_equal(a[0], gen.summary)
    assert np.array_equal(a[1], gen.get(_abi.OUT_FLOW_MEAN))
    assert np.array_equal(a[2], gen.counters[:, :4])
    eng.close()


def test_trace_upload_validation_on_gpu():
    """gfq_upload_traces validates every arrival on the GPU and reports the
    first failure in (trace, position, check) order, as a sequential scan
    would (engine.py:50-52,72-73); a failed upload leaves no traces resident."""
    from paper_2507_08954_b200.engine import Engine
    eng = Engine(0)
    good = np.array([0.5, 1.0, 1.0, 2.0])
    bad_t = np.array([0.5, 1.0, 0.9, 2.0])
    off = np.array([0, 4, 8, 12], dtype=np.int64)
    nf = np.array([2, 2, 2], dtype=np.int32)
    fl = np.zeros(12, dtype=np.int32)

    def up(arr, flow):
        eng.upload_trace_arrays(np.ascontiguousarray(arr, dtype=np.float64),
                                np.ascontiguousarray(flow, dtype=np.int32), off, nf)

    with pytest.raises(ValueError, match=r"non-decreasing \(trace 2\)"):
        up(np.concatenate([good, good, bad_t]), fl)
    f2 = fl.copy(); f2[9] = 2; f2[6] = 5                  # trace 1 fails first
    with pytest.raises(ValueError, match="flow id out of range in trace 1"):
        up(np.concatenate([good, good, bad_t]), f2)
    a3 = np.concatenate([good, good, good]); a3[5] = np.nan
    with pytest.raises(ValueError, match="finite"):
        up(a3, fl)
    up(np.concatenate([good, good, good]), fl)            # a valid upload still works
    eng.close()


def test_capacity_statuses_are_retried():
    """The engine's event pool, audit buffers and event budget are its own
    limits (the reference has none): a single simulation that hits one is
    re-run with larger ones and then matches the oracle."""
    import numpy as np
    from oracle import oracle as orc
    from test_gpu_fuzz import _workload
    from paper_2507_08954_b200 import _abi
    from paper_2507_08954_b200.engine import Engine, _run_one
    traces, tabs, dcfgs, sims, _ = _workload(np.random.default_rng(5), 5)
    eng = Engine(0)
    eng.upload_traces(traces)
    eng.upload_flowtabs(tabs)
    eng.upload_device_cfgs(dcfgs)
    s = sims[0]                                              # MQFQ
    tr, tab = traces[0], tabs[0]
    r = orc.run_packed(_abi.Sim.from_buffer_copy(s), tr.arrival, tr.flow, tr.n_flows,
                       {"warm": tab.warm, "cold": tab.cold, "mem": tab.mem,
                        "share": tab.share, "weight": tab.weight},
                       [_abi.device_cfg_from(d) for d in dcfgs[s.device_cfg: s.device_cfg + s.n_devices]],
                       want_audit=False)
    outs = _abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_DISPATCH | _abi.WANT_AUDIT
    tight = _abi.Sim.from_buffer_copy(s)
    tight.max_events = 500
    for sim, kw in ((s, {"event_capacity": 2}), (s, {"audit_util_cap": 256}), (tight, {})):
        res = _run_one(eng, sim, tr.n, outs, True, **kw)
        comp = res.completion_order(0)
        assert int(res.status[0]) == 0
        assert np.array_equal(comp, r["rec_inv"])
        assert np.array_equal(res.records(0)["complete"][comp], r["rec_complete"])
        assert np.array_equal(res.dispatch_rows(0)["vt_before"], r["d_vt_before"])
    eng.close()
