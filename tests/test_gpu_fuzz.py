"""Randomised parity: 480 random simulations (every policy; 1-3 devices;
D, T, alpha, default TTL, pool size / disabled, dynamic D, utilisation
threshold and window, PCIe bandwidth, prefetch overlap, interference,
heterogeneous profiles, a third of them with non-integral memory sizes) run as one batch and checked against the C oracle:
dispatch rows and completion records bit for bit, per-function statistics
and the run summary within 1e-9.  The batch runs through each build: the
specialised warp classes (statistics + records + dispatch rows, early
exit), the generic class (audit logs requested), flows in global memory,
CTA-per-simulation, and the forced warp build (GFQ_FLAG_WARP).  Complements the 1560 golden cases with configurations
nobody hand-picked."""

from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

POLICIES = ("mqfq", "fcfs", "batch", "sjf", "fcfs_naive")


def _workload(rng, n_sims):
    from paper_2507_08954_b200 import _abi
    from paper_2507_08954_b200.core import FunctionProfile
    from paper_2507_08954_b200.device import DeviceConfig
    from paper_2507_08954_b200.engine import sim_params
    from paper_2507_08954_b200.mqfq import SchedulerConfig
    from paper_2507_08954_b200.pack import flow_table, pack_trace
    from paper_2507_08954_b200.workload import default_profiles, gen_zipf
    traces, tabs, dcfgs, sims = [], [], [], []
    for i in range(n_sims):
        nfn = int(rng.integers(2, 40))
        cap = float(rng.choice([4096.0, 8192.0, 16384.0]))
        base = default_profiles(nfn)
        def warm_cold(p):
            w = p.warm_exec_s * float(rng.uniform(0.5, 2.0))
            return w, max(w, p.cold_exec_s * float(rng.uniform(0.5, 2.0)))
        # a third of the tables get non-integral memory sizes: those simulations
        # leave the 1-device fast classes (integer resident-memory sums) for
        # the classes that replay CPython's compensated sum in pool order
        frac = bool(rng.random() < 1 / 3)
        def mem_mb():
            m = float(rng.choice([256.0, 512.0, 1024.0, 1500.0, 3000.0]))
            return m * float(rng.uniform(0.5, 1.3)) if frac else m
        profiles = {nm: FunctionProfile(nm, *warm_cold(p),
                                        mem_mb(),
                                        float(rng.uniform(0.1, 0.7)),
                                        float(rng.choice([1.0, 1.0, 2.0, 0.5])))
                    for nm, p in base.items()}
        tr = gen_zipf(nfn, float(rng.uniform(0.6, 2.0)), float(rng.uniform(0.5, 4.0)),
                      float(rng.uniform(30.0, 240.0)), int(rng.integers(1, 10 ** 6)),
                      names=list(profiles))
        pt = pack_trace(tr.entries, profiles)
        traces.append(pt)
        tabs.append(flow_table(pt.names, profiles, None))
        pol = POLICIES[i % len(POLICIES)]
        ndev = int(rng.choice([1, 1, 1, 2, 3]))
        d_max = int(rng.integers(1, 5))
        dyn = bool(rng.random() < 0.3)
        for _ in range(ndev):
            dcfgs.append(DeviceConfig(
                mem_capacity_mb=cap, d_max=d_max, util_threshold=float(rng.uniform(0.6, 1.0)),
                pcie_mb_per_s=float(rng.choice([3000.0, 12000.0])),
                interference_beta=float(rng.uniform(0.0, 0.3)),
                monitor_period_s=float(rng.choice([0.1, 0.2, 0.5])),
                util_window_s=float(rng.choice([0.4, 1.0, 2.0])),
                pool_max_containers=int(rng.integers(2, 33)),
                pool_enabled=pol != "fcfs_naive" and bool(rng.random() < 0.9),
                dynamic_d=dyn, prefetch_overlap_s=float(rng.choice([0.0, 0.05]))))
        cfg = SchedulerConfig(t_overrun=float(rng.choice([0.0, 1.0, 5.0, 10.0, 50.0])),
                              d_max=d_max, alpha=float(rng.choice([0.0, 0.5, 2.0, 8.0])),
                              default_ttl_s=float(rng.choice([0.5, 2.0, 5.0])))
        sim = sim_params(pol, cfg, ndev, trace=i, flowtab=i, device_cfg=len(dcfgs) - ndev,
                         tau_includes_overheads=bool(rng.random() < 0.2))
        sim.max_events = 1 << 30       # heavily overloaded draws tick for a long time
        sims.append(sim)
    return traces, tabs, dcfgs, sims, _abi


BUILDS = {"fast": (0, 0), "generic": (0, 1), "flows_global": (1, 0), "cta": (2, 0), "warp": (4, 0)}
# GFQ_FUZZ_ROUNDS=N runs N independently seeded batches per build (default 1)
ROUNDS = int(os.environ.get("GFQ_FUZZ_ROUNDS", "1"))


EVENT_OVERFLOW = 1        # gfq.h GFQ_SIM_EVENT_OVERFLOW


def _check(eng, idx, sims, traces, tabs, dcfgs, _abi, flags, audit, event_capacity=0):
    """Run sims[idx] as one batch; return (mismatching, event-pool overflowed)
    indices.  An overflow is the engine's documented capacity status (callers
    re-run with a larger event_capacity, as cli.run_experiments does)."""
    from oracle import oracle as orc
    from paper_2507_08954_b200._lib import EngineError
    from paper_2507_08954_b200.engine import BatchResult
    outputs = _abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_DISPATCH
    kw = {}
    if audit:
        outputs |= _abi.WANT_AUDIT
        kw["audit_util_cap"] = 1 << 17                        # overloaded sims tick long
    eng.prepare([sims[i] for i in idx], outputs=outputs, early_exit=True, flags=flags,
                event_capacity=event_capacity, **kw)
    eng.launch()
    try:
        eng.synchronize()
    except EngineError:
        pass                                                  # per-sim status below
    res = BatchResult(eng)
    bad, over = [], []
    for j, i in enumerate(idx):
        s = sims[i]
        if int(res.status[j]) == EVENT_OVERFLOW:
            over.append(i)
            continue
        tr, tab = traces[s.trace], tabs[s.flowtab]
        dc = dcfgs[s.device_cfg: s.device_cfg + s.n_devices]
        r = orc.run_packed(_abi.Sim.from_buffer_copy(s), tr.arrival, tr.flow, tr.n_flows,
                           {"warm": tab.warm, "cold": tab.cold, "mem": tab.mem,
                            "share": tab.share, "weight": tab.weight},
                           [_abi.device_cfg_from(d) for d in dc], want_audit=False)
        rec = res.records(j)
        comp = res.completion_order(j)
        dr = res.dispatch_rows(j)
        fs = res.flow_stats(j)
        ok = (int(res.status[j]) == 0
              and np.array_equal(comp, r["rec_inv"])
              and np.array_equal(rec["complete"][comp], r["rec_complete"])
              and np.array_equal(rec["dispatch"][comp], r["rec_dispatch"])
              and np.array_equal(rec["state"][comp], r["rec_state"])
              and np.array_equal(rec["device"][comp], r["rec_device"])
              and np.array_equal(dr["inv"], r["d_inv"])
              and np.array_equal(dr["vt_before"], r["d_vt_before"])
              and np.array_equal(dr["gvt"], r["d_gvt"])
              and np.array_equal(fs["count"], r["f_count"])
              and np.allclose(fs["mean"], r["f_mean"], rtol=1e-9, atol=0)
              and np.allclose(fs["var"], r["f_var"], rtol=1e-9, atol=0)
              and abs(res.summary[j, 0] - r["weighted_avg_latency"])
              <= 1e-9 * abs(r["weighted_avg_latency"])
              and res.summary[j, 2] == r["mean_util"])
        if not ok:
            bad.append((i, s.policy, s.n_devices, int(res.status[j])))
    return bad, over


@pytest.mark.parametrize("rnd", range(ROUNDS))
@pytest.mark.parametrize("build", list(BUILDS))
def test_random_configs_match_oracle(build, rnd):
    from paper_2507_08954_b200.engine import Engine
    rng = np.random.default_rng(20261017 + 1000 * rnd)
    traces, tabs, dcfgs, sims, _abi = _workload(rng, 480 if build == "fast" else 160)
    flags, audit = BUILDS[build]
    eng = Engine(0)
    eng.upload_traces(traces)
    eng.upload_flowtabs(tabs)
    eng.upload_device_cfgs(dcfgs)
    args = (sims, traces, tabs, dcfgs, _abi, flags, audit)
    bad, over = _check(eng, list(range(len(sims))), *args)
    if over:                      # the default pool (2 slots per flow) overflowed: re-run larger
        bad2, over2 = _check(eng, over, *args, event_capacity=2048)
        bad += bad2 + [(i, "still overflows") for i in over2]
    eng.close()
    assert not bad, f"{len(bad)} of {len(sims)} random sims differ from the oracle: {bad[:10]}"
