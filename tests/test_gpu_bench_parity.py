"""Parity at the bench's full sizes (BASELINE C3 / C2 / C5 sweeps, their
exact launch configuration): a random sample of each batch against the C
oracle bit for bit (records, dispatch rows) and within 1e-9 (statistics),
plus size-independent properties over every simulation -- every arrival
completes, per-function counts add up, the histograms hold every
completion, and the stats-only bench launch gives the same statistics as a
records launch of the same batch."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine():
    from paper_2507_08954_b200.engine import Engine
    e = Engine(0)
    yield e
    e.close()


def _bench_launch(eng, w, flags=0):
    from paper_2507_08954_b200 import _abi, sweep
    eng.run(w.sims_array(), outputs=_abi.WANT_STATS | _abi.WANT_HIST, early_exit=True,
            hist_groups=w.groups, hist_rows=w.hist_rows, hist_bins=sweep.HIST_BINS,
            hist_lo_s=sweep.HIST_LO_S, hist_hi_s=sweep.HIST_HI_S, flags=flags)
    return {oid: eng.output(oid).copy() for oid in (
        _abi.OUT_STATUS, _abi.OUT_COUNTERS, _abi.OUT_SUMMARY, _abi.OUT_FLOW_COUNT,
        _abi.OUT_FLOW_MEAN, _abi.OUT_FLOW_VAR, _abi.OUT_FLOW_COLD_PCT, _abi.OUT_HIST)}


def _check(eng, w, n_sample, seed=0, flags=0, expect=None):
    """expect: batch_info() entries the bench launch must have (its build)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import oracle as orc
    from paper_2507_08954_b200 import _abi
    from paper_2507_08954_b200.engine import BatchResult
    w.upload(eng)
    bench = _bench_launch(eng, w, flags)
    info = eng.batch_info()
    for k, v in (expect or {}).items():
        assert info[k] == v, (k, info)
    assert (bench[_abi.OUT_STATUS] == 0).all()
    eng.run(w.sims_array(), outputs=_abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_DISPATCH,
            early_exit=True, flags=flags)
    for k, v in (expect or {}).items():
        assert eng.batch_info()[k] == v, (k, eng.batch_info())
    res = BatchResult(eng)
    c = res.counters
    n_arr = np.array([w.traces[s.trace].n for s in w.sims])
    # every arrival is dispatched and completes; the flow counts add up
    assert np.array_equal(c[:, 2], n_arr)
    fo = res.flow_off
    fc = res.get(_abi.OUT_FLOW_COUNT)
    assert np.array_equal(np.add.reduceat(fc, fo[:-1]) if len(fc) else fc, n_arr)
    # the bench's stats-only launch computes the same numbers
    for oid in (_abi.OUT_SUMMARY, _abi.OUT_FLOW_COUNT, _abi.OUT_FLOW_MEAN, _abi.OUT_FLOW_VAR,
                _abi.OUT_FLOW_COLD_PCT):
        assert np.array_equal(bench[oid], res.get(oid)), oid
    assert int(bench[_abi.OUT_HIST].sum()) == int(n_arr.sum())
    # a random sample against the oracle (ctypes releases the GIL: threads)
    rng = np.random.default_rng(seed)
    bad, work = [], []
    sample = sorted(rng.choice(len(w.sims), n_sample, replace=False).tolist())

    def oracle_run(i):
        s = w.sims[i]
        tr, tab = w.traces[s.trace], w.tabs[s.flowtab]
        dc = w.dcfgs[s.device_cfg: s.device_cfg + s.n_devices]
        return orc.run_packed(_abi.Sim.from_buffer_copy(s), tr.arrival, tr.flow, tr.n_flows,
                              {"warm": tab.warm, "cold": tab.cold, "mem": tab.mem,
                               "share": tab.share, "weight": tab.weight},
                              [_abi.device_cfg_from(d) for d in dc], want_audit=False,
                              early_exit=True)

    with ThreadPoolExecutor(max_workers=16) as ex:
        refs = list(ex.map(oracle_run, sample))
    for i, r in zip(sample, refs):
        rec = res.records(i)
        comp = res.completion_order(i)
        dr = res.dispatch_rows(i)
        fs = res.flow_stats(i)
        ok = (np.array_equal(comp, r["rec_inv"])
              and np.array_equal(rec["complete"][comp], r["rec_complete"])
              and np.array_equal(rec["dispatch"][comp], r["rec_dispatch"])
              and np.array_equal(rec["state"][comp], r["rec_state"])
              and np.array_equal(dr["inv"], r["d_inv"])
              and np.array_equal(dr["vt_before"], r["d_vt_before"])
              and np.array_equal(dr["gvt"], r["d_gvt"])
              and np.array_equal(fs["count"], r["f_count"])
              and np.allclose(fs["mean"], r["f_mean"], rtol=1e-9, atol=0)
              and np.allclose(fs["var"], r["f_var"], rtol=1e-9, atol=0)
              and abs(res.summary[i, 0] - r["weighted_avg_latency"])
              <= 1e-9 * abs(r["weighted_avg_latency"])
              and res.summary[i, 2] == r["mean_util"])
        if not ok:
            bad.append(i)
        # the same early exit in both (bench arms do identical work): the
        # processed events and dispatch() calls agree too
        if (int(c[i, 0]), int(c[i, 1])) != (r["n_events"], r["n_dispatch_calls"]):
            work.append((i, int(c[i, 0]), r["n_events"], int(c[i, 1]), r["n_dispatch_calls"]))
    assert not bad, f"{len(bad)} of {n_sample} sampled sims differ from the oracle: {bad[:10]}"
    assert not work, f"event / dispatch-call counts differ (sim, gpu, oracle): {work[:5]}"


def test_c3_full_sweep(engine):
    from paper_2507_08954_b200 import sweep
    _check(engine, sweep.build("c3", 0, engine=engine), 128)


def test_c2_sample_of_seeds(engine):
    from paper_2507_08954_b200 import sweep
    _check(engine, sweep.build("c2", 0, engine=engine, n_seeds=40), 96, seed=1)


def test_c5_shard_sample(engine):
    from paper_2507_08954_b200 import sweep
    _check(engine, sweep.build("c5", 0, engine=engine, n_seeds=48), 120, seed=2)


def test_c4_bench_batch_cta(engine):
    """BASELINE C4 exactly as the bench runs it: 148 simulations of 4096
    functions (37 seeds x pool 32/256 x MQFQ/FCFS, 1800 s), one per SM on the
    CTA-per-simulation build; 32 sampled against the oracle."""
    from paper_2507_08954_b200 import sweep
    _check(engine, sweep.build("c4", 0, engine=engine), 32, seed=3,
           expect={"cta_threads": 512, "flows_global": False})


def test_c4_large_batch_flows_global(engine):
    """C4 at 2368 simulations (592 seeds): the batch size where gfq_prepare
    switches to the warp build with the flow state in global scratch (16
    simulations per SM); conservation over all 2368, 32 sampled vs the oracle."""
    from paper_2507_08954_b200 import sweep
    _check(engine, sweep.build("c4", 0, engine=engine, n_seeds=592), 32, seed=4,
           expect={"cta_threads": 0, "flows_global": True})
