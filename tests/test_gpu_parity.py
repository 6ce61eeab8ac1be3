"""GPU parity: the CUDA engine against the reference's own outputs.

All 1560 golden cases (tests/golden/reference_golden.json: Appendix-B
default/medium x 5 policies, the reference's engine scenarios, 400 A1-style
fuzz instances over every device/scheduler knob, C2/C3/C4 samples, and the
acceptance suite's 1000 A8 + 100 A11 scripted oracle instances) run as ONE
batch through libgfq.so.  Dispatch traces, completion records, exec / util /
backlog audit and the processed-event stream must match the reference's
fingerprints bit for bit; per-function latency statistics and the run
summary within 1e-9 relative (north_star).
"""

from __future__ import annotations

import pytest

from cases import all_cases
from golden_check import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine():
    from paper_2507_08954_b200.engine import Engine
    e = Engine(0)
    yield e
    e.close()


@pytest.fixture(scope="module")
def full_run(engine):
    from gpu_harness import run_cases
    cases = all_cases()
    outs, res = run_cases(cases, engine, early_exit=False, event_log_cap=65536,
                          audit_util_cap=16384)
    return cases, outs


def _report(cases, outs, gold, keys=None):
    from gpu_harness import compare_to_golden
    bad = {}
    for case, out in zip(cases, outs):
        m = compare_to_golden(out, gold[case["name"]], **({"exact_keys": keys} if keys else {}))
        if m:
            bad[case["name"]] = m
    return bad


@pytest.mark.parametrize("family", ["appendix_b", "engine", "fuzz", "c3", "c2", "c4", "a8", "a11"])
def test_golden_family(full_run, family):
    cases, outs = full_run
    sel = [(c, o) for c, o in zip(cases, outs) if c["name"].split("/")[0] == family]
    bad = _report([c for c, _ in sel], [o for _, o in sel], golden())
    assert sel
    assert not bad, f"{len(bad)}/{len(sel)} differ: {dict(list(bad.items())[:6])}"


def test_early_exit_is_exact(engine, full_run):
    """The bench configuration (early exit once only keep-alive rechecks
    remain) changes no record, dispatch row, audit row or stat."""
    from gpu_harness import run_cases
    from paper_2507_08954_b200 import _abi
    cases, full = full_run
    outs, _ = run_cases(cases, engine, early_exit=True, audit_util_cap=16384,
                        outputs=_abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_DISPATCH |
                        _abi.WANT_AUDIT)
    for c, a, b in zip(cases, outs, full):
        for k in ("dispatch", "records", "exec", "util", "backlog", "summary", "per_function",
                  "transcript"):
            assert a.get(k) == b.get(k), (c["name"], k)


def test_fast_build_matches_reference(engine):
    """MQFQ-Sticky / DeviceSet sims run the specialised k_sim<false> build
    (bench configuration); its dispatch rows, records and statistics must
    match the reference like the generic build's."""
    from gpu_harness import compare_to_golden, run_cases
    from paper_2507_08954_b200 import _abi
    fast = [c for c in all_cases() if c.get("policy", "mqfq") == "mqfq" and not c.get("scripted")]
    one = [c for c in fast if len(c.get("devices", [{}])) == 1]     # k_sim<false, true>
    gold = golden()
    for cases in (one, fast):                                         # ... and <false, false>
        outs, _ = run_cases(cases, engine, early_exit=True,
                            outputs=_abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_DISPATCH)
        bad = {}
        for c, o in zip(cases, outs):
            m = compare_to_golden(o, gold[c["name"]], exact_keys=("dispatch", "records", "exec"))
            if m:
                bad[c["name"]] = m
        assert not bad, f"{len(bad)}/{len(cases)} differ: {dict(list(bad.items())[:6])}"


def test_mixed_class_batch(engine):
    """One batch whose sims span the three kernel classes (generic, MQFQ
    multi-device, MQFQ 1-device): each class runs its own launch over its
    slice of the work order; every sim must still match the reference."""
    from gpu_harness import compare_to_golden, run_cases
    from paper_2507_08954_b200 import _abi
    cases = all_cases()
    outs, _ = run_cases(cases, engine, early_exit=True,
                        outputs=_abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_DISPATCH)
    gold = golden()
    bad = {c["name"]: m for c, o in zip(cases, outs)
           if (m := compare_to_golden(o, gold[c["name"]], exact_keys=("dispatch", "records", "exec")))}
    assert not bad, f"{len(bad)}/{len(cases)} differ: {dict(list(bad.items())[:6])}"


def test_flows_global_build(engine):
    """The build that keeps per-flow state in global scratch (used when the
    flow count does not fit shared memory, e.g. C4's 4096 functions), forced
    on every golden case with every output."""
    from gpu_harness import compare_to_golden, run_cases
    from paper_2507_08954_b200 import _abi
    cases = all_cases()
    outs, _ = run_cases(cases, engine, early_exit=False, event_log_cap=65536,
                        audit_util_cap=16384, flags=_abi.FLAG_FLOWS_GLOBAL)
    gold = golden()
    bad = {c["name"]: m for c, o in zip(cases, outs)
           if (m := compare_to_golden(o, gold[c["name"]]))}
    assert not bad, f"{len(bad)}/{len(cases)} differ: {dict(list(bad.items())[:6])}"


@pytest.mark.parametrize("flags", ["cta", "cta+global"])
def test_cta_build(engine, flags):
    """The CTA-per-simulation build (one simulation per CTA, scans split over
    its warps; automatic for large flow counts), forced on every golden case
    with every scan on the CTA path (cta_min = 0), with the workspace in
    shared memory and with the flow/event part in global scratch."""
    from gpu_harness import compare_to_golden, run_cases
    from paper_2507_08954_b200 import _abi
    cases = all_cases()
    f = _abi.FLAG_CTA | (_abi.FLAG_FLOWS_GLOBAL if "global" in flags else 0)
    outs, _ = run_cases(cases, engine, early_exit=False, event_log_cap=65536,
                        audit_util_cap=16384, flags=f)
    gold = golden()
    bad = {c["name"]: m for c, o in zip(cases, outs)
           if (m := compare_to_golden(o, gold[c["name"]]))}
    assert not bad, f"{len(bad)}/{len(cases)} differ: {dict(list(bad.items())[:6])}"


@pytest.mark.parametrize("flags", ["cta", "cta+global"])
def test_cta_fast_builds(engine, flags):
    """The specialised CTA builds (MQFQ-Sticky / FCFS on a 1-device
    DeviceSet, device state in registers), forced on every such golden case
    with every scan on the CTA path: dispatch rows, records and statistics
    must match the reference."""
    from gpu_harness import compare_to_golden, run_cases
    from paper_2507_08954_b200 import _abi
    cases = [c for c in all_cases() if not c.get("scripted")
             and c.get("policy", "mqfq") in ("mqfq", "fcfs", "fcfs_naive")
             and len(c.get("devices", [{}])) == 1]
    f = _abi.FLAG_CTA | (_abi.FLAG_FLOWS_GLOBAL if "global" in flags else 0)
    outs, _ = run_cases(cases, engine, early_exit=True, flags=f,
                        outputs=_abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_DISPATCH)
    gold = golden()
    bad = {c["name"]: m for c, o in zip(cases, outs)
           if (m := compare_to_golden(o, gold[c["name"]], exact_keys=("dispatch", "records")))}
    assert cases and not bad, f"{len(bad)}/{len(cases)} differ: {dict(list(bad.items())[:6])}"


@pytest.mark.parametrize("build", ["auto", "warp"])
def test_c4_large_flow_sims_match_oracle(engine, build):
    """BASELINE C4: 4096 functions per simulation (2.1k touched), pool 32/256,
    heterogeneous memory, MQFQ + FCFS vs the oracle: the CTA-per-simulation
    build a small batch gets, and the warp build with the flow state in global
    scratch that a large batch gets (GFQ_FLAG_WARP)."""
    from c4_check import check
    from paper_2507_08954_b200 import _abi
    assert check(1, engine, _abi.FLAG_WARP if build == "warp" else 0) == []


def test_large_flow_batch_build_choice(engine):
    """Large-flow simulations: a batch of one wave per SM runs CTA-per-simulation;
    a batch that would need more than 6 CTA waves per warp-build wave runs the
    warp build with the flow state in global scratch (gfq_prepare's rule)."""
    import torch
    from paper_2507_08954_b200 import _abi, sweep
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    w = sweep.c4(n_seeds=1)
    w.upload(engine)
    s0 = w.sims[0]
    small = (_abi.Sim * n_sm)(*([s0] * n_sm))
    engine.prepare(small, outputs=_abi.WANT_STATS)
    info = engine.batch_info()
    assert info["cta_threads"] > 0 and not info["flows_global"], info
    big = (_abi.Sim * (16 * n_sm))(*([s0] * (16 * n_sm)))
    engine.prepare(big, outputs=_abi.WANT_STATS)
    info = engine.batch_info()
    assert info["cta_threads"] == 0 and info["flows_global"], info
    engine.prepare(big, outputs=_abi.WANT_STATS, flags=_abi.FLAG_CTA)
    assert engine.batch_info()["cta_threads"] > 0
