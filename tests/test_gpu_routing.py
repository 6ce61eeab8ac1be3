"""Parity at the edges of the kernel-class routing added in round 2
(gfq_prepare): the 1-device warp classes keep their per-flow counters in
u16 and sum resident memory as integers, so

* a trace of 65535+ arrivals must leave them (-> the i32 classes),
* a flow table with a non-integral mem_mb must leave them (-> the MQFQ
  multi-device class or the generic class, whose resident_mb replays
  CPython's compensated sum in pool order),

and both must still match the C oracle bit for bit (dispatch rows, records)
and within 1e-9 (statistics), in the warp and the CTA builds."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

FAST = None


@pytest.fixture(scope="module")
def engine():
    from paper_2507_08954_b200.engine import Engine
    e = Engine(0)
    yield e
    e.close()


def _rows(names, warm, mems):
    return [[nm, w, 4.0 * w, m, 0.38, 1.0] for nm, w, m in zip(names, warm, mems)]


def _long_case(policy):
    # 4 short functions at 110 rps for 620 s: ~68k arrivals, rho ~0.6 on D=4
    names = ["a", "b", "c", "d"]
    return dict(name=f"long/{policy}", trace={"gen": [4, 1.2, 110.0, 620.0, 7], "names": names},
                profiles={"explicit": _rows(names, [0.02, 0.03, 0.015, 0.025], [256.0] * 4)},
                policy=policy, sched={"t_overrun": 5.0, "alpha": 2.0},
                devices=[{"d_max": 4, "pool_max_containers": 8}])


def _frac_case(policy, i):
    # non-integral mem_mb with memory pressure: LRU swap-outs and refusals
    names = [f"f{k}" for k in range(12)]
    mems = [1000.0 + 123.456 * k + 0.1 * i for k in range(12)]
    return dict(name=f"frac/{policy}/{i}", trace={"gen": [12, 1.1, 3.0, 300.0, 100 + i],
                                                  "names": names},
                profiles={"explicit": _rows(names, [0.3 + 0.05 * k for k in range(12)], mems)},
                policy=policy, sched={"t_overrun": 2.0, "alpha": 1.0},
                devices=[{"d_max": 3, "mem_capacity_mb": 6000.5, "pool_max_containers": 10}])


def _check(engine, cases, flags=0):
    from gpu_harness import close, run_cases
    from oracle import oracle as orc
    from paper_2507_08954_b200 import _abi
    outs, _ = run_cases(cases, engine, early_exit=True, flags=flags,
                        outputs=_abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_DISPATCH)
    for c, o in zip(cases, outs):
        ref = orc.run_case(c)
        assert o.get("status") == 0, (c["name"], o)
        for k in ("dispatch", "records", "exec"):
            assert o[k] == ref[k], (c["name"], k)
        assert set(o["per_function"]) == set(ref["per_function"])
        for fn, r in ref["per_function"].items():
            g = o["per_function"][fn]
            assert g["count"] == r["count"]
            for k in ("mean_latency_s", "var_latency_s", "cold_hit_pct"):
                assert close(g[k], r[k]), (c["name"], fn, k)
        for k, v in ref["summary"].items():
            assert close(o["summary"][k], v), (c["name"], k)


def test_long_trace_leaves_u16_classes(engine):
    """65535+ arrivals: MQFQ and FCFS on one device run the i32 classes."""
    cases = [_long_case("mqfq"), _long_case("fcfs")]
    from oracle.oracle import case_inputs
    assert len(case_inputs(cases[0])[0]) >= 65535
    _check(engine, cases)


@pytest.mark.parametrize("build", ["warp", "cta"])
def test_non_integral_memory_leaves_fast_classes(engine, build):
    """Non-integral mem_mb: resident_mb is CPython's compensated sum in pool
    order (the serial path), in the warp and the CTA builds."""
    from paper_2507_08954_b200 import _abi
    cases = [_frac_case(p, i) for p in ("mqfq", "fcfs", "batch", "sjf") for i in range(3)]
    _check(engine, cases, flags=_abi.FLAG_CTA if build == "cta" else 0)


def test_mixed_integral_batch(engine):
    """Integral and non-integral tables in one batch: each simulation is
    routed on its own table."""
    from paper_2507_08954_b200 import _abi  # noqa: F401
    cases = [_frac_case("mqfq", 0), _long_case("mqfq"), _frac_case("fcfs", 1)]
    cases[1] = dict(cases[1], trace={"gen": [4, 1.2, 3.0, 300.0, 9], "names": ["a", "b", "c", "d"]})
    _check(engine, cases)
