"""GPU parity on the round-2 reference goldens (tests/golden/
reference_golden_extra.json, made by make_golden.py --extra from the
UNMODIFIED reference):

* c1  -- BASELINE C1's 10-function variant of configs/default.cfg (rate
  3.197988, 600 s, seed 1, 1,875 arrivals) under every policy;
* c4x -- BASELINE C4 at its full 4096 flows: short traces (60 / 300 s) and
  two of the bench's own 1800 s simulations (seeds 1 and 2).

Each family runs as its own batch (the 4096-flow layout would change the
build of a mixed batch), in every build that can run it: the generic
all-outputs build (event stream, audit, eviction log), the specialised
fast builds, and for c4x the CTA-per-simulation and the warp
flows-in-global builds.
"""

from __future__ import annotations

import pytest

from cases import extra_cases
from golden_check import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine():
    from paper_2507_08954_b200.engine import Engine
    e = Engine(0)
    yield e
    e.close()


def _family(name):
    return [c for c in extra_cases() if c["name"].split("/")[0] == name]


def _bad(cases, outs, keys=None):
    from gpu_harness import compare_to_golden
    gold = golden()
    return {c["name"]: m for c, o in zip(cases, outs)
            if (m := compare_to_golden(o, gold[c["name"]], **({"exact_keys": keys} if keys else {})))}


@pytest.mark.parametrize("family", ["c1", "c4x"])
@pytest.mark.parametrize("build", ["auto", "warp", "cta"])
def test_all_outputs(engine, family, build):
    """Dispatch rows, records, exec / util / backlog audit, event stream and
    eviction log bit-exact; statistics within 1e-9."""
    from gpu_harness import run_cases
    from paper_2507_08954_b200 import _abi
    flags = {"auto": 0, "warp": _abi.FLAG_WARP, "cta": _abi.FLAG_CTA}[build]
    cases = _family(family)
    outs, _ = run_cases(cases, engine, early_exit=False, event_log_cap=1 << 17,
                        audit_util_cap=1 << 16, flags=flags)
    bad = _bad(cases, outs)
    assert cases and not bad, bad


@pytest.mark.parametrize("family", ["c1", "c4x"])
@pytest.mark.parametrize("build", ["auto", "warp", "cta"])
def test_fast_builds(engine, family, build):
    """The bench's specialised builds (stats / records / dispatch outputs,
    early exit): MQFQ-Sticky and FCFS on one device with the device state in
    registers (warp and CTA), Batch / SJF / fcfs_naive in their classes."""
    from gpu_harness import run_cases
    from paper_2507_08954_b200 import _abi
    flags = {"auto": 0, "warp": _abi.FLAG_WARP, "cta": _abi.FLAG_CTA}[build]
    cases = _family(family)
    outs, _ = run_cases(cases, engine, early_exit=True, flags=flags,
                        outputs=_abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_DISPATCH)
    bad = _bad(cases, outs, keys=("dispatch", "records", "exec"))
    assert cases and not bad, bad


def test_eviction_log_nonempty():
    """The c4x goldens do exercise the eviction log (LRU admission victims and
    keep-alive swap-outs), so its fingerprint check above is not vacuous."""
    from fingerprint import fp
    empty = fp([])
    gold = golden()
    assert sum(gold[c["name"]]["fp"]["evictions"] != empty for c in _family("c4x")) >= 4
