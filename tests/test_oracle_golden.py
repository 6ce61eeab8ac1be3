"""Pin the C oracle (oracle/gfq_oracle.c) against the reference's own outputs.

tests/golden/reference_golden.json holds sha256 fingerprints of the
UNMODIFIED reference's dispatch trace, records, exec/util/backlog audit,
event stream, eviction log and per-function stats for 1560 cases
(tests/golden/make_golden.py).  Every case must match bit-for-bit before
the oracle may serve as the GPU engine's parity checker.
"""

from __future__ import annotations

import pytest

from cases import all_cases, extra_cases
from golden_check import golden, mismatches

from oracle import oracle

CASES = all_cases()
FAMILIES = sorted({c["name"].split("/")[0] for c in CASES})


@pytest.mark.parametrize("family", FAMILIES)
def test_oracle_matches_reference(family):
    gold = golden()
    bad = {}
    n = 0
    for case in CASES:
        if case["name"].split("/")[0] != family:
            continue
        out = oracle.run_case(case, want_events=True)
        m = mismatches(out, gold[case["name"]])
        n += 1
        if m:
            bad[case["name"]] = m
    assert n > 0
    assert not bad, f"{len(bad)}/{n} cases differ: {dict(list(bad.items())[:5])}"


@pytest.mark.parametrize("family", ["c1", "c4x"])
def test_oracle_matches_reference_extra(family):
    """C1's 10-function variant under every policy, and C4 at its full 4096
    flows (short traces plus two of the bench's own 1800 s simulations)."""
    gold = golden()
    cases = [c for c in extra_cases() if c["name"].split("/")[0] == family]
    bad = {}
    for case in cases:
        m = mismatches(oracle.run_case(case, want_events=True), gold[case["name"]])
        if m:
            bad[case["name"]] = m
    assert cases and not bad, bad
