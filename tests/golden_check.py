"""Compare reference-shaped outputs with a golden case (tests/golden/)."""

from __future__ import annotations

import json
import os

from fingerprint import fp, hexf, per_function_rows

_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GOLDEN = os.path.join(_DIR, "reference_golden.json")
# round-2 families (cases.extra_cases: C1's 10-function variant, C4 at 4096 flows)
GOLDEN_EXTRA = os.path.join(_DIR, "reference_golden_extra.json")
_cache = None


def golden() -> dict:
    global _cache
    if _cache is None:
        _cache = {}
        for path in (GOLDEN, GOLDEN_EXTRA):
            with open(path) as fh:
                _cache.update({c["name"]: c for c in json.load(fh)["cases"]})
    return _cache


def mismatches(out: dict, gold: dict, keys=None) -> list[str]:
    """Return the list of fingerprints / values that differ (empty = parity)."""
    bad = []
    if "transcript" in out:
        if fp(out["transcript"]) != gold["fp"]["transcript"]:
            bad.append("transcript")
        return bad
    want = keys or ("dispatch", "records", "exec", "util", "backlog", "evictions", "events")
    for k in want:
        if k in out and fp(out[k]) != gold["fp"][k]:
            bad.append(k)
    if fp(per_function_rows(out["per_function"])) != gold["fp"]["per_function"]:
        bad.append("per_function")
    for k, v in gold["summary"].items():
        if hexf(out["summary"][k]) != v:
            bad.append(f"summary.{k}")
    return bad
