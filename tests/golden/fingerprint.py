"""Canonical row serialisation + sha256 fingerprints (SURVEY App. B format):
one line per row, '\\n'-terminated, floats as float.hex(), other fields str().
"""

from __future__ import annotations

import hashlib


def _field(x) -> str:
    if isinstance(x, float):
        return x.hex()
    if isinstance(x, bool):
        return "1" if x else "0"
    if x is None:
        return "None"
    return str(x)


def rows_text(rows) -> str:
    return "".join(",".join(_field(x) for x in row) + "\n" for row in rows)


def fp(rows) -> str:
    return hashlib.sha256(rows_text(rows).encode()).hexdigest()[:16]


def hexf(x: float) -> str:
    return float(x).hex()


def per_function_rows(pf: dict):
    return [(fn, float(v["mean_latency_s"]), float(v["var_latency_s"]), int(v["count"]),
             float(v["cold_hit_pct"])) for fn, v in sorted(pf.items())]
