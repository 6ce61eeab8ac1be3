"""Domain types of the reference API (gpufairq.core, core.py:1-204).

These are host-side value types only: the per-flow queue state machine that
the reference keeps in ``FlowQueue`` (core.py:96-152) lives on the GPU in
this engine (paper_2507_08954_b200/csrc/gfq_engine.cu), laid out as
per-simulation structure-of-arrays in shared memory.  Names, fields and
validation messages match the reference so reference callers can switch
imports.
"""

from __future__ import annotations

import csv
import itertools
from dataclasses import dataclass, field
from enum import Enum


class StartState(str, Enum):
    """Container thermal state at invocation start (core.py:16-21)."""

    GPU_WARM = "gpu_warm"
    HOST_WARM = "host_warm"
    COLD = "cold"


# engine encoding (include/gfq.h GFQ_GPU_WARM..GFQ_COLD) -> enum
STATE_BY_CODE = (StartState.GPU_WARM, StartState.HOST_WARM, StartState.COLD)


class QueueState(str, Enum):
    ACTIVE = "active"
    THROTTLED = "throttled"
    INACTIVE = "inactive"


@dataclass
class FunctionProfile:
    """Static per-function model; same validation as core.py:41-51."""

    name: str
    warm_exec_s: float
    cold_exec_s: float
    mem_mb: float
    compute_share: float = 0.38
    weight: float = 1.0

    def __post_init__(self) -> None:
        checks = (
            (self.warm_exec_s <= 0, "warm_exec_s must be > 0"),
            (self.cold_exec_s < self.warm_exec_s, "cold_exec_s must be >= warm_exec_s"),
            (self.mem_mb <= 0, "mem_mb must be > 0"),
            (not 0 < self.compute_share <= 1, "compute_share must be in (0, 1]"),
            (self.weight <= 0, "weight must be > 0"),
        )
        for bad, msg in checks:
            if bad:
                raise ValueError(f"{self.name}: {msg}")


_uids = itertools.count()


@dataclass
class Invocation:
    """One request (core.py:57-73).  The engine identifies invocations by
    trace position; ``uid`` keeps the reference's process-wide counter."""

    function: str
    arrival_s: float
    start_tag: float = 0.0
    dispatch_s: float | None = None
    complete_s: float | None = None
    start_state: StartState | None = None
    uid: int = field(default=-1)

    def __post_init__(self) -> None:
        if self.uid < 0:
            self.uid = next(_uids)


@dataclass
class RunningMean:
    """All-history running mean, ``mean += (x - mean) / count`` (core.py:76-87)."""

    count: int = 0
    mean: float = 0.0

    def record(self, x: float) -> None:
        if x < 0:
            raise ValueError(f"negative sample: {x}")
        self.count += 1
        self.mean += (x - self.mean) / self.count


def record_sample(est: RunningMean, x: float) -> RunningMean:
    est.record(x)
    return est


PROFILE_COLUMNS = ["name", "warm_s", "cold_s", "mem_mb", "compute_share", "weight"]


def _strict_float(text: str) -> float:
    text = text.strip()
    if "," in text:
        raise ValueError(f"decimal comma not allowed: {text!r}")
    return float(text)


def load_profiles(path: str) -> dict[str, FunctionProfile]:
    """Strict profile CSV reader (core.py:158-187)."""
    out: dict[str, FunctionProfile] = {}
    with open(path, newline="", encoding="utf-8") as fh:
        rd = csv.reader(fh)
        try:
            header = next(rd)
        except StopIteration:
            raise ValueError(f"{path}: empty profile file, header required") from None
        if header != PROFILE_COLUMNS:
            raise ValueError(f"{path}: bad header {header!r}, expected {PROFILE_COLUMNS!r}")
        for lineno, row in enumerate(rd, start=2):
            if not row:
                continue
            if len(row) != len(PROFILE_COLUMNS):
                raise ValueError(f"{path}:{lineno}: expected {len(PROFILE_COLUMNS)} columns")
            name = row[0].strip()
            try:
                vals = [_strict_float(v) for v in row[1:]]
            except ValueError as exc:
                raise ValueError(f"{path}:{lineno}: {exc}") from None
            if name in out:
                raise ValueError(f"{path}:{lineno}: duplicate function {name!r}")
            try:
                out[name] = FunctionProfile(name, *vals)
            except ValueError as exc:
                raise ValueError(f"{path}:{lineno}: {exc}") from None
    return out


def save_profiles(profiles: dict[str, FunctionProfile], path: str) -> None:
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(PROFILE_COLUMNS)
        for p in profiles.values():
            w.writerow([p.name, p.warm_exec_s, p.cold_exec_s, p.mem_mb,
                        p.compute_share, p.weight])
