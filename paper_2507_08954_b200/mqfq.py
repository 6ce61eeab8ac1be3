"""Scheduler configuration and audit types (gpufairq.mqfq, mqfq.py:16-69).

The MQFQ-Sticky state machine (mqfq.py:72-247: global VT, throttle window,
anticipatory keep-alive, sticky candidate order, token dispatch) is the
warp-per-simulation loop of paper_2507_08954_b200/csrc/gfq_engine.cu.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .core import Invocation


@dataclass
class SchedulerConfig:
    """Same fields, defaults and validation as mqfq.py:16-32."""

    t_overrun: float = 10.0
    d_max: int = 2
    alpha: float = 2.0
    dynamic_d: bool = False
    default_ttl_s: float = 2.0
    weights: dict[str, float] = field(default_factory=dict)
    tau_includes_overheads: bool = False

    def __post_init__(self) -> None:
        if self.t_overrun < 0:
            raise ValueError("t_overrun must be >= 0")
        if self.d_max < 1:
            raise ValueError("d_max must be >= 1")
        if self.alpha < 0:
            raise ValueError("alpha must be >= 0")


@dataclass
class DispatchDecision:
    invocation: Invocation
    device: int
    token: object


@dataclass
class DispatchAudit:
    """One row per successful dispatch (mqfq.py:42-53)."""

    now: float
    function: str
    vt_before: float
    global_vt: float
    queue_len: int
    in_flight: int
    device: int
    start_state: str


def fairness_bound(d: int, t_overrun: float, tau_i: float, tau_j: float,
                   w_i: float = 1.0, w_j: float = 1.0) -> float:
    """Eq. 1: (D - 1) * (2T + tau_i/w_i - tau_j/w_j) (mqfq.py:56-69)."""
    if d < 1:
        raise ValueError("d must be >= 1")
    if w_i <= 0 or w_j <= 0:
        raise ValueError("weights must be positive")
    return (d - 1) * (2.0 * t_overrun + tau_i / w_i - tau_j / w_j)
