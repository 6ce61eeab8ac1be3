"""Policy plugin surface (gpufairq.policies, policies.py:18-77,276-289).

A ``Policy`` here is the configuration a simulation runs under: its kind
(mqfq / fcfs / batch / sjf / fcfs_naive), the profiles and the
``SchedulerConfig``.  The dispatch rules of every kind execute in the
simulation kernel (policy = a per-simulation parameter), so the reference's
per-event methods are not exposed; after a run the policy object carries
the run's ``dispatch_log`` exactly like the reference's.
"""

from __future__ import annotations

from enum import Enum

from .core import FunctionProfile
from .mqfq import DispatchAudit, SchedulerConfig


class PolicyKind(str, Enum):
    MQFQ = "mqfq"
    FCFS = "fcfs"
    BATCH = "batch"
    SJF = "sjf"
    FCFS_NAIVE = "fcfs_naive"

    @property
    def pool_disabled(self) -> bool:
        # the naive baseline runs with the container pool off (cli.py:36)
        return self is PolicyKind.FCFS_NAIVE

    @property
    def code(self) -> int:
        """include/gfq.h GFQ_POLICY_* value."""
        return _CODES[self]


_CODES = {PolicyKind.MQFQ: 0, PolicyKind.FCFS: 1, PolicyKind.BATCH: 2,
          PolicyKind.SJF: 3, PolicyKind.FCFS_NAIVE: 4}


class Policy:
    """Policy configuration + the dispatch log of the last run."""

    def __init__(self, kind: PolicyKind, profiles: dict[str, FunctionProfile],
                 cfg: SchedulerConfig):
        self.kind = kind.value
        self.policy_kind = kind
        self.profiles = profiles
        self.cfg = cfg
        self.dispatch_log: list[DispatchAudit] = []


def make_policy(kind: PolicyKind | str, profiles: dict[str, FunctionProfile],
                cfg: SchedulerConfig) -> Policy:
    """Same signature and errors as policies.py:276-289."""
    kind = PolicyKind(kind)
    return Policy(kind, profiles, cfg)
