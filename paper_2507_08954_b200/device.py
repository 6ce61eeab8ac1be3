"""Device configuration API (gpufairq.device, device.py:22-48,300-341).

The device model itself — token caps, utilization headroom, LRU memory
admission with swap-to-host, the kept-alive container pool and its cap,
interference, the utilization monitor and dynamic D, sticky multi-GPU
assignment — runs inside the simulation kernel
(paper_2507_08954_b200/csrc/gfq_engine.cu).  On the host, ``DeviceSet`` is
the same duck-typed container the reference's ``run_simulation`` accepts;
the engine reads each member's ``cfg``.
"""

from __future__ import annotations

from dataclasses import dataclass

from .core import StartState


@dataclass
class DeviceConfig:
    """Same fields, defaults and validation as device.py:22-48."""

    mem_capacity_mb: float = 16384.0
    d_max: int = 2
    util_threshold: float = 0.90
    pcie_mb_per_s: float = 12000.0
    interference_beta: float = 0.10
    monitor_period_s: float = 0.2
    util_window_s: float = 1.0
    pool_max_containers: int = 32
    pool_enabled: bool = True
    dynamic_d: bool = False
    prefetch_overlap_s: float = 0.0

    def __post_init__(self) -> None:
        if not 0 < self.util_threshold <= 1:
            raise ValueError("util_threshold must be in (0, 1]")
        if self.d_max < 1:
            raise ValueError("d_max must be >= 1")
        for name in ("mem_capacity_mb", "pcie_mb_per_s", "monitor_period_s",
                     "util_window_s"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be > 0")
        if self.pool_max_containers < 1:
            raise ValueError("pool_max_containers must be >= 1")
        if self.interference_beta < 0:
            raise ValueError("interference_beta must be >= 0")


@dataclass
class DToken:
    """Concurrency token (device.py:64-68); returned in DispatchDecision."""

    device: int
    holder: int
    start_state: StartState


class Device:
    """Host view of one modeled GPU: its index, config and eviction log
    (device.py:92; run_simulation / Simulation append each run's rows).  Its
    other mutable state (pool, running set, util samples) exists only in the
    kernel."""

    def __init__(self, index: int, cfg: DeviceConfig):
        self.index = index
        self.cfg = cfg
        self.eviction_log: list[tuple[float, str]] = []


class DeviceSet:
    """Ordered set of modeled GPUs (device.py:300-318)."""

    def __init__(self, configs: list[DeviceConfig]):
        if not configs:
            raise ValueError("at least one device required")
        self.devices = [Device(i, cfg) for i, cfg in enumerate(configs)]

    def __iter__(self):
        return iter(self.devices)

    def __len__(self) -> int:
        return len(self.devices)

    def __getitem__(self, i: int) -> Device:
        return self.devices[i]

    def configs(self) -> list[DeviceConfig]:
        return [d.cfg for d in self.devices]
