"""Experiment configuration files (gpufairq.config, config.py:1-260).

Same INI schema, defaults, strict validation and error messages as the
reference's ``load_config``: unknown sections / keys, conflicting
``d_max`` / ``dynamic_d`` values given in two sections, and incomplete or
ambiguous workload specs raise ``ConfigError`` (a ``ValueError``; the CLI
maps it to exit code 2, cli.py:260-267).  The parsed ``ExperimentConfig``
feeds the batched experiment driver (``paper_2507_08954_b200.cli``), which
runs every simulation of a compare / sweep in one engine batch.
"""

from __future__ import annotations

import configparser
import os
from dataclasses import dataclass, field

from .core import FunctionProfile, load_profiles
from .device import DeviceConfig
from .mqfq import SchedulerConfig
from .policies import PolicyKind
from .workload import (DEFAULT_COMPUTE_SHARE, DEFAULT_MEM_MB, Trace, default_profiles, gen_zipf,
                       load_trace)


class ConfigError(ValueError):
    pass


@dataclass
class ExperimentConfig:
    """Field names and defaults as config.py:38-76."""

    policy: PolicyKind = PolicyKind.MQFQ
    t_overrun: float = 10.0
    d_max: int = 2
    alpha: float = 2.0
    dynamic_d: bool = False
    default_ttl_s: float = 2.0
    tau_includes_overheads: bool = False

    device_count: int = 1
    mem_capacity_mb: float = 16384.0
    util_threshold: float = 0.90
    pcie_mb_per_s: float = 12000.0
    interference_beta: float = 0.10
    monitor_period_s: float = 0.2
    util_window_s: float = 1.0
    pool_max_containers: int = 32
    pool_enabled: bool = True
    prefetch_overlap_s: float = 0.0

    profiles_path: str | None = None
    trace_path: str | None = None
    n_functions: int | None = None
    zipf_s: float | None = None
    rate_rps: float | None = None
    duration_s: float | None = None
    copies: int | None = None
    workload_mem_mb: float = DEFAULT_MEM_MB
    workload_compute_share: float = DEFAULT_COMPUTE_SHARE

    seed: int = 1
    out_dir: str | None = None
    base_dir: str = "."
    echo: dict = field(default_factory=dict)

    def scheduler_config(self) -> SchedulerConfig:
        return SchedulerConfig(t_overrun=self.t_overrun, d_max=self.d_max, alpha=self.alpha,
                               dynamic_d=self.dynamic_d, default_ttl_s=self.default_ttl_s,
                               tau_includes_overheads=self.tau_includes_overheads)

    def device_configs(self, pool_enabled: bool | None = None) -> list[DeviceConfig]:
        """``device_count`` identical devices (config.py:84-96)."""
        one = DeviceConfig(mem_capacity_mb=self.mem_capacity_mb, d_max=self.d_max,
                           util_threshold=self.util_threshold, pcie_mb_per_s=self.pcie_mb_per_s,
                           interference_beta=self.interference_beta,
                           monitor_period_s=self.monitor_period_s,
                           util_window_s=self.util_window_s,
                           pool_max_containers=self.pool_max_containers,
                           pool_enabled=self.pool_enabled if pool_enabled is None else pool_enabled,
                           dynamic_d=self.dynamic_d, prefetch_overlap_s=self.prefetch_overlap_s)
        return [one] * self.device_count

    def build_profiles(self) -> dict[str, FunctionProfile]:
        if self.profiles_path:
            return load_profiles(self._resolve(self.profiles_path))
        n = self.n_functions
        if n is None and self.copies:
            n = 8 * self.copies
        if n is None:
            raise ConfigError("workload needs profiles_path or a generator spec")
        return default_profiles(n, mem_mb=self.workload_mem_mb,
                                compute_share=self.workload_compute_share)

    def build_trace(self, profiles: dict[str, FunctionProfile]) -> Trace:
        if self.trace_path:
            return load_trace(self._resolve(self.trace_path), known_names=set(profiles))
        names = list(profiles)
        n = len(names) if self.n_functions is None else self.n_functions
        return gen_zipf(n, self.zipf_s, self.rate_rps, self.duration_s, self.seed,
                        names=names[:n])

    def _resolve(self, path: str) -> str:
        return path if os.path.isabs(path) else os.path.join(self.base_dir, path)


def _parse_bool(text: str, key: str) -> bool:
    v = text.strip().lower()
    if v in ("true", "yes", "on", "1"):
        return True
    if v in ("false", "no", "off", "0"):
        return False
    raise ConfigError(f"bad boolean for {key}: {text!r}")


def _policy(text: str) -> PolicyKind:
    try:
        return PolicyKind(text.strip())
    except ValueError:
        raise ConfigError(f"unknown policy: {text!r}") from None


def _strip(text: str) -> str:
    return text.strip()


# (section, key) -> (ExperimentConfig attribute, parser).  Parsers that take the
# key name get it as a second argument (booleans name the key in their error).
_KEYS = {
    ("scheduler", "policy"): ("policy", _policy),
    ("scheduler", "t"): ("t_overrun", float),
    ("scheduler", "d_max"): ("d_max", int),
    ("scheduler", "alpha"): ("alpha", float),
    ("scheduler", "dynamic_d"): ("dynamic_d", _parse_bool),
    ("scheduler", "default_ttl_s"): ("default_ttl_s", float),
    ("scheduler", "tau_includes_overheads"): ("tau_includes_overheads", _parse_bool),
    ("device", "count"): ("device_count", int),
    ("device", "mem_mb"): ("mem_capacity_mb", float),
    ("device", "d_max"): ("d_max", int),
    ("device", "util_threshold"): ("util_threshold", float),
    ("device", "pcie_mb_per_s"): ("pcie_mb_per_s", float),
    ("device", "interference_beta"): ("interference_beta", float),
    ("device", "monitor_period_s"): ("monitor_period_s", float),
    ("device", "util_window_s"): ("util_window_s", float),
    ("device", "pool_max_containers"): ("pool_max_containers", int),
    ("device", "pool_enabled"): ("pool_enabled", _parse_bool),
    ("device", "dynamic_d"): ("dynamic_d", _parse_bool),
    ("device", "prefetch_overlap_s"): ("prefetch_overlap_s", float),
    ("workload", "profiles_path"): ("profiles_path", _strip),
    ("workload", "trace_path"): ("trace_path", _strip),
    ("workload", "n_functions"): ("n_functions", int),
    ("workload", "zipf_s"): ("zipf_s", float),
    ("workload", "rate_rps"): ("rate_rps", float),
    ("workload", "duration_s"): ("duration_s", float),
    ("workload", "copies"): ("copies", int),
    ("workload", "mem_mb"): ("workload_mem_mb", float),
    ("workload", "compute_share"): ("workload_compute_share", float),
    ("sim", "seed"): ("seed", int),
    ("output", "dir"): ("out_dir", _strip),
}
_SECTIONS = {s for s, _ in _KEYS}
_GENERATOR = ("n_functions", "zipf_s", "rate_rps", "duration_s", "copies")


def load_config(path: str) -> ExperimentConfig:
    """Parse and validate an experiment file (config.py:126-163)."""
    parser = configparser.ConfigParser()
    try:
        ok = parser.read(path, encoding="utf-8")
    except configparser.Error as exc:
        raise ConfigError(f"malformed config file: {exc}") from None
    if not ok:
        raise ConfigError(f"cannot read config file: {path}")
    cfg = ExperimentConfig(base_dir=os.path.dirname(os.path.abspath(path)))
    echo: dict[str, dict[str, str]] = {}
    d_max_seen: dict[str, str] = {}
    dynamic_seen: dict[str, str] = {}
    for section in parser.sections():
        if section not in _SECTIONS:
            raise ConfigError(f"unknown config section: [{section}]")
        echo[section] = {}
        for key, value in parser.items(section):
            if (section, key) not in _KEYS:
                raise ConfigError(f"unknown config key: {section}.{key}")
            echo[section][key] = value
            attr, conv = _KEYS[(section, key)]
            try:
                parsed = conv(value, key) if conv is _parse_bool else conv(value)
            except ConfigError:
                raise
            except ValueError as exc:
                raise ConfigError(f"bad value for {section}.{key}: {exc}") from None
            setattr(cfg, attr, parsed)
            if key == "d_max":
                d_max_seen[f"{section}.d_max"] = value.strip()
            elif key == "dynamic_d":
                dynamic_seen[f"{section}.dynamic_d"] = str(parsed)
    if len(set(d_max_seen.values())) > 1:
        raise ConfigError(f"conflicting d_max values: {d_max_seen}")
    if len(set(dynamic_seen.values())) > 1:
        raise ConfigError(f"conflicting dynamic_d values: {dynamic_seen}")
    _validate(cfg)
    cfg.echo = echo
    return cfg


def _validate(cfg: ExperimentConfig) -> None:
    """Workload spec completeness, input files, device count (config.py:243-271)."""
    has_trace = cfg.trace_path is not None
    has_gen = any(getattr(cfg, k) is not None for k in _GENERATOR)
    if has_trace and has_gen:
        raise ConfigError("workload: give trace_path or a generator spec, not both")
    if not has_trace and not has_gen:
        raise ConfigError("workload: needs trace_path or a generator spec "
                          f"({', '.join(sorted(_GENERATOR))})")
    if has_gen:
        missing = [k for k in ("zipf_s", "rate_rps", "duration_s") if getattr(cfg, k) is None]
        if cfg.n_functions is None and cfg.copies is None:
            missing.append("n_functions")
        if missing:
            raise ConfigError(f"workload generator spec incomplete, missing: {missing}")
    for attr, what in (("trace_path", "trace"), ("profiles_path", "profiles")):
        rel = getattr(cfg, attr)
        if rel and not os.path.exists(cfg._resolve(rel)):
            raise ConfigError(f"{what} file not found: {cfg._resolve(rel)}")
    if cfg.device_count < 1:
        raise ConfigError("device count must be >= 1")
