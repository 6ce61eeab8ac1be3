"""Batched sweeps: the BASELINE.json configurations as engine batches.

The reference runs sweeps serially, one ``run_experiment`` per grid point
(cli.py:131-163 ``cmd_sweep``; cli.py:67-116 ``cmd_compare``).  Here a sweep
is one upload of its distinct traces and flow tables plus one
``gfq_sim`` parameter block per grid point, run in a single kernel launch.

* ``c3`` — BASELINE C3 (configs[2]): F=100 default profiles, Zipf s=1.5,
  2.382870 rps (rho = 1), 600 s; T in {0,1,2,5,10,20,50,100} x alpha in
  {0,.5,1,1.5,2,3,4,8} x D in {1,2,3,4} x 16 seeds = 4096 MQFQ-Sticky sims.
* ``c2`` — BASELINE C2 (configs[1]): F=200, Zipf 1.5, the paper's Table 3
  request rates x seeds x {mqfq, fcfs, batch}, 600 s.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _abi
from .device import DeviceConfig
from .engine import sim_params
from .mqfq import SchedulerConfig
from .pack import FlowTable, PackedTrace, flow_table, pack_trace
from .workload import default_profiles, gen_zipf

C3_T = [0.0, 1.0, 2.0, 5.0, 10.0, 20.0, 50.0, 100.0]
C3_ALPHA = [0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 8.0]
C3_D = [1, 2, 3, 4]
C3_RATE = 2.382870
TABLE3_RPS = [1.12, 1.69, 1.94, 4.26, 2.69, 2.57, 2.55, 1.79, 1.12]


@dataclass
class Workload:
    name: str
    traces: list[PackedTrace]
    tabs: list[FlowTable]
    dcfgs: list
    sims: list
    groups: int
    hist_rows: int
    describe: dict

    @property
    def arrivals(self) -> int:
        return int(sum(self.traces[s.trace].n for s in self.sims))

    def upload(self, eng) -> None:
        eng.upload_traces(self.traces)
        eng.upload_flowtabs(self.tabs)
        eng.upload_device_cfgs(self.dcfgs)

    def sims_array(self):
        arr = (_abi.Sim * len(self.sims))(*self.sims)
        return arr


def gen_traces(n_fn, s, rates_seeds, duration, profiles=None, engine=None) -> list[PackedTrace]:
    """gen_zipf + pack_trace for each (rate, seed): on the GPU when an engine
    is given (gfq_generate_traces, bit-identical), else on the host."""
    profiles = profiles or default_profiles(n_fn)
    if engine is not None:
        return engine.generate_traces([(n_fn, s, rate, duration, seed, list(profiles))
                                       for rate, seed in rates_seeds])
    return [pack_trace(gen_zipf(n_fn, s, rate, duration, seed, names=list(profiles)).entries,
                       profiles) for rate, seed in rates_seeds]


def _traces(n_fn, s, rates_seeds, duration, engine=None):
    profiles = default_profiles(n_fn)
    order = {nm: i for i, nm in enumerate(profiles)}
    traces, tabs = [], []
    for pt in gen_traces(n_fn, s, rates_seeds, duration, profiles, engine):
        traces.append(pt)
        # histogram row = the function's identity (profile index), not its
        # per-trace rank, so rows line up across traces and GPUs
        tabs.append(flow_table(pt.names, profiles, None, [order[nm] for nm in pt.names]))
    return traces, tabs


def c3(seed_base: int = 1, n_seeds: int = 16, duration: float = 600.0, engine=None) -> Workload:
    seeds = list(range(seed_base, seed_base + n_seeds))
    traces, tabs = _traces(100, 1.5, [(C3_RATE, s) for s in seeds], duration, engine)
    dcfgs = [DeviceConfig(d_max=d) for d in C3_D]
    sims = []
    for ti, t in enumerate(C3_T):
        for ai, a in enumerate(C3_ALPHA):
            cfg = SchedulerConfig(t_overrun=t, alpha=a)
            for di, d in enumerate(C3_D):
                for si in range(n_seeds):
                    sims.append(sim_params("mqfq", cfg, 1, trace=si, flowtab=si, device_cfg=di,
                                           group=ti * len(C3_ALPHA) + ai))
    return Workload("c3", traces, tabs, dcfgs, sims, groups=len(C3_T) * len(C3_ALPHA),
                    hist_rows=100,
                    describe={"workload": "C3 MQFQ-Sticky sweep: T x alpha x D x seeds",
                              "functions": 100, "zipf_s": 1.5, "rate_rps": C3_RATE,
                              "duration_s": duration, "seeds": [seeds[0], seeds[-1]],
                              "grid": "8 T x 8 alpha x 4 D", "sims": len(sims)})


def c2(seed_base: int = 1, n_seeds: int = 456, duration: float = 600.0,
       policies=("mqfq", "fcfs", "batch"), engine=None) -> Workload:
    rs = [(r, s) for s in range(seed_base, seed_base + n_seeds) for r in TABLE3_RPS]
    traces, tabs = _traces(200, 1.5, rs, duration, engine)
    dcfgs = [DeviceConfig()]
    sims = []
    cfg = SchedulerConfig()
    for ti in range(len(traces)):
        for pi, pol in enumerate(policies):
            sims.append(sim_params(pol, cfg, 1, trace=ti, flowtab=ti, device_cfg=0, group=pi))
    return Workload("c2", traces, tabs, dcfgs, sims, groups=len(policies), hist_rows=200,
                    describe={"workload": "C2 Azure-shaped: Table-3 rates x seeds x policies",
                              "functions": 200, "zipf_s": 1.5, "duration_s": duration,
                              "traces": len(traces), "policies": list(policies),
                              "sims": len(sims)})


C4_MEM_MB = [256.0, 512.0, 1024.0, 1500.0, 3000.0]


def c4(seed_base: int = 1, n_seeds: int = 4, duration: float = 1800.0, rate: float = 2.0,
       policies=("mqfq", "fcfs"), engine=None) -> Workload:
    """BASELINE C4 (configs[3]): 4096 functions per simulation (Zipf 0.5, ~2.1k
    touched in 1800 s at 2 rps), heterogeneous memory (mem_mb by rank mod 5),
    16 GB device, D=4, container pool 32 or 256 -> cold starts, host-warm
    prefetch and LRU swap all exercised.  A simulation's workspace (~220 KB)
    takes a whole SM's shared memory, so these run the CTA-per-simulation
    build (k_sim_cta, 512 threads, scans split over 16 warps)."""
    from .core import FunctionProfile
    n_fn = 4096
    base = default_profiles(n_fn)
    profiles = {nm: FunctionProfile(nm, p.warm_exec_s, p.cold_exec_s, C4_MEM_MB[i % 5], 0.38, 1.0)
                for i, (nm, p) in enumerate(base.items())}
    order = {nm: i for i, nm in enumerate(profiles)}
    traces, tabs = [], []
    seeds = list(range(seed_base, seed_base + n_seeds))
    for pt in gen_traces(n_fn, 0.5, [(rate, sd) for sd in seeds], duration, profiles, engine):
        traces.append(pt)
        tabs.append(flow_table(pt.names, profiles, None, [order[nm] for nm in pt.names]))
    dcfgs = [DeviceConfig(d_max=4, pool_max_containers=pm) for pm in (32, 256)]
    sims = []
    cfg = SchedulerConfig()
    for pi, pol in enumerate(policies):
        for di in range(2):
            for si in range(n_seeds):
                sims.append(sim_params(pol, cfg, 1, trace=si, flowtab=si, device_cfg=di,
                                       group=pi * 2 + di))
    return Workload("c4", traces, tabs, dcfgs, sims, groups=2 * len(policies), hist_rows=n_fn,
                    describe={"workload": "C4 large-flow stress: 4096 functions per sim",
                              "functions": n_fn, "zipf_s": 0.5, "rate_rps": rate,
                              "duration_s": duration, "mem_mb": C4_MEM_MB, "pool": [32, 256],
                              "d_max": 4, "policies": list(policies), "sims": len(sims)})


C5_T = [0.0, 2.0, 10.0, 50.0]
C5_ALPHA = [0.0, 1.0, 2.0, 8.0]
C5_D = [1, 2, 3, 4]
C5_MEM_MB = [256.0, 512.0, 1024.0, 1500.0, 3000.0, 6000.0]
C5_SHARE = [0.2, 0.38, 0.5]
C5_RHO = [0.7, 0.9, 1.0, 1.1]


def c5(seed_base: int = 1, n_traces: int = 1563, duration: float = 600.0, engine=None) -> Workload:
    """BASELINE C5 (configs[4]) per GPU: the 1M-simulation sensitivity sweep
    is 8 x ~125k.  Every trace (F=100 functions, heterogeneous memory /
    compute share / weight by rank, load rho in {0.7,0.9,1.0,1.1}) runs 80
    configurations: MQFQ-Sticky over T x alpha x D (64) and FCFS / Batch / SJF /
    fcfs_naive over D (16)."""
    from .core import FunctionProfile
    n_fn = 100
    base = default_profiles(n_fn)
    profiles = {nm: FunctionProfile(nm, p.warm_exec_s, p.cold_exec_s, C5_MEM_MB[i % 6],
                                    C5_SHARE[i % 3], 2.0 if i % 7 == 0 else 1.0)
                for i, (nm, p) in enumerate(base.items())}
    order = {nm: i for i, nm in enumerate(profiles)}
    shares = [(k + 1) ** -1.5 for k in range(n_fn)]
    tot = sum(shares)
    mean_exec = sum(sh / tot * p.warm_exec_s for sh, p in zip(shares, profiles.values()))
    traces, tabs = [], []
    rs = [(C5_RHO[j % 4] * 1.8 / mean_exec, seed_base + j) for j in range(n_traces)]
    for pt in gen_traces(n_fn, 1.5, rs, duration, profiles, engine):
        traces.append(pt)
        tabs.append(flow_table(pt.names, profiles, None, [order[nm] for nm in pt.names]))
    dcfgs = [DeviceConfig(d_max=d) for d in C5_D] + \
            [DeviceConfig(d_max=d, pool_enabled=False) for d in C5_D]
    sims = []
    for ti in range(n_traces):
        for t in C5_T:
            for a in C5_ALPHA:
                for di in range(4):
                    sims.append(sim_params("mqfq", SchedulerConfig(t_overrun=t, alpha=a), 1,
                                           trace=ti, flowtab=ti, device_cfg=di, group=0))
        for gi, pol in enumerate(("fcfs", "batch", "sjf", "fcfs_naive")):
            for di in range(4):
                sims.append(sim_params(pol, SchedulerConfig(), 1, trace=ti, flowtab=ti,
                                       device_cfg=di + (4 if pol == "fcfs_naive" else 0),
                                       group=1 + gi))
    return Workload("c5", traces, tabs, dcfgs, sims, groups=5, hist_rows=n_fn,
                    describe={"workload": "C5 sensitivity sweep, per-GPU shard of 1M sims",
                              "functions": n_fn, "traces": n_traces, "rho": C5_RHO,
                              "policies": ["mqfq", "fcfs", "batch", "sjf", "fcfs_naive"],
                              "mem_mb": C5_MEM_MB, "compute_share": C5_SHARE,
                              "duration_s": duration, "sims": len(sims)})


def c1(variant: str = "default", engine=None) -> Workload:
    """BASELINE C1 (configs[0]): the reference's default run, one simulation.
    ``default`` is configs/default.cfg verbatim (24 functions, Zipf 1.5,
    2.69 rps, 600 s, seed 1; MQFQ-Sticky T=10, alpha=2; one 16 GB device,
    D=2, pool 32: 1,586 arrivals); ``f10`` its 10-function variant (3.197988
    rps -> 1,875 arrivals)."""
    n_fn, rate = {"default": (24, 2.69), "f10": (10, 3.197988)}[variant]
    traces, tabs = _traces(n_fn, 1.5, [(rate, 1)], 600.0, engine)
    dcfgs = [DeviceConfig(mem_capacity_mb=16384.0, d_max=2, pool_max_containers=32)]
    sims = [sim_params("mqfq", SchedulerConfig(t_overrun=10.0, d_max=2, alpha=2.0), 1,
                       trace=0, flowtab=0, device_cfg=0, group=0)]
    return Workload("c1", traces, tabs, dcfgs, sims, groups=1, hist_rows=n_fn,
                    describe={"workload": f"C1 reference default run ({variant}): one "
                                          "MQFQ-Sticky simulation, per-simulation latency",
                              "functions": n_fn, "zipf_s": 1.5, "rate_rps": rate,
                              "duration_s": 600.0, "seed": 1, "d_max": 2, "pool": 32,
                              "sims": 1})


def sim_costs(w: Workload) -> list[float]:
    """A-priori cost of each simulation for partitioning (SURVEY §8(e):
    N_arrivals x F_touched), scaled like the engine's LPT estimate by the
    policy and the device concurrency (gfq_prepare's work order)."""
    out = []
    for s in w.sims:
        tr = w.traces[s.trace]
        d = sum(w.dcfgs[s.device_cfg + k].d_max for k in range(s.n_devices))
        out.append(tr.n * (1.0 + tr.n_flows / 32.0) * (2.0 if s.policy == _abi.POLICY_MQFQ else 1.0)
                   * (1.0 + 1.0 / max(d, 1)))
    return out


def restrict(w: Workload, idx) -> Workload:
    """The same workload (traces, tables, configs) with only sims ``idx``."""
    idx = list(idx)
    return Workload(w.name, w.traces, w.tabs, w.dcfgs, [w.sims[i] for i in idx], w.groups,
                    w.hist_rows, dict(w.describe, sims=len(idx)))


def build(name: str, rank: int = 0, engine=None, **kw) -> Workload:
    """Weak-scaling shard for `rank`: a disjoint block of seeds per GPU.
    With an engine the traces are generated on its GPU."""
    if name in ("c1", "c1f10"):
        return c1("f10" if name == "c1f10" else "default", engine=engine)
    if name == "c3":
        n = kw.get("n_seeds", 16)
        return c3(seed_base=1 + rank * n, n_seeds=n, engine=engine)
    if name == "c2":
        n = kw.get("n_seeds", 456)
        return c2(seed_base=1 + rank * n, n_seeds=n, engine=engine)
    if name == "c4":
        n = kw.get("n_seeds", 37)          # 37 seeds x 2 pools x 2 policies = 148 sims, 1 per SM
        return c4(seed_base=1 + rank * n, n_seeds=n, engine=engine)
    if name == "c5":
        n = kw.get("n_seeds", 1563)
        return c5(seed_base=1 + rank * n, n_traces=n, engine=engine)
    raise ValueError(f"unknown workload {name}")


HIST_BINS = 64
HIST_LO_S = 1e-2
HIST_HI_S = 1e5
