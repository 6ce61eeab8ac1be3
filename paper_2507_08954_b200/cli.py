"""Experiment driver on the GPU engine (gpufairq.cli, cli.py:1-300).

Same sub-commands, flags, outputs and exit codes as the reference's CLI
(``run`` / ``compare`` / ``sweep`` / ``generate``; 0 ok, 2 usage or
validation error, 1 runtime / IO failure), but the serial per-experiment
loops of ``cmd_compare`` (cli.py:67-116) and ``cmd_sweep`` (cli.py:131-163)
become ONE engine batch: every policy / sweep value is a ``gfq_sim``
parameter block of the same launch, the distinct traces and flow tables are
uploaded once, and the fairness audit of all of them is one
``gfq_fairness`` call.  Per-experiment directories get the reference's
``invocations.csv`` / ``windows.csv`` / ``summary.json`` and the top level
its ``compare.csv`` / ``sweep.csv`` (p50 / p99 from the sorted completion
latencies, cli.py:119-128), byte-identical to the reference's files except
``var_latency_s`` (last place, see metrics.py).

    python -m paper_2507_08954_b200.cli compare --config default.cfg --policies mqfq,fcfs
"""

from __future__ import annotations

import argparse
import os
import sys
from dataclasses import dataclass, replace

import numpy as np

from . import _abi
from .config import ConfigError, ExperimentConfig, load_config
from ._lib import EngineError
from .engine import BatchResult, default_engine, sim_params
from .metrics import (RunArrays, WindowReport, export, percentile, run_arrays, summarize,
                      windows_from, write_atomic)
from .pack import flow_table, pack_trace
from .policies import PolicyKind
from .workload import gen_zipf, save_trace

SWEEP_PARAMS = ("T", "alpha", "d_max", "pool_max_containers", "rate_rps")
WINDOW_S = 30.0
_RETRY_EVENTS, _RETRY_OUTPUT = 1, 5          # gfq.h GFQ_SIM_EVENT_OVERFLOW / _OUTPUT_OVERFLOW


def default_out_dir() -> str:
    return os.environ.get("GPUFAIRQ_OUT", "out")


@dataclass
class Experiment:
    """One simulation of a batch: its config, output directory, and optionally
    pre-built profiles / trace shared with other experiments (cmd_compare
    materialises one trace for every policy, cli.py:86-89)."""

    cfg: ExperimentConfig
    out_dir: str | None = None
    profiles: dict | None = None
    trace: object | None = None


@dataclass
class Outcome:
    run: RunArrays
    windows: list[WindowReport]
    summary: dict

    @property
    def records(self):
        return self.run.records()


def run_experiments(exps: list[Experiment], device: int = 0, write: bool = True) -> list[Outcome]:
    """run_experiment (cli.py:27-42) for many configs in one engine batch."""
    items = []
    traces, tabs, dcfgs = [], [], []
    trace_ix: dict[int, int] = {}
    tab_ix: dict[tuple, int] = {}
    alive = []      # the id()-keyed objects stay alive, so no id is reused
    for e in exps:
        cfg = e.cfg
        profiles = e.profiles if e.profiles is not None else cfg.build_profiles()
        trace = e.trace if e.trace is not None else cfg.build_trace(profiles)
        sched = cfg.scheduler_config()
        pool = cfg.pool_enabled and not PolicyKind(cfg.policy).pool_disabled
        devs = cfg.device_configs(pool_enabled=pool)
        alive.append((trace, profiles))
        if id(trace) not in trace_ix:
            trace_ix[id(trace)] = len(traces)
            traces.append(pack_trace(trace.entries, profiles))
        ti = trace_ix[id(trace)]
        key = (ti, id(profiles), tuple(sorted(sched.weights.items())))
        if key not in tab_ix:
            tab_ix[key] = len(tabs)
            tabs.append(flow_table(traces[ti].names, profiles, sched.weights))
        sim = sim_params(PolicyKind(cfg.policy).value, sched, len(devs), trace=ti,
                         flowtab=tab_ix[key], device_cfg=len(dcfgs),
                         tau_includes_overheads=cfg.tau_includes_overheads)
        dcfgs.extend(devs)
        items.append((e, sim, traces[ti], sched))
    outcomes: list[Outcome | None] = [None] * len(items)
    eng = default_engine(device)
    todo = list(range(len(items)))
    cap, ev_cap = 1 << 15, 0
    for attempt in range(4):
        if not todo:
            break
        eng.upload_traces(traces)
        eng.upload_flowtabs(tabs)
        eng.upload_device_cfgs(dcfgs)
        sims = [items[k][1] for k in todo]
        eng.prepare(sims, outputs=_abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_AUDIT,
                    early_exit=True, audit_util_cap=cap, audit_backlog_cap=cap,
                    event_capacity=ev_cap)
        eng.launch()
        err = None
        try:
            eng.synchronize()
        except EngineError as exc:
            err = exc
        res = BatchResult(eng)
        st = [int(x) for x in res.status]
        # output-buffer / event-pool overflows are re-run with larger buffers
        # (only those sims); anything else is the engine's RuntimeError
        over = [j for j in range(len(todo)) if st[j] in (_RETRY_OUTPUT, _RETRY_EVENTS)]
        if err is not None and (attempt == 3 or any(x not in (0, _RETRY_OUTPUT, _RETRY_EVENTS)
                                                    for x in st)):
            raise err
        fair = None
        if len(over) < len(todo):
            dmax = np.array([items[k][3].d_max for k in todo], dtype=np.int32)
            rw = np.concatenate([np.ones(len(t)) for t in tabs]) if tabs else np.zeros(0)
            for (ti_, _, w), fi in tab_ix.items():
                if w:
                    wd = dict(w)
                    a = int(sum(len(t) for t in tabs[:fi]))
                    rw[a:a + len(tabs[fi])] = [float(wd.get(nm, 1.0)) for nm in traces[ti_].names]
            fair = eng.fairness(dmax, rw, WINDOW_S)
        for j, k in enumerate(todo):
            if j in over:
                continue
            e, _, pt, _ = items[k]
            run = run_arrays(res, j, pt)
            wins = windows_from(fair, j, WINDOW_S)
            summary = summarize(PolicyKind(e.cfg.policy).value, res, j, pt.names, wins,
                                e.cfg.echo, e.cfg.seed, len(run))
            outcomes[k] = Outcome(run, wins, summary)
        if any(st[j] == _RETRY_OUTPUT for j in over):
            cap *= 8
        if any(st[j] == _RETRY_EVENTS for j in over):
            # grow from the capacity that overflowed (never retry a smaller one)
            ev_cap = 4 * eng.batch_info()["event_capacity"]
        todo = [todo[j] for j in over]
    if write:
        for (e, _, _, _), o in zip(items, outcomes):
            if e.out_dir is not None:
                export(o.run, o.windows, o.summary, e.out_dir)
    return outcomes


def run_experiment(cfg: ExperimentConfig, out_dir: str, profiles=None, trace=None):
    """Drop-in for cli.run_experiment: (records, windows, summary)."""
    o = run_experiments([Experiment(cfg, out_dir, profiles, trace)])[0]
    return o.records, o.windows, o.summary


def _summary_line(summary: dict) -> str:
    return (f"policy={summary['policy']} "
            f"weighted_avg_latency_s={summary['weighted_avg_latency_s']:.3f} "
            f"cold_hit_pct={summary['cold_hit_pct']:.1f} "
            f"bound_violations={summary['bound_violations']}")


def cmd_run(args) -> int:
    cfg = load_config(args.config)
    if args.policy:
        cfg.policy = PolicyKind(args.policy)
    if args.seed is not None:
        cfg.seed = args.seed
    out_dir = args.out or cfg.out_dir or default_out_dir()
    _, _, summary = run_experiment(cfg, out_dir)
    print(_summary_line(summary))
    return 0


def cmd_compare(args) -> int:
    cfg = load_config(args.config)
    if args.seed is not None:
        cfg.seed = args.seed
    policies: list[PolicyKind] = []
    for name in args.policies.split(","):
        kind = PolicyKind(name.strip())
        if kind in policies:
            print(f"warning: policy {kind.value} listed twice, ignoring duplicate",
                  file=sys.stderr)
            continue
        policies.append(kind)
    if len(policies) < 2:
        raise ConfigError("compare needs at least 2 distinct policies")
    out_dir = args.out or cfg.out_dir or default_out_dir()
    os.makedirs(out_dir, exist_ok=True)
    profiles = cfg.build_profiles()
    trace = cfg.build_trace(profiles)           # every policy sees identical arrivals
    save_trace(trace, os.path.join(out_dir, "trace.csv"))
    exps = [Experiment(replace(cfg, policy=k, echo=dict(cfg.echo)),
                       os.path.join(out_dir, k.value), profiles, trace) for k in policies]
    lines = ["policy,weighted_avg_latency_s,p50,p99,cold_hit_pct,max_gap_worst_window"]
    for k, o in zip(policies, run_experiments(exps)):
        lat = np.sort(o.run.latencies(), kind="stable")
        worst = max((w.max_gap for w in o.windows if w.comparable), default=0.0)
        s = o.summary
        lines.append(f"{k.value},{s['weighted_avg_latency_s']:.6f},{percentile(lat, 50.0):.6f},"
                     f"{percentile(lat, 99.0):.6f},{s['cold_hit_pct']:.6f},{worst:.6f}")
        print(_summary_line(s))
    write_atomic(os.path.join(out_dir, "compare.csv"), lines)
    return 0


def _format_value(value: float) -> str:
    return str(int(value)) if value == int(value) else str(value)


def _apply_sweep_param(cfg: ExperimentConfig, param: str, value: float) -> None:
    """cli.py:170-184."""
    if param == "T":
        cfg.t_overrun = value
    elif param == "alpha":
        cfg.alpha = value
    elif param == "d_max":
        cfg.d_max = int(value)
    elif param == "pool_max_containers":
        cfg.pool_max_containers = int(value)
    elif param == "rate_rps":
        if cfg.rate_rps is None:
            raise ConfigError("rate_rps sweep needs a generator workload")
        cfg.rate_rps = value


def cmd_sweep(args) -> int:
    cfg = load_config(args.config)
    if args.seed is not None:
        cfg.seed = args.seed
    if args.param not in SWEEP_PARAMS:
        raise ConfigError(f"unknown sweep param {args.param!r}, "
                          f"choose from {', '.join(SWEEP_PARAMS)}")
    try:
        values = [float(v) for v in args.values.split(",") if v.strip()]
    except ValueError as exc:
        raise ConfigError(f"bad sweep values: {exc}") from None
    if not values:
        raise ConfigError("sweep needs at least one value")
    out_dir = args.out or cfg.out_dir or default_out_dir()
    os.makedirs(out_dir, exist_ok=True)
    exps, labels = [], []
    for v in values:
        c = replace(cfg, echo=dict(cfg.echo))
        _apply_sweep_param(c, args.param, v)
        label = _format_value(v)
        labels.append(label)
        exps.append(Experiment(c, os.path.join(out_dir, f"{args.param}_{label}")))
    lines = ["value,weighted_avg_latency_s,cold_hit_pct,mean_util"]
    for label, o in zip(labels, run_experiments(exps)):
        s = o.summary
        lines.append(f"{label},{s['weighted_avg_latency_s']:.6f},{s['cold_hit_pct']:.6f},"
                     f"{s['mean_util']:.6f}")
        print(f"{args.param}={label} " + _summary_line(s))
    write_atomic(os.path.join(out_dir, "sweep.csv"), lines)
    return 0


def cmd_generate(args) -> int:
    if args.functions < 1 or args.rate <= 0 or args.duration < 0 or args.zipf <= 0:
        raise ConfigError("generate: functions >= 1, zipf > 0, rate > 0, duration >= 0")
    trace = gen_zipf(args.functions, args.zipf, args.rate, args.duration, args.seed)
    save_trace(trace, args.out)
    print(f"wrote {len(trace.entries)} arrivals to {args.out}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="gpufairq-b200",
                                description="MQFQ-Sticky fair-queueing simulator on B200")
    sub = p.add_subparsers(dest="command", required=True)
    pols = [k.value for k in PolicyKind]
    r = sub.add_parser("run", help="run one simulation from a config file")
    r.add_argument("--config", required=True)
    r.add_argument("--policy", choices=pols)
    r.add_argument("--seed", type=int)
    r.add_argument("--out")
    r.set_defaults(func=cmd_run)
    c = sub.add_parser("compare", help="run several policies on one trace (one GPU batch)")
    c.add_argument("--config", required=True)
    c.add_argument("--policies", required=True)
    c.add_argument("--seed", type=int)
    c.add_argument("--out")
    c.set_defaults(func=cmd_compare)
    s = sub.add_parser("sweep", help="run one config across parameter values (one GPU batch)")
    s.add_argument("--config", required=True)
    s.add_argument("--param", required=True, help=f"one of {', '.join(SWEEP_PARAMS)}")
    s.add_argument("--values", required=True)
    s.add_argument("--seed", type=int)
    s.add_argument("--out")
    s.set_defaults(func=cmd_sweep)
    g = sub.add_parser("generate", help="write a synthetic Zipf trace")
    g.add_argument("--functions", type=int, required=True)
    g.add_argument("--zipf", type=float, required=True)
    g.add_argument("--rate", type=float, required=True)
    g.add_argument("--duration", type=float, required=True)
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--out", required=True)
    g.set_defaults(func=cmd_generate)
    return p


def main(argv: list[str] | None = None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return 2 if exc.code not in (0, None) else 0
    try:
        return args.func(args)
    except (ConfigError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
