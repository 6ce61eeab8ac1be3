"""Result reports and the bit-exact exporter (gpufairq.metrics, metrics.py:1-300).

The reductions themselves run on the GPU: per-function count / mean /
unbiased variance / cold %, the weighted average latency, the cold-hit
rate and the mean utilisation in ``k_reduce`` (metrics.py:63-84,195-245),
the Eq. 1 service-gap audit in ``k_fairness`` (metrics.py:106-187).  This
module shapes those device outputs into the reference's objects
(``WindowReport``, the ``summarize`` dict) and writes the reference's files
byte for byte: ``invocations.csv`` / ``windows.csv`` (LF endings, ``%.6f``
numerics) and ``summary.json`` (``json.dumps(indent=2, sort_keys=True)``),
each through a temp file + ``os.replace`` (metrics.py:253-300).

Exactness: every number written is the GPU's, bit-identical to the
reference's except ``var_latency_s``, which agrees within 1e-9 relative --
the reference squares with ``(x - mean) ** 2`` (libm ``pow``), the GPU with
``x * x``; the two differ in the last place for ~0.1% of inputs.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass, field

import numpy as np

from .engine import InvocationRecord

INVOCATION_COLUMNS = ("function,arrival_s,dispatch_s,complete_s,start_state,"
                      "device,queue_latency_s,exec_s,latency_s")
WINDOW_COLUMNS = "window_start_s,max_gap,bound,violated"
STATE_NAMES = ("gpu_warm", "host_warm", "cold")


@dataclass
class WindowReport:
    """metrics.py:42-60.  ``service`` / ``qualified`` are not materialised by
    the GPU reducer (it keeps their sum, count and an order-independent hash);
    ``n_qualified`` and ``service_sum`` carry them."""

    window_start_s: float
    window_s: float
    service: dict = field(default_factory=dict)
    qualified: list = field(default_factory=list)
    comparable: bool = False
    max_gap: float = 0.0
    bound: float = 0.0
    bound_conservative: float = 0.0
    violated: bool = False
    n_qualified: int = 0
    service_sum: float = 0.0


def windows_from(fair, i: int, window_s: float) -> list[WindowReport]:
    """WindowReports of sim ``i`` from an ``Engine.fairness`` result."""
    rows, meta = fair.windows(i)
    out = []
    for r, m in zip(rows.tolist(), meta.tolist()):
        out.append(WindowReport(window_start_s=float(r[0]), window_s=window_s,
                                comparable=bool(m[0]), max_gap=float(r[2]), bound=float(r[3]),
                                bound_conservative=float(r[4]), violated=bool(m[5]),
                                n_qualified=int(m[1]), service_sum=float(r[1])))
    return out


@dataclass
class RunArrays:
    """One finished simulation's records as columns, in completion order."""

    names: list
    flow: np.ndarray        # int32 flow rank per record
    arrival: np.ndarray
    dispatch: np.ndarray
    complete: np.ndarray
    state: np.ndarray       # int8 StartState code
    device: np.ndarray      # int8

    def __len__(self) -> int:
        return int(self.arrival.shape[0])

    def records(self) -> list[InvocationRecord]:
        nm = self.names
        return [InvocationRecord(nm[f], a, d, c, STATE_NAMES[s], dv)
                for f, a, d, c, s, dv in zip(self.flow.tolist(), self.arrival.tolist(),
                                              self.dispatch.tolist(), self.complete.tolist(),
                                              self.state.tolist(), self.device.tolist())]

    def latencies(self) -> np.ndarray:
        return self.complete - self.arrival


def run_arrays(res, i: int, pt) -> RunArrays:
    """Completion-ordered columns of sim ``i`` of a BatchResult (WANT_RECORDS)."""
    rec = res.records(i)
    pos = res.completion_order(i)
    return RunArrays(list(pt.names), pt.flow[pos], pt.arrival[pos], rec["dispatch"][pos],
                     rec["complete"][pos], rec["state"][pos], rec["device"][pos])


def per_function_summary(res, i: int, names) -> dict:
    """metrics.py:195-220 from the GPU per-flow statistics (flows with at
    least one record, in sorted-name order -- flow ranks are that order)."""
    st = res.flow_stats(i)
    out = {}
    for f, nm in enumerate(names):
        n = int(st["count"][f])
        if n:
            out[nm] = {"mean_latency_s": float(st["mean"][f]),
                       "var_latency_s": float(st["var"][f]),
                       "count": n, "cold_hit_pct": float(st["cold_pct"][f])}
    return out


def summarize(policy: str, res, i: int, names, windows: list[WindowReport], config_echo: dict,
              seed, n_records: int) -> dict:
    """metrics.py:229-245 with every number from the GPU reducers."""
    wavg, cold_pct, util = (float(x) for x in res.summary[i])
    return {
        "policy": policy,
        "weighted_avg_latency_s": wavg if n_records else 0.0,
        "per_function": per_function_summary(res, i, names),
        "cold_hit_pct": cold_pct,
        "mean_util": util,
        "bound_violations": sum(1 for w in windows if w.violated),
        "bound_conservative_violations": sum(
            1 for w in windows if w.comparable and w.max_gap > w.bound_conservative),
        "config": config_echo,
        "seed": seed,
    }


def _fmt6(a: np.ndarray) -> list:
    # '%.6f' % x is the same correctly rounded conversion as f"{x:.6f}"
    return ["%.6f" % x for x in a.tolist()]


def invocation_lines(run: RunArrays) -> list[str]:
    lines = [INVOCATION_COLUMNS]
    if not len(run):
        return lines
    names = run.names
    fn = [names[f] for f in run.flow.tolist()]
    st = [STATE_NAMES[s] for s in run.state.tolist()]
    dev = [str(d) for d in run.device.tolist()]
    a, d, c = run.arrival, run.dispatch, run.complete
    cols = [_fmt6(a), _fmt6(d), _fmt6(c), _fmt6(d - a), _fmt6(c - d), _fmt6(c - a)]
    for k in range(len(run)):
        lines.append(f"{fn[k]},{cols[0][k]},{cols[1][k]},{cols[2][k]},{st[k]},{dev[k]},"
                     f"{cols[3][k]},{cols[4][k]},{cols[5][k]}")
    return lines


def window_lines(windows: list[WindowReport]) -> list[str]:
    lines = [WINDOW_COLUMNS]
    for w in windows:
        if w.comparable:
            lines.append(f"{w.window_start_s:.6f},{w.max_gap:.6f},{w.bound:.6f},"
                         f"{'true' if w.violated else 'false'}")
        else:
            lines.append(f"{w.window_start_s:.6f},,,false")
    return lines


def export(run: RunArrays, windows: list[WindowReport], summary: dict, out_dir: str) -> list[str]:
    """invocations.csv, windows.csv, summary.json (metrics.py:253-287)."""
    os.makedirs(out_dir, exist_ok=True)
    payload = json.dumps(summary, indent=2, sort_keys=True) + "\n"
    return [write_atomic(os.path.join(out_dir, "invocations.csv"), invocation_lines(run)),
            write_atomic(os.path.join(out_dir, "windows.csv"), window_lines(windows)),
            write_atomic(os.path.join(out_dir, "summary.json"), [payload], raw=True)]


def write_atomic(path: str, lines: list[str], raw: bool = False) -> str:
    """metrics.py:290-300: temp file, then os.replace; LF, UTF-8."""
    tmp = path + ".tmp"
    try:
        with open(tmp, "w", encoding="utf-8", newline="") as fh:
            fh.write("".join(lines) if raw else "\n".join(lines) + "\n")
        os.replace(tmp, path)
    except OSError as exc:
        raise OSError(f"failed writing {path}: {exc}") from exc
    return path


def percentile(sorted_values, q: float) -> float:
    """cli.py:119-128 linear interpolation on a sorted sequence."""
    n = len(sorted_values)
    if n == 0:
        return 0.0
    if n == 1:
        return float(sorted_values[0])
    pos = (q / 100.0) * (n - 1)
    lo = int(pos)
    hi = min(lo + 1, n - 1)
    frac = pos - lo
    return float(sorted_values[lo]) * (1 - frac) + float(sorted_values[hi]) * frac
