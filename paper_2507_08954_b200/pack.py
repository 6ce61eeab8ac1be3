"""Host packing of reference-shaped inputs into the engine's HBM layout.

* A trace (``Trace.entries``, workload.py:37-46) becomes ``arrival f64[N]``
  plus ``flow i32[N]``, where a flow id is the rank of the function name
  within the trace's sorted set of names.  Python ``sorted()`` order is the
  order the reference iterates queues in (refresh_states, mqfq.py:160) and
  breaks candidate ties by (mqfq.py:213), so ranks preserve every tie.
* A flow table holds the ``FunctionProfile`` columns (core.py:30-51) of those
  flows in rank order, with the effective scheduler weight
  (``weight_of``: ``cfg.weights`` override, else ``profile.weight``,
  mqfq.py:88-92).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class PackedTrace:
    names: list[str]
    arrival: np.ndarray      # f64[N], non-decreasing
    flow: np.ndarray         # i32[N], rank into names

    @property
    def n(self) -> int:
        return int(self.arrival.shape[0])

    @property
    def n_flows(self) -> int:
        return len(self.names)


@dataclass
class FlowTable:
    warm: np.ndarray
    cold: np.ndarray
    mem: np.ndarray
    share: np.ndarray
    weight: np.ndarray
    hist_row: np.ndarray

    def __len__(self) -> int:
        return int(self.warm.shape[0])


def pack_trace(entries, profiles=None) -> PackedTrace:
    """Sorted-name ranks + arrays; validates like Simulation.__init__
    (engine.py:50-52 unknown functions, :72-73 non-decreasing times)."""
    names = sorted({nm for _, nm in entries})
    if profiles is not None:
        unknown = set(names) - set(profiles)
        if unknown:
            raise ValueError(f"trace references unknown functions: {sorted(unknown)}")
    rank = {nm: i for i, nm in enumerate(names)}
    arrival = np.fromiter((t for t, _ in entries), dtype=np.float64, count=len(entries))
    flow = np.fromiter((rank[nm] for _, nm in entries), dtype=np.int32, count=len(entries))
    if arrival.size > 1 and bool(np.any(np.diff(arrival) < 0)):
        raise ValueError("trace arrival times must be non-decreasing")
    return PackedTrace(names=names, arrival=arrival, flow=flow)


def flow_table(names, profiles, weights=None, hist_rows=None) -> FlowTable:
    weights = weights or {}
    ps = [profiles[nm] for nm in names]
    return FlowTable(
        warm=np.array([p.warm_exec_s for p in ps], dtype=np.float64),
        cold=np.array([p.cold_exec_s for p in ps], dtype=np.float64),
        mem=np.array([p.mem_mb for p in ps], dtype=np.float64),
        share=np.array([p.compute_share for p in ps], dtype=np.float64),
        weight=np.array([float(weights.get(nm, p.weight)) for nm, p in zip(names, ps)],
                        dtype=np.float64),
        hist_row=np.asarray(hist_rows if hist_rows is not None else np.arange(len(names)),
                            dtype=np.int32),
    )
