"""Python face of the B200 engine: the reference's ``run_simulation`` drop-in
and the batched sweep API, both over libgfq.so (include/gfq.h).

``run_simulation(trace, profiles, policy, devices, tau_includes_overheads)``
keeps the reference signature and return type (engine.py:214-218): it
accepts the reference's own ``Trace`` / ``FunctionProfile`` dict /
``make_policy`` result / ``DeviceSet`` (or this package's mirrors of them,
duck-typed on ``.entries``, ``.kind``, ``.cfg`` and each device's ``.cfg``)
and returns ``SimResult(records, audit)`` with ``InvocationRecord`` rows in
completion order, ``audit.dispatches`` (the DispatchAudit dispatch trace,
also appended to ``policy.dispatch_log``), ``audit.backlog``,
``audit.util`` and ``audit.exec``.

``Engine`` is the batch interface: upload traces / flow tables / device
configs once, then run thousands of independent simulations per launch
(the serial ``cmd_sweep`` / ``cmd_compare`` loops, cli.py:67-163, become one
kernel launch).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._lib import check, lib
from .core import STATE_BY_CODE
from .mqfq import DispatchAudit
from .pack import FlowTable, PackedTrace, flow_table, pack_trace

_OUT_DTYPES = {
    _abi.OUT_STATUS: np.int32, _abi.OUT_COUNTERS: np.int64, _abi.OUT_FINAL_TIME: np.float64,
    _abi.OUT_SUMMARY: np.float64, _abi.OUT_FLOW_COUNT: np.int64, _abi.OUT_FLOW_MEAN: np.float64,
    _abi.OUT_FLOW_VAR: np.float64, _abi.OUT_FLOW_COLD_PCT: np.float64,
    _abi.OUT_REC_DISPATCH: np.float64, _abi.OUT_REC_COMPLETE: np.float64,
    _abi.OUT_REC_STATE: np.int8, _abi.OUT_REC_DEVICE: np.int8, _abi.OUT_REC_ORDER: np.int32,
    _abi.OUT_REC_PURE: np.float64, _abi.OUT_DSP_INV: np.int32,
    _abi.OUT_DSP_VT_BEFORE: np.float64, _abi.OUT_DSP_GVT: np.float64,
    _abi.OUT_DSP_QLEN: np.int32, _abi.OUT_DSP_INFLIGHT: np.int32,
    _abi.OUT_UTIL_ROWS: np.float64, _abi.OUT_UTIL_META: np.int32,
    _abi.OUT_BACKLOG_TIME: np.float64, _abi.OUT_BACKLOG_META: np.int32,
    _abi.OUT_BACKLOG_COUNT: np.int64, _abi.OUT_EVENT_TIME: np.float64,
    _abi.OUT_EVENT_META: np.int64, _abi.OUT_EVENT_COUNT: np.int64, _abi.OUT_HIST: np.uint64,
    _abi.OUT_FAIR_ROWS: np.float64, _abi.OUT_FAIR_META: np.int64, _abi.OUT_FAIR_OFF: np.int64,
    _abi.OUT_FAIR_COUNT: np.int64, _abi.OUT_EVICT_TIME: np.float64,
    _abi.OUT_EVICT_META: np.int32, _abi.OUT_EVICT_COUNT: np.int64,
    _abi.OUT_DSP_EVENT: np.int32, _abi.OUT_EVICT_EVENT: np.int32, _abi.OUT_REC_START_TAG: np.float64,
}

_POLICY = {"mqfq": _abi.POLICY_MQFQ, "fcfs": _abi.POLICY_FCFS, "batch": _abi.POLICY_BATCH,
           "sjf": _abi.POLICY_SJF, "fcfs_naive": _abi.POLICY_FCFS_NAIVE}


def policy_code(kind) -> int:
    k = getattr(kind, "value", kind)
    if k not in _POLICY:
        raise ValueError(f"unknown policy: {kind}")
    return _POLICY[k]


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _stream_handle(stream) -> int | None:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(getattr(stream, "cuda_stream"))


class Engine:
    """One libgfq handle bound to one CUDA device (single logical actor)."""

    def __init__(self, device: int = 0):
        self._L = lib()
        h = C.c_void_p()
        check(self._L.gfq_create(int(device), C.byref(h)))
        self._h = h
        self.device = device
        self._keep = []
        self.n_sims = 0
        self._flow_off = None
        self._rec_off = None

    def close(self) -> None:
        if self._h:
            self._L.gfq_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---------------------------------------------------------------- inputs
    def upload_traces(self, traces) -> None:
        arrs = [np.ascontiguousarray(t.arrival, dtype=np.float64) for t in traces]
        flows = [np.ascontiguousarray(t.flow, dtype=np.int32) for t in traces]
        off = np.zeros(len(traces) + 1, dtype=np.int64)
        off[1:] = np.cumsum([a.shape[0] for a in arrs])
        arrival = np.concatenate(arrs) if arrs else np.zeros(0)
        flow = np.concatenate(flows) if flows else np.zeros(0, np.int32)
        nf = np.array([t.n_flows for t in traces], dtype=np.int32)
        arrival = np.ascontiguousarray(arrival, dtype=np.float64)
        flow = np.ascontiguousarray(flow, dtype=np.int32)
        check(self._L.gfq_upload_traces(self._h, _ptr(arrival, C.c_double), _ptr(flow, C.c_int32),
                                        _ptr(off, C.c_int64), _ptr(nf, C.c_int32), len(traces)))

    def generate_traces(self, specs) -> list[PackedTrace]:
        """GPU gen_zipf (workload.py:82-111) for many traces, made resident as
        by upload_traces.  specs: (n_functions, zipf_s, total_rate_rps,
        duration_s, seed[, names]) tuples; names default to
        default_profiles(n_functions).  Returns one PackedTrace per spec
        (names = the touched functions in sorted order; arrays fetched from
        the device)."""
        from .workload import default_profiles, zipf_rates
        nfs, rates, ranks, durs, seeds, names_all = [], [], [], [], [], []
        for spec in specs:
            n, s_, rate, dur, seed = spec[:5]
            names = list(spec[5]) if len(spec) > 5 and spec[5] is not None else None
            if n < 1:
                raise ValueError("n_functions must be >= 1")
            if rate <= 0:
                raise ValueError("total_rate_rps must be > 0")
            if names is None:
                names = list(default_profiles(n))
            if len(names) != n:
                raise ValueError("names must match n_functions")
            if not 0 <= int(seed) < 2 ** 64:
                raise ValueError("seed must be in [0, 2**64)")
            rates.extend(zipf_rates(n, s_, rate))
            order = sorted(range(n), key=lambda k: names[k])
            rk = [0] * n
            for j, k in enumerate(order):
                rk[k] = j
            ranks.extend(rk)
            nfs.append(n); durs.append(float(dur)); seeds.append(int(seed)); names_all.append(names)
        nt = len(nfs)
        nf_a = np.asarray(nfs, dtype=np.int32)
        rt_a = np.asarray(rates, dtype=np.float64)
        rk_a = np.asarray(ranks, dtype=np.int32)
        du_a = np.asarray(durs, dtype=np.float64)
        sd_a = np.asarray(seeds, dtype=np.uint64)
        touched = np.zeros(max(len(rates), 1), dtype=np.uint8)
        toff = np.zeros(nt + 1, dtype=np.int64)
        check(self._L.gfq_generate_traces(self._h, nt, _ptr(nf_a, C.c_int32), _ptr(rt_a, C.c_double),
                                          _ptr(rk_a, C.c_int32), _ptr(du_a, C.c_double),
                                          _ptr(sd_a, C.c_uint64), _ptr(touched, C.c_uint8),
                                          _ptr(toff, C.c_int64)))
        total = int(toff[-1])
        arrival = np.zeros(max(total, 1), dtype=np.float64)
        flow = np.zeros(max(total, 1), dtype=np.int32)
        check(self._L.gfq_download_traces(self._h, _ptr(arrival, C.c_double), _ptr(flow, C.c_int32),
                                          total))
        out, a = [], 0
        for t in range(nt):
            n = nfs[t]
            tn = sorted(nm for nm, hit in zip(names_all[t], touched[a:a + n]) if hit)
            a += n
            lo, hi = int(toff[t]), int(toff[t + 1])
            out.append(PackedTrace(tn, arrival[lo:hi].copy(), flow[lo:hi].copy()))
        return out

    def upload_trace_arrays(self, arrival, flow, off, n_flows) -> None:
        """Pre-packed CSR arrays (e.g. pinned host buffers), no host copy."""
        check(self._L.gfq_upload_traces(self._h, _ptr(arrival, C.c_double), _ptr(flow, C.c_int32),
                                        _ptr(off, C.c_int64), _ptr(n_flows, C.c_int32),
                                        int(n_flows.shape[0])))

    def upload_flowtab_arrays(self, warm, cold, mem, share, weight, hist_row, off) -> None:
        check(self._L.gfq_upload_flowtabs(
            self._h, _ptr(warm, C.c_double), _ptr(cold, C.c_double), _ptr(mem, C.c_double),
            _ptr(share, C.c_double), _ptr(weight, C.c_double), _ptr(hist_row, C.c_int32),
            _ptr(off, C.c_int64), int(off.shape[0]) - 1))

    def upload_flowtabs(self, tabs) -> None:
        cols = {}
        for name in ("warm", "cold", "mem", "share", "weight"):
            cols[name] = np.ascontiguousarray(
                np.concatenate([getattr(t, name) for t in tabs]) if tabs else np.zeros(0),
                dtype=np.float64)
        hist = np.ascontiguousarray(
            np.concatenate([t.hist_row for t in tabs]) if tabs else np.zeros(0, np.int32),
            dtype=np.int32)
        off = np.zeros(len(tabs) + 1, dtype=np.int64)
        off[1:] = np.cumsum([len(t) for t in tabs])
        check(self._L.gfq_upload_flowtabs(
            self._h, _ptr(cols["warm"], C.c_double), _ptr(cols["cold"], C.c_double),
            _ptr(cols["mem"], C.c_double), _ptr(cols["share"], C.c_double),
            _ptr(cols["weight"], C.c_double), _ptr(hist, C.c_int32), _ptr(off, C.c_int64),
            len(tabs)))

    def upload_device_cfgs(self, cfgs) -> None:
        structs = [c if isinstance(c, _abi.DeviceCfg) else _abi.device_cfg_from(c) for c in cfgs]
        arr = (_abi.DeviceCfg * max(len(structs), 1))(*structs)
        check(self._L.gfq_upload_device_cfgs(self._h, arr, len(structs)))

    def upload_execs(self, execs) -> None:
        e = np.ascontiguousarray(execs, dtype=np.float64)
        check(self._L.gfq_upload_execs(self._h, _ptr(e, C.c_double), int(e.shape[0])))

    # ---------------------------------------------------------------- runs
    def prepare(self, sims, outputs: int = _abi.WANT_STATS, early_exit: bool = True,
                **kw) -> None:
        if isinstance(sims, C.Array):
            arr, n = sims, len(sims)
        else:
            n = len(sims)
            arr = (_abi.Sim * max(n, 1))(*sims)
        cfg = _abi.LaunchCfg()
        cfg.outputs = int(outputs)
        cfg.early_exit = int(bool(early_exit))
        for k, v in kw.items():
            setattr(cfg, k, v)
        self._keep = [arr]
        check(self._L.gfq_prepare(self._h, arr, n, C.byref(cfg)))
        self.n_sims = n
        fo = np.zeros(n + 1, dtype=np.int64)
        ro = np.zeros(n + 1, dtype=np.int64)
        check(self._L.gfq_sim_offsets(self._h, _ptr(fo, C.c_int64), _ptr(ro, C.c_int64)))
        self._flow_off, self._rec_off = fo, ro
        self.cfg = cfg

    def launch(self, stream=None) -> None:
        check(self._L.gfq_launch(self._h, _stream_handle(stream)))

    def synchronize(self) -> None:
        check(self._L.gfq_synchronize(self._h))

    def kernel_ms(self) -> float:
        a, b = C.c_float(), C.c_float()
        check(self._L.gfq_last_kernel_ms(self._h, C.byref(a), C.byref(b)))
        return float(a.value) + float(b.value)

    def fairness(self, d_max, report_weights, window_s: float = 30.0):
        """metrics.service_gap_report for every sim of the last batch (which must
        have been run with WANT_RECORDS | WANT_AUDIT).  d_max: per-sim
        SchedulerConfig.d_max; report_weights: cfg.weights.get(f, 1.0) for every
        uploaded flow-table row.  Returns FairnessResult."""
        dm = np.ascontiguousarray(d_max, dtype=np.int32)
        rw = np.ascontiguousarray(report_weights, dtype=np.float64)
        check(self._L.gfq_fairness(self._h, float(window_s), _ptr(dm, C.c_int32),
                                   _ptr(rw, C.c_double), int(rw.shape[0])))
        return FairnessResult(self.output(_abi.OUT_FAIR_ROWS).reshape(-1, 5),
                              self.output(_abi.OUT_FAIR_META).reshape(-1, 6),
                              self.output(_abi.OUT_FAIR_OFF),
                              self.output(_abi.OUT_FAIR_COUNT).reshape(-1, 3))

    def batch_info(self) -> dict:
        """gfq_batch_info of the staged batch."""
        v = np.zeros(6, dtype=np.int32)
        check(self._L.gfq_batch_info(self._h, _ptr(v, C.c_int32), 6))
        return {"launches_per_step": int(v[0]), "cta_threads": int(v[1]),
                "flows_global": bool(v[2]), "warps_per_block": int(v[3]), "ctas": int(v[4]),
                "event_capacity": int(v[5])}

    def reduce_nccl(self, comm: "NcclComm", summary_out=None, stream=None) -> None:
        """gfq_reduce_nccl: sum the last launch's latency histograms over every
        rank of `comm` (in place) and gather the per-simulation summary rows
        into `summary_out` (a CUDA tensor of n_ranks * n_sims * 3 float64, or
        None).  Enqueued on `stream` after the launch."""
        ptr = None
        if summary_out is not None:
            ptr = C.c_void_p(summary_out.data_ptr())
        check(self._L.gfq_reduce_nccl(self._h, comm.handle, ptr, _stream_handle(stream)))

    def kernel_times(self, cap: int = 256):
        """(sim_ms, reduce_ms) arrays of the launches since the last call."""
        a = np.zeros(cap, dtype=np.float32)
        b = np.zeros(cap, dtype=np.float32)
        n = C.c_int32()
        check(self._L.gfq_kernel_times(self._h, _ptr(a, C.c_float), _ptr(b, C.c_float), cap,
                                       C.byref(n)))
        return a[:n.value].astype(np.float64), b[:n.value].astype(np.float64)

    def run(self, sims, outputs: int = _abi.WANT_STATS, early_exit: bool = True, **kw):
        self.prepare(sims, outputs, early_exit, **kw)
        self.launch()
        self.synchronize()
        return BatchResult(self)

    # ---------------------------------------------------------------- outputs
    def output(self, oid: int) -> np.ndarray:
        n, b = C.c_int64(), C.c_int32()
        check(self._L.gfq_output_info(self._h, oid, C.byref(n), C.byref(b)))
        a = np.empty(n.value, dtype=_OUT_DTYPES[oid])
        if n.value:
            check(self._L.gfq_output_copy(self._h, oid, a.ctypes.data_as(C.c_void_p),
                                          n.value * b.value))
        return a

    def output_into(self, oid: int, out: np.ndarray) -> np.ndarray:
        """Copy output `oid` into a caller-owned array (e.g. pinned host
        memory, for full-bandwidth device->host reads); returns the filled
        prefix view."""
        n, b = C.c_int64(), C.c_int32()
        check(self._L.gfq_output_info(self._h, oid, C.byref(n), C.byref(b)))
        if out.dtype != _OUT_DTYPES[oid] or out.size < n.value or not out.flags.c_contiguous:
            raise ValueError("output_into: array too small, wrong dtype or not contiguous")
        if n.value:
            check(self._L.gfq_output_copy(self._h, oid, out.ctypes.data_as(C.c_void_p),
                                          n.value * b.value))
        return out[: n.value]

    def output_device_ptr(self, oid: int) -> tuple[int, int]:
        p = C.c_void_p()
        n, b = C.c_int64(), C.c_int32()
        check(self._L.gfq_output_device_ptr(self._h, oid, C.byref(p)))
        check(self._L.gfq_output_info(self._h, oid, C.byref(n), C.byref(b)))
        return int(p.value or 0), int(n.value)

    @property
    def flow_off(self):
        return self._flow_off

    @property
    def rec_off(self):
        return self._rec_off


class NcclComm:
    """An NCCL communicator made through libgfq (gfq_nccl_comm_init), one
    rank per GPU; rank 0 makes the id (unique_id()) and shares it (e.g. with
    torch.distributed.broadcast_object_list)."""

    def __init__(self, n_ranks: int, rank: int, uid: bytes):
        self._L = lib()
        h = C.c_void_p()
        check(self._L.gfq_nccl_comm_init(C.byref(h), int(n_ranks), bytes(uid), int(rank)))
        self.handle = h

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().gfq_nccl_unique_id(buf))
        return buf.raw

    def close(self) -> None:
        if getattr(self, "handle", None):
            check(self._L.gfq_nccl_comm_destroy(self.handle))
            self.handle = None


@dataclass
class FairnessResult:
    """gfq_fairness outputs; window(i) gives sim i's rows (WindowReport fields)."""
    rows: np.ndarray        # [windows, 5] w0, service_sum, max_gap, bound, bound_conservative
    meta: np.ndarray        # [windows, 6] comparable, n_qualified, qual_hash, hi, lo, violated
    off: np.ndarray         # [sims + 1]
    count: np.ndarray       # [sims, 3] windows, comparable, violated

    def windows(self, i: int):
        a = int(self.off[i])
        k = int(self.count[i, 0])
        return self.rows[a:a + k], self.meta[a:a + k]


class BatchResult:
    """Host copies of a finished batch's outputs, sliced per simulation."""

    def __init__(self, eng: Engine):
        self.eng = eng
        self.n_sims = eng.n_sims
        self.flow_off = eng.flow_off
        self.rec_off = eng.rec_off
        self.cfg = eng.cfg
        self._cache = {}

    def get(self, oid: int) -> np.ndarray:
        if oid not in self._cache:
            self._cache[oid] = self.eng.output(oid)
        return self._cache[oid]

    @property
    def status(self):
        return self.get(_abi.OUT_STATUS)

    @property
    def counters(self):
        return self.get(_abi.OUT_COUNTERS).reshape(-1, _abi.NCOUNTERS)

    @property
    def summary(self):
        return self.get(_abi.OUT_SUMMARY).reshape(-1, 3)

    def dispatches_total(self) -> int:
        return int(self.counters[:, 2].sum())

    def flow_stats(self, i: int) -> dict:
        a, b = int(self.flow_off[i]), int(self.flow_off[i + 1])
        return {"count": self.get(_abi.OUT_FLOW_COUNT)[a:b],
                "mean": self.get(_abi.OUT_FLOW_MEAN)[a:b],
                "var": self.get(_abi.OUT_FLOW_VAR)[a:b],
                "cold_pct": self.get(_abi.OUT_FLOW_COLD_PCT)[a:b]}

    def records(self, i: int) -> dict:
        """Per-invocation arrays by trace position, plus completion order."""
        a, b = int(self.rec_off[i]), int(self.rec_off[i + 1])
        n_done = int(self.counters[i, 2])
        order = self.get(_abi.OUT_REC_ORDER)[a:b]
        return {"dispatch": self.get(_abi.OUT_REC_DISPATCH)[a:b],
                "complete": self.get(_abi.OUT_REC_COMPLETE)[a:b],
                "state": self.get(_abi.OUT_REC_STATE)[a:b],
                "device": self.get(_abi.OUT_REC_DEVICE)[a:b],
                "pure": self.get(_abi.OUT_REC_PURE)[a:b],
                # FlowQueue start tags (MQFQ, generic build with the logs; else 0)
                "start_tag": self.get(_abi.OUT_REC_START_TAG)[a:b],
                "order": order, "n": n_done}

    def completion_order(self, i: int) -> np.ndarray:
        """Trace positions in completion order (every arrival completes in a
        finished simulation, SPEC: #records == #arrivals)."""
        order = self.records(i)["order"].astype(np.int64)
        pos = np.empty(order.shape[0], dtype=np.int64)
        pos[order] = np.arange(order.shape[0])
        return pos

    def dispatch_rows(self, i: int) -> dict:
        a = int(self.rec_off[i])
        k = int(self.counters[i, 2])
        return {"inv": self.get(_abi.OUT_DSP_INV)[a:a + k],
                "vt_before": self.get(_abi.OUT_DSP_VT_BEFORE)[a:a + k],
                "gvt": self.get(_abi.OUT_DSP_GVT)[a:a + k],
                "qlen": self.get(_abi.OUT_DSP_QLEN)[a:a + k],
                "inflight": self.get(_abi.OUT_DSP_INFLIGHT)[a:a + k],
                # generic build: the processed event whose drain made each row
                "event": self.get(_abi.OUT_DSP_EVENT)[a:a + k]}

    def _cap(self, oid: int, per: int) -> int:
        return int(self.get(oid).shape[0]) // (per * max(self.n_sims, 1))

    def util_rows(self, i: int):
        cap = self._cap(_abi.OUT_UTIL_META, 2)
        k = min(int(self.counters[i, 3]), cap)
        rows = self.get(_abi.OUT_UTIL_ROWS).reshape(-1, cap, 3)[i, :k]
        meta = self.get(_abi.OUT_UTIL_META).reshape(-1, cap, 2)[i, :k]
        return rows, meta

    def backlog_rows(self, i: int):
        cap = self._cap(_abi.OUT_BACKLOG_META, 1)
        k = min(int(self.get(_abi.OUT_BACKLOG_COUNT)[i]), cap)
        t = self.get(_abi.OUT_BACKLOG_TIME).reshape(-1, cap)[i, :k]
        m = self.get(_abi.OUT_BACKLOG_META).reshape(-1, cap)[i, :k]
        return t, m

    def eviction_rows(self, i: int, events: bool = False):
        """(time, device, flow) arrays of sim i's Device.eviction_log rows,
        all devices interleaved in the order they were logged (+ the index of
        the processed event that logged each, with events=True)."""
        a = int(self.rec_off[i])
        k = int(self.get(_abi.OUT_EVICT_COUNT)[i])
        t = self.get(_abi.OUT_EVICT_TIME)[a:a + k]
        m = self.get(_abi.OUT_EVICT_META)[a:a + k].astype(np.int64)
        if events:
            return t, m & 15, m >> 4, self.get(_abi.OUT_EVICT_EVENT)[a:a + k]
        return t, m & 15, m >> 4

    def event_rows(self, i: int):
        cap = self._cap(_abi.OUT_EVENT_META, 1)
        k = min(int(self.get(_abi.OUT_EVENT_COUNT)[i]), cap)
        t = self.get(_abi.OUT_EVENT_TIME).reshape(-1, cap)[i, :k]
        m = self.get(_abi.OUT_EVENT_META).reshape(-1, cap)[i, :k]
        return t, m


# ----------------------------------------------------------------------------
# reference-shaped results (metrics.py:18-39, engine.py:26-43)

@dataclass
class InvocationRecord:
    function: str
    arrival_s: float
    dispatch_s: float
    complete_s: float
    start_state: str
    device: int

    @property
    def queue_latency_s(self) -> float:
        return self.dispatch_s - self.arrival_s

    @property
    def exec_s(self) -> float:
        return self.complete_s - self.dispatch_s

    @property
    def latency_s(self) -> float:
        return self.complete_s - self.arrival_s


@dataclass
class AuditLog:
    dispatches: list = field(default_factory=list)
    backlog: list = field(default_factory=list)
    util: list = field(default_factory=list)
    exec: list = field(default_factory=list)


@dataclass
class SimResult:
    records: list
    audit: AuditLog


def sim_params(policy_kind, sched_cfg, n_devices: int, *, trace: int = 0, flowtab: int = 0,
               device_cfg: int = 0, tau_includes_overheads: bool = False,
               group: int = -1) -> _abi.Sim:
    s = _abi.Sim()
    s.trace, s.flowtab = trace, flowtab
    s.policy = policy_code(policy_kind)
    s.device_model = _abi.DEVMODEL_DEVICESET
    s.n_devices, s.device_cfg = n_devices, device_cfg
    s.tau_includes_overheads = int(bool(tau_includes_overheads))
    s.group = group
    s.t_overrun = float(sched_cfg.t_overrun)
    s.alpha = float(sched_cfg.alpha)
    s.default_ttl_s = float(sched_cfg.default_ttl_s)
    return s


_engines: dict[int, Engine] = {}


def default_engine(device: int = 0) -> Engine:
    if device not in _engines:
        _engines[device] = Engine(device)
    return _engines[device]


def _device_cfgs(devices):
    cfgs = []
    for d in devices:
        cfgs.append(d.cfg if hasattr(d, "cfg") else d)
    if not cfgs:
        raise ValueError("at least one device required")
    return cfgs


# gfq.h per-simulation statuses that are the engine's own capacity limits,
# not the reference's behaviour: re-run with larger buffers / budget
_SIM_EVENT_OVERFLOW, _SIM_WATCHDOG, _SIM_OUTPUT_OVERFLOW = 1, 3, 5


def _run_one(eng: "Engine", sim, n_arrivals: int, outputs: int, early_exit: bool, **kw):
    """One simulation through ``eng``.  The reference has no event-pool,
    audit-buffer or event-budget limits, so a simulation that hits one of the
    engine's is re-run with 4x the capacity (16x the event budget), as
    cli.run_experiments does for a batch; other statuses raise."""
    from ._lib import EngineError
    sim = _abi.Sim.from_buffer_copy(sim)
    for attempt in range(6):
        eng.prepare([sim], outputs, early_exit, **kw)
        eng.launch()
        try:
            eng.synchronize()
            return BatchResult(eng)
        except EngineError:
            st = int(eng.output(_abi.OUT_STATUS)[0])
            if attempt == 5 or st not in (_SIM_EVENT_OVERFLOW, _SIM_WATCHDOG, _SIM_OUTPUT_OVERFLOW):
                raise
        if st == _SIM_EVENT_OVERFLOW:    # grow from the capacity that overflowed
            kw["event_capacity"] = 4 * eng.batch_info()["event_capacity"]
        elif st == _SIM_WATCHDOG:
            sim.max_events = 16 * (int(sim.max_events) or 64 * (n_arrivals + 1024))
        else:
            for k in ("audit_util_cap", "audit_backlog_cap", "event_log_cap"):
                kw[k] = 4 * int(kw.get(k, 0) or (1 << 16))
    raise AssertionError("unreachable")


def run_simulation(trace, profiles, policy, devices, tau_includes_overheads: bool = False,
                   *, device: int = 0) -> SimResult:
    """Drop-in for gpufairq.engine.run_simulation (engine.py:214-218), run by
    the CUDA engine on ``device``."""
    pt = pack_trace(trace.entries, profiles)
    cfg = policy.cfg
    tab = flow_table(pt.names, profiles, getattr(cfg, "weights", None))
    dcfgs = _device_cfgs(devices)
    eng = default_engine(device)
    eng.upload_traces([pt])
    eng.upload_flowtabs([tab])
    eng.upload_device_cfgs(dcfgs)
    sim = sim_params(policy.kind, cfg, len(dcfgs), tau_includes_overheads=tau_includes_overheads)
    res = _run_one(eng, sim, pt.n, _abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_DISPATCH |
                   _abi.WANT_AUDIT | _abi.WANT_EVICTIONS, True)
    out = to_sim_result(res, 0, pt)
    _share_dispatch_log(policy, out.audit)
    _append_eviction_logs(devices, res, 0, pt.names)
    return out


def _append_eviction_logs(devices, res: "BatchResult", i: int, names) -> None:
    """Device.eviction_log (device.py:92): the run's (time, function) rows
    appended to each device's list, as the reference's devices record them."""
    devs = list(devices)
    t, d, f = res.eviction_rows(i)
    for tt, dd, ff in zip(t.tolist(), d.tolist(), f.tolist()):
        log = getattr(devs[dd], "eviction_log", None)
        if isinstance(log, list):
            log.append((tt, names[ff]))


def _share_dispatch_log(policy, audit) -> None:
    """The reference's audit.dispatches IS the policy's dispatch_log list
    (engine.py:118): this run's rows are appended to it, earlier rows kept."""
    log = getattr(policy, "dispatch_log", None)
    if isinstance(log, list):
        log.extend(audit.dispatches)
        audit.dispatches = log


# event kinds, engine.py:20-23
ARRIVAL, COMPLETION, MONITOR_TICK, QUEUE_EXPIRY = 0, 1, 2, 3


class Simulation:
    """Drop-in for ``gpufairq.engine.Simulation`` (engine.py:46-119).

    Construction validates like the reference (unknown functions and
    decreasing arrival times raise ``ValueError``).  On first ``step()`` or
    ``run()`` the whole simulation runs on the GPU in parity mode (processed-
    event log, records, dispatch rows with the event that made each, audit,
    eviction log).  ``step()`` then replays it event by event and leaves the
    observable state where the reference's ``step()`` leaves it
    (engine.py:99-197): it returns the reference's ``(time, kind, payload)``
    tuple -- the ``Invocation`` for arrivals, its ``uid`` for completions,
    ``None`` for monitor ticks, the function name for keep-alive expiries --
    advances ``now``; a completion appends its ``InvocationRecord`` and
    ``audit.exec`` row and stamps ``complete_s``; backlog transitions and
    monitor ticks append their ``audit.backlog`` / ``audit.util`` rows; the
    dispatches of the event's drain stamp their invocations' ``dispatch_s`` /
    ``start_state`` and append their ``DispatchAudit`` rows to
    ``policy.dispatch_log``; the event's evictions go to each device's
    ``eviction_log``.  ``run()`` then shares ``policy.dispatch_log`` as
    ``audit.dispatches`` (engine.py:118).  The policy's and devices' internal
    queues and pools are not replayed.
    """

    def __init__(self, trace, profiles, policy, devices, tau_includes_overheads: bool = False,
                 *, device: int = 0):
        from .core import Invocation
        self._pt = pack_trace(trace.entries, profiles)
        self.trace, self.profiles, self.policy, self.devices = trace, profiles, policy, devices
        self.tau_includes_overheads = tau_includes_overheads
        self._device = device
        self.now = 0.0
        self.records: list = []
        self.audit = AuditLog()
        self._inv = [Invocation(function=nm, arrival_s=t) for t, nm in trace.entries]
        self._events = None
        self._pos = 0
        self._result = None

    def _ensure(self) -> None:
        if self._events is not None:
            return
        pt = self._pt
        cfg = self.policy.cfg
        eng = default_engine(self._device)
        dcfgs = _device_cfgs(self.devices)
        eng.upload_traces([pt])
        eng.upload_flowtabs([flow_table(pt.names, self.profiles, getattr(cfg, "weights", None))])
        eng.upload_device_cfgs(dcfgs)
        sim = sim_params(self.policy.kind, cfg, len(dcfgs),
                         tau_includes_overheads=self.tau_includes_overheads)
        cap = 64 * (pt.n + 1024)
        res = _run_one(eng, sim, pt.n, _abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_DISPATCH |
                       _abi.WANT_AUDIT | _abi.WANT_EVENTS | _abi.WANT_EVICTIONS, False,
                       event_log_cap=cap, audit_util_cap=cap, audit_backlog_cap=2 * pt.n + 2)
        full = to_sim_result(res, 0, pt)
        rec = res.records(0)
        self._rec_dispatch = rec["dispatch"].tolist()
        self._rec_state = [STATE_BY_CODE[int(x)] for x in rec["state"].tolist()]
        self._stag = rec["start_tag"].tolist()
        order = rec["order"]
        self._rec_of = {p: full.records[int(order[p])] for p in range(pt.n)}
        self._exec_of = {p: full.audit.exec[int(order[p])] for p in range(pt.n)}
        # dispatch rows and eviction rows, bucketed by the processed event
        # (1-based) whose drain / swap-out made them
        dr = res.dispatch_rows(0)
        self._disp_of = {}
        for j, (ev, p) in enumerate(zip(dr["event"].tolist(), dr["inv"].tolist())):
            self._disp_of.setdefault(ev, []).append((p, full.audit.dispatches[j]))
        t, d, f, e = res.eviction_rows(0, events=True)
        self._evict_of = {}
        for tt, dd, ff, ee in zip(t.tolist(), d.tolist(), f.tolist(), e.tolist()):
            self._evict_of.setdefault(ee, []).append((dd, (tt, pt.names[ff])))
        self._util_rows = full.audit.util
        self._backlog = {}
        self._ndev = max(len(dcfgs), 1)
        et, em = res.event_rows(0)
        evs = []
        for t, m in zip(et.tolist(), em.tolist()):
            kind, pay = m & 3, m >> 2
            if kind == ARRIVAL:
                evs.append((t, kind, self._inv[pay], pay))
            elif kind == COMPLETION:
                evs.append((t, kind, self._inv[pay].uid, pay))
            elif kind == MONITOR_TICK:
                evs.append((t, kind, None))
            else:
                evs.append((t, kind, pt.names[pay]))
        self._events = evs
        self._result = full

    def _backlog_change(self, t, fn, delta) -> None:
        """_backlog_change, engine.py:199-207: the row of a 0 -> 1 or 1 -> 0
        transition (the GPU run's rows, in the same order)."""
        c = self._backlog.get(fn, 0) + delta
        self._backlog[fn] = c
        if (delta > 0 and c == 1) or (delta < 0 and c == 0):
            self.audit.backlog.append((t, fn, delta > 0))

    def step(self):
        """Process the earliest event; returns (time, kind, payload) or None."""
        self._ensure()
        if self._pos >= len(self._events):
            return None
        ev = self._events[self._pos]
        self._pos += 1
        k = self._pos                                   # 1-based processed-event index
        self.now = t = ev[0]
        if ev[1] == ARRIVAL:
            ev[2].start_tag = self._stag[ev[3]]         # FlowQueue.enqueue, core.py:131-134
            self._backlog_change(t, ev[2].function, +1)
            ev = ev[:3]
        elif ev[1] == COMPLETION:
            p = ev[3]
            self._inv[p].complete_s = t
            self.records.append(self._rec_of[p])
            self._backlog_change(t, self._inv[p].function, -1)
            self.audit.exec.append(self._exec_of[p])
            ev = ev[:3]
        elif ev[1] == MONITOR_TICK:
            u0 = len(self.audit.util)
            self.audit.util.extend(self._util_rows[u0:u0 + self._ndev])
        log = getattr(self.policy, "dispatch_log", None)
        for p, row in self._disp_of.get(k, ()):
            inv = self._inv[p]
            inv.dispatch_s = self._rec_dispatch[p]
            inv.start_state = self._rec_state[p]
            (log if isinstance(log, list) else self.audit.dispatches).append(row)
        if k in self._evict_of:
            devs = list(self.devices)
            for d, row in self._evict_of[k]:
                elog = getattr(devs[d], "eviction_log", None)
                if isinstance(elog, list):
                    elog.append(row)
        return ev

    def run(self) -> SimResult:
        while self.step() is not None:
            pass
        log = getattr(self.policy, "dispatch_log", None)
        if isinstance(log, list):
            self.audit.dispatches = log                  # engine.py:118
        return SimResult(records=self.records, audit=self.audit)


def to_sim_result(res: BatchResult, i: int, pt: PackedTrace) -> SimResult:
    """Reference-shaped SimResult of simulation i (records in completion
    order, DispatchAudit rows, audit.exec / util / backlog).  The arrays are
    turned into Python lists once, and the rows are built from those."""
    names = pt.names
    rec = res.records(i)
    k = int(res.counters[i, 2])
    comp = res.completion_order(i).tolist()
    fname = [names[f] for f in pt.flow.tolist()]
    arr = pt.arrival.tolist()
    d_s, c_s, pure = rec["dispatch"].tolist(), rec["complete"].tolist(), rec["pure"].tolist()
    sv = [s.value for s in STATE_BY_CODE]
    st = [sv[x] for x in rec["state"].tolist()]
    dv = rec["device"].tolist()
    records = [InvocationRecord(fname[p], arr[p], d_s[p], c_s[p], st[p], dv[p]) for p in comp]
    exe = [(fname[p], d_s[p], c_s[p], pure[p]) for p in comp]
    dr = res.dispatch_rows(i)
    disp = [DispatchAudit(now=d_s[p], function=fname[p], vt_before=vb, global_vt=g, queue_len=q,
                          in_flight=fl, device=dv[p], start_state=st[p])
            for p, vb, g, q, fl in zip(dr["inv"][:k].tolist(), dr["vt_before"][:k].tolist(),
                                        dr["gvt"][:k].tolist(), dr["qlen"][:k].tolist(),
                                        dr["inflight"][:k].tolist())]
    audit = AuditLog(dispatches=disp, exec=exe)
    if res.cfg.outputs & _abi.WANT_AUDIT:
        rows, meta = res.util_rows(i)
        audit.util = [(r[0], m[0], r[1], r[2], m[1]) for r, m in zip(rows.tolist(), meta.tolist())]
        bt, bm = res.backlog_rows(i)
        audit.backlog = [(t, names[m >> 1], bool(m & 1)) for t, m in zip(bt.tolist(), bm.tolist())]
    return SimResult(records=records, audit=audit)


__all__ = ["Engine", "BatchResult", "Simulation", "run_simulation", "sim_params", "SimResult",
           "InvocationRecord", "AuditLog", "FlowTable", "PackedTrace", "default_engine"]
