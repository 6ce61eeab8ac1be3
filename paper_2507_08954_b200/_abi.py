"""ctypes mirrors of the structs and constants in include/gfq.h.

Kept layout-identical to the header (checked by tests/test_abi.py against
the compiled library's exported sizes)."""

from __future__ import annotations

import ctypes as C

ABI_VERSION = 3
GFQ_OK, GFQ_EINVAL, GFQ_ERUNTIME, GFQ_ECUDA, GFQ_ENOMEM = 0, 1, 2, 3, 4

POLICY_MQFQ, POLICY_FCFS, POLICY_BATCH, POLICY_SJF, POLICY_FCFS_NAIVE = 0, 1, 2, 3, 4
GPU_WARM, HOST_WARM, COLD = 0, 1, 2
EV_ARRIVAL, EV_COMPLETION, EV_MONITOR_TICK, EV_QUEUE_EXPIRY = 0, 1, 2, 3
DEVMODEL_DEVICESET, DEVMODEL_SCRIPTED = 0, 1
MAX_DEVICES = 8
NCOUNTERS = 12
FLAG_FLOWS_GLOBAL = 0x1
FLAG_CTA = 0x2
FLAG_WARP = 0x4

SIM_STATUS = {
    0: "ok",
    1: "dynamic event pool overflow",
    2: "utilization-sample buffer overflow",
    3: "watchdog: event budget exhausted (the reference would not terminate)",
    4: "event scheduled in the past",
    5: "output buffer overflow",
    6: "container pool overflow",
    7: "bad simulation parameters",
}

WANT_STATS, WANT_RECORDS, WANT_DISPATCH, WANT_AUDIT, WANT_EVENTS, WANT_HIST, WANT_EVICTIONS = (
    0x01, 0x02, 0x04, 0x08, 0x10, 0x20, 0x40)

(OUT_STATUS, OUT_COUNTERS, OUT_FINAL_TIME, OUT_SUMMARY, OUT_FLOW_COUNT,
 OUT_FLOW_MEAN, OUT_FLOW_VAR, OUT_FLOW_COLD_PCT, OUT_REC_DISPATCH,
 OUT_REC_COMPLETE, OUT_REC_STATE, OUT_REC_DEVICE, OUT_REC_ORDER, OUT_REC_PURE,
 OUT_DSP_INV, OUT_DSP_VT_BEFORE, OUT_DSP_GVT, OUT_DSP_QLEN, OUT_DSP_INFLIGHT,
 OUT_UTIL_ROWS, OUT_UTIL_META, OUT_BACKLOG_TIME, OUT_BACKLOG_META,
 OUT_BACKLOG_COUNT, OUT_EVENT_TIME, OUT_EVENT_META, OUT_EVENT_COUNT,
 OUT_HIST, OUT_FAIR_ROWS, OUT_FAIR_META, OUT_FAIR_OFF, OUT_FAIR_COUNT,
 OUT_EVICT_TIME, OUT_EVICT_META, OUT_EVICT_COUNT, OUT_DSP_EVENT, OUT_EVICT_EVENT,
 OUT_REC_START_TAG, OUT_COUNT_) = range(39)


class DeviceCfg(C.Structure):
    _fields_ = [
        ("mem_capacity_mb", C.c_double),
        ("util_threshold", C.c_double),
        ("pcie_mb_per_s", C.c_double),
        ("interference_beta", C.c_double),
        ("monitor_period_s", C.c_double),
        ("util_window_s", C.c_double),
        ("prefetch_overlap_s", C.c_double),
        ("d_max", C.c_int32),
        ("pool_max_containers", C.c_int32),
        ("pool_enabled", C.c_int32),
        ("dynamic_d", C.c_int32),
    ]


class Sim(C.Structure):
    _fields_ = [
        ("trace", C.c_int32),
        ("flowtab", C.c_int32),
        ("policy", C.c_int32),
        ("device_model", C.c_int32),
        ("n_devices", C.c_int32),
        ("device_cfg", C.c_int32),
        ("tau_includes_overheads", C.c_int32),
        ("group", C.c_int32),
        ("t_overrun", C.c_double),
        ("alpha", C.c_double),
        ("default_ttl_s", C.c_double),
        ("scripted_d", C.c_int32),
        ("scripted_deny_every", C.c_int32),
        ("exec_off", C.c_int64),
        ("exec_len", C.c_int32),
        ("reserved", C.c_int32),
        ("max_events", C.c_int64),
    ]


class LaunchCfg(C.Structure):
    _fields_ = [
        ("outputs", C.c_uint32),
        ("early_exit", C.c_int32),
        ("event_capacity", C.c_int32),
        ("sample_capacity", C.c_int32),
        ("audit_util_cap", C.c_int64),
        ("audit_backlog_cap", C.c_int64),
        ("event_log_cap", C.c_int64),
        ("hist_groups", C.c_int32),
        ("hist_rows", C.c_int32),
        ("hist_bins", C.c_int32),
        ("warps_per_block", C.c_int32),
        ("hist_lo_s", C.c_double),
        ("hist_hi_s", C.c_double),
        ("blocks", C.c_int32),
        ("flags", C.c_uint32),
    ]


def device_cfg_from(cfg) -> DeviceCfg:
    """DeviceConfig (either this package's or the reference's) -> struct."""
    return DeviceCfg(
        float(cfg.mem_capacity_mb), float(cfg.util_threshold), float(cfg.pcie_mb_per_s),
        float(cfg.interference_beta), float(cfg.monitor_period_s), float(cfg.util_window_s),
        float(cfg.prefetch_overlap_s), int(cfg.d_max), int(cfg.pool_max_containers),
        int(bool(cfg.pool_enabled)), int(bool(cfg.dynamic_d)))
