/*
 * gfq.h — C ABI of the B200-native MQFQ-Sticky simulation engine (libgfq.so).
 *
 * The reference (`gpufairq`, /root/reference/pkg/src/gpufairq) is pure
 * Python: its hot path is `run_simulation(trace, profiles, policy, devices,
 * tau_includes_overheads) -> SimResult` (engine.py:214-218), driven one
 * simulation at a time by the CLI's serial sweep/compare loops
 * (cli.py:91-107,148-157).  A per-event FFI call would be far too fine
 * grained, so this ABI sits at the simulation-batch level: the caller uploads
 * traces, per-trace flow tables and device configs once, then runs batches
 * of independent simulations.  Every entry point below names the reference
 * interface it replaces; INTEGRATION.md shows the ctypes binding a
 * maintainer adds on the reference side.
 *
 * Conventions (mirroring SURVEY.md §8(b)):
 *   - plain C types, caller-owned host buffers, engine-owned device buffers;
 *   - every call returns an int status; nonzero -> gfq_last_error() holds a
 *     message.  GFQ_EINVAL maps to the reference's ValueError, GFQ_ERUNTIME
 *     and GFQ_ECUDA to RuntimeError (cli.py:260-267 exit-code mapping);
 *   - one handle per GPU; calls on a handle are serialised by the caller
 *     (the reference's single-logical-actor contract).
 */
#ifndef GFQ_H
#define GFQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GFQ_ABI_VERSION 3

/* ---- status codes ---------------------------------------------------- */
#define GFQ_OK        0
#define GFQ_EINVAL    1   /* bad arguments           -> ValueError   */
#define GFQ_ERUNTIME  2   /* simulation logic error  -> RuntimeError */
#define GFQ_ECUDA     3   /* CUDA failure            -> RuntimeError */
#define GFQ_ENOMEM    4   /* allocation failure      -> MemoryError  */

/* ---- enums (values match the reference's declaration order) ---------- */
/* PolicyKind, policies.py:18-23 */
#define GFQ_POLICY_MQFQ        0
#define GFQ_POLICY_FCFS        1
#define GFQ_POLICY_BATCH       2
#define GFQ_POLICY_SJF         3
#define GFQ_POLICY_FCFS_NAIVE  4   /* FCFS; the caller disables the pool (cli.py:36) */

/* StartState, core.py:16-21 */
#define GFQ_GPU_WARM   0
#define GFQ_HOST_WARM  1
#define GFQ_COLD       2

/* event kinds, engine.py:20-23 */
#define GFQ_EV_ARRIVAL       0
#define GFQ_EV_COMPLETION    1
#define GFQ_EV_MONITOR_TICK  2
#define GFQ_EV_QUEUE_EXPIRY  3

/* device models */
#define GFQ_DEVMODEL_DEVICESET 0   /* DeviceSet of modeled GPUs, device.py:80-341 */
#define GFQ_DEVMODEL_SCRIPTED  1   /* ScriptedDevices + drive(), tests/oracles.py:12-35,199-238 */

/* per-simulation status (GFQ_OUT_STATUS) */
#define GFQ_SIM_OK               0
#define GFQ_SIM_EVENT_OVERFLOW   1  /* dynamic event pool full               */
#define GFQ_SIM_SAMPLE_OVERFLOW  2  /* util-sample window longer than buffer */
#define GFQ_SIM_WATCHDOG         3  /* max_events reached (reference would spin) */
#define GFQ_SIM_PAST_EVENT       4  /* event scheduled in the past, engine.py:84-85 */
#define GFQ_SIM_OUTPUT_OVERFLOW  5  /* an audit/event-log buffer was too small */
#define GFQ_SIM_POOL_OVERFLOW    6  /* container pool exceeded its buffer   */
#define GFQ_SIM_BAD_CONFIG       7  /* parameter block rejected in-kernel    */

/* ---- parameter blocks ------------------------------------------------- */

/* DeviceConfig, device.py:22-34 (same fields, same meaning). */
typedef struct gfq_device_cfg {
    double  mem_capacity_mb;
    double  util_threshold;
    double  pcie_mb_per_s;
    double  interference_beta;
    double  monitor_period_s;
    double  util_window_s;
    double  prefetch_overlap_s;
    int32_t d_max;
    int32_t pool_max_containers;
    int32_t pool_enabled;
    int32_t dynamic_d;
} gfq_device_cfg;

/* One simulation = run_simulation(trace, profiles, make_policy(kind, cfg),
 * DeviceSet(configs), tau_includes_overheads) (engine.py:214-218). */
typedef struct gfq_sim {
    int32_t trace;                  /* uploaded trace id                           */
    int32_t flowtab;                /* uploaded flow table id (profiles+weights)    */
    int32_t policy;                 /* GFQ_POLICY_*                                 */
    int32_t device_model;           /* GFQ_DEVMODEL_*                               */
    int32_t n_devices;              /* len(DeviceSet), 1..GFQ_MAX_DEVICES           */
    int32_t device_cfg;             /* first of n_devices consecutive device cfgs   */
    int32_t tau_includes_overheads; /* engine.py:135                                */
    int32_t group;                  /* histogram group, -1 = none                   */
    double  t_overrun;              /* SchedulerConfig, mqfq.py:16-32               */
    double  alpha;
    double  default_ttl_s;
    int32_t scripted_d;             /* ScriptedDevices(d, deny_every)               */
    int32_t scripted_deny_every;
    int64_t exec_off;               /* scripted exec times: execs[exec_off ..]      */
    int32_t exec_len;               /*   cycled in dispatch order (oracles.py:217)  */
    int32_t reserved;
    int64_t max_events;             /* watchdog, 0 = 64 * (arrivals + 1024)         */
} gfq_sim;

#define GFQ_MAX_DEVICES 8

/* Requested outputs (bitmask for gfq_launch_cfg.outputs). */
#define GFQ_WANT_STATS     0x01u  /* per-sim summary + per-flow stats (metrics.py:63-84,195-226) */
#define GFQ_WANT_RECORDS   0x02u  /* per-invocation records (InvocationRecord, metrics.py:18-39) */
#define GFQ_WANT_DISPATCH  0x04u  /* DispatchAudit rows in dispatch order (mqfq.py:42-53)        */
#define GFQ_WANT_AUDIT     0x08u  /* AuditLog backlog/util rows (engine.py:26-37)                */
#define GFQ_WANT_EVENTS    0x10u  /* processed-event log, Simulation.step() (engine.py:99-113)   */
#define GFQ_WANT_HIST      0x20u  /* per-(group, flow) log-binned latency histograms             */
#define GFQ_WANT_EVICTIONS 0x40u  /* Device.eviction_log rows (device.py:92,172,177,275)         */

typedef struct gfq_launch_cfg {
    uint32_t outputs;           /* GFQ_WANT_* mask                                     */
    int32_t  early_exit;        /* 1: stop once only expiry rechecks remain (exact for
                                   every output except GFQ_WANT_EVENTS and
                                   GFQ_WANT_EVICTIONS, which turn it off) */
    int32_t  event_capacity;    /* dynamic-event slots per sim, 0 = auto               */
    int32_t  sample_capacity;   /* util-sample slots per device, 0 = auto              */
    int64_t  audit_util_cap;    /* util rows per sim (GFQ_WANT_AUDIT)                  */
    int64_t  audit_backlog_cap; /* backlog rows per sim                                */
    int64_t  event_log_cap;     /* event rows per sim (GFQ_WANT_EVENTS)                */
    int32_t  hist_groups;       /* GFQ_WANT_HIST: groups x hist_rows x hist_bins u64    */
    int32_t  hist_rows;         /* rows per group (flow-table hist_row ids)            */
    int32_t  hist_bins;
    int32_t  warps_per_block;   /* 0 = auto                                            */
    double   hist_lo_s;         /* log-binned latency histogram range                 */
    double   hist_hi_s;
    int32_t  blocks;            /* 0 = auto (persistent grid)                          */
    uint32_t flags;             /* GFQ_FLAG_*                                          */
} gfq_launch_cfg;

/* gfq_launch_cfg.flags */
#define GFQ_FLAG_FLOWS_GLOBAL 0x1u /* per-flow state in global scratch (automatic when the
                                      flow count does not fit shared memory)           */
#define GFQ_FLAG_CTA          0x2u /* one simulation per CTA, every scan split over its
                                      warps (automatic for large flow counts)          */
#define GFQ_FLAG_WARP         0x4u /* never CTA-per-simulation: one simulation per warp,
                                      per-flow state in global scratch when it does not
                                      fit (many large-flow simulations at once)        */

#define GFQ_NCOUNTERS 12

/* Output ids for gfq_output_info / gfq_output_copy / gfq_output_device_ptr.
 * Per-sim arrays have n_sims elements; per-flow arrays are concatenated per
 * sim at the sim's flow offset (gfq_sim_offsets); per-invocation arrays at
 * the sim's record offset (index = trace position).                       */
enum gfq_output_id {
    GFQ_OUT_STATUS = 0,        /* int32  [sims]                                  */
    GFQ_OUT_COUNTERS,          /* int64  [sims][GFQ_NCOUNTERS]: events, dispatch()
                                  calls, dispatches, util rows, peak dynamic
                                  events, global-VT scans, keep-alive refresh
                                  scans, candidate scans, monitor ticks,
                                  window-average memo hits, misses, quiet
                                  drains                                        */
    GFQ_OUT_FINAL_TIME,        /* double [sims]  simulated clock at exit          */
    GFQ_OUT_SUMMARY,           /* double [sims][3]: weighted_avg_latency_s,
                                  cold_hit_pct, mean_util (metrics.py:229-245)   */
    GFQ_OUT_FLOW_COUNT,        /* int64  [flows]                                  */
    GFQ_OUT_FLOW_MEAN,         /* double [flows] mean latency                     */
    GFQ_OUT_FLOW_VAR,          /* double [flows] unbiased variance                */
    GFQ_OUT_FLOW_COLD_PCT,     /* double [flows]                                  */
    GFQ_OUT_REC_DISPATCH,      /* double [invocations] dispatch_s                 */
    GFQ_OUT_REC_COMPLETE,      /* double [invocations] complete_s                 */
    GFQ_OUT_REC_STATE,         /* int8   [invocations] start_state                */
    GFQ_OUT_REC_DEVICE,        /* int8   [invocations] device index               */
    GFQ_OUT_REC_ORDER,         /* int32  [invocations] completion rank            */
    GFQ_OUT_REC_PURE,          /* double [invocations] pure exec (audit.exec)     */
    GFQ_OUT_DSP_INV,           /* int32  [invocations] dispatch row -> trace pos  */
    GFQ_OUT_DSP_VT_BEFORE,     /* double [invocations]                            */
    GFQ_OUT_DSP_GVT,           /* double [invocations]                            */
    GFQ_OUT_DSP_QLEN,          /* int32  [invocations]                            */
    GFQ_OUT_DSP_INFLIGHT,      /* int32  [invocations]                            */
    GFQ_OUT_UTIL_ROWS,         /* double [sims][audit_util_cap][3]: t, inst, avg  */
    GFQ_OUT_UTIL_META,         /* int32  [sims][audit_util_cap][2]: device, eff_d */
    GFQ_OUT_BACKLOG_TIME,      /* double [sims][audit_backlog_cap]                */
    GFQ_OUT_BACKLOG_META,      /* int32  [sims][audit_backlog_cap]: flow<<1 | on  */
    GFQ_OUT_BACKLOG_COUNT,     /* int64  [sims]                                   */
    GFQ_OUT_EVENT_TIME,        /* double [sims][event_log_cap]                    */
    GFQ_OUT_EVENT_META,        /* int64  [sims][event_log_cap]: payload<<2 | kind */
    GFQ_OUT_EVENT_COUNT,       /* int64  [sims]                                   */
    GFQ_OUT_HIST,              /* uint64 [groups][rows][bins]                     */
    GFQ_OUT_FAIR_ROWS,         /* double [windows][5]: w0, service_sum, max_gap,
                                  bound, bound_conservative  (gfq_fairness)      */
    GFQ_OUT_FAIR_META,         /* int64  [windows][6]: comparable, n_qualified,
                                  qualified-set hash, hi flow, lo flow, violated */
    GFQ_OUT_FAIR_OFF,          /* int64  [sims+1] window-row offset of each sim  */
    GFQ_OUT_FAIR_COUNT,        /* int64  [sims][3]: windows, comparable, violated */
    GFQ_OUT_EVICT_TIME,        /* double [invocations] eviction time, the sim's
                                  rows from its record offset in log order
                                  (GFQ_WANT_EVICTIONS; rows <= arrivals)         */
    GFQ_OUT_EVICT_META,        /* int32  [invocations] flow << 4 | device         */
    GFQ_OUT_EVICT_COUNT,       /* int64  [sims]                                   */
    GFQ_OUT_DSP_EVENT,         /* int32  [invocations] per dispatch row: the
                                  1-based index of the processed event whose
                                  drain made it (generic build, i.e. with
                                  GFQ_WANT_AUDIT / EVENTS / EVICTIONS; 0
                                  otherwise) -- Simulation.step() replay      */
    GFQ_OUT_EVICT_EVENT,       /* int32  [invocations] per eviction row: the
                                  processed event that logged it             */
    GFQ_OUT_REC_START_TAG,     /* double [invocations] Invocation.start_tag set
                                  by FlowQueue.enqueue (core.py:131-134):
                                  MQFQ in the generic build with
                                  GFQ_WANT_RECORDS; 0 otherwise              */
    GFQ_OUT_COUNT_
};

/* ---- handle lifecycle --------------------------------------------------- */
typedef struct gfq_handle gfq_handle;

/* Thread-local message for the last nonzero status. */
const char* gfq_last_error(void);
int  gfq_abi_version(void);

/* Bind a handle to CUDA device `device`.  Replaces constructing the
 * reference's Simulation objects (engine.py:47-78) for a batch. */
int  gfq_create(int device, gfq_handle** out);
int  gfq_destroy(gfq_handle* h);

/* ---- inputs --------------------------------------------------------------- */
/* Traces: the reference's Trace.entries (workload.py:37-46), packed CSR.
 * arrival[off[t] .. off[t+1]) are non-decreasing seconds; flow[] holds the
 * rank of the function name within the trace's sorted touched-name set
 * (Python sorted() order, mqfq.py:160,213).  n_flows[t] is that set's size.
 * The per-flow arrival index (the FIFO slices every policy pops from,
 * SURVEY App. C) is built on the GPU by the trace-loader kernel.
 * Validation mirrors Simulation.__init__ (engine.py:50-52,72-73): a
 * decreasing arrival or out-of-range flow id returns GFQ_EINVAL.           */
int  gfq_upload_traces(gfq_handle* h, const double* arrival, const int32_t* flow,
                       const int64_t* off, const int32_t* n_flows, int32_t n_traces);

/* Synthetic traces generated on the GPU, in place of gfq_upload_traces: the
 * reference's gen_zipf (workload.py:82-111) for n_traces traces at once,
 * bit-identical to it (numpy 2.3 SeedSequence.spawn + PCG64 + the
 * exponential ziggurat + round(t, 6) + sort by (t, name)).  Per trace t:
 * n_functions[t] functions in the caller's order (the names= order of
 * gen_zipf); rates[] = zipf_rates(...) for them (concatenated per trace);
 * name_rank[] = each function's position in the sorted name list;
 * duration_s[t]; seed[t] (< 2^64).  Outputs (optional): touched[] (1 if the
 * function arrived at least once, same layout as rates) and
 * trace_off[n_traces + 1].  The resident traces are replaced exactly as by
 * gfq_upload_traces, with flow ids = rank among the touched names. */
int  gfq_generate_traces(gfq_handle* h, int32_t n_traces, const int32_t* n_functions,
                         const double* rates, const int32_t* name_rank,
                         const double* duration_s, const uint64_t* seed,
                         uint8_t* touched, int64_t* trace_off);

/* Copy the resident traces (uploaded or generated) back to the host:
 * arrival[total] and flow[total], total = trace_off[n_traces]. */
int  gfq_download_traces(gfq_handle* h, double* arrival, int32_t* flow, int64_t total);

/* Flow tables: FunctionProfile fields (core.py:30-51) for one trace's flows,
 * in flow-rank order, plus the effective scheduler weight (weight_of,
 * mqfq.py:88-92) and a histogram row id.  off has n_tabs+1 entries.      */
int  gfq_upload_flowtabs(gfq_handle* h, const double* warm_s, const double* cold_s,
                         const double* mem_mb, const double* compute_share,
                         const double* weight, const int32_t* hist_row,
                         const int64_t* off, int32_t n_tabs);

/* DeviceConfig array, referenced by gfq_sim.device_cfg. */
int  gfq_upload_device_cfgs(gfq_handle* h, const gfq_device_cfg* cfgs, int32_t n);

/* Scripted-device execution durations (oracles.drive exec_times). */
int  gfq_upload_execs(gfq_handle* h, const double* execs, int64_t n);

/* ---- runs ---------------------------------------------------------------- */
/* Stage a batch: validates every gfq_sim against the uploaded inputs,
 * computes per-sim flow/record offsets and allocates device outputs.
 * Replaces the serial loops of cli.cmd_sweep / cmd_compare (cli.py:67-163). */
int  gfq_prepare(gfq_handle* h, const gfq_sim* sims, int32_t n_sims,
                 const gfq_launch_cfg* cfg);

/* Per-sim offsets of the staged batch (host arrays of n_sims+1). */
int  gfq_sim_offsets(gfq_handle* h, int64_t* flow_off, int64_t* rec_off);

/* Enqueue the simulation + reducer kernels on `stream` (cudaStream_t, NULL =
 * legacy default).  Asynchronous; outputs stay in HBM. */
int  gfq_launch(gfq_handle* h, void* stream);

/* Wait for the last launch; returns GFQ_ERUNTIME if any sim's status is not
 * GFQ_SIM_OK (the message names the first failing sim). */
int  gfq_synchronize(gfq_handle* h);

/* Device time of the last launch's kernels in milliseconds (CUDA events
 * recorded on the launch stream around the sim kernel and the reducer). */
int  gfq_last_kernel_ms(gfq_handle* h, float* sim_ms, float* reduce_ms);

/* Per-launch kernel times of up to the last GFQ_TIMING_RING launches since
 * the previous call (oldest first); *n receives the count.  Lets a caller
 * time the simulation kernel alone over a region of back-to-back launches. */
#define GFQ_TIMING_RING 256
int  gfq_kernel_times(gfq_handle* h, float* sim_ms, float* reduce_ms, int32_t cap, int32_t* n);

/* How the staged batch will launch: info[0] kernel launches per gfq_launch
 * (one per active simulation class + the reducer), info[1] simulations per
 * CTA class mode (0 = warp per simulation, else CTA threads per simulation),
 * info[2] flows in global scratch (0/1), info[3] simulation warps per CTA in
 * warp mode, info[4] CTAs of the largest simulation launch, info[5] the
 * dynamic-event capacity per simulation actually used (slots; callers that
 * re-run a GFQ_SIM_EVENT_OVERFLOW simulation grow from this).  n = entries
 * wanted (<= 6). */
int  gfq_batch_info(gfq_handle* h, int32_t* info, int32_t n);

/* Output access. */
int  gfq_output_info(gfq_handle* h, int32_t id, int64_t* n_elems, int32_t* elem_bytes);
int  gfq_output_copy(gfq_handle* h, int32_t id, void* host_dst, int64_t bytes);
int  gfq_output_device_ptr(gfq_handle* h, int32_t id, void** dptr);

/* Fairness audit of the last (synchronized) batch: metrics.service_gap_report
 * (metrics.py:106-187) per simulation, on the GPU.  Needs a batch run with
 * GFQ_WANT_RECORDS | GFQ_WANT_AUDIT.  d_max[n_sims] is each sim's
 * SchedulerConfig.d_max (the reference's fallback D); report_weight holds
 * cfg.weights.get(f, 1.0) for every uploaded flow-table row (same offsets).
 * Window rows land in GFQ_OUT_FAIR_*; the call synchronizes. */
int  gfq_fairness(gfq_handle* h, double window_s, const int32_t* d_max,
                  const double* report_weight, int64_t n_weights);

/* ---- multi-GPU (one process per GPU) -------------------------------------
 * The sweep's one collective step: after a launch, sum the
 * latency histograms of every rank in place (ncclAllReduce) and gather every
 * rank's per-simulation summary rows (ncclAllGather) into summary_out, a
 * device buffer of n_ranks * n_sims * 3 doubles (NULL: histograms only).
 * Enqueued on `stream` (cudaStream_t, NULL = legacy default) after the
 * launch; all ranks must have staged batches of the same shape.  NCCL is
 * loaded at first use (dlopen "libnccl.so.2", the one already in the process
 * if any); comm is an ncclComm_t, from the helpers below or the caller's own.
 * Replaces the serial per-process result collection of cli.cmd_sweep. */
#define GFQ_NCCL_ID_BYTES 128
int  gfq_nccl_unique_id(char id[GFQ_NCCL_ID_BYTES]);
int  gfq_nccl_comm_init(void** comm, int32_t n_ranks, const char id[GFQ_NCCL_ID_BYTES], int32_t rank);
int  gfq_nccl_comm_destroy(void* comm);
int  gfq_reduce_nccl(gfq_handle* h, void* comm, void* summary_out, void* stream);

/* Convenience: prepare + launch + synchronize on the default stream.
 * The drop-in for run_simulation over a batch (engine.py:214-218). */
int  gfq_run(gfq_handle* h, const gfq_sim* sims, int32_t n_sims,
             const gfq_launch_cfg* cfg);

#ifdef __cplusplus
}
#endif
#endif /* GFQ_H */
