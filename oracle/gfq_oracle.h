/*
 * gfq_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference simulator (gpufairq engine/mqfq/device/
 * policies/metrics) for ONE simulation, used as the parity checker by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm.  Never linked into libgfq.so and never on the product path.
 */
#ifndef GFQ_ORACLE_H
#define GFQ_ORACLE_H
#include "../include/gfq.h"
#ifdef __cplusplus
extern "C" {
#endif

typedef struct gfq_oracle_out {
    /* capacities in, counts out; NULL arrays are skipped                    */
    int64_t  cap_records, n_records;          /* completion order            */
    int64_t *rec_inv; double *rec_dispatch, *rec_complete, *rec_pure;
    int8_t  *rec_state, *rec_device;
    int64_t  cap_dispatch, n_dispatch;        /* DispatchAudit rows          */
    int64_t *d_inv; int32_t *d_flow; double *d_now, *d_vt_before, *d_gvt;
    int64_t *d_qlen, *d_inflight; int8_t *d_device, *d_state;
    int64_t  cap_util, n_util;                /* AuditLog.util               */
    double  *u_time, *u_inst, *u_avg; int32_t *u_dev, *u_effd;
    int64_t  cap_backlog, n_backlog;          /* AuditLog.backlog            */
    double  *b_time; int32_t *b_flow; int8_t *b_on;
    int64_t  cap_events, n_events_logged;     /* Simulation.step() stream    */
    double  *ev_time; int8_t *ev_kind; int64_t *ev_payload;
    int64_t  cap_evictions, n_evictions;      /* Device.eviction_log         */
    double  *x_time; int32_t *x_dev, *x_flow;
    /* per flow (n_flows), metrics.per_function_summary                      */
    int64_t *f_count; double *f_mean, *f_var, *f_cold_pct;
    /* scalars                                                               */
    double   weighted_avg_latency, cold_hit_pct, mean_util, final_time;
    int64_t  n_events, n_dispatch_calls;
    int32_t  status;
    int32_t  early_exit;    /* in: 1 = stop once only keep-alive rechecks remain
                               (no tick scheduled, every arrival processed,
                               nothing pending or in flight): the engine's
                               bench-launch rule (gfq_launch_cfg.early_exit),
                               so both bench arms process the same events    */
} gfq_oracle_out;

int gfq_oracle_run(const gfq_sim* sim,
                   const double* arrival, const int32_t* flow, int64_t n, int32_t n_flows,
                   const double* warm_s, const double* cold_s, const double* mem_mb,
                   const double* compute_share, const double* weight,
                   const gfq_device_cfg* device_cfgs, const double* execs,
                   gfq_oracle_out* out);

#ifdef __cplusplus
}
#endif
#endif
