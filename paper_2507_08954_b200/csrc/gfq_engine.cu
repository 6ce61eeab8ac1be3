// gfq_engine.cu — kernels and the C ABI (include/gfq.h) of libgfq.so.
//
// Kernels
//   k_trace_index  trace loader: builds, per uploaded trace, the per-flow
//                  arrival index (CSR of trace positions grouped by flow, in
//                  arrival order).  Every policy pops queue heads from these
//                  FIFO slices (pending(f) = arrivals_f[popped
//                  : arrived]), replacing the reference's per-queue deques
//                  (core.py:110, FlowQueue.pending).
//   k_sim          persistent warp-per-simulation engine (sim_warp.cuh): each
//                  warp pulls simulations from an atomic work queue (longest
//                  first), runs the reference's event loop to completion and
//                  then reduces its own completion stream into the
//                  per-function summary (metrics.py:63-84,195-226) and the
//                  log-binned latency histograms, so no second pass over the
//                  records touches HBM.
//
// Host ABI: see include/gfq.h for the contract and the reference interface
// each entry point replaces.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <unordered_map>
#include <string>
#include <vector>

#include <cub/device/device_segmented_radix_sort.cuh>

#include "sim_warp.cuh"
#include "fairness.cuh"
#include "tracegen.cuh"

#ifndef GFQ_CTA_MIN
#define GFQ_CTA_MIN 256     // CTA builds: scans shorter than this stay on the leader warp (C4: 64 -> 256 +1%)
#endif
#ifndef GFQ_TIMELINE
#define GFQ_TIMELINE 0      // diagnostic build: per-simulation start/end time and SM in the counters
#endif

namespace gfq {

// ----------------------------------------------------------------------------
// stats reducer
enum { RED_FLOW_BYTES = 24,     // per-flow reducer scratch: naive f64 + cnt, cur, first/order i32
       RED_CHUNK = 8 };         // records a reducer lane loads ahead
//
// Per function, in completion order (metrics.py:195-220):
//   count, mean = sum(lat)/n (builtin Neumaier sum), var = sum((x-mean)**2)/(n-1),
//   cold % = 100*cold/n;
// weighted_avg_latency (metrics.py:63-77): per-function naive sums in a dict
// ordered by first completion, then sum(n*(s/n)) / total;
// cold_hit_rate (metrics.py:80-84); mean_util (metrics.py:223-226).
//
// One warp per simulation.  The completion stream is grouped by function
// with a stable counting sort (coalesced 32-record batches, __match_any_sync
// ranks), so each lane then walks its own functions' latencies in
// completion order -- every sum is the reference's sequential one, but the
// lanes run their functions in parallel instead of replaying every record
// through the whole warp.  Scratch: 24 B per flow (shared memory or global)
// and 8 B per record (global, `rec`).
__device__ __forceinline__ void reduce_one(const Params& p, unsigned char* base, double* rec, int lane, int sid) {
    const gfq_sim* sim = p.sims + sid;
    const int nf = p.trace_nf[sim->trace];
    const int nrec = (int)p.counters[(int64_t)sid * GFQ_NCOUNTERS + C_DISP];
    const int64_t roff = p.sim_roff[sid], tb = p.tab_off[sim->flowtab];
    const int F = p.L.F;
    // per flow: naive sum, record count, end cursor of its group, first
    // completion index (then: rank -> flow order)
    double* naive = (double*)base;
    int *cnt = (int*)(naive + F), *cur = cnt + F, *first = cnt + 2 * F, *order = cnt + 3 * F;
    for (int f = lane; f < nf; f += 32) { naive[f] = 0.0; cnt[f] = 0; first[f] = 0x7fffffff; }
    __syncwarp();
    // completion stream: completion time, trace position, flow | cold << 31;
    // latency = complete - arrival (InvocationRecord.latency_s)
    const double* ctime = p.comp_lat + roff;
    const int32_t* cpos = p.comp_pos + roff;
    const double* arrival = p.arrival + p.trace_off[sim->trace];
    const int32_t* meta = p.comp_meta + roff;
    int colds = 0;
    const bool want_hist = (p.outputs & GFQ_WANT_HIST) && sim->group >= 0;
    const double hl0 = want_hist ? log(p.hist_lo) : 0.0;
    const double hscale = want_hist ? (double)p.hist_bins / (log(p.hist_hi) - hl0) : 0.0;
    const int32_t* hrow = p.hist_row + tb;
    // pass 1: histograms, per-function counts and first completions
    for (int b0 = 0; b0 < nrec; b0 += 32) {
        const int k = b0 + lane;
        const bool in = k < nrec;
        double x = 0.0; int32_t m = 0;
        if (in) { x = ctime[k] - __ldg(arrival + cpos[k]); m = meta[k]; }
        const int fn = m & 0x7fffffff;
        if (want_hist) {
            // warp-aggregated: one atomic per distinct (row, bin) of the batch
            // (a sweep's simulations all hit the same few popular bins)
            int key = -1;
            if (in) {
                int b = x > 0.0 ? (int)floor((log(x) - hl0) * hscale) : 0;
                b = max(0, min(p.hist_bins - 1, b));
                key = hrow[fn] * p.hist_bins + b;
            }
            const unsigned peers = __match_any_sync(FULLMASK, key);
            if (in && lane == __ffs(peers) - 1) {
                int64_t o = (int64_t)sim->group * p.hist_rows * p.hist_bins + key;
                atomicAdd(&p.hist[o], (unsigned long long)__popc(peers));
            }
        }
        if (in) { atomicAdd(&cnt[fn], 1); atomicMin(&first[fn], k); }
        colds += __popc(__ballot_sync(FULLMASK, in && m < 0));
    }
    __syncwarp();
    // group starts (exclusive prefix of the counts, 32 flows per step)
    int carry = 0;
    for (int f0 = 0; f0 < nf; f0 += 32) {
        const int f = f0 + lane;
        const int c = f < nf ? cnt[f] : 0;
        int inc = c;
        #pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(FULLMASK, inc, d);
            if (lane >= d) inc += y;
        }
        if (f < nf) cur[f] = carry + inc - c;
        carry += __shfl_sync(FULLMASK, inc, 31);
    }
    __syncwarp();
    // pass 2: stable scatter by function; cold is carried in the sign bit
    // (latencies are >= 0, so -x with x == 0 is -0.0 and still decodes)
    for (int b0 = 0; b0 < nrec; b0 += 32) {
        const int k = b0 + lane;
        const bool in = k < nrec;
        double x = 0.0; int32_t m = 0;
        if (in) { x = ctime[k] - __ldg(arrival + cpos[k]); m = meta[k]; }
        const int fn = in ? (m & 0x7fffffff) : -1;
        const unsigned peers = __match_any_sync(FULLMASK, fn);
        if (in) {
            const int pos = cur[fn] + __popc(peers & ((1u << lane) - 1));
            rec[pos] = m < 0 ? -x : x;
        }
        __syncwarp();
        if (in && lane == 31 - __clz(peers)) cur[fn] += __popc(peers);
        __syncwarp();
    }
    // pass 3: each lane walks its functions' latencies in completion order
    const int64_t fo = p.sim_foff[sid];
    for (int f = lane; f < nf; f += 32) {
        const int c = cnt[f];
        if (c == 0) {
            if (p.outputs & GFQ_WANT_STATS) { p.f_count[fo + f] = 0; p.f_mean[fo + f] = 0.0; p.f_var[fo + f] = 0.0; p.f_cold[fo + f] = 0.0; }
            continue;
        }
        const int s0 = cur[f] - c;
        // the walks load RED_CHUNK records at a time (independent loads in
        // flight), then accumulate them in order
        double sv = 0.0, sc = 0.0, nv = 0.0;
        int cc = 0;
        for (int j0 = 0; j0 < c; j0 += RED_CHUNK) {
            double vb[RED_CHUNK];
            #pragma unroll
            for (int u = 0; u < RED_CHUNK; u++) vb[u] = j0 + u < c ? rec[s0 + j0 + u] : 0.0;
            #pragma unroll
            for (int u = 0; u < RED_CHUNK; u++) {
                if (j0 + u >= c) break;
                const double x = fabs(vb[u]);
                cc += signbit(vb[u]) ? 1 : 0;
                if (j0 + u == 0) sv = 0.0 + x;
                else {
                    const double t = sv + x;
                    if (fabs(sv) >= fabs(x)) sc += (sv - t) + x;
                    else                     sc += (x - t) + sv;
                    sv = t;
                }
                nv = nv + x;
            }
        }
        const double s = (sc != 0.0 && isfinite(sc)) ? sv + sc : sv;
        const double mean = s / (double)c;
        double vf = 0.0, vc = 0.0;
        for (int j0 = 0; j0 < c; j0 += RED_CHUNK) {
            double vb[RED_CHUNK];
            #pragma unroll
            for (int u = 0; u < RED_CHUNK; u++) vb[u] = j0 + u < c ? rec[s0 + j0 + u] : 0.0;
            #pragma unroll
            for (int u = 0; u < RED_CHUNK; u++) {
                if (j0 + u >= c) break;
                const double dx = fabs(vb[u]) - mean;
                const double v = dx * dx;                    // (x - mean) ** 2
                if (j0 + u == 0) vf = 0.0 + v;
                else {
                    const double t = vf + v;
                    if (fabs(vf) >= fabs(v)) vc += (vf - t) + v;
                    else                     vc += (v - t) + vf;
                    vf = t;
                }
            }
        }
        const double vs = (vc != 0.0 && isfinite(vc)) ? vf + vc : vf;
        naive[f] = nv;
        if (p.outputs & GFQ_WANT_STATS) {
            p.f_count[fo + f] = c;
            p.f_mean[fo + f] = mean;
            p.f_var[fo + f] = c > 1 ? vs / (double)(c - 1) : 0.0;
            p.f_cold[fo + f] = 100.0 * (double)cc / (double)c;
        }
    }
    __syncwarp();
    // weighted_avg_latency: builtin sum over functions in first-completion
    // order.  The record scratch is free again: mark each function at its
    // first completion index, then read the marks in order.
    int* mark = (int*)rec;
    for (int k = lane; k < nrec; k += 32) mark[k] = -1;
    __syncwarp();
    for (int f = lane; f < nf; f += 32) if (cnt[f] > 0) mark[first[f]] = f;
    __syncwarp();
    int nfirst = 0;
    for (int b0 = 0; b0 < nrec; b0 += 32) {
        const int k = b0 + lane;
        const int f = k < nrec ? mark[k] : -1;
        const unsigned hit = __ballot_sync(FULLMASK, f >= 0);
        if (f >= 0) order[nfirst + __popc(hit & ((1u << lane) - 1))] = f;
        nfirst += __popc(hit);
    }
    __syncwarp();
    PySum num; ps_init(num);
    for (int r = 0; r < nfirst; r++) {
        int f = order[r];
        double nn = (double)cnt[f];
        ps_add(num, nn * (naive[f] / nn));
    }
    if (lane == 0) {
        double* smy = p.summary + (int64_t)sid * 3;
        smy[0] = nrec > 0 ? ps_val(num) / (double)nrec : 0.0;
        smy[1] = nrec > 0 ? 100.0 * ((double)colds / (double)nrec) : 0.0;
    }
}


// Per-simulation member setup (every thread that touches the simulation).
template <int POL, bool ND1, bool CTA, bool FG>
__device__ __forceinline__ void sim_setup(WarpSim<POL, ND1, CTA, FG>& w, const Params& p, int sid) {
    constexpr bool G = POL == PB_GENERIC;
    const gfq_sim* sim = p.sims + sid;
    w.sim = sim;
    const int t = sim->trace;
    w.toff = p.trace_off[t];
    w.n = (int)(p.trace_off[t + 1] - w.toff);
    w.nf = p.trace_nf[t];
    w.foff = p.foff + p.foff_off[t];
    w.tb = (int)p.tab_off[sim->flowtab];
    w.mem_int = w.nf > 0 && __ldg(p.memi + w.tb) >= 0;
    w.roff = p.sim_roff[sid];
    w.policy = sim->policy;
    w.scripted_ = sim->device_model == GFQ_DEVMODEL_SCRIPTED;
    w.mqfq_ = sim->policy == GFQ_POLICY_MQFQ;
    w.fcfs_ = sim->policy == GFQ_POLICY_FCFS || sim->policy == GFQ_POLICY_FCFS_NAIVE;
    const bool scripted = G && w.scripted_;
    w.ndev = scripted ? 1 : sim->n_devices;
    w.T = sim->t_overrun; w.alpha = sim->alpha; w.dttl = sim->default_ttl_s;
    w.tau_inc = sim->tau_includes_overheads != 0;
}

// Zero the per-flow state and container counts (threads t, t+st, ...).
template <int POL, bool ND1, bool CTA, bool FG>
__device__ __forceinline__ void sim_reset_flows(WarpSim<POL, ND1, CTA, FG>& w, const Params& p, int t, int st) {
    double *vt = w.vt(), *lex = w.lex(), *tau = w.tau(), *iat = w.iat(), *larr = w.larr();
    auto *pt = w.pt(), *ph = w.ph(), *infl = w.infl(), *head = w.head(), *done = w.done(), *pend = w.pend();
    uint8_t* fst = w.fst();
    for (int f = t; f < w.nf; f += st) {
        vt[f] = 0.0; lex[f] = 0.0; tau[f] = 0.0; iat[f] = 0.0; larr[f] = 0.0;
        pt[f] = 0; ph[f] = 0; infl[f] = 0; head[f] = (typename WarpSim<POL, ND1, CTA, FG>::CI)-1; done[f] = 0; pend[f] = 0; fst[f] = 0;
    }
    uint16_t* cnt = (uint16_t*)(w.fe + p.L.o_cnt);
    for (int i = t; i < 3 * w.ndev * p.L.F; i += st) cnt[i] = 0;
    if (p.L.o_lst) {
        double* lst = (double*)(w.fe + p.L.o_lst);
        for (int f = t; f < w.nf; f += st) lst[f] = 0.0;
    }
    if (p.L.o_bmin) {
        double* bmin = (double*)(w.fe + p.L.o_bmin);
        for (int i = t; i < p.L.F / 32; i += st) bmin[i] = __longlong_as_double(0x7ff0000000000000ll);
    }
}

// Device state reset, the event loop and the per-simulation outputs (one warp).
template <int POL, bool ND1, bool CTA, bool FG>
__device__ __forceinline__ void sim_run(WarpSim<POL, ND1, CTA, FG>& w, const Params& p, int sid) {
    constexpr bool G = POL == PB_GENERIC;
    const gfq_sim* sim = w.sim;
    const int lane = w.lane;
    unsigned char* base = w.sm;
    const bool scripted = G && w.scripted_;
#if GFQ_TIMELINE
    unsigned long long tl0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl0));
#endif
    {
        if (lane < w.ndev) {
            int d = lane;
            int* dvi = (int*)(base + p.L.o_dvi) + d * DV_NI;
            double* dvd = (double*)(base + p.L.o_dvd) + d * DD_ND;
            for (int k = 0; k < DV_NI; k++) dvi[k] = 0;
            for (int k = 0; k < DD_ND; k++) dvd[k] = 0.0;
            if (scripted) {
                dvi[DV_DMAX] = sim->scripted_d; dvi[DV_EFFD] = sim->scripted_d; dvi[DV_HROK] = 1;
            } else {
                const gfq_device_cfg& c = p.dcfg[sim->device_cfg + d];
                dvi[DV_DMAX] = c.d_max; dvi[DV_EFFD] = c.d_max;
                dvi[DV_POOLMAX] = c.pool_max_containers; dvi[DV_POOLON] = c.pool_enabled != 0;
                dvi[DV_DYN] = c.dynamic_d != 0;
                dvd[DD_MEMCAP] = c.mem_capacity_mb; dvd[DD_THR] = c.util_threshold;
                dvd[DD_PCIE] = c.pcie_mb_per_s; dvd[DD_BETA] = c.interference_beta;
                dvd[DD_WINDOW] = c.util_window_s; dvd[DD_OVERLAP] = c.prefetch_overlap_s;
                dvd[DD_INVDMAX] = 1.0 / (double)c.d_max;
                dvi[DV_HROK] = !(0.0 + dvd[DD_INVDMAX] > c.util_threshold);
                dvi[DV_INSTDIRTY] = 1;                // intern the idle utilization 0.0
                dvi[DV_LKEY] = -1;                              // no previous window
                uint32_t* wk = (uint32_t*)(base + p.L.o_wkey) + d * WMEMO;
                for (int k = 0; k < WMEMO; k++) wk[k] = 0xffffffffu;   // no valid key has all bits set
                u64* wd = (u64*)(base + p.L.o_wdict) + d * WDICT;
                for (int k = 0; k < WDICT; k++) wd[k] = ~0ull;   // empty intern slots
            }
        }
        uint32_t* dg = (uint32_t*)(base + p.L.o_diag);
        if (lane < DG_N) dg[lane] = 0;
        __syncwarp();
        if (ND1) {                                 // device 0's mutable state -> registers
            const int* dvi = (const int*)(base + p.L.o_dvi);
            const double* dvd = (const double*)(base + p.L.o_dvd);
#pragma unroll
            for (int k = 0; k < DV_NSTATE; k++) w.hv[k] = dvi[k];
#pragma unroll
            for (int k = 0; k < DD_NSTATE; k++) w.hd[k] = dvd[k];
            w.win0 = dvd[DD_WINDOW];
        }
    }
    w.period = 0.0;
    if (!scripted) {                                   // engine.py:80-81
        w.period = p.dcfg[sim->device_cfg].monitor_period_s;
        for (int d = 1; d < w.ndev; d++) w.period = pymin(w.period, p.dcfg[sim->device_cfg + d].monitor_period_s);
    }
    w.now = 0.0; w.gvt = 0.0;
    w.seq = (uint32_t)w.n;
    w.cursor = 0; w.nev = 0;
    // an absent tick / pooled event keeps its time at +inf (event selection)
    w.tick_on = false; w.tick_t = __longlong_as_double(0x7ff0000000000000ll); w.tick_seq = 0;
    w.pmin_ok = true; w.pmin_t = __longlong_as_double(0x7ff0000000000000ll); w.pmin_seq = 0; w.pmin_slot = -1;
    w.tot_pend = 0; w.tot_infl = 0;
    w.fcfs_head = 0; w.fcfs_infl = 0; w.draining = -1;
    w.s_att = 0; w.s_out = 0; w.s_exec = 0;
    w.status = 0; w.any_newly = false; w.newly_n = 0;
    w.gmin_ok = false; w.gmin = ~0ull;
    w.idle_lb = __longlong_as_double(0x7ff0000000000000ll);
    w.n_events = 0;
    w.n_calls = w.n_disp = w.n_comp = w.n_util = w.n_backlog = w.n_evlog = 0;
    w.n_evict = 0;
    w.nbl = 0;
    ps_init(w.util_sum);

    // Simulation.__init__, engine.py:70-78: arrivals own seq 0..n-1, the first
    // tick (only when the trace is non-empty) seq n
    if (w.n > 0 && !scripted) w.push_tick(w.period);

    w.run();
    if (CTA) w.cta_release();

    if (lane == 0) {
        p.status[sid] = w.status;
        p.summary[(int64_t)sid * 3 + 2] = w.n_util ? ps_val(w.util_sum) / (double)w.n_util : 0.0;
        int64_t* c = p.counters + (int64_t)sid * GFQ_NCOUNTERS;
        c[C_EVENTS] = w.n_events; c[C_CALLS] = w.n_calls; c[C_DISP] = w.n_disp; c[C_UTIL] = w.n_util;
        const uint32_t* dg = (const uint32_t*)(base + p.L.o_diag);
        c[C_MAXEV] = dg[DG_MAXEV]; c[C_GSCAN] = dg[DG_GSCAN]; c[C_RSCAN] = dg[DG_RSCAN];
        c[C_CSCAN] = dg[DG_CSCAN]; c[C_TICKS] = dg[DG_TICKS]; c[C_WHIT] = dg[DG_WHIT];
        c[C_WMISS] = dg[DG_WMISS]; c[C_QUIET] = dg[DG_QUIET];
#if GFQ_PROF
        // -DGFQ_PROF=1 diagnostic build: cycles per phase (PF_*) in counters 5..11
        for (int k = 0; k < 7; k++) c[C_GSCAN + k] = dg[DG_P0 + k];
#endif
#if GFQ_TIMELINE
        // -DGFQ_TIMELINE=1 diagnostic build: start / end (ns) and SM of each simulation
        unsigned long long tl1; unsigned smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl1));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        c[C_GSCAN] = (int64_t)tl0; c[C_RSCAN] = (int64_t)tl1; c[C_CSCAN] = smid;
#endif
        p.final_time[sid] = w.now;
        if (p.outputs & GFQ_WANT_AUDIT) p.backlog_count[sid] = w.n_backlog;
        if (p.outputs & GFQ_WANT_EVENTS) p.event_count[sid] = w.n_evlog;
        if (p.outputs & GFQ_WANT_EVICTIONS) p.evict_count[sid] = w.n_evict;
        if ((p.outputs & GFQ_WANT_AUDIT) && !w.status &&
            (w.n_backlog > p.audit_backlog_cap || w.n_util > p.audit_util_cap))
            p.status[sid] = GFQ_SIM_OUTPUT_OVERFLOW;
        if ((p.outputs & GFQ_WANT_EVENTS) && !w.status && w.n_evlog > p.event_log_cap)
            p.status[sid] = GFQ_SIM_OUTPUT_OVERFLOW;
    }
    __syncwarp();
}

template <int POL, bool ND1, bool FG>
__device__ __forceinline__ void run_one(const Params& p, unsigned char* base, unsigned char* fe,
                                        int lane, int sid) {
    WarpSim<POL, ND1, false, FG> w(p, base, fe, lane, sid);
    sim_setup(w, p, sid);
    sim_reset_flows(w, p, lane, 32);
    __syncwarp();
    sim_run(w, p, sid);
}

#ifndef GFQ_MINB
#define GFQ_MINB 4
#endif
#ifndef GFQ_KTHREADS                      // k_sim block size bound (simulations per CTA x 32)
#define GFQ_KTHREADS 128
#endif

#ifndef GFQ_MINB_FG                       // flows-in-global builds (L2-latency bound)
#define GFQ_MINB_FG GFQ_MINB
#endif

#ifndef GFQ_MINB_FAST                     // 1-device warp classes (u16 per-flow state)
#define GFQ_MINB_FAST GFQ_MINB
#endif

template <int POL, bool ND1, bool FG>
__global__ void __launch_bounds__(GFQ_KTHREADS, FG ? GFQ_MINB_FG : (ND1 && POL != PB_GENERIC) ? GFQ_MINB_FAST : GFQ_MINB) k_sim(const __grid_constant__ Params p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* slice = smem + (size_t)warp * p.L.bytes;
    // FG: the flow/event part lives in this warp's global scratch slice
    unsigned char* fe = FG ? p.gscratch + (size_t)(blockIdx.x * (blockDim.x >> 5) + warp) * p.L.fe_bytes
                           : slice;
    unsigned char* base = FG ? slice : slice + p.L.fe_bytes;
    for (;;) {
        int idx = 0;
        if (lane == 0) idx = atomicAdd(p.work, 1);
        idx = __shfl_sync(FULLMASK, idx, 0);
        if (idx >= p.n_sims) break;
        run_one<POL, ND1, FG>(p, base, fe, lane, p.order[idx]);
    }
}

// CTA-per-simulation engine for large flow counts (BASELINE C4: 4096
// functions): one simulation per CTA, its whole workspace in the CTA's shared
// memory (or the flow/event part in a per-CTA global slice, FG).  Warp 0 runs
// the event loop; warps 1.. serve its flow scans and event-pool argmins
// (WarpSim::cta_scan / helper_loop, named barriers 1 and 2).
template <int POL, bool ND1, bool FG>
__global__ void __launch_bounds__(GFQ_CTA_THREADS, 1) k_sim_cta(const __grid_constant__ Params p) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_idx;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* fe = FG ? p.gscratch + (size_t)blockIdx.x * p.L.fe_bytes : smem;
    unsigned char* base = FG ? smem : smem + p.L.fe_bytes;
    if (warp == 0) ring_init(base, p.L, lane);
    for (;;) {
        if (threadIdx.x == 0) s_idx = atomicAdd(p.work, 1);
        __syncthreads();
        const int idx = s_idx;
        __syncthreads();
        if (idx >= p.n_sims) break;
        const int sid = p.order[idx];
        WarpSim<POL, ND1, true, FG> w(p, base, fe, lane, sid);
        w.wid = warp; w.nthr = blockDim.x; w.use_inf_ = 0;
        sim_setup(w, p, sid);
        sim_reset_flows(w, p, threadIdx.x, blockDim.x);
        __syncthreads();
        if (warp == 0) sim_run(w, p, sid);
        else w.helper_loop();
        __syncthreads();
    }
}

// Result reducer: one warp per finished simulation, over its completion
// stream (comp_lat / comp_meta, written in completion order by k_sim).
template <bool FG>
__global__ void __launch_bounds__(128) k_reduce(const __grid_constant__ Params p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const size_t scratch = (size_t)RED_FLOW_BYTES * p.L.F;
    unsigned char* base = FG ? p.gscratch + (size_t)(blockIdx.x * wpb + warp) * scratch
                             : smem + (size_t)warp * scratch;
    double* rec = p.rscratch + (size_t)(blockIdx.x * wpb + warp) * p.rscratch_per_warp;
    for (int sid = blockIdx.x * wpb + warp; sid < p.n_sims; sid += gridDim.x * wpb)
        if (p.status[sid] == GFQ_SIM_OK) reduce_one(p, base, rec, lane, sid);
}

// Trace validation (Simulation.__init__, engine.py:50-52,72-73), one block
// per trace: the smallest (trace, position, check) failure wins (atomicMin on
// trace << 29 | position << 2 | check; checks: 0 flow id out of range,
// 1 decreasing time, 2 non-finite or negative time -- a sequential scan's order).
__global__ void k_validate_traces(const double* arrival, const int32_t* flow, const int64_t* trace_off,
                                  const int32_t* trace_nf, unsigned long long* err) {
    const int t = blockIdx.x;
    const int64_t a = trace_off[t], b = trace_off[t + 1];
    const int nf = trace_nf[t];
    for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
        int kind = -1;
        const int f = flow[i];
        const double x = arrival[i];
        if (f < 0 || f >= nf) kind = 0;
        else if (i > a && x < arrival[i - 1]) kind = 1;
        else if (!(x >= 0.0) || !isfinite(x)) kind = 2;
        if (kind >= 0)
            atomicMin(err, ((unsigned long long)t << 29) | ((unsigned long long)(i - a) << 2) | (unsigned)kind);
    }
}

// Trace loader: one warp per trace.  Counting sort of trace positions by
// flow rank, stable (arrival order kept within a flow) via __match_any_sync.
__global__ void k_trace_index(const int32_t* flow, const int64_t* trace_off, const int32_t* trace_nf,
                              const int64_t* foff_off, int32_t* foff, int32_t* fpos, int n_traces) {
    extern __shared__ int cursor[];
    const int t = blockIdx.x;
    if (t >= n_traces) return;
    const int lane = threadIdx.x;
    const int64_t toff = trace_off[t];
    const int n = (int)(trace_off[t + 1] - toff);
    const int nf = trace_nf[t];
    const int32_t* fl = flow + toff;
    int32_t* fo = foff + foff_off[t];
    int32_t* fp = fpos + toff;
    for (int f = lane; f <= nf; f += 32) cursor[f] = 0;
    __syncwarp();
    for (int i = lane; i < n; i += 32) atomicAdd(&cursor[fl[i]], 1);
    __syncwarp();
    if (lane == 0) {
        int acc = 0;
        for (int f = 0; f < nf; f++) { int c = cursor[f]; cursor[f] = acc; fo[f] = acc; acc += c; }
        fo[nf] = acc;
    }
    __syncwarp();
    for (int b = 0; b < n; b += 32) {
        int i = b + lane;
        bool act = i < n;
        unsigned am = __ballot_sync(FULLMASK, act);
        if (act) {
            int f = fl[i];
            unsigned peers = __match_any_sync(am, f);
            int rank = __popc(peers & ((1u << lane) - 1));
            int pos = cursor[f] + rank;
            fp[pos] = i;
            __syncwarp(am);
            if (lane == 31 - __clz(peers)) cursor[f] += __popc(peers);
        }
        __syncwarp();
    }
}

}  // namespace gfq

// ============================================================================
// host side

using namespace gfq;

// the k_sim instantiation of each kernel class (see gfq_prepare)
// CTA-mode classes: 6 generic, 7 MQFQ-Sticky and 8 FCFS on a 1-device DeviceSet
// class 6: MQFQ-Sticky on a 1-device DeviceSet with the audit / event / eviction logs
enum { NCLASS = 10, CLASS_MQFQ_LOG = 6, CLASS_CTA = 7, CLASS_CTA_MQFQ1 = 8, CLASS_CTA_FCFS1 = 9 };
static inline bool is_cta_class(int k) { return k >= CLASS_CTA; }
static const void* class_kernel(int k, bool flows_global) {
    switch (k) {
        case CLASS_CTA: return flows_global ? (const void*)k_sim_cta<PB_GENERIC, false, true>
                                            : (const void*)k_sim_cta<PB_GENERIC, false, false>;
        case CLASS_CTA_MQFQ1: return flows_global ? (const void*)k_sim_cta<PB_MQFQ, true, true>
                                                  : (const void*)k_sim_cta<PB_MQFQ, true, false>;
        case CLASS_CTA_FCFS1: return flows_global ? (const void*)k_sim_cta<PB_FCFS, true, true>
                                                  : (const void*)k_sim_cta<PB_FCFS, true, false>;
        case 1: return (const void*)k_sim<PB_MQFQ, false, false>;
        case 2: return flows_global ? (const void*)k_sim<PB_MQFQ, true, true>
                                    : (const void*)k_sim<PB_MQFQ, true, false>;
        case 3: return flows_global ? (const void*)k_sim<PB_FCFS, true, true>
                                    : (const void*)k_sim<PB_FCFS, true, false>;
        case 4: return (const void*)k_sim<PB_BATCH, true, false>;
        case 5: return (const void*)k_sim<PB_SJF, true, false>;
        case CLASS_MQFQ_LOG: return (const void*)k_sim<PB_MQFQ_LOG, true, false>;
        default: return flows_global ? (const void*)k_sim<PB_GENERIC, false, true>
                                     : (const void*)k_sim<PB_GENERIC, false, false>;
    }
}


namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) { g_err = msg; return code; }

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return set_err(GFQ_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct DBuf {
    void* p = nullptr;
    size_t cap = 0;
    int ensure(size_t bytes) {
        if (bytes <= cap && p) return GFQ_OK;
        if (p) cudaFree(p);
        p = nullptr; cap = 0;
        size_t b = std::max<size_t>(bytes, 16);
        cudaError_t e = cudaMalloc(&p, b);
        if (e != cudaSuccess) return set_err(GFQ_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        cap = b;
        return GFQ_OK;
    }
    void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    template <class T> T* as() const { return (T*)p; }
};

}  // namespace

struct gfq_handle {
    int device = 0;
    int n_sm = 0;
    size_t smem_optin = 0;
    size_t smem_per_sm = 0;
    // traces
    DBuf arrival, flow, trace_off, trace_nf, foff_off, foff, fpos;
    std::vector<int64_t> h_trace_off;
    std::vector<int32_t> h_trace_nf;
    int32_t n_traces = 0;
    // flow tables
    DBuf warm, cold, mem, share, weight, hist_row, tab_off;
    DBuf memi;                      // mem_mb as integer MB per row; -1 for every row of a table that is not integral
    std::vector<int64_t> h_tab_off;
    std::vector<char> h_tab_int;    // per flow table: every mem_mb integral (memi valid)
    std::vector<double> h_mem;
    int32_t n_tabs = 0;
    // device configs, scripted execs
    DBuf dcfg, execs;
    std::vector<gfq_device_cfg> h_dcfg;
    int64_t n_execs = 0;
    // staged batch
    DBuf sims, order, sim_foff, sim_roff, work;
    std::vector<gfq_sim> h_sims;
    std::vector<int64_t> h_sim_foff, h_sim_roff;
    int32_t n_sims = 0;
    gfq_launch_cfg cfg{};
    Layout L{};
    int wpb = 0, rwpb = 4, rblocks = 1;
    int cta_threads = 0, cta_min = GFQ_CTA_MIN;
    bool rglobal = false;
    int ccount[NCLASS] = {0}, cblocks[NCLASS] = {0};   // per kernel class
    Layout Lk[NCLASS] = {};                              // per-class workspace layout
    bool prepared = false;
    DBuf out[GFQ_OUT_COUNT_];
    int64_t out_n[GFQ_OUT_COUNT_] = {0};
    int32_t out_b[GFQ_OUT_COUNT_] = {0};
    DBuf comp_lat, comp_meta, comp_pos, gscratch, fscratch, rscr, verr;
    int64_t rscr_per_warp = 1;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    // kernel classes run concurrently on side streams (fork/join on the
    // caller's stream), so one class's tail overlaps the next class's start
    cudaStream_t side[16] = {};
    cudaEvent_t fork = nullptr, join[16] = {};
    std::vector<cudaEvent_t> ring;          // GFQ_TIMING_RING x 3 events
    int ring_next = 0, ring_count = 0;
    cudaStream_t last_stream = nullptr;
    // host<->device copies of the per-batch API calls: a non-blocking stream,
    // ordered after this handle's last launch (ev[2]) and synchronised before
    // each call returns, so a call on one handle overlaps kernels of another
    // (the e2e pipeline double-buffers two handles)
    cudaStream_t xfer = nullptr;
    bool launched = false;
};

static const int32_t kOutBytes[GFQ_OUT_COUNT_] = {
    4, 8, 8, 8, 8, 8, 8, 8,   // status counters final summary fcount fmean fvar fcold
    8, 8, 1, 1, 4, 8,         // rec dispatch complete state device order pure
    4, 8, 8, 4, 4,            // dsp inv vt gvt qlen infl
    8, 4, 8, 4, 8,            // util rows/meta, backlog time/meta/count
    8, 8, 8,                  // event time/meta/count
    8,                        // hist
    8, 8, 8, 8,               // fairness rows/meta/offsets/counts
    8, 4, 8,                  // eviction log time/meta/count
    4, 4,                     // dispatch-row / eviction-row event index
    8};                       // start tags

extern "C" {

const char* gfq_last_error(void) { return g_err.c_str(); }
int gfq_abi_version(void) { return GFQ_ABI_VERSION; }

int gfq_create(int device, gfq_handle** out) {
    if (!out) return set_err(GFQ_EINVAL, "gfq_create: out is NULL");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return set_err(GFQ_EINVAL, "gfq_create: no such CUDA device");
    CK(cudaSetDevice(device));
    int major = 0, minor = 0;
    CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    if (major != 10 || minor != 0)
        return set_err(GFQ_ECUDA, "gfq_create: libgfq.so is built for sm_100a (B200) only");
    gfq_handle* h = new gfq_handle();
    h->device = device;
    CK(cudaDeviceGetAttribute(&h->n_sm, cudaDevAttrMultiProcessorCount, device));
    int optin = 0;
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    h->smem_optin = (size_t)optin;
    int per_sm_smem = 0;
    CK(cudaDeviceGetAttribute(&per_sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device));
    h->smem_per_sm = (size_t)per_sm_smem;
    for (auto& e : h->ev) CK(cudaEventCreate(&e));
    h->ring.resize(3 * GFQ_TIMING_RING);
    for (auto& e : h->ring) CK(cudaEventCreate(&e));
    CK(cudaStreamCreateWithFlags(&h->xfer, cudaStreamNonBlocking));
    *out = h;
    return GFQ_OK;
}

int gfq_destroy(gfq_handle* h) {
    if (!h) return GFQ_OK;
    cudaSetDevice(h->device);
    DBuf* all[] = {&h->gscratch, &h->fscratch, &h->rscr, &h->verr, &h->comp_pos, &h->arrival, &h->flow, &h->trace_off, &h->trace_nf, &h->foff_off, &h->foff,
                   &h->fpos, &h->warm, &h->cold, &h->mem, &h->share, &h->weight, &h->hist_row,
                   &h->tab_off, &h->dcfg, &h->execs, &h->sims, &h->order, &h->sim_foff,
                   &h->sim_roff, &h->work, &h->comp_lat, &h->comp_meta};
    for (DBuf* b : all) b->release();
    for (auto& b : h->out) b.release();
    for (auto& e : h->ev) if (e) cudaEventDestroy(e);
    for (auto& e : h->ring) if (e) cudaEventDestroy(e);
    for (auto& e : h->join) if (e) cudaEventDestroy(e);
    if (h->fork) cudaEventDestroy(h->fork);
    for (auto& q : h->side) if (q) cudaStreamDestroy(q);
    if (h->xfer) cudaStreamDestroy(h->xfer);
    delete h;
    return GFQ_OK;
}

static int index_traces(gfq_handle* h, const int64_t* off, const int32_t* n_flows, int32_t n_traces,
                        const std::vector<int64_t>& foff_off, int32_t max_nf);

int gfq_upload_traces(gfq_handle* h, const double* arrival, const int32_t* flow,
                      const int64_t* off, const int32_t* n_flows, int32_t n_traces) {
    if (!h || n_traces < 0 || (n_traces > 0 && (!off || !n_flows)))
        return set_err(GFQ_EINVAL, "gfq_upload_traces: bad arguments");
    CK(cudaSetDevice(h->device));
    CK(cudaStreamWaitEvent(h->xfer, h->ev[2], 0));      // after this handle's last launch
    if (off[0] != 0) return set_err(GFQ_EINVAL, "gfq_upload_traces: off[0] must be 0");
    int64_t total = n_traces ? off[n_traces] : 0;
    int32_t max_nf = 1;
    std::vector<int64_t> foff_off(n_traces + 1, 0);
    for (int t = 0; t < n_traces; t++) {
        int64_t a = off[t], b = off[t + 1];
        if (b < a) return set_err(GFQ_EINVAL, "gfq_upload_traces: offsets must be non-decreasing");
        if (b - a >= (1 << 27)) return set_err(GFQ_EINVAL, "gfq_upload_traces: trace longer than 2^27 arrivals");
        if (n_flows[t] < 0 || n_flows[t] > 0xffff)
            return set_err(GFQ_EINVAL, "gfq_upload_traces: n_flows out of range");
        foff_off[t + 1] = foff_off[t] + n_flows[t] + 1;
        max_nf = std::max(max_nf, n_flows[t]);
    }
    int rc;
    // padded to whole 32-entry chunks: k_sim streams the traces in by TMA
    // bulk copies of aligned 32-entry chunks (WarpSim::ring_issue)
    const int64_t padded = ((total + 31) & ~(int64_t)31) + 32;
    if ((rc = h->arrival.ensure(8 * padded)) || (rc = h->flow.ensure(4 * padded)) ||
        (rc = h->fpos.ensure(4 * total)) || (rc = h->trace_off.ensure(8 * (n_traces + 1))) ||
        (rc = h->trace_nf.ensure(4 * std::max(n_traces, 1))) ||
        (rc = h->foff_off.ensure(8 * (n_traces + 1))) || (rc = h->foff.ensure(4 * foff_off[n_traces])))
        return rc;
    if (total) {
        CK(cudaMemcpyAsync(h->arrival.p, arrival, 8 * total, cudaMemcpyHostToDevice, h->xfer));
        CK(cudaMemcpyAsync(h->flow.p, flow, 4 * total, cudaMemcpyHostToDevice, h->xfer));
    }
    CK(cudaMemcpyAsync(h->trace_off.p, off, 8 * (n_traces + 1), cudaMemcpyHostToDevice, h->xfer));
    if (n_traces) CK(cudaMemcpyAsync(h->trace_nf.p, n_flows, 4 * n_traces, cudaMemcpyHostToDevice, h->xfer));
    // per-arrival validation (engine.py:50-52,72-73) on the GPU; the first
    // failure in (trace, position, check) order is the one reported, as a
    // sequential scan would.  On failure no traces stay resident.
    if (total) {
        if ((rc = h->verr.ensure(8))) return rc;
        CK(cudaMemsetAsync(h->verr.p, 0xff, 8, h->xfer));
        k_validate_traces<<<n_traces, 256, 0, h->xfer>>>(h->arrival.as<double>(), h->flow.as<int32_t>(), h->trace_off.as<int64_t>(),
                                             h->trace_nf.as<int32_t>(), h->verr.as<unsigned long long>());
        CK(cudaGetLastError());
        unsigned long long e = 0;
        CK(cudaMemcpyAsync(&e, h->verr.p, 8, cudaMemcpyDeviceToHost, h->xfer));
        CK(cudaStreamSynchronize(h->xfer));
        if (e != ~0ull) {
            const int t = (int)(e >> 29), kind = (int)(e & 3);
            h->n_traces = 0; h->h_trace_off.assign(1, 0); h->h_trace_nf.clear(); h->prepared = false;
            if (kind == 0) return set_err(GFQ_EINVAL, "gfq_upload_traces: flow id out of range in trace " + std::to_string(t));
            if (kind == 1) return set_err(GFQ_EINVAL, "trace arrival times must be non-decreasing (trace " + std::to_string(t) + ")");
            return set_err(GFQ_EINVAL, "gfq_upload_traces: arrival times must be finite and >= 0");
        }
    }
    return index_traces(h, off, n_flows, n_traces, foff_off, max_nf);
}

// Per-flow arrival index of the resident traces (k_trace_index) and the
// host-side trace table; arrival / flow / trace_off / trace_nf are on the device.
static int index_traces(gfq_handle* h, const int64_t* off, const int32_t* n_flows, int32_t n_traces,
                        const std::vector<int64_t>& foff_off, int32_t max_nf) {
    CK(cudaMemcpyAsync(h->foff_off.p, foff_off.data(), 8 * (n_traces + 1), cudaMemcpyHostToDevice, h->xfer));
    if (n_traces) {
        size_t sm = 4 * ((size_t)max_nf + 1);
        if (sm > 48 * 1024) CK(cudaFuncSetAttribute(k_trace_index, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k_trace_index<<<n_traces, 32, sm, h->xfer>>>(h->flow.as<int32_t>(), h->trace_off.as<int64_t>(),
                                            h->trace_nf.as<int32_t>(), h->foff_off.as<int64_t>(),
                                            h->foff.as<int32_t>(), h->fpos.as<int32_t>(), n_traces);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(h->xfer));
    h->h_trace_off.assign(off, off + n_traces + 1);
    h->h_trace_nf.assign(n_flows, n_flows + n_traces);
    h->n_traces = n_traces;
    h->prepared = false;
    return GFQ_OK;
}

int gfq_generate_traces(gfq_handle* h, int32_t n_traces, const int32_t* n_functions,
                        const double* rates, const int32_t* name_rank, const double* duration_s,
                        const uint64_t* seed, uint8_t* touched, int64_t* trace_off_out) {
    if (!h || n_traces < 0 || (n_traces > 0 && (!n_functions || !rates || !name_rank || !duration_s || !seed)))
        return set_err(GFQ_EINVAL, "gfq_generate_traces: bad arguments");
    CK(cudaSetDevice(h->device));
    CK(cudaStreamWaitEvent(0, h->ev[2], 0));   // legacy-stream work after this handle's last launch
    // streams of a trace in name order: stream (t, j) is the function whose
    // name rank is j, so a stable sort by time gives (t, name) order
    std::vector<int64_t> fn_off(n_traces + 1, 0);
    for (int t = 0; t < n_traces; t++) {
        if (n_functions[t] < 1 || n_functions[t] > 0xffff)
            return set_err(GFQ_EINVAL, "n_functions must be in [1, 65535]");
        if (!isfinite(duration_s[t]))        // (a negative duration gives an empty trace, as in gen_zipf)
            return set_err(GFQ_EINVAL, "gfq_generate_traces: duration must be finite");
        fn_off[t + 1] = fn_off[t] + n_functions[t];
    }
    const int64_t nfn = fn_off[n_traces];
    std::vector<int32_t> st(nfn), sf(nfn), sr(nfn);
    for (int t = 0; t < n_traces; t++) {
        const int64_t a = fn_off[t];
        const int n = n_functions[t];
        std::vector<int32_t> inv(n, -1);
        for (int k = 0; k < n; k++) {
            const int r = name_rank[a + k];
            if (r < 0 || r >= n || inv[r] >= 0) return set_err(GFQ_EINVAL, "gfq_generate_traces: name_rank is not a permutation");
            if (!(rates[a + k] > 0) || !isfinite(rates[a + k])) return set_err(GFQ_EINVAL, "total_rate_rps must be > 0");
            inv[r] = k;
        }
        for (int j = 0; j < n; j++) { st[a + j] = t; sf[a + j] = inv[j]; sr[a + j] = j; }
    }
    DBuf d_st, d_sf, d_sr, d_fo, d_rt, d_du, d_sd, d_cnt, d_oo, d_k0, d_k1, d_v0, d_v1, d_tmp, d_map, d_tch;
    int rc;
    const size_t ns = (size_t)std::max<int64_t>(nfn, 1);
    if ((rc = d_st.ensure(4 * ns)) || (rc = d_sf.ensure(4 * ns)) || (rc = d_sr.ensure(4 * ns)) ||
        (rc = d_fo.ensure(8 * (n_traces + 1))) || (rc = d_rt.ensure(8 * ns)) ||
        (rc = d_du.ensure(8 * std::max(n_traces, 1))) || (rc = d_sd.ensure(8 * std::max(n_traces, 1))) ||
        (rc = d_cnt.ensure(8 * ns)) || (rc = d_oo.ensure(8 * ns)) || (rc = d_map.ensure(4 * ns)) ||
        (rc = d_tch.ensure(ns)))
        return rc;
    if (nfn) {
        CK(cudaMemcpy(d_st.p, st.data(), 4 * nfn, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_sf.p, sf.data(), 4 * nfn, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_sr.p, sr.data(), 4 * nfn, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_rt.p, rates, 8 * nfn, cudaMemcpyHostToDevice));
    }
    CK(cudaMemcpy(d_fo.p, fn_off.data(), 8 * (n_traces + 1), cudaMemcpyHostToDevice));
    if (n_traces) {
        CK(cudaMemcpy(d_du.p, duration_s, 8 * n_traces, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(d_sd.p, seed, 8 * n_traces, cudaMemcpyHostToDevice));
    }
    GenParams g{};
    g.n_streams = (int32_t)nfn;
    g.stream_trace = d_st.as<int32_t>(); g.stream_fn = d_sf.as<int32_t>(); g.stream_rank = d_sr.as<int32_t>();
    g.fn_off = d_fo.as<int64_t>(); g.rates = d_rt.as<double>(); g.duration = d_du.as<double>();
    g.seed = d_sd.as<unsigned long long>(); g.count = d_cnt.as<int64_t>(); g.out_off = d_oo.as<int64_t>();
    const int gb = (int)((nfn + 127) / 128);
    // pass 1: arrivals per stream
    if (nfn) { k_gen_streams<<<gb, 128>>>(g, 0); CK(cudaGetLastError()); }
    std::vector<int64_t> cnt(nfn), oo(nfn), toff(n_traces + 1, 0);
    if (nfn) CK(cudaMemcpy(cnt.data(), d_cnt.p, 8 * nfn, cudaMemcpyDeviceToHost));
    int64_t total = 0;
    for (int t = 0; t < n_traces; t++) {
        for (int64_t i = fn_off[t]; i < fn_off[t + 1]; i++) { oo[i] = total; total += cnt[i]; }
        toff[t + 1] = total;
        if (toff[t + 1] - toff[t] >= (1 << 27)) return set_err(GFQ_EINVAL, "gfq_generate_traces: trace longer than 2^27 arrivals");
    }
    if (total >= ((int64_t)1 << 31)) return set_err(GFQ_EINVAL, "gfq_generate_traces: more than 2^31 arrivals in one call");
    const size_t na = (size_t)std::max<int64_t>(total, 1);
    if ((rc = d_k0.ensure(8 * na)) || (rc = d_k1.ensure(8 * na)) || (rc = d_v0.ensure(4 * na)) || (rc = d_v1.ensure(4 * na)))
        return rc;
    if (nfn) CK(cudaMemcpy(d_oo.p, oo.data(), 8 * nfn, cudaMemcpyHostToDevice));
    g.key = d_k0.as<unsigned long long>(); g.val = d_v0.as<int32_t>();
    // pass 2: arrival times (rounded) + name ranks, streams in name order
    if (nfn) { k_gen_streams<<<gb, 128>>>(g, 1); CK(cudaGetLastError()); }
    // the engine's trace buffers (padded to whole 32-entry chunks, see upload)
    const int64_t padded = ((total + 31) & ~(int64_t)31) + 32;
    if ((rc = h->arrival.ensure(8 * padded)) || (rc = h->flow.ensure(4 * padded)) ||
        (rc = h->fpos.ensure(4 * std::max<int64_t>(total, 1))) || (rc = h->trace_off.ensure(8 * (n_traces + 1))) ||
        (rc = h->trace_nf.ensure(4 * std::max(n_traces, 1))))
        return rc;
    CK(cudaMemcpy(h->trace_off.p, toff.data(), 8 * (n_traces + 1), cudaMemcpyHostToDevice));
    if (total) {
        // stable sort of each trace by time (the fp64 bit pattern of t >= 0)
        size_t tmp = 0;
        CK(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tmp, d_k0.as<unsigned long long>(), d_k1.as<unsigned long long>(),
                                                    d_v0.as<int32_t>(), d_v1.as<int32_t>(), (int)total, n_traces,
                                                    h->trace_off.as<int64_t>(), h->trace_off.as<int64_t>() + 1));
        if ((rc = d_tmp.ensure(tmp))) return rc;
        CK(cub::DeviceSegmentedRadixSort::SortPairs(d_tmp.p, tmp, d_k0.as<unsigned long long>(), d_k1.as<unsigned long long>(),
                                                    d_v0.as<int32_t>(), d_v1.as<int32_t>(), (int)total, n_traces,
                                                    h->trace_off.as<int64_t>(), h->trace_off.as<int64_t>() + 1));
    }
    if (n_traces) {
        k_gen_flows<<<n_traces, 256>>>(d_k1.as<unsigned long long>(), d_v1.as<int32_t>(), h->trace_off.as<int64_t>(),
                                       d_fo.as<int64_t>(), d_map.as<int32_t>(), h->arrival.as<double>(),
                                       h->flow.as<int32_t>(), h->trace_nf.as<int32_t>(), d_tch.as<uint8_t>());
        CK(cudaGetLastError());
    }
    std::vector<int32_t> nfl(std::max(n_traces, 1));
    std::vector<uint8_t> tch(ns);
    if (n_traces) CK(cudaMemcpy(nfl.data(), h->trace_nf.p, 4 * n_traces, cudaMemcpyDeviceToHost));
    if (nfn) CK(cudaMemcpy(tch.data(), d_tch.p, nfn, cudaMemcpyDeviceToHost));
    std::vector<int64_t> foff_off(n_traces + 1, 0);
    int32_t max_nf = 1;
    for (int t = 0; t < n_traces; t++) {
        foff_off[t + 1] = foff_off[t] + nfl[t] + 1;
        max_nf = std::max(max_nf, nfl[t]);
        if (touched)                          // back to the caller's function order
            for (int64_t k = fn_off[t]; k < fn_off[t + 1]; k++) touched[k] = tch[fn_off[t] + name_rank[k]];
    }
    if ((rc = h->foff_off.ensure(8 * (n_traces + 1))) || (rc = h->foff.ensure(4 * std::max<int64_t>(foff_off[n_traces], 1))))
        return rc;
    if (trace_off_out) memcpy(trace_off_out, toff.data(), 8 * (n_traces + 1));
    rc = index_traces(h, toff.data(), nfl.data(), n_traces, foff_off, max_nf);
    for (DBuf* b : {&d_st, &d_sf, &d_sr, &d_fo, &d_rt, &d_du, &d_sd, &d_cnt, &d_oo, &d_k0, &d_k1, &d_v0, &d_v1, &d_tmp, &d_map, &d_tch})
        b->release();
    return rc;
}

int gfq_download_traces(gfq_handle* h, double* arrival, int32_t* flow, int64_t total) {
    if (!h || total < 0) return set_err(GFQ_EINVAL, "gfq_download_traces: bad arguments");
    const int64_t have = h->h_trace_off.empty() ? 0 : h->h_trace_off.back();
    if (total != have) return set_err(GFQ_EINVAL, "gfq_download_traces: total does not match the resident traces");
    CK(cudaSetDevice(h->device));
    CK(cudaStreamWaitEvent(0, h->ev[2], 0));   // legacy-stream work after this handle's last launch
    if (total && arrival) CK(cudaMemcpy(arrival, h->arrival.p, 8 * total, cudaMemcpyDeviceToHost));
    if (total && flow) CK(cudaMemcpy(flow, h->flow.p, 4 * total, cudaMemcpyDeviceToHost));
    return GFQ_OK;
}

int gfq_upload_flowtabs(gfq_handle* h, const double* warm_s, const double* cold_s,
                        const double* mem_mb, const double* compute_share,
                        const double* weight, const int32_t* hist_row,
                        const int64_t* off, int32_t n_tabs) {
    if (!h || n_tabs < 0 || !off) return set_err(GFQ_EINVAL, "gfq_upload_flowtabs: bad arguments");
    CK(cudaSetDevice(h->device));
    int64_t total = off[n_tabs];
    if (total >= 0x7fffffff) return set_err(GFQ_EINVAL, "gfq_upload_flowtabs: more than 2^31 flow-table rows");
    for (int64_t i = 0; i < total; i++) {       // FunctionProfile validation, core.py:41-51
        if (!(warm_s[i] > 0)) return set_err(GFQ_EINVAL, "warm_exec_s must be > 0");
        if (!(cold_s[i] >= warm_s[i])) return set_err(GFQ_EINVAL, "cold_exec_s must be >= warm_exec_s");
        if (!(mem_mb[i] > 0)) return set_err(GFQ_EINVAL, "mem_mb must be > 0");
        if (!(compute_share[i] > 0 && compute_share[i] <= 1)) return set_err(GFQ_EINVAL, "compute_share must be in (0, 1]");
        if (!(weight[i] > 0)) return set_err(GFQ_EINVAL, "weight must be > 0");
    }
    CK(cudaStreamWaitEvent(h->xfer, h->ev[2], 0));      // after this handle's last launch
    int rc;
    if ((rc = h->warm.ensure(8 * total)) || (rc = h->cold.ensure(8 * total)) ||
        (rc = h->mem.ensure(8 * total)) || (rc = h->share.ensure(8 * total)) ||
        (rc = h->weight.ensure(8 * total)) || (rc = h->hist_row.ensure(4 * total)) ||
        (rc = h->memi.ensure(4 * total)) ||
        (rc = h->tab_off.ensure(8 * (n_tabs + 1))))
        return rc;
    if (total) {
        CK(cudaMemcpyAsync(h->warm.p, warm_s, 8 * total, cudaMemcpyHostToDevice, h->xfer));
        CK(cudaMemcpyAsync(h->cold.p, cold_s, 8 * total, cudaMemcpyHostToDevice, h->xfer));
        CK(cudaMemcpyAsync(h->mem.p, mem_mb, 8 * total, cudaMemcpyHostToDevice, h->xfer));
        CK(cudaMemcpyAsync(h->share.p, compute_share, 8 * total, cudaMemcpyHostToDevice, h->xfer));
        CK(cudaMemcpyAsync(h->weight.p, weight, 8 * total, cudaMemcpyHostToDevice, h->xfer));
        if (hist_row) CK(cudaMemcpyAsync(h->hist_row.p, hist_row, 4 * total, cudaMemcpyHostToDevice, h->xfer));
        else CK(cudaMemsetAsync(h->hist_row.p, 0, 4 * total, h->xfer));
    }
    // Integral tables: every mem_mb an integer in [1, 2^20].  Then every partial
    // sum of resident_mb (device.py:114-117) is an integer far below 2^53, each
    // float addition is exact and CPython's compensated sum() equals the exact
    // integer total in any order, so the engine sums them lane-parallel.
    std::vector<int32_t> memi(total);
    std::vector<char> tab_int(n_tabs);
    for (int32_t t = 0; t < n_tabs; t++) {
        bool integral = true;
        for (int64_t i = off[t]; i < off[t + 1]; i++)
            integral = integral && mem_mb[i] <= 1048576.0 && mem_mb[i] == floor(mem_mb[i]);
        for (int64_t i = off[t]; i < off[t + 1]; i++) memi[i] = integral ? (int32_t)mem_mb[i] : -1;
        tab_int[t] = integral;
    }
    if (total) CK(cudaMemcpyAsync(h->memi.p, memi.data(), 4 * total, cudaMemcpyHostToDevice, h->xfer));
    CK(cudaMemcpyAsync(h->tab_off.p, off, 8 * (n_tabs + 1), cudaMemcpyHostToDevice, h->xfer));
    CK(cudaStreamSynchronize(h->xfer));
    h->h_tab_off.assign(off, off + n_tabs + 1);
    h->h_tab_int = tab_int;
    h->h_mem.assign(mem_mb, mem_mb + total);
    h->n_tabs = n_tabs;
    h->prepared = false;
    return GFQ_OK;
}

int gfq_upload_device_cfgs(gfq_handle* h, const gfq_device_cfg* cfgs, int32_t n) {
    if (!h || n < 0 || (n > 0 && !cfgs)) return set_err(GFQ_EINVAL, "gfq_upload_device_cfgs: bad arguments");
    for (int i = 0; i < n; i++) {               // DeviceConfig validation, device.py:36-48
        const gfq_device_cfg& c = cfgs[i];
        if (!(c.util_threshold > 0 && c.util_threshold <= 1)) return set_err(GFQ_EINVAL, "util_threshold must be in (0, 1]");
        if (c.d_max < 1) return set_err(GFQ_EINVAL, "d_max must be >= 1");
        if (!(c.mem_capacity_mb > 0) || !(c.pcie_mb_per_s > 0) || !(c.monitor_period_s > 0) || !(c.util_window_s > 0))
            return set_err(GFQ_EINVAL, "device capacities and periods must be > 0");
        if (c.pool_max_containers < 1) return set_err(GFQ_EINVAL, "pool_max_containers must be >= 1");
        if (!(c.interference_beta >= 0)) return set_err(GFQ_EINVAL, "interference_beta must be >= 0");
    }
    CK(cudaSetDevice(h->device));
    CK(cudaStreamWaitEvent(h->xfer, h->ev[2], 0));
    int rc = h->dcfg.ensure(sizeof(gfq_device_cfg) * std::max(n, 1));
    if (rc) return rc;
    if (n) CK(cudaMemcpyAsync(h->dcfg.p, cfgs, sizeof(gfq_device_cfg) * n, cudaMemcpyHostToDevice, h->xfer));
    CK(cudaStreamSynchronize(h->xfer));
    h->h_dcfg.assign(cfgs, cfgs + n);
    h->prepared = false;
    return GFQ_OK;
}

int gfq_upload_execs(gfq_handle* h, const double* execs, int64_t n) {
    if (!h || n < 0 || (n > 0 && !execs)) return set_err(GFQ_EINVAL, "gfq_upload_execs: bad arguments");
    CK(cudaSetDevice(h->device));
    CK(cudaStreamWaitEvent(h->xfer, h->ev[2], 0));
    int rc = h->execs.ensure(8 * std::max<int64_t>(n, 1));
    if (rc) return rc;
    if (n) CK(cudaMemcpyAsync(h->execs.p, execs, 8 * n, cudaMemcpyHostToDevice, h->xfer));
    CK(cudaStreamSynchronize(h->xfer));
    h->n_execs = n;
    h->prepared = false;
    return GFQ_OK;
}

static int alloc_out(gfq_handle* h, int id, int64_t n) {
    int rc = h->out[id].ensure((size_t)std::max<int64_t>(n, 1) * kOutBytes[id]);
    if (rc) return rc;
    h->out_n[id] = n;
    h->out_b[id] = kOutBytes[id];
    return GFQ_OK;
}

int gfq_prepare(gfq_handle* h, const gfq_sim* sims, int32_t n_sims, const gfq_launch_cfg* cfg) {
    if (!h || n_sims < 0 || (n_sims > 0 && !sims) || !cfg) return set_err(GFQ_EINVAL, "gfq_prepare: bad arguments");
    CK(cudaSetDevice(h->device));
    h->prepared = false;
    gfq_launch_cfg c = *cfg;
    if (c.outputs & GFQ_WANT_DISPATCH) c.outputs |= GFQ_WANT_RECORDS;   // rows read dispatch_s
    int max_nf = 1, nd = 1, P = 1, R = 1, S = 4, max_n = 0;
    std::unordered_map<int64_t, double> maxmem;
    int64_t flows = 0, recs = 0;
    std::vector<int64_t> foffs(n_sims + 1, 0), roffs(n_sims + 1, 0);
    std::vector<double> cost(n_sims);
    for (int i = 0; i < n_sims; i++) {
        const gfq_sim& s = sims[i];
        auto who = [i]() { return "sim " + std::to_string(i) + ": "; };   // built only on error
        if (s.trace < 0 || s.trace >= h->n_traces) return set_err(GFQ_EINVAL, who() + "trace id out of range");
        if (s.flowtab < 0 || s.flowtab >= h->n_tabs) return set_err(GFQ_EINVAL, who() + "flow table id out of range");
        if (s.policy < 0 || s.policy > GFQ_POLICY_FCFS_NAIVE) return set_err(GFQ_EINVAL, who() + "unknown policy");
        if (!(s.t_overrun >= 0)) return set_err(GFQ_EINVAL, who() + "t_overrun must be >= 0");
        if (!(s.alpha >= 0)) return set_err(GFQ_EINVAL, "alpha must be >= 0");
        int nf = h->h_trace_nf[s.trace];
        int64_t n = h->h_trace_off[s.trace + 1] - h->h_trace_off[s.trace];
        int64_t tabn = h->h_tab_off[s.flowtab + 1] - h->h_tab_off[s.flowtab];
        if (tabn < nf) return set_err(GFQ_EINVAL, who() + "flow table shorter than the trace's flow set");
        if (s.device_model == GFQ_DEVMODEL_SCRIPTED) {
            if (s.scripted_d < 1 || s.exec_len < 1 || s.exec_off < 0 || s.exec_off + s.exec_len > h->n_execs)
                return set_err(GFQ_EINVAL, who() + "bad scripted-device parameters");
            R = std::max(R, s.scripted_d);
        } else if (s.device_model == GFQ_DEVMODEL_DEVICESET) {
            if (s.n_devices < 1 || s.n_devices > GFQ_MAX_DEVICES)
                return set_err(GFQ_EINVAL, who() + "n_devices must be in [1, 8]");
            if (s.device_cfg < 0 || s.device_cfg + s.n_devices > (int)h->h_dcfg.size())
                return set_err(GFQ_EINVAL, who() + "device config range out of bounds");
            nd = std::max(nd, s.n_devices);
            double period = h->h_dcfg[s.device_cfg].monitor_period_s;
            for (int d = 0; d < s.n_devices; d++) period = std::min(period, h->h_dcfg[s.device_cfg + d].monitor_period_s);
            const int64_t tb = h->h_tab_off[s.flowtab];
            for (int d = 0; d < s.n_devices; d++) {
                const gfq_device_cfg& dc = h->h_dcfg[s.device_cfg + d];
                R = std::max(R, dc.d_max);
                if (dc.pool_enabled) P = std::max(P, dc.pool_max_containers + 1);
                S = std::max(S, (int)ceil(dc.util_window_s / period) + 3);
                // the reference never terminates otherwise; the
                // table's max over the trace's flows is computed once per (table, nf)
                const int64_t mk = ((int64_t)s.flowtab << 20) | nf;
                auto it = maxmem.find(mk);
                if (it == maxmem.end()) {
                    double m = -INFINITY;
                    for (int f = 0; f < nf; f++) m = std::max(m, h->h_mem[tb + f]);
                    it = maxmem.emplace(mk, m).first;
                }
                if (it->second > dc.mem_capacity_mb)
                    return set_err(GFQ_EINVAL, who() + "a function's mem_mb exceeds the device's mem_capacity_mb");
            }
        } else {
            return set_err(GFQ_EINVAL, who() + "unknown device model");
        }
        max_nf = std::max(max_nf, nf);
        max_n = std::max<int>(max_n, (int)n);
        foffs[i + 1] = foffs[i] + nf;
        roffs[i + 1] = roffs[i] + n;
        // LPT cost estimate: events grow with the trace, the flow scans with
        // nf, and the backlog (hence the simulated span and its monitor
        // ticks) shrinks with the device concurrency
        int dsum = 0;
        if (s.device_model == GFQ_DEVMODEL_SCRIPTED) dsum = s.scripted_d;
        else for (int d = 0; d < s.n_devices; d++) dsum += h->h_dcfg[s.device_cfg + d].d_max;
        cost[i] = (double)n * (1.0 + nf / 32.0) * (s.policy == GFQ_POLICY_MQFQ ? 2.0 : 1.0) *
                  (1.0 + 1.0 / (double)std::max(dsum, 1));
    }
    flows = foffs[n_sims]; recs = roffs[n_sims];
    Layout L{};
    L.F = (max_nf + 31) & ~31;
    L.ND = nd; L.P = P; L.R = R; L.S = S;
    L.E = c.event_capacity > 0 ? c.event_capacity : std::max(64, ((2 * max_nf + 2 * R * nd + 32) + 31) & ~31);
    L.flows_global = 0;
    L.cta = 0;
    // records with the logs: every simulation runs the generic build, which
    // then also keeps FlowQueue.last_start_tag and writes each start tag
    L.lst = (c.outputs & GFQ_WANT_RECORDS) &&
            (c.outputs & (GFQ_WANT_AUDIT | GFQ_WANT_EVENTS | GFQ_WANT_EVICTIONS));
    layout_finish(L);
    // Large flow counts (fewer than 4 warp-simulations' workspaces fit an SM's
    // shared memory, or GFQ_FLAG_CTA): one simulation per CTA, its scans split
    // over the CTA's warps.  The CTA gets 512 threads (256 when two such
    // simulations fit an SM).
    //
    // Unless the batch is large: then the warp build with the flow state in
    // global scratch (16 simulations per SM instead of 1-2) finishes first.
    // Measured on BASELINE C4 (4096 functions, ~2.1k touched): a warp
    // simulation takes ~6x as long as a CTA one, so the warp build wins once
    // the CTA build would need more than 6 waves per warp-build wave
    // (2368 simulations: 23M vs 9M dispatches/s).  GFQ_FLAG_CTA / GFQ_FLAG_WARP
    // force either.
    int cta_threads = 0;
    const bool big = (size_t)4 * L.bytes > h->smem_optin;    // warp build: flows in global scratch
    if (!(c.flags & GFQ_FLAG_WARP) && ((c.flags & GFQ_FLAG_CTA) || big)) {
        Layout Lc = L;
        Lc.cta = 1;
        layout_finish(Lc);
        const int cta_per_sm = (size_t)2 * Lc.bytes <= h->smem_optin ? 2 : 1;
        const long long cta_waves = (n_sims + (long long)cta_per_sm * h->n_sm - 1) / ((long long)cta_per_sm * h->n_sm);
        const long long warp_waves = (n_sims + 16ll * h->n_sm - 1) / (16ll * h->n_sm);
        if ((c.flags & GFQ_FLAG_CTA) || cta_waves <= 6 * warp_waves) {
            L = Lc;
            cta_threads = cta_per_sm == 2 ? 256 : GFQ_CTA_THREADS;
        }
    }
    // flow counts whose per-simulation state does not fit in shared memory
    // (or GFQ_FLAG_FLOWS_GLOBAL) put the flow/event part in global scratch
    const size_t smem_avail = h->smem_optin - (L.cta ? 64 : 0);     // CTA mode: + static s_idx
    // CTA mode: rather than spill the flow state to global memory, trim the
    // default event capacity (2 slots per flow) to what fits, down to 1 slot
    // per flow + 2 per token + 64; a simulation that still overflows reports
    // GFQ_SIM_EVENT_OVERFLOW (callers re-run it with a larger event_capacity)
    if (L.cta && c.event_capacity <= 0 && (size_t)L.bytes > smem_avail) {
        const int32_t over = (int32_t)(((size_t)L.bytes - smem_avail + 15) / 16);
        const int32_t e_fit = (L.E - over) & ~31;
        if (e_fit >= max_nf + 2 * R * nd + 64) {
            L.E = e_fit;
            layout_finish(L);
        }
    }
    if ((c.flags & GFQ_FLAG_FLOWS_GLOBAL) || (size_t)L.bytes > smem_avail || (big && !L.cta)) {
        L.flows_global = 1;
        layout_finish(L);
    }
    if ((size_t)L.bytes > h->smem_optin)
        return set_err(GFQ_EINVAL, "gfq_prepare: per-simulation workspace (" + std::to_string(L.bytes) +
                                       " B) exceeds shared memory; reduce flows/pool/event capacity");
    // Kernel classes (one launch each over its slice of the work order):
    //   0 generic (any policy, scripted devices, audit / event logs, large F)
    //   1 MQFQ-Sticky on a multi-device DeviceSet
    //   2..5 one policy (MQFQ / FCFS / Batch / SJF) on a 1-device DeviceSet
    //        (flows in global scratch: MQFQ / FCFS only)
    const bool logs = (c.outputs & (GFQ_WANT_AUDIT | GFQ_WANT_EVENTS | GFQ_WANT_EVICTIONS)) != 0;
    std::vector<int> cls(n_sims);
    int ccount[NCLASS] = {0};
    for (int i = 0; i < n_sims; i++) {
        const gfq_sim& s = sims[i];
        int k = 0;
        // the 1-device fast classes sum resident memory as integers only
        // (WarpSim::MEMI): a table with a non-integral mem_mb runs generic
        const bool fast1 = !logs && s.device_model == GFQ_DEVMODEL_DEVICESET && s.n_devices == 1 &&
                           h->h_tab_int[s.flowtab];
        if (L.cta) {
            k = CLASS_CTA;
            if (fast1) {
                if (s.policy == GFQ_POLICY_MQFQ) k = CLASS_CTA_MQFQ1;
                else if (s.policy == GFQ_POLICY_FCFS || s.policy == GFQ_POLICY_FCFS_NAIVE) k = CLASS_CTA_FCFS1;
            }
        } else if (logs && s.device_model == GFQ_DEVMODEL_DEVICESET) {
            // the logs asked for (run_simulation, Simulation, the CLI): MQFQ-Sticky
            // on one device has its own build, with the same u16 / integral rules
            const int64_t tn = h->h_trace_off[s.trace + 1] - h->h_trace_off[s.trace];
            if (s.policy == GFQ_POLICY_MQFQ && s.n_devices == 1 && h->h_tab_int[s.flowtab] &&
                !L.flows_global && tn < 65535)
                k = CLASS_MQFQ_LOG;
        } else if (!logs && s.device_model == GFQ_DEVMODEL_DEVICESET) {
            // (and, with the flow state in shared memory, u16 per-flow counters:
            // traces under 65535 arrivals)
            const int64_t tn = h->h_trace_off[s.trace + 1] - h->h_trace_off[s.trace];
            if (fast1 && (L.flows_global || tn < 65535)) {
                k = s.policy == GFQ_POLICY_MQFQ ? 2
                  : (s.policy == GFQ_POLICY_FCFS || s.policy == GFQ_POLICY_FCFS_NAIVE) ? 3
                  : s.policy == GFQ_POLICY_BATCH ? 4 : 5;
                if (L.flows_global && k > 3) k = 0;       // flows in global: MQFQ / FCFS builds only
            } else if (s.policy == GFQ_POLICY_MQFQ && !L.flows_global) {
                k = 1;
            }
        }
        cls[i] = k;
        ccount[k]++;
    }
    int wpb = c.warps_per_block > 0 ? std::min(c.warps_per_block, GFQ_KTHREADS / 32) : GFQ_KTHREADS / 32;
    while (wpb > 1 && (size_t)wpb * L.bytes > h->smem_optin) wpb--;
    if (L.cta) wpb = 1;                       // one simulation (workspace) per CTA
    int cblocks[NCLASS] = {0};
    // Per-class layouts: FCFS / Batch / SJF on one device (classes 3-5) never
    // pool keep-alive expiries, so their dynamic events are completions, one
    // per token at most; their smaller workspace raises their occupancy
    // (C2: 18.8 -> 13.9 KB per simulation, 12 -> 16 warps per SM).
    Layout Lk[NCLASS];
    for (int k = 0; k < NCLASS; k++) Lk[k] = L;
    if (!L.cta && !L.flows_global)
        for (int k = 2; k <= CLASS_MQFQ_LOG; k++) { Lk[k].i16 = 1; layout_finish(Lk[k]); }
    if (!L.cta && !L.flows_global && c.event_capacity <= 0) {
        const int32_t e_tok = std::max(64, (2 * R * nd + 32 + 31) & ~31);
        for (int k = 3; k <= 5; k++)
            if (e_tok < L.E) { Lk[k].E = e_tok; layout_finish(Lk[k]); }
    }
    for (int k = 0; k < NCLASS; k++) {
        if (!ccount[k]) continue;
        const void* kfn = class_kernel(k, L.flows_global);
        const size_t smem = (size_t)(is_cta_class(k) ? 1 : wpb) * Lk[k].bytes;
        const int threads = is_cta_class(k) ? cta_threads : wpb * 32;
        const int per_cta = is_cta_class(k) ? 1 : wpb;   // simulations in flight per CTA
        CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        // all of the unified L1/shared array to shared memory: occupancy is bounded
        // by per-warp simulation state; the kernel's global traffic is tiny
        CK(cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                (int)cudaSharedmemCarveoutMaxShared));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, threads, smem));
        if (per_sm < 1) return set_err(GFQ_EINVAL, "gfq_prepare: kernel does not fit on an SM");
        // then give the rest of the unified array back to L1: the read-only
        // flow tables, per-flow arrival index and trace windows of an SM's
        // simulations stay L1-resident instead of costing an L2 round trip
        // on every dispatch
        {
            const double need = (double)per_sm * (double)(smem + 1024);
            int pct = (int)ceil(100.0 * need / (double)h->smem_per_sm);
            pct = std::min(100, std::max(pct, 1));
            CK(cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
            int per_sm2 = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, kfn, threads, smem));
            if (per_sm2 < per_sm)                 // keep the occupancy
                CK(cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        (int)cudaSharedmemCarveoutMaxShared));
        }
        int blocks = c.blocks > 0 ? c.blocks : per_sm * h->n_sm;
        cblocks[k] = std::max(1, std::min(blocks, (ccount[k] + per_cta - 1) / per_cta));
    }
    // reducer: 60 B of scratch per flow per warp, shared memory or global
    int rwpb = 4;
    const bool rglobal = L.flows_global || (size_t)RED_FLOW_BYTES * L.F > h->smem_optin;
    if (!rglobal) while (rwpb > 1 && (size_t)rwpb * RED_FLOW_BYTES * L.F > h->smem_optin) rwpb--;
    int red_per_sm = 8;
    if (!rglobal) {
        CK(cudaFuncSetAttribute(k_reduce<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(rwpb * RED_FLOW_BYTES * L.F)));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&red_per_sm, k_reduce<false>, rwpb * 32,
                                                         (size_t)rwpb * RED_FLOW_BYTES * L.F));
    } else {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&red_per_sm, k_reduce<true>, rwpb * 32, 0));
    }
    int rblocks = std::max(1, std::min((n_sims + rwpb - 1) / rwpb, std::max(red_per_sm, 1) * h->n_sm));
    if (!rglobal)
        CK(cudaFuncSetAttribute(k_reduce<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(rwpb * RED_FLOW_BYTES * L.F)));
    size_t gscr = 0;
    if (L.flows_global)
        for (int k = 0; k < NCLASS; k++) gscr = std::max(gscr, (size_t)cblocks[k] * (is_cta_class(k) ? 1 : wpb) * L.fe_bytes);
    if (rglobal) gscr = std::max(gscr, (size_t)rblocks * rwpb * RED_FLOW_BYTES * L.F);
    const int64_t rper = std::max(max_n, 1);              // reducer record scratch per warp

    int rc;
    if ((rc = h->sims.ensure(sizeof(gfq_sim) * std::max(n_sims, 1))) || (rc = h->order.ensure(4 * std::max(n_sims, 1))) ||
        (rc = h->sim_foff.ensure(8 * (n_sims + 1))) || (rc = h->sim_roff.ensure(8 * (n_sims + 1))) ||
        (rc = h->work.ensure(4 * NCLASS)) || (rc = h->comp_lat.ensure(8 * std::max<int64_t>(recs, 1))) ||
        (rc = h->comp_meta.ensure(4 * std::max<int64_t>(recs, 1))) ||
        (gscr && (rc = h->gscratch.ensure(gscr))) ||
        (rc = h->comp_pos.ensure(4 * std::max<int64_t>(recs, 1))) ||
        (rc = h->rscr.ensure((size_t)8 * rblocks * rwpb * rper)))
        return rc;
    for (int id = 0; id < GFQ_OUT_COUNT_; id++) h->out_n[id] = 0;
    if ((rc = alloc_out(h, GFQ_OUT_STATUS, n_sims)) || (rc = alloc_out(h, GFQ_OUT_COUNTERS, (int64_t)GFQ_NCOUNTERS * n_sims)) ||
        (rc = alloc_out(h, GFQ_OUT_FINAL_TIME, n_sims)) || (rc = alloc_out(h, GFQ_OUT_SUMMARY, 3ll * n_sims)))
        return rc;
    if (c.outputs & GFQ_WANT_STATS)
        for (int id : {GFQ_OUT_FLOW_COUNT, GFQ_OUT_FLOW_MEAN, GFQ_OUT_FLOW_VAR, GFQ_OUT_FLOW_COLD_PCT})
            if ((rc = alloc_out(h, id, flows))) return rc;
    if (c.outputs & GFQ_WANT_RECORDS)
        for (int id : {GFQ_OUT_REC_DISPATCH, GFQ_OUT_REC_COMPLETE, GFQ_OUT_REC_STATE, GFQ_OUT_REC_DEVICE,
                       GFQ_OUT_REC_ORDER, GFQ_OUT_REC_PURE, GFQ_OUT_REC_START_TAG})
            if ((rc = alloc_out(h, id, recs))) return rc;
    if (c.outputs & GFQ_WANT_DISPATCH)
        for (int id : {GFQ_OUT_DSP_INV, GFQ_OUT_DSP_VT_BEFORE, GFQ_OUT_DSP_GVT, GFQ_OUT_DSP_QLEN, GFQ_OUT_DSP_INFLIGHT,
                       GFQ_OUT_DSP_EVENT})
            if ((rc = alloc_out(h, id, recs))) return rc;
    if (c.outputs & GFQ_WANT_AUDIT) {
        if (c.audit_util_cap <= 0) c.audit_util_cap = 1 << 16;
        if (c.audit_backlog_cap <= 0) c.audit_backlog_cap = 2 * (int64_t)max_n + 2;
        if ((rc = alloc_out(h, GFQ_OUT_UTIL_ROWS, (int64_t)n_sims * c.audit_util_cap * 3)) ||
            (rc = alloc_out(h, GFQ_OUT_UTIL_META, (int64_t)n_sims * c.audit_util_cap * 2)) ||
            (rc = alloc_out(h, GFQ_OUT_BACKLOG_TIME, (int64_t)n_sims * c.audit_backlog_cap)) ||
            (rc = alloc_out(h, GFQ_OUT_BACKLOG_META, (int64_t)n_sims * c.audit_backlog_cap)) ||
            (rc = alloc_out(h, GFQ_OUT_BACKLOG_COUNT, n_sims)))
            return rc;
    }
    if (c.outputs & GFQ_WANT_EVICTIONS)
        if ((rc = alloc_out(h, GFQ_OUT_EVICT_TIME, recs)) || (rc = alloc_out(h, GFQ_OUT_EVICT_META, recs)) ||
            (rc = alloc_out(h, GFQ_OUT_EVICT_EVENT, recs)) ||
            (rc = alloc_out(h, GFQ_OUT_EVICT_COUNT, n_sims)))
            return rc;
    if (c.outputs & GFQ_WANT_EVENTS) {
        if (c.event_log_cap <= 0) c.event_log_cap = 64 * (int64_t)max_n + 1024;
        if ((rc = alloc_out(h, GFQ_OUT_EVENT_TIME, (int64_t)n_sims * c.event_log_cap)) ||
            (rc = alloc_out(h, GFQ_OUT_EVENT_META, (int64_t)n_sims * c.event_log_cap)) ||
            (rc = alloc_out(h, GFQ_OUT_EVENT_COUNT, n_sims)))
            return rc;
    }
    if (c.outputs & GFQ_WANT_HIST) {
        if (c.hist_groups < 1 || c.hist_rows < 1 || c.hist_bins < 1 || !(c.hist_lo_s > 0) || !(c.hist_hi_s > c.hist_lo_s))
            return set_err(GFQ_EINVAL, "gfq_prepare: bad histogram parameters");
        if ((rc = alloc_out(h, GFQ_OUT_HIST, (int64_t)c.hist_groups * c.hist_rows * c.hist_bins))) return rc;
        for (int i = 0; i < n_sims; i++) if (sims[i].group >= c.hist_groups)
            return set_err(GFQ_EINVAL, "gfq_prepare: sim group out of range");
    }
    // longest-first work order (LPT) for the persistent work queue
    // per class, longest first (LPT) for the persistent work queues
    std::vector<int32_t> order(n_sims);
    for (int i = 0; i < n_sims; i++) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        return cls[a] != cls[b] ? cls[a] < cls[b] : cost[a] > cost[b]; });
    CK(cudaStreamWaitEvent(h->xfer, h->ev[2], 0));      // after this handle's last launch
    if (n_sims) {
        CK(cudaMemcpyAsync(h->sims.p, sims, sizeof(gfq_sim) * n_sims, cudaMemcpyHostToDevice, h->xfer));
        CK(cudaMemcpyAsync(h->order.p, order.data(), 4 * n_sims, cudaMemcpyHostToDevice, h->xfer));
    }
    CK(cudaMemcpyAsync(h->sim_foff.p, foffs.data(), 8 * (n_sims + 1), cudaMemcpyHostToDevice, h->xfer));
    CK(cudaMemcpyAsync(h->sim_roff.p, roffs.data(), 8 * (n_sims + 1), cudaMemcpyHostToDevice, h->xfer));
    CK(cudaStreamSynchronize(h->xfer));
    h->h_sims.assign(sims, sims + n_sims);
    h->h_sim_foff = foffs; h->h_sim_roff = roffs;
    h->n_sims = n_sims;
    h->cfg = c;
    h->L = L;
    h->wpb = wpb;
    h->cta_threads = cta_threads;
    h->cta_min = (c.flags & GFQ_FLAG_CTA) ? 0 : GFQ_CTA_MIN;
    h->rwpb = rwpb;
    h->rblocks = rblocks;
    h->rglobal = rglobal;
    h->rscr_per_warp = rper;
    for (int k = 0; k < NCLASS; k++) { h->ccount[k] = ccount[k]; h->cblocks[k] = cblocks[k]; h->Lk[k] = Lk[k]; }
    h->prepared = true;
    h->launched = false;
    return GFQ_OK;
}

int gfq_sim_offsets(gfq_handle* h, int64_t* flow_off, int64_t* rec_off) {
    if (!h || !h->prepared) return set_err(GFQ_EINVAL, "gfq_sim_offsets: no staged batch");
    if (flow_off) memcpy(flow_off, h->h_sim_foff.data(), 8 * (h->n_sims + 1));
    if (rec_off) memcpy(rec_off, h->h_sim_roff.data(), 8 * (h->n_sims + 1));
    return GFQ_OK;
}

static Params make_params(gfq_handle* h) {
    Params p{};
    p.sims = h->sims.as<gfq_sim>(); p.order = h->order.as<int32_t>(); p.n_sims = h->n_sims;
    p.arrival = h->arrival.as<double>(); p.flow = h->flow.as<int32_t>();
    p.trace_off = h->trace_off.as<int64_t>(); p.trace_nf = h->trace_nf.as<int32_t>();
    p.foff_off = h->foff_off.as<int64_t>(); p.foff = h->foff.as<int32_t>(); p.fpos = h->fpos.as<int32_t>();
    p.warm = h->warm.as<double>(); p.cold = h->cold.as<double>(); p.mem = h->mem.as<double>();
    p.memi = h->memi.as<int32_t>();
    p.share = h->share.as<double>(); p.weight = h->weight.as<double>();
    p.hist_row = h->hist_row.as<int32_t>(); p.tab_off = h->tab_off.as<int64_t>();
    p.dcfg = h->dcfg.as<gfq_device_cfg>(); p.execs = h->execs.as<double>();
    p.sim_foff = h->sim_foff.as<int64_t>(); p.sim_roff = h->sim_roff.as<int64_t>();
    p.L = h->L;
    p.cta_min = h->cta_min;
    p.outputs = h->cfg.outputs;
    p.early_exit = h->cfg.early_exit;
    p.status = h->out[GFQ_OUT_STATUS].as<int32_t>();
    p.counters = h->out[GFQ_OUT_COUNTERS].as<int64_t>();
    p.final_time = h->out[GFQ_OUT_FINAL_TIME].as<double>();
    p.summary = h->out[GFQ_OUT_SUMMARY].as<double>();
    p.f_count = h->out[GFQ_OUT_FLOW_COUNT].as<int64_t>();
    p.f_mean = h->out[GFQ_OUT_FLOW_MEAN].as<double>();
    p.f_var = h->out[GFQ_OUT_FLOW_VAR].as<double>();
    p.f_cold = h->out[GFQ_OUT_FLOW_COLD_PCT].as<double>();
    p.comp_lat = h->comp_lat.as<double>(); p.comp_meta = h->comp_meta.as<int32_t>();
    p.comp_pos = h->comp_pos.as<int32_t>();
    p.rscratch = h->rscr.as<double>(); p.rscratch_per_warp = h->rscr_per_warp;
    p.rec_dispatch = h->out[GFQ_OUT_REC_DISPATCH].as<double>();
    p.rec_complete = h->out[GFQ_OUT_REC_COMPLETE].as<double>();
    p.rec_pure = h->out[GFQ_OUT_REC_PURE].as<double>();
    p.rec_stag = h->out[GFQ_OUT_REC_START_TAG].as<double>();
    p.rec_state = h->out[GFQ_OUT_REC_STATE].as<int8_t>();
    p.rec_device = h->out[GFQ_OUT_REC_DEVICE].as<int8_t>();
    p.rec_order = h->out[GFQ_OUT_REC_ORDER].as<int32_t>();
    p.dsp_inv = h->out[GFQ_OUT_DSP_INV].as<int32_t>();
    p.dsp_vt = h->out[GFQ_OUT_DSP_VT_BEFORE].as<double>();
    p.dsp_gvt = h->out[GFQ_OUT_DSP_GVT].as<double>();
    p.dsp_qlen = h->out[GFQ_OUT_DSP_QLEN].as<int32_t>();
    p.dsp_infl = h->out[GFQ_OUT_DSP_INFLIGHT].as<int32_t>();
    p.dsp_ev = h->out[GFQ_OUT_DSP_EVENT].as<int32_t>();
    p.util_rows = h->out[GFQ_OUT_UTIL_ROWS].as<double>();
    p.util_meta = h->out[GFQ_OUT_UTIL_META].as<int32_t>();
    p.audit_util_cap = h->cfg.audit_util_cap;
    p.backlog_time = h->out[GFQ_OUT_BACKLOG_TIME].as<double>();
    p.backlog_meta = h->out[GFQ_OUT_BACKLOG_META].as<int32_t>();
    p.backlog_count = h->out[GFQ_OUT_BACKLOG_COUNT].as<int64_t>();
    p.audit_backlog_cap = h->cfg.audit_backlog_cap;
    p.event_time = h->out[GFQ_OUT_EVENT_TIME].as<double>();
    p.event_meta = h->out[GFQ_OUT_EVENT_META].as<int64_t>();
    p.event_count = h->out[GFQ_OUT_EVENT_COUNT].as<int64_t>();
    p.event_log_cap = h->cfg.event_log_cap;
    p.evict_time = h->out[GFQ_OUT_EVICT_TIME].as<double>();
    p.evict_meta = h->out[GFQ_OUT_EVICT_META].as<int32_t>();
    p.evict_ev = h->out[GFQ_OUT_EVICT_EVENT].as<int32_t>();
    p.evict_count = h->out[GFQ_OUT_EVICT_COUNT].as<int64_t>();
    p.hist = h->out[GFQ_OUT_HIST].as<unsigned long long>();
    p.hist_rows = h->cfg.hist_rows; p.hist_bins = h->cfg.hist_bins;
    p.hist_lo = h->cfg.hist_lo_s; p.hist_hi = h->cfg.hist_hi_s;
    p.work = h->work.as<int32_t>();
    p.gscratch = h->gscratch.as<unsigned char>();
    return p;
}

int gfq_launch(gfq_handle* h, void* stream) {
    if (!h || !h->prepared) return set_err(GFQ_EINVAL, "gfq_launch: no staged batch");
    CK(cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)stream;
    Params p = make_params(h);
    CK(cudaMemsetAsync(h->work.p, 0, 4 * NCLASS, st));   // one work counter per class
    if (h->cfg.outputs & GFQ_WANT_HIST)
        CK(cudaMemsetAsync(h->out[GFQ_OUT_HIST].p, 0, 8 * h->out_n[GFQ_OUT_HIST], st));
    if (h->cfg.outputs & GFQ_WANT_DISPATCH)        // written by the generic build only
        CK(cudaMemsetAsync(h->out[GFQ_OUT_DSP_EVENT].p, 0, 4 * h->out_n[GFQ_OUT_DSP_EVENT], st));
    if (h->cfg.outputs & GFQ_WANT_RECORDS)         // MQFQ arrivals in the generic build only
        CK(cudaMemsetAsync(h->out[GFQ_OUT_REC_START_TAG].p, 0, 8 * h->out_n[GFQ_OUT_REC_START_TAG], st));
    cudaEvent_t* re = &h->ring[3 * h->ring_next];
    CK(cudaEventRecord(h->ev[0], st));
    CK(cudaEventRecord(re[0], st));
    if (h->n_sims > 0) {
        int active = 0;
        for (int k = 0; k < NCLASS; k++) active += h->ccount[k] > 0;
        // several classes: fork onto side streams (not with flows in global
        // scratch, whose slices are sized for one class at a time)
        const bool fork = active > 1 && !h->L.flows_global;
        if (fork) {
            if (!h->fork) {
                CK(cudaEventCreateWithFlags(&h->fork, cudaEventDisableTiming));
                for (int k = 0; k < NCLASS; k++) {
                    CK(cudaStreamCreateWithFlags(&h->side[k], cudaStreamNonBlocking));
                    CK(cudaEventCreateWithFlags(&h->join[k], cudaEventDisableTiming));
                }
            }
            CK(cudaEventRecord(h->fork, st));
        }
        int off = 0;
        for (int k = 0; k < NCLASS; k++) {
            if (!h->ccount[k]) continue;
            Params pk = p;
            pk.L = h->Lk[k];
            const size_t smem = (size_t)h->wpb * pk.L.bytes;
            pk.order = p.order + off;
            pk.n_sims = h->ccount[k];
            pk.work = p.work + k;
            dim3 g(h->cblocks[k]), b(is_cta_class(k) ? h->cta_threads : h->wpb * 32);
            void* args[] = {&pk};
            cudaStream_t ks = st;
            if (fork) {
                ks = h->side[k];
                CK(cudaStreamWaitEvent(ks, h->fork, 0));
            }
            CK(cudaLaunchKernel(class_kernel(k, h->L.flows_global), g, b, args, smem, ks));
            if (fork) {
                CK(cudaEventRecord(h->join[k], ks));
                CK(cudaStreamWaitEvent(st, h->join[k], 0));
            }
            off += h->ccount[k];
        }
        CK(cudaGetLastError());
    }
    CK(cudaEventRecord(h->ev[1], st));
    CK(cudaEventRecord(re[1], st));
    if (h->n_sims > 0) {
        if (h->rglobal) k_reduce<true><<<h->rblocks, h->rwpb * 32, 0, st>>>(p);
        else k_reduce<false><<<h->rblocks, h->rwpb * 32, (size_t)h->rwpb * RED_FLOW_BYTES * h->L.F, st>>>(p);
        CK(cudaGetLastError());
    }
    CK(cudaEventRecord(h->ev[2], st));
    CK(cudaEventRecord(re[2], st));
    h->ring_next = (h->ring_next + 1) % GFQ_TIMING_RING;
    h->ring_count = std::min(h->ring_count + 1, (int)GFQ_TIMING_RING);
    h->last_stream = st;
    h->launched = true;
    return GFQ_OK;
}

int gfq_synchronize(gfq_handle* h) {
    if (!h || !h->launched) return set_err(GFQ_EINVAL, "gfq_synchronize: nothing launched");
    CK(cudaSetDevice(h->device));
    CK(cudaEventSynchronize(h->ev[2]));
    if (h->n_sims == 0) return GFQ_OK;
    std::vector<int32_t> st(h->n_sims);
    CK(cudaMemcpyAsync(st.data(), h->out[GFQ_OUT_STATUS].p, 4 * h->n_sims, cudaMemcpyDeviceToHost, h->xfer));
    CK(cudaStreamSynchronize(h->xfer));
    for (int i = 0; i < h->n_sims; i++)
        if (st[i] != GFQ_SIM_OK) {
            static const char* names[] = {"ok", "dynamic event pool overflow", "utilization-sample buffer overflow",
                                          "watchdog: event budget exhausted", "event scheduled in the past",
                                          "output buffer overflow", "container pool / running set overflow",
                                          "bad simulation state"};
            return set_err(GFQ_ERUNTIME, "simulation " + std::to_string(i) + " failed: " +
                                             (st[i] >= 0 && st[i] <= 7 ? names[st[i]] : "unknown"));
        }
    return GFQ_OK;
}

int gfq_last_kernel_ms(gfq_handle* h, float* sim_ms, float* reduce_ms) {
    if (!h || !h->launched) return set_err(GFQ_EINVAL, "gfq_last_kernel_ms: nothing launched");
    CK(cudaEventSynchronize(h->ev[2]));
    float a = 0, b = 0;
    CK(cudaEventElapsedTime(&a, h->ev[0], h->ev[1]));
    CK(cudaEventElapsedTime(&b, h->ev[1], h->ev[2]));
    if (sim_ms) *sim_ms = a;
    if (reduce_ms) *reduce_ms = b;
    return GFQ_OK;
}

int gfq_kernel_times(gfq_handle* h, float* sim_ms, float* reduce_ms, int32_t cap, int32_t* n) {
    if (!h || cap < 0 || !n) return set_err(GFQ_EINVAL, "gfq_kernel_times: bad arguments");
    CK(cudaSetDevice(h->device));
    int cnt = std::min(h->ring_count, (int)cap);
    int first = (h->ring_next - cnt + GFQ_TIMING_RING) % GFQ_TIMING_RING;
    for (int i = 0; i < cnt; i++) {
        cudaEvent_t* re = &h->ring[3 * ((first + i) % GFQ_TIMING_RING)];
        CK(cudaEventSynchronize(re[2]));
        float a = 0, b = 0;
        CK(cudaEventElapsedTime(&a, re[0], re[1]));
        CK(cudaEventElapsedTime(&b, re[1], re[2]));
        if (sim_ms) sim_ms[i] = a;
        if (reduce_ms) reduce_ms[i] = b;
    }
    *n = cnt;
    h->ring_count = 0;
    return GFQ_OK;
}

int gfq_batch_info(gfq_handle* h, int32_t* info, int32_t n) {
    if (!h || !h->prepared || !info || n < 0 || n > 6) return set_err(GFQ_EINVAL, "gfq_batch_info: bad arguments");
    int32_t v[6] = {0, h->L.cta ? h->cta_threads : 0, h->L.flows_global, h->wpb, 0, h->L.E};
    for (int k = 0; k < NCLASS; k++)
        if (h->ccount[k]) { v[0]++; v[4] = std::max(v[4], h->cblocks[k]); }
    if (h->n_sims > 0) v[0]++;                             // k_reduce
    for (int i = 0; i < n; i++) info[i] = v[i];
    return GFQ_OK;
}

// ---- NCCL, loaded at first use (no link-time dependency)
namespace {
struct NcclId { char internal[GFQ_NCCL_ID_BYTES]; };    // ncclUniqueId (passed by value)
struct NcclApi {
    typedef int (*GetId)(NcclId*);
    typedef int (*InitRank)(void**, int, NcclId, int);
    typedef int (*Destroy)(void*);
    typedef int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t);
    typedef int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t);
    typedef int (*Group)();
    typedef const char* (*ErrStr)(int);
    GetId get_id = nullptr; InitRank init_rank = nullptr; Destroy destroy = nullptr;
    AllReduce all_reduce = nullptr; AllGather all_gather = nullptr;
    Group group_start = nullptr, group_end = nullptr; ErrStr err = nullptr;
    bool ok = false, tried = false;
};
NcclApi g_nccl;
// nccl.h enums (stable across NCCL 2.x)
enum { NCCL_UINT64 = 5, NCCL_FLOAT64 = 8, NCCL_SUM = 0 };

int nccl_load() {
    if (g_nccl.tried) return g_nccl.ok ? GFQ_OK : set_err(GFQ_ERUNTIME, "NCCL is not available (libnccl.so.2)");
    g_nccl.tried = true;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return set_err(GFQ_ERUNTIME, std::string("dlopen libnccl.so.2: ") + dlerror());
    g_nccl.get_id = (NcclApi::GetId)dlsym(lib, "ncclGetUniqueId");
    g_nccl.init_rank = (NcclApi::InitRank)dlsym(lib, "ncclCommInitRank");
    g_nccl.destroy = (NcclApi::Destroy)dlsym(lib, "ncclCommDestroy");
    g_nccl.all_reduce = (NcclApi::AllReduce)dlsym(lib, "ncclAllReduce");
    g_nccl.all_gather = (NcclApi::AllGather)dlsym(lib, "ncclAllGather");
    g_nccl.group_start = (NcclApi::Group)dlsym(lib, "ncclGroupStart");
    g_nccl.group_end = (NcclApi::Group)dlsym(lib, "ncclGroupEnd");
    g_nccl.err = (NcclApi::ErrStr)dlsym(lib, "ncclGetErrorString");
    g_nccl.ok = g_nccl.get_id && g_nccl.init_rank && g_nccl.destroy && g_nccl.all_reduce &&
                g_nccl.all_gather && g_nccl.group_start && g_nccl.group_end && g_nccl.err;
    return g_nccl.ok ? GFQ_OK : set_err(GFQ_ERUNTIME, "libnccl.so.2 lacks the expected symbols");
}

#define NK(call)                                                                            \
    do {                                                                                    \
        int r_ = (call);                                                                    \
        if (r_ != 0) return set_err(GFQ_ERUNTIME, std::string(#call) + ": " + g_nccl.err(r_)); \
    } while (0)
}  // namespace

int gfq_nccl_unique_id(char id[GFQ_NCCL_ID_BYTES]) {
    if (!id) return set_err(GFQ_EINVAL, "gfq_nccl_unique_id: null id");
    int rc = nccl_load();
    if (rc) return rc;
    NcclId u;
    NK(g_nccl.get_id(&u));
    memcpy(id, u.internal, GFQ_NCCL_ID_BYTES);
    return GFQ_OK;
}

int gfq_nccl_comm_init(void** comm, int32_t n_ranks, const char id[GFQ_NCCL_ID_BYTES], int32_t rank) {
    if (!comm || !id || n_ranks < 1 || rank < 0 || rank >= n_ranks)
        return set_err(GFQ_EINVAL, "gfq_nccl_comm_init: bad arguments");
    int rc = nccl_load();
    if (rc) return rc;
    NcclId u;
    memcpy(u.internal, id, GFQ_NCCL_ID_BYTES);
    NK(g_nccl.init_rank(comm, n_ranks, u, rank));
    return GFQ_OK;
}

int gfq_nccl_comm_destroy(void* comm) {
    if (!comm) return GFQ_OK;
    int rc = nccl_load();
    if (rc) return rc;
    NK(g_nccl.destroy(comm));
    return GFQ_OK;
}

int gfq_reduce_nccl(gfq_handle* h, void* comm, void* summary_out, void* stream) {
    if (!h || !h->launched || !comm) return set_err(GFQ_EINVAL, "gfq_reduce_nccl: no launched batch or no communicator");
    int rc = nccl_load();
    if (rc) return rc;
    CK(cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)stream;
    NK(g_nccl.group_start());
    if (h->out_n[GFQ_OUT_HIST] > 0)
        NK(g_nccl.all_reduce(h->out[GFQ_OUT_HIST].p, h->out[GFQ_OUT_HIST].p, (size_t)h->out_n[GFQ_OUT_HIST],
                             NCCL_UINT64, NCCL_SUM, comm, st));
    if (summary_out && h->n_sims > 0)
        NK(g_nccl.all_gather(h->out[GFQ_OUT_SUMMARY].p, summary_out, (size_t)3 * h->n_sims, NCCL_FLOAT64,
                             comm, st));
    NK(g_nccl.group_end());
    return GFQ_OK;
}

int gfq_output_info(gfq_handle* h, int32_t id, int64_t* n_elems, int32_t* elem_bytes) {
    if (!h || id < 0 || id >= GFQ_OUT_COUNT_) return set_err(GFQ_EINVAL, "gfq_output_info: bad id");
    if (n_elems) *n_elems = h->out_n[id];
    if (elem_bytes) *elem_bytes = kOutBytes[id];
    return GFQ_OK;
}

int gfq_output_copy(gfq_handle* h, int32_t id, void* host_dst, int64_t bytes) {
    if (!h || id < 0 || id >= GFQ_OUT_COUNT_) return set_err(GFQ_EINVAL, "gfq_output_copy: bad id");
    int64_t have = h->out_n[id] * kOutBytes[id];
    if (bytes > have) return set_err(GFQ_EINVAL, "gfq_output_copy: request larger than the output");
    CK(cudaSetDevice(h->device));
    if (bytes) {
        CK(cudaStreamWaitEvent(h->xfer, h->ev[2], 0));  // after this handle's last launch
        CK(cudaMemcpyAsync(host_dst, h->out[id].p, bytes, cudaMemcpyDeviceToHost, h->xfer));
        CK(cudaStreamSynchronize(h->xfer));
    }
    return GFQ_OK;
}

int gfq_output_device_ptr(gfq_handle* h, int32_t id, void** dptr) {
    if (!h || id < 0 || id >= GFQ_OUT_COUNT_ || !dptr) return set_err(GFQ_EINVAL, "gfq_output_device_ptr: bad id");
    *dptr = h->out_n[id] ? h->out[id].p : nullptr;
    return GFQ_OK;
}

int gfq_fairness(gfq_handle* h, double window_s, const int32_t* d_max,
                 const double* report_weight, int64_t n_weights) {
    if (!h || !h->launched) return set_err(GFQ_EINVAL, "gfq_fairness: no finished batch");
    if (!(window_s > 0) || (h->n_sims && !d_max))
        return set_err(GFQ_EINVAL, "gfq_fairness: bad arguments");
    if ((h->cfg.outputs & (GFQ_WANT_RECORDS | GFQ_WANT_AUDIT)) != (GFQ_WANT_RECORDS | GFQ_WANT_AUDIT))
        return set_err(GFQ_EINVAL, "gfq_fairness: the batch needs GFQ_WANT_RECORDS | GFQ_WANT_AUDIT");
    int64_t rows_tab = h->h_tab_off.empty() ? 0 : h->h_tab_off.back();
    if (n_weights != rows_tab || (rows_tab && !report_weight))
        return set_err(GFQ_EINVAL, "gfq_fairness: report_weight must cover every flow-table row");
    for (int i = 0; i < h->n_sims; i++)
        if (d_max[i] < 1) return set_err(GFQ_EINVAL, "d must be >= 1");
    for (int64_t i = 0; i < n_weights; i++)
        if (!(report_weight[i] > 0)) return set_err(GFQ_EINVAL, "weights must be positive");
    CK(cudaSetDevice(h->device));
    CK(cudaStreamWaitEvent(0, h->ev[2], 0));   // legacy-stream work after this handle's last launch
    CK(cudaEventSynchronize(h->ev[2]));
    const int n = h->n_sims;
    std::vector<double> ft(std::max(n, 1));
    if (n) CK(cudaMemcpy(ft.data(), h->out[GFQ_OUT_FINAL_TIME].p, 8 * n, cudaMemcpyDeviceToHost));
    std::vector<int64_t> woff(n + 1, 0);
    for (int i = 0; i < n; i++) woff[i + 1] = woff[i] + (int64_t)ceil(ft[i] / window_s) + 2;
    int rc;
    if ((rc = alloc_out(h, GFQ_OUT_FAIR_ROWS, 5 * woff[n])) || (rc = alloc_out(h, GFQ_OUT_FAIR_META, 6 * woff[n])) ||
        (rc = alloc_out(h, GFQ_OUT_FAIR_OFF, n + 1)) || (rc = alloc_out(h, GFQ_OUT_FAIR_COUNT, 3ll * n)))
        return rc;
    DBuf dm, rw;
    if ((rc = dm.ensure(4 * std::max(n, 1))) || (rc = rw.ensure(8 * std::max<int64_t>(n_weights, 1)))) return rc;
    if (n) CK(cudaMemcpy(dm.p, d_max, 4 * n, cudaMemcpyHostToDevice));
    if (n_weights) CK(cudaMemcpy(rw.p, report_weight, 8 * n_weights, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->out[GFQ_OUT_FAIR_OFF].p, woff.data(), 8 * (n + 1), cudaMemcpyHostToDevice));
    const int wpb = 4;
    int blocks = std::max(1, std::min((n + wpb - 1) / wpb, 4 * h->n_sm));
    if ((rc = h->fscratch.ensure((size_t)blocks * wpb * 48 * h->L.F))) { dm.release(); rw.release(); return rc; }
    FairParams fp{};
    fp.window_s = window_s; fp.d_max = dm.as<int32_t>(); fp.rweight = rw.as<double>();
    fp.woff = h->out[GFQ_OUT_FAIR_OFF].as<int64_t>();
    fp.rows = h->out[GFQ_OUT_FAIR_ROWS].as<double>(); fp.meta = h->out[GFQ_OUT_FAIR_META].as<int64_t>();
    fp.count = h->out[GFQ_OUT_FAIR_COUNT].as<int64_t>(); fp.scratch = h->fscratch.as<unsigned char>();
    Params p = make_params(h);
    if (n) k_fairness<<<blocks, wpb * 32>>>(p, fp);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    dm.release(); rw.release();
    if (e != cudaSuccess) return set_err(GFQ_ECUDA, std::string("k_fairness: ") + cudaGetErrorString(e));
    return GFQ_OK;
}

int gfq_run(gfq_handle* h, const gfq_sim* sims, int32_t n_sims, const gfq_launch_cfg* cfg) {
    int rc = gfq_prepare(h, sims, n_sims, cfg);
    if (rc) return rc;
    if ((rc = gfq_launch(h, nullptr))) return rc;
    return gfq_synchronize(h);
}

}  // extern "C"
