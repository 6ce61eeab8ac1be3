// gfq_layout.h — shared (host + device) description of the per-simulation
// shared-memory workspace and the kernel parameter block.
//
// One simulation runs per warp.  Its mutable state lives in a private slice
// of the CTA's dynamic shared memory, laid out structure-of-arrays so that
// the warp's lane-parallel scans (lane i owns flows i, i+32, ...; pool
// entries i, i+32, ...; event slots i, i+32, ...) are bank-conflict free.
// Sizes are per batch (the maxima over the batch's simulations), computed
// on the host by gfq_layout_make() and mirrored on the device.
#pragma once
#include <stdint.h>
#include "../../include/gfq.h"

namespace gfq {

// flow state bits (per flow, u8)
enum : uint8_t { FL_CREATED = 1, FL_INACTIVE = 2, FL_NEWLY = 4, FL_MARKED = 8 };

// per-device int fields
enum { DV_OUT = 0, DV_EFFD, DV_HROK, DV_NP, DV_NRUN, DV_SHEAD, DV_SN, DV_INSTDIRTY, DV_INSTID,
       DV_ZAGE, DV_WCODE, DV_LKEY, DV_NSTATE,                // hot mutable state (registers
       DV_SPARE0 = DV_NSTATE,                                //  in the 1-device build);
       DV_DMAX, DV_POOLMAX, DV_POOLON, DV_DYN,               //  DeviceConfig copy
       DV_NI = 18 };
// per-device double fields: state, then a copy of the device's DeviceConfig
enum { DD_UAVG = 0, DD_INST, DD_OLDT, DD_NSTATE,
       DD_MEMCAP = DD_NSTATE, DD_THR, DD_PCIE, DD_BETA, DD_WINDOW, DD_OVERLAP, DD_INVDMAX,
       DD_ND = 12 };
// window-average memo: WDICT distinct utilization values per device,
// WMEMO direct-mapped (window code, count) -> average entries; windows of up
// to WMAXN samples are memoised (32-bit key: 7 x 4-bit ids + the count)
enum { WDICT = 15, WMEMO = 64, WMEMO_BITS = 6, WMAXN = 7 };
// flows queued for swap-out since the last _swap_out_inactive
enum { NEWLY_CAP = 32 };
// per-warp diagnostic counters (shared memory, lane 0 increments)
#ifndef GFQ_PROF
#define GFQ_PROF 0      // diagnostic build: per-simulation clock64() cycles per event-loop phase
#endif
enum { DG_MAXEV = 0, DG_GSCAN, DG_RSCAN, DG_CSCAN, DG_TICKS, DG_WHIT, DG_WMISS, DG_QUIET,
       DG_P0, DG_N = GFQ_PROF ? DG_P0 + 7 : DG_P0 };
// GFQ_PROF phases (DG_P0 + k): pool minimum, keep-alive refresh scan, drain (incl. the
// refresh), monitor ticks, arrivals, completions, expiries + swap-outs
enum { PF_POOL = 0, PF_REFRESH, PF_DRAIN, PF_TICK, PF_ARR, PF_COMP, PF_EXP };

// event kinds (engine.py:20-23)
enum { EV_ARRIVAL = 0, EV_COMPLETION = 1, EV_TICK = 2, EV_EXPIRY = 3 };

// CTA mode: the leader warp's scan command and the per-warp partial argmins
// (lexicographic (k, s, i)) the helper warps return.
enum { CTA_MAXW = 32 };
#ifndef GFQ_CTA_THREADS
#define GFQ_CTA_THREADS 512        // threads of a CTA-mode simulation (max)
#endif
struct CtaCmd {
    int32_t op, nf, nev, iarg;     // scan kind, flow count, event slots, use_inf
    int32_t pad0, pad1, nset, pad2;        // nset: backlogged-set size (large-flow builds)
    double gvt, now;
    unsigned long long pk[CTA_MAXW];
    uint32_t ps[CTA_MAXW];
    int32_t pi[CTA_MAXW];
};

struct Layout {
    int32_t F;      // flow slots (multiple of 32)
    int32_t E;      // dynamic event slots (completions + keep-alive expiries)
    int32_t ND;     // modeled devices
    int32_t P;      // container pool slots per device (pool_max + 1)
    int32_t R;      // running slots per device (max d_max)
    int32_t S;      // utilization-sample ring slots per device
    // F-dependent part ("fe"): per-flow state, dynamic events, per-flow
    // container counts.  Byte offsets from the fe base (8-byte aligned).
    int32_t o_vt, o_lex, o_tau, o_iat, o_larr;          // f64[F]
    int32_t o_pt, o_ph, o_infl, o_head, o_done, o_pend;  // i32[F] (u16[F] when i16)
    int32_t o_fst;                                       // u8[F]
    int32_t o_ev_t, o_ev_seq, o_ev_meta;                 // f64[E], u32[E], u32[E]
    int32_t o_cnt;                                       // u16[ND][3][F]: gpu-warm, host-warm, running
    int32_t fe_bytes;
    // device part: offsets from the device base
    int32_t o_dvi, o_dvd;                                // i32[ND][DV_NI], f64[ND][DD_ND]
    int32_t o_smp_t, o_smp_u;                            // f64[ND][S]
    int32_t o_run_i, o_run_d;                            // i32[ND][R][4], f64[ND][R][2]
    int32_t o_pool_m, o_pool_t;                          // u32[ND][P], f64[ND][P]
    int32_t o_wdict, o_wkey, o_wval;                     // f64[ND][WDICT], u32[ND][WMEMO], f64[ND][WMEMO]
    int32_t o_diag;                                      // u32[DG_N]
    int32_t o_newly;                                     // i32[NEWLY_CAP]
    int32_t o_cst, o_csp, o_csm;                         // completion staging: f64[32], i32[32], i32[32]
    int32_t o_rgt, o_rgf, o_mbar;                        // arrival window: f64[64], i32[64], 2 mbarriers
    int32_t o_cta;                                       // CtaCmd (CTA-per-simulation mode only)
    int32_t dev_bytes;
    // the fe part lives in shared memory in front of the device part, or (for
    // flow counts whose state does not fit) in a per-warp global scratch slice
    int32_t flows_global;
    // CTA-per-simulation mode (large flow counts): one simulation per CTA,
    // warp 0 runs the event loop, the other warps join its O(F) scans
    int32_t cta;
    int32_t bytes;                                       // shared bytes per warp (per CTA in CTA mode)
    // the six per-flow counters / cursors as u16 (the 1-device warp classes,
    // traces shorter than 65535 arrivals): a smaller workspace, more
    // simulations resident per SM
    int32_t i16;
    // large-flow builds (CTA or flows in global): the set of backlogged flows
    // (pending or in flight) as an unordered list + position index, so the
    // global-VT and candidate scans visit backlogged flows only
    int32_t o_bll, o_blp;                                // u16[F], u16[F] (fe part; 0 = none)
    // large-flow builds: per 32-flow block, a lower bound on the earliest
    // keep-alive expiry among the block's idle queues (refresh_states visits
    // only the blocks whose bound has passed)
    int32_t o_bmin;                                      // f64[F / 32] (fe part; 0 = none)
    // FlowQueue.last_start_tag per flow: batches that ask for records together
    // with the logs (the generic build: Simulation.step() replays start tags)
    int32_t lst;                                         // flag
    int32_t o_lst;                                       // f64[F] (fe part; 0 = none)
};

struct Params {
    const gfq_sim* sims;
    const int32_t* order;          // work-queue order of sims (longest first)
    int32_t n_sims;
    // traces (CSR) and their per-flow arrival index (built by the loader)
    const double* arrival;
    const int32_t* flow;
    const int64_t* trace_off;      // [n_traces + 1]
    const int32_t* trace_nf;       // [n_traces]
    const int64_t* foff_off;       // [n_traces + 1] offsets into foff
    const int32_t* foff;           // per trace: nf + 1 offsets into fpos (trace-relative)
    const int32_t* fpos;           // per trace: arrival positions grouped by flow
    // flow tables (profiles + weights)
    const double *warm, *cold, *mem, *share, *weight;
    const int32_t* memi;           // mem_mb in integer MB, or -1 for a non-integral table
    const int32_t* hist_row;
    const int64_t* tab_off;
    const gfq_device_cfg* dcfg;
    const double* execs;
    // per-sim output offsets
    const int64_t* sim_foff;       // flow offset per sim
    const int64_t* sim_roff;       // record offset per sim
    Layout L;
    uint32_t outputs;
    int32_t early_exit;
    // outputs
    int32_t* status;
    int64_t* counters;             // [sims][GFQ_NCOUNTERS]
    double* final_time;
    double* summary;               // [sims][3]
    int64_t* f_count; double* f_mean; double* f_var; double* f_cold;
    // completion-order scratch (always): latency and flow|cold<<31
    double* comp_lat; int32_t* comp_meta;
    int32_t* comp_pos;             // completion rank -> trace position (GFQ_WANT_RECORDS)
    double* rec_dispatch; double* rec_complete; double* rec_pure;
    double* rec_stag;              // Invocation.start_tag (generic build, Layout::lst)
    int8_t* rec_state; int8_t* rec_device; int32_t* rec_order;
    int32_t* dsp_inv; double* dsp_vt; double* dsp_gvt; int32_t* dsp_qlen; int32_t* dsp_infl;
    int32_t* dsp_ev;               // generic build: processed-event index of each dispatch row
    double* util_rows; int32_t* util_meta; int64_t audit_util_cap;
    double* backlog_time; int32_t* backlog_meta; int64_t* backlog_count; int64_t audit_backlog_cap;
    double* event_time; int64_t* event_meta; int64_t* event_count; int64_t event_log_cap;
    double* evict_time; int32_t* evict_meta; int64_t* evict_count;   // at the sim's record offset
    int32_t* evict_ev;             // processed-event index of each eviction row
    unsigned long long* hist; int32_t hist_rows, hist_bins; double hist_lo, hist_hi;
    int32_t* work;                 // work-queue counter
    double* rscratch;              // reducer: per-warp record scratch (rscratch_per_warp doubles)
    int64_t rscratch_per_warp;
    int32_t cta_min;               // CTA mode: scans shorter than this stay on the leader warp
    unsigned char* gscratch;       // per-warp fe slices when L.flows_global
};

inline int32_t align8(int32_t x) { return (x + 7) & ~7; }

inline void layout_finish(Layout& L) {
    const int32_t F = L.F, E = L.E, ND = L.ND, P = L.P, R = L.R, S = L.S;
    int32_t o = 0;
    auto take = [&](int32_t bytes) { int32_t r = o; o = align8(o + bytes); return r; };
    L.o_vt = take(8 * F); L.o_lex = take(8 * F); L.o_tau = take(8 * F);
    L.o_iat = take(8 * F); L.o_larr = take(8 * F);
    const int32_t iw = L.i16 ? 2 : 4;
    L.o_pt = take(iw * F); L.o_ph = take(iw * F); L.o_infl = take(iw * F);
    L.o_head = take(iw * F); L.o_done = take(iw * F); L.o_pend = take(iw * F);
    L.o_fst = take(F);
    L.o_ev_t = take(8 * E); L.o_ev_seq = take(4 * E); L.o_ev_meta = take(4 * E);
    L.o_cnt = take(2 * 3 * ND * F);
    if (L.cta || L.flows_global) { L.o_bll = take(2 * F); L.o_blp = take(2 * F); L.o_bmin = take(8 * (F / 32)); }
    else L.o_bll = L.o_blp = L.o_bmin = 0;
    L.o_lst = L.lst ? take(8 * F) : 0;
    L.fe_bytes = o;
    o = 0;
    auto take16 = [&](int32_t bytes) { o = (o + 15) & ~15; return take(bytes); };
    if (L.cta) {                                 // CTA mode only (WarpSim::RING / CSTAGE)
        L.o_rgt = take16(8 * 64); L.o_rgf = take16(4 * 64); L.o_mbar = take16(24);   // TMA targets, mbarriers + parity
        L.o_cst = take(8 * 32); L.o_csp = take(4 * 32); L.o_csm = take(4 * 32);
    } else {
        L.o_rgt = L.o_rgf = L.o_mbar = L.o_cst = L.o_csp = L.o_csm = 0;
    }
    L.o_dvi = take(4 * DV_NI * ND); L.o_dvd = take(8 * DD_ND * ND);
    L.o_smp_t = take(8 * ND * S); L.o_smp_u = take(8 * ND * S);
    L.o_run_i = take(4 * 4 * ND * R); L.o_run_d = take(8 * 2 * ND * R);
    L.o_pool_m = take(4 * ND * P); L.o_pool_t = take(8 * ND * P);
    L.o_wdict = take(8 * WDICT * ND); L.o_wkey = take(4 * WMEMO * ND); L.o_wval = take(8 * WMEMO * ND);
    L.o_diag = take(4 * DG_N);
    L.o_newly = take(4 * NEWLY_CAP);
    L.o_cta = L.cta ? take((int32_t)sizeof(CtaCmd)) : 0;
    L.dev_bytes = (o + 15) & ~15;
    L.fe_bytes = (L.fe_bytes + 15) & ~15;                // keep every slice 16-byte aligned
    L.bytes = L.flows_global ? L.dev_bytes : L.fe_bytes + L.dev_bytes;
}

}  // namespace gfq
