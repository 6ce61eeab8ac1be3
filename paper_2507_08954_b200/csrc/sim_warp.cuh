// sim_warp.cuh — one MQFQ-Sticky discrete-event simulation per warp.
//
// This is the B200 restatement of the reference's hot path
//   Simulation.run -> _drain -> Policy.dispatch -> DeviceSet.assign -> Device.*
//   (gpufairq engine.py:115-197, mqfq.py:190-239, policies.py:116-273,
//    device.py:124-341)
// executed by all 32 lanes of a warp in lock-step:
//
//   * scalar simulation state (clock, global VT, event cursor, counters) is
//     warp-uniform and lives in registers; every lane computes it;
//   * per-flow state (vt, last_exec, tau/iat estimators, queue cursors) is a
//     structure-of-arrays slice of shared memory; the O(F) passes of the
//     reference (recompute_global_vt, refresh_states, the candidate filter and
//     its two stable sorts) become lane-parallel scans (lane i owns flows
//     i, i+32, ...) closed by redux.sync reductions on order-preserving keys;
//   * the container pool is an ordered array (list semantics: append,
//     remove-with-shift) with per-(device, flow) warm/host-warm/running
//     counts; order-sensitive float sums (CPython 3.12 Neumaier sum()) are
//     replayed serially through warp shuffles in list order;
//   * dynamic events (completions, keep-alive expiries) sit in a slot pool
//     with a cached (time, seq) minimum; arrivals stream from the trace
//     (their seq is the trace index, engine.py:70-75); the single monitor
//     tick is kept in registers.
//
// Three exact short-circuits remove most of the reference's per-call O(F)
// work without changing any observable result:
//   (A) the minimum vt over backlogged queues (recompute_global_vt) is cached
//       and only rescanned when the queue holding it is charged or drains;
//   (B) refresh_states can only change a queue's INACTIVE bit (THROTTLED vs
//       ACTIVE is unobservable), and only for idle queues whose
//       keep-alive has run out; a rounding-safe lower bound on the earliest
//       such time skips the scan until it can fire;
//   (C) when every modeled device refuses on the function-independent checks
//       (tokens, utilization headroom; device.py:134-139) the dispatch returns
//       None whatever the candidate, so candidate selection is skipped (the
//       scripted token provider counts attempts and is never short-circuited).
//
// Every floating-point operation is written in the reference's operation
// order and the file is compiled with -fmad=false, so dispatch order,
// DispatchAudit rows and completion records are bit-identical to the
// reference (tests/test_gpu_parity.py).
//
// Code layout: drain(), dispatch_once(), provider_assign() and the device
// model each have exactly ONE inlined call site so the kernel stays compact
// (the instruction cache, not the ALUs, bounds a latency-bound event loop).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>
#include "gfq_layout.h"

namespace gfq {

#define FULLMASK 0xffffffffu
#ifndef GFQ_DIAG
#define GFQ_DIAG 0      // per-warp diagnostic counters (scans, ticks, memo hits, ...)
#endif
#define FI __device__ __forceinline__
typedef unsigned long long u64;
// Latency-bound builds only (CTA mode: one event-loop warp per SM): the
// arrival window in shared memory fed by TMA bulk copies, and the completion
// stream staged in shared memory with a coalesced write-back.  The
// warp-per-simulation builds run 16 event loops per SM, which hide the L2
// latency these remove but not the instruction-cache footprint they add
// (measured: each costs ~10% on C3).
#ifndef GFQ_RING
#define GFQ_RING 1
#endif
#ifndef GFQ_CSTAGE
#define GFQ_CSTAGE 1
#endif

// ------------------------------------------------------------------------
// warp primitives

FI u64 okey(double x) {                                   // order-preserving key
    u64 b = (u64)__double_as_longlong(x);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
FI double from_key(u64 k) {                               // inverse of okey
    u64 b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}
FI unsigned wmin32(unsigned v) { return __reduce_min_sync(FULLMASK, v); }
FI unsigned wor32(unsigned v) { return __reduce_or_sync(FULLMASK, v); }
FI u64 wmin64(u64 v) {
    unsigned hi = wmin32((unsigned)(v >> 32));
    unsigned lo = wmin32(((unsigned)(v >> 32) == hi) ? (unsigned)v : 0xffffffffu);
    return ((u64)hi << 32) | lo;
}
// Uniform shared-memory state is read-modify-written by all 32 lanes with
// identical values (each lane loads X, then stores the same new X).
//  * No barrier after such a store: whichever lane's store a later load
//    observes, the value is the same, and a lane's own store is ordered
//    before its own later loads.
//  * None before it either (USYNC() is empty): the warp runs the scalar
//    code converged -- every branch there is on warp-uniform values -- so all
//    lanes execute a load before any lane executes the store after it.  The
//    regions that diverge (lane-strided scans, lane-0 writes) end in a
//    *_sync reduction or an explicit __syncwarp(), which reconverge the warp
//    before scalar code continues.  -DGFQ_STRICT_SYNC=1 restores a
//    __syncwarp() before every uniform store (the parity suite passes on
//    both builds).
#ifndef GFQ_STRICT_SYNC
#define GFQ_STRICT_SYNC 0
#endif
#if GFQ_STRICT_SYNC
#define USYNC() __syncwarp()
#else
#define USYNC() do { } while (0)
#endif
template <class T>
FI void ust(T& ref, T v) { USYNC(); ref = v; }

// Python max(a, b) / min(a, b): the first argument wins ties.
FI double pymax(double a, double b) { return b > a ? b : a; }
FI double pymin(double a, double b) { return b < a ? b : a; }

// CPython 3.12 builtin sum() over floats (bltinmodule.c builtin_sum_impl):
// the first item is added to the int start 0, then Neumaier compensation,
// the compensation is added once at the end when nonzero and finite.
//
// Starting from f = 0.0, c = 0.0, the general step below applied to the first
// item computes exactly CPython's `0 + x` with a zero compensation term, so
// no item count or first-item branch is needed (and an empty sum is 0.0).
struct PySum { double f, c; };
FI void ps_init(PySum& s) { s.f = 0.0; s.c = 0.0; }
FI void ps_add(PySum& s, double x) {
    // c += (f - t) + x if |f| >= |x| else (x - t) + f: the operands are
    // selected first, so one compensation term is computed, not two
    const double t = s.f + x;
    const bool big = fabs(s.f) >= fabs(x);
    const double a = big ? s.f : x, b = big ? x : s.f;
    s.c += (a - t) + b;
    s.f = t;
}
FI double ps_val(const PySum& s) {
    if (s.c != 0.0 && isfinite(s.c)) return s.f + s.c;
    return s.f;
}

// Lower bound on the time at which `now - lex >= ttl` (fp64, as the
// reference evaluates it) can first hold: below it the rounded difference is
// provably < ttl.  Relative margin 2^-50 >> the 2 ulps of rounding involved.
FI double expiry_lb(double lex, double ttl) {
    double x = lex + ttl;
    return x - fabs(x) * 8.881784197001252e-16;
}

// pool entry meta: fn | thermal << 24 | evictable << 26 | swapping << 27
FI int pm_fn(uint32_t m) { return (int)(m & 0xffffffu); }
FI int pm_th(uint32_t m) { return (int)((m >> 24) & 3u); }
FI bool pm_ev(uint32_t m) { return (m >> 26) & 1u; }
FI bool pm_sw(uint32_t m) { return (m >> 27) & 1u; }
FI uint32_t pm_make(int fn, int th, int ev) {
    return (uint32_t)fn | ((uint32_t)th << 24) | ((uint32_t)ev << 26);
}

enum { C_EVENTS = 0, C_CALLS, C_DISP, C_UTIL, C_MAXEV, C_GSCAN, C_RSCAN, C_CSCAN, C_TICKS,
       C_WHIT, C_WMISS, C_QUIET };

// ------------------------------------------------------------------------
// the per-warp simulation

// Build classes: PB_GENERIC handles every policy, the scripted token provider
// and the audit / event logs; the others are one policy on a DeviceSet.
enum { PB_GENERIC = 0, PB_MQFQ = 1, PB_FCFS = 2, PB_BATCH = 3, PB_SJF = 4,
       PB_MQFQ_LOG = 5 };   // MQFQ-Sticky on one device WITH the audit / event / eviction logs

// Once per warp slice at kernel start: the arrival window's two mbarriers
// (see WarpSim::ring_start) and their phase-parity word.
FI void ring_init(unsigned char* dev_base, const Layout& L, int lane) {
    if (lane == 0) {
        const uint32_t mb = (uint32_t)__cvta_generic_to_shared(dev_base + L.o_mbar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb + 8) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        *(uint32_t*)(dev_base + L.o_mbar + 16) = 0;
    }
    __syncwarp();
}

// CTA-mode scan kinds (the leader warp's command to the helper warps)
enum { OP_EXIT = 0, OP_GVT, OP_CAND, OP_BATCH, OP_SJF, OP_EVMIN };

// lexicographic (k, s, i) argmin candidate
struct Arg { u64 k; uint32_t s; int i; };
FI Arg arg_none() { Arg a; a.k = ~0ull; a.s = 0xffffffffu; a.i = 0x7fffffff; return a; }
FI Arg warp_argmin(Arg a) {
    Arg r;
    r.k = wmin64(a.k);
    r.s = wmin32(a.k == r.k ? a.s : 0xffffffffu);
    r.i = (int)wmin32(a.k == r.k && a.s == r.s ? (unsigned)a.i : 0x7fffffffu);
    return r;
}
// named barrier over the n threads of the simulation's CTA.  The non-.aligned
// form: a warp may reach it with its lanes not yet reconverged (after the
// lane-0 command writes), which bar.sync (= barrier.sync.aligned) forbids.
FI void cta_bar(int id, int n) { asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// CTA = one simulation per CTA (large flow counts): warp 0
// (the leader) runs everything below; the O(F) flow scans and the event-pool
// argmin are split over all the CTA's warps (cta_scan / helper_loop).
#ifndef GFQ_FG_UNROLL
#define GFQ_FG_UNROLL 8
#endif
template <int POL, bool ND1, bool CTA = false, bool FG = false>
struct WarpSim {
    static constexpr bool G = POL == PB_GENERIC;
    // the build writes the logs (utilization / backlog audit, processed-event
    // log, eviction log, per-row event indices, start tags): the generic
    // build, and the MQFQ 1-device build the drop-ins use (run_simulation,
    // Simulation, the CLI ask for every log)
    static constexpr bool LG = G || POL == PB_MQFQ_LOG;
    // FG: the flow/event part lives in global scratch; its lane-strided scans
    // keep several loads in flight (a smem build keeps them rolled: its hot
    // code size is what bounds it)
    static constexpr int SCAN_UNROLL = FG ? GFQ_FG_UNROLL : 1;
    static constexpr bool RING = CTA && GFQ_RING;
    static constexpr bool CSTAGE = CTA && GFQ_CSTAGE;
    // large-flow builds: the global-VT / candidate scans visit the set of
    // backlogged flows (pending or in flight: at most the queued invocations
    // plus the tokens out) instead of every touched flow
    static constexpr bool SETS = CTA || FG;
    // the 1-device fast classes run integral flow tables only (gfq_prepare)
    static constexpr bool MEMI = !G && ND1;
    const Params& P;
    unsigned char* const sm;   // device part of this warp's state (shared memory)
    unsigned char* const fe;   // flow/event part (shared memory, or global scratch)
    const int lane;
    const int sid;

    // ---- shared-memory views (offsets live in the kernel's param space)
    FI double* vt() const { return (double*)(fe + P.L.o_vt); }
    FI double* lex() const { return (double*)(fe + P.L.o_lex); }
    FI double* tau() const { return (double*)(fe + P.L.o_tau); }
    FI double* iat() const { return (double*)(fe + P.L.o_iat); }
    FI double* larr() const { return (double*)(fe + P.L.o_larr); }
    // per-flow counters / cursors: u16 in the 1-device warp classes (Layout::i16;
    // gfq_prepare routes traces of 65535+ arrivals elsewhere), i32 otherwise.
    // head() is only read while the queue has pending work, so its empty
    // marker (-1, stored as 0xffff) is never compared.
    static constexpr bool I16 = !G && ND1 && !CTA && !FG;
    typedef typename std::conditional<I16, uint16_t, int32_t>::type CI;
    FI CI* pt() const { return (CI*)(fe + P.L.o_pt); }
    FI CI* ph() const { return (CI*)(fe + P.L.o_ph); }
    FI CI* infl() const { return (CI*)(fe + P.L.o_infl); }
    FI CI* head() const { return (CI*)(fe + P.L.o_head); }
    FI CI* done() const { return (CI*)(fe + P.L.o_done); }
    FI CI* pend() const { return (CI*)(fe + P.L.o_pend); }
    FI uint8_t* fst() const { return (uint8_t*)(fe + P.L.o_fst); }
    FI uint16_t* BLL() const { return (uint16_t*)(fe + P.L.o_bll); }   // backlogged set (SETS)
    FI uint16_t* BLP() const { return (uint16_t*)(fe + P.L.o_blp); }   // flow -> its slot
    FI double* BMIN() const { return (double*)(fe + P.L.o_bmin); }     // per-block expiry bound (SETS)
    FI double* ev_t() const { return (double*)(fe + P.L.o_ev_t); }
    FI uint32_t* ev_seq() const { return (uint32_t*)(fe + P.L.o_ev_seq); }
    FI uint32_t* ev_meta() const { return (uint32_t*)(fe + P.L.o_ev_meta); }
    // per-device fields; in the 1-device build the mutable ones are registers
    int hv[DV_NSTATE]; double hd[DD_NSTATE];
    double win0;                       // 1-device build: device 0's util_window_s (read every tick)
    FI int& DV(int d, int k) {
        if (ND1 && k < DV_NSTATE) return hv[k];
        return ((int*)(sm + P.L.o_dvi))[d * DV_NI + k];
    }
    FI double& DD(int d, int k) {
        if (ND1 && k < DD_NSTATE) return hd[k];
        return ((double*)(sm + P.L.o_dvd))[d * DD_ND + k];
    }
    FI int NDEV() const { return ND1 ? 1 : ndev; }
    FI void diag(int k, unsigned v = 1) { if (GFQ_DIAG && lane == 0) ((uint32_t*)(sm + P.L.o_diag))[k] += v; }
    FI long long pclk() const { return GFQ_PROF ? (long long)clock64() : 0ll; }
    FI void prof(int k, long long t0) {
        if (GFQ_PROF && lane == 0) ((uint32_t*)(sm + P.L.o_diag))[DG_P0 + k] += (uint32_t)(clock64() - t0);
    }
    FI double& UAVG(int d) { return DD(d, DD_UAVG); }
    FI double& SMPT(int d, int i) const { return ((double*)(sm + P.L.o_smp_t))[d * P.L.S + i]; }
    FI double& SMPU(int d, int i) const { return ((double*)(sm + P.L.o_smp_u))[d * P.L.S + i]; }
    FI int& RI(int d, int r, int k) const { return ((int*)(sm + P.L.o_run_i))[(d * P.L.R + r) * 4 + k]; }
    FI double& RD(int d, int r, int k) const { return ((double*)(sm + P.L.o_run_d))[(d * P.L.R + r) * 2 + k]; }
    FI uint32_t& PM(int d, int i) const { return ((uint32_t*)(sm + P.L.o_pool_m))[d * P.L.P + i]; }
    FI double& PT(int d, int i) const { return ((double*)(sm + P.L.o_pool_t))[d * P.L.P + i]; }
    FI double& WDICTV(int d, int i) const { return ((double*)(sm + P.L.o_wdict))[d * WDICT + i]; }
    FI uint32_t& WKEY(int d, int i) const { return ((uint32_t*)(sm + P.L.o_wkey))[d * WMEMO + i]; }
    FI double& WVAL(int d, int i) const { return ((double*)(sm + P.L.o_wval))[d * WMEMO + i]; }
    FI int* NEWLY() const { return (int*)(sm + P.L.o_newly); }
    FI double* CST() const { return (double*)(sm + P.L.o_cst); }      // completion staging
    FI int* CSP() const { return (int*)(sm + P.L.o_csp); }
    FI int* CSM() const { return (int*)(sm + P.L.o_csm); }
    FI double* RGT() const { return (double*)(sm + P.L.o_rgt); }      // arrival window
    FI int* RGF() const { return (int*)(sm + P.L.o_rgf); }
    FI uint16_t& CNT(int d, int kind, int f) const {   // kind: 0 gpu-warm, 1 host-warm, 2 running
        return ((uint16_t*)(fe + P.L.o_cnt))[(d * 3 + kind) * P.L.F + f];
    }

    // ---- per-simulation inputs
    const gfq_sim* sim;
    int64_t toff, roff;
    int tb;
    bool tau_inc;
    bool mem_int;                      // the flow table's mem_mb are integers (resident_mb)
    const int* foff;
    int n, nf, ndev;
    int policy;
    bool scripted_, mqfq_, fcfs_;
    // G = generic build (every policy, the scripted token provider, audit and
    // event logs); !G = the MQFQ-Sticky / DeviceSet build the sweeps run
#define SCRIPTED (G && scripted_)
#define MQFQ (G ? mqfq_ : (POL == PB_MQFQ || POL == PB_MQFQ_LOG))
#define FCFS (G ? fcfs_ : POL == PB_FCFS)
#define BATCH (G ? policy == GFQ_POLICY_BATCH : POL == PB_BATCH)
#define SJF (G ? policy == GFQ_POLICY_SJF : POL == PB_SJF)
    double T, alpha, dttl, period;

    // read-only inputs through the non-coherent path (L1-resident: the flow
    // tables of an SM's simulations and their trace windows are small)
    FI double arr(int i) const { return __ldg(P.arrival + toff + i); }
    FI int flw(int i) const { return __ldg(P.flow + toff + i); }
    FI double warm(int f) const { return __ldg(P.warm + tb + f); }
    FI double cold(int f) const { return __ldg(P.cold + tb + f); }
    FI double mem(int f) const { return __ldg(P.mem + tb + f); }
    FI uint32_t memi(int f) const { return (uint32_t)__ldg(P.memi + tb + f); }
    FI double share(int f) const { return __ldg(P.share + tb + f); }
    FI double weight(int f) const { return __ldg(P.weight + tb + f); }

    // ---- arrival window: the trace streams through a 2 x 32-entry ring in
    // shared memory, each 32-entry chunk (32-aligned global trace index)
    // fetched by one TMA bulk copy (cp.async.bulk, mbarrier completion) a
    // chunk ahead of the cursor.  The parity word (bit h = the phase parity to
    // wait for on half h) sits in shared memory next to the mbarriers.
    FI int ring_last() const { return (int)((toff + n - 1) >> 5); }   // n > 0
    FI uint32_t mbar_addr(int h) const {
        return (uint32_t)__cvta_generic_to_shared(sm + P.L.o_mbar + 8 * h);
    }
    FI void ring_issue(int c) {        // lane 0: fetch chunk c into half c & 1
        const int h = c & 1;
        const uint32_t mb = mbar_addr(h);
        const uint32_t dt = (uint32_t)__cvta_generic_to_shared(RGT() + 32 * h);
        const uint32_t df = (uint32_t)__cvta_generic_to_shared(RGF() + 32 * h);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(384) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                     ::"r"(dt), "l"(P.arrival + (int64_t)c * 32), "r"(mb) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];"
                     ::"r"(df), "l"(P.flow + (int64_t)c * 32), "r"(mb) : "memory");
    }
    FI void ring_wait_chunk(int c) {   // every lane waits for chunk c
        const int h = c & 1;
        const uint32_t ph = *ring_ph_slot();
        const uint32_t mb = mbar_addr(h), par = (ph >> h) & 1u;
        uint32_t done = 0;
        #pragma unroll 1
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(mb), "r"(par) : "memory");
        __syncwarp();
        if (lane == 0) *ring_ph_slot() = ph ^ (1u << h);
        __syncwarp();
    }
    // The two mbarriers are initialised once per warp slice when the kernel
    // starts (ring_init) and keep their phases across the simulations the
    // warp runs; the parity bits live next to them between simulations.
    FI uint32_t* ring_ph_slot() const { return (uint32_t*)(sm + P.L.o_mbar + 16); }
    FI void ring_start() {
        if (n <= 0) return;
        const int c0 = (int)(toff >> 5);
        if (lane == 0) {
            ring_issue(c0);
            if (c0 < ring_last()) ring_issue(c0 + 1);
        }
        __syncwarp();
        ring_wait_chunk(c0);
    }
    // the cursor moved to trace position i: entering a new chunk waits for it
    // (fetched one chunk ago) and fetches the next one into the other half,
    // whose previous chunk has been fully consumed
    FI void ring_enter(int i) {
        const int64_t g = toff + i;
        if ((g & 31) != 0) return;
        const int c = (int)(g >> 5);
        ring_wait_chunk(c);
        if (c < ring_last()) {
            if (lane == 0) ring_issue(c + 1);
            __syncwarp();
        }
    }
    // no bulk copy may outlive the simulation: the chunk after the last one
    // entered (the cursor's, or the final entry's) is in flight unless it
    // does not exist
    FI void ring_drain() {
        if (n > 0) {
            const int c = (int)((toff + min(cursor, n - 1)) >> 5);
            if (c < ring_last()) ring_wait_chunk(c + 1);
        }
    }
    FI double ring_t(int i) const { return RGT()[(toff + i) & 63]; }
    FI int ring_f(int i) const { return RGF()[(toff + i) & 63]; }

    // ---- uniform scalar state (registers)
    double now, gvt;
    uint32_t seq;
    int cursor;                        // next trace position to arrive
    int nev;                           // occupied event slots
    bool tick_on; double tick_t; uint32_t tick_seq;
    bool pmin_ok; double pmin_t; uint32_t pmin_seq; int pmin_slot;
    int tot_pend, tot_infl;
    int fcfs_head, fcfs_infl, draining;
    int s_att, s_out, s_exec;
    int status;
    bool any_newly;
    int newly_n;                       // flows queued for swap-out (list in shared memory)
    bool gmin_ok; u64 gmin;            // (A) cached min okey(vt) over backlogged queues
    double idle_lb;                    // (B) no keep-alive can expire before this
    int n_events;
    int n_calls, n_disp, n_comp, n_util, n_backlog, n_evlog;
    int nbl;                           // SETS: backlogged-set size
    int n_evict;                       // Device.eviction_log rows (generic build)
    PySum util_sum;

    FI WarpSim(const Params& p, unsigned char* s, unsigned char* f, int l, int id)
        : P(p), sm(s), fe(f), lane(l), sid(id) {}

    // ---- CTA mode
    int wid, nthr;                     // warp index in the CTA, CTA threads
    int use_inf_;                      // candidate order uses in_flight (helpers' copy)
    FI CtaCmd* cmd() const { return (CtaCmd*)(sm + P.L.o_cta); }
    FI bool cta_on(int n) const { return CTA && n >= P.cta_min; }

    // This warp's share of a scan (every warp of the CTA runs it; flows
    // f = wid*32 + lane + k*nthr), reduced over the warp.
    FI Arg cta_part(int op) {
        Arg a = arg_none();
        const bool set_op = SETS && op != OP_EVMIN;
        const int lim = op == OP_EVMIN ? nev : set_op ? nbl : nf;
        #pragma unroll 1
        for (int b = wid * 32; b < lim; b += nthr) {
            const bool in = b + lane < lim;
            const int f = set_op ? (in ? (int)BLL()[b + lane] : 0) : b + lane;
            if (op == OP_GVT) {
                if (in && pt()[f] - done()[f] > 0) { u64 k = okey(vt()[f]); if (k < a.k) a.k = k; }
            } else if (op == OP_CAND) {
                if (in) {
                    int pe = pend()[f];
                    if (pe > 0 && vt()[f] - gvt <= T) {
                        unsigned inf = use_inf_ ? (unsigned)infl()[f] : 0u;
                        u64 k = ((u64)inf << 48) | ((u64)(0xffffffffu - (unsigned)pe) << 16) | (u64)f;
                        if (k < a.k) a.k = k;
                    }
                }
            } else if (op == OP_BATCH) {
                if (in && pend()[f] > 0) a.k = min(a.k, (u64)(unsigned)head()[f]);
            } else if (op == OP_SJF) {
                if (in && pend()[f] > 0) {
                    u64 k = okey(tau()[f]);
                    if (k < a.k || (k == a.k && f < a.i)) { a.k = k; a.i = f; }
                }
            } else if (op == OP_EVMIN) {
                if (in) {
                    u64 k = okey(ev_t()[f]); uint32_t q = ev_seq()[f];
                    if (k < a.k || (k == a.k && q < a.s)) { a.k = k; a.s = q; a.i = f; }
                }
            }
        }
        return warp_argmin(a);
    }

    // Leader: publish the command, do warp 0's share, combine every warp's.
    FI Arg cta_scan(int op) {
        CtaCmd* c = cmd();
        __syncwarp();
        if (lane == 0) {
            c->op = op; c->nf = nf; c->nev = nev; c->iarg = use_inf_; c->nset = nbl;
            c->gvt = gvt; c->now = now;
        }
        cta_bar(1, nthr);
        Arg a = cta_part(op);
        if (lane == 0) { c->pk[0] = a.k; c->ps[0] = a.s; c->pi[0] = a.i; }
        cta_bar(2, nthr);
        Arg b = arg_none();
        if (lane < (nthr >> 5)) { b.k = c->pk[lane]; b.s = c->ps[lane]; b.i = c->pi[lane]; }
        return warp_argmin(b);
    }

    // Helper warps: serve the leader's scans until it sends OP_EXIT.
    FI void helper_loop() {
        CtaCmd* c = cmd();
        #pragma unroll 1
        for (;;) {
            cta_bar(1, nthr);
            const int op = c->op;
            if (op == OP_EXIT) break;
            nf = c->nf; nev = c->nev; use_inf_ = c->iarg; gvt = c->gvt; now = c->now; nbl = c->nset;
            Arg a = cta_part(op);
            if (lane == 0) { c->pk[wid] = a.k; c->ps[wid] = a.s; c->pi[wid] = a.i; }
            cta_bar(2, nthr);
        }
    }
    FI void cta_release() {            // leader, end of the simulation
        __syncwarp();
        if (lane == 0) cmd()->op = OP_EXIT;
        cta_bar(1, nthr);
    }

    FI void fail(int st) { if (!status) status = st; }
#define UNLIKELY(x) __builtin_expect(!!(x), 0)
#define LIKELY(x) __builtin_expect(!!(x), 1)
    FI double ttl(int f) const {                          // FlowQueue.ttl, core.py:140-152
        if (alpha == 0.0) return 0.0;
        if (pt()[f] >= 2) return alpha * iat()[f];       // iat.count = arrivals - 1
        return dttl;
    }

    // ==================================================================
    // event pool (engine.py:83-87: heap of (time, seq, kind, payload))

    // the next monitor tick (now + period, never in the past: period > 0)
    FI void push_tick(double t) { tick_on = true; tick_t = t; tick_seq = seq++; }

    FI void push(double t, int kind, uint32_t payload) {
        if (UNLIKELY(t < now)) { fail(GFQ_SIM_PAST_EVENT); return; }     // engine.py:84-85
        uint32_t s = seq++;
        if (UNLIKELY(nev >= P.L.E)) { fail(GFQ_SIM_EVENT_OVERFLOW); return; }
        int slot = nev++;
        if (GFQ_DIAG && lane == 0) { uint32_t* dg = (uint32_t*)(sm + P.L.o_diag); dg[DG_MAXEV] = max(dg[DG_MAXEV], (uint32_t)nev); }
        USYNC();
        ev_t()[slot] = t; ev_seq()[slot] = s; ev_meta()[slot] = ((uint32_t)kind << 30) | payload;
        // (no trailing sync: every lane stored the same value)
        if (pmin_ok && (pmin_slot < 0 || t < pmin_t || (t == pmin_t && s < pmin_seq))) {
            pmin_t = t; pmin_seq = s; pmin_slot = slot;
        }
    }

    FI void pool_min() {                                  // lane-parallel argmin
        if (cta_on(nev)) {
            Arg a = cta_scan(OP_EVMIN);
            pmin_ok = true;
            if (a.i == 0x7fffffff) { pmin_slot = -1; pmin_t = __longlong_as_double(0x7ff0000000000000ll); return; }
            pmin_slot = a.i; pmin_t = from_key(a.k); pmin_seq = a.s;
            return;
        }
        u64 bt = ~0ull; uint32_t bs = 0xffffffffu; int bslot = -1;
        #pragma unroll SCAN_UNROLL
        for (int i = lane; i < nev; i += 32) {
            u64 k = okey(ev_t()[i]); uint32_t s = ev_seq()[i];
            if (k < bt || (k == bt && s < bs)) { bt = k; bs = s; bslot = i; }
        }
        u64 m = wmin64(bt);
        uint32_t ms = wmin32(bt == m ? bs : 0xffffffffu);
        int src = __ffs(__ballot_sync(FULLMASK, bt == m && bs == ms && bslot >= 0)) - 1;
        pmin_ok = true;
        if (src < 0) { pmin_slot = -1; pmin_t = __longlong_as_double(0x7ff0000000000000ll); return; }
        pmin_slot = __shfl_sync(FULLMASK, bslot, src);
        pmin_t = from_key(m); pmin_seq = ms;
    }

    FI void pool_remove(int slot) {
        int last = --nev;
        if (slot != last) {
            double t = ev_t()[last]; uint32_t s = ev_seq()[last], m = ev_meta()[last];
            USYNC();
            ev_t()[slot] = t; ev_seq()[slot] = s; ev_meta()[slot] = m;
        }
        pmin_ok = false;
    }

    // Backlogged set (SETS builds): unordered list + position index.  A flow
    // enters when its backlog (arrived - completed) leaves 0 and leaves when it
    // returns to 0; every scan over it reduces order-independently (min keys
    // that end in the flow id), so results equal the full scans'.
    FI void bl_add(int f) {
        USYNC();
        BLL()[nbl] = (uint16_t)f; BLP()[f] = (uint16_t)nbl;
        nbl++;
    }
    FI void bl_remove(int f) {
        const int p = BLP()[f];
        const int last = BLL()[nbl - 1];
        USYNC();
        BLL()[p] = (uint16_t)last; BLP()[last] = (uint16_t)p;
        nbl--;
    }
    FI int scan_n() const { return SETS ? nbl : nf; }                 // flows a set scan visits
    FI int scan_f(int i) const { return SETS ? (int)BLL()[i] : i; }   // i-th of them

    // ==================================================================
    // device model (device.py)

    FI int container_state(int d, int fn) {         // device.py:104-112
        if (!DV(d, DV_POOLON)) return GFQ_COLD;
        if (CNT(d, 0, fn) > 0) return GFQ_GPU_WARM;
        if (CNT(d, 1, fn) > 0) return GFQ_HOST_WARM;
        return GFQ_COLD;
    }

    // _idle_entry, device.py:96-102: first entry (list order) with the max
    // last_used_s among (fn, thermal); -1 if none
    FI int idle_entry(int d, int fn, int th) {
        int np = DV(d, DV_NP);
        u64 bk = ~0ull; int bi = 0x7fffffff;
        #pragma unroll 1
        for (int i = lane; i < np; i += 32) {
            uint32_t m = PM(d, i);
            if (pm_fn(m) == fn && pm_th(m) == th) {
                u64 k = ~okey(PT(d, i));
                if (k < bk) { bk = k; bi = i; }
            }
        }
        u64 mk = wmin64(bk);
        int r = (int)wmin32(bk == mk ? (unsigned)bi : 0x7fffffffu);
        return r == 0x7fffffff ? -1 : r;
    }

    // list.remove at position i (shift left), keeping the per-flow counts
    FI void pool_erase(int d, int i) {
        int np = DV(d, DV_NP);
        uint32_t m = PM(d, i);
        #pragma unroll 1
        for (int base = i; base < np - 1; base += 32) {
            int j = base + lane;
            uint32_t mm = 0; double tt = 0.0;
            bool act = j < np - 1;
            if (act) { mm = PM(d, j + 1); tt = PT(d, j + 1); }
            __syncwarp();
            if (act) { PM(d, j) = mm; PT(d, j) = tt; }
        }
        int k = pm_th(m) == GFQ_GPU_WARM ? 0 : 1;
        ust(CNT(d, k, pm_fn(m)), (uint16_t)(CNT(d, k, pm_fn(m)) - 1));
        ust(DV(d, DV_NP), np - 1);
    }

    // resident_mb, device.py:114-117: sum(idle GPU_WARM mem) + sum(running
    // mem), each a builtin Neumaier sum in list order (replayed via shuffles)
    FI double resident_mb(int d) {
        int np = DV(d, DV_NP);
        if (MEMI || mem_int) {
            // integral table (gfq_upload_flowtabs): both builtin sums are exact
            // integers, so one lane-parallel integer sum gives the same double.
            // Per lane < 2^32 (entries <= 2^20 MB each); the halves reduce
            // without overflow and recombine exactly.
            uint32_t acc = 0;
            #pragma unroll 1
            for (int i = lane; i < np; i += 32) {
                const uint32_t m = PM(d, i);
                if (pm_th(m) == GFQ_GPU_WARM) acc += memi(pm_fn(m));
            }
            const int nr = DV(d, DV_NRUN);
            #pragma unroll 1
            for (int r = lane; r < nr; r += 32) acc += memi(RI(d, r, 1));
            const uint32_t lo = __reduce_add_sync(FULLMASK, acc & 0xffffu);
            const uint32_t hi = __reduce_add_sync(FULLMASK, acc >> 16);
            return (double)hi * 65536.0 + (double)lo;
        }
        PySum a; ps_init(a);
        #pragma unroll 1
        for (int base = 0; base < np; base += 32) {
            int i = base + lane;
            double v = 0.0; bool g = false;
            if (i < np) { uint32_t m = PM(d, i); g = pm_th(m) == GFQ_GPU_WARM; if (g) v = mem(pm_fn(m)); }
            unsigned gm = __ballot_sync(FULLMASK, g);
            #pragma unroll 1
            while (gm) {
                int j = __ffs(gm) - 1; gm &= gm - 1;
                ps_add(a, __shfl_sync(FULLMASK, v, j));
            }
        }
        PySum b; ps_init(b);
        int nr = DV(d, DV_NRUN);
        #pragma unroll 1
        for (int r = 0; r < nr; r++) ps_add(b, mem(RI(d, r, 1)));
        return ps_val(a) + ps_val(b);
    }

    // admit_memory, device.py:147-179.  Victims are idle GPU_WARM entries in
    // a stable ascending last_used_s order; roll back if the deficit stays.
    FI bool admit_memory(int d, int fn) {
        if (CNT(d, 0, fn) > 0) return true;               // idle GPU_WARM exists
        double needed = mem(fn);
        double free_mb = DD(d, DD_MEMCAP) - resident_mb(d);
        if (LIKELY(free_mb >= needed)) return true;
        int np = DV(d, DV_NP);
        int nsw = 0;
        #pragma unroll 1
        while (free_mb < needed) {
            u64 bk = ~0ull; int bi = 0x7fffffff;
            #pragma unroll 1
            for (int i = lane; i < np; i += 32) {
                uint32_t m = PM(d, i);
                if (pm_th(m) == GFQ_GPU_WARM && !pm_sw(m)) {
                    u64 k = okey(PT(d, i));
                    if (k < bk) { bk = k; bi = i; }
                }
            }
            u64 mk = wmin64(bk);
            int v = (int)wmin32(bk == mk ? (unsigned)bi : 0x7fffffffu);
            if (v == 0x7fffffff) break;
            uint32_t m = PM(d, v);
            ust(PM(d, v), m | (1u << 27));                 // tentatively HOST_WARM
            free_mb += mem(pm_fn(m));
            nsw++;
            if (LG) evict_log(d, pm_fn(m));                // eviction_log.append, in victim order
        }
        bool ok = free_mb >= needed;
        if (LG && !ok) n_evict -= nsw;                     // rollback pops them (device.py:175-177)
        if (nsw) {   // commit (-> HOST_WARM) or roll back, one entry at a time
            #pragma unroll 1
            for (int base = 0; base < np; base += 32) {
                int i = base + lane;
                bool s = i < np && pm_sw(PM(d, i));
                unsigned smk = __ballot_sync(FULLMASK, s);
                #pragma unroll 1
                while (smk) {
                    int j = __ffs(smk) - 1; smk &= smk - 1;
                    int idx = base + j;
                    uint32_t m = PM(d, idx) & ~(1u << 27);
                    if (ok) {
                        int f = pm_fn(m);
                        ust(CNT(d, 0, f), (uint16_t)(CNT(d, 0, f) - 1));
                        ust(CNT(d, 1, f), (uint16_t)(CNT(d, 1, f) + 1));
                        m = (m & ~(3u << 24)) | ((uint32_t)GFQ_HOST_WARM << 24);
                    }
                    ust(PM(d, idx), m);
                }
            }
        }
        return ok;
    }

    // the function-independent part of try_acquire_token (device.py:134-139)
    FI bool token_free(int d) {
        int out = DV(d, DV_OUT);
        return out < DV(d, DV_EFFD) && (out == 0 || DV(d, DV_HROK));
    }

    // (C): every device refuses whatever the function
    FI bool certain_refusal() {
        if (SCRIPTED) return false;
        #pragma unroll 1
        for (int d = 0; d < NDEV(); d++) if (token_free(d)) return false;
        return true;
    }

    // try_acquire_token, device.py:124-145 -> start state or -1
    FI int try_acquire_token(int d, int fn) {
        if (!token_free(d)) return -1;
        int st = container_state(d, fn);
        if (st != GFQ_GPU_WARM) {
            if (!admit_memory(d, fn)) return -1;
        }
        ust(DV(d, DV_OUT), DV(d, DV_OUT) + 1);
        return st;
    }

    // ScriptedDevices.assign (tests/oracles.py:25-32) or DeviceSet.assign
    // (device.py:320-341): devices tried in sorted (pref, outstanding, index)
    // order, first grant wins.  A refusal leaves a device unchanged, so the
    // order is re-derived by repeated minimum selection.
    FI int provider_assign(int fn, int& st) {
        if (SCRIPTED) {
            s_att += 1;
            if (sim->scripted_deny_every && s_att % sim->scripted_deny_every == 0) return -1;
            if (s_out >= sim->scripted_d) return -1;
            s_out += 1;
            st = GFQ_GPU_WARM;
            return 0;
        }
        unsigned tried = 0;
        #pragma unroll 1
        for (int k = 0; k < NDEV(); k++) {
            int best = 0; int bkey = 0x7fffffff;
            #pragma unroll 1
            for (int d = 0; d < NDEV(); d++) {
                if (tried & (1u << d)) continue;
                int key = (container_state(d, fn) << 20) | (DV(d, DV_OUT) << 4) | d;
                if (key < bkey) { bkey = key; best = d; }
            }
            tried |= 1u << best;
            int r = try_acquire_token(best, fn);
            if (r >= 0) { st = r; return best; }
        }
        return -1;
    }

    FI int max_effective_d() {                      // device.py:317-318
        if (SCRIPTED) return sim->scripted_d;
        int m = DV(0, DV_EFFD);
        #pragma unroll 1
        for (int i = 1; i < NDEV(); i++) m = max(m, DV(i, DV_EFFD));
        return m;
    }

    // ---- running set (Device.running dict, insertion order)
    FI void run_append(int d, int inv, int fn, int st, double duration, double pure) {
        int nr = DV(d, DV_NRUN);
        if (UNLIKELY(nr >= P.L.R)) { fail(GFQ_SIM_POOL_OVERFLOW); return; }
        USYNC();
        RI(d, nr, 0) = inv; RI(d, nr, 1) = fn; RI(d, nr, 2) = st;
        RD(d, nr, 0) = duration; RD(d, nr, 1) = pure;
        DV(d, DV_NRUN) = nr + 1;
        ust(CNT(d, 2, fn), (uint16_t)(CNT(d, 2, fn) + 1));
        if (!SCRIPTED) ust(DV(d, DV_INSTDIRTY), 1);
    }
    FI bool run_remove(int d, int inv, double& duration, double& pure, int& st, int& fn) {
        int nr = DV(d, DV_NRUN);
        int ri = -1;
        #pragma unroll 1
        for (int r = 0; r < nr; r++) if (RI(d, r, 0) == inv) { ri = r; break; }
        if (ri < 0) { fail(GFQ_SIM_BAD_CONFIG); return false; }   // RuntimeError
        fn = RI(d, ri, 1);
        st = RI(d, ri, 2); duration = RD(d, ri, 0); pure = RD(d, ri, 1);
        #pragma unroll 1
        for (int r = ri; r < nr - 1; r++) {
            int a = RI(d, r + 1, 0), b = RI(d, r + 1, 1), c = RI(d, r + 1, 2);
            double x = RD(d, r + 1, 0), y = RD(d, r + 1, 1);
            USYNC();
            RI(d, r, 0) = a; RI(d, r, 1) = b; RI(d, r, 2) = c; RD(d, r, 0) = x; RD(d, r, 1) = y;
        }
        ust(DV(d, DV_NRUN), nr - 1);
        ust(CNT(d, 2, fn), (uint16_t)(CNT(d, 2, fn) - 1));
        if (!SCRIPTED) ust(DV(d, DV_INSTDIRTY), 1);
        return true;
    }

    // start_invocation, device.py:183-218
    FI void start_invocation(int d, int fn, int st, int inv, double& duration, double& pure) {
        double base;
        if (st == GFQ_GPU_WARM) {
            base = warm(fn);
        } else if (st == GFQ_HOST_WARM) {
            double transfer = pymax(0.0, mem(fn) / DD(d, DD_PCIE) - DD(d, DD_OVERLAP));
            base = warm(fn) + transfer;
        } else {
            base = cold(fn);
        }
        if (st != GFQ_COLD) {            // claim the freshest idle container of that class
            int claimed = idle_entry(d, fn, st);
            if (claimed >= 0) pool_erase(d, claimed);
        }
        int concurrent = DV(d, DV_NRUN) + 1;
        double factor = 1.0 + DD(d, DD_BETA) * (double)(concurrent - 1);
        duration = base * factor;
        pure = warm(fn) * factor;
        run_append(d, inv, fn, st, duration, pure);
    }

    // _enforce_pool_cap, device.py:239-258: destroy min by
    // (not spare, not evictable, last_used_s), first in list order on ties;
    // spare = another pooled container of the function exists and none runs
    FI void enforce_pool_cap(int d) {
        int cap = DV(d, DV_POOLMAX);
        #pragma unroll 1
        for (;;) {
            int np = DV(d, DV_NP), nr = DV(d, DV_NRUN);
            if (LIKELY(!(np + nr > cap && np > 0))) break;
            unsigned bk01 = 0xffffffffu; u64 bk2 = ~0ull; int bi = 0x7fffffff;
            #pragma unroll 1
            for (int i = lane; i < np; i += 32) {
                uint32_t m = PM(d, i); int f = pm_fn(m);
                bool spare = (int)CNT(d, 0, f) + (int)CNT(d, 1, f) > 1 && CNT(d, 2, f) == 0;
                unsigned k01 = ((unsigned)!spare << 1) | (unsigned)!pm_ev(m);
                u64 k2 = okey(PT(d, i));
                if (k01 < bk01 || (k01 == bk01 && k2 < bk2)) { bk01 = k01; bk2 = k2; bi = i; }
            }
            unsigned m01 = wmin32(bk01);
            u64 m2 = wmin64(bk01 == m01 ? bk2 : ~0ull);
            int v = (int)wmin32(bk01 == m01 && bk2 == m2 ? (unsigned)bi : 0x7fffffffu);
            pool_erase(d, v);
        }
    }

    // Device.complete, device.py:220-237
    FI bool device_complete(int d, int inv, int& fn, double& duration, double& pure, int& st) {
        if (!run_remove(d, inv, duration, pure, st, fn)) return false;
        ust(DV(d, DV_OUT), DV(d, DV_OUT) - 1);
        if (!DV(d, DV_POOLON)) return true;
        int np = DV(d, DV_NP);
        if (UNLIKELY(np >= P.L.P)) { fail(GFQ_SIM_POOL_OVERFLOW); return false; }
        // the re-pooled entry is (fn, GPU_WARM, mem[fn], now, evictable=False)
        // whether or not a container was claimed at start (device.py:226-236)
        USYNC();
        PM(d, np) = pm_make(fn, GFQ_GPU_WARM, 0);
        PT(d, np) = now;
        DV(d, DV_NP) = np + 1;
        ust(CNT(d, 0, fn), (uint16_t)(CNT(d, 0, fn) + 1));
        enforce_pool_cap(d);
        return true;
    }

    // instantaneous_util, device.py:279-280
    FI double instantaneous_util(int d) {
        PySum a; ps_init(a);
        int nr = DV(d, DV_NRUN);
        #pragma unroll 1
        for (int r = 0; r < nr; r++) ps_add(a, share(RI(d, r, 1)));
        return pymin(1.0, ps_val(a));
    }

    // monitor_tick, device.py:282-297 -> effective_d; inst = the util sample.
    // instantaneous_util is cached per device (it only changes when the
    // running set does).  The window average is a builtin Neumaier sum in
    // window order; it is memoised exactly: each device interns its distinct
    // sample values (<= WDICT) as 4-bit ids, the window is the shift register
    // of the ids of its samples, and (ids, count) fixes the summed sequence.
    // The tick's utilization sample (instantaneous_util, cached while the
    // running set is unchanged) and its interned id.
    FI double tick_util(int d, int& id_out) {
        double util = DD(d, DD_INST);
        int id = DV(d, DV_INSTID);
        if (DV(d, DV_INSTDIRTY)) {              // the running set changed since the last tick
            util = instantaneous_util(d);
            // intern: open-addressed table of WDICT slots (id = slot + 1),
            // empty slots hold an all-ones pattern (a NaN, never a utilization)
            const u64 ub = (u64)__double_as_longlong(util);
            int sl = (int)((((uint32_t)ub ^ (uint32_t)(ub >> 32)) * 0x9E3779B1u) >> 28);
            if (sl >= WDICT) sl = 0;
            id = 0;
            #pragma unroll 1
            for (int k = 0; k < WDICT; k++) {
                const u64 v = (u64)__double_as_longlong(WDICTV(d, sl));
                if (v == ub) { id = sl + 1; break; }
                if (v == ~0ull) {
                    USYNC();
                    WDICTV(d, sl) = util;
                    USYNC();
                    id = sl + 1;
                    break;
                }
                if (++sl == WDICT) sl = 0;
            }
            DD(d, DD_INST) = util; DV(d, DV_INSTDIRTY) = 0; DV(d, DV_INSTID) = id;
        }
        id_out = id;
        return util;
    }

    FI int monitor_tick(int d, double util, int id) {
        const int S = P.L.S;
        int head = DV(d, DV_SHEAD), ns = DV(d, DV_SN);
        // No overflow check: samples are a tick period apart and a window
        // keeps those newer than now - window, so at most
        // ceil(window / period) + 2 are held here, and gfq_prepare sizes
        // S = ceil(window / period) + 3 (the min period over the devices).
        int w = head + ns; if (w >= S) w -= S;
        const uint32_t code = ((uint32_t)DV(d, DV_WCODE) << 4) | (uint32_t)id;
        const int zage = id ? min(DV(d, DV_ZAGE) + 1, 15) : 0;
        USYNC();
        SMPT(d, w) = now; SMPU(d, w) = util;
        double oldt = ns == 0 ? now : DD(d, DD_OLDT);    // time of the oldest sample
        ns++;
        double horizon = now - (ND1 ? win0 : DD(d, DD_WINDOW));
        #pragma unroll 1
        while (ns > 0 && oldt <= horizon) {
            head++; if (head >= S) head = 0; ns--;
            oldt = SMPT(d, head);                          // ns >= 1: the new sample stays
        }
        double avg;
        // memo key: the window's ids and count (valid while the last ns ids
        // are all interned); 0xffffffff (never a key: count <= 7) marks empty
        const bool memo = ns <= WMAXN && zage >= ns;
        uint32_t key = 0xffffffffu; int slot = 0;
        if (memo) {
            key = (code & ((1u << (4 * ns)) - 1u)) | ((uint32_t)ns << 28);
            slot = (int)((key * 0x9E3779B1u) >> (32 - WMEMO_BITS));
        }
        int effd = DV(d, DV_EFFD), hrok = DV(d, DV_HROK);
        if (memo && key == (uint32_t)DV(d, DV_LKEY)) {
            // same window as the last tick: the same average, and (the key is
            // only kept for a fixed D) the same effective_d and headroom flag
            avg = UAVG(d);
        } else {
            if (LIKELY(memo && WKEY(d, slot) == key)) {
                avg = WVAL(d, slot);
                diag(DG_WHIT);
            } else {
                diag(DG_WMISS);
                PySum a; ps_init(a);
                int j = head;
                #pragma unroll 1
                for (int k = 0; k < ns; k++) { ps_add(a, SMPU(d, j)); j++; if (j >= S) j = 0; }
                avg = ps_val(a) / (double)ns;
                // a real barrier here (memo misses only): the slot may be
                // rewritten a few ticks later with no warp collective in
                // between, and racecheck cannot see convergence as ordering
                if (memo) { __syncwarp(); WKEY(d, slot) = key; WVAL(d, slot) = avg; }
            }
            const bool dyn = DV(d, DV_DYN);
            // a fixed D and an unchanged average leave effective_d and the
            // headroom check as they were
            if (dyn || __double_as_longlong(avg) != __double_as_longlong(UAVG(d))) {
                const int dmax = DV(d, DV_DMAX);
                const double thr = DD(d, DD_THR), inv = DD(d, DD_INVDMAX);
                if (!dyn) effd = dmax;
                else if (avg > thr) effd = max(effd - 1, 1);
                else if (avg < thr - inv) effd = min(effd + 1, dmax);
                hrok = !(avg + inv > thr);                              // device.py:137-139
            }
            if (dyn) key = 0xffffffffu;                  // dynamic D moves every tick
        }
        if (!ND1) __syncwarp();                          // 1-device build: registers
        DV(d, DV_SHEAD) = head; DV(d, DV_SN) = ns; UAVG(d) = avg; DV(d, DV_EFFD) = effd;
        DV(d, DV_HROK) = hrok; DV(d, DV_ZAGE) = zage;
        DV(d, DV_WCODE) = (int)code; DV(d, DV_LKEY) = (int)key;
        DD(d, DD_OLDT) = oldt;
        return effd;
    }

    // ==================================================================
    // scheduler (mqfq.py) and baseline policies (policies.py)

    // (A) recompute_global_vt, mqfq.py:114-127.  INACTIVE => not backlogged,
    // so the filter is "backlogged"; the minimum is cached (gmin).
    FI void recompute_gvt() {
        if (!gmin_ok && cta_on(scan_n())) {
            diag(DG_GSCAN);
            gmin = cta_scan(OP_GVT).k;
            gmin_ok = true;
        }
        if (UNLIKELY(!gmin_ok)) {
            diag(DG_GSCAN);
            u64 bk = ~0ull;
            const int ns = scan_n();
            #pragma unroll SCAN_UNROLL
            for (int i = lane; i < ns; i += 32) {
                const int f = scan_f(i);
                if (SETS || pt()[f] - done()[f] > 0) { u64 k = okey(vt()[f]); if (k < bk) bk = k; }
            }
            gmin = wmin64(bk);
            gmin_ok = true;
        }
        if (gmin != ~0ull) gvt = pymax(gvt, from_key(gmin));
    }

    // unstall, mqfq.py:129-139 (same backlogged set, ignoring the raise rule)
    FI void unstall() {
        if (tot_infl > 0) return;
        // the failed dispatch() that precedes every unstall (engine.py:177-181)
        // left the cached minimum valid
        if (!gmin_ok) { fail(GFQ_SIM_BAD_CONFIG); return; }
        if (gmin == ~0ull) return;
        double mv = from_key(gmin);
        if (gvt < mv) gvt = mv;
    }

    // (B) refresh_states, mqfq.py:159-161 / _update_state, mqfq.py:143-157,
    // restricted to what is observable: idle queues whose keep-alive expired
    // become INACTIVE (and are queued for swap-out).
    FI void refresh_states() {
        if (LIKELY(now < idle_lb)) return;
        diag(DG_RSCAN);
        const long long p0 = pclk();
        refresh_scan();
        prof(PF_REFRESH, p0);
    }
    FI void refresh_scan() {
        if (SETS) { refresh_blocks(); return; }   // every CTA build is a SETS build
        u64 lbk = ~0ull;
        bool newly = false;
        #pragma unroll 1
        for (int base = 0; base < nf; base += 32) {      // warp-uniform trip count
            const int f = base + lane;
            bool idle = false, mk = false;
            uint8_t s = 0;
            double le = 0.0, tt = 0.0;
            if (f < nf) {
                s = fst()[f];
                idle = (s & (FL_CREATED | FL_INACTIVE)) == FL_CREATED && pt()[f] - done()[f] == 0;
                if (idle) { le = lex()[f]; tt = ttl(f); mk = now - le >= tt; }
            }
            if (!SCRIPTED) {                               // compact the marked flows into the list
                unsigned bm = __ballot_sync(FULLMASK, mk);
                int pos = newly_n + __popc(bm & ((1u << lane) - 1));
                if (mk && pos < NEWLY_CAP) NEWLY()[pos] = f;
                newly_n += __popc(bm);
            }
            if (mk) {
                fst()[f] = (uint8_t)(s | FL_INACTIVE | (SCRIPTED ? 0 : FL_NEWLY));
                newly = true;
            } else if (idle) {
                u64 k = okey(expiry_lb(le, tt));
                if (k < lbk) lbk = k;
            }
        }
        __syncwarp();
        if (wor32(newly) && !SCRIPTED) any_newly = true;
        u64 m = wmin64(lbk);
        idle_lb = m == ~0ull ? __longlong_as_double(0x7ff0000000000000ll) : from_key(m);
    }

    // Large-flow builds: refresh_states over the 32-flow blocks whose expiry
    // bound has passed.  BMIN[b] is a lower bound on expiry_lb() of every idle
    // queue in block b: lowered when a queue of the block drains
    // (policy_on_completion), never raised except here, where the block is
    // rescanned and gets its exact bound.  A queue can only be expired when
    // now >= its expiry_lb >= its block's bound, so every expired queue lies
    // in a visited block and the marks equal the full scan's; idle_lb becomes
    // the minimum over all the blocks' bounds (still a valid lower bound).
    // One warp does it all (the leader in CTA builds).
    FI void refresh_blocks() {
        const int nb = (nf + 31) >> 5;
        u64 lbk = ~0ull;
        bool newly = false;
        #pragma unroll 1
        for (int base = 0; base < nb; base += 32) {
            const int b = base + lane;
            const double bm = b < nb ? BMIN()[b] : __longlong_as_double(0x7ff0000000000000ll);
            const bool hit = b < nb && bm <= now;
            if (!hit) { u64 k = okey(bm); if (k < lbk) lbk = k; }
            unsigned hm = __ballot_sync(FULLMASK, hit);
            #pragma unroll 1
            while (hm) {
                const int bb = base + __ffs(hm) - 1; hm &= hm - 1;
                const int f = bb * 32 + lane;
                bool idle = false, mk = false;
                uint8_t s = 0;
                double le = 0.0, tt = 0.0;
                if (f < nf) {
                    s = fst()[f];
                    idle = (s & (FL_CREATED | FL_INACTIVE)) == FL_CREATED && pt()[f] - done()[f] == 0;
                    if (idle) { le = lex()[f]; tt = ttl(f); mk = now - le >= tt; }
                }
                if (!SCRIPTED) {
                    unsigned bm2 = __ballot_sync(FULLMASK, mk);
                    int pos = newly_n + __popc(bm2 & ((1u << lane) - 1));
                    if (mk && pos < NEWLY_CAP) NEWLY()[pos] = f;
                    newly_n += __popc(bm2);
                }
                u64 k = ~0ull;
                if (mk) {
                    fst()[f] = (uint8_t)(s | FL_INACTIVE | (SCRIPTED ? 0 : FL_NEWLY));
                    newly = true;
                } else if (idle) {
                    k = okey(expiry_lb(le, tt));
                }
                const u64 m = wmin64(k);
                __syncwarp();
                if (lane == 0) BMIN()[bb] = m == ~0ull ? __longlong_as_double(0x7ff0000000000000ll) : from_key(m);
                if (m < lbk) lbk = m;
            }
        }
        __syncwarp();
        if (wor32(newly) && !SCRIPTED) any_newly = true;
        const u64 m = wmin64(lbk);
        idle_lb = m == ~0ull ? __longlong_as_double(0x7ff0000000000000ll) : from_key(m);
    }

    // candidates (mqfq.py:200-205) + the two stable sorts (mqfq.py:213-215):
    // lexicographic min of (in_flight if D != 1, -len(pending), name)
    FI int mqfq_candidate() {
        diag(DG_CSCAN);
        bool use_inf = max_effective_d() != 1;
        if (cta_on(scan_n())) {
            use_inf_ = use_inf;
            u64 m = cta_scan(OP_CAND).k;
            return m == ~0ull ? -1 : (int)(m & 0xffffu);
        }
        u64 bk = ~0ull;
        const int ns = scan_n();
        #pragma unroll SCAN_UNROLL
        for (int i = lane; i < ns; i += 32) {
            const int f = scan_f(i);
            int pe = pend()[f];
            if (pe > 0 && vt()[f] - gvt <= T) {
                unsigned inf = use_inf ? (unsigned)infl()[f] : 0u;
                u64 k = ((u64)inf << 48) | ((u64)(0xffffffffu - (unsigned)pe) << 16) | (u64)f;
                if (k < bk) bk = k;
            }
        }
        u64 m = wmin64(bk);
        return m == ~0ull ? -1 : (int)(m & 0xffffu);
    }

    // BatchPolicy._oldest_nonempty, policies.py:197-208: key (arrival_s, uid)
    // == smallest trace position among the queue heads
    FI int batch_candidate() {
        int dr = draining;
        if (dr >= 0 && (pend()[dr] > 0 || infl()[dr] > 0))
            return pend()[dr] == 0 ? -1 : dr;                // hold for late arrivals
        diag(DG_CSCAN);
        if (cta_on(scan_n())) {
            u64 m = cta_scan(OP_BATCH).k;
            return m == ~0ull ? -1 : flw((int)m);
        }
        unsigned bk = 0xffffffffu;
        const int ns = scan_n();
        #pragma unroll SCAN_UNROLL
        for (int i = lane; i < ns; i += 32) {
            const int f = scan_f(i);
            if (pend()[f] > 0) bk = min(bk, (unsigned)head()[f]);
        }
        unsigned m = wmin32(bk);
        return m == 0xffffffffu ? -1 : flw((int)m);
    }

    // SjfPolicy.dispatch, policies.py:245-262: min tau.mean, name order on ties
    FI int sjf_candidate() {
        diag(DG_CSCAN);
        if (cta_on(scan_n())) {
            Arg a = cta_scan(OP_SJF);
            return a.k == ~0ull ? -1 : a.i;
        }
        u64 bk = ~0ull; int bf = 0x7fffffff;
        const int ns = scan_n();
        #pragma unroll SCAN_UNROLL
        for (int i = lane; i < ns; i += 32) {
            const int f = scan_f(i);
            if (pend()[f] > 0) {
                u64 k = okey(tau()[f]);
                if (k < bk || (SETS && k == bk && f < bf)) { bk = k; bf = f; }   // name order on ties
            }
        }
        u64 m = wmin64(bk);
        if (m == ~0ull) return -1;
        return (int)wmin32(bk == m ? (unsigned)bf : 0x7fffffffu);
    }

    FI void audit_dispatch(int inv, double vt_before, double g, int qlen, int infl_after) {
        int k = n_disp++;
        if (P.outputs & GFQ_WANT_DISPATCH) {
            if (lane == 0) {
                int64_t o = roff + k;
                P.dsp_inv[o] = inv; P.dsp_vt[o] = vt_before; P.dsp_gvt[o] = g;
                P.dsp_qlen[o] = qlen; P.dsp_infl[o] = infl_after;
                if (LG) P.dsp_ev[o] = n_events;        // Simulation.step() replay
            }
            __syncwarp();                    // reconverge after the lane-0 write
        }
    }

    // One Policy.dispatch call for every policy kind; returns the started
    // invocation's trace position (or -1) with its function/device/state.
    FI int dispatch_once(int& fn_out, int& dev_out, int& st_out) {
        n_calls++;
        int fn = -1;
        if (MQFQ) {
            recompute_gvt();
            refresh_states();
            if (tot_pend > 0 && !certain_refusal()) fn = mqfq_candidate();
        } else if (tot_pend > 0 && !certain_refusal()) {
            if (FCFS) fn = fcfs_head < cursor ? flw(fcfs_head) : -1;   // policies.py:129-139
            else if (BATCH) fn = batch_candidate();
            else if (SJF) fn = sjf_candidate();
        }
        if (fn < 0) return -1;
        int st = 0;
        int dev = provider_assign(fn, st);
        if (dev < 0) return -1;
        int inv;
        if (FCFS) {
            inv = fcfs_head++;
            fcfs_infl++;
            audit_dispatch(inv, 0.0, 0.0, (cursor - fcfs_head) + 1, fcfs_infl);
        } else {
            // FlowQueue.pending.popleft()
            inv = head()[fn];
            int k = ph()[fn] + 1;
            int nxt = k < pt()[fn] ? __ldg(P.fpos + toff + __ldg(foff + fn) + k) : -1;
            int pe = pend()[fn] - 1, ninf = infl()[fn] + 1;
            double vt_before = vt()[fn];
            double nvt = vt_before;
            if (MQFQ) nvt = vt_before + tau()[fn] / weight(fn);          // mqfq.py:223
            USYNC();
            ph()[fn] = k; head()[fn] = nxt; pend()[fn] = pe; infl()[fn] = ninf;
            if (MQFQ) { vt()[fn] = nvt; lex()[fn] = now; }
            if (BATCH) draining = fn;
            if (MQFQ) {
                if (gmin_ok && nvt != vt_before && okey(vt_before) == gmin) gmin_ok = false;
                audit_dispatch(inv, vt_before, gvt, pe + 1, ninf);
                // mqfq.py:238 recomputes the global VT here; _drain always calls
                // dispatch() again next (engine.py:175-184), which recomputes it
                // before any read, and nothing in between reads it: done there
            } else {
                audit_dispatch(inv, 0.0, 0.0, pe + 1, ninf);
            }
        }
        tot_pend--; tot_infl++;
        fn_out = fn; dev_out = dev; st_out = st;
        return inv;
    }

    // on_arrival of every policy (mqfq.py:186-188 + core.py:120-138;
    // policies.py:126-127,172-173,242-243)
    FI void policy_on_arrival(int inv, int fn) {
        uint8_t s = fst()[fn];
        int p0 = pt()[fn], pe = pend()[fn], d0 = done()[fn];
        double v = vt()[fn], le = lex()[fn], im = iat()[fn];
        int hd = head()[fn];
        if (UNLIKELY(!(s & FL_CREATED))) {                // queue_for, mqfq.py:94-99
            s = FL_CREATED | FL_INACTIVE;
            v = 0.0;
            le = MQFQ ? now : 0.0;
        }
        tot_pend++;
        if (!FCFS) {
            if (MQFQ && (s & FL_INACTIVE)) {              // reactivation clamp, core.py:128-130
                v = pymax(v, gvt);
                s &= (uint8_t)~FL_INACTIVE;
            }
            if (pe == 0) hd = inv;                        // pending.append
            if (MQFQ && p0 >= 1) {                        // iat.record(now - last_arrival)
                double x = now - larr()[fn];
                im = im + (x - im) / (double)p0;
            }
            if (MQFQ && p0 == d0 && gmin_ok) {            // (A) queue becomes backlogged
                u64 k = okey(v);
                if (k < gmin) gmin = k;
            }
            if (LG && MQFQ && P.L.o_lst) {                 // FlowQueue.enqueue start tag, core.py:131-134
                double* lst = (double*)(fe + P.L.o_lst);
                const double stag = pymax(lst[fn], v + (double)pe * tau()[fn]);
                ust(lst[fn], stag);
                if (lane == 0) P.rec_stag[roff + inv] = stag;
                __syncwarp();
            }
        }
        USYNC();
        fst()[fn] = s; pt()[fn] = p0 + 1; pend()[fn] = pe + 1;
        vt()[fn] = v; lex()[fn] = le; iat()[fn] = im; head()[fn] = hd;
        if (MQFQ) larr()[fn] = now;
    }

    // on_completion of every policy (mqfq.py:241-247; policies.py:141-142,210-213,264-267)
    FI void policy_on_completion(int fn, double exec_s) {
        tot_infl--;
        int dn = done()[fn] + 1;
        if (FCFS) { fcfs_infl -= 1; ust(done()[fn], (CI)dn); return; }
        int inf = infl()[fn] - 1;
        double tm = tau()[fn];
        tm = tm + (exec_s - tm) / (double)dn;            // tau.count == completions
        USYNC();
        done()[fn] = dn; infl()[fn] = inf; tau()[fn] = tm;
        if (MQFQ) lex()[fn] = now;
        if (MQFQ && pt()[fn] == dn) {                     // queue drained (idle)
            if (gmin_ok && okey(vt()[fn]) == gmin) gmin_ok = false;          // (A)
            const double lb = expiry_lb(now, ttl(fn));
            idle_lb = pymin(idle_lb, lb);                                    // (B)
            if (SETS) ust(BMIN()[fn >> 5], pymin(BMIN()[fn >> 5], lb));
        }
    }

    // ==================================================================
    // engine (engine.py)

    FI void backlog_audit(int fn, bool on) {
        if (!LG) return;
        int k = n_backlog++;
        if ((LG && (P.outputs & GFQ_WANT_AUDIT)) && lane == 0 && k < P.audit_backlog_cap) {
            int64_t o = (int64_t)sid * P.audit_backlog_cap + k;
            P.backlog_time[o] = now; P.backlog_meta[o] = (fn << 1) | (on ? 1 : 0);
        }
        if (LG) __syncwarp();
    }

    // Device.eviction_log row (device.py:92): lane 0 writes (now, device, flow)
    // at the simulation's record offset (evictions <= completions: a container
    // turns GPU_WARM only when an invocation completes into the pool)
    FI void evict_log(int d, int fn) {
        const int k = n_evict++;
        if ((P.outputs & GFQ_WANT_EVICTIONS) && lane == 0) {
            const int64_t o = P.sim_roff[sid] + k;
            P.evict_time[o] = now; P.evict_meta[o] = (fn << 4) | d; P.evict_ev[o] = n_events;
        }
    }
    // Device.swap_out's log rows (device.py:270-275) for this call's newly
    // inactive flows: per function (ascending: one refresh_states pass, or
    // the single expiring flow), per device, GPU_WARM entries in pool order.
    // Enumerated by repeated warp argmin over (device, flow, pool index).
    FI void swap_out_log() {
        #pragma unroll 1
        for (int d = 0; d < NDEV(); d++) {
            const int np = DV(d, DV_NP);
            u64 last = 0; bool first = true;
            #pragma unroll 1
            while (true) {
                u64 bk = ~0ull;
                #pragma unroll 1
                for (int i = lane; i < np; i += 32) {
                    const uint32_t m = PM(d, i);
                    if (pm_th(m) == GFQ_GPU_WARM && (fst()[pm_fn(m)] & FL_NEWLY)) {
                        const u64 k = ((u64)pm_fn(m) << 32) | (u64)i;
                        if ((first || k > last) && k < bk) bk = k;
                    }
                }
                const u64 mk = wmin64(bk);
                if (mk == ~0ull) break;
                evict_log(d, (int)(mk >> 32));
                last = mk; first = false;
            }
        }
    }

    // _swap_out_inactive, engine.py:199-203 (+ Device.swap_out / mark_evictable)
    FI void swap_out_inactive() {
        if (LIKELY(!any_newly)) return;
        any_newly = false;
        if (LG && (P.outputs & GFQ_WANT_EVICTIONS)) swap_out_log();
        if (newly_n <= NEWLY_CAP) {
            // no idle container of any listed function on any device: swap_out
            // and mark_evictable change nothing, and a later unmark_evictable
            // finds nothing to clear (containers pooled later are not
            // evictable), so only the NEWLY flags go
            bool has = false;
            if (lane < newly_n) {
                const int f = NEWLY()[lane];
                #pragma unroll 1
                for (int d = 0; d < NDEV(); d++) has |= (CNT(d, 0, f) | CNT(d, 1, f)) != 0;
            }
            if (!__any_sync(FULLMASK, has)) {
                if (lane < newly_n) { const int f = NEWLY()[lane]; fst()[f] = (uint8_t)(fst()[f] & ~FL_NEWLY); }
                __syncwarp();
                newly_n = 0;
                return;
            }
        }
        #pragma unroll 1
        for (int d = 0; d < NDEV(); d++) {
            int np = DV(d, DV_NP);
            #pragma unroll 1
            for (int i = lane; i < np; i += 32) {
                uint32_t m = PM(d, i);
                if (fst()[pm_fn(m)] & FL_NEWLY) {
                    m |= (1u << 26);                                    // evictable
                    if (pm_th(m) == GFQ_GPU_WARM) m = (m & ~(3u << 24)) | ((uint32_t)GFQ_HOST_WARM << 24);
                    PM(d, i) = m;
                }
            }
        }
        __syncwarp();
        if (newly_n <= NEWLY_CAP) {          // the listed flows (usually one)
            #pragma unroll 1
            for (int k = 0; k < newly_n; k++) {
                const int f = NEWLY()[k];
                #pragma unroll 1
                for (int d = 0; d < NDEV(); d++) {
                    uint16_t g = CNT(d, 0, f), hw = CNT(d, 1, f);
                    __syncwarp();
                    CNT(d, 1, f) = (uint16_t)(hw + g); CNT(d, 0, f) = 0;
                    __syncwarp();
                }
                ust(fst()[f], (uint8_t)((fst()[f] & ~FL_NEWLY) | FL_MARKED));
            }
        } else {                             // list overflow: scan every flow
            #pragma unroll SCAN_UNROLL
            for (int f = lane; f < nf; f += 32) {
                uint8_t s = fst()[f];
                if (s & FL_NEWLY) {
                    #pragma unroll 1
                    for (int d = 0; d < NDEV(); d++) { CNT(d, 1, f) += CNT(d, 0, f); CNT(d, 0, f) = 0; }
                    fst()[f] = (uint8_t)((s & ~FL_NEWLY) | FL_MARKED);
                }
            }
            __syncwarp();
        }
        newly_n = 0;
    }

    // _start, engine.py:187-197
    FI void start(int inv, int fn, int dev, int st) {
        double duration, pure;
        if (SCRIPTED) {
            // drive(): completion at now + next(exec_iter) (oracles.py:235-236)
            duration = P.execs[sim->exec_off + (s_exec % sim->exec_len)];
            s_exec++;
            pure = duration;
            run_append(0, inv, fn, st, duration, pure);
        } else {
            start_invocation(dev, fn, st, inv, duration, pure);
        }
        if (status) return;
        if (P.outputs & GFQ_WANT_RECORDS) {
            if (lane == 0) {
                int64_t o = roff + inv;
                P.rec_dispatch[o] = now; P.rec_state[o] = (int8_t)st; P.rec_device[o] = (int8_t)dev;
                P.rec_pure[o] = pure;
            }
            __syncwarp();
        }
        push(now + duration, EV_COMPLETION, (uint32_t)inv | ((uint32_t)dev << 27));
    }

    // _drain, engine.py:173-185 (the swap-out after the loop is done by the
    // caller, once per event)
    // A drain whose single dispatch() call provably returns None and is not
    // retried after unstall (engine.py:177-181): the global-VT recompute is
    // idempotent (the cached minimum is valid and already applied), no
    // keep-alive can expire yet (B), and either nothing is pending or every
    // device refuses (C) while something is in flight.  Such a drain is one
    // counted dispatch() call and no state change.
    FI bool quiet_drain() {
        if (MQFQ && !(gmin_ok && now < idle_lb)) return false;
        return tot_pend == 0 || (tot_infl > 0 && certain_refusal());
    }

    FI void drain() {
        if (quiet_drain()) { n_calls++; diag(DG_QUIET); return; }
        bool retried = false;
        #pragma unroll 1
        for (;;) {
            int fn, dev, st;
            int inv = dispatch_once(fn, dev, st);
            if (inv < 0) {
                if (!retried && tot_infl == 0 && tot_pend > 0) {
                    if (MQFQ) unstall();
                    retried = true;
                    continue;
                }
                break;
            }
            retried = false;
            start(inv, fn, dev, st);
            if (status) return;
        }
    }

    FI void on_arrival(int inv, int fn) {                 // engine.py:121-129
        if (SETS && pt()[fn] - done()[fn] == 0) bl_add(fn);            // backlog 0 -> 1
        if (!SCRIPTED) {
            if (pt()[fn] - done()[fn] == 0) backlog_audit(fn, true);   // _backlog_change(+1)
            if (UNLIKELY(fst()[fn] & FL_MARKED)) {         // unmark_evictable on every device
                #pragma unroll 1
                for (int d = 0; d < NDEV(); d++) {
                    int np = DV(d, DV_NP);
                    #pragma unroll 1
                    for (int i = lane; i < np; i += 32) {
                        uint32_t m = PM(d, i);
                        if (pm_fn(m) == fn) PM(d, i) = m & ~(1u << 26);
                    }
                }
                ust(fst()[fn], (uint8_t)(fst()[fn] & ~FL_MARKED));
            }
        }
        policy_on_arrival(inv, fn);
        if (!SCRIPTED && !tick_on) push_tick(now + period);
    }

    // Completion stream (InvocationRecords in completion order, read by the
    // reducer and the fairness audit): staged 32 at a time in shared memory
    // and written back by the whole warp, coalesced.
    FI void comp_flush(int cnt) {
        __syncwarp();
        if (lane < cnt) {
            const int64_t o = roff + ((n_comp - 1) & ~31) + lane;
            P.comp_lat[o] = CST()[lane];
            P.comp_pos[o] = CSP()[lane];
            P.comp_meta[o] = CSM()[lane];
        }
        __syncwarp();
    }

    FI void on_completion(int inv, int dev) {             // engine.py:131-153
        int fn = 0;
        double duration = 0.0, pure = 0.0; int st = 0;
        if (SCRIPTED) {
            s_out -= 1;
            if (!run_remove(0, inv, duration, pure, st, fn)) return;
            policy_on_completion(fn, duration);
        } else {
            if (!device_complete(dev, inv, fn, duration, pure, st)) return;
            policy_on_completion(fn, tau_inc ? duration : pure);
        }
        int k = n_comp++;
        if (lane == 0) {
            const int cm = fn | ((st == GFQ_COLD) ? (int)0x80000000 : 0);
            if (CSTAGE) {
                CST()[k & 31] = now;        // latency = now - arrival, taken by the reducer
                CSP()[k & 31] = inv;
                CSM()[k & 31] = cm;
            } else {
                P.comp_lat[roff + k] = now; P.comp_pos[roff + k] = inv; P.comp_meta[roff + k] = cm;
            }
            if (P.outputs & GFQ_WANT_RECORDS) {
                P.rec_complete[roff + inv] = now;
                P.rec_order[roff + inv] = k;
            }
        }
        __syncwarp();
        if (CSTAGE && (k & 31) == 31) comp_flush(32);
        if (SETS && pt()[fn] - done()[fn] == 0) bl_remove(fn);         // backlog 1 -> 0
        if (!SCRIPTED && pt()[fn] - done()[fn] == 0) {     // _backlog_change(-1)
            backlog_audit(fn, false);
            if (MQFQ) push(now + ttl(fn), EV_EXPIRY, (uint32_t)fn);
        }
    }

    FI void on_monitor() {                                // engine.py:155-165
        #pragma unroll 1
        for (int d = 0; d < NDEV(); d++) {
            int id;
            const double inst = tick_util(d, id);
            // the mean-utilization sum first: its fp64 chain overlaps the
            // window work below (adding +0.0, nothing running, leaves a
            // Neumaier sum of non-negative terms bit-for-bit unchanged)
            if (inst != 0.0) ps_add(util_sum, inst);
            int eff = monitor_tick(d, inst, id);
            int k = n_util++;
            if ((LG && (P.outputs & GFQ_WANT_AUDIT)) && lane == 0 && k < P.audit_util_cap) {
                int64_t o = (int64_t)sid * P.audit_util_cap + k;
                P.util_rows[o * 3 + 0] = now; P.util_rows[o * 3 + 1] = inst;
                P.util_rows[o * 3 + 2] = UAVG(d);
                P.util_meta[o * 2 + 0] = d; P.util_meta[o * 2 + 1] = eff;
            }
            if (LG) __syncwarp();
        }
        if (cursor < n || tot_pend > 0 || tot_infl > 0) push_tick(now + period);
        else { tick_on = false; tick_t = __longlong_as_double(0x7ff0000000000000ll); }
    }

    FI void on_expiry(int fn) {                           // engine.py:167-171
        // expiry_check, mqfq.py:163-176 (the recheck is pushed before the
        // swap-out; the swap-out creates no event, so the order is immaterial)
        uint8_t s = fst()[fn];
        if ((s & FL_CREATED) && pt()[fn] - done()[fn] == 0) {
            double le = lex()[fn], tt = ttl(fn);
            bool inact = now - le >= tt;
            if (inact && !(s & FL_INACTIVE)) {
                ust(fst()[fn], (uint8_t)(s | FL_INACTIVE | FL_NEWLY));
                if (newly_n < NEWLY_CAP) ust(NEWLY()[newly_n], fn);
                newly_n++;
                any_newly = true;
            } else if (!inact && (s & FL_INACTIVE)) {
                // unreachable: INACTIVE is absorbing while idle (lex and ttl
                // only change on dispatch/arrival); kept for fidelity
                ust(fst()[fn], (uint8_t)(s & ~FL_INACTIVE));
            }
            if (!inact) {
                double due = le + tt;
                if (due > now) push(due, EV_EXPIRY, (uint32_t)fn);
            }
        }
    }

    FI void log_event(double t, int kind, long long payload) {
        if (!LG) return;
        int k = n_evlog++;
        if ((LG && (P.outputs & GFQ_WANT_EVENTS)) && lane == 0 && k < P.event_log_cap) {
            int64_t o = (int64_t)sid * P.event_log_cap + k;
            P.event_time[o] = t;
            P.event_meta[o] = (int64_t)((payload << 2) | kind);
        }
        if (LG) __syncwarp();
    }

    // Simulation.run / step, engine.py:99-119
    FI void run() {
        long long me = sim->max_events > 0 ? sim->max_events : 64ll * ((long long)n + 1024);
        const int max_events = (int)min(me, 0x7fffffffll);
        const double INF = __longlong_as_double(0x7ff0000000000000ll);
        if (RING) ring_start();
        double t_arr = n > 0 ? (RING ? ring_t(0) : arr(0)) : INF;
        // trailing keep-alive expiries still log events and swap-out evictions
        const bool early = P.early_exit && !(LG && (P.outputs & (GFQ_WANT_EVENTS | GFQ_WANT_EVICTIONS)));
        #pragma unroll 1
        for (;;) {
            if (!pmin_ok) { const long long p0 = pclk(); pool_min(); prof(PF_POOL, p0); }
            if (!tick_on) {            // no tick scheduled: the run is ending
                if (cursor >= n && pmin_slot < 0) break;
                // exact early exit: only keep-alive rechecks remain, which change
                // no record, dispatch row, audit row or statistic
                if (early && cursor >= n && tot_pend == 0 && tot_infl == 0) break;
            }
            // earliest (time, seq): arrivals (seq = trace index < every dynamic
            // seq) win time ties.  An absent tick or pooled event keeps its time
            // at +inf (tick_t / pmin_t invariants), and with neither present and
            // no arrival left the loop has ended above, so no +inf tie remains.
            int kind; double t;
            if ((t_arr <= tick_t) & (t_arr <= pmin_t) & (t_arr != INF)) { kind = EV_ARRIVAL; t = t_arr; }
            else if ((tick_t < pmin_t) | ((tick_t == pmin_t) & (tick_seq < pmin_seq))) { kind = EV_TICK; t = tick_t; }
            else { kind = 4; t = pmin_t; }
            if (UNLIKELY(n_events >= max_events)) { fail(GFQ_SIM_WATCHDOG); break; }
            now = t;
            n_events++;
            bool dr = true;
            const long long p0 = pclk();
            if (kind == EV_ARRIVAL) {
                int inv = cursor++;
                const int fn = RING ? ring_f(inv) : flw(inv);
                if (cursor < n) {
                    if (RING) { ring_enter(cursor); t_arr = ring_t(cursor); }
                    else t_arr = arr(cursor);
                } else {
                    t_arr = INF;
                }
                log_event(t, EV_ARRIVAL, inv);
                on_arrival(inv, fn);
                prof(PF_ARR, p0);
            } else if (kind == EV_TICK) {
                // A run of ticks: while the drain after a tick is provably quiet
                // (one counted dispatch() call, no state change) and the next
                // event is again the tick, stay in this loop.  A tick whose drain
                // may dispatch falls through to the common drain() below.
                // During the run nothing but the tick is pushed, so the next
                // arrival and the pooled minimum stay put, and both win a
                // time tie with the tick (an arrival's seq is its trace index;
                // a pooled event was pushed before the tick): the run ends at
                // the first tick with time >= lim.
                const double lim = pymin(t_arr, pmin_t);
                // quiet_drain() with the terms a run cannot change hoisted: no
                // dispatch, completion or refresh happens inside it, so only
                // the clock (keep-alive bound) and the device window's
                // effective_d / headroom flag move from tick to tick
                const bool q_gvt = !MQFQ || gmin_ok;
                const bool q_idle = tot_pend == 0, q_busy = tot_infl > 0;
                #pragma unroll 1
                for (;;) {
                    tick_on = false;
                    diag(DG_TICKS);
                    log_event(now, EV_TICK, -1);
                    on_monitor();
                    // bitwise, not short-circuit: one branch per test
                    const bool quiet = q_gvt & (!MQFQ | (now < idle_lb)) &
                                       (q_idle | (q_busy & certain_refusal()));
                    if ((status != 0) | !quiet) break;
                    n_calls++;
                    diag(DG_QUIET);
                    dr = false;
                    if (!tick_on | (n_events >= max_events) | (tick_t >= lim)) break;
                    now = tick_t;
                    n_events++;
                    dr = true;
                }
                prof(PF_TICK, p0);
            } else {
                int slot = pmin_slot;
                uint32_t meta = ev_meta()[slot];
                pool_remove(slot);
                uint32_t pay = meta & 0x3fffffffu;
                if ((meta >> 30) == EV_COMPLETION) {
                    int inv = (int)(pay & 0x7ffffffu);
                    log_event(t, EV_COMPLETION, inv);
                    on_completion(inv, (int)(pay >> 27));
                    prof(PF_COMP, p0);
                } else {
                    log_event(t, EV_EXPIRY, (long long)pay);
                    on_expiry((int)pay);
                    prof(PF_EXP, p0);
                    dr = false;
                }
            }
            if (UNLIKELY(status)) break;
            if (dr) { const long long p1 = pclk(); drain(); prof(PF_DRAIN, p1); }
            if (UNLIKELY(status)) break;
            if (!SCRIPTED) { const long long p1 = pclk(); swap_out_inactive(); prof(PF_EXP, p1); }
        }
        if (RING) ring_drain();
        if (CSTAGE && (n_comp & 31)) comp_flush(n_comp & 31);
    }
};

#undef SCRIPTED
#undef MQFQ
#undef FCFS
#undef BATCH
#undef SJF
}  // namespace gfq
