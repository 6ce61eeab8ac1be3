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
//     i, i+32, ...) closed by redux.sync argmin reductions on
//     order-preserving integer keys;
//   * the container pool is an ordered array (list semantics: append,
//     remove-with-shift) whose searches are lane-parallel and whose
//     order-sensitive float sums (CPython 3.12 Neumaier sum()) are replayed
//     serially through warp shuffles in list order;
//   * dynamic events (completions, keep-alive expiries) sit in a small slot
//     pool with a cached (time, seq) minimum; arrivals stream from the trace
//     (their seq is the trace index, engine.py:70-75) and the single monitor
//     tick is kept in registers.
//
// Every floating-point operation is written in the reference's operation
// order and the file is compiled with -fmad=false, so dispatch order,
// DispatchAudit rows and completion records are bit-identical to the
// reference (tests/test_gpu_parity.py checks them against oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "gfq_layout.h"

namespace gfq {

#define FULLMASK 0xffffffffu
typedef unsigned long long u64;

// ------------------------------------------------------------------------
// warp primitives

__device__ __forceinline__ u64 okey(double x) {  // order-preserving key
    u64 b = (u64)__double_as_longlong(x);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ u64 wmin64(u64 v) {
    unsigned hi = __reduce_min_sync(FULLMASK, (unsigned)(v >> 32));
    unsigned lo = __reduce_min_sync(FULLMASK, ((unsigned)(v >> 32) == hi) ? (unsigned)v : 0xffffffffu);
    return ((u64)hi << 32) | lo;
}
__device__ __forceinline__ double from_key(u64 k) {          // inverse of okey
    u64 b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}
// Store a warp-uniform value to shared memory: every lane has finished
// reading the old value before any lane writes (RMW-safe under independent
// thread scheduling), and the write is visible to all lanes afterwards.
template <class T>
__device__ __forceinline__ void ust(T& ref, T v) { __syncwarp(); ref = v; __syncwarp(); }

__device__ __forceinline__ unsigned wmin32(unsigned v) { return __reduce_min_sync(FULLMASK, v); }
__device__ __forceinline__ unsigned wor32(unsigned v) { return __reduce_or_sync(FULLMASK, v); }

// Python max(a, b) / min(a, b): the first argument wins ties.
__device__ __forceinline__ double pymax(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ double pymin(double a, double b) { return b < a ? b : a; }

// CPython 3.12 builtin sum() over floats (bltinmodule.c builtin_sum_impl):
// the first item is added to the int start 0, then Neumaier compensation,
// the compensation is added once at the end when nonzero and finite.
struct PySum { double f, c; int n; };
__device__ __forceinline__ void ps_init(PySum& s) { s.f = 0.0; s.c = 0.0; s.n = 0; }
__device__ __forceinline__ void ps_add(PySum& s, double x) {
    if (s.n++ == 0) { s.f = 0.0 + x; return; }
    double t = s.f + x;
    if (fabs(s.f) >= fabs(x)) s.c += (s.f - t) + x;
    else                      s.c += (x - t) + s.f;
    s.f = t;
}
__device__ __forceinline__ double ps_val(const PySum& s) {
    if (s.n == 0) return 0.0;
    if (s.c != 0.0 && isfinite(s.c)) return s.f + s.c;
    return s.f;
}

// pool entry meta: fn | thermal << 24 | evictable << 26 | swapping << 27
__device__ __forceinline__ int pm_fn(uint32_t m) { return (int)(m & 0xffffffu); }
__device__ __forceinline__ int pm_th(uint32_t m) { return (int)((m >> 24) & 3u); }
__device__ __forceinline__ bool pm_ev(uint32_t m) { return (m >> 26) & 1u; }
__device__ __forceinline__ bool pm_sw(uint32_t m) { return (m >> 27) & 1u; }
__device__ __forceinline__ uint32_t pm_make(int fn, int th, int ev) {
    return (uint32_t)fn | ((uint32_t)th << 24) | ((uint32_t)ev << 26);
}

struct Decision { int inv, fn, dev, st; bool ok; };

// ------------------------------------------------------------------------
// the per-warp simulation

struct WarpSim {
    const Params* P;
    const Layout* L;
    int lane;
    // smem slices
    double *vt, *lex, *tau, *iat, *larr;
    int *pt, *ph, *infl, *head, *done;
    uint8_t* fst;
    double* ev_t; uint32_t* ev_seq; uint32_t* ev_meta;
    int* dvi; double* dvd;
    double *smp_t, *smp_u;
    int* run_i; double* run_d;
    uint32_t* pool_m; double* pool_t;
    uint16_t* cnt;
    // inputs
    int sid;
    const gfq_sim* sim;
    const double* arr; const int* flw; const int* foff; const int* fpos;
    const double *warm, *cold, *mem, *share, *weight;
    const gfq_device_cfg* dc;
    const double* execs;
    int n, nf, ndev, policy;
    bool scripted, mqfq, fcfs;
    double T, alpha, dttl, period;
    int64_t roff, foffs;
    // uniform scalar state
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
    long long n_events, n_calls, n_disp, n_comp, n_util, n_backlog, n_evlog;
    PySum util_sum;

    // ---------------- accessors
    __device__ __forceinline__ int& DV(int d, int k) { return dvi[d * 8 + k]; }
    __device__ __forceinline__ double& UAVG(int d) { return dvd[d * 2]; }
    __device__ __forceinline__ uint16_t& GCNT(int d, int f) { return cnt[(d * 2) * L->F + f]; }
    __device__ __forceinline__ uint16_t& HCNT(int d, int f) { return cnt[(d * 2 + 1) * L->F + f]; }
    __device__ __forceinline__ uint32_t& PM(int d, int i) { return pool_m[d * L->P + i]; }
    __device__ __forceinline__ double& PT(int d, int i) { return pool_t[d * L->P + i]; }
    __device__ __forceinline__ int& RI(int d, int r, int k) { return run_i[(d * L->R + r) * 4 + k]; }
    __device__ __forceinline__ double& RD(int d, int r, int k) { return run_d[(d * L->R + r) * 2 + k]; }

    __device__ __forceinline__ void fail(int st) { if (!status) status = st; }

    // ---------------- flow helpers
    __device__ __forceinline__ int pending(int f) const { return pt[f] - ph[f]; }
    __device__ __forceinline__ double ttl(int f) const {     // FlowQueue.ttl, core.py:140-152
        if (alpha == 0.0) return 0.0;
        if (pt[f] >= 2) return alpha * iat[f];              // iat.count = arrivals - 1
        return dttl;
    }

    // ==================================================================
    // event pool (engine.py:83-87: heap of (time, seq, kind, payload))

    __device__ void push(double t, int kind, uint32_t payload) {
        if (t < now) { fail(GFQ_SIM_PAST_EVENT); return; }     // engine.py:84-85
        uint32_t s = seq++;
        if (kind == EV_TICK) { tick_on = true; tick_t = t; tick_seq = s; return; }
        if (nev >= L->E) { fail(GFQ_SIM_EVENT_OVERFLOW); return; }
        int slot = nev++;
        ev_t[slot] = t; ev_seq[slot] = s; ev_meta[slot] = ((uint32_t)kind << 30) | payload;
        if (pmin_ok && (pmin_slot < 0 || t < pmin_t || (t == pmin_t && s < pmin_seq))) {
            pmin_t = t; pmin_seq = s; pmin_slot = slot;
        }
        __syncwarp();
    }

    __device__ void pool_min() {                               // lane-parallel argmin
        u64 bt = ~0ull; uint32_t bs = 0xffffffffu; int bslot = -1;
        for (int i = lane; i < nev; i += 32) {
            u64 k = okey(ev_t[i]); uint32_t s = ev_seq[i];
            if (k < bt || (k == bt && s < bs)) { bt = k; bs = s; bslot = i; }
        }
        u64 m = wmin64(bt);
        uint32_t ms = wmin32(bt == m ? bs : 0xffffffffu);
        int src = __ffs(__ballot_sync(FULLMASK, bt == m && bs == ms && bslot >= 0)) - 1;
        pmin_ok = true;
        if (src < 0) { pmin_slot = -1; return; }
        pmin_slot = __shfl_sync(FULLMASK, bslot, src);
        pmin_t = ev_t[pmin_slot]; pmin_seq = ms;
    }

    __device__ void pool_remove(int slot) {
        int last = --nev;
        if (slot != last) { ev_t[slot] = ev_t[last]; ev_seq[slot] = ev_seq[last]; ev_meta[slot] = ev_meta[last]; }
        __syncwarp();
        pmin_ok = false;
    }

    // ==================================================================
    // device model (device.py)

    // container_state, device.py:104-112
    __device__ __forceinline__ int container_state(int d, int fn) {
        if (!dc[d].pool_enabled) return GFQ_COLD;
        if (GCNT(d, fn) > 0) return GFQ_GPU_WARM;
        if (HCNT(d, fn) > 0) return GFQ_HOST_WARM;
        return GFQ_COLD;
    }

    // _idle_entry, device.py:96-102: first entry (list order) with the max
    // last_used_s among (fn, thermal).  Returns -1 if none.
    __device__ int idle_entry(int d, int fn, int th) {
        int np = DV(d, DV_NP);
        u64 bk = ~0ull; int bi = 0x7fffffff;
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
    __device__ void pool_erase(int d, int i) {
        int np = DV(d, DV_NP);
        uint32_t m = PM(d, i);
        int fn = pm_fn(m), th = pm_th(m);
        __syncwarp();
        for (int base = i; base < np - 1; base += 32) {
            int j = base + lane;
            uint32_t mm = 0; double tt = 0.0;
            bool act = j < np - 1;
            if (act) { mm = PM(d, j + 1); tt = PT(d, j + 1); }
            __syncwarp();
            if (act) { PM(d, j) = mm; PT(d, j) = tt; }
            __syncwarp();
        }
        if (th == GFQ_GPU_WARM) ust(GCNT(d, fn), (uint16_t)(GCNT(d, fn) - 1));
        else ust(HCNT(d, fn), (uint16_t)(HCNT(d, fn) - 1));
        ust(DV(d, DV_NP), np - 1);
    }

    // resident_mb, device.py:114-117: sum(idle GPU_WARM mem) + sum(running mem)
    // in list order (two builtin Neumaier sums), replayed through shuffles.
    __device__ double resident_mb(int d) {
        int np = DV(d, DV_NP);
        PySum a; ps_init(a);
        for (int base = 0; base < np; base += 32) {
            int i = base + lane;
            double v = 0.0; bool g = false;
            if (i < np) { uint32_t m = PM(d, i); g = pm_th(m) == GFQ_GPU_WARM; if (g) v = mem[pm_fn(m)]; }
            unsigned gm = __ballot_sync(FULLMASK, g);
            while (gm) {
                int j = __ffs(gm) - 1; gm &= gm - 1;
                ps_add(a, __shfl_sync(FULLMASK, v, j));
            }
        }
        PySum b; ps_init(b);
        int nr = DV(d, DV_NRUN);
        for (int r = 0; r < nr; r++) ps_add(b, mem[RI(d, r, 1)]);
        return ps_val(a) + ps_val(b);
    }

    // admit_memory, device.py:147-179.  Victims are idle GPU_WARM entries in
    // a stable ascending last_used_s order; roll back if the deficit stays.
    __device__ bool admit_memory(int d, int fn) {
        if (GCNT(d, fn) > 0) return true;                 // idle GPU_WARM exists
        double needed = mem[fn];
        double free_mb = dc[d].mem_capacity_mb - resident_mb(d);
        if (free_mb >= needed) return true;
        int np = DV(d, DV_NP);
        int nsw = 0;
        while (free_mb < needed) {
            u64 bk = ~0ull; int bi = 0x7fffffff;
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
            free_mb += mem[pm_fn(m)];
            nsw++;
        }
        bool ok = free_mb >= needed;
        if (nsw) {
            // commit (thermal -> HOST_WARM) or roll back, one entry at a time so
            // the per-flow counts are updated without races
            for (int base = 0; base < np; base += 32) {
                int i = base + lane;
                bool s = i < np && pm_sw(PM(d, i));
                unsigned sm = __ballot_sync(FULLMASK, s);
                while (sm) {
                    int j = __ffs(sm) - 1; sm &= sm - 1;
                    int idx = base + j;
                    uint32_t m = PM(d, idx) & ~(1u << 27);
                    if (ok) {
                        int f = pm_fn(m);
                        ust(GCNT(d, f), (uint16_t)(GCNT(d, f) - 1));
                        ust(HCNT(d, f), (uint16_t)(HCNT(d, f) + 1));
                        m = (m & ~(3u << 24)) | ((uint32_t)GFQ_HOST_WARM << 24);
                    }
                    ust(PM(d, idx), m);
                }
            }
        }
        return ok;
    }

    // try_acquire_token, device.py:124-145 -> start state or -1
    __device__ int try_acquire_token(int d, int fn) {
        int out = DV(d, DV_OUT);
        if (out >= DV(d, DV_EFFD)) return -1;
        if (out >= 1 && UAVG(d) + 1.0 / (double)dc[d].d_max > dc[d].util_threshold) return -1;
        int st = container_state(d, fn);
        if (st != GFQ_GPU_WARM) {
            if (!admit_memory(d, fn)) return -1;
        }
        ust(DV(d, DV_OUT), out + 1);
        return st;
    }

    // DeviceSet.assign, device.py:320-341
    __device__ int assign(int fn, int& st) {
        if (ndev == 1) { st = try_acquire_token(0, fn); return st >= 0 ? 0 : -1; }
        int key[GFQ_MAX_DEVICES]; int order[GFQ_MAX_DEVICES];
#pragma unroll
        for (int i = 0; i < GFQ_MAX_DEVICES; i++) {
            if (i < ndev) {
                int cs = container_state(i, fn);   // pref 0/1/2 == GPU/HOST/COLD
                key[i] = (cs << 20) | (DV(i, DV_OUT) << 4) | i;
                order[i] = i;
            }
        }
        for (int i = 1; i < ndev; i++) {               // sorted(key=(pref, outstanding, index))
            int v = order[i]; int j = i - 1;
            while (j >= 0 && key[order[j]] > key[v]) { order[j + 1] = order[j]; j--; }
            order[j + 1] = v;
        }
        for (int k = 0; k < ndev; k++) {
            int r = try_acquire_token(order[k], fn);
            if (r >= 0) { st = r; return order[k]; }
        }
        return -1;
    }

    __device__ int max_effective_d() {                 // device.py:317-318
        if (scripted) return sim->scripted_d;
        int m = DV(0, DV_EFFD);
        for (int i = 1; i < ndev; i++) m = max(m, DV(i, DV_EFFD));
        return m;
    }

    // ScriptedDevices.assign (tests/oracles.py:25-32) or DeviceSet.assign
    __device__ int provider_assign(int fn, int& st) {
        if (scripted) {
            s_att += 1;
            if (sim->scripted_deny_every && s_att % sim->scripted_deny_every == 0) return -1;
            if (s_out >= sim->scripted_d) return -1;
            s_out += 1;
            st = GFQ_GPU_WARM;
            return 0;
        }
        return assign(fn, st);
    }

    // start_invocation, device.py:183-218 -> running entry
    __device__ void start_invocation(int d, int fn, int st, int inv, double& duration, double& pure) {
        double base; int claimed = -1;
        if (st == GFQ_GPU_WARM) {
            base = warm[fn];
            claimed = idle_entry(d, fn, GFQ_GPU_WARM);
        } else if (st == GFQ_HOST_WARM) {
            double transfer = pymax(0.0, mem[fn] / dc[d].pcie_mb_per_s - dc[d].prefetch_overlap_s);
            base = warm[fn] + transfer;
            claimed = idle_entry(d, fn, GFQ_HOST_WARM);
        } else {
            base = cold[fn];
        }
        if (claimed >= 0) pool_erase(d, claimed);
        int nr = DV(d, DV_NRUN);
        int concurrent = nr + 1;
        double factor = 1.0 + dc[d].interference_beta * (double)(concurrent - 1);
        duration = base * factor;
        pure = warm[fn] * factor;
        run_append(d, inv, fn, st, duration, pure);
    }

    __device__ void run_append(int d, int inv, int fn, int st, double duration, double pure) {
        int nr = DV(d, DV_NRUN);
        if (nr >= L->R) { fail(GFQ_SIM_POOL_OVERFLOW); return; }
        __syncwarp();
        RI(d, nr, 0) = inv; RI(d, nr, 1) = fn; RI(d, nr, 2) = st;
        RD(d, nr, 0) = duration; RD(d, nr, 1) = pure;
        DV(d, DV_NRUN) = nr + 1;
        __syncwarp();
    }

    // remove the running entry of `inv` (dict delete keeps insertion order)
    __device__ bool run_remove(int d, int inv, double& duration, double& pure, int& st) {
        int nr = DV(d, DV_NRUN);
        int ri = -1;
        for (int r = 0; r < nr; r++) if (RI(d, r, 0) == inv) { ri = r; break; }
        if (ri < 0) { fail(GFQ_SIM_BAD_CONFIG); return false; }   // RuntimeError
        st = RI(d, ri, 2); duration = RD(d, ri, 0); pure = RD(d, ri, 1);
        for (int r = ri; r < nr - 1; r++) {
            int a = RI(d, r + 1, 0), b = RI(d, r + 1, 1), c = RI(d, r + 1, 2);
            double x = RD(d, r + 1, 0), y = RD(d, r + 1, 1);
            __syncwarp();
            RI(d, r, 0) = a; RI(d, r, 1) = b; RI(d, r, 2) = c; RD(d, r, 0) = x; RD(d, r, 1) = y;
        }
        ust(DV(d, DV_NRUN), nr - 1);
        return true;
    }

    // _enforce_pool_cap, device.py:239-258: destroy min by
    // (not spare, not evictable, last_used_s), first in list order on ties
    __device__ void enforce_pool_cap(int d) {
        int cap = dc[d].pool_max_containers;
        for (;;) {
            int np = DV(d, DV_NP), nr = DV(d, DV_NRUN);
            if (!(np + nr > cap && np > 0)) break;
            unsigned bk01 = 0xffffffffu; u64 bk2 = ~0ull; int bi = 0x7fffffff;
            for (int i = lane; i < np; i += 32) {
                uint32_t m = PM(d, i); int f = pm_fn(m);
                bool running = false;
                for (int r = 0; r < nr; r++) running |= RI(d, r, 1) == f;
                bool spare = (int)GCNT(d, f) + (int)HCNT(d, f) > 1 && !running;
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

    // Device.complete, device.py:220-237 -> running entry fields
    __device__ bool device_complete(int d, int inv, int fn, double& duration, double& pure, int& st) {
        if (!run_remove(d, inv, duration, pure, st)) return false;
        ust(DV(d, DV_OUT), DV(d, DV_OUT) - 1);
        if (!dc[d].pool_enabled) return true;
        int np = DV(d, DV_NP);
        if (np >= L->P) { fail(GFQ_SIM_POOL_OVERFLOW); return false; }
        // the re-pooled entry is (fn, GPU_WARM, mem[fn], now, evictable=False)
        // whether or not a container was claimed at start (device.py:226-236)
        __syncwarp();
        PM(d, np) = pm_make(fn, GFQ_GPU_WARM, 0);
        PT(d, np) = now;
        DV(d, DV_NP) = np + 1;
        ust(GCNT(d, fn), (uint16_t)(GCNT(d, fn) + 1));
        enforce_pool_cap(d);
        return true;
    }

    // set_evictable over all entries of fn (mark/unmark_evictable, device.py:260-268)
    __device__ void set_evictable(int d, int fn, bool v) {
        int np = DV(d, DV_NP);
        for (int i = lane; i < np; i += 32) {
            uint32_t m = PM(d, i);
            if (pm_fn(m) == fn) PM(d, i) = v ? (m | (1u << 26)) : (m & ~(1u << 26));
        }
        __syncwarp();
    }

    // instantaneous_util, device.py:279-280
    __device__ double instantaneous_util(int d) {
        PySum a; ps_init(a);
        int nr = DV(d, DV_NRUN);
        for (int r = 0; r < nr; r++) ps_add(a, share[RI(d, r, 1)]);
        return pymin(1.0, ps_val(a));
    }

    // monitor_tick, device.py:282-297 -> (effective_d, inst util)
    __device__ int monitor_tick(int d, double& inst) {
        double util = instantaneous_util(d);
        inst = util;
        int S = L->S;
        int head = DV(d, DV_SHEAD), ns = DV(d, DV_SN);
        if (ns >= S) { fail(GFQ_SIM_SAMPLE_OVERFLOW); return DV(d, DV_EFFD); }
        int w = head + ns; if (w >= S) w -= S;
        smp_t[d * S + w] = now; smp_u[d * S + w] = util;
        ns++;
        double horizon = now - dc[d].util_window_s;
        while (ns > 0 && smp_t[d * S + head] <= horizon) { head++; if (head >= S) head = 0; ns--; }
        PySum a; ps_init(a);
        int j = head;
        for (int k = 0; k < ns; k++) { ps_add(a, smp_u[d * S + j]); j++; if (j >= S) j = 0; }
        double avg = ps_val(a) / (double)ns;
        int effd = DV(d, DV_EFFD);
        const gfq_device_cfg& c = dc[d];
        if (!c.dynamic_d) effd = c.d_max;
        else if (avg > c.util_threshold) effd = max(effd - 1, 1);
        else if (avg < c.util_threshold - 1.0 / (double)c.d_max) effd = min(effd + 1, c.d_max);
        __syncwarp();
        DV(d, DV_SHEAD) = head; DV(d, DV_SN) = ns; UAVG(d) = avg; DV(d, DV_EFFD) = effd;
        __syncwarp();
        return effd;
    }

    // ==================================================================
    // scheduler (mqfq.py) and baseline policies (policies.py)

    // recompute_global_vt, mqfq.py:114-127 (INACTIVE => not backlogged, so
    // the filter is just "backlogged")
    __device__ __forceinline__ u64 min_backlogged_vt() {
        u64 bk = ~0ull;
        for (int f = lane; f < nf; f += 32)
            if (pt[f] - done[f] > 0) { u64 k = okey(vt[f]); if (k < bk) bk = k; }
        return wmin64(bk);
    }

    __device__ void recompute_gvt() {
        u64 m = min_backlogged_vt();
        if (m != ~0ull) gvt = pymax(gvt, from_key(m));
    }

    // unstall, mqfq.py:129-139
    __device__ void unstall() {
        if (tot_infl > 0) return;
        u64 m = min_backlogged_vt();
        if (m == ~0ull) return;
        double mv = from_key(m);
        if (gvt < mv) gvt = mv;
    }

    // _update_state for an idle queue (mqfq.py:143-157); only the INACTIVE
    // bit is observable downstream
    __device__ __forceinline__ bool idle_update(int f, uint8_t& s) {
        bool inact = now - lex[f] >= ttl(f);
        bool newly = inact && !(s & FL_INACTIVE);
        s = inact ? (uint8_t)(s | FL_INACTIVE) : (uint8_t)(s & ~FL_INACTIVE);
        if (newly && !scripted) s |= FL_NEWLY;
        return newly;
    }

    __device__ void audit_dispatch(int inv, double vt_before, double g, int qlen, int infl_after) {
        long long k = n_disp++;
        if (P->outputs & GFQ_WANT_DISPATCH) {
            if (lane == 0) {
                int64_t o = roff + k;
                P->dsp_inv[o] = inv; P->dsp_vt[o] = vt_before; P->dsp_gvt[o] = g;
                P->dsp_qlen[o] = qlen; P->dsp_infl[o] = infl_after;
            }
        }
    }

    // pop the head of flow f (FlowQueue.pending.popleft)
    __device__ __forceinline__ int pop_head(int f) {
        int inv = head[f];
        int k = ph[f] + 1;
        int nxt = k < pt[f] ? fpos[foff[f] + k] : -1;
        __syncwarp();
        ph[f] = k;
        head[f] = nxt;
        __syncwarp();
        return inv;
    }

    // MqfqScheduler.dispatch, mqfq.py:190-239
    __device__ Decision mqfq_dispatch() {
        Decision dd; dd.ok = false;
        recompute_gvt();
        // refresh_states (name order) fused with the candidate filter and the
        // two stable sorts: head = lexicographic min of
        // (in_flight if D != 1, -len(pending), name)
        bool use_inf = max_effective_d() != 1;
        u64 bk = ~0ull;
        bool newly = false;
        for (int f = lane; f < nf; f += 32) {
            uint8_t s = fst[f];
            if (!(s & FL_CREATED)) continue;
            int pend = pending(f), inf = infl[f];
            if (pend == 0 && inf == 0) {
                uint8_t s0 = s;
                newly |= idle_update(f, s);
                if (s != s0) fst[f] = s;
            } else if (pend > 0 && vt[f] - gvt <= T) {
                u64 k = ((u64)(use_inf ? (unsigned)inf : 0u) << 48) |
                        ((u64)(0xffffffffu - (unsigned)pend) << 16) | (u64)f;
                if (k < bk) bk = k;
            }
        }
        __syncwarp();
        if (wor32(newly)) any_newly = true;
        u64 m = wmin64(bk);
        if (m == ~0ull) return dd;
        int h = (int)(m & 0xffffu);
        int st = 0;
        int dev = provider_assign(h, st);
        if (dev < 0) return dd;
        double vt_before = vt[h];
        int inv = pop_head(h);
        double nvt = vt_before + tau[h] / weight[h];
        int ninf = infl[h] + 1;
        __syncwarp();
        vt[h] = nvt; infl[h] = ninf; lex[h] = now;
        __syncwarp();
        audit_dispatch(inv, vt_before, gvt, pending(h) + 1, ninf);
        recompute_gvt();
        dd.inv = inv; dd.fn = h; dd.dev = dev; dd.st = st; dd.ok = true;
        return dd;
    }

    // FcfsPolicy.dispatch, policies.py:129-139 (one global FIFO = trace order)
    __device__ Decision fcfs_dispatch() {
        Decision dd; dd.ok = false;
        if (fcfs_head == cursor) return dd;
        int inv = fcfs_head;
        int fn = flw[inv];
        int st = 0;
        int dev = provider_assign(fn, st);
        if (dev < 0) return dd;
        fcfs_head++;
        fcfs_infl++;
        audit_dispatch(inv, 0.0, 0.0, (cursor - fcfs_head) + 1, fcfs_infl);
        dd.inv = inv; dd.fn = fn; dd.dev = dev; dd.st = st; dd.ok = true;
        return dd;
    }

    // BatchPolicy._oldest_nonempty, policies.py:197-208: key (arrival_s, uid)
    // == smallest trace position among the queue heads
    __device__ int batch_oldest() {
        unsigned bk = 0xffffffffu;
        for (int f = lane; f < nf; f += 32)
            if (pending(f) > 0) bk = min(bk, (unsigned)head[f]);
        unsigned m = wmin32(bk);
        return m == 0xffffffffu ? -1 : flw[m];
    }

    // BatchPolicy.dispatch, policies.py:175-195
    __device__ Decision batch_dispatch() {
        Decision dd; dd.ok = false;
        int dr = draining;
        if (dr >= 0 && (pending(dr) > 0 || infl[dr] > 0)) {
            if (pending(dr) == 0) return dd;            // hold for late arrivals
        } else {
            dr = batch_oldest();
            if (dr < 0) return dd;
        }
        int st = 0;
        int dev = provider_assign(dr, st);
        if (dev < 0) return dd;
        draining = dr;
        int inv = pop_head(dr);
        int ninf = infl[dr] + 1;
        __syncwarp();
        infl[dr] = ninf;
        __syncwarp();
        audit_dispatch(inv, 0.0, 0.0, pending(dr) + 1, ninf);
        dd.inv = inv; dd.fn = dr; dd.dev = dev; dd.st = st; dd.ok = true;
        return dd;
    }

    // SjfPolicy.dispatch, policies.py:245-262: min tau.mean, name order on ties
    __device__ Decision sjf_dispatch() {
        Decision dd; dd.ok = false;
        u64 bk = ~0ull; int bf = 0x7fffffff;
        for (int f = lane; f < nf; f += 32) {
            if (pending(f) > 0) { u64 k = okey(tau[f]); if (k < bk) { bk = k; bf = f; } }
        }
        u64 m = wmin64(bk);
        if (m == ~0ull) return dd;
        int sh = (int)wmin32(bk == m ? (unsigned)bf : 0x7fffffffu);
        int st = 0;
        int dev = provider_assign(sh, st);
        if (dev < 0) return dd;
        int inv = pop_head(sh);
        int ninf = infl[sh] + 1;
        __syncwarp();
        infl[sh] = ninf;
        __syncwarp();
        audit_dispatch(inv, 0.0, 0.0, pending(sh) + 1, ninf);
        dd.inv = inv; dd.fn = sh; dd.dev = dev; dd.st = st; dd.ok = true;
        return dd;
    }

    __device__ Decision policy_dispatch() {
        n_calls++;
        Decision d;
        if (mqfq) d = mqfq_dispatch();
        else if (policy == GFQ_POLICY_BATCH) d = batch_dispatch();
        else if (policy == GFQ_POLICY_SJF) d = sjf_dispatch();
        else d = fcfs_dispatch();
        if (d.ok) { tot_pend--; tot_infl++; }
        return d;
    }

    // on_arrival of every policy (mqfq.py:186-188 + core.py:120-138;
    // policies.py:126-127,172-173,242-243)
    __device__ void policy_on_arrival(int inv, int fn) {
        uint8_t s = fst[fn];
        int p0 = pt[fn], h0 = ph[fn];
        double v = vt[fn], le = lex[fn], im = iat[fn];
        int hd = head[fn];
        if (!(s & FL_CREATED)) {                          // queue_for, mqfq.py:94-99
            s = FL_CREATED | FL_INACTIVE;
            v = 0.0;
            le = mqfq ? now : 0.0;
        }
        tot_pend++;
        if (!fcfs) {
            if (mqfq && (s & FL_INACTIVE)) {              // reactivation clamp, core.py:128-130
                v = pymax(v, gvt);
                s &= (uint8_t)~FL_INACTIVE;
            }
            if (p0 == h0) hd = inv;                       // pending.append
            if (mqfq && p0 >= 1) {                        // iat.record(now - last_arrival)
                double x = now - larr[fn];
                im = im + (x - im) / (double)p0;
            }
        }
        __syncwarp();
        fst[fn] = s; pt[fn] = p0 + 1;                     // pt also drives the engine backlog count
        vt[fn] = v; lex[fn] = le; iat[fn] = im; head[fn] = hd;
        if (mqfq) larr[fn] = now;
        __syncwarp();
    }

    // on_completion of every policy (mqfq.py:241-247; policies.py:141-142,210-213,264-267)
    __device__ void policy_on_completion(int fn, double exec_s) {
        tot_infl--;
        int dn = done[fn] + 1;
        if (fcfs) { fcfs_infl -= 1; ust(done[fn], dn); return; }
        int inf = infl[fn] - 1;
        double tm = tau[fn];
        tm = tm + (exec_s - tm) / (double)dn;            // tau.count == completions
        __syncwarp();
        done[fn] = dn; infl[fn] = inf; tau[fn] = tm;
        if (mqfq) lex[fn] = now;
        __syncwarp();
    }

    // ==================================================================
    // engine (engine.py)

    __device__ void backlog_audit(int fn, bool on) {
        long long k = n_backlog++;
        if ((P->outputs & GFQ_WANT_AUDIT) && lane == 0) {
            if (k < P->audit_backlog_cap) {
                int64_t o = (int64_t)sid * P->audit_backlog_cap + k;
                P->backlog_time[o] = now; P->backlog_meta[o] = (fn << 1) | (on ? 1 : 0);
            }
        }
    }

    // _swap_out_inactive, engine.py:199-203 (+ Device.swap_out / mark_evictable)
    __device__ void swap_out_inactive() {
        if (!any_newly) return;
        any_newly = false;
        for (int d = 0; d < ndev; d++) {
            int np = DV(d, DV_NP);
            for (int i = lane; i < np; i += 32) {
                uint32_t m = PM(d, i);
                if (fst[pm_fn(m)] & FL_NEWLY) {
                    m |= (1u << 26);                                    // evictable
                    if (pm_th(m) == GFQ_GPU_WARM) m = (m & ~(3u << 24)) | ((uint32_t)GFQ_HOST_WARM << 24);
                    PM(d, i) = m;
                }
            }
        }
        __syncwarp();
        for (int f = lane; f < nf; f += 32) {
            uint8_t s = fst[f];
            if (s & FL_NEWLY) {
                for (int d = 0; d < ndev; d++) { HCNT(d, f) += GCNT(d, f); GCNT(d, f) = 0; }
                fst[f] = (uint8_t)((s & ~FL_NEWLY) | FL_MARKED);
            }
        }
        __syncwarp();
    }

    // _start, engine.py:187-197
    __device__ void start(const Decision& dd) {
        double duration, pure;
        if (scripted) {
            // drive(): completion at now + next(exec_iter) (oracles.py:235-236)
            duration = execs[sim->exec_off + (s_exec % sim->exec_len)];
            s_exec++;
            pure = duration;
            run_append(0, dd.inv, dd.fn, dd.st, duration, pure);
            if (status) return;
        } else {
            start_invocation(dd.dev, dd.fn, dd.st, dd.inv, duration, pure);
            if (status) return;
        }
        if ((P->outputs & GFQ_WANT_RECORDS) && lane == 0) {
            int64_t o = roff + dd.inv;
            P->rec_dispatch[o] = now; P->rec_state[o] = (int8_t)dd.st; P->rec_device[o] = (int8_t)dd.dev;
            P->rec_pure[o] = pure;
        }
        push(now + duration, EV_COMPLETION, (uint32_t)dd.inv | ((uint32_t)dd.dev << 27));
    }

    // _drain, engine.py:173-185
    __device__ void drain() {
        for (;;) {
            Decision d = policy_dispatch();
            if (!d.ok && tot_infl == 0 && tot_pend > 0) {
                if (mqfq) unstall();
                d = policy_dispatch();
            }
            if (!d.ok || status) break;
            start(d);
            if (status) return;
        }
        if (!scripted) swap_out_inactive();
    }

    __device__ void on_arrival(int inv) {                  // engine.py:121-129
        int fn = flw[inv];
        if (scripted) { policy_on_arrival(inv, fn); drain(); return; }
        if (pt[fn] - done[fn] == 0) backlog_audit(fn, true);   // _backlog_change(+1)
        if (fst[fn] & FL_MARKED) {                          // unmark_evictable on every device
            for (int d = 0; d < ndev; d++) set_evictable(d, fn, false);
            ust(fst[fn], (uint8_t)(fst[fn] & ~FL_MARKED));
        }
        policy_on_arrival(inv, fn);
        if (!tick_on) push(now + period, EV_TICK, 0);
        drain();
    }

    __device__ void on_completion(int inv, int dev) {     // engine.py:131-153
        int fn = flw[inv];
        double duration = 0.0, pure = 0.0; int st = 0;
        if (scripted) {
            s_out -= 1;
            if (!run_remove(0, inv, duration, pure, st)) return;
            policy_on_completion(fn, duration);
        } else {
            if (!device_complete(dev, inv, fn, duration, pure, st)) return;
            policy_on_completion(fn, sim->tau_includes_overheads ? duration : pure);
        }
        long long k = n_comp++;
        if (lane == 0) {
            int64_t o = roff + k;
            P->comp_lat[o] = now - arr[inv];
            P->comp_meta[o] = fn | ((st == GFQ_COLD) ? (int)0x80000000 : 0);
            if (P->outputs & GFQ_WANT_RECORDS) {
                P->rec_complete[roff + inv] = now;
                P->rec_order[roff + inv] = (int32_t)k;
            }
        }
        if (!scripted) {
            if (pt[fn] - done[fn] == 0) {                   // _backlog_change(-1)
                backlog_audit(fn, false);
                if (mqfq) push(now + ttl(fn), EV_EXPIRY, (uint32_t)fn);
            }
        }
        drain();
    }

    __device__ void on_monitor() {                         // engine.py:155-165
        for (int d = 0; d < ndev; d++) {
            double inst;
            int eff = monitor_tick(d, inst);
            long long k = n_util++;
            if ((P->outputs & GFQ_WANT_AUDIT) && lane == 0 && k < P->audit_util_cap) {
                int64_t o = (int64_t)sid * P->audit_util_cap + k;
                P->util_rows[o * 3 + 0] = now; P->util_rows[o * 3 + 1] = inst;
                P->util_rows[o * 3 + 2] = UAVG(d);
                P->util_meta[o * 2 + 0] = d; P->util_meta[o * 2 + 1] = eff;
            }
            ps_add(util_sum, inst);
        }
        if (cursor < n || tot_pend > 0 || tot_infl > 0) push(now + period, EV_TICK, 0);
        else tick_on = false;
        drain();
    }

    __device__ void on_expiry(int fn) {                    // engine.py:167-171
        // expiry_check, mqfq.py:163-176
        bool has = false; double due = 0.0;
        uint8_t s = fst[fn];
        if ((s & FL_CREATED) && pending(fn) == 0 && infl[fn] == 0) {
            uint8_t s0 = s;
            if (idle_update(fn, s)) any_newly = true;
            __syncwarp();
            if (s != s0) fst[fn] = s;
            __syncwarp();
            if (!(s & FL_INACTIVE)) {
                due = lex[fn] + ttl(fn);
                if (due > now) has = true;
            }
        }
        swap_out_inactive();
        if (has) push(due, EV_EXPIRY, (uint32_t)fn);
    }

    // ==================================================================

    __device__ void log_event(double t, int kind, long long payload) {
        long long k = n_evlog++;
        if ((P->outputs & GFQ_WANT_EVENTS) && lane == 0 && k < P->event_log_cap) {
            int64_t o = (int64_t)sid * P->event_log_cap + k;
            P->event_time[o] = t;
            P->event_meta[o] = (int64_t)((payload << 2) | kind);
        }
    }

    __device__ void run() {
        long long max_events = sim->max_events > 0 ? sim->max_events : 64ll * ((long long)n + 1024);
        double t_arr = n > 0 ? arr[0] : 0.0;
        for (;;) {
            if (status) break;
            // candidates: next arrival (seq = trace index), the tick, the pool min
            bool has_arr = cursor < n;
            if (!pmin_ok) pool_min();
            bool has_pool = pmin_slot >= 0 && nev > 0;
            if (!has_arr && !tick_on && !has_pool) break;
            if (P->early_exit && !has_arr && !tick_on && tot_pend == 0 && tot_infl == 0 &&
                !(P->outputs & GFQ_WANT_EVENTS))
                break;                                      // only expiry rechecks remain
            int kind; double t; uint32_t sq;
            if (has_arr) { kind = EV_ARRIVAL; t = t_arr; sq = (uint32_t)cursor; }
            else { kind = -1; t = 0.0; sq = 0xffffffffu; }
            if (tick_on && (kind < 0 || tick_t < t || (tick_t == t && tick_seq < sq))) {
                kind = EV_TICK; t = tick_t; sq = tick_seq;
            }
            if (has_pool && (kind < 0 || pmin_t < t || (pmin_t == t && pmin_seq < sq))) {
                kind = 4; t = pmin_t; sq = pmin_seq;
            }
            if (n_events >= max_events) { fail(GFQ_SIM_WATCHDOG); break; }
            now = t;
            n_events++;
            if (kind == EV_ARRIVAL) {
                int inv = cursor++;
                if (cursor < n) t_arr = arr[cursor];
                log_event(t, EV_ARRIVAL, inv);
                on_arrival(inv);
            } else if (kind == EV_TICK) {
                tick_on = false;
                log_event(t, EV_TICK, -1);
                on_monitor();
            } else {
                int slot = pmin_slot;
                uint32_t meta = ev_meta[slot];
                pool_remove(slot);
                int k = (int)(meta >> 30);
                uint32_t pay = meta & 0x3fffffffu;
                if (k == EV_COMPLETION) {
                    int inv = (int)(pay & 0x7ffffffu);
                    log_event(t, EV_COMPLETION, inv);
                    on_completion(inv, (int)(pay >> 27));
                } else {
                    log_event(t, EV_EXPIRY, (long long)pay);
                    on_expiry((int)pay);
                }
            }
        }
    }
};

}  // namespace gfq
