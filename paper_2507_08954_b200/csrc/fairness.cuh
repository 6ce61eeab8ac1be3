// fairness.cuh — the fairness-audit reducer: metrics.service_gap_report
// (gpufairq metrics.py:106-187) over a finished parity-mode batch, one warp
// per simulation.
//
// Per window [w0, w0 + window_s) (w0 accumulated from 0 while w0 < the last
// completion time):
//   * qualified = functions backlogged for the whole window: an on-transition
//     at or before w0 and no off-transition before w1 (_backlog_intervals +
//     `s <= w0 and e >= w1`), swept over the AuditLog.backlog rows in order;
//   * service[f] = sum over exec rows (completion order) overlapping the
//     window of pure * overlap / (complete - dispatch), qualified f only, with
//     the window's (count, naive sum) of pure per function;
//   * normalised = service / cfg.weights.get(f, 1.0); hi / lo = max / min of
//     (normalised, name); d_eff = max effective D of the util rows with
//     w0 <= t < w1 (else cfg.d_max); tau = window mean else run mean else 0;
//   * bound = (d_eff - 1) * (2T + tau_hi/w_hi - tau_lo/w_lo) (fairness_bound,
//     mqfq.py:56-69), bound_conservative with the pair's times added,
//     violated = max_gap > bound.
// Lane (f mod 32) owns function f; every row stream is read 32 rows at a time
// and replayed in order through shuffles, so per-function float sums keep the
// reference's order.
#pragma once
#include "sim_warp.cuh"

namespace gfq {

struct FairParams {
    double window_s;
    const int32_t* d_max;          // [sims] SchedulerConfig.d_max (fallback D)
    const double* rweight;         // [flow-table rows] cfg.weights.get(f, 1.0)
    const int64_t* woff;           // [sims + 1] window-row offsets (capacity)
    double* rows;                  // [windows][5]: w0, service_sum, max_gap, bound, bound_cons
    int64_t* meta;                 // [windows][6]: comparable, n_qual, qual_hash, hi, lo, violated
    int64_t* count;                // [sims][3]: windows, comparable, violated
    unsigned char* scratch;        // per-warp F * 48 B
};

template <class T>
FI T shfl(T v, int j) { return __shfl_sync(FULLMASK, v, j); }

__device__ void fair_one(const Params& p, const FairParams& fp, unsigned char* scr, int lane,
                         int sid) {
    const gfq_sim* sim = p.sims + sid;
    const int nf = p.trace_nf[sim->trace];
    const int F = p.L.F;
    const int nrec = (int)p.counters[(int64_t)sid * GFQ_NCOUNTERS + C_DISP];
    const int64_t roff = p.sim_roff[sid];
    const int64_t tb = p.tab_off[sim->flowtab];
    const double T = sim->t_overrun;
    int64_t* cnt = fp.count + (int64_t)sid * 3;
    const int64_t wbase = fp.woff[sid], wcap = fp.woff[sid + 1] - wbase;
    // scratch: on, rn, wn, q (i32[F]); on_since, rs, svc, ws (f64[F])
    int* on = (int*)scr; int* rn = on + F; int* wn = on + 2 * F; int* q = on + 3 * F;
    double* on_since = (double*)(scr + 16 * (size_t)F);
    double* rs = on_since + F; double* svc = on_since + 2 * F; double* ws = on_since + 3 * F;
    for (int f = lane; f < nf; f += 32) { on[f] = 0; rn[f] = 0; rs[f] = 0.0; on_since[f] = 0.0; }
    __syncwarp();
    if (p.status[sid] != GFQ_SIM_OK || nrec == 0) {
        if (lane == 0) { cnt[0] = 0; cnt[1] = 0; cnt[2] = 0; }
        return;
    }
    const double* rc = p.rec_complete + roff;
    const double* rd = p.rec_dispatch + roff;
    const double* rp = p.rec_pure + roff;
    const int32_t* cpos = p.comp_pos + roff;        // completion rank -> trace position
    const int32_t* cmeta = p.comp_meta + roff;
    // end = max complete; maxdur = max (complete - dispatch)
    double end = 0.0, maxdur = 0.0;
    for (int k = lane; k < nrec; k += 32) {
        int i = cpos[k];
        end = fmax(end, rc[i]);
        maxdur = fmax(maxdur, rc[i] - rd[i]);
    }
    for (int o = 16; o; o >>= 1) {
        end = fmax(end, shfl(end, lane ^ o));
        maxdur = fmax(maxdur, shfl(maxdur, lane ^ o));
    }
    // run_mean_exec: per function (count, naive sum of pure) in exec-row order
    for (int base = 0; base < nrec; base += 32) {
        int k = base + lane;
        int fn = 0; double pu = 0.0;
        if (k < nrec) { fn = cmeta[k] & 0x7fffffff; pu = rp[cpos[k]]; }
        int nb = min(32, nrec - base);
        for (int j = 0; j < nb; j++) {
            int fj = shfl(fn, j); double pj = shfl(pu, j);
            if ((fj & 31) == lane) { rn[fj] += 1; rs[fj] = rs[fj] + pj; }
        }
    }
    __syncwarp();
    const int64_t bcap = p.audit_backlog_cap, ucap = p.audit_util_cap;
    const int nb_rows = (int)min((int64_t)p.backlog_count[sid], bcap);
    const double* bt = p.backlog_time + (int64_t)sid * bcap;
    const int32_t* bm = p.backlog_meta + (int64_t)sid * bcap;
    const int nu_rows = (int)min((int64_t)p.counters[(int64_t)sid * GFQ_NCOUNTERS + C_UTIL], ucap);
    const double* ur = p.util_rows + (int64_t)sid * ucap * 3;
    const int32_t* um = p.util_meta + (int64_t)sid * ucap * 2;
    const double* rw = fp.rweight + tb;
    int bptr = 0, uptr = 0, eptr = 0;
    int64_t nw = 0, ncomp = 0, nviol = 0;
    double w0 = 0.0;
    while (w0 < end) {
        const double w1 = w0 + fp.window_s;
        // backlog transitions at or before w0 update the per-function state
        while (bptr < nb_rows && bt[bptr] <= w0) {
            int m = bm[bptr]; int f = m >> 1;
            if ((f & 31) == lane) { if (m & 1) { on[f] = 1; on_since[f] = bt[bptr]; } else on[f] = 0; }
            bptr++;
        }
        __syncwarp();
        for (int f = lane; f < nf; f += 32) {
            q[f] = on[f] && on_since[f] <= w0;
            svc[f] = 0.0; wn[f] = 0; ws[f] = 0.0;
        }
        __syncwarp();
        // ... and an off-transition before w1 breaks the interval
        for (int b = bptr; b < nb_rows && bt[b] < w1; b++) {
            int m = bm[b]; int f = m >> 1;
            if (!(m & 1) && (f & 31) == lane) q[f] = 0;
        }
        __syncwarp();
        // exec rows overlapping the window, in completion order
        while (eptr < nrec && rc[cpos[eptr]] <= w0) eptr++;
        for (int base = eptr; base < nrec; base += 32) {
            int k = base + lane;
            double c = 0.0, d = 0.0, pu = 0.0; int fn = 0;
            if (k < nrec) { int i = cpos[k]; c = rc[i]; d = rd[i]; pu = rp[i]; fn = cmeta[k] & 0x7fffffff; }
            int nbk = min(32, nrec - base);
            bool stop = false;
            for (int j = 0; j < nbk; j++) {
                double cj = shfl(c, j), dj = shfl(d, j), pj = shfl(pu, j); int fj = shfl(fn, j);
                if (cj - maxdur >= w1) { stop = true; break; }     // no later row can overlap
                double got = pymax(0.0, pymin(cj, w1) - pymax(dj, w0));   // _overlap
                if (got > 0.0 && (fj & 31) == lane && q[fj]) {
                    svc[fj] += pj * got / (cj - dj);
                    wn[fj] += 1; ws[fj] = ws[fj] + pj;
                }
            }
            if (stop) break;
        }
        __syncwarp();
        // d_eff: max effective D of the util rows in [w0, w1)
        while (uptr < nu_rows && ur[uptr * 3] < w0) uptr++;
        int deff = -1;
        while (uptr < nu_rows && ur[uptr * 3] < w1) { deff = max(deff, um[uptr * 2 + 1]); uptr++; }
        if (deff < 0) deff = fp.d_max[sid];
        // per-window reductions over the qualified functions
        u64 hk = 0ull, lk = ~0ull; int hf = -1, lf = 0x7fffffff;
        unsigned nq = 0, qh = 0;
        for (int f = lane; f < nf; f += 32) {
            if (!q[f]) continue;
            nq++;
            qh += (unsigned)f * 2654435761u + 1u;
            u64 k = okey(svc[f] / rw[f]);
            if (k > hk || (k == hk && f > hf)) { hk = k; hf = f; }
            if (k < lk || (k == lk && f < lf)) { lk = k; lf = f; }
        }
        nq = __reduce_add_sync(FULLMASK, nq);
        qh = __reduce_add_sync(FULLMASK, qh);
        double ssum = 0.0;                                     // naive, in name order
        for (int base = 0; base < nf; base += 32) {
            int f = base + lane;
            double v = (f < nf && q[f]) ? svc[f] : 0.0;
            unsigned qm = __ballot_sync(FULLMASK, f < nf && q[f]);
            while (qm) { int j = __ffs(qm) - 1; qm &= qm - 1; ssum = ssum + shfl(v, j); }
        }
        double max_gap = 0.0, bound = 0.0, bcons = 0.0; int comparable = nq > 0, viol = 0;
        int hi = -1, lo = -1;
        if (comparable) {
            // hi = max (key, f): top 32 bits, then low 32, then f
            unsigned h1 = __reduce_max_sync(FULLMASK, (unsigned)(hk >> 32));
            unsigned h2 = __reduce_max_sync(FULLMASK, (unsigned)(hk >> 32) == h1 ? (unsigned)hk : 0u);
            u64 hmax = ((u64)h1 << 32) | h2;
            hi = (int)__reduce_max_sync(FULLMASK, hk == hmax ? (unsigned)hf : 0u);
            u64 lmin = wmin64(lk);
            lo = (int)wmin32(lk == lmin ? (unsigned)lf : 0xffffffffu);
            const double whi = rw[hi], wlo = rw[lo];
            const double nhi = svc[hi] / whi, nlo = svc[lo] / wlo;
            const double thi = wn[hi] > 0 ? ws[hi] / (double)wn[hi] : (rn[hi] > 0 ? rs[hi] / (double)rn[hi] : 0.0);
            const double tlo = wn[lo] > 0 ? ws[lo] / (double)wn[lo] : (rn[lo] > 0 ? rs[lo] / (double)rn[lo] : 0.0);
            max_gap = nhi - nlo;
            bound = (double)(deff - 1) * (2.0 * T + thi / whi - tlo / wlo);
            bcons = (double)(deff - 1) * (2.0 * T + thi / whi + tlo / wlo);
            viol = max_gap > bound;
        }
        if (lane == 0 && nw < wcap) {
            int64_t o = wbase + nw;
            double* r = fp.rows + o * 5;
            r[0] = w0; r[1] = ssum; r[2] = max_gap; r[3] = bound; r[4] = bcons;
            int64_t* m = fp.meta + o * 6;
            m[0] = comparable; m[1] = nq; m[2] = qh; m[3] = hi; m[4] = lo; m[5] = viol;
        }
        nw++; ncomp += comparable; nviol += viol;
        __syncwarp();
        w0 = w1;
    }
    if (lane == 0) { cnt[0] = nw; cnt[1] = ncomp; cnt[2] = nviol; }
}

__global__ void __launch_bounds__(128) k_fairness(const __grid_constant__ Params p,
                                                  const __grid_constant__ FairParams fp) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    unsigned char* scr = fp.scratch + (size_t)(blockIdx.x * wpb + warp) * 48 * p.L.F;
    for (int sid = blockIdx.x * wpb + warp; sid < p.n_sims; sid += gridDim.x * wpb)
        fair_one(p, fp, scr, lane, sid);
}

}  // namespace gfq
