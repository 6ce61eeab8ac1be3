// tracegen.cuh — GPU trace generator: the reference's gen_zipf
// (gpufairq/workload.py:82-111) for thousands of traces at once, written
// straight into the engine's trace buffers (no host round trip).
//
// Per trace: function k (original order) gets rate r_k (host-computed,
// zipf_rates, workload.py:73-79) and its own numpy substream
// SeedSequence(seed).spawn(n)[k] -> PCG64; t += (1/r_k) * Exp(1) until
// t >= duration, each arrival rounded to 6 decimals (Python round(t, 6));
// then the whole trace sorted by (t, name).
//
//   k_gen_streams  one thread per (trace, function) stream, two passes
//                  (count, then write): numpy's SeedSequence pool hashing
//                  and generate_state (bit_generator.pyx), PCG64 XSL-RR 128/64
//                  (pcg64.h), the exponential ziggurat with numpy's own tables
//                  (distributions.c standard_exponential_zig), and round(t, 6)
//                  by exact 128-bit integer arithmetic.  Streams of a trace are
//                  laid out in name order, so a stable sort by time gives the
//                  reference's (t, name) order.
//   (CUB segmented radix sort, stable, keyed by the fp64 bit pattern of t)
//   k_gen_flows    per trace: which functions arrived, and each arrival's flow
//                  id = rank of its name among those (pack_trace's encoding).
#pragma once
#include <stdint.h>
#include "zig_exp_tables.h"

namespace gfq {

struct GenParams {
    int32_t n_streams;
    const int32_t* stream_trace;    // [streams] trace of the stream
    const int32_t* stream_fn;       // [streams] function index k (spawn key, rate)
    const int32_t* stream_rank;     // [streams] name rank of that function
    const int64_t* fn_off;          // [traces + 1] offsets into rates
    const double* rates;            // [functions] per trace, original order
    const double* duration;         // [traces]
    const unsigned long long* seed; // [traces]
    int64_t* count;                 // [streams] arrivals (pass 1)
    const int64_t* out_off;         // [streams] first output slot (pass 2)
    unsigned long long* key;        // [arrivals] fp64 bits of round(t, 6)
    int32_t* val;                   // [arrivals] name rank
};

namespace tg {

typedef unsigned __int128 u128;
__device__ __forceinline__ uint32_t hashmix(uint32_t v, uint32_t& hc) {
    v ^= hc;
    hc *= 0x931E8875u;
    v *= hc;
    return v ^ (v >> 16);
}
__device__ __forceinline__ uint32_t mixw(uint32_t x, uint32_t y) {
    uint32_t r = 0xCA01F9DDu * x - 0x4973F715u * y;
    return r ^ (r >> 16);
}

// SeedSequence(seed).spawn(n)[k].pool: entropy = seed words (little-endian
// 32-bit, zero-padded to the pool size because a spawn key follows) + [k]
__device__ void seed_pool(unsigned long long seed, uint32_t k, uint32_t pool[4]) {
    uint32_t ent[7];
    int ne = 0;
    if (seed == 0) ent[ne++] = 0;
    for (unsigned long long s = seed; s; s >>= 32) ent[ne++] = (uint32_t)s;
    while (ne < 4) ent[ne++] = 0;
    ent[ne++] = k;
    uint32_t hc = 0x43B0D7E5u;
    for (int i = 0; i < 4; i++) pool[i] = hashmix(ent[i], hc);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = mixw(pool[d], hashmix(pool[s], hc));
    for (int s = 4; s < ne; s++)
        for (int d = 0; d < 4; d++) pool[d] = mixw(pool[d], hashmix(ent[s], hc));
}

struct Pcg64 {
    u128 state, inc;
    __device__ void step() {
        const u128 mult = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
        state = state * mult + inc;
    }
    __device__ unsigned long long next64() {          // step, then XSL-RR output
        step();
        const unsigned long long hi = (unsigned long long)(state >> 64), lo = (unsigned long long)state;
        const unsigned rot = (unsigned)(hi >> 58);
        const unsigned long long x = hi ^ lo;
        return (x >> rot) | (x << ((64u - rot) & 63u));
    }
    __device__ double next_double() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
    // PCG64(seed_seq): generate_state(4, uint64) -> initstate, initseq (pcg64_set_seed)
    __device__ void seed_from(const uint32_t pool[4]) {
        uint32_t hc = 0x8B51F9DDu, w[8];
        for (int i = 0; i < 8; i++) {
            uint32_t v = pool[i & 3] ^ hc;
            hc *= 0x58F38DEDu;
            v *= hc;
            w[i] = v ^ (v >> 16);
        }
        unsigned long long v64[4];
        for (int i = 0; i < 4; i++) v64[i] = (unsigned long long)w[2 * i] | ((unsigned long long)w[2 * i + 1] << 32);
        const u128 initstate = ((u128)v64[0] << 64) | v64[1];
        const u128 initseq = ((u128)v64[2] << 64) | v64[3];
        inc = (initseq << 1) | 1;
        state = 0;
        step();
        state += initstate;
        step();
    }
};

// standard_exponential_zig (numpy distributions.c)
__device__ double std_exponential(Pcg64& g) {
    for (;;) {
        unsigned long long ri = g.next64() >> 3;
        const int idx = (int)(ri & 0xFF);
        ri >>= 8;
        const double x = (double)ri * __longlong_as_double((long long)__ldg(zig_we_bits + idx));
        if (ri < __ldg(zig_ke + idx)) return x;
        if (idx == 0) return 7.69711747013104972 - log1p(-g.next_double());
        const double f0 = __longlong_as_double((long long)__ldg(zig_fe_bits + idx - 1));
        const double f1 = __longlong_as_double((long long)__ldg(zig_fe_bits + idx));
        if ((f0 - f1) * g.next_double() + f1 < exp(-x)) return x;
    }
}

// Python round(x, 6) for 0 <= x < 2^53 / 10^6: the double nearest to x's
// exact value rounded (half-even) to 6 decimals = N / 1e6 with N exact
__device__ double round6(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    const int ex = (int)((b >> 52) & 0x7FF);
    const unsigned long long frac = b & ((1ull << 52) - 1);
    const unsigned long long m = ex ? (frac | (1ull << 52)) : frac;
    const int e = ex ? ex - 1075 : -1074;
    const u128 p = (u128)m * 1000000u;
    unsigned long long n;
    if (e >= 0) {
        n = (unsigned long long)(p << e);
    } else if (-e >= 127) {
        n = 0;
    } else {
        const int sh = -e;
        const u128 q = p >> sh, rem = p & (((u128)1 << sh) - 1), half = (u128)1 << (sh - 1);
        n = (unsigned long long)q;
        if (rem > half || (rem == half && (n & 1))) n++;
    }
    return (double)n / 1000000.0;
}

}  // namespace tg

__global__ void k_gen_streams(const GenParams g, int write) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= g.n_streams) return;
    const int t = g.stream_trace[s], k = g.stream_fn[s];
    uint32_t pool[4];
    tg::seed_pool(g.seed[t], (uint32_t)k, pool);
    tg::Pcg64 rng;
    rng.seed_from(pool);
    const double scale = 1.0 / g.rates[g.fn_off[t] + k];     // rng.exponential(1.0 / rate)
    const double dur = g.duration[t];
    const int32_t rank = g.stream_rank[s];
    double tt = 0.0;
    int64_t n = 0;
    const int64_t o = write ? g.out_off[s] : 0;
    for (;;) {
        tt += scale * tg::std_exponential(rng);
        if (tt >= dur) break;
        if (write) {
            g.key[o + n] = (unsigned long long)__double_as_longlong(tg::round6(tt));
            g.val[o + n] = rank;
        }
        n++;
    }
    if (!write) g.count[s] = n;
}

// Per trace (one CTA): touched functions (by name rank), the rank of each
// arrival's name among them, and the fp64 arrival times.
__global__ void k_gen_flows(const unsigned long long* key, const int32_t* val, const int64_t* trace_off,
                            const int64_t* fn_off, int32_t* flow_rank_scratch, double* arrival,
                            int32_t* flow, int32_t* n_flows, uint8_t* touched_by_rank) {
    const int t = blockIdx.x;
    const int64_t a = trace_off[t], b = trace_off[t + 1];
    const int64_t f0 = fn_off[t];
    const int nf = (int)(fn_off[t + 1] - f0);
    uint8_t* tch = touched_by_rank + f0;
    int32_t* map = flow_rank_scratch + f0;
    for (int j = threadIdx.x; j < nf; j += blockDim.x) tch[j] = 0;
    __syncthreads();
    for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) tch[val[i]] = 1;
    __syncthreads();
    if (threadIdx.x == 0) {
        int c = 0;
        for (int j = 0; j < nf; j++) { map[j] = c; c += tch[j]; }
        n_flows[t] = c;
    }
    __syncthreads();
    for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
        arrival[i] = __longlong_as_double((long long)key[i]);
        flow[i] = map[val[i]];
    }
}

}  // namespace gfq
