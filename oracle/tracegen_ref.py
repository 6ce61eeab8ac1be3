"""TEST INFRASTRUCTURE ONLY (parity checker for the GPU trace generator).

Pure-Python restatement of what the reference's gen_zipf
(gpufairq/workload.py:82-111) computes through numpy 2.3
(numpy/random/bit_generator.pyx SeedSequence, pcg64.h PCG64 XSL-RR,
distributions.c standard_exponential_zig): integer-exact, used by
tests/test_tracegen_host.py to pin each stage against numpy itself, and as
the readable statement of the algorithm the CUDA kernel
(paper_2507_08954_b200/csrc/tracegen.cuh) implements.
"""
from __future__ import annotations

import math

M32 = 0xFFFFFFFF
M64 = (1 << 64) - 1
M128 = (1 << 128) - 1
INIT_A, MULT_A, INIT_B, MULT_B = 0x43B0D7E5, 0x931E8875, 0x8B51F9DD, 0x58F38DED
MIX_L, MIX_R = 0xCA01F9DD, 0x4973F715
PCG_MULT = (0x2360ED051FC65DA4 << 64) | 0x4385DF649FCCF645
ZIG_R = 7.69711747013104972


def _words(n: int) -> list[int]:
    if n == 0:
        return [0]
    out = []
    while n:
        out.append(n & M32)
        n >>= 32
    return out


def seed_pool(seed: int, spawn: tuple[int, ...]) -> list[int]:
    """SeedSequence(seed, spawn_key=spawn).pool (bit_generator.pyx mix_entropy)."""
    run = _words(seed)
    sp = [w for k in spawn for w in _words(k)]
    if sp and len(run) < 4:
        run = run + [0] * (4 - len(run))
    ent = run + sp
    hc = [INIT_A]

    def hashmix(v):
        v ^= hc[0]
        hc[0] = (hc[0] * MULT_A) & M32
        v = (v * hc[0]) & M32
        return v ^ (v >> 16)

    def mix(x, y):
        r = (MIX_L * x - MIX_R * y) & M32
        return r ^ (r >> 16)

    pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(4)]
    for s in range(4):
        for d in range(4):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(4, len(ent)):
        for d in range(4):
            pool[d] = mix(pool[d], hashmix(ent[s]))
    return pool


def generate_state64(pool: list[int], n: int) -> list[int]:
    hc = INIT_B
    w = []
    for i in range(2 * n):
        v = pool[i % 4] ^ hc
        hc = (hc * MULT_B) & M32
        v = (v * hc) & M32
        w.append(v ^ (v >> 16))
    return [w[2 * i] | (w[2 * i + 1] << 32) for i in range(n)]


class PCG64:
    """numpy PCG64 seeded from a SeedSequence pool (pcg64.h, _pcg64.pyx)."""

    def __init__(self, pool):
        v = generate_state64(pool, 4)
        initstate = (v[0] << 64) | v[1]
        initseq = (v[2] << 64) | v[3]
        self.inc = ((initseq << 1) | 1) & M128
        self.state = 0
        self._step()
        self.state = (self.state + initstate) & M128
        self._step()

    def _step(self):
        self.state = (self.state * PCG_MULT + self.inc) & M128

    def next64(self) -> int:
        self._step()
        hi, lo = self.state >> 64, self.state & M64
        rot = hi >> 58
        x = hi ^ lo
        return ((x >> rot) | (x << ((64 - rot) & 63))) & M64

    def next_double(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)


def standard_exponential(rng: PCG64, ke, we, fe) -> float:
    while True:
        ri = rng.next64() >> 3
        idx = ri & 0xFF
        ri >>= 8
        x = ri * we[idx]
        if ri < ke[idx]:
            return x
        if idx == 0:
            return ZIG_R - math.log1p(-rng.next_double())
        if (fe[idx - 1] - fe[idx]) * rng.next_double() + fe[idx] < math.exp(-x):
            return x


def round6(x: float) -> float:
    """Python round(x, 6) via exact integer arithmetic (what the kernel does)."""
    m, e = math.frexp(x)
    mi = int(m * (1 << 53))
    e -= 53
    p = mi * 10 ** 6
    if e >= 0:
        n = p << e
    else:
        sh = -e
        n, rem = p >> sh, p & ((1 << sh) - 1)
        half = 1 << (sh - 1)
        if rem > half or (rem == half and (n & 1)):
            n += 1
    return n / 1e6


def stream(seed: int, k: int, rate: float, duration: float, ke, we, fe) -> list[float]:
    """Arrival times of function rank k (workload.py:99-108)."""
    rng = PCG64(seed_pool(seed, (k,)))
    scale = 1.0 / rate
    t, out = 0.0, []
    while True:
        t += scale * standard_exponential(rng, ke, we, fe)
        if t >= duration:
            return out
        out.append(round6(t))
