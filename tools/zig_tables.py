"""Recover numpy's exponential-ziggurat tables (ke_double, we_double,
fe_double; numpy/random/src/distributions/ziggurat_constants.h) for the GPU
trace generator, and write paper_2507_08954_b200/data/zig_exp.npz.

numpy does not export them.  we[] and ke[] are read off Generator.exponential
itself, driven by a scripted bit generator (a bitgen_t capsule whose
next_uint64 returns chosen words): idx = (u >> 3) & 0xff, ri = u >> 11,
fast path x = ri * we[idx] iff ri < ke[idx].  fe[] (used only on the 1.1%
rejection path) is located in numpy's random extension binaries next to the
recovered we[] bytes.  tests/test_tracegen_host.py checks all three tables by
replaying numpy's own PCG64 word stream through them (>= 10^6 draws, so the
rejection path runs ~10^4 times) against Generator.standard_exponential.

    python tools/zig_tables.py
"""
import ctypes
import glob
import os
import threading

import numpy as np

NEXT64 = ctypes.CFUNCTYPE(ctypes.c_uint64, ctypes.c_void_p)
NEXT32 = ctypes.CFUNCTYPE(ctypes.c_uint32, ctypes.c_void_p)
NEXTD = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_void_p)


class BitgenT(ctypes.Structure):
    _fields_ = [("state", ctypes.c_void_p), ("next_uint64", NEXT64), ("next_uint32", NEXT32),
                ("next_double", NEXTD), ("next_raw", NEXT64)]


class Scripted:
    """A numpy bit generator that replays scripted 64-bit words / doubles."""

    def __init__(self):
        self.words, self.doubles, self.calls = [], [], 0
        self._n64 = NEXT64(self._next64)
        self._n32 = NEXT32(lambda st: 0)
        self._nd = NEXTD(self._nextd)
        self._s = BitgenT(None, self._n64, self._n32, self._nd, self._n64)
        new = ctypes.pythonapi.PyCapsule_New
        new.restype = ctypes.py_object
        new.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p]
        self.capsule = new(ctypes.addressof(self._s), b"BitGenerator", None)
        self.lock = threading.Lock()

    def _next64(self, st):
        self.calls += 1
        return self.words.pop(0) if self.words else (1 << 11) | (1 << 3)   # ri 1, idx 1

    def _nextd(self, st):
        self.calls += 1
        return self.doubles.pop(0) if self.doubles else 0.0

    def draw(self, words, doubles=()):
        self.words, self.doubles, self.calls = list(words), list(doubles), 0
        return self.gen.standard_exponential(), self.calls


def recover():
    sg = Scripted()
    sg.gen = np.random.Generator(sg)
    we = np.zeros(256)
    ke = np.zeros(256, dtype=np.uint64)
    for idx in range(256):
        word = lambda ri: (ri << 11) | (idx << 3)
        # ke: smallest ri that leaves the fast path (monotone)
        lo, hi = 0, 1 << 53
        while lo < hi:
            mid = (lo + hi) // 2
            _, calls = sg.draw([word(mid)], [0.5])
            if calls == 1:
                lo = mid + 1
            else:
                hi = mid
        ke[idx] = lo
        # ri = 2^20 (exact scaling).  Below ke the fast path returns x; with
        # ke[idx] <= ri (ke is 0 for some layers) the rejection test with
        # U = 0 still accepts a tiny x (fe[idx] < exp(-x) ~ 1) and returns it
        ri = 1 << 20
        x, calls = sg.draw([word(ri)], [0.0])
        assert calls == (1 if ri < lo else 2), (idx, calls)
        we[idx] = x / ri
        assert we[idx] * ri == x
    return sg, we, ke


def find_fe(we):
    pat = we.astype("<f8").tobytes()
    d = os.path.dirname(np.random.__file__)
    for so in sorted(glob.glob(os.path.join(d, "*.so"))):
        blob = open(so, "rb").read()
        i = blob.find(pat)
        if i >= 0:            # the compiler places fe_double right before we_double
            for a in (i - len(pat), i + len(pat)):
                fe = np.frombuffer(blob[a: a + len(pat)], dtype="<f8").copy()
                if fe[0] == 1.0 and np.all(np.diff(fe) < 0):
                    return fe, os.path.basename(so)
    raise SystemExit("we_double bytes not found in numpy's random extensions")


def main():
    sg, we, ke = recover()
    fe, src = find_fe(we)
    assert fe[0] == 1.0 and np.all(np.diff(fe) < 0), "fe_double candidate is not decreasing from 1"
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_2507_08954_b200", "data", "zig_exp.npz")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    np.savez(out, ke=ke, we=we, fe=fe, numpy_version=np.__version__)
    print(f"ke/we recovered by probing, fe from {src}; wrote {out}")


if __name__ == "__main__":
    main()
