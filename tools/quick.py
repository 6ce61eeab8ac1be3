"""A/B timing of libgfq builds on one workload: for each .so given, load it
in a fresh process (GFQ_LIB), run the workload W + K times and print the
best and median k_sim + k_reduce time and dispatch decisions/s.

    python tools/quick.py [--workload c3] [--seeds N] [--steps K] lib1.so [lib2.so ...]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, numpy as np
sys.path.insert(0, %r)
from paper_2507_08954_b200 import _abi, sweep
from paper_2507_08954_b200.engine import Engine
eng = Engine(0)
kw = {"n_seeds": %d} if %d else {}
w = sweep.build(%r, 0, engine=eng, **kw)
w.upload(eng)
arr = w.sims_array()
ms = []
for i in range(%d):
    eng.run(arr, outputs=_abi.WANT_STATS, early_exit=True)
    ms.append(eng.kernel_ms())
c = eng.output(_abi.OUT_COUNTERS).reshape(-1, _abi.NCOUNTERS)
st = eng.output(_abi.OUT_STATUS)
disp = int(c[:, 2].sum())
ms = ms[3:]
print(json.dumps({"ms_best": min(ms), "ms_med": float(np.median(ms)), "disp": disp,
                  "events": int(c[:, 0].sum()), "bad_status": int((st != 0).sum())}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--seeds", type=int, default=0)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    for rep in range(2):
        for lib in a.libs:
            code = CHILD % (ROOT, a.seeds, a.seeds, a.workload, a.steps + 3)
            env = dict(os.environ, GFQ_LIB=os.path.abspath(lib))
            r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
            except Exception:
                print(lib, "FAILED", r.stderr[-800:])
                continue
            print(f"{os.path.basename(lib):28s} best {d['ms_best']:8.3f} ms  med {d['ms_med']:8.3f} ms  "
                  f"{d['disp'] / d['ms_best'] / 1e3:8.1f} M disp/s  events {d['events']}  "
                  f"bad {d['bad_status']}", flush=True)


if __name__ == "__main__":
    main()
