"""A small random batch (tests/test_gpu_fuzz.py's generator) through every
build -- fast warp classes, generic with audit, flows in global memory,
CTA per simulation, forced warp -- checked against the oracle.  Sized to run
under compute-sanitizer (see tools/sanitize.sh).

    python tools/sanitize_batch.py [n_sims]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)
from test_gpu_fuzz import _check, _workload  # noqa: E402

from paper_2507_08954_b200.engine import Engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
traces, tabs, dcfgs, sims, _abi = _workload(np.random.default_rng(7), n)
eng = Engine(0)
eng.upload_traces(traces)
eng.upload_flowtabs(tabs)
eng.upload_device_cfgs(dcfgs)
for flags, audit in ((0, 0), (0, 1), (_abi.FLAG_FLOWS_GLOBAL, 0), (_abi.FLAG_CTA, 0), (_abi.FLAG_WARP, 0)):
    bad, over = _check(eng, list(range(len(sims))), sims, traces, tabs, dcfgs, _abi, flags, audit)
    print("flags", flags, "audit", audit, "mismatches", len(bad), "event-pool overflows", len(over),
          flush=True)
    assert not bad
