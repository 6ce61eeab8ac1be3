"""C4 (4096 functions per simulation) through the engine vs the oracle:
dispatch rows and completion records bit-exact, statistics within 1e-9."""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as orc
from paper_2507_08954_b200 import _abi, sweep
from paper_2507_08954_b200.engine import Engine


def check(n_seeds: int = 1, eng: Engine | None = None, flags: int = 0) -> list[str]:
    w = sweep.c4(n_seeds=n_seeds)
    own = eng is None
    eng = eng or Engine(0)
    w.upload(eng)
    res = eng.run(w.sims_array(), outputs=_abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_DISPATCH,
                  flags=flags)
    bad = []
    for i, s in enumerate(w.sims):
        tr, tab = w.traces[s.trace], w.tabs[s.flowtab]
        r = orc.run_packed(_abi.Sim.from_buffer_copy(s), tr.arrival, tr.flow, tr.n_flows,
                           {"warm": tab.warm, "cold": tab.cold, "mem": tab.mem,
                            "share": tab.share, "weight": tab.weight},
                           [_abi.device_cfg_from(w.dcfgs[s.device_cfg])], want_audit=False)
        rec = res.records(i)
        comp = res.completion_order(i)
        dr = res.dispatch_rows(i)
        ok = (np.array_equal(comp, r["rec_inv"]) and
              np.array_equal(rec["complete"][comp], r["rec_complete"]) and
              np.array_equal(rec["dispatch"][comp], r["rec_dispatch"]) and
              np.array_equal(rec["state"][comp], r["rec_state"]) and
              np.array_equal(dr["inv"], r["d_inv"]) and
              np.array_equal(dr["vt_before"], r["d_vt_before"]) and
              np.array_equal(dr["gvt"], r["d_gvt"]))
        fs = res.flow_stats(i)
        ok = ok and np.array_equal(fs["count"], r["f_count"]) and \
            np.allclose(fs["mean"], r["f_mean"], rtol=1e-9, atol=0) and \
            np.allclose(fs["var"], r["f_var"], rtol=1e-9, atol=0)
        ok = ok and abs(res.summary[i, 0] - r["weighted_avg_latency"]) <= 1e-9 * r["weighted_avg_latency"]
        if not ok:
            bad.append(f"c4 sim {i}")
    if own:
        eng.close()
    return bad


if __name__ == "__main__":
    print("C4 parity mismatches:", check(1))
