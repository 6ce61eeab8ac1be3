"""Diagnostic runner (GPU box): all golden cases through the engine, per-family
pass counts, and for the first failures the first differing row vs the oracle."""
import os
import sys
import time
from collections import Counter, defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), HERE, os.path.join(HERE, "golden")]

from cases import all_cases  # noqa: E402
from golden_check import golden  # noqa: E402
from gpu_harness import compare_to_golden, first_diff, run_cases  # noqa: E402

from oracle import oracle as orc  # noqa: E402

fams = sys.argv[1:] or None
cases = [c for c in all_cases() if fams is None or c["name"].split("/")[0] in fams]
t0 = time.time()
from paper_2507_08954_b200.engine import Engine  # noqa: E402
eng = Engine(0)
outs, res = run_cases(cases, eng, early_exit=False, event_log_cap=65536, audit_util_cap=16384)
print(f"ran {len(cases)} cases in {time.time() - t0:.1f}s")
g = golden()
ok, tot = Counter(), Counter()
fails = defaultdict(list)
for c, o in zip(cases, outs):
    fam = c["name"].split("/")[0]
    tot[fam] += 1
    m = compare_to_golden(o, g[c["name"]])
    if m:
        fails[fam].append((c, o, m))
    else:
        ok[fam] += 1
for fam in tot:
    print(f"{fam:12s} {ok[fam]}/{tot[fam]}")
shown = 0
for fam, lst in fails.items():
    for c, o, m in lst[:3]:
        print("FAIL", c["name"], m, "status", o.get("status"))
        if o.get("status"):
            continue
        ref = orc.run_case(c, want_events=True)
        for k in ("transcript", "dispatch", "records", "exec", "util", "backlog", "events"):
            if k in o and k in ref:
                d = first_diff(o[k], ref[k])
                if d:
                    print(f"   {k}: first diff at {d[0]}:\n      gpu={d[1]}\n      ref={d[2]}")
        for k in ("summary",):
            if o[k] != ref[k]:
                print("   summary gpu", o[k], "ref", ref[k])
        shown += 1
print("TOTAL", sum(ok.values()), "/", sum(tot.values()))

# ---- fast builds (MQFQ / DeviceSet, no audit logs): dispatch rows, records,
# exec rows and statistics against the same golden fingerprints.  The
# single-device subset runs k_sim<false,true>, the full MQFQ set k_sim<false,false>.
from paper_2507_08954_b200 import _abi  # noqa: E402
fast = [c for c in cases if c.get("policy", "mqfq") == "mqfq" and not c.get("scripted")]
one = [c for c in fast if len(c.get("devices", [{}])) == 1]
for label, sel in (("FAST 1-device build", one), ("FAST multi-device build", fast)):
    outs2, _ = run_cases(sel, eng, outputs=_abi.WANT_STATS | _abi.WANT_RECORDS |
                         _abi.WANT_DISPATCH, early_exit=True)
    bad2 = []
    for c, o in zip(sel, outs2):
        m = compare_to_golden(o, g[c["name"]], exact_keys=("dispatch", "records", "exec"))
        if m:
            bad2.append((c["name"], m))
    print(label + ":", len(sel) - len(bad2), "/", len(sel), bad2[:5])

# ---- one batch spanning all three kernel classes (no audit logs): generic
# (other policies, scripted), multi-device MQFQ and 1-device MQFQ launches
outs3, _ = run_cases(cases, eng, outputs=_abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_DISPATCH,
                     early_exit=True)
bad3 = []
for c, o in zip(cases, outs3):
    m = compare_to_golden(o, g[c["name"]], exact_keys=("dispatch", "records", "exec"))
    if m:
        bad3.append((c["name"], m))
print("MIXED-class batch:", len(cases) - len(bad3), "/", len(cases), bad3[:5])


# ---- flows-in-global build forced on every case (generic, all outputs)
outs4, _ = run_cases(cases, eng, early_exit=False, event_log_cap=65536, audit_util_cap=16384,
                     flags=_abi.FLAG_FLOWS_GLOBAL)
bad4 = [(c["name"], m) for c, o in zip(cases, outs4) if (m := compare_to_golden(o, g[c["name"]]))]
print("FLOWS-GLOBAL build:", len(cases) - len(bad4), "/", len(cases), bad4[:5])
