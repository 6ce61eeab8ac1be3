"""Dump GPU fairness rows for a few cases (for diffing against the reference)."""
import json, os, sys
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), HERE, os.path.join(HERE, "golden")]
from cases import all_cases
from fingerprint import fp
from test_gpu_fairness import fairness_rows, run_fairness
from paper_2507_08954_b200.engine import Engine
gold = {c["name"]: c for c in json.load(open(os.path.join(HERE, "golden", "fairness_golden.json")))["cases"]}
cases = [c for c in all_cases() if not c.get("scripted")]
eng = Engine(0)
allrows = run_fairness(cases, eng)
bad = []
dump = {}
for c, rows in zip(cases, allrows):
    if fp(rows) != gold[c["name"]]["fp"]:
        bad.append(c["name"])
        if len(dump) < 6:
            dump[c["name"]] = [[x if not isinstance(x, float) else x.hex() for x in r] for r in rows]
print("fairness ok", len(cases) - len(bad), "/", len(cases), bad[:10])
os.makedirs("gpurun_out", exist_ok=True)
json.dump(dump, open("gpurun_out/fair_dump.json", "w"))
