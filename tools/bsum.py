"""Summarise a bench.py JSON line from stdin: value, sims, kernel ms."""
import json
import sys

for ln in sys.stdin.read().splitlines():
    ln = ln.strip()
    if not ln.startswith("{"):
        continue
    d = json.loads(ln)
    c = d.get("config", {})
    print(f"{sys.argv[1] if len(sys.argv) > 1 else ''} sims={c.get('sims')} "
          f"value={d['value']/1e6:.2f}M/s kernel={d.get('kernel_ms', {}).get('k_sim_mean', d.get('kernel_ms', {}).get('mean', 0)):.2f}ms "
          f"e2e={d.get('e2e', {}).get('value', 0)/1e6:.2f}M/s")
