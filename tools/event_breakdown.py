"""Warp-instructions of the simulation kernel per event kind.

    python tools/event_breakdown.py <capture.ncu-rep> <libgfq.so> <kernel-substring> \
        <events> <ticks> <arrivals> <completions> [out.txt]

Executed instructions per SASS address come from the capture's source page;
nvdisasm -gi gives each address its inline chain (innermost frame first), and
the outermost frame inside WarpSim's event loop decides the bucket:

  arrival     on_arrival (+ the arrival branch of run())
  completion  on_completion and below (Device.complete, pool cap, stats stream)
  tick        the monitor tick: on_monitor / monitor_tick / tick_util and the
              tick-run lines of run() (quiet-drain test, successor push)
  expiry      on_expiry
  drain       drain(): every dispatch() call after an arrival / completion /
              non-quiet tick (candidate scan, global VT, keep-alive refresh,
              token + memory admission, start, completion push)
  pool        the dynamic-event pool minimum (pool_min / pool_remove)
  swap        _swap_out_inactive
  loop        event selection and the rest of run()
  setup       per-simulation setup / teardown (sim_run, kernel prologue)

The event counts come from a -DGFQ_DIAG=1 bench line of the same workload
(ticks) and the engine's counters (events, dispatches = arrivals =
completions); expiries = events - ticks - arrivals - completions.
"""

from __future__ import annotations

import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_funcs import func_ranges, owner  # noqa: E402
from ncu_lines import sass_page  # noqa: E402

BUCKET = {
    "on_arrival": "arrival", "policy_on_arrival": "arrival",
    "on_completion": "completion", "device_complete": "completion",
    "policy_on_completion": "completion", "comp_flush": "completion",
    "on_monitor": "tick", "monitor_tick": "tick", "tick_util": "tick",
    "on_expiry": "expiry",
    "drain": "drain",
    "pool_min": "pool", "pool_remove": "pool",
    "swap_out_inactive": "swap",
}


def inline_chains(so: str, kernel: str):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
    chains = {}
    for fn in os.listdir(d):
        if not fn.endswith(".cubin"):
            continue
        txt = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, fn)], capture_output=True,
                             text=True).stdout
        cur_fn, frames, pending = None, [], False
        for ln in txt.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                cur_fn = m.group(1)
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at)?', ln)
            if m:
                if not pending:
                    frames = []
                    pending = True
                frames.append((os.path.basename(m.group(1)), int(m.group(2))))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and cur_fn and kernel in cur_fn:
                chains[int(m.group(1), 16)] = list(frames)
                pending = False
    return chains


def main():
    rep, so, kernel = sys.argv[1], sys.argv[2], sys.argv[3]
    events, ticks, arrivals, completions = (int(x) for x in sys.argv[4:8])
    out_path = sys.argv[8] if len(sys.argv) > 8 else None
    csrc = os.path.join(os.path.dirname(so), "csrc")
    ranges = {f: func_ranges(os.path.join(csrc, f)) for f in os.listdir(csrc)
              if f.endswith((".cuh", ".cu"))}
    warp_src = open(os.path.join(csrc, "sim_warp.cuh")).read().splitlines()
    # run()'s tick-run block and arrival branch, by their source markers
    tick_lo = next(i for i, s in enumerate(warp_src) if "kind == EV_TICK" in s) + 1
    tick_hi = next(i for i in range(tick_lo, len(warp_src)) if "int slot = pmin_slot;" in warp_src[i])
    arr_lo = next(i for i, s in enumerate(warp_src) if "if (kind == EV_ARRIVAL) {" in s) + 1
    data = sass_page(rep)
    chains = inline_chains(so, kernel)
    agg = defaultdict(int)
    for a, x, _ in data:                             # a: offset from the kernel's start
        fr = chains.get(a, [])
        bucket = None
        for f, line in reversed(fr):                 # outermost first
            if f not in ranges:
                continue
            name = owner(ranges[f], line)
            if f == "sim_warp.cuh" and name == "run":
                if tick_lo <= line < tick_hi:
                    bucket = "tick"
                elif arr_lo <= line < tick_lo - 1:
                    bucket = "arrival"
                else:
                    bucket = "loop"
                continue                              # an inner frame may be more specific
            if name in BUCKET:
                bucket = BUCKET[name]
                break
            if f == "gfq_engine.cu" and bucket is None:
                bucket = "setup"
        agg[bucket or "loop"] += x
    tot = sum(agg.values())
    expiries = events - ticks - arrivals - completions
    per = {"arrival": arrivals, "completion": completions, "tick": ticks, "expiry": expiries,
           "drain": arrivals, "pool": events, "swap": events, "loop": events, "setup": None}
    lines = [f"# per-event-kind warp-instructions: {os.path.basename(rep)} ({kernel})",
             f"# events {events}, ticks {ticks}, arrivals {arrivals}, completions {completions}, "
             f"expiries {expiries}; total {tot / 1e9:.2f} G warp-instructions "
             f"({tot / max(events, 1):.0f} per event, {tot / max(arrivals, 1):.0f} per dispatch)", "",
             f"{'bucket':12s} {'G inst':>8s} {'share':>6s} {'per unit':>9s}  unit"]
    for b in ("tick", "arrival", "completion", "expiry", "drain", "pool", "swap", "loop", "setup"):
        v = agg.get(b, 0)
        n = per[b]
        unit = {"drain": "dispatch", "pool": "event", "swap": "event", "loop": "event",
                "setup": "-"}.get(b, b)
        lines.append(f"{b:12s} {v / 1e9:8.3f} {100 * v / tot:5.1f}% "
                     f"{(v / n if n else 0):9.0f}  {unit}")
    txt = "\n".join(lines) + "\n"
    print(txt)
    if out_path:
        open(out_path, "w").write(txt)


if __name__ == "__main__":
    main()
