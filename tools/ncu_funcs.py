"""Aggregate an ncu capture's executed instructions / stall samples by the
enclosing source FUNCTION (exclusive, innermost inlined frame), using the
line table of the profiled .so and the csrc sources next to it.

    python tools/ncu_funcs.py <report.ncu-rep> <libgfq.so> [kernel-substring] [csrc-dir]
"""
import os
import re
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_lines import line_table, sass_page  # noqa: E402

DEF = re.compile(r"^\s*(?:template\s*<[^>]*>\s*)?(?:FI|__device__|__global__|static)[^;{]*?\b(\w+)\s*\([^;]*\)\s*(?:const\s*)?\{")


def func_ranges(path):
    lines = open(path).read().splitlines()
    starts = []
    for i, ln in enumerate(lines):
        m = DEF.match(ln)
        if m:
            starts.append((i + 1, m.group(1)))
    return starts


def owner(starts, line):
    name = "?"
    for s, nm in starts:
        if s <= line:
            name = nm
        else:
            break
    return name


def main():
    rep, so = sys.argv[1], sys.argv[2]
    kernel = sys.argv[3] if len(sys.argv) > 3 else "k_sim"
    csrc = sys.argv[4] if len(sys.argv) > 4 else os.path.join(os.path.dirname(so), "csrc")
    data = sass_page(rep)
    table = line_table(so, kernel)
    ranges = {}
    agg = defaultdict(lambda: [0, 0])
    for a, x, s in data:
        k = table.get(a)
        key = "?"
        if k and ":" in k:
            f, l = k.rsplit(":", 1)
            p = os.path.join(csrc, f)
            if os.path.exists(p):
                if f not in ranges:
                    ranges[f] = func_ranges(p)
                key = f"{f}:{owner(ranges[f], int(l))}"
            else:
                key = f
        agg[key][0] += x
        agg[key][1] += s
    tx = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"executed {tx/1e9:.2f} G warp-instructions")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        if v[0] / tx < 0.003:
            continue
        print(f"{v[0]/1e6:8.0f}M {100*v[0]/tx:5.1f}%  stall {100*v[1]/ts:5.1f}%  {k}")


if __name__ == "__main__":
    main()
