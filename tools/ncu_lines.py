"""Attribute an ncu capture's per-SASS-instruction metrics to CUDA source lines.

    python tools/ncu_lines.py <report.ncu-rep> <libgfq.so> [kernel-substring] [top]

ncu's source page gives executed-instruction counts and stall samples per
SASS address; nvdisasm's line table maps each address to file:line.  Prints
the hottest source lines and the hot-code footprint.
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def sass_page(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, iex = hdr.index("Address"), hdr.index("Instructions Executed")
    ismp = hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[ia], 16), int(r[iex] or 0), int(r[ismp] or 0)))
        except (ValueError, IndexError):
            pass
    data.sort()
    base = data[0][0]
    return [(a - base, x, s) for a, x, s in data]


def line_table(so, kernel):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
    table = {}
    for fn in os.listdir(d):
        if not fn.endswith(".cubin"):
            continue
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, fn)], capture_output=True,
                             text=True).stdout
        cur_fn, cur_line = None, None
        for ln in txt.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                cur_fn = m.group(1)
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and cur_fn and kernel in cur_fn:
                table[int(m.group(1), 16)] = cur_line
    return table


def main():
    rep, so = sys.argv[1], sys.argv[2]
    kernel = sys.argv[3] if len(sys.argv) > 3 else "k_sim"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    data = sass_page(rep)
    table = line_table(so, kernel)
    agg = defaultdict(lambda: [0, 0, 0])
    for a, x, s in data:
        k = table.get(a, "?")
        agg[k][0] += x
        agg[k][1] += s
        agg[k][2] += 1
    tx = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"SASS instrs {len(data)}, executed {tx/1e9:.2f} G, stall samples {ts}")
    src = {}
    for k, _ in agg.items():
        if k and ":" in k:
            f, l = k.rsplit(":", 1)
            path = os.path.join(os.path.dirname(so), "csrc", f)
            if os.path.exists(path):
                src.setdefault(f, open(path).read().splitlines())
    print(f"{'exec':>8} {'exec%':>6} {'stall%':>6} {'#sass':>5}  line")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        text = ""
        if k and ":" in k:
            f, l = k.rsplit(":", 1)
            lines = src.get(f)
            if lines and int(l) - 1 < len(lines):
                text = lines[int(l) - 1].strip()[:70]
        print(f"{v[0]/1e6:7.0f}M {100*v[0]/tx:5.1f}% {100*v[1]/ts:5.1f}% {v[2]:5d}  {k:22s} {text}")


if __name__ == "__main__":
    main()
