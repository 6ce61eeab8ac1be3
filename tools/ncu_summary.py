"""Summarise one ncu --set full capture of the dominant simulation kernel.

    python tools/ncu_summary.py <capture.ncu-rep> <name> <workload> <sims> [algorithmic_bytes]

Writes profiles/<name>.txt (human summary) and profiles/ncu_k_sim_<workload>.json,
the numbers bench.py ties to its live launch time for the SM-issue roofline:
warp-instructions per launch (smsp__inst_executed.sum), issue / warp-active
percentages, DRAM bytes per launch, and the engine-source hash of the build
that was captured (bench.py reports whether it matches the running build).
"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import _norm_kernel, kernel_sass_hashes, source_hash  # noqa: E402

rep, name, workload, sims = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
algo_bytes = float(sys.argv[5]) if len(sys.argv) > 5 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = {h[i]: (v[i], u[i]) for i in range(len(h))}
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
        "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sass__inst_executed_local_loads",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
out = [f"# {name}: ncu --set full --clock-control none, one launch of the dominant kernel "
       f"({workload}, {sims} simulations; engine source {source_hash()})", ""]
for k in keys:
    if k in d:
        out.append(f"{k:60s} {d[k][0]} {d[k][1]}")
st = [(k, float(x[0])) for k, x in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
tot = sum(x for _, x in st) or 1
out += ["", "stall reasons (pc sampling, share of samples):"]
for k, x in sorted(st, key=lambda kv: -kv[1])[:10]:
    out.append(f"  {k[33:]:40s} {100 * x / tot:5.1f}%")
rd = float(d["dram__bytes_read.sum"][0]) * mult[d["dram__bytes_read.sum"][1]]
wr = float(d["dram__bytes_write.sum"][0]) * mult[d["dram__bytes_write.sum"][1]]
inst = float(d["smsp__inst_executed.sum"][0])
cyc = float(d["sm__cycles_elapsed.avg"][0])
n_sm = 148
out += ["", f"dram bytes per launch (read+write): {rd + wr:.0f}",
        f"issue utilisation over elapsed cycles: {inst / (cyc * n_sm * 4):.3f} "
        f"(warp-instructions / (cycles x {n_sm} SMs x 4))"]
if algo_bytes:
    out.append(f"algorithmic bytes per launch: {algo_bytes:.0f} "
               f"(traffic/algorithmic = {(rd + wr) / algo_bytes:.2f})")
open(f"profiles/{name}.txt", "w").write("\n".join(out) + "\n")
json.dump({"capture": f"profiles/{name}.txt", "workload": workload, "sims": sims,
           "kernel": d["Kernel Name"][0], "source_hash": source_hash(),
           "kernel_sass_hash": kernel_sass_hashes().get(_norm_kernel(d["Kernel Name"][0])),
           "inst_executed_per_launch": inst, "cycles_elapsed": cyc,
           "duration_ms": float(d["gpu__time_duration.sum"][0]),
           "issue_frac_elapsed": inst / (cyc * n_sm * 4),
           "dram_bytes_per_launch": rd + wr,
           "sm_inst_issued_pct": float(d["sm__inst_issued.avg.pct_of_peak_sustained_active"][0]),
           "warps_active_pct": float(d["sm__warps_active.avg.pct_of_peak_sustained_active"][0])},
          open(f"profiles/ncu_k_sim_{workload}.json", "w"), indent=1)
print("\n".join(out))
