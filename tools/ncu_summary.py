"""Write profiles/<name>.txt (+ profiles/ncu_k_sim.json) from an ncu --set full capture."""
import csv
import io
import json
import subprocess
import sys

rep, name, algo_bytes = sys.argv[1], sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else 0
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
out = [f"# {name}: ncu --set full --clock-control none, one k_sim launch (C3 4096-sim sweep)", ""]
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
out += ["", f"dram bytes per launch (read+write): {rd + wr:.0f}"]
if algo_bytes:
    out.append(f"algorithmic bytes per launch: {algo_bytes:.0f} (traffic/algorithmic = {(rd + wr) / algo_bytes:.2f})")
open(f"profiles/{name}.txt", "w").write("\n".join(out) + "\n")
json.dump({"capture": f"profiles/{name}.txt", "dram_bytes_per_launch": rd + wr,
           "sm_inst_issued_pct": float(d["sm__inst_issued.avg.pct_of_peak_sustained_active"][0])},
          open("profiles/ncu_k_sim.json", "w"), indent=1)
print("\n".join(out))
