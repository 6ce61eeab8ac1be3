"""Generate tests/golden/cli_golden.json by running the UNMODIFIED reference
CLI (gpufairq.cli.main, imported read-only from /root/reference/pkg/src) on
the commands in CLI_COMMANDS.  Run in the build container only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cli_golden.py

For every file a command writes it stores the sha256 and size; summary.json
files are also stored parsed (their ``var_latency_s`` values are compared
within 1e-9 relative, see paper_2507_08954_b200/metrics.py), and the top
level compare.csv / sweep.csv verbatim.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
CFG = os.path.join(HERE, "cli")

# (name, argv without --out); config paths are relative to tests/golden/cli
CLI_COMMANDS = [
    ("compare_default", ["compare", "--config", "default.cfg",
                         "--policies", "mqfq,fcfs,batch,sjf,fcfs_naive"]),
    ("compare_medium", ["compare", "--config", "medium.cfg", "--policies", "mqfq,fcfs,sjf,batch"]),
    ("compare_twodev", ["compare", "--config", "twodev.cfg", "--policies", "mqfq,fcfs,sjf"]),
    ("sweep_T", ["sweep", "--config", "default.cfg", "--param", "T", "--values", "0,1,5,10"]),
    ("sweep_alpha", ["sweep", "--config", "default.cfg", "--param", "alpha",
                     "--values", "0,0.5,2,4"]),
    ("sweep_dmax", ["sweep", "--config", "default.cfg", "--param", "d_max", "--values", "1,2,4"]),
    ("sweep_pool", ["sweep", "--config", "medium.cfg", "--param", "pool_max_containers",
                    "--values", "4,8,16"]),
    ("sweep_rate", ["sweep", "--config", "small.cfg", "--param", "rate_rps",
                    "--values", "0.5,1,3"]),
    ("run_small_naive", ["run", "--config", "small.cfg", "--policy", "fcfs_naive"]),
    ("run_small_seed", ["run", "--config", "small.cfg", "--seed", "11"]),
    ("run_twodev", ["run", "--config", "twodev.cfg"]),
    ("compare_files", ["compare", "--config", "files.cfg", "--policies", "mqfq,fcfs,batch,sjf"]),
    ("sweep_files_T", ["sweep", "--config", "files.cfg", "--param", "T", "--values", "0,2,8"]),
]


def snapshot(out_dir: str) -> dict:
    files = {}
    for root, _, names in os.walk(out_dir):
        for nm in sorted(names):
            p = os.path.join(root, nm)
            rel = os.path.relpath(p, out_dir)
            data = open(p, "rb").read()
            ent = {"sha256": hashlib.sha256(data).hexdigest(), "size": len(data)}
            if nm == "summary.json":
                ent["json"] = json.loads(data)
            elif rel in ("compare.csv", "sweep.csv"):
                ent["text"] = data.decode()
            files[rel] = ent
    return files


def main() -> None:
    sys.path.insert(0, "/root/reference/pkg/src")
    from gpufairq.cli import main as ref_main
    out = {}
    cwd = os.getcwd()
    os.chdir(CFG)
    try:
        for name, argv in CLI_COMMANDS:
            with tempfile.TemporaryDirectory() as td:
                rc = ref_main(argv + ["--out", td])
                out[name] = {"argv": argv, "rc": rc, "files": snapshot(td)}
                print(name, rc, len(out[name]["files"]), "files")
    finally:
        os.chdir(cwd)
    with open(os.path.join(HERE, "cli_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
