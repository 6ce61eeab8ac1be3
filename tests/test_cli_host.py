"""Host side of the experiment driver (no GPU): config parsing, validation
and CLI exit codes as the reference's tests/test_cli.py checks them
(test_cli.py:54-79,114-116,138-142,155-180), the exporter's formatting, and
the generate sub-command (trace bytes vs the reference's gen_zipf)."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2507_08954_b200.cli import main
from paper_2507_08954_b200.config import ConfigError, load_config

HERE = os.path.dirname(os.path.abspath(__file__))
CFG = os.path.join(HERE, "golden", "cli")
BASE = open(os.path.join(CFG, "small.cfg")).read()


def _cfg(tmp_path, text):
    p = tmp_path / "exp.cfg"
    p.write_text(text)
    return str(p)


def test_load_default_config_fields():
    c = load_config(os.path.join(CFG, "medium.cfg"))
    assert (c.n_functions, c.zipf_s, c.rate_rps, c.duration_s, c.seed) == (19, 1.5, 2.0, 1500.0, 7)
    assert (c.util_threshold, c.util_window_s, c.pcie_mb_per_s) == (0.97, 0.4, 3000.0)
    assert c.workload_compute_share == 0.46
    assert c.echo["device"]["pcie_mb_per_s"] == "3000"
    d = c.device_configs()
    assert len(d) == 1 and d[0].util_threshold == 0.97
    t = load_config(os.path.join(CFG, "twodev.cfg"))
    assert t.device_count == 2 and t.dynamic_d and t.d_max == 3
    assert len(t.device_configs(pool_enabled=False)) == 2
    assert not t.device_configs(pool_enabled=False)[0].pool_enabled


@pytest.mark.parametrize("mutate,needle", [
    (lambda s: s.replace("alpha = 2", "alpha = 2\nbananas = 3"), "bananas"),
    (lambda s: s + "[mystery]\nx = 1\n", "mystery"),
    (lambda s: s.replace("[workload]", "[workload]\ntrace_path = ghost.csv"), "not both"),
    (lambda s: s.replace("policy = mqfq", "policy = lottery"), "unknown policy"),
    (lambda s: s.replace("count = 1", "count = 1\nd_max = 3"), "conflicting d_max"),
    (lambda s: s.replace("zipf_s = 1.5\n", ""), "missing"),
    (lambda s: s.replace("alpha = 2", "alpha = two"), "bad value for scheduler.alpha"),
    (lambda s: s.replace("count = 1", "count = 1\npool_enabled = maybe"), "bad boolean"),
    (lambda s: s.replace("count = 1", "count = 0"), "device count"),
])
def test_config_errors_exit_2(tmp_path, capsys, mutate, needle):
    path = _cfg(tmp_path, mutate(BASE))
    with pytest.raises(ConfigError):
        load_config(path)
    assert main(["run", "--config", path, "--out", str(tmp_path / "o")]) == 2
    assert needle in capsys.readouterr().err


def test_cli_usage_errors(tmp_path, capsys):
    path = _cfg(tmp_path, BASE)
    assert main(["compare", "--config", path, "--policies", "mqfq",
                 "--out", str(tmp_path / "x")]) == 2
    assert main(["sweep", "--config", path, "--param", "gamma", "--values", "1,2",
                 "--out", str(tmp_path / "x")]) == 2
    assert "gamma" in capsys.readouterr().err
    assert main(["sweep", "--config", path, "--param", "T", "--values", "a,b",
                 "--out", str(tmp_path / "x")]) == 2
    assert main(["bogus"]) == 2
    assert main(["run", "--config", str(tmp_path / "missing.cfg")]) == 2


def test_generate_matches_reference_trace(tmp_path):
    """generate writes the same bytes as the reference's gen_zipf + save_trace
    (hash recorded from the reference: tests/golden/cli/generate.sha256)."""
    out = tmp_path / "t.csv"
    assert main(["generate", "--functions", "24", "--zipf", "1.5", "--rate", "2.69",
                 "--duration", "600", "--seed", "3", "--out", str(out)]) == 0
    want = open(os.path.join(CFG, "generate.sha256")).read().split()[0]
    assert hashlib.sha256(out.read_bytes()).hexdigest() == want
    empty = tmp_path / "e.csv"
    assert main(["generate", "--functions", "4", "--zipf", "1.5", "--rate", "1.0",
                 "--duration", "0", "--out", str(empty)]) == 0
    assert empty.read_text() == "arrival_s,function\n"


def test_exporter_formatting(tmp_path):
    """invocations.csv / windows.csv / summary.json layout (metrics.py:253-287)."""
    from paper_2507_08954_b200.metrics import RunArrays, WindowReport, export, percentile
    run = RunArrays(["a", "b"], np.array([1, 0], np.int32), np.array([0.1, 0.25]),
                    np.array([0.5, 0.25]), np.array([2.0000004, 1.5]), np.array([2, 0], np.int8),
                    np.array([0, 1], np.int8))
    wins = [WindowReport(0.0, 30.0, comparable=True, max_gap=1.25, bound=2.0, violated=False),
            WindowReport(30.0, 30.0)]
    export(run, wins, {"b": 1, "a": [1.5]}, str(tmp_path))
    inv = (tmp_path / "invocations.csv").read_text().splitlines()
    assert inv[0].startswith("function,arrival_s,")
    assert inv[1] == "b,0.100000,0.500000,2.000000,cold,0,0.400000,1.500000,1.900000"
    assert inv[2] == "a,0.250000,0.250000,1.500000,gpu_warm,1,0.000000,1.250000,1.250000"
    assert (tmp_path / "windows.csv").read_text() == (
        "window_start_s,max_gap,bound,violated\n0.000000,1.250000,2.000000,false\n"
        "30.000000,,,false\n")
    assert json.loads((tmp_path / "summary.json").read_text()) == {"a": [1.5], "b": 1}
    assert (tmp_path / "summary.json").read_text().endswith("}\n")
    assert not [p for p in os.listdir(tmp_path) if p.endswith(".tmp")]
    assert percentile([], 50) == 0.0 and percentile([3.0], 99) == 3.0
    assert percentile([1.0, 2.0, 3.0, 4.0], 50.0) == 2.5
