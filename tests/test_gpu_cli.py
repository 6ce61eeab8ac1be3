"""Batched experiment driver + exporter (paper_2507_08954_b200.cli / .metrics)
against the reference CLI's own output files (tests/golden/cli_golden.json,
made by tests/golden/make_cli_golden.py from the unmodified reference).

Every file the reference writes -- per-experiment invocations.csv,
windows.csv, summary.json, and the top-level trace.csv, compare.csv,
sweep.csv -- must be byte-identical; summary.json is compared parsed, with
``var_latency_s`` within 1e-9 relative (the reference squares with libm
``pow``, see metrics.py) and everything else exact.
"""

from __future__ import annotations

import hashlib
import json
import os

import pytest

from make_cli_golden import CFG, CLI_COMMANDS

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _gold():
    return json.load(open(os.path.join(HERE, "golden", "cli_golden.json")))


def _same_summary(a, b, path=""):
    if isinstance(a, dict):
        assert isinstance(b, dict) and sorted(a) == sorted(b), path
        for k in a:
            _same_summary(a[k], b[k], f"{path}.{k}")
    elif path.endswith("var_latency_s"):
        assert abs(a - b) <= 1e-9 * max(abs(a), abs(b)), (path, a, b)
    else:
        assert a == b and type(a) is type(b), (path, a, b)


@pytest.mark.parametrize("name,argv", CLI_COMMANDS, ids=[c[0] for c in CLI_COMMANDS])
def test_cli_matches_reference_files(name, argv, tmp_path, monkeypatch):
    from paper_2507_08954_b200.cli import main
    gold = _gold()[name]
    monkeypatch.chdir(CFG)
    out = tmp_path / "out"
    assert main(argv + ["--out", str(out)]) == gold["rc"]
    got = {}
    for root, _, names in os.walk(out):
        for nm in names:
            p = os.path.join(root, nm)
            got[os.path.relpath(p, out)] = open(p, "rb").read()
    assert sorted(got) == sorted(gold["files"])
    for rel, ent in gold["files"].items():
        data = got[rel]
        if hashlib.sha256(data).hexdigest() == ent["sha256"]:
            continue
        assert rel.endswith("summary.json"), f"{name}/{rel} differs from the reference"
        _same_summary(json.loads(data), ent["json"], rel)


def test_run_experiment_dropin(tmp_path):
    """cli.run_experiment returns (records, windows, summary) like the reference."""
    from paper_2507_08954_b200.cli import run_experiment
    from paper_2507_08954_b200.config import load_config
    cfg = load_config(os.path.join(CFG, "small.cfg"))
    records, windows, summary = run_experiment(cfg, str(tmp_path / "o"))
    assert len(records) == sum(v["count"] for v in summary["per_function"].values())
    assert [r.complete_s for r in records] == sorted(r.complete_s for r in records)
    assert all(w.window_s == 30.0 for w in windows)
    assert (tmp_path / "o" / "summary.json").exists()


def test_compare_is_one_batch(tmp_path, monkeypatch):
    """compare runs every policy in a single engine launch."""
    from paper_2507_08954_b200 import cli, engine
    calls = []
    orig = engine.Engine.launch

    def counting(self, stream=None):
        calls.append(self.n_sims)
        return orig(self, stream)

    monkeypatch.setattr(engine.Engine, "launch", counting)
    monkeypatch.chdir(CFG)
    assert cli.main(["compare", "--config", "default.cfg", "--policies", "mqfq,fcfs,sjf",
                     "--out", str(tmp_path)]) == 0
    assert calls == [3]
