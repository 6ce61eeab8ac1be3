"""Two ranks, each running libgfq (sharing the one GPU of this box, gloo
for the collective): the strong split of one fixed C3 sweep
(dist.partition), histograms all-reduced and summary rows all-gathered,
must equal a single-process run of the whole sweep bit for bit
(the reference's serial sweep loop, cli.py:148-157)."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_libgfq_strong_split(tmp_path):
    out = tmp_path / "dist.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(HERE, "dist_worker.py"), str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    res = json.loads(out.read_text())
    assert res["world"] == 2 and res["parts"] == [256, 256]
    assert res["ids_cover"]
    assert res["hist_equal"] and res["hist_total"] == res["arrivals"]
    assert res["summary_equal"] and res["dispatches_equal"]
