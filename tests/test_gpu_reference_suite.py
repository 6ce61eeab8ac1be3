"""The reference's OWN test suite, run against the CUDA engine.

tests/refshim puts a ``gpufairq`` package ahead of the unmodified reference
on PYTHONPATH: every reference module loads unchanged from the reference's
directory except ``gpufairq.engine``, which becomes this repo's drop-in
``Simulation`` / ``run_simulation`` over libgfq.so.  The reference's
test_engine.py (Simulation.step / run, keep-alive, determinism),
test_acceptance.py (A1-A11: 1000 fuzz runs + the medium workload through
run_simulation, the CLI's byte-identical exports), test_metrics.py and
test_cli.py (the reference CLI, whose cli.py:16 imports run_simulation from
.engine) must pass unmodified, and the shim's call log proves the
simulations went through the GPU engine (reference callers:
test_engine.py:17,136,149; test_acceptance.py:63,116,155,314).
"""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

from refsuite import ROOT, SHIM, locate

pytestmark = pytest.mark.gpu

FILES = ["test_engine.py", "test_acceptance.py", "test_metrics.py", "test_cli.py"]


def test_reference_suite_through_the_gpu_engine(tmp_path):
    loc = locate()
    if loc is None:
        pytest.skip("reference not installed (tools/install_ref.sh)")
    src, tests = loc
    log = tmp_path / "shim_calls.log"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([SHIM, ROOT, src]),
               GFQ_REF_SRC=src, GFQ_SHIM_LOG=str(log), PYTHONDONTWRITEBYTECODE="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-x",
           "--rootdir", tests, *FILES]
    r = subprocess.run(cmd, cwd=tests, env=env, capture_output=True, text=True, timeout=1500)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-25:])
    assert r.returncode == 0, tail
    calls = log.read_text().split()
    # A1 alone makes 1000 run_simulation calls; test_engine builds Simulations
    assert calls.count("run_simulation") >= 1000, (len(calls), tail)
    assert calls.count("Simulation") >= 10, (len(calls), tail)
    assert " passed" in tail and "failed" not in tail, tail


def test_shim_resolves_engine_to_libgfq():
    """In the shim, gpufairq.engine is this repo's engine and every other
    module is the reference's own file."""
    loc = locate()
    if loc is None:
        pytest.skip("reference not installed (tools/install_ref.sh)")
    src, _ = loc
    code = ("import gpufairq, gpufairq.engine as e, gpufairq.mqfq as m, gpufairq.cli as c;"
            "print(e.LIBGFQ); print(m.__file__); print(c.run_simulation is e.run_simulation);"
            "print(gpufairq.Simulation is e.Simulation)")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([SHIM, ROOT, src]), GFQ_REF_SRC=src)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         check=True).stdout.split("\n")
    assert out[0].endswith("libgfq.so")
    assert out[1].startswith(os.path.join(src, "gpufairq"))
    assert out[2] == "True" and out[3] == "True"
