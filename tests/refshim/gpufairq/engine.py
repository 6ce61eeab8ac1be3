"""``gpufairq.engine`` served by the CUDA engine (see refshim/gpufairq/__init__.py).

Same public names as the reference module (engine.py:20-23,26-43,46,214):
event kinds, AuditLog, SimResult, Simulation, run_simulation.  Every call
is counted in ``CALLS`` (and, when ``GFQ_SHIM_LOG`` names a file, appended
there) so a test can prove the reference's suite ran through libgfq.
"""

import os

import paper_2507_08954_b200.engine as _gpu
from paper_2507_08954_b200._lib import lib as _lib

ARRIVAL, COMPLETION, MONITOR_TICK, QUEUE_EXPIRY = (_gpu.ARRIVAL, _gpu.COMPLETION,
                                                   _gpu.MONITOR_TICK, _gpu.QUEUE_EXPIRY)
AuditLog = _gpu.AuditLog
SimResult = _gpu.SimResult
LIBGFQ = _lib()._name                      # the loaded libgfq.so (raises if it is missing)
CALLS = {"run_simulation": 0, "Simulation": 0}


def _count(kind: str) -> None:
    CALLS[kind] += 1
    log = os.environ.get("GFQ_SHIM_LOG")
    if log:
        with open(log, "a") as fh:
            fh.write(kind + "\n")


class Simulation(_gpu.Simulation):
    __doc__ = _gpu.Simulation.__doc__

    def __init__(self, *args, **kw):
        super().__init__(*args, **kw)
        _count("Simulation")


def run_simulation(trace, profiles, policy, devices, tau_includes_overheads=False):
    _count("run_simulation")
    return _gpu.run_simulation(trace, profiles, policy, devices, tau_includes_overheads)
