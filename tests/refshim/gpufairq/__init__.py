"""Backend shim: the UNMODIFIED reference package ``gpufairq`` with its
simulation engine swapped for this repo's CUDA engine (test infrastructure).

Put ``tests/refshim`` ahead of the reference on PYTHONPATH.  This package
then loads every reference module (core, device, mqfq, policies, workload,
metrics, config, cli) from the reference's own directory, unchanged, except
``gpufairq.engine``: that resolves to ``refshim/gpufairq/engine.py``, which
re-exports ``paper_2507_08954_b200.engine`` -- the drop-in ``Simulation`` /
``run_simulation`` over libgfq.so.  The reference's own tests and CLI
(``cli.py:16`` imports ``run_simulation`` from ``.engine``) then exercise
the GPU engine with the reference's own Trace / FunctionProfile / policy /
DeviceSet objects.

The reference directory comes from ``GFQ_REF_SRC``, else the first of
``baseline/_ref`` (tools/install_ref.sh) and ``/root/reference/pkg/src``
that holds ``gpufairq``.
"""

import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(_HERE)))


def _real_dir() -> str:
    cands = [os.environ.get("GFQ_REF_SRC", ""), os.path.join(_ROOT, "baseline", "_ref"),
             "/root/reference/pkg/src"]
    for c in cands:
        d = os.path.join(c, "gpufairq") if c else ""
        if d and os.path.isfile(os.path.join(d, "__init__.py")) and os.path.abspath(d) != _HERE:
            return d
    raise ImportError("refshim: the reference gpufairq package was not found "
                      "(run tools/install_ref.sh or set GFQ_REF_SRC)")


REFERENCE_DIR = _real_dir()
__path__ = [_HERE, REFERENCE_DIR]          # shim modules (engine) first, then the reference's

# the reference's own package __init__, run unchanged in this namespace
with open(os.path.join(REFERENCE_DIR, "__init__.py")) as _fh:
    exec(compile(_fh.read(), os.path.join(REFERENCE_DIR, "__init__.py"), "exec"), globals())
