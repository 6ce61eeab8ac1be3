"""Where the UNMODIFIED reference lives for the drop-in tests (test
infrastructure): baseline/_ref (tools/install_ref.sh; travels to the GPU
box) or, in the build container, /root/reference/pkg."""

from __future__ import annotations

import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "refshim")


def locate():
    """(src dir holding gpufairq/, reference tests dir) or None."""
    for src, tests in ((os.path.join(ROOT, "baseline", "_ref"),
                        os.path.join(ROOT, "baseline", "_ref", "refpkg", "tests")),
                       ("/root/reference/pkg/src", "/root/reference/pkg/tests")):
        if os.path.isfile(os.path.join(src, "gpufairq", "__init__.py")) and os.path.isdir(tests):
            return src, tests
    return None
