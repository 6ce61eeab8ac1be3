"""CPU checks of the C-ABI boundary: libgfq.so loads and exports every
entry point include/gfq.h declares; the ctypes mirrors match the header."""

from __future__ import annotations

import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gfq.h")


def header_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(gfq_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_2507_08954_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libgfq.so not built")
    L = C.CDLL(_lib.LIB_PATH)       # loads without a GPU (no CUDA call at load)
    missing = [f for f in header_functions() if not hasattr(L, f)]
    assert not missing, missing
    assert set(header_functions()) == set(_lib.EXPORTS)


def test_struct_layouts_match_header():
    from paper_2507_08954_b200 import _abi
    # sizes implied by include/gfq.h (all members naturally aligned)
    assert C.sizeof(_abi.DeviceCfg) == 7 * 8 + 4 * 4
    assert C.sizeof(_abi.Sim) == 8 * 4 + 3 * 8 + 2 * 4 + 8 + 2 * 4 + 8
    assert C.sizeof(_abi.LaunchCfg) == 4 * 4 + 3 * 8 + 4 * 4 + 2 * 8 + 2 * 4


def test_header_constants_match_abi():
    from paper_2507_08954_b200 import _abi
    src = open(HEADER).read()
    consts = dict(re.findall(r"#define\s+(GFQ_[A-Z_]+)\s+(0x[0-9a-fA-F]+u?|\d+)", src))
    assert int(consts["GFQ_POLICY_SJF"]) == _abi.POLICY_SJF
    assert int(consts["GFQ_ABI_VERSION"]) == _abi.ABI_VERSION
    assert int(consts["GFQ_WANT_EVENTS"].rstrip("u"), 16) == _abi.WANT_EVENTS
    for nm in ("FLOWS_GLOBAL", "CTA", "WARP"):
        assert int(consts["GFQ_FLAG_" + nm].rstrip("u"), 16) == getattr(_abi, "FLAG_" + nm)
    enum = re.search(r"enum gfq_output_id \{(.*?)\};", src, re.S).group(1)
    names = re.findall(r"(GFQ_OUT_[A-Z_]+)", enum)
    assert names.index("GFQ_OUT_HIST") == _abi.OUT_HIST
    assert names.index("GFQ_OUT_COUNT_") == _abi.OUT_COUNT_


def test_no_cpu_fallback_when_library_missing(monkeypatch, tmp_path):
    """The product path fails loudly instead of falling back."""
    from paper_2507_08954_b200 import _lib
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError):
        _lib.lib()
