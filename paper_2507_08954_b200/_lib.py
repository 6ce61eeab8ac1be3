"""ctypes binding of libgfq.so (include/gfq.h).

The CUDA engine is the only implementation of the simulation path in this
package: if the shared library is missing or cannot be loaded this module
raises instead of falling back to anything else.  Build it with
``python -m paper_2507_08954_b200.build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import _abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GFQ_LIB") or os.path.join(HERE, "libgfq.so")

_lib = None
_lock = threading.Lock()

_P = C.POINTER
_SIGS = {
    "gfq_last_error": (C.c_char_p, []),
    "gfq_abi_version": (C.c_int, []),
    "gfq_create": (C.c_int, [C.c_int, _P(C.c_void_p)]),
    "gfq_destroy": (C.c_int, [C.c_void_p]),
    "gfq_upload_traces": (C.c_int, [C.c_void_p, _P(C.c_double), _P(C.c_int32), _P(C.c_int64),
                                    _P(C.c_int32), C.c_int32]),
    "gfq_upload_flowtabs": (C.c_int, [C.c_void_p] + [_P(C.c_double)] * 5 +
                            [_P(C.c_int32), _P(C.c_int64), C.c_int32]),
    "gfq_upload_device_cfgs": (C.c_int, [C.c_void_p, _P(_abi.DeviceCfg), C.c_int32]),
    "gfq_upload_execs": (C.c_int, [C.c_void_p, _P(C.c_double), C.c_int64]),
    "gfq_prepare": (C.c_int, [C.c_void_p, _P(_abi.Sim), C.c_int32, _P(_abi.LaunchCfg)]),
    "gfq_sim_offsets": (C.c_int, [C.c_void_p, _P(C.c_int64), _P(C.c_int64)]),
    "gfq_launch": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gfq_synchronize": (C.c_int, [C.c_void_p]),
    "gfq_last_kernel_ms": (C.c_int, [C.c_void_p, _P(C.c_float), _P(C.c_float)]),
    "gfq_batch_info": (C.c_int, [C.c_void_p, _P(C.c_int32), C.c_int32]),
    "gfq_generate_traces": (C.c_int, [C.c_void_p, C.c_int32, _P(C.c_int32), _P(C.c_double),
                                      _P(C.c_int32), _P(C.c_double), _P(C.c_uint64),
                                      _P(C.c_uint8), _P(C.c_int64)]),
    "gfq_download_traces": (C.c_int, [C.c_void_p, _P(C.c_double), _P(C.c_int32), C.c_int64]),
    "gfq_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "gfq_nccl_comm_init": (C.c_int, [_P(C.c_void_p), C.c_int32, C.c_char_p, C.c_int32]),
    "gfq_nccl_comm_destroy": (C.c_int, [C.c_void_p]),
    "gfq_reduce_nccl": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gfq_kernel_times": (C.c_int, [C.c_void_p, _P(C.c_float), _P(C.c_float), C.c_int32,
                                   _P(C.c_int32)]),
    "gfq_output_info": (C.c_int, [C.c_void_p, C.c_int32, _P(C.c_int64), _P(C.c_int32)]),
    "gfq_output_copy": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64]),
    "gfq_output_device_ptr": (C.c_int, [C.c_void_p, C.c_int32, _P(C.c_void_p)]),
    "gfq_fairness": (C.c_int, [C.c_void_p, C.c_double, _P(C.c_int32), _P(C.c_double), C.c_int64]),
    "gfq_run": (C.c_int, [C.c_void_p, _P(_abi.Sim), C.c_int32, _P(_abi.LaunchCfg)]),
}
EXPORTS = tuple(_SIGS)


class EngineError(RuntimeError):
    """Nonzero status from libgfq (GFQ_ERUNTIME / GFQ_ECUDA)."""


def lib() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build the CUDA engine first "
                    "(python -m paper_2507_08954_b200.build); there is no CPU fallback")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            if L.gfq_abi_version() != _abi.ABI_VERSION:
                raise ImportError("libgfq.so ABI version mismatch; rebuild it")
            _lib = L
    return _lib


def check(rc: int) -> None:
    """Map a GFQ_* status to the reference's exception types (cli.py:260-267)."""
    if rc == _abi.GFQ_OK:
        return
    msg = lib().gfq_last_error().decode(errors="replace")
    if rc == _abi.GFQ_EINVAL:
        raise ValueError(msg)
    if rc == _abi.GFQ_ENOMEM:
        raise MemoryError(msg)
    raise EngineError(msg)
