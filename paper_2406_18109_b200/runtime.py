"""ctypes binding of ``libdk_b200.so`` (declared in ``include/dk_b200.h``).

There is no fallback: if the library is missing or fails to load, importing
the backend raises.  Status codes become the backend's exceptions, which
``GpuSession`` maps onto the reference's own exception types
(``executor.py:28-37``, ``kernels.py:22-35``).
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint8, c_uint64, c_void_p

from .errors import (
    BackendError,
    BoundsError,
    CollectiveError,
    CompileError,
    DeviceOOMError,
    PrivilegeError,
    UnsupportedError,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdk_b200.so")

DK_F64, DK_I32 = 0, 1


class dk_view(ctypes.Structure):
    _fields_ = [
        ("ptr", c_uint64),
        ("rank", c_int32),
        ("dtype", c_int32),
        ("ext", c_int64 * 4),
        ("stride", c_int64 * 4),
    ]


_SIGS = {
    "dk_last_error": (c_char_p, []),
    "dk_version": (c_int, []),
    "dk_init": (c_int, [c_int]),
    "dk_shutdown": (c_int, []),
    "dk_set_stream": (c_int, [c_uint64]),
    "dk_get_stream": (c_int, [POINTER(c_uint64)]),
    "dk_sync": (c_int, []),
    "dk_device_info": (c_int, [POINTER(c_int), POINTER(c_int64), POINTER(c_int64)]),
    "dk_launch_count": (c_int, [POINTER(c_int64)]),
    "dk_graph_begin": (c_int, []),
    "dk_graph_end": (c_int, [POINTER(c_uint64)]),
    "dk_graph_launch": (c_int, [c_uint64]),
    "dk_graph_destroy": (c_int, [c_uint64]),
    "dk_store_create": (c_int, [c_int64, c_int, POINTER(c_int64), c_int]),
    "dk_store_ensure": (c_int, [c_int64, c_int64, c_int64]),
    "dk_store_free": (c_int, [c_int64]),
    "dk_store_ptr": (c_int, [c_int64, POINTER(c_uint64)]),
    "dk_store_bytes_mapped": (c_int, [c_int64, POINTER(c_int64)]),
    "dk_store_upload_rect": (c_int, [c_int64, POINTER(c_int64), POINTER(c_int64), c_void_p]),
    "dk_store_download_rect": (c_int, [c_int64, POINTER(c_int64), POINTER(c_int64), c_void_p]),
    "dk_store_fill": (c_int, [c_int64, c_int64, c_int64, c_double]),
    "dk_pcg64_rejects": (
        c_int,
        [POINTER(c_uint64), POINTER(c_uint64), c_int64, POINTER(c_int64), c_int64, POINTER(c_int64)],
    ),
    "dk_pcg64_fill": (
        c_int,
        [c_int64, POINTER(c_int64), POINTER(c_int64), POINTER(c_uint64), POINTER(c_uint64), c_int, c_double,
         POINTER(c_int64), c_int64],
    ),
    "dk_scratch_alloc": (c_int, [c_int64, POINTER(c_uint64)]),
    "dk_scratch_free": (c_int, [c_uint64]),
    "dk_memset_zero": (c_int, [c_uint64, c_int64]),
    "dk_memcpy_d2h": (c_int, [c_void_p, c_uint64, c_int64]),
    "dk_memcpy_h2d": (c_int, [c_uint64, c_void_p, c_int64]),
    "dk_host_alloc": (c_int, [c_int64, POINTER(c_void_p)]),
    "dk_host_free": (c_int, [c_void_p]),
    "dk_memcpy_d2h_async": (c_int, [c_void_p, c_uint64, c_int64]),
    "dk_stream_new": (c_int, [POINTER(c_uint64)]),
    "dk_event_new": (c_int, [POINTER(c_uint64)]),
    "dk_event_record": (c_int, [c_uint64]),
    "dk_stream_wait_event": (c_int, [c_uint64]),
    "dk_event_sync": (c_int, [c_uint64]),
    "dk_event_elapsed_ms": (c_int, [c_uint64, c_uint64, POINTER(ctypes.c_float)]),
    "dk_kernel_compile": (c_int, [c_char_p, c_int64, POINTER(c_int64)]),
    "dk_kernel_source": (c_int, [c_int64, c_char_p, c_int64, POINTER(c_int64)]),
    "dk_kernel_num_reductions": (c_int, [c_int64, POINTER(c_int)]),
    "dk_jit_stats": (c_int, [POINTER(c_int64), POINTER(c_int64), POINTER(c_int64), POINTER(c_double)]),
    "dk_kernel_codegen": (
        c_int,
        [c_char_p, c_int64, POINTER(dk_view), c_int, POINTER(c_double), c_int, c_char_p, c_int64, POINTER(c_int64)],
    ),
    "dk_launch": (c_int, [c_int64, POINTER(dk_view), c_int, POINTER(c_double), c_int, c_uint64]),
    "dk_accum": (c_int, [POINTER(dk_view), c_uint64, c_int64, c_int64, c_int]),
    "dk_builtin": (c_int, [c_char_p, POINTER(dk_view), c_int, POINTER(c_int32)]),
    "dk_spmv_csr_dot": (c_int, [POINTER(dk_view), c_uint64, c_int64, POINTER(c_int)]),
    "dk_comm_unique_id": (c_int, [POINTER(c_uint8)]),
    "dk_comm_init": (c_int, [c_int, c_int, POINTER(c_uint8)]),
    "dk_comm_destroy": (c_int, []),
    "dk_comm_exchange": (
        c_int,
        [c_int, POINTER(c_int64), POINTER(c_int32), POINTER(c_int32), POINTER(c_int64), POINTER(c_int64)],
    ),
    "dk_comm_allgather_f64": (c_int, [c_uint64, c_uint64, c_int64]),
    "dk_comm_barrier": (c_int, []),
    "dk_p2p_init": (c_int, [POINTER(c_int)]),
    "dk_timestamp": (c_int, [c_uint64, c_int64]),
    "dk_launch_pub": (c_int, [c_int64, POINTER(dk_view), c_int, POINTER(c_double), c_int, c_int64, c_int]),
    "dk_p2p_wait": (c_int, [c_int64, POINTER(c_int32), POINTER(c_uint64)]),
    "dk_launch_pub_ex": (c_int, [c_int64, POINTER(dk_view), c_int, POINTER(c_double), c_int, c_int64, c_int, c_int,
                                 c_int]),
    "dk_p2p_block": (c_int, [c_int64, c_int, c_int, POINTER(c_uint64)]),
    "dk_p2p_wait_fold": (
        c_int,
        [c_int64, POINTER(c_int32), c_int, POINTER(c_uint64), POINTER(c_int64), POINTER(c_int64), POINTER(c_int32)],
    ),
    "dk_dma_send": (c_int, [c_int, POINTER(c_int64), POINTER(c_int32), POINTER(c_int64), POINTER(c_int64)]),
    "dk_dma_recv": (c_int, [c_int, POINTER(c_int64), POINTER(c_int32), POINTER(c_int64), POINTER(c_int64)]),
    "dk_p2p_exchange": (
        c_int,
        [c_int, POINTER(c_int64), POINTER(c_int32), POINTER(c_int32), POINTER(c_int64), POINTER(c_int64)],
    ),
}

# board geometry of the peer-memory reduction exchange (include/dk_b200.h)
P2P_SLOTS = 4
P2P_POINTS = 16
P2P_RED = 32
P2P_MAIL_BYTES = 1 << 20
P2P_FOLDS = 64
# dk_spmv_csr_dot's partials buffer: per-CTA partials, the ticket word, the folded total
SPMV_DOT_PARTS = 4096
SPMV_DOT_TOTAL = SPMV_DOT_PARTS + 1
SPMV_DOT_DOUBLES = SPMV_DOT_PARTS + 2

EXPORTED = tuple(_SIGS)

_ERRS = {
    1: BackendError,
    2: CompileError,
    3: BackendError,
    4: DeviceOOMError,
    5: BackendError,
    6: CollectiveError,
    7: PrivilegeError,
    8: BoundsError,
    9: UnsupportedError,
}

_lib = None


def load(path: str = LIB_PATH):
    """Load the backend library (raises if it is absent -- never falls back)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 backend has no CPU fallback)"
        )
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = _lib.dk_last_error().decode(errors="replace")
        raise _ERRS.get(rc, BackendError)(msg)


def i64s(vals) -> ctypes.Array:
    vals = list(vals)
    return (c_int64 * max(len(vals), 1))(*vals)
