"""ctypes binding of libucp_b200.so (the C ABI in include/ucp_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2406_18820_b200._build``). There is no fallback: if the
library or a CUDA device is missing, every compute entry point raises
:class:`NativeUnavailableError`.
"""

from __future__ import annotations

import ctypes
import os

from . import _build
from ._errors import NativeUnavailableError

LIB_NAME = "libucp_b200.so"
LIB_PATH = os.environ.get("UCP_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), LIB_NAME)  # env override: kernel A/B experiments

# exported symbols declared in include/ucp_b200.h
EXPORTS = ("ucp_version", "ucp_build_id", "ucp_status_reset", "ucp_runtile_scan", "ucp_convert_gather",
           "ucp_load_scatter",
           "ucp_reshard_fused", "ucp_gen_state", "ucp_adam_step", "ucp_compare", "ucp_peek",
           "ucp_dev_alloc", "ucp_dev_free", "ucp_ipc_export", "ucp_ipc_open", "ucp_ipc_close")
ABI_VERSION = 3

_lib = None

_c = ctypes
_P = _c.c_void_p
_SIGS = {
    "ucp_version": (_c.c_int, []),
    "ucp_build_id": (_c.c_char_p, []),
    "ucp_status_reset": (_c.c_int, [_P, _P]),
    "ucp_runtile_scan": (_c.c_int, [_P, _P, _P]),
    "ucp_convert_gather": (_c.c_int, [_P, _c.c_int64, _P, _P, _P, _P, _P, _P, _P]),
    "ucp_load_scatter": (_c.c_int, [_P, _c.c_int64, _P, _P, _P, _P, _P, _P, _P]),
    "ucp_reshard_fused": (_c.c_int, [_P, _c.c_int64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "ucp_adam_step": (_c.c_int, [_P, _P, _P, _c.c_uint64, _c.c_uint64, _c.c_uint64] +
                      [_c.c_double] * 8 + [_P]),
    "ucp_gen_state": (_c.c_int, [_c.c_uint64, _c.c_uint64, _c.c_uint64, _c.c_int, _P, _P]),
    "ucp_compare": (_c.c_int, [_P, _P, _c.c_uint64, _P, _P]),
    "ucp_peek": (_c.c_int, [_P, _P, _c.c_uint64]),
    "ucp_dev_alloc": (_c.c_int, [_c.c_uint64, _P]),
    "ucp_dev_free": (_c.c_int, [_P]),
    "ucp_ipc_export": (_c.c_int, [_P, _P]),
    "ucp_ipc_open": (_c.c_int, [_P, _P]),
    "ucp_ipc_close": (_c.c_int, [_P]),
}


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load and type the library (no CUDA device needed)."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailableError(
            f"{path} is missing; build it with __graft_entry__.build() (no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.ucp_version() != ABI_VERSION:
        raise NativeUnavailableError(f"{path}: ABI {lib.ucp_version()} != {ABI_VERSION}")
    _check_build_id(path, lib.ucp_build_id(), _build.kernel_id())
    if path == LIB_PATH:
        _lib = lib
    return lib


def build_id(lib_handle=None) -> str:
    """The build id baked into the loaded libucp_b200.so."""
    raw = (lib_handle or lib()).ucp_build_id().decode()
    return raw.split(":", 1)[1]


def _check_build_id(path: str, raw: bytes, want: str | None) -> None:
    """Refuse a library not built from the sources next to it (a stale or
    foreign .so). Sources absent (an installed copy): nothing to check."""
    got = raw.decode().split(":", 1)[-1]
    if want is not None and got != want:
        raise NativeUnavailableError(
            f"{path} was built from other sources (build id {got}, sources {want}); "
            "rebuild with __graft_entry__.build()")


def lib() -> ctypes.CDLL:
    return load_library()


# --------------------------------------------------------------------------- comm library

COMM_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libucp_b200_comm.so")
COMM_EXPORTS = ("ucp_comm_version", "ucp_comm_build_id", "ucp_comm_unique_id", "ucp_comm_init", "ucp_alltoallv",
                "ucp_comm_destroy")
_comm = None
_COMM_SIGS = {
    "ucp_comm_version": (_c.c_int, []),
    "ucp_comm_build_id": (_c.c_char_p, []),
    "ucp_comm_unique_id": (_c.c_int, [_P]),
    "ucp_comm_init": (_c.c_int, [_c.c_int, _c.c_int, _P, _P]),
    "ucp_alltoallv": (_c.c_int, [_P, _P, _P, _P, _P, _P]),
    "ucp_comm_destroy": (_c.c_int, [_P]),
}


def comm_lib() -> ctypes.CDLL:
    """libucp_b200_comm.so (NCCL all-to-all-v of the rank-homed exchange)."""
    global _comm
    if _comm is None:
        if not os.path.exists(COMM_PATH):
            raise NativeUnavailableError(f"{COMM_PATH} is missing; run __graft_entry__.build()")
        lib = ctypes.CDLL(COMM_PATH)
        for name, (res, args) in _COMM_SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _check_build_id(COMM_PATH, lib.ucp_comm_build_id(), _build.comm_id())
        _comm = lib
    return _comm
