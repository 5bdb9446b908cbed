"""ctypes binding of libsht.so (include/sht.h).

The library is built in-tree by ``_build.build()`` (``__graft_entry__.build()``
calls it) and loaded from this package directory.  There is no fallback: if
the shared library is missing the product raises instead of computing
anything on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import ConfigurationError, ProtocolError

# SHT_LIB overrides the library for A/B timing of two builds (tools/); the
# default is the in-tree build
LIB_PATH = Path(os.environ.get("SHT_LIB") or Path(__file__).resolve().parent / "libsht.so")

SHT_OK = 0
SHT_ERR_CONFIG = 1
SHT_ERR_CUDA = 2
SHT_ERR_COMM = 3
SHT_FLAG_RECOMPUTE_LEGENDRE = 1
SHT_FLAG_PROFILE_PHASES = 2

# every symbol include/sht.h declares (checked by tests/test_boundary.py)
EXPORTS = (
    "sht_version", "sht_plan_create", "sht_inv_trans", "sht_dir_trans", "sht_local_layout",
    "sht_phase_ms", "sht_phase_ms_avg", "sht_work", "sht_kernel_launches", "sht_transport", "sht_nccl_get_unique_id", "sht_plan_destroy", "sht_plan_close", "sht_wait", "sht_last_error",
    "sht_plan_validate", "sht_gauss_nodes", "sht_partition", "sht_alltoall_rows", "sht_alltoall_order", "sht_fft_plan_info",
    "sht_plan_set_gp_layout", "sht_gp_layout", "sht_inv_trans_gp", "sht_dir_trans_gp", "sht_gp_bands",
    "sht_halo_create", "sht_halo_exchange", "sht_halo_stencil_step", "sht_halo_counts", "sht_halo_destroy",
)

_lib = None

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
f32p = C.POINTER(C.c_float)


def load() -> C.CDLL:
    """Open libsht.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    lib = C.CDLL(str(LIB_PATH))
    lib.sht_version.restype = C.c_int
    lib.sht_last_error.restype = C.c_char_p
    lib.sht_plan_create.argtypes = [C.c_int, C.c_int, i32p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                    C.POINTER(C.c_void_p)]
    lib.sht_inv_trans.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.sht_dir_trans.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.sht_local_layout.argtypes = [C.c_void_p, i64p, i64p, i32p, i32p, i32p, i32p]
    lib.sht_phase_ms.argtypes = [C.c_void_p, f32p, C.c_int]
    lib.sht_phase_ms_avg.argtypes = [C.c_void_p, C.c_int, f32p, C.c_int]
    lib.sht_work.argtypes = [C.c_void_p, f64p, f64p, f64p]
    lib.sht_kernel_launches.argtypes = [C.c_void_p, i32p]
    lib.sht_transport.argtypes = [C.c_void_p, i32p]
    lib.sht_nccl_get_unique_id.argtypes = [C.c_void_p]
    lib.sht_plan_destroy.argtypes = [C.c_void_p]
    lib.sht_plan_destroy.restype = None
    lib.sht_plan_close.argtypes = [C.c_void_p]
    lib.sht_wait.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
    lib.sht_plan_validate.argtypes = [C.c_int, C.c_int, i32p, C.c_int, C.c_int]
    lib.sht_gauss_nodes.argtypes = [C.c_int, f64p, f64p, f64p]
    lib.sht_partition.argtypes = [C.c_int, C.c_int, i32p, C.c_int, i32p, i32p]
    lib.sht_alltoall_rows.argtypes = [C.c_int, C.c_int, i32p, C.c_int, i64p]
    lib.sht_alltoall_order.argtypes = [C.c_int, C.c_int, i32p]
    lib.sht_fft_plan_info.argtypes = [C.c_int, i32p, i32p, i32p, i32p]
    lib.sht_plan_set_gp_layout.argtypes = [C.c_void_p, C.c_int, C.c_int]
    lib.sht_gp_layout.argtypes = [C.c_void_p, i64p, i32p, i32p, i32p, i32p]
    lib.sht_inv_trans_gp.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.sht_dir_trans_gp.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.sht_gp_bands.argtypes = [C.c_int, C.c_int, i32p, C.c_int, i32p]
    lib.sht_halo_create.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_int64, i64p, i64p, i64p, i64p,
                                    C.c_int, i32p, i64p, i64p, i64p, C.POINTER(C.c_void_p)]
    lib.sht_halo_exchange.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.sht_halo_stencil_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.sht_halo_counts.argtypes = [C.c_void_p, i64p, i64p]
    lib.sht_halo_destroy.argtypes = [C.c_void_p]
    lib.sht_halo_destroy.restype = None
    for name in EXPORTS:
        if name not in ("sht_version", "sht_last_error", "sht_plan_destroy", "sht_halo_destroy"):
            getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a C-ABI status onto the reference's error classes (errors.py:9-39)."""
    if rc == SHT_OK:
        return
    msg = (load().sht_last_error() or b"").decode(errors="replace")
    if rc == SHT_ERR_CONFIG:
        raise ConfigurationError(msg)
    if rc == SHT_ERR_COMM:
        raise ProtocolError(msg)
    raise RuntimeError(f"libsht CUDA error: {msg}")
