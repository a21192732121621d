"""ctypes binding of ``librcp_b200.so`` (the C ABI in ``include/rcp_b200.h``).

The shared library is built in-tree by ``paper_1710_00125_b200.build`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no fallback: if the
library is missing or fails to load, every entry point raises
:class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_NAME = "librcp_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

# Status codes (include/rcp_b200.h).
RCP_OK = 0
RCP_ERR_INVALID_ARG = 1
RCP_ERR_NOT_SYMMETRIC = 2
RCP_ERR_NONFINITE_INPUT = 3
RCP_ERR_NUMERICAL = 4
RCP_ERR_NEED_NORMALS = 5
RCP_ERR_CUDA = 6
RCP_ERR_WORKSPACE = 7
RCP_ERR_UNSUPPORTED = 8

RCP_NUM_ZERO_1X1 = 1
RCP_NUM_SINGULAR_2X2 = 2
RCP_NUM_NONFINITE = 3
RCP_NUM_DET_BOUND = 4

# Every symbol include/rcp_b200.h declares (checked by tests/test_native_abi.py).
EXPORTED_SYMBOLS = (
    "rcp_workspace_bytes",
    "rcp_factor",
    "rcp_factor_host_l",
    "rcp_factor_host",
    "rcp_factor_diag",
    "rcp_solve",
    "rcp_solve_workspace_bytes",
    "rcp_reconstruct",
    "rcp_version",
    "rcp_lower_to_host",
    "rcp_batched_workspace_bytes",
    "rcp_factor_batched",
    "rcp_solve_batched",
    "rcp_factor_dist",
    "rcp_worker_workspace_bytes",
    "rcp_dist_prepare",
    "rcp_schur_worker",
    "rcp_device_alloc",
    "rcp_device_free",
    "rcp_ipc_export",
    "rcp_ipc_import",
    "rcp_ipc_close",
    "rcp_schur_tile_plan",
)


class NativeUnavailable(RuntimeError):
    """The CUDA library could not be loaded (no CPU fallback exists)."""


class RcpConfig(ctypes.Structure):
    _fields_ = [("p", ctypes.c_int32), ("b", ctypes.c_int32), ("q", ctypes.c_int32), ("robust_r", ctypes.c_int32),
                ("strategy", ctypes.c_int32)]


class RcpStats(ctypes.Structure):
    _fields_ = [
        ("rho_cheap", ctypes.c_double),
        ("max_multiplier", ctypes.c_double),
        ("amax", ctypes.c_double),
        ("dmax", ctypes.c_double),
        ("recompute_count", ctypes.c_int64),
        ("n_panels", ctypes.c_int64),
        ("n_steps", ctypes.c_int64),
        ("n_2x2", ctypes.c_int64),
        ("deficient_from", ctypes.c_int64),
        ("num_kind", ctypes.c_int32),
        ("num_step", ctypes.c_int32),
        ("t_factor_ms", ctypes.c_double),
        ("t_schur_ms", ctypes.c_double),
        ("t_panel_ms", ctypes.c_double),
        ("schur_flops", ctypes.c_double),
        ("n_launches", ctypes.c_int64),
        ("mults", ctypes.c_int64),
        ("adds", ctypes.c_int64),
        ("divs", ctypes.c_int64),
        ("comps", ctypes.c_int64),
        ("panel_prof_ms", ctypes.c_double * 16),
        ("message", ctypes.c_char * 160),
    ]


class RcpDiag(ctypes.Structure):
    _fields_ = [
        ("track_full", ctypes.c_int32),
        ("audit", ctypes.c_int32),
        ("snapshots", ctypes.c_void_p),
        ("drift", ctypes.c_void_p),
        ("omega_orig", ctypes.c_void_p),
        ("cap", ctypes.c_int64),
        ("n_snapshots", ctypes.c_int64),
        ("n_drift", ctypes.c_int64),
    ]


class RcpBatchStats(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int32),
        ("num_kind", ctypes.c_int32),
        ("num_step", ctypes.c_int32),
        ("recompute_count", ctypes.c_int32),
        ("deficient_from", ctypes.c_int32),
        ("n_2x2", ctypes.c_int32),
        ("n_steps", ctypes.c_int32),
        ("n_panels", ctypes.c_int32),
        ("rho_cheap", ctypes.c_double),
        ("max_multiplier", ctypes.c_double),
        ("amax", ctypes.c_double),
        ("dmax", ctypes.c_double),
        ("mults", ctypes.c_int64),
        ("adds", ctypes.c_int64),
        ("divs", ctypes.c_int64),
        ("comps", ctypes.c_int64),
    ]


# numpy view of an array of rcp_batch_stats (same layout, 96 bytes)
BATCH_STATS_DTYPE = [
    ("status", "<i4"), ("num_kind", "<i4"), ("num_step", "<i4"), ("recompute_count", "<i4"),
    ("deficient_from", "<i4"), ("n_2x2", "<i4"), ("n_steps", "<i4"), ("n_panels", "<i4"),
    ("rho_cheap", "<f8"), ("max_multiplier", "<f8"), ("amax", "<f8"), ("dmax", "<f8"),
    ("mults", "<i8"), ("adds", "<i8"), ("divs", "<i8"), ("comps", "<i8"),
]


DRAW_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                           ctypes.POINTER(ctypes.c_double))

_lib = None


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the ctypes handle of the CUDA library."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    if path is None and os.environ.get("RCP_B200_LIB"):
        path = os.environ["RCP_B200_LIB"]  # alternative build (experiments)
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise NativeUnavailable(
            f"{p} not found: build it with `python -m paper_1710_00125_b200.build` "
            "(nvcc, sm_100a); there is no CPU fallback")
    try:
        lib = ctypes.CDLL(str(p))
    except OSError as exc:  # pragma: no cover - environment dependent
        raise NativeUnavailable(f"failed to load {p}: {exc}") from exc
    vp, i64, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t
    lib.rcp_workspace_bytes.argtypes = [i64, ctypes.POINTER(RcpConfig)]
    lib.rcp_workspace_bytes.restype = sz
    lib.rcp_factor.argtypes = [ctypes.POINTER(RcpConfig), i64, vp, i64, vp, DRAW_FN, vp, vp, sz,
                               vp, vp, vp, vp, vp, vp, vp, ctypes.POINTER(RcpStats), vp]
    lib.rcp_factor.restype = ctypes.c_int
    lib.rcp_factor_host_l.argtypes = [ctypes.POINTER(RcpConfig), i64, vp, i64, vp, DRAW_FN, vp, vp, sz,
                                      vp, vp, vp, vp, vp, vp, vp, ctypes.POINTER(RcpStats), vp, vp]
    lib.rcp_factor_host_l.restype = ctypes.c_int
    lib.rcp_factor_host.argtypes = [ctypes.POINTER(RcpConfig), i64, vp, i64, vp, DRAW_FN, vp, vp, sz,
                                    vp, vp, vp, vp, vp, vp, vp, ctypes.POINTER(RcpStats), vp, vp]
    lib.rcp_factor_host.restype = ctypes.c_int
    lib.rcp_factor_diag.argtypes = [ctypes.POINTER(RcpConfig), i64, vp, i64, vp, DRAW_FN, vp, vp, sz,
                                    vp, vp, vp, vp, vp, vp, vp, ctypes.POINTER(RcpStats), ctypes.POINTER(RcpDiag), vp]
    lib.rcp_factor_diag.restype = ctypes.c_int
    lib.rcp_solve.argtypes = [i64, vp, vp, vp, vp, vp, i64, vp, vp, vp, sz, ctypes.POINTER(ctypes.c_int32), vp]
    lib.rcp_solve.restype = ctypes.c_int
    lib.rcp_solve_workspace_bytes.argtypes = [i64, i64]
    lib.rcp_solve_workspace_bytes.restype = sz
    lib.rcp_reconstruct.argtypes = [i64, vp, vp, vp, vp, vp, vp]
    lib.rcp_reconstruct.restype = ctypes.c_int
    lib.rcp_batched_workspace_bytes.argtypes = [i64, ctypes.POINTER(RcpConfig)]
    lib.rcp_batched_workspace_bytes.restype = sz
    lib.rcp_factor_batched.argtypes = [ctypes.POINTER(RcpConfig), i64, i64, vp, i64, i64, vp, i64, vp, sz,
                                       vp, vp, vp, vp, vp, vp, vp]
    lib.rcp_factor_batched.restype = ctypes.c_int
    lib.rcp_solve_batched.argtypes = [i64, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    lib.rcp_solve_batched.restype = ctypes.c_int
    lib.rcp_factor_dist.argtypes = [ctypes.POINTER(RcpConfig), i64, vp, i64, vp, DRAW_FN, vp, vp, sz,
                                    vp, vp, vp, vp, vp, vp, vp, ctypes.POINTER(RcpStats), ctypes.c_int, ctypes.c_int,
                                    vp, sz, vp]
    lib.rcp_factor_dist.restype = ctypes.c_int
    lib.rcp_worker_workspace_bytes.argtypes = [i64, ctypes.POINTER(RcpConfig)]
    lib.rcp_worker_workspace_bytes.restype = sz
    lib.rcp_dist_prepare.argtypes = [i64, ctypes.POINTER(RcpConfig), vp, vp]
    lib.rcp_dist_prepare.restype = ctypes.c_int
    lib.rcp_schur_worker.argtypes = [ctypes.POINTER(RcpConfig), i64, ctypes.c_int, ctypes.c_int, vp, vp, sz, vp]
    lib.rcp_schur_worker.restype = ctypes.c_int
    lib.rcp_lower_to_host.argtypes = [i64, vp, vp, vp]
    lib.rcp_lower_to_host.restype = ctypes.c_int
    lib.rcp_device_alloc.argtypes = [sz, ctypes.POINTER(ctypes.c_void_p)]
    lib.rcp_device_alloc.restype = ctypes.c_int
    lib.rcp_device_free.argtypes = [vp]
    lib.rcp_device_free.restype = ctypes.c_int
    lib.rcp_ipc_export.argtypes = [vp, vp]
    lib.rcp_ipc_export.restype = ctypes.c_int
    lib.rcp_ipc_import.argtypes = [vp, ctypes.POINTER(ctypes.c_void_p)]
    lib.rcp_ipc_import.restype = ctypes.c_int
    lib.rcp_ipc_close.argtypes = [vp]
    lib.rcp_ipc_close.restype = ctypes.c_int
    lib.rcp_schur_tile_plan.argtypes = [i64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, vp, vp,
                                        vp, i64]
    lib.rcp_schur_tile_plan.restype = i64
    lib.rcp_version.argtypes = []
    lib.rcp_version.restype = ctypes.c_char_p
    _lib = lib
    return lib
