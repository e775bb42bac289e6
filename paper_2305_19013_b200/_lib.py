"""ctypes binding of libekcg_b200.so (C ABI declared in include/ekcg_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing, the
product path raises.  Every pointer argument is a raw device address (int).
"""

from __future__ import annotations

import ctypes
from ctypes import c_double, c_int, c_longlong, c_uint64, c_void_p
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libekcg_b200.so"
_lib = None

# name -> (restype, argtypes)
SIGNATURES = {
    "ekcg_split": (c_int, [c_void_p, c_void_p, c_void_p, c_longlong, c_int, c_int, c_void_p, c_void_p]),
    "ekcg_split_axpy": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_double, c_void_p,
                                c_longlong, c_int, c_int, c_void_p, c_void_p]),
    "ekcg_axpy_cols": (c_int, [c_void_p, c_int, c_void_p, c_int, c_void_p, c_double, c_longlong, c_int, c_void_p,
                               c_void_p]),
    "ekcg_spmm_csr": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int, c_longlong,
                              c_int, c_void_p, c_void_p]),
    "ekcg_spmm_stencil": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_int, c_int, c_void_p, c_void_p]),
    "ekcg_spmm_csr_kernel": (c_int, [c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int,
                                     c_longlong, c_int, c_void_p, c_void_p]),
    "ekcg_stencil_coefs": (c_int, [c_void_p, c_void_p, c_void_p]),
    "ekcg_spmm_stencil_kernel": (c_int, [c_int, c_void_p, c_void_p, c_int, c_void_p, c_int, c_int, c_void_p,
                                         c_void_p]),
    "ekcg_gram_chunks": (c_int, [c_longlong, c_int, c_int, c_int]),
    "ekcg_gram": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_int, c_int, c_longlong, c_void_p,
                          c_void_p, c_void_p]),
    "ekcg_reduce": (c_int, [c_void_p, c_int, c_longlong, c_void_p, c_void_p, c_void_p]),
    "ekcg_block_update": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_int, c_void_p, c_int,
                                  c_int, c_double, c_double, c_longlong, c_void_p, c_void_p]),
    "ekcg_tri_apply": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_int, c_int, c_longlong, c_void_p, c_void_p]),
    "ekcg_vec_chunks": (c_int, [c_longlong]),
    "ekcg_xr_update": (c_int, [c_void_p, c_int, c_void_p, c_int, c_void_p, c_int, c_void_p, c_void_p,
                               c_longlong, c_void_p, c_void_p, c_void_p]),
    "ekcg_sumsq": (c_int, [c_void_p, c_longlong, c_void_p, c_void_p, c_void_p]),
    "ekcg_block_diag_apply": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int, c_void_p,
                                      c_int, c_longlong, c_int, c_void_p, c_void_p]),
    "ekcg_block_trsv": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p, c_int, c_void_p, c_int,
                                c_int, c_void_p, c_void_p]),
    "ekcg_copy_cols": (c_int, [c_void_p, c_int, c_void_p, c_int, c_longlong, c_int, c_void_p, c_void_p]),
    "ekcg_sub": (c_int, [c_void_p, c_void_p, c_void_p, c_longlong, c_void_p, c_void_p]),
    "ekcg_prechol": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_int, c_double, c_void_p]),
    "ekcg_cholinv": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_int, c_double, c_void_p]),
    "ekcg_cholesky": (c_int, [c_void_p, c_int, c_double, c_void_p, c_void_p, c_void_p]),
    "ekcg_ctrl_bytes": (c_int, []),
    "ekcg_start": (c_int, [c_void_p, c_void_p, c_double, c_void_p, c_void_p]),
    "ekcg_finish": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_void_p, c_void_p]),
    "ekcg_store_norm": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_void_p]),
    "ekcg_launch_count": (c_uint64, []),
    "ekcg_fused_partials": (c_int, [c_longlong, c_int]),
    "ekcg_update_prechol": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_int, c_void_p, c_int, c_int,
                                    c_longlong, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_double, c_void_p]),
    "ekcg_update_vec": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_int, c_int, c_longlong, c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_void_p]),
    "ekcg_stencil_cholinv": (c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                                     c_int, c_double, c_int, c_void_p]),
    "ekcg_cluster_cg": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_longlong, c_int, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p]),
    "ekcg_cluster_solve_fits": (c_int, [c_longlong, c_int, c_int]),
    "ekcg_cluster_solve": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_longlong, c_int, c_int, c_int, c_int,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_longlong, c_void_p, c_void_p,
                                   c_void_p, c_double, c_void_p, c_void_p]),
    "ekcg_stencil_xr": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p, c_int, c_void_p,
                                c_void_p]),
}


class EkcgStencil(ctypes.Structure):
    """Mirror of `EkcgStencil` in include/ekcg_b200.h."""

    _fields_ = [
        ("dim", c_int), ("nx", c_int), ("ny", c_int), ("nz", c_int),
        ("cx", c_double), ("cy", c_double), ("cz", c_double),
        ("kfield", c_void_p),
        ("tx", c_int), ("ty", c_int), ("tz", c_int),
        ("fx", c_int), ("fy", c_int),
        ("kconst", c_double),
        ("row_begin", c_longlong), ("row_end", c_longlong),
        ("kself", c_void_p),
        ("hx", c_void_p), ("hy", c_void_p), ("hz", c_void_p),
        ("coef", c_void_p),
    ]


class KernelError(RuntimeError):
    pass


def library_path() -> Path:
    return _LIB_PATH


def load():
    """Load (building first if stale and nvcc is present) and bind the library."""
    global _lib
    if _lib is not None:
        return _lib
    from . import build as _build
    if _build.needs_build():  # compile in-tree when missing or older than its sources
        _build.build()
    lib = ctypes.CDLL(str(_LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def call(name, *args):
    """Invoke a C-ABI entry; raise KernelError on a nonzero status."""
    rc = getattr(load(), name)(*args)
    if rc != 0:
        kind = "invalid argument" if rc == -1 else "CUDA launch error"
        raise KernelError(f"{name} failed: {kind} ({rc})")
    return rc


def query(name, *args):
    return getattr(load(), name)(*args)
