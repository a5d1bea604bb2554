"""ctypes binding of libcfgpu.so (include/cfgpu.h).

The product path is CUDA only: if the library or a CUDA device is missing
every entry point raises -- there is no CPU fallback anywhere in this
package.  Device memory and streams come from PyTorch (plumbing only); the
compute is the hand-written sm_100a kernels behind the C ABI.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CF_LIB", os.path.join(_HERE, "libcfgpu.so"))  # CF_LIB: tuning experiments only

CF_OK = 0
CF_BREAKDOWN = 1
CF_NOT_CONVERGED = 2
CF_EINVAL = -1
CF_ECUDA = -2
CF_ENOMEM = -3
CF_EIO = -4

ORDER_CSR = 0
ORDER_SYM = 1

PRECOND_NONE = 0
PRECOND_JACOBI = 1
PRECOND_DIC = 2
CG_FORM_TWO = 1  # include/cfgpu.h CF_CG_FORM_*
CG_FORM_SPASS = 2

_lib = None

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double
_pd = ctypes.POINTER(ctypes.c_double)
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pf = ctypes.POINTER(ctypes.c_float)

_SIGNATURES = {
    "cf_last_error": ([], ctypes.c_char_p),
    "cf_version": ([], _int),
    "cf_device_sms": ([], _int),
    "cf_dot": ([_vp, _vp, _i64, _pd, _vp], _int),
    "cf_axpy": ([_vp, _dbl, _vp, _i64, _vp], _int),
    "cf_add": ([_vp, _vp, _vp, _i64, _vp], _int),
    "cf_scale": ([_dbl, _vp, _vp, _i64, _vp], _int),
    "cf_mul": ([_vp, _vp, _vp, _i64, _vp], _int),
    "cf_max_abs": ([_vp, _i64, _pd, _vp], _int),
    "cf_csr_spmv": ([_i64, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    "cf_sym_spmv": ([_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    "cf_stencil7_apply": ([_int, _int, _int, _dbl, _int, _vp, _vp, _vp], _int),
    "cf_level_schedule": ([_i64, _vp, _vp, _vp, _vp], _int),
    "cf_dic_factor": ([_i64, _vp, _vp, _vp, _vp, _vp, _vp, _int, _vp, _vp, _vp], _int),
    "cf_dic_apply": ([_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _int, _vp, _vp, _vp, _vp], _int),
    "cf_dic_divide": ([_i64, _vp, _vp, _vp, _vp], _int),
    "cf_cg_set_dic": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _int], _int),
    "cf_cg_create": ([ctypes.POINTER(_vp), _int, _int, _int, _dbl, _int, _vp], _int),
    "cf_cg_destroy": ([_vp], _int),
    "cf_cg_solve": ([_vp, _vp, _vp, _vp, _dbl, _i64, _int, _vp, _pi64, _pd, _vp], _int),
    "cf_cg_last_loop_ms": ([_vp, _pf], _int),
    "cf_cg_last_form": ([_vp, ctypes.POINTER(_int), _pi64], _int),
    "cf_nccl_unique_id": ([_vp], _int),
    "cf_dcg_create": ([ctypes.POINTER(_vp), _int, _int, _int, _dbl, _int, _int, _int, _vp, _int, _vp, _int, _int,
                       _vp], _int),
    "cf_dcg_destroy": ([_vp], _int),
    "cf_dcg_solve": ([_vp, _vp, _vp, _dbl, _i64, _int, _pi64, _pd, _vp], _int),
    "cf_dcg_last_loop_ms": ([_vp, _pf], _int),
    "cf_pcg_create": ([ctypes.POINTER(_vp), _int, _int, _int, _dbl, _int, _int, _int, _int, _vp, _vp], _int),
    "cf_pcg_export_size": ([], _int),
    "cf_pcg_export": ([_vp, _vp, _int], _int),
    "cf_pcg_import": ([_vp, _vp, _int], _int),
    "cf_pcg_destroy": ([_vp], _int),
    "cf_pcg_solve": ([_vp, _vp, _vp, _dbl, _i64, _int, _pi64, _pd, _vp], _int),
    "cf_pcg_last_loop_ms": ([_vp, _pf], _int),
    "cf_pcg_form": ([_vp, ctypes.POINTER(_int)], _int),
    "cf_pcg_debug_io": ([_vp, _int, _int, _vp, _i64], _int),
    "cf_forces_bc": ([_vp, _vp, _vp, _int, _int, _int, _int, _dbl, _int, _vp], _int),
    "cf_advect": ([_vp, _vp, _vp, _vp, _vp, _vp, _int, _int, _int, _int, _dbl, _dbl, _vp], _int),
    "cf_divergence": ([_vp, _vp, _vp, _int, _int, _int, _int, _dbl, _dbl, _vp, _pd, _vp], _int),
    "cf_pressure_correct": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp, _int, _int, _int, _int, _dbl, _dbl,
                             _pd, _vp], _int),
    "cf_forces_bc_slab": ([_vp, _vp, _vp] + [_int] * 9 + [_dbl, _int, _vp], _int),
    "cf_advect_slab": ([_vp] * 6 + [_int] * 9 + [_dbl, _dbl, _vp], _int),
    "cf_divergence_slab": ([_vp] * 3 + [_int] * 9 + [_dbl, _dbl, _vp, _pd, _vp], _int),
    "cf_pressure_correct_slab": ([_vp] * 7 + [_int] * 9 + [_dbl, _dbl, _pd, _vp], _int),
    "cf_helmholtz": ([_int, _int, _vp, _vp, _int, _int, _int, _int, _dbl, _dbl, _int, _int, _vp], _int),
    "cf_diffuse": ([_vp, _vp, _vp, _vp, _vp, _vp, _int, _int, _int, _int, _dbl, _dbl, _int, _int, _vp], _int),
    "cf_diffuse_slab": ([_vp] * 6 + [_int] * 9 + [_dbl, _dbl, _int, _int, _vp], _int),
    "cf_sample_velocity":([_vp, _vp, _vp, _int, _int, _int, _int, _dbl, _dbl, _dbl, _dbl, _pd, _vp],
                           _int),
    "cf_snapshot_cells": ([_vp, _vp, _vp, _vp, _int, _int, _int, _int, _int, _int, _vp, _vp], _int),
    "cf_format_double": ([_dbl, ctypes.c_char_p, _int], _int),
    "cf_snapshot_write": ([ctypes.c_char_p, _vp, _int, _int, _int, _dbl, _int], _int),
    "cf_csv_write_columns": ([ctypes.c_char_p, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _int], _int),
}

EXPORTED = tuple(_SIGNATURES)


def open_library(path: str = LIB_PATH):
    """dlopen libcfgpu.so and declare every prototype (no CUDA call is made)."""
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build the CUDA extension first (python -c "
            "'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


def load_library():
    """The loaded library; raises unless a CUDA device is visible."""
    global _lib
    if _lib is None:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_2504_03697_b200 needs a CUDA (sm_100a) device; "
                               "no CPU fallback exists")
        torch.cuda.init()
        _lib = open_library()
    return _lib


_host = None


def host_library():
    """The library for its host-only entry points (level schedule, snapshot
    CSV formatting): those make no CUDA call, so no device is required."""
    global _host
    if _lib is not None:
        return _lib
    if _host is None:
        _host = open_library()
    return _host


def last_error() -> str:
    return (_lib if _lib is not None else host_library()).cf_last_error().decode(errors="replace")


def check(rc: int, what: str) -> int:
    if rc < 0:
        msg = f"{what}: {last_error()}"
        if rc == CF_EINVAL:
            raise ValueError(msg)
        if rc == CF_ENOMEM:
            raise MemoryError(msg)
        if rc == CF_EIO:
            raise OSError(msg)
        raise RuntimeError(msg)
    return rc


def stream() -> int:
    import torch

    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int:
    """Device pointer of a CUDA float64/int32 tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    return t.data_ptr()


def dbl_out():
    return ctypes.c_double()


def byref(x):
    return ctypes.byref(x)


def np_ptr(a: np.ndarray):
    return a.ctypes.data_as(_pd)
