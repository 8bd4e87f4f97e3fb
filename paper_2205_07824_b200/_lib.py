"""ctypes binding of libldgb200.so (the C ABI in include/ldgb200.h).

There is no fallback: if the library is missing or no CUDA device is
present, every entry point raises.  Device pointers come from PyTorch CUDA
tensors (``tensor.data_ptr()``); streams are torch's current stream.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

import os

LIB_PATH = Path(os.environ.get("LDGB200_LIB",
                             Path(__file__).resolve().parent / "lib" / "libldgb200.so"))
MAX_N1 = 9
MAX_NCU = 5

FACE_INTERIOR, FACE_DIRICHLET, FACE_NEUMANN = 0, 1, 2
FACE_SIDE_RIGHT = 4
FACE_SWITCH = 8
FACE_MAP_SHIFT = 8


class LdgNativeError(RuntimeError):
    pass


class LdgTables(C.Structure):
    _fields_ = [
        ("nd", C.c_int32), ("n1", C.c_int32), ("ncu", C.c_int32), ("ne", C.c_int32),
        ("n_maps", C.c_int32), ("trace_centered", C.c_int32),
        ("grad_centered", C.c_int32), ("flux_uses_u", C.c_int32),
        ("geo", C.c_void_p), ("fnbr", C.c_void_p), ("finfo", C.c_void_p),
        ("ftau", C.c_void_p), ("nmap", C.c_void_p),
        ("d1", C.c_double * (MAX_N1 * MAX_N1)),
        ("m1", C.c_double * (MAX_N1 * MAX_N1)),
        ("s1", C.c_double * (MAX_N1 * MAX_N1)),
        ("clo", C.c_double * MAX_N1),
        ("chi", C.c_double * MAX_N1),
        ("au", C.c_double * (MAX_NCU * 3 * MAX_NCU)),
        ("aq", C.c_double * (MAX_NCU * 3 * MAX_NCU * 3)),
        ("mass_coef", C.c_double * MAX_NCU),
    ]


class LdgDenseTables(C.Structure):
    _fields_ = [
        ("nd", C.c_int32), ("nb", C.c_int32), ("nqf", C.c_int32), ("nface", C.c_int32),
        ("nperm", C.c_int32), ("ncu", C.c_int32), ("ne", C.c_int32),
        ("trace_centered", C.c_int32), ("grad_centered", C.c_int32), ("flux_uses_u", C.c_int32),
        ("geo", C.c_void_p), ("fnorm", C.c_void_p), ("fsj", C.c_void_p), ("fnbr", C.c_void_p),
        ("finfo", C.c_void_p), ("ftau", C.c_void_p), ("dr", C.c_void_p), ("kr", C.c_void_p),
        ("lift", C.c_void_p), ("fluxop", C.c_void_p), ("phif", C.c_void_p), ("phio", C.c_void_p),
        ("au", C.c_double * (MAX_NCU * 3 * MAX_NCU)),
        ("aq", C.c_double * (MAX_NCU * 3 * MAX_NCU * 3)),
    ]


_lib = None
_host_lib = None

_SIGS = {
    "ldg_version": ([], C.c_int),
    "ldg_last_error": ([], C.c_char_p),
    "ldg_create": ([C.POINTER(LdgTables), C.POINTER(C.c_void_p)], C.c_int),
    "ldg_create_dense": ([C.POINTER(LdgDenseTables), C.POINTER(C.c_void_p)], C.c_int),
    "ldg_destroy": ([C.c_void_p], C.c_int),
    "ldg_last_bad_element": ([C.c_void_p], C.c_int64),
    "ldg_compute_mixed": ([C.c_void_p] * 5, C.c_int),
    "ldg_scratch_doubles": ([C.c_void_p], C.c_int64),
    "ldg_set_export_layout": ([C.c_void_p, C.c_int], C.c_int),
    "ldg_set_ghost_rows": ([C.c_void_p, C.c_int, C.c_void_p], C.c_int),
    "ldg_set_option": ([C.c_void_p, C.c_char_p, C.c_int], C.c_int),
    "ldg_set_ghost_rows_dense": ([C.c_void_p, C.c_int, C.c_void_p, C.c_void_p], C.c_int),
    "ldg_residual": ([C.c_void_p] * 7, C.c_int),
    "ldg_residual_tangent": ([C.c_void_p] * 5, C.c_int),
    "ldg_operator_pass": ([C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 6, C.c_int),
    "ldg_operator_pass_range": ([C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 5
                                + [C.c_int, C.c_int, C.c_void_p], C.c_int),
    "ldg_apply_host": ([C.c_void_p, C.c_int] + [C.c_void_p] * 7 + [C.c_int, C.c_void_p,
                                                                 C.c_void_p, C.c_void_p],
                       C.c_int),
    "ldg_apply_host_staged": ([C.c_void_p, C.c_int] + [C.c_void_p] * 8
                              + [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ldg_flux_from_mixed": ([C.c_void_p, C.c_int] + [C.c_void_p] * 6, C.c_int),
    "ldg_mass_apply": ([C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p], C.c_int),
    "ldg_mass_inv_apply": ([C.c_void_p] * 4, C.c_int),
    "ldg_reduce_scratch_doubles": ([], C.c_int64),
    "ldg_dot": ([C.c_int64] + [C.c_void_p] * 5, C.c_int),
    "ldg_nrm2": ([C.c_int64] + [C.c_void_p] * 4, C.c_int),
    "ldg_axpy": ([C.c_int64, C.c_double, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p,
                  C.c_void_p], C.c_int),
    "ldg_div_scalar": ([C.c_int64] + [C.c_void_p] * 4, C.c_int),
    "ldg_div_scalar_guarded": ([C.c_int64, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                                C.c_void_p], C.c_int),
    "ldg_mgs_step": ([C.c_int64] + [C.c_void_p] * 7, C.c_int),
    "ldg_cgs_dots": ([C.c_int64, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                      C.c_void_p, C.c_void_p], C.c_int),
    "ldg_cgs_update": ([C.c_int64, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                        C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ldg_combine": ([C.c_int64, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                     C.c_void_p], C.c_int),
    "ldg_color_distance2": ([C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p],
                            C.c_int),
    "ldg_bj_tile_elems": ([], C.c_int),
    "ldg_bj_block_keys": ([C.c_int64, C.c_int] + [C.c_void_p] * 3, C.c_int),
    "ldg_bj_class_verify": ([C.c_int64, C.c_int] + [C.c_void_p] * 4, C.c_int),
    "ldg_bj_apply_tiles": ([C.c_int64, C.c_int] + [C.c_void_p] * 6, C.c_int),
    "ldg_comm_unique_id": ([C.c_void_p], C.c_int),
    "ldg_comm_init": ([C.c_void_p, C.c_int, C.c_int, C.c_void_p], C.c_int),
    "ldg_comm_init_local": ([C.c_void_p, C.c_int], C.c_int),
    "ldg_set_halo_plan": ([C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                           C.c_int] + [C.c_void_p] * 9, C.c_int),
    "ldg_apply_dist": ([C.c_void_p, C.c_int] + [C.c_void_p] * 6, C.c_int),
    "ldg_comm_destroy": ([C.c_void_p], C.c_int),
    "ldg_face_nbar": ([C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 4,
                      C.c_int),
    "ldg_probe_fp64": ([C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ldg_probe_fp64_mode": ([C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ldg_dcgs_dots": ([C.c_int64, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ldg_dcgs_update": ([C.c_int64, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                         C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ldg_bj_probe_colour": ([C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int64, C.c_void_p,
                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ldg_bj_probe_vector": ([C.c_int64, C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_void_p,
                             C.c_void_p], C.c_int),
    "ldg_bj_extract": ([C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p,
                        C.c_void_p], C.c_int),
    "ldg_bj_invert": ([C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
                      C.c_int),
    "ldg_bj_invert_global": ([C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
                      C.c_int),
    "ldg_bj_apply": ([C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
                     C.c_int),
    "ldg_permute_gather": ([C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
                           C.c_int),
    "ldg_permute_scatter": ([C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
                            C.c_int),
    "ldg_jit_last_error": ([], C.c_char_p),
    "ldg_jit_compile": ([C.c_char_p, C.c_char_p, C.c_void_p, C.c_int, C.c_void_p,
                         C.POINTER(C.c_int64)], C.c_int),
    "ldg_jit_load": ([C.c_void_p, C.c_int64, C.POINTER(C.c_void_p)], C.c_int),
    "ldg_jit_unload": ([C.c_void_p], C.c_int),
    "ldg_jit_launch": ([C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                        C.c_int64, C.c_void_p], C.c_int),
    "ldg_jit_attr": ([C.c_void_p, C.c_char_p] + [C.POINTER(C.c_int)] * 3, C.c_int),
}

EXPORTED = tuple(_SIGS)


def load(require_gpu=True):
    """Load the native library (building it first if sources are newer)."""
    global _lib, _host_lib
    if _lib is not None:
        return _lib
    if not require_gpu and _host_lib is not None:
        return _host_lib
    if not LIB_PATH.exists():
        try:
            from .build import build
            build()
        except Exception as e:  # pragma: no cover - surfaced loudly
            raise LdgNativeError(f"libldgb200.so missing and build failed: {e}") from e
    lib = C.CDLL(str(LIB_PATH))
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if not require_gpu:
        _host_lib = lib        # host-only entry points (setup, NVRTC); not GPU-verified
        return lib
    import torch
    if not torch.cuda.is_available():
        raise LdgNativeError("the B200 LDG path needs a CUDA device; no CPU fallback")
    _lib = lib
    return lib


def check(rc, what, jit=False):
    if rc == 0:
        return
    msg = ""
    lib = _lib if _lib is not None else _host_lib
    if lib is not None:
        msg = (lib.ldg_jit_last_error() if jit else lib.ldg_last_error()).decode()
    raise LdgNativeError(f"{what} failed (code {rc}): {msg}")


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def as_c(arr, dtype):
    a = np.ascontiguousarray(arr, dtype=dtype)
    return a, a.ctypes.data_as(C.c_void_p)
