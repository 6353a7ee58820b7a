"""ctypes declarations of include/bgk.h (argument marshalling only).

The shared library ``libbgk_b200.so`` is built in-tree by
``paper_2408_02350_b200.build.build_library()`` (nvcc, sm_100a).  There is no
fallback: if the library is missing or fails to load, importing the binding
raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbgk_b200.so")

BGK_OK = 0
STATUS = {0: "BGK_OK", 1: "BGK_E_INVALID_ARG", 2: "BGK_E_CAPACITY", 3: "BGK_E_DEFICIENT_STENCIL",
          4: "BGK_E_DEGENERATE_STATE", 5: "BGK_E_OUT_OF_DOMAIN", 6: "BGK_E_CUDA", 7: "BGK_E_WALL"}
BUF_MOMENT_SUMS, BUF_WALL_FLUX, BUF_F = 0, 1, 2
PHASES = ("geometry", "transport", "moment_sums", "relax", "boundary_interp", "boundary_fill")


class BgkConfig(C.Structure):
    _fields_ = [("dims", C.c_int32), ("Nv", C.c_int32), ("vmax", C.c_double), ("L", C.c_double),
                ("h", C.c_double), ("h2", C.c_double), ("alpha_w", C.c_double), ("dt", C.c_double),
                ("R", C.c_double), ("kb", C.c_double), ("dmol", C.c_double), ("T_wall", C.c_double),
                ("U_lid", C.c_double * 3), ("dx", C.c_double), ("ale", C.c_int32),
                ("col_begin", C.c_int32), ("col_end", C.c_int32), ("max_neighbors", C.c_int32),
                ("wls_order", C.c_int32), ("manage", C.c_int32), ("m_min", C.c_int32),
                ("r_merge", C.c_double), ("max_particles", C.c_int64), ("staging", C.c_int32)]


_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64

# name -> argtypes (all return bgk_status as int unless noted)
SIGNATURES = {
    "bgk_workspace_size": [_P, _I64, _P],
    "bgk_init_cloud": [_P, _P, _P, _P, _I64, _P, C.c_size_t, _P, _P],
    "bgk_build_neighbors": [_P, _P, _P, _I64, _P, _P],
    "bgk_wls_coeffs": [_P, _P],
    "bgk_get_wls": [_P, _P, _P, _P, _P, _P],
    "bgk_step": [_P, _I, _P],
    "bgk_step_transport": [_P, _P],
    "bgk_step_relax": [_P, _P],
    "bgk_step_boundary": [_P, _P],
    "bgk_run_phase": [_P, _I, _P],
    "bgk_buffer": [_P, _I, _P, _P],
    "bgk_moments": [_P, _P, _P, _P, _P],
    "bgk_moments_partial": [_P, _P],
    "bgk_moments_finalize": [_P, _P, _P, _P, _P],
    "bgk_get_macro": [_P, _P, _P],
    "bgk_get_f": [_P, _P, _P],
    "bgk_set_f": [_P, _P, _P],
    "bgk_get_positions": [_P, _P, _P],
    "bgk_get_neighbors": [_P, _P, _P, _P, _P],
    "bgk_stable_dt": [_P, _P, _P],
    "bgk_launches_per_step": [_P, _P],
    "bgk_sync": [_P, _P],
    "bgk_destroy": [_P],
    "bgk_manage": [_P, _P, _P],
    "bgk_count": [_P, _P, _P, _P, _P],
    "bgk_manage_report": [_P, _P],
    "bgk_get_kind": [_P, _P, _P],
    "bgk_transport_info": [_P, _P],
    "bgk_graph_info": [_P, _P],
    "bgk_stage_f": [_P, _P, _P],
    "bgk_use_staged_f": [_P, _P],
}
OTHER = {"bgk_last_error": (C.c_char_p, [_P, _P]), "bgk_version": (C.c_char_p, [])}
EXPORTED = sorted(list(SIGNATURES) + list(OTHER))

_lib = None


def load(path: str = LIB_PATH):
    """Load the library (raises OSError/ImportError if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("BGK_LIB_PATH", path)   # experiment builds (tools/); default is the in-tree library
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with paper_2408_02350_b200.build.build_library() "
                          "(the CUDA path has no CPU fallback)")
    L = C.CDLL(path)
    for name, args in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = C.c_int
        fn.argtypes = args
    for name, (res, args) in OTHER.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


class BgkError(RuntimeError):
    def __init__(self, status: int, msg: str = "", particle: int = -1):
        self.status, self.particle = status, particle
        super().__init__(f"{STATUS.get(status, status)}: {msg} (particle {particle})")
