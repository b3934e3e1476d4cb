"""ctypes binding of the C ABI (include/csflow_b200.h).

There is no CPU fallback: if the sm_100a library is missing or a CUDA device
is absent, every compute entry point raises ``ExtensionMissing``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ExtensionMissing

LIB_PATH = os.environ.get("CSB_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libcsflow_b200.so")

_p = ctypes.c_void_p
_d = ctypes.c_double
_i = ctypes.c_int
_ll = ctypes.c_longlong
_sz = ctypes.c_size_t
_dp = ctypes.c_void_p  # device pointers travel as integers
_hp = ctypes.POINTER(ctypes.c_double)

# name -> (restype, argtypes); the ABI test checks every header symbol is here
SIGNATURES = {
    "csb_version": (_i, []),
    "csb_launch_count": (ctypes.c_ulonglong, []),
    "csb_create": (_i, [ctypes.POINTER(_p)]),
    "csb_destroy": (None, [_p]),
    "csb_last_error": (ctypes.c_char_p, [_p]),
    "csb_set_model": (_i, [_p, _i, _hp, _hp, _hp, _hp, _hp, _hp, _hp, _d, _d]),
    "csb_set_mechanism": (_i, [_p, _i, _hp, _hp, _hp, _hp, _i]),
    "csb_set_grid": (_i, [_p, _i, _i, _i, _dp, _dp, _dp, _dp]),
    "csb_set_bc": (_i, [_p, _i, _i, _d, _i, _hp]),
    "csb_workspace_bytes": (_sz, [_p, _i]),
    "csb_set_workspace": (_i, [_p, _dp, _sz]),
    "csb_status": (_i, [_p, ctypes.POINTER(ctypes.c_ulonglong), ctypes.POINTER(_ll),
                        ctypes.POINTER(_ll), _p]),
    "csb_residual": (_i, [_p, _dp, _dp, _dp, _i, _p]),
    "csb_cons_to_prim": (_i, [_p, _ll, _dp, _dp, _p]),
    "csb_production_rates": (_i, [_p, _ll, _dp, _dp, _p]),
    "csb_source_jacobian": (_i, [_p, _ll, _dp, _dp, _dp, _p]),
    "csb_spectral_radii": (_i, [_p, _dp, _dp, _dp, _p]),
    "csb_local_time_step": (_i, [_p, _ll, _dp, _dp, _dp, _d, _d, _dp, _dp, _p]),
    "csb_time_step": (_i, [_p, _dp, _d, _dp, _dp, _p]),
    "csb_assemble": (_i, [_p, _dp, _dp, _i, _i, _d, _d, _dp, _p]),
    "csb_operator_field": (_i, [_p, _dp, _i, _dp, _p]),
    "csb_lusgs": (_i, [_p, _dp, _dp, _dp, _p]),
    "csb_apply_update": (_i, [_p, _ll, _dp, _dp, _i, _dp, _p]),
    "csb_correct": (_i, [_p, _i, _ll, _i, _dp, _dp, _dp, _dp, _p]),
    "csb_residual_norms": (_i, [_p, _ll, _dp, _dp, _p]),
    "csb_implicit_step": (_i, [_p, _dp, _dp, _d, _i, _i, _dp, _dp, _p]),
    "csb_profile_step": (_i, [_p, _dp, _dp, _d, _i, _dp, ctypes.POINTER(ctypes.c_float), _p]),
    "csb_implicit_step_ex": (_i, [_p, _dp, _dp, _d, _i, _i, _dp, _dp, _dp, _i, _p]),
    "csb_iteration": (_i, [_p, _dp, _d, _i, _i, _i, _dp, _dp, _dp, _p]),
    "csb_transpose": (_i, [_ll, _i, _dp, _dp, _i, _p]),
    "csb_batched_inverse": (_i, [_i, _ll, _dp, _dp, _dp, _dp, _dp, _p]),
    "csb_fp64_peak": (_i, [_i, _dp, _p]),
    "csb_dual_time_rhs": (_i, [_p, _ll, _dp, _dp, _dp, _dp, _dp, _d, _d, _dp, _p]),
    "csb_implicit_step_rhs": (_i, [_p, _dp, _dp, _d, _i, _i, _d, _d, _dp, _p]),
    "csb_sum_squares": (_i, [_p, _ll, _dp, _dp, _p]),
    "csb_march_begin": (_i, [_p, _p, _dp, _dp, _dp, _i, _dp, _p]),
    "csb_march_run": (_i, [_p, _i, _i, _i, _p]),
    "csb_march_state": (_i, [_p, ctypes.POINTER(_i), ctypes.POINTER(_d), _p]),
    "csb_march_end": (None, [_p]),
    "csb_fill_nodes": (_i, [_i, _i, _i, _i, _dp, _dp, _dp, _dp, _dp, _p]),
    "csb_grid_metrics": (_i, [_i, _i, _i, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _p]),
    "csb_primitive": (_i, [_p, _ll, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _p]),
    "csb_wall_heat_flux": (_i, [_p, _i, _dp, _dp, _dp, _dp, _p]),
    "csb_argmax_pick": (_i, [_ll, _dp, _dp, _dp, _p]),
}

class MarchParams(ctypes.Structure):
    """csb_march_params (include/csflow_b200.h)."""

    _fields_ = [("scheme", _i), ("offdiag_paper", _i), ("first_order", _i), ("max_retries", _i),
                ("abs_floor", _d), ("drop_factor", _d)]


_LIB = None


def load():
    """Load the shared library (no CUDA call is made by loading)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ExtensionMissing(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a).  There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def hp(arr):
    """Host float64 numpy array -> ctypes double pointer (caller keeps arr alive)."""
    return arr.ctypes.data_as(_hp)
