"""ctypes binding of ``libsmg.so`` (the sm_100a hot path, ``include/smg.h``).

The library is built in-tree (``paper_1512_02390_b200/libsmg.so``) by
``__graft_entry__.build()`` / ``make -C paper_1512_02390_b200/csrc``.  There is
no CPU fallback: if the library or a CUDA device is missing, every compute
entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SMG_LIB: an alternative build of the same library (e.g. the phase-profile build, tools/fdt_phases.py)
LIB_PATH = os.environ.get("SMG_LIB") or os.path.join(_HERE, "libsmg.so")

SMG_EINVAL = -1
SMG_EUNSUPPORTED = -2

_vp = C.c_void_p
_dp = C.c_void_p            # device pointers are passed as integers
_hp = C.POINTER(C.c_double)  # host arrays
_i64 = C.c_int64

# name -> (restype, argtypes); every symbol declared in include/smg.h
SIGNATURES = {
    "smg_last_error": (C.c_char_p, []),
    "smg_version": (C.c_int, []),
    "smg_launch_count": (C.c_int64, []),
    "smg_device_ok": (C.c_int, []),
    "smg_debug_fdt_phases": (C.c_int, [C.POINTER(C.c_ulonglong), C.c_int]),
    "smg_op_create": (C.c_int, [C.POINTER(_vp), C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                C.c_double, _hp, _hp, _dp]),
    "smg_op_destroy": (C.c_int, [_vp]),
    "smg_op_residual": (C.c_int, [_vp, _dp, _dp, _dp, _vp]),
    "smg_op_ws_doubles": (C.c_size_t, [_vp]),
    "smg_op_residual_norm2": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _dp, _vp]),
    "smg_schwarz_create": (C.c_int, [C.POINTER(_vp), C.c_int, C.c_int, C.c_int, C.c_int, _hp, _hp,
                                     _hp, _hp, _hp, _hp, _dp]),
    "smg_schwarz_destroy": (C.c_int, [_vp]),
    "smg_schwarz_ws_doubles": (C.c_size_t, [_vp]),
    "smg_schwarz_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "smg_schwarz_correct": (C.c_int, [_vp, _dp, _dp, _dp, _vp]),
    "smg_schwarz_smooth": (C.c_int, [_vp, _vp, _dp, _dp, _dp, _dp, C.c_int, C.c_int, _vp]),
    "smg_fd_solve_blocks": (C.c_int, [_vp, _dp, _dp, C.c_int, C.c_int, _vp]),
    "smg_transfer_create": (C.c_int, [C.POINTER(_vp), C.c_int, C.c_int, C.c_int, C.c_int, _hp]),
    "smg_transfer_destroy": (C.c_int, [_vp]),
    "smg_prolongate": (C.c_int, [_vp, _dp, _dp, C.c_int, _vp]),
    "smg_prolongate_chain": (C.c_int, [C.POINTER(_vp), C.c_int, _dp, C.POINTER(_vp), _vp]),
    "smg_restrict": (C.c_int, [_vp, _dp, _dp, _vp]),
    "smg_residual_restrict": (C.c_int, [_vp, _vp, _dp, _dp, _dp, _dp, _vp]),
    "smg_transfer_ws_doubles": (C.c_size_t, [_vp]),
    "smg_restrict_ws": (C.c_int, [_vp, _dp, _dp, _dp, _vp]),
    "smg_residual_restrict_ws": (C.c_int, [_vp, _vp, _dp, _dp, _dp, _dp, _dp, _dp, _vp]),
    "smg_op_residual_norm2_ws": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _dp, _dp, _vp]),
    "smg_op_apply_dot": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _dp, _vp]),
    "smg_op_ring_doubles": (C.c_size_t, [_vp]),
    "smg_op_residual_ws": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _vp]),
    "smg_schwarz_smooth_ws": (C.c_int, [_vp, _vp, _dp, _dp, _dp, _dp, _dp, C.c_int, C.c_int, _vp]),
    "smg_coarse_create": (C.c_int, [C.POINTER(_vp), C.c_int, C.c_int, C.c_double, C.c_double]),
    "smg_coarse_destroy": (C.c_int, [_vp]),
    "smg_coarse_ws_doubles": (C.c_size_t, [_vp]),
    "smg_coarse_pinv": (C.c_int, [_vp, _dp, _dp, _dp, _vp]),
    "smg_mult_create": (C.c_int, [C.POINTER(_vp), C.c_int, C.c_int, C.c_int, C.c_int, _hp, _hp, _hp, _hp, _dp]),
    "smg_mult_destroy": (C.c_int, [_vp]),
    "smg_mult_sweep": (C.c_int, [_vp, _vp, _dp, _dp, C.c_int, _vp]),
    "smg_coarse_cg": (C.c_int, [_vp, _dp, _dp, _dp, C.c_double, C.c_int, C.POINTER(C.c_int), _vp]),
    "smg_coarse_cg_ws_doubles": (C.c_size_t, [_i64]),
    "smg_coarse_pcg_ws_doubles": (C.c_size_t, [_vp]),
    "smg_coarse_pcg": (C.c_int, [_vp, _vp, _dp, _dp, _dp, C.c_double, C.c_int, C.c_double, C.POINTER(C.c_int), _vp]),
    "smg_reduce_ws_doubles": (C.c_size_t, []),
    "smg_dot": (C.c_int, [_dp, _dp, _i64, _dp, _dp, _vp]),
    "smg_dot2": (C.c_int, [_dp, _dp, _dp, _i64, _dp, _dp, _vp]),
    "smg_axpby": (C.c_int, [C.c_double, _dp, C.c_double, _dp, _i64, _vp]),
    "smg_cg_update": (C.c_int, [_dp, _dp, _dp, _dp, _i64, _dp, _dp, _dp, _vp]),
    "smg_cg_update2": (C.c_int, [_dp, _dp, _dp, _dp, _dp, _i64, _dp, _dp, _dp, _vp]),
    "smg_cg_beta": (C.c_int, [_dp, _dp, _dp, _i64, _dp, _dp, _vp]),
    "smg_cg_beta_finish": (C.c_int, [_dp, _vp]),
    "smg_halo_available": (C.c_int, []),
    "smg_halo_nccl_version": (C.c_int, []),
    "smg_halo_unique_id": (C.c_int, [C.c_char_p, C.c_int]),
    "smg_halo_create": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]),
    "smg_halo_destroy": (C.c_int, [_vp]),
    "smg_halo_exchange": (C.c_int, [_vp, _dp, _i64, _i64, _i64, _i64, C.c_int, C.c_int, _vp]),
    "smg_halo_ws_doubles": (_i64, [_i64, C.c_int, C.c_int]),
    "smg_halo_exchange_add": (C.c_int, [_vp, _dp, _i64, _i64, _i64, _i64, C.c_int, C.c_int, _dp, _vp]),
    "smg_halo_allreduce": (C.c_int, [_vp, _dp, _i64, _vp]),
    "smg_halo_allgather": (C.c_int, [_vp, _dp, _dp, _i64, _vp]),
    "smg_cg_direction": (C.c_int, [_dp, _dp, _i64, _dp, _vp]),
    "smg_project_mean": (C.c_int, [_dp, _i64, _dp, _vp]),
    "smg_sum": (C.c_int, [_dp, _i64, _dp, _dp, _vp]),
    "smg_sum_partials": (C.c_int, [_dp, C.c_int, _dp, _vp]),
    "smg_problem_field": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, _hp, _hp,
                                    C.c_double, C.c_double, _dp, _vp]),
    "smg_element_mean": (C.c_int, [C.c_int, C.c_int, C.c_int, _hp, _dp, _dp, _vp]),
}

_lib = None


def load(require_device: bool = True):
    """Load libsmg.so once; raise loudly if it (or, optionally, a device) is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libsmg.so not found at {LIB_PATH}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_device:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1512_02390_b200 needs a CUDA device (B200, sm_100a); "
                               "there is no CPU fallback")
        torch.cuda.init()
        if not _lib.smg_device_ok():
            raise RuntimeError(_lib.smg_last_error().decode())
    return _lib


def lib():
    return load(True)


def check(rc: int, what: str = ""):
    if rc == 0:
        return
    msg = _lib.smg_last_error().decode() if _lib is not None else "libsmg not loaded"
    if rc == SMG_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"{what}: {msg}" if what else msg)


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def hptr(a: np.ndarray):
    """ctypes double* into a contiguous float64 numpy array (kept alive by the caller)."""
    return a.ctypes.data_as(_hp)


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def host(a):
    """Host float64 contiguous array -> ctypes double* (keeps a reference)."""
    import numpy as np
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_hp)


class Handle:
    """Owns a libsmg handle; destroyed with the Python object."""

    def __init__(self, raw, destroy):
        self._raw = raw
        self._destroy = destroy

    @property
    def raw(self):
        return self._raw

    def __del__(self):
        try:
            if self._raw and _lib is not None:
                getattr(_lib, self._destroy)(self._raw)
        except Exception:
            pass
        self._raw = None
