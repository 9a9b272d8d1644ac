"""ctypes loader for the B200 engine (paper_1408_3839_b200/_lib/liblatham_b200.so).

The product path has no CPU fallback: if the shared library is missing or no CUDA
device is visible, constructing a :class:`Context` raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "liblatham_b200.so")

_P = ctypes.POINTER
_d = ctypes.c_double
_i64 = ctypes.c_int64
_dp = _P(ctypes.c_double)
_ip = _P(ctypes.c_int64)
_vp = ctypes.c_void_p


class Error(RuntimeError):
    """latham::Error (errors.hpp:10-13)."""


class DimensionError(Error):
    pass


class BoundsError(Error):
    pass


class StructureError(Error):
    pass


class DefinitenessError(Error):
    pass


class ResourceCapError(Error):
    pass


class DeviceError(Error):
    pass


_ERRORS = {1: DimensionError, 2: BoundsError, 3: StructureError, 4: DefinitenessError, 5: ResourceCapError,
           6: Error, 7: DeviceError}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() (make -C paper_1408_3839_b200/csrc)")
        L = ctypes.CDLL(LIB_PATH)
        sig = {
            "lt_create": ([ctypes.c_int, _P(_vp)], ctypes.c_int),
            "lt_destroy": ([_vp], None),
            "lt_last_error": ([], ctypes.c_char_p),
            "lt_stream": ([_vp], _vp),
            "lt_stream_wait": ([_vp, _vp], ctypes.c_int),
            "lt_stream_join": ([_vp, _vp], ctypes.c_int),
            "lt_launch_count": ([_vp], _i64),
            "lt_set_stage_timing": ([_vp, ctypes.c_int], ctypes.c_int),
            "lt_set_diagnostics": ([_vp, ctypes.c_int], ctypes.c_int),
            "lt_stage_count": ([_vp], _i64),
            "lt_stage_get": ([_vp, _i64, ctypes.c_char_p, _i64, _dp, _ip], ctypes.c_int),
            "lt_op_separable_count": ([_vp], _i64),
            "lt_op_separable": ([_vp, _dp], ctypes.c_int),
            "lt_separable_residual": ([_vp, _vp, _dp], ctypes.c_int),
            "lt_solve_periodic_factorized": ([_vp, _vp, _vp, ctypes.c_double, _dp], ctypes.c_int),
            "lt_solve_periodic_factorized_gen": ([_vp, _ip, _i64, _i64, _ip, _dp, _i64, _dp, _i64, _ip, _dp, _i64,
                                                  _dp, ctypes.c_double, _dp], ctypes.c_int),
            "lt_factorized_block_diagonalize": ([_vp, ctypes.c_int, _ip, _i64, _i64, _dp, _dp], ctypes.c_int),
            "lt_box_circulant_defect": ([_vp, _vp, _dp, _dp], ctypes.c_int),
            "lt_stage_timeline_count": ([_vp], _i64),
            "lt_stage_timeline_get": ([_vp, _i64, ctypes.c_char_p, _i64, ctypes.POINTER(ctypes.c_int), _dp, _dp],
                                      ctypes.c_int),
            "lt_solve_core": ([_vp, _vp, ctypes.c_int, _dp, _ip], ctypes.c_int),
            "lt_sys_upload": ([_vp, _vp, _P(_vp)], ctypes.c_int),
            "lt_sys_free": ([_vp], None),
            "lt_solve_core_dev": ([_vp, _vp, ctypes.c_int, _vp, _i64, _i64, _ip], ctypes.c_int),
            "lt_solve_core_dev_on": ([_vp, _vp, ctypes.c_int, _vp, _i64, _i64, _ip, _vp], ctypes.c_int),
            "lt_core_layout": ([_vp, _vp, ctypes.c_int, _ip, _ip], ctypes.c_int),
            "lt_assemble_core_dev": ([_vp, _vp, ctypes.c_int, _i64, _i64, ctypes.c_int, _vp, _vp], ctypes.c_int),
            "lt_spectrum_dev": ([_vp, _vp, ctypes.c_int, _vp, _vp, _vp, _i64, _i64], ctypes.c_int),
            "lt_assemble": ([_vp, _vp, ctypes.c_int, ctypes.c_int, _P(_vp)], ctypes.c_int),
            "lt_assemble_core": ([_vp, _vp, ctypes.c_int, _P(_vp), _P(_vp)], ctypes.c_int),
            "lt_combine": ([_vp, _d, _vp, _d, _vp, _P(_vp)], ctypes.c_int),
            "lt_op_free": ([_vp], None),
            "lt_op_info": ([_vp, _ip], None),
            "lt_op_dense": ([_vp, _dp], ctypes.c_int),
            "lt_op_blocks": ([_vp, _ip, _dp], ctypes.c_int),
            "lt_solve_periodic_ops": ([_vp, _vp, _vp, _dp], ctypes.c_int),
            "lt_solve_periodic": ([_vp, _ip, _i64, _i64, _ip, _dp, _i64, _ip, _dp, _dp], ctypes.c_int),
            "lt_block_diagonalize": ([_vp, _ip, _i64, _i64, _ip, _dp, _dp], ctypes.c_int),
            "lt_solve_box_dense": ([_vp, _i64, _dp, _dp, _i64, _dp], ctypes.c_int),
            "lt_pencil_eig": ([_vp, _i64, _i64, _dp, _dp, _dp], ctypes.c_int),
            "lt_solve_box_dense_vectors": ([_vp, _i64, _dp, _dp, _i64, _dp, _dp], ctypes.c_int),
            "lt_pencil_eigvec": ([_vp, _i64, _i64, _dp, _dp, _dp, _dp], ctypes.c_int),
            "lt_solve_periodic_ops_vectors": ([_vp, _vp, _vp, _dp, _dp], ctypes.c_int),
            "lt_solve_periodic_vectors": ([_vp, _ip, _i64, _i64, _ip, _dp, _i64, _ip, _dp, _dp, _dp], ctypes.c_int),
            "lt_solve_periodic_factorized_vectors": ([_vp, _vp, _vp, ctypes.c_double, _dp, _dp], ctypes.c_int),
            "lt_reconstruct_eigenvectors": ([_vp, _ip, _i64, _dp, _i64, _dp], ctypes.c_int),
            "lt_bc_full_eigenvector": ([_vp, _ip, _i64, _dp, _i64, _i64, _dp], ctypes.c_int),
            "lt_sinc_quadrature": ([_vp, _i64, _dp, _dp], ctypes.c_int),
            "lt_overlap_constant": ([_vp, _vp, _ip], ctypes.c_int),
            "lt_newton_master": ([_vp, _i64, _d, _i64, _dp], ctypes.c_int),
            "lt_potential": ([_vp, _vp, ctypes.c_int, _i64, _ip, _ip, _dp, _dp, _i64], ctypes.c_int),
            "lt_assembled_window_sum": ([_vp, _i64, _i64, _dp, _i64, _ip, _i64, _dp], ctypes.c_int),
            "lt_profiles": ([_vp, _vp, _i64, _ip, _ip, _ip, _dp, _i64], ctypes.c_int),
            "lt_create_multi": ([_P(ctypes.c_int), ctypes.c_int, _P(_vp)], ctypes.c_int),
            "lt_destroy_multi": ([_vp], None),
            "lt_multi_ndev": ([_vp], ctypes.c_int),
            "lt_multi_ctx": ([_vp, ctypes.c_int], _vp),
            "lt_solve_core_multi": ([_vp, _vp, ctypes.c_int, ctypes.c_int, _dp, _ip], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def check(rc: int):
    if rc != 0:
        msg = lib().lt_last_error().decode()
        raise _ERRORS.get(rc, Error)(msg)


# symbols declared in include/latham_b200.h (checked by tests/test_abi.py)
EXPORTS = (
    "lt_create_multi", "lt_destroy_multi", "lt_multi_ndev", "lt_multi_ctx", "lt_solve_core_multi",
    "lt_create", "lt_destroy", "lt_last_error", "lt_stream", "lt_stream_wait", "lt_stream_join", "lt_launch_count", "lt_set_stage_timing", "lt_set_diagnostics",
    "lt_stage_count", "lt_stage_get", "lt_stage_timeline_count", "lt_stage_timeline_get",
    "lt_op_separable_count", "lt_op_separable", "lt_separable_residual", "lt_solve_periodic_factorized",
    "lt_solve_periodic_factorized_gen", "lt_factorized_block_diagonalize", "lt_box_circulant_defect", "lt_solve_core", "lt_sys_upload",
    "lt_sys_free", "lt_solve_core_dev", "lt_solve_core_dev_on", "lt_core_layout", "lt_assemble_core_dev", "lt_spectrum_dev", "lt_assemble", "lt_assemble_core", "lt_combine", "lt_op_free", "lt_op_info",
    "lt_op_dense", "lt_op_blocks", "lt_solve_periodic_ops", "lt_solve_periodic", "lt_block_diagonalize",
    "lt_solve_box_dense", "lt_pencil_eig", "lt_solve_box_dense_vectors", "lt_pencil_eigvec",
    "lt_solve_periodic_ops_vectors", "lt_solve_periodic_vectors", "lt_solve_periodic_factorized_vectors",
    "lt_reconstruct_eigenvectors", "lt_bc_full_eigenvector", "lt_sinc_quadrature", "lt_overlap_constant", "lt_newton_master",
    "lt_potential", "lt_assembled_window_sum", "lt_profiles",
)
