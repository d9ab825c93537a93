"""ctypes binding of the C-ABI in include/psigpu.h (libpsigpu.so).

The library is built in-tree (see :mod:`paper_0904_0939_b200.build`) and
loaded from this package directory.  There is no CPU fallback: if the
library is missing, every entry point raises ImportError; if no CUDA device
is visible, every compute call raises DeviceError.  ctypes releases the GIL
for the duration of each call, like the reference's ``nogil`` numba kernels
(kernels.py:1-7).
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint, c_void_p

from .errors import raise_for_status

LIB_NAME = "libpsigpu.so"
# PSG_LIB overrides the in-tree library (developer A/B builds)
LIB_PATH = os.environ.get("PSG_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                     LIB_NAME)

F_WRITE = 1
RUN_LINEAR_NORM = 1   # psg_run_params.flags: linear renormalisation pairs
RUN_EXACT = 2         # psg_run_params.flags: norm / measure steps through the per-step path
F_NORM = 2
F_MEASURE = 4
F_CHECK = 8
Q_NUM, Q_DEN, Q_R2, Q_NORM = 0, 1, 2, 3

# scalar slots filled by psg_read_sums (include/psigpu.h)
S_E, S_NORM2, S_RRMS, S_N2, S_FACTOR, S_STATUS = 4, 5, 6, 7, 8, 9
NSCAL = 16

_dp = POINTER(c_double)
_lp = POINTER(c_int64)


class RunParams(ctypes.Structure):
    _fields_ = [
        ("steps", c_int64),
        ("measure_every", c_int64),
        ("norm_every", c_int64),
        ("reimpose_every", c_int64),
        ("step_offset", c_int64),
        ("n_impose", c_int32),
        ("impose_axis", c_int32 * 3),
        ("impose_sign", c_int32 * 3),
        ("flags", c_int32),
    ]


# name -> (restype, argtypes); every symbol include/psigpu.h declares
SIGNATURES = {
    "psg_abi_version": (c_int, []),
    "psg_last_error": (ctypes.c_char_p, []),
    "psg_device_count": (c_int, []),
    "psg_row_pitch": (c_int64, [c_int64]),
    "psg_trim_memory": (c_int, [c_int]),
    "psg_fill_uniform": (c_int, [c_void_p, ctypes.c_uint64]),
    "psg_get_potential": (c_int, [c_void_p, _dp, c_int64, c_int64]),
    "psg_fill_potential": (c_int, [c_void_p, c_int, _dp, c_int, _lp]),
    "psg_copy_to_host": (c_int, [c_int, c_void_p, c_void_p, c_int64]),
    "psg_host_alloc": (c_void_p, [c_int64]),
    "psg_host_free": (None, [c_void_p, c_int64]),
    "psg_copy_to_device": (c_int, [c_int, c_void_p, c_void_p, c_int64]),
    "psg_pairwise_sum_device": (c_int, [_dp, c_int64, _dp]),
    "psg_selftest_division": (c_int, [c_int64, ctypes.c_uint64, c_double, c_double,
                                      POINTER(ctypes.c_uint64)]),
    "psg_kernel_stencil_update": (c_int, [_dp, _dp, _dp, _dp, c_int64, c_int64, c_int64, c_int64]),
    "psg_kernel_stencil_update_v": (
        c_int, [_dp, _dp, c_double, c_double, c_double, _dp, c_int64, c_int64, c_int64, c_int64]),
    "psg_kernel_norm_plane_sums": (c_int, [_dp, c_int64, c_int64, c_int64, c_int64, _dp]),
    "psg_kernel_energy_plane_sums": (
        c_int, [_dp, _dp, c_double, c_int64, c_int64, c_int64, c_int64, _dp, _dp]),
    "psg_kernel_radius2_plane_sums": (
        c_int, [_dp, c_int64, c_double, c_double, c_int64, c_int64, c_int64, c_int64, _dp, _dp]),
    "psg_kernel_dot_plane_sums": (c_int, [_dp, _dp, c_int64, c_int64, c_int64, c_int64, _dp]),
    "psg_create": (c_int, [c_int, c_int64, c_int64, c_int64, c_double, c_double, c_double,
                           POINTER(c_void_p)]),
    "psg_create_ex": (c_int, [c_int, c_int64, c_int64, c_int64, c_double, c_double, c_double,
                              c_uint, c_int64, POINTER(c_void_p)]),
    "psg_destroy": (c_int, [c_void_p]),
    "psg_field_bytes": (c_int64, [c_void_p]),
    "psg_mem_info": (c_int, [c_int, _lp, _lp]),
    "psg_host_find_singular": (c_int, [_dp, c_int64, c_double, _lp]),
    "psg_stream": (c_void_p, [c_void_p]),
    "psg_sync": (c_int, [c_void_p]),
    "psg_geometry": (c_int, [c_void_p, _lp, _lp, _lp]),
    "psg_plane_ptr": (c_void_p, [c_void_p, c_int, c_int64]),
    "psg_set_field": (c_int, [c_void_p, _dp, c_int64, c_int64]),
    "psg_get_field": (c_int, [c_void_p, _dp, c_int64, c_int64]),
    "psg_set_potential": (c_int, [c_void_p, _dp, c_int64, c_int64, _lp]),
    "psg_set_coefficients": (c_int, [c_void_p, _dp, _dp, c_int64, c_int64]),
    "psg_sweep": (c_int, [c_void_p, c_int64, c_int64, c_uint]),
    "psg_swap": (c_int, [c_void_p, c_int]),
    "psg_reduce": (c_int, [c_void_p, c_int64, c_int64, c_uint, c_int]),
    "psg_plane_sums_ptr": (c_void_p, [c_void_p]),
    "psg_combine": (c_int, [c_void_p, c_uint]),
    "psg_read_sums": (c_int, [c_void_p, _dp, _dp]),
    "psg_measure": (c_int, [c_void_p, c_int64, c_int64]),
    "psg_dot": (c_int, [c_void_p, c_void_p, c_int64, c_int64]),
    "psg_materialize": (c_int, [c_void_p]),
    "psg_scale": (c_int, [c_void_p, c_double]),
    "psg_impose": (c_int, [c_void_p, c_int, c_int, c_int]),
    "psg_resample": (c_int, [c_void_p, c_void_p, _lp, _dp]),
    "psg_run": (c_int, [c_void_p, POINTER(RunParams), _dp, c_int64, _lp]),
    "psg_nccl_available": (c_int, []),
    "psg_nccl_unique_id": (c_int, [c_void_p]),
    "psg_comm_create": (c_int, [c_int, c_int, c_int, c_void_p, POINTER(c_void_p)]),
    "psg_comm_destroy": (c_int, [c_void_p]),
    "psg_comm_halo_messages": (c_int64, [c_void_p]),
    "psg_run_dist": (c_int, [c_void_p, c_void_p, c_int, c_int, POINTER(RunParams), _dp, c_int64,
                             _lp]),
    "psg_measure_dist": (c_int, [c_void_p, c_void_p, c_int, c_int, _dp]),
    "psg_ipc_create": (c_int, [c_void_p, c_int, c_int, c_void_p, POINTER(c_void_p)]),
    "psg_ipc_connect": (c_int, [c_void_p, c_void_p]),
    "psg_ipc_destroy": (c_int, [c_void_p]),
    "psg_run_ipc": (c_int, [c_void_p, c_void_p, POINTER(RunParams), _dp, c_int64, _lp]),
    "psg_measure_ipc": (c_int, [c_void_p, c_void_p, _dp]),
    "psg_ipc_halo_planes": (c_int64, [c_void_p]),
    "psg_run_multi": (c_int, [POINTER(c_void_p), c_int, POINTER(RunParams), _dp, c_int64, _lp]),
    "psg_measure_multi": (c_int, [POINTER(c_void_p), c_int, _dp]),
    "psg_tune": (c_int, [c_void_p, c_int, c_int, c_int]),
    "psg_norm_partials": (c_int, [c_void_p, c_int64, c_int64]),
    "psg_use_factor": (c_int, [c_void_p]),
    "psg_zero_sums": (c_int, [c_void_p]),
    "psg_set_factor": (c_int, [c_void_p, c_double]),
    "psg_axpy": (c_int, [c_void_p, c_void_p, c_double]),
    "psg_copy_plane": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int, c_int64]),
    "psg_launch_count": (c_int64, [c_void_p]),
    "psg_fused_pass_count": (c_int64, [c_void_p]),
    "psg_pass": (c_int, [c_void_p, c_int]),
    "psg_set_temporal": (c_int, [c_void_p, c_int]),
    "psg_set_option": (c_int, [c_void_p, c_int, c_int]),
}

_lib = None


def load():
    """Load libpsigpu.so from the package directory (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_0904_0939_b200.build` "
            "(there is no CPU fallback for the hot path)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().psg_last_error()
    return msg.decode() if msg else ""


def check(code: int) -> None:
    if code:
        raise_for_status(code, last_error())


def dptr(arr):
    """double* of a C-contiguous float64 numpy array."""
    return arr.ctypes.data_as(_dp)


def lptr(arr):
    return arr.ctypes.data_as(_lp)


def device_count() -> int:
    return int(load().psg_device_count())
