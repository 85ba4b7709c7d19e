"""ctypes binding of libmcb200.so (include/mcb200.h).

This is the only way the package reaches device code: there is no CPU
fallback.  Importing the package without the built library, or calling a
device entry point without a CUDA device, raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os

from .errors import (ConfigError, DegenerateFitError, DeviceError, EmptyActiveSetError,
                     InvalidStructureError, OutOfGridError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MCB200_LIB") or os.path.join(_HERE, "libmcb200.so")

MC_OK = 0
MC_ERR_INVALID_STRUCTURE = -1
MC_ERR_DEGENERATE_FIT = -2
MC_ERR_CONFIG = -3
MC_ERR_OUT_OF_GRID = -4
MC_ERR_EMPTY_ACTIVE_SET = -5
MC_ERR_CUDA_BASE = -100

FLAG_DEGENERATE = 1
FLAG_NO_CONVERGE = 2
FLAG_NON_FINITE = 4
FLAG_ADJ_FALLBACK = 8
FLAG_SIG_OVERFLOW = 16
FLAG_OUT_OF_GRID = 32

MC_F32 = 0
MC_F64 = 1

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double

# name -> argtypes (all return int status)
_SIGS = {
    "mc_center": [_P, ctypes.c_int, _I64, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "mc_cov_f64": [_P, _P, _I32, _I32, _I32, _P, _P],
    "mc_cov_pairs": [_P, _P, _P, _P, _I64, _I32, _P, _P, _P],
    "mc_fit_dense": [_P, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P],
    "mc_fit_list_msd": [_P, _I64, _P, _P, _P, _P, _P, _P],
    "mc_fit_full": [_P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "mc_rot_grad": [_P, _P, _P, _P, _I64, _I32, _I32, _P, _P, _P, _P],
    "mc_jacobi4": [_P, _I64, _P, _P, _P, _P],
    "mc_jacobi_n": [_P, _I64, _I32, _D, _I32, _P, _P, _P, _P],
    "mc_window_pairs": [_I32, _I32, _I32, _P, _P, _P],
    "mc_close_scan": [_P, _P, _I32, _I32, _I32, _P, _P, _I32, _D, _P, _P, _P, _P, _P],
    "mc_xy_eig": [_P, _P, _I64, _I32, _P, _P, _P, _P, _P, _P, _P],
    "mc_pathcv_weights": [_I32, _I32, _I32, _D, _D, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                          _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "mc_pathcv_weights_nl": [_I32, _I32, _I32, _D, _D, _I32, _P, _P, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                             _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "mc_neighbour_topm": [_P, ctypes.c_int, _I32, _I32, _I64, _P, _I32, _P, _P],
    "mc_mtd_bias_direct": [_P, _I32, _I32, _P, _P, _P, _I32, _P, _P, _P],
    "mc_mtd_grid_deposit": [_P, _P, _P, _I32, _P, _P, _P, _P, _P, _D, _D, _P, _P],
    "mc_mtd_grid_eval": [_P, _P, _P, _I32, _P, _P, _P, _P, _I32, _P, _P, _P, _P],
    "mc_mtd_force": [_P, _I32, _I32, _P, _P, _P, ctypes.c_int, _I32, _P, _P],
    "mc_pathcv_grad": [_I32, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I32,
                       _P, _P, _P, _P, _P, _P],
    "mc_center_split": [_P, ctypes.c_int, _I64, _I32, _I32, _P, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P],
    "mc_msd_tf32": [_P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _P, _I64, _I32, _P],
    "mc_msd_tf32_2sm": [_P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _P, _I64, _I32, _P],
    "mc_center_split16": [_P, ctypes.c_int, _I64, _I32, _I32, _P, _P, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P,
                          _P, _P],
    "mc_msd_f16": [_P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _I64, _I32, _P],
    "mc_msd_f16_2sm": [_P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _P, _I64, _I32, _P],
    "mc_pathcv_grad_block": [_I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _P],
    "mc_toysim_run": [_I32, _I32, _I32, _I32, _I64, _I32, _I32, _I32, _I32] + [_D] * 10 + [ctypes.c_uint64]
    + [_P] * 17 + [_I32, _I32, _P, _P, _P],
    "mc_shard_rescale": [_I32, _I32, _P, _P, _P, _P, _P, _P],
    "mc_candidates": [_P, _I32, _I32, _I64, _D, _D, _P, _D, _P, _P, _P, _I32, _P, _P, _P, _P, _P],
    "mc_grad_i8_wide_plan": [_I32, _I32, _I32, _P, _P, _P, _P, _P],
    "mc_pathcv_grad_i8_wide": [_I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P,
                               _P, _I32, _I32, _P, _I32, _P, _P, _I64, _P, _P],
    "mc_center_split16_uniform": [_P, _I64, _I32, _I32, _D, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "mc_candidates_life": [_P, _I32, _I32, _I64, _D, _D, _P, _D, _P, _I32, _P, _P, _P, _P, _P],
    "mc_refine_i8_close": [_P, _P, _P, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _P, _P],
    "mc_prune_plan": [_P, _I32, _I32, _I64, _P, _P, _P, _P, _D, _P, _P, _I32, _I32, _D, _I32, _I32, _P, _P, _P, _P, _P,
                      _P],
    "mc_band_tiles": [_P, _I32, _P, _P, _I32, _I32, _I32, _P, _P, _P, _P, _P],
    "mc_gather_rows": [_P, _I32, _I64, _P, _I32, _P, _P],
    "mc_sort_by_key": [_P, _I32, _I32, _P, _P, _P],
    "mc_refine": [_P, _P, _P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _P, _P, _P, _I32, _P, _P, _P, _I64, _P, _P, _D, _P,
                  _P],
    "mc_cov_dmma": [_P, _P, _P, _P, _P, _P, _P, _D, _I32, _I32, _I32, _P, _P],
    "mc_close_grad_fix": [_I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _P],
    "mc_pair_grad": [_I64, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                     _P, _P],
    "mc_property_map": [_I32, _I32, _P, _P, _P, _D, _P, _P, _P, _P],
    "mc_ldig_prep": [_P, _P, _I32, _I32, _I32, _I32, _P, _P, _P],
    "mc_row_digits": [_P, _P, _P, _P, _P, _I32, _I32, _I32, _P, _P, _P, _I32, _P],
    "mc_refine_i8": [_P, _P, _P, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _I32, _P, _P, _P, _I64, _P, _P],
    "mc_pathcv_grad_i8": [_I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _I32, _P, _P, _P, _P, _P, _P, _P,
                          _P, _P, _I32, _I32, _P, _P, _I64, _P],
}

# optional entry points (none at present)
_OPTIONAL = {}

_lib = None


def load():
    """Load libmcb200.so (once).  Raises DeviceError if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    for name, args in _OPTIONAL.items():
        fn = getattr(lib, name, None)
        if fn is not None:
            fn.argtypes = args
            fn.restype = ctypes.c_int
    lib.mc_version.restype = ctypes.c_int
    lib.mc_grad_i8_workspace_size.argtypes = [_I32, _I32]
    lib.mc_grad_i8_workspace_size.restype = _I64
    lib.mc_grad_i8_wide_header_size.argtypes = [_I32, _I32]
    lib.mc_grad_i8_wide_header_size.restype = _I64
    _lib = lib
    return lib


def exported_symbols():
    """Names declared in include/mcb200.h that the loaded library must export."""
    return ["mc_version", "mc_grad_i8_workspace_size", "mc_grad_i8_wide_header_size", *_SIGS.keys()]


def check(status, what=""):
    if status == MC_OK:
        return
    if status == MC_ERR_INVALID_STRUCTURE:
        raise InvalidStructureError(f"{what}: invalid structure")
    if status == MC_ERR_DEGENERATE_FIT:
        raise DegenerateFitError(f"{what}: degenerate fit")
    if status == MC_ERR_CONFIG:
        raise ConfigError(f"{what}: invalid configuration / arguments")
    if status == MC_ERR_OUT_OF_GRID:
        raise OutOfGridError(f"{what}: collective variable outside the bias grid")
    if status == MC_ERR_EMPTY_ACTIVE_SET:
        raise EmptyActiveSetError(f"{what}: empty active set")
    if status <= MC_ERR_CUDA_BASE:
        raise DeviceError(f"{what}: CUDA error {MC_ERR_CUDA_BASE - status}")
    raise DeviceError(f"{what}: status {status}")


COUNTERS = {"launches": 0}
_PROFILE = None  # list of (name, start_event, end_event) while profiling


def start_profile():
    global _PROFILE
    _PROFILE = []


def stop_profile():
    """Stop recording; returns {name: (count, total_ms)} (synchronises)."""
    global _PROFILE
    import torch

    rec, _PROFILE = _PROFILE, None
    torch.cuda.synchronize()
    out = {}
    for name, e0, e1 in rec or []:
        c, t = out.get(name, (0, 0.0))
        out[name] = (c + 1, t + e0.elapsed_time(e1))
    return out


def call(name, *args):
    """Invoke one C entry point (each launches exactly one kernel)."""
    lib = load()
    fn = getattr(lib, name)
    COUNTERS["launches"] += 1
    if _PROFILE is not None:
        import torch

        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        st = fn(*args)
        e1.record()
        _PROFILE.append((name, e0, e1))
    else:
        st = fn(*args)
    check(st, name)


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
