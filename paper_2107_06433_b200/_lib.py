"""ctypes binding of libswmd.so (the sm_100a kernels behind include/swmd.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no fallback: if the
library is missing or no CUDA device is present, every compute entry point
raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libswmd.so")
SOURCES = [os.path.join(_HERE, "csrc", "swmd.cu")]
INCLUDE = os.path.abspath(os.path.join(_HERE, "..", "include"))

ERR_WORDS = 4
NO_EVENT = (1 << 63) - 1
EINVAL = 1000
EVR = 1001

_lib = None


class NativeUnavailable(RuntimeError):
    """libswmd.so could not be loaded or no CUDA device is visible."""


class NativeError(RuntimeError):
    """A libswmd entry point returned a nonzero status."""


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double

# name -> argtypes (all return int)
_SIGS = {
    "swmd_abi_version": [],
    "swmd_device_sm_count": [],
    "swmd_err_reset": [_P, _P],
    "swmd_solve_reset": [_P, _P, _P],
    "swmd_row_norms_f64": [_P, _I64, _I32, _I64, _P, _P],
    "swmd_cost_build_f64": [_P, _I64, _I32, _I64, _P, _I32, _P, _D, _I32, _P, _P, _I64,
                            _P, _P, _P, _P, _I64, _P],
    "swmd_precompute_f64": [_P, _I64, _I32, _I64, _P, _D, _P, _P, _P, _P],
    "swmd_cost_build_compact_f64": [_P, _I64, _P, _I64, _I32, _I64, _P, _P, _I32, _P, _D, _P,
                                    _P, _P, _I64, _P],
    "swmd_cost_build_compact_reset_f64": [_P, _I64, _P, _I64, _I32, _I64, _P, _P, _I32, _P, _D,
                                          _P, _P, _P, _I64, _P, _P, _P],
    "swmd_solve_f64": [_P, _P, _P, _I64, _P, _P, _P, _P, _I32, _I64, _I32, _I32, _P, _P, _P,
                       _I64, _I64, _I32, _I32, _P, _P, _P],
    "swmd_solve_f64_reset_done": [_P, _P, _P, _I64, _P, _P, _P, _P, _I32, _I64, _I32, _I32, _P,
                                  _P, _P, _I64, _I64, _I32, _I32, _P, _P, _P],
    "swmd_solve_hot_f64": [_P, _P, _P, _I64, _P, _P, _P, _P, _I32, _I64, _I32, _I32, _P, _P, _P,
                           _I64, _I64, _I32, _I32, _P, _P, _P, _I32, _P, _P, _I32],
    "swmd_fused_iteration_f64": [_P, _P, _P, _I64, _P, _P, _I32, _I64, _P, _P, _I64, _P, _P],
    "swmd_fused_final_f64": [_P, _P, _P, _I64, _P, _P, _I32, _I64, _P, _P, _I64, _P, _P],
    "swmd_sddmm_f64": [_P, _P, _P, _P, _I64, _P, _I32, _I64, _P, _P, _I64, _P, _P],
    "swmd_spmm_f64": [_P, _P, _P, _P, _I64, _P, _I32, _I64, _P, _P],
    "swmd_update_u_f64": [_P, _P, _I64, _I32, _P, _P],
    "swmd_unfused_row_width": [_I32],
    "swmd_unfused_iterate_f64": [_P, _P, _P, _I64, _P, _P, _I32, _I64, _P, _P, _I64, _P, _I32,
                                 _I64, _I64, _P, _P],
    "swmd_unfused_final_f64": [_P, _P, _P, _I64, _P, _P, _I32, _I64, _P, _I64, _P, _I32, _I64,
                               _I64, _P, _P],
    "swmd_l2_flush": [_P, _I64, _P],
    "swmd_select_query": [_P, _I64, _P, _I64],
    "swmd_host_copy": [_P, _P, _I64, _I32],
    "swmd_row_norms_f32": [_P, _I64, _I32, _I64, _P, _P],
    "swmd_cost_build_batch_f32": [_P, _I64, _I32, _I64, _P, _P, _I32, ctypes.c_float, _P, _P,
                                  _I64, _P, _P, _P],
    "swmd_solve_f32": [_P, _P, _P, _I64, _P, _P, _P, _P, _I32, _I64, _I32, _I32, _P, _P, _P,
                       _I64, _I64, _I32, _P, _P, _P],
    "swmd_solve_group_f32": [_P, _P, _P, _I64, _P, _I32, _P, _P, _P, _P, _I64, _I32, _P, _P,
                             _I64, _I64, _P, _P],
    "swmd_topk_f64": [_P, _I64, _I32, _I64, _P, _P, _P, _I64, _P],
    "swmd_csr_to_csc_f64": [_P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _I64, _P, _P],
    "swmd_csr_to_csc_scratch_bytes": [_I64],
    "swmd_sample_crc": [_P, _I64, _I64],
    "swmd_content_hash": [_P, _I64, _I32],
    "swmd_topk_scratch_bytes": [_I64, _I32],
    "swmd_plan_create": [_P, _P, _I32],
    "swmd_plan_destroy": [_P],
    "swmd_plan_run": [_P, _P, _I64, _D, _I32, _I32, _P, _P, _P, _P],
    "swmd_plan_run_device": [_P, _P, _I64, _D, _I32, _I32, _P, _P, _P],
    "swmd_plan_run_selected": [_P, _P, _P, _I64, _D, _I32, _I32, _P, _P, _P],
    "swmd_schedule_order": [_P, _I64, _I32, _I32, _I32, _I32, _P],
    "swmd_solve_slots_f64": [_I32, _P],
    "swmd_solve_reg_rounds_f64": [_I32],
}
_RESTYPE = {"swmd_select_query": ctypes.c_int64, "swmd_topk_scratch_bytes": ctypes.c_int64,
            "swmd_csr_to_csc_scratch_bytes": ctypes.c_int64,
            "swmd_sample_crc": ctypes.c_int64, "swmd_content_hash": ctypes.c_int64}

EXPORTED = tuple(_SIGS)


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library and declare every exported signature (no GPU needed)."""
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(path)
    for name, argtypes in _SIGS.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            if os.path.abspath(path) != os.path.abspath(LIB_PATH):
                continue      # an older experiment build (SWMD_LIB): only what it has
            raise
        fn.argtypes = argtypes
        fn.restype = _RESTYPE.get(name, ctypes.c_int)
    return lib


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = load(os.environ.get("SWMD_LIB", LIB_PATH))   # override: build experiments
    return _lib


def lib_or_none():
    try:
        return lib()
    except (NativeUnavailable, OSError):
        return None


def call(name: str, *args) -> None:
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        if rc == EVR:
            raise NativeError(f"{name}: query length outside the supported range (code {rc})")
        if rc == EINVAL:
            raise NativeError(f"{name}: invalid argument (code {rc})")
        raise NativeError(f"{name}: CUDA error {rc}")
