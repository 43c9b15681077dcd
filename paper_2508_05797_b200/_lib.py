"""ctypes loader for libcdc_b200.so (the C ABI of include/cdc_b200.h).

The library is the product: there is no CPU fallback.  If the shared object is
missing, importing the package raises.
"""
from __future__ import annotations

import ctypes
import os

from .build import LIB

# CDC_LIB selects another build of the same library (tuning variants under build/)
_DEFAULT_LIB = LIB
LIB = os.environ.get("CDC_LIB", LIB)
if not os.path.exists(LIB):
    raise ImportError(
        f"{LIB} is missing: build it with `python paper_2508_05797_b200/build.py` "
        "(or __graft_entry__.build()); there is no CPU fallback")

lib = ctypes.CDLL(LIB)


class cdc_params(ctypes.Structure):
    _fields_ = [
        ("algo", ctypes.c_int32),
        ("window", ctypes.c_uint32),
        ("max_size", ctypes.c_uint64),
        ("seg_bytes", ctypes.c_uint64),
        ("halo_bytes", ctypes.c_uint64),
    ]


_P = ctypes.POINTER(cdc_params)
_u64, _u32, _i32, _vp, _sz = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t

SIGNATURES = {
    "cdc_abi_version": ([], ctypes.c_int),
    "cdc_last_error": ([], ctypes.c_char_p),
    "cdc_last_launch_count": ([], ctypes.c_int),
    "cdc_window_for_avg": ([_i32, _u64, ctypes.POINTER(_u32)], ctypes.c_int),
    "cdc_params_default": ([_P, _i32, _u64], ctypes.c_int),
    "cdc_max_boundaries": ([_P, _u64], _u64),
    "cdc_workspace_size": ([_P, _u64, _u64, _u64, ctypes.POINTER(_sz)], ctypes.c_int),
    "cdc_chunk": ([_P, _vp, _u64, _vp, _u64, _vp, _vp, _sz, _vp], ctypes.c_int),
    "cdc_chunk_batch": ([_P, _vp, _vp, _u64, _u64, _u64, _vp, _u64, _vp, _vp, _vp, _sz, _vp], ctypes.c_int),
    "cdc_chunk_host": ([_P, _vp, _u64, _vp, _u64, ctypes.POINTER(_u64)], ctypes.c_int),
    "cdc_chunk_batch_host": ([_P, _vp, _vp, _u64, _vp, _u64, _vp, ctypes.POINTER(_u64)], ctypes.c_int),
    "cdc_plan_segments": ([_P, _u64, _vp, _u64, ctypes.POINTER(_u64)], ctypes.c_int),
    "cdc_chain": ([_P, _vp, _u64, _u64, _u64, _vp, _u64, _vp, _vp], ctypes.c_int),
    "cdc_first_common": ([_vp, _u64, _vp, _u64, _vp, _vp], ctypes.c_int),
    "cdc_extreme_byte_search": ([_vp, _vp, _vp, _u64, _i32, _vp, _vp, _vp], ctypes.c_int),
    "cdc_range_scan": ([_vp, _vp, _vp, _vp, _u64, _i32, _vp, _vp], ctypes.c_int),
    "cdc_profile_enable": ([ctypes.c_int], ctypes.c_int),
    "cdc_profile_query": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "cdc_debug_timing": ([_vp], ctypes.c_int),
    "cdc_plan_info": ([_P, _u64, _u64, _u64, ctypes.POINTER(_u64)], ctypes.c_int),
    "cdc_stats": ([_P, _u64, _u64, _u64, _vp, ctypes.POINTER(_u64), _vp], ctypes.c_int),
    "cdc_fetched": ([_P, _u64, _u64, _u64, _vp, ctypes.POINTER(_u64), _vp], ctypes.c_int),
    "cdc_set_kphase": ([ctypes.c_int], ctypes.c_int),
    "cdc_set_dense": ([ctypes.c_int], ctypes.c_int),
    "cdc_profile_collect": ([ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_u64), ctypes.POINTER(_u64)],
                            ctypes.c_int),
}

for _name, (_args, _res) in SIGNATURES.items():
    if LIB != _DEFAULT_LIB and not hasattr(lib, _name):
        continue  # an older tuning build under build/ (CDC_LIB) may lack newer entry points
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res


class CdcError(RuntimeError):
    pass


def check(rc: int) -> None:
    if rc != 0:
        raise CdcError(f"cdc error {rc}: {lib.cdc_last_error().decode()}")
