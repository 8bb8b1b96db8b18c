"""ctypes binding of libbbsi_cuda.so (C ABI: include/bbsi_cuda.h).

There is no fallback: if the library is missing or exports are absent this
module raises at import / first use.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("BBSI_LIB") or Path(__file__).resolve().parent / "_lib" / "libbbsi_cuda.so")

# Every symbol include/bbsi_cuda.h declares, with its ctypes signature.
_vp, _ip, _i, _ll, _d = C.c_void_p, C.POINTER(C.c_int), C.c_int, C.c_longlong, C.c_double
SIGNATURES = {
    "bbsi_cuda_version": (_i, []),
    "bbsi_cuda_last_error": (C.c_char_p, []),
    "bbsi_cuda_device_count": (_i, []),
    "bbsi_cuda_release_workspace": (None, []),
    "bbsi_cuda_rgf_tridiag_z": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_rgf_ndiag_z": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_rgf_fused_z": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_rgf_extended_z": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_ddrgf_z": (_i, [_i, _i, _i, _vp, _vp, _vp, _i, _i, _i, _vp, _vp, _vp]),
    "bbsi_cuda_rgf_batched_dev": (_i, [_i, _i, _i, _i, _vp, _ll, _vp, _vp, _vp]),
    "bbsi_cuda_dyson_rgf_dev": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_dyson_fill_h_dev": (_i, [_i, _i, _i, C.c_uint64, _vp, _vp]),
    "bbsi_dyson_fill_h_host": (None, [_i, _i, _i, C.c_uint64, _vp]),
    "bbsi_cuda_dyson_fill_h_rows_dev": (_i, [_i, _i, _i, C.c_uint64, _i, _i, _vp, _vp]),
    "bbsi_random_spd_like_z": (_i, [_i, _i, _i, _vp, C.c_uint64, _d, _vp]),
    "bbsi_cuda_zgemm_dev": (_i, [_i, _i, _i, _vp, _vp, _ll, _ll, _vp, _ll, _ll, _vp, _vp, _ll, _ll, _i, _vp]),
    "bbsi_cuda_zinv_dev": (_i, [_i, _i, _i, _vp, _ll, _ll, _vp, _vp]),
    "bbsi_cuda_dyson_rgf_z": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _i]),
    "bbsi_cuda_ddrgf_dev": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_dyson_ddrgf_dev": (_i, [_i, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp]),
    "bbsi_cuda_ddrgf_plan_dev": (_i, [_i, _i, _vp, _i, _vp, _vp, _vp, _vp]),
    "bbsi_ddrgf_reference_counters": (None, [_ll, _vp, _i, _vp]),
    "bbsi_cuda_ddrgf_num_tasks": (_i, [_i, _i]),
    "bbsi_cuda_ddrgf_packet_bytes": (_ll, [_i, _i]),
    "bbsi_cuda_ddrgf_phase2_bytes": (_ll, [_i, _i]),
    "bbsi_cuda_ddrgf_phase1_dev": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_ddrgf_phase2_dev": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_ddrgf_phase3_dev": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_ddrgf_halo_dev": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _vp]),
    "bbsi_cuda_ddrgf_couplings_dev": (_i, [_i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_nccl_available": (_i, []),
    "bbsi_cuda_nccl_unique_id": (_i, [_vp]),
    "bbsi_cuda_nccl_comm_init": (_i, [_vp, _i, _i, _vp]),
    "bbsi_cuda_nccl_comm_destroy": (None, [_vp]),
    "bbsi_cuda_ddrgf_rank_layers": (_i, [_i, _i, _i, _i, _ip, _ip, _ip, _ip]),
    "bbsi_cuda_ddrgf_rank_dev": (_i, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_ddrgf_rank_plan_dev": (_i, [_vp, _i, _i, _vp, _i, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_ddrgf_multi_z": (_i, [_i, _i, _i, _vp, _vp, _vp, _i, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_dyson_rgf_multi_z": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp]),
    "bbsi_cuda_rgf_many_z": (_i, [_i, _i, _i, _vp, _i, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_dyson_rgf_sigma_dev": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bbsi_cuda_launch_count": (_ll, []),
    "bbsi_cuda_profile_enable": (None, [_i]),
    "bbsi_cuda_profile_collect": (_i, [_vp, _i]),
    "bbsi_cuda_fp64_peak_tflops": (_d, [_d, _i]),
    "bbsi_cuda_bench_kernels": (_i, [_i, _i, _i, _vp]),
}

_lib = None


def lib():
    """Loads the native library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the bbsi GPU path has no CPU fallback)")
        lib_ = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib_, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib_
    return _lib


def last_error() -> str:
    return lib().bbsi_cuda_last_error().decode()
