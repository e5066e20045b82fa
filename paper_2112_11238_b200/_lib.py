"""ctypes binding of the C-ABI in include/mumode_gpu.h (libmumode_b200.so).

The library is built in-tree for sm_100a (``make -C paper_2112_11238_b200/csrc``
or ``__graft_entry__.build()``). There is no CPU implementation behind this
binding: if the shared object is missing the import fails loudly, and every
compute entry point needs a B200.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libmumode_b200.so"

I64 = ctypes.c_int64
I64P = ctypes.POINTER(ctypes.c_int64)
DP = ctypes.POINTER(ctypes.c_double)
DPP = ctypes.POINTER(DP)
VP = ctypes.c_void_p
H = ctypes.c_void_p

# name -> (restype, argtypes); the complete exported surface of mumode_gpu.h
SIGNATURES = {
    "mumode_handle_create": (ctypes.c_int, [ctypes.POINTER(H), ctypes.c_int]),
    "mumode_handle_destroy": (ctypes.c_int, [H]),
    "mumode_set_stream": (ctypes.c_int, [H, VP]),
    "mumode_get_stream": (VP, [H]),
    "mumode_last_error": (ctypes.c_char_p, []),
    "mumode_version": (ctypes.c_char_p, []),
    "mumode_launch_count": (I64, [H]),
    "mumode_set_kernel_policy": (ctypes.c_int, [H, ctypes.c_int]),
    "mumode_mode_product_f64": (ctypes.c_int, [H, ctypes.c_int, I64P, ctypes.c_int, I64, VP, VP, VP]),
    "mumode_mode_product_c128": (ctypes.c_int, [H, ctypes.c_int, I64P, ctypes.c_int, I64, VP, VP, VP]),
    "mumode_tucker_f64": (ctypes.c_int, [H, ctypes.c_int, I64P, I64P, VP, ctypes.POINTER(VP), VP, ctypes.c_int]),
    "mumode_tucker_c128": (ctypes.c_int, [H, ctypes.c_int, I64P, I64P, VP, ctypes.POINTER(VP), VP, ctypes.c_int]),
    "mumode_tucker_promote": (ctypes.c_int, [H, ctypes.c_int, I64P, I64P, VP, ctypes.POINTER(VP), VP, ctypes.c_int]),
    "mumode_tucker_range_f64": (ctypes.c_int, [H, ctypes.c_int, I64P, I64P, VP, ctypes.POINTER(VP), VP, ctypes.c_int, ctypes.c_int]),
    "mumode_tucker_range_scatter_f64": (ctypes.c_int, [H, ctypes.c_int, I64P, I64P, VP, ctypes.POINTER(VP), ctypes.c_int,
                                                       ctypes.c_int, ctypes.c_int, I64P, I64, ctypes.POINTER(VP)]),
    "mumode_tucker_range_scatter_c128": (ctypes.c_int, [H, ctypes.c_int, I64P, I64P, VP, ctypes.POINTER(VP), ctypes.c_int,
                                                        ctypes.c_int, ctypes.c_int, I64P, I64, ctypes.POINTER(VP)]),
    "mumode_slab_pack_f64": (ctypes.c_int, [H, I64, I64, ctypes.c_int, I64P, VP, VP]),
    "mumode_slab_unpack_f64": (ctypes.c_int, [H, I64, I64, ctypes.c_int, I64P, VP, VP]),
    "mumode_comm_unique_id": (ctypes.c_int, [VP]),
    "mumode_comm_create": (ctypes.c_int, [ctypes.POINTER(VP), ctypes.c_int, VP, ctypes.c_int, ctypes.c_int]),
    "mumode_comm_wrap": (ctypes.c_int, [ctypes.POINTER(VP), ctypes.c_int, VP, ctypes.c_int, ctypes.c_int]),
    "mumode_comm_destroy": (ctypes.c_int, [VP]),
    "mumode_comm_set_exchange": (ctypes.c_int, [VP, ctypes.c_int]),
    "mumode_comm_set_overlap_sms": (ctypes.c_int, [VP, ctypes.c_int]),
    "mumode_comm_create_local": (ctypes.c_int, [ctypes.POINTER(VP), ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "mumode_comm_ipc_handle_bytes": (ctypes.c_int, []),
    "mumode_comm_ipc_export": (ctypes.c_int, [VP, ctypes.c_int, I64P, I64P, ctypes.c_int, VP]),
    "mumode_comm_ipc_import": (ctypes.c_int, [VP, ctypes.c_int, I64P, I64P, ctypes.c_int, VP]),
    "mumode_comm_poll": (ctypes.c_int, [H, VP, I64]),
    "mumode_dist_local_f64": (ctypes.c_int, [H, ctypes.c_int, ctypes.c_int, ctypes.c_int, I64P, I64P, VP,
                                             ctypes.POINTER(VP), VP, VP, ctypes.c_int]),
    "mumode_dist_tucker_phase_f64": (ctypes.c_int, [H, VP, ctypes.c_int, I64P, I64P, VP, ctypes.POINTER(VP), VP, ctypes.c_int]),
    "mumode_dist_tucker_phase_c128": (ctypes.c_int, [H, VP, ctypes.c_int, I64P, I64P, VP, ctypes.POINTER(VP), VP, ctypes.c_int]),
    "mumode_slab_plan": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, I64P, I64P, I64P, I64P]),
    "mumode_dist_plan": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, I64P, I64P, ctypes.c_int, ctypes.c_int,
                                        I64P, ctypes.c_int, ctypes.POINTER(ctypes.c_int), I64P, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_int)]),
    "mumode_dist_return_plan": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, I64P, I64P, ctypes.c_int,
                                               ctypes.POINTER(ctypes.c_int)]),
    "mumode_dist_expint_f64": (ctypes.c_int, [H, VP, ctypes.c_int, I64P, ctypes.POINTER(VP), VP, VP, ctypes.c_int]),
    "mumode_dist_tucker_f64": (ctypes.c_int, [H, VP, ctypes.c_int, I64P, I64P, VP, ctypes.POINTER(VP), VP, ctypes.c_int]),
    "mumode_dist_tucker_c128": (ctypes.c_int, [H, VP, ctypes.c_int, I64P, I64P, VP, ctypes.POINTER(VP), VP, ctypes.c_int]),
    "mumode_kronsumv_f64": (ctypes.c_int, [H, ctypes.c_int, I64P, VP, ctypes.POINTER(VP), VP]),
    "mumode_kronsumv_c128": (ctypes.c_int, [H, ctypes.c_int, I64P, VP, ctypes.POINTER(VP), VP]),
    "mumode_expint_f64": (ctypes.c_int, [H, ctypes.c_int, I64P, ctypes.POINTER(VP), VP, VP, ctypes.c_int]),
    "mumode_kronsum_solve_f64": (ctypes.c_int, [H, ctypes.c_int, I64P, ctypes.POINTER(VP), ctypes.POINTER(VP), ctypes.POINTER(VP), VP, VP]),
    "mumode_host_mode_product_f64": (ctypes.c_int, [H, ctypes.c_int, I64P, ctypes.c_int, I64, VP, VP, VP]),
    "mumode_host_mode_product_c128": (ctypes.c_int, [H, ctypes.c_int, I64P, ctypes.c_int, I64, VP, VP, VP]),
    "mumode_host_tucker_f64": (ctypes.c_int, [H, ctypes.c_int, I64P, I64P, VP, ctypes.POINTER(VP), VP, ctypes.c_int]),
    "mumode_host_tucker_f64_async": (ctypes.c_int, [H, ctypes.c_int, I64P, I64P, VP, ctypes.POINTER(VP), VP]),
    "mumode_host_wait": (ctypes.c_int, [H]),
    "mumode_host_tucker_c128": (ctypes.c_int, [H, ctypes.c_int, I64P, I64P, VP, ctypes.POINTER(VP), VP, ctypes.c_int]),
    "mumode_host_tucker_promote": (ctypes.c_int, [H, ctypes.c_int, I64P, I64P, VP, ctypes.POINTER(VP), VP, ctypes.c_int]),
    "mumode_host_kronsumv_f64": (ctypes.c_int, [H, ctypes.c_int, I64P, VP, ctypes.POINTER(VP), VP]),
    "mumode_host_kronsumv_c128": (ctypes.c_int, [H, ctypes.c_int, I64P, VP, ctypes.POINTER(VP), VP]),
    "mumode_host_expint_f64": (ctypes.c_int, [H, ctypes.c_int, I64P, ctypes.POINTER(VP), VP, VP, ctypes.c_int]),
    "mumode_probe_fp64_peak": (ctypes.c_int, [H, ctypes.POINTER(ctypes.c_double)]),
    "mumode_expm_f64": (ctypes.c_int, [I64, VP, VP]),
    "mumode_inverse_f64": (ctypes.c_int, [I64, VP, VP]),
    "mumode_lu_factor_f64": (ctypes.c_int, [I64, VP, VP, VP]),
    "mumode_lu_factor_c128": (ctypes.c_int, [I64, VP, VP, VP]),
    "mumode_itucker_f64": (ctypes.c_int, [H, ctypes.c_int, I64P, VP, ctypes.POINTER(VP), ctypes.POINTER(VP), VP]),
    "mumode_itucker_c128": (ctypes.c_int, [H, ctypes.c_int, I64P, VP, ctypes.POINTER(VP), ctypes.POINTER(VP), VP]),
    "mumode_host_itucker_f64": (ctypes.c_int, [H, ctypes.c_int, I64P, VP, ctypes.POINTER(VP), ctypes.POINTER(VP), VP]),
    "mumode_host_itucker_c128": (ctypes.c_int, [H, ctypes.c_int, I64P, VP, ctypes.POINTER(VP), ctypes.POINTER(VP), VP]),
    "mumode_extract_tridiag_f64": (ctypes.c_int, [I64, VP, VP, VP]),
    "mumode_symtridiag_eig_f64": (ctypes.c_int, [I64, VP, VP, VP, VP]),
    "mumode_rng_create": (ctypes.c_int, [ctypes.POINTER(VP), ctypes.c_uint64]),
    "mumode_rng_destroy": (ctypes.c_int, [VP]),
    "mumode_rng_normal": (ctypes.c_int, [VP, VP, I64, ctypes.c_int]),
    "mumode_rng_u64": (ctypes.c_int, [VP, VP, I64]),
}

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is not built; run __graft_entry__.build() or "
                "`make -C paper_2112_11238_b200/csrc`. The mu-mode engine has no CPU fallback.")
        so = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(so, name)
            fn.restype = res
            fn.argtypes = args
        _lib = so
    return _lib


def i64_array(vals) -> ctypes.Array:
    vals = [int(v) for v in vals]
    return (ctypes.c_int64 * max(1, len(vals)))(*vals)


def ptr_array(ptrs) -> ctypes.Array:
    return (VP * max(1, len(ptrs)))(*[VP(int(p)) for p in ptrs])
