"""ctypes binding of librsc_b200.so (the C ABI declared in include/rsc_b200.h).

The product path has no CPU fallback: importing a compute entry point without the
built library, or calling it without a CUDA device, raises immediately.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RSC_B200_LIB", os.path.join(_HERE, "librsc_b200.so"))  # override: experiments only

# numpy mirror of rsc_gemm_problem (include/rsc_b200.h); 128 bytes, naturally aligned
GEMM_DTYPE = np.dtype(
    [
        ("A", "u8"), ("B", "u8"), ("C", "u8"),
        ("sA", "i8"), ("sB", "i8"), ("sC", "i8"),
        ("b_rows", "u8"), ("c_rows", "u8"), ("c_cols", "u8"),
        ("M", "i4"), ("N", "i4"), ("K", "i4"),
        ("lda", "i4"), ("ldb", "i4"), ("ldc", "i4"),
        ("batch", "i4"), ("atomic", "i4"),
        ("alpha", "f8"), ("beta", "f8"),
        ("ext_r", "i4"), ("ext_c", "i4"),
    ]
)
assert GEMM_DTYPE.itemsize == 128

# every symbol include/rsc_b200.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "rsc_gemm_grouped",
    "rsc_gemm_grouped_balanced",
    "rsc_gemm_set_workspace",
    "rsc_potrf_batched",
    "rsc_trsm_batched",
    "rsc_trsm_right_batched",
    "rsc_trtri_diag_batched",
    "rsc_qrcp_workspace_bytes",
    "rsc_qrcp_batched",
    "rsc_csr_to_dense_batched",
    "rsc_spmm_csr",
    "rsc_spmm_csr_batched",
    "rsc_spmv_csr",
    "rsc_trsv_batched",
    "rsc_gemv_batched",
    "rsc_gemv_multi",
    "rsc_gemv_desc_bytes",
    "rsc_gemv_describe",
    "rsc_gemv_multi_dev",
    "rsc_apply_tasks",
    "rsc_apply_cluster_tasks",
    "rsc_flow_describe",
    "rsc_apply_flow",
    "rsc_apply_flow_trace",
    "rsc_flow_deps",
    "rsc_identity_batched",
    "rsc_transpose_batched",
    "rsc_copy2d_batched",
    "rsc_gather_rows",
    "rsc_scatter_add_rows",
    "rsc_dot",
    "rsc_pcg_update_xr",
    "rsc_pcg_update_p",
    "rsc_sym_etree",
    "rsc_sym_etree_par",
    "rsc_sym_postorder",
    "rsc_sym_colcounts",
    "rsc_sym_amalgamate",
    "rsc_sym_rows_compute",
    "rsc_sym_rows_compute_par",
    "rsc_sym_rows_fetch",
    "rsc_sym_full_csr",
    "rsc_sym_permute_lower",
    "rsc_nd_split_geometric",
    "rsc_nd_geometric",
    "rsc_csr_windows",
    "rsc_plan_pairs",
    "rsc_hash64",
    "rsc_plan_pairs_fetch",
    "rsc_plan_tree_maps",
    "rsc_plan_tree_maps_fetch",
    "rsc_pcg64_block_states",
    "rsc_pcg64_seed_states",
    "rsc_normal_workspace_bytes",
    "rsc_normal_pcg64",
    "rsc_log1p_fdlibm",
    "rsc_normal_debug_limits",
    "rsc_schur_update",
    "rsc_offdiag_products",
    "rsc_interior_factor_batched",
    "rsc_tree_trsm",
    "rsc_apply_sweep",
    "rsc_nccl_available",
    "rsc_nccl_unique_id",
    "rsc_nccl_comm_init",
    "rsc_nccl_allreduce_sum_f64",
    "rsc_nccl_broadcast_f64",
    "rsc_nccl_comm_destroy",
    "rsc_launch_counter",
    "rsc_version",
    "rsc_device_arch",
)

_lib = None

P = ctypes.c_void_p
I = ctypes.c_int
D = ctypes.c_double
LL = ctypes.c_longlong

_SIGS = {
    "rsc_gemm_grouped": (I, [I, I, P, I, P]),
    "rsc_gemm_grouped_balanced": (I, [I, I, P, I, I, P]),
    "rsc_gemm_set_workspace": (I, [P, P, LL, I]),
    "rsc_potrf_batched": (I, [I, P, P, P, P, P, P]),
    "rsc_trsm_batched": (I, [I, I, I, P, P, P, P, P, P, P, P]),
    "rsc_trsm_right_batched": (I, [I, P, P, P, P, P, P, P, P, P]),
    "rsc_trtri_diag_batched": (I, [I, P, P, P, P, P]),
    "rsc_qrcp_workspace_bytes": (LL, [I, P, P]),
    "rsc_qrcp_batched": (I, [I, P, P, P, P, P, P, P, P, P]),
    "rsc_csr_to_dense_batched": (I, [I, P, P, P, P, P, P, P]),
    "rsc_spmm_csr": (I, [I, I, P, P, P, P, I, D, D, P, I, P]),
    "rsc_spmm_csr_batched": (I, [I, P, P, P, P, P, P, P, D, D, P, P, P]),
    "rsc_spmv_csr": (I, [I, P, P, P, P, P, P]),
    "rsc_trsv_batched": (I, [I, P, P, P, P, P, I, P]),
    "rsc_gemv_batched": (I, [I, P, P, P, P, P, P, P, P, I, D, P]),
    "rsc_gemv_multi": (I, [I, P, P, P, P, P, P, P, P, P, P, P]),
    "rsc_gemv_desc_bytes": (I, []),
    "rsc_gemv_describe": (I, [I, P, P, P, P, P, P, P, P, P, P, P, P]),
    "rsc_gemv_multi_dev": (I, [P, P, LL, P]),
    "rsc_apply_tasks": (I, [P, P, I, P]),
    "rsc_apply_cluster_tasks": (I, [P, P, I, I, P]),
    "rsc_flow_describe": (LL, [I, P, P, P, P, P, P, P, P, P, P, P, P]),
    "rsc_apply_flow": (I, [P, P, P, P, P, P, I, I, P]),
    "rsc_apply_flow_trace": (I, [P, P, P, P, P, P, I, I, P, P]),
    "rsc_flow_deps": (LL, [I, P, P, P, P, P, P, P, I, P, P, P, LL, LL, P, P, P, LL]),

    "rsc_gather_rows": (I, [I, I, P, P, I, P, I, P]),
    "rsc_identity_batched": (I, [I, P, P, P, P]),
    "rsc_transpose_batched": (I, [I, P, P, P, P, P, P]),
    "rsc_copy2d_batched": (I, [I, P, P, P, P, P, P, I, P]),
    "rsc_scatter_add_rows": (I, [I, I, P, D, P, I, P, I, P]),
    "rsc_dot": (I, [I, P, P, P, P, P]),
    "rsc_pcg_update_xr": (I, [I, P, P, P, P, P, P, P]),
    "rsc_pcg_update_p": (I, [I, P, P, P, P, P]),
    "rsc_sym_etree": (I, [LL, P, P, P]),
    "rsc_sym_etree_par": (I, [LL, P, P, LL, P, P]),
    "rsc_sym_postorder": (I, [LL, P, P]),
    "rsc_sym_colcounts": (I, [LL, P, P, P, P, P]),
    "rsc_sym_amalgamate": (LL, [LL, P, P, P, I, P, P, P]),
    "rsc_sym_rows_compute": (ctypes.c_void_p, [LL, P, P, P, P]),
    "rsc_sym_rows_compute_par": (ctypes.c_void_p, [LL, P, P, P, LL, P, P]),
    "rsc_sym_rows_fetch": (I, [ctypes.c_void_p, P, P]),
    "rsc_sym_full_csr": (LL, [LL, P, P, P, I, P, P, P]),
    "rsc_sym_permute_lower": (I, [LL, P, P, P, P, P, P]),
    "rsc_nd_split_geometric": (I, [LL, P, ctypes.c_int, P, P, P, P, P, P]),
    "rsc_nd_geometric": (LL, [LL, ctypes.c_int, P, P, P, LL, P, LL, P, P, P, P, P, P, P]),
    "rsc_csr_windows": (I, [LL, LL] + [P] * 16),
    "rsc_hash64": (ctypes.c_ulonglong, [P, LL]),
    "rsc_plan_pairs": (ctypes.c_void_p, [LL, P, P, P, LL, P, P, P, P, P, P]),
    "rsc_plan_pairs_fetch": (I, [ctypes.c_void_p] + [P] * 7),
    "rsc_plan_tree_maps": (ctypes.c_void_p, [LL, P, P, P, P, P, P, P, P]),
    "rsc_plan_tree_maps_fetch": (I, [ctypes.c_void_p, P, P]),
    "rsc_pcg64_block_states": (I, [I, I, P, P, P, P]),
    "rsc_pcg64_seed_states": (I, [I, P, P]),
    "rsc_normal_workspace_bytes": (ctypes.c_size_t, [I, P]),
    "rsc_normal_pcg64": (I, [I, P, P, P, P, ctypes.c_size_t, P]),
    "rsc_log1p_fdlibm": (D, [D]),
    "rsc_normal_debug_limits": (I, [I, I]),
    "rsc_schur_update": (I, [P, I, I, P, I, I, I] + [P] * 10),
    "rsc_offdiag_products": (I, [I, P, I, I, I, P, I, I, I] + [P] * 11),
    "rsc_interior_factor_batched": (I, [I] + [P] * 9),
    "rsc_tree_trsm": (I, [I, I, I] + [P] * 16 + [I, I, P, P]),
    "rsc_apply_sweep": (I, [I] + [P] * 12),
    "rsc_nccl_available": (I, []),
    "rsc_nccl_unique_id": (I, [P]),
    "rsc_nccl_comm_init": (I, [I, P, I, P]),
    "rsc_nccl_allreduce_sum_f64": (I, [P, P, P, LL, P]),
    "rsc_nccl_broadcast_f64": (I, [P, P, P, LL, I, P]),
    "rsc_nccl_comm_destroy": (I, [P]),
    "rsc_launch_counter": (LL, [I]),
    "rsc_version": (ctypes.c_char_p, []),
    "rsc_device_arch": (I, []),
}


class NativeLibraryMissing(RuntimeError):
    """librsc_b200.so is not built (run __graft_entry__.build())."""


def load():
    """Load (once) and return the native library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} not found; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed with status {rc}")


def ptr_array(ptrs):
    """Host array of device pointers (uint64) for the batched entry points."""
    return np.ascontiguousarray(np.asarray(ptrs, dtype=np.uint64))


def int_array(vals):
    return np.ascontiguousarray(np.asarray(vals, dtype=np.int32))


def addr(a):
    """ctypes address of a host numpy array (or None)."""
    return None if a is None else a.ctypes.data
