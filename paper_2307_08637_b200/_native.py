"""ctypes binding of liblsort_cuda.so (the C-ABI declared in include/lsort_cuda.h).

The shared library is the product: hand-written sm_100a kernels plus the C++
orchestrator. This module only declares its entry points. There is no
fallback: if the library is missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "liblsort_cuda.so")

LSORT_OK, LSORT_EINVAL, LSORT_ENAN, LSORT_ENOMEM, LSORT_ECUDA, LSORT_ENCCL, LSORT_EINTERNAL, LSORT_EIO = range(8)
KEY_U64, KEY_F64, KEY_ENC_F64 = 0, 1, 2
MEM_DEVICE, MEM_HOST = 0, 1
MAX_TREE = 1024
MAX_RMI = 2048
FLAG_PHASE_TIMING = 1
FLAG_STRICT_POLICY = 2  # reference Alg. 5 models only (no GPU quality fallback)
FLAG_CLUSTER = 4  # experimental fused cluster (DSMEM) last level
FLAG_TEST_DIRECT_OVERFLOW = 8  # test only: force the padded level 0 to overflow
FLAG_TEST_NO_PADDED_MEM = 16  # test only: as if the padded one-pass buffers could not be allocated


class lsort_cfg(C.Structure):
    _fields_ = [
        ("rmi_bucket_count", C.c_uint32), ("tree_bucket_count", C.c_uint32),
        ("min_rmi_input", C.c_uint64), ("max_duplicate_fraction", C.c_double),
        ("radix_base_case", C.c_uint32), ("insertion_base_case", C.c_uint32),
        ("first_sample_cap", C.c_uint32), ("rmi_sample_cap", C.c_uint32),
        ("sample_fraction", C.c_double), ("seed", C.c_uint64), ("workers", C.c_uint32),
        ("base_case_capacity", C.c_uint32), ("bucket_target", C.c_uint32), ("flags", C.c_uint32),
    ]


class lsort_rmi_header(C.Structure):
    _fields_ = [("root_slope", C.c_double), ("root_intercept", C.c_double),
                ("key_base", C.c_double), ("key_scale", C.c_double),
                ("submodels", C.c_uint32), ("reserved", C.c_uint32)]


class lsort_rmi_entry(C.Structure):
    _fields_ = [("slope", C.c_double), ("intercept", C.c_double), ("lo", C.c_double), ("hi", C.c_double)]


class lsort_tree(C.Structure):
    _fields_ = [("levels", C.c_uint32), ("leaf_origin", C.c_uint32), ("nsplitters", C.c_uint32),
                ("bucket_count", C.c_uint32), ("tree", C.c_uint64 * MAX_TREE),
                ("splitters", C.c_uint64 * MAX_TREE), ("eq_offset", C.c_uint32 * (MAX_TREE + 1))]


class lsort_model_info(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("nbuckets", C.c_uint32), ("first_sample", C.c_uint64),
                ("rmi_sample", C.c_uint64), ("duplicate_fraction", C.c_double)]


class lsort_stats(C.Structure):
    _fields_ = [("ms_total", C.c_double), ("ms_h2d", C.c_double), ("ms_d2h", C.c_double),
                ("levels", C.c_uint32), ("level0_kind", C.c_uint32),
                ("partitioned_keys", C.c_uint64), ("base_case_keys", C.c_uint64),
                ("fill_keys", C.c_uint64), ("segments", C.c_uint64), ("base_segments", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("ms_models", C.c_double), ("ms_classify", C.c_double), ("ms_scatter", C.c_double),
                ("ms_base", C.c_double), ("ms_fill", C.c_double), ("ms_level0_classify", C.c_double),
                ("ms_level0_scatter", C.c_double), ("level0_keys", C.c_uint64), ("round2_buckets", C.c_uint64), ("direct_keys", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = [
    "lsort_cfg_default", "lsort_cuda_ctx_create", "lsort_cuda_ctx_destroy", "lsort_cuda_last_error",
    "lsort_cuda_set_stream", "lsort_cuda_sort", "lsort_cuda_sort_batch", "lsort_cuda_sort_many", "lsort_read_keys", "lsort_write_keys", "lsort_cuda_sort_forward", "lsort_cuda_rmi_train", "lsort_cuda_classify_rmi",
    "lsort_cuda_tree_build", "lsort_cuda_classify_tree", "lsort_cuda_build_model",
    "lsort_cuda_block_sort", "lsort_cuda_verify", "lsort_gen_keys", "lsort_cuda_decode_inplace", "lsort_cuda_learned_pivots", "lsort_cuda_pivot_quality", "lsort_cuda_eta",
    "lsort_cuda_sort_buckets", "lsort_nccl_available", "lsort_nccl_unique_id",
    "lsort_cuda_dist_create", "lsort_cuda_dist_destroy", "lsort_cuda_dist_last_error", "lsort_cuda_dist_set_stream",
    "lsort_cuda_sort_dist", "lsort_cuda_dist_result", "lsort_cuda_sort_multi", "lsort_cuda_dist_emulate",
    "lsort_dist_plan", "lsort_cuda_sort_classic", "lsort_cuda_model_counting_sort",
]

_lib = None


def lib():
    """Load liblsort_cuda.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not built: run `python -m paper_2307_08637_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u64, u32, i32, f64 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_double
    P = C.POINTER
    L.lsort_cfg_default.restype = None
    L.lsort_cfg_default.argtypes = [P(lsort_cfg)]
    L.lsort_cuda_ctx_create.restype = i32
    L.lsort_cuda_ctx_create.argtypes = [P(vp), i32, vp, C.c_size_t]
    L.lsort_cuda_ctx_destroy.restype = i32
    L.lsort_cuda_ctx_destroy.argtypes = [vp]
    L.lsort_cuda_last_error.restype = C.c_char_p
    L.lsort_cuda_last_error.argtypes = [vp]
    L.lsort_cuda_set_stream.restype = i32
    L.lsort_cuda_set_stream.argtypes = [vp, vp]
    L.lsort_cuda_sort.restype = i32
    L.lsort_cuda_sort.argtypes = [vp, vp, u64, i32, i32, P(lsort_cfg), P(lsort_stats), P(u64)]
    L.lsort_cuda_sort_classic.restype = i32
    L.lsort_cuda_sort_classic.argtypes = [vp, vp, u64, i32, i32, P(lsort_cfg), P(lsort_stats), P(u64)]
    L.lsort_cuda_model_counting_sort.restype = i32
    L.lsort_cuda_model_counting_sort.argtypes = [vp, P(lsort_rmi_header), vp, f64, f64, vp, u64, vp]
    L.lsort_cuda_sort_forward.restype = i32
    L.lsort_cuda_sort_forward.argtypes = [vp, vp, u64, i32, P(lsort_cfg), P(lsort_rmi_header), vp, C.c_uint32,
                                          C.c_uint32, vp, u64, P(lsort_stats), P(u64)]
    L.lsort_read_keys.restype = i32
    L.lsort_read_keys.argtypes = [C.c_char_p, vp, u64, P(u64), C.c_char_p, C.c_size_t]
    L.lsort_write_keys.restype = i32
    L.lsort_write_keys.argtypes = [C.c_char_p, vp, u64, C.c_char_p, C.c_size_t]
    L.lsort_cuda_sort_many.restype = i32
    L.lsort_cuda_sort_many.argtypes = [vp, P(vp), P(u64), C.c_uint32, i32, P(lsort_cfg), P(lsort_stats), P(u64)]
    L.lsort_cuda_sort_batch.restype = i32
    L.lsort_cuda_sort_batch.argtypes = [vp, P(vp), P(u64), C.c_uint32, i32, P(lsort_cfg), P(lsort_stats),
                                        P(u64)]
    L.lsort_cuda_rmi_train.restype = i32
    L.lsort_cuda_rmi_train.argtypes = [vp, vp, u64, u32, P(lsort_rmi_header), vp]
    L.lsort_cuda_classify_rmi.restype = i32
    L.lsort_cuda_classify_rmi.argtypes = [vp, P(lsort_rmi_header), vp, u32, f64, f64, vp, u64, i32, vp, vp]
    L.lsort_cuda_tree_build.restype = i32
    L.lsort_cuda_tree_build.argtypes = [vp, vp, u64, u32, i32, P(lsort_tree)]
    L.lsort_cuda_classify_tree.restype = i32
    L.lsort_cuda_classify_tree.argtypes = [vp, P(lsort_tree), vp, u64, i32, vp, vp]
    L.lsort_cuda_build_model.restype = i32
    L.lsort_cuda_build_model.argtypes = [vp, vp, u64, i32, P(lsort_cfg), P(lsort_model_info),
                                         P(lsort_rmi_header), vp, P(lsort_tree)]
    L.lsort_cuda_block_sort.restype = i32
    L.lsort_cuda_block_sort.argtypes = [vp, vp, u64]
    L.lsort_cuda_verify.restype = i32
    L.lsort_cuda_verify.argtypes = [vp, vp, u64, i32, P(u64), P(u64)]
    L.lsort_cuda_learned_pivots.restype = i32
    L.lsort_cuda_learned_pivots.argtypes = [vp, P(lsort_rmi_header), vp, u32, vp, u64, i32, vp, vp, P(u32)]
    L.lsort_cuda_pivot_quality.restype = i32
    L.lsort_cuda_pivot_quality.argtypes = [vp, vp, u64, i32, vp, u32, u32, P(f64), vp]
    L.lsort_cuda_eta.restype = i32
    L.lsort_cuda_sort_buckets.restype = i32
    L.lsort_cuda_sort_buckets.argtypes = [vp, vp, u64, i32, P(lsort_cfg), P(lsort_rmi_header), vp, u32, u32, vp, vp,
                                          u64, P(lsort_stats)]
    L.lsort_cuda_eta.argtypes = [vp, vp, u64, i32, u64, P(f64)]
    L.lsort_gen_keys.restype = i32
    L.lsort_gen_keys.argtypes = [i32, u64, u64, u64, u64, vp, i32]
    L.lsort_cuda_decode_inplace.restype = i32
    L.lsort_cuda_decode_inplace.argtypes = [vp, vp, u64]
    # multi-GPU driver (dist.cu)
    L.lsort_nccl_available.restype = i32
    L.lsort_nccl_available.argtypes = []
    L.lsort_nccl_unique_id.restype = i32
    L.lsort_nccl_unique_id.argtypes = [vp]
    L.lsort_cuda_dist_create.restype = i32
    L.lsort_cuda_dist_create.argtypes = [P(vp), i32, i32, i32, vp]
    L.lsort_cuda_dist_destroy.restype = i32
    L.lsort_cuda_dist_destroy.argtypes = [vp]
    L.lsort_cuda_dist_last_error.restype = C.c_char_p
    L.lsort_cuda_dist_last_error.argtypes = [vp]
    L.lsort_cuda_dist_set_stream.restype = i32
    L.lsort_cuda_dist_set_stream.argtypes = [vp, vp]
    L.lsort_cuda_sort_dist.restype = i32
    L.lsort_cuda_sort_dist.argtypes = [vp, vp, u64, i32, vp, u64, P(u64), P(lsort_cfg), P(lsort_stats), P(u64)]
    L.lsort_cuda_dist_result.restype = i32
    L.lsort_cuda_dist_result.argtypes = [vp, P(vp), P(u64)]
    L.lsort_cuda_sort_multi.restype = i32
    L.lsort_cuda_sort_multi.argtypes = [u32, vp, vp, vp, i32, vp, vp, vp, P(lsort_cfg), vp, vp, C.c_char_p,
                                        C.c_size_t]
    L.lsort_cuda_dist_emulate.restype = i32
    L.lsort_cuda_dist_emulate.argtypes = [i32, u32, vp, vp, i32, vp, vp, vp, P(lsort_cfg), vp, vp, C.c_char_p,
                                          C.c_size_t]
    L.lsort_dist_plan.restype = i32
    L.lsort_dist_plan.argtypes = [u32, u32, vp, vp, u32, vp, vp, vp, vp, vp, P(u32)]
    _lib = L
    return L
