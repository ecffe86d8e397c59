"""ctypes binding of the C ABI in include/featgrind_b200.h.

This is the same binding a host application would write against the shared
library.  It loads the in-tree ``libfgb200.so`` and fails
loudly when it is missing: there is no CPU fallback for any op.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import DataError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfgb200.so")

FG_OK, FG_EUSAGE, FG_EDATA, FG_ECUDA = 0, 1, 2, 3
OUT_F32, OUT_BF16, OUT_F64 = 0, 1, 2
CODEC_SQ, CODEC_VQ = 1, 2
METRIC_EUCLIDEAN, METRIC_COSINE = 0, 1
RNG_WORDS = 264

vp = C.c_void_p
i32, i64, u64, u32 = C.c_int32, C.c_int64, C.c_uint64, C.c_uint32
ci = C.c_int


class CodecDesc(C.Structure):
    """Mirror of ``fg_codec_desc``."""
    _fields_ = [("kind", i32), ("bits", i32), ("n", i64), ("d", i64),
                ("row_stride", i64), ("rows", vp), ("table", vp),
                ("width", i32), ("length", i32), ("num_parts", i32),
                ("elem_bits", i32), ("table_lp", vp), ("table_h", vp), ("part_scale", vp)]


_SIGS = {
    "fg_last_error": (C.c_char_p, []),
    "fg_version": (ci, []),
    "fg_launch_count": (i64, []),
    "fg_sm_count": (ci, [C.POINTER(ci)]),
    "fg_set_l2_fetch_granularity": (ci, [ci]),
    "fg_get_l2_fetch_granularity": (ci, [C.POINTER(ci)]),
    "fg_stream_to_rows": (ci, [vp, i64, i64, i64, vp, i64, vp]),
    "fg_rows_to_stream": (ci, [vp, i64, i64, i64, vp, i64, vp]),
    "fg_bits_pack": (ci, [vp, i64, ci, vp, vp, vp]),
    "fg_bits_unpack": (ci, [vp, i64, i64, i64, ci, vp, vp]),
    "fg_bit_rows_gather": (ci, [vp, i64, i64, vp, i64, vp, vp, vp]),
    "fg_sq_encode": (ci, [vp, ci, i64, i64, ci, vp, vp, vp, i64, vp]),
    "fg_sq_gather_dequant": (ci, [C.POINTER(CodecDesc), vp, ci, i64, vp, ci, vp, vp]),
    "fg_count_nonzero": (ci, [vp, i64, vp, vp]),
    "fg_gather_nonzero_sample": (ci, [vp, i64, i64, i64, vp, vp, i64, vp]),
    "fg_nonzero_sample_workspace_bytes": (i64, [i64]),
    "fg_gather_nonzero_sample_chunk": (ci, [vp, i64, i64, i64, i64, vp, vp, i64, vp]),
    "fg_select_ranks": (ci, [vp, i64, C.POINTER(i64), ci, C.POINTER(C.c_float), vp, i64, vp]),
    "fg_select_workspace_bytes": (i64, []),
    "fg_vq_assign": (ci, [vp, ci, i64, i64, ci, ci, ci, vp, vp, ci, ci, vp, i64, vp, vp]),
    "fg_vq_assign_fp64": (ci, [vp, ci, i64, i64, ci, ci, ci, vp, vp, ci, ci, vp, i64, vp, vp]),
    "fg_codes_to_rows": (ci, [vp, i64, ci, ci, vp, i64, vp]),
    "fg_segment_sums": (ci, [vp, i64, ci, vp, vp, ci, vp, vp, vp]),
    "fg_kmeanspp_batched": (ci, [vp, vp, vp, i64, i64, ci, ci, vp, vp, vp, vp, vp, vp]),
    "fg_vq_gather_decode": (ci, [C.POINTER(CodecDesc), vp, ci, i64, vp, ci, vp, vp]),
    "fg_kmeans_assign": (ci, [vp, i64, ci, vp, ci, ci, vp, vp, vp, vp]),
    "fg_kmeans_assign_tc": (ci, [vp, i64, ci, vp, ci, ci, vp, vp, vp]),
    "fg_gather_dequant_mean": (ci, [C.POINTER(CodecDesc), vp, vp, vp, i64, vp, i64, ci, vp]),
    "fg_gather_dequant_wsum": (ci, [C.POINTER(CodecDesc), vp, vp, vp, vp, i64, vp, i64, ci,
                                    vp]),
    "fg_block_edge_weights": (ci, [ci, vp, vp, vp, vp, vp, i64, vp, vp]),
    "fg_block_mean_fwd": (ci, [vp, i64, vp, vp, vp, i64, vp, i64, ci, vp, vp]),
    "fg_block_mean_fwd_bits": (ci, [vp, i64, vp, vp, vp, i64, vp, i64, vp, vp, vp]),
    "fg_input_block_mean_supported": (ci, [i64, i64, i64]),
    "fg_input_block_mean_fwd": (ci, [vp, i64, vp, i64, vp, vp, vp, i64, i64, vp, vp, i64, vp,
                                     vp]),
    "fg_block_mean_bwd": (ci, [vp, i64, vp, vp, vp, i64, vp, vp]),
    "fg_f32_to_bf16": (ci, [vp, i64, vp, vp, vp]),
    "fg_block_transpose_scratch_bytes": (i64, [i64]),
    "fg_block_transpose": (ci, [vp, vp, i64, vp, vp, i64, ci, i64, vp, vp, vp, vp, vp, i64, vp]),
    "fg_block_transpose_ex": (ci, [vp, vp, i64, vp, vp, i64, ci, i64, vp, vp, vp, vp, vp, vp, i64,
                                   vp]),
    "fg_block_mean_bwd_t": (ci, [vp, i64, i64, vp, vp, vp, vp, i64, vp, vp, vp]),
    "fg_block_mean_bwd_t_bits": (ci, [vp, i64, i64, vp, vp, vp, vp, i64, vp, vp, vp]),
    "fg_block_mean_wgrad_supported": (ci, [i64, i64]),
    "fg_block_mean_wgrad_scratch_bytes": (i64, [i64, i64]),
    "fg_block_mean_wgrad": (ci, [vp, i64, vp, vp, vp, i64, vp, vp, ci, i64, vp, i64, vp, vp,
                                 i64, vp]),
    "fg_relu_mask_bits": (ci, [vp, i64, i64, vp, vp]),
    "fg_gat_softmax_fwd": (ci, [vp, vp, i64, vp, vp, i64, vp, ci, C.c_float, vp, vp, vp]),
    "fg_gat_softmax_bwd": (ci, [vp, i64, vp, vp, vp, vp, vp, i64, vp, ci, C.c_float, vp, vp, vp]),
    "fg_gat_agg_fwd": (ci, [vp, i64, ci, vp, vp, vp, i64, vp, vp, vp]),
    "fg_gat_agg_bwd": (ci, [vp, i64, ci, vp, vp, vp, i64, vp, vp, vp, vp, vp]),
    "fg_gat_xagg_fwd": (ci, [vp, i64, ci, vp, vp, i64, vp, vp, vp]),
    "fg_gat_xagg_bwd": (ci, [vp, i64, ci, vp, i64, vp, vp, vp, i64, vp]),
    "fg_gat_code_scores": (ci, [C.POINTER(CodecDesc), vp, vp, vp, i64, i64, ci, vp, vp, vp, vp]),
    "fg_gat_code_scores_bwd_blocks": (i64, [i64]),
    "fg_gat_code_scores_bwd": (ci, [C.POINTER(CodecDesc), vp, vp, vp, i64, i64, ci, vp, vp, i64,
                                    vp, vp]),
    "fg_gat_code_xagg_fwd": (ci, [C.POINTER(CodecDesc), vp, vp, i64, ci, vp, vp, i64, vp, vp,
                                  i64, vp]),
    "fg_gat_elu_fwd": (ci, [vp, ci, i64, vp, i64, i64, vp, vp]),
    "fg_cat_rows_bf16": (ci, [vp, i64, vp, i64, i64, vp, i64, vp]),
    "fg_gat_agg_bwd_t_supported": (ci, [i64, ci]),
    "fg_gat_agg_bwd_t": (ci, [vp, i64, ci, vp, vp, vp, vp, vp, i64, vp, vp, vp, vp]),
    "fg_gat_input_attn_fwd": (ci, [C.POINTER(CodecDesc), vp, vp, i64, ci, vp, vp, i64, i64, vp,
                                   C.c_float, vp, vp, vp, vp, i64, vp]),
    "fg_gat_input_attn_bwd_blocks": (i64, []),
    "fg_gat_input_attn_bwd": (ci, [C.POINTER(CodecDesc), vp, vp, i64, ci, vp, vp, vp, vp, vp,
                                   i64, vp, C.c_float, vp, vp, vp]),
    "fg_gat_elu_bwd": (ci, [vp, vp, i64, vp, ci, vp]),
    "fg_gat_code_xagg_bwd": (ci, [C.POINTER(CodecDesc), vp, vp, i64, ci, vp, i64, vp, vp, vp,
                                  vp]),
    "fg_softmax_ce": (ci, [vp, ci, ci, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp]),
    "fg_adam_step": (ci, [vp, vp, vp, vp, i64, vp, C.c_float, C.c_float, C.c_float, C.c_float,
                          C.c_float, vp, vp]),
    "fg_f32_to_bf16_plain": (ci, [vp, i64, vp, vp]),
    "fg_rng_init": (ci, [vp, u64, u64, u64, u64, ci, u32]),
    "fg_rng_read": (ci, [vp, C.POINTER(u64), C.POINTER(u64), C.POINTER(ci), C.POINTER(u32)]),
    "fg_rng_permutation_host": (ci, [vp, vp, i64]),
    "fg_sample_layer": (ci, [vp, vp, i64, vp, vp, i64, ci, vp, vp, vp, i64, vp, vp, vp, i64,
                             vp, vp]),
    "fg_sample_workspace_bytes": (i64, [i64]),
    "fg_bitmap_words": (i64, [i64]),
    "fg_bitmap_mark": (ci, [vp, vp, i64, vp, i64, vp]),
    "fg_bitmap_mark64": (ci, [vp, vp, i64, vp, i64, vp]),
    "fg_bitmap_compact": (ci, [vp, i64, vp, i64, vp, vp, vp, i64, vp]),
    "fg_bitmap_workspace_bytes": (i64, [i64]),
    "fg_bitmap_rank": (ci, [vp, vp, i64, vp, vp, vp, vp]),
    "fg_sort_ids": (ci, [vp, vp, i64, vp, vp, i64, vp]),
    "fg_bitmap_clear": (ci, [vp, vp, i64, vp, i64, vp]),
    "fg_synth_features": (ci, [ci, u64, i64, i64, i64, vp, ci, vp, vp]),
    "fg_synth_feature_rows": (ci, [ci, u64, vp, i64, i64, vp, ci, vp, vp]),
    "fg_graph_degrees": (ci, [u64, i64, i64, C.c_double, C.c_double, i64, vp, vp]),
    "fg_graph_emit": (ci, [u64, i64, i64, C.c_double, C.c_double, i64, i64, i64, vp, i64, vp,
                           vp]),
    "fg_graph_labels": (ci, [u64, i64, i64, vp, vp]),
    "fg_csr_self_loops": (ci, [vp, vp, i64, vp, vp]),
}

_lib = None


def lib():
    """The loaded library (built in-tree by ``__graft_entry__.build()``)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"featgrind-b200 CUDA library not built: {LIB_PATH} is missing. "
                "Run `python -m paper_2207_14696_b200.build` (there is no CPU fallback).")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


class CudaError(RuntimeError):
    pass


def check(rc: int, what: str = "") -> None:
    if rc == FG_OK:
        return
    msg = lib().fg_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc in (FG_EDATA, FG_EUSAGE):
        raise DataError(msg)
    raise CudaError(msg)


def call(name: str, *args):
    """Invoke an ``int``-returning entry point and raise on failure."""
    check(getattr(lib(), name)(*args), name)


def ptr(t) -> int | None:
    """Device/host address of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_handle(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


_l2_set = False


def require_cuda():
    global _l2_set
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("featgrind-b200 requires a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    lib()
    if not _l2_set:
        _l2_set = True
        g = int(os.environ.get("FG_L2_FETCH", "0"))
        if g:
            torch.cuda.init()
            call("fg_set_l2_fetch_granularity", g)


def l2_fetch_granularity() -> int:
    v = C.c_int()
    call("fg_get_l2_fetch_granularity", C.byref(v))
    return v.value
