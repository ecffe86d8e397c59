"""Torch-facing wrappers of the fused aggregate kernels.

* ``gather_dequant_mean`` — layer-1 SAGE mean straight from compressed rows
  (``fg_gather_dequant_mean``): the north-star hot path.  Its input is a
  constant (features are not trained), so it has no backward.
* ``BlockMean`` — mean over a sampled block of hidden bf16 rows addressed by
  local index, with a scatter backward (``fg_block_mean_fwd/bwd``).

Both produce static-capacity outputs (rows past the live destination count
are zeros) so a whole training step has fixed shapes and can be captured in
one CUDA graph.
"""

from __future__ import annotations

import ctypes

import torch

from . import _native as N


def padded_dim(d: int) -> int:
    """Row pitch of aggregate buffers: 16-element aligned so the following
    bf16 GEMM gets an aligned K (d=100 -> 112)."""
    return (d + 15) // 16 * 16


def alloc_aggregate(max_dst: int, d: int, dtype=torch.bfloat16, device="cuda"):
    """Zeroed [max_dst, padded_dim(d)] buffer; the fused kernel only writes
    live rows and the first d columns, so padding stays exactly zero."""
    return torch.zeros((max_dst, padded_dim(d)), dtype=dtype, device=device)


def gather_dequant_mean(codec, indptr, src, n_dst, max_dst: int, out=None,
                        out_dtype=torch.bfloat16):
    """out[v, :d] = mean_{e in indptr[v]:indptr[v+1]} decode(codec, src[e])
    for live v < n_dst (rows past n_dst are not written)."""
    if out is None:
        out = alloc_aggregate(max_dst, codec.d, out_dtype, indptr.device)
    assert out.shape[0] >= max_dst and out.shape[1] >= codec.d and out.is_contiguous()
    code = N.OUT_BF16 if out.dtype == torch.bfloat16 else N.OUT_F32
    N.call("fg_gather_dequant_mean", ctypes.byref(codec.desc), N.ptr(indptr), N.ptr(src),
           N.ptr(n_dst), max_dst, N.ptr(out), out.shape[1], code, N.stream_handle())
    return out


class BlockMean(torch.autograd.Function):
    """h_dst[v] = mean over picks e of v of act(h_src[local[e]]) (bf16, fp32
    accumulate), act = ReLU when ``relu`` (fused on load; its derivative is
    applied in the backward's fp32 -> bf16 conversion)."""

    @staticmethod
    def forward(ctx, h_src, indptr, local, n_dst, max_dst: int, relu: bool = False):
        h_src = h_src.contiguous()
        H = h_src.shape[1]
        out = torch.empty((max_dst, H), dtype=torch.bfloat16, device=h_src.device)
        N.call("fg_block_mean_fwd", N.ptr(h_src), H, N.ptr(indptr), N.ptr(local), N.ptr(n_dst),
               max_dst, N.ptr(out), int(relu), N.stream_handle())
        if relu:
            ctx.save_for_backward(indptr, local, n_dst, h_src)
        else:
            ctx.save_for_backward(indptr, local, n_dst)
        ctx.relu = relu
        ctx.max_dst = max_dst
        ctx.n_src = h_src.shape[0]
        return out

    @staticmethod
    def backward(ctx, g):
        if ctx.relu:
            indptr, local, n_dst, h_src = ctx.saved_tensors
        else:
            indptr, local, n_dst = ctx.saved_tensors
            h_src = None
        g = g.contiguous().to(torch.bfloat16)
        H = g.shape[1]
        acc = torch.zeros((ctx.n_src, H), dtype=torch.float32, device=g.device)
        s = N.stream_handle()
        N.call("fg_block_mean_bwd", N.ptr(g), H, N.ptr(indptr), N.ptr(local), N.ptr(n_dst),
               ctx.max_dst, N.ptr(acc), s)
        gh = torch.empty((ctx.n_src, H), dtype=torch.bfloat16, device=g.device)
        N.call("fg_f32_to_bf16", N.ptr(acc), acc.numel(), N.ptr(h_src), N.ptr(gh), s)
        return gh, None, None, None, None, None


def block_mean(h_src, indptr, local, n_dst, max_dst: int, relu: bool = False):
    return BlockMean.apply(h_src, indptr, local, n_dst, max_dst, relu)
