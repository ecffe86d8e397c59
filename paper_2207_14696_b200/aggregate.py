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


def gather_dequant_mean(codec, indptr, src, n_dst, max_dst: int, out=None,
                        out_dtype=torch.bfloat16):
    """out[v] = mean_{e in indptr[v]:indptr[v+1]} decode(codec, src[e])."""
    if out is None:
        out = torch.empty((max_dst, codec.d), dtype=out_dtype, device=indptr.device)
    code = N.OUT_BF16 if out.dtype == torch.bfloat16 else N.OUT_F32
    N.call("fg_gather_dequant_mean", ctypes.byref(codec.desc), N.ptr(indptr), N.ptr(src),
           N.ptr(n_dst), max_dst, N.ptr(out), code, N.stream_handle())
    return out


class BlockMean(torch.autograd.Function):
    """h_dst[v] = mean over picks e of v of h_src[local[e]] (bf16, fp32 acc)."""

    @staticmethod
    def forward(ctx, h_src, indptr, local, n_dst, max_dst: int):
        h_src = h_src.contiguous()
        H = h_src.shape[1]
        out = torch.empty((max_dst, H), dtype=torch.bfloat16, device=h_src.device)
        N.call("fg_block_mean_fwd", N.ptr(h_src), H, N.ptr(indptr), N.ptr(local), N.ptr(n_dst),
               max_dst, N.ptr(out), N.stream_handle())
        ctx.save_for_backward(indptr, local, n_dst)
        ctx.max_dst = max_dst
        ctx.n_src = h_src.shape[0]
        return out

    @staticmethod
    def backward(ctx, g):
        indptr, local, n_dst = ctx.saved_tensors
        g = g.contiguous().to(torch.bfloat16)
        H = g.shape[1]
        acc = torch.zeros((ctx.n_src, H), dtype=torch.float32, device=g.device)
        s = N.stream_handle()
        N.call("fg_block_mean_bwd", N.ptr(g), H, N.ptr(indptr), N.ptr(local), N.ptr(n_dst),
               ctx.max_dst, N.ptr(acc), s)
        gh = torch.empty((ctx.n_src, H), dtype=torch.bfloat16, device=g.device)
        N.call("fg_f32_to_bf16", N.ptr(acc), acc.numel(), N.ptr(gh), s)
        return gh, None, None, None, None


def block_mean(h_src, indptr, local, n_dst, max_dst: int):
    return BlockMean.apply(h_src, indptr, local, n_dst, max_dst)
