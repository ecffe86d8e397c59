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
import os

import torch

from . import _native as N


def padded_dim(d: int) -> int:
    """Row pitch of aggregate buffers: 16-element aligned (so the following
    bf16 GEMM gets an aligned K) with at least one spare column, which holds
    a constant 1 so the first layer's bias rides inside its weight GEMM
    (d=100 -> 112, d=128 -> 144)."""
    return (d + 1 + 15) // 16 * 16


def alloc_aggregate(max_dst: int, d: int, dtype=torch.bfloat16, device="cuda",
                    ones_col: bool = True):
    """[max_dst, padded_dim(d)] buffer, zero except column d = 1 (bias
    input).  The fused kernel only writes live rows and the first d
    columns, so the padding keeps these values."""
    out = torch.zeros((max_dst, padded_dim(d)), dtype=dtype, device=device)
    if ones_col:
        out[:, d] = 1
    return out


def gather_dequant_mean(codec, indptr, src, n_dst, max_dst: int, out=None,
                        out_dtype=torch.bfloat16, edge_w=None):
    """out[v, :d] = mean_{e in indptr[v]:indptr[v+1]} decode(codec, src[e])
    for live v < n_dst (rows past n_dst are not written); with ``edge_w``
    the edge-weighted sum sum_e edge_w[e] decode(codec, src[e]) instead
    (aggregator variants, ``fg_gather_dequant_wsum``)."""
    if out is None:
        out = alloc_aggregate(max_dst, codec.d, out_dtype, indptr.device)
    assert out.shape[0] >= max_dst and out.shape[1] >= codec.d and out.is_contiguous()
    code = N.OUT_BF16 if out.dtype == torch.bfloat16 else N.OUT_F32
    if edge_w is None:
        N.call("fg_gather_dequant_mean", ctypes.byref(codec.desc), N.ptr(indptr), N.ptr(src),
               N.ptr(n_dst), max_dst, N.ptr(out), out.shape[1], code, N.stream_handle())
    else:
        N.call("fg_gather_dequant_wsum", ctypes.byref(codec.desc), N.ptr(indptr), N.ptr(src),
               N.ptr(edge_w), N.ptr(n_dst), max_dst, N.ptr(out), out.shape[1], code,
               N.stream_handle())
    return out


AGGREGATORS = ("mean", "gcn")  # FG_AGG_MEAN, FG_AGG_GCN


def edge_weights(kind: str, graph, dst_nodes, indptr, src_nodes, n_dst, max_dst: int, out):
    """Per-edge weights of a sampled block (``fg_block_edge_weights``):
    'mean' -> 1/cnt_v; 'gcn' -> sqrt(deg v) / (cnt_v sqrt(deg u)), the sampled
    estimator of D^-1/2 A D^-1/2 over full-graph degrees."""
    N.call("fg_block_edge_weights", AGGREGATORS.index(kind), N.ptr(graph.row_offsets),
           N.ptr(dst_nodes), N.ptr(indptr), N.ptr(src_nodes), N.ptr(n_dst), max_dst, N.ptr(out),
           N.stream_handle())
    return out


class BlockMean(torch.autograd.Function):
    """h_dst[v] = mean over picks e of v of act(h_src[local[e]]) (bf16, fp32
    accumulate), act = ReLU when ``relu`` (fused on load; its derivative is
    applied in the backward's fp32 -> bf16 conversion)."""

    @staticmethod
    def forward(ctx, h_src, indptr, local, n_dst, max_dst: int, relu: bool = False,
                trans=None, bias_col: bool = False, edge_w=None):
        h_src = h_src.contiguous()
        H = h_src.shape[1]
        ld = H + 8 if bias_col else H
        assert edge_w is None or trans is not None, "edge weights need the gather backward"
        out = torch.empty((max_dst, ld), dtype=torch.bfloat16, device=h_src.device)
        N.call("fg_block_mean_fwd", N.ptr(h_src), H, N.ptr(indptr), N.ptr(local), N.ptr(n_dst),
               max_dst, N.ptr(out), ld, int(relu), N.ptr(edge_w), N.stream_handle())
        t_indptr, t_dst, t_w, n_src = trans if trans is not None else (indptr, indptr, n_dst,
                                                                        n_dst)
        ctx.save_for_backward(indptr, local, n_dst, h_src if relu else indptr, t_indptr, t_dst,
                              t_w, n_src)
        ctx.relu = relu
        ctx.H = H
        ctx.gather_bwd = trans is not None
        ctx.max_dst = max_dst
        ctx.n_src = h_src.shape[0]
        return out

    @staticmethod
    def backward(ctx, g):
        indptr, local, n_dst, h_src, t_indptr, t_dst, t_w, n_src = ctx.saved_tensors
        if not ctx.relu:
            h_src = None
        g = g.contiguous().to(torch.bfloat16)
        H = ctx.H
        if ctx.gather_bwd:  # gather over the block's transpose, no float atomics
            gh = torch.empty((ctx.n_src, H), dtype=torch.bfloat16, device=g.device)
            N.call("fg_block_mean_bwd_t", N.ptr(g), H, g.shape[1], N.ptr(t_indptr), N.ptr(t_dst),
                   N.ptr(t_w), N.ptr(n_src), ctx.n_src, N.ptr(h_src), N.ptr(gh),
                   N.stream_handle())
            return gh, None, None, None, None, None, None, None, None
        if g.shape[1] != H:
            g = g[:, :H].contiguous()
        acc = torch.zeros((ctx.n_src, H), dtype=torch.float32, device=g.device)
        s = N.stream_handle()
        N.call("fg_block_mean_bwd", N.ptr(g), H, N.ptr(indptr), N.ptr(local), N.ptr(n_dst),
               ctx.max_dst, N.ptr(acc), s)
        gh = torch.empty((ctx.n_src, H), dtype=torch.bfloat16, device=g.device)
        N.call("fg_f32_to_bf16", N.ptr(acc), acc.numel(), N.ptr(h_src), N.ptr(gh), s)
        return gh, None, None, None, None, None, None, None, None


def block_mean(h_src, indptr, local, n_dst, max_dst: int, relu: bool = False, trans=None,
               bias_col: bool = False, edge_w=None):
    """``trans`` = (t_indptr, t_dst, t_w, n_src) of the block (DeviceSampler
    with need_transpose) switches the backward to the gather form; ``bias_col``
    appends a [1, 0 x 7] column block (output width H + 8) so the next
    layer's bias is a column of its weight; ``edge_w`` turns the mean into
    the edge-weighted sum (the transpose must carry the same weights)."""
    return BlockMean.apply(h_src, indptr, local, n_dst, max_dst, relu, trans, bias_col, edge_w)


def wgrad_supported(h_dim: int, p_dim: int) -> bool:
    return bool(N.lib().fg_block_mean_wgrad_supported(h_dim, p_dim))


def relu_mask_bits(h, out=None):
    """Packed ReLU mask of bf16 rows h [rows, H]: uint8 [rows, H/8]."""
    rows, H = h.shape
    if out is None:
        out = torch.empty((rows, H // 8), dtype=torch.uint8, device=h.device)
    N.call("fg_relu_mask_bits", N.ptr(h), rows, H, N.ptr(out), N.stream_handle())
    return out


def wgrad_scratch(H: int, P: int, device) -> torch.Tensor:
    nb = N.lib().fg_block_mean_wgrad_scratch_bytes(H, P)
    return torch.empty((nb + 3) // 4, dtype=torch.float32, device=device)


def block_mean_wgrad(g, indptr, local, n_dst, max_dst: int, h_mask, x, dw=None, scratch=None,
                     H: int | None = None, edge_w=None):
    """dW = dH^T x for the block mean a[v] = mean_e relu(h[local[e]]) with
    upstream gradient g = dL/da, computed as an edge-tiled GEMM
    (``fg_block_mean_wgrad``: per-edge terms relu'(h[l_e]) * g[v_e] / cnt_v
    are built in shared memory and consumed by tcgen05 MMAs; neither they
    nor dH reach HBM).  g: [>= max_dst, >= H] bf16, x: [cap_src, P] bf16,
    h_mask: [cap_src, H] bf16 pre-activations, [cap_src, H/8] uint8 packed
    ReLU bits (``relu_mask_bits``), or None; returns dw [H, P] fp32."""
    H = H or (h_mask.shape[1] if h_mask is not None else g.shape[1] - 8)
    P = x.shape[1]
    if dw is None:
        dw = torch.empty((H, P), dtype=torch.float32, device=x.device)
    if scratch is None:
        scratch = wgrad_scratch(H, P, x.device)
    N.call("fg_block_mean_wgrad", N.ptr(g), g.stride(0), N.ptr(indptr), N.ptr(local),
           N.ptr(n_dst), max_dst, N.ptr(edge_w), N.ptr(h_mask),
           0 if h_mask is None else (2 if h_mask.dtype == torch.uint8 else 1),
           H, N.ptr(x), P, N.ptr(dw), N.ptr(scratch), scratch.numel() * 4, N.stream_handle())
    return dw


class InputBlockMean(torch.autograd.Function):
    """a = block_mean(relu(x @ W^T)) for the SAGE input layer (bias folded in
    W via x's ones column).  Forward: one bf16 GEMM + the block-mean gather;
    backward: ``block_mean_wgrad`` (edge-tiled fused tcgen05 dW), no dx (x
    is the decoded input aggregate, not a parameter)."""

    @staticmethod
    def forward(ctx, x, w, indptr, local, n_dst, max_dst, bias_col, scratch, edge_w):
        h = torch.mm(x, w.to(torch.bfloat16).t())
        h_src = h.contiguous()
        H = h_src.shape[1]
        ld = H + 8 if bias_col else H
        out = torch.empty((max_dst, ld), dtype=torch.bfloat16, device=h.device)
        N.call("fg_block_mean_fwd", N.ptr(h_src), H, N.ptr(indptr), N.ptr(local), N.ptr(n_dst),
               max_dst, N.ptr(out), ld, 1, N.ptr(edge_w), N.stream_handle())
        ctx.save_for_backward(x, h_src, indptr, local, n_dst)
        ctx.max_dst, ctx.scratch, ctx.edge_w = max_dst, scratch, edge_w
        return out

    @staticmethod
    def backward(ctx, ga):
        x, h, indptr, local, n_dst = ctx.saved_tensors
        dw = block_mean_wgrad(ga.contiguous(), indptr, local, n_dst, ctx.max_dst, h, x,
                              scratch=ctx.scratch, edge_w=ctx.edge_w)
        return None, dw, None, None, None, None, None, None, None


def input_block_mean(x, w, indptr, local, n_dst, max_dst: int, bias_col: bool = True,
                     scratch=None, edge_w=None):
    return InputBlockMean.apply(x, w, indptr, local, n_dst, max_dst, bias_col, scratch, edge_w)


class SoftmaxCE(torch.autograd.Function):
    """Mean cross-entropy over the live seed rows of padded logits (classes
    past ``num_classes`` are padding), labels gathered on the device
    (``fg_softmax_ce``: one fused kernel computing loss and d loss / d
    logits)."""

    @staticmethod
    def forward(ctx, logits, labels, row_node, n_valid, num_classes):
        logits = logits.contiguous()
        rows, ld = logits.shape
        grad = torch.empty_like(logits)
        row_loss = torch.empty(rows, dtype=torch.float32, device=logits.device)
        loss = torch.empty((), dtype=torch.float32, device=logits.device)
        ctr = torch.zeros(1, dtype=torch.int32, device=logits.device)
        N.call("fg_softmax_ce", N.ptr(logits), int(logits.dtype == torch.bfloat16),
               num_classes or ld, ld, rows, N.ptr(n_valid), N.ptr(labels), N.ptr(row_node),
               N.ptr(grad), N.ptr(row_loss), N.ptr(loss), N.ptr(ctr), N.stream_handle())
        ctx.save_for_backward(grad)
        return loss

    @staticmethod
    def backward(ctx, g):
        (grad,) = ctx.saved_tensors
        return grad * g.to(grad.dtype), None, None, None, None


def softmax_ce(logits, labels, row_node, n_valid, num_classes: int | None = None):
    return SoftmaxCE.apply(logits, labels, row_node, n_valid, num_classes)


def kgemm(a, b, out, chunks: int | None = None, min_k: int = 32768):
    """out [M, N] fp32 = a^T b for bf16 a [K, M], b [K, N].  Past min_k rows
    K is cut into `chunks` slices multiplied by one batched GEMM (fp32 out)
    and summed: for K ~ 1e5 with M, N <= 400 cuBLAS's single-GEMM choice (no
    split-K) runs several times slower.  A K % chunks tail is one more GEMM.
    Default chunks: 64, or 32 for outputs past 64 K elements (the fp32
    partials are written and summed once more)."""
    K = a.shape[0]
    if K < min_k:
        return torch.mm(a.t(), b, out_dtype=torch.float32, out=out)
    if chunks is None:
        chunks = int(os.environ.get("FG_KGEMM_CHUNKS", "0")) or (
            32 if a.shape[1] * b.shape[1] > 65536 else 64)
    kc = K // chunks
    Kc = kc * chunks
    part = torch.bmm(a[:Kc].view(chunks, kc, -1).transpose(1, 2), b[:Kc].view(chunks, kc, -1),
                     out_dtype=torch.float32)
    torch.sum(part, 0, out=out)
    if Kc < K:
        out += torch.mm(a[Kc:].t(), b[Kc:], out_dtype=torch.float32)
    return out
