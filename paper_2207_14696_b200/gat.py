"""Graph attention network (GAT) on compressed features — BASELINE config E's
second aggregator variant (PAPER.md:259-261 and 1048-1055 list GAT among the
trained models; the reference has no model code).

Per layer and head k (fg_gat.cu):
    z = h W;  el = <z, a_l[k]>;  er = <z, a_r[k]>
    q[v] = mean_{e in v} er[l_e]                  (destination query)
    alpha[e] = softmax_{e in v} LeakyReLU(el[l_e] + q[v])
    out[v] = sum_e alpha[e] z[l_e] + b
Standard GAT scores a destination with its own projected features; under the
reference's block semantics (pipeline.py:203-221) a destination that did not
sample itself has no representation at the layer below, so the
query is the mean of its sampled neighbours' er.

Input layer: the sources of the last block are its picks (one row per pick),
read straight from the codec's code rows by the scores / attention-weighted
aggregation kernels (decoded in registers) and projected by one block-
diagonal GEMM; hidden layers project the previous layer's output.
Edge operators are CUDA kernels wrapped as autograd Functions; the GEMMs,
LeakyReLU/ELU and the loss are torch/cuBLAS plus the fused softmax-CE kernel.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

from . import _native as N
from . import ddp
from .aggregate import kgemm as _kgemm, softmax_ce
from .sampler import DeviceSampler


class GatAttention(torch.autograd.Function):
    """alpha [E_cap, heads] from per-source scores el, er [src_rows, heads]."""

    @staticmethod
    def forward(ctx, el, er, indptr, local, n_dst, max_dst: int, e_cap: int, slope: float):
        heads = el.shape[1]
        el, er = el.float().contiguous(), er.float().contiguous()
        alpha = torch.zeros((e_cap, heads), dtype=torch.float32, device=el.device)
        q = torch.empty((max_dst, heads), dtype=torch.float32, device=el.device)
        N.call("fg_gat_softmax_fwd", N.ptr(el), N.ptr(er), heads, N.ptr(indptr), N.ptr(local),
               max_dst, N.ptr(n_dst), heads, slope, N.ptr(alpha), N.ptr(q), N.stream_handle())
        ctx.save_for_backward(el, q, alpha, indptr, local if local is not None else indptr, n_dst)
        ctx.has_local, ctx.max_dst, ctx.slope = local is not None, max_dst, slope
        return alpha

    @staticmethod
    def backward(ctx, dalpha):
        el, q, alpha, indptr, local, n_dst = ctx.saved_tensors
        local = local if ctx.has_local else None
        heads = el.shape[1]
        del_ = torch.zeros_like(el)
        der = torch.zeros_like(el)
        N.call("fg_gat_softmax_bwd", N.ptr(el), heads, N.ptr(q), N.ptr(alpha),
               N.ptr(dalpha.float().contiguous()), N.ptr(indptr), N.ptr(local), ctx.max_dst,
               N.ptr(n_dst), heads, ctx.slope, N.ptr(del_), N.ptr(der), N.stream_handle())
        return del_, der, None, None, None, None, None, None


class GatAggregate(torch.autograd.Function):
    """out[v] = sum_e alpha[e, head] z[l_e] (fp32 [max_dst, hf])."""

    @staticmethod
    def forward(ctx, z, alpha, indptr, local, n_dst, max_dst: int):
        z = z.to(torch.bfloat16).contiguous()
        hf, heads = z.shape[1], alpha.shape[1]
        out = torch.empty((max_dst, hf), dtype=torch.float32, device=z.device)
        N.call("fg_gat_agg_fwd", N.ptr(z), hf, heads, N.ptr(alpha), N.ptr(indptr), N.ptr(local),
               max_dst, N.ptr(n_dst), N.ptr(out), N.stream_handle())
        ctx.save_for_backward(z, alpha, indptr, local if local is not None else indptr, n_dst)
        ctx.has_local, ctx.max_dst = local is not None, max_dst
        return out

    @staticmethod
    def backward(ctx, dout):
        z, alpha, indptr, local, n_dst = ctx.saved_tensors
        local = local if ctx.has_local else None
        hf, heads = z.shape[1], alpha.shape[1]
        dz = torch.zeros(z.shape, dtype=torch.float32, device=z.device)
        dalpha = torch.zeros_like(alpha)
        N.call("fg_gat_agg_bwd", N.ptr(z), hf, heads, N.ptr(alpha), N.ptr(indptr), N.ptr(local),
               ctx.max_dst, N.ptr(n_dst), N.ptr(dout.float().contiguous()), N.ptr(dz),
               N.ptr(dalpha), N.stream_handle())
        return dz, dalpha, None, None, None, None


class PickSource:
    """The last block's picks as the input layer reads them: decoded once by
    the codec's gather kernel into bf16 rows (one per pick, pick order).
    The code-reading form of the same kernels (``decoded=False``: elements
    decoded in registers from the code rows, SQ any k / VQ 8-bit) is kept for
    A/B: measured slower on the B200 (products-shape SQ8: per-thread byte
    decodes are less coalesced than one bf16 row gather + cuBLAS)."""

    def __init__(self, codec, picks, n_picks, e_cap: int, decoded: bool = True):
        import ctypes
        self.codec, self.picks, self.n_picks, self.e_cap = codec, picks, n_picks, int(e_cap)
        self.d = codec.d
        desc = codec.desc
        direct = not decoded and ((desc.kind == N.CODEC_SQ and desc.elem_bits == 32) or
                                  (desc.kind == N.CODEC_VQ and desc.bits == 8))
        self.x = None if direct else codec.gather(picks, out_dtype=torch.bfloat16, check=False)
        self._desc = ctypes.byref(desc)

    def head(self):
        """(codec desc, decoded rows or None, picks) -- the kernels' first args."""
        return (self._desc, N.ptr(self.x), N.ptr(self.picks))


class PickScores(torch.autograd.Function):
    """s = x c^T for the decoded picks x [E, d] (bf16) and c [2H, d]; the
    backward dc = ds^T x has K = E (~5e5): split into 64 chunks reduced by
    one batched GEMM instead of a single skinny cuBLAS call."""

    @staticmethod
    def forward(ctx, x, c):
        ctx.save_for_backward(x)
        return torch.mm(x, c.to(x.dtype).t()).float()

    @staticmethod
    def backward(ctx, ds):
        (x,) = ctx.saved_tensors
        E, d = x.shape
        ch = 64
        pad = (-E) % ch
        xs = x if not pad else torch.cat([x, x.new_zeros(pad, d)])
        gs = ds.to(x.dtype)
        gs = gs if not pad else torch.cat([gs, gs.new_zeros(pad, gs.shape[1])])
        part = torch.bmm(gs.view(ch, -1, gs.shape[1]).transpose(1, 2), xs.view(ch, -1, d))
        return None, part.float().sum(0)


class GatInputScores(torch.autograd.Function):
    """el, er [e_cap, H] = per-pick scores x_e . c[k] from the code rows;
    backward dc = sum_e ds_e x_e^T (deterministic block partials)."""

    @staticmethod
    def forward(ctx, c, src, heads: int):
        c = c.float().contiguous()
        el = torch.empty((src.e_cap, heads), dtype=torch.float32, device=c.device)
        er = torch.empty_like(el)
        N.call("fg_gat_code_scores", *src.head(), N.ptr(src.n_picks), src.e_cap, src.d, heads,
               N.ptr(c), N.ptr(el), N.ptr(er), N.stream_handle())
        ctx.src, ctx.heads = src, heads
        return el, er

    @staticmethod
    def backward(ctx, del_, der):
        src, heads = ctx.src, ctx.heads
        nb = N.lib().fg_gat_code_scores_bwd_blocks(src.e_cap)
        part = torch.empty((nb, 2 * heads, src.d), dtype=torch.float32, device=del_.device)
        z = torch.zeros((src.e_cap, heads), dtype=torch.float32, device=del_.device)
        del_ = z if del_ is None else del_.float().contiguous()
        der = z if der is None else der.float().contiguous()
        N.call("fg_gat_code_scores_bwd", *src.head(), N.ptr(src.n_picks), src.e_cap, src.d, heads,
               N.ptr(del_), N.ptr(der), heads, N.ptr(part), N.stream_handle())
        return part.sum(0), None, None


class GatInputXagg(torch.autograd.Function):
    """A [max_dst, H*d] bf16 = per head the alpha-weighted sum of the picks'
    decoded rows; backward dalpha[e, k] = <dA[v, k], x_e>."""

    @staticmethod
    def forward(ctx, alpha, src, indptr, n_dst, max_dst: int, heads: int):
        alpha = alpha.float().contiguous()
        A = torch.empty((max_dst, heads * src.d), dtype=torch.bfloat16, device=alpha.device)
        N.call("fg_gat_code_xagg_fwd", *src.head(), src.d, heads, N.ptr(alpha), N.ptr(indptr),
               max_dst, N.ptr(n_dst), N.ptr(A), 0, N.stream_handle())
        ctx.save_for_backward(indptr, n_dst)
        ctx.src, ctx.max_dst, ctx.heads = src, max_dst, heads
        return A

    @staticmethod
    def backward(ctx, dA):
        indptr, n_dst = ctx.saved_tensors
        src, heads = ctx.src, ctx.heads
        dalpha = torch.zeros((src.e_cap, heads), dtype=torch.float32, device=dA.device)
        dA = dA.to(torch.bfloat16).contiguous()
        N.call("fg_gat_code_xagg_bwd", *src.head(), src.d, heads, N.ptr(indptr), ctx.max_dst,
               N.ptr(n_dst), N.ptr(dA), N.ptr(dalpha), N.stream_handle())
        return dalpha, None, None, None, None, None


class GatLayer(nn.Module):
    def __init__(self, in_dim: int, out_per_head: int, heads: int, out_pad: int | None = None):
        super().__init__()
        self.heads, self.f = heads, out_per_head
        width = out_pad or out_per_head * heads
        self.lin = nn.Linear(in_dim, width, bias=False)
        if out_pad:  # padded classes: zero rows (their z, alpha-weighted sums and grads stay 0)
            with torch.no_grad():
                self.lin.weight[out_per_head * heads:] = 0
        self.width = width
        self.attn_l = nn.Parameter(torch.randn(heads, width // heads) * 0.1)
        self.attn_r = nn.Parameter(torch.randn(heads, width // heads) * 0.1)
        self.bias = nn.Parameter(torch.zeros(width))

    def forward(self, h, indptr, local, n_dst, max_dst, e_cap, slope=0.2):
        if local is None:
            return self._forward_input(h, indptr, n_dst, max_dst, e_cap, slope)
        z = self.lin(h)                                           # [src, width]
        # el/er = z . a per head = h (W_k^T a_k): one skinny GEMM on h
        H, f = self.heads, self.width // self.heads
        w = self.lin.weight.view(H, f, -1)
        c = torch.cat([torch.einsum("hfd,hf->hd", w, self.attn_l),
                       torch.einsum("hfd,hf->hd", w, self.attn_r)])  # [2H, in]
        s = torch.mm(h, c.to(h.dtype).t()).float()
        el, er = s[:, :H], s[:, H:]
        alpha = GatAttention.apply(el, er, indptr, local, n_dst, max_dst, e_cap, slope)
        return GatAggregate.apply(z, alpha, indptr, local, n_dst, max_dst) + self.bias

    def _forward_input(self, src, indptr, n_dst, max_dst, e_cap, slope):
        """Same math for the input layer, rearranged by linearity: scores
        el = x (W_k^T a_l[k]) per pick (one skinny GEMM on the decoded picks),
        the attention-weighted sum of the picks' rows per head (A,
        [N_dst, H*d] bf16, one kernel), then out = A . blockdiag(W_k^T) + b:
        one GEMM, no per-pick projection.  Every step is differentiable: dA
        flows back to the attention (round 1's head projection dropped it, so
        layer 0's attention vectors never trained)."""
        H, f = self.heads, self.width // self.heads
        d = src.d
        w = self.lin.weight.view(H, f, d)                       # [H, F, d]
        c = torch.cat([torch.einsum("hfd,hf->hd", w, self.attn_l),
                       torch.einsum("hfd,hf->hd", w, self.attn_r)])  # [2H, d]
        if src.x is not None:  # decoded rows: the scores are one skinny GEMM
            sc = PickScores.apply(src.x, c)
            el, er = sc[:, :H].contiguous(), sc[:, H:].contiguous()
        else:
            el, er = GatInputScores.apply(c, src, H)
        alpha = GatAttention.apply(el, er, indptr, None, n_dst, max_dst, e_cap, slope)
        A = GatInputXagg.apply(alpha, src, indptr, n_dst, max_dst, H)   # [N, H*d] bf16
        w_bd = torch.block_diag(*[w[k].t() for k in range(H)])         # [H*d, H*F]
        # bias folded into the GEMM; the output stays in the autocast dtype
        return torch.addmm(self.bias.to(A.dtype), A, w_bd.to(A.dtype))


class GatModel(nn.Module):
    """L GAT layers: hidden layers `heads` heads of hidden/heads features
    (concatenated, ELU), output layer one head of num_classes (padded to 8)."""

    def __init__(self, in_dim: int, hidden: int, num_classes: int, num_layers: int,
                 heads: int = 4):
        super().__init__()
        self.num_classes = num_classes
        c_pad = (num_classes + 7) // 8 * 8
        layers = []
        for i in range(num_layers):
            last = i == num_layers - 1
            d_in = in_dim if i == 0 else hidden
            if last:
                layers.append(GatLayer(d_in, num_classes, 1, out_pad=c_pad))
            else:
                layers.append(GatLayer(d_in, hidden // heads, heads))
        self.layers = nn.ModuleList(layers)

    def forward(self, src, sb, caps, pick_cap):
        """src: the last block's picks (PickSource: code rows or decoded rows)."""
        L = len(self.layers)
        h = src
        for i, layer in enumerate(self.layers):
            l = L - 1 - i  # block feeding layer i
            local = None if l == L - 1 else sb.local[l]
            e_cap = pick_cap if l == L - 1 else sb.local[l].numel()
            h = layer(h, sb.indptr[l], local, sb.n_nodes[l], caps[l], e_cap)
            if i < L - 1:
                h = F.elu(h)
        return h


def _round_up(n: int, m: int) -> int:
    return (n + m - 1) // m * m


class _LayerViews:
    """One GatLayer's parameters as views of the trainer's flat fp32 / bf16
    parameter buffers and flat gradient (attn_l, attn_r adjacent: one [2,
    heads, F] view each), plus the input layer's persistent block-diagonal
    bf16 weight (zero off the diagonal; the diagonal blocks are refreshed
    from the bf16 shadow every step)."""

    def __init__(self, layer, flat, grad, flat_bf16):
        def off(p):
            return (p.data_ptr() - flat.data_ptr()) // flat.element_size()

        self.heads = layer.heads
        self.width = layer.width
        self.F = layer.width // layer.heads
        self.D = layer.lin.weight.shape[1]
        w, al, ar, b = layer.lin.weight, layer.attn_l, layer.attn_r, layer.bias
        assert off(ar) == off(al) + al.numel(), "attn_l / attn_r must be adjacent"
        ow, oa, ob = off(w), off(al), off(b)
        na, nw, nb = 2 * al.numel(), w.numel(), b.numel()
        shp_a = (2, self.heads, self.F)
        self.W = flat[ow:ow + nw].view(w.shape)
        self.Wb = flat_bf16[ow:ow + nw].view(w.shape)
        self.attn = flat[oa:oa + na].view(shp_a)
        self.b = flat[ob:ob + nb]
        self.bb = flat_bf16[ob:ob + nb]
        self.dW = grad[ow:ow + nw].view(w.shape)
        self.dattn = grad[oa:oa + na].view(shp_a)
        self.db = grad[ob:ob + nb]
        self.wbd = None

    def refresh_block_diag(self):
        """wbd [Hh*D + 8, Hh*F]: wbd[k*D + j, k*F + f] = W[k*F + f, j], row
        Hh*D = the bias (the input's ones column), zeros elsewhere."""
        Hh, F, D = self.heads, self.F, self.D
        if self.wbd is None:
            self.wbd = torch.zeros((Hh * D + 8, Hh * F), dtype=torch.bfloat16,
                                   device=self.W.device)
        self.wbd[:Hh * D].view(Hh, D, Hh, F).diagonal(dim1=0, dim2=2).copy_(
            self.Wb.view(Hh, F, D).permute(2, 1, 0))
        self.wbd[Hh * D].copy_(self.bb)


@dataclass
class GatConfig:
    fanouts: tuple = (15, 10, 5)
    batch_size: int = 1024
    hidden: int = 256
    heads: int = 4
    lr: float = 3e-3
    seed: int = 0
    use_graph: bool = True
    explicit: bool = True
    pipeline: bool = True


class GatTrainer:
    """Single-process (or one-rank-of-DDP) GAT trainer over device-resident
    data: sample (pipelined on a side stream) -> GAT layers (input layer over
    the decoded picks) -> fused softmax-CE -> explicit backward into one flat
    gradient -> flat all-reduce -> flat Adam; one CUDA graph per sampler slot."""

    def __init__(self, graph, codec, labels, num_classes: int, cfg: GatConfig,
                 process_group=None):
        self.cfg, self.codec, self.labels = cfg, codec, labels
        self.device = labels.device
        self.pg = process_group
        self.world = torch.distributed.get_world_size(process_group) if process_group else 1
        torch.manual_seed(cfg.seed)
        L = len(cfg.fanouts)
        # FG_GAT_GATHER=1: transposes with edge ids of the non-input blocks for
        # the gather-form aggregation backward (fg_gat_agg_bwd_t; measured
        # 1.228 vs 1.169 ms/step with the atomic form: a warp walks a hub
        # source's entries serially)
        self._gather = os.environ.get("FG_GAT_GATHER", "0") == "1"
        self.sampler = DeviceSampler(graph, cfg.fanouts, cfg.batch_size, need_local=True,
                                     need_transpose=self._gather, need_eid=self._gather)
        # pipelined like SageTrainer: batch b+1 is sampled into the other slot
        # on a side stream while batch b trains (one shared PCG64 stream)
        self.samplers = [self.sampler]
        self.pipeline = cfg.pipeline
        if self.pipeline:
            self.samplers.append(DeviceSampler(graph, cfg.fanouts, cfg.batch_size,
                                               need_local=True, need_transpose=self._gather,
                                               need_eid=self._gather, share=self.sampler))
            self.side = torch.cuda.Stream(self.device,
                                          priority=int(os.environ.get("FG_SIDE_PRIORITY", "-1")))
        self.graphs = {}
        self._primed, self._next = False, 0
        self.steps_run = 0
        self.caps = self.sampler.caps
        self.pick_cap = self.sampler.pcaps[L - 1]
        self.model = GatModel(codec.d, cfg.hidden, num_classes, L, cfg.heads).to(self.device)
        # one flat fp32 buffer each for params / grads (the parameters and their
        # .grad are views): one memset, one all-reduce and one Adam kernel per
        # step instead of per-tensor foreach launches
        from .sage import FlatAdam
        params = list(self.model.parameters())
        total = sum(p.numel() for p in params)
        self.flat_param = torch.zeros(total, dtype=torch.float32, device=self.device)
        self.flat_grad = torch.zeros(total, dtype=torch.float32, device=self.device)
        off = 0
        for p in params:
            n = p.numel()
            self.flat_param[off:off + n].copy_(p.data.reshape(-1))
            p.data = self.flat_param[off:off + n].view_as(p)
            p.grad = self.flat_grad[off:off + n].view_as(p)
            off += n
        if self.world > 1:
            torch.distributed.broadcast(self.flat_param, 0, group=self.pg)
        # bf16 shadow of the parameters (written by the Adam kernel): the
        # explicit step's GEMM operands
        self.flat_bf16 = torch.zeros(total, dtype=torch.bfloat16, device=self.device)
        self.opt = FlatAdam(self.flat_param, self.flat_grad, lr=cfg.lr, param_bf16=self.flat_bf16)
        self.loss_buf = torch.zeros((), dtype=torch.float32, device=self.device)
        self.ce_ctr = torch.zeros(1, dtype=torch.int32, device=self.device)
        # explicit forward/backward (no autograd/autocast glue); FG_GAT_EXPLICIT=0
        # keeps the autograd model step (A/B and the gradient tests' reference)
        self.explicit = (cfg.explicit and L > 1
                         and os.environ.get("FG_GAT_EXPLICIT", "1") != "0")
        self._views = [_LayerViews(layer, self.flat_param, self.flat_grad, self.flat_bf16)
                       for layer in self.model.layers]
        self._ones = torch.ones(max(self.caps), dtype=torch.float32, device=self.device)
        self._wstream = torch.cuda.Stream(self.device)
        # FG_GAT_OVERLAP=1: the forward's z GEMM and the backward's dz zero
        # fills on the side stream too (measured 1.047 vs 1.038 ms: contention)
        self._overlap = os.environ.get("FG_GAT_OVERLAP", "0") == "1"
        desc = codec.desc
        self._direct = (os.environ.get("FG_GAT_DIRECT", "0") == "1" and desc.kind == N.CODEC_SQ
                        and desc.bits == 8 and desc.elem_bits == 32 and desc.row_stride % 2 == 0)
        self.graph = None

    def _decode(self, sb):
        L = len(self.cfg.fanouts)
        return PickSource(self.codec, sb.picks[L - 1], sb.n_picks[L - 1], self.pick_cap)

    def _body(self, k: int = 0):
        """One step.  Serial: sample slot 0's loaded seeds, then train.
        Pipelined: train the batch already in slot k while the side stream
        samples the next batch (seeds already loaded) into slot 1-k."""
        if not self.pipeline:
            return self._train(self.sampler.sample_loaded())
        cur = torch.cuda.current_stream()
        self.side.wait_stream(cur)
        with torch.cuda.stream(self.side):
            self.samplers[1 - k].sample_loaded()
        self._train(self.samplers[k].batch_view())
        cur.wait_stream(self.side)

    def _train(self, sb):
        if self.explicit:
            self.forward_backward(sb)
        else:
            x = self._decode(sb)
            with torch.autocast("cuda", dtype=torch.bfloat16):
                logits = self.model(x, sb, self.caps, self.pick_cap)
            loss = softmax_ce(logits.contiguous(), self.labels, sb.nodes[0], sb.n_nodes[0],
                              self.model.num_classes)
            self.flat_grad.zero_()
            loss.backward()
            self.loss_buf.copy_(loss.detach())
        ddp.average_flat_(self.flat_grad, self.pg)
        self.opt.step()

    def forward_backward(self, sb) -> None:
        """GatModel's loss and every parameter gradient for batch sb, written
        out (same math as the autograd model, bf16 GEMM operands from the
        Adam kernel's shadow, fp32 scores / attention / gradients): loss ->
        loss_buf, gradients -> flat_grad (every element written: no zero
        fill).  Layer i reads block l = L-1-i; the input layer's sources are
        the decoded picks (one row per pick).

        forward   c = [a_l . W_k ; a_r . W_k]  (scores el|er = src c^T, one GEMM)
                  alpha = softmax_v LeakyReLU(el[l_e] + mean_e er[l_e])
                  input: A = sum_e alpha x_e per head, o = A blockdiag(W_k^T) + b
                  other: o = sum_e alpha z[l_e] + b,  z = h W^T
                  h_next = ELU(o); logits = o of the last layer
        backward  dz, dalpha (agg), ds = [del|der] (softmax), dW = dz^T h
                  (input: the diagonal blocks of do^T A), dc = ds^T src,
                  dW += a . dc, d[a_l|a_r] = W . dc, dh = dz W + ds c,
                  do_prev = ELU'(h) dh"""
        L = len(self.cfg.fanouts)
        s = N.stream_handle()
        dev = self.device
        f32, bf16 = torch.float32, torch.bfloat16
        # the picks: decoded bf16 rows, one per pick (k_sq_gather); FG_GAT_DIRECT=1
        # reads 8-bit SQ code rows in place instead (no decoded matrix, but a
        # dependent pick-id load per row: measured 1.225 vs 1.169 ms/step)
        L1 = L - 1
        # parameter-only operands of every layer (score vectors c, their bf16
        # copy, the input layer's block-diagonal weight, the backward's
        # [W; c; 0]) on the side stream, beside the pick decode
        if self._views[0].wbd is None:
            self._views[0].refresh_block_diag()
        pre = []
        with self._side_branch():
            for i, v in enumerate(self._views):
                Hh, Fh, D = v.heads, v.F, v.D
                c = torch.bmm(v.attn.permute(1, 0, 2), v.W.view(Hh, Fh, D))    # [Hh, 2, D]
                c = c.permute(1, 0, 2).reshape(2 * Hh, D)                       # [el | er] rows
                cb = c.to(bf16)
                if i == 0:
                    v.refresh_block_diag()
                    wcat = None
                else:
                    w2 = v.width + 2 * Hh
                    wcat = torch.cat([v.Wb, cb, cb.new_zeros((_round_up(w2, 8) - w2, D))])
                pre.append((c, cb, wcat))
            ev_pre = torch.cuda.Event()
            ev_pre.record(self._wstream)
        main = torch.cuda.current_stream()
        for t in pre:
            for x in t:
                if x is not None:
                    x.record_stream(main)
        src = PickSource(self.codec, sb.picks[L1], sb.n_picks[L1], self.pick_cap,
                         decoded=not self._direct)
        main.wait_event(ev_pre)
        saved = []
        h = src
        for i, v in enumerate(self._views):
            l = L - 1 - i
            Hh, Fh, D = v.heads, v.F, v.D
            c, cb, _ = pre[i]
            first = i == 0
            local = None if first else sb.local[l]
            e_cap = self.pick_cap if first else sb.local[l].numel()
            alpha = torch.empty((e_cap, Hh), dtype=f32, device=dev)
            q = torch.empty((self.caps[l], Hh), dtype=f32, device=dev)
            if first:
                # one pass over the picks (fg_gat_input_attn_fwd): scores,
                # softmax and A = [per-head alpha-weighted pick sums | 1 0..0],
                # rows padded to a multiple of 64 (zero rows) for the chunked
                # K-GEMMs; o = A [blockdiag(W_k^T); b; 0] (bias via the ones column)
                sc = torch.empty((e_cap, 2 * Hh), dtype=f32, device=dev)
                rows = _round_up(self.caps[l], 64)
                A = torch.empty((rows, Hh * D + 8), dtype=bf16, device=dev)
                N.call("fg_gat_input_attn_fwd", *src.head(), D, Hh, N.ptr(c), N.ptr(sb.indptr[l]),
                       self.caps[l], rows, N.ptr(sb.n_nodes[l]), 0.2, N.ptr(sc), N.ptr(alpha),
                       N.ptr(q), N.ptr(A), Hh * D + 8, s)
                o = torch.mm(A, v.wbd)                                          # bf16
                z = A
                bias, in_f32 = None, 0
            else:
                if self._overlap:
                    with self._side_branch(h):  # z = h W^T beside the score path
                        z = torch.mm(h, v.Wb.t())                               # [src rows, Wd]
                    z.record_stream(torch.cuda.current_stream())
                else:
                    z = torch.mm(h, v.Wb.t())
                sc = torch.mm(h, cb.t(), out_dtype=f32)                     # [src rows, 2Hh]
                N.call("fg_gat_softmax_fwd", N.ptr(sc), N.ptr(sc[:, Hh:]), 2 * Hh,
                       N.ptr(sb.indptr[l]), N.ptr(local), self.caps[l], N.ptr(sb.n_nodes[l]),
                       Hh, 0.2, N.ptr(alpha), N.ptr(q), s)
                if self._overlap:
                    torch.cuda.current_stream().wait_stream(self._wstream)
                o = torch.empty((self.caps[l], v.width), dtype=f32, device=dev)
                N.call("fg_gat_agg_fwd", N.ptr(z), v.width, Hh, N.ptr(alpha), N.ptr(sb.indptr[l]),
                       N.ptr(local), self.caps[l], N.ptr(sb.n_nodes[l]), N.ptr(o), s)
                bias, in_f32 = v.b, 1
            saved.append((h, c, cb, sc, alpha, q, z, local, e_cap))
            if i < L - 1:
                h = torch.empty(o.shape, dtype=bf16, device=dev)
                N.call("fg_gat_elu_fwd", N.ptr(o), in_f32, o.shape[1], N.ptr(bias), o.shape[0],
                       o.shape[1], N.ptr(h), s)
            else:
                h = o.add_(v.b)
        logits = h
        C, ld = self.model.num_classes, logits.shape[1]
        do = torch.empty_like(logits)
        row_loss = torch.empty(logits.shape[0], dtype=f32, device=dev)
        N.call("fg_softmax_ce", N.ptr(logits), 0, C, ld, logits.shape[0], N.ptr(sb.n_nodes[0]),
               N.ptr(self.labels), N.ptr(sb.nodes[0]), N.ptr(do), N.ptr(row_loss),
               N.ptr(self.loss_buf), N.ptr(self.ce_ctr), s)
        # ---- backward
        # the atomic aggregation backward's zeroed dz buffers, filled on the
        # side stream while the loss and the last layer's first kernels run
        gather = self._gather and sb.t_eid
        dz_pre = {}
        if not gather and self._overlap:
            with self._side_branch():
                for i in range(1, L):
                    dz_pre[i] = torch.zeros((saved[i][0].shape[0], self._views[i].width),
                                            dtype=f32, device=dev)
            ev_fill = torch.cuda.Event()
            ev_fill.record(self._wstream)
            for t in dz_pre.values():
                t.record_stream(torch.cuda.current_stream())
        for i in range(L - 1, -1, -1):
            v = self._views[i]
            l = L - 1 - i
            Hh, Fh, D = v.heads, v.F, v.D
            h, c, cb, sc, alpha, q, z, local, e_cap = saved[i]
            if i == 0:
                A = z
                dA = torch.mm(do, v.wbd[:Hh * D].t())                          # [rows, Hh*D]
                with self._side_branch(do, A):
                    # do^T A: the diagonal blocks are dW_k, the ones column db
                    full = _kgemm(do, A, torch.empty((v.width, A.shape[1]), dtype=f32,
                                                     device=dev))
                    v.dW.view(Hh, Fh, D).copy_(full[:, :Hh * D].view(Hh, Fh, Hh, D)
                                               .diagonal(dim1=0, dim2=2).permute(2, 0, 1))
                    v.db.copy_(full[:, Hh * D])
                # dalpha, the softmax backward and dc = [del|der]^T x in one
                # pass over the picks (fg_gat_input_attn_bwd)
                dalpha = torch.empty((e_cap, Hh), dtype=f32, device=dev)
                part = torch.empty((N.lib().fg_gat_input_attn_bwd_blocks(), 2 * Hh, D),
                                   dtype=f32, device=dev)
                N.call("fg_gat_input_attn_bwd", *src.head(), D, Hh, N.ptr(sc), N.ptr(alpha),
                       N.ptr(q), N.ptr(dA), N.ptr(sb.indptr[l]), self.caps[l],
                       N.ptr(sb.n_nodes[l]), 0.2, N.ptr(dalpha), N.ptr(part), s)
                with self._side_branch(part):
                    self._attn_grads(v, part.sum(0))
            else:
                ds = torch.zeros((h.shape[0], 2 * Hh), dtype=f32, device=dev)
                with self._side_branch(do):
                    torch.mv(do.t(), self._ones[:do.shape[0]], out=v.db)
                teid = sb.t_eid[l] if sb.t_eid else None
                if teid is not None and N.lib().fg_gat_agg_bwd_t_supported(v.width, Hh):
                    # gather form over the block's transpose: dz in bf16, no
                    # zero fill / atomics / cast
                    t_indptr, t_dst, _, n_src = sb.trans[l]
                    dzb = torch.empty((h.shape[0], v.width), dtype=bf16, device=dev)
                    dalpha = torch.empty((e_cap, Hh), dtype=f32, device=dev)
                    N.call("fg_gat_agg_bwd_t", N.ptr(z), v.width, Hh, N.ptr(alpha),
                           N.ptr(t_indptr), N.ptr(t_dst), N.ptr(teid), N.ptr(n_src), h.shape[0],
                           N.ptr(do), N.ptr(dzb), N.ptr(dalpha), s)
                    dz = dzb
                else:
                    if i in dz_pre:
                        torch.cuda.current_stream().wait_event(ev_fill)
                        dz = dz_pre.pop(i)
                    else:
                        dz = torch.zeros((h.shape[0], v.width), dtype=f32, device=dev)
                    dalpha = torch.zeros((e_cap, Hh), dtype=f32, device=dev)
                    N.call("fg_gat_agg_bwd", N.ptr(z), v.width, Hh, N.ptr(alpha),
                           N.ptr(sb.indptr[l]), N.ptr(local), self.caps[l], N.ptr(sb.n_nodes[l]),
                           N.ptr(do), N.ptr(dz), N.ptr(dalpha), s)
                N.call("fg_gat_softmax_bwd", N.ptr(sc), 2 * Hh, N.ptr(q), N.ptr(alpha),
                       N.ptr(dalpha), N.ptr(sb.indptr[l]), N.ptr(local), self.caps[l],
                       N.ptr(sb.n_nodes[l]), Hh, 0.2, N.ptr(ds), N.ptr(ds[:, Hh:]), s)
                # g = [dz | ds | 0] (bf16, 8-aligned width) against [W; c; 0]:
                # one K-GEMM gives dW and dc, one GEMM gives dh = dz W + ds c
                w2 = v.width + 2 * Hh
                Wp = _round_up(w2, 8)
                gcat = torch.empty((h.shape[0], Wp), dtype=bf16, device=dev)
                if dz.dtype == f32:
                    N.call("fg_cat_rows_bf16", N.ptr(dz), v.width, N.ptr(ds), 2 * Hh, h.shape[0],
                           N.ptr(gcat), Wp, s)
                else:  # gather form: dz already bf16
                    gcat[:, :v.width].copy_(dz)
                    gcat[:, v.width:w2].copy_(ds)
                    if Wp > w2:
                        gcat[:, w2:].zero_()
                with self._side_branch(gcat, h):
                    full = _kgemm(gcat, h, torch.empty((Wp, D), dtype=f32, device=dev))
                    v.dW.copy_(full[:v.width])
                    self._attn_grads(v, full[v.width:w2])
            if i == 0:
                break
            dh = torch.mm(gcat, pre[i][2])                                      # [src rows, D] bf16
            # ELU'(o) from its output h; fp32 for a hidden layer's aggregation
            # backward, bf16 for the input layer's GEMMs
            nxt = torch.empty(dh.shape, dtype=f32 if i - 1 > 0 else bf16, device=dev)
            N.call("fg_gat_elu_bwd", N.ptr(dh), N.ptr(h), dh.numel(), N.ptr(nxt),
                   int(i - 1 > 0), s)
            do = nxt
        # the weight-gradient branch ran on its own stream: join before the
        # all-reduce / Adam read flat_grad
        torch.cuda.current_stream().wait_stream(self._wstream)

    @staticmethod
    def _attn_grads(v, dc):
        """From dc = d[c] ([2H, D]: el rows then er rows): d[a_l | a_r][k, f] =
        <W[kF+f], dc[row k]> and dW += a . dc."""
        Hh, Fh, D = v.heads, v.F, v.D
        dcv = dc.view(2, Hh, D).permute(1, 0, 2)                                # [Hh, 2, D]
        v.dattn.copy_(torch.bmm(v.W.view(Hh, Fh, D), dcv.transpose(1, 2)).permute(2, 0, 1))
        v.dW.view(Hh, Fh, D).baddbmm_(v.attn.permute(1, 2, 0), dcv)

    def _side_branch(self, *inputs):
        """Context: the ops inside run on the side stream after the main
        stream's work so far (the weight-gradient branch, which only feeds
        flat_grad and so overlaps the rest of the backward; a forward GEMM
        independent of the score path); the inputs are marked in use there."""
        import contextlib
        main = torch.cuda.current_stream()
        ws = self._wstream
        ws.wait_stream(main)
        for t in inputs:
            t.record_stream(ws)

        @contextlib.contextmanager
        def ctx():
            with torch.cuda.stream(ws):
                yield
        return ctx()

    # epoch / step API and CUDA-graph capture: SageTrainer's (same slot
    # logic, same attribute names; one graph per sampler slot)
    from .sage import SageTrainer as _S
    begin_epoch = _S.begin_epoch
    prepare = _S.prepare
    _load_seeds_staged = _S._load_seeds_staged
    replay = _S.replay
    step = _S.step
    capture = _S.capture
    del _S

    @torch.no_grad()
    def evaluate(self, ids, seed: int = 12345, max_batches: int | None = None) -> float:
        smp = DeviceSampler(self.sampler.g, self.cfg.fanouts, self.cfg.batch_size,
                            need_local=True)
        nb = smp.begin_epoch(ids, seed)
        if max_batches:
            nb = min(nb, max_batches)
        L = len(self.cfg.fanouts)
        correct = torch.zeros((), dtype=torch.int64, device=self.device)
        total = torch.zeros((), dtype=torch.int64, device=self.device)
        self.model.eval()
        for b in range(nb):
            sb = smp.sample(b)
            src = PickSource(self.codec, sb.picks[L - 1], sb.n_picks[L - 1], smp.pcaps[L - 1])
            with torch.autocast("cuda", dtype=torch.bfloat16):
                logits = self.model(src, sb, smp.caps, smp.pcaps[L - 1])
            valid = torch.arange(smp.caps[0], device=self.device) < sb.n_nodes[0]
            y = self.labels[sb.nodes[0].long()].long()
            pred = logits[:, :self.model.num_classes].argmax(1)
            correct += ((pred == y) & valid).sum()
            total += valid.sum()
        self.model.train()
        return float(correct.item()) / max(1, int(total.item()))

    def reference_state(self) -> dict:
        return {k: v.detach().float().cpu().clone() for k, v in self.model.state_dict().items()}
