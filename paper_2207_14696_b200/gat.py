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
from .aggregate import softmax_ce
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
               max_dst, N.ptr(n_dst), N.ptr(A), N.stream_handle())
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
        Hh, F, D = self.heads, self.F, self.D
        if self.wbd is None:
            self.wbd = torch.zeros((Hh * D, Hh * F), dtype=torch.bfloat16, device=self.W.device)
        # wbd[k*D + j, k*F + f] = W[k*F + f, j]
        self.wbd.view(Hh, D, Hh, F).diagonal(dim1=0, dim2=2).copy_(
            self.Wb.view(Hh, F, D).permute(2, 1, 0))


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


class GatTrainer:
    """Single-process (or one-rank-of-DDP) GAT trainer over device-resident
    data: sample -> GAT layers (input layer straight from the picks' code
    rows) -> fused softmax-CE -> autograd backward into one flat gradient ->
    flat all-reduce -> flat Adam; one CUDA graph per step."""

    def __init__(self, graph, codec, labels, num_classes: int, cfg: GatConfig,
                 process_group=None):
        self.cfg, self.codec, self.labels = cfg, codec, labels
        self.device = labels.device
        self.pg = process_group
        self.world = torch.distributed.get_world_size(process_group) if process_group else 1
        torch.manual_seed(cfg.seed)
        L = len(cfg.fanouts)
        self.sampler = DeviceSampler(graph, cfg.fanouts, cfg.batch_size, need_local=True)
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
        self.graph = None

    def _decode(self, sb):
        L = len(self.cfg.fanouts)
        return PickSource(self.codec, sb.picks[L - 1], sb.n_picks[L - 1], self.pick_cap)

    def _body(self, k: int = 0):
        sb = self.sampler.sample_loaded()
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
        x = self._decode(sb).x  # [pick_cap, d] bf16, pick order
        saved = []
        h = x
        for i, v in enumerate(self._views):
            l = L - 1 - i
            Hh, Fh, D = v.heads, v.F, v.D
            c = torch.bmm(v.attn.permute(1, 0, 2), v.W.view(Hh, Fh, D))     # [Hh, 2, D]
            c = c.permute(1, 0, 2).reshape(2 * Hh, D)                       # [el | er] rows
            cb = c.to(bf16)
            sc = torch.mm(h, cb.t(), out_dtype=f32)                         # [src rows, 2Hh]
            first = i == 0
            local = None if first else sb.local[l]
            e_cap = self.pick_cap if first else sb.local[l].numel()
            alpha = torch.empty((e_cap, Hh), dtype=f32, device=dev)
            q = torch.empty((self.caps[l], Hh), dtype=f32, device=dev)
            N.call("fg_gat_softmax_fwd", N.ptr(sc), N.ptr(sc[:, Hh:]), 2 * Hh,
                   N.ptr(sb.indptr[l]), N.ptr(local), self.caps[l], N.ptr(sb.n_nodes[l]), Hh,
                   0.2, N.ptr(alpha), N.ptr(q), s)
            if first:
                A = torch.empty((self.caps[l], Hh * D), dtype=bf16, device=dev)
                N.call("fg_gat_code_xagg_fwd", None, N.ptr(h), None, D, Hh, N.ptr(alpha),
                       N.ptr(sb.indptr[l]), self.caps[l], N.ptr(sb.n_nodes[l]), N.ptr(A), s)
                v.refresh_block_diag()
                o = torch.addmm(v.bb, A, v.wbd)                                # bf16
                z = A
            else:
                z = torch.mm(h, v.Wb.t())                                       # [src rows, Wd]
                o = torch.empty((self.caps[l], v.width), dtype=f32, device=dev)
                N.call("fg_gat_agg_fwd", N.ptr(z), v.width, Hh, N.ptr(alpha), N.ptr(sb.indptr[l]),
                       N.ptr(local), self.caps[l], N.ptr(sb.n_nodes[l]), N.ptr(o), s)
                o += v.b
            saved.append((h, c, cb, sc, alpha, q, z, local, e_cap))
            h = F.elu(o).to(bf16) if i < L - 1 else o
        logits = h
        C, ld = self.model.num_classes, logits.shape[1]
        do = torch.empty_like(logits)
        row_loss = torch.empty(logits.shape[0], dtype=f32, device=dev)
        N.call("fg_softmax_ce", N.ptr(logits), 0, C, ld, logits.shape[0], N.ptr(sb.n_nodes[0]),
               N.ptr(self.labels), N.ptr(sb.nodes[0]), N.ptr(do), N.ptr(row_loss),
               N.ptr(self.loss_buf), N.ptr(self.ce_ctr), s)
        # ---- backward
        for i in range(L - 1, -1, -1):
            v = self._views[i]
            l = L - 1 - i
            Hh, Fh, D = v.heads, v.F, v.D
            h, c, cb, sc, alpha, q, z, local, e_cap = saved[i]
            torch.sum(do, 0, dtype=f32, out=v.db)
            ds = torch.zeros((h.shape[0], 2 * Hh), dtype=f32, device=dev)
            if i == 0:
                A = z
                dA = torch.mm(do, v.wbd.t())                                    # [N, Hh*D] bf16
                # dW_k = do_k^T A_k: the diagonal blocks only (strided batched GEMM)
                dWk = torch.bmm(do.view(-1, Hh, Fh).permute(1, 2, 0),
                                A.view(-1, Hh, D).permute(1, 0, 2))
                v.dW.view(Hh, Fh, D).copy_(dWk)
                dalpha = torch.empty((e_cap, Hh), dtype=f32, device=dev)
                N.call("fg_gat_code_xagg_bwd", None, N.ptr(h), None, D, Hh, N.ptr(sb.indptr[l]),
                       self.caps[l], N.ptr(sb.n_nodes[l]), N.ptr(dA), N.ptr(dalpha), s)
                N.call("fg_gat_softmax_bwd", N.ptr(sc), 2 * Hh, N.ptr(q), N.ptr(alpha),
                       N.ptr(dalpha), N.ptr(sb.indptr[l]), None, self.caps[l],
                       N.ptr(sb.n_nodes[l]), Hh, 0.2, N.ptr(ds), N.ptr(ds[:, Hh:]), s)
                nb = N.lib().fg_gat_code_scores_bwd_blocks(e_cap)
                part = torch.empty((nb, 2 * Hh, D), dtype=f32, device=dev)
                N.call("fg_gat_code_scores_bwd", None, N.ptr(h), None, N.ptr(sb.n_picks[l]), e_cap,
                       D, Hh, N.ptr(ds), N.ptr(ds[:, Hh:]), 2 * Hh, N.ptr(part), s)
                dc = part.sum(0)
            else:
                dz = torch.zeros((h.shape[0], v.width), dtype=f32, device=dev)
                dalpha = torch.zeros((e_cap, Hh), dtype=f32, device=dev)
                N.call("fg_gat_agg_bwd", N.ptr(z), v.width, Hh, N.ptr(alpha), N.ptr(sb.indptr[l]),
                       N.ptr(local), self.caps[l], N.ptr(sb.n_nodes[l]), N.ptr(do), N.ptr(dz),
                       N.ptr(dalpha), s)
                N.call("fg_gat_softmax_bwd", N.ptr(sc), 2 * Hh, N.ptr(q), N.ptr(alpha),
                       N.ptr(dalpha), N.ptr(sb.indptr[l]), N.ptr(local), self.caps[l],
                       N.ptr(sb.n_nodes[l]), Hh, 0.2, N.ptr(ds), N.ptr(ds[:, Hh:]), s)
                dzb, dsb = dz.to(bf16), ds.to(bf16)
                torch.mm(dzb.t(), h, out_dtype=f32, out=v.dW)
                dc = torch.mm(dsb.t(), h, out_dtype=f32)                      # [2Hh, D]
            dcv = dc.view(2, Hh, D).permute(1, 0, 2)                            # [Hh, 2, D]
            # d[a_l | a_r][k, f] = <W[kF+f], dc[el|er row k]>;  dW += a . dc
            v.dattn.copy_(torch.bmm(v.W.view(Hh, Fh, D), dcv.transpose(1, 2)).permute(2, 0, 1))
            v.dW.view(Hh, Fh, D).baddbmm_(v.attn.permute(1, 2, 0), dcv)
            if i == 0:
                break
            dh = torch.addmm(torch.mm(dzb, v.Wb), dsb, cb)                      # [src rows, D] bf16
            # ELU'(o) from its output h: 1 where h > 0, h + 1 elsewhere
            do = torch.ops.aten.elu_backward(dh, 1.0, 1.0, 1.0, True, h)
            if i - 1 > 0:
                do = do.float()

    def begin_epoch(self, train_ids, epoch: int = 0) -> int:
        r = torch.distributed.get_rank(self.pg) if self.world > 1 else 0
        shard = ddp.shard_ids(train_ids, r, self.world)
        self._nb = self.sampler.begin_epoch(shard, ddp.rank_seed(self.cfg.seed, epoch, r,
                                                                 self.world))
        self._nb = ddp.agree_num_batches(self._nb, self.pg, self.device)
        return self._nb

    def capture(self, warmup_batches: int = 3):
        rng_save = self.sampler.rng.clone()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for b in range(warmup_batches):
                self.sampler.load_seeds(b % self._nb)
                self._body()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._body()
        torch.cuda.synchronize()
        self.sampler.rng.copy_(rng_save)

    # same step API as SageTrainer (serial sampling: one slot)
    pipeline = False

    @property
    def samplers(self):
        return [self.sampler]

    def prepare(self, b: int, seeds_host=None) -> None:
        if seeds_host is not None:
            self.sampler.load_seeds_host(seeds_host)
        else:
            self.sampler.load_seeds(b)

    def replay(self, b: int):
        if self.graph is not None:
            self.graph.replay()
        else:
            self._body()
        return self.loss_buf

    def step(self, b: int, seeds_host=None):
        self.prepare(b, seeds_host)
        return self.replay(b)

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
