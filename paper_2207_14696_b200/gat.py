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
decoded on the device by the codec's gather-dequant kernel (bf16) and
projected by one GEMM; hidden layers project the previous layer's output.
Edge operators are CUDA kernels wrapped as autograd Functions; the GEMMs,
LeakyReLU/ELU and the loss are torch/cuBLAS plus the fused softmax-CE kernel.
"""

from __future__ import annotations

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
        N.call("fg_gat_softmax_fwd", N.ptr(el), N.ptr(er), N.ptr(indptr), N.ptr(local), max_dst,
               N.ptr(n_dst), heads, slope, N.ptr(alpha), N.ptr(q), N.stream_handle())
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
        N.call("fg_gat_softmax_bwd", N.ptr(el), N.ptr(q), N.ptr(alpha),
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


def _chunked_sum_bmm(a, b, ch: int = 64):
    """sum_n a[n]^T b[n] for a [N, p], b [N, q] with N ~ 1e5: 64 K-chunks in
    one batched GEMM, then a sum (cuBLAS picks an 8-CTA kernel for the
    single skinny K = N product)."""
    n = a.shape[0]
    pad = (-n) % ch
    if pad:
        a = torch.cat([a, a.new_zeros(pad, a.shape[1])])
        b = torch.cat([b, b.new_zeros(pad, b.shape[1])])
    return torch.bmm(a.view(ch, -1, a.shape[1]).transpose(1, 2),
                     b.view(ch, -1, b.shape[1])).sum(0)


class HeadProject(torch.autograd.Function):
    """out[n, k*F:(k+1)*F] = agg[n, k*d:(k+1)*d] @ w[k]^T, w [H, F, d]."""

    @staticmethod
    def forward(ctx, agg, w):
        n = agg.shape[0]
        H, f, d = w.shape
        a = agg.view(n, H, d).transpose(0, 1).to(torch.bfloat16)          # [H, n, d]
        out = torch.bmm(a, w.to(torch.bfloat16).transpose(1, 2))           # [H, n, F]
        ctx.save_for_backward(a, w)
        return out.transpose(0, 1).reshape(n, H * f).float()

    @staticmethod
    def backward(ctx, dout):
        a, w = ctx.saved_tensors
        H, f, d = w.shape
        n = a.shape[1]
        g = dout.view(n, H, f).transpose(0, 1).to(torch.bfloat16)          # [H, n, F]
        dw = torch.stack([_chunked_sum_bmm(g[k], a[k]) for k in range(H)])  # [H, F, d]
        return None, dw.float()


class GatInputAggregate(torch.autograd.Function):
    """A[v, k*d:(k+1)*d] = sum_e alpha[e,k] x[e] over decoded pick rows x
    (constant input: no dx)."""

    @staticmethod
    def forward(ctx, x, alpha, indptr, n_dst, max_dst: int):
        x = x.to(torch.bfloat16).contiguous()
        d, heads = x.shape[1], alpha.shape[1]
        out = torch.empty((max_dst, heads * d), dtype=torch.float32, device=x.device)
        N.call("fg_gat_xagg_fwd", N.ptr(x), d, heads, N.ptr(alpha), N.ptr(indptr), max_dst,
               N.ptr(n_dst), N.ptr(out), N.stream_handle())
        ctx.save_for_backward(x, indptr, n_dst)
        ctx.max_dst, ctx.heads, ctx.e_cap = max_dst, heads, alpha.shape[0]
        return out

    @staticmethod
    def backward(ctx, dout):
        x, indptr, n_dst = ctx.saved_tensors
        dalpha = torch.zeros((ctx.e_cap, ctx.heads), dtype=torch.float32, device=x.device)
        N.call("fg_gat_xagg_bwd", N.ptr(x), x.shape[1], ctx.heads, N.ptr(indptr), ctx.max_dst,
               N.ptr(n_dst), N.ptr(dout.float().contiguous()), N.ptr(dalpha), ctx.e_cap,
               N.stream_handle())
        return None, dalpha, None, None, None


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

    def _forward_input(self, x, indptr, n_dst, max_dst, e_cap, slope):
        """Same math for the input layer, rearranged by linearity: scores
        el = x (W_k^T a_l[k]) per pick, the attention-weighted sum of the
        decoded picks per head, then one [N_dst, d] x [d, F] product per head
        -- no per-pick projection (518 K x 256 at products shape)."""
        H, f = self.heads, self.width // self.heads
        d = x.shape[1]
        w = self.lin.weight.view(H, f, d)                       # [H, F, d]
        c = torch.cat([torch.einsum("hfd,hf->hd", w, self.attn_l),
                       torch.einsum("hfd,hf->hd", w, self.attn_r)])  # [2H, d]
        s = PickScores.apply(x.to(torch.bfloat16), c)           # [E, 2H]
        alpha = GatAttention.apply(s[:, :H], s[:, H:], indptr, None, n_dst, max_dst, e_cap, slope)
        agg = GatInputAggregate.apply(x, alpha, indptr, n_dst, max_dst)   # [N, H*d]
        return HeadProject.apply(agg, w) + self.bias


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

    def forward(self, x_picks, sb, caps, pick_cap):
        """x_picks: decoded input rows of the last block's picks [pick_cap, d]."""
        L = len(self.layers)
        h = x_picks
        for i, layer in enumerate(self.layers):
            l = L - 1 - i  # block feeding layer i
            local = None if l == L - 1 else sb.local[l]
            e_cap = pick_cap if l == L - 1 else sb.local[l].numel()
            h = layer(h, sb.indptr[l], local, sb.n_nodes[l], caps[l], e_cap)
            if i < L - 1:
                h = F.elu(h)
        return h


@dataclass
class GatConfig:
    fanouts: tuple = (15, 10, 5)
    batch_size: int = 1024
    hidden: int = 256
    heads: int = 4
    lr: float = 3e-3
    seed: int = 0
    use_graph: bool = True


class GatTrainer:
    """Single-process (or one-rank-of-DDP) GAT trainer over device-resident
    data: sample -> decode the last block's picks (codec gather-dequant, bf16)
    -> GAT layers -> fused softmax-CE -> autograd backward -> flat all-reduce
    -> Adam; one CUDA graph per step."""

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
        self.opt = torch.optim.Adam(self.model.parameters(), lr=cfg.lr, capturable=True)
        self.loss_buf = torch.zeros((), dtype=torch.float32, device=self.device)
        self.graph = None

    def _decode(self, sb):
        L = len(self.cfg.fanouts)
        return self.codec.gather(sb.picks[L - 1], out_dtype=torch.bfloat16, check=False)

    def _body(self, k: int = 0):
        sb = self.sampler.sample_loaded()
        x = self._decode(sb)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            logits = self.model(x, sb, self.caps, self.pick_cap)
        loss = softmax_ce(logits.contiguous(), self.labels, sb.nodes[0], sb.n_nodes[0],
                          self.model.num_classes)
        self.opt.zero_grad(set_to_none=False)
        loss.backward()
        if self.world > 1:
            for p in self.model.parameters():
                ddp.average_flat_(p.grad.view(-1), self.pg)
        self.opt.step()
        self.loss_buf.copy_(loss.detach())

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
            x = self.codec.gather(sb.picks[L - 1], out_dtype=torch.bfloat16, check=False)
            with torch.autocast("cuda", dtype=torch.bfloat16):
                logits = self.model(x, sb, smp.caps, smp.pcaps[L - 1])
            valid = torch.arange(smp.caps[0], device=self.device) < sb.n_nodes[0]
            y = self.labels[sb.nodes[0].long()].long()
            pred = logits[:, :self.model.num_classes].argmax(1)
            correct += ((pred == y) & valid).sum()
            total += valid.sum()
        self.model.train()
        return float(correct.item()) / max(1, int(total.item()))

    def reference_state(self) -> dict:
        return {k: v.detach().float().cpu().clone() for k, v in self.model.state_dict().items()}
