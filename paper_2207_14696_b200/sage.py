"""GraphSAGE mini-batch training on compressed features (new layer L4; the
reference has no trainer).

Model (mean aggregator): the reference defines aggregation as
the row-stochastic mean over stored neighbours including the self-loop
(factors.py:108-114).  Restricted to the sampled blocks:
    h_{L-1}[v] = act(W_1 · mean_{u in picks(v)} x_u + b_1)   (fused kernel)
    h_l[v]     = act(W · mean_{u in picks(v)} h_{l+1}[u] + b)
with fanouts[0] applied at the seeds (pipeline.py:207 convention),
so the input-side aggregation uses fanouts[-1].

One step = sample (device PCG64 stream) -> fused gather-dequant-mean ->
bf16 SAGE layers fwd/bwd -> (NCCL all-reduce of the flat gradient) -> Adam.
Every buffer has a static capacity, so the whole step is captured once into
a CUDA graph and replayed per batch; the only per-step host traffic is the
seed ids in and the loss out.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

from . import ddp
from . import _native as N
from .aggregate import (alloc_aggregate, block_mean, gather_dequant_mean, input_block_mean, kgemm,
                        padded_dim, softmax_ce, wgrad_scratch, wgrad_supported)
from .sampler import DeviceSampler


class SageModel(nn.Module):
    """Every layer is a bias-free Linear over an input that carries a
    constant-1 column: layer 0 reads the padded aggregate (column in_dim = 1),
    layer i > 0 reads the block-mean output widened by a [1, 0 x 7] block
    (column hidden = 1).  Biases therefore live in weight columns and their
    gradients come out of the weight GEMMs (no reductions over the ~1e5-row
    activations in backward).  Initialisation matches nn.Linear."""

    def __init__(self, in_dim: int, hidden: int, num_classes: int, num_layers: int,
                 dropout: float = 0.0, in_pitch: int | None = None):
        super().__init__()
        dims = [in_dim] + [hidden] * (num_layers - 1) + [num_classes]
        self.in_dims = dims[:-1]
        self.out_dims = dims[1:]
        self.num_classes = num_classes
        # the class dimension is padded to a multiple of 8 (zero weight rows:
        # their logits are 0, their gradients 0, Adam leaves them at 0) so
        # every GEMM operand is 16-byte aligned (aligned cuBLAS kernels)
        c_pad = (num_classes + 7) // 8 * 8
        lins = []
        for i in range(num_layers):
            pitch = (in_pitch or in_dim + 1) if i == 0 else dims[i] + 8
            rows = c_pad if i == num_layers - 1 else dims[i + 1]
            lin = nn.Linear(pitch, rows, bias=False)
            ref = nn.Linear(dims[i], dims[i + 1])
            with torch.no_grad():
                lin.weight.zero_()
                lin.weight[:dims[i + 1], :dims[i]] = ref.weight
                lin.weight[:dims[i + 1], dims[i]] = ref.bias
            lins.append(lin)
        self.lins = nn.ModuleList(lins)
        self.dropout = dropout
        self.fuse_input = True

    def fused_input_ok(self) -> bool:
        """Input layer + first hidden block mean through ``input_block_mean``
        (backward = edge-tiled tcgen05 dW, fg_wgrad.cu) when there is a hidden
        block, no dropout, and the shape is one the kernel takes."""
        w = self.lins[0].weight
        return (self.fuse_input and len(self.lins) > 1 and not self.dropout
                and wgrad_supported(w.shape[0], w.shape[1]))

    def forward(self, agg_in, sb, caps, wgrad_scratch=None):
        """agg_in: [caps[L-1], pitch] mean of decoded inputs over the last
        block (+ ones column); sb: SampledBatch; returns logits [caps[0], C]."""
        L = len(self.lins)
        first = 1
        if self.training and self.fused_input_ok():
            l = L - 2
            h = input_block_mean(agg_in, self.lins[0].weight, sb.indptr[l], sb.local[l],
                                 sb.n_nodes[l], caps[l], True, wgrad_scratch,
                                 sb.ew[l] if sb.ew else None)
            h = self.lins[1](h)
            first = 2
        else:
            h = self.lins[0](agg_in)
        for i in range(first, L):
            l = L - 1 - i  # block index feeding this layer
            trans = sb.trans[l] if sb.trans else None
            ew = sb.ew[l] if sb.ew else None
            if self.dropout and self.training:
                h = F.dropout(F.relu(h), self.dropout)
                a = block_mean(h.to(torch.bfloat16), sb.indptr[l], sb.local[l], sb.n_nodes[l],
                               caps[l], trans=trans, bias_col=True, edge_w=ew)
            else:  # ReLU fused into the block-mean gather
                a = block_mean(h.to(torch.bfloat16), sb.indptr[l], sb.local[l], sb.n_nodes[l],
                               caps[l], relu=True, trans=trans, bias_col=True, edge_w=ew)
            h = self.lins[i](a)
        return h

    def reference_state(self) -> dict:
        """Weights as plain (weight, bias) Linear layers (for the CPU oracle)."""
        out = {}
        for i, (lin, d) in enumerate(zip(self.lins, self.in_dims)):
            w = lin.weight.detach().float().cpu()
            o = self.out_dims[i]
            out[f"lins.{i}.weight"] = w[:o, :d].clone()
            out[f"lins.{i}.bias"] = w[:o, d].clone()
        return out


class FlatAdam:
    """torch.optim.Adam(betas=(0.9, 0.999), eps=1e-8) over one flat buffer,
    one kernel per step (``fg_adam_step``), device-side step counter; keeps
    an optional bf16 shadow of the parameters for the next forward."""

    def __init__(self, param, grad, lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.0,
                 param_bf16=None):
        from . import _native as N
        self.N = N
        self.p, self.g, self.pb = param, grad, param_bf16
        self.m = torch.zeros_like(param)
        self.v = torch.zeros_like(param)
        self.t = torch.zeros(2, dtype=torch.int64, device=param.device)  # [step, block ctr]
        self.lr, self.b1, self.b2, self.eps, self.wd = lr, betas[0], betas[1], eps, weight_decay
        if self.pb is not None:
            N.call("fg_f32_to_bf16_plain", N.ptr(param), param.numel(), N.ptr(self.pb),
                   N.stream_handle())

    def step(self):
        N = self.N
        N.call("fg_adam_step", N.ptr(self.p), N.ptr(self.g), N.ptr(self.m), N.ptr(self.v),
               self.p.numel(), N.ptr(self.t), self.lr, self.b1, self.b2, self.eps, self.wd,
               N.ptr(self.pb) if self.pb is not None else None, N.stream_handle())


@dataclass
class TrainConfig:
    fanouts: tuple = (15, 10, 5)
    batch_size: int = 1024
    hidden: int = 256
    lr: float = 3e-3
    seed: int = 0
    dropout: float = 0.0
    use_graph: bool = True
    agg_dtype: torch.dtype = torch.bfloat16
    # sample batch b+1 on a side stream while batch b trains (two sampler
    # slots sharing one PCG64 stream: the batches are the same as serial)
    pipeline: bool = True
    # "mean" (SAGE-mean, the reference's row-stochastic D^-1 A) or "gcn"
    # (Kipf's D^-1/2 A D^-1/2, sampled estimator; BASELINE config E)
    aggregator: str = "mean"


class SageTrainer:
    """Single-process (or one-rank-of-DDP) trainer over device-resident data."""

    def __init__(self, graph, codec, labels, num_classes: int, cfg: TrainConfig,
                 process_group=None):
        self.cfg = cfg
        self.codec = codec
        self.labels = labels
        self.device = labels.device
        self.pg = process_group
        self.world = torch.distributed.get_world_size(process_group) if process_group else 1
        torch.manual_seed(cfg.seed)
        L = len(cfg.fanouts)
        # input layer sees the 16-aligned padded aggregate (zero columns past d)
        self.model = SageModel(codec.d, cfg.hidden, num_classes, L, cfg.dropout,
                               in_pitch=padded_dim(codec.d)).to(self.device)
        # the fused input layer needs no transpose of its block (block L-2)
        fused = self.model.fused_input_ok()
        tl = range(L - 2) if fused else None
        self.sampler = DeviceSampler(graph, cfg.fanouts, cfg.batch_size, need_local=True,
                                     need_transpose=True, transpose_layers=tl,
                                     aggregator=cfg.aggregator)
        self.samplers = [self.sampler]
        self.pipeline = cfg.pipeline
        if self.pipeline:
            self.samplers.append(DeviceSampler(graph, cfg.fanouts, cfg.batch_size,
                                               need_local=True, need_transpose=True,
                                               transpose_layers=tl, share=self.sampler,
                                               aggregator=cfg.aggregator))
            # high priority: the latency-bound sampler kernels take SMs as soon as
            # the wide training kernels free them
            self.side = torch.cuda.Stream(self.device,
                                          priority=int(os.environ.get("FG_SIDE_PRIORITY", "-1")))
        self.caps = self.sampler.caps
        # flat gradient buffer: one all-reduce per step
        # one flat fp32 buffer each for params, grads and Adam moments: a
        # single all-reduce and a single optimizer kernel per step
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
        if self.world > 1:  # identical initial weights on every rank
            torch.distributed.broadcast(self.flat_param, 0, group=self.pg)
        # bf16 shadow of the parameters (written by the Adam kernel): the
        # explicit step's GEMM operands, so no per-step weight casts
        self.flat_bf16 = torch.zeros(total, dtype=torch.bfloat16, device=self.device)
        self.w_bf16, self.w_grad = [], []
        off = 0
        for p in params:
            n = p.numel()
            self.w_bf16.append(self.flat_bf16[off:off + n].view_as(p))
            self.w_grad.append(self.flat_grad[off:off + n].view_as(p))
            off += n
        self.opt = FlatAdam(self.flat_param, self.flat_grad, lr=cfg.lr, param_bf16=self.flat_bf16)
        # explicit forward/backward (no autograd) unless dropout is on
        self.explicit = not cfg.dropout
        self.loss_buf = torch.zeros((), dtype=torch.float32, device=self.device)
        self.ce_ctr = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.agg = alloc_aggregate(self.caps[L - 1], codec.d, cfg.agg_dtype, self.device)
        w0 = self.model.lins[0].weight
        self.wgrad_scratch = None
        self.relu_bits = None
        if fused:
            self.wgrad_scratch = wgrad_scratch(w0.shape[0], w0.shape[1], self.device)
        # h0's packed ReLU mask, written by the first block mean's forward and
        # read by the dW0 kernel or, on the GEMM path (MAG: P > 256), by the
        # block-mean backward instead of the bf16 h0 rows (FG_RELU_BITS=0:
        # the backward reads h0 itself)
        if (self.explicit and L > 1 and w0.shape[0] % 8 == 0
                and os.environ.get("FG_RELU_BITS", "1") != "0"):
            self.relu_bits = torch.empty((self.caps[L - 1], w0.shape[0] // 8),
                                         dtype=torch.uint8, device=self.device)
        # forward: input projection fused with the first block mean
        # (fg_infwd.cu) when the shape allows -- mean aggregator only (products
        # step 0.258 -> 0.247 ms; GCN's weighted variant measured no gain);
        # FG_INFWD=0 keeps GEMM + block mean, FG_INFWD=2 forces it for GCN too
        mode = os.environ.get("FG_INFWD", "1")
        self.infwd = bool(fused and self.relu_bits is not None and self.explicit
                          and (mode == "2" or (mode == "1" and cfg.aggregator == "mean"))
                          and N.lib().fg_input_block_mean_supported(
                              w0.shape[0], w0.shape[1], cfg.fanouts[L - 2]))
        # dW0 on the GEMM path (MAG240M-shape: K = 153,600 aggregate rows,
        # 256 x 784 output): K cut into 16 slices by one batched GEMM + a
        # sum (tools/gemm_probe.py on the B200: 65 vs 90 us for one cuBLAS
        # GEMM; 32 slices: 77 us).  FG_SAGE_KGEMM=0/1 forces it off/on.
        kg = os.environ.get("FG_SAGE_KGEMM", "auto")
        self.kgemm = kg == "1" or (kg == "auto" and not fused)
        self.kgemm_chunks = int(os.environ.get("FG_SAGE_KGEMM_CHUNKS", "16"))
        self.graph = None
        self.graphs = {}
        self._primed, self._next = False, 0
        self.steps_run = 0

    # ------------------------------------------------------------- step
    def _train(self, sb):
        if self.explicit:
            return self._train_explicit(sb)
        return self._train_autograd(sb)

    def _body(self, k: int = 0):
        """One step.  Serial: sample slot 0's loaded seeds, then train.
        Pipelined: train the batch already in slot k on the current stream
        while the side stream samples the next batch (seeds already loaded)
        into slot 1-k; the side stream first waits for the work already
        queued (the previous step still reading slot 1-k) and is joined
        before the step ends."""
        if not self.pipeline:
            return self._train(self.sampler.sample_loaded())
        cur = torch.cuda.current_stream()
        self.side.wait_stream(cur)
        with torch.cuda.stream(self.side):
            self.samplers[1 - k].sample_loaded()
        self._train(self.samplers[k].batch_view())
        cur.wait_stream(self.side)

    def _train_explicit(self, sb):
        """One training step with the backward written out (SageModel's
        math, bf16 GEMMs on the Adam kernel's bf16 weight shadow, fp32 weight
        gradients straight into the flat gradient buffer): no autograd
        bookkeeping, weight casts, gradient zero-fill or accumulation kernels.

        forward   in_0 = agg;  h_i = in_i W_i^T;  in_{i+1} = mean_block(relu h_i) (+ ones col)
        backward  dW_i = dh_i^T in_i;  d in_i = dh_i W_i[:, :H];
                  dh_{i-1} = relu'(h_{i-1}) * mean_block^T(d in_i)
        with the input layer's dW_0 from the edge-tiled tcgen05 kernel when
        the shape allows (fg_block_mean_wgrad)."""
        L = len(self.cfg.fanouts)
        caps = self.caps
        s = N.stream_handle()
        ew = sb.ew or [None] * L
        gather_dequant_mean(self.codec, sb.indptr[L - 1], sb.picks[L - 1], sb.n_nodes[L - 1],
                            caps[L - 1], out=self.agg, edge_w=ew[L - 1])
        W, dW = self.w_bf16, self.w_grad
        ins, hs = [self.agg], []
        fused = self.wgrad_scratch is not None
        for i in range(L):
            if i == 0 and self.infwd:
                # h0 = agg W0^T and its block mean in one tcgen05 kernel (h0
                # stays on chip; its ReLU bits go to the dW0 kernel)
                l, H = L - 2, W[0].shape[0]
                a = torch.empty((caps[l], H + 8), dtype=torch.bfloat16, device=self.device)
                N.call("fg_input_block_mean_fwd", N.ptr(self.agg), self.agg.shape[1],
                       N.ptr(W[0]), H, N.ptr(sb.indptr[l]), N.ptr(sb.local[l]),
                       N.ptr(sb.n_nodes[l]), caps[l], self.cfg.fanouts[l], N.ptr(ew[l]),
                       N.ptr(a), H + 8, N.ptr(self.relu_bits), s)
                hs.append(None)
                ins.append(a)
                continue
            h = torch.mm(ins[i], W[i].t())
            hs.append(h)

            if i < L - 1:
                l = L - 2 - i  # block feeding layer i+1
                H = h.shape[1]
                a = torch.empty((caps[l], H + 8), dtype=torch.bfloat16, device=self.device)
                if i == 0 and self.relu_bits is not None:
                    # h0's ReLU mask as bits for the edge-tiled dW0 (mask_kind 2)
                    N.call("fg_block_mean_fwd_bits", N.ptr(h), H, N.ptr(sb.indptr[l]),
                           N.ptr(sb.local[l]), N.ptr(sb.n_nodes[l]), caps[l], N.ptr(a), H + 8,
                           N.ptr(ew[l]), N.ptr(self.relu_bits), s)
                else:
                    N.call("fg_block_mean_fwd", N.ptr(h), H, N.ptr(sb.indptr[l]),
                           N.ptr(sb.local[l]), N.ptr(sb.n_nodes[l]), caps[l], N.ptr(a), H + 8,
                           1, N.ptr(ew[l]), s)
                ins.append(a)
        logits = hs[-1]
        ld = logits.shape[1]
        dh = torch.empty_like(logits)
        row_loss = torch.empty(logits.shape[0], dtype=torch.float32, device=self.device)
        N.call("fg_softmax_ce", N.ptr(logits), 1, self.model.num_classes, ld, logits.shape[0],
               N.ptr(sb.n_nodes[0]), N.ptr(self.labels), N.ptr(sb.nodes[0]), N.ptr(dh),
               N.ptr(row_loss), N.ptr(self.loss_buf), N.ptr(self.ce_ctr), s)
        for i in range(L - 1, -1, -1):
            if self.kgemm:  # K ~ 1e5 rows (MAG's GEMM-path dW0): chunked batched GEMM
                kgemm(dh, ins[i], dW[i], chunks=self.kgemm_chunks)
            else:
                torch.mm(dh.t(), ins[i], out_dtype=torch.float32, out=dW[i])
            if i == 0:
                break
            H = W[i - 1].shape[0]
            din = torch.mm(dh, W[i][:, :H])
            l = L - 1 - i  # block feeding layer i
            if fused and i == 1:
                N.call("fg_block_mean_wgrad", N.ptr(din), H, N.ptr(sb.indptr[l]),
                       N.ptr(sb.local[l]), N.ptr(sb.n_nodes[l]), caps[l], N.ptr(ew[l]),
                       *((N.ptr(self.relu_bits), 2) if self.relu_bits is not None
                         else (N.ptr(hs[0]), 1)), H,
                       N.ptr(self.agg), self.agg.shape[1], N.ptr(dW[0]),
                       N.ptr(self.wgrad_scratch), self.wgrad_scratch.numel() * 4, s)
                break
            t_indptr, t_dst, t_w, n_src = sb.trans[l]
            dh = torch.empty_like(hs[i - 1])
            if i == 1 and self.relu_bits is not None:
                N.call("fg_block_mean_bwd_t_bits", N.ptr(din), H, H, N.ptr(t_indptr),
                       N.ptr(t_dst), N.ptr(t_w), N.ptr(n_src), dh.shape[0],
                       N.ptr(self.relu_bits), N.ptr(dh), s)
            else:
                N.call("fg_block_mean_bwd_t", N.ptr(din), H, H, N.ptr(t_indptr), N.ptr(t_dst),
                       N.ptr(t_w), N.ptr(n_src), dh.shape[0], N.ptr(hs[i - 1]), N.ptr(dh), s)
        ddp.average_flat_(self.flat_grad, self.pg)
        self.opt.step()

    def _train_autograd(self, sb):
        L = len(self.cfg.fanouts)
        gather_dequant_mean(self.codec, sb.indptr[L - 1], sb.picks[L - 1], sb.n_nodes[L - 1],
                            self.caps[L - 1], out=self.agg,
                            edge_w=sb.ew[L - 1] if sb.ew else None)
        with torch.autocast("cuda", dtype=torch.bfloat16):
            logits = self.model(self.agg, sb, self.caps, self.wgrad_scratch)
        loss = softmax_ce(logits, self.labels, sb.nodes[0], sb.n_nodes[0],
                          self.model.num_classes)
        self.flat_grad.zero_()
        loss.backward()
        ddp.average_flat_(self.flat_grad, self.pg)
        self.opt.step()
        self.loss_buf.copy_(loss.detach())

    def capture(self, warmup_batches: int = 3):
        """Warm up eagerly (allocations, cuBLAS handles, kernel attributes),
        then capture the step into CUDA graphs (one per sampler slot).  The
        PCG64 stream is restored afterwards, so the epoch's batches are
        unchanged by the warm-up (the warm-up steps do update the model)."""
        rng_save = self.sampler.rng.clone()
        nxt = self._next
        if self.world > 1 and torch.distributed.get_backend(self.pg) != "nccl":
            # a host-side (gloo) all-reduce cannot live in a CUDA graph: the
            # step stays eager (NCCL's all-reduce is captured below)
            self.graphs, self.graph = {}, None
            return
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for b in range(warmup_batches):
                self.prepare(b)
                self._body(b % len(self.samplers))
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        for k in range(len(self.samplers)):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._body(k)
            self.graphs[k] = g
        torch.cuda.synchronize()
        self.graph = self.graphs[0]
        self.sampler.rng.copy_(rng_save)
        self._primed, self._next = False, nxt

    def begin_epoch(self, train_ids, epoch: int = 0) -> int:
        """Seeds are sharded like DDP: rank r takes ids[r::W] with seed
        seed*W + r + epoch."""
        import time
        t0 = time.perf_counter()
        r = torch.distributed.get_rank(self.pg) if self.world > 1 else 0
        shard = ddp.shard_ids(train_ids, r, self.world)
        t1 = time.perf_counter()
        self._nb = self.sampler.begin_epoch(shard, ddp.rank_seed(self.cfg.seed, epoch, r,
                                                                 self.world))
        t2 = time.perf_counter()
        self._nb = ddp.agree_num_batches(self._nb, self.pg, self.device)
        self._primed, self._next = False, 0
        self.begin_epoch_timing = {"shard_s": t1 - t0, "sampler_s": t2 - t1,
                                   "agree_s": time.perf_counter() - t2}
        return self._nb

    def prepare(self, b: int, seeds_host: torch.Tensor | None = None) -> None:
        """Stage the inputs of step b.  Serial: batch b's seeds (from the
        device permutation, or copied from pinned host memory).  Pipelined:
        batch b must already be sampled into slot b % 2 (the previous step
        did it; otherwise it is sampled here first), and this loads the seeds
        of batch b+1 -- ``seeds_host`` if given, else the permutation slice
        (wrapping at the epoch end) -- for the step to sample."""
        if not self.pipeline:
            if seeds_host is not None:
                self.sampler.load_seeds_host(seeds_host)
            else:
                self.sampler.load_seeds(b)
            return
        if not (self._primed and self._next == b):
            cur = self.samplers[b % 2]
            cur.load_seeds(b % self._nb)
            cur.sample_loaded()
        nxt = self.samplers[(b + 1) % 2]
        if seeds_host is not None:
            self._load_seeds_staged(nxt, seeds_host)
        else:
            nxt.load_seeds((b + 1) % self._nb)
        self._primed, self._next = True, b + 1

    def _load_seeds_staged(self, smp, seeds_host) -> None:
        """Pipelined end-to-end input: the H2D copy of batch b+1's seeds runs
        on a copy stream into one of two device staging buffers, so it
        overlaps the step still running (the slot's own seed layer is read by
        that step's loss until it ends); the main stream then only waits for
        it and moves the 4 KB device to device.  The staging buffer of the
        same parity is rewritten only after its previous device copy ran.
        Unsorted, non-int32 or pageable seeds take the plain path."""
        import numpy as np
        if not (seeds_host.dtype == torch.int32 and seeds_host.is_pinned()
                and 0 < seeds_host.numel() <= smp.bs):
            smp.load_seeds_host(seeds_host)
            return
        a = seeds_host.numpy()
        if not bool(np.all(a[1:] >= a[:-1])):
            smp.load_seeds_host(seeds_host)
            return
        if getattr(self, "_h2d", None) is None:
            self._h2d = torch.cuda.Stream(self.device)
            self._stage = [torch.empty(smp.bs, dtype=torch.int32, device=self.device)
                           for _ in range(2)]
            self._stage_ready = [torch.cuda.Event() for _ in range(2)]
            self._stage_done = [torch.cuda.Event() for _ in range(2)]
            self._stage_used = [False, False]
            self._stage_i = 0
        j = self._stage_i
        self._stage_i ^= 1
        cnt = seeds_host.numel()
        if self._stage_used[j]:
            self._h2d.wait_event(self._stage_done[j])
        with torch.cuda.stream(self._h2d):
            self._stage[j][:cnt].copy_(seeds_host, non_blocking=True)
            self._stage_ready[j].record()
        cur = torch.cuda.current_stream()
        cur.wait_event(self._stage_ready[j])
        smp.nodes[0][:cnt].copy_(self._stage[j][:cnt], non_blocking=True)
        smp.n_nodes[0].fill_(cnt)
        self._stage_done[j].record(cur)
        self._stage_used[j] = True

    def replay(self, b: int):
        """Run step b (after ``prepare(b)``) from its CUDA graph, or eagerly."""
        k = b % len(self.samplers)
        if k in self.graphs:
            self.graphs[k].replay()
        else:
            self._body(k)
        self.steps_run += 1
        return self.loss_buf

    def step(self, b: int, seeds_host: torch.Tensor | None = None):
        """One training step on batch b (see ``prepare`` for ``seeds_host``)."""
        self.prepare(b, seeds_host)
        return self.replay(b)

    # -------------------------------------------------------- evaluation
    @torch.no_grad()
    def evaluate(self, ids, seed: int = 12345, max_batches: int | None = None) -> float:
        """Accuracy over ``ids`` with the same sampled-block model."""
        smp = DeviceSampler(self.sampler.g, self.cfg.fanouts, self.cfg.batch_size,
                            need_local=True, aggregator=self.cfg.aggregator,
                            need_transpose=self.cfg.aggregator != "mean")
        nb = smp.begin_epoch(ids, seed)
        if max_batches:
            nb = min(nb, max_batches)
        L = len(self.cfg.fanouts)
        agg = alloc_aggregate(smp.caps[L - 1], self.codec.d, self.cfg.agg_dtype, self.device)
        correct = torch.zeros((), dtype=torch.int64, device=self.device)
        total = torch.zeros((), dtype=torch.int64, device=self.device)
        self.model.eval()
        for b in range(nb):
            sb = smp.sample(b)
            gather_dequant_mean(self.codec, sb.indptr[L - 1], sb.picks[L - 1],
                                sb.n_nodes[L - 1], smp.caps[L - 1], out=agg,
                                edge_w=sb.ew[L - 1] if sb.ew else None)
            with torch.autocast("cuda", dtype=torch.bfloat16):
                logits = self.model(agg, sb, smp.caps)
            valid = torch.arange(smp.caps[0], device=self.device) < sb.n_nodes[0]
            y = self.labels[sb.nodes[0].long()].long()
            pred = logits[:, :self.model.num_classes].argmax(1)
            correct += ((pred == y) & valid).sum()
            total += valid.sum()
        self.model.train()
        return float(correct.item()) / max(1, int(total.item()))
