"""CPU fp32 GraphSAGE oracle trainer — TEST INFRASTRUCTURE ONLY.

The reference has no trainer, so "accuracy within
0.5 points of the reference" is defined against this oracle: plain PyTorch
fp32 on the CPU, fed by the restated reference sampler (oracle/sampler.py,
pipeline.py:185-222) and the restated reference decoders (oracle/codecs.py),
with the row-stochastic mean aggregation of factors.py:108-114 restricted to
the sampled blocks.  Same model structure as paper_2207_14696_b200.sage.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

from .aggregate import block_mean as np_block_mean
from .aggregate import block_wsum, gcn_weights
from .sampler import sample_batches_oracle


class OracleSage(nn.Module):
    def __init__(self, in_dim, hidden, num_classes, num_layers):
        super().__init__()
        dims = [in_dim] + [hidden] * (num_layers - 1) + [num_classes]
        self.lins = nn.ModuleList(nn.Linear(dims[i], dims[i + 1]) for i in range(num_layers))

    def forward(self, agg_in, blocks):
        """blocks[l] = (counts, local[, weights]) for l < L-1 (local indexes
        layer l+1); with weights the block is the weighted sum (GCN)."""
        L = len(self.lins)
        h = self.lins[0](agg_in)
        for i in range(1, L):
            h = F.relu(h)
            l = L - 1 - i
            counts, local = blocks[l][0], blocks[l][1]
            seg = torch.repeat_interleave(torch.arange(counts.numel()), counts)
            if len(blocks[l]) > 2:
                a = torch.zeros(counts.numel(), h.shape[1]).index_add_(
                    0, seg, h[local] * blocks[l][2][:, None])
            else:
                a = torch.zeros(counts.numel(), h.shape[1]).index_add_(0, seg, h[local])
                a = a / counts.clamp_min(1)[:, None].float()
            h = self.lins[i](a)
        return h


def batch_tensors(batch, decode_rows, aggregator="mean", off=None):
    """Input aggregate (float64 -> fp32) and hidden blocks of one batch;
    aggregator 'gcn' weights every block by gcn_weights (needs row offsets)."""
    L = len(batch.layers)
    last = batch.layers[-1]
    dec = decode_rows(last.picks)
    if aggregator == "gcn":
        w = gcn_weights(off, last.nodes, last.counts, last.picks)
        agg = torch.from_numpy(block_wsum(dec, last.counts, w).astype(np.float32))
    else:
        agg = torch.from_numpy(np_block_mean(dec, last.counts).astype(np.float32))
    blocks = []
    for l in range(L - 1):
        lay = batch.layers[l]
        nxt = batch.layers[l + 1].nodes
        local = np.searchsorted(nxt, lay.picks)
        blk = (torch.from_numpy(lay.counts), torch.from_numpy(local))
        if aggregator == "gcn":
            wl = gcn_weights(off, lay.nodes, lay.counts, lay.picks).astype(np.float32)
            blk = blk + (torch.from_numpy(wl),)
        blocks.append(blk)
    return agg, blocks


def train_epoch(model, opt, off, col, labels, train_ids, fanouts, bs, seed, decode_rows,
                max_batches=None, aggregator="mean"):
    batches, _ = sample_batches_oracle(off, col, train_ids, fanouts, bs, seed,
                                       max_batches=max_batches)
    losses = []
    for b in batches:
        agg, blocks = batch_tensors(b, decode_rows, aggregator, off)
        logits = model(agg, blocks)
        loss = F.cross_entropy(logits, torch.from_numpy(labels[b.seeds]).long())
        opt.zero_grad()
        loss.backward()
        opt.step()
        losses.append(float(loss))
    return losses


@torch.no_grad()
def evaluate(model, off, col, labels, ids, fanouts, bs, seed, decode_rows, max_batches=None,
             aggregator="mean"):
    batches, _ = sample_batches_oracle(off, col, ids, fanouts, bs, seed, max_batches=max_batches)
    correct = total = 0
    for b in batches:
        agg, blocks = batch_tensors(b, decode_rows, aggregator, off)
        pred = model(agg, blocks).argmax(1).numpy()
        correct += int((pred == labels[b.seeds]).sum())
        total += b.seeds.size
    return correct / max(1, total)


# ------------------------------------------------------------------- GAT
class _OracleGatLayer(nn.Module):
    """CPU fp32 restatement of paper_2207_14696_b200.gat.GatLayer (same
    parameter names, so GPU weights load directly)."""

    def __init__(self, in_dim, out_per_head, heads, out_pad=None):
        super().__init__()
        self.heads = heads
        width = out_pad or out_per_head * heads
        self.width = width
        self.lin = nn.Linear(in_dim, width, bias=False)
        self.attn_l = nn.Parameter(torch.zeros(heads, width // heads))
        self.attn_r = nn.Parameter(torch.zeros(heads, width // heads))
        self.bias = nn.Parameter(torch.zeros(width))

    def forward(self, h, counts, local, slope=0.2):
        z = self.lin(h)
        zh = z.view(-1, self.heads, self.width // self.heads)
        el = (zh * self.attn_l).sum(-1)
        er = (zh * self.attn_r).sum(-1)
        nd = counts.numel()
        seg = torch.repeat_interleave(torch.arange(nd), counts)
        cnt = counts.clamp_min(1).float()[:, None]
        q = torch.zeros(nd, self.heads).index_add_(0, seg, er[local]) / cnt
        s = F.leaky_relu(el[local] + q[seg], slope)
        mx = torch.full((nd, self.heads), -float("inf")).index_reduce_(0, seg, s, "amax")
        p = torch.exp(s - mx[seg])
        den = torch.zeros(nd, self.heads).index_add_(0, seg, p)
        alpha = p / den[seg]
        msg = (alpha[:, :, None] * zh[local]).reshape(-1, self.width)
        return torch.zeros(nd, self.width).index_add_(0, seg, msg) + self.bias


class OracleGat(nn.Module):
    def __init__(self, in_dim, hidden, num_classes, num_layers, heads=4):
        super().__init__()
        self.num_classes = num_classes
        c_pad = (num_classes + 7) // 8 * 8
        self.layers = nn.ModuleList(
            _OracleGatLayer(in_dim if i == 0 else hidden, num_classes, 1, c_pad)
            if i == num_layers - 1 else
            _OracleGatLayer(in_dim if i == 0 else hidden, hidden // heads, heads)
            for i in range(num_layers))

    def forward(self, x_picks, blocks):
        """x_picks: decoded rows of the last block's picks; blocks[l] =
        (counts, local) with the last block's local = arange(picks)."""
        L = len(self.layers)
        h = x_picks
        for i, layer in enumerate(self.layers):
            counts, local = blocks[L - 1 - i]
            h = layer(h, counts, local)
            if i < L - 1:
                h = F.elu(h)
        return h[:, :self.num_classes]


def gat_batch_tensors(batch, decode_rows):
    L = len(batch.layers)
    last = batch.layers[-1]
    x = torch.from_numpy(np.asarray(decode_rows(last.picks), np.float32))
    blocks = []
    for l in range(L):
        lay = batch.layers[l]
        if l == L - 1:
            local = np.arange(lay.picks.size)
        else:
            local = np.searchsorted(batch.layers[l + 1].nodes, lay.picks)
        blocks.append((torch.from_numpy(lay.counts), torch.from_numpy(local)))
    return x, blocks


def gat_train_epoch(model, opt, off, col, labels, train_ids, fanouts, bs, seed, decode_rows):
    batches, _ = sample_batches_oracle(off, col, train_ids, fanouts, bs, seed)
    for b in batches:
        x, blocks = gat_batch_tensors(b, decode_rows)
        loss = F.cross_entropy(model(x, blocks), torch.from_numpy(labels[b.seeds]).long())
        opt.zero_grad()
        loss.backward()
        opt.step()


@torch.no_grad()
def gat_evaluate(model, off, col, labels, ids, fanouts, bs, seed, decode_rows):
    batches, _ = sample_batches_oracle(off, col, ids, fanouts, bs, seed)
    correct = total = 0
    for b in batches:
        x, blocks = gat_batch_tensors(b, decode_rows)
        pred = model(x, blocks).argmax(1).numpy()
        correct += int((pred == labels[b.seeds]).sum())
        total += b.seeds.size
    return correct / max(1, total)
