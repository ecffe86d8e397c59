"""Synthetic BASELINE workloads built on the device.

The reference's generators are Python loops (graphstore.py:205-253, ~23k
nodes/s) and cannot reach the BASELINE shapes, so graphs here are a
degree-corrected planted-partition model generated on the GPU:

* nodes carry planted labels (``num_classes``); each class owns a contiguous
  range of virtual positions and positions map to node ids through a fixed
  Feistel bijection, so hubs are spread over the id space;
* edge e is a pure function of (seed, e) (counter-based hash): endpoint
  ranks follow a power law (w ∝ (rank+1)^-alpha) inside a class; with
  probability ``homophily`` the second endpoint stays in the first's class;
* the CSR is built in node-range chunks that each regenerate the edge stream
  (fg_graph_degrees / fg_graph_emit kernels), de-duplicated, symmetric, with
  self-loops (the reference always samples with self-loops,
  test_pipeline.py:13-14): int64 offsets, int32 sorted columns.

Features are row-addressable (``fg_synth_features``): class-conditional
Gaussians, so the trainer has signal; codecs are built by streaming row
chunks through the device encoders, so the raw matrix never needs to exist
whole (MAG240M-shape is 750 GB in fp32).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .graph import DeviceGraph

# BASELINE.json configs (node counts: PAPER.md:219-221 / OGB; split sizes are
# the OGB train splits, external to the reference — SURVEY.md §6)
SHAPES = {
    "arxiv": dict(n=169_343, d=128, avg_deg=13.7, classes=40, train=90_941),
    "products": dict(n=2_449_029, d=100, avg_deg=50.5, classes=47, train=196_615),
    "papers100m": dict(n=111_059_956, d=128, avg_deg=29.1, classes=172, train=1_207_179),
    "mag240m": dict(n=244_160_499, d=768, avg_deg=27.9, classes=153, train=1_112_392),
}


@dataclass
class SynthGraph:
    graph: DeviceGraph
    labels: torch.Tensor       # int32 [n] on device
    num_classes: int
    train_ids: np.ndarray      # sorted int64 host
    val_ids: np.ndarray


def generate_graph(n: int, avg_deg: float, num_classes: int, *, seed: int = 0,
                   alpha: float = 0.8, homophily: float = 0.75, device="cuda",
                   chunk_entries: int = 1 << 28) -> tuple[DeviceGraph, torch.Tensor]:
    """Power-law planted-partition graph built on the device in node-range
    chunks (fg_graph_degrees / fg_graph_emit): valid CSR with sorted,
    duplicate-free rows, symmetric adjacency and all self-loops.  Memory is
    O(nnz) for the result plus O(chunk_entries) scratch, so MAG240M-shape
    graphs (~7e9 stored entries) build on one B200."""
    dev = torch.device(device)
    E = int(round(n * avg_deg / 2))
    s = N.stream_handle(dev)
    deg = torch.zeros(n, dtype=torch.int32, device=dev)
    N.call("fg_graph_degrees", seed, n, num_classes, alpha, homophily, E, N.ptr(deg), s)
    raw = deg.long() + 1                      # + self loop
    cum = torch.cumsum(raw, 0)
    total_raw = int(cum[-1].item())
    # chunk boundaries: node ranges whose raw entry count fits the budget
    bounds = [0]
    while bounds[-1] < n:
        lo = bounds[-1]
        base = int(cum[lo - 1].item()) if lo > 0 else 0
        hi = int(torch.searchsorted(cum, torch.tensor(base + chunk_entries, device=dev),
                                    right=True).item())
        bounds.append(max(hi, lo + 1) if hi < n else n)
    del cum
    col = torch.empty(total_raw, dtype=torch.int32, device=dev)
    counts = torch.zeros(n, dtype=torch.int64, device=dev)
    cursor = torch.zeros(1, dtype=torch.int64, device=dev)
    pos = 0
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        cap = int(deg[lo:hi].sum().item())
        keys = torch.empty(cap + (hi - lo), dtype=torch.int64, device=dev)
        cursor.zero_()
        N.call("fg_graph_emit", seed, n, num_classes, alpha, homophily, E, lo, hi,
               N.ptr(cursor), cap, N.ptr(keys), s)
        m = int(cursor.item())
        assert m == cap, (m, cap)
        loc = torch.arange(hi - lo, device=dev, dtype=torch.int64)
        keys[m:] = loc * n + (loc + lo)        # self loops
        keys = torch.unique(keys)              # sorted: by local source, then target
        counts[lo:hi] = torch.bincount(keys // n, minlength=hi - lo)
        col[pos:pos + keys.numel()] = (keys % n).to(torch.int32)
        pos += keys.numel()
        del keys
    col = col[:pos].clone()
    off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    off[1:] = torch.cumsum(counts, 0)
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    N.call("fg_graph_labels", seed, n, num_classes, N.ptr(labels), s)
    return DeviceGraph(n, off, col, True), labels


def split_ids(n: int, train: int, val: int, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    r = np.random.default_rng(seed + 1)
    perm = r.permutation(n)
    return np.sort(perm[:train]), np.sort(perm[train:train + val])


def make_shape(name: str, *, seed: int = 0, scale: float = 1.0, device="cuda") -> SynthGraph:
    s = SHAPES[name]
    n = max(1000, int(s["n"] * scale))
    g, labels = generate_graph(n, s["avg_deg"], s["classes"], seed=seed, device=device)
    tr = max(1, int(s["train"] * scale))
    va = max(1, min(n - tr, tr // 5))
    train, val = split_ids(n, tr, va, seed)
    return SynthGraph(g, labels, s["classes"], train, val)


def synth_features(rows: int, d: int, *, row0: int = 0, kind: int = 3, seed: int = 0,
                   labels: torch.Tensor | None = None, num_classes: int = 1,
                   device="cuda") -> torch.Tensor:
    out = torch.empty((rows, d), dtype=torch.float32, device=device)
    N.call("fg_synth_features", kind, seed, row0, rows, d, N.ptr(labels), num_classes,
           N.ptr(out), N.stream_handle())
    return out


def synth_feature_rows(ids, d: int, *, kind: int = 3, seed: int = 0,
                       labels: torch.Tensor | None = None, num_classes: int = 1) -> torch.Tensor:
    """Rows ``ids`` (int64 device tensor) of the same row-addressable matrix."""
    ids = ids.to(torch.int64).contiguous()
    out = torch.empty((ids.numel(), d), dtype=torch.float32, device=ids.device)
    N.call("fg_synth_feature_rows", kind, seed, N.ptr(ids), ids.numel(), d, N.ptr(labels),
           num_classes, N.ptr(out), N.stream_handle())
    return out


def build_sq_codec(n: int, d: int, k: int, *, labels, num_classes: int, seed: int = 0,
                   chunk_rows: int = 1 << 20, kind: int = 3, group=None):
    """fit_sq over the row-addressable matrix (streamed: the exact reference
    fit, sq.py:84-111, never needs the whole matrix), then chunked encode.
    With a process group each rank encodes its own row block and one
    all-gather assembles the replica (ddp.allgather_rows_)."""
    from . import ddp
    from .sq import DeviceSqCodec, fit_sq_stream, sq_row_stride
    dev = labels.device

    def chunks():
        for r0 in range(0, n, chunk_rows):
            m = min(chunk_rows, n - r0)
            yield synth_features(m, d, row0=r0, kind=kind, seed=seed, labels=labels,
                                 num_classes=num_classes, device=dev)

    params = fit_sq_stream(chunks, k, device=dev)
    rank, world = ddp.world_of(group)
    if world == 1:
        dc = DeviceSqCodec.empty(params, n, d, dev)
        r0 = 0
        for x in chunks():
            dc.encode_rows_(x, r0)
            r0 += x.shape[0]
        return dc
    buf = ddp.padded_rows(n, sq_row_stride(d, k), world, dev)
    dc = DeviceSqCodec(params, n, d, buf[:n])
    b0, b1, _ = ddp.row_block(n, rank, world)
    for r0 in range(b0, b1, chunk_rows):
        m = min(chunk_rows, b1 - r0)
        dc.encode_rows_(synth_features(m, d, row0=r0, kind=kind, seed=seed, labels=labels,
                                       num_classes=num_classes, device=dev), r0)
    ddp.allgather_rows_(buf, n, group)
    return dc


def build_vq_codec(n: int, d: int, width: int, length: int, *, labels, num_classes: int,
                   seed: int = 0, chunk_rows: int = 1 << 20, kind: int = 3,
                   max_iters: int = 50, restarts: int = 4, metric: str = "cosine",
                   group=None):
    """fit_vq on the reference's default uniform sample (min(1, 1e6/n)),
    then chunked device encode of every row.  With a process group, parts are
    fitted round-robin across ranks and rows encoded per rank block, then
    all-gathered."""
    from . import ddp
    from .vq import DeviceVqCodec, VqParams, _fit_from_sample, vq_row_stride
    dev = labels.device
    rank, world = ddp.world_of(group)
    p = VqParams(width, length, metric=metric, kmeans_max_iters=max_iters, restarts=restarts,
                 seed=seed)
    frac = min(1.0, 1_000_000 / n)
    rows = min(max(math.ceil(frac * n - 1e-9), 1), n)
    rng = np.random.default_rng(p.seed)
    pick = np.sort(rng.choice(n, size=rows, replace=False)) if rows < n else np.arange(n)
    full = synth_features(n, d, kind=kind, seed=seed, labels=labels, num_classes=num_classes,
                          device=dev) if n * d <= (1 << 31) else None
    if full is not None:
        sample = full[torch.from_numpy(pick).to(dev)]
    else:  # only the fit sample rows are ever generated
        sample = synth_feature_rows(torch.from_numpy(pick).to(dev), d, kind=kind, seed=seed,
                                    labels=labels, num_classes=num_classes)
    import sys
    import time
    t0 = time.perf_counter()
    codec = _fit_from_sample(sample.double(), p, d, 32, rng, group=group)
    del sample
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if world == 1:
        dc = DeviceVqCodec.empty(p, d, codec.codebooks, n, dev)
        b0, b1, buf = 0, n, None
    else:
        buf = ddp.padded_rows(n, vq_row_stride(len(codec.codebooks), p.bits_per_code), world,
                              dev)
        dc = DeviceVqCodec(p, d, codec.codebooks, n, buf[:n], dev)
        b0, b1, _ = ddp.row_block(n, rank, world)
    for r0 in range(b0, b1, chunk_rows):
        m = min(chunk_rows, b1 - r0)
        x = full[r0:r0 + m] if full is not None else synth_features(
            m, d, row0=r0, kind=kind, seed=seed, labels=labels, num_classes=num_classes,
            device=dev)
        dc.encode_rows_(x, r0)
    if buf is not None:
        ddp.allgather_rows_(buf, n, group)
    torch.cuda.synchronize()
    print(f"[synth] vq codec: fit_vq on {rows} sample rows {t1 - t0:.1f} s, encode {n} rows "
          f"{time.perf_counter() - t1:.1f} s", file=sys.stderr, flush=True)
    return dc, codec
