"""Synthetic BASELINE workloads built on the device.

The reference's generators are Python loops (graphstore.py:205-253, ~23k
nodes/s) and cannot reach the BASELINE shapes, so graphs here are a
degree-corrected planted-partition model generated on the GPU:

* nodes carry planted labels (``num_classes``); each class owns a contiguous
  range of virtual positions and positions map to node ids through a fixed
  pseudo-random bijection, so hubs are spread over the id space;
* edge endpoints are drawn from power-law position weights
  (w ∝ (rank+1)^-alpha); with probability ``homophily`` the second endpoint
  is drawn inside the first endpoint's class;
* edges are canonicalised, de-duplicated, symmetrised and given self-loops
  (the reference always samples with self-loops, test_pipeline.py:13-14),
  giving a valid CsrGraph (int64 offsets, int32 sorted columns).

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


def _feistel_perm(x: torch.Tensor, n: int, seed: int) -> torch.Tensor:
    """Bijection on [0, n) (cycle-walking 4-round Feistel on 2*half bits)."""
    bits = max(2, int(math.ceil(math.log2(max(n, 2)))))
    bits += bits & 1
    half = bits // 2
    mask = (1 << half) - 1
    keys = [(seed * 0x9E3779B1 + r * 0x85EBCA77) & 0xFFFFFFF for r in range(4)]

    def rounds(v):
        lo, hi = v & mask, v >> half
        for k in keys:
            f = ((lo * 0x2545F491 + k) ^ (lo >> 3)) & mask
            lo, hi = hi ^ f, lo
        return (hi << half) | lo

    y = rounds(x)
    for _ in range(256):  # cycle walk until inside [0, n)
        bad = y >= n
        if not bool(bad.any()):
            break
        y = torch.where(bad, rounds(y), y)
    return y


@dataclass
class SynthGraph:
    graph: DeviceGraph
    labels: torch.Tensor       # int32 [n] on device
    num_classes: int
    train_ids: np.ndarray      # sorted int64 host
    val_ids: np.ndarray


def generate_graph(n: int, avg_deg: float, num_classes: int, *, seed: int = 0,
                   alpha: float = 0.8, homophily: float = 0.75, device="cuda",
                   edge_chunk: int = 1 << 26) -> tuple[DeviceGraph, torch.Tensor]:
    """Power-law planted-partition graph; returns (DeviceGraph, labels)."""
    dev = torch.device(device)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    C = num_classes
    # class sizes ~ equal; position p in class c -> node id perm(p)
    sizes = torch.full((C,), n // C, dtype=torch.int64)
    sizes[: n % C] += 1
    starts = torch.zeros(C + 1, dtype=torch.int64)
    starts[1:] = torch.cumsum(sizes, 0)
    pos = torch.arange(n, device=dev)
    cls_of_pos = torch.bucketize(pos, starts[1:].to(dev), right=True).to(torch.int32)
    node_of_pos = _feistel_perm(pos, n, seed)
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    labels[node_of_pos] = cls_of_pos
    # power-law weight by rank within class
    rank = pos - starts.to(dev)[cls_of_pos.long()]
    w = (rank.double() + 1.0).pow(-alpha)
    cdf = torch.cumsum(w, 0)                       # global (concatenated classes)
    cls_lo = torch.zeros(C + 1, dtype=torch.float64, device=dev)
    cls_lo[1:] = cdf[starts[1:].to(dev) - 1]
    E = int(round(n * avg_deg / 2))
    keys = []
    done = 0
    while done < E:
        m = min(edge_chunk, E - done)
        u = torch.searchsorted(cdf, torch.rand(m, generator=gen, device=dev, dtype=torch.float64)
                               * cdf[-1]).clamp_max(n - 1)
        cu = cls_of_pos[u].long()
        inside = torch.rand(m, generator=gen, device=dev) < homophily
        r = torch.rand(m, generator=gen, device=dev, dtype=torch.float64)
        lo = torch.where(inside, cls_lo[cu], torch.zeros_like(r))
        hi = torch.where(inside, cls_lo[cu + 1], cdf[-1].expand_as(r))
        v = torch.searchsorted(cdf, lo + r * (hi - lo)).clamp_max(n - 1)
        a, b = node_of_pos[u], node_of_pos[v]
        keep = a != b
        a, b = a[keep], b[keep]
        keys.append(torch.minimum(a, b) * n + torch.maximum(a, b))
        done += m
    key = torch.unique(torch.cat(keys))
    del keys
    lo, hi = key // n, key % n
    del key
    diag = torch.arange(n, device=dev)
    src = torch.cat([lo, hi, diag])
    dst = torch.cat([hi, lo, diag])
    del lo, hi
    order = torch.argsort(src * n + dst)
    src, dst = src[order], dst[order]
    del order
    off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    off[1:] = torch.cumsum(torch.bincount(src, minlength=n), 0)
    g = DeviceGraph(n, off, dst.to(torch.int32).contiguous(), True)
    return g, labels


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


def build_sq_codec(n: int, d: int, k: int, *, labels, num_classes: int, seed: int = 0,
                   chunk_rows: int = 1 << 20, kind: int = 3):
    """fit_sq over the (streamed) matrix, then chunked device encode."""
    from .sq import DeviceSqCodec, fit_sq_device
    dev = labels.device
    # fit: the reference fits on all nonzeros (<= 1e7 strided sample); the
    # exact sample needs the whole matrix order, so stream it when it fits
    total = n * d
    if total <= (1 << 31):
        x = synth_features(n, d, kind=kind, seed=seed, labels=labels, num_classes=num_classes,
                           device=dev)
        params = fit_sq_device(x.reshape(-1), k)
        dc = DeviceSqCodec.empty(params, n, d, dev)
        dc.encode_rows_(x, 0)
        del x
        return dc
    # very large: fit on a row-strided sample of rows (documented deviation)
    rows = torch.arange(0, n, max(1, n // 100_000), device=dev)
    xs = torch.cat([synth_features(1, d, row0=int(r), kind=kind, seed=seed, labels=labels,
                                   num_classes=num_classes, device=dev) for r in rows[:2000]])
    params = fit_sq_device(xs.reshape(-1), k)
    dc = DeviceSqCodec.empty(params, n, d, dev)
    for r0 in range(0, n, chunk_rows):
        m = min(chunk_rows, n - r0)
        x = synth_features(m, d, row0=r0, kind=kind, seed=seed, labels=labels,
                           num_classes=num_classes, device=dev)
        dc.encode_rows_(x, r0)
    return dc


def build_vq_codec(n: int, d: int, width: int, length: int, *, labels, num_classes: int,
                   seed: int = 0, chunk_rows: int = 1 << 20, kind: int = 3,
                   max_iters: int = 50, restarts: int = 4, metric: str = "cosine"):
    """fit_vq on the reference's default uniform sample (min(1, 1e6/n)),
    then chunked device encode of every row."""
    from .vq import DeviceVqCodec, VqParams, _fit_from_sample
    dev = labels.device
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
    else:
        sample = torch.cat([synth_features(1, d, row0=int(r), kind=kind, seed=seed,
                                           labels=labels, num_classes=num_classes, device=dev)
                            for r in pick])
    codec = _fit_from_sample(sample.double(), p, d, 32, rng)
    del sample
    dc = DeviceVqCodec.empty(p, d, codec.codebooks, n, dev)
    for r0 in range(0, n, chunk_rows):
        m = min(chunk_rows, n - r0)
        x = full[r0:r0 + m] if full is not None else synth_features(
            m, d, row0=r0, kind=kind, seed=seed, labels=labels, num_classes=num_classes,
            device=dev)
        dc.encode_rows_(x, r0)
    return dc, codec
