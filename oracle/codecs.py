"""numpy restatement of the reference codecs — TEST INFRASTRUCTURE ONLY.

Restates, operation for operation where floating point is involved:
  * bitpack  : pkg/src/featgrind/bitpack.py:17-83 (MSB-first row-major stream)
  * SQ       : pkg/src/featgrind/sq.py:84-153 (fit / quantize / dequantize)
  * VQ       : pkg/src/featgrind/vq.py:154-344 (k-means fit, assign, decode)

The float64 expression order matters for bit-exactness, so every
floating-point line below keeps the reference's evaluation order; the
integer plumbing (packing, gathering) is written independently.
Pinned against tests/golden/*.npz produced by importing the reference.
"""

from __future__ import annotations

import math

import numpy as np

FIT_SAMPLE_CAP = 10_000_000          # sq.py:35
AUTO_VQ_SAMPLE = 1_000_000           # vq.py:39


# ------------------------------------------------------------------ bitpack

def pack_msb(codes, bits: int) -> bytes:
    """bitpack.py:17-36 — codes flattened row-major, MSB-first, zero tail."""
    flat = np.asarray(codes, dtype=np.int64).reshape(-1)
    if flat.size and (flat.min() < 0 or (flat.max() >> bits)):
        raise ValueError("code overflow")
    bitplanes = [(flat >> (bits - 1 - b)) & 1 for b in range(bits)]
    stream = np.stack(bitplanes, axis=1).astype(np.uint8).reshape(-1) if flat.size \
        else np.zeros(0, np.uint8)
    return np.packbits(stream).tobytes()


def unpack_msb(payload, bits: int, count: int, start_bit: int = 0) -> np.ndarray:
    """bitpack.py:39-55."""
    raw = np.frombuffer(bytes(payload), dtype=np.uint8)
    stream = np.unpackbits(raw)[start_bit:start_bit + count * bits]
    if stream.size != count * bits:
        raise ValueError("short stream")
    weights = np.int64(1) << np.arange(bits - 1, -1, -1, dtype=np.int64)
    return stream.reshape(count, bits).astype(np.int64) @ weights


def row_codes(payload, row_elems: int, bits: int, rows) -> np.ndarray:
    """Codes of selected rows of a continuous row-major stream
    (bitpack.py:58-83 gather, then per-element weights as sq.py:145-146)."""
    rows = np.asarray(rows, dtype=np.int64)
    raw = np.unpackbits(np.frombuffer(bytes(payload), dtype=np.uint8))
    rb = row_elems * bits
    if rows.size and (rows.max() + 1) * rb > raw.size:
        raise ValueError("rows past stream end")
    cols = rows[:, None] * rb + np.arange(rb, dtype=np.int64)[None, :]
    bitmat = raw[cols].reshape(rows.size, row_elems, bits).astype(np.int64)
    weights = np.int64(1) << np.arange(bits - 1, -1, -1, dtype=np.int64)
    return bitmat @ weights


# ----------------------------------------------------------------------- SQ

def sq_fit(values: np.ndarray, k: int, clip: float = 0.005) -> tuple[float, float]:
    """sq.py:84-111: quantiles of log2|x| over nonzeros (strided sample)."""
    flat = np.asarray(values).reshape(-1)
    nz = flat[flat != 0]
    if nz.size == 0:
        if k == 1:
            return 0.0, 0.0
        raise ValueError("all-zero")
    if nz.size > FIT_SAMPLE_CAP:
        nz = nz[np.linspace(0, nz.size - 1, FIT_SAMPLE_CAP).astype(np.int64)]
    logs = np.log2(np.abs(nz.astype(np.float64)))
    lo, hi = np.quantile(logs, [clip, 1.0 - clip])
    return float(lo), float(hi)


def sq_codes(values: np.ndarray, k: int, e_min: float, e_max: float) -> np.ndarray:
    """sq.py:114-128 element codes (int64), same float64 op order."""
    x = np.asarray(values).astype(np.float64, copy=False)
    if k == 1:
        return (x >= 0).astype(np.int64)
    mag = np.abs(x)
    lg = np.log2(np.where(mag == 0, 1.0, mag))
    lg = np.where(mag == 0, e_min, lg)
    lg = np.clip(lg, e_min, e_max)
    half = 1 << (k - 1)
    off = np.floor((lg - e_min) / (e_max - e_min) * half).astype(np.int64)
    off = np.clip(off, 0, half - 1)
    return np.where(x >= 0, half + off, half - 1 - off)


def sq_decode_codes(q: np.ndarray, k: int, e_min: float, e_max: float,
                    elem_bits: int = 32) -> np.ndarray:
    """sq.py:144-153 bucket midpoints from integer codes."""
    q = np.asarray(q, dtype=np.int64)
    half = 1 << (k - 1)
    pos = q >= half
    steps = np.where(pos, q - half + 0.5, half - 0.5 - q)
    mags = np.exp2(steps * ((e_max - e_min) / half) + e_min)
    out = np.where(pos, mags, -mags)
    return out.astype(np.float32 if elem_bits == 32 else np.float64)


def sq_lut(k: int, e_min: float, e_max: float, elem_bits: int = 32) -> np.ndarray:
    return sq_decode_codes(np.arange(1 << k), k, e_min, e_max, elem_bits)


def sq_dequant_rows(payload, n: int, d: int, k: int, e_min: float, e_max: float,
                    rows=None, elem_bits: int = 32) -> np.ndarray:
    rows = np.arange(n) if rows is None else np.asarray(rows, dtype=np.int64)
    if rows.size and (rows.min() < 0 or rows.max() >= n):
        raise IndexError("row id out of range")
    q = row_codes(payload, d, k, rows)
    return sq_decode_codes(q, k, e_min, e_max, elem_bits).reshape(rows.size, d)


# ----------------------------------------------------------------------- VQ

def part_bounds(d: int, width: int) -> list[tuple[int, int]]:
    return [(lo, min(lo + width, d)) for lo in range(0, d, width)]


def sqdist(x: np.ndarray, c: np.ndarray) -> np.ndarray:
    """vq.py:154-156 (keep the exact expression order)."""
    d2 = (x * x).sum(axis=1)[:, None] + (c * c).sum(axis=1)[None, :] - 2.0 * (x @ c.T)
    return np.maximum(d2, 0.0)


def vq_assign_part(pts64: np.ndarray, book: np.ndarray, metric: str) -> np.ndarray:
    """vq.py:306-316 nearest entry, ties -> lowest index."""
    cb = book.astype(np.float64)
    if metric == "cosine":
        nrm = np.linalg.norm(pts64, axis=1)
        sims = (pts64 / np.where(nrm > 0, nrm, 1.0)[:, None]) @ cb.T
        out = np.argmax(sims, axis=1)
        out[nrm == 0] = 0
        return out.astype(np.int32)
    return np.argmin(sqdist(pts64, cb), axis=1).astype(np.int32)


def vq_assign(values: np.ndarray, books, width: int, metric: str) -> np.ndarray:
    """vq.py:319-327."""
    x = np.asarray(values).astype(np.float64, copy=False)
    bounds = part_bounds(x.shape[1], width)
    codes = np.empty((x.shape[0], len(bounds)), np.int32)
    for p, (lo, hi) in enumerate(bounds):
        codes[:, p] = vq_assign_part(x[:, lo:hi], books[p], metric)
    return codes


def vq_decode(codes: np.ndarray, books, d: int, width: int, rows=None) -> np.ndarray:
    """vq.py:330-344 exact float32 copies."""
    sel = codes if rows is None else codes[np.asarray(rows, dtype=np.int64)]
    out = np.empty((sel.shape[0], d), np.float32)
    for p, (lo, hi) in enumerate(part_bounds(d, width)):
        out[:, lo:hi] = books[p][sel[:, p]]
    return out


def _bincount_sums(pts, assign, k):
    """vq.py:159-164."""
    counts = np.bincount(assign, minlength=k).astype(np.float64)
    sums = np.empty((k, pts.shape[1]))
    for j in range(pts.shape[1]):
        sums[:, j] = np.bincount(assign, weights=pts[:, j], minlength=k)
    return sums, counts


def _seed_centroids(pts, k, rng):
    """vq.py:166-181 k-means++ D^2 seeding."""
    cents = np.empty((k, pts.shape[1]))
    cents[0] = pts[int(rng.integers(pts.shape[0]))]
    d2 = sqdist(pts, cents[:1]).ravel()
    for c in range(1, k):
        tot = d2.sum()
        if tot <= 0:
            cents[c:] = pts[int(rng.integers(pts.shape[0]))]
            return cents
        pick = int(np.searchsorted(np.cumsum(d2), rng.random() * tot))
        cents[c] = pts[min(pick, pts.shape[0] - 1)]
        d2 = np.minimum(d2, sqdist(pts, cents[c:c + 1]).ravel())
    return cents


def lloyd(pts, k, metric, max_iters, tol, rng):
    """vq.py:184-228; returns (centroids, objective, history)."""
    cents = _seed_centroids(pts, k, rng)
    hist: list[float] = []
    prev = math.inf
    obj = math.inf
    for _ in range(max_iters):
        if metric == "cosine":
            sims = pts @ cents.T
            a = np.argmax(sims, axis=1)
            cost = 1.0 - sims[np.arange(pts.shape[0]), a]
        else:
            d2 = sqdist(pts, cents)
            a = np.argmin(d2, axis=1)
            cost = d2[np.arange(pts.shape[0]), a]
        obj = float(cost.sum())
        hist.append(obj)
        sums, counts = _bincount_sums(pts, a, k)
        live = counts > 0
        nxt = cents.copy()
        if metric == "cosine":
            nr = np.linalg.norm(sums, axis=1)
            ok = live & (nr > 0)
            nxt[ok] = sums[ok] / nr[ok, None]
        else:
            nxt[live] = sums[live] / counts[live, None]
        far = cost.copy()
        for c in np.flatnonzero(~live):
            i = int(np.argmax(far))
            nxt[c] = pts[i]
            far[i] = -math.inf
        cents = nxt
        if prev - obj <= tol * max(abs(prev), 1e-12):
            break
        prev = obj
    if metric == "cosine":
        final = float((1.0 - (pts @ cents.T).max(axis=1)).sum())
    else:
        final = float(sqdist(pts, cents).min(axis=1).sum())
    hist.append(final)
    return cents, final, hist


def fit_part(pts, metric, capacity, seeds, restarts, max_iters, tol):
    """vq.py:231-254."""
    uniq = np.unique(pts, axis=0)
    if uniq.shape[0] <= capacity:
        return uniq.astype(np.float32), 0.0
    best = None
    for r in range(restarts):
        cand = lloyd(pts, capacity, metric, max_iters, tol,
                     np.random.default_rng(int(seeds[r])))
        if best is None or cand[1] < best[1]:
            best = cand
    cents, obj, _ = best
    if metric == "cosine":
        nr = np.linalg.norm(cents, axis=1)
        cents = cents / np.where(nr > 0, nr, 1.0)[:, None]
    return cents.astype(np.float32), obj


def vq_fit(values, width, length, metric="cosine", fit_sample_fraction=None,
           max_iters=50, tol=1e-4, restarts=4, seed=0):
    """vq.py:257-303; returns (codebooks list, per-part objectives)."""
    x = np.asarray(values)
    n, d = x.shape
    frac = fit_sample_fraction if fit_sample_fraction is not None \
        else min(1.0, AUTO_VQ_SAMPLE / n)
    rows = min(max(math.ceil(frac * n - 1e-9), 1), n)
    rng = np.random.default_rng(seed)
    sample = x[np.sort(rng.choice(n, size=rows, replace=False))] if rows < n else x
    sample = sample.astype(np.float64, copy=False)
    books, objs = [], []
    for lo, hi in part_bounds(d, width):
        pts = sample[:, lo:hi]
        zero_slot = False
        if metric == "cosine":
            nr = np.linalg.norm(pts, axis=1)
            keep = nr > 0
            zero_slot = not keep.all()
            pts = pts[keep] / nr[keep][:, None]
            if pts.shape[0] == 0:
                books.append(np.zeros((1, hi - lo), np.float32))
                objs.append(0.0)
                continue
        seeds = rng.integers(0, 2 ** 63 - 1, size=restarts)
        cb, obj = fit_part(pts, metric, length - 1 if zero_slot else length,
                           seeds, restarts, max_iters, tol)
        if zero_slot:
            cb = np.concatenate([np.zeros((1, cb.shape[1]), np.float32), cb])
        books.append(cb)
        objs.append(obj)
    return books, objs
