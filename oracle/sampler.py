"""Restatement of ``sample_batches`` that also records blocks — TEST INFRA ONLY.

Follows pkg/src/featgrind/pipeline.py:185-222 call-for-call on the same numpy
``Generator`` (``default_rng(seed)`` → ``permutation`` → per batch, per layer,
per node in ascending id: ``choice(nbrs, f, replace=False)`` when
``deg > f``), so its seeds / frontier / edges_touched equal the reference's
(pinned in tests/test_oracle.py::test_sampler_oracle_matches_reference against tests/golden/sampler_golden.npz).
In addition it keeps what the reference discards: for every
layer the expanded node list, the per-node pick counts and the picks in
``choice`` output order — the "sampled blocks" the GPU sampler must match.

``engine="pcg"`` drives the same algorithm from oracle/pcg64.py instead of
numpy, which is how the draw-level restatement itself is pinned.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .pcg64 import Pcg64Stream


@dataclass
class OracleLayer:
    nodes: np.ndarray      # int64, sorted unique: the nodes expanded here
    counts: np.ndarray     # int64 per node: min(f, deg)
    picks: np.ndarray      # int64, concatenated picks in node order
    fanout: int


@dataclass
class OracleBatch:
    seeds: np.ndarray
    frontier: np.ndarray
    edges_touched: int
    layers: list[OracleLayer] = field(default_factory=list)
    rng_state_after: dict | None = None


def _choice_numpy(rng, nbrs, f):
    return rng.choice(nbrs, size=f, replace=False)


def _choice_pcg(stream: Pcg64Stream, nbrs, f):
    idx = stream.choice_noreplace(int(nbrs.size), f)
    return nbrs[np.asarray(idx, dtype=np.int64)]


def sample_batches_oracle(row_offsets, col_indices, train_ids, fanouts,
                          batch_size, seed=0, engine="numpy",
                          max_batches=None, rng_state=None):
    """Returns (list[OracleBatch], final numpy-style rng state dict)."""
    off = np.asarray(row_offsets, dtype=np.int64)
    col = np.asarray(col_indices)
    n = off.size - 1
    ids = np.unique(np.asarray(train_ids, dtype=np.int64))
    if ids.size == 0:
        raise ValueError("train_ids must be non-empty")
    if ids.min() < 0 or ids.max() >= n:
        raise ValueError("train id out of range")
    rng = np.random.default_rng(seed)
    if rng_state is not None:
        rng.bit_generator.state = rng_state
    if engine == "numpy":
        perm = rng.permutation(ids)
        draw, src = _choice_numpy, rng
    else:
        stream = Pcg64Stream.from_numpy(rng.bit_generator.state)
        perm = np.asarray(stream.permute(ids), dtype=np.int64)
        draw, src = _choice_pcg, stream
    out: list[OracleBatch] = []
    for lo in range(0, perm.size, batch_size):
        if max_batches is not None and len(out) >= max_batches:
            break
        seeds = np.sort(perm[lo:lo + batch_size])
        cur = seeds
        every = [seeds]
        edges = 0
        layers: list[OracleLayer] = []
        for f in fanouts:
            parts, counts = [], np.zeros(cur.size, np.int64)
            for i, u in enumerate(cur):
                nb = col[off[u]:off[u + 1]]
                if nb.size <= f:
                    parts.append(nb.astype(np.int64))
                    counts[i] = nb.size
                else:
                    parts.append(np.asarray(draw(src, nb, f), dtype=np.int64))
                    counts[i] = f
            picks = np.concatenate(parts) if parts else np.zeros(0, np.int64)
            edges += int(counts.sum())
            layers.append(OracleLayer(cur, counts, picks, int(f)))
            cur = np.unique(picks).astype(np.int64) if parts else np.zeros(0, np.int64)
            every.append(cur)
        b = OracleBatch(seeds, np.unique(np.concatenate(every)), edges, layers)
        b.rng_state_after = (rng.bit_generator.state if engine == "numpy"
                             else src.as_numpy_state())
        out.append(b)
    final = rng.bit_generator.state if engine == "numpy" else src.as_numpy_state()
    return out, final


class HostRows:
    """Row source over host CSR arrays (the protocol of
    ``sample_batches_oracle_rows``): ``rows(ids) -> (start, deg)`` and
    ``take(pos) -> cols`` for absolute int64 positions into col_indices."""

    def __init__(self, row_offsets, col_indices):
        self.off = np.asarray(row_offsets, dtype=np.int64)
        self.col = np.asarray(col_indices)
        self.n = self.off.size - 1

    def rows(self, ids):
        ids = np.asarray(ids, dtype=np.int64)
        return self.off[ids], self.off[ids + 1] - self.off[ids]

    def take(self, pos):
        return self.col[np.asarray(pos, dtype=np.int64)].astype(np.int64)


def sample_batches_oracle_rows(src, n, train_ids, fanouts, batch_size, seed=0,
                               max_batches=None):
    """``sample_batches_oracle`` over a row source that serves CSR rows on
    demand (``HostRows`` or a device-backed one in the tests), so graphs too
    large to copy to the host (papers100M / MAG240M shape: 13-27 GB of
    columns) can still be checked batch by batch.

    Same draws as pipeline.py:205-214: ``rng.choice(nbrs, f, replace=False)``
    is ``nbrs[rng.choice(len(nbrs), f, replace=False)]`` in numpy (the array
    form indexes the integer form's output: identical draws and stream
    state, tests/test_oracle.py::test_row_source_oracle_equals_array_oracle),
    so only the degrees and the picked positions are fetched per layer."""
    ids = np.unique(np.asarray(train_ids, dtype=np.int64))
    if ids.size == 0:
        raise ValueError("train_ids must be non-empty")
    if ids.min() < 0 or ids.max() >= n:
        raise ValueError("train id out of range")
    rng = np.random.default_rng(seed)
    perm = rng.permutation(ids)
    out: list[OracleBatch] = []
    for lo in range(0, perm.size, batch_size):
        if max_batches is not None and len(out) >= max_batches:
            break
        seeds = np.sort(perm[lo:lo + batch_size])
        cur = seeds
        every = [seeds]
        edges = 0
        layers: list[OracleLayer] = []
        for f in fanouts:
            start, deg = src.rows(cur)
            counts = np.minimum(deg, f).astype(np.int64)
            pos = np.empty(int(counts.sum()), np.int64)
            o = 0
            for i in range(cur.size):
                dg, s0 = int(deg[i]), int(start[i])
                if dg <= f:
                    pos[o:o + dg] = np.arange(s0, s0 + dg)
                    o += dg
                else:
                    pos[o:o + f] = s0 + rng.choice(dg, size=f, replace=False)
                    o += f
            picks = src.take(pos) if pos.size else np.zeros(0, np.int64)
            edges += int(counts.sum())
            layers.append(OracleLayer(cur, counts, picks, int(f)))
            cur = np.unique(picks).astype(np.int64)
            every.append(cur)
        b = OracleBatch(seeds, np.unique(np.concatenate(every)), edges, layers)
        b.rng_state_after = rng.bit_generator.state
        out.append(b)
    return out, rng.bit_generator.state


def state_after_permutation(train_ids, seed=0):
    """PCG64 state right after ``permutation`` (start of batch 0) and perm."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(np.unique(np.asarray(train_ids, dtype=np.int64)))
    return perm, rng.bit_generator.state
