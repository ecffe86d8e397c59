"""Mean-aggregation oracle — TEST INFRASTRUCTURE ONLY.

The reference defines aggregation only as the row-stochastic operator
M = D̂⁻¹Â over stored neighbours (pkg/src/featgrind/factors.py:108-114;
PAPER.md:672-687).  Restricted to a sampled block, destination v averages
the decoded input rows of its picks.  This oracle decodes those rows with
the restated reference decoders (oracle/codecs.py) and accumulates in
float64; destinations with no picks produce zeros.

GCN variant (BASELINE config E; no reference counterpart): Kipf's symmetric
D^-1/2 A D^-1/2 with full-graph degrees (self-loops included), estimated
from the cnt_v sampled neighbours: w_vu = sqrt(deg v) / (cnt_v sqrt(deg u)).
"""

from __future__ import annotations

import numpy as np


def block_mean(decoded_rows: np.ndarray, counts: np.ndarray) -> np.ndarray:
    """decoded_rows: (E, d) rows in pick order; counts: picks per dst."""
    counts = np.asarray(counts, dtype=np.int64)
    x = np.asarray(decoded_rows, dtype=np.float64)
    out = np.zeros((counts.size, x.shape[1]), np.float64)
    if x.shape[0] == 0:
        return out
    seg = np.repeat(np.arange(counts.size), counts)
    np.add.at(out, seg, x)
    nz = counts > 0
    out[nz] /= counts[nz, None]
    return out


def mean_tolerance_ok(got: np.ndarray, ref: np.ndarray, decoded_rows: np.ndarray,
                      counts: np.ndarray, rel: float) -> tuple[bool, float]:
    """|got - ref| <= rel * mean_u |x_u| + 1e-30, per destination and element
    (a plain relative error breaks near zero)."""
    scale = block_mean(np.abs(decoded_rows), counts)
    err = np.abs(np.asarray(got, np.float64) - ref)
    bound = rel * scale + 1e-30
    worst = float(np.max(err / bound)) if err.size else 0.0
    return bool((err <= bound).all()), worst


def gcn_weights(row_offsets: np.ndarray, dst_nodes: np.ndarray, counts: np.ndarray,
                src_nodes: np.ndarray) -> np.ndarray:
    """Per-pick weights (pick order) of the sampled GCN aggregation, float64."""
    off = np.asarray(row_offsets, np.int64)
    deg = (off[1:] - off[:-1]).astype(np.float64)
    counts = np.asarray(counts, np.int64)
    dst = np.repeat(np.asarray(dst_nodes, np.int64), counts)
    cnt = np.repeat(counts, counts).astype(np.float64)
    return np.sqrt(deg[dst]) / (cnt * np.sqrt(deg[np.asarray(src_nodes, np.int64)]))


def block_wsum(decoded_rows: np.ndarray, counts: np.ndarray, w: np.ndarray) -> np.ndarray:
    """out[v] = sum over v's picks of w_e x_e (float64)."""
    counts = np.asarray(counts, dtype=np.int64)
    x = np.asarray(decoded_rows, dtype=np.float64) * np.asarray(w, np.float64)[:, None]
    out = np.zeros((counts.size, x.shape[1]), np.float64)
    if x.shape[0]:
        np.add.at(out, np.repeat(np.arange(counts.size), counts), x)
    return out


def wsum_tolerance_ok(got, ref, decoded_rows, counts, w, rel):
    """|got - ref| <= rel * sum_e |w_e x_e| + 1e-30 (the weighted analogue of
    mean_tolerance_ok)."""
    scale = block_wsum(np.abs(decoded_rows), counts, np.abs(w))
    err = np.abs(np.asarray(got, np.float64) - ref)
    bound = rel * scale + 1e-30
    worst = float(np.max(err / bound)) if err.size else 0.0
    return bool((err <= bound).all()), worst
