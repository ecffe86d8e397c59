"""Mean-aggregation oracle — TEST INFRASTRUCTURE ONLY.

The reference defines aggregation only as the row-stochastic operator
M = D̂⁻¹Â over stored neighbours (pkg/src/featgrind/factors.py:108-114;
PAPER.md:672-687).  Restricted to a sampled block, destination v averages
the decoded input rows of its picks.  This oracle decodes those rows with
the restated reference decoders (oracle/codecs.py) and accumulates in
float64; destinations with no picks produce zeros.
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
