"""Graph and feature containers (drop-in for pkg/src/featgrind/graphstore.py).

``FeatureMatrix`` and ``CsrGraph`` keep the reference's field names and
invariants (graphstore.py:46-163): dense finite float32/float64 rows; CSR with
int64 ``row_offsets``, int32 ``col_indices``, sorted duplicate-free rows, a
symmetric adjacency and all-or-none self-loops.  ``DeviceGraph`` is the
HBM-resident replica the sampler reads (same two arrays, on the GPU).

Host validation is O(nnz log nnz), like the reference's; graphs built by the
synthetic generator are valid by construction and skip it
(``CsrGraph.trusted``), which is what makes 10^9-edge graphs loadable.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import DataError


@dataclass(frozen=True)
class FeatureMatrix:
    """Dense (n, d) float32/float64 matrix with finite values."""

    values: np.ndarray

    def __post_init__(self) -> None:
        v = self.values
        if not isinstance(v, np.ndarray) or v.ndim != 2:
            raise DataError("features must be a 2-d numpy array")
        if v.dtype not in (np.float32, np.float64):
            raise DataError(f"features must be float32 or float64, got {v.dtype}")
        finite = np.isfinite(v)
        if not finite.all():
            i, j = np.argwhere(~finite)[0]
            raise DataError(f"non-finite feature value at ({i}, {j})")
        object.__setattr__(self, "values", np.ascontiguousarray(v))

    @property
    def n(self) -> int:
        return self.values.shape[0]

    @property
    def d(self) -> int:
        return self.values.shape[1]

    @property
    def elem_bits(self) -> int:
        return 64 if self.values.dtype == np.float64 else 32

    def nbytes(self) -> int:
        return self.n * self.d * self.elem_bits // 8


def _validate_csr(n: int, off: np.ndarray, col: np.ndarray) -> bool:
    """Checks graphstore.py:94-126's invariants; returns has_self_loops."""
    if off.shape != (n + 1,) or off[0] != 0 or off[-1] != col.size:
        raise DataError("row_offsets must be (n+1,) spanning col_indices")
    deg = np.diff(off)
    if (deg < 0).any():
        raise DataError("row_offsets must be non-decreasing")
    if col.size and (col.min() < 0 or col.max() >= n):
        raise DataError("column index out of range")
    row = np.repeat(np.arange(n, dtype=np.int64), deg)
    key = row * n + col.astype(np.int64)
    if col.size > 1 and not (np.diff(key) > 0).all():
        # keys strictly increase iff every row is sorted and duplicate free
        raise DataError("neighbor lists must be sorted and duplicate-free")
    tkey = np.sort(col.astype(np.int64) * n + row)
    if not np.array_equal(tkey, key):
        raise DataError("adjacency must be symmetric")
    loops = int((row == col).sum())
    if loops not in (0, n):
        raise DataError("self-loops must be present on all nodes or none")
    return loops == n


@dataclass(frozen=True)
class CsrGraph:
    """Undirected graph in CSR form (graphstore.py:80-163)."""

    n: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    has_self_loops: bool = field(init=False)

    def __post_init__(self) -> None:
        if self.n < 1:
            raise DataError("graph must have at least one node")
        off = np.ascontiguousarray(self.row_offsets, dtype=np.int64)
        col = np.ascontiguousarray(self.col_indices, dtype=np.int32)
        object.__setattr__(self, "row_offsets", off)
        object.__setattr__(self, "col_indices", col)
        object.__setattr__(self, "has_self_loops", _validate_csr(self.n, off, col))

    @classmethod
    def trusted(cls, n: int, row_offsets: np.ndarray, col_indices: np.ndarray,
                has_self_loops: bool) -> "CsrGraph":
        """Wrap arrays known to satisfy the invariants (no O(nnz) checks)."""
        g = object.__new__(cls)
        object.__setattr__(g, "n", int(n))
        object.__setattr__(g, "row_offsets", np.ascontiguousarray(row_offsets, dtype=np.int64))
        object.__setattr__(g, "col_indices", np.ascontiguousarray(col_indices, dtype=np.int32))
        object.__setattr__(g, "has_self_loops", bool(has_self_loops))
        return g

    @property
    def nnz(self) -> int:
        return int(self.col_indices.size)

    def degrees(self, include_self: bool = False) -> np.ndarray:
        deg = np.diff(self.row_offsets)
        if self.has_self_loops and not include_self:
            deg = deg - 1
        return deg.astype(np.int64)

    def num_undirected_edges(self) -> int:
        return (self.nnz - (self.n if self.has_self_loops else 0)) // 2

    def neighbors(self, i: int) -> np.ndarray:
        return self.col_indices[self.row_offsets[i]:self.row_offsets[i + 1]]

    def equals(self, other: "CsrGraph") -> bool:
        return (self.n == other.n and np.array_equal(self.row_offsets, other.row_offsets)
                and np.array_equal(self.col_indices, other.col_indices))

    def to_device(self, device=None) -> "DeviceGraph":
        import torch
        dev = torch.device(device or "cuda")
        return DeviceGraph(self.n, torch.from_numpy(self.row_offsets).to(dev),
                           torch.from_numpy(self.col_indices).to(dev), self.has_self_loops)


@dataclass
class DeviceGraph:
    """HBM-resident CSR replica: int64 offsets (n+1), int32 columns (nnz)."""

    n: int
    row_offsets: "object"   # torch.int64 cuda tensor
    col_indices: "object"   # torch.int32 cuda tensor
    has_self_loops: bool = True

    @property
    def nnz(self) -> int:
        return int(self.col_indices.numel())

    def to_host(self) -> CsrGraph:
        return CsrGraph.trusted(self.n, self.row_offsets.cpu().numpy(),
                                self.col_indices.cpu().numpy(), self.has_self_loops)

    def nbytes(self) -> int:
        return self.row_offsets.numel() * 8 + self.col_indices.numel() * 4


def sorted_unique_ids(a) -> np.ndarray:
    """np.unique(a) as int64 (pipeline.py:194), with a linear-time fast path
    for ids that are already strictly increasing (train splits usually are):
    numpy's unique sorts (~0.5 s for 1.1 M ids on the bench host)."""
    a = np.asarray(a, dtype=np.int64).reshape(-1)
    if a.size < 2 or bool(np.all(a[1:] > a[:-1])):
        return a.copy()  # always a fresh array, like np.unique (callers permute it)
    return np.unique(a)


# ------------------------------------------------------- FMAT1 / CSRG1 files
# graphstore.py:364-426.  Byte-identical files (formats.py); the loaders run
# the same container validation, with CSR violations re-raised as
# FormatError.  deviceio.load_csrg_device streams the same CSRG1 file
# straight into HBM.

def save_features(f: FeatureMatrix, path: str) -> None:
    """FMAT1: 32-byte header then row-major little-endian payload."""
    from . import formats
    formats.write_fmat(path, f.values)


def load_features(path: str) -> FeatureMatrix:
    from . import formats
    return FeatureMatrix(formats.read_fmat(path))


def save_graph(g, path: str) -> None:
    """CSRG1: header, u64 row offsets, u32 column indices (a DeviceGraph is
    copied to the host first)."""
    from . import formats
    if isinstance(g, DeviceGraph):
        g = g.to_host()
    formats.write_csrg(path, g.n, g.row_offsets, g.col_indices, g.has_self_loops)


def load_graph(path: str) -> CsrGraph:
    from . import formats
    from .errors import FormatError
    n, off, col, loops = formats.read_csrg(path)
    try:
        g = CsrGraph(n, off, col)
    except DataError as e:
        raise FormatError(f"{path}: {e}") from e
    if g.has_self_loops != loops:
        raise FormatError(f"{path}: self-loop flag does not match contents")
    return g
