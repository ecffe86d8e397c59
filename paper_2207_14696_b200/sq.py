"""Log-domain scalar quantization, B200 path (drop-in for pkg/src/featgrind/sq.py).

Public names, signatures, dataclasses and errors are the reference's
(sq.py:39-194).  The heavy work runs in sm_100a kernels through the C ABI:

* ``quantize_sq``  -> ``fg_sq_encode``: compares |x| against 2^(k-1)-1
  thresholds.  The thresholds are derived on the host by bisection over
  float bit patterns of the reference's own float64 expression
  (sq.py:119-127), which is monotone in |x|; the resulting codes are
  bit-identical by construction (and pinned by tests/golden).
* ``dequantize_sq`` -> ``fg_sq_gather_dequant``: a 2^k-entry LUT holding the
  reference decode (sq.py:144-153) of every code; decode is one lookup.
* ``fit_sq`` -> device nonzero compaction / strided sampling and an exact
  radix select of the four order statistics np.quantile interpolates; the
  host applies numpy's log2 and the quantile lerp to those four values.

``DeviceSqCodec`` is the HBM-resident form the training path reads.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import formats
from .errors import DataError, FormatError
from .graph import FeatureMatrix

__all__ = ["SqParams", "SqCodec", "fit_sq", "quantize_sq", "dequantize_sq",
           "sq_compression_ratio", "save_sq", "load_sq", "DeviceSqCodec",
           "sq_decode_table", "sq_thresholds"]

SQF_HEADER_BYTES = formats.SQF_HEADER_BYTES
FIT_SAMPLE_CAP = 10_000_000
DEFAULT_CLIP_TAIL_FRACTION = 0.005


@dataclass(frozen=True)
class SqParams:
    """Bit width and fitted exponent range (sq.py:39-58)."""

    k: int
    e_min: float
    e_max: float
    clip_tail_fraction: float = DEFAULT_CLIP_TAIL_FRACTION

    def __post_init__(self) -> None:
        if not 1 <= self.k <= 8:
            raise DataError(f"k must be in [1, 8], got {self.k}")
        if not 0.0 <= self.clip_tail_fraction <= 0.2:
            raise DataError("clip_tail_fraction must be in [0, 0.2]")
        if not (np.isfinite(self.e_min) and np.isfinite(self.e_max)):
            raise DataError("exponent range must be finite")
        if self.k >= 2 and not self.e_min < self.e_max:
            raise DataError("e_min must be < e_max for k >= 2")
        if self.e_min > self.e_max:
            raise DataError("e_min must be <= e_max")


@dataclass(frozen=True)
class SqCodec:
    """Params plus the packed MSB-first row-major payload (sq.py:61-81)."""

    params: SqParams
    n: int
    d: int
    payload: bytes
    elem_bits: int = 32

    def __post_init__(self) -> None:
        if self.n < 0 or self.d < 1:
            raise DataError("invalid codec dimensions")
        if self.elem_bits not in (32, 64):
            raise DataError("elem_bits must be 32 or 64")
        expect = (self.n * self.d * self.params.k + 7) // 8
        if len(self.payload) != expect:
            raise DataError(f"payload must be {expect} bytes, got {len(self.payload)}")

    def bytes_per_row(self) -> int:
        return (self.d * self.params.k + 7) // 8


# ---------------------------------------------------------- host tables

def _ref_offsets(mag: np.ndarray, p: SqParams) -> np.ndarray:
    """The reference's bucket offset of non-negative magnitudes (float64),
    evaluated with exactly sq.py:120-127's operations and order."""
    logs = np.log2(np.where(mag == 0, 1.0, mag))
    logs = np.where(mag == 0, p.e_min, logs)
    np.clip(logs, p.e_min, p.e_max, out=logs)
    half = 1 << (p.k - 1)
    scaled = (logs - p.e_min) / (p.e_max - p.e_min) * half
    off = np.floor(scaled).astype(np.int64)
    np.clip(off, 0, half - 1, out=off)
    return off


def sq_thresholds(p: SqParams, elem_bits: int = 32) -> np.ndarray:
    """t_j = smallest |x| (float32 or float64) whose reference offset >= j,
    j = 1 .. 2^(k-1)-1; +inf when no finite value reaches j."""
    half = 1 << (p.k - 1)
    if half <= 1:
        return np.zeros(0, np.float32 if elem_bits == 32 else np.float64)
    if elem_bits == 32:
        ftype, itype, top = np.float32, np.uint32, np.uint32(0x7F800000)  # +inf pattern
    else:
        ftype, itype, top = np.float64, np.uint64, np.uint64(0x7FF0000000000000)
    want = np.arange(1, half, dtype=np.int64)
    lo = np.zeros(want.size, itype)              # pattern of +0.0
    hi = np.full(want.size, top, itype)           # exclusive upper bound (inf)
    # invariant: off(lo-1 pattern) < j (or lo == 0), answer in [lo, hi]
    while True:
        active = lo < hi
        if not active.any():
            break
        mid = lo + (hi - lo) // itype(2)
        vals = mid.view(ftype).astype(np.float64)
        reach = _ref_offsets(vals, p) >= want
        hi = np.where(active & reach, mid, hi)
        lo = np.where(active & ~reach, mid + itype(1), lo)
    return lo.view(ftype).copy()   # lo == top -> +inf: never reached


def sq_decode_table(p: SqParams, elem_bits: int = 32) -> np.ndarray:
    """Reference decode (sq.py:144-153) of every code 0 .. 2^k-1."""
    q = np.arange(1 << p.k, dtype=np.int64)
    half = 1 << (p.k - 1)
    span = p.e_max - p.e_min
    steps = np.where(q >= half, q - half + 0.5, half - 0.5 - q)
    mags = np.exp2(steps * (span / half) + p.e_min)
    out = np.where(q >= half, mags, -mags)
    return out.astype(np.float32 if elem_bits == 32 else np.float64)


def sq_row_stride(d: int, k: int) -> int:
    """Device row stride: whole 16-code chunks, rounded to 32 B sectors."""
    need = max((d * k + 7) // 8, ((d + 15) // 16) * 2 * k)
    return ((need + 31) // 32) * 32


# ------------------------------------------------------------ device codec

class DeviceSqCodec:
    """HBM-resident SQ codec: strided code rows + decode LUT."""

    def __init__(self, params: SqParams, n: int, d: int, rows, elem_bits: int = 32):
        import torch
        self.params, self.n, self.d, self.elem_bits = params, int(n), int(d), elem_bits
        self.row_stride = sq_row_stride(d, params.k)
        self.rows = rows  # uint8 [n, row_stride]
        self.lut = torch.from_numpy(sq_decode_table(params, elem_bits)).to(rows.device)
        self._closed = False
        self._desc = N.CodecDesc(N.CODEC_SQ, params.k, self.n, self.d, self.row_stride,
                                 N.ptr(rows), N.ptr(self.lut), 0, 0, 0, elem_bits, None)

    # -- construction
    @classmethod
    def empty(cls, params: SqParams, n: int, d: int, device="cuda", elem_bits: int = 32):
        import torch
        rows = torch.zeros((n, sq_row_stride(d, params.k)), dtype=torch.uint8, device=device)
        return cls(params, n, d, rows, elem_bits)

    @classmethod
    def from_codec(cls, c: SqCodec, device="cuda") -> "DeviceSqCodec":
        import torch
        N.require_cuda()
        dc = cls.empty(c.params, c.n, c.d, device, c.elem_bits)
        if c.n:
            stream = torch.frombuffer(bytearray(c.payload), dtype=torch.uint8).to(device)
            N.call("fg_stream_to_rows", N.ptr(stream), stream.numel(), c.n, c.d * c.params.k,
                   N.ptr(dc.rows), dc.row_stride, N.stream_handle())
        return dc

    def encode_rows_(self, x, row0: int = 0) -> None:
        """Quantize a device block x [m, d] (float32/float64) into rows
        [row0, row0+m) -- the streaming encode used for matrices that never
        exist whole in memory."""
        import torch
        self._check_open()
        x = x.contiguous()
        m = x.shape[0]
        is64 = x.dtype == torch.float64
        thr = torch.from_numpy(sq_thresholds(self.params, 64 if is64 else 32)).to(x.device)
        dst = self.rows[row0:row0 + m]
        N.call("fg_sq_encode", N.ptr(x), int(is64), m, self.d, self.params.k,
               None if is64 else N.ptr(thr), N.ptr(thr) if is64 else None,
               N.ptr(dst), self.row_stride, N.stream_handle())

    def to_codec(self) -> SqCodec:
        import torch
        self._check_open()
        nbytes = (self.n * self.d * self.params.k + 7) // 8
        stream = torch.empty(nbytes, dtype=torch.uint8, device=self.rows.device)
        if nbytes:
            N.call("fg_rows_to_stream", N.ptr(self.rows), self.n, self.d * self.params.k,
                   self.row_stride, N.ptr(stream), nbytes, N.stream_handle())
        return SqCodec(self.params, self.n, self.d, stream.cpu().numpy().tobytes(), self.elem_bits)

    # -- access
    @property
    def desc(self) -> N.CodecDesc:
        self._check_open()
        return self._desc

    def gather(self, ids, out_dtype=None, check: bool = True):
        """Decode rows ``ids`` (device int32/int64 tensor) -> [len(ids), d]."""
        import torch
        self._check_open()
        if out_dtype is None:
            out_dtype = torch.float64 if self.elem_bits == 64 else torch.float32
        code = {torch.float32: N.OUT_F32, torch.bfloat16: N.OUT_BF16,
                torch.float64: N.OUT_F64}[out_dtype]
        out = torch.empty((ids.numel(), self.d), dtype=out_dtype, device=self.rows.device)
        err = torch.zeros(1, dtype=torch.int32, device=self.rows.device)
        N.call("fg_sq_gather_dequant", C_ref(self._desc), N.ptr(ids),
               int(ids.dtype == torch.int32), ids.numel(), N.ptr(out), code, N.ptr(err),
               N.stream_handle())
        if check and int(err.item()) != 0:
            raise DataError("row id out of range")
        return out

    def nbytes(self) -> int:
        return self.rows.numel()

    def close(self) -> None:
        """Release device memory; later use raises DataError."""
        self.rows = None
        self.lut = None
        self._closed = True

    def _check_open(self):
        if self._closed:
            raise DataError("operation on a closed codec handle")


def C_ref(desc):
    import ctypes
    return ctypes.byref(desc)


# --------------------------------------------------------------- public API

def _device_values(f: FeatureMatrix):
    import torch
    N.require_cuda()
    return torch.from_numpy(f.values).cuda()


def _quantile_lerp(lo_val: float, hi_val: float, m: int, q: float) -> float:
    """numpy 'linear' quantile interpolation (numpy/lib/_function_base_impl.py
    _quantile/_lerp) given the two neighbouring order statistics."""
    v = (m - 1) * np.float64(q)
    prev = np.floor(v)
    t = v - prev
    a, b = np.float64(lo_val), np.float64(hi_val)
    diff = b - a
    r = a + diff * t
    if t >= 0.5:
        r = b - diff * (1 - t)
    return float(r)


def _order_stat_ranks(m: int, q: float) -> tuple[int, int]:
    v = (m - 1) * np.float64(q)
    if v >= m - 1:
        return m - 1, m - 1
    if v < 0:
        return 0, 0
    prev = int(np.floor(v))
    return prev, prev + 1


def fit_sq(f: FeatureMatrix, k: int,
           clip_tail_fraction: float = DEFAULT_CLIP_TAIL_FRACTION) -> SqParams:
    """sq.py:84-111 on the device (see module docstring)."""
    import torch
    if not 1 <= k <= 8:
        raise DataError(f"k must be in [1, 8], got {k}")
    if not 0.0 <= clip_tail_fraction <= 0.2:
        raise DataError("clip_tail_fraction must be in [0, 0.2]")
    x = _device_values(f).reshape(-1)
    return fit_sq_device(x, k, clip_tail_fraction)


def _params_from_sample(sample_abs, m: int, k: int, clip: float,
                        sorted_host=None) -> SqParams:
    """e_min/e_max from the fit sample (|x| of the strided nonzeros): exact
    radix-select of the four order statistics np.quantile interpolates, then
    numpy's log2 + quantile lerp on those values (sq.py:107-108)."""
    import ctypes
    import torch
    qs = [clip, 1.0 - clip]
    ranks = sorted({r for q in qs for r in _order_stat_ranks(m, q)})
    if sorted_host is None:
        sel_ws = torch.empty(N.lib().fg_select_workspace_bytes(), dtype=torch.uint8,
                             device=sample_abs.device)
        rk = (ctypes.c_int64 * len(ranks))(*ranks)
        outv = (ctypes.c_float * len(ranks))()
        N.call("fg_select_ranks", N.ptr(sample_abs), m, rk, len(ranks), outv, N.ptr(sel_ws),
               sel_ws.numel(), N.stream_handle())
        stats = {r: float(np.float32(outv[i])) for i, r in enumerate(ranks)}
    else:
        stats = {r: float(sorted_host[r]) for r in ranks}
    logs = {r: float(np.log2(np.abs(np.array([v], dtype=np.float64)))[0])
            for r, v in stats.items()}
    e_min, e_max = (_quantile_lerp(logs[_order_stat_ranks(m, q)[0]],
                                   logs[_order_stat_ranks(m, q)[1]], m, q) for q in qs)
    if k >= 2 and not e_min < e_max:
        raise DataError("constant log-magnitude data: exponent range is empty")
    return SqParams(k, float(e_min), float(e_max), clip)


def fit_sq_device(x, k: int, clip_tail_fraction: float = DEFAULT_CLIP_TAIL_FRACTION) -> SqParams:
    """fit_sq over a flat device tensor in row-major order."""
    import torch
    dev = x.device
    if x.dtype == torch.float32:
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        N.call("fg_count_nonzero", N.ptr(x), x.numel(), N.ptr(cnt), N.stream_handle())
        nnz = int(cnt.item())
    else:
        nnz = int((x != 0).sum().item())
    if nnz == 0:
        if k == 1:
            return SqParams(1, 0.0, 0.0, clip_tail_fraction)
        raise DataError("cannot fit an exponent range on an all-zero matrix")
    m = min(nnz, FIT_SAMPLE_CAP)
    if x.dtype == torch.float32:
        sample = torch.empty(m, dtype=torch.float32, device=dev)
        ws = torch.empty(max(N.lib().fg_nonzero_sample_workspace_bytes(x.numel()), 1),
                         dtype=torch.uint8, device=dev)
        N.call("fg_gather_nonzero_sample", N.ptr(x), x.numel(), nnz, FIT_SAMPLE_CAP,
               N.ptr(sample), N.ptr(ws), ws.numel(), N.stream_handle())
        return _params_from_sample(sample, m, k, clip_tail_fraction)
    # float64 features: exact order statistics with a device sort
    nz = x[x != 0]
    if nnz > FIT_SAMPLE_CAP:
        pick = torch.from_numpy(np.linspace(0, nnz - 1, FIT_SAMPLE_CAP).astype(np.int64))
        nz = nz[pick.to(dev)]
    srt = torch.sort(nz.abs()).values.cpu().numpy()
    return _params_from_sample(None, m, k, clip_tail_fraction, sorted_host=srt)


def fit_sq_stream(chunks, k: int, clip_tail_fraction: float = DEFAULT_CLIP_TAIL_FRACTION,
                  device="cuda") -> SqParams:
    """fit_sq over a matrix that only exists as a sequence of row chunks
    (``chunks()`` yields float32 device tensors in row order, and can be
    called twice): pass 1 counts nonzeros per chunk, pass 2 gathers the
    reference's linspace-strided sample with global ranks.  Same result as
    fit_sq on the whole matrix."""
    import torch
    cnt = torch.zeros(1, dtype=torch.int64, device=device)
    per = []
    for x in chunks():
        N.call("fg_count_nonzero", N.ptr(x), x.numel(), N.ptr(cnt), N.stream_handle())
        per.append(int(cnt.item()))
    nnz = sum(per)
    if nnz == 0:
        if k == 1:
            return SqParams(1, 0.0, 0.0, clip_tail_fraction)
        raise DataError("cannot fit an exponent range on an all-zero matrix")
    m = min(nnz, FIT_SAMPLE_CAP)
    sample = torch.empty(m, dtype=torch.float32, device=device)
    base = 0
    for x, c in zip(chunks(), per):
        ws = torch.empty(max(N.lib().fg_nonzero_sample_workspace_bytes(x.numel()), 1),
                         dtype=torch.uint8, device=device)
        N.call("fg_gather_nonzero_sample_chunk", N.ptr(x), x.numel(), base, nnz, FIT_SAMPLE_CAP,
               N.ptr(sample), N.ptr(ws), ws.numel(), N.stream_handle())
        base += c
    return _params_from_sample(sample, m, k, clip_tail_fraction)


def quantize_sq(f: FeatureMatrix, p: SqParams) -> SqCodec:
    """sq.py:114-129 on the device; payload bit-identical to the reference."""
    x = _device_values(f)
    dc = DeviceSqCodec.empty(p, f.n, f.d, x.device, f.elem_bits)
    if f.n:
        dc.encode_rows_(x, 0)
    return dc.to_codec()


def _codec_on_device(c: SqCodec) -> DeviceSqCodec:
    cache = c.__dict__.get("_device_cache")
    if cache is None:
        cache = DeviceSqCodec.from_codec(c)
        object.__setattr__(c, "_device_cache", cache)
    return cache


def dequantize_sq(c: SqCodec, rows: np.ndarray | None = None) -> FeatureMatrix:
    """sq.py:132-153: bucket midpoints for a row subset (or all rows)."""
    import torch
    if rows is None:
        ids = np.arange(c.n, dtype=np.int64)
    else:
        ids = np.asarray(rows, dtype=np.int64)
        if ids.size and (ids.min() < 0 or ids.max() >= c.n):
            raise DataError("row id out of range")
    if ids.size == 0:
        return FeatureMatrix(np.zeros((0, c.d), np.float32 if c.elem_bits == 32 else np.float64))
    dc = _codec_on_device(c)
    out = dc.gather(torch.from_numpy(ids).cuda())
    return FeatureMatrix(out.cpu().numpy())


def sq_compression_ratio(c: SqCodec) -> tuple[float, float]:
    """sq.py:156-165: (payload-only ratio, ratio including the header)."""
    raw = c.n * c.d * (c.elem_bits // 8)
    return c.elem_bits / c.params.k, raw / (SQF_HEADER_BYTES + len(c.payload))


def save_sq(c: SqCodec, path: str) -> None:
    p = c.params
    formats.write_sqf(path, p.k, c.n, c.d, p.e_min, p.e_max, p.clip_tail_fraction, c.payload)


def load_sq(path: str) -> SqCodec:
    k, n, d, e_min, e_max, clip, payload = formats.read_sqf(path)
    try:
        return SqCodec(SqParams(k, e_min, e_max, clip), n, d, payload)
    except DataError as e:
        raise FormatError(f"{path}: {e}") from e
