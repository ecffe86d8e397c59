"""Streaming device loaders for the reference's on-disk formats (SURVEY.md
§8(f) row 2): SQF1 (sq.py:168-194), VQF1 (vq.py:365-439) and CSRG1
(graphstore.py:364-426) go file -> mmap -> pinned staging -> HBM in chunks,
never materialising the whole payload in host memory (MAG240M-shape: 23 GB of
codes, 29 GB of CSR).  Code streams are converted to the device row layout
by ``fg_stream_to_rows`` chunk by chunk; the bytes on disk are exactly the
reference's (files written by the reference load unchanged).

Two pinned buffers alternate: the host copy of chunk i+1 overlaps the
host->device copy and conversion of chunk i.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _native as N
from . import formats
from .errors import DataError, FormatError


def _stream_file(path: str, offset: int, nbytes: int, chunk_bytes: int, consume, device):
    """Call consume(dev_uint8_chunk, byte_off) for consecutive chunks of
    [offset, offset+nbytes) of the file (chunk_bytes may be shortened by
    consume's alignment: it receives whole chunks and returns nothing)."""
    if nbytes == 0:
        return
    mm = np.memmap(path, dtype=np.uint8, mode="r", offset=offset, shape=(nbytes,))
    cap = min(chunk_bytes, nbytes)
    pinned = [torch.empty(cap, dtype=torch.uint8).pin_memory() for _ in range(2)]
    dev = [torch.empty(cap, dtype=torch.uint8, device=device) for _ in range(2)]
    done = [None, None]
    pos, i = 0, 0
    while pos < nbytes:
        m = min(cap, nbytes - pos)
        k = i & 1
        if done[k] is not None:
            done[k].synchronize()          # pinned[k]'s previous copy finished
        np.copyto(pinned[k].numpy()[:m], mm[pos:pos + m])
        dev[k][:m].copy_(pinned[k][:m], non_blocking=True)
        consume(dev[k][:m], pos)
        ev = torch.cuda.Event()
        ev.record()
        done[k] = ev
        pos += m
        i += 1
    torch.cuda.current_stream().synchronize()
    del mm


def _rows_chunk_bytes(row_bits: int, chunk_bytes: int) -> int:
    """Chunk size covering whole rows, starting each chunk on a byte boundary
    (a multiple of 8 rows always does)."""
    rows = max(8, (chunk_bytes * 8 // max(row_bits, 1)) // 8 * 8)
    return rows * row_bits // 8


def _stream_rows(path, offset, n, row_bits, rows_out, stride, chunk_bytes, device):
    """MSB-first code stream of n rows (row r at bit r*row_bits) -> device rows."""
    total = (n * row_bits + 7) // 8
    step = _rows_chunk_bytes(row_bits, chunk_bytes)

    def consume(chunk, byte_off):
        r0 = byte_off * 8 // row_bits
        m = min(n - r0, (chunk.numel() * 8) // row_bits if byte_off + chunk.numel() < total
                else n - r0)
        N.call("fg_stream_to_rows", N.ptr(chunk), chunk.numel(), m, row_bits,
               N.ptr(rows_out) + r0 * stride, stride, N.stream_handle())
    _stream_file(path, offset, total, step, consume, device)


def load_sq_device(path: str, device="cuda", chunk_bytes: int = 256 << 20):
    """SQF1 file -> DeviceSqCodec (same result as
    DeviceSqCodec.from_codec(load_sq(path)), without reading the payload
    into host memory)."""
    from .sq import DeviceSqCodec, SqParams
    with open(path, "rb") as fh:
        hdr = fh.read(formats.SQF_HEADER.size)
    _, _, k, n, d, e_min, e_max, clip = formats._header(hdr, formats.SQF_HEADER,
                                                        formats.SQF_MAGIC, "SQF1", path)
    want = formats.SQF_HEADER.size + (n * d * k + 7) // 8
    if os.path.getsize(path) != want:
        raise FormatError(f"{path}: expected {want} bytes, found {os.path.getsize(path)}")
    try:  # load_sq (sq.py:190-194): invalid params are format errors
        params = SqParams(k, e_min, e_max, clip)
        if n < 0 or d < 1:
            raise DataError("invalid codec dimensions")
    except DataError as e:
        raise FormatError(f"{path}: {e}") from e
    dc = DeviceSqCodec.empty(params, n, d, device)
    _stream_rows(path, formats.SQF_HEADER.size, n, d * k, dc.rows, dc.row_stride, chunk_bytes,
                 device)
    return dc


def load_vq_device(path: str, device="cuda", chunk_bytes: int = 256 << 20):
    """VQF1 file -> DeviceVqCodec.  Packed layouts (and byte-aligned 8-bit
    codes, the same bytes) stream straight to device rows; byte-aligned
    16-bit codes take the host path (load_vq + from_codec)."""
    from .vq import CODE_LAYOUTS, METRICS, DeviceVqCodec, VqParams, load_vq
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        hdr = fh.read(formats.VQF_HEADER_BYTES)
    metric_id, layout_id, width, length, num_parts, n, d = formats.read_vqf_header(hdr, path)
    if metric_id >= len(METRICS) or layout_id >= len(CODE_LAYOUTS):
        raise FormatError(f"{path}: unknown metric or layout id")
    try:  # mirror load_vq (vq.py:405-409, 438-439): bad params are format errors
        params = VqParams(width, length, METRICS[metric_id], CODE_LAYOUTS[layout_id])
        if params.num_parts(d) != num_parts:
            raise FormatError(f"{path}: num_parts inconsistent with width and d")
        if width > d:
            raise FormatError(f"{path}: need 1 <= width <= d")
    except DataError as e:
        if isinstance(e, FormatError):
            raise
        raise FormatError(f"{path}: {e}") from e
    bits = params.bits_per_code
    if params.code_layout != "packed" and bits > 8:
        return DeviceVqCodec.from_codec(load_vq(path), device)
    pos = formats.VQF_HEADER_BYTES
    books = []
    with open(path, "rb") as fh:
        fh.seek(pos)
        for sl in params.part_slices(d):
            w = sl.stop - sl.start
            raw = fh.read(length * w * 4)
            if len(raw) != length * w * 4:
                raise FormatError(f"{path}: truncated codebooks")
            books.append(np.frombuffer(raw, "<f4").reshape(length, w).copy())
            pos += length * w * 4
    row_bits = num_parts * bits
    if size - pos != (n * row_bits + 7) // 8:
        raise FormatError(f"{path}: code payload size mismatch")
    dc = DeviceVqCodec.empty(params, d, tuple(books), n, device)
    _stream_rows(path, pos, n, row_bits, dc.rows, dc.row_stride, chunk_bytes, device)
    return dc


def load_csrg_device(path: str, device="cuda", chunk_bytes: int = 256 << 20):
    """CSRG1 file -> DeviceGraph (int64 offsets / int32 columns in HBM),
    streamed; cheap device checks (monotone offsets, columns in range)
    replace the reference's host lexsort validation (graphstore.py:116-119)."""
    from .graph import DeviceGraph
    with open(path, "rb") as fh:
        hdr = fh.read(formats.CSRG_HEADER.size)
    _, _, flags, n, nnz = formats._header(hdr, formats.CSRG_HEADER, formats.CSRG_MAGIC, "CSRG1",
                                          path)
    want = formats.CSRG_HEADER.size + (n + 1) * 8 + nnz * 4
    if os.path.getsize(path) != want:
        raise FormatError(f"{path}: expected {want} bytes, found {os.path.getsize(path)}")
    off = torch.empty(n + 1, dtype=torch.int64, device=device)
    col = torch.empty(nnz, dtype=torch.int32, device=device)
    for t, offset, nbytes in ((off, formats.CSRG_HEADER.size, (n + 1) * 8),
                              (col, formats.CSRG_HEADER.size + (n + 1) * 8, nnz * 4)):
        flat = t.view(torch.uint8)

        def consume(chunk, byte_off, flat=flat):
            flat[byte_off:byte_off + chunk.numel()].copy_(chunk)
        _stream_file(path, offset, nbytes, chunk_bytes, consume, device)
    bad = (off[0] != 0) | (off[-1] != nnz) | (off[1:] < off[:-1]).any()
    if nnz:
        bad |= (col.min() < 0) | (col.max() >= n)
    if bool(bad):
        raise FormatError(f"{path}: invalid CSR (offsets or column range)")
    # self-loops all-or-none and matching the header flag (graphstore.py:
    # 125-127, 423-425): one binary search per row on the device
    cnt = torch.zeros(1, dtype=torch.int64, device=device)
    N.call("fg_csr_self_loops", N.ptr(off), N.ptr(col), n, N.ptr(cnt), N.stream_handle())
    loops = int(cnt.item())
    if loops not in (0, n):
        raise FormatError(f"{path}: self-loops must be present on all nodes or none")
    if (loops == n and n > 0) != bool(flags & 1):
        raise FormatError(f"{path}: self-loop flag does not match contents")
    return DeviceGraph(n, off, col, bool(flags & 1))
