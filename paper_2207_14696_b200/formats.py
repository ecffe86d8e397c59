"""Binary file formats, byte-compatible with the reference.

  FMAT1 / CSRG1 : pkg/src/featgrind/graphstore.py:33-39, 364-426
  SQF1          : pkg/src/featgrind/sq.py:30-33, 168-194
  VQF1          : pkg/src/featgrind/vq.py:31-37, 365-439

All little-endian; headers are fixed-size structs.  Loaders raise
FormatError on truncation / bad magic / size mismatch with the reference's
messages.  Pinned against reference-written byte images in tests/golden.
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import DataError, FormatError

FMAT_MAGIC = b"FMAT1\x00\x00\x00"
CSRG_MAGIC = b"CSRG1\x00\x00\x00"
SQF_MAGIC = b"SQF1\x00\x00\x00\x00"
VQF_MAGIC = b"VQF1\x00\x00\x00\x00"

FMAT_HEADER = struct.Struct("<8sIIQQ")       # magic, version, elem_bits, n, d
CSRG_HEADER = struct.Struct("<8sIIQQ")       # magic, version, flags, n, nnz
SQF_HEADER = struct.Struct("<8sIIQQddd")     # magic, version, k, n, d, e_min, e_max, clip
VQF_HEADER = struct.Struct("<8sIBBHIIIQQ")   # magic, version, metric, layout, pad,
                                             # width, length, num_parts, n, d
SQF_HEADER_BYTES = SQF_HEADER.size
VQF_HEADER_BYTES = VQF_HEADER.size


def _read(path: str) -> bytes:
    with open(path, "rb") as fh:
        return fh.read()


def _header(raw: bytes, hdr: struct.Struct, magic: bytes, tag: str, path: str):
    if len(raw) < hdr.size:
        raise FormatError(f"{path}: truncated {tag} header")
    fields = hdr.unpack_from(raw)
    if fields[0] != magic:
        raise FormatError(f"{path}: not an {tag} file" if tag[0] in "AEFIOS"
                          else f"{path}: not a {tag} file")
    if fields[1] != 1:
        raise FormatError(f"{path}: unsupported {tag} version {fields[1]}")
    return fields


# ------------------------------------------------------------------ FMAT1

def write_fmat(path: str, values: np.ndarray) -> None:
    eb = 64 if values.dtype == np.float64 else 32
    with open(path, "wb") as fh:
        fh.write(FMAT_HEADER.pack(FMAT_MAGIC, 1, eb, values.shape[0], values.shape[1]))
        fh.write(np.ascontiguousarray(values, dtype="<f8" if eb == 64 else "<f4").tobytes())


def read_fmat(path: str) -> np.ndarray:
    raw = _read(path)
    _, _, eb, n, d = _header(raw, FMAT_HEADER, FMAT_MAGIC, "FMAT1", path)
    if eb not in (32, 64):
        raise FormatError(f"{path}: elem_bits must be 32 or 64, got {eb}")
    want = FMAT_HEADER.size + n * d * (eb // 8)
    if len(raw) != want:
        raise FormatError(f"{path}: expected {want} bytes, found {len(raw)}")
    dt = "<f8" if eb == 64 else "<f4"
    return np.frombuffer(raw, dtype=dt, offset=FMAT_HEADER.size).reshape(n, d).copy()


# ------------------------------------------------------------------ CSRG1

def write_csrg(path: str, n: int, row_offsets, col_indices, self_loops: bool) -> None:
    with open(path, "wb") as fh:
        fh.write(CSRG_HEADER.pack(CSRG_MAGIC, 1, 1 if self_loops else 0, n, len(col_indices)))
        fh.write(np.asarray(row_offsets).astype("<u8").tobytes())
        fh.write(np.asarray(col_indices).astype("<u4").tobytes())


def read_csrg(path: str):
    raw = _read(path)
    _, _, flags, n, nnz = _header(raw, CSRG_HEADER, CSRG_MAGIC, "CSRG1", path)
    want = CSRG_HEADER.size + (n + 1) * 8 + nnz * 4
    if len(raw) != want:
        raise FormatError(f"{path}: expected {want} bytes, found {len(raw)}")
    off = np.frombuffer(raw, "<u8", n + 1, CSRG_HEADER.size).astype(np.int64)
    col = np.frombuffer(raw, "<u4", nnz, CSRG_HEADER.size + (n + 1) * 8).astype(np.int32)
    return n, off, col, bool(flags & 1)


# ------------------------------------------------------------------- SQF1

def write_sqf(path: str, k: int, n: int, d: int, e_min: float, e_max: float,
              clip: float, payload: bytes) -> None:
    with open(path, "wb") as fh:
        fh.write(SQF_HEADER.pack(SQF_MAGIC, 1, k, n, d, e_min, e_max, clip))
        fh.write(payload)


def read_sqf(path: str):
    raw = _read(path)
    _, _, k, n, d, e_min, e_max, clip = _header(raw, SQF_HEADER, SQF_MAGIC, "SQF1", path)
    want = SQF_HEADER.size + (n * d * k + 7) // 8
    if len(raw) != want:
        raise FormatError(f"{path}: expected {want} bytes, found {len(raw)}")
    return k, n, d, e_min, e_max, clip, raw[SQF_HEADER.size:]


# ------------------------------------------------------------------- VQF1

def write_vqf(path: str, metric_id: int, layout_id: int, width: int, length: int,
              num_parts: int, n: int, d: int, padded_books: list[np.ndarray],
              code_bytes: bytes | None) -> None:
    with open(path, "wb") as fh:
        fh.write(VQF_HEADER.pack(VQF_MAGIC, 1, metric_id, layout_id, 0, width, length,
                                 num_parts, n, d))
        for cb in padded_books:
            fh.write(np.ascontiguousarray(cb, dtype="<f4").tobytes())
        if code_bytes:
            fh.write(code_bytes)


def read_vqf_header(raw: bytes, path: str):
    _, _, metric_id, layout_id, _pad, width, length, num_parts, n, d = _header(
        raw, VQF_HEADER, VQF_MAGIC, "VQF1", path)
    return metric_id, layout_id, width, length, num_parts, n, d


def check_payload(got: int, want: int, path: str, what: str) -> None:
    if got != want:
        raise FormatError(f"{path}: {what}")


__all__ = ["FormatError", "DataError", "write_fmat", "read_fmat", "write_csrg", "read_csrg",
           "write_sqf", "read_sqf", "write_vqf", "read_vqf_header", "SQF_HEADER_BYTES",
           "VQF_HEADER_BYTES"]
