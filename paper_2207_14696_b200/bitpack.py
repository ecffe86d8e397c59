"""MSB-first code bitstreams (pkg/src/featgrind/bitpack.py:17-83), on the GPU.

Same names, arguments, return types and errors as the reference module;
the bit work runs in ``fg_bits_pack`` / ``fg_bits_unpack`` /
``fg_bit_rows_gather`` (csrc/fg_bitpack.cu).  Inputs are host arrays or
bytes (the reference's interface): they are copied to the device, and the
results copied back.  No CPU fallback.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .errors import DataError


def _dev_bytes(payload):
    import torch
    buf = np.frombuffer(payload, dtype=np.uint8) if isinstance(payload, (bytes, bytearray)) \
        else np.ascontiguousarray(payload, dtype=np.uint8).reshape(-1)
    return torch.from_numpy(buf.copy()).cuda() if buf.size else torch.zeros(1, dtype=torch.uint8,
                                                                            device="cuda"), buf.size


def _check_bits(bits: int) -> None:
    if not 1 <= bits <= 32:
        raise DataError(f"code width must be in [1, 32], got {bits}")


def pack_codes(codes: np.ndarray, bits: int) -> bytes:
    """bitpack.py:17-36: row-major codes -> ceil(size*bits/8) bytes."""
    import torch
    _check_bits(bits)
    N.require_cuda()
    flat = np.ascontiguousarray(codes).reshape(-1).astype(np.int64)
    nbytes = (flat.size * bits + 7) // 8
    if nbytes == 0:
        return b""
    d = torch.from_numpy(flat).cuda()
    out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.call("fg_bits_pack", N.ptr(d), flat.size, bits, N.ptr(out), N.ptr(err), N.stream_handle())
    if int(err.item()):
        raise DataError(f"codes do not fit in {bits} bits")
    return out.cpu().numpy().tobytes()


def unpack_codes(payload, bits: int, count: int, start_bit: int = 0) -> np.ndarray:
    """bitpack.py:39-55: ``count`` codes from ``start_bit``, int64."""
    import torch
    _check_bits(bits)
    N.require_cuda()
    d, nbytes = _dev_bytes(payload)
    need = start_bit + count * bits
    if need > nbytes * 8:
        raise DataError(f"bitstream too short: need {need} bits, have {nbytes * 8}")
    out = torch.empty(max(count, 1), dtype=torch.int64, device="cuda")
    N.call("fg_bits_unpack", N.ptr(d), nbytes, start_bit, count, bits, N.ptr(out),
           N.stream_handle())
    return out[:count].cpu().numpy()


def gather_bit_rows(payload, row_bits: int, row_ids) -> np.ndarray:
    """bitpack.py:58-83: (len(row_ids), row_bits) uint8 matrix of raw bits,
    rows in any order, repeats allowed."""
    import torch
    rows = np.asarray(row_ids, dtype=np.int64).reshape(-1)
    if rows.size == 0:
        return np.zeros((0, row_bits), dtype=np.uint8)
    N.require_cuda()
    d, nbytes = _dev_bytes(payload)
    r = torch.from_numpy(rows.copy()).cuda()
    out = torch.empty((rows.size, row_bits), dtype=torch.uint8, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.call("fg_bit_rows_gather", N.ptr(d), nbytes, row_bits, N.ptr(r), rows.size, N.ptr(out),
           N.ptr(err), N.stream_handle())
    if int(err.item()):
        raise DataError("row ids exceed the packed stream")
    return out.cpu().numpy()
