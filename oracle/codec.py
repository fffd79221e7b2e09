"""Oracle: low-bit row codec (TEST INFRASTRUCTURE ONLY).

Restates ``halobit/codec.py`` in float64 numpy:

* bit widths 1..8, 16 and the 32-bit passthrough (codec.py:28, 35-52);
* per-row metadata ``row_min = f32(min)``, ``row_scale = f32((max-min)/B)``
  computed in float64 before the cast (codec.py:178-184);
* stochastic rounding ``code = clip(floor(hbar) + (u < hbar - floor(hbar)), 0, B)``
  with ``hbar = (x - f64(row_min)) / f64(row_scale)`` on rows with
  ``row_scale > 0``; one uniform per element of the block, row-major, drawn
  for constant rows too (codec.py:185-194);
* LSB-first packing, code bit ``j`` of column ``c`` at row bit ``c*b + j``,
  rows padded to whole bytes, b=16 as little-endian u16 (codec.py:100-134);
* dequantization ``f64(scale) * code + f64(min)`` (codec.py:199-207);
* the wire block ``<BBHII`` header {version=1, bits, 0, rows, dim} +
  interleaved f32 (min, scale) per row + payload (codec.py:22-25, 71-76);
* byte accounting (codec.py:104-121).
"""

from __future__ import annotations

import struct

import numpy as np

HEADER = struct.Struct("<BBHII")
HEADER_BYTES = HEADER.size  # 12
WIRE_VERSION = 1
VALID_BITS = tuple(range(1, 9)) + (16, 32)


class OracleCodecError(ValueError):
    pass


def row_bytes(d: int, b: int) -> int:
    return (d * b + 7) // 8


def payload_bytes(rows: int, d: int, b: int) -> int:
    """codec.py:110-114 — fp32 basis for the passthrough."""
    return rows * d * 4 if b == 32 else rows * row_bytes(d, b)


def metadata_bytes(rows: int, b: int) -> int:
    """codec.py:117-121."""
    return 0 if b == 32 else 8 * rows


def pack(codes: np.ndarray, b: int) -> bytes:
    """(rows, d) integer codes → packed payload bytes (codec.py:124-134)."""
    codes = np.asarray(codes)
    if codes.size and (codes.min() < 0 or codes.max() >= (1 << b)):
        raise OracleCodecError("code out of range")
    if b == 16:
        return codes.astype("<u2").tobytes()
    rows, d = codes.shape
    planes = (codes.astype(np.uint16)[:, :, None] >> np.arange(b, dtype=np.uint16)) & 1
    return np.packbits(planes.astype(np.uint8).reshape(rows, d * b), axis=1,
                       bitorder="little").tobytes()


def unpack(raw: bytes, rows: int, d: int, b: int) -> np.ndarray:
    """Inverse of ``pack`` (codec.py:137-145)."""
    if len(raw) != rows * row_bytes(d, b):
        raise OracleCodecError("payload length mismatch")
    if b == 16:
        return np.frombuffer(raw, dtype="<u2").reshape(rows, d).astype(np.int64)
    by = np.frombuffer(raw, dtype=np.uint8).reshape(rows, row_bytes(d, b))
    bits = np.unpackbits(by, axis=1, bitorder="little", count=d * b).reshape(rows, d, b)
    return (bits.astype(np.int64) << np.arange(b, dtype=np.int64)).sum(axis=2)


def quantize(m: np.ndarray, b: int, u: np.ndarray | None):
    """Quantize a float64 (rows, d) block.

    ``u`` — the (rows*d) uniforms for this block (row-major), ignored for
    b=32.  Returns ``(row_min f32, row_scale f32, codes int64)`` or, for
    b=32, ``(None, None, m)``.
    """
    m = np.atleast_2d(np.asarray(m, dtype=np.float64))
    if not np.isfinite(m).all():
        raise OracleCodecError("non-finite values in quantizer input")
    if b == 32:
        return None, None, m.copy()
    rows, d = m.shape
    B = (1 << b) - 1
    lo = m.min(axis=1) if d else np.zeros(rows)
    hi = m.max(axis=1) if d else np.zeros(rows)
    rmin = lo.astype(np.float32)
    rscale = ((hi - lo) / B).astype(np.float32)
    codes = np.zeros((rows, d), dtype=np.int64)
    live = rscale.astype(np.float64) > 0.0
    uu = np.asarray(u, dtype=np.float64).reshape(rows, d)
    if live.any():
        hbar = (m[live] - rmin[live].astype(np.float64)[:, None]) \
            / rscale[live].astype(np.float64)[:, None]
        fl = np.floor(hbar)
        codes[live] = np.clip(fl + (uu[live] < hbar - fl), 0, B).astype(np.int64)
    return rmin, rscale, codes


def dequantize(rmin, rscale, codes, b: int) -> np.ndarray:
    """codec.py:199-207 (separate f64 multiply then add)."""
    if b == 32:
        return np.array(codes, dtype=np.float64, copy=True)
    return rscale.astype(np.float64)[:, None] * codes + rmin.astype(np.float64)[:, None]


def wire_block(rmin, rscale, codes, b: int, rows: int, d: int) -> bytes:
    """Header + interleaved (min, scale) + payload (codec.py:71-76).

    The passthrough block carries fp32 rows here (the accounting basis,
    codec.py:110-114) — the reference keeps f64 in its in-process object.
    """
    head = HEADER.pack(WIRE_VERSION, b, 0, rows, d)
    if b == 32:
        return head + np.asarray(codes, dtype="<f4").tobytes()
    meta = np.empty((rows, 2), dtype="<f4")
    meta[:, 0] = rmin
    meta[:, 1] = rscale
    return head + meta.tobytes() + pack(codes, b)


def parse_wire_block(raw: bytes):
    """Inverse of ``wire_block`` → (bits, rows, d, rmin, rscale, codes)."""
    ver, b, _, rows, d = HEADER.unpack_from(raw)
    if ver != WIRE_VERSION:
        raise OracleCodecError("bad wire version")
    if b == 32:
        vals = np.frombuffer(raw[HEADER_BYTES:], dtype="<f4").reshape(rows, d)
        return b, rows, d, None, None, vals.astype(np.float64)
    meta = np.frombuffer(raw[HEADER_BYTES:HEADER_BYTES + 8 * rows], dtype="<f4").reshape(rows, 2)
    codes = unpack(raw[HEADER_BYTES + 8 * rows:], rows, d, b)
    return b, rows, d, meta[:, 0].copy(), meta[:, 1].copy(), codes
