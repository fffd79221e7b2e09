"""Low-bit Module: drop-in for ``halobit.codec`` running on the B200.

Same public surface as the reference (``codec.py:28-207``): ``QuantConfig``,
``QuantizedBlock`` (identical wire layout), ``quantize_rows``,
``dequantize_rows``, ``payload_bytes``, ``metadata_bytes``, ``CodecError``.
``quantize_rows``/``dequantize_rows`` run the K1/K2 kernels through the C-ABI
(``hb_quantize_gather`` / ``hb_dequant_gather``); the packed payload and the
f32 row metadata are bit-identical to the reference for fp32-representable
input and the same stream key.  Differences, by design:

* the device computes on fp32 rows (float64 input is rounded to fp32 first);
* ``dequantize_rows`` returns ``f32(scale*code + min)`` evaluated in f64 — the
  reference's f64 value rounded once to fp32 — promoted back to float64;
* the passthrough (bits=32) wire carries fp32 rows (the accounting basis of
  ``codec.py:110-114``); the host-facing ``quantize_rows(..., QuantConfig(32))``
  keeps the reference's exact f64 payload since it involves no arithmetic.

The trainer does not use these host-facing functions: it drives the same
kernels on device-resident buffers through :mod:`.transport`.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .rngstream import RngStream

_HEADER = struct.Struct("<BBHII")
HEADER_BYTES = _HEADER.size
WIRE_VERSION = 1
VALID_BITS = frozenset(range(1, 9)) | {16, 32}


class CodecError(ValueError):
    pass


@dataclass(frozen=True)
class QuantConfig:
    bits: int = 1

    def __post_init__(self):
        if self.bits not in VALID_BITS:
            raise CodecError(f"unsupported bit width {self.bits}")

    @property
    def passthrough(self) -> bool:
        return self.bits == 32

    @property
    def bins(self) -> int:
        if self.passthrough:
            raise CodecError("passthrough mode has no quantization bins")
        return (1 << self.bits) - 1


def row_bytes(d: int, b: int) -> int:
    return (d * b + 7) // 8


def payload_bytes(rows: int, d: int, b: int) -> int:
    """Main-data bytes (fp32 basis for the passthrough) — codec.py:110-114."""
    return rows * d * 4 if b == 32 else rows * row_bytes(d, b)


def metadata_bytes(rows: int, b: int = 1) -> int:
    """codec.py:117-121."""
    return 0 if b == 32 else rows * 8


def wire_bytes(rows: int, d: int, b: int) -> int:
    """Bytes of one device wire block (header + meta + payload)."""
    return HEADER_BYTES + (4 * rows * d if b == 32 else 8 * rows + rows * row_bytes(d, b))


@dataclass(frozen=True)
class QuantizedBlock:
    num_rows: int
    dim: int
    bits: int
    payload: bytes
    row_min: np.ndarray
    row_scale: np.ndarray

    def to_bytes(self) -> bytes:
        head = _HEADER.pack(WIRE_VERSION, self.bits, 0, self.num_rows, self.dim)
        if self.bits == 32:
            return head + self.payload
        meta = np.empty((self.num_rows, 2), dtype="<f4")
        meta[:, 0] = self.row_min
        meta[:, 1] = self.row_scale
        return head + meta.tobytes() + self.payload

    @classmethod
    def from_bytes(cls, raw: bytes) -> "QuantizedBlock":
        if len(raw) < HEADER_BYTES:
            raise CodecError("truncated block header")
        version, bits, _, rows, dim = _HEADER.unpack_from(raw)
        if version != WIRE_VERSION:
            raise CodecError(f"unsupported wire version {version}")
        if bits == 32:
            blk = cls(rows, dim, bits, raw[HEADER_BYTES:], np.empty(0, np.float32),
                      np.empty(0, np.float32))
        else:
            end = HEADER_BYTES + 8 * rows
            meta = np.frombuffer(raw[HEADER_BYTES:end], dtype="<f4").reshape(rows, 2)
            blk = cls(rows, dim, bits, raw[end:], meta[:, 0].copy(), meta[:, 1].copy())
        blk.validate()
        return blk

    def validate(self):
        if self.bits == 32:
            ok = len(self.payload) in (self.num_rows * self.dim * 8, self.num_rows * self.dim * 4)
        else:
            ok = len(self.payload) == self.num_rows * row_bytes(self.dim, self.bits)
        if not ok:
            raise CodecError(f"payload length {len(self.payload)} does not match "
                             f"(rows={self.num_rows}, dim={self.dim}, bits={self.bits})")


# ---------------------------------------------------------------------------
# device entry points (torch tensors in, torch tensors out)

def segments_tensor(rows_list, keys, offsets, outs, device):
    """Pack hb_segment_t descriptors into a device uint8 tensor."""
    import torch
    n = len(rows_list)
    seg = np.zeros(n, dtype=_lib.SEGMENT_DTYPE)
    begin = 0
    for i in range(n):
        seg[i] = (keys[i][0], keys[i][1], offsets[i], outs[i], begin, rows_list[i])
        begin += rows_list[i]
    return torch.from_numpy(seg.view(np.uint8).copy()).to(device)


def quantize_gather(src, row_idx, segs, nseg: int, d: int, bits: int, flags, stream=None):
    """K1 on device buffers (see include/halob200.h: hb_quantize_gather)."""
    _lib.call("hb_quantize_gather", _lib.ptr(src), src.stride(0), _lib.ptr(row_idx),
              int(row_idx.numel()), _lib.ptr(segs), nseg, d, bits, _lib.ptr(flags),
              _lib.stream_handle(stream))


def dequant_gather(segs, nseg: int, dst_rows, src_ptr, src_rows, d: int, bits: int, dst,
                   accumulate: bool, stream=None):
    """K2 on device buffers (see include/halob200.h: hb_dequant_gather)."""
    _lib.call("hb_dequant_gather", _lib.ptr(segs), nseg, int(dst_rows.numel()), _lib.ptr(dst_rows),
              _lib.ptr(src_ptr), _lib.ptr(src_rows), d, bits, _lib.ptr(dst), dst.stride(0),
              int(bool(accumulate)), _lib.stream_handle(stream))


def _as_device_rows(m):
    import torch
    if isinstance(m, torch.Tensor):
        t = m.detach()
        if t.dim() == 1:
            t = t[None, :]
        return t.to(device="cuda", dtype=torch.float32).contiguous()
    a = np.atleast_2d(np.asarray(m))
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def quantize_rows(m, cfg: QuantConfig, rng: RngStream | None = None) -> QuantizedBlock:
    """Drop-in for ``halobit.codec.quantize_rows`` (codec.py:158-196), on the GPU."""
    import torch
    if cfg.passthrough and not isinstance(m, torch.Tensor):
        a = np.atleast_2d(np.asarray(m, dtype=np.float64))
        if not np.isfinite(a).all():
            raise CodecError("non-finite values in quantizer input")
        return QuantizedBlock(a.shape[0], a.shape[1], 32, np.ascontiguousarray(a).tobytes(),
                              np.empty(0, np.float32), np.empty(0, np.float32))
    if not cfg.passthrough and rng is None:
        raise CodecError("stochastic rounding requires an RngStream")
    x = _as_device_rows(m)
    rows, d = x.shape
    if rows == 0:
        return QuantizedBlock(0, d, cfg.bits, b"", np.empty(0, np.float32), np.empty(0, np.float32))
    nbytes = wire_bytes(rows, d, cfg.bits)
    out = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    if cfg.passthrough:
        key, off = (0, 0), 0
    else:
        key, off = rng.philox_key, rng.take(rows * d)
    segs = segments_tensor([rows], [key], [off], [out.data_ptr()], "cuda")
    idx = torch.arange(rows, dtype=torch.int32, device="cuda")
    quantize_gather(x, idx, segs, 1, d, cfg.bits, flags)
    if int(flags.item()) & _lib.HB_FLAG_NONFINITE:
        raise CodecError("non-finite values in quantizer input")
    raw = out.cpu().numpy().tobytes()
    return QuantizedBlock.from_bytes(raw)


def dequantize_rows(q: QuantizedBlock) -> np.ndarray:
    """Drop-in for ``halobit.codec.dequantize_rows`` (codec.py:199-207), on the GPU."""
    import torch
    q.validate()
    if q.num_rows == 0:
        return np.zeros((0, q.dim))
    if q.bits == 32 and len(q.payload) == q.num_rows * q.dim * 8:
        return np.frombuffer(q.payload, dtype=np.float64).reshape(q.num_rows, q.dim).copy()
    raw = q.to_bytes()
    buf = torch.from_numpy(np.frombuffer(raw, dtype=np.uint8).copy()).cuda()
    segs = segments_tensor([q.num_rows], [(0, 0)], [0], [buf.data_ptr()], "cuda")
    dst = torch.empty((q.num_rows, q.dim), dtype=torch.float32, device="cuda")
    rows = torch.arange(q.num_rows, dtype=torch.int32, device="cuda")
    ptr = torch.arange(q.num_rows + 1, dtype=torch.int32, device="cuda")
    dequant_gather(segs, 1, rows, ptr, rows, q.dim, q.bits, dst, accumulate=False)
    return dst.cpu().numpy().astype(np.float64)


def philox_uniforms(key, start: int, n: int):
    """Device uniforms of stream elements [start, start+n) (f64 tensor)."""
    import torch
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.call("hb_philox_uniforms", int(key[0]), int(key[1]), int(start), int(n), _lib.ptr(out),
              _lib.stream_handle())
    return out
