"""Oracle: keyed Philox4x64-10 uniform streams (TEST INFRASTRUCTURE ONLY).

Reference: ``halobit/rngstream.py``
* ``_derive_key`` (rngstream.py:19-23): blake2b-128 over the unit-separator
  joined ``str()`` of the key parts; the 16 digest bytes are two little-endian
  uint64 words = the Philox key.
* ``RngStream.uniforms`` (rngstream.py:38-39) draws ``Generator.random(n)``
  from ``np.random.Philox(key=...)`` (numpy, third-party, pinned ``numpy>=1.24``
  by ``pkg/pyproject.toml:10-13``; numpy 2.3.5 here).

numpy's Philox (Random123 Philox4x64-10) increments its 256-bit counter before
each block, so block ``j`` (0-based) is ``philox(ctr=[j+1,0,0,0], key)`` and
yields 4 uint64 words consumed in order; ``Generator.random`` maps a word ``w``
to ``(w >> 11) * 2**-53``.  Hence element ``i`` of a stream is
``philox([i//4 + 1, 0, 0, 0], key)[i % 4] >> 11`` scaled by ``2**-53``.

``philox4x64_10`` below is a from-scratch numpy restatement of that block
function (the formula the CUDA kernel implements); ``stream_uniforms`` uses
numpy's own Philox (the reference's exact dependency) for speed.  Both are
checked against each other and against the golden vectors.
"""

from __future__ import annotations

import hashlib

import numpy as np

M0 = np.uint64(0xD2E7470EE14C6C93)
M1 = np.uint64(0xCA5A826395121157)
W0 = np.uint64(0x9E3779B97F4A7C15)
W1 = np.uint64(0xBB67AE8584CAA73B)
_MASK32 = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def derive_key(parts) -> tuple:
    """(k0, k1) uint64 Philox key for a structural key tuple.

    Follows rngstream.py:19-23 (``"\\x1f".join(str(p))`` → blake2b, 16 bytes,
    read as two little-endian uint64).
    """
    text = "\x1f".join(str(p) for p in parts).encode()
    dig = hashlib.blake2b(text, digest_size=16).digest()
    return int.from_bytes(dig[:8], "little"), int.from_bytes(dig[8:], "little")


def _mulhilo(a: np.uint64, b: np.ndarray):
    """128-bit product of uint64 ``a`` (scalar) and array ``b`` → (hi, lo)."""
    b = b.astype(np.uint64)
    al, ah = a & _MASK32, a >> _S32
    bl, bh = b & _MASK32, b >> _S32
    p0 = al * bl
    p1 = al * bh
    p2 = ah * bl
    p3 = ah * bh
    mid = (p0 >> _S32) + (p1 & _MASK32) + (p2 & _MASK32)
    lo = (p0 & _MASK32) | ((mid & _MASK32) << _S32)
    hi = p3 + (p1 >> _S32) + (p2 >> _S32) + (mid >> _S32)
    return hi, lo


def philox4x64_10(ctr0: np.ndarray, key) -> np.ndarray:
    """Philox4x64-10 block for counters ``[ctr0, 0, 0, 0]`` → (n, 4) uint64."""
    with np.errstate(over="ignore"):
        c0 = np.asarray(ctr0, dtype=np.uint64)
        c1 = np.zeros_like(c0)
        c2 = np.zeros_like(c0)
        c3 = np.zeros_like(c0)
        k0, k1 = np.uint64(key[0]), np.uint64(key[1])
        for r in range(10):
            if r:
                k0 = k0 + W0
                k1 = k1 + W1
            hi0, lo0 = _mulhilo(M0, c0)
            hi1, lo1 = _mulhilo(M1, c2)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return np.stack([c0, c1, c2, c3], axis=1)


def uniforms_restated(key, start: int, n: int) -> np.ndarray:
    """Elements [start, start+n) of a stream via the restated block function."""
    if n == 0:
        return np.zeros(0)
    first, last = start // 4, (start + n - 1) // 4
    blocks = philox4x64_10(np.arange(first + 1, last + 2, dtype=np.uint64), key)
    words = blocks.reshape(-1)[start - 4 * first: start - 4 * first + n]
    return (words >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


class Stream:
    """One keyed stream consumed sequentially (rngstream.py:26-39)."""

    def __init__(self, *parts):
        self.key = derive_key(parts)
        self._gen = np.random.Generator(
            np.random.Philox(key=np.array(self.key, dtype=np.uint64)))
        self.consumed = 0

    def uniforms(self, n: int) -> np.ndarray:
        self.consumed += n
        return self._gen.random(n)


def keyed_generator(*parts) -> np.random.Generator:
    """rngstream.py:42-45 — used for weight init / dropout / SBM synthesis."""
    return np.random.Generator(
        np.random.Philox(key=np.array(derive_key(parts), dtype=np.uint64)))
