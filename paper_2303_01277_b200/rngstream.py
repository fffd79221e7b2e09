"""Keyed Philox streams (reference ``rngstream.py:1-45``).

The host only derives the 128-bit key (blake2b of the structural key tuple,
``rngstream.py:19-23``); the uniforms themselves are generated on the device
inside the quantize kernel (Philox4x64-10, counter ``i//4 + 1``, word
``i % 4``, ``(w >> 11) * 2^-53`` — numpy's ``Philox`` + ``Generator.random``).

``RngStream`` keeps the reference's single-owner semantics: it hands out
contiguous element ranges (``take``), so several blocks quantized from one
stream continue where the previous block stopped, exactly like repeated
``uniforms(n)`` calls (``transport.py:184-188``).
"""

from __future__ import annotations

import hashlib

import numpy as np

FORWARD = "forward"
BACKWARD = "backward"


def derive_key(parts: tuple) -> tuple:
    """Two little-endian uint64 words of blake2b-128 over the joined key."""
    text = "\x1f".join(str(p) for p in parts).encode()
    dig = hashlib.blake2b(text, digest_size=16).digest()
    return int.from_bytes(dig[:8], "little"), int.from_bytes(dig[8:], "little")


class RngStream:
    """Single-owner uniform stream for one (partition, epoch, layer, phase)."""

    def __init__(self, global_seed: int, partition: int, epoch: int, layer: int, phase: str):
        self.key = (global_seed, partition, epoch, layer, phase)
        self.philox_key = derive_key(self.key)
        self.offset = 0

    def take(self, n: int) -> int:
        """Reserve the next ``n`` elements; returns their starting index."""
        start = self.offset
        self.offset += int(n)
        return start

    def uniforms(self, n: int) -> np.ndarray:
        """Host copy of the next ``n`` uniforms (host-side tests/tools only;
        the device path never materialises them)."""
        start = self.take(n)
        gen = np.random.Generator(np.random.Philox(key=np.array(self.philox_key, dtype=np.uint64)))
        if start:
            gen.random(start)
        return gen.random(n)


def keyed_generator(*parts) -> np.random.Generator:
    """Host generator for init / dataset synthesis (``rngstream.py:42-45``)."""
    return np.random.Generator(np.random.Philox(key=np.array(derive_key(tuple(parts)),
                                                             dtype=np.uint64)))
