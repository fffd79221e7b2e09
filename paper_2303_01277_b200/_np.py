"""numpy helpers.  ``np.unique`` is pathologically slow on large int64 arrays in
this numpy build (hash path: 140 s for 57M keys vs 2 s sort+mask), so the
host-side graph code uses these sort-based equivalents."""

from __future__ import annotations

import numpy as np


def sorted_unique(a: np.ndarray) -> np.ndarray:
    """Equivalent of ``np.unique(a)`` for 1-D arrays."""
    a = np.sort(np.asarray(a).ravel())
    if a.size == 0:
        return a
    keep = np.empty(a.size, dtype=bool)
    keep[0] = True
    np.not_equal(a[1:], a[:-1], out=keep[1:])
    return a[keep]


def sorted_unique_index(a_sorted: np.ndarray):
    """(unique values, first index) of an already sorted 1-D array."""
    if a_sorted.size == 0:
        return a_sorted, np.zeros(0, dtype=np.int64)
    keep = np.empty(a_sorted.size, dtype=bool)
    keep[0] = True
    np.not_equal(a_sorted[1:], a_sorted[:-1], out=keep[1:])
    idx = np.flatnonzero(keep)
    return a_sorted[idx], idx


def setdiff_sorted(a_sorted_unique: np.ndarray, b_sorted_unique: np.ndarray) -> np.ndarray:
    """Elements of ``a`` not in ``b`` (both sorted & unique)."""
    if b_sorted_unique.size == 0 or a_sorted_unique.size == 0:
        return a_sorted_unique
    pos = np.searchsorted(b_sorted_unique, a_sorted_unique)
    pos = np.minimum(pos, b_sorted_unique.size - 1)
    return a_sorted_unique[b_sorted_unique[pos] != a_sorted_unique]
