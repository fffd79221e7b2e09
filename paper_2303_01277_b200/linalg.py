"""Sparse container + device numerics entry points.

``CsrMatrix`` mirrors ``halobit.linalg.CsrMatrix`` (reference
``linalg.py:20-62``): same fields (int64 ``row_ptr``/``col_idx``, float64
``values``), same invariants, but the validation is vectorised (the reference
checks column order with a per-row Python loop, ``linalg.py:36-39``).

The device-side products (``spmm``, ``softmax_cross_entropy``, ``adam_step``,
...) live in :mod:`paper_2303_01277_b200.ops` and run through the C-ABI
library; there is no host fallback.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp


class ShapeError(ValueError):
    pass


@dataclass(frozen=True)
class CsrMatrix:
    rows: int
    cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    validate: bool = field(default=True, repr=False, compare=False)

    def __post_init__(self):
        if not self.validate:
            return
        rp, ci, v = self.row_ptr, self.col_idx, self.values
        if len(rp) != self.rows + 1 or rp[-1] != len(ci) or len(ci) != len(v):
            raise ShapeError("inconsistent CSR arrays")
        if np.any(np.diff(rp) < 0):
            raise ShapeError("row_ptr must be nondecreasing")
        if len(ci) and (ci.min() < 0 or ci.max() >= self.cols):
            raise ShapeError("column index out of range")
        if len(ci) > 1:
            step = np.diff(ci)
            row_start = np.zeros(len(ci), dtype=bool)
            row_start[rp[:-1][rp[:-1] < len(ci)]] = True
            if np.any((step <= 0) & ~row_start[1:]):
                raise ShapeError("columns not strictly increasing within a row")

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @classmethod
    def from_scipy(cls, a) -> "CsrMatrix":
        a = sp.csr_matrix(a)
        a.sort_indices()
        a.sum_duplicates()
        return cls(a.shape[0], a.shape[1], a.indptr.astype(np.int64),
                   a.indices.astype(np.int64), a.data.astype(np.float64))

    def to_scipy(self) -> sp.csr_matrix:
        return sp.csr_matrix((self.values, self.col_idx, self.row_ptr),
                             shape=(self.rows, self.cols))

    @classmethod
    def identity(cls, n: int) -> "CsrMatrix":
        return cls.from_scipy(sp.identity(n, format="csr"))

    def to_dense(self) -> np.ndarray:
        return self.to_scipy().toarray()

    def transpose(self) -> "CsrMatrix":
        """CSR of the transpose (stable: rows of A^T keep ascending columns)."""
        n = self.rows
        r = np.repeat(np.arange(n, dtype=np.int64), np.diff(self.row_ptr))
        o = np.argsort(self.col_idx, kind="stable")
        rp = np.zeros(self.cols + 1, dtype=np.int64)
        np.cumsum(np.bincount(self.col_idx, minlength=self.cols), out=rp[1:])
        return CsrMatrix(self.cols, n, rp, r[o], self.values[o], validate=False)
