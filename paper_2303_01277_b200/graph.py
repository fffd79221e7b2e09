"""Graph, adjacency normalisation and partitioning (host side, run once).

Drop-in for ``halobit.graph`` (reference ``graph.py:28-256``): same types,
same fields, same index-map semantics, but vectorised (numpy/scipy) so the
BASELINE shapes (233k nodes / 114M edges, 2.4M nodes / 62M edges) build in
seconds instead of the reference's per-node Python loops
(``graph.py:163-164, 179-196, 245-246``).  Index maps are proven identical to
the reference's on its own fixtures (``tests/test_graph.py``).

The partition is the *input contract* of the device halo path: the send sets
``S_k``, the receive slots ``R_k`` and the block's column order (local rows
first, then halo rows, each sorted by global id — ``graph.py:218-229``) decide
which rows are quantized, in which order the Philox stream is consumed and
where received rows land.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
from scipy.sparse import csgraph

from ._np import sorted_unique
from .linalg import CsrMatrix

STRATEGIES = ("contiguous", "bfs_blocks", "hash")


class GraphConfigError(ValueError):
    pass


@dataclass
class Graph:
    """``graph.py:28-53``.  ``features`` may be float32 for large graphs."""

    num_nodes: int
    edges: np.ndarray
    features: np.ndarray
    labels: np.ndarray
    train_mask: np.ndarray
    val_mask: np.ndarray
    test_mask: np.ndarray
    num_classes: int = 0

    def __post_init__(self):
        if self.edges.size and self.edges.max() >= self.num_nodes:
            raise GraphConfigError("edge endpoint out of range")
        if self.features.shape[0] != self.num_nodes:
            raise GraphConfigError("feature row count mismatch")
        tv, tt, vt = (self.train_mask & self.val_mask, self.train_mask & self.test_mask,
                      self.val_mask & self.test_mask)
        if tv.any() or tt.any() or vt.any():
            raise GraphConfigError("masks must be disjoint")
        if self.num_classes == 0:
            self.num_classes = int(self.labels.max()) + 1 if self.num_nodes else 0

    @property
    def feature_dim(self) -> int:
        return self.features.shape[1]


@dataclass(frozen=True)
class PartitionPlan:
    """``graph.py:56-67``."""

    num_partitions: int
    assignment: np.ndarray

    def __post_init__(self):
        counts = np.bincount(self.assignment, minlength=self.num_partitions)
        if len(counts) > self.num_partitions or np.any(counts == 0):
            raise GraphConfigError("every partition must own at least one node")

    def nodes_of(self, part: int) -> np.ndarray:
        return np.flatnonzero(self.assignment == part)


@dataclass
class Partition:
    """``graph.py:70-100``: one worker's local rows, halo and peer index maps."""

    id: int
    num_partitions: int
    local_nodes: np.ndarray
    halo_nodes: np.ndarray
    send_sets: list
    recv_sets: list
    adj_block: CsrMatrix
    mean_block: CsrMatrix | None
    features: np.ndarray
    labels: np.ndarray
    train_mask: np.ndarray
    val_mask: np.ndarray
    test_mask: np.ndarray

    @property
    def num_local(self) -> int:
        return len(self.local_nodes)

    @property
    def num_halo(self) -> int:
        return len(self.halo_nodes)

    def send_global_ids(self, peer: int) -> np.ndarray:
        return self.local_nodes[self.send_sets[peer]]

    def recv_global_ids(self, peer: int) -> np.ndarray:
        return self.halo_nodes[self.recv_sets[peer]]


def clean_edges(g: Graph) -> np.ndarray:
    """Drop input self-loops and duplicates, sorted by (src, dst)
    (``graph.py:103-109``), via a 1-D int64 key instead of ``unique(axis=0)``."""
    e = np.asarray(g.edges, dtype=np.int64).reshape(-1, 2)
    if e.size == 0:
        return e.reshape(0, 2)
    key = e[:, 0] * np.int64(g.num_nodes) + e[:, 1]
    if len(key) > 1 and np.all(key[1:] > key[:-1]) and not np.any(e[:, 0] == e[:, 1]):
        return e  # already sorted, unique and loop-free (the generators emit this form)
    e = e[e[:, 0] != e[:, 1]]
    key = sorted_unique(e[:, 0] * np.int64(g.num_nodes) + e[:, 1])
    return np.stack([key // g.num_nodes, key % g.num_nodes], axis=1)


def _adjacency_csr(g: Graph) -> sp.csr_matrix:
    e = clean_edges(g)
    n = g.num_nodes
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(e[:, 0], minlength=n), out=rp[1:])
    return sp.csr_matrix((np.ones(len(e)), e[:, 1], rp), shape=(n, n))


def normalize_adjacency(g: Graph, degree_with_self_loops: bool = True) -> CsrMatrix:
    """D^-1/2 (A + I) D^-1/2 (``graph.py:120-132``).  Entry (i, j) is
    ``dinv[i] * dinv[j]`` — one f64 rounding, the value the reference's
    diagonal scalings produce."""
    a = _adjacency_csr(g)
    n = g.num_nodes
    cnt = np.diff(a.indptr)
    deg = cnt.astype(np.float64)
    if degree_with_self_loops:
        deg = deg + 1.0
    deg[deg == 0] = 1.0
    dinv = 1.0 / np.sqrt(deg)
    # insert the diagonal into every (column-sorted) row in O(nnz)
    rows = np.repeat(np.arange(n, dtype=np.int64), cnt)
    cols = a.indices.astype(np.int64)
    after = cols > rows
    pos = np.arange(len(cols), dtype=np.int64) + rows + after
    below = np.bincount(rows, weights=~after, minlength=n).astype(np.int64)
    dpos = a.indptr[:-1].astype(np.int64) + np.arange(n, dtype=np.int64) + below
    nnz = len(cols) + n
    ci = np.empty(nnz, dtype=np.int64)
    v = np.empty(nnz, dtype=np.float64)
    ci[pos] = cols
    v[pos] = dinv[rows] * dinv[cols]
    ci[dpos] = np.arange(n)
    v[dpos] = dinv * dinv
    rp = a.indptr.astype(np.int64) + np.arange(n + 1, dtype=np.int64)
    return CsrMatrix(n, n, rp, ci, v, validate=False)


def mean_adjacency(g: Graph) -> CsrMatrix:
    """D^-1 A, isolated rows all-zero (``graph.py:135-141``)."""
    a = _adjacency_csr(g)
    deg = np.diff(a.indptr).astype(np.float64)
    deg[deg == 0] = 1.0
    inv = 1.0 / deg
    rows = np.repeat(np.arange(g.num_nodes), np.diff(a.indptr))
    return CsrMatrix(g.num_nodes, g.num_nodes, a.indptr.astype(np.int64),
                     a.indices.astype(np.int64), inv[rows] * 1.0, validate=False)


def _hash_node(seed: int, node: int, n_parts: int) -> int:
    dig = hashlib.blake2b(f"{seed}:{node}".encode(), digest_size=8).digest()
    return int.from_bytes(dig, "little") % n_parts


def _bfs_order(g: Graph, start: int) -> np.ndarray:
    """Level-synchronous BFS with sorted adjacency, restarting from the smallest
    unseen node (``graph.py:176-202``) — FIFO order equals level order."""
    e = clean_edges(g)
    n = g.num_nodes
    if e.size:
        both = np.concatenate([e, e[:, ::-1]])
        a = sp.csr_matrix((np.ones(len(both)), (both[:, 0], both[:, 1])), shape=(n, n))
        a.sum_duplicates()
        a.sort_indices()
    else:
        a = sp.csr_matrix((n, n))
    seen = np.zeros(n, dtype=bool)
    out = []
    nxt = start
    while True:
        order = csgraph.breadth_first_order(a, nxt, directed=True, return_predecessors=False)
        out.append(order)
        seen[order] = True
        rest = np.flatnonzero(~seen)
        if rest.size == 0:
            break
        nxt = int(rest[0])
    return np.concatenate(out).astype(np.int64)


def partition_nodes(g: Graph, n: int, strategy: str = "contiguous", seed: int = 0) -> PartitionPlan:
    """``graph.py:149-173``: contiguous / bfs_blocks / hash."""
    if n < 1 or n > g.num_nodes:
        raise GraphConfigError(f"cannot split {g.num_nodes} nodes into {n} partitions")
    if strategy not in STRATEGIES:
        raise GraphConfigError(f"unknown strategy {strategy!r}")
    if strategy == "hash":
        assign = np.array([_hash_node(seed, v, n) for v in range(g.num_nodes)], dtype=np.int64)
        return PartitionPlan(n, assign)
    order = np.arange(g.num_nodes) if strategy == "contiguous" else \
        _bfs_order(g, seed % g.num_nodes)
    bounds = np.linspace(0, g.num_nodes, n + 1).astype(int)
    assign = np.zeros(g.num_nodes, dtype=np.int64)
    for p in range(n):
        assign[order[bounds[p]:bounds[p + 1]]] = p
    return PartitionPlan(n, assign)


def _row_slice(a: CsrMatrix, rows: np.ndarray):
    """COO (row-in-slice, col, val) of ``a[rows]`` without scipy fancy indexing."""
    rp = a.row_ptr
    cnt = rp[rows + 1] - rp[rows]
    starts = np.repeat(rp[rows] - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt)
    idx = starts + np.arange(cnt.sum(), dtype=np.int64)
    return np.repeat(np.arange(len(rows), dtype=np.int64), cnt), a.col_idx[idx], a.values[idx]


def build_partition(g: Graph, a_hat: CsrMatrix, plan: PartitionPlan, n: int,
                    mean_hat: CsrMatrix | None = None) -> Partition:
    """``graph.py:205-256``, vectorised.

    * halo = sorted global ids adjacent (in Â) to a local node, minus locals;
    * block columns: local first, then halo, each sorted by global id;
    * ``recv_sets[k]`` = ascending halo slots owned by k;
    * ``send_sets[k]`` = ascending local rows with >= 1 Â-neighbour owned by k.
    """
    local = np.sort(plan.nodes_of(n))
    owner = plan.assignment
    nl = len(local)
    contiguous = nl > 0 and local[-1] - local[0] + 1 == nl
    if contiguous:
        lo = int(local[0])
        k0, k1 = int(a_hat.row_ptr[lo]), int(a_hat.row_ptr[lo + nl])
        rp_loc = a_hat.row_ptr[lo:lo + nl + 1] - k0
        r = np.repeat(np.arange(nl, dtype=np.int64), np.diff(rp_loc))
        c, v = a_hat.col_idx[k0:k1], a_hat.values[k0:k1]
        is_local = (c >= lo) & (c < lo + nl)
    else:
        r, c, v = _row_slice(a_hat, local)
        is_local = owner[c] == n
    halo = sorted_unique(c[~is_local])
    ncols = nl + len(halo)

    def block(rr, cc, vv, loc):
        """Columns local-first then halo, each sorted by global id: within a
        row of a column-sorted matrix that is a stable local/halo partition."""
        if contiguous:
            newc = np.where(loc, cc - lo, nl + np.searchsorted(halo, cc))
        else:
            cmap = np.full(g.num_nodes, -1, dtype=np.int64)
            cmap[local] = np.arange(nl)
            cmap[halo] = nl + np.arange(len(halo))
            newc = cmap[cc]
        cnt = np.bincount(rr, minlength=nl)
        rp = np.zeros(nl + 1, dtype=np.int64)
        np.cumsum(cnt, out=rp[1:])
        nloc = np.bincount(rr, weights=loc, minlength=nl).astype(np.int64)
        cl = np.cumsum(loc) - loc                       # locals before this entry (global)
        ch = np.cumsum(~loc) - (~loc)                   # halos before this entry (global)
        start = rp[:-1][rr]
        cl0 = np.concatenate([[0], np.cumsum(nloc)])[rr]
        ch0 = (rp[:-1] - np.concatenate([[0], np.cumsum(nloc)[:-1]]))[rr]
        pos = np.where(loc, start + (cl - cl0), start + nloc[rr] + (ch - ch0))
        ci = np.empty(len(cc), dtype=np.int64)
        vo = np.empty(len(cc), dtype=np.float64)
        ci[pos] = newc
        vo[pos] = vv
        return CsrMatrix(nl, ncols, rp, ci, vo, validate=False)

    adj_block = block(r, c, v, is_local)
    mean_block = None
    if mean_hat is not None:
        if contiguous:
            m0, m1 = int(mean_hat.row_ptr[lo]), int(mean_hat.row_ptr[lo + nl])
            mrp = mean_hat.row_ptr[lo:lo + nl + 1] - m0
            mr = np.repeat(np.arange(nl, dtype=np.int64), np.diff(mrp))
            mc, mv = mean_hat.col_idx[m0:m1], mean_hat.values[m0:m1]
            mloc = (mc >= lo) & (mc < lo + nl)
        else:
            mr, mc, mv = _row_slice(mean_hat, local)
            mloc = owner[mc] == n
        mean_block = block(mr, mc, mv, mloc)

    recv_sets, send_sets = [], []
    halo_owner = owner[halo]
    # S_k: local rows with >= 1 neighbour owned by k (graph.py:238-247), from the
    # halo entries only: unique (owner, row) keys, already ordered by row per owner
    hr, hc = r[~is_local], c[~is_local]
    keys = sorted_unique(owner[hc] * np.int64(max(nl, 1)) + hr)
    kown, krow = keys // max(nl, 1), keys % max(nl, 1)
    bounds = np.searchsorted(kown, np.arange(plan.num_partitions + 1))
    for k in range(plan.num_partitions):
        if k == n:
            recv_sets.append(np.empty(0, dtype=np.int64))
            send_sets.append(np.empty(0, dtype=np.int64))
            continue
        recv_sets.append(np.flatnonzero(halo_owner == k).astype(np.int64))
        send_sets.append(krow[bounds[k]:bounds[k + 1]].astype(np.int64))

    return Partition(
        id=n, num_partitions=plan.num_partitions, local_nodes=local, halo_nodes=halo,
        send_sets=send_sets, recv_sets=recv_sets, adj_block=adj_block, mean_block=mean_block,
        features=g.features[local], labels=g.labels[local], train_mask=g.train_mask[local],
        val_mask=g.val_mask[local], test_mask=g.test_mask[local])


def build_partitions(g: Graph, n: int, strategy: str = "contiguous", seed: int = 0,
                     model: str = "gcn", degree_with_self_loops: bool = True):
    """Convenience: Â (and M for SAGE), plan and all partitions."""
    a_hat = normalize_adjacency(g, degree_with_self_loops)
    mean_hat = mean_adjacency(g) if model == "sage" else None
    plan = partition_nodes(g, n, strategy, seed)
    return a_hat, mean_hat, [build_partition(g, a_hat, plan, k, mean_hat) for k in range(n)]
