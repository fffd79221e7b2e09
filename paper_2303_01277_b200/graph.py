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
    e = e[e[:, 0] != e[:, 1]]
    key = np.unique(e[:, 0] * np.int64(g.num_nodes) + e[:, 1])
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
    deg = np.diff(a.indptr).astype(np.float64)
    if degree_with_self_loops:
        deg = deg + 1.0
    deg[deg == 0] = 1.0
    dinv = 1.0 / np.sqrt(deg)
    # insert the diagonal into every row, keeping columns sorted
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(a.indptr))
    cols = a.indices.astype(np.int64)
    key = np.concatenate([rows * n + cols, np.arange(n, dtype=np.int64) * (n + 1)])
    key.sort()
    r, c = key // n, key % n
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=rp[1:])
    return CsrMatrix(n, n, rp, c, dinv[r] * dinv[c], validate=False)


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
    r, c, v = _row_slice(a_hat, local)
    is_local = owner[c] == n
    halo = np.unique(c[~is_local])
    col_map = np.full(g.num_nodes, -1, dtype=np.int64)
    col_map[local] = np.arange(len(local))
    col_map[halo] = len(local) + np.arange(len(halo))
    ncols = len(local) + len(halo)

    def block(rr, cc, vv):
        newc = col_map[cc]
        key = rr * ncols + newc
        o = np.argsort(key, kind="stable")
        rp = np.zeros(len(local) + 1, dtype=np.int64)
        np.cumsum(np.bincount(rr, minlength=len(local)), out=rp[1:])
        return CsrMatrix(len(local), ncols, rp, newc[o], vv[o], validate=False)

    adj_block = block(r, c, v)
    mean_block = None
    if mean_hat is not None:
        mr, mc, mv = _row_slice(mean_hat, local)
        keep = col_map[mc] >= 0
        mean_block = block(mr[keep], mc[keep], mv[keep])

    recv_sets, send_sets = [], []
    halo_owner = owner[halo]
    c_owner = owner[c]
    for k in range(plan.num_partitions):
        if k == n:
            recv_sets.append(np.empty(0, dtype=np.int64))
            send_sets.append(np.empty(0, dtype=np.int64))
            continue
        recv_sets.append(np.flatnonzero(halo_owner == k).astype(np.int64))
        send_sets.append(np.unique(r[c_owner == k]).astype(np.int64))

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
