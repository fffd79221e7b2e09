"""Vectorised graph/partition code vs the reference's outputs (CPU only)."""

import hashlib

import numpy as np
import pytest

from conftest import load_json, load_npz
from paper_2303_01277_b200.datasets import CONFIG1, PlantedSpec, generate_planted, generate_sbm
from paper_2303_01277_b200.graph import (Graph, GraphConfigError, PartitionPlan, build_partition,
                                         mean_adjacency, normalize_adjacency, partition_nodes)
from paper_2303_01277_b200.linalg import CsrMatrix, ShapeError


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def small_graph():
    z = load_npz("graph_small.npz")
    return z, Graph(num_nodes=len(z["labels"]), edges=z["edges"], features=z["features"],
                    labels=z["labels"], train_mask=z["train"], val_mask=z["val"],
                    test_mask=z["test"])


def split_csr(flat, rows):
    rp = flat[:rows + 1].astype(np.int64)
    nnz = int(rp[-1])
    return rp, flat[rows + 1:rows + 1 + nnz].astype(np.int64), flat[rows + 1 + nnz:]


def test_small_adjacencies_identical():
    z, g = small_graph()
    n = g.num_nodes
    for name, got in (("ahat", normalize_adjacency(g)), ("mean", mean_adjacency(g))):
        rp, ci, v = split_csr(z[name], n)
        np.testing.assert_array_equal(got.row_ptr, rp)
        np.testing.assert_array_equal(got.col_idx, ci)
        np.testing.assert_array_equal(got.values, v)


@pytest.mark.parametrize("strategy", ["contiguous", "bfs_blocks", "hash"])
def test_partitions_identical_to_reference(strategy):
    z, g = small_graph()
    a, mh = normalize_adjacency(g), mean_adjacency(g)
    plan = partition_nodes(g, 3, strategy, 5)
    np.testing.assert_array_equal(plan.assignment, z[f"{strategy}_assign"])
    for k in range(3):
        p = build_partition(g, a, plan, k, mh)
        pre = f"{strategy}_{k}_"
        np.testing.assert_array_equal(p.local_nodes, z[pre + "local"])
        np.testing.assert_array_equal(p.halo_nodes, z[pre + "halo"])
        for j in range(3):
            np.testing.assert_array_equal(p.send_sets[j], z[pre + f"send{j}"])
            np.testing.assert_array_equal(p.recv_sets[j], z[pre + f"recv{j}"])
        for blk, key in ((p.adj_block, "A"), (p.mean_block, "M")):
            rp, ci, v = split_csr(z[pre + key], p.num_local)
            np.testing.assert_array_equal(blk.row_ptr, rp)
            np.testing.assert_array_equal(blk.col_idx, ci)
            np.testing.assert_array_equal(blk.values, v)


def test_config1_graph_and_partitions_identical():
    info = load_json("graph_hashes.json")
    g = generate_sbm(CONFIG1)
    c = info["config1_sbm"]
    assert sha(g.edges) == c["edges"] and sha(g.features) == c["features"]
    assert sha(g.labels) == c["labels"]
    assert sha(g.train_mask, g.val_mask, g.test_mask) == c["masks"]
    a = normalize_adjacency(g)
    assert sha(a.row_ptr, a.col_idx, a.values) == info["config1_ahat"]
    plan = partition_nodes(g, 2)
    for k, want in enumerate(info["config1_parts"]):
        p = build_partition(g, a, plan, k)
        assert sha(p.halo_nodes) == want["halo"]
        assert [sha(s) for s in p.send_sets] == want["send"]
        assert [sha(r) for r in p.recv_sets] == want["recv"]
        assert sha(p.adj_block.row_ptr, p.adj_block.col_idx, p.adj_block.values) == want["block"]


def test_send_recv_identity_on_planted_graph():
    g = generate_planted(PlantedSpec(num_nodes=3000, num_edges=60000, feature_dim=16,
                                     num_classes=5, cut=0.05, seed=3))
    assert abs(len(g.edges) - 60000) <= 2
    a = normalize_adjacency(g)
    plan = partition_nodes(g, 4)
    parts = [build_partition(g, a, plan, k) for k in range(4)]
    for n in range(4):
        slots = np.concatenate([parts[n].recv_sets[k] for k in range(4)])
        np.testing.assert_array_equal(np.sort(slots), np.arange(parts[n].num_halo))
        for k in range(4):
            if k != n:
                np.testing.assert_array_equal(parts[n].send_global_ids(k),
                                              parts[k].recv_global_ids(n))


def test_csr_validation_and_transpose():
    with pytest.raises(ShapeError):
        CsrMatrix(1, 2, np.array([0, 2]), np.array([0, 0]), np.array([1.0, 1.0]))
    with pytest.raises(ShapeError):
        CsrMatrix(1, 2, np.array([0, 1]), np.array([5]), np.array([1.0]))
    rng = np.random.default_rng(2)
    dense = (rng.random((6, 4)) < 0.4) * rng.standard_normal((6, 4))
    import scipy.sparse as sp
    m = CsrMatrix.from_scipy(sp.csr_matrix(dense))
    np.testing.assert_array_equal(m.transpose().to_dense(), dense.T)


def test_partition_errors():
    g = Graph(3, np.zeros((0, 2), dtype=np.int64), np.eye(3), np.zeros(3, dtype=np.int64),
              np.ones(3, bool), np.zeros(3, bool), np.zeros(3, bool))
    with pytest.raises(GraphConfigError):
        partition_nodes(g, 4)
    with pytest.raises(GraphConfigError):
        partition_nodes(g, 2, "metis")
    with pytest.raises(GraphConfigError):
        PartitionPlan(3, np.array([0, 0, 1, 1]))
