"""Host-side planning logic (no GPU)."""

import numpy as np
import pytest


def test_agg_order_choice_reddit_shapes():
    """Reddit-shaped SAGE 602-256-256-41 (114.6M nnz, 8 partitions on one
    GPU: 233k local + 461k halo rows): the 41-wide output layer aggregates
    after the projection; equal widths keep the reference order."""
    from paper_2303_01277_b200.trainer import choose_agg_order
    nnz, nl, rows = 114_615_892, 232_965, 232_965 + 461_000
    assert choose_agg_order(3, 256, 41, nnz, nl, rows, "sage", "cublas") == "post"
    assert choose_agg_order(2, 256, 256, nnz, nl, rows, "sage", "cublas") == "pre"
    assert choose_agg_order(1, 602, 256, nnz, nl, rows, "sage", "cublas") == "pre"
    # widening layers never aggregate after the projection
    assert choose_agg_order(2, 100, 128, 62_000_000, 300_000, 500_000, "sage", "tcgen05") == "pre"


def test_agg_order_validation():
    from paper_2303_01277_b200.trainer import AGG_ORDERS
    assert AGG_ORDERS == ("pre", "post", "auto")


def test_agg_order_with_tcgen05_rates():
    """With the tcgen05 GEMM rate the 602->256 first layer also aggregates
    after the projection (the SpMM saving outweighs the extra GEMM rows)."""
    from paper_2303_01277_b200.trainer import choose_agg_order
    nnz, nl, rows = 114_615_892, 232_965, 232_965 + 461_000
    assert choose_agg_order(1, 602, 256, nnz, nl, rows, "sage", "tcgen05") == "post"
    assert choose_agg_order(3, 256, 41, nnz, nl, rows, "sage", "tcgen05") == "post"
    assert choose_agg_order(2, 256, 256, nnz, nl, rows, "sage", "tcgen05") == "pre"


def test_wire_accounting_matches_oracle():
    """codec byte accounting (codec.py:104-121) vs the oracle restatement."""
    from oracle import codec as oc
    from paper_2303_01277_b200.codec import HEADER_BYTES, metadata_bytes, payload_bytes, wire_bytes
    assert HEADER_BYTES == oc.HEADER_BYTES == 12
    for rows in (0, 1, 7, 1000):
        for d in (1, 3, 41, 64, 100, 602):
            for b in (1, 2, 3, 4, 8, 16, 32):
                assert payload_bytes(rows, d, b) == oc.payload_bytes(rows, d, b)
                assert metadata_bytes(rows, b) == oc.metadata_bytes(rows, b)
                assert wire_bytes(rows, d, b) == HEADER_BYTES + payload_bytes(rows, d, b) + metadata_bytes(rows, b)


def _small_parts(n=4, strategy="hash"):
    from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
    from paper_2303_01277_b200.graph import build_partitions
    g = generate_sbm(SbmSpec(nodes_per_community=30, communities=4, feature_dim=8, seed=4))
    return g, build_partitions(g, n, strategy, 0, "sage")[2]


@pytest.mark.parametrize("owner", [[0, 0, 0, 0], [0, 1, 0, 1], [0, 0, 1, 1]])
def test_exchange_buffer_layout(owner):
    """Receive/send buffers: every message 16-byte aligned and sized to its wire
    block, remote groups contiguous per peer rank, local deliveries inside
    the receive buffer, K1 stream offsets restart per sender and advance over
    non-empty peers in ascending order (transport.py:184-188)."""
    from paper_2303_01277_b200.codec import wire_bytes
    from paper_2303_01277_b200.transport import ExchangeBuffers, RankLayout
    _, parts = _small_parts()
    for rank in sorted(set(owner)):
        lay = RankLayout({p.id: p for p in parts if owner[p.id] == rank}, owner, rank)
        for plan in (lay.fwd, lay.bwd):
            for bits in (1, 32):
                b = ExchangeBuffers(lay, plan, 8, bits, "cpu", parities=2)
                for (s, d), off in b.recv_off.items():
                    assert off % 16 == 0
                for (s, d), off in b.send_off.items():
                    assert off % 16 == 0 and owner[d] != rank
                for r, (o, n) in b.send_group.items():
                    msgs = [m for m in plan.send_msgs if owner[m.dst] == r]
                    assert n >= sum(wire_bytes(m.rows, 8, bits) for m in msgs)
                last = {}
                for m in plan.send_msgs:
                    assert b.elem_off[(m.src, m.dst)] == last.get(m.src, 0)
                    last[m.src] = b.elem_off[(m.src, m.dst)] + m.rows * 8
                tab = b.send_table(3, 2, 1, 0)
                for i, m in enumerate(plan.send_msgs):
                    base = b.recv[0].data_ptr() if owner[m.dst] == rank else b.send.data_ptr()
                    assert int(tab["out"][i]) - base == (b.recv_off if owner[m.dst] == rank else b.send_off)[
                        (m.src, m.dst)]


def test_tiled_csr_decomposition_is_exact():
    """ops.TiledCsr (built with torch ops, here on CPU) splits the matrix into
    64x64 tiles + a residual CSR that together hold every nonzero exactly once,
    with per-tile record caps and row offsets consistent."""
    import numpy as np
    import scipy.sparse as sp
    import torch
    from paper_2303_01277_b200 import ops
    rng = np.random.default_rng(1)
    dense = np.zeros((300, 500), dtype=np.float32)
    dense[64:128, 128:192] = rng.standard_normal((64, 64))           # > MAXREC? no: 4096 > 1024 -> split
    mask = rng.random((300, 500)) < 0.08
    dense[mask] = rng.standard_normal(mask.sum())
    a = sp.csr_matrix(dense)
    A = ops.DeviceCsr(300, 500, a.indptr, a.indices, a.data, "cpu")
    T = ops.TiledCsr(A, threshold=20)
    rebuilt = np.zeros_like(dense)
    nz = T.tile_nz.numpy()
    ro = T.tile_rowoff.numpy().astype(np.int64) & 0xFFFF
    off = T.tile_off.numpy()
    tp = T.tile_ptr.numpy()
    for b in range(T.nblocks):
        for t in range(tp[b], tp[b + 1]):
            recs = nz[off[t]:off[t + 1]]
            assert ro[t, 64] <= 1024 and off[t] % 2 == 0
            for r in range(64):
                for k in range(ro[t, r], ro[t, r + 1]):
                    c = int(T.tile_win[t]) * 64 + recs[k, 0]
                    rebuilt[b * 64 + r, c] += recs[k, 1:2].view(np.float32)[0]
    rp, rc, rv = T.res_ptr.numpy(), T.res_col.numpy(), T.res_val.numpy()
    for r in range(300):
        for k in range(rp[r], rp[r + 1]):
            rebuilt[r, rc[k]] += rv[k]
    np.testing.assert_array_equal(rebuilt, dense)
    assert T.tiled_nnz + len(rc) == a.nnz
    assert T.ntiles > int((tp[1:] - tp[:-1] > 0).sum())                # the dense block was split


def _tile_dense(T):
    """Rebuild the dense matrix a TiledCsr describes (tiles + residual)."""
    import torch
    out = np.zeros((T.rows, T.cols))
    tp, win = T.tile_ptr.numpy(), T.tile_win.numpy()
    off, ro = T.tile_off.numpy(), T.tile_rowoff.numpy().astype(np.int64) & 0xFFFF
    rs = T.row_scale.double().numpy() if T.row_scale is not None else np.ones(T.rows)
    cs = T.col_scale.double().numpy() if T.col_scale is not None else np.ones(T.cols)
    for b in range(T.nblocks):
        for t in range(tp[b], tp[b + 1]):
            for lr in range(T.RB):
                r = b * T.RB + lr
                for k in range(ro[t, lr], ro[t, lr + 1]):
                    if T.binary:
                        assert ro[t, lr] % 4 == 0                 # row runs start on whole words
                        j = int(T.tile_nz[off[t] + k])
                        if j == 0xFF:                             # word padding: only at a run's end
                            assert all(int(T.tile_nz[off[t] + kk]) == 0xFF for kk in range(k, ro[t, lr + 1]))
                            break
                        c = win[t] * T.W + j
                        out[r, c] += rs[r] * cs[c]
                    else:
                        c = win[t] * T.W + int(T.tile_nz[off[t] + k, 0])
                        out[r, c] += float(T.tile_nz[off[t] + k, 1:2].view(torch.float32))
    rp, rc, rv = T.res_ptr.numpy(), T.res_col.numpy(), T.res_val.numpy()
    for r in range(T.rows):
        for k in range(rp[r], rp[r + 1]):
            out[r, rc[k]] += rs[r] * cs[rc[k]] if T.binary else rv[k]
    return out


@pytest.mark.parametrize("kind", ["general", "mean", "mean_T", "gcn"])
def test_tiled_layout_reconstructs_matrix(kind):
    """ops.TiledCsr (built with torch ops, no kernel) describes exactly the
    input matrix: 64-row / 8-byte-record tiles for general values, 128-row /
    one-byte-record tiles plus diagonal scalings for the trainer's operators
    (graph.py:120-141)."""
    import scipy.sparse as sp
    from paper_2303_01277_b200 import ops
    rng = np.random.default_rng(3)
    rows, cols = 300, 420
    pat = (rng.random((rows, cols)) < 0.01)
    pat[130:250, 64:128] |= rng.random((120, 64)) < 0.5
    pat = pat.astype(np.float64)
    if kind == "general":
        a = pat * rng.standard_normal(pat.shape)
    elif kind.startswith("mean"):
        a = pat / np.maximum(pat.sum(1), 1)[:, None]
        if kind == "mean_T":
            a = a.T.copy()
    else:
        np.fill_diagonal(pat, 1.0)
        dinv = 1 / np.sqrt(rng.integers(1, 50, cols))
        a = dinv[:rows, None] * pat * dinv[None, :]
    m = sp.csr_matrix(a.astype(np.float32))
    A = ops.DeviceCsr(m.shape[0], m.shape[1], m.indptr, m.indices, m.data, "cpu")
    T = ops.TiledCsr(A, threshold=100, block_rows=128 if kind == "gcn" else None)
    assert T.binary == (kind != "general")
    assert T.RB == (128 if kind == "gcn" else 120 if T.binary else 64) and 0 < T.tiled_fraction < 1
    np.testing.assert_allclose(_tile_dense(T), m.toarray(), rtol=3e-7, atol=0)


def test_factor_scales_deterministic_first_nonzero():
    """GCN partition blocks: a halo column's factor is derived from its first
    nonzero in CSR order (not an arbitrary one: the candidates differ in their
    last bits, and picking any of them made identical runs differ)."""
    torch = pytest.importorskip("torch")
    from paper_2303_01277_b200 import ops
    from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
    from paper_2303_01277_b200.graph import build_partitions
    g = generate_sbm(SbmSpec(nodes_per_community=20, communities=4, feature_dim=8, seed=13))
    for p in build_partitions(g, 3, "contiguous", 0, "gcn")[2]:
        a = p.adj_block
        d = ops.DeviceCsr.from_csr(a, torch.device("cpu"))
        r, c = ops.factor_scales(d)
        rp, ci = np.asarray(a.row_ptr), np.asarray(a.col_idx)
        v = np.asarray(a.values, dtype=np.float32).astype(np.float64)     # device values are fp32
        rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
        diag = np.zeros(len(rp) - 1)
        diag[rows[ci == rows]] = np.sqrt(v[ci == rows])
        for j in range(len(rp) - 1, a.cols):          # halo columns: no diagonal entry
            e = np.flatnonzero(ci == j)
            if len(e):
                assert float(c[j]) == np.float32(v[e[0]] / diag[rows[e[0]]])

