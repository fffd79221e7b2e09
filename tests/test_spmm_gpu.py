"""K3/K4 CSR SpMM vs the reference's ``linalg.spmm`` (linalg.py:71-75).

Golden outputs come from the reference itself (tests/golden/make_golden.py,
``spmm_cases``) on fp32-representable inputs; the device accumulates in fp32,
so the tolerance is |y - y_ref| <= 1e-5 * (|A| @ |X|) elementwise + 1e-30."""

import numpy as np
import pytest

from conftest import load_json, load_npz

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _bound(rp, ci, v, x):
    import scipy.sparse as sp
    a = sp.csr_matrix((np.abs(v.astype(np.float64)), ci, rp), shape=(len(rp) - 1, x.shape[0]))
    return a @ np.abs(x.astype(np.float64))


def _run(rp, ci, v, x, ncols, ld_pad=0, ld_out_pad=0, algo="auto", window=0, stream_col=None):
    from paper_2303_01277_b200 import ops
    rows, d = len(rp) - 1, x.shape[1]
    A = ops.DeviceCsr(rows, ncols, rp, ci, v, "cuda")
    ldx = d + ld_pad
    X = torch.zeros(ncols, ldx, device="cuda")
    X[:, :d] = torch.from_numpy(x)
    Y = torch.full((rows, d + ld_out_pad), 7.0, device="cuda")
    ops.spmm(A, X, Y, d, algo=algo, window=window, stream_col=stream_col)
    torch.cuda.synchronize()
    out = Y.cpu().numpy()
    if ld_out_pad:
        assert np.all(out[:, d:] == 7.0)          # padding columns untouched
    return out[:, :d].astype(np.float64)


@pytest.mark.parametrize("algo,window,halo", [("rows", 0, False), ("rows", 4, False), ("rows", 16, False),
                                              ("rows", 0, True)])
def test_spmm_matches_reference_golden(algo, window, halo):
    """halo: the upper half of X's rows is read with the L2 evict-first hint."""
    meta, z = load_json("spmm_cases.json"), load_npz("spmm_cases.npz")
    for m in meta:
        k, name = m["key"], m["mat"]
        rp, ci, v = z[name + "_rp"], z[name + "_ci"], z[name + "_v"]
        x, y = z[k + "_x"], z[k + "_y"]
        # 16-byte aligned rows (vector path) and unaligned rows (scalar path)
        for pad in ((-x.shape[1]) % 4, (-x.shape[1]) % 4 + 1):
            got = _run(rp, ci, v, x, m["cols"], ld_pad=pad, ld_out_pad=pad, algo=algo, window=window,
                       stream_col=m["cols"] // 2 if halo else None)
            tol = 1e-5 * _bound(rp, ci, v, x) + 1e-30
            assert np.all(np.abs(got - y) <= tol), (k, pad, np.abs(got - y).max())


@pytest.mark.parametrize("d", [3, 8, 20, 44, 47, 65, 96, 101, 126, 128, 200, 300, 512, 1024, 1100])
def test_spmm_random_power_law_rows(d):
    """Skewed row lengths (0 .. 2000 nonzeros) at every width class."""
    import scipy.sparse as sp
    rng = np.random.default_rng(d)
    rows, cols = 700, 5000
    lens = np.minimum((rng.pareto(1.2, rows) * 8).astype(int), 2000)
    lens[::97] = 0
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(cols, n, replace=False)) for n in lens]).astype(np.int64)
    v = rng.standard_normal(len(ci)).astype(np.float32)
    x = rng.standard_normal((cols, d)).astype(np.float32)
    ref = sp.csr_matrix((v.astype(np.float64), ci, rp), shape=(rows, cols)) @ x.astype(np.float64)
    got = _run(rp, ci, v, x, cols, ld_pad=(-d) % 4, algo="rows")
    tol = 1e-5 * _bound(rp, ci, v, x) + 1e-30
    assert np.all(np.abs(got - ref) <= tol), np.abs(got - ref).max()


def _tiled_run(rp, ci, v, x, ncols, threshold, ld_pad=0, factored=None, block_rows=None, window=64,
               block_order=None):
    from paper_2303_01277_b200 import ops
    rows, d = len(rp) - 1, x.shape[1]
    A = ops.DeviceCsr(rows, ncols, rp, ci, v, "cuda")
    T = ops.TiledCsr(A, threshold=threshold, factored=factored, block_rows=block_rows, window=window,
                     block_order=block_order)
    X = torch.zeros(ncols, d + ld_pad, device="cuda")
    X[:, :d] = torch.from_numpy(x)
    Y = torch.full((rows, d + ld_pad), 7.0, device="cuda")
    ops.spmm_tiled(T, X, Y, d)
    torch.cuda.synchronize()
    out = Y.cpu().numpy()
    assert np.all(out[:, d:] == 7.0)
    return out[:, :d].astype(np.float64), T


@pytest.mark.parametrize("factored", [None, False])
@pytest.mark.parametrize("threshold", [1, 64, 10**9])
def test_spmm_tiled_matches_reference_golden(threshold, factored):
    """All-tiles / mixed / all-residual splits against the reference's spmm.
    factored None: the reference's own aggregation blocks (Â block, its
    transpose, the SAGE mean block) take the one-byte-record kernel with
    their diagonal scalings; False: every matrix through the general kernel."""
    meta, z = load_json("spmm_cases.json"), load_npz("spmm_cases.npz")
    for m in meta:
        k, name = m["key"], m["mat"]
        rp, ci, v = z[name + "_rp"], z[name + "_ci"], z[name + "_v"]
        x, y = z[k + "_x"], z[k + "_y"]
        got, T = _tiled_run(rp, ci, v, x, m["cols"], threshold, ld_pad=(-x.shape[1]) % 4, factored=factored)
        assert T.binary == (factored is None and name in ("ahat_block", "ahat_block_T", "mean_block")), name
        tol = 1e-5 * _bound(rp, ci, v, x) + 1e-30
        assert np.all(np.abs(got - y) <= tol), (k, threshold, np.abs(got - y).max())


def _community_pattern(rng, rows, comm, halo_cols, lo=20, hi=120):
    ci, rp = [], [0]
    for r in range(rows):
        c0 = (r // comm) * comm
        intra = rng.choice(comm, size=rng.integers(lo, hi), replace=False) + c0
        halo = rows + rng.choice(halo_cols, size=rng.integers(0, 4), replace=False)
        c = np.sort(np.concatenate([intra, halo]))
        ci.append(c)
        rp.append(rp[-1] + len(c))
    return np.asarray(rp, dtype=np.int64), np.concatenate(ci).astype(np.int64)


@pytest.mark.parametrize("rb", [64, 120, 128])
@pytest.mark.parametrize("kind", ["mean", "mean_T", "gcn", "gcn_T"])
@pytest.mark.parametrize("d", [41, 100, 128, 256, 602])
@pytest.mark.parametrize("threshold", [1, 64])
def test_spmm_tiled_factored_operators(kind, d, threshold, rb):
    """The trainer's aggregation operators on community blocks (the Reddit
    shape in miniature): SAGE mean D^-1 A (row scale), its transpose (column
    scale, applied through the scratch copy of X), GCN Â = D^-1/2 (A+I)
    D^-1/2 blocks with halo columns and their transposes (both scales), vs
    scipy f64 at the fp32 tolerance."""
    import scipy.sparse as sp
    rng = np.random.default_rng(31 + d)
    rows, comm, halo = 1500, 300, 2000
    rp, ci = _community_pattern(rng, rows, comm, halo)
    cols = rows + halo
    pat = sp.csr_matrix((np.ones(len(ci)), ci, rp), shape=(rows, cols))
    if kind.startswith("mean"):
        deg = np.maximum(np.diff(rp), 1).astype(np.float64)
        a = sp.diags(1.0 / deg) @ pat
    else:
        pat = pat.tolil()
        pat.setdiag(1.0)                          # self loops on the square part
        pat = pat.tocsr()
        dinv = 1.0 / np.sqrt(rng.integers(1, 400, cols).astype(np.float64))
        a = sp.diags(dinv[:rows]) @ pat @ sp.diags(dinv)
    if kind.endswith("_T"):
        a = a.T
    a = sp.csr_matrix(a)
    a.sort_indices()
    v = a.data.astype(np.float32)
    rp2, ci2 = a.indptr.astype(np.int64), a.indices.astype(np.int64)
    x = rng.standard_normal((a.shape[1], d)).astype(np.float32)
    ref = sp.csr_matrix((v.astype(np.float64), ci2, rp2), shape=a.shape) @ x.astype(np.float64)
    got, T = _tiled_run(rp2, ci2, v, x, a.shape[1], threshold, ld_pad=(-d) % 4, factored=True, block_rows=rb)
    assert T.binary and T.RB == rb
    for order in ("lpt", "light7"):
        # the work-item order changes which CTA runs a block, not the result
        got_o, _ = _tiled_run(rp2, ci2, v, x, a.shape[1], threshold, ld_pad=(-d) % 4, factored=True,
                              block_rows=rb, block_order=order)
        assert np.array_equal(got_o, got)
    assert (T.row_scale is None) == (kind == "mean_T") and (T.col_scale is None) == (kind == "mean")
    tol = 1e-5 * _bound(rp2, ci2, v, x) + 1e-30
    assert np.all(np.abs(got - ref) <= tol), np.abs(got - ref).max()


@pytest.mark.parametrize("rb", [64, 120, 128])
@pytest.mark.parametrize("d", [41, 256])
def test_spmm_tiled_factored_splits_dense_tiles(d, rb):
    """A fully dense 128x64 block (8192 one-byte records) exceeds a factored
    tile's 2048-record slot and becomes several tiles of the same window;
    the second launch reuses the self-resetting work counter."""
    import scipy.sparse as sp
    rng = np.random.default_rng(5 + d)
    rows, cols = 300, 400
    pat = (rng.random((rows, cols)) < 0.05).astype(np.float64)
    pat[128:256, 64:128] = 1.0
    deg = np.maximum(pat.sum(1), 1.0)
    a = sp.csr_matrix(pat / deg[:, None])
    rp, ci, v = a.indptr.astype(np.int64), a.indices.astype(np.int64), a.data.astype(np.float32)
    x = rng.standard_normal((cols, d)).astype(np.float32)
    ref = sp.csr_matrix((v.astype(np.float64), ci, rp), shape=a.shape) @ x.astype(np.float64)
    for _ in range(2):
        got, T = _tiled_run(rp, ci, v, x, cols, 64, ld_pad=(-d) % 4, factored=True, block_rows=rb)
        assert T.ntiles > int((T.tile_ptr[1:] - T.tile_ptr[:-1]).gt(0).sum())
        tol = 1e-5 * _bound(rp, ci, v, x) + 1e-30
        assert np.all(np.abs(got - ref) <= tol), np.abs(got - ref).max()
        assert int(T.work.abs().sum()) == 0       # counter pair re-armed by the last CTA


@pytest.mark.parametrize("d", [41, 100, 128, 256, 602])
def test_spmm_tiled_community_blocks(d):
    import scipy.sparse as sp
    rng = np.random.default_rng(11 + d)
    rows, comm = 1500, 300
    cols = rows + 2000
    ci, rp = [], [0]
    for r in range(rows):
        c0 = (r // comm) * comm
        intra = rng.choice(comm, size=rng.integers(20, 120), replace=False) + c0
        halo = rows + rng.choice(2000, size=rng.integers(0, 4), replace=False)
        c = np.sort(np.concatenate([intra, halo]))
        ci.append(c)
        rp.append(rp[-1] + len(c))
    ci = np.concatenate(ci).astype(np.int64)
    rp = np.asarray(rp, dtype=np.int64)
    v = rng.standard_normal(len(ci)).astype(np.float32)
    x = rng.standard_normal((cols, d)).astype(np.float32)
    ref = sp.csr_matrix((v.astype(np.float64), ci, rp), shape=(rows, cols)) @ x.astype(np.float64)
    got, T = _tiled_run(rp, ci, v, x, cols, 64, ld_pad=(-d) % 4)
    assert 0.5 < T.tiled_fraction < 1.0          # both paths exercised
    tol = 1e-5 * _bound(rp, ci, v, x) + 1e-30
    assert np.all(np.abs(got - ref) <= tol), np.abs(got - ref).max()


@pytest.mark.parametrize("d", [41, 128, 256])
def test_spmm_tiled_splits_dense_tiles(d):
    """A fully dense 64x64 block (4096 records) exceeds a tile's record slot
    and is split into several tiles of the same window."""
    import scipy.sparse as sp
    rng = np.random.default_rng(d)
    rows, cols = 200, 400
    dense = np.zeros((rows, cols), dtype=np.float32)
    dense[64:128, 128:192] = rng.standard_normal((64, 64))
    mask = rng.random((rows, cols)) < 0.05
    dense[mask] = rng.standard_normal(mask.sum())
    a = sp.csr_matrix(dense)
    rp, ci, v = a.indptr.astype(np.int64), a.indices.astype(np.int64), a.data.astype(np.float32)
    x = rng.standard_normal((cols, d)).astype(np.float32)
    ref = a.astype(np.float64) @ x.astype(np.float64)
    got, T = _tiled_run(rp, ci, v, x, cols, 64, ld_pad=(-d) % 4)
    assert T.ntiles > int((T.tile_ptr[1:] - T.tile_ptr[:-1]).gt(0).sum())   # some window has >1 tile
    tol = 1e-5 * _bound(rp, ci, v, x) + 1e-30
    assert np.all(np.abs(got - ref) <= tol), np.abs(got - ref).max()


@pytest.fixture(params=[0, 1, 2, 3], ids=["g8", "g4x3_or_balanced_pairs", "tail_pairs16", "tail_pairs8"])
def narrow_variant(request):
    from paper_2303_01277_b200 import ops
    ops.spmm_set_narrow(request.param)
    yield request.param
    ops.spmm_set_narrow(1)


@pytest.mark.parametrize("window", [64, 128, 255])
@pytest.mark.parametrize("kind", ["mean", "mean_T", "gcn"])
@pytest.mark.parametrize("d", [33, 36, 41, 44, 47, 48, 20])
def test_spmm_tiled_factored_narrow_variants(kind, d, window, narrow_variant):
    """Every narrow consumer layout (d <= 48; tail pairs for 32 < d <= 48,
    odd and even record runs), with 64- and 128-column windows, vs scipy f64."""
    import scipy.sparse as sp
    rng = np.random.default_rng(7 * d + len(kind))
    rows, comm, halo = 1300, 260, 900
    rp, ci = _community_pattern(rng, rows, comm, halo)
    cols = rows + halo
    pat = sp.csr_matrix((np.ones(len(ci)), ci, rp), shape=(rows, cols))
    if kind.startswith("mean"):
        deg = np.maximum(np.diff(rp), 1).astype(np.float64)
        a = sp.diags(1.0 / deg) @ pat
    else:
        pat = pat.tolil()
        pat.setdiag(1.0)
        pat = pat.tocsr()
        dinv = 1.0 / np.sqrt(rng.integers(1, 400, cols).astype(np.float64))
        a = sp.diags(dinv[:rows]) @ pat @ sp.diags(dinv)
    if kind.endswith("_T"):
        a = a.T
    a = sp.csr_matrix(a)
    a.sort_indices()
    v = a.data.astype(np.float32)
    rp2, ci2 = a.indptr.astype(np.int64), a.indices.astype(np.int64)
    x = rng.standard_normal((a.shape[1], d)).astype(np.float32)
    ref = sp.csr_matrix((v.astype(np.float64), ci2, rp2), shape=a.shape) @ x.astype(np.float64)
    for threshold in (1, 64):
        got, T = _tiled_run(rp2, ci2, v, x, a.shape[1], threshold, ld_pad=(-d) % 4, factored=True, block_rows=64,
                            window=window)
        assert T.binary and T.W == window
        tol = 1e-5 * _bound(rp2, ci2, v, x) + 1e-30
        assert np.all(np.abs(got - ref) <= tol), (threshold, np.abs(got - ref).max())
        if window == 255 and d > 32:           # 128-row blocks with 255-column windows
            got, T = _tiled_run(rp2, ci2, v, x, a.shape[1], threshold, ld_pad=(-d) % 4, factored=True,
                                block_rows=128, window=window)
            assert T.RB == 128 and T.W == 255
        tol = 1e-5 * _bound(rp2, ci2, v, x) + 1e-30
        assert np.all(np.abs(got - ref) <= tol), (threshold, np.abs(got - ref).max())
