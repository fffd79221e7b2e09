"""Factored tiled SpMM launches on the Reddit-shaped aggregation matrix for
ncu captures (not a benchmark):
  python tools/prof_spmm_bin.py <d> <window> <narrow variant> [launches] [block rows] [transpose]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(d=41, window=64, variant=1, launches=2, block_rows=64, transpose=0):
    import torch
    from bench import build_graph
    from paper_2303_01277_b200 import ops
    from paper_2303_01277_b200.trainer import _stack_csr
    from paper_2303_01277_b200.transport import RankLayout
    g, parts = build_graph("reddit")
    lay = RankLayout(parts, [0] * len(parts), 0)
    rp, ci, v = _stack_csr(lay, "mean")
    A = ops.DeviceCsr(lay.NL, lay.NL + lay.NH, rp, ci, v, "cuda")
    if transpose:
        from paper_2303_01277_b200.trainer import _transpose_device
        A = _transpose_device(A)
    T = ops.TiledCsr(A, factored=True, block_rows=block_rows, window=window)
    ops.spmm_set_narrow(variant)
    ld = (d + 3) // 4 * 4
    X = torch.randn(A.cols, ld, device="cuda")
    Y = torch.zeros(A.rows, ld, device="cuda")
    for _ in range(launches):
        ops.spmm_tiled(T, X, Y, d)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
