"""One rows-kernel and one tiled-kernel SpMM launch on the Reddit-shaped
aggregation matrix (for ncu; not a benchmark)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(d=256, config="reddit"):
    import torch
    from bench import build_graph
    from paper_2303_01277_b200 import ops
    from paper_2303_01277_b200.trainer import _stack_csr
    from paper_2303_01277_b200.transport import RankLayout
    g, parts = build_graph(config)
    lay = RankLayout(parts, [0] * len(parts), 0)
    rp, ci, v = _stack_csr(lay, "mean")
    A = ops.DeviceCsr(lay.NL, lay.NL + lay.NH, rp, ci, v, "cuda")
    T = ops.TiledCsr(A) if config == "reddit" else None
    ld = (d + 3) // 4 * 4
    X = torch.randn(A.cols, ld, device="cuda")
    Y = torch.zeros(A.rows, ld, device="cuda")
    for _ in range(2):
        ops.spmm(A, X, Y, d, algo="rows", stream_col=lay.NL)
        if T is not None:
            ops.spmm_tiled(T, X, Y, d)
    torch.cuda.synchronize()
    ops.spmm(A, X, Y, d, algo="rows", stream_col=lay.NL)
    if T is not None:
        ops.spmm_tiled(T, X, Y, d)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 256, sys.argv[2] if len(sys.argv) > 2 else "reddit")
