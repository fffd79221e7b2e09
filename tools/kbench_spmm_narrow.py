"""Narrow factored SpMM (32 < d <= 48) on the Reddit-shaped aggregation
operators, 64-row blocks x 255-column windows, per consumer variant
(hb_spmm_set_narrow): CUDA-event time per launch, max |diff| vs variant 1.
One JSON line per (operator, variant).
  python tools/kbench_spmm_narrow.py [d] [reps] [block rows] [variants...]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(d=41, reps=20, block_rows=64, *variants):
    import torch
    from bench import build_graph
    from paper_2303_01277_b200 import ops
    from paper_2303_01277_b200.trainer import _stack_csr, _transpose_device
    from paper_2303_01277_b200.transport import RankLayout
    variants = variants or (1, 4, 5, 1)
    g, parts = build_graph("reddit")
    lay = RankLayout(parts, [0] * len(parts), 0)
    rp, ci, v = _stack_csr(lay, "mean")
    A = ops.DeviceCsr(lay.NL, lay.NL + lay.NH, rp, ci, v, "cuda")
    At = _transpose_device(A)
    del g
    ld = (d + 3) // 4 * 4
    for name, M in (("mean", A), ("mean_T", At)):
        X = torch.randn(M.cols, ld, device="cuda")
        T = ops.TiledCsr(M, factored=True, block_rows=block_rows, window=255)
        ref = None
        for var in variants:
            ops.spmm_set_narrow(var)
            Y = torch.zeros(M.rows, ld, device="cuda")
            for _ in range(2):
                ops.spmm_tiled(T, X, Y, d)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                ops.spmm_tiled(T, X, Y, d)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            diff = None if ref is None else float((Y[:, :d] - ref).abs().max())
            if ref is None:
                ref = Y[:, :d].clone()
            print(json.dumps({"op": name, "d": d, "block_rows": block_rows, "variant": var, "ms": round(ms, 4), "nnz": M.nnz,
                              "max_diff_vs_first": diff,
                              "gathered_gbps": round(4.0 * M.nnz * d / ms / 1e6, 1)}), flush=True)
        ops.spmm_set_narrow(1)


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
