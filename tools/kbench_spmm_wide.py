"""Wide factored SpMM on the Reddit-shaped aggregation operators: row-run
tiles (hb_spmm_tiled_bin, 64/128-row blocks) vs column-major tiles
(hb_spmm_tiled_cm).  CUDA-event time per launch (L2 not flushed: X is larger
than L2), max |diff| between formats, entries per nonzero.  One JSON line per
(operator, format).   python tools/kbench_spmm_wide.py [d] [reps]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(d=256, reps=10):
    import torch
    from bench import build_graph
    from paper_2303_01277_b200 import ops
    from paper_2303_01277_b200.trainer import _stack_csr, _transpose_device
    from paper_2303_01277_b200.transport import RankLayout
    g, parts = build_graph("reddit")
    lay = RankLayout(parts, [0] * len(parts), 0)
    rp, ci, v = _stack_csr(lay, "mean")
    A = ops.DeviceCsr(lay.NL, lay.NL + lay.NH, rp, ci, v, "cuda")
    At = _transpose_device(A)
    del g
    ld = (d + 3) // 4 * 4
    for name, M in (("mean", A), ("mean_T", At)):
        X = torch.randn(M.cols, ld, device="cuda")
        ref = None
        for fmt, rb in (("rows", 64), ("rows", 128), ("cm", 128)):
            T = ops.TiledCsr(M, factored=True, block_rows=rb, fmt=fmt)
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
            out = {"op": name, "fmt": fmt, "rb": rb, "d": d, "ms": round(ms, 4), "nnz": M.nnz,
                   "tiled_fraction": round(T.tiled_fraction, 4), "max_diff_vs_first": diff,
                   "gathered_gbps": round(4.0 * M.nnz * d / ms / 1e6, 1)}
            if fmt == "cm":
                out["entries_per_tiled_nnz"] = round(T.cm_entries / max(1, T.tiled_nnz), 4)
            print(json.dumps(out), flush=True)
            del T


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
