"""Wide factored SpMM (hb_spmm_tiled_bin) on the Reddit-shaped aggregation
operators at several row-block heights: CUDA-event time per launch (X is
larger than L2), max |diff| against the first variant.  One JSON line per
(operator, block rows).   python tools/kbench_spmm_wide.py [d] [reps] [rbs...]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(d=256, reps=10, *variants):
    import torch
    from bench import build_graph
    from paper_2303_01277_b200 import ops
    from paper_2303_01277_b200.trainer import _stack_csr, _transpose_device
    from paper_2303_01277_b200.transport import RankLayout
    runs = []
    for v in variants or ("64", "120", "128"):
        f = v.split(":")
        if len(f) == 1:
            runs += [(int(f[0]), 64, o) for o in (None, "lpt", "light296", "light592", None)]
        else:
            runs.append((int(f[0]), int(f[1]), f[2] if len(f) > 2 and f[2] else None))
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
        for rb, win, order in runs:
            T = ops.TiledCsr(M, factored=True, block_rows=rb, window=win, block_order=order)
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
            print(json.dumps({"op": name, "rb": rb, "window": win, "order": order, "d": d, "ms": round(ms, 4), "nnz": M.nnz,
                              "tiles": T.ntiles, "tiled_fraction": round(T.tiled_fraction, 4),
                              "max_diff_vs_first": diff,
                              "gathered_gbps": round(4.0 * M.nnz * d / ms / 1e6, 1)}), flush=True)
            del T


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:3]], *sys.argv[3:])
