"""L2 capacity knee for the row-gather SpMM: 1M rows x 26 uniform random
columns drawn from a working set of W MB of 512-byte X rows (d = 128)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402
from paper_2303_01277_b200 import ops  # noqa: E402


def main():
    dev = "cuda"
    nrows, deg, d = 1 << 20, 26, 128
    rp = torch.arange(0, (nrows + 1) * deg, deg, dtype=torch.int64, device=dev)
    vals = torch.full((nrows * deg,), 1.0 / deg, device=dev)
    Y = torch.empty(nrows, d, device=dev)
    for mb in [4, 8, 16, 24, 32, 48, 64, 80, 96, 128, 192, 256, 512, 1024]:
        rows = mb * (1 << 20) // 512
        X = torch.randn(rows, d, device=dev)
        for mode in ("uniform", "sorted_rows"):
            ci = torch.randint(0, rows, (nrows * deg,), dtype=torch.int32, device=dev)
            if mode == "sorted_rows":
                ci = ci.view(nrows, deg).sort(dim=1).values.reshape(-1).contiguous()
            A = object.__new__(ops.DeviceCsr)
            A.rows, A.cols, A.row_ptr, A.col_idx, A.values, A.nnz = nrows, rows, rp, ci, vals, nrows * deg
            for _ in range(3):
                ops.spmm(A, X, Y, d)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                ops.spmm(A, X, Y, d)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            print(json.dumps({"working_set_mb": mb, "mode": mode, "ms": round(ms, 4),
                              "gather_gbps": round(nrows * deg * 512 / ms / 1e6, 1)}), flush=True)
        del X


main()
