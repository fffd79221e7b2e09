"""Launch the factored tiled SpMM at every panel variant on a small mean
matrix and report which launches fail (debug aid)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import scipy.sparse as sp
import torch
from paper_2303_01277_b200 import ops

rng = np.random.default_rng(0)
pat = (rng.random((300, 400)) < 0.2).astype(np.float64)
a = sp.csr_matrix(pat / np.maximum(pat.sum(1), 1)[:, None])
A = ops.DeviceCsr(300, 400, a.indptr, a.indices, a.data, "cuda")
T = ops.TiledCsr(A, threshold=1, factored=True)
for d in (1, 41, 64, 100, 128, 132, 256):
    X = torch.randn(400, (d + 3) // 4 * 4, device="cuda")
    Y = torch.zeros(300, (d + 3) // 4 * 4, device="cuda")
    try:
        ops.spmm_tiled(T, X, Y, d)
        torch.cuda.synchronize()
        ref = torch.from_numpy(a.toarray()).float().cuda() @ X[:, :d]
        print(d, "ok", float((Y[:, :d] - ref).abs().max()))
    except Exception as e:
        print(d, "FAIL", e)
