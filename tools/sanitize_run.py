"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck):
a few epochs of each model on a small graph (K1, K2, both SpMM kernels,
tcgen05 GEMMs, K8), CUDA-graph epochs (the pinned-buffer fetch kernel, the
device-guarded Adam), plus wide and narrow tiled SpMM (general records, and
factored one-byte records: 120-row blocks, 255-column windows with balanced
tail pairs), the row-parallel gather, dual / ReLU-only tall GEMMs, a split-K
weight-gradient GEMM and the peer-exchange counter kernels."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from paper_2303_01277_b200 import ops
    from paper_2303_01277_b200.codec import QuantConfig
    from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
    from paper_2303_01277_b200.graph import build_partitions
    from paper_2303_01277_b200.trainer import DeviceRank, ModelConfig, TrainMode
    from paper_2303_01277_b200.transport import RankLayout
    g = generate_sbm(SbmSpec(nodes_per_community=60, communities=4, feature_dim=40, seed=2))
    for model, bits in (("sage", 1), ("gcn", 2)):
        _, _, parts = build_partitions(g, 3, "hash", 0, model)
        lay = RankLayout({p.id: p for p in parts}, [0] * 3, 0)
        eng = DeviceRank(lay, ModelConfig((40, 24, 6), model), TrainMode("async", 2), QuantConfig(bits), 1, 0.01,
                         int(g.train_mask.sum()))
        for e in range(1, 4):
            eng.run_epoch(e)
        geng = DeviceRank(lay, ModelConfig((40, 24, 6), model), TrainMode("sync", 0), QuantConfig(bits), 1, 0.01,
                          int(g.train_mask.sum()))
        for e in range(1, 6):
            geng.run_epoch_graphed(e)
        while geng._deferred:
            geng.finish_epoch()
        for kw in (dict(factored=True), dict(factored=True, block_rows=64, window=255)):
            Tb = ops.TiledCsr(eng.A, threshold=1, **kw)
            Xb = torch.randn(eng.A.cols, 256, device="cuda")
            Yb = torch.zeros(eng.A.rows, 256, device="cuda")
            ops.spmm_tiled(Tb, Xb, Yb, 256 if kw.get("window", 64) == 64 else 41)
        T = ops.TiledCsr(eng.A, threshold=1, factored=False)
        X = torch.randn(eng.A.cols, 256, device="cuda")
        Y = torch.zeros(eng.A.rows, 256, device="cuda")
        ops.spmm_tiled(T, X, Y, 256)
        ops.spmm_tiled(T, X, Y, 40)                       # narrow: a lane group per row
        ops.spmm(eng.A, X, Y, 100)                        # row-parallel gather (d <= 128)
    # tall GEMMs: dual operand, ReLU-only output, TMA-store epilogue
    H = torch.randn(20000, 100, device="cuda")
    AG = torch.randn(20000, 100, device="cuda")
    W = torch.randn(200, 128, device="cuda")
    Z = torch.empty(20000, 128, device="cuda")
    R = torch.empty(20000, 128, device="cuda")
    wsb = torch.empty(1 << 20, device="cuda")
    ops.gemm2(H, W[:100], AG, W[100:], Z, relu_out=R, ws=wsb)
    ops.gemm2(H, W[:100], AG, W[100:], None, relu_out=R, ws=wsb)
    ops.gemm(H, W[:100], Z, relu_out=R, ws=wsb)
    A = torch.randn(5000, 300, device="cuda")
    m = torch.randn(5000, 64, device="cuda")
    G = torch.empty(300, 64, device="cuda")
    ws = torch.empty(64 * 300 * 64, device="cuda")
    ops.gemm(A.t(), m, G, ws=ws)
    from paper_2303_01277_b200 import _lib
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    addrs = torch.tensor([cnt.data_ptr(), cnt.data_ptr() + 8], dtype=torch.int64, device="cuda")
    _lib.call("hb_p2p_signal", addrs.data_ptr(), 2, _lib.stream_handle())
    _lib.call("hb_p2p_wait", cnt.data_ptr(), 1, None, flags.data_ptr(), 2, 10**9, _lib.stream_handle())
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
