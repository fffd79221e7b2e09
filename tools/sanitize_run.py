"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck):
a few epochs of each model on a small graph (K1, K2, both SpMM kernels,
tcgen05 GEMMs, K8) plus wide and narrow tiled SpMM, the row-parallel gather,
dual / ReLU-only tall GEMMs and a split-K weight-gradient GEMM."""
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
        T = ops.TiledCsr(eng.A, threshold=1)
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
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
