"""Run one GEMM shape a few times (for ncu -k captures; not a benchmark).
  python tools/prof_gemm.py M N K kind    kind: nn | tn | nt"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(M, N, K, kind):
    import torch
    from paper_2303_01277_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(0)

    def mat(r, c):
        return torch.randn(r, (c + 3) // 4 * 4, device="cuda", generator=g)[:, :c]
    A = mat(K, M).t() if kind == "tn" else mat(M, K)
    B = mat(N, K).t() if kind == "nt" else mat(K, N)
    C = mat(M, N)
    ws = torch.empty(64 * 602 * 256, device="cuda")
    for _ in range(3):
        ops.gemm(A, B, C, ws=ws)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
