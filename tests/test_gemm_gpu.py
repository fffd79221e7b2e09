"""tcgen05 3xTF32 GEMM (K5-K7) vs an fp64 torch reference.

Tolerance: max |C - C_ref| <= 1e-5 * (sum_k |A||B|) elementwise bound scale,
i.e. fp32-GEMM accuracy (plain TF32 would be ~1e-3)."""

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _check(A, B, C, beta=0.0, C0=None):
    ref = A.double() @ B.double()
    if beta:
        ref = ref + beta * C0.double()
    scale = (A.double().abs() @ B.double().abs()).max().item() + 1e-30
    err = (C.double() - ref).abs().max().item()
    assert err <= 2e-6 * scale, (err, scale)


@pytest.mark.parametrize("M,N,K", [(128, 256, 32), (1000, 256, 602), (233, 41, 256), (5, 7, 3),
                                   (4096, 128, 1204), (300, 64, 100)])
def test_gemm_shapes_row_major(M, N, K):
    from paper_2303_01277_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(K, N, device="cuda", generator=g)
    C = torch.empty(M, N, device="cuda")
    ops.gemm(A, B, C)
    _check(A, B, C)


def test_gemm_transposed_operands_and_beta_relu():
    from paper_2303_01277_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(3)
    P = torch.randn(2000, 604, device="cuda", generator=g)[:, :602]   # padded ld
    W = torch.randn(602, 256, device="cuda", generator=g)
    m = torch.randn(2000, 256, device="cuda", generator=g)
    # G = P^T m (A col-major view, split-K with workspace)
    G = torch.empty(602, 256, device="cuda")
    ws = torch.empty(64 * 602 * 256, device="cuda")
    ops.gemm(P.t(), m, G, ws=ws)
    _check(P.t(), m, G)
    # T = m W^T (B is a transposed view)
    T = torch.empty(2000, 602, device="cuda")
    ops.gemm(m, W.t(), T)
    _check(m, W.t(), T)
    # Z = P W + 1.0 * Z0 with fused ReLU output
    Z0 = torch.randn(2000, 256, device="cuda", generator=g)
    Z = Z0.clone()
    H = torch.zeros(2000, 260, device="cuda")
    ops.gemm(P, W, Z, beta=1.0, relu_out=H)
    _check(P, W, Z, beta=1.0, C0=Z0)
    assert torch.equal(H[:, :256], torch.clamp(Z, min=0))
