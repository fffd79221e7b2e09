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


def _pad(rows, cols, g, ld=None):
    ld = ld or (cols + 3) // 4 * 4
    return torch.randn(rows, ld, device="cuda", generator=g)[:, :cols]


@pytest.fixture(params=[0, 1, 3], ids=["tma", "simt_staged", "tma_a_in_tmem"])
def gemm_path(request):
    from paper_2303_01277_b200 import ops
    ops.gemm_set_path(request.param)
    yield request.param
    ops.gemm_set_path(0)


@pytest.mark.parametrize("M,N,K", [(128, 64, 32), (1000, 256, 602), (5000, 41, 256), (777, 602, 100),
                                   (300, 128, 1204), (64, 200, 40)])
def test_gemm_forward_layout(M, N, K, gemm_path):
    """Z = P W: A K-major (padded rows), B MN-major (padded rows)."""
    from paper_2303_01277_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M + 3 * N + 7 * K)
    A, B = _pad(M, K, g), _pad(K, N, g)
    C = torch.empty(M, N, device="cuda")
    ops.gemm(A, B, C)
    _check(A, B, C)


@pytest.mark.parametrize("M,N,K", [(602, 256, 20000), (256, 41, 9000), (1204, 256, 4096), (100, 128, 700)])
def test_gemm_weight_grad_split_k(M, N, K, gemm_path):
    """G = P^T m: both operands MN-major, long K -> deterministic split-K."""
    from paper_2303_01277_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    P, m = _pad(K, M, g), _pad(K, N, g)
    G = torch.empty(M, N, device="cuda")
    ws = torch.empty(64 * M * N, device="cuda")
    ops.gemm(P.t(), m, G, ws=ws)
    _check(P.t(), m, G)
    G2 = torch.empty(M, N, device="cuda")
    ops.gemm(P.t(), m, G2, ws=ws)
    assert torch.equal(G, G2)           # fixed-order reduction: replay is bit-identical


@pytest.mark.parametrize("M,N,K", [(3000, 256, 256), (1000, 602, 41), (500, 256, 128)])
def test_gemm_input_grad_layout(M, N, K, gemm_path):
    """T = m W^T: A K-major, B K-major (transposed weight view)."""
    from paper_2303_01277_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M * 3 + N + K)
    m, W = _pad(M, K, g), _pad(N, K, g)
    T = torch.empty(M, N, device="cuda")
    ops.gemm(m, W.t(), T)
    _check(m, W.t(), T)


def test_gemm_accumulate_relu_and_split_relu(gemm_path):
    from paper_2303_01277_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(17)
    A, B = _pad(2000, 256, g), _pad(256, 41, g)
    Z0 = _pad(2000, 41, g).contiguous()
    Z = Z0.clone()
    H = torch.zeros(2000, 44, device="cuda")
    ops.gemm(A, B, Z, beta=1.0, relu_out=H[:, :41])
    _check(A, B, Z, beta=1.0, C0=Z0)
    assert torch.equal(H[:, :41], torch.clamp(Z, min=0))
    if gemm_path == 1:
        return           # the SIMT-staged kernel has no ReLU epilogue under split-K
    # split-K with the ReLU copy applied by the reduction
    P, m = _pad(30000, 128, g), _pad(30000, 64, g)
    G = torch.empty(128, 64, device="cuda")
    R = torch.empty(128, 64, device="cuda")
    ws = torch.empty(64 * 128 * 64, device="cuda")
    ops.gemm(P.t(), m, G, ws=ws, relu_out=R)
    _check(P.t(), m, G)
    assert torch.equal(R, torch.clamp(G, min=0))


@pytest.mark.parametrize("N,K,kind", [(256, 602, "nn"), (41, 256, "nn"), (256, 256, "nt"), (602, 41, "nt")])
def test_gemm_presplit_weight_operand(N, K, kind, gemm_path):
    """Tall GEMMs (>= 2 tiles per SM) with a weight-sized B take the path that
    splits B into tf32 hi / lo once (workspace) instead of per CTA."""
    from paper_2303_01277_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(N + K)
    M = 40_000
    A = _pad(M, K, g)
    B = _pad(K, N, g) if kind == "nn" else _pad(N, K, g).t()
    C0 = torch.randn(M, N, device="cuda", generator=g)
    C = C0.clone()
    H = torch.zeros(M, (N + 3) // 4 * 4, device="cuda")
    ws = torch.empty(64 * 602 * 256, device="cuda")
    ops.gemm(A, B, C, beta=1.0, relu_out=H[:, :N], ws=ws)
    _check(A, B, C, beta=1.0, C0=C0)
    assert torch.equal(H[:, :N], torch.clamp(C, min=0))


@pytest.mark.parametrize("M,N,K", [(40000, 128, 100), (40001, 41, 256), (37900, 256, 602), (38000, 94, 128)])
@pytest.mark.parametrize("ws_on", [True, False])
def test_tall_gemm_tma_store_epilogue(M, N, K, ws_on):
    """Tall GEMMs (>= 148 output tiles) run the A-in-TMEM kernel whose epilogue
    stages through shared memory and TMA bulk-stores C and the ReLU copy."""
    from paper_2303_01277_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K + 4, device="cuda", generator=g)[:, :K]
    B = torch.randn(K, N, device="cuda", generator=g)
    ldc = (N + 3) // 4 * 4
    C = torch.full((M, ldc), 7.0, device="cuda")[:, :N]
    H = torch.full((M, ldc + 4), 7.0, device="cuda")
    ws = torch.empty(4 << 20, device="cuda") if ws_on else None
    ops.gemm(A, B, C, relu_out=H[:, :N], ws=ws)
    _check(A, B, C)
    assert torch.equal(H[:, :N], torch.clamp(C, min=0))
    assert bool((H[:, N:] == 7.0).all())                      # nothing written past N
    if ldc > N:
        full = C.as_strided((M, ldc), (ldc, 1))
        assert bool((full[:, N:] == 7.0).all())


@pytest.mark.parametrize("M", [40000, 40001, 700])
@pytest.mark.parametrize("ws_on", [True, False])
def test_gemm2_dual(M, ws_on):
    """C = A1 B1 + A2 B2 (the SAGE combine and its input gradient) in one pass,
    K1 not a multiple of the 32-wide K block, B operands as transposed views."""
    from paper_2303_01277_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M)
    d, dout = 100, 128
    H = torch.randn(M, 104, device="cuda", generator=g)[:, :d]
    AGG = torch.randn(M, 104, device="cuda", generator=g)[:, :d]
    W = torch.randn(2 * d, dout, device="cuda", generator=g)
    ws = torch.empty(4 << 20, device="cuda") if ws_on else None
    Z = torch.empty(M, dout, device="cuda")
    R = torch.empty(M, dout + 4, device="cuda")
    ops.gemm2(H, W[:d], AGG, W[d:], Z, relu_out=R[:, :dout], ws=ws)
    _check(torch.cat([H, AGG], 1), W, Z)
    assert torch.equal(R[:, :dout], torch.clamp(Z, min=0))
    # input gradient: j = S W_bot^T + m W_top^T
    S = torch.randn(M, dout, device="cuda", generator=g)
    m = torch.randn(M, dout, device="cuda", generator=g)
    J = torch.empty(M, 104, device="cuda")[:, :d]
    ops.gemm2(S, W[d:].t(), m, W[:d].t(), J, ws=ws)
    _check(torch.cat([S, m], 1), torch.cat([W[d:].t(), W[:d].t()], 0), J)
    # beta accumulate
    J0 = J.clone()
    ops.gemm2(S, W[d:].t(), m, W[:d].t(), J, beta=1.0, ws=ws)
    _check(torch.cat([S, m], 1), torch.cat([W[d:].t(), W[:d].t()], 0), J, beta=1.0, C0=J0)


def test_relu_only_store():
    """C = NULL: only relu(A B) / relu(A1 B1 + A2 B2) is written."""
    from paper_2303_01277_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(9)
    M, K, N = 40000, 100, 128
    A1 = torch.randn(M, 104, device="cuda", generator=g)[:, :K]
    A2 = torch.randn(M, 104, device="cuda", generator=g)[:, :K]
    W = torch.randn(2 * K, N, device="cuda", generator=g)
    ws = torch.empty(4 << 20, device="cuda")
    R = torch.full((M, N + 4), 3.0, device="cuda")
    ops.gemm2(A1, W[:K], A2, W[K:], None, relu_out=R[:, :N], ws=ws)
    Z = torch.empty(M, N, device="cuda")
    ops.gemm2(A1, W[:K], A2, W[K:], Z, ws=ws)
    assert torch.equal(R[:, :N], torch.clamp(Z, min=0))
    assert bool((R[:, N:] == 3.0).all())
    R2 = torch.full((M, N), 3.0, device="cuda")
    ops.gemm(A1, W[:K], None, relu_out=R2, ws=ws)
    ops.gemm(A1, W[:K], Z, ws=ws)
    assert torch.equal(R2, torch.clamp(Z, min=0))


@pytest.mark.parametrize("M,K,N", [(2000, 512, 256), (1500, 1204, 256), (700, 256, 41)])
def test_relu_only_store_small_m_long_k(M, K, N):
    """C = NULL on shapes where split-K would be chosen (tiles < SMs, many K
    blocks): the launcher must keep one split and store only the ReLU copy."""
    from paper_2303_01277_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M + K + N)
    Kp, Np = (K + 3) // 4 * 4, (N + 3) // 4 * 4
    A = torch.randn(M, Kp, device="cuda", generator=g)[:, :K]
    W = torch.randn(K, Np, device="cuda", generator=g)[:, :N]
    ws = torch.empty(64 * K * Np, device="cuda")
    R = torch.full((M, Np), 3.0, device="cuda")
    ops.gemm(A, W, None, relu_out=R[:, :N], ws=ws)
    # the same single-split path with C stored (a workspace that holds the
    # pre-split weight but not M x N partials: split-K off), so the ReLU copy
    # must be the bit-identical clamp of it
    Z = torch.empty(M, N, device="cuda")
    ops.gemm(A, W, Z, ws=torch.empty(2 * N * Kp, device="cuda"))
    _check(A, W, Z)
    assert torch.equal(R[:, :N], torch.clamp(Z, min=0))
    # and the split-K path (C only) agrees within the 3xTF32 tolerance
    Zs = torch.empty(M, N, device="cuda")
    ops.gemm(A, W, Zs, ws=ws)
    _check(A, W, Zs)


def test_simt_split_k_relu_out(gemm_path):
    """SIMT-staged path with a ReLU copy on a small-M, long-K shape: C and the
    ReLU copy both written (split-K is not taken when relu_out is set)."""
    from paper_2303_01277_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(23)
    A, B = _pad(600, 1024, g), _pad(1024, 64, g)
    C = torch.empty(600, 64, device="cuda")
    R = torch.full((600, 64), 7.0, device="cuda")
    ws = torch.empty(64 * 600 * 64, device="cuda")
    ops.gemm(A, B, C, ws=ws, relu_out=R)
    _check(A, B, C)
    assert torch.equal(R, torch.clamp(C, min=0))
