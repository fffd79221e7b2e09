"""K8 elementwise ops vs the oracle (linalg.py:78-140 restated in oracle/epoch.py).

Tolerances: ReLU / relu' masks exact; softmax-CE loss rel 1e-6 (f64 loss
accumulation on device, fp32 logits) and gradient abs 1e-7; Adam one step
rel 1e-6 + abs 1e-6 (f64 update math, fp32 storage of w, m, v)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


@pytest.mark.parametrize("n,d,ld", [(1000, 256, 256), (777, 41, 44), (50, 41, 41), (3, 5, 7)])
def test_relu_and_relu_grad_mul(n, d, ld):
    from paper_2303_01277_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(n + d)
    z = torch.randn(n, ld, device="cuda", generator=g)
    z[0, 0] = float("nan")
    y = torch.full((n, ld), 9.0, device="cuda")
    ops.relu(z, y, n, d)
    zz = z[:, :d].cpu().numpy()
    np.testing.assert_array_equal(y[:, :d].cpu().numpy(), np.maximum(zz, 0.0))   # NaN propagates like numpy
    assert torch.all(y[:, d:] == 9.0)
    j = torch.randn(n, ld, device="cuda", generator=g)
    m = torch.full((n, ld), 9.0, device="cuda")
    ops.relu_grad_mul(j, y, m, n, d)
    want = np.where(y[:, :d].cpu().numpy() > 0, j[:, :d].cpu().numpy(), 0.0)
    np.testing.assert_array_equal(m[:, :d].cpu().numpy(), want)


@pytest.mark.parametrize("n,C", [(5000, 41), (300, 4), (64, 100), (20000, 47), (700, 160)])
def test_softmax_xent_matches_oracle(n, C):
    from oracle.epoch import xent
    from paper_2303_01277_b200 import ops
    rng = np.random.default_rng(C)
    logits = (rng.standard_normal((n, C)) * 3).astype(np.float32)
    labels = rng.integers(0, C, n)
    mask = rng.random(n) < 0.6
    norm = float(mask.sum() + 17)              # global normaliser (trainer.py:397)
    loss_ref, grad_ref = xent(logits.astype(np.float64), labels, mask, norm)
    ld = (C + 3) // 4 * 4
    L = torch.zeros(n, ld, device="cuda")
    L[:, :C] = torch.from_numpy(logits).cuda()
    lab = torch.from_numpy(labels.astype(np.int32)).cuda()
    msk = torch.from_numpy(mask.astype(np.uint8)).cuda()
    # the unmasked rows are written (zeros) ...
    grad = torch.full((n, ld), 5.0, device="cuda")
    row_loss = torch.full((n,), 3.0, dtype=torch.float64, device="cuda")
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    ops.softmax_xent(L, C, lab, msk, norm, grad, row_loss, loss)
    assert float(loss) == pytest.approx(loss_ref, rel=1e-6)
    np.testing.assert_allclose(grad[:, :C].cpu().numpy(), grad_ref, atol=1e-7)
    # ... or kept (keep_unmasked: the trainer's buffers hold zeros there)
    grad2 = torch.zeros(n, ld, device="cuda")
    row_loss2 = torch.zeros(n, dtype=torch.float64, device="cuda")
    loss2 = torch.zeros(1, dtype=torch.float64, device="cuda")
    ops.softmax_xent(L, C, lab, msk, norm, grad2, row_loss2, loss2, keep_unmasked=True)
    assert float(loss2) == float(loss)
    assert torch.equal(grad2[:, :C], grad[:, :C])


def test_adam_matches_oracle():
    from oracle.epoch import Adam
    from paper_2303_01277_b200 import ops
    rng = np.random.default_rng(3)
    w0 = rng.standard_normal(5000).astype(np.float32)
    opt = Adam(0.01)
    w_ref = w0.astype(np.float64)
    w = torch.from_numpy(w0.copy()).cuda()
    m, v = torch.zeros_like(w), torch.zeros_like(w)
    for t in range(1, 4):
        gr = rng.standard_normal(5000).astype(np.float32)
        w_ref = opt.step(w_ref, gr.astype(np.float64))
        ops.adam_step(w, torch.from_numpy(gr).cuda(), m, v, 0.01, t)
    np.testing.assert_allclose(w.cpu().numpy(), w_ref, rtol=1e-6, atol=1e-6)   # fp32 storage of w, m, v


@pytest.mark.parametrize("n,C", [(1000, 100), (20000, 7)])
def test_sigmoid_bce_multilabel_vs_torch_f64(n, C):
    """Multi-label extension (not in the reference): masked sigmoid BCE loss
    and gradient vs a torch float64 restatement (mean over labels, global
    normaliser); rel 1e-6 on the loss, 1e-7 absolute on the gradient."""
    from paper_2303_01277_b200 import ops
    rng = np.random.default_rng(n + C)
    z = torch.from_numpy((rng.standard_normal((n, C)) * 4).astype(np.float32)).cuda()
    y = torch.from_numpy((rng.random((n, C)) < 0.1).astype(np.uint8)).cuda()
    mask = torch.from_numpy((rng.random(n) < 0.7).astype(np.uint8)).cuda()
    norm = float(mask.sum()) + 5.0
    zd, yd, md = z.double(), y.double(), mask.bool()
    per = torch.nn.functional.binary_cross_entropy_with_logits(zd, yd, reduction="none")
    loss_ref = float(per[md].sum() / (norm * C))
    grad_ref = torch.where(md[:, None], (torch.sigmoid(zd) - yd) / (norm * C), torch.zeros_like(zd))
    ld = (C + 3) // 4 * 4
    L = torch.zeros(n, ld, device="cuda")
    L[:, :C] = z
    grad = torch.full((n, ld), 5.0, device="cuda")
    row_loss = torch.zeros(n, dtype=torch.float64, device="cuda")
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    ops.sigmoid_bce(L, C, y, mask, norm, grad, row_loss, loss)
    assert float(loss) == pytest.approx(loss_ref, rel=1e-6)
    assert float((grad[:, :C].double() - grad_ref).abs().max()) <= 1e-7
    counts = torch.zeros(9, dtype=torch.int64, device="cuda")
    em = torch.from_numpy(rng.integers(0, 4, n).astype(np.uint8)).cuda()
    ops.multilabel_counts(L, C, y, em, counts)
    pred, tgt = z > 0, y.bool()
    for k in range(3):
        sel = em == k + 1
        want = [int((pred & tgt)[sel].sum()), int((pred & ~tgt)[sel].sum()), int((~pred & tgt)[sel].sum())]
        assert counts[3 * k:3 * k + 3].tolist() == want
