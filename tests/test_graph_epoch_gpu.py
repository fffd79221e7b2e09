"""CUDA-graph epochs (DeviceRank.run_epoch_graphed) vs eager epochs.

A replayed graph must train bit-identically to the eager epoch loop: the
per-epoch words (K1 descriptor tables with the epoch's Philox keys, Adam's
bias corrections) are re-uploaded per replay, and the host bookkeeping (slot
tags and their staleness checks, byte meters, kernel counts) is re-applied.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _engine(model="sage", bits=1, mode=("sync", 0), widths=(32, 16, 4), seed=3):
    from paper_2303_01277_b200.codec import QuantConfig
    from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
    from paper_2303_01277_b200.graph import build_partitions
    from paper_2303_01277_b200.trainer import DeviceRank, ModelConfig, TrainMode
    from paper_2303_01277_b200.transport import RankLayout
    g = generate_sbm(SbmSpec(nodes_per_community=40, communities=4, feature_dim=widths[0], seed=seed))
    parts = build_partitions(g, 4, "contiguous", 0, model)[2]
    lay = RankLayout({p.id: p for p in parts}, [0] * 4, 0)
    return DeviceRank(lay, ModelConfig(widths, model), TrainMode(*mode), QuantConfig(bits), 5, 0.01,
                      int(g.train_mask.sum()))


def _run_graphed(eng, epochs, swap=None):
    losses = []
    for e in range(1, epochs + 1):
        if swap is not None:
            eng.swap_features(swap[e % 2])
        eng.run_epoch_graphed(e)
        if e > 1:
            eng.finish_epoch()
            losses.append(eng.epoch_loss)
    eng.finish_epoch()
    losses.append(eng.epoch_loss)
    return losses


@pytest.mark.parametrize("model,bits,mode", [
    ("sage", 1, ("sync", 0)), ("gcn", 1, ("async", 0)), ("sage", 2, ("async", 2)),
    ("gcn", 32, ("sync", 0)), ("sage", 1, ("async", 1)), ("gcn", 4, ("async", 3)),
])
def test_graphed_epochs_bit_identical(model, bits, mode):
    a, b = _engine(model, bits, mode), _engine(model, bits, mode)
    assert b.graphable()
    la = []
    for e in range(1, 10):
        a.run_epoch(e)
        la.append(a.epoch_loss)
    lb = _run_graphed(b, 9)
    assert la == lb
    assert len(b._graphs) >= 2                     # epochs 3.. came from graph replays
    for wa, wb in zip(a.weights_host(), b.weights_host()):
        assert np.array_equal(wa, wb)
    assert a.total_stats() == b.total_stats()
    assert a.slots == b.slots
    assert a.launches == b.launches
    assert a.adam_t == b.adam_t


def test_graphed_epochs_with_swapped_inputs():
    """The e2e input pipeline alternates two feature buffers: graphs are keyed
    by the layer-1 input buffer, so each replay reads the buffer it was given."""
    a, b = _engine(), _engine()
    spare = torch.empty_like(b.Ht[1])
    spare.copy_(b.Ht[1])
    bufs = [b.Ht[1], spare]
    la = []
    for e in range(1, 8):
        a.run_epoch(e)
        la.append(a.epoch_loss)
    assert _run_graphed(b, 7, swap=bufs) == la
    for wa, wb in zip(a.weights_host(), b.weights_host()):
        assert np.array_equal(wa, wb)


def test_graphed_failed_epoch_leaves_weights():
    """A non-finite input under a replayed graph: the device-guarded Adam skips
    the update and finish_epoch raises the reference's abort."""
    from paper_2303_01277_b200.trainer import TrainingError
    eng = _engine()
    for e in range(1, 6):
        eng.run_epoch_graphed(e)
    while eng._deferred:
        eng.finish_epoch()
    assert eng._graphs
    before = [w.copy() for w in eng.weights_host()]
    eng.Ht[1][0, 0] = float("nan")
    eng.run_epoch_graphed(6)
    with pytest.raises(TrainingError, match="aborted"):
        eng.finish_epoch()
    for w0, w1 in zip(before, eng.weights_host()):
        assert np.array_equal(w0, w1)
