"""The oracle epoch (``oracle/epoch.py``) replays the reference's own training
traces (``tests/golden/train_traces.json``, produced by ``halobit.train`` in the
build container by ``tests/golden/make_golden.py``) bit for bit: per-epoch
loss, byte meters, mode, and — where recorded — the final weights, plus the
centralized evaluation (``trainer.py:115-144``) on config 1.

This pins the oracle the GPU trajectory tests (async / SAGE / dropout /
modes) are checked against.  CPU only.
"""

import numpy as np
import pytest

from oracle.epoch import OracleTrainer, accuracies, full_forward


def _parts(g, n, model):
    from paper_2303_01277_b200.graph import build_partitions
    a, m, parts = build_partitions(g, n, "contiguous", 0, model)
    return a, m, parts


SMALL = {
    # trace name: (n, widths, model, variant, staleness, bits, epochs, seed, dropout)
    "small_sage_async2_b4": (3, (32, 16, 4), "sage", "async", 2, 4, 6, 3, 0.0),
    "small_gcn_sync_b32": (4, (32, 16, 4), "gcn", "sync", 0, 32, 10, 2, 0.0),
    "small_gcn_async0_b1_drop": (2, (32, 8, 4), "gcn", "async", 0, 1, 5, 5, 0.3),
}


def _check_epochs(o, want, epochs):
    prev = o.totals()
    for e in range(1, epochs + 1):
        mode = o.run_epoch(e)
        t = o.totals()
        w = want["metrics"][e - 1]
        assert mode == w["mode_this_epoch"]
        assert o.loss == w["train_loss"], (e, o.loss, w["train_loss"])
        got = (t["main"] - prev["main"], t["meta"] - prev["meta"], t["header"] - prev["header"],
               t["allreduce"] - prev["allreduce"], t["messages"] - prev["messages"])
        assert got == (w["main_bytes"], w["meta_bytes"], w["header_bytes"], w["allreduce_bytes"],
                       w["messages"]), e
        prev = t


@pytest.mark.parametrize("name", sorted(SMALL))
def test_small_traces_bit_identical(name, traces):
    from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
    n, widths, model, variant, st, bits, epochs, seed, drop = SMALL[name]
    g = generate_sbm(SbmSpec(nodes_per_community=25, communities=4, seed=4))
    _, _, parts = _parts(g, n, model)
    o = OracleTrainer(parts, widths, model, variant, st, bits, seed, dropout=drop,
                      global_norm=int(g.train_mask.sum()))
    want = traces[name]
    _check_epochs(o, want, epochs)
    for w, ref in zip(o.weights, want["final_weights"]):
        np.testing.assert_array_equal(w, np.asarray(ref))


@pytest.mark.parametrize("bits", [1, 32])
def test_config1_trace_with_evaluation(bits, traces):
    """BASELINE config 1 (2-layer GCN 64-32-4, 2 partitions, sync), seed 1:
    losses, byte meters and the centralized accuracies of all 20 epochs."""
    from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
    spec = SbmSpec(nodes_per_community=2500, communities=4, p_in=0.006, p_out=0.0006,
                   feature_dim=64, feature_noise=1.0, seed=1)
    g = generate_sbm(spec)
    a_hat, _, parts = _parts(g, 2, "gcn")
    o = OracleTrainer(parts, (64, 32, 4), "gcn", "sync", 0, bits, 1, global_norm=int(g.train_mask.sum()))
    want = traces[f"config1_seed1_b{bits}"]
    prev = o.totals()
    for e in range(1, 21):
        o.run_epoch(e)
        w = want["metrics"][e - 1]
        assert o.loss == w["train_loss"], e
        t = o.totals()
        assert t["main"] - prev["main"] == w["main_bytes"]
        assert t["meta"] - prev["meta"] == w["meta_bytes"]
        prev = t
        acc = accuracies(full_forward(g.features, a_hat, o.weights, "gcn"), g.labels,
                         (g.train_mask, g.val_mask, g.test_mask))
        assert acc == {k: w[k] for k in ("train_acc", "val_acc", "test_acc")}, e
