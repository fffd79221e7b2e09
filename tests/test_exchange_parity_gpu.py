"""Every halo exchange of an epoch, byte for byte, on the benchmark's own
row widths and padded row strides.

The device epoch runs through ``DeviceRank`` exactly as ``bench.py`` drives
it (16-byte padded rows: d=602 sits in a 604-float row, so the 1-bit K1
takes its TMA/half-warp kernel with a Philox frame offset that alternates row
to row).  After epoch 1 every (layer, phase) receive buffer still holds the
wire blocks K1 wrote, and the exchange inputs are still in place (forward:
the local rows of ``Ht[l]``; backward: the halo rows of ``JF[l]``).  The
oracle (``oracle/epoch.py`` ``exchange``, a restatement of
``transport.py:172-205`` + ``codec.py:158-196``) is fed those same fp32 rows
(promoted to f64) and must produce identical bytes for every message of every
layer's forward and backward exchange.  K2 is checked too: forward halo rows
equal ``f32(oracle dequant)`` exactly; backward local rows equal
``f32(j + sum_k recv_k)`` accumulated in f64 in ascending peer order
(``trainer.py:214-216``).

Widths cover every residue class mod 4 (602 = 2, 41 = 1, 103 = 3, 300 = 0,
257 = 1, 43 = 3) at bits 1 and 2, contiguous and hash partitions.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


CASES = [
    ((602, 256, 256, 41), "sage", "contiguous"),      # the bench's Reddit widths
    ((602, 41, 103, 300, 5), "sage", "hash"),
    ((300, 100, 257, 43, 7), "gcn", "contiguous"),
]


@pytest.mark.parametrize("bits", [1, 2])
@pytest.mark.parametrize("widths,model,strategy", CASES)
def test_every_exchange_bit_exact(widths, model, strategy, bits):
    from oracle.epoch import OracleTrainer
    from paper_2303_01277_b200.codec import QuantConfig
    from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
    from paper_2303_01277_b200.graph import build_partitions
    from paper_2303_01277_b200.trainer import DeviceRank, ModelConfig, TrainMode
    from paper_2303_01277_b200.transport import RankLayout

    g = generate_sbm(SbmSpec(nodes_per_community=60, communities=4, p_in=0.2, p_out=0.02,
                             feature_dim=widths[0], seed=31))
    n = 4
    parts = build_partitions(g, n, strategy, 0, model)[2]
    lay = RankLayout({p.id: p for p in parts}, [0] * n, 0)
    eng = DeviceRank(lay, ModelConfig(widths, model), TrainMode(), QuantConfig(bits), 17, 0.01,
                     int(g.train_mask.sum()))
    # snapshot the backward K2 destinations around the accumulate (the next
    # layer's relu' mask is applied to them in place afterwards)
    before, after = {}, {}
    orig_recv = eng._recv

    def recv(bufs, parity, dst, accumulate):
        if accumulate:
            before[id(bufs)] = dst[:eng.NL].double().cpu().numpy()
        orig_recv(bufs, parity, dst, accumulate)
        if accumulate:
            after[id(bufs)] = dst[:eng.NL].cpu().numpy()
    eng._recv = recv
    eng.run_epoch(1)
    torch.cuda.synchronize()
    L, NL = len(widths) - 1, eng.NL
    o = OracleTrainer(parts, widths, model, "sync", 0, bits, 17)
    checked = 0
    for phase, bufs_by_layer in (("forward", eng.xf), ("backward", eng.xb)):
        for l, bufs in bufs_by_layer.items():
            d = widths[l - 1]
            if phase == "forward":
                src = eng.Ht[l][:, :d].double().cpu().numpy()
                rows = {p.id: (lay.loc_base[p.id], p.send_sets) for p in lay.parts}
            else:
                src = eng.JF[l][:, :d].double().cpu().numpy()
                rows = {p.id: (NL + lay.halo_base[p.id], p.recv_sets) for p in lay.parts}
            outgoing = [{k: src[base + np.asarray(sets[k])] for k in range(n) if k != pid and len(sets[k])}
                        for pid, (base, sets) in sorted(rows.items())]
            o.wire_log = []
            received = o.exchange(1, l, phase, outgoing)
            got = bufs.recv[0].cpu().numpy().tobytes()
            assert len(o.wire_log) == bufs.n_recv > 0
            for s, dst, _, _, _, raw in o.wire_log:
                off = bufs.recv_off[(s, dst)]
                assert got[off:off + len(raw)] == raw, (phase, l, d, s, dst)
                checked += 1
            if phase == "forward":
                H = eng.Ht[l][:, :d].cpu().numpy()
                for p in lay.parts:
                    hb = NL + lay.halo_base[p.id]
                    for k, mat in received[p.id].items():
                        np.testing.assert_array_equal(H[hb + p.recv_sets[k]], mat.astype(np.float32))
            else:
                want = before[id(bufs)].copy()
                for p in lay.parts:
                    lb = lay.loc_base[p.id]
                    for k in sorted(received[p.id]):
                        want[lb + p.send_sets[k], :d] += received[p.id][k]
                got_j = after[id(bufs)][:, :d]
                np.testing.assert_array_equal(got_j, want[:, :d].astype(np.float32))
    assert checked > 0
