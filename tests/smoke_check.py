"""One small device epoch checked against the CPU oracle (used by smoke())."""

from __future__ import annotations

import numpy as np


def run_smoke() -> None:
    import torch
    from oracle.epoch import OracleTrainer
    from paper_2303_01277_b200.codec import QuantConfig
    from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
    from paper_2303_01277_b200.graph import build_partitions
    from paper_2303_01277_b200.trainer import DeviceRank, ModelConfig, TrainMode
    from paper_2303_01277_b200.transport import RankLayout

    assert torch.cuda.is_available(), "smoke() needs cuda:0"
    g = generate_sbm(SbmSpec(nodes_per_community=40, communities=4, feature_dim=64, seed=1))
    _, _, parts = build_partitions(g, 2, model="sage")
    lay = RankLayout({p.id: p for p in parts}, [0, 0], 0)
    eng = DeviceRank(lay, ModelConfig((64, 32, 4), "sage"), TrainMode("sync", 0), QuantConfig(1),
                     1, 0.01, int(g.train_mask.sum()), device="cuda:0")
    eng.run_epoch(1)          # forward + backward + Adam, 1-bit halos
    torch.cuda.synchronize()
    feats = [np.asarray(p.features, dtype=np.float32).astype(np.float64) for p in parts]
    o = OracleTrainer(parts, (64, 32, 4), "sage", "sync", 0, 1, 1, features=feats)
    o.wire_log = []
    o.run_epoch(1)
    # 1) first-layer halo messages are bit-exact
    bufs = eng.xf[1]
    got = bufs.recv[0].cpu().numpy().tobytes()
    n = 0
    for s, d, e, l, ph, raw in o.wire_log:
        if l == 1 and ph == "forward":
            off = bufs.recv_off[(s, d)]
            assert got[off:off + len(raw)] == raw, f"wire block {s}->{d} differs"
            n += 1
    assert n == 2
    # 2) the epoch-1 loss agrees (first forward uses exact halos on both sides
    #    up to fp32 rounding of later layers)
    assert abs(eng.epoch_loss - o.loss) <= 1e-3 * abs(o.loss), (eng.epoch_loss, o.loss)
    # 3) the TMA-tiled SpMM (used for wide layers) agrees with the row kernel
    from paper_2303_01277_b200 import ops
    A = eng.A
    T = ops.TiledCsr(A, threshold=1)
    X = torch.randn(A.cols, 256, device="cuda:0")
    Y1 = torch.zeros(A.rows, 256, device="cuda:0")
    Y2 = torch.zeros_like(Y1)
    ops.spmm(A, X, Y1, 256, algo="rows")
    ops.spmm_tiled(T, X, Y2, 256)
    torch.cuda.synchronize()
    err = (Y1 - Y2).abs().max().item()
    assert err <= 1e-5 * max(1.0, Y1.abs().max().item()), err
    print(f"smoke ok: loss {eng.epoch_loss:.6f} (oracle {o.loss:.6f}), {n} wire blocks bit-exact, "
          f"{eng.launches} kernel launches, tiled SpMM vs row SpMM max|diff| {err:.2e} "
          f"({T.ntiles} tiles)")
