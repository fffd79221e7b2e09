"""Which kernels slow down while the next step's features (562 MB pinned H2D at
Reddit shape) are uploaded on a copy stream?  Per-kernel CUDA-event totals of
one eager epoch, alone and with the upload issued at the epoch's start, for
whole / chunked copies and for a copy issued after layer 1 (GEMM phase).
Prints one JSON line.   python tools/probes/upload_contention_probe.py [config]
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))


def main(config="reddit"):
    import numpy as np
    import torch
    from bench import LOSS, MODEL, PARTITIONS, WIDTHS, build_graph
    from paper_2303_01277_b200.codec import QuantConfig
    from paper_2303_01277_b200.profiling import KernelTimer
    from paper_2303_01277_b200.trainer import DeviceRank, ModelConfig, TrainMode
    from paper_2303_01277_b200.transport import RankLayout
    g, parts = build_graph(config)
    lay = RankLayout(parts, [0] * PARTITIONS, 0)
    eng = DeviceRank(lay, ModelConfig(WIDTHS[config], MODEL[config], loss=LOSS[config]), TrainMode("sync", 0),
                     QuantConfig(1), 0, 0.01, int(g.train_mask.sum()))
    feats = np.concatenate([np.asarray(p.features, dtype=np.float32) for p in lay.parts])
    host = torch.zeros((feats.shape[0], eng.Ht[1].shape[1]), dtype=torch.float32).pin_memory()
    host[:, :feats.shape[1]] = torch.from_numpy(feats)
    spare = torch.empty_like(eng.Ht[1][:eng.NL])
    del g, feats
    ep = 0
    for _ in range(3):
        ep += 1
        eng.run_epoch(ep)
    torch.cuda.synchronize()
    cs = torch.cuda.Stream()
    E = lambda: torch.cuda.Event(enable_timing=True)   # noqa: E731

    def upload(chunks):
        rows = host.shape[0]
        with torch.cuda.stream(cs):
            cs.wait_stream(torch.cuda.current_stream())
            for c in range(chunks):
                r0, r1 = rows * c // chunks, rows * (c + 1) // chunks
                spare[r0:r1].copy_(host[r0:r1], non_blocking=True)

    def epoch(chunks=0, reps=3):
        nonlocal ep
        tot, wall = {}, 0.0
        for _ in range(reps):
            t = KernelTimer()
            eng.timer = t
            torch.cuda.synchronize()
            a, b = E(), E()
            a.record()
            if chunks:
                upload(chunks)
            ep += 1
            eng.run_epoch(ep, check=False)
            b.record()
            torch.cuda.synchronize()
            wall += a.elapsed_time(b) / reps
            for k, v in t.summary().items():
                tot[k] = tot.get(k, 0.0) + v["ms"] / reps
        eng.timer = KernelTimer()
        eng.timer.enabled = False
        return {"epoch_ms": round(wall, 3), **{k: round(v, 3) for k, v in sorted(tot.items())}}

    out = {"config": config, "alone": epoch(), "upload_1": epoch(1), "upload_16": epoch(16), "alone2": epoch()}
    print(json.dumps(out))


if __name__ == "__main__":
    main(*sys.argv[1:2])
