"""Does the per-step feature upload (562 MB pinned H2D at Reddit shape) overlap
with an epoch?  Measures, on the Reddit bench engine:
  * epoch alone, upload alone (one copy, and in chunks),
  * the upload on a copy stream issued at the start of an epoch (whole / chunked),
    with per-chunk events giving the copy bandwidth while the epoch runs.
Not a benchmark: prints one JSON line per measurement.
  python tools/probes/upload_overlap_probe.py [config]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))


def main(config="reddit"):
    import numpy as np
    import torch
    from bench import LOSS, MODEL, PARTITIONS, WIDTHS, build_graph
    from paper_2303_01277_b200.codec import QuantConfig
    from paper_2303_01277_b200.trainer import DeviceRank, ModelConfig, TrainMode
    from paper_2303_01277_b200.transport import RankLayout
    g, parts = build_graph(config)
    lay = RankLayout(parts, [0] * PARTITIONS, 0)
    eng = DeviceRank(lay, ModelConfig(WIDTHS[config], MODEL[config], loss=LOSS[config]), TrainMode("sync", 0),
                     QuantConfig(1), 0, 0.01, int(g.train_mask.sum()))
    feats = np.concatenate([np.asarray(p.features, dtype=np.float32) for p in lay.parts])
    ldf = eng.Ht[1].shape[1]
    host = torch.zeros((feats.shape[0], ldf), dtype=torch.float32).pin_memory()
    host[:, :feats.shape[1]] = torch.from_numpy(feats)
    spare = torch.empty_like(eng.Ht[1][:eng.NL])
    del g, feats
    ep = 0
    for _ in range(3):
        ep += 1
        eng.run_epoch(ep)
    torch.cuda.synchronize()
    cs = torch.cuda.Stream()
    nbytes = host.numel() * 4
    E = lambda: torch.cuda.Event(enable_timing=True)   # noqa: E731

    def epoch_alone(n=5):
        nonlocal ep
        a, b = E(), E()
        a.record()
        for _ in range(n):
            ep += 1
            eng.run_epoch(ep, check=False)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    def upload(dst, chunks, stream):
        rows = host.shape[0]
        evs = [E()]
        with torch.cuda.stream(stream):
            evs[0].record(stream)
            for c in range(chunks):
                r0, r1 = rows * c // chunks, rows * (c + 1) // chunks
                dst[r0:r1].copy_(host[r0:r1], non_blocking=True)
                e = E()
                e.record(stream)
                evs.append(e)
        return evs

    out = {"config": config, "upload_bytes": nbytes}
    out["epoch_ms"] = epoch_alone()
    for chunks in (1, 8, 32):
        upload(spare, chunks, cs)
        torch.cuda.synchronize()
        evs = upload(spare, chunks, cs)
        torch.cuda.synchronize()
        ms = evs[0].elapsed_time(evs[-1])
        out[f"upload_alone_{chunks}"] = {"ms": ms, "gbs": nbytes / ms / 1e6}
    for chunks in (1, 8, 32):
        torch.cuda.synchronize()
        a, b = E(), E()
        a.record()
        evs = upload(spare, chunks, cs)
        ep += 1
        eng.run_epoch(ep, check=False)
        b.record()
        torch.cuda.current_stream().wait_stream(cs)
        c = E()
        c.record()
        torch.cuda.synchronize()
        per = [evs[i].elapsed_time(evs[i + 1]) for i in range(len(evs) - 1)]
        out[f"overlap_{chunks}"] = {"epoch_ms": a.elapsed_time(b), "both_ms": a.elapsed_time(c),
                                    "upload_ms": evs[0].elapsed_time(evs[-1]),
                                    "upload_gbs": nbytes / evs[0].elapsed_time(evs[-1]) / 1e6,
                                    "chunk_ms_min": min(per), "chunk_ms_max": max(per)}
    # serial (what bench's e2e does today): upload then epoch on one stream
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        eng.Ht[1][:eng.NL].copy_(host, non_blocking=True)
        ep += 1
        eng.run_epoch(ep, check=False)
    torch.cuda.synchronize()
    out["serial_wall_ms"] = (time.perf_counter() - t0) * 1e3 / 3
    print(json.dumps(out))


if __name__ == "__main__":
    main(*sys.argv[1:2])
