"""Host-side profile of the epoch issue path (cProfile over a few epochs after
warm-up; not a benchmark).  python tools/prof_host.py [config] [epochs]"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(config="reddit", epochs=5):
    import torch
    from bench import MODEL, PARTITIONS, WIDTHS, build_graph
    from paper_2303_01277_b200.codec import QuantConfig
    from paper_2303_01277_b200.trainer import DeviceRank, ModelConfig, TrainMode
    from paper_2303_01277_b200.transport import RankLayout
    g, parts = build_graph(config)
    lay = RankLayout(parts, [0] * PARTITIONS, 0)
    eng = DeviceRank(lay, ModelConfig(WIDTHS[config], MODEL[config]), TrainMode("sync", 0), QuantConfig(1), 0,
                     0.01, int(g.train_mask.sum()))
    del g
    for e in range(1, 4):
        eng.run_epoch(e)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    for e in range(4, 4 + epochs):
        eng.run_epoch(e, check=False)
    pr.disable()
    host = (time.perf_counter() - t0) * 1e3 / epochs
    torch.cuda.synchronize()
    print(f"host issue ms/epoch under cProfile: {host:.2f}")
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "reddit", int(sys.argv[2]) if len(sys.argv) > 2 else 5)
