"""Build the bench workload and run a few epochs (for ncu -k <kernel> captures;
not a benchmark).  python tools/prof_epoch.py [config] [epochs]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(config="reddit", epochs=2):
    import torch
    from bench import LOSS, MODEL, PARTITIONS, WIDTHS, build_graph
    from paper_2303_01277_b200.codec import QuantConfig
    from paper_2303_01277_b200.trainer import DeviceRank, ModelConfig, TrainMode
    from paper_2303_01277_b200.transport import RankLayout
    g, parts = build_graph(config)
    lay = RankLayout(parts, [0] * PARTITIONS, 0)
    eng = DeviceRank(lay, ModelConfig(WIDTHS[config], MODEL[config], loss=LOSS[config]), TrainMode("sync", 0), QuantConfig(1), 0,
                     0.01, int(g.train_mask.sum()))
    del g
    for e in range(1, epochs + 1):
        eng.run_epoch(e)
    torch.cuda.synchronize()
    print("loss", eng.epoch_loss)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "reddit", int(sys.argv[2]) if len(sys.argv) > 2 else 2)
