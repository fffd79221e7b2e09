"""Run train() repeatedly on small graphs and report bitwise run-to-run
differences (final weights, per-epoch losses) per configuration, to locate a
non-deterministic kernel.  usage: python tools/probes/determinism_probe.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    from paper_2303_01277_b200.codec import QuantConfig
    from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
    from paper_2303_01277_b200.graph import build_partitions
    from paper_2303_01277_b200.trainer import ModelConfig, TrainMode, train
    g = generate_sbm(SbmSpec(nodes_per_community=20, communities=4, feature_dim=32, seed=13))
    parts = build_partitions(g, 3, "contiguous", 0, "gcn")[2]
    cfgs = [("async", 2, 2, 0.2), ("sync", 0, 2, 0.2), ("async", 2, 32, 0.0), ("sync", 0, 32, 0.0),
            ("sync", 0, 2, 0.0), ("async", 2, 2, 0.0), ("sync", 0, 32, 0.2)]
    reps = int(os.environ.get("REPS", "6"))
    for variant, st, bits, drop in cfgs:
        runs = [train(g, parts, ModelConfig((32, 8, 4), dropout=drop), TrainMode(variant, st), QuantConfig(bits),
                      4, 7) for _ in range(reps)]
        w0 = runs[0].final_weights
        wd = [max(float(np.abs(a - b).max()) for a, b in zip(w0, r.final_weights)) for r in runs[1:]]
        ld = [max(abs(a.train_loss - b.train_loss) for a, b in zip(runs[0].metrics, r.metrics)) for r in runs[1:]]
        first = []
        for r in runs[1:]:
            e = next((i + 1 for i, (a, b) in enumerate(zip(runs[0].metrics, r.metrics))
                      if a.train_loss != b.train_loss), None)
            first.append(e)
        print(f"{variant},{st} bits={bits} drop={drop}: wdiff={wd} lossdiff={ld} first_epoch={first}", flush=True)


if __name__ == "__main__":
    main()
