"""First-train()-in-process vs later runs (bitwise).  argv: ev(0/1) epochs bits variant st drop"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2303_01277_b200.codec import QuantConfig
from paper_2303_01277_b200.trainer import ModelConfig, TrainMode, train
from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
from paper_2303_01277_b200.graph import build_partitions
ev, ep, bits, var, st, drop = bool(int(sys.argv[1])), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5]), float(sys.argv[6])
g = generate_sbm(SbmSpec(nodes_per_community=20, communities=4, feature_dim=32, seed=13))
parts = build_partitions(g, 3, "contiguous", 0, "gcn")[2]
rs = [train(g, parts, ModelConfig((32, 8, 4), dropout=drop), TrainMode(var, st), QuantConfig(bits), ep, 7,
            evaluate_each_epoch=ev) for _ in range(int(os.environ.get("REPS", "3")))]
print(sys.argv[1:], [[float(np.abs(a - b).max()) for a, b in zip(rs[0].final_weights, r.final_weights)] for r in rs[1:]],
      [[a.train_loss - b.train_loss for a, b in zip(rs[0].metrics, r.metrics)] for r in rs[1:]])
