"""Is the first async 2-bit train() different because it is the first in the process (lazy
module loading makes the host run ahead) or because of its own state?  argv: warm(0/1)"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2303_01277_b200.codec import QuantConfig
from paper_2303_01277_b200.trainer import ModelConfig, TrainMode, train
from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
from paper_2303_01277_b200.graph import build_partitions
g = generate_sbm(SbmSpec(nodes_per_community=20, communities=4, feature_dim=32, seed=13))
parts = build_partitions(g, 3, "contiguous", 0, "gcn")[2]
if int(sys.argv[1]):
    train(g, parts, ModelConfig((32, 8, 4)), TrainMode("sync", 0), QuantConfig(32), 2, 7, evaluate_each_epoch=False)
rs = [train(g, parts, ModelConfig((32, 8, 4), dropout=0.2), TrainMode("async", 2), QuantConfig(2), 4, 7,
            evaluate_each_epoch=False) for _ in range(3)]
print(sys.argv[1:], os.environ.get("CUDA_LAUNCH_BLOCKING"), [m.train_loss for m in rs[0].metrics],
      [[float(np.abs(a - b).max()) for a, b in zip(rs[0].final_weights, r.final_weights)] for r in rs[1:]])
