"""train() after poisoning the caching allocator with NaN-filled freed blocks: a
read of never-written device memory then shows up as a changed result."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2303_01277_b200.codec import QuantConfig
from paper_2303_01277_b200.trainer import ModelConfig, TrainMode, train
from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
from paper_2303_01277_b200.graph import build_partitions
g = generate_sbm(SbmSpec(nodes_per_community=20, communities=4, feature_dim=32, seed=13))
parts = build_partitions(g, 3, "contiguous", 0, "gcn")[2]
def run(bits, var, st, ep=4):
    return train(g, parts, ModelConfig((32, 8, 4), dropout=0.2), TrainMode(var, st), QuantConfig(bits), ep, 7,
                 evaluate_each_epoch=False)
for cfg in [(2, "async", 2), (2, "sync", 0), (32, "async", 2), (1, "async", 0), (1, "async", 1)]:
    a = run(*cfg)
    torch.cuda.synchronize(); torch.cuda.empty_cache()
    junk = [torch.full((1 << k,), float("nan"), device="cuda") for k in range(8, 24)]
    junk += [torch.full((3 * (1 << k),), 12345.0, device="cuda") for k in range(8, 22)]
    del junk
    b = run(*cfg)
    print(cfg, [float(np.abs(x - y).max()) for x, y in zip(a.final_weights, b.final_weights)],
          [m.train_loss for m in b.metrics], flush=True)
