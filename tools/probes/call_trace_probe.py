"""Log the C-ABI call sequence (names + small scalar args) of the first train() in
the process and of a second identical one; print the first difference."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2303_01277_b200 import _lib
from paper_2303_01277_b200.codec import QuantConfig
from paper_2303_01277_b200.trainer import ModelConfig, TrainMode, train
from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
from paper_2303_01277_b200.graph import build_partitions
log = []
orig = _lib.call
def call(name, *args):
    log.append((name, tuple(a if isinstance(a, float) or (isinstance(a, int) and abs(a) < (1 << 32)) else "P"
                            for a in args)))
    return orig(name, *args)
_lib.call = call
import paper_2303_01277_b200.ops as ops
ops._lib.call = call
g = generate_sbm(SbmSpec(nodes_per_community=20, communities=4, feature_dim=32, seed=13))
parts = build_partitions(g, 3, "contiguous", 0, "gcn")[2]
logs = []
for _ in range(2):
    log.clear()
    train(g, parts, ModelConfig((32, 8, 4), dropout=0.2), TrainMode("async", 2), QuantConfig(2), 4, 7,
          evaluate_each_epoch=False)
    logs.append(list(log))
a, b = logs
print(len(a), len(b))
for i, (x, y) in enumerate(zip(a, b)):
    if x != y:
        print("first diff at", i, "\n", x, "\n", y)
        for j in range(max(0, i - 3), min(len(a), i + 8)):
            print(j, a[j], "|", b[j] if j < len(b) else None)
        break
else:
    print("identical call sequences")
