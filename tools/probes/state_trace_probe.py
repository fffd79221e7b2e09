"""After every C-ABI call of train(), hash every device tensor the DeviceRank
holds; compare the first train() in the process with a second identical one."""
import os, sys, hashlib
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2303_01277_b200 import _lib, trainer
from paper_2303_01277_b200.codec import QuantConfig
from paper_2303_01277_b200.trainer import ModelConfig, TrainMode, train
from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
from paper_2303_01277_b200.graph import build_partitions
eng = [None]
init = trainer.DeviceRank.__init__
def hooked(self, *a, **k):
    init(self, *a, **k)
    eng[0] = self
trainer.DeviceRank.__init__ = hooked

def tensors(obj, prefix, out, depth=0):
    if depth > 3:
        return
    if isinstance(obj, torch.Tensor):
        if obj.is_cuda:
            out[prefix] = obj
    elif isinstance(obj, (list, tuple)):
        for i, x in enumerate(obj):
            tensors(x, f"{prefix}[{i}]", out, depth + 1)
    elif isinstance(obj, dict):
        for i, (k, x) in enumerate(obj.items()):
            kk = f"#{i}" if "1398" in repr(k) or (isinstance(k, int) and k > (1 << 32)) else repr(k)
            tensors(x, f"{prefix}[{kk}]", out, depth + 1)
    elif hasattr(obj, "__dict__") and type(obj).__module__.startswith("paper_2303"):
        for k, x in vars(obj).items():
            tensors(x, f"{prefix}.{k}", out, depth + 1)

log = []
orig = _lib.call
def call(name, *args):
    r = orig(name, *args)
    if eng[0] is not None:
        torch.cuda.synchronize()
        ts = {}
        tensors(eng[0], "eng", ts)
        h = {k: hashlib.md5(t.detach().contiguous().view(-1).view(torch.uint8).cpu().numpy().tobytes()).hexdigest()[:8]
             for k, t in ts.items() if t.numel()}
        log.append((name, h))
    return r
_lib.call = call
g = generate_sbm(SbmSpec(nodes_per_community=20, communities=4, feature_dim=32, seed=13))
parts = build_partitions(g, 3, "contiguous", 0, "gcn")[2]
logs = []
for _ in range(2):
    log.clear(); eng[0] = None
    train(g, parts, ModelConfig((32, 8, 4), dropout=0.2), TrainMode("async", 2), QuantConfig(2), 4, 7,
          evaluate_each_epoch=False)
    logs.append(list(log))
a, b = logs
print(len(a), len(b))
for i, ((n1, h1), (n2, h2)) in enumerate(zip(a, b)):
    diff = sorted(k for k in set(h1) | set(h2) if h1.get(k) != h2.get(k))
    if diff:
        print("first diff after call", i, n1, n2, diff[:20])
        print("calls before:", [x[0] for x in a[max(0, i - 6):i + 1]])
        break
else:
    print("identical")
