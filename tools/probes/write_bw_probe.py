import torch, json
x = torch.empty(460000, 604, device="cuda")
for _ in range(3): x.fill_(1.0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): x.fill_(2.0)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(json.dumps({"fill_bytes": x.numel() * 4, "ms": ms, "gbps": x.numel() * 4 / ms / 1e6}))
y = torch.empty_like(x)
e0.record()
for _ in range(20): y.copy_(x)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(json.dumps({"copy_bytes": 2 * x.numel() * 4, "ms": ms, "gbps": 2 * x.numel() * 4 / ms / 1e6}))
