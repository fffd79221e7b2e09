"""Per-kernel CUDA-event timing used by bench.py (and NVTX-free by design).

``KernelTimer`` brackets each instrumented launch with a pair of CUDA events
recorded on the launching (current) stream and accumulates the algorithmic
bytes the caller attributes to that launch.  ``DeviceRank`` calls
``timer(name, nbytes)`` around its K1/K2/K3/K4 launches when a timer is set.
"""

from __future__ import annotations

from contextlib import contextmanager, nullcontext


class KernelTimer:
    def __init__(self):
        import torch
        self.torch = torch
        self.records = []        # (name, nbytes, flops, start_event, end_event)
        self.enabled = True

    @contextmanager
    def __call__(self, name: str, nbytes: int = 0, flops: int = 0):
        if not self.enabled:
            yield
            return
        s = self.torch.cuda.Event(enable_timing=True)
        e = self.torch.cuda.Event(enable_timing=True)
        s.record()
        try:
            yield
        finally:
            e.record()
            self.records.append((name, int(nbytes), int(flops), s, e))

    def summary(self) -> dict:
        """name -> {launches, ms, bytes, flops, gbps, tflops} (call after a sync)."""
        out = {}
        for name, nb, fl, s, e in self.records:
            d = out.setdefault(name, dict(launches=0, ms=0.0, bytes=0, flops=0))
            d["launches"] += 1
            d["ms"] += s.elapsed_time(e)
            d["bytes"] += nb
            d["flops"] += fl
        for d in out.values():
            sec = d["ms"] / 1e3
            d["gbps"] = d["bytes"] / sec / 1e9 if sec > 0 else 0.0
            d["tflops"] = d["flops"] / sec / 1e12 if sec > 0 else 0.0
        return out

    def reset(self):
        self.records = []


def null_timer(name: str, nbytes: int = 0, flops: int = 0):
    return nullcontext()
