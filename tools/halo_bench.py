"""Halo quantize/exchange microbenchmark (BASELINE.json configs[4]).

Per GPU a boundary set of R rows x d columns (fp32, rows scaled by U(0.1, 5)
as SURVEY 8d specifies) is split evenly over the peers; each step runs
  K1  hb_quantize_gather  (gather + Philox4x64-10 stochastic rounding + pack,
                           wire blocks written per peer)
  X   the exchange: NCCL all-to-all of the packed blocks on a side stream
      (N > 1); at N = 1 the blocks are written straight into the local
      receive buffer by K1 (8-way loopback, like the 8 hosted partitions)
  K2  hb_dequant_gather   (unpack + dequantize + scatter into halo rows)
for 1-bit and fp32 passthrough (bits 32).  Times are CUDA events on the
launching streams, max over ranks.  One JSON line per case on rank 0:
K1/K2 algorithmic GB/s and fraction of the measured HBM peak, Philox
G elements/s, wire bytes, halo GB/s over the exchange span (N > 1), and the
effective fp32-equivalent GB/s (R*d*4 / (K1 + X + K2)).

  python tools/halo_bench.py [--rows 10000 100000 1000000 10000000] [--d 128 256 512 1024]
  torchrun --nproc-per-node N tools/halo_bench.py ...
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    return json.loads(p.read_text())["hbm_gbs"] if p.exists() else 6650.0


def run_case(R, d, bits, world, rank, reps, warm):
    import torch
    import torch.distributed as dist
    from paper_2303_01277_b200.codec import dequant_gather, segments_tensor, wire_bytes
    from paper_2303_01277_b200.rngstream import derive_key
    dev = torch.device("cuda")
    ld = (d + 3) // 4 * 4
    peers = max(1, world - 1) if world > 1 else 7
    R = R // peers * peers                      # equal per-peer blocks: symmetric all-to-all splits
    g = torch.Generator(device=dev).manual_seed(2303 + rank)
    nsrc = R + R // 4
    src = torch.randn(nsrc, ld, device=dev, generator=g) * (0.1 + 4.9 * torch.rand(nsrc, 1, device=dev, generator=g))
    rows_idx = torch.randperm(nsrc, device=dev, generator=g)[:R].sort().values.to(torch.int32)
    counts = [R // peers] * peers
    sizes = [(wire_bytes(c, d, bits) + 15) // 16 * 16 for c in counts]
    send = torch.zeros(sum(sizes), dtype=torch.uint8, device=dev)
    recv = torch.zeros_like(send) if world > 1 else send
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    key = derive_key((2303, rank, 1, 1, "forward")) if bits != 32 else (0, 0)
    eoff = np.concatenate([[0], np.cumsum(counts)[:-1]]) * d
    segs_send = segments_tensor(counts, [key] * peers, [int(e) for e in eoff],
                                [send.data_ptr() + int(o) for o in offs], "cuda")
    segs_recv = segments_tensor(counts, [(0, 0)] * peers, [0] * peers,
                                [recv.data_ptr() + int(o) for o in offs], "cuda")
    dst = torch.zeros(R, ld, device=dev)
    dst_rows = torch.arange(R, dtype=torch.int32, device=dev)
    src_ptr = torch.arange(R + 1, dtype=torch.int32, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    from paper_2303_01277_b200.codec import quantize_gather
    comm = torch.cuda.Stream() if world > 1 else None
    split = [int(s) for s in sizes]

    def step(ev):
        ev[0].record()
        quantize_gather(src, rows_idx, segs_send, peers, d, bits, flags)
        ev[1].record()
        if world > 1:
            cur = torch.cuda.current_stream()
            with torch.cuda.stream(comm):
                comm.wait_stream(cur)
                ev[2].record(comm)
                # send block i goes to the i-th other rank; blocks arrive in
                # source-rank order into the same equal-sized slots
                sp = [0 if r == rank else split[0] for r in range(world)]
                dist.all_to_all_single(recv, send, sp, sp)
                ev[3].record(comm)
            cur.wait_stream(comm)
        else:
            ev[2].record()
            ev[3].record()
        dequant_gather(segs_recv, peers, dst_rows, src_ptr, dst_rows, d, bits, dst, False)
        ev[4].record()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(reps)]
    for _ in range(warm):
        step([torch.cuda.Event(enable_timing=True) for _ in range(5)])
    torch.cuda.synchronize()
    for ev in evs:
        step(ev)
    torch.cuda.synchronize()
    k1 = np.mean([e[0].elapsed_time(e[1]) for e in evs])
    xx = np.mean([e[2].elapsed_time(e[3]) for e in evs])
    k2 = np.mean([e[3].elapsed_time(e[4]) for e in evs])
    tot = np.mean([e[0].elapsed_time(e[4]) for e in evs])
    t = torch.tensor([k1, xx, k2, tot], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    k1, xx, k2, tot = t.tolist()
    wire = sum(wire_bytes(c, d, bits) for c in counts)
    k1_bytes = R * d * 4 + R * 4 + wire
    k2_bytes = wire + R * d * 4 + 12 * R
    hbm = _peaks()
    return {"rows": R, "d": d, "bits": bits, "n_gpus": world, "k1_ms": k1, "exchange_ms": xx, "k2_ms": k2,
            "step_ms": tot, "wire_bytes": wire,
            "k1_gbps": k1_bytes / k1 / 1e6, "k1_hbm_frac": k1_bytes / k1 / 1e6 / hbm,
            "k1_philox_gelem_s": (R * d / k1 / 1e6) if bits != 32 else None,
            "k2_gbps": k2_bytes / k2 / 1e6, "k2_hbm_frac": k2_bytes / k2 / 1e6 / hbm,
            "halo_gbps": (wire / xx / 1e6) if world > 1 and xx > 0 else None,
            "effective_fp32_gbps": R * d * 4 / tot / 1e6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, nargs="*", default=[10_000, 100_000, 1_000_000, 10_000_000])
    ap.add_argument("--d", type=int, nargs="*", default=[128, 256, 512, 1024])
    ap.add_argument("--bits", type=int, nargs="*", default=[1, 32])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--max-elems", type=float, default=2.6e9, help="skip cases with R*d above this")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    for R in a.rows:
        for d in a.d:
            if R * d > a.max_elems:
                continue
            for b in a.bits:
                res = run_case(R, d, b, world, rank, a.reps, a.warmup)
                if rank == 0:
                    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in res.items()}),
                          flush=True)
                torch.cuda.empty_cache()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
