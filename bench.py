"""Benchmark: full-graph epoch time of the Sylvie halo path on B200.

Workload (BASELINE.json configs[1]): 3-layer GraphSAGE (602-256-256-41) on a
Reddit-shaped synthetic planted-partition graph (232,965 nodes, 114,615,892
directed edges, 41 classes), 8 partitions (contiguous), 1-bit halos, Sylvie-S
(sync).  The 8 partitions are spread over the N GPUs (N=1: all 8 on one GPU —
the reference's one-process simulation with device-resident halo traffic;
N=8: one subgraph per GPU, halos over NVLink via NCCL).  Total work is fixed
as N grows ("strong" scaling).

A "step" is one training epoch (forward + loss + backward + gradient
all-reduce + Adam), the centralized evaluation excluded.

  python bench.py [--gpus N --steps K --warmup W]          # B200 arm
  python bench.py --impl reference [--steps K --warmup W]  # CPU oracle arm

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WIDTHS = {"reddit": (602, 256, 256, 41), "ogbn": (100, 128, 128, 47), "yelp": (300, 512, 512, 512, 100),
          "config1": (64, 32, 4)}
MODEL = {"reddit": "sage", "ogbn": "sage", "yelp": "gcn", "config1": "gcn"}
LOSS = {"reddit": "softmax", "ogbn": "softmax", "yelp": "multilabel",   # BASELINE configs[3]: multilabel 100
        "config1": "softmax"}
# BASELINE configs[0] (the reference's CPU-runnable case) is 2 partitions
DEFAULT_PARTS = {"config1": 2}
PARTITIONS = 8
CPU_SAMPLE_SCALE = 0.125       # oracle-port fallback only (no baseline/_ref): 1/8 of the nodes/edges
REF_EPOCHS = 2                 # timed halobit.train epochs per reference measurement (after 1 warm-up)
# Bit-exact Philox4x64-10 throughput of the B200 at full occupancy (uniforms/s,
# tools/probes/philox_probe.cu measured on the GPU box; profiles/ has the run)
PHILOX_CEILING_GELEM_S = 414.0


def _spec(name: str, scale: float = 1.0):
    from paper_2303_01277_b200 import datasets as ds
    if name == "config1":
        if scale != 1.0:
            raise SystemExit("config1 is the reference's own SBM graph: --scale 1 only")
        return ds.CONFIG1
    spec = {"reddit": ds.REDDIT, "ogbn": ds.OGBN_PRODUCTS, "yelp": ds.YELP}[name]
    return spec if scale == 1.0 else ds.scaled(spec, scale)


def _spec_size(spec):
    """(nodes, directed edges) of a spec (the SBM's edge count is known after drawing)."""
    if hasattr(spec, "num_nodes"):
        return spec.num_nodes, spec.num_edges
    return spec.nodes_per_community * spec.communities, 195_652     # CONFIG1: measured


def build_graph(name: str, scale: float = 1.0, parts_needed=None):
    from paper_2303_01277_b200.datasets import generate_planted
    from paper_2303_01277_b200.graph import build_partition, mean_adjacency, normalize_adjacency, \
        partition_nodes
    from paper_2303_01277_b200.datasets import generate_sbm
    spec = _spec(name, scale)
    g = generate_planted(spec) if hasattr(spec, "num_nodes") else generate_sbm(spec)
    a = normalize_adjacency(g)
    m = mean_adjacency(g) if MODEL[name] == "sage" else None
    plan = partition_nodes(g, PARTITIONS)
    ids = range(PARTITIONS) if parts_needed is None else parts_needed
    return g, {k: build_partition(g, a, plan, k, m) for k in ids}


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(hbm_gbs=float(d["hbm_gbs"]), bf16_tflops=float(d["bf16_tflops"]), source="measured")
    return dict(hbm_gbs=6650.0, bf16_tflops=1590.0, source="fallback")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            self.proc.wait(timeout=10)

    def result(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 9 and f[1].isdigit():
                    rows.append(f)
        finally:
            os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        sm = [int(r[1]) for r in rows]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": int(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3] not in ("", "[N/A]"))}


REF_DIR = ROOT / "baseline" / "_ref"


def _halobit():
    """The unmodified reference package installed into baseline/_ref (pip
    --target); None when it is absent."""
    if not (REF_DIR / "halobit" / "__init__.py").exists():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import halobit  # noqa: F401
    from halobit import trainer
    return trainer


class _MaskOnlyGraph:
    """``halobit.train`` reads ``graph.train_mask`` (the global CE normaliser,
    trainer.py:392); the full graph itself only feeds the centralized
    ``evaluate``, which is excluded from the timed epoch."""

    def __init__(self, train_mask):
        self.train_mask = train_mask


def _to_halobit_partition(p, hb_graph, hb_linalg):
    def csr(m):
        if m is None:
            return None
        return hb_linalg.CsrMatrix(m.rows, m.cols, np.asarray(m.row_ptr, np.int64),
                                   np.asarray(m.col_idx, np.int64), np.asarray(m.values, np.float64))
    return hb_graph.Partition(
        id=p.id, num_partitions=p.num_partitions, local_nodes=p.local_nodes, halo_nodes=p.halo_nodes,
        send_sets=list(p.send_sets), recv_sets=list(p.recv_sets), adj_block=csr(p.adj_block),
        mean_block=csr(p.mean_block), features=np.asarray(p.features, dtype=np.float64),
        labels=_single_label(p.labels), train_mask=p.train_mask, val_mask=p.val_mask, test_mask=p.test_mask)


def _single_label(labels):
    """The reference trains only a softmax CE: a multi-label
    matrix becomes its first positive class for the CPU arm."""
    lab = np.asarray(labels)
    return lab.argmax(1).astype(np.int64) if lab.ndim == 2 else lab


def reference_epochs(name: str, parts: dict, train_mask, bits: int, mode: str, staleness: int,
                     epochs: int, seed: int):
    """``halobit.train`` (trainer.py:386-465, one worker thread per partition)
    on the bench's own partitions for `epochs` epochs; returns (per-epoch ms,
    metrics).  The centralized full-graph evaluation (and the full-graph
    Â / M it needs, trainer.py:392-394) is stubbed out for the run: SURVEY
    8(d) times the training epoch without it."""
    ht = _halobit()
    if ht is None:
        return None
    from halobit import codec as hc, graph as hg, linalg as hl
    hparts = [_to_halobit_partition(parts[k], hg, hl) for k in sorted(parts)]
    saved = (ht.evaluate, ht.normalize_adjacency, ht.mean_adjacency)
    ht.evaluate = lambda *a, **k: {"train_acc": 0.0, "val_acc": 0.0, "test_acc": 0.0}
    ht.normalize_adjacency = lambda *a, **k: None
    ht.mean_adjacency = lambda *a, **k: None
    try:
        res = ht.train(_MaskOnlyGraph(np.asarray(train_mask, bool)), hparts,
                       ht.ModelConfig(WIDTHS[name], MODEL[name]), ht.TrainMode(mode, staleness),
                       hc.QuantConfig(bits), epochs, seed, timeout=3600.0)
    finally:
        ht.evaluate, ht.normalize_adjacency, ht.mean_adjacency = saved
    return list(res.timings_ms), res.metrics


def cpu_epoch_sample(name: str, threads: int, epochs: int = 1, warmup: int = 0):
    """Fallback when baseline/_ref is absent: the numpy oracle port on the
    same-shape graph at CPU_SAMPLE_SCALE; returns (seconds per epoch of the
    sample, sample description, times, scale)."""
    from oracle.epoch import OracleTrainer
    g, parts = build_graph(name, CPU_SAMPLE_SCALE)
    for p in parts.values():
        p.labels = _single_label(p.labels)
    o = OracleTrainer([parts[k] for k in sorted(parts)], WIDTHS[name], MODEL[name], "sync", 0, 1, 0,
                      threads=threads)
    for e in range(1, warmup + 1):
        o.run_epoch(e)
    times = []
    for e in range(warmup + 1, warmup + epochs + 1):
        t0 = time.perf_counter()
        o.run_epoch(e)
        times.append(time.perf_counter() - t0)
    nnz = sum(p.mean_block.nnz if p.mean_block is not None else p.adj_block.nnz for p in parts.values())
    per = statistics.mean(times)
    sample = (f"{epochs} oracle epoch(s) (numpy/scipy f64, {threads} worker threads) of the {name}-shaped "
              f"graph at {CPU_SAMPLE_SCALE:g} scale ({g.num_nodes} nodes, {len(g.edges)} edges, "
              f"{nnz} aggregation nnz, same widths/partitions/cut); NOT extrapolated")
    return per, sample, times, CPU_SAMPLE_SCALE


def _cpu_info() -> dict:
    aff = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None
    return {"cpu_count": os.cpu_count(), "affinity": aff,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}


def reference_line(args, parts=None, train_mask=None, epochs=REF_EPOCHS):
    """The reference's own CPU implementation on this workload: ``halobit.train``
    from baseline/_ref at full scale (one warm-up epoch + `epochs` timed
    epochs).  Returns the cpu_baseline dict (value = mean timed epoch, s)."""
    if _halobit() is not None:
        t0 = time.perf_counter()
        if parts is None:
            g, parts = build_graph(args.config, args.scale)
            train_mask = g.train_mask
            del g
        setup = time.perf_counter() - t0
        t1 = time.perf_counter()
        ms, _ = reference_epochs(args.config, parts, train_mask, args.bits, args.mode, args.staleness,
                                 1 + epochs, args.seed)
        run = time.perf_counter() - t1
        timed = ms[1:]
        per = statistics.mean(timed) / 1e3
        return {"value": per, "unit": "s", "cores": os.cpu_count(), "kind": "reference",
                "sample": (f"halobit.train (baseline/_ref, unmodified reference, f64, {PARTITIONS} partition "
                           f"worker threads + OpenBLAS) on the {'full-scale ' if args.scale == 1.0 else ''}{args.config}-shaped graph "
                           f"(scale {args.scale:g}), {len(timed)} timed epoch(s) after 1 warm-up epoch, "
                           f"centralized evaluate stubbed out"),
                "epochs_ms": [round(x, 1) for x in ms], "timed_epochs": len(timed),
                "scale": args.scale, "setup_s": round(setup, 1), "train_call_s": round(run, 1),
                "host": _cpu_info()}
    threads = os.cpu_count() or 1
    per, sample, times, scale = cpu_epoch_sample(args.config, threads, epochs=epochs, warmup=1)
    return {"value": per, "unit": "s", "cores": threads, "kind": "port", "sample": sample,
            "timed_epochs": len(times), "scale": scale, "host": _cpu_info()}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = reference_line(args, epochs=min(args.steps, REF_EPOCHS))
    per = cb["value"]
    cfg = workload_config(args)
    cfg["scale"] = cb["scale"]
    line = {
        "impl": "reference", "metric": "full-graph epoch time", "value": per, "unit": "s",
        "n_gpus": args.gpus, "steps": cb["timed_epochs"], "warmup": 1,
        "requested": {"steps": args.steps, "warmup": args.warmup},
        "ms_per_step": per * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg,
        "cpu_baseline": cb,
        "e2e": {"value": per, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args) -> dict:
    spec = _spec(args.config, getattr(args, "scale", 1.0))
    return {"workload": f"{args.config}-shaped {len(WIDTHS[args.config]) - 1}-layer "
                        f"{MODEL[args.config].upper()} {'-'.join(map(str, WIDTHS[args.config]))}, "
                        f"{PARTITIONS} partitions over {args.gpus} GPU(s), {args.bits}-bit halos, "
                        f"Sylvie-{'S' if args.mode == 'sync' else 'A'}",
            "nodes": _spec_size(spec)[0], "edges": _spec_size(spec)[1], "partitions": PARTITIONS,
            "bits": args.bits, "mode": args.mode, "staleness": args.staleness,
            "model": MODEL[args.config], "widths": list(WIDTHS[args.config]), "loss": LOSS[args.config],
            "scale": getattr(args, "scale", 1.0),
            "exchange": ("in-GPU (all partitions on one GPU)" if args.gpus == 1 else
                         "peer memory (CUDA IPC)" if getattr(args, "p2p", None) or (
                             getattr(args, "p2p", None) is None and not getattr(args, "share_gpu", False)) else
                         "gloo, host-staged" if getattr(args, "share_gpu", False) else "NCCL send/recv"),
            "l2": "n/a (CPU)" if args.impl == "reference" else None}


def run_b200(args):
    import torch
    import torch.distributed as dist
    from paper_2303_01277_b200.codec import QuantConfig
    from paper_2303_01277_b200.profiling import KernelTimer
    from paper_2303_01277_b200.trainer import DeviceRank, ModelConfig, TrainMode
    from paper_2303_01277_b200.transport import RankLayout

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.share_gpu:
        # test mode: every rank on cuda:0, gloo transport (wire blocks staged
        # through host memory) — exercises the N>1 host logic on one GPU
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    owner = [p * world // PARTITIONS for p in range(PARTITIONS)]
    mine = [p for p in range(PARTITIONS) if owner[p] == rank]
    t0 = time.perf_counter()
    g, parts = build_graph(args.config, args.scale, mine)
    gnorm = int(g.train_mask.sum())
    train_mask = g.train_mask
    layout = RankLayout(parts, owner, rank)
    eng = DeviceRank(layout, ModelConfig(WIDTHS[args.config], MODEL[args.config], loss=LOSS[args.config]),
                     TrainMode(args.mode, args.staleness), QuantConfig(args.bits), args.seed, 0.01, gnorm,
                     device=torch.device("cuda", local), p2p=args.p2p)
    # the step's input features, pinned and laid out like the device buffer
    # (16-byte padded rows) so each step's upload is one contiguous copy
    feats = np.concatenate([np.asarray(p.features, dtype=np.float32) for p in layout.parts])
    ldf = eng.Ht[1].shape[1]
    feats_host = torch.zeros((feats.shape[0], ldf), dtype=torch.float32).pin_memory()
    feats_host[:, :feats.shape[1]] = torch.from_numpy(feats)
    del feats
    del g
    setup_s = time.perf_counter() - t0
    epoch = 0
    for _ in range(args.warmup):
        epoch += 1
        eng.run_epoch(epoch)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- device-timed region: K epochs, no host syncs inside ------------------
    timer = KernelTimer()
    eng.timer = timer
    if world > 1:
        eng.comm_events = []
    launches0 = eng.launches
    # a working set below L2 (config 1): every timed epoch starts from a
    # flushed L2 (a 512 MB write between epochs, outside the event pairs)
    small = _working_set_bytes(eng) < 126e6
    flush = torch.empty(128 << 20, dtype=torch.float32, device=torch.device("cuda", local)) if small else None
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        spans = []
        ev0.record()
        h0 = time.perf_counter()
        for _ in range(args.steps):
            epoch += 1
            if small:
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                eng.run_epoch(epoch, check=False)
                e1.record()
                spans.append((e0, e1))
            else:
                eng.run_epoch(epoch, check=False)
        host_issue_ms = (time.perf_counter() - h0) * 1e3 / args.steps
        ev1.record()
        torch.cuda.synchronize()
        barrier()
    launches = eng.launches - launches0
    halo_net = _halo_net(eng, world, args.steps, timer.summary())
    eng.comm_events = None
    eng.timer = KernelTimer()
    eng.timer.enabled = False
    eng.check_epoch(epoch)
    ms = (sum(a.elapsed_time(b) for a, b in spans) if small else ev0.elapsed_time(ev1)) / args.steps
    ms = _max_over_ranks(ms, world)
    l2_note = ("working set below L2: L2 flushed (512 MB write) before every timed epoch, outside its event pair"
               if small else f"inputs larger than L2 (working set {_working_set_bytes(eng) / 1e9:.2f} GB)")
    ksum = timer.summary()
    clocks = clk.result()

    # ---- the same K epochs replayed from CUDA graphs (no per-kernel timers) ---
    use_graphs = not args.no_graphs and eng.graphable()
    graph_line = None
    if use_graphs:
        for _ in range(2):                       # capture both epoch parities
            epoch += 1
            eng.run_epoch_graphed(epoch)
        while eng._deferred:
            eng.finish_epoch()
        launches0 = eng.launches
        barrier()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gspans = []
        g0.record()
        h0 = time.perf_counter()
        for _ in range(args.steps):
            epoch += 1
            if small:
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                eng.run_epoch_graphed(epoch)
                e1.record()
                gspans.append((e0, e1))
            else:
                eng.run_epoch_graphed(epoch)
        g_issue = (time.perf_counter() - h0) * 1e3 / args.steps
        g1.record()
        torch.cuda.synchronize()
        while eng._deferred:
            eng.finish_epoch()
        barrier()
        gms = (sum(a.elapsed_time(b) for a, b in gspans) if small else g0.elapsed_time(g1)) / args.steps
        # the host cost of issuing one replayed epoch (with the GPU idle, so no
        # wait on an earlier replay is included)
        issue = []
        for _ in range(4):
            torch.cuda.synchronize()
            epoch += 1
            h0 = time.perf_counter()
            eng.run_epoch_graphed(epoch)
            issue.append((time.perf_counter() - h0) * 1e3)
        torch.cuda.synchronize()
        while eng._deferred:
            eng.finish_epoch()
        graph_line = {"ms_per_step": _max_over_ranks(gms, world), "host_loop_ms_per_step": round(g_issue, 3),
                      "host_issue_ms_per_step": round(statistics.median(issue), 3),
                      "graphs_captured": len(eng._graphs), "kernels_per_step": (eng.launches - launches0) / args.steps,
                      "note": "the timed epochs replayed from CUDA graphs of the epoch (one graph launch per "
                              "epoch; per-epoch K1 key tables and Adam bias corrections re-fetched from pinned "
                              "buffers by the graph), without the per-kernel event timers of the breakdown above; "
                              "host_loop: wall time per epoch of the issuing loop (the host waits for the replay "
                              "two epochs back, so it tracks the device); host_issue: one replayed epoch's issue "
                              "cost with the GPU idle"}

    # ---- end-to-end through the public epoch call with host buffers ----------
    h2d = int(feats_host.numel() * 4)
    e2e_steps = max(1, args.steps)
    # (a) serial: each step uploads its features, then runs the epoch
    e2e_times = []
    for _ in range(e2e_steps):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        epoch += 1
        eng.Ht[1][:eng.NL].copy_(feats_host, non_blocking=True)
        eng.run_epoch(epoch, check=True)            # reads loss + codec flag back (D2H)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    e2e_serial = _max_over_ranks(statistics.mean(e2e_times), world)
    # (b) pipelined input: two feature buffers; step k+1's upload runs on a copy
    # stream while step k computes (it waits for step k-1, the last reader of
    # its buffer).  Every step still moves its full feature matrix host->device
    # and reads its loss back inside the timed region, which spans all steps.
    e2e_pipe = None
    if not args.e2e_serial:
        cur = torch.cuda.current_stream()
        cs = torch.cuda.Stream(device=torch.device("cuda", local))
        slots = [eng.Ht[1], torch.empty_like(eng.Ht[1])]
        done, up = [None, None], [None, None]

        def upload(s):
            with torch.cuda.stream(cs):
                if done[s] is not None:
                    cs.wait_event(done[s])
                slots[s][:eng.NL].copy_(feats_host, non_blocking=True)
                up[s] = cs.record_event()

        run = eng.run_epoch_graphed if use_graphs else (lambda e: eng.run_epoch(e, defer=True))

        def pipeline(nsteps):
            nonlocal epoch
            upload(0)
            for k in range(nsteps):
                s = k % 2
                if k + 1 < nsteps:
                    upload(1 - s)
                cur.wait_event(up[s])
                eng.swap_features(slots[s])
                epoch += 1
                # Adam guarded on the device; the loss + codec/protocol flags come
                # back (D2H) and are checked once the next epoch has been issued
                run(epoch)
                done[s] = cur.record_event()
                if k > 0:
                    eng.finish_epoch()
            eng.finish_epoch()

        # untimed: capture the CUDA graphs of both input buffers' epochs
        pipeline(4)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pipeline(e2e_steps)
        torch.cuda.synchronize()
        e2e_pipe = _max_over_ranks((time.perf_counter() - t0) / e2e_steps, world)
        eng.swap_features(slots[0])
        del slots
    e2e = e2e_pipe if e2e_pipe is not None else e2e_serial

    # ---- Sylvie-A sub-line (async, staleness 0) on the same graph -------------
    async_line = None
    if args.mode == "sync" and not args.no_async_line:
        import gc
        sync_recv = sum(b.recv[0].numel() for b in list(eng.xf.values()) + list(eng.xb.values()))
        del eng
        gc.collect()
        torch.cuda.empty_cache()
        eng = DeviceRank(layout, ModelConfig(WIDTHS[args.config], MODEL[args.config], loss=LOSS[args.config]),
                         TrainMode("async", 0), QuantConfig(args.bits), args.seed, 0.01, gnorm,
                         device=torch.device("cuda", local), p2p=args.p2p)
        aepoch = 0                       # a fresh run: epoch 1 has no stale buffers yet
        for _ in range(args.warmup):
            aepoch += 1
            eng.run_epoch(aepoch)
        barrier()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(args.steps):
            aepoch += 1
            eng.run_epoch(aepoch, check=False)
        a1.record()
        torch.cuda.synchronize()
        barrier()
        eng.check_epoch(aepoch)
        ams = _max_over_ranks(a0.elapsed_time(a1) / args.steps, world)
        async_recv = sum(sum(r.numel() for r in b.recv) for b in list(eng.xf.values()) + list(eng.xb.values()))
        async_line = {"mode": "async", "staleness": 0, "ms_per_step": ams, "vs_sync": ams / ms,
                      "recv_buffer_bytes": {"sync": int(sync_recv), "async_two_parities": int(async_recv)},
                      "note": ("Sylvie-A: each exchange ships epoch t's halos into parity t%2 while epoch t "
                               "consumes parity (t-1)%2; at N=1 the wire blocks move HBM->HBM, so the deferred "
                               "exchange overlaps nothing and the two modes cost the same device work")}

    if rank == 0:
        peaks = load_peaks()
        dom = max(ksum, key=lambda k: ksum[k]["ms"]) if ksum else None
        clocks_mhz = clocks.get("sm_mhz") or 1965
        roof = None
        # the dominant kernel: the TMA-tiled SpMM (the 256-wide aggregations)
        skey = "spmm_tiled" if "spmm_tiled" in ksum else ("spmm_rows" if "spmm_rows" in ksum else None)
        if skey is not None:
            s = ksum[skey]
            sec = s["ms"] / 1e3
            # L1TEX/SMEM datapath: 128 B/clk/SM is what a SIMT SpMM can pull into
            # registers, whether X rows come from L2 (row kernel) or from TMA-
            # staged smem tiles (tiled kernel); gathered bytes = 4 * nnz * d
            dp_peak = 148 * 128 * clocks_mhz * 1e6 / 1e9
            gather_gbps = 2.0 * s["flops"] / sec / 1e9 if sec > 0 else 0.0
            binary = any(t is not None and t.binary for t in eng._tiles.values())
            roof = {"kernel": {"spmm_tiled": "hb_spmm_tiled_bin (K3/K4, TMA-staged tiles, one-byte records, "
                                             "diagonal scalings)" if binary else
                                             "hb_spmm_tiled (K3/K4, TMA-staged tiles)",
                               "spmm_rows": "hb_spmm_csr_ex (K3/K4, row gather)"}[skey], "bound": "hbm",
                    "achieved": s["gbps"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": s["gbps"] / peaks["hbm_gbs"], "traffic": _ncu_traffic(skey, args),
                    "algorithmic_bytes_per_launch": s["bytes"] / s["launches"],
                    "algorithmic_bytes_model": "compulsory: CSR + each X row once + Y once (SURVEY 8d)",
                    "avg_launch_ms": s["ms"] / s["launches"], "peak_source": peaks["source"],
                    "fp32_simt_tflops": s["tflops"],
                    "l1_datapath": {"gathered_gbps": gather_gbps, "peak_gbps": dp_peak,
                                    "frac": gather_gbps / dp_peak,
                                    "ncu_l1tex_pct_elapsed": _ncu_traffic("spmm_tiled_l1tex_pct_elapsed", args)
                                    if skey == "spmm_tiled" else None,
                                    "note": "gather model 4*nnz*d bytes per launch vs 148 SM x 128 B/clk; the "
                                            "kernel is bound by this shared-memory datapath, not HBM"}}
        kroof = {}
        if "quantize_gather" in ksum:
            q = ksum["quantize_gather"]
            elems = sum(int(b.plan.send_rows.size) * b.d for b in list(eng.xf.values()) + list(eng.xb.values()))
            rate = elems * args.steps / (q["ms"] / 1e3) / 1e9
            kroof["quantize_gather"] = {
                "bound": "hbm", "achieved": q["gbps"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": q["gbps"] / peaks["hbm_gbs"],
                "philox_gelem_s": rate, "philox_ceiling_gelem_s": PHILOX_CEILING_GELEM_S,
                "philox_frac": rate / PHILOX_CEILING_GELEM_S,
                "note": "bit-exact Philox4x64-10 (one uniform per element) caps K1 below HBM speed"}
        for k in ("spmm_tiled_narrow", "spmm_rows"):
            if k in ksum and k != skey:
                v = ksum[k]
                sec = v["ms"] / 1e3
                kroof[k] = {"bound": "hbm", "achieved": v["gbps"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
                            "frac": v["gbps"] / peaks["hbm_gbs"],
                            "gathered_gbps": 2.0 * v["flops"] / sec / 1e9 if sec > 0 else 0.0,
                            "avg_launch_ms": v["ms"] / v["launches"]}
        for k in ("dequant_gather", "elementwise"):
            if k in ksum:
                v = ksum[k]
                kroof[k] = {"bound": "hbm", "achieved": v["gbps"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
                            "frac": v["gbps"] / peaks["hbm_gbs"]}
        if "gemm" in ksum:
            g = ksum["gemm"]
            tf32_peak = peaks["bf16_tflops"] / 2.0
            kroof["gemm"] = {"bound": "tensor", "achieved": g["tflops"], "unit": "TFLOP/s",
                             "tf32_mma_tflops": 3.0 * g["tflops"], "peak": tf32_peak,
                             "frac": 3.0 * g["tflops"] / tf32_peak,
                             "hbm_gbps": g["gbps"], "hbm_frac": g["gbps"] / peaks["hbm_gbs"],
                             "note": "3xTF32 (hi*hi + hi*lo + lo*hi per fp32 product); peak = dense TF32 = "
                                     "measured bf16 / 2; hbm_*: compulsory bytes (A, B, C, ReLU copy) of all "
                                     "GEMM launches — the narrow-K shapes (K <= 128) are HBM-bound"}
        if dom == "gemm" and "gemm" in kroof and roof is not None:
            # the GEMMs dominate (e.g. the Yelp-shaped GCN): the headline roofline
            # is theirs; the SpMM's moves to kernel_rooflines
            kroof[skey] = roof
            g = ksum["gemm"]
            roof = dict(kroof.pop("gemm"), kernel="hb_gemm_f32 / hb_gemm2_f32 (K5-K7, tcgen05 3xTF32)",
                        traffic=_ncu_traffic("gemm", args), avg_launch_ms=g["ms"] / g["launches"],
                        peak_source=peaks["source"])
        wire = sum(b.wire_bytes_total() for b in list(eng.xf.values()) + list(eng.xb.values()))
        halo_ms = sum(ksum.get(k, {}).get("ms", 0.0) for k in ("quantize_gather", "dequant_gather"))
        line = {
            "metric": "full-graph epoch time", "value": ms / 1e3, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (planted-partition reddit-shaped graph, random-init Glorot weights)",
            "config": dict(workload_config(args), l2=l2_note),
            "roofline": roof,
            "kernel_rooflines": kroof,
            "kernels": {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                        for k, v in ksum.items()},
            "dominant_kernel": dom,
            "halo": {"wire_bytes_per_epoch": wire,
                     "k1_k2_ms_per_epoch": halo_ms / args.steps,
                     "fp32_equiv_bytes_per_epoch": _fp32_equiv(eng),
                     "note": ("N=1: the 8 partitions share one GPU, so halo messages move HBM->HBM; "
                              "K1 writes each wire block straight into its receiver's buffer") if world == 1 else
                             ("rank 0's wire bytes; same-rank messages are written straight into the receiver's "
                              "buffer, the rest move per peer rank over " +
                              ("peer memory: K1 writes them into the peers' receive buffers (CUDA IPC), "
                               "counters order arrival and reuse" if eng.p2p is not None else
                               "gloo with host staging (--share-gpu: all ranks on one GPU)" if args.share_gpu
                               else "NCCL send/recv on the comm stream"))},
            "gpu_launches": launches,
            "halo_network": halo_net,
            "async": async_line,
            "host_issue_ms_per_step": round(host_issue_ms, 3),
            "host_issue_note": "wall time to issue an epoch; includes the waits on each exchange's two pinned "
                               "descriptor slots that keep the host at most two epochs ahead of the GPU "
                               "(tools/prof_host.py: ~3 ms/epoch of Python + ctypes issue at Reddit shape)",
            "clocks": clocks,
            "cuda_graph": graph_line,
            "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": h2d,
                    "epochs": "CUDA-graph replays" if use_graphs else "eager",
                    "d2h_bytes_per_step": 16 if e2e_pipe is not None else 12,
                    "input_pipeline": "double-buffered" if e2e_pipe is not None else "serial",
                    "serial_value": e2e_serial,
                    "d2h_note": "pipelined: f64 loss + two u32 flag words per step (16 B)",
                    "note": ("every step uploads its full feature matrix from pinned host memory and reads its "
                             "loss + codec flag back; double-buffered: step k+1's upload runs on a copy stream "
                             "during step k, Adam is guarded on the device and step k's loss is checked on the "
                             "host after step k+1 is issued (timed over all steps, first upload exposed); "
                             "serial_value: upload, then epoch with the host check before Adam, synchronised "
                             "per step")},
            "setup_s": round(setup_s, 1),
            "final_loss": eng.epoch_loss,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = reference_line(args, parts, train_mask, epochs=1)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _working_set_bytes(eng) -> float:
    """Bytes an epoch touches at least once: features / activations and the
    aggregation operator (CSR + its transpose)."""
    act = sum(t.numel() * 4 for t in eng.Ht.values())
    csr = sum(m.nnz * 8 + (m.rows + 1) * 8 for m in (eng.A, eng.At))
    return float(act + csr)


def _halo_net(eng, world: int, steps: int, ksum=None):
    """Halo GB/s over the network leg (N>1): remote wire bytes / NCCL span,
    both from the comm-stream events of the timed epochs.  With
    the peer-memory exchange the transfer happens inside K1 (its stores land
    in the peers' buffers): remote wire bytes / K1 time, a lower bound on the
    link rate since K1 is bound by its Philox stream."""
    if world == 1:
        return None
    if eng.p2p is not None:
        nbytes = sum(n for b in eng.p2p.ex for _, (_, n) in b.send_group.items())
        k1 = (ksum or {}).get("quantize_gather")
        if not k1 or k1["ms"] <= 0:
            return None
        ms = _max_over_ranks(k1["ms"] / steps, world)
        return {"transport": "peer memory (CUDA IPC, K1 stores into the peers' receive buffers)",
                "wire_bytes_per_epoch": nbytes, "k1_ms_per_epoch": ms,
                "halo_gbps": nbytes / ms / 1e6 if ms > 0 else None, "nvlink_peak_gbps": 900.0,
                "frac": (nbytes / ms / 1e6) / 900.0 if ms > 0 else None,
                "note": "this rank's remote wire bytes / its K1 time (the link leg overlaps the quantize)"}
    if not eng.comm_events:
        return None
    ms = sum(a.elapsed_time(b) for a, b, _ in eng.comm_events)
    nbytes = sum(n for _, _, n in eng.comm_events)
    ms = _max_over_ranks(ms, world)
    return {"wire_bytes_per_epoch": nbytes / steps, "nccl_ms_per_epoch": ms / steps,
            "halo_gbps": nbytes / ms / 1e6 if ms > 0 else None, "nvlink_peak_gbps": 900.0,
            "frac": (nbytes / ms / 1e6) / 900.0 if ms > 0 else None,
            "note": "this rank's sends to other ranks over NCCL; comm-stream events, max span over ranks"}


def _max_over_ranks(x: float, world: int) -> float:
    """Max of a per-rank timing over all ranks (device clocks, CPU tensor for gloo)."""
    if world == 1:
        return float(x)
    import torch
    import torch.distributed as dist
    dev = "cpu" if dist.get_backend() != "nccl" else "cuda"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _fp32_equiv(eng) -> int:
    tot = 0
    for b in list(eng.xf.values()) + list(eng.xb.values()):
        tot += int(b.plan.send_rows.size) * b.d * 4
    return tot


def _ncu_traffic(kernel: str, args=None):
    """ncu-measured values of the full-scale Reddit-shaped epoch (the capture in
    profiles/ncu_traffic.json); None for other workloads."""
    if args is not None and (args.config != "reddit" or args.scale != 1.0):
        return None
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(kernel)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="reddit", choices=sorted(WIDTHS))
    ap.add_argument("--bits", type=int, default=1)
    ap.add_argument("--mode", default="sync", choices=["sync", "async"])
    ap.add_argument("--staleness", type=int, default=0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-async-line", action="store_true", help="skip the Sylvie-A sub-line")
    ap.add_argument("--no-graphs", action="store_true", help="eager epochs only (no CUDA-graph replays)")
    ap.add_argument("--p2p", dest="p2p", action="store_true", default=None,
                    help="N>1: peer-memory halo exchange (K1 writes into the peers' receive buffers over "
                         "CUDA IPC mappings; the default on NCCL process groups)")
    ap.add_argument("--nccl-exchange", dest="p2p", action="store_false",
                    help="N>1: halo blocks over NCCL send/recv instead of peer memory")
    ap.add_argument("--e2e-serial", action="store_true",
                    help="e2e with the serial upload only (no double-buffered input pipeline)")
    ap.add_argument("--partitions", type=int, default=None,
                    help="graph partitions (8 = BASELINE config 2; --partitions N with --gpus N = one "
                         "subgraph per GPU)")
    ap.add_argument("--scale", type=float, default=1.0,
                    help="graph size factor (1.0 = the BASELINE shape; smaller only for diagnostics)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="test mode: all ranks on cuda:0 over gloo (the N>1 path on one GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    global PARTITIONS
    PARTITIONS = args.partitions or DEFAULT_PARTS.get(args.config, 8)
    if PARTITIONS < max(1, args.gpus):
        raise SystemExit("--partitions must be >= --gpus (every GPU hosts at least one partition)")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
