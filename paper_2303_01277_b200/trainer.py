"""Sylvie-S / Sylvie-A training on the B200: drop-in for ``halobit.trainer``.

Public surface kept from the reference (``trainer.py:32-465``):
``ModelConfig``, ``TrainMode``, ``staleness_adaptor``, ``MetricsRecord``,
``TrainResult``, ``TrainingError``, ``init_weights``, ``train`` — same
arguments, same semantics, same exceptions.  Underneath, each rank (one per
GPU; a single rank hosts all partitions in the one-GPU case, exactly like the
reference's one-process simulation) runs the epoch on device-resident buffers:

  forward, layer l:   halo exchange (K1 -> [NCCL] -> K2)  |  Sylvie-A: consume
                      epoch t-1 halo, ship epoch t halo for t+1
                      p = A h~ (K3 SpMM)  [SAGE: p = [h~_local | M h~]]
                      z = p W (GEMM);  h = relu(z)
  loss:               masked softmax-CE with the global normaliser (K8)
  backward, layer l:  m = j * relu'(z);  G = p^T m;  j_full = A^T (m W^T) (K4)
                      halo gradient exchange, ascending-peer integration (K2)
  all-reduce(G), NaN check, Adam.

Numerics are fp32 (f64 in the reference); the codec decisions are bit-exact
given identical fp32 inputs (see codec.py).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import ops
from .codec import CodecError, QuantConfig, quantize_gather, dequant_gather
from .graph import Graph, Partition
from .linalg import ShapeError
from .profiling import null_timer
from .rngstream import BACKWARD, FORWARD, derive_key, keyed_generator
from .transport import SEG_BYTES, ExchangeBuffers, ProtocolError, RankLayout, TransportStats, nccl_exchange

MODELS = ("gcn", "sage")


class TrainingError(RuntimeError):
    pass


LOSSES = ("softmax", "multilabel")


@dataclass(frozen=True)
class ModelConfig:
    """``trainer.py:32-45``.  ``loss`` is an extension (default = the
    reference's masked softmax CE): "multilabel" trains a sigmoid BCE over a
    (nodes x classes) 0/1 label matrix and evaluates micro-F1 (the Yelp-shaped
    "multilabel 100" config; not in the reference)."""

    widths: tuple
    model: str = "gcn"
    dropout: float = 0.0
    loss: str = "softmax"

    def __post_init__(self):
        if len(self.widths) < 2 or any(w <= 0 for w in self.widths):
            raise TrainingError("widths must list input, hidden(s), and output dims")
        if self.model not in MODELS:
            raise TrainingError(f"unknown model {self.model!r}")
        if not (0.0 <= self.dropout < 1.0):
            raise TrainingError("dropout must be in [0, 1)")
        if self.loss not in LOSSES:
            raise TrainingError(f"unknown loss {self.loss!r}")

    @property
    def num_layers(self) -> int:
        return len(self.widths) - 1


@dataclass(frozen=True)
class TrainMode:
    variant: str = "sync"
    staleness: int = 0

    def __post_init__(self):
        if self.variant not in ("sync", "async"):
            raise TrainingError(f"unknown mode {self.variant!r}")
        if self.staleness < 0:
            raise TrainingError("staleness interval must be >= 0")


def staleness_adaptor(epoch: int, mode: TrainMode) -> str:
    """Bounded Staleness Adaptor (trainer.py:70-76)."""
    if mode.variant == "sync":
        return "sync"
    if mode.staleness > 0 and epoch % mode.staleness == 0:
        return "sync"
    return "async"


@dataclass
class MetricsRecord:
    epoch: int
    mode_this_epoch: str
    train_loss: float
    train_acc: float
    val_acc: float
    test_acc: float
    main_bytes: int
    meta_bytes: int
    header_bytes: int
    allreduce_bytes: int
    messages: int
    wall_ms: int = 0


@dataclass
class TrainResult:
    metrics: list
    final_weights: list
    timings_ms: list = field(default_factory=list)


def init_weights(cfg: ModelConfig, seed: int) -> list:
    """Glorot-uniform from keyed Philox (trainer.py:102-112); float64 host arrays."""
    out = []
    for l in range(1, cfg.num_layers + 1):
        fan_in = cfg.widths[l - 1] * (2 if cfg.model == "sage" else 1)
        lim = np.sqrt(6.0 / (fan_in + cfg.widths[l]))
        out.append(keyed_generator(seed, "init", l).uniform(-lim, lim, size=(fan_in, cfg.widths[l])))
    return out


def _ld(d: int) -> int:
    return (d + 3) // 4 * 4


def _stack_csr(layout: RankLayout, which: str):
    """Block-diagonal CSR over all hosted partitions, columns remapped into the
    rank's [local | halo] row space (graph.py:218-229 column order per part)."""
    rps, cols, vals = [np.zeros(1, dtype=np.int64)], [], []
    nnz = 0
    for p in layout.parts:
        m = p.adj_block if which == "adj" else p.mean_block
        c = np.asarray(m.col_idx, dtype=np.int64)
        nl = p.num_local
        c = np.where(c < nl, layout.loc_base[p.id] + c,
                     layout.NL + layout.halo_base[p.id] + (c - nl))
        rps.append(np.asarray(m.row_ptr[1:], dtype=np.int64) + nnz)
        nnz += int(m.row_ptr[-1])
        cols.append(c)
        vals.append(np.asarray(m.values))
    rp = np.concatenate(rps)
    ci = np.concatenate(cols) if cols else np.zeros(0, np.int64)
    v = np.concatenate(vals) if vals else np.zeros(0)
    return rp, ci, v


def _transpose_device(a: "ops.DeviceCsr") -> "ops.DeviceCsr":
    """CSR of A^T built on the device (stable by row, so each row of A^T keeps
    ascending columns) — the reference precomputes the same transpose on the
    host (trainer.py:164-165)."""
    import torch
    dev = a.row_ptr.device
    counts = a.row_ptr[1:] - a.row_ptr[:-1]
    rows = torch.repeat_interleave(torch.arange(a.rows, device=dev, dtype=torch.int32), counts)
    order = torch.sort(a.col_idx.long(), stable=True).indices
    t = ops.DeviceCsr.__new__(ops.DeviceCsr)
    t.rows, t.cols, t.nnz = a.cols, a.rows, a.nnz
    t.col_idx = rows[order].contiguous()
    t.values = a.values[order].contiguous()
    rp = torch.zeros(a.cols + 1, dtype=torch.int64, device=dev)
    rp[1:] = torch.cumsum(torch.bincount(a.col_idx.long(), minlength=a.cols), 0)
    t.row_ptr = rp
    t.work = torch.zeros(2, dtype=torch.int32, device=dev)    # the dynamic row schedule's counter pair
    return t


class EpochGraph:
    """One training epoch captured as a CUDA graph (``DeviceRank.run_epoch_graphed``).

    The epoch's launches are identical from epoch to epoch except for a few
    per-epoch words: each exchange's K1 descriptor table (the Philox keys
    derive from the epoch, rngstream.py:19-23) and Adam's bias corrections
    (linalg.py:127-140).  Those reach the device through memcpy nodes that
    read pinned host buffers owned by the graph; ``replay`` re-fills them for
    the replayed epoch, then launches the graph.  The host bookkeeping of an
    epoch (slot tags with their staleness checks, byte meters, Adam's step
    count) is recorded at capture and re-applied per replay."""

    def __init__(self, torch):
        self.graph = torch.cuda.CUDAGraph()
        self.fills = []            # callables(epoch) re-filling the pinned buffers
        self._host = {}            # id(owner) -> pinned host tensor
        self.consumed = []         # (layer, phase) slots consumed (tag checks)
        self.set_slots = []        # (layer, phase) slots this epoch fills
        self.stats = {}            # partition -> byte-meter deltas
        self.launches = 0
        self.done = None           # event after the last replay (its pinned buffers are free)
        # N > 1 with the peer-memory exchange: the epoch's PeerLinks calls (re-run
        # before each replay for the counter targets) and the targets' buffers
        self.p2p_calls = []
        self.p2p_host = self.p2p_dev = None
        self.p2p_n = 0

    def p2p_slot(self, target: int) -> int:
        """Device address of the next wait-target slot (its capture-time value
        is the target the first replay uses)."""
        i = self.p2p_n
        if i >= self.p2p_host.numel():
            raise RuntimeError("more peer waits per epoch than target slots")
        self.p2p_n += 1
        self.p2p_host[i] = target
        return self.p2p_dev.data_ptr() + 8 * i

    def pinned(self, owner, nbytes: int):
        return self._host[id(owner)][:nbytes]

    def alloc(self, torch, owner, nbytes: int, dtype=None):
        t = torch.zeros(max(1, nbytes), dtype=dtype or torch.uint8).pin_memory()
        self._host[id(owner)] = t
        return t

    def add_fill(self, fn):
        self.fills.append(fn)


class DeviceRank:
    """One rank's share of the training: buffers, exchanges, epoch loop."""

    def __init__(self, layout: RankLayout, cfg: ModelConfig, mode: TrainMode, quant: QuantConfig,
                 seed: int, lr: float, global_norm: int, device=None, group=None, probe=None,
                 features=None, agg_order=None, timeout: float = 60.0, p2p: bool | None = None):
        import torch
        self.torch = torch
        self.dev = torch.device(device or "cuda")
        self.layout, self.cfg, self.mode, self.quant = layout, cfg, mode, quant
        self.seed, self.lr, self.norm = seed, lr, float(global_norm)
        self.timeout = float(timeout)
        self.group, self.probe = group, probe
        self.world = 1
        if group is not None or _dist_initialized():
            import torch.distributed as dist
            self.world = dist.get_world_size(group)
        L, W = cfg.num_layers, cfg.widths
        self.L = L
        NL, NH = layout.NL, layout.NH
        self.NL, self.NH = NL, NH
        dev = self.dev
        f32 = torch.float32
        layout.to(dev)
        # graph operators
        which = "mean" if cfg.model == "sage" else "adj"
        rp, ci, v = _stack_csr(layout, which)
        self.A = ops.DeviceCsr(NL, NL + NH, rp, ci, v, dev)
        self.At = _transpose_device(self.A)
        # activations: Ht[l] = [local ; halo] input of layer l (ld padded to 16 B)
        self.Ht = {l: torch.zeros((NL + NH, _ld(W[l - 1])), dtype=f32, device=dev)
                   for l in range(1, L + 1)}
        feats = features if features is not None else \
            np.concatenate([np.asarray(p.features, dtype=np.float32) for p in layout.parts])
        self.Ht[1][:NL, :W[0]] = torch.from_numpy(np.ascontiguousarray(feats, dtype=np.float32)).to(dev)
        self.drop = cfg.dropout > 0.0
        self.Hd = {l: torch.zeros_like(self.Ht[l]) for l in range(1, L + 1)} if self.drop else self.Ht
        self.spmm_impl = os.environ.get("HB_SPMM", "auto")
        if self.spmm_impl not in ("auto", "rows", "tiled"):
            raise TrainingError(f"unknown SpMM implementation {self.spmm_impl!r}")
        self._tiles = {}
        # factored SpMM rows of <= 48 columns: 255-column windows (1.03-1.07 ms
        # vs 1.41-1.43 with 64 at d = 41 on Reddit, profiles/r2_kbench_spmm_narrow_windows.jsonl)
        self.narrow_window = int(os.environ.get("HB_NARROW_WINDOW", "255"))
        self.gemm_impl = os.environ.get("HB_GEMM", "tcgen05")
        if self.gemm_impl not in GEMM_FLOPS:
            raise TrainingError(f"unknown GEMM implementation {self.gemm_impl!r}")
        # aggregation order per layer (see choose_agg_order)
        order = agg_order or os.environ.get("HB_AGG_ORDER", "auto")
        if order not in AGG_ORDERS:
            raise TrainingError(f"unknown aggregation order {order!r}")
        self.post = {}
        for l in range(1, L + 1):
            o = order if order != "auto" else choose_agg_order(
                l, W[l - 1], W[l], self.A.nnz, NL, NL + NH, cfg.model, self.gemm_impl)
            self.post[l] = o == "post"
        # pre: AGG = A h~ (width d_in); post: Y = h~ W_bot, AGG = A Y (width d_out)
        self.AGG = {l: torch.zeros((NL, _ld(W[l] if self.post[l] else W[l - 1])), dtype=f32, device=dev)
                    for l in range(1, L + 1)}
        self.Y = {l: torch.zeros((NL + NH, _ld(W[l])), dtype=f32, device=dev)
                  for l in range(1, L + 1) if self.post[l]}
        self.S = {l: torch.zeros((NL + NH, _ld(W[l])), dtype=f32, device=dev)
                  for l in range(1, L + 1) if self.post[l]}
        self.Z = {l: torch.zeros((NL, _ld(W[l])), dtype=f32, device=dev)[:, :W[l]] for l in range(1, L + 1)}
        self.JF = {l: torch.zeros((NL + NH, _ld(W[l - 1])), dtype=f32, device=dev) for l in range(2, L + 1)}
        self.T = {l: torch.zeros((NL, _ld(W[l - 1])), dtype=f32, device=dev)
                  for l in range(2, L + 1) if not self.post[l]}
        self.JL = torch.zeros((NL, _ld(W[L])), dtype=f32, device=dev)
        self.row_loss = torch.zeros(max(1, NL), dtype=torch.float64, device=dev)
        self.loss_dev = torch.zeros(1, dtype=torch.float64, device=dev)
        self.xent_partials = torch.zeros(ops.XENT_PARTIALS, dtype=torch.float64, device=dev)
        self.flags = torch.zeros(1, dtype=torch.int32, device=dev)
        self._deferred, self._snap, self._snap_next = [], [], 0       # run_epoch(defer=True) bookkeeping
        self._graphs, self._cap = {}, None                           # run_epoch_graphed
        self.adam_bc = torch.zeros(2, dtype=torch.float64, device=dev)  # (1-b1^t, 1-b2^t) for graph replays
        self.proto_flags = torch.zeros(1, dtype=torch.int32, device=dev)   # written on the comm stream only
        self.counts = torch.zeros(9, dtype=torch.int64, device=dev)
        self.multilabel = cfg.loss == "multilabel"
        if self.multilabel:
            labels = np.concatenate([np.asarray(p.labels).reshape(p.num_local, -1) for p in layout.parts])
            if labels.shape[1] != W[L]:
                raise TrainingError(f"multilabel labels have {labels.shape[1]} columns, output width {W[L]}")
            self.labels = torch.from_numpy(np.ascontiguousarray(labels, dtype=np.uint8)).to(dev)
        else:
            labels = np.concatenate([np.asarray(p.labels) for p in layout.parts]).astype(np.int32)
            self.labels = torch.from_numpy(labels).to(dev)
        tm = np.concatenate([np.asarray(p.train_mask, dtype=bool) for p in layout.parts])
        self.train_mask = torch.from_numpy(tm.astype(np.uint8)).to(dev)
        em = np.zeros(NL, dtype=np.uint8)
        off = 0
        for p in layout.parts:
            n = p.num_local
            em[off:off + n][np.asarray(p.train_mask, bool)] = 1
            em[off:off + n][np.asarray(p.val_mask, bool)] = 2
            em[off:off + n][np.asarray(p.test_mask, bool)] = 3
            off += n
        self.eval_mask = torch.from_numpy(em).to(dev)
        # parameters (replicated; identical Glorot init on every rank, no broadcast)
        # Stored with 16-byte row strides (columns padded to a multiple of 4, pad
        # entries stay exactly 0 through Adam) so every GEMM operand is
        # TMA-describable; W / G are the logical (fan_in x d_out) views.
        w0 = init_weights(cfg, seed)
        self.Wp, self.Gp = [], []
        gsize = sum(w.shape[0] * _ld(w.shape[1]) for w in w0)
        self.gflat = torch.zeros(gsize, dtype=f32, device=dev)
        off = 0
        for w in w0:
            r, c = w.shape
            wp = torch.zeros((r, _ld(c)), dtype=f32, device=dev)
            wp[:, :c] = torch.from_numpy(w.astype(np.float32)).to(dev)
            self.Wp.append(wp)
            self.Gp.append(self.gflat[off:off + wp.numel()].view_as(wp))
            off += wp.numel()
        self.W = [wp[:, :w.shape[1]] for wp, w in zip(self.Wp, w0)]
        self.G = [gp[:, :w.shape[1]] for gp, w in zip(self.Gp, w0)]
        # split-K workspace for the weight-gradient GEMM (G = P^T m, K = rows)
        gmax = max(w.numel() for w in self.Wp)
        self.gemm_ws = torch.empty(64 * gmax, dtype=f32, device=dev)
        self.adam_m = [torch.zeros_like(w) for w in self.Wp]
        self.adam_v = [torch.zeros_like(w) for w in self.Wp]
        self.adam_t = 0
        # exchange buffers
        par = 2 if mode.variant == "async" else 1
        self.xf = {l: ExchangeBuffers(layout, layout.fwd, W[l - 1], quant.bits, dev, par)
                   for l in range(1, L + 1)}
        self.xb = {l: ExchangeBuffers(layout, layout.bwd, W[l - 1], quant.bits, dev, par)
                   for l in range(2, L + 1)}
        self.xeval = None
        # peer-memory halo exchange (K1 writes into the peers' receive buffers;
        # transport.PeerLinks) instead of NCCL send/recv: the default for N > 1
        # on an NCCL process group (one node, NVLink); HB_P2P=0/1 overrides,
        # gloo groups (host-staged test runs) use it only when asked
        if p2p is None:
            env = os.environ.get("HB_P2P")
            if env is not None:
                p2p = env == "1"
            else:
                from .transport import host_staged
                p2p = self.world > 1 and not host_staged(group)
        self.p2p = None
        if p2p and self.world > 1:
            from .transport import PeerLinks
            try:
                self.p2p = PeerLinks(list(self.xf.values()) + list(self.xb.values()), group, dev, self.timeout,
                                     parities=par)
            except Exception as exc:         # e.g. no CUDA IPC between these processes
                if os.environ.get("HB_P2P") == "1":
                    raise
                import warnings
                warnings.warn(f"peer-memory halo exchange unavailable ({exc}); using NCCL send/recv")
                for b in list(self.xf.values()) + list(self.xb.values()):
                    b.peer_recv, b.peer_off = None, None
        self.slots = {}
        self.stats = {p: TransportStats() for p in layout.ids}
        self.epoch_loss = 0.0
        self.comm_stream = torch.cuda.Stream(device=dev) if self.world > 1 else None
        self.comm_events = None      # list -> (start, end, remote wire bytes) per NCCL exchange
        self.launches = 0
        self.timer = null_timer

    # -- exchange helpers -----------------------------------------------------
    def _count(self, bufs: ExchangeBuffers):
        for p, (mb, md, hd, ms) in bufs.stats_delta().items():
            s = self.stats[p]
            s.main_bytes_sent += mb
            s.metadata_bytes_sent += md
            s.header_bytes_sent += hd
            s.messages_sent += ms

    def _send(self, bufs: ExchangeBuffers, src, epoch: int, layer: int, parity: int, count=True,
              defer: bool = False):
        """K1 for every hosted sender (+ NCCL for remote peers on the comm stream)."""
        torch = self.torch
        # K1 below overwrites the send buffer: an exchange still in flight on
        # the comm stream (Sylvie-A, or a drained slot at an adaptor-sync
        # epoch) must have left it first
        self._wait_comm(bufs)
        p2p = self.p2p if self.p2p is not None and id(bufs) in self.p2p.index else None
        if p2p is not None:
            p2p.before_send(bufs, parity, self.proto_flags)     # the peers no longer read what K1 overwrites
        if bufs.n_send:
            segs = bufs.upload_send_table(self.seed, epoch, layer, parity)
            R = int(bufs.plan.send_rows.size)
            nbytes = R * bufs.d * 4 + R * 4 + bufs.wire_bytes_total()
            with self.timer("quantize_gather", nbytes):
                quantize_gather(src, bufs.plan.dev["send_rows"], segs, bufs.n_send, bufs.d,
                                bufs.bits, self.flags)
            self.launches += 1
            if self.probe and count:      # the evaluation forward is centralized in the reference: no events
                self._probe_out(bufs, epoch, layer)
        if p2p is not None:
            p2p.after_send(bufs, parity)                         # the blocks are in the peers' buffers
        elif self.world > 1:
            ev = torch.cuda.current_stream().record_event()
            with torch.cuda.stream(self.comm_stream):
                self.comm_stream.wait_event(ev)
                if self.comm_events is not None:     # halo GB/s: the NCCL span on the comm stream
                    t0 = torch.cuda.Event(enable_timing=True)
                    t0.record(self.comm_stream)
                nccl_exchange(bufs, parity, self.group, tag=(epoch, layer, bufs.plan.phase),
                              flags=self.proto_flags)
                done = self.comm_stream.record_event()
                if self.comm_events is not None:
                    t1 = torch.cuda.Event(enable_timing=True)
                    t1.record(self.comm_stream)
                    self.comm_events.append((t0, t1, sum(n for _, n in bufs.send_group.values())))
            if defer:
                # Sylvie-A: the exchange overlaps the rest of this epoch and the
                # next one up to the consuming K2 (_recv waits on `done`)
                bufs.comm_done[parity] = done
            else:
                torch.cuda.current_stream().wait_event(done)
        if count:
            self._count(bufs)

    def _wait_comm(self, bufs: ExchangeBuffers, parity=None):
        for p in range(len(bufs.comm_done)) if parity is None else (parity,):
            ev = bufs.comm_done[p]
            if ev is not None:
                self.torch.cuda.current_stream().wait_event(ev)
                bufs.comm_done[p] = None

    def _recv(self, bufs: ExchangeBuffers, parity: int, dst, accumulate: bool):
        """K2: forward scatter into halo rows / backward ascending-peer integration."""
        p2p = self.p2p if self.p2p is not None and id(bufs) in self.p2p.index else None
        if bufs.n_recv == 0:
            if p2p is not None:
                p2p.after_recv(bufs, parity)
            return
        self._wait_comm(bufs, parity)
        if p2p is not None:
            p2p.before_recv(bufs, parity, self.proto_flags)
        pd = bufs.plan.dev
        nd, ns = int(bufs.plan.dst_rows.size), int(bufs.plan.src_rows.size)
        nbytes = bufs.wire_bytes_total() + nd * bufs.d * 4 * (2 if accumulate else 1) + 4 * (2 * nd + ns)
        with self.timer("dequant_gather", nbytes):
            dequant_gather(bufs.recv_segs[parity], bufs.n_recv, pd["dst_rows"], pd["src_ptr"],
                           pd["src_rows"], bufs.d, bufs.bits, dst, accumulate)
        self.launches += 1
        if p2p is not None:
            p2p.after_recv(bufs, parity)                         # the senders may overwrite it now

    def _probe_out(self, bufs, epoch, layer):
        for m in bufs.plan.send_msgs:
            p = self.layout.parts[self.layout.ids.index(m.src)]
            if bufs.plan.phase == FORWARD:
                gids = p.local_nodes[p.send_sets[m.dst]]
            else:
                gids = p.halo_nodes[p.recv_sets[m.dst]]
            self.probe("exchange_out", part=m.src, peer=m.dst, epoch=epoch, layer=layer,
                       phase=bufs.plan.phase, global_ids=gids)

    def _consume(self, epoch: int, layer: int, phase: str) -> int:
        """trainer.py:232-246 — tags are tracked on the host."""
        if self._cap is not None:
            self._cap.consumed.append((layer, phase))
        tag = self.slots.get((layer, phase))
        if tag is None:
            if epoch > 1:
                raise ProtocolError(f"buffer underflow: ({layer}, {phase}) never filled before epoch {epoch}")
            return 0
        if tag != epoch - 1:
            raise ProtocolError(f"staleness violation on ({layer}, {phase}): buffer from epoch {tag}, "
                                f"consuming at epoch {epoch}")
        return tag

    def _dropout(self, src, dst, epoch: int, layer: int, d: int):
        lay = self.layout
        for p in lay.parts:
            key = derive_key((self.seed, "dropout", p.id, epoch, layer))
            lb, hb = lay.loc_base[p.id], lay.NL + lay.halo_base[p.id]
            if p.num_local:
                ops.dropout(src[lb:], p.num_local, 0, d, key, self.cfg.dropout, dst[lb:])
            if p.num_halo:
                ops.dropout(src[hb:], p.num_halo, p.num_local, d, key, self.cfg.dropout, dst[hb:])
            self.launches += 2

    # -- forward / backward -----------------------------------------------------
    def forward(self, epoch: int, epoch_mode: str, training: bool = True):
        torch = self.torch
        W, L, NL = self.cfg.widths, self.L, self.NL
        sync_variant = self.mode.variant == "sync"
        for l in range(1, L + 1):
            d = W[l - 1]
            H = self.Ht[l]
            if not training:
                bufs = self.xeval[l]
                self._send(bufs, H, epoch, l, 0, count=False)
                self._recv(bufs, 0, H, False)
            elif sync_variant:
                bufs = self.xf[l]
                self._send(bufs, H, epoch, l, 0)
                self._recv(bufs, 0, H, False)
            elif epoch_mode == "sync":
                bufs = self.xf[l]
                if epoch > 1:
                    self._consume(epoch, l, FORWARD)
                self._send(bufs, H, epoch, l, epoch % 2)
                self._recv(bufs, epoch % 2, H, False)
                self.slots[(l, FORWARD)] = epoch
            else:
                bufs = self.xf[l]
                tag = self._consume(epoch, l, FORWARD)
                if tag == 0:
                    H[NL:].zero_()
                else:
                    self._recv(bufs, (epoch - 1) % 2, H, False)
                if self.probe:
                    self._probe_halo(epoch, l, tag, H, d)
                self._send(bufs, H, epoch, l, epoch % 2, defer=True)
                self.slots[(l, FORWARD)] = epoch
            Hd = H
            if training and self.drop:
                Hd = self.Hd[l]
                self._dropout(H, Hd, epoch, l, d)
            self._layer_forward(l, Hd)
        return self.Z[L]

    # -- dense combine + aggregation of one layer --------------------------------
    def _mm(self, a, b, out, accumulate: bool = False, relu_out=None):
        """out (+)= a @ b (trainer.py:294,313,318-321).  out None: only
        relu_out = relu(a @ b) is stored (tcgen05 path)."""
        nl, nc = a.shape[0], b.shape[1]
        # compulsory bytes: A, B once, C written (and read when accumulating), the ReLU copy
        nbytes = 4 * (a.shape[0] * a.shape[1] + b.shape[0] * nc + nl * nc * (
            (out is not None) + bool(accumulate) + (relu_out is not None)))
        with self.timer("gemm", nbytes, 2 * a.shape[0] * a.shape[1] * b.shape[1]):
            if self.gemm_impl == "cublas":
                if accumulate:
                    out.addmm_(a, b)
                else:
                    self.torch.mm(a, b, out=out)
                if relu_out is not None:
                    ops.relu(out, relu_out, nl, nc)
                    self.launches += 1
            else:
                ops.gemm(a, b, out, beta=1.0 if accumulate else 0.0, relu_out=relu_out, ws=self.gemm_ws)
                self.launches += 1

    def _mm2(self, a1, b1, a2, b2, out, relu_out=None):
        """out = a1 @ b1 + a2 @ b2: the SAGE combine over [h | A h] (trainer.py:294,318-321)
        in one GEMM pass, without materialising the concatenation.  out None:
        only relu_out = relu(...) is stored (tcgen05 path)."""
        nl, nc = a1.shape[0], b1.shape[1]
        nbytes = 4 * (nl * (a1.shape[1] + a2.shape[1]) + (b1.shape[0] + b2.shape[0]) * nc + nl * nc * (
            (out is not None) + (relu_out is not None)))
        with self.timer("gemm", nbytes, 2 * a1.shape[0] * (a1.shape[1] + a2.shape[1]) * b1.shape[1]):
            if self.gemm_impl == "cublas":
                self.torch.mm(a1, b1, out=out)
                out.addmm_(a2, b2)
                if relu_out is not None:
                    ops.relu(out, relu_out, nl, nc)
                    self.launches += 1
            else:
                ops.gemm2(a1, b1, a2, b2, out, relu_out=relu_out, ws=self.gemm_ws)
                self.launches += 1

    def _tiled(self, a, d: int = 0):
        """Tiled (TMA-staged) layout of `a`, built on first use; None when too
        little of the matrix falls into dense tiles to pay off.  Rows of 33-48
        columns use their own factored layout with 255-column windows
        (HB_NARROW_WINDOW) when the operator factors."""
        key = id(a)
        if key not in self._tiles:
            # forward operator: the 296 lightest row blocks go out last (d = 256
            # on Reddit: 4.15 vs 4.22-4.27 ms, DRAM 2.0 vs 1.05 GB per launch;
            # heaviest-first over all blocks: 4.07 ms but 5.5 GB); the
            # transpose keeps ascending blocks (profiles/r2_kbench_spmm_wide.jsonl)
            t = ops.TiledCsr(a, block_order="light296" if a is self.A else None)
            self._tiles[key] = t if t.tiled_fraction >= 0.5 else None
        t = self._tiles[key]
        if t is not None and t.binary and 32 < d <= 48 and self.narrow_window != 64:
            nkey = (key, "narrow")
            if nkey not in self._tiles:
                self._tiles[nkey] = ops.TiledCsr(a, factored=True, block_rows=64, window=self.narrow_window)
            t = self._tiles[nkey]
        return t

    def _spmm(self, a, x, y, d: int):
        """K3/K4: the TMA-staged tiled kernel where the matrix has dense
        (community) blocks, the row-gather kernel otherwise."""
        # auto: the tiled kernel for wide (> 128) and narrow (<= 64, row-per-
        # lane-group consumers) panels of community-structured blocks
        t = self._tiled(a, d) if (self.spmm_impl == "tiled" or (self.spmm_impl == "auto" and (d > 128 or d <= 64))) \
            else None
        name = "spmm_rows" if t is None else ("spmm_tiled_narrow" if d <= 64 else "spmm_tiled")
        with self.timer(name, *_spmm_cost(a, d)):
            if t is not None:
                ops.spmm_tiled(t, x, y, d)
            else:
                ops.spmm(a, x, y, d, stream_col=self.NL if a is self.A else None)
        self.launches += 1

    def _layer_forward(self, l: int, Hd):
        """p = A h~ (SAGE: [h~_local | M h~]); z = p W; h = relu(z) (trainer.py:290-295).

        pre order (the reference's): AGG = A h~ at width d_in, then the GEMM.
        post order: Y = h~ W_bot over local+halo rows, AGG = A Y at width d_out,
        z = h~_local W_top + AGG — the same z up to fp32 summation order, with
        the SpMM at the narrower width (DGL applies the same reordering)."""
        W, NL = self.cfg.widths, self.NL
        d, dout = W[l - 1], W[l]
        sage = self.cfg.model == "sage"
        Wl = self.W[l - 1]
        Wtop, Wbot = (Wl[:d], Wl[d:]) if sage else (None, Wl)
        Z, agg = self.Z[l], self.AGG[l]
        hout = self.Ht[l + 1][:NL, :dout] if l < self.L else None
        if not self.post[l]:
            self._spmm(self.A, Hd, agg, d)
            # a hidden layer's z is never read again (the backward masks with
            # h > 0): the tcgen05 epilogue stores only h = relu(z)
            zout = None if (hout is not None and self.gemm_impl != "cublas") else Z
            if sage:
                self._mm2(Hd[:NL, :d], Wtop, agg[:, :d], Wbot, zout, relu_out=hout)
            else:
                self._mm(agg[:, :d], Wbot, zout, relu_out=hout)
            return
        Y = self.Y[l]
        self._mm(Hd[:, :d], Wbot, Y[:, :dout])
        if sage:
            self._spmm(self.A, Y, Z, dout)           # aggregate straight into z, then z += h~ W_top
            self._mm(Hd[:NL, :d], Wtop, Z, accumulate=True, relu_out=hout)
        else:
            self._spmm(self.A, Y, agg, dout)
            if hout is not None:
                ops.relu(agg, self.Ht[l + 1], NL, dout)
                self.launches += 1
            else:
                Z.copy_(agg[:, :dout])

    def _layer_backward(self, l: int, m, JF):
        """G = p^T m; j_full = A^T (m W_bot^T) (+ SAGE local m W_top^T)
        (trainer.py:313-321).  post order: S = A^T m at width d_out, then
        G_bot = h~^T S and j_full = S W_bot^T."""
        W, NL = self.cfg.widths, self.NL
        d, dout = W[l - 1], W[l]
        sage = self.cfg.model == "sage"
        Hd = self.Hd[l] if self.drop else self.Ht[l]
        Wl, G = self.W[l - 1], self.G[l - 1]
        Gtop, Gbot = (G[:d], G[d:]) if sage else (None, G)
        Wtop, Wbot = (Wl[:d], Wl[d:]) if sage else (None, Wl)
        if sage:
            self._mm(Hd[:NL, :d].t(), m, Gtop)
        if not self.post[l]:
            agg = self.AGG[l]
            self._mm(agg[:, :d].t(), m, Gbot)
            if JF is None:
                return
            T = self.T[l]
            self._mm(m, Wbot.t(), T[:, :d])
            self._spmm(self.At, T, JF, d)
        else:
            S = self.S[l]
            self._spmm(self.At, m, S, dout)
            self._mm(Hd[:, :d].t(), S[:, :dout], Gbot)
            if JF is None:
                return
            if sage:
                # local rows: j = S W_bot^T + m W_top^T in one pass; halo rows: S W_bot^T
                self._mm2(S[:NL, :dout], Wbot.t(), m, Wtop.t(), JF[:NL, :d])
                if JF.shape[0] > NL:
                    self._mm(S[NL:, :dout], Wbot.t(), JF[NL:, :d])
                return
            self._mm(S[:, :dout], Wbot.t(), JF[:, :d])
        if sage:
            self._mm(m, Wtop.t(), JF[:NL, :d], accumulate=True)

    def _probe_halo(self, epoch, layer, tag, H, d):
        lay = self.layout
        for p in lay.parts:
            hb = lay.NL + lay.halo_base[p.id]
            data = H[hb:hb + p.num_halo, :d].double().cpu().numpy()
            self.probe("halo_consumed", part=p.id, epoch=epoch, layer=layer, phase=FORWARD,
                       tag=tag, data=data)

    def _probe_grads(self, bufs, parity, epoch, layer, tag):
        """Sylvie-A backward 'halo_consumed' (trainer.py:333-337): the stale
        per-peer gradient rows each hosted partition integrates, decoded from
        the wire blocks in its receive buffer."""
        from .codec import QuantizedBlock, dequantize_rows, wire_bytes
        raw = bufs.recv[parity]
        per = {q: {} for q in self.layout.ids}
        for m in bufs.plan.recv_msgs:
            o = bufs.recv_off[(m.src, m.dst)]
            blk = raw[o:o + wire_bytes(m.rows, bufs.d, bufs.bits)].cpu().numpy().tobytes()
            per[m.dst][m.src] = dequantize_rows(QuantizedBlock.from_bytes(blk))
        for q in self.layout.ids:
            self.probe("halo_consumed", part=q, epoch=epoch, layer=layer, phase=BACKWARD, tag=tag,
                       data=per[q])

    def backward(self, epoch: int, epoch_mode: str, logits):
        torch = self.torch
        W, L, NL = self.cfg.widths, self.L, self.NL
        sync_variant = self.mode.variant == "sync"
        C = W[L]
        # JL / row_loss rows outside the train mask are zero from allocation and
        # never written: the CE kernel skips them
        loss_fn = ops.sigmoid_bce if self.multilabel else ops.softmax_xent
        loss_fn(logits, C, self.labels, self.train_mask, self.norm, self.JL,
                self.row_loss, self.loss_dev, keep_unmasked=True, partials=self.xent_partials)
        self.launches += 2
        J = self.JL
        for l in range(L, 0, -1):
            d, dout = W[l - 1], W[l]
            if l < L:
                with self.timer("elementwise", 12 * NL * dout):
                    ops.relu_grad_mul(J, self.Ht[l + 1], J, NL, dout)
                self.launches += 1
            m = J[:, :dout]
            if l == 1:
                self._layer_backward(l, m, None)
                break
            JF = self.JF[l]
            self._layer_backward(l, m, JF)
            if self.drop:
                self._dropout(JF, JF, epoch, l, d)
            bufs = self.xb[l]
            if sync_variant:
                self._send(bufs, JF, epoch, l, 0)
                self._recv(bufs, 0, JF, True)
            elif epoch_mode == "sync":
                if epoch > 1:
                    self._consume(epoch, l, BACKWARD)
                self._send(bufs, JF, epoch, l, epoch % 2)
                self._recv(bufs, epoch % 2, JF, True)
                self.slots[(l, BACKWARD)] = epoch
            else:
                if epoch > 1:
                    tag = self._consume(epoch, l, BACKWARD)
                    self._recv(bufs, (epoch - 1) % 2, JF, True)
                    if self.probe:
                        self._probe_grads(bufs, (epoch - 1) % 2, epoch, l, tag)
                self._send(bufs, JF, epoch, l, epoch % 2, defer=True)
                self.slots[(l, BACKWARD)] = epoch
            J = JF[:NL]
        return self.loss_dev

    def step(self, epoch: int):
        """All-reduce, Adam (trainer.py:358-366); returns nothing, loss stays on device."""
        self.reduce(epoch)
        self.adam()

    def reduce(self, epoch: int):
        """Gradient + loss all-reduce (trainer.py:358-360)."""
        if self.world > 1:
            # every NCCL call of the rank is issued from the comm stream, so the
            # all-reduce queues behind any deferred (Sylvie-A) halo exchange in
            # host issue order — identical on all ranks — and never runs
            # concurrently with it on another stream
            torch = self.torch
            cur = torch.cuda.current_stream()
            with torch.cuda.stream(self.comm_stream):
                self.comm_stream.wait_stream(cur)
                reduce_gradients(self.gflat, self.loss_dev, self.group)
            cur.wait_stream(self.comm_stream)

    def adam(self, guarded: bool = False):
        """adam_step per layer (trainer.py:365-366); guarded: skipped on the
        device when the epoch's loss is not finite or a flag is set."""
        self.adam_t += 1
        guard = (self.loss_dev, self.flags, self.proto_flags) if guarded else None
        bc = None
        if self._cap is not None:
            # graph capture: the bias corrections come from device memory,
            # uploaded from a pinned pair the replays re-fill
            cap = self._cap
            host = cap.pinned(self.adam_bc, 16).view(self.torch.float64)

            def fill(_epoch, h=host):
                h[0], h[1] = 1.0 - 0.9 ** self.adam_t, 1.0 - 0.999 ** self.adam_t
            fill(0)
            ops.upload(self.adam_bc, host)
            cap.add_fill(fill)
            bc = self.adam_bc
        for w, g, m, v in zip(self.Wp, self.Gp, self.adam_m, self.adam_v):
            ops.adam_step(w, g, m, v, self.lr, self.adam_t, guard=guard, bc=bc)
            self.launches += 1

    def swap_features(self, buf):
        """Make `buf` layer 1's input ([local ; halo] x ld, shaped like Ht[1]);
        returns the previous buffer.  For double-buffered input pipelines: the
        next epoch's features are uploaded into the spare buffer while this
        epoch runs.  Halo rows need no copy (the layer-1 exchange rewrites them
        every epoch)."""
        old = self.Ht[1]
        if buf.shape != old.shape or buf.dtype != old.dtype or buf.stride() != old.stride() \
                or buf.device != old.device:
            raise ShapeError(f"feature buffer {tuple(buf.shape)} does not match layer 1's input {tuple(old.shape)}")
        self.Ht[1] = buf
        return old

    def run_epoch(self, epoch: int, check: bool = True, defer: bool = False) -> str:
        """One epoch.  check: the reference's host checks before Adam
        (trainer.py:358-366; a host synchronisation).  defer: Adam is guarded
        on the device instead (skipped when the loss is not finite or a codec /
        protocol flag is set) and the epoch's loss and flags are copied to
        pinned host memory; ``finish_epoch`` raises or records the loss later,
        so the host can issue the next epoch first.  A failed epoch leaves the
        weights untouched either way."""
        epoch_mode = staleness_adaptor(epoch, self.mode)
        logits = self.forward(epoch, epoch_mode)
        self.backward(epoch, epoch_mode, logits)
        self.reduce(epoch)
        if defer:
            self.adam(guarded=True)
            self._defer_tail(epoch)
            return epoch_mode
        if check:                 # on the all-reduced loss, before Adam (trainer.py:358-366)
            self.check_epoch(epoch)
        self.adam()
        return epoch_mode

    def _defer_tail(self, epoch: int):
        """Copy the epoch's loss and flags to a pinned slot (read by finish_epoch)."""
        torch = self.torch
        if not self._snap:
            self._snap = [tuple(torch.zeros(1, dtype=t.dtype).pin_memory()
                                for t in (self.loss_dev, self.flags, self.proto_flags)) for _ in range(3)]
        slot = self._snap[self._snap_next % len(self._snap)]
        self._snap_next += 1
        for host, dev in zip(slot, (self.loss_dev, self.flags, self.proto_flags)):
            host.copy_(dev.view(-1)[:1], non_blocking=True)
        self._deferred.append((epoch, torch.cuda.current_stream().record_event(), slot))
        if len(self._deferred) >= len(self._snap):      # at most len(_snap) epochs in flight
            self.finish_epoch()

    def graphable(self) -> bool:
        """CUDA-graph epochs: one rank, or several with the peer-memory halo
        exchange (the gradient all-reduce and Adam then run eagerly after the
        replay; NCCL halo exchanges are not captured); no dropout (its
        per-epoch keys are launch arguments), no probe (host callbacks inside
        the epoch), the tcgen05 GEMMs."""
        return (self.world == 1 or self.p2p is not None) and not self.drop and self.probe is None \
            and self.gemm_impl != "cublas"

    def run_epoch_graphed(self, epoch: int) -> str:
        """``run_epoch(epoch, defer=True)`` replayed from a CUDA graph of the
        epoch: one graph launch instead of ~40 kernel launches + descriptor
        uploads from Python, so the host issue time no longer tracks the device
        time.  Graphs are keyed by (epoch mode, epoch parity, layer-1 input
        buffer); the first two epochs (the Sylvie-A pipeline's start-up, and
        first-use allocations) run eagerly, and a graph is captured the first
        time its key comes up.  Falls back to eager epochs when not
        ``graphable()``."""
        if not self.graphable() or epoch <= 2:
            return self.run_epoch(epoch, defer=True)
        torch = self.torch
        epoch_mode = staleness_adaptor(epoch, self.mode)
        key = (epoch_mode, epoch % 2, self.Ht[1].data_ptr())
        ent = self._graphs.get(key)
        if ent is None:
            self._graphs[key] = self._capture_epoch(epoch, epoch_mode)
        else:
            if ent.done is not None:
                ent.done.synchronize()          # its pinned buffers are free again
            for layer, phase in ent.consumed:
                self._consume(epoch, layer, phase)
            if self.world == 1:
                self.adam_t += 1                # Adam is part of the graph
            for fill in ent.fills:
                fill(epoch)
            if ent.p2p_calls:
                vals = self.p2p.replay_targets(ent.p2p_calls)
                ent.p2p_host.numpy()[:len(vals)] = vals
            ent.graph.replay()
            ent.done = torch.cuda.current_stream().record_event()
            if self.world > 1:
                self.reduce(epoch)
                self.adam(guarded=True)
            for k in ent.set_slots:
                self.slots[k] = epoch
            for p, delta in ent.stats.items():
                st = self.stats[p]
                for k, v in delta.items():
                    setattr(st, k, getattr(st, k) + v)
            self.launches += ent.launches
        self._defer_tail(epoch)
        return epoch_mode

    def _capture_epoch(self, epoch: int, epoch_mode: str) -> EpochGraph:
        """Capture (and run) one epoch as a CUDA graph."""
        torch = self.torch
        ent = EpochGraph(torch)
        bufs = list(self.xf.values()) + list(self.xb.values())
        for b in bufs:
            ent.alloc(torch, b, b.n_send * SEG_BYTES)
        ent.alloc(torch, self.adam_bc, 16)
        stats0 = {p: s.snapshot() for p, s in self.stats.items()}
        slots0 = dict(self.slots)
        launches0 = self.launches
        timer, self.timer = self.timer, null_timer
        if getattr(self, "_cap_stream", None) is None:
            self._cap_stream = torch.cuda.Stream(device=self.dev)
        for b in bufs:
            b.capture = ent
        self._cap = ent
        p2p = self.p2p
        if p2p is not None:
            ent.p2p_host = torch.zeros(1024, dtype=torch.int64).pin_memory()
            ent.p2p_dev = torch.zeros(1024, dtype=torch.int64, device=self.dev)
            p2p.capture = ent
        # no finalizers mid-capture: a collected pinned buffer or event of an
        # earlier engine would make an API call that invalidates the capture
        import gc
        gc.collect()
        gc_was = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.graph(ent.graph, stream=self._cap_stream, capture_error_mode="thread_local"):
                if p2p is not None:
                    ops.upload(ent.p2p_dev, ent.p2p_host)     # this replay's peer-wait targets
                logits = self.forward(epoch, epoch_mode)
                self.backward(epoch, epoch_mode, logits)
                if self.world == 1:
                    self.reduce(epoch)
                    self.adam(guarded=True)
        finally:
            if gc_was:
                gc.enable()
            for b in bufs:
                b.capture = None
            self._cap = None
            if p2p is not None:
                p2p.capture = None
            self.timer = timer
        ent.launches = self.launches - launches0
        ent.stats = {p: {k: v - stats0[p][k] for k, v in s.snapshot().items()} for p, s in self.stats.items()}
        ent.set_slots = [k for k, v in self.slots.items() if v == epoch and slots0.get(k) != epoch]
        ent.graph.replay()                      # a capture records the work; this runs it
        ent.done = torch.cuda.current_stream().record_event()
        if self.world > 1:                      # the all-reduce and Adam stay eager
            self.reduce(epoch)
            self.adam(guarded=True)
        return ent

    def finish_epoch(self):
        """Host checks of the oldest deferred epoch (``run_epoch(defer=True)``)."""
        epoch, ev, (loss_h, flags_h, proto_h) = self._deferred.pop(0)
        self._check(epoch, ev, lambda: float(loss_h[0]), lambda: int(flags_h[0]), lambda: int(proto_h[0]))

    def check_epoch(self, epoch: int):
        """Host checks of the reference (codec.py:167-168, trainer.py:361-363),
        after waiting at most ``timeout`` seconds for the epoch to finish on
        the device (the reference's recv timeout, transport.py:115-124: with
        NCCL a stalled or diverged peer leaves the comm stream waiting)."""
        self._check(epoch, self.torch.cuda.current_stream().record_event(), lambda: float(self.loss_dev.item()),
                    lambda: int(self.flags.item()), lambda: int(self.proto_flags.item()))

    def _check(self, epoch, event, loss_fn, flags_fn, proto_fn):
        wait_device(event, self.timeout,
                    f"epoch {epoch} did not complete within {self.timeout:g} s (a peer rank stalled "
                    "or the ranks diverged)")
        if proto_fn():
            raise ProtocolError(f"tag mismatch in an exchange of epoch {epoch}: the ranks diverged")
        if flags_fn() & 1:
            raise TrainingError(f"worker {self.layout.ids[0]} aborted: "
                                f"{CodecError('non-finite values in quantizer input')}")
        loss = loss_fn()
        if not math.isfinite(loss):
            raise TrainingError(f"worker {self.layout.ids[0]} aborted: NaN/inf loss at epoch {epoch}: "
                                "learning rate too high or codec error")
        self.epoch_loss = loss

    def evaluate(self) -> dict:
        """Full-precision forward (no dropout, passthrough halos) + argmax
        accuracy on every mask (trainer.py:115-144), on device."""
        if self.xeval is None:
            self.xeval = {l: ExchangeBuffers(self.layout, self.layout.fwd, self.cfg.widths[l - 1], 32,
                                             self.dev, 1) for l in range(1, self.L + 1)}
        logits = self.forward(0, "sync", training=False)
        if self.multilabel:
            ops.multilabel_counts(logits, self.cfg.widths[-1], self.labels, self.eval_mask, self.counts)
        else:
            ops.argmax_accuracy(logits, self.cfg.widths[-1], self.labels, self.eval_mask, self.counts)
        if self.world > 1:
            import torch.distributed as dist
            from .transport import host_staged
            if host_staged(self.group):
                c = self.counts.cpu()
                dist.all_reduce(c, group=self.group)
                self.counts.copy_(c)
            else:
                dist.all_reduce(self.counts, group=self.group)
        return _accuracies(self.counts.cpu().numpy(), self.multilabel)

    def weights_host(self) -> list:
        return [w.double().cpu().numpy() for w in self.W]

    def total_stats(self) -> dict:
        t = TransportStats()
        for s in self.stats.values():
            t.main_bytes_sent += s.main_bytes_sent
            t.metadata_bytes_sent += s.metadata_bytes_sent
            t.header_bytes_sent += s.header_bytes_sent
            t.messages_sent += s.messages_sent
            t.allreduce_bytes += s.allreduce_bytes
        return t.snapshot()


def wait_device(event, timeout: float, what: str, poll=None):
    """Block until `event` completes, raising ProtocolError after `timeout`
    seconds (a spin for the first ~50 us, then 50-us sleeps)."""
    import time
    done = poll or event.query
    t0 = time.monotonic()
    spins = 0
    while not done():
        if time.monotonic() - t0 > timeout:
            raise ProtocolError(f"timed out: {what}")
        spins += 1
        if spins > 64:
            time.sleep(5e-5)


def _accuracies(c, multilabel: bool) -> dict:
    """train/val/test accuracy from argmax counts; micro-F1 for multi-label."""
    names = ("train_acc", "val_acc", "test_acc")
    if multilabel:
        out = {}
        for k, n in enumerate(names):
            tp, fp, fn = (float(x) for x in c[3 * k:3 * k + 3])
            out[n] = 2 * tp / (2 * tp + fp + fn) if (2 * tp + fp + fn) else 0.0
        return out
    return {n: (float(c[2 * k + 1]) / float(c[2 * k]) if c[2 * k] else 0.0) for k, n in enumerate(names)}


def reduce_gradients(gflat, loss, group=None):
    """``Fabric.all_reduce_sum`` of the weight gradients and the loss
    (transport.py:126-148, trainer.py:358-360): one flat all-reduce each, so
    every replica applies bit-identical updates."""
    import torch.distributed as dist
    from .transport import host_staged
    if gflat.is_cuda and host_staged(group):        # gloo test runs: stage through host memory
        g, l_ = gflat.cpu(), loss.cpu()
        dist.all_reduce(g, group=group)
        dist.all_reduce(l_, group=group)
        gflat.copy_(g)
        loss.copy_(l_)
        return
    dist.all_reduce(gflat, group=group)
    dist.all_reduce(loss, group=group)


AGG_ORDERS = ("pre", "post", "auto")
# Effective rates behind the per-layer aggregation-order choice, measured on
# the B200 (bench r1): the SpMM moves ~17 TB/s of gathered X rows out of L2;
# the GEMM rate depends on the implementation.
SPMM_GATHER_BPS = 17e12
GEMM_FLOPS = {"cublas": 40e12, "tcgen05": 150e12}


def choose_agg_order(layer: int, d_in: int, d_out: int, nnz: int, nl: int, nrows: int, model: str,
                     gemm_impl: str = "cublas") -> str:
    """'pre' (aggregate the d_in-wide input, the reference's order) or 'post'
    (project to d_out first, aggregate the d_out-wide product), whichever
    moves fewer bytes/flops under the measured rates.  Layer 1 has no
    backward SpMM in 'pre' order (no j_full), but always has one in 'post'
    (for G_bot = h~^T A^T m)."""
    fan = 2 if model == "sage" else 1
    bwd = 1 if layer > 1 else 0
    rate = GEMM_FLOPS.get(gemm_impl, GEMM_FLOPS["cublas"])
    spmm = lambda w: 4.0 * nnz * w / SPMM_GATHER_BPS  # noqa: E731
    pre = spmm(d_in) * (1 + bwd) + 2.0 * nl * fan * d_in * d_out * (2 + bwd) / rate
    post = 2 * spmm(d_out) + 2.0 * d_in * d_out * (nrows + (fan - 1) * nl) * (2 + bwd) / rate
    return "post" if post < pre else "pre"


def _spmm_cost(a, d: int):
    """(compulsory HBM bytes, flops) of one SpMM launch: CSR arrays + every X
    row read once + Y written once; 2 flops per nonzero per column."""
    nbytes = 8 * (a.rows + 1) + 8 * a.nnz + 4 * a.cols * d + 4 * a.rows * d
    return nbytes, 2 * a.nnz * d


def _dist_initialized() -> bool:
    try:
        import torch.distributed as dist
        return dist.is_available() and dist.is_initialized()
    except Exception:
        return False


def full_forward(features, a_hat, weights: list, cfg: ModelConfig, mean_hat=None, device=None):
    """``halobit.trainer.full_forward`` (trainer.py:115-126) on the device:
    the single-machine full-precision forward (no dropout) through the
    row-gather SpMM and the tcgen05 GEMMs; returns the logits as a float32
    device tensor (n x C).  ``a_hat`` / ``mean_hat`` are ``CsrMatrix`` (or
    ``ops.DeviceCsr``); ``weights`` the (fan_in x d_out) arrays."""
    import torch
    dev = torch.device(device or "cuda")
    def dcsr(m):
        return m if isinstance(m, ops.DeviceCsr) else ops.DeviceCsr.from_csr(m, dev)
    agg = dcsr(mean_hat if cfg.model == "sage" else a_hat)
    x = np.asarray(features)
    n = x.shape[0]
    h = torch.zeros((n, _ld(x.shape[1])), dtype=torch.float32, device=dev)
    h[:, :x.shape[1]] = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(dev)
    for l, w in enumerate(weights, start=1):
        din, dout = cfg.widths[l - 1], cfg.widths[l]
        wp = torch.zeros((w.shape[0], _ld(dout)), dtype=torch.float32, device=dev)
        wp[:, :dout] = torch.from_numpy(np.asarray(w, dtype=np.float32)).to(dev)
        p = torch.zeros((n, _ld(din)), dtype=torch.float32, device=dev)
        ops.spmm(agg, h, p, din)
        z = torch.zeros((n, _ld(dout)), dtype=torch.float32, device=dev)
        if cfg.model == "sage":
            ops.gemm2(h[:, :din], wp[:din, :dout], p[:, :din], wp[din:, :dout], z[:, :dout])
        else:
            ops.gemm(p[:, :din], wp[:, :dout], z[:, :dout])
        if l < cfg.num_layers:
            ops.relu(z, z, n, dout)
        h = z
    return h[:, :cfg.widths[-1]]


def evaluate(weights: list, graph: Graph, cfg: ModelConfig, a_hat=None, mean_hat=None,
             device=None) -> dict:
    """``halobit.trainer.evaluate`` (trainer.py:129-144): centralized argmax
    accuracy on the train / val / test masks, computed on the device."""
    import torch
    from .graph import mean_adjacency, normalize_adjacency
    if a_hat is None and cfg.model != "sage":
        a_hat = normalize_adjacency(graph)
    if cfg.model == "sage" and mean_hat is None:
        mean_hat = mean_adjacency(graph)
    dev = torch.device(device or "cuda")
    logits = full_forward(graph.features, a_hat, weights, cfg, mean_hat, device=dev)
    n, C = logits.shape
    em = np.zeros(n, dtype=np.uint8)
    em[np.asarray(graph.train_mask, bool)] = 1
    em[np.asarray(graph.val_mask, bool)] = 2
    em[np.asarray(graph.test_mask, bool)] = 3
    counts = torch.zeros(9, dtype=torch.int64, device=dev)
    mask = torch.from_numpy(em).to(dev)
    if cfg.loss == "multilabel":
        labels = torch.from_numpy(np.ascontiguousarray(graph.labels, dtype=np.uint8)).to(dev)
        ops.multilabel_counts(logits, C, labels, mask, counts)
    else:
        labels = torch.from_numpy(np.asarray(graph.labels).astype(np.int32)).to(dev)
        ops.argmax_accuracy(logits, C, labels, mask, counts)
    return _accuracies(counts.cpu().numpy(), cfg.loss == "multilabel")


def train(graph: Graph, partitions: list, model_cfg: ModelConfig, mode: TrainMode,
          quant_cfg: QuantConfig, epochs: int, seed: int, lr: float = 0.01, probe=None,
          timeout: float = 60.0, device=None, evaluate_each_epoch: bool = True,
          agg_order: str | None = None) -> TrainResult:
    """Drop-in for ``halobit.train`` (trainer.py:386-465) on one GPU: every
    partition is hosted by this process's device (the reference's one-process
    simulation, with device-resident halo traffic)."""
    import time
    n = len(partitions)
    global_norm = max(1, int(np.asarray(graph.train_mask).sum()))
    layout = RankLayout({p.id: p for p in partitions}, [0] * n, 0)
    eng = DeviceRank(layout, model_cfg, mode, quant_cfg, seed, lr, global_norm, device=device,
                     probe=probe, agg_order=agg_order, timeout=timeout)
    if epochs == 0:
        return TrainResult([], init_weights(model_cfg, seed))
    ar_per_epoch = (4 * sum(int(w.numel()) for w in eng.W)) if n > 1 else 0
    metrics, timings = [], []
    prev = eng.total_stats()
    for epoch in range(1, epochs + 1):
        t0 = time.perf_counter()
        try:
            epoch_mode = eng.run_epoch(epoch)
        except ProtocolError as e:
            raise TrainingError(f"worker {layout.ids[0]} aborted: {e}") from e
        for p in layout.ids:
            eng.stats[p].allreduce_bytes += ar_per_epoch
        stats = eng.total_stats()
        accs = eng.evaluate() if evaluate_each_epoch else dict(train_acc=0.0, val_acc=0.0, test_acc=0.0)
        if probe:
            wts = eng.weights_host()
            probe("weights", epoch=epoch, weights=[[w.copy() for w in wts] for _ in range(n)])
        metrics.append(MetricsRecord(
            epoch=epoch, mode_this_epoch=epoch_mode, train_loss=eng.epoch_loss,
            main_bytes=stats["main_bytes_sent"] - prev["main_bytes_sent"],
            meta_bytes=stats["metadata_bytes_sent"] - prev["metadata_bytes_sent"],
            header_bytes=stats["header_bytes_sent"] - prev["header_bytes_sent"],
            allreduce_bytes=stats["allreduce_bytes"] - prev["allreduce_bytes"],
            messages=stats["messages_sent"] - prev["messages_sent"], **accs))
        prev = stats
        timings.append((time.perf_counter() - t0) * 1000.0)
    return TrainResult(metrics, eng.weights_host(), timings)
