"""Halo exchange on device buffers: drop-in for ``halobit.transport``'s
``exchange`` + ``Fabric`` on the B200.

Reference (``transport.py:90-205``, driven by ``trainer.py:175-223``): for each
(partition, epoch, layer, phase) the sender gathers its boundary rows per peer,
quantizes them peer-by-peer (ascending) from one keyed stream, ships one
message per non-empty peer; the receiver dequantizes and scatters
(forward: into its halo slots) or accumulates (backward: into its local rows,
ascending peer order).

B200 design:
* A rank hosts one or more partitions (one per GPU in production; the
  single-GPU case hosts all of them, which is exactly the reference's
  one-process simulation).  Its rows live in HBM as one contiguous
  ``[local rows of all hosted partitions ; halo rows of all hosted partitions]``
  matrix per layer, so one SpMM, one GEMM and one K1/K2 launch cover every
  hosted partition.
* K1 (``hb_quantize_gather``) gathers, quantizes, packs and writes each
  message's wire block straight into its destination: the receiver's slot in
  the local receive buffer (same-rank peer) or the send buffer for the peer
  rank.  Messages to one rank are contiguous, so one NCCL send/recv pair per
  peer rank moves them (``torch.distributed`` over NCCL/NVLink, on a side
  stream).
* K2 (``hb_dequant_gather``) consumes the receive buffer: forward writes halo
  rows, backward accumulates into local rows with sources in ascending peer
  order (f64 sum, one fp32 rounding).
* Receive buffers are double-buffered by epoch parity for the Sylvie-A
  pipeline: epoch t consumes parity (t-1)%2 while its fresh sends land in
  parity t%2 (``trainer.py:232-246``).
* Byte meters are exact functions of the plan (``transport.py:105-114``):
  they count what the device actually moves.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._np import sorted_unique_index
from .codec import HEADER_BYTES, metadata_bytes, payload_bytes, wire_bytes
from .rngstream import BACKWARD, FORWARD, derive_key

DEFAULT_TIMEOUT = 60.0


class ProtocolError(RuntimeError):
    pass


@dataclass
class TransportStats:
    """``transport.py:62-71``."""

    main_bytes_sent: int = 0
    metadata_bytes_sent: int = 0
    header_bytes_sent: int = 0
    messages_sent: int = 0
    allreduce_bytes: int = 0

    def snapshot(self) -> dict:
        return dict(self.__dict__)


class PoisonableBarrier:
    """``transport.py:74-87`` (host-side epoch barrier for probes/eval)."""

    def __init__(self, parties: int):
        self._barrier = threading.Barrier(parties)

    def wait(self, timeout: float = DEFAULT_TIMEOUT):
        try:
            self._barrier.wait(timeout)
        except threading.BrokenBarrierError:
            raise ProtocolError("barrier poisoned: a worker aborted") from None

    def poison(self):
        self._barrier.abort()


SEG_BYTES = 40          # sizeof(hb_segment_t)


def _align16(n: int) -> int:
    return (n + 15) & ~15


@dataclass
class _Msg:
    src: int          # sending partition
    dst: int          # receiving partition
    rows: int
    row_begin: int    # position in the flattened send (or receive) row list


class PhasePlan:
    """Static (layer-independent) index maps of one phase on one rank."""

    def __init__(self, phase, send_msgs, send_rows, recv_msgs, dst_rows, src_ptr, src_rows):
        self.phase = phase
        self.send_msgs = send_msgs      # list[_Msg], sorted by (src, dst)
        self.send_rows = send_rows      # int32 numpy, source row per flattened send row
        self.recv_msgs = recv_msgs      # list[_Msg], sorted by (src, dst)
        self.dst_rows = dst_rows        # int32 numpy, K2 destination rows
        self.src_ptr = src_ptr          # int32 numpy CSR over dst_rows
        self.src_rows = src_rows        # int32 numpy, flattened receive indices
        self.dev = None

    def to(self, device):
        import torch

        def t(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(device)
        self.dev = dict(send_rows=t(self.send_rows), dst_rows=t(self.dst_rows),
                        src_ptr=t(self.src_ptr), src_rows=t(self.src_rows))
        return self


class RankLayout:
    """Row layout of the partitions one rank hosts.

    ``owner[p]`` is the rank of partition p; ``parts`` maps hosted partition
    id → Partition (each with ``send_sets``/``recv_sets`` per peer,
    ``graph.py:70-100``).
    """

    def __init__(self, parts: dict, owner, rank: int):
        self.rank = rank
        self.owner = list(owner)
        self.num_partitions = len(self.owner)
        self.ids = sorted(parts)
        self.parts = [parts[i] for i in self.ids]
        self.nl = {p.id: p.num_local for p in self.parts}
        self.nh = {p.id: p.num_halo for p in self.parts}
        self.loc_base, self.halo_base = {}, {}
        a = b = 0
        for p in self.parts:
            self.loc_base[p.id], self.halo_base[p.id] = a, b
            a += p.num_local
            b += p.num_halo
        self.NL, self.NH = a, b
        self.ranks = sorted(set(self.owner))
        self.fwd = self._phase_plan(FORWARD)
        self.bwd = self._phase_plan(BACKWARD)

    def _phase_plan(self, phase) -> PhasePlan:
        fwd = phase == FORWARD
        send_msgs, send_rows = [], []
        pos = 0
        for p in self.parts:
            for q in range(self.num_partitions):
                if q == p.id:
                    continue
                idx = p.send_sets[q] if fwd else p.recv_sets[q]
                if len(idx) == 0:
                    continue
                send_msgs.append(_Msg(p.id, q, len(idx), pos))
                pos += len(idx)
                if fwd:
                    send_rows.append(self.loc_base[p.id] + np.asarray(idx))
                else:
                    send_rows.append(self.NL + self.halo_base[p.id] + np.asarray(idx))
        # receive side: messages (p -> q) for hosted q, sorted by (p, q)
        recv = []
        for q in self.parts:
            for p in range(self.num_partitions):
                if p == q.id:
                    continue
                idx = q.recv_sets[p] if fwd else q.send_sets[p]
                if len(idx):
                    recv.append((p, q.id, np.asarray(idx)))
        recv.sort(key=lambda m: (m[0], m[1]))
        recv_msgs, dst, srcp = [], [], []
        pos = 0
        for p, qid, idx in recv:
            recv_msgs.append(_Msg(p, qid, len(idx), pos))
            if fwd:
                dst.append(self.NL + self.halo_base[qid] + idx)
            else:
                dst.append(self.loc_base[qid] + idx)
            srcp.append(np.full(len(idx), p, dtype=np.int64))
            pos += len(idx)
        cat = (lambda xs: np.concatenate(xs).astype(np.int64)) if recv else \
            (lambda xs: np.zeros(0, dtype=np.int64))
        dst_all, src_part = cat(dst), cat(srcp)
        flat = np.arange(len(dst_all), dtype=np.int64)
        if fwd:
            dst_rows, src_ptr, src_rows = dst_all, np.arange(len(dst_all) + 1), flat
        else:
            # integrate j[S_k] += recv_k in ascending peer order (trainer.py:214-216):
            # destination-major CSR, sources sorted by (dst row, peer)
            o = np.lexsort((src_part, dst_all))
            d_sorted = dst_all[o]
            dst_rows, starts = sorted_unique_index(d_sorted)
            src_ptr = np.append(starts, len(d_sorted))
            src_rows = flat[o]
        srows = np.concatenate(send_rows).astype(np.int64) if send_rows else np.zeros(0, np.int64)
        return PhasePlan(phase, send_msgs, srows, recv_msgs, dst_rows, src_ptr, src_rows)

    def to(self, device):
        self.fwd.to(device)
        self.bwd.to(device)
        return self


class ExchangeBuffers:
    """Wire buffers + descriptor tables for one (layer, phase, d, bits)."""

    def __init__(self, layout: RankLayout, plan: PhasePlan, d: int, bits: int, device,
                 parities: int = 1):
        import torch
        self.layout, self.plan, self.d, self.bits = layout, plan, d, bits
        me = layout.rank
        size = [_align16(wire_bytes(m.rows, d, bits)) for m in plan.recv_msgs]
        # receive buffer: groups by source rank, (src, dst) order inside a group
        self.recv_off, self.recv_group = {}, {}
        off = 0
        for r in layout.ranks:
            g0 = off
            for m, sz in zip(plan.recv_msgs, size):
                if layout.owner[m.src] == r:
                    self.recv_off[(m.src, m.dst)] = off
                    off += sz
            if off > g0:
                self.recv_group[r] = (g0, off - g0)
        self.recv_bytes = off
        # send buffer: messages to remote ranks, grouped by destination rank
        self.send_off, self.send_group = {}, {}
        off = 0
        for r in layout.ranks:
            if r == me:
                continue
            g0 = off
            for m in plan.send_msgs:
                if layout.owner[m.dst] == r:
                    self.send_off[(m.src, m.dst)] = off
                    off += _align16(wire_bytes(m.rows, d, bits))
            if off > g0:
                self.send_group[r] = (g0, off - g0)
        self.send_bytes = off
        self.recv = [torch.zeros(max(16, self.recv_bytes), dtype=torch.uint8, device=device)
                     for _ in range(parities)]
        self.send = torch.zeros(max(16, self.send_bytes), dtype=torch.uint8, device=device)
        # element offsets of each sender's stream: peers ascending, empty skipped
        self.elem_off = {}
        acc = {}
        for m in plan.send_msgs:
            self.elem_off[(m.src, m.dst)] = acc.get(m.src, 0)
            acc[m.src] = acc.get(m.src, 0) + m.rows * d
        # static receive-side descriptors per parity
        self.recv_segs = []
        for par in range(parities):
            seg = np.zeros(len(plan.recv_msgs), dtype=_lib.SEGMENT_DTYPE)
            base = self.recv[par].data_ptr()
            for i, m in enumerate(plan.recv_msgs):
                seg[i] = (0, 0, 0, base + self.recv_off[(m.src, m.dst)], m.row_begin, m.rows)
            self.recv_segs.append(torch.from_numpy(seg.view(np.uint8).copy()).to(device))
        self.n_send = len(plan.send_msgs)
        self.n_recv = len(plan.recv_msgs)
        self.comm_done = [None] * parities     # CUDA events of in-flight remote exchanges
        # K1 descriptor tables change every epoch (keys): staged through two
        # pinned host slots so the upload is asynchronous (no stream sync)
        self._dev = torch.device(device)
        self._seg_dev = torch.zeros(max(1, self.n_send) * SEG_BYTES, dtype=torch.uint8, device=device)
        self._seg_host = None
        self._seg_ev = [None, None]
        self._seg_slot = 0
        self.capture = None                    # an EpochGraph while one is being captured
        # peer-memory exchange (PeerLinks): receiving rank's mapped receive
        # buffer base per (rank, parity), message offsets on the receiver
        self.peer_recv, self.peer_off = None, None

    def send_table(self, seed: int, epoch: int, layer: int, parity: int) -> np.ndarray:
        """hb_segment_t rows for this exchange (keys depend on the epoch)."""
        me = self.layout.rank
        seg = np.zeros(self.n_send, dtype=_lib.SEGMENT_DTYPE)
        keys = {}
        for i, m in enumerate(self.plan.send_msgs):
            if m.src not in keys:
                keys[m.src] = derive_key((seed, m.src, epoch, layer, self.plan.phase)) \
                    if self.bits != 32 else (0, 0)
            r = self.layout.owner[m.dst]
            if r == me:
                out = self.recv[parity].data_ptr() + self.recv_off[(m.src, m.dst)]
            elif self.peer_recv is not None:
                # peer-memory exchange: straight into the receiving rank's buffer
                out = self.peer_recv[(r, parity)] + self.peer_off[(m.src, m.dst)]
            else:
                out = self.send.data_ptr() + self.send_off[(m.src, m.dst)]
            k = keys[m.src]
            seg[i] = (k[0], k[1], self.elem_off[(m.src, m.dst)], out, m.row_begin, m.rows)
        return seg

    def upload_send_table(self, seed: int, epoch: int, layer: int, parity: int):
        """Device copy of ``send_table(...)`` (stream-ordered, host does not block)."""
        import torch
        tab = self.send_table(seed, epoch, layer, parity).view(np.uint8)
        if self._dev.type != "cuda":
            self._seg_dev.copy_(torch.from_numpy(tab.copy()))
            return self._seg_dev
        cap = self.capture
        if cap is not None:
            # inside a CUDA-graph capture: the copy becomes a memcpy node reading
            # a pinned buffer the graph owns (allocated before the capture);
            # each replay re-fills it with the replayed epoch's table first
            host = cap.pinned(self, tab.size)
            host.numpy()[:] = tab
            _lib.call("hb_upload_async", self._seg_dev.data_ptr(), host.data_ptr(), tab.size,
                      _lib.stream_handle())
            cap.add_fill(lambda e, b=host: b.numpy().__setitem__(
                slice(None), self.send_table(seed, e, layer, parity).view(np.uint8)))
            return self._seg_dev
        if self._seg_host is None:
            self._seg_host = [torch.empty(tab.size, dtype=torch.uint8).pin_memory() for _ in range(2)]
        k = self._seg_slot = self._seg_slot ^ 1
        if self._seg_ev[k] is not None:
            self._seg_ev[k].synchronize()          # the copy from this slot two uploads ago
        self._seg_host[k].numpy()[:] = tab
        # a kernel reading the mapped pinned slot (hb_upload_async), not a
        # copy-engine transfer that would queue behind a feature upload
        _lib.call("hb_upload_async", self._seg_dev.data_ptr(), self._seg_host[k].data_ptr(), tab.size,
                  _lib.stream_handle())
        self._seg_ev[k] = torch.cuda.current_stream(self._dev).record_event()
        return self._seg_dev

    def stats_delta(self) -> dict:
        """Per sending partition byte meters of one exchange (transport.py:105-114)."""
        out = {}
        for m in self.plan.send_msgs:
            s = out.setdefault(m.src, [0, 0, 0, 0])
            s[0] += payload_bytes(m.rows, self.d, self.bits)
            s[1] += metadata_bytes(m.rows, self.bits)
            s[2] += HEADER_BYTES
            s[3] += 1
        return out

    def wire_bytes_total(self) -> int:
        return sum(wire_bytes(m.rows, self.d, self.bits) for m in self.plan.send_msgs)


def host_staged(group=None) -> bool:
    """True when the process group cannot move device buffers itself (gloo:
    used by the multi-process tests that share one GPU); the wire blocks are
    then staged through host memory.  Production runs NCCL (device to device
    over NVLink)."""
    import torch.distributed as dist
    return dist.get_backend(group) != "nccl"


class PeerLinks:
    """Peer-memory halo exchange (``hb_p2p_*``, N > 1 with one process per GPU).

    Replaces the NCCL send/recv of ``nccl_exchange`` for the halo blocks (the
    reference's ``exchange``, transport.py:172-205): every rank exports its
    receive buffers once as CUDA IPC handles; the other ranks map them, and
    K1 writes each remote message's wire block straight into the receiver's
    buffer (NVLink / NVSwitch peer stores) — the transfer happens inside the
    quantize kernel.  Arrival and buffer reuse are ordered by monotonically
    increasing 64-bit counters, one block per rank: ``cnt[e, p, 0]`` counts
    arrivals into this rank's receive buffer of exchange e, parity p;
    ``cnt[e, p, 1 + r]`` counts receiver r's consumptions of what this rank
    wrote there.  All ranks run the same exchange schedule, so a rank derives
    every target from its own history:

    * before K1 (use n of (e, p)): wait until each remote receiver r has
      consumed (e, p) as often as this rank has (``cnt[e, p, 1 + r] >=
      own consumptions``) — the data about to be overwritten is no longer
      read, Sylvie-A re-reads included;
    * after K1: +1 on each remote receiver's ``cnt[e, p, 0]``;
    * before K2: wait until ``cnt[e, p, 0] >= own sends into (e, p) x remote
      senders`` — the latest blocks have all arrived;
    * after K2: +1 on each remote sender's ``cnt[e, p, 1 + me]``.

    A wait that times out sets FLAG_PROTOCOL in the rank's device flag word."""

    def __init__(self, exchanges: list, group, device, timeout: float, parities: int = 2):
        import torch
        import torch.distributed as dist
        self.torch = torch
        self.ex = list(exchanges)
        self.index = {id(b): i for i, b in enumerate(self.ex)}
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.timeout_ns = int(timeout * 1e9)
        E, P, W = len(self.ex), parities, self.world
        self.cnt = torch.zeros((E, P, 1 + W), dtype=torch.int64, device=device)
        self.sends = np.zeros((E, P), dtype=np.int64)
        self.consumes = np.zeros((E, P), dtype=np.int64)
        me = self.rank

        def export(t):
            h = (ctypes.c_char * 64)()
            off = ctypes.c_int64()
            _lib.call("hb_ipc_get_handle", t.data_ptr(), h, ctypes.byref(off))
            return bytes(h), int(off.value)
        # every rank takes part in each collective whatever happens locally, so
        # a failure anywhere makes all ranks fall back together
        try:
            mine = {"cnt": export(self.cnt),
                    "recv": [[export(b.recv[p]) for p in range(len(b.recv))] for b in self.ex],
                    "recv_off": [dict(b.recv_off) for b in self.ex]}
        except Exception:
            mine = None
        allr = [None] * W
        dist.all_gather_object(allr, mine, group=group)
        if any(x is None for x in allr):
            raise RuntimeError("a rank could not export its receive buffers as CUDA IPC handles")
        self.opened = []
        bases = {}

        def open_(h):
            # one mapping per exported allocation: the caching allocator packs
            # small buffers (the counters) into shared segments, and a handle
            # is opened once per process
            if h[0] not in bases:
                base = ctypes.c_void_p()
                _lib.call("hb_ipc_open_handle", h[0], ctypes.byref(base))
                bases[h[0]] = base.value
                self.opened.append(base.value)
            return bases[h[0]] + h[1]
        try:
            self._map(allr, open_, me, W, E, P)
            ok = 1
        except Exception:
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32,
                            device="cpu" if host_staged(group) else device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if not int(flag.item()):
            self.close()
            for b in self.ex:
                b.peer_recv, b.peer_off = None, None
            raise RuntimeError("a rank could not map its peers' receive buffers")

    def _map(self, allr, open_, me, W, E, P):
        torch = self.torch
        device = self.cnt.device
        cnt_addr = {r: (self.cnt.data_ptr() if r == me else open_(allr[r]["cnt"])) for r in range(W)}
        stride = self.cnt.stride()
        el = self.cnt.element_size()

        def caddr(r, e, p, k):
            return cnt_addr[r] + el * (e * stride[0] + p * stride[1] + k * stride[2])
        self.send_ranks, self.recv_ranks = [], []
        sig_send, sig_recv = [], []
        for e, b in enumerate(self.ex):
            sr = sorted(b.send_group)                       # remote ranks this rank writes to
            rr = sorted(r for r in b.recv_group if r != me)  # remote ranks writing here
            self.send_ranks.append(sr)
            self.recv_ranks.append(rr)
            b.peer_recv = {(r, p): open_(allr[r]["recv"][e][p]) for r in sr for p in range(len(b.recv))}
            b.peer_off = {}
            for r in sr:
                b.peer_off.update({k: v for k, v in allr[r]["recv_off"][e].items()})
            sig_send.append([[caddr(r, e, p, 0) for r in sr] for p in range(P)])
            sig_recv.append([[caddr(r, e, p, 1 + me) for r in rr] for p in range(P)])
        # device arrays of counter addresses for hb_p2p_signal, per (e, p)
        self._sig = {}
        for e in range(E):
            for p in range(P):
                for kind, lst in (("send", sig_send[e][p]), ("recv", sig_recv[e][p])):
                    if lst:
                        self._sig[(kind, e, p)] = torch.tensor(lst, dtype=torch.int64, device=device)

    # CUDA-graph epochs (DeviceRank.run_epoch_graphed): while an EpochGraph is
    # being captured, every wait reads its target from a device slot the graph
    # uploads from its pinned buffer at the start of each replay; before a
    # replay the recorded calls are re-run in "fill" mode, which only advances
    # the counters and writes the targets the eager path would have used
    capture = None
    _fill = None

    def _wait(self, e, p, k, target, flags, stream):
        if self._fill is not None:
            self._fill.append(int(target))
            return
        addr = self.cnt.data_ptr() + self.cnt.element_size() * (
            e * self.cnt.stride(0) + p * self.cnt.stride(1) + k * self.cnt.stride(2))
        cap = self.capture
        if cap is not None:
            slot = cap.p2p_slot(int(target))
            _lib.call("hb_p2p_wait", addr, 0, slot, _lib.ptr(flags), FLAG_PROTOCOL, self.timeout_ns,
                      _lib.stream_handle(stream))
            return
        if target <= 0:
            return
        _lib.call("hb_p2p_wait", addr, int(target), None, _lib.ptr(flags), FLAG_PROTOCOL, self.timeout_ns,
                  _lib.stream_handle(stream))

    def _signal(self, kind, e, p, stream):
        if self._fill is not None:
            return
        a = self._sig.get((kind, e, p))
        if a is not None:
            _lib.call("hb_p2p_signal", a.data_ptr(), a.numel(), _lib.stream_handle(stream))

    def _record(self, name, bufs, parity):
        if self.capture is not None:
            self.capture.p2p_calls.append((name, bufs, parity))

    def before_send(self, bufs, parity, flags, stream=None):
        """Before K1 writes into the peers' (e, parity) buffers."""
        self._record("before_send", bufs, parity)
        e = self.index[id(bufs)]
        for r in self.send_ranks[e]:
            self._wait(e, parity, 1 + r, self.consumes[e, parity], flags, stream)

    def after_send(self, bufs, parity, stream=None):
        self._record("after_send", bufs, parity)
        e = self.index[id(bufs)]
        self.sends[e, parity] += 1
        self._signal("send", e, parity, stream)

    def before_recv(self, bufs, parity, flags, stream=None):
        """Before K2 reads the (e, parity) receive buffer."""
        self._record("before_recv", bufs, parity)
        e = self.index[id(bufs)]
        self._wait(e, parity, 0, self.sends[e, parity] * len(self.recv_ranks[e]), flags, stream)

    def after_recv(self, bufs, parity, stream=None):
        self._record("after_recv", bufs, parity)
        e = self.index[id(bufs)]
        self.consumes[e, parity] += 1
        self._signal("recv", e, parity, stream)

    def replay_targets(self, calls) -> list:
        """Advance the counters through a captured epoch's calls and return
        the wait targets in capture order (no launches)."""
        out = []
        self._fill = out
        try:
            for name, bufs, parity in calls:
                if name in ("before_send", "before_recv"):
                    getattr(self, name)(bufs, parity, None)
                else:
                    getattr(self, name)(bufs, parity)
        finally:
            self._fill = None
        return out

    def close(self):
        for base in self.opened:
            try:
                _lib.call("hb_ipc_close", base)
            except Exception:
                pass
        self.opened = []


ENVELOPE_MAGIC = int.from_bytes(b"HBM1", "little")
_PHASE_CODE = {FORWARD: 0, BACKWARD: 1}
FLAG_PROTOCOL = 2          # device flag bit: an envelope did not match its exchange's tag


def envelope(src_rank: int, dst_rank: int, tag) -> list:
    """The ``Message`` envelope of one rank-to-rank group (transport.py:23-59:
    magic "HBM1", src, dst and the tag (epoch, layer, phase)) as 6 int64."""
    epoch, layer, phase = tag
    return [ENVELOPE_MAGIC, src_rank, dst_rank, int(epoch), int(layer), _PHASE_CODE[phase]]


def nccl_exchange(bufs: ExchangeBuffers, parity: int, group=None, tag=None, flags=None):
    """Move the remote groups with NCCL send/recv (one pair per peer rank).
    Called on the comm stream; a no-op on a single rank.

    tag = (epoch, layer, phase): every group travels with its 48-byte envelope
    (not byte-metered, like the reference's ``Message`` header) and the
    receiver checks it against its own tag — the reference's tag check in
    ``Fabric.recv`` (transport.py:115-124).  A mismatch raises ProtocolError
    at once when the exchange is host-staged (gloo), and sets FLAG_PROTOCOL in
    the device word ``flags`` on the NCCL path (read at the epoch check)."""
    import torch
    import torch.distributed as dist
    stage = bufs.send.is_cuda and host_staged(group)
    me = bufs.layout.rank
    ops, landing, envs = [], [], []
    env_dev = bufs.send.device if not stage else torch.device("cpu")
    for r, (o, n) in bufs.send_group.items():
        t = bufs.send[o:o + n]
        ops.append(dist.P2POp(dist.isend, t.cpu() if stage else t, r, group=group))
        if tag is not None:
            e = torch.tensor(envelope(me, r, tag), dtype=torch.int64, device=env_dev)
            ops.append(dist.P2POp(dist.isend, e, r, group=group))
    for r, (o, n) in bufs.recv_group.items():
        if r == me:
            continue
        t = bufs.recv[parity][o:o + n]
        h = t.cpu() if stage else t
        if stage:
            landing.append((t, h))
        ops.append(dist.P2POp(dist.irecv, h, r, group=group))
        if tag is not None:
            e = torch.empty(6, dtype=torch.int64, device=env_dev)
            envs.append((r, e))
            ops.append(dist.P2POp(dist.irecv, e, r, group=group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for t, h in landing:
        t.copy_(h, non_blocking=False)
    for r, e in envs:
        want = torch.tensor(envelope(r, me, tag), dtype=torch.int64, device=e.device)
        if e.device.type == "cpu":
            if not torch.equal(e, want):
                got = e.tolist()
                raise ProtocolError(f"tag mismatch from rank {r}: got (epoch {got[3]}, layer {got[4]}, "
                                    f"phase {got[5]}), expected {tuple(tag)}")
        elif flags is not None:
            flags.bitwise_or_(torch.ne(e, want).any().to(flags.dtype) * FLAG_PROTOCOL)
