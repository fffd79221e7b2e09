"""Multi-rank halo exchange over torch.distributed (gloo, world sizes 2, 4 and
8, CPU).

The N>1 device path (one rank per GPU, NCCL) runs the same host code as here:
``RankLayout`` splits the partitions over ranks, ``ExchangeBuffers`` lays the
wire blocks out (receive buffer grouped by source rank, send buffer grouped
by destination rank), ``send_table`` gives K1 its per-message keys, stream
offsets and output addresses, and ``nccl_exchange`` moves one contiguous
group per peer rank.  On CPU the K1 launch is replaced by the oracle writing
the reference's ``QuantizedBlock`` bytes to exactly the addresses
``send_table`` hands K1; after the gloo exchange every receiving rank must
hold, at its planned offsets, the bytes the reference's ``exchange``
(transport.py:172-205) would deliver — keyed per sender by
(seed, partition, epoch, layer, phase), stream offsets restarting per
exchange and advancing over non-empty peers in ascending order.  The K2 index
maps (forward: halo slots R_k; backward: ascending-peer integration into S_k,
trainer.py:208-216) are replayed in numpy against the same semantics.
"""

import ctypes
import os
import socket
import traceback

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

SEED, EPOCH, LAYER, D = 5, 3, 2, 20


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# world size -> partition owners (non-contiguous: every rank's partitions are
# interleaved with other ranks')
OWNERS = {2: [0, 1, 0, 1], 4: [1, 0, 3, 2, 1, 0, 3, 2], 8: [3, 0, 6, 1, 7, 2, 5, 4]}


def _parts(n):
    from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
    from paper_2303_01277_b200.graph import build_partitions
    g = generate_sbm(SbmSpec(nodes_per_community=25 if n == 4 else 15, communities=n, feature_dim=D, seed=3))
    return build_partitions(g, n, "hash", 0, "gcn")[2]


def _rows(p, peer, phase):
    """Rows partition p sends to `peer` (trainer.py:175-206): forward its local
    rows S_peer (fp32 features), backward its halo-gradient rows R_peer
    (synthetic fp32 values keyed by the partition)."""
    from paper_2303_01277_b200.rngstream import FORWARD
    if phase == FORWARD:
        return np.asarray(p.features, dtype=np.float32)[p.send_sets[peer]].astype(np.float64)
    halo = np.random.default_rng(100 + p.id).standard_normal((p.num_halo, D)).astype(np.float32)
    return halo[p.recv_sets[peer]].astype(np.float64)


def _block(rows, key, offset, bits):
    from oracle.codec import quantize, wire_block
    from oracle.rng import uniforms_restated
    u = uniforms_restated(key, offset, rows.size) if bits != 32 else None
    rmin, rscale, codes = quantize(rows, bits, u)
    return wire_block(rmin, rscale, codes, bits, rows.shape[0], rows.shape[1])


def _expected_blocks(parts, phase, bits):
    """(src, dst) -> wire bytes, restated independently of the planner."""
    from oracle.rng import derive_key
    out = {}
    for p in parts:
        key = derive_key((SEED, p.id, EPOCH, LAYER, phase))
        off = 0
        for q in range(len(parts)):          # peers ascending, empty ones skipped
            if q == p.id:
                continue
            rows = _rows(p, q, phase)
            if rows.shape[0] == 0:
                continue
            out[(p.id, q)] = _block(rows, key, off, bits)
            off += rows.size
    return out


def _check(rank, world):
    from oracle.codec import dequantize, parse_wire_block
    from paper_2303_01277_b200.rngstream import BACKWARD, FORWARD
    from paper_2303_01277_b200.transport import ExchangeBuffers, RankLayout, nccl_exchange
    owner = OWNERS[world]
    parts = _parts(len(owner))
    lay = RankLayout({p.id: p for p in parts if owner[p.id] == rank}, owner, rank)
    checked = 0
    # every rank plans the same P2P traffic: what rank a sends to rank b is
    # what b expects from a, for every (layer width, bits, phase)
    for plan in (lay.fwd, lay.bwd):
        for bits in (1, 32):
            bufs = ExchangeBuffers(lay, plan, D, bits, "cpu", parities=1)
            mine = {"send": {r: n for r, (o, n) in bufs.send_group.items()},
                    "recv": {r: n for r, (o, n) in bufs.recv_group.items() if r != rank}}
            allp = [None] * world
            dist.all_gather_object(allp, mine)
            for a in range(world):
                for b in range(world):
                    if a != b:
                        assert allp[a]["send"].get(b, 0) == allp[b]["recv"].get(a, 0), (a, b, bits)
    for phase, plan in ((FORWARD, lay.fwd), (BACKWARD, lay.bwd)):
        for bits in (1, 4, 32):
            want = _expected_blocks(parts, phase, bits)
            bufs = ExchangeBuffers(lay, plan, D, bits, "cpu", parities=2)
            parity = EPOCH % 2
            tab = bufs.send_table(SEED, EPOCH, LAYER, parity)
            # "K1": write each message's block where send_table points
            for i, m in enumerate(plan.send_msgs):
                p = parts[m.src]
                rows = _rows(p, m.dst, phase)
                blk = _block(rows, (int(tab["key0"][i]), int(tab["key1"][i])), int(tab["elem_offset"][i]), bits)
                assert blk == want[(m.src, m.dst)], (m.src, m.dst)
                ctypes.memmove(int(tab["out"][i]), blk, len(blk))
            nccl_exchange(bufs, parity)
            got_all = bufs.recv[parity].numpy().tobytes()
            hosted = set(lay.ids)
            expect_msgs = sorted(k for k in want if k[1] in hosted)
            assert sorted((m.src, m.dst) for m in plan.recv_msgs) == expect_msgs
            for (s, d) in expect_msgs:
                off = bufs.recv_off[(s, d)]
                assert got_all[off:off + len(want[(s, d)])] == want[(s, d)], (phase, bits, s, d)
                checked += 1
            # K2 index maps, replayed: build what _assemble_halo / _integrate produce
            recv_rows = np.zeros((int(plan.src_rows.size), D))
            for m in plan.recv_msgs:
                off = bufs.recv_off[(m.src, m.dst)]
                b, r, dd, rmin, rscale, codes = parse_wire_block(got_all[off:off + len(want[(m.src, m.dst)])])
                recv_rows[m.row_begin:m.row_begin + m.rows] = dequantize(rmin, rscale, codes, b)
            total = lay.NL + lay.NH
            dev = np.zeros((total, D))
            for i, t in enumerate(plan.dst_rows):
                acc = 0.0
                for k in range(plan.src_ptr[i], plan.src_ptr[i + 1]):
                    acc = acc + recv_rows[plan.src_rows[k]]
                dev[t] += acc
            ref = np.zeros((total, D))
            for q in lay.parts:
                for p in range(len(parts)):
                    if p == q.id or (p, q.id) not in want:
                        continue
                    b, r, dd, rmin, rscale, codes = parse_wire_block(want[(p, q.id)])
                    vals = dequantize(rmin, rscale, codes, b)
                    if phase == FORWARD:          # halo[R_p] = recv_p
                        ref[lay.NL + lay.halo_base[q.id] + np.asarray(q.recv_sets[p])] = vals
                    else:                         # j[S_p] += recv_p, ascending p
                        ref[lay.loc_base[q.id] + np.asarray(q.send_sets[p])] += vals
            np.testing.assert_array_equal(dev, ref)
    # replicas agree after the gradient all-reduce (trainer.reduce_gradients)
    from paper_2303_01277_b200.trainer import reduce_gradients
    g = torch.full((7,), float(rank + 1))
    loss = torch.tensor([0.25 * (rank + 1)], dtype=torch.float64)
    reduce_gradients(g, loss)
    tot = world * (world + 1) / 2
    assert torch.all(g == tot) and float(loss) == 0.25 * tot
    return checked


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        q.put((rank, "ok", _check(rank, world)))
    except Exception:
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multi_rank_halo_exchange_matches_reference_semantics(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, info in results:
        assert status == "ok", f"rank {rank}:\n{info}"
        assert info > 0


def _tag_worker(rank, world, port, q):
    """Both ranks run one exchange; rank 1 is one epoch ahead (a diverged
    rank).  Each receiver's envelope check must raise ProtocolError
    (transport.py:115-124), and a matching exchange must pass."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        from paper_2303_01277_b200.rngstream import FORWARD
        from paper_2303_01277_b200.transport import ExchangeBuffers, ProtocolError, RankLayout, nccl_exchange
        dist.init_process_group("gloo", rank=rank, world_size=world)
        owner = OWNERS[2]
        parts = _parts(4)
        lay = RankLayout({p.id: p for p in parts if owner[p.id] == rank}, owner, rank)
        bufs = ExchangeBuffers(lay, lay.fwd, D, 1, "cpu")
        nccl_exchange(bufs, 0, tag=(3, 1, FORWARD))            # agreeing tags: no error
        try:
            nccl_exchange(bufs, 0, tag=(3 + rank, 1, FORWARD))
            q.put((rank, "fail", "no ProtocolError on a diverged tag"))
        except ProtocolError as e:
            q.put((rank, "ok", str(e)))
    except Exception:
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_envelope_tag_mismatch_raises_protocol_error():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tag_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, info in results:
        assert status == "ok", f"rank {rank}:\n{info}"
        assert "tag mismatch" in info


def test_wait_device_times_out():
    """train(timeout=) / DeviceRank(timeout=): a device epoch that never
    completes (a stalled peer on the NCCL path) raises ProtocolError, which
    train() reports as TrainingError (trainer.py:386-388, 457-464)."""
    import time
    from paper_2303_01277_b200.trainer import wait_device
    from paper_2303_01277_b200.transport import ProtocolError
    t0 = time.monotonic()
    with pytest.raises(ProtocolError, match="timed out"):
        wait_device(None, 0.05, "stalled", poll=lambda: False)
    assert time.monotonic() - t0 < 2.0
    wait_device(None, 0.05, "done", poll=lambda: True)
