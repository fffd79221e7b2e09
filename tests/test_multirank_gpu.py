"""The multi-rank device path (DeviceRank with world size 2) on one B200.

Two processes share cuda:0 and talk over gloo (NCCL refuses two ranks on one
device), so the wire blocks are staged through host memory
(`transport.host_staged`); everything else — the per-rank layouts, K1 writing
remote messages into the send buffer and local ones straight into the
receiver's slot, the per-peer-rank send/recv groups, comm-stream ordering and
Sylvie-A deferral, the gradient/loss all-reduce — is the production N>1 code.

The same runs with the peer-memory exchange (``DeviceRank(p2p=True)``,
``transport.PeerLinks``): each rank maps the other's receive buffers through
CUDA IPC handles, K1 writes the remote wire blocks straight into them, and
the arrival / reuse counters order K1 and K2 across the two processes — must
train bit-identically to the host-staged exchange (same blocks, same K2
inputs).

Checks against the single-process run of the same 4 partitions:
* passthrough (bits 32): global losses every epoch rel 1e-5 and final weights
  max-abs/max 1e-5 (fp32 summation order of the all-reduce differs), sync and
  Sylvie-A;
* 1-bit: byte meters summed over ranks equal the single-rank meters every
  epoch, and the epoch-1 loss matches (identical inputs to the first
  exchange).
"""

import os
import socket
import traceback

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

EPOCHS = 4
CASES = [("sync", 0, 32), ("async", 0, 32), ("async", 2, 32), ("sync", 0, 1)]
GRAPH_CASES = [("sync", 0, 1), ("async", 0, 1), ("async", 2, 2)]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup():
    from paper_2303_01277_b200.datasets import SbmSpec, generate_sbm
    from paper_2303_01277_b200.graph import build_partitions
    g = generate_sbm(SbmSpec(nodes_per_community=60, communities=4, feature_dim=32, seed=8))
    return g, build_partitions(g, 4, "hash", 0, "sage")[2]


def _run(rank, world, owner, variant, st, bits, p2p=False, graphed=False, epochs=EPOCHS):
    from paper_2303_01277_b200.codec import QuantConfig
    from paper_2303_01277_b200.trainer import DeviceRank, ModelConfig, TrainMode
    from paper_2303_01277_b200.transport import RankLayout
    g, parts = _setup()
    lay = RankLayout({p.id: p for p in parts if owner[p.id] == rank}, owner, rank)
    eng = DeviceRank(lay, ModelConfig((32, 16, 8), "sage"), TrainMode(variant, st), QuantConfig(bits), 3, 0.01,
                     int(g.train_mask.sum()), device="cuda:0", p2p=p2p)
    assert (eng.p2p is not None) == bool(p2p and world > 1 and os.environ.get("HB_FORCE_FALLBACK") is None)
    losses, meters = [], []
    prev = eng.total_stats()
    if graphed:
        # epochs 3.. replayed from CUDA graphs (peer waits with per-replay targets)
        assert eng.graphable() == (eng.p2p is not None or world == 1)
        for e in range(1, epochs + 1):
            eng.run_epoch_graphed(e)
            if e > 1:
                eng.finish_epoch()
                losses.append(eng.epoch_loss)
        eng.finish_epoch()
        losses.append(eng.epoch_loss)
        torch.cuda.synchronize()
        return losses, len(eng._graphs), [w.double().cpu().numpy() for w in eng.W]
    for e in range(1, epochs + 1):
        eng.run_epoch(e)
        losses.append(eng.epoch_loss)
        t = eng.total_stats()
        meters.append(tuple(t[k] - prev[k] for k in ("main_bytes_sent", "metadata_bytes_sent",
                                                   "header_bytes_sent", "messages_sent")))
        prev = t
    torch.cuda.synchronize()
    return losses, meters, [w.double().cpu().numpy() for w in eng.W]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        out = {c: _run(rank, world, [0, 1, 1, 0], *c) for c in CASES}
        out.update({("p2p",) + c: _run(rank, world, [0, 1, 1, 0], *c, p2p=True) for c in CASES})
        for c in GRAPH_CASES:
            out[("p2p_eager6",) + c] = _run(rank, world, [0, 1, 1, 0], *c, p2p=True, epochs=6)
            out[("p2p_graph6",) + c] = _run(rank, world, [0, 1, 1, 0], *c, p2p=True, graphed=True, epochs=6)
        q.put((rank, "ok", out))
    except Exception:
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_single_rank():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, status, info = q.get(timeout=600)
        assert status == "ok", f"rank {rank}:\n{info}"
        res[rank] = info
    for p in procs:
        p.join(timeout=60)
    for case in CASES:
        single = _run(0, 1, [0, 0, 0, 0], *case)
        l0, m0, w0 = res[0][case]
        l1, m1, w1 = res[1][case]
        assert l0 == l1                                            # both ranks see the all-reduced loss
        np.testing.assert_allclose(w0[0], w1[0], rtol=0, atol=0)   # replicas bit-identical
        summed = [tuple(a + b for a, b in zip(x, y)) for x, y in zip(m0, m1)]
        assert summed == single[1], case
        if case[2] == 32:
            np.testing.assert_allclose(l0, single[0], rtol=1e-5)
            scale = max(np.abs(w).max() for w in single[2])
            assert max(np.abs(a - b).max() for a, b in zip(w0, single[2])) / scale < 1e-5, case
        else:
            assert l0[0] == pytest.approx(single[0][0], rel=1e-6)
        # the peer-memory exchange moves the same blocks: bit-identical training
        lp, mp_, wp = res[0][("p2p",) + case]
        assert lp == l0 and mp_ == m0, case
        for a, b in zip(wp, w0):
            np.testing.assert_array_equal(a, b)
        assert res[1][("p2p",) + case][0] == l1
    # CUDA-graph epochs over the peer-memory exchange: bit-identical to eager epochs
    for case in GRAPH_CASES:
        for r in (0, 1):
            le, _, we = res[r][("p2p_eager6",) + case]
            lg, ngraphs, wg = res[r][("p2p_graph6",) + case]
            assert ngraphs >= 2, case
            assert lg == le, (r, case)
            for a, b in zip(wg, we):
                np.testing.assert_array_equal(a, b)


def test_p2p_counter_kernels():
    """hb_p2p_signal adds 1 (system-scope release) to every counter of its
    address list; hb_p2p_wait returns once the counter reaches the target and
    gives up after its timeout with the flag bit set instead of hanging."""
    from paper_2303_01277_b200 import _lib
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    addrs = torch.tensor([cnt.data_ptr() + 8 * i for i in (0, 2, 2)], dtype=torch.int64, device="cuda")
    _lib.call("hb_p2p_signal", addrs.data_ptr(), 3, _lib.stream_handle())
    _lib.call("hb_p2p_wait", cnt.data_ptr() + 16, 2, None, flags.data_ptr(), 2, 10**9, _lib.stream_handle())
    tgt = torch.tensor([3], dtype=torch.int64, device="cuda")      # target from device memory
    _lib.call("hb_p2p_wait", cnt.data_ptr() + 16, 99, tgt.data_ptr(), flags.data_ptr(), 2, 2 * 10**6,
              _lib.stream_handle())
    torch.cuda.synchronize()
    assert cnt.tolist() == [1, 0, 2, 0] and int(flags) == 2        # 2 < 3: the device target timed out
    flags.zero_()
    _lib.call("hb_p2p_wait", cnt.data_ptr() + 8, 1, None, flags.data_ptr(), 2, 2 * 10**6, _lib.stream_handle())
    torch.cuda.synchronize()
    assert int(flags) == 2


def _fallback_worker(rank, world, port, q):
    """Rank 1 cannot export its buffers: both ranks must agree to fall back to
    the (here host-staged) send/recv exchange and train identically to it."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.pop("HB_P2P", None)
    os.environ["HB_FORCE_FALLBACK"] = "1"         # _run: expect no peer links after the failure
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2303_01277_b200 import _lib
        if rank == 1:
            real = _lib.call

            def broken(name, *args):
                if name == "hb_ipc_get_handle":
                    raise _lib.HaloLibError("hb_ipc_get_handle: simulated failure")
                return real(name, *args)
            _lib.call = broken
        import warnings
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            out = _run(rank, world, [0, 1, 1, 0], "sync", 0, 1, p2p=True)
        q.put((rank, "ok", (out, [str(x.message) for x in w])))
    except Exception:
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_p2p_setup_failure_falls_back_on_every_rank():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fallback_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, status, info = q.get(timeout=600)
        assert status == "ok", f"rank {rank}:\n{info}"
        res[rank] = info
    for p in procs:
        p.join(timeout=60)
    (l0, m0, _), warn0 = res[0]
    (l1, _, _), warn1 = res[1]
    assert any("peer-memory halo exchange unavailable" in s for s in warn0)
    assert any("peer-memory halo exchange unavailable" in s for s in warn1)
    assert l0 == l1


def _world4_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        out = {}
        for c in (("sync", 0, 1), ("async", 2, 2)):
            out[("staged",) + c] = _run(rank, world, [0, 1, 2, 3], *c)
            out[("p2p",) + c] = _run(rank, world, [0, 1, 2, 3], *c, p2p=True)
        q.put((rank, "ok", out))
    except Exception:
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_four_ranks_peer_memory_matches_staged():
    """Four processes on one GPU, one partition each: every rank maps three
    peers' receive buffers; the peer-memory exchange trains bit-identically to
    the host-staged one (sync 1-bit, Sylvie-A with the adaptor at 2 bits)."""
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_world4_worker, args=(r, 4, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, status, info = q.get(timeout=900)
        assert status == "ok", f"rank {rank}:\n{info}"
        res[rank] = info
    for p in procs:
        p.join(timeout=60)
    for c in (("sync", 0, 1), ("async", 2, 2)):
        for r in range(4):
            ls, ms, ws = res[r][("staged",) + c]
            lp, mp_, wp = res[r][("p2p",) + c]
            assert lp == ls and mp_ == ms, (r, c)
            for a, b in zip(wp, ws):
                np.testing.assert_array_equal(a, b)
