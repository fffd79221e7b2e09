"""Generate golden vectors from the REAL reference (halobit) in the build container.

Run once here (``python tests/golden/make_golden.py``); the outputs are
committed under ``tests/golden/`` so tests on the GPU box (where
``/root/reference`` does not exist) can pin the oracle and the CUDA path.

Every vector comes from the reference's own public functions:
``rngstream.RngStream`` / ``_derive_key`` (rngstream.py:19-39),
``codec.quantize_rows`` / ``dequantize_rows`` / ``QuantizedBlock.to_bytes``
(codec.py:71-207), ``datasets.generate_sbm`` (datasets.py:136-171),
``graph.normalize_adjacency`` / ``partition_nodes`` / ``build_partition``
(graph.py:120-256) and ``trainer.train`` (trainer.py:386-465).
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from halobit.codec import QuantConfig, dequantize_rows, quantize_rows  # noqa: E402
from halobit.datasets import SbmSpec, generate_sbm  # noqa: E402
from halobit.graph import (build_partition, mean_adjacency,  # noqa: E402
                           normalize_adjacency, partition_nodes)
from halobit.rngstream import RngStream, _derive_key  # noqa: E402
from halobit.linalg import CsrMatrix, spmm  # noqa: E402
from halobit.trainer import ModelConfig, TrainMode, train  # noqa: E402

KEY_TUPLES = [
    (0, 0, 1, 1, "forward"), (1, 0, 1, 1, "forward"), (1, 1, 3, 2, "backward"),
    (123, 0, 1, 1, "forward"), (2303, 7, 1, 1, "forward"), (42, 3, 100, 4, "backward"),
    (1, "dropout", 0, 1, 1), (0, "init", 1),
]


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def special_rows(rng, rows, d):
    """fp32-representable rows incl. the edge cases SURVEY §8(d) lists."""
    x = rng.standard_normal((rows, d)).astype(np.float32)
    x *= rng.uniform(0.1, 5.0, size=(rows, 1)).astype(np.float32)
    if rows >= 8:
        x[1] = np.maximum(x[1], 0)             # ReLU-like: ties at 0 (the min)
        x[2] = 3.25                            # constant row → scale 0
        x[3, : d // 2] = x[3].min()            # duplicated minimum
        x[3, d // 2:] = x[3].max()             # duplicated maximum
        x[4] = 0.0                             # all-zero row
        x[5] = np.float32(-0.0)
        x[5, 0] = 1.0
        x[6] = (np.arange(d) % 3).astype(np.float32)  # lattice endpoints at b=1
        x[7] *= np.float32(1e-30)              # tiny range
    return x


def codec_cases():
    rng = np.random.default_rng(2303)
    cases = {}
    meta = []
    ci = 0
    for d in (1, 7, 64, 100, 128, 300, 602, 1024):
        for bits in (1, 2, 3, 4, 5, 7, 8, 16, 32):
            rows = 16 if d >= 300 else 37
            x = special_rows(rng, rows, d)
            key = (ci, 1, 1, 1, "forward")
            q = quantize_rows(x.astype(np.float64), QuantConfig(bits), RngStream(*key))
            # QuantizedBlock.to_bytes() cannot serialize the passthrough block
            # (empty metadata arrays, codec.py:73-75); keep the f64 payload.
            wire = q.to_bytes() if bits != 32 else q.payload
            deq = dequantize_rows(q)
            cases[f"x{ci}"] = x
            cases[f"wire{ci}"] = np.frombuffer(wire, dtype=np.uint8)
            cases[f"deq{ci}"] = deq
            meta.append(dict(case=ci, d=d, bits=bits, rows=rows, key=list(key)))
            ci += 1
    np.savez_compressed(OUT / "codec_cases.npz", **cases)
    (OUT / "codec_cases.json").write_text(json.dumps(meta, indent=1))


def stream_cases():
    out = {}
    keys = {}
    for i, k in enumerate(KEY_TUPLES):
        kk = _derive_key(k)
        keys[i] = dict(parts=list(k), key=[int(kk[0]), int(kk[1])])
        st = RngStream(*k) if len(k) == 5 and isinstance(k[4], str) and k[4] in ("forward", "backward") else None
        if st is None:
            gen = np.random.Generator(np.random.Philox(key=kk))
            u = gen.random(4099)
        else:
            u = st.uniforms(4099)
        out[f"u{i}"] = u
        # a far window: stream elements [1_000_001, 1_000_001 + 37)
        gen = np.random.Generator(np.random.Philox(key=kk))
        gen.random(1_000_001)
        out[f"far{i}"] = gen.random(37)
    np.savez_compressed(OUT / "streams.npz", **out)
    (OUT / "streams.json").write_text(json.dumps(keys, indent=1))


def multi_peer_case():
    """One exchange of partition 1 to peers {0, 2(empty), 3}: the stream runs
    on across peers in ascending order (transport.py:184-192)."""
    rng = np.random.default_rng(7)
    out = {}
    st = RngStream(5, 1, 2, 3, "backward")
    for peer, rows in ((0, 5), (2, 0), (3, 9)):
        x = rng.standard_normal((rows, 100)).astype(np.float32)
        out[f"x{peer}"] = x
        if rows:
            out[f"wire{peer}"] = np.frombuffer(
                quantize_rows(x.astype(np.float64), QuantConfig(1), st).to_bytes(), dtype=np.uint8)
    np.savez_compressed(OUT / "multi_peer.npz", **out)


def graph_cases():
    info = {}
    spec = SbmSpec(nodes_per_community=2500, communities=4, p_in=0.006, p_out=0.0006,
                   feature_dim=64, feature_noise=1.0, seed=1)
    g = generate_sbm(spec)
    info["config1_sbm"] = dict(edges=sha(g.edges), features=sha(g.features), labels=sha(g.labels),
                               masks=sha(g.train_mask, g.val_mask, g.test_mask),
                               num_edges=int(len(g.edges)))
    a = normalize_adjacency(g)
    info["config1_ahat"] = sha(a.row_ptr, a.col_idx, a.values)
    plan = partition_nodes(g, 2, "contiguous", 0)
    parts = [build_partition(g, a, plan, k) for k in range(2)]
    info["config1_parts"] = [dict(
        halo=sha(p.halo_nodes), send=[sha(s) for s in p.send_sets],
        recv=[sha(r) for r in p.recv_sets],
        block=sha(p.adj_block.row_ptr, p.adj_block.col_idx, p.adj_block.values),
        nl=int(p.num_local), nh=int(p.num_halo)) for p in parts]
    # small graph: every strategy, SAGE mean block too
    small = {}
    gs = generate_sbm(SbmSpec(nodes_per_community=30, communities=3, seed=6))
    a = normalize_adjacency(gs)
    mh = mean_adjacency(gs)
    small["ahat"] = [a.row_ptr, a.col_idx, a.values]
    small["mean"] = [mh.row_ptr, mh.col_idx, mh.values]
    blob = {"edges": gs.edges, "features": gs.features, "labels": gs.labels,
            "train": gs.train_mask, "val": gs.val_mask, "test": gs.test_mask}
    for strat in ("contiguous", "bfs_blocks", "hash"):
        plan = partition_nodes(gs, 3, strat, 5)
        blob[f"{strat}_assign"] = plan.assignment
        for k in range(3):
            p = build_partition(gs, a, plan, k, mh)
            pre = f"{strat}_{k}_"
            blob[pre + "local"] = p.local_nodes
            blob[pre + "halo"] = p.halo_nodes
            for j in range(3):
                blob[pre + f"send{j}"] = p.send_sets[j]
                blob[pre + f"recv{j}"] = p.recv_sets[j]
            blob[pre + "A"] = np.concatenate([p.adj_block.row_ptr.astype(np.float64),
                                              p.adj_block.col_idx.astype(np.float64),
                                              p.adj_block.values])
            blob[pre + "M"] = np.concatenate([p.mean_block.row_ptr.astype(np.float64),
                                              p.mean_block.col_idx.astype(np.float64),
                                              p.mean_block.values])
    for k, v in (("ahat", small["ahat"]), ("mean", small["mean"])):
        blob[k] = np.concatenate([v[0].astype(np.float64), v[1].astype(np.float64), v[2]])
    np.savez_compressed(OUT / "graph_small.npz", **blob)
    (OUT / "graph_hashes.json").write_text(json.dumps(info, indent=1))


def spmm_cases():
    """``linalg.spmm`` (linalg.py:71-75) and ``CsrMatrix.transpose`` (:62-63)
    on the small graph's blocks and on ragged random CSR (empty rows, rows
    longer than a warp's 32-entry chunk, a dense row), fp32-representable
    inputs, f64 outputs."""
    import scipy.sparse as sp
    rng = np.random.default_rng(2303)
    out, meta = {}, []
    gs = generate_sbm(SbmSpec(nodes_per_community=30, communities=3, seed=6))
    a = normalize_adjacency(gs)
    plan = partition_nodes(gs, 3, "contiguous", 5)
    p = build_partition(gs, a, plan, 1, mean_adjacency(gs))
    mats = {"ahat_block": p.adj_block, "mean_block": p.mean_block, "ahat_block_T": p.adj_block.transpose()}
    dens = np.zeros((200, 300))
    lens = rng.integers(0, 60, size=200)
    lens[:7] = 0                      # empty rows
    lens[10] = 300                    # one dense row
    lens[11:14] = [31, 32, 33]        # chunk boundaries
    for r, ln in enumerate(lens):
        cols = rng.choice(300, size=ln, replace=False)
        dens[r, cols] = rng.standard_normal(ln).astype(np.float32)
    mats["ragged"] = CsrMatrix.from_scipy(sp.csr_matrix(dens))
    mats["ragged_T"] = mats["ragged"].transpose()
    for name, m in mats.items():
        vals = np.asarray(m.values, dtype=np.float32)
        out[name + "_rp"], out[name + "_ci"], out[name + "_v"] = m.row_ptr, m.col_idx, vals
        mm = CsrMatrix(m.rows, m.cols, m.row_ptr, m.col_idx, vals.astype(np.float64))
        widths = {"ahat_block": (1, 5, 32, 41, 64, 100, 132), "mean_block": (5, 41, 128),
                  "ahat_block_T": (5, 41, 100)}.get(name, (1, 41, 64, 256))
        for d in widths:
            x = rng.standard_normal((m.cols, d)).astype(np.float32)
            key = f"{name}_d{d}"
            out[key + "_x"] = x
            out[key + "_y"] = spmm(mm, x.astype(np.float64))   # reference output on the fp32 inputs
            meta.append(dict(key=key, mat=name, rows=int(m.rows), cols=int(m.cols), d=d,
                             nnz=int(len(m.col_idx))))
    np.savez_compressed(OUT / "spmm_cases.npz", **out)
    (OUT / "spmm_cases.json").write_text(json.dumps(meta, indent=1))


def _run(g, n, widths, model, mode, bits, epochs, seed, dropout=0.0):
    a = normalize_adjacency(g)
    mh = mean_adjacency(g) if model == "sage" else None
    plan = partition_nodes(g, n, "contiguous", 0)
    parts = [build_partition(g, a, plan, k, mh) for k in range(n)]
    res = train(g, parts, ModelConfig(widths=widths, model=model, dropout=dropout), mode,
                QuantConfig(bits), epochs, seed)
    return dict(metrics=[m.__dict__ for m in res.metrics],
                final_weights=[w.tolist() for w in res.final_weights])


def train_traces():
    traces = {}
    # BASELINE configs[0] (config 1): 2-layer GCN (64, 32, 4), 2 partitions, 1-bit, sync.
    spec = SbmSpec(nodes_per_community=2500, communities=4, p_in=0.006, p_out=0.0006,
                   feature_dim=64, feature_noise=1.0, seed=1)
    g = generate_sbm(spec)
    for seed in (1, 2, 3):
        for bits in (1, 32):
            t = _run(g, 2, (64, 32, 4), "gcn", TrainMode("sync", 0), bits, 20, seed)
            t.pop("final_weights")
            traces[f"config1_seed{seed}_b{bits}"] = t
    small = generate_sbm(SbmSpec(nodes_per_community=25, communities=4, seed=4))
    traces["small_sage_async2_b4"] = _run(small, 3, (32, 16, 4), "sage",
                                          TrainMode("async", 2), 4, 6, 3)
    traces["small_gcn_sync_b32"] = _run(small, 4, (32, 16, 4), "gcn",
                                        TrainMode("sync", 0), 32, 10, 2)
    traces["small_gcn_async0_b1_drop"] = _run(small, 2, (32, 8, 4), "gcn",
                                              TrainMode("async", 0), 1, 5, 5, dropout=0.3)
    (OUT / "train_traces.json").write_text(json.dumps(traces))


CLI_CASES = {
    # name: halobit.cli.ExperimentConfig fields (out is set per case)
    "cli_config1_b1": dict(synthetic="sbm:k=4,n=2500,pin=0.006,pout=0.0006,d=64,noise=1.0", parts=2,
                           model="gcn", layers=2, hidden=32, bits=1, epochs=12, seed=1, warmup=3),
    "cli_config1_b32": dict(synthetic="sbm:k=4,n=2500,pin=0.006,pout=0.0006,d=64,noise=1.0", parts=2,
                            model="gcn", layers=2, hidden=32, bits=32, epochs=12, seed=1, warmup=3),
    "cli_sage_async_b2": dict(synthetic="sbm:k=4,n=60,pin=0.2,pout=0.02,d=24", parts=3, partition="hash",
                              model="sage", layers=3, hidden=16, bits=2, mode="async", staleness=2,
                              epochs=6, seed=4, warmup=2),
}


def cli_cases():
    """``halobit.cli.run_experiment`` artefacts (cli.py:122-198): metrics.csv
    verbatim, summary.json without the wall-clock field."""
    import tempfile
    from halobit.cli import ExperimentConfig, run_experiment
    for name, kw in CLI_CASES.items():
        with tempfile.TemporaryDirectory() as d:
            run_experiment(ExperimentConfig(out=d, **kw))
            (OUT / f"{name}_metrics.csv").write_text((Path(d) / "metrics.csv").read_text())
            summ = json.loads((Path(d) / "summary.json").read_text())
            summ.pop("total_wall_ms")
            summ["config"].pop("out")
            (OUT / f"{name}_summary.json").write_text(json.dumps(summ, indent=1) + "\n")


if __name__ == "__main__":
    if sys.argv[1:] == ["spmm"]:
        spmm_cases()
        sys.exit(0)
    if sys.argv[1:] == ["cli"]:
        cli_cases()
        sys.exit(0)
    spmm_cases()
    stream_cases()
    codec_cases()
    multi_peer_case()
    graph_cases()
    train_traces()
    cli_cases()
    print("golden vectors written to", OUT)
