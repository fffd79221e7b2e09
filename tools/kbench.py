"""Microbenchmarks of the halo-path kernels on synthetic inputs (GPU box).

  python tools/kbench.py codec [--rows R --d D --bits B --segs S]
  python tools/kbench.py spmm  [--config reddit]      (real planted graph, all SpMM shapes)

Times each kernel with CUDA events over several launches (inputs > L2), prints
one JSON line per case with achieved algorithmic GB/s.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def _time(fn, reps=10, warm=3):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def codec(args):
    import torch
    from paper_2303_01277_b200 import codec as C
    from paper_2303_01277_b200.rngstream import derive_key
    rng = np.random.default_rng(0)
    R, d, b, S = args.rows, args.d, args.bits, args.segs
    ld = (d + 3) // 4 * 4
    nsrc = int(R * 1.5)
    src = torch.randn(nsrc, ld, device="cuda") * torch.rand(nsrc, 1, device="cuda") * 3
    idx = np.sort(rng.choice(nsrc, size=R, replace=False)).astype(np.int32)
    bounds = np.linspace(0, R, S + 1).astype(int)
    rows = np.diff(bounds)
    sizes = [(C.wire_bytes(int(r), d, b) + 15) // 16 * 16 for r in rows]
    out = torch.zeros(sum(sizes), dtype=torch.uint8, device="cuda")
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    keys = [derive_key((0, s // 7, 1, 1, "forward")) for s in range(S)]
    eoff = [int((bounds[s] - bounds[(s // 7) * 7]) * d) for s in range(S)]
    segs = C.segments_tensor([int(r) for r in rows], keys, eoff,
                             [out.data_ptr() + int(o) for o in offs], "cuda")
    ridx = torch.from_numpy(idx).cuda()
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    ms = _time(lambda: C.quantize_gather(src, ridx, segs, S, d, b, flags))
    nbytes = R * d * 4 + R * 4 + sum(C.wire_bytes(int(r), d, b) for r in rows)
    print(json.dumps({"kernel": "quantize_gather", "rows": R, "d": d, "bits": b, "ms": ms,
                      "gbps": nbytes / ms / 1e6, "gelem_s": R * d / ms / 1e6}), flush=True)
    # K2 forward scatter into a halo region
    dst = torch.zeros(nsrc, ld, device="cuda")
    drow = torch.from_numpy(rng.permutation(nsrc)[:R].astype(np.int32)).cuda()
    ptr = torch.arange(R + 1, dtype=torch.int32, device="cuda")
    srows = torch.arange(R, dtype=torch.int32, device="cuda")
    ms2 = _time(lambda: C.dequant_gather(segs, S, drow, ptr, srows, d, b, dst, False))
    nb2 = sum(C.wire_bytes(int(r), d, b) for r in rows) + R * d * 4 + 12 * R
    print(json.dumps({"kernel": "dequant_gather", "rows": R, "d": d, "bits": b, "ms": ms2,
                      "gbps": nb2 / ms2 / 1e6}), flush=True)


def spmm(args):
    import torch
    sys.path.insert(0, str(ROOT))
    from bench import build_graph
    from paper_2303_01277_b200 import ops
    from paper_2303_01277_b200.trainer import _stack_csr, _transpose_device
    from paper_2303_01277_b200.transport import RankLayout
    t0 = time.time()
    g, parts = build_graph(args.config)
    lay = RankLayout(parts, [0] * len(parts), 0)
    which = "mean" if args.config != "yelp" else "adj"
    rp, ci, v = _stack_csr(lay, which)
    A = ops.DeviceCsr(lay.NL, lay.NL + lay.NH, rp, ci, v, "cuda")
    At = _transpose_device(A)
    print(json.dumps({"setup_s": time.time() - t0, "NL": lay.NL, "NH": lay.NH, "nnz": A.nnz}), flush=True)
    tiled = {}
    cases = (("A", A, 602), ("A", A, 256), ("At", At, 256), ("A", A, 128), ("At", At, 128), ("A", A, 100),
             ("A", A, 64), ("A", A, 41), ("At", At, 41), ("A", A, 47), ("At", At, 47), ("A", A, 512),
             ("At", At, 512), ("A", A, 300))
    if args.d_list:
        cases = tuple(c for c in cases if c[2] in args.d_list)
    for name, M, d in cases:
        ld = (d + 3) // 4 * 4
        X = torch.randn(M.cols, ld, device="cuda")
        Y = torch.zeros(M.rows, ld, device="cuda")
        comp = 8 * (M.rows + 1) + 8 * M.nnz + 4 * M.cols * d + 4 * M.rows * d
        variants = [("rows", 0)] + ([("tiled", 0), ("tiled_bin64", 0), ("tiled_bin128", 0)] if args.config == "reddit" else []) + \
            ([("tiled_bin64w128", 0), ("tiled_bin64w255", 0), ("tiled_bin128w255", 0)]
             if args.config == "reddit" and d <= 48 else []) + \
            ([("rows", 4), ("rows", 16)] if d <= 64 else []) + ([("rows", 1), ("rows", 4)] if d > 256 else [])
        if args.tiled_only:
            variants = [v for v in variants if v[0].startswith("tiled")]
        for algo, win in variants:
            if algo.startswith("tiled"):
                key = (name, algo)
                if key not in tiled:
                    t0 = time.time()
                    spec = algo[len("tiled_bin"):] if algo.startswith("tiled_bin") else None
                    rb = int(spec.split("w")[0]) if spec else None
                    win = int(spec.split("w")[1]) if spec and "w" in spec else 64
                    tiled[key] = ops.TiledCsr(M, factored=rb is not None, block_rows=rb, window=win)
                    torch.cuda.synchronize()
                    print(json.dumps({"tiled": name, "algo": algo, "build_s": round(time.time() - t0, 2),
                                      "tiles": tiled[key].ntiles,
                                      "tiled_fraction": round(tiled[key].tiled_fraction, 4)}), flush=True)
                T = tiled[key]
                if T.binary and d <= 48 and T.RB == 64:           # (both window sizes)
                    for nv in (0, 1, 2, 3):         # narrow consumer layouts (hb_spmm_set_narrow)
                        ops.spmm_set_narrow(nv)
                        ms = _time(lambda: ops.spmm_tiled(T, X, Y, d), reps=5)
                        print(json.dumps({"kernel": "spmm", "mat": name, "d": d, "algo": algo, "narrow": nv,
                                          "ms": round(ms, 3),
                                          "gather_gbps": round((8 * M.nnz + 4 * M.nnz * d) / ms / 1e6, 1)}),
                              flush=True)
                    ops.spmm_set_narrow(1)
                ms = _time(lambda: ops.spmm_tiled(T, X, Y, d), reps=5)
            else:
                sc = lay.NL if name == "A" else None
                ms = _time(lambda: ops.spmm(M, X, Y, d, algo=algo, window=win, stream_col=sc), reps=5)
            print(json.dumps({"kernel": "spmm", "mat": name, "d": d, "algo": algo, "window": win,
                              "ms": round(ms, 3), "compulsory_gbps": round(comp / ms / 1e6, 1),
                              "gather_gbps": round((8 * M.nnz + 4 * M.nnz * d) / ms / 1e6, 1),
                              "tflops": round(2 * M.nnz * d / ms / 1e9, 2)}), flush=True)


def gemm(args):
    import torch
    from paper_2303_01277_b200 import ops
    NL = 232_965
    g = torch.Generator(device="cuda").manual_seed(0)
    cases = [("Z=P W   (l1 half)", NL, 256, 602, "nn"), ("Z=P W   (l2 half)", NL, 256, 256, "nn"),
             ("Z=P W   (l3 half)", NL, 41, 256, "nn"), ("G=P^T m (l1 half)", 602, 256, NL, "tn"),
             ("G=P^T m (l3 half)", 256, 41, NL, "tn"), ("T=m W^T (l2)", NL, 256, 256, "nt"),
             ("T=m W^T (l3)", NL, 256, 41, "nt")]
    if args.config == "ogbn":
        NL = 2_449_029
        cases = [("Z=P W   (l1 half)", NL, 128, 100, "nn"), ("Z=P W   (l2 half)", NL, 128, 128, "nn"),
                 ("Y=H W   (l3 bot)", NL, 47, 128, "nn"), ("G=P^T m (l2 half)", 128, 128, NL, "tn"),
                 ("T=m W^T (l2)", NL, 128, 128, "nt"), ("dual Z=[H|AH] W (l1)", NL, 128, 100, "dual"),
                 ("dual Z=[H|AH] W (l2)", NL, 128, 128, "dual"), ("dual j=[S|m] W^T (l3)", NL, 128, 47, "dualt"), ("dual j=[S|m] W^T (l2)", NL, 128, 128, "dualt")]
    if args.config == "yelp":
        NL = 716_847
        cases = [("Z=AH W (l1)", NL, 512, 300, "nn"), ("Z=AH W (l2)", NL, 512, 512, "nn"),
                 ("Y=H W (l4)", NL, 100, 512, "nn"), ("G=P^T m (l2)", 512, 512, NL, "tn"),
                 ("T=m W^T (l2)", NL, 512, 512, "nt"), ("T=m W^T (l4)", NL, 512, 100, "nt")]
    ws = torch.empty(64 * 602 * 256, device="cuda")
    def mat(r, c):   # row-major with a 16-byte row stride, like the trainer's buffers
        return torch.randn(r, (c + 3) // 4 * 4, device="cuda", generator=g)[:, :c]
    for name, M, N, K, kind in cases:
        if kind.startswith("dual"):
            A1, A2 = mat(M, K), mat(M, K)
            if kind == "dual":
                W = mat(2 * K, N)
                B1, B2 = W[:K], W[K:]
            else:   # the trainer's W_bot^T / W_top^T views of one padded (2K x N) weight
                W = mat(2 * N, K)
                B1, B2 = W[N:].t(), W[:N].t()
            C = mat(M, N)
            ms = _time(lambda: ops.gemm2(A1, B1, A2, B2, C, ws=ws), reps=5)
            ms2 = _time(lambda: (ops.gemm(A1, B1, C, ws=ws), ops.gemm(A2, B2, C, beta=1.0, ws=ws)), reps=5)
            print(json.dumps({"gemm": name, "M": M, "N": N, "K": 2 * K, "dual_ms": round(ms, 4),
                              "two_pass_ms": round(ms2, 4),
                              "dual_hbm_gbps": round(4 * M * (2 * K + N) / ms / 1e6, 1)}), flush=True)
            continue
        if kind == "nn":
            A, B = mat(M, K), mat(K, N)
        elif kind == "tn":
            A, B = mat(K, M).t(), mat(K, N)
        else:
            A, B = mat(M, K), mat(N, K).t()
        C = mat(M, N)
        ms = _time(lambda: ops.gemm(A, B, C, ws=ws), reps=5)
        ops.gemm_set_path(1)
        ms_v1 = _time(lambda: ops.gemm(A, B, C, ws=ws), reps=5)
        ops.gemm_set_path(0)
        ms_cb = _time(lambda: torch.mm(A, B, out=C), reps=5)
        fl = 2.0 * M * N * K
        if args.config in ("ogbn", "yelp"):
            print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "tcgen05_ms": round(ms, 4),
                              "tf32x3_frac": round(3 * fl / ms / 1e9 / 826.0, 3),
                              "hbm_gbps": round(4 * (M * K + M * N + K * N) / ms / 1e6, 1),
                              "cublas_fp32_ms": round(ms_cb, 4)}), flush=True)
            continue
        print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "tcgen05_tma_ms": round(ms, 4),
                          "tcgen05_simt_staged_ms": round(ms_v1, 4), "cublas_fp32_ms": round(ms_cb, 4),
                          "tcgen05_tflops": round(fl / ms / 1e9, 1), "cublas_tflops": round(fl / ms_cb / 1e9, 1)}),
              flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["codec", "spmm", "gemm"])
    ap.add_argument("--rows", type=int, default=461_644)
    ap.add_argument("--d", type=int, default=602)
    ap.add_argument("--bits", type=int, default=1)
    ap.add_argument("--segs", type=int, default=56)
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--d-list", type=int, nargs="*", default=None)
    ap.add_argument("--tiled-only", action="store_true")
    a = ap.parse_args()
    {"codec": codec, "spmm": spmm, "gemm": gemm}[a.what](a)
