"""Thin torch-tensor wrappers over the C-ABI kernels (no host fallback).

Each wrapper names the reference function it replaces.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import ptr, stream_handle


class DeviceCsr:
    """CSR matrix resident in HBM: int64 row_ptr, int32 col_idx, fp32 values,
    plus the {next row chunk, warps finished} counter pair its dynamically
    scheduled SpMM launches use (zero between launches)."""

    def __init__(self, rows: int, cols: int, row_ptr, col_idx, values, device):
        import torch
        self.rows, self.cols = int(rows), int(cols)
        self.row_ptr = torch.from_numpy(np.ascontiguousarray(row_ptr, dtype=np.int64)).to(device)
        self.col_idx = torch.from_numpy(np.ascontiguousarray(col_idx, dtype=np.int32)).to(device)
        self.values = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float32)).to(device)
        self.nnz = int(self.col_idx.numel())
        self.work = torch.zeros(2, dtype=torch.int32, device=device)

    @classmethod
    def from_csr(cls, m, device):
        return cls(m.rows, m.cols, m.row_ptr, m.col_idx, m.values, device)


def factor_scales(a: DeviceCsr):
    """Diagonal factorisation of the values, if there is one:
    values[i, j] == r[i] * c[j] over a 0/1 pattern, for the trainer's
    aggregation operators (graph.py:120-141):

    * row-constant rows (SAGE mean D^-1 A):          r = row value, c = None;
    * column-constant columns (its transpose A^T D^-1): r = None, c = column value;
    * GCN D^-1/2 (A+I) D^-1/2 and its partition blocks / their transposes
      (self loops on the square part): r = c = sqrt(diag) there, the other
      rows' / columns' factors from their nonzeros; values within 2^-21
      relative of r[i] c[j].

    Returns (r, c) fp32 device tensors (either may be None), or None when the
    values do not factor (general matrices keep per-nonzero values)."""
    import torch
    if a.nnz == 0:
        return None
    dev = a.row_ptr.device
    v = a.values
    counts = a.row_ptr[1:] - a.row_ptr[:-1]
    rows = torch.repeat_interleave(torch.arange(a.rows, device=dev, dtype=torch.int64), counts)
    col = a.col_idx.long()
    nonempty = counts > 0
    first = torch.zeros(a.rows, dtype=v.dtype, device=dev)
    first[nonempty] = v[a.row_ptr[:-1][nonempty]]
    if bool((v == first[rows]).all()):
        return first, None
    cfirst = torch.zeros(a.cols, dtype=v.dtype, device=dev).scatter_(0, col, v)
    if bool((v == cfirst[col]).all()):
        return None, cfirst
    # GCN: the self loops give r = c = sqrt(diag) on the square part; rows /
    # columns without a diagonal entry (the halo columns of a partition block,
    # the halo rows of its transpose) take their factor from any nonzero whose
    # other factor is known
    m = min(a.rows, a.cols)
    dmask = col == rows
    if not bool(dmask.any()):
        return None
    vd = v.double()
    nan = float("nan")
    r = torch.full((a.rows,), nan, dtype=torch.float64, device=dev)
    c = torch.full((a.cols,), nan, dtype=torch.float64, device=dev)
    di = rows[dmask]
    if bool((vd[dmask] <= 0).any()):
        return None
    r[di] = vd[dmask].sqrt()
    c[di] = r[di]
    del m
    # a missing factor comes from the row's (column's) first qualifying
    # nonzero in CSR order: scatter_ with repeated indices would keep an
    # arbitrary one, and the candidates differ in their last bits, which made
    # two identical runs differ (min-index scatter_reduce is order-independent)
    nnz_idx = torch.arange(v.numel(), device=dev)
    for fill, known, fk, ok in ((r, c, rows, col), (c, r, col, rows)):
        sel = torch.isnan(fill[fk]) & ~torch.isnan(known[ok])
        if bool(sel.any()):
            first_nz = torch.full((fill.numel(),), v.numel(), dtype=torch.int64, device=dev)
            first_nz.scatter_reduce_(0, fk[sel], nnz_idx[sel], reduce="amin")
            tgt = (first_nz < v.numel()).nonzero().view(-1)
            e = first_nz[tgt]
            fill[tgt] = vd[e] / known[ok[e]]
    rr, cc = r[rows], c[col]
    if bool(torch.isnan(rr).any() | torch.isnan(cc).any()):
        return None
    if not bool(((vd - rr * cc).abs() <= 2.0 ** -21 * vd.abs()).all()):
        return None
    return torch.nan_to_num(r, nan=0.0).float(), torch.nan_to_num(c, nan=0.0).float()
    return None


class TiledCsr:
    """The K3/K4 tiled layout of a ``DeviceCsr`` (built on the device, once per
    matrix): dense (row block x 64-column window) tiles holding at least
    ``threshold`` nonzeros — their X windows are staged in shared memory by TMA
    and reused across the block's rows — and a residual CSR for the rest.
    Tile records keep the CSR's (row, column) order, so each row still sums its
    tile contributions in ascending column order, then its residual ones.

    Two record formats:
    * general (``hb_spmm_tiled``): 64-row blocks, 8-byte {col, val} records;
    * factored (``hb_spmm_tiled_bin``, when ``factor_scales`` finds the values
      to be r[i] c[j] over a 0/1 pattern — the trainer's aggregation
      operators): 64- or 128-row blocks, one-byte column records, r / c
      applied as diagonal scalings; ``window=128`` (64-row blocks, rows of
      at most 48 columns) doubles the nonzeros per (row, tile)."""

    def __init__(self, a: DeviceCsr, threshold: int = 64, factored: bool | None = None,
                 block_rows: int | None = None, window: int = 64, block_order: str | None = None):
        import torch
        dev = a.row_ptr.device
        scales = factor_scales(a) if factored in (None, True) else None
        if factored is True and scales is None:
            raise ValueError("matrix values do not factor into diagonal scalings of a 0/1 pattern")
        self.binary = scales is not None
        self.row_scale, self.col_scale = scales if self.binary else (None, None)
        if self.binary:
            import os
            # 120-row blocks (30 consumer warps x 4 rows): the staged X window
            # serves 120 rows (profiles/r2_kbench_spmm_wide.jsonl)
            rb = block_rows or int(os.environ.get("HB_BIN_RB", "120"))
            if rb not in (64, 120, 128):
                raise ValueError(f"factored tiles are 64, 120 or 128 rows, not {rb}")
            self.RB, self.ROWOFF, self.MAXREC = rb, (72 if rb == 64 else 136), 2048
        else:
            self.RB, self.ROWOFF, self.MAXREC = 64, 72, 1024
        if window not in (64, 128, 255) or (window != 64 and not self.binary) or \
                (window == 128 and self.RB != 64) or (window != 64 and self.RB == 120):
            raise ValueError("128-column windows need factored 64-row tiles, 255-column ones factored tiles")
        if window == 255 and self.RB == 128:
            self.MAXREC = 4096
        self.W = window
        self.rows, self.cols, self.nnz = a.rows, a.cols, a.nnz
        self.work = torch.zeros(2, dtype=torch.int32, device=dev)
        self._xs = {}
        RB, W = self.RB, self.W
        self.nblocks = (a.rows + RB - 1) // RB
        nwin = (a.cols + W - 1) // W
        counts_row = a.row_ptr[1:] - a.row_ptr[:-1]
        rows = torch.repeat_interleave(torch.arange(a.rows, device=dev, dtype=torch.int64), counts_row)
        col = a.col_idx.long()
        key = (rows // RB) * nwin + col // W
        order = torch.sort(key, stable=True).indices          # (block, window) groups, CSR order inside
        skey = key[order]
        del key
        uniq, cnt = torch.unique_consecutive(skey, return_counts=True)
        dense_g = cnt >= threshold
        gid = torch.repeat_interleave(torch.arange(len(uniq), device=dev), cnt)
        dense_nz = dense_g[gid]
        grp_key, grp_cnt = uniq[dense_g], cnt[dense_g]
        # a tile holds at most `cap` records (the kernel's smem record slot;
        # factored tiles pad each row's run to whole 4-byte words, up to 3
        # bytes per row); denser (block, window) groups become several tiles
        # of the same window
        cap = self.MAXREC - 3 * RB if self.binary else self.MAXREC
        nsplit = (grp_cnt + cap - 1) // cap
        sub_of_grp = torch.repeat_interleave(torch.arange(grp_key.numel(), device=dev), nsplit)
        first_sub = torch.zeros(grp_key.numel() + 1, dtype=torch.int64, device=dev)
        first_sub[1:] = torch.cumsum(nsplit, 0)
        j = torch.arange(sub_of_grp.numel(), device=dev) - first_sub[sub_of_grp]
        tile_key = grp_key[sub_of_grp]
        tile_cnt = torch.clamp(grp_cnt[sub_of_grp] - j * cap, max=cap)
        self.ntiles = int(tile_key.numel())
        tile_blk = tile_key // nwin
        self.tile_win = (tile_key % nwin).to(torch.int32).contiguous()
        tp = torch.zeros(self.nblocks + 1, dtype=torch.int64, device=dev)
        tp[1:] = torch.cumsum(torch.bincount(tile_blk, minlength=self.nblocks), 0)
        self.tile_ptr = tp.to(torch.int32)
        didx = order[dense_nz]                                # original nonzero ids, tile order
        grp_of = (torch.cumsum(dense_g.long(), 0) - 1)[gid[dense_nz]]
        gstart = torch.zeros(grp_key.numel() + 1, dtype=torch.int64, device=dev)
        gstart[1:] = torch.cumsum(grp_cnt, 0)
        grank = torch.arange(didx.numel(), device=dev) - gstart[grp_of]
        tile_of = first_sub[grp_of] + grank // cap
        rank = grank % cap                                    # position in the tile (rows ascending)
        rel = col[didx] - self.tile_win.long()[tile_of] * W
        lr = rows[didx] % RB
        per = torch.bincount(tile_of * RB + lr, minlength=self.ntiles * RB).view(self.ntiles, RB)
        ro = torch.zeros((self.ntiles, self.ROWOFF), dtype=torch.int64, device=dev)
        if self.binary:
            # row runs padded to 4-byte words (0xFF fills the padding): the
            # kernel reads a row's records one word at a time
            pc = (per + 3) // 4 * 4
            ro[:, 1:RB + 1] = torch.cumsum(pc, 1)
            start = torch.zeros((self.ntiles, RB), dtype=torch.int64, device=dev)
            start[:, 1:] = torch.cumsum(per, 1)[:, :-1]       # unpadded start of each row in the tile
            padded = (ro[:, RB] + 15) // 16 * 16
            off = torch.zeros(self.ntiles + 1, dtype=torch.int64, device=dev)
            off[1:] = torch.cumsum(padded, 0)
            pos = off[tile_of] + ro[tile_of, lr] + (rank - start[tile_of, lr])
            rec = torch.full((max(16, int(off[-1].item())),), 0xFF, dtype=torch.uint8, device=dev)
            rec[pos] = rel.to(torch.uint8)
            self.tile_nz = rec
            self.tile_off = off                               # byte offsets
        else:
            ro[:, 1:RB + 1] = torch.cumsum(per, 1)
            padded = (tile_cnt + 1) // 2 * 2                  # 16-byte aligned record runs
            off = torch.zeros(self.ntiles + 1, dtype=torch.int64, device=dev)
            off[1:] = torch.cumsum(padded, 0)
            pos = off[tile_of] + rank
            nz = torch.zeros((int(off[-1].item()), 2), dtype=torch.int32, device=dev)
            nz[pos, 0] = rel.to(torch.int32)
            nz[pos, 1] = a.values[didx].view(torch.int32)
            self.tile_nz = nz
            self.tile_off = off                               # record (8-byte) offsets
        self.tile_rowoff = ro.to(torch.int16).contiguous()     # values <= MAXREC, read as uint16
        # work-item order (hb_spmm_tiled_bin block_order): ascending blocks by
        # default (the CTAs in flight share X windows in L2); "lpt": heaviest
        # block first; "lightK": ascending, but the K lightest blocks last,
        # lightest at the very end (the dynamically scheduled tail is made of
        # light blocks while most of the matrix keeps its L2 locality)
        self.block_order = None
        if block_order is not None:
            blk_nnz = torch.zeros(self.nblocks, dtype=torch.int64, device=dev)
            blk_nnz.index_add_(0, torch.div(rows, RB, rounding_mode="floor"), torch.ones_like(rows))
            if block_order == "lpt":
                order = torch.sort(-blk_nnz, stable=True).indices
            elif block_order.startswith("light") and block_order[5:].isdigit():
                k = min(self.nblocks, int(block_order[5:]))
                light = torch.sort(blk_nnz, stable=True).indices[:k]
                is_light = torch.zeros(self.nblocks, dtype=torch.bool, device=dev)
                is_light[light] = True
                order = torch.cat([torch.nonzero(~is_light).view(-1), light.flip(0)])
            else:
                raise ValueError(f"unknown block order {block_order!r}")
            self.block_order = order.to(torch.int32).contiguous()
        keep = torch.ones(a.nnz, dtype=torch.bool, device=dev)
        keep[didx] = False
        rp = torch.zeros(a.rows + 1, dtype=torch.int64, device=dev)
        rp[1:] = torch.cumsum(torch.bincount(rows[keep], minlength=a.rows), 0)
        self.res_ptr = rp
        self.res_col = a.col_idx[keep].contiguous()
        self.res_val = a.values[keep].contiguous()
        self.tiled_nnz = int(didx.numel())

    @property
    def tiled_fraction(self) -> float:
        return self.tiled_nnz / max(1, self.nnz)

    def col_scaled_scratch(self, ld: int, device):
        """The c X copy hb_spmm_tiled_bin writes when there is a column scale."""
        import torch
        if ld not in self._xs:
            self._xs[ld] = torch.empty((self.cols, ld), dtype=torch.float32, device=device)
        return self._xs[ld]


def spmm_tiled(t: TiledCsr, x, out, d: int | None = None, stream=None):
    """``linalg.spmm`` (linalg.py:71-75) through the TMA-staged tiled kernel
    (the factored one-byte-record kernel when ``t.binary``)."""
    d = x.shape[1] if d is None else d
    if t.binary:
        xs = t.col_scaled_scratch(x.stride(0), x.device) if t.col_scale is not None else None
        _lib.call("hb_spmm_tiled_bin", t.rows, t.cols, t.nblocks, ptr(t.tile_ptr), ptr(t.tile_win),
                  ptr(t.tile_off), ptr(t.tile_rowoff), ptr(t.tile_nz), ptr(t.res_ptr), ptr(t.res_col),
                  ptr(t.row_scale), ptr(t.col_scale), ptr(x), x.stride(0), d, ptr(out), out.stride(0),
                  ptr(xs), xs.stride(0) if xs is not None else 0, ptr(t.work), t.RB, t.W, ptr(t.block_order),
                  stream_handle(stream))
        return out
    _lib.call("hb_spmm_tiled", t.rows, t.cols, t.nblocks, ptr(t.tile_ptr), ptr(t.tile_win), ptr(t.tile_off),
              ptr(t.tile_rowoff), ptr(t.tile_nz), ptr(t.res_ptr), ptr(t.res_col), ptr(t.res_val), ptr(x),
              x.stride(0), d, ptr(out), out.stride(0), ptr(t.work), stream_handle(stream))
    return out


SPMM_ALGOS = {"auto": 0, "rows": 1}


def spmm(a: DeviceCsr, x, out, d: int | None = None, stream=None, algo: str = "auto", window: int = 0,
         stream_col: int | None = None):
    """``linalg.spmm`` (linalg.py:71-75): out[:rows, :d] = A @ x[:, :d].
    Columns >= stream_col (halo copies) are read L2-evict-first."""
    d = x.shape[1] if d is None else d
    sc = 2**31 - 1 if stream_col is None else int(stream_col)
    _lib.call("hb_spmm_csr_ex", a.rows, ptr(a.row_ptr), ptr(a.col_idx), ptr(a.values), ptr(x),
              x.stride(0), d, ptr(out), out.stride(0), a.nnz, SPMM_ALGOS[algo], int(window), sc,
              ptr(a.work), stream_handle(stream))
    return out


def gemm(A, B, C, beta: float = 0.0, relu_out=None, ws=None, stream=None):
    """C (+)= A @ B on tcgen05 (3xTF32), A/B any 2-D strided fp32 views
    (trainer.py:294,313,318-321).  Returns C."""
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    if C is None:       # store only relu(A B)
        assert relu_out is not None and beta == 0.0
    else:
        assert C.shape[0] == M and C.shape[1] == N and C.stride(1) == 1
    _lib.call("hb_gemm_f32", M, N, K, ptr(A), A.stride(0), A.stride(1), ptr(B), B.stride(0),
              B.stride(1), ptr(C), C.stride(0) if C is not None else 0, float(beta), ptr(relu_out),
              relu_out.stride(0) if relu_out is not None else 0, ptr(ws),
              ws.numel() if ws is not None else 0, stream_handle(stream))
    return C


def gemm2(A1, B1, A2, B2, C, beta: float = 0.0, relu_out=None, ws=None, stream=None):
    """C = A1 @ B1 + A2 @ B2 (+ beta C) in one tcgen05 pass where the operands
    allow: the SAGE combine [h | A h] [W_top; W_bot] without the concatenation
    (trainer.py:294,318-321).  Returns C."""
    M, K1 = A1.shape
    M2, K2 = A2.shape
    assert M == M2 and B1.shape[0] == K1 and B2.shape[0] == K2 and B1.shape[1] == B2.shape[1]
    N = B1.shape[1]
    if C is None:       # store only relu(A1 B1 + A2 B2)
        assert relu_out is not None and beta == 0.0
    else:
        assert C.shape[0] == M and C.shape[1] == N and C.stride(1) == 1
    _lib.call("hb_gemm2_f32", M, N, K1, ptr(A1), A1.stride(0), A1.stride(1), ptr(B1), B1.stride(0), B1.stride(1),
              K2, ptr(A2), A2.stride(0), A2.stride(1), ptr(B2), B2.stride(0), B2.stride(1), ptr(C),
              C.stride(0) if C is not None else 0,
              float(beta), ptr(relu_out), relu_out.stride(0) if relu_out is not None else 0, ptr(ws),
              ws.numel() if ws is not None else 0, stream_handle(stream))
    return C


def spmm_set_narrow(variant: int):
    """Consumer layout of the factored tiled SpMM for d <= 48 (tuning / tests);
    the meaning depends on the tile window, see hb_spmm_set_narrow (1 is the
    default)."""
    _lib.call("hb_spmm_set_narrow", int(variant))


def gemm_set_path(path: int):
    """0: TMA warp-specialised tcgen05 kernels where operands allow; 1: SIMT-staged kernel;
    3: the A-in-TMEM kernel for every shape."""
    _lib.call("hb_gemm_set_path", int(path))


XENT_PARTIALS = 256      # HB_XENT_PARTIALS


def softmax_xent(logits, C: int, labels, mask, norm: float, grad, row_loss, loss_out, stream=None,
                 keep_unmasked: bool = False, partials=None):
    """``linalg.softmax_cross_entropy`` (linalg.py:87-112) on device.
    keep_unmasked: grad / row_loss rows outside the mask already hold zeros.
    partials: XENT_PARTIALS doubles of scratch (allocated here if omitted)."""
    import torch
    n = labels.numel()
    if partials is None and n > 16 * 1024:
        partials = torch.empty(XENT_PARTIALS, dtype=torch.float64, device=logits.device)
    _lib.call("hb_softmax_xent", ptr(logits), logits.stride(0), n, C, ptr(labels), ptr(mask),
              float(norm), ptr(grad), grad.stride(0), ptr(row_loss), ptr(loss_out), int(bool(keep_unmasked)),
              ptr(partials), stream_handle(stream))


def sigmoid_bce(logits, C: int, labels, mask, norm: float, grad, row_loss, loss_out, stream=None,
                keep_unmasked: bool = False, partials=None):
    """Multi-label sigmoid BCE (extension; include/halob200.h hb_sigmoid_bce).
    labels: uint8 (n x C) 0/1 matrix."""
    import torch
    n = labels.shape[0]
    if partials is None and n > 16 * 1024:
        partials = torch.empty(XENT_PARTIALS, dtype=torch.float64, device=logits.device)
    _lib.call("hb_sigmoid_bce", ptr(logits), logits.stride(0), n, C, ptr(labels), labels.stride(0), ptr(mask),
              float(norm), ptr(grad), grad.stride(0), ptr(row_loss), ptr(loss_out), int(bool(keep_unmasked)),
              ptr(partials), stream_handle(stream))


def multilabel_counts(logits, C: int, labels, mask, counts, stream=None):
    """TP / FP / FN per mask value (hb_multilabel_counts), counts: int64[9]."""
    _lib.call("hb_multilabel_counts", ptr(logits), logits.stride(0), labels.shape[0], C, ptr(labels),
              labels.stride(0), ptr(mask), ptr(counts), stream_handle(stream))


def relu(z, y, n: int, d: int, stream=None):
    """``linalg.relu`` (linalg.py:78-80)."""
    _lib.call("hb_relu", ptr(z), z.stride(0), n, d, ptr(y), y.stride(0), stream_handle(stream))


def relu_grad_mul(j, h, m, n: int, d: int, stream=None):
    """``j * relu_grad(z)`` (trainer.py:312, linalg.py:83-84) with h = relu(z)."""
    _lib.call("hb_relu_grad_mul", ptr(j), j.stride(0), ptr(h), h.stride(0), n, d, ptr(m),
              m.stride(0), stream_handle(stream))


def adam_step(w, g, m, v, lr, t, b1=0.9, b2=0.999, eps=1e-8, stream=None, guard=None, bc=None):
    """``linalg.adam_step`` (linalg.py:127-140) in place on device tensors.
    guard = (loss f64, flags u32, flags2 u32 or None) device tensors: the step is
    skipped on the device when the loss is not finite or a flag is set.
    bc: device f64[2] holding (1-b1^t, 1-b2^t) (needs guard; t is then unused):
    the launch's arguments do not change with the epoch (CUDA-graph replays)."""
    if bc is not None:
        loss, flags, flags2 = guard
        _lib.call("hb_adam_step_dev", ptr(w), ptr(g), ptr(m), ptr(v), w.numel(), float(lr), float(b1),
                  float(b2), float(eps), ptr(bc), ptr(loss), ptr(flags), ptr(flags2), stream_handle(stream))
    elif guard is None:
        _lib.call("hb_adam_step", ptr(w), ptr(g), ptr(m), ptr(v), w.numel(), float(lr), float(b1),
                  float(b2), float(eps), 1.0 - b1 ** t, 1.0 - b2 ** t, stream_handle(stream))
    else:
        loss, flags, flags2 = guard
        _lib.call("hb_adam_step_guarded", ptr(w), ptr(g), ptr(m), ptr(v), w.numel(), float(lr), float(b1),
                  float(b2), float(eps), 1.0 - b1 ** t, 1.0 - b2 ** t, ptr(loss), ptr(flags), ptr(flags2),
                  stream_handle(stream))


def upload(dst, host, stream=None):
    """Stream-ordered copy of the pinned host tensor `host` into `dst` (same
    byte size) through hb_upload_async: capturable as a graph memcpy node."""
    n = host.numel() * host.element_size()
    if dst.numel() * dst.element_size() < n:
        raise ValueError("upload: destination smaller than the host buffer")
    _lib.call("hb_upload_async", ptr(dst), host.data_ptr(), n, stream_handle(stream))


def argmax_accuracy(logits, C: int, labels, mask, counts, stream=None):
    """Counts for ``evaluate`` (trainer.py:129-144)."""
    _lib.call("hb_argmax_accuracy", ptr(logits), logits.stride(0), labels.numel(), C,
              ptr(labels), ptr(mask), ptr(counts), stream_handle(stream))


def dropout(x, nrows: int, row0: int, d: int, key, p: float, out, stream=None):
    """Keyed dropout of ``trainer.py:285-289`` (mask regenerated, never stored)."""
    _lib.call("hb_dropout", ptr(x), x.stride(0), nrows, row0, d, int(key[0]), int(key[1]),
              float(p), ptr(out), out.stride(0), stream_handle(stream))
