"""Oracle: the distributed Sylvie epoch, restated sequentially (TEST INFRASTRUCTURE ONLY).

The reference runs one thread per partition that meet at in-process queues
(``halobit/trainer.py:386-465``, ``transport.py:90-205``).  Because every
random draw is keyed by (seed, partition, epoch, layer, phase) and the
all-reduce sums in partition order, the result does not depend on thread
interleaving, so this oracle simulates all partitions layer-synchronously in
one thread (optionally running the per-partition dense/sparse products on a
thread pool, as the reference's workers do).

Restated pieces (reference file:line):
* send/recv gathers ``h[S_k]`` / ``j_full[nl + R_k]`` — trainer.py:175-206;
* halo assembly ``halo[R_k] = recv_k`` (zeros elsewhere) — trainer.py:208-212;
* integration ``j[S_k] += recv_k`` in ascending peer order — trainer.py:214-216;
* one keyed stream per exchange consumed over peers in ascending order, empty
  sets skipped — trainer.py:220-223, transport.py:172-205;
* Sylvie-A slots: consume epoch t-1 data (epoch 1: zeros / no integration),
  adaptor-forced sync epochs drain then refresh — trainer.py:232-246,250-351;
* ``staleness_adaptor`` — trainer.py:70-76;
* GCN ``p = A h~`` / SAGE ``p = [h~[:nl] | M h~]``, ``z = p W``, ReLU except
  the last layer, dropout on ``h~`` with keyed Philox masks — trainer.py:280-299;
* backward ``m = j * relu'(z)``, ``G = p^T m``, ``j_full = A^T (m W^T)`` (SAGE:
  ``M^T (m W_bot^T)`` + ``m W_top^T`` on local rows) — trainer.py:302-351;
* all-reduce in partition order, NaN check, Adam — trainer.py:353-372,
  transport.py:126-148, linalg.py:87-140;
* byte meters — transport.py:105-114, 146-147.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.sparse as sp

from . import codec as ocodec
from .rng import Stream, keyed_generator

FWD, BWD = "forward", "backward"


class OracleProtocolError(RuntimeError):
    pass


def staleness_mode(epoch: int, variant: str, staleness: int) -> str:
    """trainer.py:70-76."""
    if variant == "sync":
        return "sync"
    return "sync" if staleness > 0 and epoch % staleness == 0 else "async"


def glorot_weights(widths, model: str, seed: int) -> list:
    """trainer.py:102-112 (keyed Philox, identical replica on every partition)."""
    out = []
    for l in range(1, len(widths)):
        fan_in = widths[l - 1] * (2 if model == "sage" else 1)
        lim = np.sqrt(6.0 / (fan_in + widths[l]))
        out.append(keyed_generator(seed, "init", l).uniform(-lim, lim, size=(fan_in, widths[l])))
    return out


def xent(logits, labels, mask, norm):
    """linalg.py:87-112: masked softmax-CE with a global normalizer."""
    grad = np.zeros_like(logits)
    idx = np.flatnonzero(np.asarray(mask, dtype=bool))
    if idx.size == 0:
        return 0.0, grad
    z = logits[idx] - logits[idx].max(axis=1, keepdims=True)
    ez = np.exp(z)
    den = ez.sum(axis=1)
    y = np.asarray(labels)[idx]
    loss = -(z[np.arange(idx.size), y] - np.log(den)).sum() / norm
    g = ez / den[:, None]
    g[np.arange(idx.size), y] -= 1.0
    grad[idx] = g / norm
    return float(loss), grad


class Adam:
    """linalg.py:115-140 (bias-corrected Adam)."""

    def __init__(self, lr, b1=0.9, b2=0.999, eps=1e-8):
        self.lr, self.b1, self.b2, self.eps = lr, b1, b2, eps
        self.t, self.m, self.v = 0, None, None

    def step(self, w, g):
        if self.m is None:
            self.m, self.v = np.zeros_like(w), np.zeros_like(w)
        self.t += 1
        self.m = self.b1 * self.m + (1.0 - self.b1) * g
        self.v = self.b2 * self.v + (1.0 - self.b2) * g * g
        mh = self.m / (1.0 - self.b1 ** self.t)
        vh = self.v / (1.0 - self.b2 ** self.t)
        return w - self.lr * mh / (np.sqrt(vh) + self.eps)


def _csr(m):
    """Accept a scipy matrix or any object exposing ``to_scipy()``."""
    if m is None:
        return None
    if sp.issparse(m):
        return sp.csr_matrix(m)
    return m.to_scipy()


class _Part:
    """Flattened view of one partition (either package's Partition type)."""

    def __init__(self, p):
        self.id = int(p.id)
        self.n = int(p.num_partitions)
        self.nl = len(p.local_nodes)
        self.nh = len(p.halo_nodes)
        self.S = [np.asarray(s, dtype=np.int64) for s in p.send_sets]
        self.R = [np.asarray(r, dtype=np.int64) for r in p.recv_sets]
        self.A = _csr(p.adj_block)
        self.M = _csr(p.mean_block)
        self.At = self.A.T.tocsr()
        self.Mt = self.M.T.tocsr() if self.M is not None else None
        self.x = np.asarray(p.features, dtype=np.float64)
        self.labels = np.asarray(p.labels)
        self.train_mask = np.asarray(p.train_mask, dtype=bool)


class OracleTrainer:
    """Sequential restatement of ``halobit.train`` minus the centralized eval."""

    def __init__(self, parts, widths, model="gcn", variant="sync", staleness=0,
                 bits=1, seed=0, lr=0.01, global_norm=None, dropout=0.0,
                 threads: int = 1, features=None):
        self.P = [_Part(p) for p in parts]
        if features is not None:  # e.g. fp32-rounded features for GPU parity
            for q, f in zip(self.P, features):
                q.x = np.asarray(f, dtype=np.float64)
        self.n = len(self.P)
        self.widths, self.model = tuple(widths), model
        self.variant, self.staleness = variant, staleness
        self.bits, self.seed, self.dropout = bits, seed, dropout
        self.L = len(widths) - 1
        if global_norm is None:
            global_norm = max(1, int(sum(q.train_mask.sum() for q in self.P)))
        self.norm = global_norm
        self.weights = glorot_weights(widths, model, seed)
        self.adam = [Adam(lr) for _ in self.weights]
        self.slots = {}
        self.stats = [dict(main=0, meta=0, header=0, messages=0, allreduce=0)
                      for _ in self.P]
        self.loss = 0.0
        self.pool = ThreadPoolExecutor(threads) if threads > 1 else None
        self.wire_log = None  # set to a list to record (part, peer, epoch, layer, phase, bytes)

    # -- helpers ------------------------------------------------------------
    def _map(self, fn, items):
        if self.pool is None:
            return [fn(i) for i in items]
        return list(self.pool.map(fn, items))

    def exchange(self, epoch, layer, phase, outgoing):
        """outgoing[p] = {peer: rows} → received[q] = {peer: rows} (f64).

        transport.py:172-205 per partition: one keyed stream, peers ascending,
        empty sets skipped; bytes metered per transport.py:105-114.
        """
        b = self.bits
        received = [dict() for _ in self.P]
        for q in self.P:
            st = Stream(self.seed, q.id, epoch, layer, phase)
            for peer in sorted(outgoing[q.id]):
                mat = outgoing[q.id][peer]
                if mat.shape[0] == 0:
                    continue
                rows, d = mat.shape
                u = st.uniforms(rows * d) if b != 32 else None
                rmin, rscale, codes = ocodec.quantize(mat, b, u)
                s = self.stats[q.id]
                s["main"] += ocodec.payload_bytes(rows, d, b)
                s["meta"] += ocodec.metadata_bytes(rows, b)
                s["header"] += ocodec.HEADER_BYTES
                s["messages"] += 1
                if self.wire_log is not None:
                    self.wire_log.append((q.id, peer, epoch, layer, phase,
                                          ocodec.wire_block(rmin, rscale, codes, b, rows, d)))
                received[peer][q.id] = ocodec.dequantize(rmin, rscale, codes, b)
        return [dict(sorted(r.items())) for r in received]

    def _fwd_out(self, hs):
        return [{k: hs[q.id][q.S[k]] for k in range(self.n)
                 if k != q.id and len(q.S[k])} for q in self.P]

    def _bwd_out(self, jf):
        return [{k: jf[q.id][q.nl + q.R[k]] for k in range(self.n)
                 if k != q.id and len(q.R[k])} for q in self.P]

    def _halo(self, q, recv, d):
        halo = np.zeros((q.nh, d))
        for k, mat in recv.items():
            halo[q.R[k]] = mat
        return halo

    def _consume(self, epoch, layer, phase):
        ent = self.slots.get((layer, phase))
        if ent is None:
            if epoch > 1:
                raise OracleProtocolError(f"buffer underflow ({layer}, {phase}) at {epoch}")
            return 0, [dict() for _ in self.P]
        tag, data = ent
        if tag != epoch - 1:
            raise OracleProtocolError(f"staleness violation ({layer}, {phase})")
        return tag, data

    # -- one epoch ------------------------------------------------------------
    def run_epoch(self, epoch: int, probe=None) -> str:
        mode = staleness_mode(epoch, self.variant, self.staleness)
        sync_variant = self.variant == "sync"
        L, P = self.L, self.P
        hs = [q.x for q in P]
        caches = [[] for _ in P]
        for l in range(1, L + 1):
            d = self.widths[l - 1]
            if sync_variant:
                recv = self.exchange(epoch, l, FWD, self._fwd_out(hs))
            elif mode == "sync":
                if epoch > 1:
                    self._consume(epoch, l, FWD)
                recv = self.exchange(epoch, l, FWD, self._fwd_out(hs))
                self.slots[(l, FWD)] = (epoch, recv)
            else:
                tag, recv = self._consume(epoch, l, FWD)
                if probe:
                    for q in P:
                        probe("halo_consumed", part=q.id, epoch=epoch, layer=l,
                              phase=FWD, tag=tag, data=self._halo(q, recv[q.id], d))
                fresh = self.exchange(epoch, l, FWD, self._fwd_out(hs))
                self.slots[(l, FWD)] = (epoch, fresh)
            W = self.weights[l - 1]

            def fwd(i, l=l, d=d, W=W, recv=recv):
                q = P[i]
                ht = np.vstack([hs[i], self._halo(q, recv[i], d)]) if q.nh else hs[i]
                mask = None
                if self.dropout > 0.0:
                    gen = keyed_generator(self.seed, "dropout", q.id, epoch, l)
                    mask = (gen.random(ht.shape) >= self.dropout) / (1.0 - self.dropout)
                    ht = ht * mask
                if self.model == "sage":
                    p = np.hstack([ht[:q.nl], q.M @ ht])
                else:
                    p = q.A @ ht
                z = p @ W
                return (np.maximum(z, 0.0) if l < L else z), (p, z, mask)
            res = self._map(fwd, range(len(P)))
            hs = [r[0] for r in res]
            for i, r in enumerate(res):
                caches[i].append(r[1])
        logits = hs
        losses, js = [], []
        for i, q in enumerate(P):
            lo, g = xent(logits[i], q.labels, q.train_mask, self.norm)
            losses.append(lo)
            js.append(g)
        grads = [[None] * L for _ in P]
        for l in range(L, 0, -1):
            W = self.weights[l - 1]
            dprev = self.widths[l - 1]

            def bwd(i, l=l, W=W, dprev=dprev):
                q = P[i]
                p, z, mask = caches[i][l - 1]
                m = js[i] if l == L else js[i] * (z > 0.0)
                g = p.T @ m
                jf = None
                if l > 1:
                    if self.model == "sage":
                        jf = q.Mt @ (m @ W[dprev:].T)
                        jf[:q.nl] += m @ W[:dprev].T
                    else:
                        jf = q.At @ (m @ W.T)
                    if mask is not None:
                        jf = jf * mask
                return g, jf
            res = self._map(bwd, range(len(P)))
            for i in range(len(P)):
                grads[i][l - 1] = res[i][0]
            if l == 1:
                break
            jfs = [r[1] for r in res]
            js = [np.ascontiguousarray(jfs[i][:P[i].nl]) for i in range(len(P))]
            if sync_variant or mode == "sync":
                if not sync_variant and epoch > 1:
                    self._consume(epoch, l, BWD)
                recv = self.exchange(epoch, l, BWD, self._bwd_out(jfs))
                if not sync_variant:
                    self.slots[(l, BWD)] = (epoch, recv)
                self._integrate(js, recv)
            else:
                if epoch > 1:
                    tag, stale = self._consume(epoch, l, BWD)
                    self._integrate(js, stale)
                fresh = self.exchange(epoch, l, BWD, self._bwd_out(jfs))
                self.slots[(l, BWD)] = (epoch, fresh)
        # all-reduce in partition order (transport.py:139-147)
        total = []
        for l in range(L):
            acc = grads[0][l].copy()
            for i in range(1, len(P)):
                acc += grads[i][l]
            total.append(acc)
        if len(P) > 1:
            for s in self.stats:
                s["allreduce"] += sum(g.size for g in total) * 4
        tl = losses[0]
        for x in losses[1:]:
            tl += x
        if not np.isfinite(tl):
            raise OracleProtocolError(f"NaN/inf loss at epoch {epoch}")
        self.loss = float(tl)
        self.last_grads = total          # (test hook) the all-reduced gradients this epoch
        self.weights = [a.step(w, g) for w, g, a in zip(self.weights, total, self.adam)]
        return mode

    def _integrate(self, js, recv):
        for i, q in enumerate(self.P):
            for k, mat in recv[i].items():
                js[i][q.S[k]] += mat

    def totals(self) -> dict:
        out = dict(main=0, meta=0, header=0, messages=0, allreduce=0)
        for s in self.stats:
            for k in out:
                out[k] += s[k]
        return out


def full_forward(features, a_hat, weights, model="gcn", mean_hat=None):
    """trainer.py:115-126 (centralized, full precision, no dropout)."""
    h = np.asarray(features, dtype=np.float64)
    A = _csr(a_hat)
    M = _csr(mean_hat)
    for l, w in enumerate(weights, start=1):
        p = np.hstack([h, M @ h]) if model == "sage" else A @ h
        z = p @ w
        h = np.maximum(z, 0.0) if l < len(weights) else z
    return h


def accuracies(logits, labels, masks) -> dict:
    """trainer.py:129-144."""
    pred = logits.argmax(axis=1)
    out = {}
    for name, m in zip(("train_acc", "val_acc", "test_acc"), masks):
        m = np.asarray(m, dtype=bool)
        out[name] = float((pred[m] == np.asarray(labels)[m]).mean()) if m.any() else 0.0
    return out
