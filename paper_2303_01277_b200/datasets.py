"""Synthetic graphs (host side, run once).

* ``SbmSpec`` / ``generate_sbm`` — the reference's dense O(n^2) SBM
  (``datasets.py:116-171``), reproduced draw-for-draw (same keyed Philox
  generators) so BASELINE config 1 is the identical graph on both sides.
* ``PlantedSpec`` / ``generate_planted`` — the scalable planted-partition
  generator SURVEY §8(f) rank 1 asks for: O(E) memory/time, emits the same
  ``Graph`` type, so the Reddit / ogbn-products / Yelp shapes (configs 2-4)
  become buildable.  Communities are contiguous id ranges (as in the
  reference SBM, ``datasets.py:142``); each undirected edge joins a uniform
  node to a uniform node of its own community with probability ``1 - cut``,
  else to a uniform node of the whole graph.  Labels = community mod
  classes; features = tiled one-hot(label) + Gaussian noise (as
  ``datasets.py:154-158``), generated as float32.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._np import setdiff_sorted, sorted_unique
from .graph import Graph
from .rngstream import keyed_generator


class DatasetError(ValueError):
    pass


@dataclass(frozen=True)
class SbmSpec:
    nodes_per_community: int = 125
    communities: int = 4
    p_in: float = 0.15
    p_out: float = 0.01
    feature_dim: int = 32
    feature_noise: float = 1.0
    seed: int = 0

    def __post_init__(self):
        if not (0.0 <= self.p_out < self.p_in <= 1.0):
            raise DatasetError("require 0 <= p_out < p_in <= 1")
        if self.feature_dim < self.communities:
            raise DatasetError("feature_dim must be >= number of communities")


def _split_masks(n, perm, fractions):
    n_train = int(round(fractions[0] * n))
    n_val = int(round(fractions[1] * n))
    masks = [np.zeros(n, dtype=bool) for _ in range(3)]
    masks[0][perm[:n_train]] = True
    masks[1][perm[n_train:n_train + n_val]] = True
    masks[2][perm[n_train + n_val:]] = True
    return masks


def generate_sbm(spec: SbmSpec) -> Graph:
    """Draw-for-draw reproduction of the reference SBM (``datasets.py:136-171``)."""
    n = spec.nodes_per_community * spec.communities
    labels = np.repeat(np.arange(spec.communities), spec.nodes_per_community)
    rng = keyed_generator(spec.seed, "sbm-edges")
    draw = rng.random((n, n))
    same = labels[:, None] == labels[None, :]
    upper = np.triu(draw < np.where(same, spec.p_in, spec.p_out), k=1)
    del draw
    src, dst = np.nonzero(upper)
    e = np.concatenate([np.stack([src, dst], 1), np.stack([dst, src], 1)])
    e = e[np.lexsort((e[:, 1], e[:, 0]))]
    reps = -(-spec.feature_dim // spec.communities)
    base = np.tile(np.eye(spec.communities)[labels], (1, reps))[:, :spec.feature_dim]
    feats = base + spec.feature_noise * keyed_generator(spec.seed, "sbm-features") \
        .standard_normal((n, spec.feature_dim))
    perm = keyed_generator(spec.seed, "sbm-masks").permutation(n)
    tr, va, te = _split_masks(n, perm, (0.6, 0.2))
    return Graph(num_nodes=n, edges=e, features=feats, labels=labels, train_mask=tr,
                 val_mask=va, test_mask=te, num_classes=spec.communities)


@dataclass(frozen=True)
class PlantedSpec:
    num_nodes: int
    num_edges: int                 # target directed edges (both directions stored)
    feature_dim: int
    num_classes: int
    communities: int = 0           # 0 -> num_classes
    cut: float = 0.03              # fraction of undirected edges with a uniform endpoint
    feature_noise: float = 1.0
    train_frac: float = 0.6
    val_frac: float = 0.2
    seed: int = 0
    multilabel: bool = False       # labels: (nodes x classes) 0/1 matrix (Yelp-shaped config)

    def __post_init__(self):
        if self.num_nodes < 2 or self.num_edges < 0 or not (0.0 <= self.cut <= 1.0):
            raise DatasetError("bad planted-partition spec")


def _tri_decode(t: np.ndarray):
    """Index t of the strict lower triangle (row-major) -> (a, b), a > b."""
    a = ((1.0 + np.sqrt(1.0 + 8.0 * t.astype(np.float64))) // 2).astype(np.int64)
    a -= (a * (a - 1) // 2 > t)           # guard float rounding at the boundaries
    a += ((a + 1) * a // 2 <= t)
    return a, t - a * (a - 1) // 2


def generate_planted(spec: PlantedSpec) -> Graph:
    """O(E) planted-partition graph.  Intra-community edges are sampled without
    replacement from each community's pair set (so there are no duplicates to
    discard); cut edges join uniform node pairs; the union is deduplicated once."""
    n = spec.num_nodes
    C = spec.communities or spec.num_classes
    bounds = np.linspace(0, n, C + 1).astype(np.int64)
    sizes = np.diff(bounds)
    comm = np.repeat(np.arange(C), sizes)
    target_und = spec.num_edges // 2
    n_cut = int(round(target_und * spec.cut))
    n_intra = target_und - n_cut
    pairs = sizes * (sizes - 1) // 2
    if n_intra > pairs.sum():
        raise DatasetError("communities too small for the requested intra-community degree")
    share = n_intra * pairs / max(1, pairs.sum())
    k = np.floor(share).astype(np.int64)
    k[np.argsort(-(share - k))[: n_intra - k.sum()]] += 1
    rng = keyed_generator(spec.seed, "planted-edges")
    keys = []
    for c in range(C):
        if k[c] == 0:
            continue
        t = rng.choice(pairs[c], size=k[c], replace=False)
        a, b = _tri_decode(t)
        keys.append((bounds[c] + b) * n + (bounds[c] + a))      # (min, max) pair key
    intra = np.concatenate(keys) if keys else np.empty(0, dtype=np.int64)
    und = np.sort(intra)              # distinct by construction (disjoint communities)
    cut_keys = np.empty(0, dtype=np.int64)
    while len(cut_keys) < n_cut:
        need = n_cut - len(cut_keys)
        u = rng.integers(0, n, size=int(need * 1.05) + 16, dtype=np.int64)
        v = rng.integers(0, n, size=len(u), dtype=np.int64)
        ok = u != v
        ck = sorted_unique(np.minimum(u[ok], v[ok]) * n + np.maximum(u[ok], v[ok]))
        ck = setdiff_sorted(setdiff_sorted(ck, und), cut_keys)
        if len(ck) > need:
            ck = np.sort(rng.choice(ck, size=need, replace=False))
        cut_keys = np.sort(np.concatenate([cut_keys, ck]))
    und = np.sort(np.concatenate([und, cut_keys]))
    lo, hi = und // n, und % n
    both = np.concatenate([lo * n + hi, hi * n + lo])
    both.sort()
    edges = np.empty((len(both), 2), dtype=np.int64)
    np.floor_divide(both, n, out=edges[:, 0])
    np.remainder(both, n, out=edges[:, 1])
    del both
    labels = comm % spec.num_classes
    d = spec.feature_dim
    frng = keyed_generator(spec.seed, "planted-features")
    feats = frng.standard_normal((n, d), dtype=np.float32)
    feats *= np.float32(spec.feature_noise)
    cls_of_col = np.arange(d) % spec.num_classes
    # tiled one-hot: column j carries the signal of class j % num_classes
    for start in range(0, n, 1 << 15):
        blk = slice(start, min(n, start + (1 << 15)))
        feats[blk] += labels[blk, None] == cls_of_col[None, :]
    perm = keyed_generator(spec.seed, "planted-masks").permutation(n)
    tr, va, te = _split_masks(n, perm, (spec.train_frac, spec.val_frac))
    out_labels = _multilabels(spec, comm, labels) if spec.multilabel else labels.astype(np.int64)
    return Graph(num_nodes=n, edges=edges, features=feats, labels=out_labels,
                 train_mask=tr, val_mask=va, test_mask=te, num_classes=spec.num_classes)


def _multilabels(spec: PlantedSpec, comm: np.ndarray, primary: np.ndarray) -> np.ndarray:
    """(nodes x classes) 0/1 labels: each community owns a label set (its
    primary class — the one the features carry — plus ~5 % of the others);
    every node takes its community's set with 1 % of the entries flipped."""
    K = spec.num_classes
    rng = keyed_generator(spec.seed, "planted-multilabels")
    ncomm = int(comm.max()) + 1 if len(comm) else 0
    sets = rng.random((ncomm, K)) < 0.05
    sets[np.arange(ncomm), np.arange(ncomm) % K] = True
    out = np.empty((len(comm), K), dtype=np.uint8)
    for start in range(0, len(comm), 1 << 16):
        blk = slice(start, min(len(comm), start + (1 << 16)))
        flip = rng.random((blk.stop - blk.start, K)) < 0.01
        out[blk] = sets[comm[blk]] ^ flip
    out[np.arange(len(comm)), primary] = 1
    return out


# BASELINE.json configs (shapes from PAPER.md Table "dataset info" and the
# model table; see DESIGN.md for the exact numbers used).
CONFIG1 = SbmSpec(nodes_per_community=2500, communities=4, p_in=0.006, p_out=0.0006,
                  feature_dim=64, feature_noise=1.0, seed=1)
REDDIT = PlantedSpec(num_nodes=232_965, num_edges=114_615_892, feature_dim=602,
                     num_classes=41, cut=0.005, train_frac=0.66, val_frac=0.10, seed=2303)
OGBN_PRODUCTS = PlantedSpec(num_nodes=2_449_029, num_edges=61_859_140, feature_dim=100,
                            num_classes=47, cut=0.03, train_frac=0.08, val_frac=0.02, seed=2303)
YELP = PlantedSpec(num_nodes=716_847, num_edges=13_954_820, feature_dim=300,
                   num_classes=100, cut=0.05, train_frac=0.75, val_frac=0.10, seed=2303, multilabel=True)


def scaled(spec: PlantedSpec, factor: float) -> PlantedSpec:
    """Same shape (degree, widths, classes, cut) at ``factor`` x the nodes."""
    from dataclasses import replace
    return replace(spec, num_nodes=max(64, int(spec.num_nodes * factor)),
                   num_edges=int(spec.num_edges * factor))
