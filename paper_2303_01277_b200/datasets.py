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

    def __post_init__(self):
        if self.num_nodes < 2 or self.num_edges < 0 or not (0.0 <= self.cut <= 1.0):
            raise DatasetError("bad planted-partition spec")


def generate_planted(spec: PlantedSpec) -> Graph:
    n = spec.num_nodes
    C = spec.communities or spec.num_classes
    bounds = np.linspace(0, n, C + 1).astype(np.int64)
    comm = np.repeat(np.arange(C), np.diff(bounds))
    target_und = spec.num_edges // 2
    rng = keyed_generator(spec.seed, "planted-edges")
    keys = np.empty(0, dtype=np.int64)
    over = 1.03
    while len(keys) < target_und:
        need = int((target_und - len(keys)) * over) + 1024
        src = rng.integers(0, n, size=need, dtype=np.int64)
        intra = rng.random(need) >= spec.cut
        c = comm[src]
        lo, sz = bounds[c], bounds[c + 1] - bounds[c]
        dst = np.where(intra, lo + (rng.random(need) * sz).astype(np.int64),
                       rng.integers(0, n, size=need, dtype=np.int64))
        ok = src != dst
        a, b = np.minimum(src[ok], dst[ok]), np.maximum(src[ok], dst[ok])
        keys = np.unique(np.concatenate([keys, a * n + b]))
        over *= 1.5
    if len(keys) > target_und:
        keys = np.sort(rng.choice(keys, size=target_und, replace=False))
    a, b = keys // n, keys % n
    both = np.concatenate([a * n + b, b * n + a])
    both.sort()
    edges = np.stack([both // n, both % n], axis=1)
    labels = comm % spec.num_classes
    d = spec.feature_dim
    frng = keyed_generator(spec.seed, "planted-features")
    feats = frng.standard_normal((n, d), dtype=np.float32)
    feats *= np.float32(spec.feature_noise)
    cols = np.arange(d)
    # tiled one-hot: column j carries the signal of class j % num_classes
    for start in range(0, n, 1 << 16):
        blk = slice(start, min(n, start + (1 << 16)))
        feats[blk] += (labels[blk, None] == (cols[None, :] % spec.num_classes)).astype(np.float32)
    perm = keyed_generator(spec.seed, "planted-masks").permutation(n)
    tr, va, te = _split_masks(n, perm, (spec.train_frac, spec.val_frac))
    return Graph(num_nodes=n, edges=edges, features=feats, labels=labels.astype(np.int64),
                 train_mask=tr, val_mask=va, test_mask=te, num_classes=spec.num_classes)


# BASELINE.json configs (shapes from PAPER.md Table "dataset info" and the
# model table; see DESIGN.md for the exact numbers used).
CONFIG1 = SbmSpec(nodes_per_community=2500, communities=4, p_in=0.006, p_out=0.0006,
                  feature_dim=64, feature_noise=1.0, seed=1)
REDDIT = PlantedSpec(num_nodes=232_965, num_edges=114_615_892, feature_dim=602,
                     num_classes=41, cut=0.005, train_frac=0.66, val_frac=0.10, seed=2303)
OGBN_PRODUCTS = PlantedSpec(num_nodes=2_449_029, num_edges=61_859_140, feature_dim=100,
                            num_classes=47, cut=0.03, train_frac=0.08, val_frac=0.02, seed=2303)
YELP = PlantedSpec(num_nodes=716_847, num_edges=13_954_820, feature_dim=300,
                   num_classes=100, cut=0.05, train_frac=0.75, val_frac=0.10, seed=2303)


def scaled(spec: PlantedSpec, factor: float) -> PlantedSpec:
    """Same shape (degree, widths, classes, cut) at ``factor`` x the nodes."""
    from dataclasses import replace
    return replace(spec, num_nodes=max(64, int(spec.num_nodes * factor)),
                   num_edges=int(spec.num_edges * factor))
