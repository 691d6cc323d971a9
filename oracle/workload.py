"""Synthetic workload built from the oracle alone — TEST INFRASTRUCTURE.

``bench.py``'s reference arm and CPU baseline build their bounded sample
with this module so that nothing of the product package (and none of its
native code) runs on the CPU leg: graph (oracle/graph.py), dataset
(dataset.py:75-98: f32 U[0,1) - 0.5 widened to f64, labels uniform, first
round(0.5 n) of one PCG64 permutation as the train mask), switching-aware
labels (oracle/partition.py), plan (oracle/plan.py) and Glorot weights
(model.py:67-89; the GraphSAGE / GAT layouts are the builder-defined ones in
paper_2605_11517_b200/model.py).

Seeds follow the reference CLI (cli.py:179,203,215,304): graph S, dataset
S+1, partitioner S+2, model S+3.
"""

from __future__ import annotations

import time
from types import SimpleNamespace

import numpy as np

from . import graph as _graph
from . import partition as _partition
from . import plan as _plan


def dataset(n, feature_dim, num_classes, seed, train_fraction=0.5):
    gen = np.random.Generator(np.random.PCG64(seed))
    x = gen.random((n, feature_dim), dtype=np.float32).astype(np.float64) - 0.5
    y = gen.integers(0, num_classes, size=n, dtype=np.int64)
    order = gen.permutation(n)
    mask = np.zeros(n, dtype=bool)
    mask[order[: max(1, int(round(train_fraction * n)))]] = True
    return x, y, mask


def weights(F, C, L, H, seed, mode="mean_self_loop", heads=4):
    widths = [F] + [H] * (L - 1) + [C]
    gen = np.random.Generator(np.random.PCG64(seed))
    out = []
    for l, (fi, fo) in enumerate(zip(widths[:-1], widths[1:])):
        if mode == "gat":
            dh = fo if l == L - 1 else fo // heads
            b = np.sqrt(6.0 / (fi + heads * dh))
            w = gen.uniform(-b, b, size=(fi, heads * dh))
            ab = np.sqrt(6.0 / (dh + 1))
            out.append(np.concatenate([w, gen.uniform(-ab, ab, size=(2, heads * dh))], axis=0))
            continue
        b = np.sqrt(6.0 / (fi + fo))
        if mode == "sage_mean":
            root = gen.uniform(-b, b, size=(fi, fo))
            out.append(np.concatenate([root, gen.uniform(-b, b, size=(fi, fo))], axis=1))
        else:
            out.append(gen.uniform(-b, b, size=(fi, fo)))
    return out


def build(scale, deg, F, C, L, H, P, mode="mean_self_loop", heads=4, seed=0):
    """Everything one epoch of the workload needs, from the oracle only."""
    t0 = time.perf_counter()
    ptr, idx = _graph.kronecker(scale, deg, seed)
    x, y, mask = dataset(len(ptr) - 1, F, C, seed + 1)
    topos = None
    if mode not in ("sage_mean", "gat"):
        part = _partition.partition(ptr, idx, P, seed=seed + 2)
        topos = _plan.build_plan(ptr, idx, part["labels"], P)
    w = weights(F, C, L, H, seed + 3, mode, heads)
    return SimpleNamespace(src_ptr=ptr, dst_idx=idx, num_vertices=len(ptr) - 1,
                           num_edges=int(idx.size), features=x, labels=y, train_mask=mask,
                           topologies=topos, weights=w, mode=mode, heads=heads, layers=L,
                           build_s=time.perf_counter() - t0)


def epoch_seconds(s, lr=0.01, epochs=1):
    """Wall time of one training epoch of the sample in the oracle."""
    t0 = time.perf_counter()
    if s.mode == "sage_mean":
        from . import sage_gat
        sage_gat.train_sage(s.features, s.labels, s.train_mask, s.src_ptr, s.dst_idx, s.weights,
                            epochs, lr)
    elif s.mode == "gat":
        from . import sage_gat
        sage_gat.train_gat(s.features, s.labels, s.train_mask, s.src_ptr, s.dst_idx, s.weights,
                           s.heads, epochs, lr)
    else:
        from . import gcn
        gcn.train_partitioned(s.features, s.labels, s.train_mask, s.topologies, s.weights,
                              epochs, lr, mode=s.mode)
    return (time.perf_counter() - t0) / epochs
