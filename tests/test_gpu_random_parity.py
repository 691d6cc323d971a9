"""Seeded random sweep of small configurations through the public API on
the GPU, each against the float64 oracle (GCN: the reference restatement;
GraphSAGE / GAT: the builder oracle): graph size and degree, directed or
symmetric, feature / hidden / class widths (multiples of 4 or not), depth
1-4, partition count, aggregation mode."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from conftest import rel_l2  # noqa: E402
from oracle import gcn, plan as oplan, sage_gat  # noqa: E402
import paper_2605_11517_b200 as g2  # noqa: E402

MODES = ["mean_self_loop", "symmetric_norm", "sage_mean", "gat"]


def _case(seed):
    rng = np.random.default_rng(seed)
    mode = MODES[seed % 4]
    scale = int(rng.integers(6, 10))
    deg = int(rng.integers(1, 20))
    L = int(rng.integers(1, 5))
    F = int(rng.integers(1, 40))
    C = int(rng.integers(1, 12))
    heads = int(rng.integers(1, 4)) if mode == "gat" else 1
    H = 4 * heads * int(rng.integers(1, 5)) if mode == "gat" else int(rng.integers(1, 48))
    P = int(rng.integers(1, 9))
    directed = bool(rng.integers(0, 2))
    if mode == "gat":
        directed = bool((seed // 4) % 2)
    return mode, scale, deg, L, F, C, H, heads, P, directed


@pytest.mark.parametrize("seed", range(48))
def test_random_configuration_matches_oracle(seed):
    mode, scale, deg, L, F, C, H, heads, P, directed = _case(seed)
    g = g2.generate_kronecker(scale, deg, seed=seed)
    if directed:
        src = np.repeat(np.arange(g.num_vertices), np.diff(g.src_ptr))
        keep = np.random.default_rng(seed).random(g.num_edges) < 0.6
        g = g2.build_csr(np.stack([src[keep], g.dst_idx[keep]], 1), g.num_vertices)
    ds = g2.make_random_dataset(g, feature_dim=F, num_classes=C, seed=seed + 1)
    labels = g2.random_partition(g.num_vertices, P, seed)
    plan = g2.build_partition_plan(g, labels, P)
    model = g2.create_model(F, C, num_layers=L, hidden_dim=H, seed=seed + 2, aggregation_mode=mode,
                            heads=heads)
    epochs, lr = 2, 0.05
    trained, trace, _ = g2.partitioned_train(ds, plan, model, epochs=epochs, lr=lr)
    if mode == "gat":
        W, _, ref = sage_gat.train_gat(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                       model.weights, heads, epochs, lr)
    elif mode == "sage_mean":
        W, _, ref = sage_gat.train_sage(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                        model.weights, epochs, lr)
    else:
        topos = oplan.build_plan(g.src_ptr, g.dst_idx, labels, P)
        W, _, ref = gcn.train_partitioned(ds.features, ds.labels, ds.train_mask, topos, model.weights,
                                          epochs, lr, mode=mode)
    for (_, l1, _), (_, l2, _) in zip(trace, ref):
        assert abs(l1 - l2) <= 1e-4 * max(abs(l2), 1e-12), (l1, l2)
    for a, b in zip(trained.weights, W):
        assert rel_l2(a, b) < 1e-4


@pytest.mark.parametrize("seed", range(16))
def test_random_streaming_configuration_matches_oracle(seed):
    """The layer-streaming engine (small row chunks, partial HBM feature
    cache) on random transform-first configurations."""
    from paper_2605_11517_b200.stream import StreamSession
    rng = np.random.default_rng(1000 + seed)
    mode = ["mean_self_loop", "symmetric_norm", "sage_mean"][seed % 3]
    scale, deg = int(rng.integers(7, 10)), int(rng.integers(2, 20))
    L = int(rng.integers(2, 5))
    F = int(rng.integers(8, 48))
    H = int(rng.integers(1, F + 1))                    # hidden layers transform-first
    C = int(rng.integers(1, H + 1)) if mode == "sage_mean" else int(rng.integers(1, 40))
    g = g2.generate_kronecker(scale, deg, seed=seed)
    ds = g2.make_random_dataset(g, feature_dim=F, num_classes=C, seed=seed + 1)
    ds.features = ds.features.astype(np.float32)
    P = int(rng.integers(1, 6))
    labels = g2.random_partition(g.num_vertices, P, seed)
    plan = g2.build_partition_plan(g, labels, P)
    model = g2.create_model(F, C, num_layers=L, hidden_dim=H, seed=seed + 2, aggregation_mode=mode)
    rows = int(rng.integers(64, 400))
    ss = StreamSession(ds, plan, model, chunk_rows=rows, x_cache_bytes=int(rng.integers(0, 3)) * rows * 4 *
                       ((F + 3) // 4 * 4))
    trained, trace = ss.train(2, 0.05)
    if mode == "sage_mean":
        W, _, ref = sage_gat.train_sage(np.asarray(ds.features, np.float64), ds.labels, ds.train_mask,
                                        g.src_ptr, g.dst_idx, model.weights, 2, 0.05)
    else:
        topos = oplan.build_plan(g.src_ptr, g.dst_idx, labels, P)
        W, _, ref = gcn.train_partitioned(np.asarray(ds.features, np.float64), ds.labels, ds.train_mask,
                                          topos, model.weights, 2, 0.05, mode=mode)
    for (_, l1, _), (_, l2, _) in zip(trace, ref):
        assert abs(l1 - l2) <= 1e-4 * max(abs(l2), 1e-12), (l1, l2)
    for a, b in zip(trained.weights, W):
        assert rel_l2(a, b) < 1e-4
