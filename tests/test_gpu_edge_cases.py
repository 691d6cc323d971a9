"""Degenerate inputs through the public API on the GPU, against the oracle:
a graph without edges, a single vertex, partitions left empty, a lone
train vertex, and one class."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from conftest import rel_l2  # noqa: E402
from oracle import gcn, plan as oplan  # noqa: E402
import paper_2605_11517_b200 as g2  # noqa: E402


def _check(g, labels, P, F=6, C=3, L=2, H=4, mode="mean_self_loop", mask=None, epochs=2):
    ds = g2.make_random_dataset(g, feature_dim=F, num_classes=C, seed=1)
    if mask is not None:
        ds.train_mask = mask
    plan = g2.build_partition_plan(g, labels, P)
    model = g2.create_model(F, C, num_layers=L, hidden_dim=H, seed=2, aggregation_mode=mode)
    trained, trace, _ = g2.partitioned_train(ds, plan, model, epochs=epochs, lr=0.1)
    topos = oplan.build_plan(g.src_ptr, g.dst_idx, labels, P)
    W, _, ref = gcn.train_partitioned(ds.features, ds.labels, ds.train_mask, topos, model.weights,
                                      epochs, 0.1, mode=mode)
    for (_, l1, _), (_, l2, _) in zip(trace, ref):
        assert abs(l1 - l2) <= 1e-4 * max(abs(l2), 1e-12)
    for a, b in zip(trained.weights, W):
        assert rel_l2(a, b) < 1e-4
    return trained, trace


@pytest.mark.parametrize("mode", ["mean_self_loop", "symmetric_norm"])
def test_graph_without_edges(mode):
    g = g2.build_csr(np.zeros((0, 2), dtype=np.int64), 50)
    labels = (np.arange(50) % 3).astype(np.int32)
    _check(g, labels, 3, mode=mode)


def test_single_vertex():
    g = g2.build_csr(np.zeros((0, 2), dtype=np.int64), 1)
    _check(g, np.zeros(1, dtype=np.int32), 1, mask=np.ones(1, dtype=bool))


def test_empty_partitions_and_one_class():
    g = g2.generate_kronecker(8, 6, seed=3)
    labels = np.zeros(g.num_vertices, dtype=np.int32)
    labels[::5] = 3                       # partitions 1 and 2 empty
    _check(g, labels, 4, C=1)


def test_one_train_vertex():
    g = g2.generate_kronecker(8, 6, seed=4)
    mask = np.zeros(g.num_vertices, dtype=bool)
    mask[17] = True
    labels = g2.random_partition(g.num_vertices, 3, 0)
    _check(g, labels, 3, mask=mask)


@pytest.mark.parametrize("mode", ["sage_mean", "gat"])
def test_sage_gat_without_edges(mode):
    from oracle import sage_gat
    g = g2.build_csr(np.zeros((0, 2), dtype=np.int64), 40)
    ds = g2.make_random_dataset(g, feature_dim=8, num_classes=3, seed=1)
    plan = g2.build_partition_plan(g, (np.arange(40) % 2).astype(np.int32), 2)
    model = g2.create_model(8, 3, num_layers=2, hidden_dim=8, seed=2, aggregation_mode=mode, heads=2)
    trained, trace, _ = g2.partitioned_train(ds, plan, model, epochs=2, lr=0.1)
    if mode == "gat":
        W, _, ref = sage_gat.train_gat(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                       model.weights, 2, 2, 0.1)
    else:
        W, _, ref = sage_gat.train_sage(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                        model.weights, 2, 0.1)
    for (_, l1, _), (_, l2, _) in zip(trace, ref):
        assert abs(l1 - l2) <= 1e-4 * abs(l2)
    for a, b in zip(trained.weights, W):
        assert rel_l2(a, b) < 1e-4


def test_streaming_without_edges(monkeypatch):
    monkeypatch.setenv("GRD_ENGINE", "stream")
    g = g2.build_csr(np.zeros((0, 2), dtype=np.int64), 64)
    _check(g, (np.arange(64) % 4).astype(np.int32), 4, F=8, C=3, H=4)


def test_per_partition_operators_on_empty_partition():
    """layer_forward / regather_backward / scatter_accumulate of a partition
    with no targets return empty results of the right shapes (the
    reference's empty-partition plans, test_training.py:91-96)."""
    g = g2.generate_kronecker(7, 6, seed=3)
    labels = np.zeros(g.num_vertices, dtype=np.int32)
    labels[::2] = 2                            # partition 1 empty
    plan = g2.build_partition_plan(g, labels, 3)
    topo = plan.topologies[1]
    assert topo.targets.size == 0 and topo.gather_map.size == 0
    model = g2.create_model(5, 3, num_layers=2, hidden_dim=4, seed=1)
    out = g2.layer_forward(0, np.zeros((0, 5)), topo, model)
    assert out.shape == (0, 4)
    acts = np.random.default_rng(0).normal(size=(g.num_vertices, 5))
    ga, gw = g2.regather_backward(0, 1, np.zeros((0, 4)), np.zeros((0, 4)), acts, plan, model)
    assert ga.shape == (0, 5) and gw.shape == (5, 4) and not gw.any()
    glob = np.ones((g.num_vertices, 5))
    res = g2.scatter_accumulate(ga, topo.gather_map, glob)
    assert res is glob and np.array_equal(glob, np.ones((g.num_vertices, 5)))


@pytest.mark.parametrize("keep", ["0", "1"])
@pytest.mark.parametrize("mode", ["mean_self_loop", "symmetric_norm"])
@pytest.mark.parametrize("F,C,L,H", [(6, 3, 3, 12), (12, 20, 2, 8), (5, 9, 3, 7)])
def test_aggregate_first_kept_vs_regathered(keep, mode, F, C, L, H, monkeypatch):
    """Aggregate-first GCN layers (hidden: N kept from the forward; last: N
    still in place) and the regather (GRD_KEEP_AGG=0) both match the oracle
    over two epochs."""
    monkeypatch.setenv("GRD_KEEP_AGG", keep)
    g = g2.generate_kronecker(9, 6, seed=4)
    labels = g2.random_partition(g.num_vertices, 3, 2)
    _check(g, labels, 3, F=F, C=C, L=L, H=H, mode=mode)
