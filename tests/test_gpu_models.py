"""GPU parity of the builder-defined GraphSAGE-mean / GAT layers against the
float64 oracle (oracle/sage_gat.py).  Tolerance as the north star: 1e-4
L2-relative on weights and gradients, 1e-4 relative on the loss."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from conftest import rel_l2  # noqa: E402
from oracle import sage_gat  # noqa: E402
import paper_2605_11517_b200 as g2  # noqa: E402

TOL = 1e-4


def _setup(scale, deg, F, C, L, H, P, mode):
    g = g2.generate_kronecker(scale, deg, seed=scale)
    ds = g2.make_random_dataset(g, feature_dim=F, num_classes=C, seed=scale + 1)
    part = g2.switching_aware_partition(g, P, g2.PartitionerParams(seed=scale + 2))
    plan = g2.build_partition_plan(g, part.labels, P)
    model = g2.create_model(F, C, num_layers=L, hidden_dim=H, seed=scale + 3, aggregation_mode=mode)
    return g, ds, plan, model


@pytest.mark.parametrize("F,H,C,L", [(6, 12, 3, 3), (16, 8, 5, 2), (10, 10, 4, 3), (3, 37, 7, 2)])
def test_sage_matches_oracle(F, H, C, L):
    g, ds, plan, model = _setup(9, 8, F, C, L, H, 4, "sage_mean")
    trained, trace, _ = g2.partitioned_train(ds, plan, model, epochs=3, lr=0.05)
    W, grads, ref = sage_gat.train_sage(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                        model.weights, 3, 0.05)
    for (_, l, a), (_, rl, ra) in zip(trace, ref):
        assert abs(l - rl) <= TOL * abs(rl)
        assert abs(a - ra) <= 2.0 / ds.train_mask.sum()
    for a, b in zip(trained.weights, W):
        assert a.shape == b.shape and rel_l2(a, b) < TOL
    # gradients of the first epoch: later epochs' gradients may cross a ReLU
    # kink when the weights differ in the 7th digit (a discontinuity, not
    # rounding), so they are compared where the weights are identical
    one, _, _ = g2.partitioned_train(ds, plan, model, epochs=1, lr=0.05)
    _, grads1, _ = sage_gat.train_sage(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                       model.weights, 1, 0.05)
    for a, b in zip(one.weight_grads, grads1):
        assert rel_l2(a, b) < TOL


def test_sage_power_law_graph_with_hubs():
    # scale-12 RMAT: hub rows exceed the heavy-row threshold in both directions
    g, ds, plan, model = _setup(12, 16, 20, 6, 2, 24, 8, "sage_mean")
    assert g.out_degrees().max() > 256
    trained, trace, _ = g2.partitioned_train(ds, plan, model, epochs=2, lr=0.05)
    W, grads, ref = sage_gat.train_sage(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                        model.weights, 2, 0.05)
    assert abs(trace[-1][1] - ref[-1][1]) <= TOL * abs(ref[-1][1])
    for a, b in zip(trained.weights, W):
        assert rel_l2(a, b) < TOL


@pytest.mark.parametrize("F,H,C,L,heads,scale", [(6, 16, 3, 3, 4, 10), (12, 8, 5, 2, 2, 10),
                                                  (8, 32, 7, 2, 4, 12), (5, 12, 4, 3, 3, 9)])
def test_gat_per_partition_engine(F, H, C, L, heads, scale):
    """GAT through the literal per-(layer, partition) schedule: GA_p
    gathered, P_ext / attention / aggregate over the partition's in-edges in
    gather-row space, regather backward, ascending-pid scatter.  Equal to
    the layer-wise engine within 1e-5, to the float64 oracle within 1e-4;
    per-partition weight-gradient probes sum to the epoch's gradient
    (scale 12: hub rows past the heavy-row threshold inside partitions)."""
    g, ds, plan, model = _setup(scale, 8, F, C, L, H, 5, "gat")
    model = g2.create_model(F, C, num_layers=L, hidden_dim=H, seed=scale + 3,
                            aggregation_mode="gat", heads=heads)
    seen = {}
    pp, trace, _ = g2.partitioned_train(
        ds, plan, model, 1, 0.05, partition_order=lambda l, ph: range(5),
        grad_probe=lambda e, l, p, ga, gw: seen.__setitem__((l, p), gw))
    lw, ltrace, _ = g2.partitioned_train(ds, plan, model, 1, 0.05)
    assert abs(trace[0][1] - ltrace[0][1]) <= 1e-6 * abs(ltrace[0][1])
    for a, b in zip(pp.weight_grads, lw.weight_grads):
        assert a.shape == b.shape and rel_l2(a, b) < 1e-5
    for a, b in zip(pp.weights, lw.weights):
        assert rel_l2(a, b) < 1e-6
    for l in range(L):
        total = sum(seen[(l, p)] for p in range(5))
        assert total.shape == pp.weight_grads[l].shape
        assert rel_l2(total, pp.weight_grads[l]) < 1e-6
    _, grads, ref = sage_gat.train_gat(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                       model.weights, heads, 1, 0.05)
    assert abs(trace[0][1] - ref[0][1]) <= TOL * abs(ref[0][1])
    for a, b in zip(pp.weight_grads, grads):
        assert rel_l2(a, b) < TOL


def test_gat_per_partition_order_invariant():
    """Partition order only changes which partition runs first: forward
    outputs are disjoint target rows, gradients are summed in ascending
    partition id, so the weights are bitwise equal."""
    g, ds, plan, _ = _setup(10, 8, 6, 3, 3, 16, 5, "gat")
    model = g2.create_model(6, 3, num_layers=3, hidden_dim=16, seed=7, aggregation_mode="gat", heads=4)
    a, ta, _ = g2.partitioned_train(ds, plan, model, 2, 0.05, partition_order=lambda l, ph: range(5))
    b, tb, _ = g2.partitioned_train(ds, plan, model, 2, 0.05,
                                    partition_order=lambda l, ph: [3, 0, 4, 2, 1])
    assert ta == tb
    assert all(np.array_equal(x, y) for x, y in zip(a.weights, b.weights))


def test_gat_offloaded_tiers(tmp_path):
    """GAT through the executing SSO manager (layers, gradients and topology
    in the storage tier): ledger equal to the byte model's, weights to the
    HBM-resident engine's."""
    from paper_2605_11517_b200.hierarchy import HierarchyConfig, TierSession, simulate_epoch
    g, ds, plan, _ = _setup(9, 8, 6, 3, 3, 12, 4, "gat")
    model = g2.create_model(6, 3, num_layers=3, hidden_dim=16, seed=5, aggregation_mode="gat", heads=4)
    cfg = HierarchyConfig(host_capacity=20_000, bytes_per_value=4)
    sess = TierSession(plan, model.dims, "GRINNDER", cfg, aggregation_mode="gat",
                       directory=str(tmp_path))
    trained, trace, ledger = g2.partitioned_train(ds, plan, model, 2, 0.05, hierarchy=sess)
    sim = simulate_epoch(plan, model.dims, "GRINNDER", cfg, epochs=2, aggregation_mode="gat")
    assert ledger.events == sim.events
    resident, rtrace, _ = g2.partitioned_train(ds, plan, model, 2, 0.05)
    for (_, a, _), (_, b, _) in zip(trace, rtrace):
        assert abs(a - b) <= 1e-5 * abs(b)
    for a, b in zip(trained.weights, resident.weights):
        assert rel_l2(a, b) < 1e-5
    sess.close()


@pytest.mark.parametrize("F,H,C,L", [(6, 12, 3, 3), (16, 8, 5, 2), (3, 37, 7, 2)])
def test_sage_per_partition_engine(F, H, C, L):
    """GraphSAGE through the literal per-(layer, partition) schedule (K1
    gather of GA_p, mean over the partition's in-edges, regather backward,
    ascending-pid scatter): equal to the layer-wise engine within 1e-5 and
    to the float64 oracle within 1e-4; the per-partition weight-gradient
    probes sum to the epoch's gradient."""
    g, ds, plan, model = _setup(10, 8, F, C, L, H, 5, "sage_mean")
    seen = {}
    pp, trace, _ = g2.partitioned_train(
        ds, plan, model, 1, 0.05, partition_order=lambda l, ph: range(5),
        grad_probe=lambda e, l, p, ga, gw: seen.__setitem__((l, p), gw))
    lw, ltrace, _ = g2.partitioned_train(ds, plan, model, 1, 0.05)
    assert abs(trace[0][1] - ltrace[0][1]) <= 1e-6 * abs(ltrace[0][1])
    for a, b in zip(pp.weight_grads, lw.weight_grads):
        assert a.shape == b.shape and rel_l2(a, b) < 1e-5
    for l in range(L):
        total = sum(seen[(l, p)] for p in range(5))
        assert total.shape == pp.weight_grads[l].shape
        assert rel_l2(total, pp.weight_grads[l]) < 1e-6
    W, grads, ref = sage_gat.train_sage(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                        model.weights, 1, 0.05)
    assert abs(trace[0][1] - ref[0][1]) <= TOL * abs(ref[0][1])
    for a, b in zip(pp.weight_grads, grads):
        assert rel_l2(a, b) < TOL


def test_sage_offloaded_tiers(tmp_path):
    """GraphSAGE through the executing SSO manager: the ledger equals the
    byte model's, the weights the HBM-resident engine's."""
    from paper_2605_11517_b200.hierarchy import HierarchyConfig, TierSession, simulate_epoch
    g, ds, plan, model = _setup(9, 8, 6, 3, 3, 12, 4, "sage_mean")
    cfg = HierarchyConfig(host_capacity=20_000, bytes_per_value=4)
    sess = TierSession(plan, model.dims, "GRINNDER", cfg, aggregation_mode="sage_mean",
                       directory=str(tmp_path))
    trained, trace, ledger = g2.partitioned_train(ds, plan, model, 2, 0.05, hierarchy=sess)
    sim = simulate_epoch(plan, model.dims, "GRINNDER", cfg, epochs=2, aggregation_mode="sage_mean")
    assert ledger.events == sim.events
    resident, rtrace, _ = g2.partitioned_train(ds, plan, model, 2, 0.05)
    for (_, a, _), (_, b, _) in zip(trace, rtrace):
        assert abs(a - b) <= 1e-5 * abs(b)
    for a, b in zip(trained.weights, resident.weights):
        assert rel_l2(a, b) < 1e-5
    sess.close()


def test_sage_cached_session_is_bitwise_identical():
    # regression: padding columns of the loss gradient must stay zero across
    # epochs of a reused session (GraphSAGE GEMMs run over padded widths)
    g, ds, plan, model = _setup(9, 8, 6, 3, 3, 12, 4, "sage_mean")
    a, ta, _ = g2.partitioned_train(ds, plan, model, epochs=1, lr=0.05)
    g2.partitioned_train(ds, plan, model, epochs=3, lr=0.05)
    b, tb, _ = g2.partitioned_train(ds, plan, model, epochs=1, lr=0.05)
    assert ta == tb
    assert all(np.array_equal(x, y) for x, y in zip(a.weight_grads, b.weight_grads))


@pytest.mark.parametrize("F,H,C,L,heads", [(6, 16, 3, 3, 4), (12, 8, 5, 2, 2), (8, 32, 7, 2, 4)])
def test_gat_matches_oracle(F, H, C, L, heads):
    g = g2.generate_kronecker(9, 8, seed=9)
    ds = g2.make_random_dataset(g, feature_dim=F, num_classes=C, seed=10)
    part = g2.switching_aware_partition(g, 4, g2.PartitionerParams(seed=11))
    plan = g2.build_partition_plan(g, part.labels, 4)
    model = g2.create_model(F, C, num_layers=L, hidden_dim=H, seed=12, aggregation_mode="gat",
                            heads=heads)
    one, tr1, _ = g2.partitioned_train(ds, plan, model, epochs=1, lr=0.05)
    W1, grads1, ref1 = sage_gat.train_gat(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                          model.weights, heads, 1, 0.05)
    assert abs(tr1[0][1] - ref1[0][1]) <= TOL * abs(ref1[0][1])
    for a, b in zip(one.weight_grads, grads1):
        assert a.shape == b.shape and rel_l2(a, b) < TOL
    trained, trace, _ = g2.partitioned_train(ds, plan, model, epochs=3, lr=0.05)
    W, _, ref = sage_gat.train_gat(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                   model.weights, heads, 3, 0.05)
    for (_, l, _), (_, rl, _) in zip(trace, ref):
        assert abs(l - rl) <= TOL * abs(rl)
    for a, b in zip(trained.weights, W):
        assert rel_l2(a, b) < TOL


def test_gat_hub_rows():
    g = g2.generate_kronecker(12, 16, seed=3)
    ds = g2.make_random_dataset(g, feature_dim=8, num_classes=4, seed=4)
    plan = g2.build_partition_plan(g, g2.random_partition(g.num_vertices, 4, 5), 4)
    model = g2.create_model(8, 4, num_layers=2, hidden_dim=16, seed=6, aggregation_mode="gat", heads=4)
    one, tr, _ = g2.partitioned_train(ds, plan, model, epochs=1, lr=0.05)
    _, grads, ref = sage_gat.train_gat(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                       model.weights, 4, 1, 0.05)
    assert abs(tr[0][1] - ref[0][1]) <= TOL * abs(ref[0][1])
    for a, b in zip(one.weight_grads, grads):
        assert rel_l2(a, b) < TOL


@pytest.mark.parametrize("keep", ["0", "1"])
def test_gat_kept_vs_regathered(keep, monkeypatch):
    """Hidden GAT layers' [P | s | t] and attention kept from the forward
    (default) or recomputed in the backward (GRD_GAT_KEEP=0, the regather):
    both match the float64 oracle."""
    monkeypatch.setenv("GRD_GAT_KEEP", keep)
    g = g2.generate_kronecker(11, 12, seed=8)
    ds = g2.make_random_dataset(g, feature_dim=12, num_classes=5, seed=9)
    plan = g2.build_partition_plan(g, g2.random_partition(g.num_vertices, 3, 5), 3)
    model = g2.create_model(12, 5, num_layers=3, hidden_dim=16, seed=10, aggregation_mode="gat", heads=4)
    one, tr, _ = g2.partitioned_train(ds, plan, model, epochs=1, lr=0.05)
    sess = g2.training.session_for(ds, plan, model) if hasattr(g2, "training") else None
    if sess is not None:
        assert bool(sess.engine.gat_kept) == (keep == "1")
    _, grads, ref = sage_gat.train_gat(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                       model.weights, 4, 1, 0.05)
    assert abs(tr[0][1] - ref[0][1]) <= TOL * abs(ref[0][1])
    for a, b in zip(one.weight_grads, grads):
        assert rel_l2(a, b) < TOL


@pytest.mark.parametrize("mode,keep", [("sage_mean", "1"), ("sage_mean", "0"), ("gat", "1"),
                                       ("gat", "0")])
def test_baseline_widths_match_oracle(mode, keep, monkeypatch):
    """configs[1] / configs[2] at their real widths (F = 100, hidden 256 —
    GAT 4 heads x 64 concatenated, mean over heads on the last layer —
    C = 47, L = 3, P = 8 switching-aware partitions) on a scale-14
    average-degree-30 Kronecker graph (the products degree), kept forward
    state and regather backward: one epoch's loss, weight gradients and
    trained weights against the float64 oracle."""
    monkeypatch.setenv("GRD_KEEP_AGG", keep)
    monkeypatch.setenv("GRD_GAT_KEEP", keep)
    g, ds, plan, model = _setup(14, 30, 100, 47, 3, 256, 8, mode)
    trained, trace, _ = g2.partitioned_train(ds, plan, model, epochs=1, lr=0.01)
    if mode == "gat":
        W, grads, ref = sage_gat.train_gat(ds.features, ds.labels, ds.train_mask, g.src_ptr,
                                           g.dst_idx, model.weights, 4, 1, 0.01)
    else:
        W, grads, ref = sage_gat.train_sage(ds.features, ds.labels, ds.train_mask, g.src_ptr,
                                            g.dst_idx, model.weights, 1, 0.01)
    assert abs(trace[0][1] - ref[0][1]) <= TOL * abs(ref[0][1])
    for a, b in zip(trained.weight_grads, grads):
        assert a.shape == b.shape and rel_l2(a, b) < TOL
    for a, b in zip(trained.weights, W):
        assert rel_l2(a, b) < TOL
    plan.device_cache.clear()


@pytest.mark.parametrize("heads,H,C,scale", [(4, 32, 7, 12), (2, 16, 5, 11), (3, 12, 4, 10), (1, 8, 3, 9)])
def test_gat_fused_backward_matches_unfused(heads, H, C, scale, monkeypatch):
    """The fused pull backward (one gO_v gather per edge for dP, ds and the
    edge score gradients; GRD_GAT_FUSED_BWD=1, the default) against the
    separate edge-backward / pull / source-score kernels: same gradients
    up to fp32 summation order, both within 1e-4 of the float64 oracle
    (scale 12: hub rows split into heavy segments on both CSRs)."""
    g = g2.generate_kronecker(scale, 16, seed=3)
    ds = g2.make_random_dataset(g, feature_dim=8, num_classes=C, seed=4)
    plan = g2.build_partition_plan(g, g2.random_partition(g.num_vertices, 4, 5), 4)
    model = g2.create_model(8, C, num_layers=3, hidden_dim=H, seed=6, aggregation_mode="gat", heads=heads)
    out = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("GRD_GAT_FUSED_BWD", fused)
        plan.device_cache.clear()
        out[fused] = g2.partitioned_train(ds, plan, model, epochs=1, lr=0.05)
        sess = g2.training.session_for(ds, plan, model)
        assert sess.engine.gat_fused == (fused == "1")
    (a, ta, _), (b, tb, _) = out["1"], out["0"]
    assert abs(ta[0][1] - tb[0][1]) <= 1e-7 * abs(tb[0][1])
    for x, y in zip(a.weight_grads, b.weight_grads):
        assert rel_l2(x, y) < 2e-6
    _, grads, ref = sage_gat.train_gat(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                       model.weights, heads, 1, 0.05)
    for x, y in zip(a.weight_grads, grads):
        assert rel_l2(x, y) < TOL
    plan.device_cache.clear()
