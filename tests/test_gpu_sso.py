"""Structured storage offloading on real tensors: layers in the host tier,
partitions staged through pinned buffers.  Same results as the HBM-resident
engines, and the ledger of the real run equals the simulated / reference one
event for event (the reference's test_simulate.py:479-493 property)."""

from __future__ import annotations

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from conftest import GOLDEN, rel_l2  # noqa: E402
import paper_2605_11517_b200 as g2  # noqa: E402
from paper_2605_11517_b200.hierarchy import (HierarchyConfig, PolicySpec, TierSession,  # noqa: E402
                                             simulate_epoch)


def test_offloaded_training_matches_resident_and_reference_ledger():
    z = np.load(GOLDEN / "ledger_cases.npz")
    g = g2.generate_kronecker(7, 6, seed=3)
    plan = g2.build_partition_plan(g, z["labels"], 4)
    ds = g2.make_random_dataset(g, feature_dim=6, num_classes=3, seed=2)
    model = g2.create_model(6, 3, num_layers=3, hidden_dim=5, seed=4)
    for name in ("layer_lru", "partition_lru", "vertex", "no_bypass", "tight"):
        cfg = HierarchyConfig(**json.loads(str(z[f"{name}/config"])))
        session = TierSession(plan, model.dims, PolicySpec("GRINNDER",
                              bypass_enabled=name != "no_bypass"), cfg)
        trained, trace, ledger = g2.partitioned_train(ds, plan, model, epochs=2, lr=0.05,
                                                      hierarchy=session)
        assert [list(e) for e in ledger.events] == json.loads(str(z[f"{name}/events"]))
        resident, rtrace, _ = g2.partitioned_train(ds, plan, model, epochs=2, lr=0.05)
        for (_, a, _), (_, b, _) in zip(trace, rtrace):
            assert abs(a - b) <= 1e-5 * abs(b)
        for a, b in zip(trained.weights, resident.weights):
            assert rel_l2(a, b) < 1e-5


def test_offloaded_per_partition_probe_matches_resident():
    g = g2.generate_kronecker(9, 8, seed=5)
    labels = g2.switching_aware_partition(g, 6, g2.PartitionerParams(seed=1)).labels
    plan = g2.build_partition_plan(g, labels, 6)
    ds = g2.make_random_dataset(g, feature_dim=12, num_classes=4, seed=3)
    model = g2.create_model(12, 4, num_layers=2, hidden_dim=16, seed=2, aggregation_mode="symmetric_norm")
    session = TierSession(plan, model.dims, "GRINNDER", HierarchyConfig(host_capacity=10_000,
                                                                       bytes_per_value=4))
    seen_a, seen_b = {}, {}
    g2.partitioned_train(ds, plan, model, 1, 0.05, hierarchy=session,
                         grad_probe=lambda e, l, p, ga, gw: seen_a.__setitem__((l, p), (ga, gw)))
    sim = simulate_epoch(plan, model.dims, "GRINNDER", HierarchyConfig(host_capacity=10_000,
                                                                     bytes_per_value=4))
    assert session.ledger.events == sim.events
    g2.partitioned_train(ds, plan, model, 1, 0.05, partition_order=lambda l, ph: range(6),
                         grad_probe=lambda e, l, p, ga, gw: seen_b.__setitem__((l, p), (ga, gw)))
    for k in seen_b:
        assert np.array_equal(seen_a[k][0], seen_b[k][0])   # same kernels, same order
        assert np.array_equal(seen_a[k][1], seen_b[k][1])


def test_offloaded_with_empty_partition():
    """A partition with no targets (and so no gathered rows) in the host-tier
    path: same result as the resident engine, ledger equals the simulation."""
    g = g2.generate_kronecker(8, 6, seed=7)
    labels = (np.arange(g.num_vertices) % 3).astype(np.int32)
    labels[labels == 1] = 2                   # partition 1 empty
    plan = g2.build_partition_plan(g, labels, 3)
    ds = g2.make_random_dataset(g, feature_dim=8, num_classes=3, seed=2)
    model = g2.create_model(8, 3, num_layers=2, hidden_dim=8, seed=4)
    cfg = HierarchyConfig(host_capacity=10_000, bytes_per_value=4)
    session = TierSession(plan, model.dims, "GRINNDER", cfg)
    trained, trace, ledger = g2.partitioned_train(ds, plan, model, epochs=2, lr=0.05, hierarchy=session)
    sim = simulate_epoch(plan, model.dims, "GRINNDER", cfg)
    assert ledger.events[:len(sim.events)] == sim.events
    resident, rtrace, _ = g2.partitioned_train(ds, plan, model, epochs=2, lr=0.05)
    for (_, a, _), (_, b, _) in zip(trace, rtrace):
        assert abs(a - b) <= 1e-5 * abs(b)
    for a, b in zip(trained.weights, resident.weights):
        assert rel_l2(a, b) < 1e-5
