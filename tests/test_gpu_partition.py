"""Switching-aware partitioner on the GPU (partition.switching_aware_partition
(..., device="cuda"): the sm_100a analysis kernel grd_sa_analyze, the
sequential host objective sum and device-sort relocation) against the
native host partitioner and the reference's own config-1 result: labels,
objective trace (f64 bits), initial objective, iteration count, convergence
flag and per-iteration maximum sizes all equal."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2605_11517_b200 as g2  # noqa: E402
from paper_2605_11517_b200.partition import PartitionerParams, switching_aware_partition  # noqa: E402


def _same(a, b):
    np.testing.assert_array_equal(a.labels, b.labels)
    assert a.objective_trace == b.objective_trace
    assert a.initial_objective == b.initial_objective
    assert a.iterations == b.iterations
    assert a.converged == b.converged
    assert a.max_size_per_iteration == b.max_size_per_iteration


@pytest.mark.parametrize("scale,deg,P,depth", [
    (7, 6, 3, 2), (8, 8, 4, 2), (8, 8, 4, 3), (9, 4, 6, 2), (12, 12, 16, 2), (13, 8, 33, 2),
    (11, 16, 2, 4), (12, 6, 40, 3), (11, 8, 300, 2),   # p > 256: int32 labels in the kernel
])
def test_gpu_partitioner_matches_host(scale, deg, P, depth):
    g = g2.generate_kronecker(scale, deg, seed=scale)
    params = PartitionerParams(seed=scale + 2, group_depth=depth)
    host = switching_aware_partition(g, P, params)
    dev = switching_aware_partition(g, P, params, device="cuda")
    assert host.iterations > 0
    _same(dev, host)


def test_gpu_partitioner_directed_isolated_and_hubs():
    """Directed graph (every third edge dropped), isolated vertices (no
    out-edges), and a hub row longer than a warp's stride many times over."""
    g = g2.generate_kronecker(11, 10, seed=5)
    src = np.repeat(np.arange(g.num_vertices), np.diff(g.src_ptr))
    keep = (np.arange(g.num_edges) % 3) != 1
    keep &= src % 7 != 0                        # vertices 0, 7, 14, ... lose every out-edge
    edges = np.stack([src[keep], g.dst_idx[keep]], 1)
    hub = np.stack([np.full(1500, 3), np.arange(10, 1510)], 1)
    gd = g2.build_csr(np.concatenate([edges, hub]), g.num_vertices)
    for P, alpha, beta in [(5, 1.1, 1.1), (8, 1.0, 1.5)]:
        params = PartitionerParams(seed=9, alpha_balance=alpha, beta=beta, epsilon=1e-4, patience=3)
        _same(switching_aware_partition(gd, P, params, device="cuda"),
              switching_aware_partition(gd, P, params))


def test_gpu_partitioner_max_iters_and_edgeless():
    g = g2.generate_kronecker(10, 8, seed=1)
    params = PartitionerParams(seed=4, max_iters=2)
    dev = switching_aware_partition(g, 4, params, device="cuda")
    assert dev.iterations <= 2
    _same(dev, switching_aware_partition(g, 4, params))
    empty = g2.build_csr(np.zeros((0, 2), dtype=np.int64), 50)
    _same(switching_aware_partition(empty, 3, PartitionerParams(seed=1), device="cuda"),
          switching_aware_partition(empty, 3, PartitionerParams(seed=1)))


def test_gpu_partitioner_config1_matches_reference(config1_golden):
    gold = config1_golden
    g = g2.generate_kronecker(17, 8, seed=0, device="cuda")
    res = switching_aware_partition(g, 8, PartitionerParams(seed=2), device="cuda")
    np.testing.assert_array_equal(res.labels, gold["sa_labels"].astype(np.int32))
    assert res.objective_trace == gold["sa_objective_trace"].tolist()
    assert res.initial_objective == float(gold["sa_initial_objective"])
    assert res.iterations == int(gold["sa_iterations"])
    assert res.converged == bool(gold["sa_converged"])
    assert res.max_size_per_iteration == gold["sa_max_sizes"].tolist()
