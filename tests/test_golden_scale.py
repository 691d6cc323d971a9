"""Integer artefacts at BASELINE scales, bit-exact with the reference itself.

Fixtures (tests/golden/make_golden.py, run against /root/reference):
  papers_s22.npz    configs[3]'s model on generate_kronecker(22, 12, 0):
                    4,194,304 V / 50,331,648 E, P = 16 switching-aware
                    partitions (seed 2), F = H = 128, C = 172, L = 3 — graph,
                    dataset, SA labels / objective trace, plan digests and
                    the reference's one-epoch loss / W / grad W
  products_s21.npz  configs[1]/[2]'s graph generate_kronecker(21, 30, 0):
                    2,097,152 V / 62,914,560 E, P = 8 SA partitions — graph,
                    SA labels / trace and plan digests

The host generator, partitioner and plan builder run here on CPU; the GPU
generator and GPU plan builder are checked against the same reference
digests in tests/test_gpu_golden_scale.py.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2605_11517_b200 import (PartitionerParams, build_partition_plan, generate_kronecker,
                                   make_random_dataset, switching_aware_partition)

pytestmark = pytest.mark.slow


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def load(name):
    path = GOLDEN / name
    if not path.exists():
        pytest.skip(f"{name} not generated (tests/golden/make_golden.py)")
    return dict(np.load(path))


def plan_digest(t) -> str:
    return digest(t.targets, t.gather_map, t.tgt_ptr, t.src_pos, t.edge_local_target, t.self_pos,
                  t.target_indeg, t.gather_indeg)


def check_integers(gold, g, P, ds=None):
    """Graph, switching-aware partitioner result and plan vs the reference."""
    assert g.num_vertices == int(gold["num_vertices"])
    assert g.num_edges == int(gold["num_edges"])
    assert digest(g.src_ptr, g.dst_idx) == str(gold["graph_digest"])
    if ds is not None:
        assert digest(ds.features) == str(gold["features_digest"])
        assert digest(ds.labels, ds.train_mask) == str(gold["labels_digest"])
    res = switching_aware_partition(g, P, PartitionerParams(seed=2))
    assert digest(res.labels) == str(gold["sa_labels_digest"])
    assert res.objective_trace == gold["sa_objective_trace"].tolist()
    assert res.initial_objective == float(gold["sa_initial_objective"])
    assert res.iterations == int(gold["sa_iterations"])
    assert res.converged == bool(gold["sa_converged"])
    assert res.max_size_per_iteration == gold["sa_max_sizes"].tolist()
    plan = build_partition_plan(g, res.labels, P)
    np.testing.assert_array_equal([t.gather_map.size for t in plan.topologies], gold["gather_rows"])
    for q, t in enumerate(plan.topologies):
        assert plan_digest(t) == str(gold[f"plan_digest_{q}"]), f"partition {q}"
    return res, plan


def test_papers_s22_host_integers_match_reference():
    gold = load("papers_s22.npz")
    scale, deg, F, C, L, H, P = [int(x) for x in gold["spec"]]
    g = generate_kronecker(scale, deg, seed=0)
    ds = make_random_dataset(g, feature_dim=F, num_classes=C, seed=1)
    check_integers(gold, g, P, ds)


def test_products_s21_host_integers_match_reference():
    gold = load("products_s21.npz")
    g = generate_kronecker(21, 30, seed=0)
    check_integers(gold, g, 8)
