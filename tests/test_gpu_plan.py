"""GPU plan builder (build_partition_plan(..., device="cuda")): every
FlatPlan array bit-identical to the native host plan, which is pinned to
the reference's plan.py (tests/test_native_host.py, test_oracle_golden.py)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2605_11517_b200 as g2  # noqa: E402

FIELDS = ("part_ptr", "perm", "in_ptr", "in_src", "in_src_pos", "gather_ptr", "gather_map",
          "self_pos", "in_degree")


@pytest.mark.parametrize("scale,deg,P,directed", [(9, 8, 4, False), (12, 16, 8, False),
                                                  (11, 12, 6, True), (14, 10, 32, False)])
def test_gpu_plan_matches_host(scale, deg, P, directed):
    g = g2.generate_kronecker(scale, deg, seed=scale)
    if directed:
        src = np.repeat(np.arange(g.num_vertices), np.diff(g.src_ptr))
        keep = (np.arange(g.num_edges) % 3) != 1
        g = g2.build_csr(np.stack([src[keep], g.dst_idx[keep]], 1), g.num_vertices)
    labels = g2.switching_aware_partition(g, P, g2.PartitionerParams(seed=1)).labels
    labels[::97] = P - 1          # uneven partitions, one maybe empty-ish
    host = g2.build_partition_plan(g, labels, P)
    dev = g2.build_partition_plan(g, labels, P, device="cuda")
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(dev.flat, f), getattr(host.flat, f), err_msg=f)
    t0, t1 = host.topology(P // 2), dev.topology(P // 2)
    np.testing.assert_array_equal(t0.gather_map, t1.gather_map)
    np.testing.assert_array_equal(t0.src_pos, t1.src_pos)


def test_gpu_plan_empty_partition():
    g = g2.generate_kronecker(8, 6, seed=3)
    labels = np.zeros(g.num_vertices, dtype=np.int32)
    labels[1::2] = 2                      # partition 1 empty
    host = g2.build_partition_plan(g, labels, 3)
    dev = g2.build_partition_plan(g, labels, 3, device="cuda")
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(dev.flat, f), getattr(host.flat, f), err_msg=f)
