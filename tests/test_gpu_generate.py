"""GPU Kronecker generator (graph.generate_kronecker(..., device="cuda")):
bit-identical to the native host generator, which is itself pinned to the
reference (tests/test_native_host.py, tests/test_oracle_golden.py)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2605_11517_b200 as g2  # noqa: E402


@pytest.mark.parametrize("scale,deg,seed", [
    (4, 3, 0),        # tiny, one 1024-pair round
    (5, 30, 1),       # nearly complete graph: many rounds before the target
    (10, 8, 2),
    (12, 16, 3),
    (17, 8, 0),       # BASELINE configs[0]
])
def test_gpu_generator_matches_host(scale, deg, seed):
    host = g2.generate_kronecker(scale, deg, seed=seed)
    dev = g2.generate_kronecker(scale, deg, seed=seed, device="cuda")
    assert dev.num_vertices == host.num_vertices and dev.num_edges == host.num_edges
    np.testing.assert_array_equal(dev.src_ptr, host.src_ptr)
    np.testing.assert_array_equal(dev.dst_idx, host.dst_idx)


@pytest.mark.parametrize("n,F,seed", [(1000, 128, 1), (777, 7, 3), (50, 100, 15)])
def test_gpu_feature_rows_match_dataset(n, F, seed):
    """grd_feature_rows: any rows of make_random_dataset's feature matrix,
    bit-exact, without the others (a sharded run's per-rank rows)."""
    from paper_2605_11517_b200.dataset import random_feature_rows
    ds = g2.make_random_dataset(g2.build_csr([], n), feature_dim=F, num_classes=3, seed=seed,
                                feature_dtype=np.float32)
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(n, size=n // 3, replace=False))
    got = random_feature_rows(F, seed, rows=rows).cpu().numpy()
    np.testing.assert_array_equal(got[:, :F], ds.features[rows])
    assert not got[:, F:].any()
    got = random_feature_rows(F, seed, row0=5, n_rows=n - 5).cpu().numpy()
    np.testing.assert_array_equal(got[:, :F], ds.features[5:])
