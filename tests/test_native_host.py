"""Host-side native code (generator, partitioner, plan) — bit-exact with
the reference (golden digests) and with the oracle.  Runs on CPU."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from oracle import graph as ograph, partition as opart, plan as oplan
from paper_2605_11517_b200 import (PartitionerParams, build_csr, build_partition_plan,
                                   generate_kronecker, random_partition,
                                   switching_aware_partition)


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("scale,deg,seed", [(4, 2, 0), (6, 6, 3), (8, 8, 0), (9, 5, 17), (10, 12, 4)])
def test_generator_matches_oracle(scale, deg, seed):
    g = generate_kronecker(scale, deg, seed)
    ptr, dst = ograph.kronecker(scale, deg, seed)
    np.testing.assert_array_equal(g.src_ptr, ptr)
    np.testing.assert_array_equal(g.dst_idx, dst)
    g.validate()


def test_generator_thread_count_invariant():
    a = generate_kronecker(12, 8, 5, num_threads=1)
    b = generate_kronecker(12, 8, 5, num_threads=7)
    np.testing.assert_array_equal(a.dst_idx, b.dst_idx)


def test_generator_rejects_bad_args():
    with pytest.raises(ValueError):
        generate_kronecker(3, 4, 0)
    with pytest.raises(ValueError):
        generate_kronecker(6, 0, 0)


def test_build_csr_dedup_and_order():
    g = build_csr([(2, 1), (0, 2), (2, 0), (0, 2), (2, 1), (1, 0)], 3)
    assert g.src_ptr.tolist() == [0, 1, 2, 4]
    assert g.dst_idx.tolist() == [2, 0, 1, 0]
    empty = build_csr([], 4)
    assert empty.num_edges == 0 and empty.src_ptr.tolist() == [0] * 5
    with pytest.raises(ValueError):
        build_csr([(0, 5)], 3)


@pytest.mark.parametrize("scale,deg,P,depth", [(7, 6, 3, 2), (8, 8, 4, 2), (8, 8, 4, 3), (9, 4, 6, 2)])
def test_partitioner_matches_oracle(scale, deg, P, depth):
    g = generate_kronecker(scale, deg, scale)
    res = switching_aware_partition(g, P, PartitionerParams(seed=scale + 2, group_depth=depth))
    ref = opart.partition(g.src_ptr, g.dst_idx, P, group_depth=depth, seed=scale + 2)
    np.testing.assert_array_equal(res.labels, ref["labels"])
    assert res.objective_trace == ref["objective_trace"]
    assert res.initial_objective == ref["initial_objective"]
    assert res.iterations == ref["iterations"]
    assert res.converged == ref["converged"]
    assert res.max_size_per_iteration == ref["max_size_per_iteration"]


def test_partitioner_capacity_and_single_partition():
    g = generate_kronecker(8, 8, 1)
    res = switching_aware_partition(g, 4, PartitionerParams(seed=1, beta=1.2, alpha_balance=1.1))
    cap = int(np.floor(1.2 * g.num_vertices / 4 + 1e-9))
    assert max(res.max_size_per_iteration[1:]) <= cap
    one = switching_aware_partition(g, 1)
    assert one.iterations == 0 and one.converged and not one.labels.any()


def test_random_partition_balanced():
    lab = random_partition(103, 5, seed=2)
    counts = np.bincount(lab, minlength=5)
    assert counts.max() - counts.min() <= 1
    np.testing.assert_array_equal(lab, opart.random_labels(103, 5, 2))


def test_config1_generator_partitioner_plan_exact(config1_golden):
    gold = config1_golden
    g = generate_kronecker(17, 8, seed=0)
    assert _digest(g.src_ptr, g.dst_idx) == str(gold["graph_digest"])
    res = switching_aware_partition(g, 8, PartitionerParams(seed=2))
    np.testing.assert_array_equal(res.labels, gold["sa_labels"].astype(np.int32))
    assert res.objective_trace == gold["sa_objective_trace"].tolist()
    assert res.initial_objective == float(gold["sa_initial_objective"])
    assert res.iterations == int(gold["sa_iterations"])
    assert res.converged == bool(gold["sa_converged"])
    assert res.max_size_per_iteration == gold["sa_max_sizes"].tolist()
    plan = build_partition_plan(g, res.labels, 8)
    for q, t in enumerate(plan.topologies):
        assert _digest(t.targets, t.gather_map, t.tgt_ptr, t.src_pos, t.edge_local_target,
                       t.self_pos, t.target_indeg, t.gather_indeg) == str(gold[f"plan_digest_{q}"])


@pytest.mark.parametrize("scale,deg,P", [(6, 4, 3), (8, 8, 5), (9, 6, 8)])
def test_plan_matches_oracle(scale, deg, P):
    g = generate_kronecker(scale, deg, scale)
    labels = random_partition(g.num_vertices, P, seed=scale)
    plan = build_partition_plan(g, labels, P)
    ref = oplan.build_plan(g.src_ptr, g.dst_idx, labels, P)
    for a, b in zip(plan.topologies, ref):
        for f in ("targets", "gather_map", "tgt_ptr", "src_pos", "edge_local_target", "self_pos",
                  "target_indeg", "gather_indeg"):
            np.testing.assert_array_equal(getattr(a, f), getattr(b, f))


def test_plan_kat_and_edge_cases():
    # reference test_training.py:45-56 — partition 0 gathers [0, 1, 4, 6, 7]
    g = build_csr([(4, 0), (6, 1), (7, 1), (0, 1), (1, 0), (2, 3), (3, 2), (5, 4)], 8)
    plan = build_partition_plan(g, np.array([0, 0, 1, 1, 2, 2, 3, 3], dtype=np.int32), 4)
    assert plan.gather_maps[0].tolist() == [0, 1, 4, 6, 7]
    assert plan.target_ranges[0].tolist() == [0, 1]
    # empty partitions (test_training.py:91-96)
    g2 = build_csr([(0, 1), (1, 0)], 2)
    plan2 = build_partition_plan(g2, np.zeros(2, dtype=np.int32), 3)
    assert plan2.empty_partitions == [1, 2]
    assert plan2.topologies[1].num_edges == 0
    with pytest.raises(ValueError):
        build_partition_plan(g2, np.array([0, 3], dtype=np.int32), 3)
    with pytest.raises(ValueError):
        build_partition_plan(g2, np.zeros(3, dtype=np.int32), 1)
    # single partition = whole graph
    g3 = generate_kronecker(6, 6, seed=3)
    p3 = build_partition_plan(g3, np.zeros(g3.num_vertices, dtype=np.int32), 1)
    np.testing.assert_array_equal(p3.gather_maps[0], np.arange(g3.num_vertices))
    assert p3.topologies[0].num_edges == g3.num_edges


def test_csr_transpose_is_the_stable_argsort():
    """grd_csr_transpose == the transposed edge order np.argsort(kind="stable")
    gives (np.add.at's order in a partition's backward, training.py:141)."""
    import ctypes
    from paper_2605_11517_b200 import _lib
    rng = np.random.default_rng(5)
    for n_rows, n_cols, nnz in ((0, 3, 0), (7, 1, 20), (500, 97, 4000), (50, 1000, 300)):
        deg = np.bincount(rng.integers(0, max(n_rows, 1), nnz), minlength=n_rows)[:n_rows] if n_rows else []
        ptr = np.zeros(n_rows + 1, dtype=np.int64)
        np.cumsum(deg, out=ptr[1:])
        idx = rng.integers(0, n_cols, int(ptr[-1])).astype(np.int32)
        col_ptr = np.empty(n_cols + 1, dtype=np.int64)
        rows = np.empty(idx.size, dtype=np.int32)
        assert _lib.lib().grd_csr_transpose(n_rows, ptr.ctypes.data, idx.ctypes.data, n_cols,
                                            col_ptr.ctypes.data, rows.ctypes.data) == 0
        local = np.repeat(np.arange(n_rows), np.diff(ptr))
        want = local[np.argsort(idx, kind="stable")]
        assert np.array_equal(rows, want)
        assert np.array_equal(np.diff(col_ptr), np.bincount(idx, minlength=n_cols))
    bad = np.array([0, 1], dtype=np.int64)
    assert _lib.lib().grd_csr_transpose(1, bad.ctypes.data, np.array([5], np.int32).ctypes.data, 2,
                                        np.empty(3, np.int64).ctypes.data,
                                        np.empty(1, np.int32).ctypes.data) < 0


def test_csr_same_rows_detects_symmetry():
    """grd_csr_same_rows(G, transpose(G)) == 1 exactly for symmetric graphs
    (the streaming engine then keeps one CSR for both directions)."""
    from paper_2605_11517_b200 import _lib, build_csr, generate_kronecker

    def same(g):
        n, m = g.num_vertices, g.num_edges
        tp = np.empty(n + 1, np.int64)
        ti = np.empty(max(m, 1), np.int32)
        L = _lib.lib()
        _lib.check(L.grd_csr_transpose(n, _lib.ptr(g.src_ptr), _lib.ptr(g.dst_idx), n,
                                       _lib.ptr(tp), _lib.ptr(ti)))
        assert np.all(np.diff(tp) >= 0)
        for v in range(0, n, max(1, n // 50)):        # rows ascending
            assert np.all(np.diff(ti[tp[v]:tp[v + 1]]) > 0)
        eq = np.zeros(1, np.int32)
        _lib.check(L.grd_csr_same_rows(n, _lib.ptr(g.src_ptr), _lib.ptr(g.dst_idx), _lib.ptr(tp),
                                       _lib.ptr(ti), 4, _lib.ptr(eq)))
        return bool(eq[0])

    g = generate_kronecker(12, 8, seed=3)
    assert same(g)
    src = np.repeat(np.arange(g.num_vertices), np.diff(g.src_ptr))
    keep = np.arange(g.num_edges) != 17
    assert not same(build_csr(np.stack([src[keep], g.dst_idx[keep]], 1), g.num_vertices))
    assert same(build_csr(np.zeros((0, 2), np.int64), 5))


def _aligned(nbytes, align=4096):
    raw = np.zeros(nbytes + align, dtype=np.uint8)
    pad = (-raw.ctypes.data) % align
    return raw[pad: pad + nbytes]


def test_direct_io_roundtrip(tmp_path):
    """Storage-tier I/O (grd_direct_*): aligned multi-threaded write / read
    round trip, zero fill past EOF, alignment errors raise ValueError."""
    from paper_2605_11517_b200 import _lib
    L = _lib.lib()
    al = int(L.grd_direct_alignment())
    assert al == 4096
    path = str(tmp_path / "tier.bin").encode()
    fd, direct = np.zeros(1, np.int32), np.zeros(1, np.int32)
    n = 3 * (8 << 20) + 5 * al                     # several 8 MiB slices + a tail
    _lib.check(L.grd_direct_open(path, 1, n, _lib.ptr(fd), _lib.ptr(direct)))
    src = _aligned(n)
    src[:] = np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)
    _lib.check(L.grd_direct_write(int(fd[0]), 0, n, _lib.ptr(src), 4))
    _lib.check(L.grd_direct_close(int(fd[0])))
    _lib.check(L.grd_direct_open(path, 0, 0, _lib.ptr(fd), _lib.ptr(direct)))
    dst = _aligned(n + 2 * al)
    dst[:] = 7
    _lib.check(L.grd_direct_read(int(fd[0]), 0, n + 2 * al, _lib.ptr(dst), 3))
    np.testing.assert_array_equal(dst[:n], src)
    assert not dst[n:].any()                       # past EOF reads as zeros
    part = _aligned(2 * al)
    _lib.check(L.grd_direct_read(int(fd[0]), 4 * al, 2 * al, _lib.ptr(part), 2))
    np.testing.assert_array_equal(part, src[4 * al: 6 * al])
    with pytest.raises(ValueError):
        _lib.check(L.grd_direct_read(int(fd[0]), 100, al, _lib.ptr(part), 1))
    _lib.check(L.grd_direct_close(int(fd[0])))


def test_file_backing_of_mmapped_features(tmp_path):
    """load_dataset(..., mmap_features=True) keeps the features in their file;
    file_backing() finds (path, offset of row 0) for the storage tier."""
    import paper_2605_11517_b200 as g2
    from paper_2605_11517_b200.tiers import file_backing
    g = g2.generate_kronecker(8, 4, seed=1)
    ds = g2.make_random_dataset(g, feature_dim=12, num_classes=3, seed=2)
    ds.save(tmp_path)
    mm = g2.load_dataset(tmp_path, mmap_features=True)
    assert mm.features.dtype == np.float32
    np.testing.assert_array_equal(mm.features, ds.features.astype(np.float32))
    path, off = file_backing(mm.features)
    assert path.endswith("features.bin") and off == 16
    raw = np.fromfile(path, dtype=np.uint8)
    row5 = raw[off + 5 * 48: off + 6 * 48].view(np.float32)
    np.testing.assert_array_equal(row5, mm.features[5])
    assert file_backing(np.zeros((3, 4), np.float32)) is None


@pytest.mark.parametrize("n,F,C,seed", [(1000, 128, 10, 1), (999, 7, 5, 3), (57, 3, 47, 11)])
def test_labels_mask_without_features_match_dataset(n, F, C, seed):
    """random_labels_mask jumps the PCG64 stream past the feature draws (odd
    draw counts leave numpy's buffered half) and equals make_random_dataset."""
    from paper_2605_11517_b200 import make_random_dataset
    from paper_2605_11517_b200.dataset import random_labels_mask
    ds = make_random_dataset(build_csr([], n), feature_dim=F, num_classes=C, seed=seed)
    labels, mask = random_labels_mask(n, F, C, seed)
    np.testing.assert_array_equal(labels, ds.labels)
    np.testing.assert_array_equal(mask, ds.train_mask)


@pytest.mark.parametrize("scale,deg,P", [(8, 6, 3), (10, 8, 5)])
def test_gat_partition_specs_are_consistent(scale, deg, P):
    """The per-partition GAT specs (engine.DevicePartition.gat_specs, host
    side on CPU tensors): the forward rows are the targets with output row
    self_pos; every pull edge of gather row g maps (edge_perm) to a forward
    edge whose source is g and whose target's gather row is the pull
    edge's neighbour, each forward edge exactly once, targets ascending."""
    from paper_2605_11517_b200.engine import DevicePartition
    g = generate_kronecker(scale, deg, seed=scale)
    plan = build_partition_plan(g, random_partition(g.num_vertices, P, 1), P)
    for q in range(P):
        part = DevicePartition.from_plan(plan, q, "cpu")
        fwd, pull, perm = part.gat_specs()
        tgt_ptr, src_pos, self_pos = part._csr
        assert np.array_equal(fwd.out_idx.numpy(), self_pos)
        E = src_pos.size
        perm = perm.numpy()[:E]
        assert np.array_equal(np.sort(perm), np.arange(E))
        tgt_of_edge = np.repeat(np.arange(part.num_targets), np.diff(tgt_ptr))
        ptr = pull.row_ptr.numpy()
        idx = pull.idx.numpy()
        assert ptr[-1] == E and ptr.size == part.num_gather + 1
        rows = np.repeat(np.arange(part.num_gather), np.diff(ptr))
        assert np.array_equal(src_pos[perm], rows)
        assert np.array_equal(self_pos[tgt_of_edge[perm]], idx)
        for r in range(part.num_gather):   # targets ascending within a pull row
            t = tgt_of_edge[perm[ptr[r]:ptr[r + 1]]]
            assert np.all(np.diff(t) >= 0)
