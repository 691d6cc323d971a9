"""Host-side logic of the sharded (multi-GPU) engine with the gloo backend,
world size 2 and 3, on CPU: partition-to-rank assignment, ownership, halo
lists, local CSRs and the halo request exchange."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2605_11517_b200 as g2
from paper_2605_11517_b200.distributed import (Communicator, _csr_rows, assign_partitions,
                                               build_shard_plan)


def _setup(scale=9, deg=8, P=6):
    g = g2.generate_kronecker(scale, deg, seed=1)
    labels = g2.switching_aware_partition(g, P, g2.PartitionerParams(seed=3)).labels
    return g, g2.build_partition_plan(g, labels, P)


def test_assign_partitions_contiguous_and_balanced():
    g, plan = _setup(P=8)
    for world in (1, 2, 3, 4, 8):
        ranks = assign_partitions(plan, world)
        assert (np.diff(ranks) >= 0).all() and ranks[0] == 0 and ranks[-1] == world - 1
        assert set(ranks.tolist()) == set(range(world))
    with pytest.raises(ValueError):
        assign_partitions(plan, 9)


def test_csr_rows_helper():
    ptr = np.array([0, 2, 2, 5], dtype=np.int64)
    idx = np.array([7, 8, 9, 10, 11])
    p, i = _csr_rows(ptr, idx, np.array([2, 0, 1]))
    assert p.tolist() == [0, 3, 5, 5] and i.tolist() == [9, 10, 11, 7, 8]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, plan = _setup()
    comm = Communicator()
    sp = build_shard_plan(g, plan, rank, world, comm)
    # exchange the owned global ids along the send lists: what arrives must
    # be exactly this rank's halo, in its (owner, id) order
    import torch
    send = torch.from_numpy(sp.owned[sp.send_idx].astype(np.float32)).reshape(-1, 1).contiguous()
    recv = torch.empty((sp.halo.size, 1), dtype=torch.float32)
    comm.all_to_all_rows(recv, send, sp.recv_counts, sp.send_counts)
    # GAT's transposed pull: partial sums over the local in-CSR's transpose,
    # halo rows returned to their owners by the reverse exchange
    tp, ti, tperm = sp.local_transpose()
    srcs = np.repeat(np.arange(sp.n_local), np.diff(tp))
    assert np.array_equal(np.repeat(np.arange(sp.n_own), np.diff(sp.in_ptr))[tperm], ti)
    assert np.array_equal(sp.in_idx[tperm], srcs)
    part = np.zeros(sp.n_local)
    np.add.at(part, srcs, sp.owned[ti].astype(np.float64))
    rsend = torch.from_numpy(part[sp.n_own:]).reshape(-1, 1).contiguous()
    rrecv = torch.empty((sp.send_idx.size, 1), dtype=torch.float64)
    comm.all_to_all_rows(rrecv, rsend, sp.send_counts, sp.recv_counts)
    pulled = part[: sp.n_own].copy()
    np.add.at(pulled, sp.send_idx, rrecv.numpy().ravel())
    np.savez(os.path.join(out, f"r{rank}.npz"), owned=sp.owned, halo=sp.halo, got=recv.numpy().ravel(),
             pulled=pulled,
             in_ptr=sp.in_ptr, in_idx=sp.in_idx, out_ptr=sp.out_ptr, out_idx=sp.out_idx,
             recv_counts=sp.recv_counts, send_counts=sp.send_counts)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shard_plans_cover_the_graph(tmp_path, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g, plan = _setup()
    shards = [dict(np.load(tmp_path / f"r{r}.npz")) for r in range(world)]
    owned = np.concatenate([s["owned"] for s in shards])
    assert np.array_equal(np.sort(owned), np.arange(g.num_vertices))
    owner = np.empty(g.num_vertices, dtype=np.int64)
    for r, s in enumerate(shards):
        owner[s["owned"]] = r
    for r, s in enumerate(shards):
        local = np.concatenate([s["owned"], s["halo"]])
        assert (owner[s["halo"]] != r).all()
        keys = owner[s["halo"]] * g.num_vertices + s["halo"]
        assert (np.diff(keys) > 0).all()                      # (owner, id) order
        assert np.array_equal(s["got"].astype(np.int64), s["halo"])
        # local in-CSR = the plan's in-edges of the owned targets
        for k in range(0, s["owned"].size, 37):
            v = s["owned"][k]
            want = np.sort(g.edge_sources()[g.dst_idx == v])
            have = np.sort(local[s["in_idx"][s["in_ptr"][k]:s["in_ptr"][k + 1]]])
            assert np.array_equal(want, have)
            outs = np.sort(g.neighbors(v))
            assert np.array_equal(outs, np.sort(local[s["out_idx"][s["out_ptr"][k]:s["out_ptr"][k + 1]]]))
        # transposed pull + reverse exchange = sum over every out-edge
        want = np.array([g.neighbors(u).astype(np.float64).sum() for u in s["owned"]])
        assert np.array_equal(s["pulled"], want)
        # what r sends to t is what t receives from r
        for t, st in enumerate(shards):
            if t != r:
                assert s["send_counts"][t] == st["recv_counts"][r]


def test_lean_shard_plan_equals_plan_based_shard_on_symmetric_graphs():
    """The plan-free shard builder (symmetric graphs) gives the same owned
    rows, halo, halo owners and per-row neighbour sets as build_shard_plan."""
    import paper_2605_11517_b200 as g2
    from paper_2605_11517_b200.distributed import LabelPlan, build_shard_plan, lean_shard_plan
    g = g2.generate_kronecker(10, 8, seed=3)
    labels = g2.switching_aware_partition(g, 6, g2.PartitionerParams(seed=1)).labels
    plan = g2.build_partition_plan(g, labels, 6)
    lp = LabelPlan(g, labels, 6)
    for world in (1, 2, 3):
        for rank in range(world):
            a = build_shard_plan(g, plan, rank, world)
            b = lean_shard_plan(g, lp, rank, world)
            np.testing.assert_array_equal(a.part_rank, b.part_rank)
            np.testing.assert_array_equal(a.owned, b.owned)
            np.testing.assert_array_equal(a.halo, b.halo)
            np.testing.assert_array_equal(a.halo_owner, b.halo_owner)
            np.testing.assert_array_equal(a.in_ptr, b.in_ptr)
            for r in range(a.n_own):
                sa = np.sort(a.in_idx[a.in_ptr[r]:a.in_ptr[r + 1]])
                sb = np.sort(b.in_idx[b.in_ptr[r]:b.in_ptr[r + 1]])
                np.testing.assert_array_equal(sa, sb)
