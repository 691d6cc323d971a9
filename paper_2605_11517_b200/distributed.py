"""Partition parallelism across GPUs.

One process per GPU.  Rank r owns a contiguous block of partition ids
(balanced by edges + targets) and therefore the targets of those partitions.
Its local row space is ``[owned vertices (perm order) | halo vertices]``,
the halo being every in-neighbour of an owned target and every out-neighbour
of an owned vertex that another rank owns, ordered by (owner rank, vertex id)
— the reference's (owner, id) gather order (plan.py:106-108) lifted to ranks,
so halo lists are deterministic and identical on every run.

Per layer the engine exchanges only the rows an aggregation actually reads:
forward, the transformed rows ``P = X W`` (transform-first) or the layer
input (aggregate-first); backward, the pre-scaled gradient rows for the
transposed pull.  Exchanges are one ``all_to_all_single`` each (packed by
a gather kernel, received in place into the contiguous halo block).  GAT's
transposed pull needs per-edge attention that only the target's owner
holds, so it runs over the transpose of the local in-CSR instead: halo rows
collect partial sums that a reverse all-to-all returns to their owners,
added in ascending source-rank order (``ShardDeviceGraph.reverse_add``).  The
weight gradients of all layers live in one flat buffer
(``engine._Weights.grad_bucket``) and are summed with one ``all_reduce``
before the replicated SGD step, and the loss/accuracy partial sums with a
second one.  Halo rows are received in place into the halo block when the
exchanged buffer's rows are exactly ld(width) wide (else through a scratch
buffer and one unpack kernel).  Choices that change which exchanges a rank
issues (keeping the forward state instead of regathering) are agreed by an
all-reduce MIN, so every rank runs the same collective sequence.  Owner-side accumulation replaces the paper's host atomics, so
results are deterministic for a fixed world size.

Transports: ``nccl`` (CUDA tensors over NVLink/NVSwitch) in production;
``gloo`` stages through host memory, which lets the same engine run with two
ranks on one GPU (tests) and lets the host-side shard logic run on CPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["LabelPlan", "ShardPlan", "Communicator", "assign_partitions", "build_shard_plan",
           "lean_shard_plan"]


def assign_partitions(plan, world: int) -> np.ndarray:
    """rank of every partition: contiguous blocks balanced by E_p + T_p."""
    t, g, e = plan.partition_sizes()
    cost = (e + t).astype(np.float64)
    P = plan.num_partitions
    if world > P:
        raise ValueError(f"{world} ranks need at least {world} partitions, plan has {P}")
    ranks = np.zeros(P, dtype=np.int64)
    prefix = np.concatenate([[0.0], np.cumsum(cost)])
    total = prefix[-1]
    start = 0
    for r in range(world):
        left = world - r
        if left == 1:
            ranks[start:] = r
            break
        # smallest block end whose prefix reaches the rank's fair share,
        # leaving at least one partition per remaining rank
        target = prefix[start] + (total - prefix[start]) / left
        end = int(np.searchsorted(prefix, target, side="left"))
        end = min(max(end, start + 1), P - (left - 1))
        ranks[start:end] = r
        start = end
    return ranks


def _csr_rows(ptr: np.ndarray, idx: np.ndarray, rows: np.ndarray):
    """Sub-CSR of the given rows (in that order): (row_ptr, column indices)."""
    lo, hi = ptr[rows], ptr[rows + 1]
    counts = hi - lo
    out_ptr = np.zeros(rows.size + 1, dtype=np.int64)
    np.cumsum(counts, out=out_ptr[1:])
    if out_ptr[-1] == 0:
        return out_ptr, np.zeros(0, dtype=idx.dtype)
    starts = np.repeat(lo - out_ptr[:-1], counts)
    pos = np.arange(out_ptr[-1], dtype=np.int64) + starts
    return out_ptr, idx[pos]


@dataclass
class ShardPlan:
    """Host-side description of one rank's shard (all numpy)."""

    rank: int
    world: int
    part_rank: np.ndarray        # [P] owning rank of each partition
    owned: np.ndarray            # [n_own] global ids, perm order
    halo: np.ndarray             # [n_halo] global ids, (owner, id) order
    halo_owner: np.ndarray       # [n_halo]
    recv_counts: np.ndarray      # [world] halo rows received from each rank
    in_ptr: np.ndarray           # local in-CSR over owned targets (int64)
    in_idx: np.ndarray           # local ids of in-neighbours (int32)
    out_ptr: np.ndarray          # local out-CSR over owned vertices
    out_idx: np.ndarray
    send_idx: np.ndarray | None = None      # [sum send] local ids, grouped by dest rank
    send_counts: np.ndarray | None = None   # [world]

    @property
    def n_own(self) -> int:
        return int(self.owned.size)

    @property
    def n_local(self) -> int:
        return int(self.owned.size + self.halo.size)

    @property
    def local_ids(self) -> np.ndarray:
        return np.concatenate([self.owned, self.halo])

    def local_transpose(self):
        """Transpose of the local in-CSR: rows = every local id (owned and
        halo sources), neighbours = the owned targets it feeds, ascending,
        and for each such edge its position in the in-CSR.  GAT's
        transposed pull reads the per-edge attention computed here; rows of
        halo sources hold partial sums for their owners (reverse exchange)."""
        n = self.n_local
        deg = np.diff(self.in_ptr)
        tgt = np.repeat(np.arange(self.n_own, dtype=np.int32), deg)
        order = np.argsort(self.in_idx, kind="stable")
        ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(self.in_idx, minlength=n), out=ptr[1:])
        return ptr, tgt[order], order.astype(np.int32)


def build_shard_plan(graph, plan, rank: int, world: int, comm=None) -> ShardPlan:
    """Shard of ``rank``: ownership, halo, local CSRs; with ``comm`` also the
    send lists (each rank requests its halo rows from their owners once)."""
    f = plan.flat
    n = plan.num_vertices
    part_rank = assign_partitions(plan, world)
    mine = np.flatnonzero(part_rank == rank)
    p0, p1 = int(mine[0]), int(mine[-1]) + 1
    r0, r1 = int(f.part_ptr[p0]), int(f.part_ptr[p1])
    owned = f.perm[r0:r1].astype(np.int64)
    owner = part_rank[plan.labels.astype(np.int64)]
    e0, e1 = int(f.in_ptr[r0]), int(f.in_ptr[r1])
    in_nbr = f.in_src[e0:e1].astype(np.int64)
    out_ptr_g, out_nbr = _csr_rows(graph.src_ptr, graph.dst_idx.astype(np.int64), owned)
    cand = np.unique(np.concatenate([in_nbr, out_nbr]))
    halo = cand[owner[cand] != rank]
    order = np.lexsort((halo, owner[halo]))
    halo = halo[order]
    halo_owner = owner[halo]
    lid = np.full(n, -1, dtype=np.int64)
    lid[owned] = np.arange(owned.size)
    lid[halo] = owned.size + np.arange(halo.size)
    in_ptr = (f.in_ptr[r0:r1 + 1] - f.in_ptr[r0]).astype(np.int64)
    sp = ShardPlan(
        rank=rank, world=world, part_rank=part_rank, owned=owned, halo=halo,
        halo_owner=halo_owner, recv_counts=np.bincount(halo_owner, minlength=world).astype(np.int64),
        in_ptr=in_ptr, in_idx=lid[in_nbr].astype(np.int32),
        out_ptr=out_ptr_g, out_idx=lid[out_nbr].astype(np.int32))
    if comm is not None:
        # tell every owner which of its rows we need, in our halo order
        requests = comm.exchange_ids(halo, sp.recv_counts)
        sp.send_counts = requests.counts
        sp.send_idx = lid[requests.ids].astype(np.int32)
        if (sp.send_idx < 0).any() or (sp.send_idx >= owned.size).any():
            raise RuntimeError("halo request for a row this rank does not own")
    return sp


@dataclass
class _Requests:
    ids: np.ndarray
    counts: np.ndarray


class LabelPlan:
    """What a shard needs of a partition plan, from the labels alone (no
    whole-graph gather maps): per-partition sizes for the rank assignment,
    global in-degrees for the degree scales.  Lets every rank of a
    configs[3]-size run skip the ~16 GB host plan (lean_shard_plan)."""

    def __init__(self, graph, labels: np.ndarray, num_partitions: int):
        from types import SimpleNamespace
        self.labels = np.asarray(labels, dtype=np.int32)
        self.num_partitions = int(num_partitions)
        self.num_vertices = int(graph.num_vertices)
        indeg = np.bincount(np.asarray(graph.dst_idx), minlength=self.num_vertices)
        self.flat = SimpleNamespace(in_degree=indeg.astype(np.int32))
        self._t = np.bincount(self.labels, minlength=self.num_partitions).astype(np.int64)
        self._e = np.bincount(self.labels, weights=indeg.astype(np.float64),
                              minlength=self.num_partitions).astype(np.int64)
        self.device_cache: dict = {}

    def partition_sizes(self):
        return self._t, np.zeros_like(self._t), self._e


def lean_shard_plan(graph, lplan: LabelPlan, rank: int, world: int, comm=None) -> ShardPlan:
    """build_shard_plan for a symmetric graph (the generators' graphs are)
    without the whole plan: owned rows = the targets of the rank's
    partitions (partition by partition, ascending ids — the plan's perm
    order), in-neighbours = out-neighbours (neighbours ascending by id
    instead of by gather position: only the float summation order
    differs), halo in (owner rank, id) order, send lists exchanged."""
    n = lplan.num_vertices
    labels = lplan.labels.astype(np.int64)
    part_rank = assign_partitions(lplan, world)
    mine = np.flatnonzero(part_rank == rank)
    owned = np.flatnonzero(np.isin(labels, mine))
    owned = owned[np.argsort(labels[owned], kind="stable")]
    owner = part_rank[labels]
    # int32 neighbour ids (no int64 copy of the whole edge array: 13 GB
    # per rank at configs[3])
    ptr, nbr = _csr_rows(graph.src_ptr, np.asarray(graph.dst_idx, dtype=np.int32), owned)
    cand = np.unique(nbr).astype(np.int64)
    halo = cand[owner[cand] != rank]
    halo = halo[np.lexsort((halo, owner[halo]))]
    halo_owner = owner[halo]
    lid = np.full(n, -1, dtype=np.int64)
    lid[owned] = np.arange(owned.size)
    lid[halo] = owned.size + np.arange(halo.size)
    local = lid[nbr].astype(np.int32)
    sp = ShardPlan(
        rank=rank, world=world, part_rank=part_rank, owned=owned, halo=halo,
        halo_owner=halo_owner, recv_counts=np.bincount(halo_owner, minlength=world).astype(np.int64),
        in_ptr=ptr, in_idx=local, out_ptr=ptr, out_idx=local)
    if comm is not None:
        requests = comm.exchange_ids(halo, sp.recv_counts)
        sp.send_counts = requests.counts
        sp.send_idx = lid[requests.ids].astype(np.int32)
        if (sp.send_idx < 0).any() or (sp.send_idx >= owned.size).any():
            raise RuntimeError("halo request for a row this rank does not own")
    return sp


class Communicator:
    """torch.distributed wrapper: ``nccl`` moves CUDA tensors directly,
    ``gloo`` stages them through host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        self.device_native = self.backend == "nccl"

    def exchange_ids(self, ids: np.ndarray, counts: np.ndarray) -> _Requests:
        """all-to-all of int64 id lists (setup only, host tensors or CUDA for nccl)."""
        import torch
        dev = torch.device("cuda") if self.device_native else torch.device("cpu")
        cnt = torch.from_numpy(np.asarray(counts, dtype=np.int64)).to(dev)
        recv_cnt = torch.empty_like(cnt)
        self.dist.all_to_all_single(recv_cnt, cnt, group=self.group)
        rc = recv_cnt.cpu().numpy()
        send = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int64)).to(dev)
        recv = torch.empty(int(rc.sum()), dtype=torch.int64, device=dev)
        self.dist.all_to_all_single(recv, send, [int(x) for x in rc], [int(x) for x in counts],
                                    group=self.group)
        return _Requests(ids=recv.cpu().numpy(), counts=rc.astype(np.int64))

    def all_to_all_rows(self, recv, send, recv_counts, send_counts, async_op: bool = False):
        """Row all-to-all of contiguous 2-D tensors (rows split by rank).
        ``async_op``: NCCL returns the work handle (``wait()`` makes the
        current stream wait for it); host-staged gloo completes before
        returning (None)."""
        rs = [int(x) for x in recv_counts]
        ss = [int(x) for x in send_counts]
        if self.device_native:
            work = self.dist.all_to_all_single(recv, send, rs, ss, group=self.group, async_op=async_op)
            return work if async_op else None
        r_host = recv.new_empty(recv.shape, device="cpu")
        self.dist.all_to_all_single(r_host, send.cpu(), rs, ss, group=self.group)
        recv.copy_(r_host)
        return None

    def all_reduce_sum(self, t) -> None:
        if self.device_native:
            self.dist.all_reduce(t, group=self.group)
            return
        h = t.cpu()
        self.dist.all_reduce(h, group=self.group)
        t.copy_(h)

    def all_reduce_min(self, t) -> None:
        op = self.dist.ReduceOp.MIN
        if self.device_native:
            self.dist.all_reduce(t, op=op, group=self.group)
            return
        h = t.cpu()
        self.dist.all_reduce(h, op=op, group=self.group)
        t.copy_(h)

    def barrier(self) -> None:
        self.dist.barrier(group=self.group)
