"""Device engine of the partition-wise GCN training step.

Two execution paths share the same kernels (ops.py -> libgrinder_b200.so):

* ``LayerwiseEngine`` — the fast path.  All partitions of a layer are one
  launch over the concatenated plan (rows = targets of partition 0, then 1,
  ...; edges pre-composed to global source ids ``gather_map[src_pos]``), so
  the gathered block GA_p is never materialised in HBM.  Per layer the
  engine picks the cheaper association of the GCN layer:

    transform-first (d_out <= d_in):  P = X W,  out = act(A_hat P)
        backward: H = A_hat^T gp,  dW = X^T H,  dX = H W^T
    aggregate-first (d_out >  d_in):  N = A_hat X,  out = act(N W)
        backward: N recomputed (regather), dW = N^T gp, dX = A_hat^T (gp W^T)

  Both equal the reference's (A_hat GA) W (training.py:72-83,103-143) up to
  fp32 rounding; transform-first aggregates at the narrower width and
  needs no forward recompute.  The transposed aggregation A_hat^T is a
  deterministic pull over the graph's own CSR (out-edges), so no float
  atomics and no per-partition scatter are needed.  Degree scales, ReLU
  masks and the next layer's pre-scale are fused into the producing
  kernel's epilogue, and the SGD step into the weight-gradient reduction.

* ``PartitionEngine`` — the literal per-(layer, partition) schedule of
  training.py:259-358: gather GA_p, layer forward, regather (or snapshot)
  in backward, per-partition grad_GA / grad_W, ascending-pid scatter.  It
  serves the reference's per-partition operators, ``grad_probe``,
  ``use_snapshots`` and tier-manager hooks.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib, ops
from .distributed import _csr_rows
from .ops import AggSpec, ld_of

__all__ = ["DeviceGraph", "DevicePartition", "LayerOps", "LayerwiseEngine", "PartitionEngine",
           "ShardDeviceGraph", "dropout_mask"]


def dropout_mask(dropout_rate: float, dropout_seed: int, epoch: int, layer: int,
                 shape: tuple[int, int]) -> np.ndarray | None:
    """Seeded keep-mask / keep (training.py:178-185), drawn on the host."""
    if dropout_rate == 0.0:
        return None
    seq = np.random.SeedSequence(dropout_seed, spawn_key=(epoch, layer))
    keep = 1.0 - dropout_rate
    return (np.random.Generator(np.random.PCG64(seq)).random(shape) < keep) / keep


def _degree_sched() -> bool:
    import os
    return os.environ.get("GRD_AGG_ROW_ORDER", "degree") == "degree"


def _degree_order(ptr: np.ndarray) -> np.ndarray | None:
    """Rows by descending degree (stable), or None for the given order
    (GRD_AGG_ROW_ORDER=plan).  Every row's sum is unchanged (same edges in
    the same order), only the order rows are scheduled in: measured -8 % on
    the products-shaped 256-wide aggregation (tools/agg_order.py) — warps
    get rows of similar length and the hub rows start first."""
    if not _degree_sched():
        return None
    return np.argsort(-np.diff(ptr), kind="stable")


def _reorder_rows(ptr: np.ndarray, idx: np.ndarray, order: np.ndarray):
    """CSR rows taken in ``order`` (edges of a row keep their order); also
    the new position of every old edge."""
    cnt = np.diff(ptr)[order]
    new_ptr = np.zeros(order.size + 1, dtype=np.int64)
    np.cumsum(cnt, out=new_ptr[1:])
    old_start = np.repeat(ptr[order] - new_ptr[:-1], cnt)
    old_pos = np.arange(new_ptr[-1], dtype=np.int64) + old_start   # old position of each new edge
    return new_ptr, idx[old_pos], old_pos


class DeviceGraph:
    """HBM-resident plan of one (graph, labeling): forward in-CSR (rows =
    targets, scheduled by descending degree, output row = vertex), the
    out-CSR for the transposed pull (likewise), and per-vertex degree scales."""

    def __init__(self, graph, plan, device):
        f = plan.flat
        self.device = device
        self.num_vertices = plan.num_vertices
        self.num_edges = int(f.in_ptr[-1])
        self.num_partitions = plan.num_partitions
        self.part_ptr = f.part_ptr.copy()
        # rows computed on this device / rows held (owned + halo); one device
        # owns every vertex and holds no halo
        self.n_own = self.n_local = plan.num_vertices
        self.comm = None
        # forward: rows = targets, output row = vertex, self = vertex
        fo = _degree_order(f.in_ptr)
        self._fwd_order = fo
        if fo is None:
            self.fwd = AggSpec.build(f.in_ptr, f.in_src, device, out_idx=f.perm)
        else:
            ptr, idx, _ = _reorder_rows(f.in_ptr, f.in_src, fo)
            self.fwd = AggSpec.build(ptr, idx, device, out_idx=f.perm[fo])
            del ptr, idx
        # transposed pull: rows = vertices, neighbours = out-edges (u -> v)
        bo = _degree_order(graph.src_ptr)
        self._bwd_order = bo
        if bo is None:
            self.bwd = AggSpec.build(graph.src_ptr, graph.dst_idx, device)
        else:
            ptr, idx, _ = _reorder_rows(graph.src_ptr, graph.dst_idx, bo)
            self.bwd = AggSpec.build(ptr, idx, device, out_idx=bo.astype(np.int32))
            del ptr, idx
        self._deg = f.in_degree.astype(np.float64)
        self._scales: dict[str, torch.Tensor] = {}
        self._partitions: dict[int, "DevicePartition"] = {}
        self.plan = plan
        self.graph = graph

    def exchange(self, buf: torch.Tensor, width: int) -> None:
        """Fill the halo rows of ``buf`` from their owners (no-op on one device)."""
        return None

    def out_to_in_perm(self) -> torch.Tensor:
        """For every out-edge (graph CSR order) its position in the forward
        in-CSR (GAT reads per-edge attention in the transposed pull)."""
        if getattr(self, "_o2i", None) is None:
            f, g = self.plan.flat, self.graph
            n = np.int64(self.num_vertices)
            # the device CSRs' row orders (see __init__)
            in_ptr, in_src, perm = f.in_ptr, f.in_src, f.perm
            if self._fwd_order is not None:
                in_ptr, in_src, _ = _reorder_rows(f.in_ptr, f.in_src, self._fwd_order)
                perm = f.perm[self._fwd_order]
            out_ptr, out_dst = g.src_ptr, g.dst_idx
            out_rows = np.arange(self.num_vertices, dtype=np.int64)
            if self._bwd_order is not None:
                out_ptr, out_dst, _ = _reorder_rows(g.src_ptr, g.dst_idx, self._bwd_order)
                out_rows = self._bwd_order.astype(np.int64)
            tgt = np.repeat(perm.astype(np.int64), np.diff(in_ptr))
            key_in = in_src.astype(np.int64) * n + tgt
            order = np.argsort(key_in, kind="stable")
            src = np.repeat(out_rows, np.diff(out_ptr))
            key_out = src * n + out_dst.astype(np.int64)
            pos = order[np.searchsorted(key_in[order], key_out)]
            # at least one element: an edgeless graph still passes a valid pointer
            self._o2i = torch.from_numpy(np.concatenate([pos.astype(np.int32),
                                                         np.zeros(1, np.int32)])).to(self.device)
        return self._o2i

    def local_rows(self, arr: np.ndarray) -> np.ndarray:
        """Rows of a per-vertex host array in this device's row order."""
        return arr

    def exchange_agg(self, which: str, y: torch.Tensor, out: torch.Tensor, width: int, **kw) -> None:
        """``agg_sum`` over the ``which`` ("fwd" / "bwd") CSR reading ``y``,
        after its halo rows are filled (sharded: overlapped, see below)."""
        ops.agg_sum(getattr(self, which), y, out, width, **kw)

    def gat_pull(self):
        """(spec, edge_perm) of GAT's transposed pull: the graph's out-CSR
        with each out-edge's position in the forward in-CSR."""
        return self.bwd, self.out_to_in_perm()

    def reverse_add(self, buf: torch.Tensor, width: int) -> None:
        """Add halo rows' partial sums into their owners' rows (no-op on one device)."""
        return None

    def scale(self, name: str | None) -> torch.Tensor | None:
        if name is None:
            return None
        t = self._scales.get(name)
        if t is None:
            t = torch.from_numpy(_degree_scale(name, self._deg).astype(np.float32)).to(self.device)
            self._scales[name] = t
        return t

    def partition(self, q: int) -> "DevicePartition":
        part = self._partitions.get(q)
        if part is None:
            part = DevicePartition.from_plan(self.plan, q, self.device)
            self._partitions[q] = part
        return part


class ShardDeviceGraph(DeviceGraph):
    """One rank's shard (distributed.ShardPlan) on its GPU: local rows are
    [owned | halo]; aggregations run over the owned rows only and read halo
    rows filled by ``exchange`` (one all-to-all per call)."""

    def __init__(self, graph, plan, shard, comm, device):
        self.device = device
        self.num_vertices = plan.num_vertices
        self.num_edges = int(shard.in_ptr[-1])
        self.num_partitions = plan.num_partitions
        self.plan = plan
        self.shard = shard
        self.comm = comm
        self.n_own, self.n_local = shard.n_own, shard.n_local
        self.fwd = AggSpec.build(shard.in_ptr, shard.in_idx, device)
        self.bwd = AggSpec.build(shard.out_ptr, shard.out_idx, device)
        self._deg = plan.flat.in_degree[shard.local_ids].astype(np.float64)
        self._scales = {}
        self._partitions = {}
        self.send_idx = torch.from_numpy(shard.send_idx.astype(np.int32)).to(device)
        self.n_send = int(shard.send_idx.size)
        self.n_recv = int(shard.halo.size)
        self.recv_ident = torch.arange(self.n_recv, dtype=torch.int32, device=device)
        self._bufs: dict = {}

    def _buf(self, key: str, rows: int, ld: int) -> torch.Tensor:
        t = self._bufs.get(key)
        if t is None or t.numel() < max(rows * ld, 1):
            # zeroed once: padding columns of packed rows stay 0 (a halo row
            # received in place carries the sender's padding into the block)
            t = torch.zeros(max(rows * ld, 1), dtype=torch.float32, device=self.device)
            self._bufs[key] = t
        return t[: rows * ld].view(rows, ld)

    def exchange(self, buf: torch.Tensor, width: int) -> None:
        self._exchange_finish(self._exchange_start(buf, width), buf, width)

    def _exchange_start(self, buf: torch.Tensor, width: int):
        """Pack the rows other ranks need and start the all-to-all.  When
        ``buf``'s rows are exactly ld(width) wide the halo block
        ``buf[n_own:]`` is contiguous and receives the rows in place;
        otherwise they land in a scratch buffer and are unpacked."""
        ld = ld_of(width)
        send = self._buf("send", self.n_send, ld)
        direct = buf.dim() == 2 and buf.shape[1] == ld and buf.stride(0) == ld \
            and buf.stride(1) == 1
        recv = buf[self.n_own:self.n_own + self.n_recv] if direct else \
            self._buf("recv", self.n_recv, ld)
        if self.n_send:
            ops.gather_rows(buf, self.send_idx, send, width)
        work = self.comm.all_to_all_rows(recv, send, self.shard.recv_counts,
                                         self.shard.send_counts, async_op=True)
        return work, direct

    def _exchange_finish(self, started, buf: torch.Tensor, width: int) -> None:
        """Wait for the all-to-all (a stream wait under NCCL) and, when the
        rows went to the scratch buffer, unpack them into the halo block."""
        work, direct = started
        if work is not None:
            work.wait()
        if self.n_recv and not direct:
            recv = self._buf("recv", self.n_recv, ld_of(width))
            ops.gather_rows(recv, self.recv_ident, buf[self.n_own:], width)

    def local_rows(self, arr: np.ndarray) -> np.ndarray:
        return arr[self.shard.local_ids]

    def _split(self, which: str):
        """(interior, boundary) row subsets of the fwd / bwd CSR: interior
        rows read owned rows only, so they run while the halo is in flight."""
        key = "_split_" + which
        sp = getattr(self, key, None)
        if sp is None:
            sh = self.shard
            ptr, idx = (sh.in_ptr, sh.in_idx) if which == "fwd" else (sh.out_ptr, sh.out_idx)
            n = ptr.size - 1
            rows_of = np.repeat(np.arange(n, dtype=np.int64), np.diff(ptr))
            halo = np.bincount(rows_of[idx >= self.n_own], minlength=n) > 0
            sp = []
            deg = np.diff(ptr)
            for rows in (np.flatnonzero(~halo), np.flatnonzero(halo)):
                if _degree_sched():                       # descending degree, stable
                    rows = rows[np.argsort(-deg[rows], kind="stable")]
                p2, i2 = _csr_rows(ptr, idx, rows)
                sp.append(AggSpec.build(p2, i2, self.device, out_idx=rows.astype(np.int32)))
            sp = tuple(sp)
            setattr(self, key, sp)
        return sp

    def exchange_agg(self, which: str, y: torch.Tensor, out: torch.Tensor, width: int, **kw) -> None:
        """Halo exchange of ``y`` overlapped with the aggregation of the
        interior rows (NCCL: the all-to-all runs on its own stream while the
        interior rows aggregate; gloo: synchronous), then the boundary rows."""
        interior, boundary = self._split(which)
        work = self._exchange_start(y, width)
        if interior.n_rows:
            ops.agg_sum(interior, y, out, width, **kw)
        self._exchange_finish(work, y, width)
        if boundary.n_rows:
            ops.agg_sum(boundary, y, out, width, **kw)

    def gat_pull(self):
        if getattr(self, "_gat_pull", None) is None:
            ptr, idx, perm = self.shard.local_transpose()
            self._gat_pull = (AggSpec.build(ptr, idx, self.device),
                              torch.from_numpy(np.concatenate([perm, [0]]).astype(np.int32)).to(self.device))
        return self._gat_pull

    def reverse_add(self, buf: torch.Tensor, width: int) -> None:
        """The forward exchange reversed: halo rows of ``buf`` (partial sums
        for rows other ranks own) go back to their owners, which add them
        into the rows they sent, one source rank after another (fixed
        order: deterministic for a given world size)."""
        ld = ld_of(width)
        send = self._buf("rsend", self.n_recv, ld)
        recv = self._buf("rrecv", self.n_send, ld)
        if self.n_recv:
            ops.gather_rows(buf[self.n_own:], self.recv_ident, send, width)
        self.comm.all_to_all_rows(recv, send, self.shard.send_counts, self.shard.recv_counts)
        r0 = 0
        for cnt in (int(x) for x in self.shard.send_counts):
            if cnt:
                ops.scatter_add_rows(recv[r0:r0 + cnt], self.send_idx[r0:r0 + cnt], buf, width)
            r0 += cnt

    def partition(self, q: int):
        raise NotImplementedError("per-partition operators run on one device")


class DevicePartition:
    """One partition's local topology on the device (plan.py:21-48) plus its
    CSC-by-gather-row transpose for the local backward pull."""

    def __init__(self, pid, targets, gather_map, tgt_ptr, src_pos, self_pos, target_indeg,
                 gather_indeg, device):
        self.pid = pid
        self.dev = device
        self.num_targets = int(len(targets))
        self.num_gather = int(len(gather_map))
        tgt_ptr = np.ascontiguousarray(tgt_ptr, dtype=np.int64)
        src_pos = np.asarray(src_pos, dtype=np.int64)
        self_pos = np.asarray(self_pos, dtype=np.int64)
        self.targets = torch.from_numpy(np.ascontiguousarray(targets, dtype=np.int32)).to(device)
        self.gather_map = torch.from_numpy(np.ascontiguousarray(gather_map, dtype=np.int32)).to(device)
        self.fwd = AggSpec.build(tgt_ptr, src_pos, device, self_idx=self_pos)
        self._csr = (tgt_ptr, src_pos, self_pos)
        self._bwd = None
        self._deg = {"targets": np.asarray(target_indeg, dtype=np.float64),
                     "gather": np.asarray(gather_indeg, dtype=np.float64)}
        self._scales: dict = {}

    @property
    def bwd(self) -> AggSpec:
        """Transposed local aggregation, built on first use (a forward-only
        stage of the SSO manager never needs it): for gather row g, its
        targets in ascending order (np.add.at's edge order, training.py:141),
        self last."""
        if self._bwd is None:
            tgt_ptr, src_pos, self_pos = self._csr
            csc_ptr = np.empty(self.num_gather + 1, dtype=np.int64)
            csc_rows = np.empty(src_pos.size, dtype=np.int32)
            src32 = np.ascontiguousarray(src_pos, dtype=np.int32)
            _lib.check(_lib.lib().grd_csr_transpose(self.num_targets, tgt_ptr.ctypes.data,
                                                    src32.ctypes.data, self.num_gather,
                                                    csc_ptr.ctypes.data, csc_rows.ctypes.data),
                       "csr_transpose")
            self_t = np.full(self.num_gather, -1, dtype=np.int32)
            self_t[self_pos] = np.arange(self.num_targets, dtype=np.int32)
            self._bwd = AggSpec.build(csc_ptr, csc_rows, self.dev, self_idx=self_t)
        return self._bwd

    def gat_specs(self):
        """(fwd, pull, edge_perm) of a GAT layer over this partition, in
        gather-position space: the forward rows are the targets with output /
        self row self_pos[t] (so t_v, the self loop, O and gO all live at the
        target's gather row), the pull's rows are the gather rows with their
        targets' gather rows as neighbours (ascending target), and edge_perm
        maps each pull edge to its forward edge (per-edge attention).  A
        gather row that is not a target gets no self term in the backward:
        its gO row and delta_self entry are zero."""
        if getattr(self, "_gat", None) is None:
            tgt_ptr, src_pos, self_pos = self._csr
            fwd = AggSpec.build(tgt_ptr, src_pos, self.dev, out_idx=self_pos)
            tgt = np.repeat(np.arange(self.num_targets, dtype=np.int64), np.diff(tgt_ptr))
            order = np.argsort(src_pos, kind="stable")
            ptr = np.zeros(self.num_gather + 1, dtype=np.int64)
            np.cumsum(np.bincount(src_pos, minlength=self.num_gather), out=ptr[1:])
            pull = AggSpec.build(ptr, self_pos[tgt[order]], self.dev)
            perm = torch.from_numpy(np.concatenate([order.astype(np.int32), np.zeros(1, np.int32)]))
            self._gat = (fwd, pull, perm.to(self.dev))
        return self._gat

    @classmethod
    def from_topology(cls, topo, device) -> "DevicePartition":
        return cls(topo.partition_id, topo.targets, topo.gather_map, topo.tgt_ptr, topo.src_pos,
                   topo.self_pos, topo.target_indeg, topo.gather_indeg, device)

    @classmethod
    def from_plan(cls, plan, q: int, device) -> "DevicePartition":
        f = plan.flat
        r0, r1 = int(f.part_ptr[q]), int(f.part_ptr[q + 1])
        e0, e1 = int(f.in_ptr[r0]), int(f.in_ptr[r1])
        g0, g1 = int(f.gather_ptr[q]), int(f.gather_ptr[q + 1])
        targets = f.perm[r0:r1]
        gmap = f.gather_map[g0:g1]
        return cls(q, targets, gmap, f.in_ptr[r0:r1 + 1] - f.in_ptr[r0], f.in_src_pos[e0:e1],
                   f.self_pos[r0:r1], f.in_degree[targets], f.in_degree[gmap], device)

    def scale(self, name: str | None, rows: str) -> torch.Tensor | None:
        """Degree scale over the target rows or gather rows of this partition."""
        if name is None:
            return None
        key = (name, rows)
        t = self._scales.get(key)
        if t is None:
            t = torch.from_numpy(_degree_scale(name, self._deg[rows]).astype(np.float32)).to(self.dev)
            self._scales[key] = t
        return t


def _degree_scale(name: str, deg: np.ndarray) -> np.ndarray:
    if name == "inv_deg1":
        return 1.0 / (deg + 1.0)
    if name == "inv_deg":        # GraphSAGE mean over in-neighbours (0 if none)
        out = np.zeros_like(deg)
        np.divide(1.0, deg, out=out, where=deg > 0)
        return out
    if name == "s":
        return 1.0 / np.sqrt(deg + 1.0)
    if name == "s_inv_deg1":
        return 1.0 / (np.sqrt(deg + 1.0) * (deg + 1.0))
    raise KeyError(name)


class _LayerCfg:
    def __init__(self, layer: int, dims: list[int], mode: str, row_normalize: bool, last: bool,
                 heads: int = 1):
        self.layer = layer
        self.d_in, self.d_out = dims[layer], dims[layer + 1]
        self.transform_first = self.d_out <= self.d_in
        self.sym = mode == "symmetric_norm"
        self.sage = mode == "sage_mean"
        self.gat = mode == "gat"
        self.rownorm = row_normalize
        self.last = last
        self.ld_in, self.ld_out = ld_of(self.d_in), ld_of(self.d_out)
        if self.gat:
            self.heads = heads
            self.dh = self.d_out if last else self.d_out // heads
            self.dhp = ld_of(self.dh)
            if not last and self.dhp != self.dh:
                raise ValueError("GAT hidden head width must be a multiple of 4")
            self.hdp = heads * self.dhp
            self.n_ext = self.hdp + 2 * heads        # [P | s | t] columns
            self.ld_ext = ld_of(self.n_ext)

    # scale applied to the upstream gradient before this layer's pull (TF)
    # or after its dgrad GEMM (AF): mean -> 1/(deg+1), sym -> 1/sqrt(deg+1)
    @property
    def pre_scale(self) -> str:
        return "s" if self.sym else "inv_deg1"


class _Weights:
    """fp32 device copies of W_l and dW_l, zero padded to [ld(d_in), ld(d_out)].
    GraphSAGE layers keep [W_root | W_nbr] as [ld(d_in), 2 ld(d_out)] with the
    neighbour block starting at column ld(d_out) (16-byte aligned); layers in
    ``stacked`` keep them stacked along K instead, [W_root ; W_nbr] as
    [2 ld(d_in), ld(d_out)], for the one-GEMM form [X | mean(X)] W."""

    def __init__(self, model, device, stacked=frozenset()):
        self.w = []
        self.dw = []
        self.blocks = 2 if model.kind == "sage" else 1
        self.gat = model.kind == "gat"
        self.stacked = frozenset(stacked) if self.blocks == 2 else frozenset()
        if self.gat:
            self._init_gat(model, device)
            return
        shapes = []
        for l, w in enumerate(model.weights):
            d_in, d_out = w.shape[0], w.shape[1] // self.blocks
            shape = (2 * ld_of(d_in), ld_of(d_out)) if l in self.stacked else \
                (ld_of(d_in), self.blocks * ld_of(d_out))
            self.w.append(torch.zeros(shape, dtype=torch.float32, device=device))
            shapes.append(shape)
        self.dw = self._bucket(shapes, device)
        self.load(model)

    def _bucket(self, shapes, device) -> list[torch.Tensor]:
        """Weight-gradient tensors as views of one flat buffer (``grad_bucket``),
        so a sharded run sums every layer's gradient with one all-reduce."""
        sizes = [a * b for a, b in shapes]
        self.grad_bucket = torch.zeros(sum(sizes), dtype=torch.float32, device=device)
        out, off = [], 0
        for (a, b), n in zip(shapes, sizes):
            out.append(self.grad_bucket[off:off + n].view(a, b))
            off += n
        return out

    # GAT: W per head padded to dhp columns [ld(d_in), H*dhp]; att = [a_src; a_dst]
    # as [2, H, dhp]; the fused transform matrix W_ext [ld(d_in), ld_ext] is
    # rebuilt from them before every use.
    def _init_gat(self, model, device):
        H = model.heads
        self.heads = H
        self.att, self.datt, self.wext, self.dwext, self.shape = [], [], [], [], []
        for l, wp in enumerate(model.weights):
            d_in = wp.shape[0] - 2
            dh = wp.shape[1] // H
            dhp = ld_of(dh)
            n_ext = H * dhp + 2 * H
            self.shape.append((d_in, dh, dhp))
            self.w.append(torch.zeros((ld_of(d_in), H * dhp), dtype=torch.float32, device=device))
            self.dw.append(torch.zeros_like(self.w[-1]))
            self.att.append(torch.zeros((2, H, dhp), dtype=torch.float32, device=device))
            self.datt.append(torch.zeros_like(self.att[-1]))
            self.wext.append(torch.zeros((ld_of(d_in), ld_of(n_ext)), dtype=torch.float32, device=device))
        # the fused [W | W a_src | W a_dst] gradient is what ranks sum
        self.dwext = self._bucket([tuple(t.shape) for t in self.wext], device)
        self.load(model)

    def _gat_load(self, model) -> None:
        for l, wp in enumerate(model.weights):
            d_in, dh, dhp = self.shape[l]
            H = self.heads
            w32 = np.asarray(wp, dtype=np.float32)
            w = np.zeros((d_in, H, dhp), np.float32)
            w[:, :, :dh] = w32[:d_in].reshape(d_in, H, dh)
            self.w[l][:d_in].copy_(torch.from_numpy(w.reshape(d_in, H * dhp)))
            att = np.zeros((2, H, dhp), np.float32)
            att[:, :, :dh] = w32[d_in:].reshape(2, H, dh)
            self.att[l].copy_(torch.from_numpy(att))

    def _gat_export(self, model) -> None:
        ws, gs = [], []
        for l in range(len(self.w)):
            d_in, dh, dhp = self.shape[l]
            H = self.heads
            for src, att, out in ((self.w[l], self.att[l], ws), (self.dw[l], self.datt[l], gs)):
                w = src[:d_in].double().cpu().numpy().reshape(d_in, H, dhp)[:, :, :dh]
                a = att.double().cpu().numpy()[:, :, :dh]
                out.append(np.concatenate([w.reshape(d_in, H * dh), a.reshape(2, H * dh)], axis=0))
        model.weights, model.weight_grads = ws, gs

    def params(self) -> list[torch.Tensor]:
        """Every trained device tensor (what an SGD step modifies)."""
        return self.w + (self.att if self.gat else [])

    def _views(self, t: torch.Tensor, w: np.ndarray, l: int):
        d_in, d_out = w.shape[0], w.shape[1] // self.blocks
        if l in self.stacked:
            li = ld_of(d_in)
            return [(t[b * li: b * li + d_in, :d_out], slice(b * d_out, (b + 1) * d_out))
                    for b in range(self.blocks)]
        ld = ld_of(d_out)
        return [(t[:d_in, b * ld: b * ld + d_out], slice(b * d_out, (b + 1) * d_out))
                for b in range(self.blocks)]

    def load(self, model) -> None:
        if self.gat:
            self._gat_load(model)
            return
        for l, (t, w) in enumerate(zip(self.w, model.weights)):
            w32 = torch.from_numpy(np.asarray(w, dtype=np.float32))
            for view, cols in self._views(t, w, l):
                view.copy_(w32[:, cols])

    def export(self, model) -> None:
        if self.gat:
            self._gat_export(model)
            return

        def host(tensors):
            out = []
            for l, (t, w) in enumerate(zip(tensors, model.weights)):
                out.append(np.concatenate([v.double().cpu().numpy() for v, _ in self._views(t, w, l)],
                                          axis=1))
            return out
        model.weights, model.weight_grads = host(self.w), host(self.dw)


class _EngineBase:
    _fuse_sage_root = False

    def __init__(self, dg: DeviceGraph, model, features: torch.Tensor, labels: np.ndarray,
                 train_mask: np.ndarray, mask_count: int | None = None):
        self.dg = dg
        dev = dg.device
        self.device = dev
        self.V = dg.n_own            # rows computed here
        self.NL = dg.n_local         # rows held (owned + halo)
        self.comm = dg.comm
        self.dims = model.dims
        self.L = model.num_layers
        self.mode = model.aggregation_mode
        self.model = model
        self.cfg = [_LayerCfg(l, self.dims, self.mode, model.row_normalize, l == self.L - 1,
                              model.heads) for l in range(self.L)]
        # GraphSAGE aggregate-first layer 0 over a features buffer with room
        # for mean(X) beside X: out = [X | mean(X)] [W_root ; W_nbr], one GEMM
        # (and one weight-gradient GEMM) instead of two with a read-back of out
        c0 = self.cfg[0]
        self.xn = None
        if (self._fuse_sage_root and c0.sage and not c0.transform_first
                and features.stride(0) >= 2 * c0.ld_in):
            self.xn = torch.as_strided(features, (dg.n_local, 2 * c0.ld_in), (features.stride(0), 1))
        self.wts = _Weights(model, dev, stacked={0} if self.xn is not None else ())
        self.acts = [features] + [ops.zeros_rows(self.NL, d, dev) for d in self.dims[1:]]
        self.labels = torch.from_numpy(np.asarray(labels, dtype=np.int32)).to(dev)
        self.mask = torch.from_numpy(np.asarray(train_mask, dtype=np.uint8)).to(dev)
        self.mask_count = int(np.count_nonzero(train_mask)) if mask_count is None else int(mask_count)
        if self.mask_count == 0:
            raise ValueError("loss mask selects no vertices")
        self.stats = torch.zeros(4, dtype=torch.float64, device=dev)
        self.partials = ops.loss_partials(self.V, dev)
        self.maxw = max(self.dims)
        self.dropout_rate = model.dropout_rate
        self.dropout_seed = model.dropout_seed
        self.dmask = [None] * self.L
        self.xd = ops.zeros_rows(self.NL, self.maxw, dev) if self.dropout_rate > 0 else None
        if self.comm is not None and (self.dropout_rate > 0 or model.row_normalize):
            raise NotImplementedError("dropout / row_normalize run on one device")

    def set_dropout(self, epoch: int) -> None:
        if self.dropout_rate == 0.0:
            return
        for l in range(self.L):
            m = dropout_mask(self.dropout_rate, self.dropout_seed, epoch, l, (self.V, self.dims[l]))
            t = ops.zeros_rows(self.V, self.dims[l], self.device)
            t[:, : self.dims[l]] = torch.from_numpy(m.astype(np.float32)).to(self.device)
            self.dmask[l] = t

    def layer_input(self, l: int) -> torch.Tensor:
        """A_l, or A_l * M_l under dropout (recomputed on every use)."""
        x = self.acts[l]
        if self.dmask[l] is None:
            return x
        ops.mul_rows(x, self.dmask[l], self.xd, self.V, self.dims[l])
        return self.xd


class LayerwiseEngine(_EngineBase):
    """Fused layer-wide epoch over an HBM-resident graph (module docstring)."""

    _fuse_sage_root = True

    def __init__(self, dg, model, features, labels, train_mask, mask_count=None):
        super().__init__(dg, model, features, labels, train_mask, mask_count)
        dev = self.device
        wide = 2 * ld_of(self.maxw) if model.kind == "sage" else self.maxw
        if model.kind == "gat":
            wide = max([self.maxw] + [c.ld_ext for c in self.cfg])
            self._gat_buffers(dg, model)
        self.t1 = ops.zeros_rows(self.NL, wide, dev)
        self.g = ops.zeros_rows(self.NL, wide, dev)
        self.h = ops.zeros_rows(self.NL, wide, dev)
        if model.kind == "sage":
            self.t2 = ops.zeros_rows(self.NL, self.maxw, dev)
        elif model.kind != "gat":
            self.t2 = None
        # GraphSAGE, transform-first last layer: the loss also writes its
        # gradient pre-scaled by 1/deg, the source scale of the pull that
        # follows (once per row instead of once per edge)
        cl = self.cfg[-1]
        self.g2 = ops.zeros_rows(self.NL, cl.d_out, dev) if (cl.sage and cl.transform_first) else None
        # aggregate-first GCN layers: the forward's normalised aggregate N is
        # kept for the backward's dW = N^T gp when it fits, instead of the
        # reference's regather (GRD_KEEP_AGG=0 regathers).  Decided after
        # every engine buffer above exists, so the free-HBM margin is what
        # the lazily allocated scratch really has left.
        self.keep_on = os.environ.get("GRD_KEEP_AGG", "1") != "0"
        self.n_kept = {}
        if self.keep_on:
            hidden = [l for l, c in enumerate(self.cfg)
                      if not (c.transform_first or c.sage or c.gat or c.rownorm or c.last)]
            need = sum(self.NL * ld_of(self.cfg[l].d_in) * 4 for l in hidden)
            if hidden and self._keep_fits(need):
                self.n_kept = {l: ops.zeros_rows(self.NL, self.cfg[l].d_in, dev) for l in hidden}
        if model.kind == "gat":
            self._alloc_gat_kept(model)
        # one device: SGD fused into the weight-gradient reduction; sharded:
        # local weight gradients are all-reduced first, SGD at epoch end
        self.defer_sgd = self.comm is not None
        self._gh = (self.g, self.h)

    # ---------------------------------------------------------- forward --
    def _forward_layer(self, l: int, x: torch.Tensor, out: torch.Tensor, relu: bool) -> None:
        c, dg = self.cfg[l], self.dg
        W = self.wts.w[l]
        s = dg.scale("s") if c.sym else None
        if c.transform_first:
            ops.gemm(x, W, self.t1, self.V, c.d_out, c.d_in, row_scale=s)
            # halo rows of P = X W, overlapped with the interior rows
            dg.exchange_agg("fwd", self.t1, out, c.d_out, post_div_deg=not c.sym, post_scale=s, relu=relu)
        else:
            n = self.n_kept.get(l, self.t1)
            self._input_agg(l, x, n, c.d_in, src_scale=s, post_div_deg=not c.sym, post_scale=s)
            ops.gemm(n, W, out, self.V, c.d_out, c.d_in, relu_out=relu)

    def _input_agg(self, l: int, x: torch.Tensor, out: torch.Tensor, width: int, **kw) -> None:
        """Aggregate-first layers read the layer input's halo rows (the
        features' halo is filled once at upload)."""
        if l > 0:
            self.dg.exchange_agg("fwd", x, out, width, **kw)
        else:
            ops.agg_sum(self.dg.fwd, x, out, width, **kw)

    def _w(self, W):
        """SGD target of a weight-gradient call (None: deferred past the all-reduce)."""
        return None if self.defer_sgd else W

    # ------------------------------------------------ GraphSAGE-mean layer --
    # out = act(X W_root + mean_in(X) W_nbr); weights [W_root | W_nbr].
    def _forward_sage(self, l: int, x: torch.Tensor, out: torch.Tensor, relu: bool) -> None:
        c, dg = self.cfg[l], self.dg
        W = self.wts.w[l]
        if c.transform_first:
            # Y = X [W_root | W_nbr] (one GEMM, its two column halves written to
            # two dense planes), out = Y_root + mean_in(Y_nbr): the gathered
            # Y_nbr rows are not interleaved with Y_root (narrow rows: whole
            # sectors instead of half-used ones)
            lo = c.ld_out
            plane = self.t1.view(-1)
            yr = plane[: self.NL * lo].view(self.NL, lo)
            yn = plane[self.NL * lo: 2 * self.NL * lo].view(self.NL, lo)
            ops.gemm(x, W, yr, self.V, 2 * lo, c.d_in, c2=yn, split=lo)
            dg.exchange_agg("fwd", yn, out, c.d_out, post_div_deg=2, no_self=True,
                            add_y=yr, relu=relu)                    # halo rows of X W_nbr
        elif l == 0 and self.xn is not None:
            # N = mean_in(X) beside X, out = [X | N] [W_root ; W_nbr]
            n = self.xn[:, c.ld_in: 2 * c.ld_in]
            self._input_agg(l, x, n, c.d_in, post_div_deg=2, no_self=True)
            ops.gemm(self.xn, W, out, self.V, c.d_out, 2 * c.ld_in, relu_out=relu)
        else:
            # N = mean_in(X), out = X W_root + N W_nbr
            n = self.t1[:, : c.ld_in]
            self._input_agg(l, x, n, c.d_in, post_div_deg=2, no_self=True)
            ops.gemm(x, W[:, : c.ld_out], out, self.V, c.d_out, c.d_in)
            ops.gemm(n, W[:, c.ld_out:], out, self.V, c.d_out, c.d_in, accumulate=True, relu_out=relu)

    def _backward_sage(self, l: int, x: torch.Tensor, lr: float) -> None:
        """g holds gp = dL/dpre of layer l (ReLU mask applied by the producer);
        leaves dL/dA_l (masked for layer l-1) in h, then swaps g and h."""
        c, dg = self.cfg[l], self.dg
        W, dW = self.wts.w[l], self.wts.dw[l]
        inv_deg = dg.scale("inv_deg")
        ref, _ = self._consumer_epilogue(l - 1) if l > 0 else (None, None)
        if c.transform_first:
            # [gp | H_nbr] with H_nbr = mean_in^T gp (pull over out-edges, 1/deg_v per edge)
            gcat = self.g[:, : 2 * c.ld_out]
            if c.last and getattr(self, "g2", None) is not None:
                # the loss wrote gp / deg as well: an unscaled pull
                dg.exchange_agg("bwd", self.g2, gcat[:, c.ld_out:], c.d_out, no_self=True)
            else:
                dg.exchange_agg("bwd", gcat[:, : c.ld_out], gcat[:, c.ld_out:], c.d_out, src_scale=inv_deg,
                                no_self=True)                      # halo rows of gp
            if l > 0:
                ops.gemm(gcat, W, self.h, self.V, c.d_in, 2 * c.ld_out, trans_b=True, relu_ref=ref)
            ops.wgrad_sgd(x, gcat, dW, c.d_in, 2 * c.ld_out, self.V, w=self._w(W), lr=lr)
        elif l == 0 and self.xn is not None:
            # N = mean_in(X) is still beside X in the features buffer (nothing
            # else writes those columns): no regather
            gp = self.g[:, : c.ld_out]
            ops.wgrad_sgd(self.xn, gp, dW, 2 * c.ld_in, c.d_out, self.V, w=self._w(W), lr=lr)
        else:
            gp = self.g[:, : c.ld_out]
            n = self.t1[:, : c.ld_in]
            ops.agg_sum(dg.fwd, x, n, c.d_in, post_div_deg=2, no_self=True)     # regather
            if l > 0:
                gn = self.t2[:, : c.ld_in]
                ops.gemm(gp, W[:, c.ld_out:], gn, self.V, c.d_in, c.d_out, trans_b=True)
                dg.exchange_agg("bwd", gn, self.h, c.d_in, src_scale=inv_deg, no_self=True)
                ops.gemm(gp, W[:, : c.ld_out], self.h, self.V, c.d_in, c.d_out, trans_b=True,
                         accumulate=True, relu_ref=ref)
            ops.wgrad_sgd(x, gp, dW[:, : c.ld_out], c.d_in, c.d_out, self.V, w=self._w(W[:, : c.ld_out]),
                          lr=lr)
            ops.wgrad_sgd(n, gp, dW[:, c.ld_out:], c.d_in, c.d_out, self.V, w=self._w(W[:, c.ld_out:]),
                          lr=lr)
        self.g, self.h = self.h, self.g

    # ---------------------------------------------------------------- GAT --
    def _gat_buffers(self, dg, model) -> None:
        dev = self.device
        H = model.heads
        E = dg.fwd.nnz
        self.alpha = torch.zeros(max(E * H, 1), dtype=torch.float32, device=dev)
        self.delta = torch.zeros_like(self.alpha)
        self.alpha_self = torch.zeros(self.NL * H, dtype=torch.float32, device=dev)
        self.delta_self = torch.zeros_like(self.alpha_self)
        self.pull, self.edge_perm = dg.gat_pull()
        # the transposed pull reads alpha in its own edge order: one permuting
        # row gather per layer (16-byte rows at 4 heads) instead of a
        # dependent edge_perm load per edge inside the pull (GRD_GAT_ALPHA_T=0
        # keeps the permuted addressing)
        self.alpha_t = None
        if H % 4 == 0 and self.pull.nnz > 0 and E > 0 and os.environ.get("GRD_GAT_ALPHA_T", "1") != "0":
            self.alpha_t = torch.zeros(self.pull.nnz * H, dtype=torch.float32, device=dev)
        # compact [s | t] score table (32 B per vertex at 4 heads): the
        # edge-softmax's per-edge score gathers stay in L2
        self.st = ops.zeros_rows(self.NL, 2 * H, dev)
        # t2: the last layer's per-head aggregate O (kept for the backward's
        # gO.O term); t3: its per-head upstream gradient
        hdp = self.cfg[-1].hdp
        self.t2 = ops.zeros_rows(self.NL, hdp, dev)
        self.t3 = ops.zeros_rows(self.NL, hdp, dev)
        self.gat_kept = {}
        self.gat_keep_on = os.environ.get("GRD_GAT_KEEP", "1") != "0"
        # fused backward over the pull (GRD_GAT_FUSED_BWD=0: the separate
        # edge backward, pull and source-score kernels)
        self.gat_fused = os.environ.get("GRD_GAT_FUSED_BWD", "1") != "0"
        self.cdot = torch.zeros(max(self.NL * H, 1), dtype=torch.float32, device=dev)

    def _keep_fits(self, need: int) -> bool:
        """Whether `need` more bytes of kept forward state leave a margin of
        free HBM (max(4 GB, 10 % of the device)) for the lazily allocated
        scratch (heavy-row partials, exchange buffers, graph capture)."""
        if not str(self.device).startswith("cuda"):
            return False
        free, total = torch.cuda.mem_get_info(torch.device(self.device))
        fits = need + max(4 << 30, total // 10) < free
        if self.comm is not None:
            # the kept and the regathering backward issue different
            # exchanges: every rank must make the same choice (all keep or
            # none), or the all-to-alls pair up wrongly
            flag = torch.tensor([1.0 if fits else 0.0], dtype=torch.float32, device=self.device)
            self.comm.all_reduce_min(flag)
            fits = bool(flag.item() > 0.5)
        return fits

    def _alloc_gat_kept(self, model) -> None:
        """Hidden layers' [P | s | t] and attention kept from the forward when
        they fit (a few GB at the products shape): the backward then skips the
        regather (transform GEMM + edge softmax).  The last layer's are still
        in t1 / alpha when its backward runs.  GRD_GAT_KEEP=0, or too little
        free HBM, recomputes them as the reference's regather does."""
        if not self.gat_keep_on:
            return
        H = model.heads
        E = self.dg.fwd.nnz
        hidden = [l for l, c in enumerate(self.cfg) if c.gat and not c.last]
        need = sum(self.NL * ops.ld_of(self.cfg[l].ld_ext) * 4 + (max(E, 1) + self.NL) * H * 4
                   for l in hidden)
        if hidden and self._keep_fits(need):
            for l in hidden:
                self.gat_kept[l] = (ops.zeros_rows(self.NL, self.cfg[l].ld_ext, self.device),
                                    torch.zeros_like(self.alpha), torch.zeros_like(self.alpha_self))

    def _gat_bufs(self, l: int):
        """(P_ext, alpha, alpha_self) buffers of layer l: kept per layer, or
        the shared ones (t1 / alpha) that the backward recomputes."""
        kept = self.gat_kept.get(l)
        if kept is not None:
            return kept[0][:, : self.cfg[l].ld_ext], kept[1], kept[2]
        return self.t1[:, : self.cfg[l].ld_ext], self.alpha, self.alpha_self

    def _gat_transform(self, l: int, x: torch.Tensor):
        """P_ext = X [W | W a_src | W a_dst] and the attention (forward, and
        recomputed in backward when not kept: the regather)."""
        c, dg = self.cfg[l], self.dg
        wt = self.wts
        d_in, dh, dhp = wt.shape[l]
        pext, alpha, alpha_self = self._gat_bufs(l)
        ops.gat_build_wext(wt.w[l], wt.att[l], d_in, c.heads, dh, dhp, wt.wext[l])
        ops.gemm(x, wt.wext[l], pext, self.V, c.n_ext, c.d_in)
        dg.exchange(pext, c.n_ext)                # halo rows of [P | s | t]
        ops.gat_pack_scores(pext, self.NL, c.heads, c.dhp, self.st)
        ops.gat_softmax(dg.fwd, pext, c.heads, c.dhp, alpha, alpha_self, st=self.st)
        return pext, alpha, alpha_self

    def _forward_gat(self, l: int, x: torch.Tensor, out: torch.Tensor) -> None:
        c, dg = self.cfg[l], self.dg
        pext, alpha, alpha_self = self._gat_transform(l, x)
        dst = self.t2[:, : c.hdp] if c.last else out
        ops.agg_sum(dg.fwd, pext[:, : c.hdp], dst, c.hdp, edge_w=alpha, self_w=alpha_self,
                    heads=c.heads, head_ld=c.dhp, relu=not c.last)
        if c.last:
            ops.head_mean(dst, self.V, c.heads, c.dh, c.dhp, out)

    def _backward_gat(self, l: int, x: torch.Tensor, lr: float) -> None:
        c, dg = self.cfg[l], self.dg
        wt = self.wts
        d_in, dh, dhp = wt.shape[l]
        if c.last:
            go, o_fwd = self.t3[:, : c.hdp], self.t2[:, : c.hdp]
            ops.head_mean(self.g, self.V, c.heads, c.dh, c.dhp, go, backward=True)
        else:
            # ReLU mask applied by the producer, so gO.relu(O) = gO.O
            go, o_fwd = self.g[:, : c.hdp], self.acts[l + 1]
        if l in self.gat_kept or (c.last and self.gat_keep_on):
            # kept from the forward (the last layer's still sit in t1 / alpha,
            # and wext[l] is the forward's)
            pext, alpha, alpha_self = self._gat_bufs(l)
        else:
            pext, alpha, alpha_self = self._gat_transform(l, x)
        gext = self.h[:, : c.ld_ext]
        if self.gat_fused:
            self._gat_fused_bwd(l, pext, alpha, alpha_self, go, o_fwd, gext)
        else:
            self._gat_unfused_bwd(l, pext, alpha, alpha_self, go, o_fwd, gext)
        dg.reverse_add(gext, c.hdp + c.heads)
        ops.wgrad_sgd(x, gext, wt.dwext[l], c.d_in, c.n_ext, self.V)
        if l > 0:
            ref, _ = self._consumer_epilogue(l - 1)
            ops.gemm(gext, wt.wext[l], self.g, self.V, c.d_in, c.n_ext, trans_b=True, relu_ref=ref)
        if not self.defer_sgd:
            ops.gat_param_grads(wt.dwext[l], wt.w[l], wt.att[l], d_in, c.heads, dh, dhp, wt.dw[l],
                                wt.datt[l], lr)

    def _gat_alpha_pull_order(self, alpha, c):
        """Attention permuted into the pull's edge order (None: addressed per edge)."""
        if self.alpha_t is None:
            return None
        ne = self.pull.nnz
        ops.gather_rows(alpha.view(-1, c.heads), self.edge_perm[:ne], self.alpha_t.view(ne, c.heads),
                        c.heads)
        return self.alpha_t

    def _gat_fused_bwd(self, l, pext, alpha, alpha_self, go, o_fwd, gext) -> None:
        """c = gO.O per target; one pass over the pull (u -> v) gathering gO_v
        once per edge for dP_u, ds_u and the edge score gradients; dt_v summed
        over the forward CSR."""
        c, dg = self.cfg[l], self.dg
        if self.NL > self.V:
            go[self.V:].zero_()    # halo rows: no self term, no stale gradient
        ops.gat_row_dots(go, o_fwd, self.NL, c.heads, c.dhp, self.cdot)
        ops.gat_pack_scores(pext, self.NL, c.heads, c.dhp, self.st)   # this layer's t_v
        alpha_t = self._gat_alpha_pull_order(alpha, c)
        ops.gat_pull_bwd(self.pull, pext, c.heads, c.dhp, self.edge_perm, alpha, alpha_self, go,
                         self.cdot, self.delta, self.delta_self, gext, alpha_t=alpha_t, st=self.st)
        ops.gat_dst_grad(dg.fwd, c.heads, c.dhp, self.delta, self.delta_self, gext)

    def _gat_unfused_bwd(self, l, pext, alpha, alpha_self, go, o_fwd, gext) -> None:
        c, dg = self.cfg[l], self.dg
        ops.gat_softmax_bwd(dg.fwd, pext, c.heads, c.dhp, alpha, alpha_self, go, o_fwd,
                            self.delta, self.delta_self, gext)   # s_u beside the gathered P_u row
        if self.NL > self.V:
            go[self.V:].zero_()    # halo rows: no self term, no stale gradient
        # dP_u = sum_v alpha_uv gO_v and ds_u = sum_v delta_uv over u's out-edges
        # (sharded: owned targets only; halo rows are partials for their owners)
        alpha_t = self._gat_alpha_pull_order(alpha, c)
        if alpha_t is not None:
            ops.agg_sum(self.pull, go, gext[:, : c.hdp], c.hdp, edge_w=alpha_t,
                        self_w=alpha_self, heads=c.heads, head_ld=c.dhp)
        else:
            ops.agg_sum(self.pull, go, gext[:, : c.hdp], c.hdp, edge_w=alpha,
                        edge_w_perm=self.edge_perm, self_w=alpha_self, heads=c.heads, head_ld=c.dhp)
        ops.gat_src_grad(self.pull, c.heads, c.dhp, self.edge_perm, self.delta, self.delta_self, gext)

    def forward(self) -> None:
        for l, c in enumerate(self.cfg):
            x = self.layer_input(l)
            out = self.acts[l + 1]
            if c.sage:
                self._forward_sage(l, x, out, relu=not c.last)
                continue
            if c.gat:
                self._forward_gat(l, x, out)
                continue
            self._forward_layer(l, x, out, relu=not c.last and not c.rownorm)
            if c.rownorm:
                ops.rownorm_fwd(out, out, self.V, c.d_out, relu=not c.last)

    # --------------------------------------------------------- backward --
    def _consumer_epilogue(self, l: int):
        """(relu_ref, row_scale) the producer of dA_{l+1} applies for layer l."""
        c = self.cfg[l]
        if c.rownorm:
            return None, None
        ref = None if c.last else self.acts[l + 1]
        scale = self.dg.scale(c.pre_scale) if c.transform_first and not (c.sage or c.gat) else None
        return ref, scale

    def loss(self) -> None:
        c = self.cfg[-1]
        _, scale = self._consumer_epilogue(self.L - 1)
        extra = {} if getattr(self, "g2", None) is None else dict(grad2=self.g2,
                                                                   grad2_scale=self.dg.scale("inv_deg"))
        ops.softmax_xent(self.acts[-1], self.V, c.d_out, self.labels, self.mask, self.mask_count,
                         self.g, self.stats, self.partials, grad_scale=scale, **extra)
        if self.comm is not None:
            self.comm.all_reduce_sum(self.stats)   # {loss, acc, sums}: partial / global count

    def backward(self, lr: float) -> None:
        dg = self.dg
        for l in reversed(range(self.L)):
            c = self.cfg[l]
            W, dW = self.wts.w[l], self.wts.dw[l]
            x = self.layer_input(l)
            if c.sage:
                self._backward_sage(l, x, lr)
                continue
            if c.gat:
                self._backward_gat(l, x, lr)
                continue
            s = dg.scale("s") if c.sym else None
            have_n = False
            if c.rownorm:
                # regather + recompute pre-activation, then the row-norm backward
                if c.transform_first:
                    ops.gemm(x, W, self.t1, self.V, c.d_out, c.d_in, row_scale=s)
                    ops.agg_sum(dg.fwd, self.t1, self.h, c.d_out, post_div_deg=not c.sym, post_scale=s)
                else:
                    ops.agg_sum(dg.fwd, x, self.t1, c.d_in, src_scale=s, post_div_deg=not c.sym,
                                post_scale=s)
                    ops.gemm(self.t1, W, self.h, self.V, c.d_out, c.d_in)
                    have_n = True
                ops.rownorm_bwd(self.h, self.g, self.g, self.V, c.d_out,
                                a_out=None if c.last else self.acts[l + 1],
                                row_scale=dg.scale(c.pre_scale) if c.transform_first else None)
            prev = self._consumer_epilogue(l - 1) if l > 0 else (None, None)
            dmask = self.dmask[l]
            if c.transform_first:
                # H = A_hat^T (gp * pre_scale)
                dg.exchange_agg("bwd", self.g, self.h, c.d_out, post_scale=s)
                if l > 0:
                    ops.gemm(self.h, W, self.g, self.V, c.d_in, c.d_out, trans_b=True,
                             row_scale=prev[1], elem_mul=dmask, relu_ref=prev[0])
                ops.wgrad_sgd(x, self.h, dW, c.d_in, c.d_out, self.V, w=self._w(W), lr=lr)
            else:
                n = self.n_kept.get(l, self.t1)
                # the forward's aggregate is kept (hidden layers, when it fits)
                # or still in t1 (the last layer: only the loss ran since)
                kept = l in self.n_kept or (c.last and self.keep_on)
                if not have_n and not kept:   # regather: recompute the normalised aggregate
                    ops.agg_sum(dg.fwd, x, n, c.d_in, src_scale=s, post_div_deg=not c.sym,
                                post_scale=s)
                ops.gemm(self.g, W, self.h, self.V, c.d_in, c.d_out, trans_b=True,
                         row_scale=dg.scale(c.pre_scale))
                ops.wgrad_sgd(n, self.g, dW, c.d_in, c.d_out, self.V, w=self._w(W), lr=lr)
                if l > 0:
                    post = self._combine(s is not None, prev[1])
                    dg.exchange_agg("bwd", self.h, self.g, c.d_in, post_scale=post,
                                    mask_ref=None if dmask is not None else prev[0])
                    if dmask is not None:
                        ops.mul_rows(self.g, dmask, self.g, self.V, c.d_in)
                        if prev[0] is not None:
                            ops.mask_scale_rows(self.g, self.g, self.V, c.d_in, ref=prev[0])

    def _combine(self, sym: bool, consumer_scale) -> torch.Tensor | None:
        if consumer_scale is None:
            return self.dg.scale("s") if sym else None
        if not sym:
            return consumer_scale
        # s * (consumer pre-scale): s*s = 1/(deg+1) (mean consumer is impossible
        # here: one model has one mode), so the consumer's scale is s.
        return self.dg.scale("inv_deg1")

    def sgd_after_allreduce(self, lr: float) -> None:
        """Sharded runs: sum the local weight gradients over ranks, then the
        replicated SGD step (training.py:343,352-354)."""
        wt = self.wts
        self.comm.all_reduce_sum(wt.grad_bucket)     # every layer in one all-reduce
        if wt.gat:
            for l, c in enumerate(self.cfg):
                d_in, dh, dhp = wt.shape[l]
                ops.gat_param_grads(wt.dwext[l], wt.w[l], wt.att[l], d_in, c.heads, dh, dhp,
                                    wt.dw[l], wt.datt[l], lr)
            return
        for W, dW in zip(self.wts.w, self.wts.dw):
            ops.wgrad_sgd(W, W, dW, dW.shape[0], dW.shape[1], 0, accumulate=True, w=W, lr=lr)

    def epoch(self, lr: float) -> None:
        self.g, self.h = self._gh    # canonical buffer roles (layers may swap them)
        self.forward()
        self.loss()
        self.backward(lr)
        if self.defer_sgd:
            self.sgd_after_allreduce(lr)


class LayerOps:
    """Per-(layer, partition) operators on device tensors (training.py:72-143):
    forward of one partition from its gathered rows GA_p and the
    regather-based backward returning (grad_GA, grad_W)."""

    def __init__(self, model, device, weights: "_Weights | None" = None):
        self.device = device
        self.dims = model.dims
        self.L = model.num_layers
        self.cfg = [_LayerCfg(l, self.dims, model.aggregation_mode, model.row_normalize,
                              l == self.L - 1, model.heads) for l in range(self.L)]
        if model.kind == "gat" and model.row_normalize:
            raise NotImplementedError("GAT layers have no row normalisation")
        self.wts = weights if weights is not None else _Weights(model, device)

    # ------------------------------------------ weight-gradient plumbing --
    def grad_sink(self, l: int) -> torch.Tensor:
        """Where a layer's per-partition weight gradients are summed: dW, or
        GAT's fused dW_ext (linear in the partition sums, converted once)."""
        return self.wts.dwext[l] if self.wts.gat else self.wts.dw[l]

    def sgd(self, lr: float) -> None:
        """W -= lr dW for every layer (GAT: dW, datt from dW_ext first)."""
        wt = self.wts
        for l in range(self.L):
            if wt.gat:
                c = self.cfg[l]
                d_in, dh, dhp = wt.shape[l]
                ops.gat_param_grads(wt.dwext[l], wt.w[l], wt.att[l], d_in, c.heads, dh, dhp,
                                    wt.dw[l], wt.datt[l], lr)
            else:
                w, dw = wt.w[l], wt.dw[l]
                ops.wgrad_sgd(w, w, dw, dw.shape[0], dw.shape[1], 0, accumulate=True, w=w, lr=lr)

    def layer_forward(self, l: int, ga: torch.Tensor, part: DevicePartition) -> torch.Tensor:
        """out = act(norm(aggregate(GA)) @ W) for one partition (training.py:86-100)."""
        c = self.cfg[l]
        if c.sage:
            return self._sage_forward(l, ga, part)
        if c.gat:
            return self._gat_forward(l, ga, part)
        W = self.wts.w[l]
        pre = self._pre(l, ga, part)
        if c.rownorm:
            ops.rownorm_fwd(pre, pre, part.num_targets, c.d_out, relu=not c.last)
        return pre

    def _pre(self, l: int, ga: torch.Tensor, part: DevicePartition, relu_default: bool = True):
        c = self.cfg[l]
        W = self.wts.w[l]
        dev = self.device
        relu = relu_default and not c.last and not c.rownorm
        out = ops.zeros_rows(part.num_targets, c.d_out, dev)
        s_g = part.scale("s", "gather") if c.sym else None
        s_t = part.scale("s", "targets") if c.sym else None
        if c.transform_first:
            p = ops.zeros_rows(part.num_gather, c.d_out, dev)
            ops.gemm(ga, W, p, part.num_gather, c.d_out, c.d_in, row_scale=s_g)
            ops.agg_sum(part.fwd, p, out, c.d_out, post_div_deg=not c.sym, post_scale=s_t, relu=relu)
        else:
            n = self._norm(l, ga, part)
            ops.gemm(n, W, out, part.num_targets, c.d_out, c.d_in, relu_out=relu)
        return out

    def _norm(self, l: int, ga: torch.Tensor, part: DevicePartition) -> torch.Tensor:
        c = self.cfg[l]
        n = ops.zeros_rows(part.num_targets, c.d_in, self.device)
        ops.agg_sum(part.fwd, ga, n, c.d_in,
                    src_scale=part.scale("s", "gather") if c.sym else None,
                    post_div_deg=not c.sym,
                    post_scale=part.scale("s", "targets") if c.sym else None)
        return n

    def grad_w_host(self, l: int, grad_w: torch.Tensor, to_host) -> np.ndarray:
        """A per-partition weight gradient in the model's host layout
        (GraphSAGE: [dW_root | dW_nbr] side by side, d_out columns each)."""
        c = self.cfg[l]
        if c.sage:
            return np.concatenate([to_host(grad_w[:, : c.ld_out], c.d_out, c.d_in),
                                   to_host(grad_w[:, c.ld_out:], c.d_out, c.d_in)], axis=1)
        if c.gat:      # dW_ext -> (dW, datt) stacked as the model's [W ; a_src ; a_dst]
            d_in, dh, dhp = self.wts.shape[l]
            dw = torch.zeros_like(self.wts.w[l])
            datt = torch.zeros_like(self.wts.att[l])
            ops.gat_param_grads(grad_w, self.wts.w[l], self.wts.att[l], d_in, c.heads, dh, dhp,
                                dw, datt, 0.0)
            w = to_host(dw, c.heads * dhp, d_in).reshape(d_in, c.heads, dhp)[:, :, :dh]
            a = datt.double().cpu().numpy()[:, :, :dh]
            return np.concatenate([w.reshape(d_in, c.heads * dh), a.reshape(2, c.heads * dh)])
        return to_host(grad_w, c.d_out, c.d_in)

    # ------------------------------------------------- GAT, per partition --
    # The layer over one partition's gathered rows GA (G rows): P_ext = GA
    # W_ext, the edge softmax over each target's in-edges + self loop, the
    # attention-weighted sum; every per-vertex quantity lives at the
    # target's gather row (DevicePartition.gat_specs), the T output rows are
    # gathered from there.
    def _gat_regather(self, l: int, ga: torch.Tensor, part: DevicePartition):
        """(P_ext, alpha, alpha_self, O) of one partition; O per head, in
        gather-row space, ReLU applied for hidden layers."""
        c = self.cfg[l]
        wt = self.wts
        d_in, dh, dhp = wt.shape[l]
        G, dev = part.num_gather, self.device
        fwd, _, _ = part.gat_specs()
        ops.gat_build_wext(wt.w[l], wt.att[l], d_in, c.heads, dh, dhp, wt.wext[l])
        pext = ops.zeros_rows(G, c.ld_ext, dev)
        ops.gemm(ga, wt.wext[l], pext, G, c.n_ext, c.d_in)
        alpha = torch.zeros(max(fwd.nnz * c.heads, 1), dtype=torch.float32, device=dev)
        alpha_self = torch.zeros(max(G * c.heads, 1), dtype=torch.float32, device=dev)
        ops.gat_softmax(fwd, pext, c.heads, c.dhp, alpha, alpha_self)
        o = ops.zeros_rows(G, c.hdp, dev)
        ops.agg_sum(fwd, pext[:, : c.hdp], o, c.hdp, edge_w=alpha, self_w=alpha_self,
                    heads=c.heads, head_ld=c.dhp, relu=not c.last)
        return pext, alpha, alpha_self, o

    def _gat_forward(self, l: int, ga: torch.Tensor, part: DevicePartition) -> torch.Tensor:
        c = self.cfg[l]
        T = part.num_targets
        out = ops.zeros_rows(T, c.d_out, self.device)
        if T == 0:
            return out
        _, _, _, o = self._gat_regather(l, ga, part)
        if c.last:
            ot = ops.zeros_rows(T, c.hdp, self.device)
            ops.gather_rows(o, part.fwd.self_idx, ot, c.hdp)
            ops.head_mean(ot, T, c.heads, c.dh, c.dhp, out)
        else:
            ops.gather_rows(o, part.fwd.self_idx, out, c.hdp)
        return out

    def _gat_backward(self, l: int, ga: torch.Tensor, a_out: torch.Tensor, grad_out: torch.Tensor,
                      part: DevicePartition) -> tuple[torch.Tensor, torch.Tensor]:
        """Regather P_ext / attention / O from GA, then: delta and dt (edge
        softmax backward), dP = sum alpha gO and ds over the pull, dW_ext =
        GA^T dP_ext, grad_GA = dP_ext W_ext^T."""
        c = self.cfg[l]
        wt = self.wts
        T, G, dev = part.num_targets, part.num_gather, self.device
        grad_w = torch.zeros_like(wt.wext[l])
        grad_ga = ops.zeros_rows(G, c.d_in, dev)
        if T == 0:
            return grad_ga, grad_w
        fwd, pull, perm = part.gat_specs()
        pext, alpha, alpha_self, o = self._gat_regather(l, ga, part)
        gt = ops.zeros_rows(T, c.hdp, dev)
        if c.last:
            ops.head_mean(grad_out, T, c.heads, c.dh, c.dhp, gt, backward=True)
        else:      # ReLU mask from the layer's output, so gO.relu(O) = gO.O
            ops.mask_scale_rows(grad_out, gt, T, c.d_out, ref=a_out)
        go = ops.zeros_rows(G, c.hdp, dev)
        ops.scatter_add_rows(gt, part.fwd.self_idx, go, c.hdp)
        delta = torch.zeros_like(alpha)
        delta_self = torch.zeros_like(alpha_self)
        gext = ops.zeros_rows(G, c.ld_ext, dev)
        ops.gat_softmax_bwd(fwd, pext, c.heads, c.dhp, alpha, alpha_self, go, o, delta,
                            delta_self, gext)
        ops.agg_sum(pull, go, gext[:, : c.hdp], c.hdp, edge_w=alpha, edge_w_perm=perm,
                    self_w=alpha_self, heads=c.heads, head_ld=c.dhp)
        ops.gat_src_grad(pull, c.heads, c.dhp, perm, delta, delta_self, gext)
        ops.wgrad_sgd(ga, gext, grad_w, c.d_in, c.n_ext, G)
        ops.gemm(gext, wt.wext[l], grad_ga, G, c.d_in, c.n_ext, trans_b=True)
        return grad_ga, grad_w

    # ---------------------------------------------- GraphSAGE-mean, per partition --
    # out_t = X_t W_root + mean_{u in in(t)} X_u W_nbr over the partition's
    # gathered rows: X_t = GA[self_pos], the mean over src_pos (no self),
    # weights [W_root | W_nbr] at columns [0, ld_out) / [ld_out, 2 ld_out).
    def _sage_parts(self, l: int, ga: torch.Tensor, part: DevicePartition):
        c = self.cfg[l]
        T = part.num_targets
        xt = ops.zeros_rows(T, c.d_in, self.device)
        if T:
            ops.gather_rows(ga, part.fwd.self_idx, xt, c.d_in)
        n = ops.zeros_rows(T, c.d_in, self.device)
        ops.agg_sum(part.fwd, ga, n, c.d_in, post_div_deg=2, no_self=True)
        return xt, n

    def _sage_forward(self, l: int, ga: torch.Tensor, part: DevicePartition) -> torch.Tensor:
        c = self.cfg[l]
        W = self.wts.w[l]
        xt, n = self._sage_parts(l, ga, part)
        out = ops.zeros_rows(part.num_targets, c.d_out, self.device)
        ops.gemm(xt, W[:, : c.ld_out], out, part.num_targets, c.d_out, c.d_in)
        ops.gemm(n, W[:, c.ld_out:], out, part.num_targets, c.d_out, c.d_in, accumulate=True,
                 relu_out=not c.last)
        return out

    def _sage_backward(self, l: int, ga: torch.Tensor, a_out: torch.Tensor, grad_out: torch.Tensor,
                       part: DevicePartition) -> tuple[torch.Tensor, torch.Tensor]:
        """dW_root = X_t^T gp, dW_nbr = N_t^T gp (N regathered); grad_GA: the
        neighbour rows receive (gp W_nbr^T / deg_t) pulled over the
        partition's CSC (no self), the target rows gp W_root^T."""
        c = self.cfg[l]
        W = self.wts.w[l]
        T, G = part.num_targets, part.num_gather
        gp = ops.zeros_rows(T, c.d_out, self.device)
        ops.mask_scale_rows(grad_out, gp, T, c.d_out, ref=None if c.last else a_out)
        xt, n = self._sage_parts(l, ga, part)
        grad_w = torch.zeros_like(W)
        ops.wgrad_sgd(xt, gp, grad_w[:, : c.ld_out], c.d_in, c.d_out, T)
        ops.wgrad_sgd(n, gp, grad_w[:, c.ld_out:], c.d_in, c.d_out, T)
        gn = ops.zeros_rows(T, c.d_in, self.device)
        ops.gemm(gp, W[:, c.ld_out:], gn, T, c.d_in, c.d_out, trans_b=True,
                 row_scale=part.scale("inv_deg", "targets"))
        grad_ga = ops.zeros_rows(G, c.d_in, self.device)
        ops.agg_sum(part.bwd, gn, grad_ga, c.d_in, no_self=True)
        gx = ops.zeros_rows(T, c.d_in, self.device)
        ops.gemm(gp, W[:, : c.ld_out], gx, T, c.d_in, c.d_out, trans_b=True)
        if T:
            ops.scatter_add_rows(gx, part.fwd.self_idx, grad_ga, c.d_in)
        return grad_ga, grad_w

    def backward_from_ga(self, l: int, ga: torch.Tensor, a_out: torch.Tensor, grad_out: torch.Tensor,
                         part: DevicePartition) -> tuple[torch.Tensor, torch.Tensor]:
        """(grad_GA [G, d_in], grad_W [d_in, d_out]) of one partition
        (training.py:103-143), recomputing from the (re)gathered input."""
        c = self.cfg[l]
        if c.sage:
            return self._sage_backward(l, ga, a_out, grad_out, part)
        if c.gat:
            return self._gat_backward(l, ga, a_out, grad_out, part)
        W = self.wts.w[l]
        dev = self.device
        T, G = part.num_targets, part.num_gather
        pre_scale = part.scale(c.pre_scale, "targets") if c.transform_first else None
        gp = ops.zeros_rows(T, c.d_out, dev)
        if c.rownorm:
            pre = self._pre(l, ga, part, relu_default=False)
            ops.rownorm_bwd(pre, grad_out, gp, T, c.d_out, a_out=None if c.last else a_out,
                            row_scale=pre_scale)
        else:
            ops.mask_scale_rows(grad_out, gp, T, c.d_out, ref=None if c.last else a_out,
                                row_scale=pre_scale)
        s_g = part.scale("s", "gather") if c.sym else None
        grad_w = torch.zeros_like(self.wts.w[l])
        grad_ga = ops.zeros_rows(G, c.d_in, dev)
        if c.transform_first:
            h = ops.zeros_rows(G, c.d_out, dev)
            ops.agg_sum(part.bwd, gp, h, c.d_out, post_scale=s_g)
            ops.wgrad_sgd(ga, h, grad_w, c.d_in, c.d_out, G)
            ops.gemm(h, W, grad_ga, G, c.d_in, c.d_out, trans_b=True)
        else:
            n = self._norm(l, ga, part)
            ops.wgrad_sgd(n, gp, grad_w, c.d_in, c.d_out, T)
            gn = ops.zeros_rows(T, c.d_in, dev)
            ops.gemm(gp, W, gn, T, c.d_in, c.d_out, trans_b=True,
                     row_scale=part.scale(c.pre_scale, "targets"))
            ops.agg_sum(part.bwd, gn, grad_ga, c.d_in, post_scale=s_g)
        return grad_ga, grad_w


class PartitionEngine(_EngineBase):
    """Per-(layer, partition) execution, literally following training.py:259-358."""

    def __init__(self, dg, model, features, labels, train_mask, mask_count=None):
        super().__init__(dg, model, features, labels, train_mask, mask_count)
        self.grad_cur = ops.zeros_rows(self.V, self.maxw, self.device)
        self.grad_prev = ops.zeros_rows(self.V, self.maxw, self.device)
        self.ops = LayerOps(model, self.device, self.wts)
        self.eye = {}

    def _add_into(self, dst: torch.Tensor, src: torch.Tensor) -> None:
        rows = src.shape[0]
        idx = self.eye.get(rows)
        if idx is None:
            idx = torch.arange(rows, dtype=torch.int32, device=self.device)
            self.eye[rows] = idx
        ops.scatter_add_rows(src, idx, dst, src.shape[1])

    # ---- the epoch -----------------------------------------------------
    def epoch(self, epoch: int, lr: float, order_of, hierarchy=None, use_snapshots=False,
              grad_probe=None, to_host=None) -> None:
        dg = self.dg
        P = dg.num_partitions
        snapshots = {}
        if hierarchy is not None:
            hierarchy.begin_epoch()
        for l, c in enumerate(self.cfg):
            x = self.layer_input(l)
            out = self.acts[l + 1]
            out.zero_()
            for pid in order_of(l, "forward"):
                part = dg.partition(pid)
                ga = ops.zeros_rows(part.num_gather, c.d_in, self.device)
                ops.gather_rows(x, part.gather_map, ga, c.d_in)
                res = self.ops.layer_forward(l, ga, part)
                ops.scatter_add_rows(res, part.targets, out, c.d_out)
                if use_snapshots:
                    snapshots[(l, pid)] = ga
                if hierarchy is not None:
                    hierarchy.forward_partition(l, pid)
            if hierarchy is not None:
                hierarchy.end_forward_layer(l)
        c = self.cfg[-1]
        ops.softmax_xent(self.acts[-1], self.V, c.d_out, self.labels, self.mask, self.mask_count,
                         self.grad_cur, self.stats, self.partials)
        self.check_loss(epoch)
        if hierarchy is not None:
            hierarchy.loss_stage()
        for l in range(self.L):
            self.ops.grad_sink(l).zero_()
        for l in reversed(range(self.L)):
            c = self.cfg[l]
            x = self.layer_input(l)
            results = {}
            for pid in order_of(l, "backward"):
                part = dg.partition(pid)
                if use_snapshots:
                    ga = snapshots.pop((l, pid))
                else:
                    ga = ops.zeros_rows(part.num_gather, c.d_in, self.device)
                    ops.gather_rows(x, part.gather_map, ga, c.d_in)
                a_out = ops.zeros_rows(part.num_targets, c.d_out, self.device)
                ops.gather_rows(self.acts[l + 1], part.targets, a_out, c.d_out)
                g = ops.zeros_rows(part.num_targets, c.d_out, self.device)
                ops.gather_rows(self.grad_cur, part.targets, g, c.d_out)
                results[pid] = self.ops.backward_from_ga(l, ga, a_out, g, part)
                if hierarchy is not None:
                    hierarchy.backward_partition(l, pid)
            if l > 0:
                self.grad_prev.zero_()
            for pid in range(P):
                grad_ga, grad_w = results[pid]
                if grad_probe is not None:
                    grad_probe(epoch, l, pid, to_host(grad_ga, c.d_in),
                               self.ops.grad_w_host(l, grad_w, to_host))
                self._add_into(self.ops.grad_sink(l), grad_w)
                if l > 0:
                    ops.scatter_add_rows(grad_ga, dg.partition(pid).gather_map, self.grad_prev, c.d_in)
            if l > 0 and self.dmask[l] is not None:
                ops.mul_rows(self.grad_prev, self.dmask[l], self.grad_prev, self.V, c.d_in)
            if hierarchy is not None:
                hierarchy.end_backward_layer(l)
            self.grad_cur, self.grad_prev = self.grad_prev, self.grad_cur
        self.ops.sgd(lr)
        if hierarchy is not None:
            hierarchy.end_epoch()

    def check_loss(self, epoch: int) -> None:
        loss = float(self.stats[0].item())
        if not np.isfinite(loss):
            raise ValueError(f"non-finite loss {loss} at epoch {epoch}; "
                             f"reduce the learning rate or check the inputs")
