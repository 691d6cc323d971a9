"""Partition execution plans (reference: grinder/plan.py).

``build_partition_plan`` runs natively (``grd_plan_create``) and stores the
plan as flat concatenated arrays — the layout the device engine uploads to
HBM once — while ``plan.topologies`` still exposes the reference's
per-partition ``PartitionTopology`` view (int64 arrays, identical values:
targets, gather map sorted by (owner, id), ``tgt_ptr``/``src_pos`` grouped
by local target with ascending gather positions, ``self_pos``, global
in-degrees; plan.py:21-136).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graph import CsrGraph

__all__ = ["FlatPlan", "PartitionPlan", "PartitionTopology", "build_partition_plan"]


@dataclass
class PartitionTopology:
    """One partition's local 1-hop topology (plan.py:21-48)."""

    partition_id: int
    targets: np.ndarray
    gather_map: np.ndarray
    tgt_ptr: np.ndarray
    src_pos: np.ndarray
    edge_local_target: np.ndarray
    self_pos: np.ndarray
    target_indeg: np.ndarray
    gather_indeg: np.ndarray

    @property
    def num_edges(self) -> int:
        return int(self.src_pos.shape[0])

    @property
    def is_empty(self) -> bool:
        return self.targets.size == 0


@dataclass
class FlatPlan:
    """Concatenated plan arrays (see include/grinder_b200.h, grd_plan_export)."""

    part_ptr: np.ndarray     # int64 [P+1] offsets into perm
    perm: np.ndarray         # int32 [V]   targets, partition by partition
    in_ptr: np.ndarray       # int64 [V+1] edge offsets per perm row
    in_src: np.ndarray       # int32 [E]   global source of each edge
    in_src_pos: np.ndarray   # int32 [E]   gather-map position of the source
    gather_ptr: np.ndarray   # int64 [P+1]
    gather_map: np.ndarray   # int32 [sum G]
    self_pos: np.ndarray     # int32 [V]   (perm order)
    in_degree: np.ndarray    # int32 [V]


class PartitionPlan:
    """All per-partition topologies of one labeling (plan.py:51-72)."""

    def __init__(self, labels: np.ndarray, num_partitions: int, num_vertices: int,
                 flat: FlatPlan):
        self.labels = np.asarray(labels, dtype=np.int32)
        self.num_partitions = int(num_partitions)
        self.num_vertices = int(num_vertices)
        self.flat = flat
        self.in_degrees = flat.in_degree.astype(np.int64)
        sizes = np.diff(flat.part_ptr)
        self.empty_partitions = [int(q) for q in np.flatnonzero(sizes == 0)]
        self._topologies: list[PartitionTopology] | None = None
        self.device_cache: dict = {}   # per-device uploads, filled by the engine

    def topology(self, q: int) -> PartitionTopology:
        f = self.flat
        r0, r1 = int(f.part_ptr[q]), int(f.part_ptr[q + 1])
        e0, e1 = int(f.in_ptr[r0]), int(f.in_ptr[r1])
        g0, g1 = int(f.gather_ptr[q]), int(f.gather_ptr[q + 1])
        targets = f.perm[r0:r1].astype(np.int64)
        gmap = f.gather_map[g0:g1].astype(np.int64)
        tgt_ptr = f.in_ptr[r0:r1 + 1] - f.in_ptr[r0]
        counts = np.diff(tgt_ptr)
        return PartitionTopology(
            partition_id=q,
            targets=targets,
            gather_map=gmap,
            tgt_ptr=tgt_ptr.astype(np.int64),
            src_pos=f.in_src_pos[e0:e1].astype(np.int64),
            edge_local_target=np.repeat(np.arange(r1 - r0, dtype=np.int64), counts),
            self_pos=f.self_pos[r0:r1].astype(np.int64),
            target_indeg=self.in_degrees[targets],
            gather_indeg=self.in_degrees[gmap],
        )

    @property
    def topologies(self) -> list[PartitionTopology]:
        if self._topologies is None:
            self._topologies = [self.topology(q) for q in range(self.num_partitions)]
        return self._topologies

    @property
    def gather_maps(self) -> list[np.ndarray]:
        return [t.gather_map for t in self.topologies]

    @property
    def target_ranges(self) -> list[np.ndarray]:
        return [t.targets for t in self.topologies]

    def gather_rows_total(self) -> int:
        return int(self.flat.gather_ptr[-1])

    def partition_sizes(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """Per-partition (targets T, gather rows G, edges E)."""
        f = self.flat
        t = np.diff(f.part_ptr)
        g = np.diff(f.gather_ptr)
        e = f.in_ptr[f.part_ptr[1:]] - f.in_ptr[f.part_ptr[:-1]]
        return t, g, e


def _flat_plan_gpu(graph: CsrGraph, lab32: np.ndarray, p: int, device) -> FlatPlan:
    """The FlatPlan by device sorts (same arrays as grd_plan_create, bit for
    bit): edges ordered by (perm row of the target, owner of the source,
    source id) through two stable sorts of the CSR's source-ordered edge
    list; gather maps as the sorted unique (partition, owner, id) keys of
    every in-edge and target, whose inverse gives src_pos and self_pos."""
    import torch
    dev = torch.device(device)
    n = graph.num_vertices
    with torch.cuda.device(dev):
        lab = torch.from_numpy(lab32).to(dev).long()
        ptr = torch.from_numpy(np.ascontiguousarray(graph.src_ptr, dtype=np.int64)).to(dev)
        dst = torch.from_numpy(np.ascontiguousarray(graph.dst_idx, dtype=np.int32)).to(dev).long()
        m = dst.numel()
        src = torch.repeat_interleave(torch.arange(n, device=dev), ptr[1:] - ptr[:-1])
        perm = torch.sort(lab, stable=True).indices
        rank = torch.empty_like(perm)
        rank[perm] = torch.arange(n, device=dev)
        part_ptr = torch.zeros(p + 1, dtype=torch.int64, device=dev)
        part_ptr[1:] = torch.cumsum(torch.bincount(lab, minlength=p), 0)
        in_degree = torch.bincount(dst, minlength=n)
        # CSR edges are in source order: stable by owner(source) gives
        # (owner, id); stable by the target's perm row groups the rows
        o1 = torch.sort(lab[src], stable=True).indices
        src, dst = src[o1], dst[o1]
        del o1
        o2 = torch.sort(rank[dst], stable=True).indices
        src, dst = src[o2], dst[o2]
        del o2
        in_ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        in_ptr[1:] = torch.cumsum(in_degree[perm], 0)
        # gather maps: unique (partition, owner, id) over in-edges and targets
        q_e = lab[dst]
        keys = torch.cat([(q_e * p + lab[src]) * n + src, (lab * p + lab) * n + torch.arange(n, device=dev)])
        del q_e
        uniq, inv = torch.unique(keys, sorted=True, return_inverse=True)
        del keys
        gq = uniq // n // p
        gather_ptr = torch.zeros(p + 1, dtype=torch.int64, device=dev)
        gather_ptr[1:] = torch.cumsum(torch.bincount(gq, minlength=p), 0)
        gather_map = (uniq % n).int()
        del uniq, gq
        in_src_pos = (inv[:m] - gather_ptr[lab[dst]]).int()
        self_all = inv[m:] - gather_ptr[lab]
        self_pos = self_all[perm].int()
        del inv, self_all

        def h(t, dt):
            return t.to(torch.int64 if dt == np.int64 else torch.int32).cpu().numpy().astype(dt, copy=False)
        flat = FlatPlan(part_ptr=h(part_ptr, np.int64), perm=h(perm, np.int32), in_ptr=h(in_ptr, np.int64),
                        in_src=h(src, np.int32), in_src_pos=h(in_src_pos, np.int32),
                        gather_ptr=h(gather_ptr, np.int64), gather_map=h(gather_map, np.int32),
                        self_pos=h(self_pos, np.int32), in_degree=h(in_degree, np.int32))
    torch.cuda.empty_cache()
    return flat


def build_partition_plan(graph: CsrGraph, labels: np.ndarray,
                         num_partitions: int | None = None,
                         num_threads: int | None = None, device=None) -> PartitionPlan:
    """Gather maps and local topologies for every partition (plan.py:75-136).
    ``device="cuda"`` builds the same plan with device sorts."""
    n = graph.num_vertices
    labels = np.asarray(labels)
    if labels.shape != (n,):
        raise ValueError(f"labels shape {labels.shape} != ({n},)")
    p = int(num_partitions) if num_partitions is not None else int(labels.max()) + 1
    if labels.size and (labels.min() < 0 or labels.max() >= p):
        raise ValueError("labels out of range for num_partitions")
    lab32 = np.ascontiguousarray(labels, dtype=np.int32)
    if device is not None and str(device).startswith("cuda"):
        return PartitionPlan(lab32, p, n, _flat_plan_gpu(graph, lab32, p, device))
    src_ptr = np.ascontiguousarray(graph.src_ptr, dtype=np.int64)
    dst_idx = np.ascontiguousarray(graph.dst_idx, dtype=np.int32)
    L = _lib.lib()
    handle = _lib.c_vp()
    threads = num_threads if num_threads is not None else (os.cpu_count() or 1)
    _lib.check(L.grd_plan_create(n, _lib.ptr(src_ptr), _lib.ptr(dst_idx), _lib.ptr(lab32), p,
                                 threads, handle), "build_partition_plan")
    try:
        m = np.zeros(1, dtype=np.int64)
        gt = np.zeros(1, dtype=np.int64)
        _lib.check(L.grd_plan_sizes(handle, _lib.ptr(m), _lib.ptr(gt)))
        e, g = int(m[0]), int(gt[0])
        flat = FlatPlan(
            part_ptr=np.empty(p + 1, np.int64), perm=np.empty(n, np.int32),
            in_ptr=np.empty(n + 1, np.int64), in_src=np.empty(e, np.int32),
            in_src_pos=np.empty(e, np.int32), gather_ptr=np.empty(p + 1, np.int64),
            gather_map=np.empty(g, np.int32), self_pos=np.empty(n, np.int32),
            in_degree=np.empty(n, np.int32))
        _lib.check(L.grd_plan_export(handle, *(_lib.ptr(a) for a in (
            flat.part_ptr, flat.perm, flat.in_ptr, flat.in_src, flat.in_src_pos,
            flat.gather_ptr, flat.gather_map, flat.self_pos, flat.in_degree))))
    finally:
        L.grd_plan_destroy(handle)
    return PartitionPlan(lab32, p, n, flat)
