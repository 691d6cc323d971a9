"""Partition plan restated with explicit per-partition loops (numpy).

TEST INFRASTRUCTURE (see oracle/__init__.py).  Restates plan.py:75-136:
targets = vertices labelled q; gather map = targets plus every in-neighbour
of a target, sorted by (owner label, vertex id); edges into the partition
grouped by local target with ascending gather position; global in-degrees.
"""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np


def build_plan(src_ptr, dst_idx, labels, num_partitions):
    """List of SimpleNamespace topologies with the reference's field names."""
    n = len(src_ptr) - 1
    labels = np.asarray(labels, dtype=np.int64)
    src_of_edge = np.repeat(np.arange(n, dtype=np.int64), np.diff(src_ptr))
    dst_of_edge = np.asarray(dst_idx, dtype=np.int64)
    indeg = np.bincount(dst_of_edge, minlength=n).astype(np.int64)
    owner_of_dst = labels[dst_of_edge]
    plan = []
    for q in range(num_partitions):
        targets = np.flatnonzero(labels == q)
        into = owner_of_dst == q
        e_src, e_dst = src_of_edge[into], dst_of_edge[into]
        members = np.union1d(targets, e_src)
        gmap = members[np.lexsort((members, labels[members]))]
        pos_of = {int(v): i for i, v in enumerate(gmap)}
        src_pos = np.array([pos_of[int(u)] for u in e_src], dtype=np.int64)
        local_t = np.searchsorted(targets, e_dst)
        k = np.lexsort((src_pos, local_t))
        src_pos, local_t = src_pos[k], local_t[k]
        tgt_ptr = np.zeros(targets.size + 1, dtype=np.int64)
        np.cumsum(np.bincount(local_t, minlength=targets.size), out=tgt_ptr[1:])
        plan.append(SimpleNamespace(
            partition_id=q, targets=targets, gather_map=gmap, tgt_ptr=tgt_ptr, src_pos=src_pos,
            edge_local_target=local_t,
            self_pos=np.array([pos_of[int(v)] for v in targets], dtype=np.int64),
            target_indeg=indeg[targets], gather_indeg=indeg[gmap]))
    return plan
