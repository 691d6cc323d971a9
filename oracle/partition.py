"""Switching-aware partitioner restated in plain Python (small graphs only).

TEST INFRASTRUCTURE (see oracle/__init__.py).  Restates partition.py:
random start (:103-111), per-vertex analysis (:140-200: objective term
1 + count_own/deg - size_own/denom summed in vertex order, top-`depth`
preferences by (count desc, id asc)), candidate order = lexsort over the
preference slots then id (:296), grouped relocation against pre-iteration
sizes (:203-251), and the stop rule (:292-319).
"""

from __future__ import annotations

import math

import numpy as np


def random_labels(n, p, seed):
    perm = np.random.Generator(np.random.PCG64(seed)).permutation(n)
    lab = np.empty(n, dtype=np.int32)
    lab[perm] = np.arange(n, dtype=np.int32) % p
    return lab


def _analyze(adj, labels, sizes, denom, p, depth):
    objective, prefs, candidates = 0.0, [], 0
    for v, nbrs in enumerate(adj):
        counts = {}
        for u in nbrs:
            counts[labels[u]] = counts.get(labels[u], 0) + 1
        own = int(labels[v])
        if nbrs:
            objective += 1.0 + counts.get(own, 0) / len(nbrs) - sizes[own] / denom
        else:
            objective += 1.0 - sizes[own] / denom
        ranked = sorted(counts.items(), key=lambda kv: (-kv[1], kv[0]))[:depth]
        slots = [int(q) for q, _ in ranked] + [p] * (depth - len(ranked))
        if not ranked or slots[0] == own:
            slots = [p] * depth
        else:
            candidates += 1
        prefs.append(slots)
    return objective, prefs, candidates


def _relocate(prefs, labels, sizes, cap, p):
    order = sorted((v for v in range(len(prefs)) if prefs[v][0] != p),
                   key=lambda v: (tuple(prefs[v]), v))
    i = 0
    while i < len(order):
        target = prefs[order[i]][0]
        j = i
        while j < len(order) and prefs[order[j]][0] == target:
            j += 1
        block = order[i:j]
        best, best_len, start = 0, 0, 0
        for k in range(1, len(block) + 1):
            if k == len(block) or prefs[block[k]][1:] != prefs[block[start]][1:]:
                if k - start > best_len:
                    best, best_len = start, k - start
                start = k
        room = max(0, cap - sizes[target])
        for v in block[best:best + min(best_len, room)]:
            labels[v] = target
        i = j


def partition(src_ptr, dst_idx, p, alpha_balance=1.1, beta=1.1, epsilon=0.001, patience=5,
              group_depth=2, max_iters=50, seed=0):
    """Returns dict(labels, objective_trace, initial_objective, iterations,
    converged, max_size_per_iteration)."""
    n = len(src_ptr) - 1
    adj = [list(dst_idx[src_ptr[v]:src_ptr[v + 1]]) for v in range(n)]
    denom = alpha_balance * n / p
    labels = random_labels(n, p, seed)
    sizes = np.bincount(labels, minlength=p).tolist()
    cap = math.floor(beta * n / p + 1e-9)
    prev, prefs, cand = _analyze(adj, labels, sizes, denom, p, group_depth)
    out = dict(initial_objective=prev, objective_trace=[], max_size_per_iteration=[max(sizes)],
               iterations=0, converged=False)
    streak, stopped = 0, False
    for _ in range(max_iters):
        if cand == 0:
            out["converged"], stopped = True, True
            break
        _relocate(prefs, labels, sizes, cap, p)
        out["iterations"] += 1
        sizes = np.bincount(labels, minlength=p).tolist()
        cur, prefs, cand = _analyze(adj, labels, sizes, denom, p, group_depth)
        out["objective_trace"].append(cur)
        out["max_size_per_iteration"].append(max(sizes))
        rel = (cur - prev) / abs(prev) if prev != 0.0 else (0.0 if cur == 0.0 else math.inf)
        streak = streak + 1 if rel < epsilon else 0
        prev = cur
        if streak >= patience:
            out["converged"], stopped = True, True
            break
    if not stopped:
        out["converged"] = cand == 0
    out["labels"] = labels
    return out
