"""Switching-aware partitioner (reference: grinder/partition.py).

The iterative grouped relocation runs in the native library
(``grd_sa_partition``, OpenMP over vertices); its convergence decisions see
the same f64 objective bits as the reference's numba kernels because the
per-vertex terms are evaluated in the same operation order and summed
sequentially in vertex order.  The balanced random start stays with numpy's
PCG64 ``permutation`` on the host (partition.py:103-111) so the initial
labels are the reference's by construction.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _lib
from .graph import CsrGraph

__all__ = [
    "PartitionQuality",
    "PartitionResult",
    "PartitionerParams",
    "expansion_ratio",
    "partition_objective",
    "partition_score",
    "random_partition",
    "relocation_capacity",
    "switching_aware_partition",
    "vertex_preferences",
]


@dataclass
class PartitionerParams:
    """Knobs of :func:`switching_aware_partition` (partition.py:40-64)."""

    alpha_balance: float = 1.1
    beta: float = 1.1
    epsilon: float = 0.001
    patience: int = 5
    group_depth: int = 2
    max_iters: int = 50
    seed: int = 0

    def __post_init__(self) -> None:
        checks = [
            (self.alpha_balance >= 1.0, f"alpha_balance must be >= 1, got {self.alpha_balance}"),
            (self.beta >= self.alpha_balance,
             f"beta ({self.beta}) must be >= alpha_balance ({self.alpha_balance})"),
            (self.epsilon > 0.0, f"epsilon must be positive, got {self.epsilon}"),
            (self.patience >= 1, f"patience must be >= 1, got {self.patience}"),
            (self.group_depth >= 2, f"group_depth must be >= 2, got {self.group_depth}"),
            (self.max_iters >= 1, f"max_iters must be >= 1, got {self.max_iters}"),
        ]
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)


@dataclass
class PartitionResult:
    labels: np.ndarray
    num_partitions: int
    objective_trace: list[float]
    initial_objective: float
    converged: bool
    iterations: int
    max_size_per_iteration: list[int]


@dataclass
class PartitionQuality:
    per_partition_alpha: list[float]
    mean_alpha: float
    dependency_matrix: list[list[int]]
    max_balance: float
    objective: float


def relocation_capacity(beta: float, num_vertices: int, num_partitions: int,
                        part_size: int) -> int:
    """Room left in a partition: floor(beta*|V|/p + 1e-9) - size, >= 0."""
    return max(0, math.floor(beta * num_vertices / num_partitions + 1e-9) - part_size)


def random_partition(num_vertices: int, num_partitions: int, seed: int = 0) -> np.ndarray:
    """Shuffled round-robin labels (sizes within one), int32."""
    if num_partitions < 1:
        raise ValueError(f"num_partitions must be >= 1, got {num_partitions}")
    shuffled = np.random.Generator(np.random.PCG64(seed)).permutation(num_vertices)
    labels = np.empty(num_vertices, dtype=np.int32)
    labels[shuffled] = np.arange(num_vertices, dtype=np.int32) % num_partitions
    return labels


def partition_score(graph: CsrGraph, labels: np.ndarray, vertex: int, part: int,
                    alpha_balance: float, num_partitions: int) -> float:
    """One vertex's affinity for one partition, the per-vertex term the
    switching-aware objective sums (partition.py:114-124): 1 + (share of the
    vertex's out-neighbours labelled ``part``) - |part| / (alpha V / P)."""
    row = graph.dst_idx[int(graph.src_ptr[vertex]):int(graph.src_ptr[vertex + 1])]
    labels = np.asarray(labels)
    share = float(np.sum(labels[row] == part)) / row.size if row.size else 0.0
    fair = alpha_balance * graph.num_vertices / num_partitions
    return 1.0 + share - float(np.sum(labels == part)) / fair


def vertex_preferences(graph: CsrGraph, labels: np.ndarray, vertex: int,
                       num_partitions: int, depth: int = 2) -> list[int]:
    """The partitions a vertex's out-neighbours fall in, most frequent first
    and ties by ascending id, at most ``depth`` of them (partition.py:
    127-137); empty for an isolated vertex."""
    row = graph.dst_idx[int(graph.src_ptr[vertex]):int(graph.src_ptr[vertex + 1])]
    if row.size == 0:
        return []
    counts = np.bincount(np.asarray(labels)[row], minlength=num_partitions)
    ranked = sorted(np.flatnonzero(counts).tolist(), key=lambda q: (-int(counts[q]), q))
    return ranked[:depth]


def partition_objective(graph: CsrGraph, labels: np.ndarray, num_partitions: int,
                        alpha_balance: float = 1.1) -> float:
    """Sum over vertices of 1 + own-neighbour share - size penalty
    (partition.py:324-336; numpy pairwise sum as in the reference)."""
    n = graph.num_vertices
    labels = np.asarray(labels)
    size_of = np.bincount(labels, minlength=num_partitions)
    src = graph.edge_sources()
    own = np.bincount(src[labels[graph.dst_idx] == labels[src]], minlength=n).astype(np.float64)
    deg = graph.out_degrees().astype(np.float64)
    share = np.zeros(n)
    np.divide(own, deg, out=share, where=deg > 0)
    per_vertex = 1.0 + share - size_of[labels] / (alpha_balance * n / num_partitions)
    return float(np.sum(per_vertex))


def switching_aware_partition(graph: CsrGraph, num_partitions: int,
                              params: PartitionerParams | None = None,
                              num_threads: int | None = None, device=None) -> PartitionResult:
    """Iterative grouped relocation under a hard capacity (partition.py:254-321).
    ``device="cuda"`` runs the iterations on the GPU (same labels, trace and
    iteration count, bit for bit: :func:`_sa_partition_gpu`)."""
    params = params or PartitionerParams()
    n, p = graph.num_vertices, num_partitions
    if p < 1:
        raise ValueError(f"num_partitions must be >= 1, got {p}")
    if p == 1:
        labels = np.zeros(n, dtype=np.int32)
        return PartitionResult(labels, 1, [], partition_objective(graph, labels, 1, params.alpha_balance),
                               True, 0, [n])
    labels = random_partition(n, p, params.seed)
    if device is not None and str(device).startswith("cuda") and _gpu_fits(n, p, params.group_depth):
        return _sa_partition_gpu(graph, p, params, labels, device)
    src_ptr = np.ascontiguousarray(graph.src_ptr, dtype=np.int64)
    dst_idx = np.ascontiguousarray(graph.dst_idx, dtype=np.int32)
    trace = np.zeros(params.max_iters, dtype=np.float64)
    sizes = np.zeros(params.max_iters + 1, dtype=np.int64)
    init = np.zeros(1, dtype=np.float64)
    iters = np.zeros(1, dtype=np.int32)
    conv = np.zeros(1, dtype=np.int32)
    knobs = _lib.GrdPartitionerParams(params.alpha_balance, params.beta, params.epsilon,
                                      params.patience, params.group_depth, params.max_iters, 0)
    threads = num_threads if num_threads is not None else (os.cpu_count() or 1)
    _lib.check(_lib.lib().grd_sa_partition(
        n, _lib.ptr(src_ptr), _lib.ptr(dst_idx), p, knobs, _lib.ptr(labels), _lib.ptr(trace),
        _lib.ptr(sizes), _lib.ptr(init), _lib.ptr(iters), _lib.ptr(conv), threads),
        "switching_aware_partition")
    k = int(iters[0])
    return PartitionResult(labels=labels, num_partitions=p,
                           objective_trace=[float(x) for x in trace[:k]],
                           initial_objective=float(init[0]), converged=bool(conv[0]),
                           iterations=k, max_size_per_iteration=[int(x) for x in sizes[:k + 1]])


def _gpu_fits(n: int, p: int, depth: int) -> bool:
    """The device path packs (preference slots, vertex id) into one int64
    sort key and keeps a per-warp histogram of p counters."""
    return p <= 1024 and (p + 1) ** depth * max(n, 1) < (1 << 62)


def _relocate_sorted(prefs, lab, sizes, p: int, cap_limit: int) -> None:
    """_relocate_kernel (partition.py:203-251) on torch tensors (any device):
    ``prefs`` [depth, n] int32 preference slots, ``lab`` [n] int32 labels
    (updated in place), ``sizes`` [p] int64 pre-iteration sizes.  Candidates
    (slot 0 != p) are ordered by one sort of (slot_0, .., slot_{d-1}, id)
    packed base p+1; equal (target, tail) keys are the reference's runs,
    and per target block the first longest run moves its first
    min(len, capacity) vertices."""
    import torch
    dev = lab.device
    depth, n = prefs.shape
    base = p + 1
    ids = torch.nonzero(prefs[0] != p).squeeze(1)
    key = prefs[0][ids].long()
    for s_ in range(1, depth):
        key = key * base + prefs[s_][ids].long()
    order = torch.sort(key * n + ids).values
    del key, ids
    gval, gcount = torch.unique_consecutive(order // n, return_counts=True)
    if gval.numel() == 0:
        return
    tgt = gval // base ** (depth - 1)
    gstart = torch.cumsum(gcount, 0) - gcount
    best = torch.zeros(p, dtype=torch.int64, device=dev).scatter_reduce(
        0, tgt, gcount, "amax", include_self=False)
    G = gval.numel()
    first = torch.full((p,), G, dtype=torch.int64, device=dev)
    win = gcount == best[tgt]
    first.scatter_reduce_(0, tgt[win], torch.arange(G, device=dev)[win], "amin")
    ts = torch.nonzero(first < G).squeeze(1)
    g = first[ts]
    take = torch.minimum(gcount[g], (cap_limit - sizes[ts]).clamp_min(0))
    for t, a, k in zip(ts.tolist(), gstart[g].tolist(), take.tolist()):
        if k:
            lab[order[a:a + k] % n] = t


def _sa_partition_gpu(graph: CsrGraph, p: int, params: PartitionerParams, labels: np.ndarray,
                      device) -> PartitionResult:
    """switching_aware_partition's iterations on the GPU (partition.py:279-321).

    Per iteration: the analysis pass is the sm_100a kernel grd_sa_analyze
    (terms, preference slots, candidate count; neighbour labels read through
    dst_idx, so the reference's dst_part refresh is fused away); the f64
    objective is the sequential sum of the terms in vertex order on the host
    (grd_sum_sequential: the reference's loop order, hence its bits); the
    candidate order — np.lexsort(prefs[::-1]) restricted to candidates — is
    one device sort of (slot_0, .., slot_{d-1}, vertex id) packed base p+1
    into an int64 key; the relocation (partition.py:203-251) is segment
    arithmetic on the sorted keys: equal (target, tail) keys are the
    reference's runs, the first longest run of every target block wins and
    its first min(len, capacity) vertices (ascending id) move."""
    import torch
    dev = torch.device(device)
    n = graph.num_vertices
    depth = params.group_depth
    denom = params.alpha_balance * n / p
    cap_limit = math.floor(params.beta * n / p + 1e-9)
    L = _lib.lib()
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        src_ptr = torch.from_numpy(np.ascontiguousarray(graph.src_ptr, dtype=np.int64)).to(dev)
        dst_idx = torch.from_numpy(np.ascontiguousarray(graph.dst_idx, dtype=np.int32)).to(dev)
        if dst_idx.numel() == 0:        # edgeless graph: a valid (never read) pointer
            dst_idx = torch.zeros(1, dtype=torch.int32, device=dev)
        lab = torch.from_numpy(labels).to(dev)
        lab_prev = torch.empty_like(lab)
        prefs = torch.empty((depth, n), dtype=torch.int32, device=dev)
        # two analysis slots: while the host sums one pass's terms (the
        # sequential f64 objective that fixes the convergence bits), the GPU
        # already runs the next relocation + analysis speculatively; a stop
        # decision restores the labels from before that relocation
        terms = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(2)]
        terms_host = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        cand = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(2)]
        copy_stream = torch.cuda.Stream(dev)
        pool = ThreadPoolExecutor(max_workers=1)
        slot = [0]

        def analyze():
            """Launch one analysis pass: (future of its objective, candidates,
            sizes, max size); the terms' D2H and host sum run beside the GPU."""
            b = slot[0]
            slot[0] ^= 1
            sizes = torch.bincount(lab, minlength=p)
            cand[b].zero_()
            _lib.check(L.grd_sa_analyze(n, src_ptr.data_ptr(), dst_idx.data_ptr(), lab.data_ptr(),
                                        sizes.data_ptr(), p, depth, denom, terms[b].data_ptr(),
                                        prefs.data_ptr(), cand[b].data_ptr(), stream), "sa_analyze")
            done = torch.cuda.Event()
            done.record()
            copy_stream.wait_event(done)
            with torch.cuda.stream(copy_stream):
                terms_host[b].copy_(terms[b], non_blocking=True)
            copied = torch.cuda.Event()
            copied.record(copy_stream)
            res = np.zeros(1, dtype=np.float64)

            def total() -> float:
                copied.synchronize()
                _lib.check(L.grd_sum_sequential(terms_host[b].data_ptr(), n, _lib.ptr(res)),
                           "sum_sequential")
                return float(res[0])
            fut = pool.submit(total)
            return fut, int(cand[b].item()), sizes, int(sizes.max().item())

        try:
            fut, num_candidates, sizes, smax = analyze()
            obj_prev = fut.result()
            initial_objective = obj_prev
            trace: list[float] = []
            max_sizes = [smax]
            converged, iterations, streak = False, 0, 0
            pending = None
            while True:
                # reference loop (partition.py:292-321): max_iters relocations,
                # stop early on no candidates or on the patience rule
                if iterations >= params.max_iters:
                    converged = num_candidates == 0
                    break
                if num_candidates == 0:
                    converged = True
                    break
                if pending is None:
                    _relocate_sorted(prefs, lab, sizes, p, cap_limit)
                    pending = analyze()
                fut, nc_cur, sizes_cur, smax = pending
                pending = None
                iterations += 1
                speculate = iterations < params.max_iters and nc_cur != 0
                if speculate:                   # the next iteration, before this one's decision
                    lab_prev.copy_(lab)
                    _relocate_sorted(prefs, lab, sizes_cur, p, cap_limit)
                    pending = analyze()
                obj_cur = fut.result()
                trace.append(obj_cur)
                max_sizes.append(smax)
                if obj_prev != 0.0:
                    rel = (obj_cur - obj_prev) / abs(obj_prev)
                else:
                    rel = 0.0 if obj_cur == 0.0 else math.inf
                if rel < params.epsilon:
                    streak += 1
                    if streak >= params.patience:
                        converged = True
                        if pending is not None:     # undo the speculative relocation
                            lab.copy_(lab_prev)
                            pending[0].result()
                            pending = None
                        break
                else:
                    streak = 0
                obj_prev = obj_cur
                num_candidates, sizes = nc_cur, sizes_cur
        finally:
            if pending is not None:
                pending[0].result()
            pool.shutdown(wait=True)
        out_labels = lab.cpu().numpy().astype(np.int32)
        del src_ptr, dst_idx, lab, lab_prev, terms, prefs
    torch.cuda.empty_cache()
    return PartitionResult(labels=out_labels, num_partitions=p, objective_trace=trace,
                           initial_objective=initial_objective, converged=converged,
                           iterations=iterations, max_size_per_iteration=max_sizes)


def expansion_ratio(graph: CsrGraph, labels: np.ndarray, num_partitions: int,
                    alpha_balance: float = 1.1) -> PartitionQuality:
    """Gather-set expansion alpha_p = |targets U in-neighbours| / |targets|,
    dependency matrix and balance of a labeling (partition.py:339-373)."""
    n, p = graph.num_vertices, num_partitions
    lab = np.asarray(labels, dtype=np.int64)
    counts = np.bincount(lab, minlength=p)
    # (needing partition, vertex) pairs: in-edge sources and the targets.
    need = np.unique(np.concatenate([lab[graph.dst_idx] * n + graph.edge_sources(),
                                     lab * n + np.arange(n, dtype=np.int64)]))
    needer, vertex = need // n, need % n
    dep = np.zeros((p, p), dtype=np.int64)
    np.add.at(dep, (needer, lab[vertex]), 1)
    required = np.bincount(needer, minlength=p)
    alphas = [float(required[q] / counts[q]) if counts[q] else 0.0 for q in range(p)]
    used = [a for q, a in enumerate(alphas) if counts[q]]
    return PartitionQuality(
        per_partition_alpha=alphas,
        mean_alpha=float(sum(used) / len(used)) if used else 0.0,
        dependency_matrix=dep.tolist(),
        max_balance=float(counts.max() / (n / p)) if n else 0.0,
        objective=partition_objective(graph, lab.astype(np.int32), p, alpha_balance),
    )
