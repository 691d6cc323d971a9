"""CSR graphs and the Kronecker generator (reference: grinder/graph.py).

``CsrGraph`` keeps the reference's field names and invariants
(graph.py:33-84): ``src_ptr`` int64 offsets of length |V|+1 and ``dst_idx``
int32 destinations; an edge u->v means "v aggregates u".  The generator
runs in the native library and reproduces numpy's PCG64 stream, so
``generate_kronecker(scale, d, seed)`` returns the reference's graph bit for
bit (graph.py:158-209) in a fraction of the time — on the host cores, or
with ``device="cuda"`` as an sm_100a kernel plus device sorts.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["CsrGraph", "DegreeStats", "build_csr", "degree_stats", "export_edge_list",
           "generate_kronecker", "KRONECKER_INITIATOR"]

# Skewed 2x2 initiator (graph.py:30).
KRONECKER_INITIATOR = (0.57, 0.19, 0.19, 0.05)


@dataclass
class CsrGraph:
    """Directed graph in CSR form; ids are dense ``0..|V|-1``."""

    num_vertices: int
    num_edges: int
    src_ptr: np.ndarray
    dst_idx: np.ndarray

    def out_degrees(self) -> np.ndarray:
        return np.diff(self.src_ptr)

    def neighbors(self, vertex: int) -> np.ndarray:
        lo, hi = self.src_ptr[vertex], self.src_ptr[vertex + 1]
        return self.dst_idx[lo:hi]

    def edge_sources(self) -> np.ndarray:
        """Source vertex of every edge, aligned with ``dst_idx``."""
        return np.repeat(np.arange(self.num_vertices, dtype=np.int64), self.out_degrees())

    def in_degrees(self) -> np.ndarray:
        return np.bincount(self.dst_idx, minlength=self.num_vertices).astype(np.int64)

    def validate(self) -> None:
        """Raise ValueError on the first violated CSR invariant."""
        n, m = self.num_vertices, self.num_edges
        if self.src_ptr.shape != (n + 1,):
            raise ValueError("src_ptr length must be num_vertices + 1")
        if self.src_ptr[0] != 0 or self.src_ptr[-1] != m:
            raise ValueError("src_ptr must start at 0 and end at num_edges")
        if (np.diff(self.src_ptr) < 0).any():
            raise ValueError("src_ptr must be monotonically non-decreasing")
        if self.dst_idx.shape != (m,):
            raise ValueError("dst_idx length must be num_edges")
        if m and (int(self.dst_idx.min()) < 0 or int(self.dst_idx.max()) >= n):
            raise ValueError("dst_idx entries must be in [0, num_vertices)")
        pair = self.edge_sources() * np.int64(n) + self.dst_idx
        if np.unique(pair).size != m:
            raise ValueError("duplicate destination within a source adjacency")


def _pairs_to_csr(src: np.ndarray, dst: np.ndarray, n: int) -> CsrGraph:
    """CSR from endpoint arrays: first occurrence of a pair survives and every
    source keeps its surviving edges in input order (graph.py:87-116)."""
    src = np.asarray(src, dtype=np.int64).ravel()
    dst = np.asarray(dst, dtype=np.int64).ravel()
    if src.size:
        lo = min(int(src.min()), int(dst.min()))
        hi = max(int(src.max()), int(dst.max()))
        if lo < 0:
            raise ValueError("edge endpoints must be non-negative")
        if hi >= n:
            raise ValueError("edge endpoint out of range")
        _, first = np.unique(src * np.int64(n) + dst, return_index=True)
        survivors = np.sort(first)
        src, dst = src[survivors], dst[survivors]
        by_src = np.argsort(src, kind="stable")
        src, dst = src[by_src], dst[by_src]
    ptr = np.zeros(n + 1, dtype=np.int64)
    if src.size:
        np.cumsum(np.bincount(src, minlength=n), out=ptr[1:])
    return CsrGraph(num_vertices=n, num_edges=int(src.size), src_ptr=ptr,
                    dst_idx=dst.astype(np.int32))


def build_csr(edge_list, num_vertices: int) -> CsrGraph:
    """Directed CSR from (src, dst) pairs; duplicates dropped (first wins)."""
    if num_vertices < 0:
        raise ValueError("num_vertices must be non-negative")
    pairs = np.asarray(edge_list, dtype=np.int64)
    if pairs.size == 0:
        pairs = pairs.reshape(0, 2)
    if pairs.ndim != 2 or pairs.shape[1] != 2:
        raise ValueError("edge_list must be pairs of (src, dst)")
    return _pairs_to_csr(pairs[:, 0], pairs[:, 1], num_vertices)


def _pcg64_words(seed: int) -> np.ndarray:
    """{state_hi, state_lo, inc_hi, inc_lo} of numpy's PCG64(seed)."""
    st = np.random.PCG64(seed).state["state"]
    mask = (1 << 64) - 1
    s, inc = int(st["state"]), int(st["inc"])
    return np.array([s >> 64, s & mask, inc >> 64, inc & mask], dtype=np.uint64)


_M128 = (1 << 128) - 1
_PCG_MULT = (0x2360ED051FC65DA4 << 64) | 0x4385DF649FCCF645


def _pcg_jump(delta: int, inc: int) -> tuple[int, int]:
    """(mul, add) with advance(state, delta) = mul * state + add (mod 2**128)."""
    cur_mult, cur_plus, acc_mult, acc_plus = _PCG_MULT, inc, 1, 0
    while delta > 0:
        if delta & 1:
            acc_mult = (acc_mult * cur_mult) & _M128
            acc_plus = (acc_plus * cur_mult + cur_plus) & _M128
        cur_plus = ((cur_mult + 1) * cur_plus) & _M128
        cur_mult = (cur_mult * cur_mult) & _M128
        delta >>= 1
    return acc_mult, acc_plus


def _words(*xs: int) -> np.ndarray:
    return np.array([w for x in xs for w in (x >> 64, x & ((1 << 64) - 1))], dtype=np.uint64)


def _first_occurrence(keys, target: int):
    """Positions of the first `target` first occurrences (ascending) and the
    number of distinct keys (np.unique(return_index) semantics).  Sorted in
    buckets (key mod nb: equal keys share a bucket, and the power-law key
    distribution still spreads evenly) so no single sort reaches the 2**31
    elements a device sort takes; the first occurrences are marked in a
    position mask, whose nonzero positions come out ascending."""
    import torch
    n = keys.numel()
    first = torch.zeros(n, dtype=torch.bool, device=keys.device)
    nb = max(1, -(-n // (1 << 29)))
    for b in range(nb):
        sel = None if nb == 1 else torch.nonzero(torch.remainder(keys, nb) == b).squeeze(1)
        k = keys if sel is None else keys[sel]
        sk, perm = torch.sort(k, stable=True)
        head = torch.ones_like(sk, dtype=torch.bool)
        head[1:] = sk[1:] != sk[:-1]
        idx = perm[head]
        first[idx if sel is None else sel[idx]] = True
        del sel, k, sk, perm, head, idx
    count = int(first.sum().item())
    return torch.nonzero(first).squeeze(1)[:target], count


def _generate_kronecker_gpu(scale: int, avg_degree: int, seed: int, device) -> CsrGraph:
    """generate_kronecker on the GPU: the rounds' pairs by the native
    sm_100a kernel (grd_kronecker_keys, bit-exact PCG64 replay), first-
    occurrence deduplication and the CSR build by device sorts."""
    import torch
    dev = torch.device(device)
    n = 1 << scale
    target = (avg_degree * n) // 2
    cum = np.cumsum(np.asarray(KRONECKER_INITIATOR, dtype=np.float64))
    w = _pcg64_words(seed)
    state = (int(w[0]) << 64) | int(w[1])
    inc = (int(w[2]) << 64) | int(w[3])
    collected, unique_count = [], 0
    allk, first_idx = None, None
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        for _ in range(64):
            remaining = target - unique_count
            if remaining <= 0:
                break
            batch = max(4 * remaining, 1024)
            keys = torch.empty(batch, dtype=torch.int64, device=dev)
            jm, ja = _pcg_jump(batch, inc)
            words = _words(state, inc, jm, ja)
            _lib.check(_lib.lib().grd_kronecker_keys(scale, batch, _lib.ptr(words), _lib.ptr(cum),
                                                     keys.data_ptr(), stream), "kronecker_keys")
            m2, a2 = _pcg_jump(scale * batch, inc)
            state = (m2 * state + a2) & _M128
            collected.append(keys[keys >= 0])
            del keys
            allk = torch.cat(collected) if len(collected) > 1 else collected[0]
            first_idx, unique_count = _first_occurrence(allk, target)
        keys = allk[first_idx] if allk is not None else torch.zeros(0, dtype=torch.int64, device=dev)
        del collected, allk, first_idx
        lo, hi = keys // n, keys % n
        del keys
        # _csr_from_pairs(concat(lo, hi), concat(hi, lo)): stable by source
        src = torch.cat([lo, hi]).to(torch.int32)
        dst = torch.cat([hi, lo]).to(torch.int32)
        del lo, hi
        order = torch.sort(src, stable=True).indices
        dst_idx = dst[order].cpu().numpy()
        counts = torch.bincount(src, minlength=n)
        src_ptr = np.zeros(n + 1, dtype=np.int64)
        src_ptr[1:] = torch.cumsum(counts, 0).cpu().numpy()
    return CsrGraph(num_vertices=n, num_edges=int(dst_idx.size), src_ptr=src_ptr,
                    dst_idx=np.ascontiguousarray(dst_idx, dtype=np.int32))


def generate_kronecker(scale: int, avg_degree: int, seed: int,
                       num_threads: int | None = None, device=None) -> CsrGraph:
    """Symmetric power-law graph of 2**scale vertices (graph.py:158-209).

    Identical output to the reference for every (scale, avg_degree, seed):
    the native generator replays numpy's PCG64 draws level by level with
    jump-ahead per thread and keeps first-occurrence unique pairs.
    ``device="cuda"`` runs the rounds on the GPU (same graph, bit for bit).
    """
    if scale < 4:
        raise ValueError("scale must be at least 4")
    if avg_degree < 1:
        raise ValueError("avg_degree must be positive")
    if device is not None and str(device).startswith("cuda"):
        return _generate_kronecker_gpu(scale, avg_degree, seed, device)
    n = 1 << scale
    cap = 2 * ((avg_degree * n) // 2)
    src_ptr = np.empty(n + 1, dtype=np.int64)
    dst_idx = np.empty(max(cap, 1), dtype=np.int32)
    cum = np.cumsum(np.asarray(KRONECKER_INITIATOR, dtype=np.float64))
    words = _pcg64_words(seed)
    m = np.zeros(1, dtype=np.int64)
    threads = num_threads if num_threads is not None else (os.cpu_count() or 1)
    _lib.check(_lib.lib().grd_kronecker_generate(
        scale, avg_degree, _lib.ptr(words), _lib.ptr(cum), _lib.ptr(src_ptr),
        _lib.ptr(dst_idx), cap, _lib.ptr(m), threads), "generate_kronecker")
    edges = int(m[0])
    dst = dst_idx[:edges] if edges < dst_idx.size else dst_idx
    return CsrGraph(num_vertices=n, num_edges=edges, src_ptr=src_ptr,
                    dst_idx=np.ascontiguousarray(dst[:edges]))


def export_edge_list(graph: CsrGraph) -> np.ndarray:
    """int64 [E, 2] (source, destination) pairs in CSR order (graph.py:149-152)."""
    return np.stack([graph.edge_sources().astype(np.int64), graph.dst_idx.astype(np.int64)], axis=1)


@dataclass
class DegreeStats:
    """Out-degree histogram, mean (= |E| / |V| exactly), max and population variance."""

    histogram: np.ndarray
    mean: float
    max: int
    variance: float


def degree_stats(graph: CsrGraph) -> DegreeStats:
    """Summary of the out-degree distribution (graph.py:306-327)."""
    deg = graph.out_degrees()
    n = graph.num_vertices
    return DegreeStats(histogram=np.bincount(deg, minlength=1),
                       mean=graph.num_edges / n if n else 0.0,
                       max=int(deg.max()) if deg.size else 0,
                       variance=float(deg.var()) if deg.size else 0.0)
