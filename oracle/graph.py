"""Kronecker generator and CSR construction restated (numpy).

TEST INFRASTRUCTURE (see oracle/__init__.py).  Restates graph.py:87-146
(first-occurrence dedup, stable per-source order) and graph.py:158-209
(recursive quadrant picks from the (0.57, 0.19, 0.19, 0.05) initiator drawn
level by level from one PCG64 stream, self-loops dropped, first-occurrence
unique pairs truncated to avg_degree * n / 2, both directions stored).
"""

from __future__ import annotations

import numpy as np


def csr_from_pairs(src, dst, n):
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    seen, keep = set(), []
    for i, key in enumerate(zip(src.tolist(), dst.tolist())):
        if key not in seen:
            seen.add(key)
            keep.append(i)
    src, dst = src[keep], dst[keep]
    order = np.argsort(src, kind="stable")
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=ptr[1:])
    return ptr, dst[order].astype(np.int32)


def kronecker(scale, avg_degree, seed):
    n = 1 << scale
    want = avg_degree * n // 2
    cum = np.cumsum([0.57, 0.19, 0.19, 0.05])
    gen = np.random.Generator(np.random.PCG64(seed))
    keys, seen = [], set()
    for _ in range(64):
        if len(seen) >= want:
            break
        batch = max(4 * (want - len(seen)), 1024)
        a = np.zeros(batch, dtype=np.int64)
        b = np.zeros(batch, dtype=np.int64)
        for _level in range(scale):
            quad = np.searchsorted(cum, gen.random(batch), side="right")
            a = (a << 1) | (quad >> 1)
            b = (b << 1) | (quad & 1)
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        for k in (lo * n + hi)[lo != hi].tolist():
            if k not in seen:
                seen.add(k)
                keys.append(k)
    keys = np.asarray(keys[:want], dtype=np.int64)
    lo, hi = keys // n, keys % n
    return csr_from_pairs(np.concatenate([lo, hi]), np.concatenate([hi, lo]), n)
