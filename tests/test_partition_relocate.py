"""The GPU partitioner's relocation step (partition._relocate_sorted: one
packed-key sort + segment arithmetic) against the oracle's restatement of
_relocate_kernel (partition.py:203-251), on CPU tensors: every iteration of
a full partitioner run, with the oracle's own analysis producing the
preference slots, moves exactly the same vertices."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import partition as op  # noqa: E402
from paper_2605_11517_b200 import generate_kronecker  # noqa: E402
from paper_2605_11517_b200.partition import _relocate_sorted  # noqa: E402


@pytest.mark.parametrize("scale,deg,P,depth,beta", [
    (7, 6, 3, 2, 1.1), (8, 8, 4, 3, 1.1), (9, 4, 6, 2, 1.3), (8, 10, 16, 2, 1.2), (7, 12, 5, 4, 1.5),
])
def test_relocate_sorted_matches_oracle(scale, deg, P, depth, beta):
    g = generate_kronecker(scale, deg, seed=scale)
    n = g.num_vertices
    adj = [list(g.dst_idx[g.src_ptr[v]:g.src_ptr[v + 1]]) for v in range(n)]
    labels = op.random_labels(n, P, scale + 2)
    denom = 1.1 * n / P
    cap = int(np.floor(beta * n / P + 1e-9))
    moved_total = 0
    for _ in range(6):
        sizes = np.bincount(labels, minlength=P).astype(np.int64)
        _, prefs, cand = op._analyze(adj, labels, sizes, denom, P, depth)
        if cand == 0:
            break
        want = labels.copy()
        op._relocate(prefs, want, sizes, cap, P)
        got = torch.from_numpy(labels.astype(np.int32))
        _relocate_sorted(torch.tensor(prefs, dtype=torch.int32).T.contiguous(), got,
                         torch.from_numpy(sizes), P, cap)
        np.testing.assert_array_equal(got.numpy(), want)
        moved_total += int(np.count_nonzero(want != labels))
        labels = want
    assert moved_total > 0
