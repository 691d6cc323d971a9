"""The builder-defined GraphSAGE / GAT oracles (no reference exists; parity
unpinned by the reference): checked against hand-written loops and central
differences in float64."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import sage_gat
from paper_2605_11517_b200 import create_model, generate_kronecker, make_random_dataset


def _loop_sage(x, w, src_ptr, dst_idx, last):
    n, d_out = x.shape[0], w.shape[1] // 2
    ins = {v: [] for v in range(n)}
    for u in range(n):
        for v in dst_idx[src_ptr[u]:src_ptr[u + 1]]:
            ins[int(v)].append(u)
    out = np.zeros((n, d_out))
    for v in range(n):
        acc = x[v] @ w[:, :d_out]
        if ins[v]:
            acc = acc + np.mean([x[u] for u in ins[v]], axis=0) @ w[:, d_out:]
        out[v] = acc if last else np.maximum(acc, 0)
    return out


def test_sage_forward_matches_loops():
    g = generate_kronecker(6, 4, seed=1)
    rng = np.random.default_rng(0)
    x = rng.normal(size=(g.num_vertices, 5))
    w = rng.normal(size=(5, 6))
    got = sage_gat.sage_forward(torch.from_numpy(x), [torch.from_numpy(w)],
                                sage_gat._graph(g.src_ptr, g.dst_idx)).numpy()
    np.testing.assert_allclose(got, _loop_sage(x, w, g.src_ptr, g.dst_idx, True), rtol=1e-12, atol=1e-12)


def test_sage_gradients_central_differences():
    g = generate_kronecker(6, 5, seed=2)
    ds = make_random_dataset(g, feature_dim=4, num_classes=3, seed=3)
    model = create_model(4, 3, num_layers=2, hidden_dim=5, seed=4, aggregation_mode="sage_mean")
    graph = sage_gat._graph(g.src_ptr, g.dst_idx)
    x = torch.from_numpy(ds.features)
    ws = [torch.tensor(w, requires_grad=True) for w in model.weights]
    loss, _ = sage_gat.masked_xent(sage_gat.sage_forward(x, ws, graph), ds.labels, ds.train_mask)
    grads = torch.autograd.grad(loss, ws)
    rng = np.random.default_rng(1)
    eps = 1e-6
    for li, w in enumerate(model.weights):
        for _ in range(6):
            i, j = rng.integers(w.shape[0]), rng.integers(w.shape[1])
            vals = []
            for sgn in (1, -1):
                ww = [t.copy() for t in model.weights]
                ww[li][i, j] += sgn * eps
                lo, _ = sage_gat.masked_xent(
                    sage_gat.sage_forward(x, [torch.from_numpy(t) for t in ww], graph),
                    ds.labels, ds.train_mask)
                vals.append(float(lo))
            fd = (vals[0] - vals[1]) / (2 * eps)
            assert fd == pytest.approx(float(grads[li][i, j]), rel=1e-5, abs=1e-9)


def _loop_gat(x, wp, src_ptr, dst_idx, heads, last):
    n, d_in = x.shape[0], wp.shape[0] - 2
    dh = wp.shape[1] // heads
    W, a_s, a_d = wp[:d_in], wp[d_in].reshape(heads, dh), wp[d_in + 1].reshape(heads, dh)
    P = (x @ W).reshape(n, heads, dh)
    ins = {v: [v] for v in range(n)}
    for u in range(n):
        for v in dst_idx[src_ptr[u]:src_ptr[u + 1]]:
            ins[int(v)].insert(-1, u)
    out = np.zeros((n, heads, dh))
    for v in range(n):
        for h in range(heads):
            z = np.array([P[u, h] @ a_s[h] + P[v, h] @ a_d[h] for u in ins[v]])
            z = np.where(z > 0, z, 0.2 * z)
            al = np.exp(z - z.max())
            al /= al.sum()
            out[v, h] = sum(a * P[u, h] for a, u in zip(al, ins[v]))
    return out.mean(axis=1) if last else np.maximum(out.reshape(n, heads * dh), 0)


def test_gat_forward_matches_loops():
    g = generate_kronecker(6, 4, seed=1)
    rng = np.random.default_rng(0)
    x = rng.normal(size=(g.num_vertices, 5))
    for last in (False, True):
        wp = rng.normal(size=(7, 6)) * 0.5
        got = sage_gat.gat_forward(torch.from_numpy(x), [torch.from_numpy(wp)] if last else
                                   [torch.from_numpy(wp), torch.zeros(8, 2, dtype=torch.float64)][:1],
                                   sage_gat._graph(g.src_ptr, g.dst_idx), 2).numpy()
        want = _loop_gat(x, wp, g.src_ptr, g.dst_idx, 2, last=True)
        if last:
            np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-12)


def test_gat_gradients_central_differences():
    g = generate_kronecker(6, 5, seed=2)
    ds = make_random_dataset(g, feature_dim=4, num_classes=3, seed=3)
    model = create_model(4, 3, num_layers=2, hidden_dim=4, seed=4, aggregation_mode="gat", heads=2)
    graph = sage_gat._graph(g.src_ptr, g.dst_idx)
    x = torch.from_numpy(ds.features)
    ws = [torch.tensor(w, requires_grad=True) for w in model.weights]
    loss, _ = sage_gat.masked_xent(sage_gat.gat_forward(x, ws, graph, 2), ds.labels, ds.train_mask)
    grads = torch.autograd.grad(loss, ws)
    rng = np.random.default_rng(1)
    eps = 1e-6
    for li, w in enumerate(model.weights):
        for _ in range(6):
            i, j = rng.integers(w.shape[0]), rng.integers(w.shape[1])
            vals = []
            for sgn in (1, -1):
                ww = [t.copy() for t in model.weights]
                ww[li][i, j] += sgn * eps
                lo, _ = sage_gat.masked_xent(
                    sage_gat.gat_forward(x, [torch.from_numpy(t) for t in ww], graph, 2),
                    ds.labels, ds.train_mask)
                vals.append(float(lo))
            fd = (vals[0] - vals[1]) / (2 * eps)
            assert fd == pytest.approx(float(grads[li][i, j]), rel=1e-5, abs=1e-9)
