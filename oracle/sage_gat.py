"""Float64 CPU oracles for the builder-defined GraphSAGE-mean and GAT layers.

TEST INFRASTRUCTURE (see oracle/__init__.py).  The reference has neither
layer (model.py:18 lists GCN modes only; SPEC.md:354 puts them out of scope),
so parity for these is UNPINNED by the reference: the conventions are the
builder's, following PyG defaults without biases, and this
oracle states them in plain torch float64 with autograd gradients
(validated by central differences in tests/test_oracle_sage_gat.py).

GraphSAGE-mean layer, weights W = [W_root | W_nbr] (d_in x 2 d_out):
    out_v = X_v W_root + (1/deg_v) sum_{u -> v} X_u W_nbr   (mean = 0 if deg_v = 0)
    ReLU on every layer but the last.
Epoch: masked mean softmax cross-entropy (model.py:102-122 semantics), one
SGD step W -= lr dW, trace records the pre-update loss / accuracy.
"""

from __future__ import annotations

import warnings

import numpy as np
import torch


def _graph(src_ptr, dst_idx):
    n = len(src_ptr) - 1
    src = torch.from_numpy(np.repeat(np.arange(n, dtype=np.int64), np.diff(src_ptr)))
    dst = torch.from_numpy(np.asarray(dst_idx, dtype=np.int64))
    deg = torch.bincount(dst, minlength=n).to(torch.float64)
    return n, src, dst, deg


def _mean_in(n, src, dst, deg, y):
    """(1/deg_v) sum_{u -> v} y_u as a sparse product (no E x d buffer)."""
    w = 1.0 / deg[dst]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")   # "sparse CSR support is in beta"
        a = torch.sparse_coo_tensor(torch.stack([dst, src]), w, (n, n)).coalesce().to_sparse_csr()
        return a @ y


def sage_forward(x, weights, graph):
    n, src, dst, deg = graph
    h = x
    for l, w in enumerate(weights):
        d_out = w.shape[1] // 2
        h_new = h @ w[:, :d_out] + _mean_in(n, src, dst, deg, h @ w[:, d_out:])
        h = torch.relu(h_new) if l < len(weights) - 1 else h_new
    return h


def masked_xent(logits, labels, mask):
    rows = torch.from_numpy(np.flatnonzero(mask))
    lab = torch.from_numpy(np.asarray(labels, dtype=np.int64))[rows]
    logp = torch.log_softmax(logits[rows], dim=1)
    loss = -logp[torch.arange(rows.numel()), lab].sum() / rows.numel()
    acc = float((logits[rows].argmax(dim=1) == lab).double().mean())
    return loss, acc


def train_sage(features, labels, mask, src_ptr, dst_idx, weights, epochs, lr):
    """Returns (weights, last gradients, trace) as float64 numpy."""
    graph = _graph(src_ptr, dst_idx)
    x = torch.from_numpy(np.asarray(features, dtype=np.float64))
    ws = [torch.tensor(np.asarray(w, dtype=np.float64), requires_grad=True) for w in weights]
    trace, grads = [], [np.zeros_like(np.asarray(w)) for w in weights]
    for epoch in range(epochs):
        loss, acc = masked_xent(sage_forward(x, ws, graph), labels, mask)
        trace.append((epoch, float(loss.detach()), acc))
        gs = torch.autograd.grad(loss, ws)
        with torch.no_grad():
            for w, g in zip(ws, gs):
                w -= lr * g
        grads = [g.numpy().copy() for g in gs]
    return [w.detach().numpy().copy() for w in ws], grads, trace


# ---------------------------------------------------------------------------
# GAT (builder-defined): per head h,
#   P = X W_h,  e_uv = LeakyReLU_0.2(a_src_h . P_u + a_dst_h . P_v) over
#   u in in(v) U {v},  alpha = softmax_u(e),  O_v = sum_u alpha_uv P_u;
#   hidden layers: ReLU(concat_h O), last layer: mean_h O.
# weights[l] = [[W], [a_src (flattened H x dh)], [a_dst]]  shape (d_in + 2, H dh)
# ---------------------------------------------------------------------------
NEG_SLOPE = 0.2


def gat_forward(x, weights, graph, heads):
    n, src, dst, _ = graph
    loops = torch.arange(n)
    s_all = torch.cat([src, loops])
    d_all = torch.cat([dst, loops])
    h = x
    for l, wp in enumerate(weights):
        d_in = wp.shape[0] - 2
        hd = wp.shape[1]
        dh = hd // heads
        W, a_s, a_d = wp[:d_in], wp[d_in].reshape(heads, dh), wp[d_in + 1].reshape(heads, dh)
        P = (h @ W).reshape(n, heads, dh)
        s = (P * a_s).sum(-1)
        t = (P * a_d).sum(-1)
        z = torch.nn.functional.leaky_relu(s[s_all] + t[d_all], NEG_SLOPE)
        zmax = torch.full((n, heads), -torch.inf, dtype=z.dtype).scatter_reduce(
            0, d_all[:, None].expand(-1, heads), z, reduce="amax", include_self=True)
        e = torch.exp(z - zmax[d_all])
        den = torch.zeros((n, heads), dtype=z.dtype).index_add(0, d_all, e)
        alpha = e / den[d_all]
        O = torch.zeros((n, heads, dh), dtype=z.dtype).index_add(0, d_all, alpha[..., None] * P[s_all])
        last = l == len(weights) - 1
        h = O.mean(dim=1) if last else torch.relu(O.reshape(n, hd))
    return h


def train_gat(features, labels, mask, src_ptr, dst_idx, weights, heads, epochs, lr):
    graph = _graph(src_ptr, dst_idx)
    x = torch.from_numpy(np.asarray(features, dtype=np.float64))
    ws = [torch.tensor(np.asarray(w, dtype=np.float64), requires_grad=True) for w in weights]
    trace, grads = [], []
    for epoch in range(epochs):
        loss, acc = masked_xent(gat_forward(x, ws, graph, heads), labels, mask)
        trace.append((epoch, float(loss.detach()), acc))
        gs = torch.autograd.grad(loss, ws)
        with torch.no_grad():
            for w, g in zip(ws, gs):
                w -= lr * g
        grads = [g.numpy().copy() for g in gs]
    return [w.detach().numpy().copy() for w in ws], grads, trace
