"""Float64 CPU restatement of the reference GCN layer, loss and epoch.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Each function names the
reference lines it restates; the arithmetic primitives are the same numpy
calls the reference relies on (fancy-index gathers, ``np.add.reduceat``
segment sums, ``np.add.at`` scatter, OpenBLAS matmul), so this module is
also the CPU baseline ``bench.py`` times.

A topology is any object with the reference's PartitionTopology fields
(plan.py:21-48): targets, gather_map, tgt_ptr, src_pos, edge_local_target,
self_pos, target_indeg, gather_indeg.
"""

from __future__ import annotations

import numpy as np

MEAN, SYM = "mean_self_loop", "symmetric_norm"


def _edge_coeff(topo) -> np.ndarray:
    """1/sqrt((d_u+1)(d_v+1)) per edge (training.py:54-57)."""
    du = topo.gather_indeg[topo.src_pos] + 1.0
    dv = topo.target_indeg[topo.edge_local_target] + 1.0
    return 1.0 / np.sqrt(du * dv)


def segment_sums(rows: np.ndarray, ptr: np.ndarray, count: int) -> np.ndarray:
    """Sum of rows[ptr[i]:ptr[i+1]] per segment; empty segments give 0
    (training.py:38-45, np.add.reduceat over the non-empty starts)."""
    res = np.zeros((count, rows.shape[1]))
    live = np.flatnonzero(ptr[1:] > ptr[:-1])
    if live.size:
        res[live] = np.add.reduceat(rows, ptr[live], axis=0)
    return res


def aggregate(ga: np.ndarray, topo, mode: str) -> np.ndarray:
    """Neighbour sum plus the implicit self row (training.py:48-58)."""
    nbr = ga[topo.src_pos]
    own = ga[topo.self_pos]
    if mode == SYM:
        nbr = nbr * _edge_coeff(topo)[:, None]
        own = own * (1.0 / (topo.target_indeg + 1.0))[:, None]
    return segment_sums(nbr, topo.tgt_ptr, len(topo.targets)) + own


def normalize(agg: np.ndarray, topo, mode: str) -> np.ndarray:
    """Mean mode divides by (in-degree + 1); sym is pre-weighted (:61-65)."""
    if mode == MEAN:
        return agg / (topo.target_indeg + 1.0)[:, None]
    return agg


def _unit_rows(pre: np.ndarray):
    norms = np.sqrt((pre * pre).sum(axis=1, keepdims=True))
    unit = np.zeros_like(pre)
    np.divide(pre, norms, out=unit, where=norms > 0)
    return unit, norms


def layer_apply(weight, ga, topo, mode, row_normalize=False, last=False):
    """(out, pre) of one layer on gathered rows (training.py:72-83)."""
    pre = normalize(aggregate(ga, topo, mode), topo, mode) @ weight
    out = _unit_rows(pre)[0] if row_normalize else pre
    if not last:
        out = np.maximum(out, 0.0)
    return out, pre


def layer_backward(weight, ga, a_out, grad_out, topo, mode, row_normalize=False, last=False):
    """(grad_GA, grad_W) of one layer from regathered rows (training.py:103-143)."""
    norm = normalize(aggregate(ga, topo, mode), topo, mode)
    gy = grad_out if last else grad_out * (a_out > 0)
    if row_normalize:
        unit, norms = _unit_rows(norm @ weight)
        gp = np.zeros_like(gy)
        np.divide(gy - unit * (unit * gy).sum(axis=1, keepdims=True), norms, out=gp,
                  where=norms > 0)
    else:
        gp = gy
    grad_w = norm.T @ gp
    gn = gp @ weight.T
    if mode == MEAN:
        per_target = gn / (topo.target_indeg + 1.0)[:, None]
        edge_vals = per_target[topo.edge_local_target]
        self_vals = per_target
    else:
        edge_vals = gn[topo.edge_local_target] * _edge_coeff(topo)[:, None]
        self_vals = gn * (1.0 / (topo.target_indeg + 1.0))[:, None]
    grad_ga = np.zeros_like(ga)
    np.add.at(grad_ga, topo.src_pos, edge_vals)     # sequential in edge order
    grad_ga[topo.self_pos] += self_vals
    return grad_ga, grad_w


def softmax_xent(logits, labels, mask):
    """Masked mean cross entropy and d/dlogits (model.py:102-122)."""
    rows = np.flatnonzero(mask)
    if rows.size == 0:
        raise ValueError("loss mask selects no vertices")
    with np.errstate(over="ignore", invalid="ignore", divide="ignore"):
        z = logits - logits.max(axis=1, keepdims=True)
        e = np.exp(z)
        prob = e / e.sum(axis=1, keepdims=True)
        loss = float(-np.sum(np.log(prob[rows, labels[rows]])) / rows.size)
    grad = np.zeros_like(logits)
    grad[rows] = prob[rows]
    grad[rows, labels[rows]] -= 1.0
    grad /= rows.size
    return loss, grad


def accuracy(logits, labels, mask) -> float:
    """Masked argmax accuracy (model.py:125-129)."""
    rows = np.flatnonzero(mask)
    return float(np.mean(np.argmax(logits[rows], axis=1) == labels[rows]))


def dropout_keep(rate, seed, epoch, layer, shape):
    """Seeded keep-mask / keep (training.py:178-185)."""
    if rate == 0.0:
        return None
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed, spawn_key=(epoch, layer))))
    return (gen.random(shape) < 1.0 - rate) / (1.0 - rate)


def train_partitioned(features, labels, mask, topologies, weights, epochs, lr, mode=MEAN,
                      row_normalize=False, dropout_rate=0.0, dropout_seed=0, order=None,
                      probe=None, snapshots=False):
    """The partition-wise epoch loop of training.py:259-358, f64.

    Returns (weights, last weight gradients, trace).  Forward/backward visit
    partitions in ``order(layer, phase)`` (default ascending); gradient
    accumulation always replays ascending partition ids.
    """
    W = [np.array(w, dtype=np.float64, copy=True) for w in weights]
    L = len(W)
    n = features.shape[0]
    P = len(topologies)
    order = order or (lambda layer, phase: range(P))
    trace, grads = [], [np.zeros_like(w) for w in W]
    for epoch in range(epochs):
        acts = [features]
        kept = {}
        for l in range(L):
            keep = dropout_keep(dropout_rate, dropout_seed, epoch, l, (n, W[l].shape[0]))
            out = np.zeros((n, W[l].shape[1]))
            for q in order(l, "forward"):
                t = topologies[q]
                ga = acts[l][t.gather_map]
                if keep is not None:
                    ga = ga * keep[t.gather_map]
                out[t.targets] = layer_apply(W[l], ga, t, mode, row_normalize, l == L - 1)[0]
                if snapshots:
                    kept[(l, q)] = ga
            acts.append(out)
        loss, grad = softmax_xent(acts[-1], labels, mask)
        if not np.isfinite(loss):
            raise ValueError(f"non-finite loss {loss} at epoch {epoch}")
        trace.append((epoch, loss, accuracy(acts[-1], labels, mask)))
        grads = [np.zeros_like(w) for w in W]
        for l in reversed(range(L)):
            keep = dropout_keep(dropout_rate, dropout_seed, epoch, l, (n, W[l].shape[0]))
            res = {}
            for q in order(l, "backward"):
                t = topologies[q]
                if snapshots:
                    ga = kept.pop((l, q))
                else:
                    ga = acts[l][t.gather_map]
                    if keep is not None:
                        ga = ga * keep[t.gather_map]
                res[q] = layer_backward(W[l], ga, acts[l + 1][t.targets], grad[t.targets], t, mode,
                                        row_normalize, l == L - 1)
            back = np.zeros((n, W[l].shape[0])) if l > 0 else None
            for q in range(P):
                g_ga, g_w = res[q]
                if probe is not None:
                    probe(epoch, l, q, g_ga, g_w)
                grads[l] += g_w
                if l > 0:
                    back[topologies[q].gather_map] += g_ga
            if l > 0 and keep is not None:
                back *= keep
            grad = back
        for w, g in zip(W, grads):
            w -= lr * g
    return W, grads, trace
