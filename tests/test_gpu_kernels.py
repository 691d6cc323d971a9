"""Kernel-level parity of the sm_100a library against float64 numpy."""

from __future__ import annotations

import os
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from conftest import rel_l2  # noqa: E402
from oracle import gcn  # noqa: E402
from paper_2605_11517_b200 import ops  # noqa: E402

DEV = "cuda"


def _dev(mat, width=None):
    mat = np.asarray(mat)
    t = ops.zeros_rows(mat.shape[0], mat.shape[1] if width is None else width, DEV)
    t[:, : mat.shape[1]] = torch.from_numpy(mat.astype(np.float32))
    return t


def _host(t, cols):
    return t[:, :cols].double().cpu().numpy()


def _random_csr(rng, n_rows, n_src, max_deg, hubs=()):
    deg = rng.integers(0, max_deg + 1, size=n_rows)
    for r, d in hubs:
        deg[r] = d
    ptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(deg, out=ptr[1:])
    idx = rng.integers(0, n_src, size=int(ptr[-1])).astype(np.int32)
    return ptr, idx


@pytest.mark.parametrize("width", [1, 3, 4, 10, 16, 33, 64, 100, 128, 256, 300])
def test_agg_sum_matches_numpy(width):
    rng = np.random.default_rng(width)
    n_rows, n_src = 700, 500
    ptr, idx = _random_csr(rng, n_rows, n_src, 40, hubs=[(5, 1000), (77, 129), (300, 5000)])
    out_idx = rng.permutation(n_rows).astype(np.int32)
    self_idx = rng.integers(-1, n_src, size=n_rows).astype(np.int32)
    y = rng.normal(size=(n_src, width))
    src_scale = rng.uniform(0.1, 1.0, size=n_src)
    post_scale = rng.uniform(0.1, 2.0, size=n_rows)
    spec = ops.AggSpec.build(ptr, idx, DEV, out_idx=out_idx, self_idx=self_idx)
    assert spec.n_segs > 0
    yt = _dev(y)
    out = ops.zeros_rows(n_rows, width, DEV)
    ss = torch.from_numpy(src_scale.astype(np.float32)).to(DEV)
    ps = torch.from_numpy(post_scale.astype(np.float32)).to(DEV)
    ops.agg_sum(spec, yt, out, width, src_scale=ss, post_scale=ps, post_div_deg=True, relu=True)
    want = np.zeros((n_rows, width))
    for r in range(n_rows):
        acc = (src_scale[idx[ptr[r]:ptr[r + 1]], None] * y[idx[ptr[r]:ptr[r + 1]]]).sum(axis=0)
        if self_idx[r] >= 0:
            acc = acc + src_scale[self_idx[r]] * y[self_idx[r]]
        acc = acc / (ptr[r + 1] - ptr[r] + 1) * post_scale[out_idx[r]]
        want[out_idx[r]] = np.maximum(acc, 0.0)
    got = _host(out, width)
    assert rel_l2(got, want) < 1e-6
    # deterministic: a second launch is bitwise identical (heavy rows included)
    out2 = ops.zeros_rows(n_rows, width, DEV)
    ops.agg_sum(spec, yt, out2, width, src_scale=ss, post_scale=ps, post_div_deg=True, relu=True)
    assert torch.equal(out, out2)
    # padding columns stay zero
    if out.shape[1] > width:
        assert not out[:, width:].any()


def test_agg_sum_mask_ref_and_defaults():
    rng = np.random.default_rng(0)
    n = 300
    ptr, idx = _random_csr(rng, n, n, 12, hubs=[(3, 600)])
    y = rng.normal(size=(n, 8))
    ref = rng.normal(size=(n, 8))
    spec = ops.AggSpec.build(ptr, idx, DEV)
    out = ops.zeros_rows(n, 8, DEV)
    ops.agg_sum(spec, _dev(y), out, 8, mask_ref=_dev(ref))
    want = np.stack([y[idx[ptr[r]:ptr[r + 1]]].sum(axis=0) + y[r] for r in range(n)])
    want = np.where(ref > 0, want, 0.0)
    assert rel_l2(_host(out, 8), want) < 1e-6


@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False)])
@pytest.mark.parametrize("m,n,k", [(1000, 64, 128), (257, 10, 64), (131, 47, 100), (64, 256, 300),
                                   (1300, 96, 64), (2000, 512, 100),
                                   (1300, 256, 70)])   # CTA pairs with an odd M-tile count
def test_gemm_matches_numpy(ta, tb, m, n, k):
    rng = np.random.default_rng(m + n + k)
    a = rng.normal(size=(k, m) if ta else (m, k))
    b = rng.normal(size=(n, k) if tb else (k, n))
    rs = rng.uniform(0.5, 1.5, size=m)
    em = rng.uniform(0.0, 2.0, size=(m, n))
    rr = rng.normal(size=(m, n))
    c = ops.zeros_rows(m, n, DEV)
    ops.gemm(_dev(a), _dev(b), c, m, n, k, trans_a=ta, trans_b=tb,
             row_scale=torch.from_numpy(rs.astype(np.float32)).to(DEV), elem_mul=_dev(em),
             relu_ref=_dev(rr))
    full = (a.T if ta else a) @ (b.T if tb else b)
    want = np.where(rr > 0, full * rs[:, None] * em, 0.0)
    assert rel_l2(_host(c, n), want) < 5e-6   # 3xTF32 on tcgen05


def test_gemm_relu_out_and_accumulate():
    rng = np.random.default_rng(1)
    a, b, c0 = rng.normal(size=(50, 12)), rng.normal(size=(12, 9)), rng.normal(size=(50, 9))
    c = _dev(c0)
    ops.gemm(_dev(a), _dev(b), c, 50, 9, 12, relu_out=True, accumulate=True)
    assert rel_l2(_host(c, 9), np.maximum(c0 + a @ b, 0)) < 5e-6   # relu(C + AB)


@pytest.mark.parametrize("m,n,k", [(128, 64, 131072), (64, 10, 5000), (100, 47, 1), (256, 256, 70000),
                                   (384, 10, 20000), (512, 96, 9000),
                                   (384, 128, 30000)])  # split-K on CTA pairs, odd M-tile count
def test_wgrad_sgd(m, n, k):
    rng = np.random.default_rng(k)
    a = rng.normal(size=(k, m)).astype(np.float32)
    b = rng.normal(size=(k, n)).astype(np.float32)
    w0 = rng.normal(size=(m, n))
    dw = ops.zeros_rows(m, n, DEV)
    w = _dev(w0)
    ops.wgrad_sgd(_dev(a), _dev(b), dw, m, n, k, w=w, lr=0.25)
    want = a.astype(np.float64).T @ b.astype(np.float64)
    # fp32 accumulation of up to 8192 zero-mean products per split-K chunk
    tol = 3e-5
    assert rel_l2(_host(dw, n), want) < tol
    assert rel_l2(_host(w, n), w0 - 0.25 * want) < tol
    dw2 = ops.zeros_rows(m, n, DEV)
    ops.wgrad_sgd(_dev(a), _dev(b), dw2, m, n, k)
    assert torch.equal(dw, dw2)
    ops.wgrad_sgd(_dev(a), _dev(b), dw2, m, n, k, accumulate=True)
    assert rel_l2(_host(dw2, n), 2 * want) < tol


@pytest.mark.parametrize("n,c", [(1000, 10), (777, 47), (300, 172), (64, 1)])
def test_softmax_xent(n, c):
    rng = np.random.default_rng(c)
    logits = rng.normal(size=(n, c)) * 3
    labels = rng.integers(0, c, size=n)
    mask = rng.random(n) < 0.5
    mask[0] = True
    loss, grad = gcn.softmax_xent(logits, labels, mask)
    acc = gcn.accuracy(logits, labels, mask)
    g = ops.zeros_rows(n, c, DEV)
    stats = torch.zeros(4, dtype=torch.float64, device=DEV)
    ops.softmax_xent(_dev(logits), n, c, torch.from_numpy(labels.astype(np.int32)).to(DEV),
                     torch.from_numpy(mask.astype(np.uint8)).to(DEV), int(mask.sum()), g, stats,
                     ops.loss_partials(n, DEV))
    s = stats.cpu().numpy()
    assert s[0] == pytest.approx(loss, rel=1e-5)
    assert s[1] == pytest.approx(acc, abs=1.5 / mask.sum())
    assert rel_l2(_host(g, c), grad) < 1e-5


def test_gather_and_scatter_rows():
    rng = np.random.default_rng(3)
    src = rng.normal(size=(100, 20))
    idx = rng.permutation(100)[:60].astype(np.int32)
    it = torch.from_numpy(idx).to(DEV)
    dst = ops.zeros_rows(60, 20, DEV)
    ops.gather_rows(_dev(src), it, dst, 20)
    np.testing.assert_array_equal(_host(dst, 20), src[idx].astype(np.float32))
    acc = _dev(np.ones((100, 20)))
    ops.scatter_add_rows(dst, it, acc, 20)
    want = np.ones((100, 20), dtype=np.float32)
    want[idx] += src[idx].astype(np.float32)
    np.testing.assert_array_equal(_host(acc, 20), want)


def test_rownorm_kernels():
    rng = np.random.default_rng(5)
    pre = rng.normal(size=(50, 7))
    pre[3] = 0.0
    out = ops.zeros_rows(50, 7, DEV)
    ops.rownorm_fwd(_dev(pre), out, 50, 7, relu=True)
    norms = np.linalg.norm(pre, axis=1, keepdims=True)
    unit = np.divide(pre, norms, out=np.zeros_like(pre), where=norms > 0)
    assert rel_l2(_host(out, 7), np.maximum(unit, 0)) < 1e-6
    g, a = rng.normal(size=(50, 7)), rng.normal(size=(50, 7))
    gp = ops.zeros_rows(50, 7, DEV)
    ops.rownorm_bwd(_dev(pre), _dev(g), gp, 50, 7, a_out=_dev(a))
    gy = g * (a > 0)
    want = np.divide(gy - unit * (unit * gy).sum(1, keepdims=True), norms,
                     out=np.zeros_like(gy), where=norms > 0)
    assert rel_l2(_host(gp, 7), want) < 1e-6


@pytest.mark.parametrize("heads,dh,scale,deg", [(2, 4, 9, 8), (2, 5, 9, 8), (4, 16, 9, 8), (1, 7, 9, 8),
                                                (4, 64, 12, 16), (8, 8, 12, 16), (3, 12, 11, 24)])
@pytest.mark.parametrize("use_st", [False, True])
def test_gat_kernels_match_autograd(heads, dh, scale, deg, use_st):
    """Edge softmax forward/backward, the weighted pulls and the score
    gradients against torch float64 autograd of the same layer (the larger
    graphs have hub rows above the 128-edge segmentation threshold); scores
    read from P_ext's columns or from the packed [s | t] table."""
    from paper_2605_11517_b200 import generate_kronecker
    from paper_2605_11517_b200.engine import DeviceGraph
    g = generate_kronecker(scale, deg, seed=2)
    n = g.num_vertices
    from paper_2605_11517_b200 import build_partition_plan, random_partition
    plan = build_partition_plan(g, random_partition(n, 3, 1), 3)
    dg = DeviceGraph(g, plan, DEV)
    rng = np.random.default_rng(heads * 10 + dh)
    dhp = (dh + 3) // 4 * 4
    hdp = heads * dhp
    P = rng.normal(size=(n, heads, dh))
    s = rng.normal(size=(n, heads))
    t = rng.normal(size=(n, heads))
    gO = rng.normal(size=(n, heads, dh))
    pext = np.zeros((n, hdp + 2 * heads))
    for h in range(heads):
        pext[:, h * dhp:h * dhp + dh] = P[:, h]
    pext[:, hdp:hdp + heads] = s
    pext[:, hdp + heads:] = t
    go = np.zeros((n, hdp))
    for h in range(heads):
        go[:, h * dhp:h * dhp + dh] = gO[:, h]
    E = dg.fwd.nnz
    alpha = torch.zeros(E * heads, device=DEV)
    alpha_self = torch.zeros(n * heads, device=DEV)
    pe = _dev(pext)
    st_tab = None
    if use_st:
        st_tab = ops.zeros_rows(n, 2 * heads, DEV)
        ops.gat_pack_scores(pe, n, heads, dhp, st_tab)
        pe[:, hdp:hdp + 2 * heads] = float("nan")   # the softmax must not read P_ext's scores
    ops.gat_softmax(dg.fwd, pe, heads, dhp, alpha, alpha_self, st=st_tab)
    if use_st:
        pe[:, hdp:hdp + 2 * heads] = torch.from_numpy(pext[:, hdp:]).float().to(DEV)   # bwd reads them
    O = ops.zeros_rows(n, hdp, DEV)
    ops.agg_sum(dg.fwd, pe[:, :hdp], O, hdp, edge_w=alpha, self_w=alpha_self, heads=heads, head_ld=dhp)
    dlt, dlt_s = torch.zeros_like(alpha), torch.zeros_like(alpha_self)
    gext = ops.zeros_rows(n, hdp + 2 * heads, DEV)
    god = _dev(go)
    ops.gat_softmax_bwd(dg.fwd, pe, heads, dhp, alpha, alpha_self, god, O, dlt, dlt_s, gext)
    perm = dg.out_to_in_perm()
    ops.agg_sum(dg.bwd, god, gext[:, :hdp], hdp, edge_w=alpha, edge_w_perm=perm, self_w=alpha_self,
                heads=heads, head_ld=dhp)
    ops.gat_src_grad(dg.bwd, heads, dhp, perm, dlt, dlt_s, gext)
    # reference
    src = torch.from_numpy(np.concatenate([g.edge_sources(), np.arange(n)]))
    dst = torch.from_numpy(np.concatenate([g.dst_idx.astype(np.int64), np.arange(n)]))
    Pt = torch.tensor(P, requires_grad=True)
    st = torch.tensor(s, requires_grad=True)
    tt = torch.tensor(t, requires_grad=True)
    z = torch.nn.functional.leaky_relu(st[src] + tt[dst], 0.2)
    zmax = torch.full((n, heads), -torch.inf, dtype=z.dtype).scatter_reduce(
        0, dst[:, None].expand(-1, heads), z, reduce="amax", include_self=True)
    e = torch.exp(z - zmax[dst])
    den = torch.zeros((n, heads), dtype=z.dtype).index_add(0, dst, e)
    al = e / den[dst]
    Or = torch.zeros((n, heads, dh), dtype=z.dtype).index_add(0, dst, al[..., None] * Pt[src])
    (Or * torch.from_numpy(gO)).sum().backward()
    Og = _host(O, hdp).reshape(n, heads, dhp)[:, :, :dh]
    assert rel_l2(Og, Or.detach().numpy()) < 1e-6
    ge = _host(gext, hdp + 2 * heads)
    dP = ge[:, :hdp].reshape(n, heads, dhp)[:, :, :dh]
    assert rel_l2(dP, Pt.grad.numpy()) < 1e-6
    assert rel_l2(ge[:, hdp:hdp + heads], st.grad.numpy()) < 1e-5
    assert rel_l2(ge[:, hdp + heads:], tt.grad.numpy()) < 1e-5
    # the fused pull backward (one gO_v gather per edge): dP, the score
    # gradients against autograd, delta against the edge backward's (light
    # rows sum in the unfused pull's order; its heavy segments stride their
    # edges over lane groups, so those rows round differently)
    cdot = torch.zeros(n * heads, device=DEV)
    ops.gat_row_dots(god, O, n, heads, dhp, cdot)
    dlt2, dlt2_s = torch.zeros_like(alpha), torch.zeros_like(alpha_self)
    gext2 = ops.zeros_rows(n, hdp + 2 * heads, DEV)
    ops.gat_pull_bwd(dg.bwd, pe, heads, dhp, perm, alpha, alpha_self, god, cdot, dlt2, dlt2_s, gext2,
                     st=st_tab)
    ops.gat_dst_grad(dg.fwd, heads, dhp, dlt2, dlt2_s, gext2)
    ge2 = _host(gext2, hdp + 2 * heads)
    dP2 = ge2[:, :hdp].reshape(n, heads, dhp)[:, :, :dh]
    assert rel_l2(dP2, Pt.grad.numpy()) < 1e-6
    assert rel_l2(ge2[:, :hdp], ge[:, :hdp]) < 1e-6
    assert rel_l2(ge2[:, hdp:hdp + heads], st.grad.numpy()) < 1e-5
    assert rel_l2(ge2[:, hdp + heads:], tt.grad.numpy()) < 1e-5
    assert rel_l2(dlt2.cpu().numpy(), dlt.cpu().numpy()) < 1e-6
    assert rel_l2(dlt2_s.cpu().numpy(), dlt_s.cpu().numpy()) < 1e-6


def test_gemm_bf16x3_opt_in_path():
    """The opt-in bf16x3 forward GEMM (GRD_GEMM_PREC=bf16x3, read once per
    process, so it runs in a child): ~4e-6 against float64 on the epilogue
    variants; the product default stays 3xTF32 (grd_gemm_tc.cu explains why)."""
    import subprocess
    import sys
    code = r'''
import numpy as np, torch
from paper_2605_11517_b200 import ops
rng = np.random.default_rng(3)
dev = "cuda"
def pad(x):
    t = ops.zeros_rows(x.shape[0], x.shape[1], dev); t[:, :x.shape[1]] = torch.from_numpy(x).float(); return t
worst = 0.0
for m, n, k, tb in [(1000, 47, 13, 0), (777, 100, 300, 1), (5000, 256, 256, 0), (300, 512, 70, 0)]:
    a = rng.normal(size=(m, k)); b = rng.normal(size=(n, k) if tb else (k, n)); c0 = rng.normal(size=(m, n))
    rr = rng.normal(size=(m, n))
    c = pad(c0)
    acc = k <= 128          # (accumulating launches stay 3xTF32; check both entries)
    if not acc:
        c = pad(np.zeros_like(c0))
    ops.gemm(pad(a), pad(b), c, m, n, k, trans_b=bool(tb), relu_ref=pad(rr), accumulate=acc)
    want = np.where(rr > 0, (c0 if acc else 0.0) + a @ (b.T if tb else b), 0.0)
    got = c[:, :n].double().cpu().numpy()
    worst = max(worst, np.linalg.norm(got - want) / np.linalg.norm(want))
print(worst)
'''
    env = dict(os.environ, GRD_GEMM_PREC="bf16x3")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         cwd=str(Path(__file__).resolve().parents[1]), timeout=300)
    assert out.returncode == 0, out.stderr
    assert float(out.stdout.strip().splitlines()[-1]) < 2e-5


@pytest.mark.parametrize("m,n2,k", [(1000, 48, 100), (2000, 256, 96), (300, 12, 7)])
def test_gemm_split_output(m, n2, k):
    """Columns >= split of one GEMM land in a second dense matrix (the
    GraphSAGE [Y_root | Y_nbr] planes)."""
    rng = np.random.default_rng(m + n2)
    a = rng.normal(size=(m, k))
    b = rng.normal(size=(k, 2 * n2))
    c1 = ops.zeros_rows(m, n2, DEV)
    c2 = ops.zeros_rows(m, n2, DEV)
    ldb = (n2 + 3) // 4 * 4
    bp = np.zeros((k, 2 * ldb))
    bp[:, :n2], bp[:, ldb:ldb + n2] = b[:, :n2], b[:, n2:]
    ops.gemm(_dev(a), _dev(bp), c1, m, 2 * ldb, k, c2=c2, split=ldb, relu_out=True)
    full = np.maximum(a @ b, 0)
    assert rel_l2(_host(c1, n2), full[:, :n2]) < 5e-6
    assert rel_l2(_host(c2, n2), full[:, n2:]) < 5e-6


@pytest.mark.parametrize("heads", [1, 2, 4, 8])
def test_gat_softmax_small_tail(heads):
    """The low-degree tail at 4 lanes per row (AggSpec.n_small) gives the
    same attention as the warp-per-row kernel, also when forced onto rows
    longer than it is meant for (hub rows included)."""
    from paper_2605_11517_b200 import generate_kronecker, build_partition_plan, random_partition
    from paper_2605_11517_b200.engine import DeviceGraph
    g = generate_kronecker(12, 16, seed=5)
    n = g.num_vertices
    dg = DeviceGraph(g, build_partition_plan(g, random_partition(n, 2, 1), 2), DEV)
    spec = dg.fwd
    assert 0 < spec.n_small < spec.n_rows
    dhp = 4
    hdp = heads * dhp
    rng = np.random.default_rng(heads)
    pe = _dev(rng.normal(size=(n, hdp + 2 * heads)))
    E = spec.nnz
    out = {}
    default = (spec.n_small, spec.n_mid)
    assert spec.n_mid > 0
    cases = {"warp": (0, 0), "default": default, "small_all": (spec.n_rows, 0),
             "mid_all": (0, spec.n_rows), "split": (spec.n_rows // 2, spec.n_rows - spec.n_rows // 2)}
    for name, (ks, km) in cases.items():
        spec.n_small, spec.n_mid = ks, km
        alpha = torch.zeros(E * heads, device=DEV)
        alpha_self = torch.zeros(n * heads, device=DEV)
        ops.gat_softmax(spec, pe, heads, dhp, alpha, alpha_self)
        out[name] = (alpha.cpu(), alpha_self.cpu())
    spec.n_small, spec.n_mid = default
    for name in cases:
        assert torch.allclose(out[name][0], out["warp"][0], rtol=1e-5, atol=1e-7), name
        assert torch.allclose(out[name][1], out["warp"][1], rtol=1e-5, atol=1e-7), name
    # every row's attention sums to one
    s = out["small_all"][1].view(n, heads).double()
    ptr = spec.row_ptr.cpu().numpy()
    oi = spec.out_idx.cpu().numpy() if spec.out_idx is not None else np.arange(n)
    a = out["small_all"][0].view(E, heads).double().numpy()
    rs = np.add.reduceat(np.vstack([a, np.zeros((1, heads))]), ptr[:-1], axis=0)[:n]
    rs[ptr[1:] == ptr[:-1]] = 0.0
    tot = s.numpy()[oi] + rs
    assert np.allclose(tot, 1.0, atol=1e-5)


@pytest.mark.parametrize("heads", [1, 4, 8])
def test_gat_src_grad_lane_groups(heads):
    """ds_u from the lane-grouped low-degree rows equals the warp-per-row
    sums (any split of the rows between the tiers) and a float64 reference."""
    from paper_2605_11517_b200 import generate_kronecker, build_partition_plan, random_partition
    from paper_2605_11517_b200.engine import DeviceGraph
    g = generate_kronecker(12, 16, seed=7)
    n = g.num_vertices
    dg = DeviceGraph(g, build_partition_plan(g, random_partition(n, 2, 1), 2), DEV)
    spec = dg.bwd
    assert spec.n_small > 0 and spec.n_mid > 0
    dhp = 4
    hdp = heads * dhp
    E = spec.nnz
    rng = np.random.default_rng(heads)
    delta = rng.normal(size=(E, heads))
    dself = rng.normal(size=(n, heads))
    d_t = torch.from_numpy(delta).float().reshape(-1).to(DEV)
    ds_t = torch.from_numpy(dself).float().reshape(-1).to(DEV)
    perm = dg.out_to_in_perm()
    default = (spec.n_small, spec.n_mid)
    cases = {"warp": (0, 0), "default": default, "small_all": (spec.n_rows, 0),
             "mid_all": (0, spec.n_rows)}
    res = {}
    for name, (ks, km) in cases.items():
        spec.n_small, spec.n_mid = ks, km
        gext = ops.zeros_rows(n, hdp + 2 * heads, DEV)
        ops.gat_src_grad(spec, heads, dhp, perm, d_t, ds_t, gext)
        res[name] = gext[:, hdp:hdp + heads].cpu().double().numpy()
    spec.n_small, spec.n_mid = default
    # float64 reference: ds_u = sum over out-edges of delta + self
    # float64 host sums over the transposed CSR (perm: its edges -> delta rows)
    ptr = spec.row_ptr.cpu().numpy()
    pm = perm.cpu().numpy()[:E].astype(np.int64)
    rows = np.repeat(np.arange(spec.n_rows), np.diff(ptr))
    per_row = np.zeros((spec.n_rows, heads))
    np.add.at(per_row, rows, delta[pm])
    oi = spec.out_idx.cpu().numpy() if spec.out_idx is not None else np.arange(n)
    ref = dself.copy()
    ref[oi] += per_row
    for name in cases:
        assert np.allclose(res[name], res["warp"], rtol=1e-5, atol=1e-5), name
        assert np.allclose(res[name], ref, rtol=1e-4, atol=1e-4), name


@pytest.mark.parametrize("tma", ["1", "0"])
@pytest.mark.parametrize("m,n,k", [(1000, 47, 128), (300, 128, 64), (2050, 256, 96)])
def test_gemm_output_columns_and_rows_exact(tma, m, n, k, monkeypatch):
    """The epilogue writes exactly rows [0, m) and columns [0, round_up(n, 4))
    of C — padding columns as zeros, nothing past them, nothing below row m —
    whether chunks leave by per-row stores or by TMA through shared memory
    (GRD_GEMM_TMA_STORE; read once per process, so a child process runs the
    opposite setting)."""
    import subprocess
    import sys
    code = f"""
import sys; sys.path.insert(0, {str(Path(__file__).resolve().parents[1])!r})
import numpy as np, torch
from paper_2605_11517_b200 import ops
m, n, k = {m}, {n}, {k}
rng = np.random.default_rng(3)
a = ops.zeros_rows(m, k, 'cuda'); a[:, :k] = torch.from_numpy(rng.normal(size=(m, k)).astype(np.float32)).cuda()
b = ops.zeros_rows(k, n, 'cuda'); b[:, :n] = torch.from_numpy(rng.normal(size=(k, n)).astype(np.float32)).cuda()
npad = (n + 3) // 4 * 4
big = torch.full((m + 37, npad + 8), 7.0, device='cuda')
c = big[:m, :]
ops.gemm(a, b, c, m, n, k)
want = a[:, :k].double() @ b[:, :n].double()
err = float((c[:, :n].double() - want).norm() / want.norm())
assert err < 5e-6, err
assert torch.all(c[:, n:npad] == 0), 'padding columns'
assert torch.all(big[:m, npad:] == 7.0), 'columns past the padding'
assert torch.all(big[m:] == 7.0), 'rows past m'
print('ok')
"""
    env = dict(os.environ, GRD_GEMM_TMA_STORE=tma)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("loring", ["0", "1", "2", "3"])
def test_gemm_lo_ring_depths(loring):
    """The lo-tile ring (GRD_GEMM_LORING slots; 0 = lo tiles inside every
    stage) and the epilogue's staging tiles per warp (GRD_GEMM_EPI_BUFS) on
    every operand mode: K-major A with the packed weight resident
    or staged, trans_b, CTA pairs (256-wide tiles), MN-major weight
    gradients with split-K and CTA pairs; with and without TMA-store
    epilogues.  Read once per process, so each setting runs in a child."""
    import subprocess
    import sys
    code = f"""
import sys; sys.path.insert(0, {str(Path(__file__).resolve().parents[1])!r})
import numpy as np, torch
from paper_2605_11517_b200 import ops
rng = np.random.default_rng(7)
def dev(x): 
    t = ops.zeros_rows(x.shape[0], x.shape[1], 'cuda'); t[:, :x.shape[1]] = torch.from_numpy(x.astype(np.float32)).cuda(); return t
for m, n, k, tb in [(70000, 128, 128, 0), (5000, 172, 128, 0), (5000, 128, 172, 1), (9000, 256, 256, 0),
                    (3000, 47, 300, 0), (40000, 512, 100, 0), (1300, 256, 70, 1)]:
    a = rng.normal(size=(m, k)); b = rng.normal(size=(n, k) if tb else (k, n))
    rs = rng.uniform(0.5, 1.5, size=m).astype(np.float32)
    c = ops.zeros_rows(m, n, 'cuda')
    ops.gemm(dev(a), dev(b), c, m, n, k, trans_b=bool(tb), row_scale=torch.from_numpy(rs).cuda())
    want = (a @ (b.T if tb else b)) * rs[:, None]
    got = c[:, :n].double().cpu().numpy()
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err < 5e-6, (m, n, k, tb, err)
for m, n, k in [(128, 128, 200000), (128, 172, 50000), (256, 256, 70000), (100, 47, 3000), (384, 128, 30000)]:
    a = rng.normal(size=(k, m)).astype(np.float32); b = rng.normal(size=(k, n)).astype(np.float32)
    dw = ops.zeros_rows(m, n, 'cuda')
    ops.wgrad_sgd(dev(a), dev(b), dw, m, n, k)
    want = a.astype(np.float64).T @ b.astype(np.float64)
    got = dw[:, :n].double().cpu().numpy()
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err < 5e-6, (m, n, k, err)
print('ok')
"""
    # TMA-store epilogue with two / one staging tiles per warp, and per-row stores
    for tma, ebufs in (("1", "2"), ("1", "1"), ("0", "2")):
        env = dict(os.environ, GRD_GEMM_LORING=loring, GRD_GEMM_TMA_STORE=tma, GRD_GEMM_EPI_BUFS=ebufs)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and "ok" in r.stdout, (tma, ebufs, r.stdout + r.stderr)
