"""Layer-streaming engine (stream.py) for graphs whose layers exceed HBM:
same epoch as the HBM-resident engine and the pinned oracle, with small row
chunks so every chunked path (split heavy rows, chunk-local outputs with
global self rows, double-buffered host streaming, host-kept deep layers)
runs on a small graph.

Tolerance: weights and weight gradients within 1e-4 L2-relative of the
oracle (north star) and within 1e-5 of the resident engine (same kernels,
different split-K summation order); loss within 1e-5 relative.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from conftest import rel_l2  # noqa: E402
from oracle import gcn, plan as oplan  # noqa: E402
import paper_2605_11517_b200 as g2  # noqa: E402
from paper_2605_11517_b200.stream import StreamSession  # noqa: E402
from paper_2605_11517_b200.training import TrainSession  # noqa: E402


def _setup(scale, deg, F, C, L, H, mode, directed=False, f32=True):
    g = g2.generate_kronecker(scale, deg, seed=scale)
    if directed:   # drop every other edge: a non-symmetric graph
        src = np.repeat(np.arange(g.num_vertices), np.diff(g.src_ptr))
        keep = (np.arange(g.num_edges) % 3) != 1
        g = g2.build_csr(np.stack([src[keep], g.dst_idx[keep]], 1), g.num_vertices)
    ds = g2.make_random_dataset(g, feature_dim=F, num_classes=C, seed=scale + 1)
    if f32:
        ds.features = ds.features.astype(np.float32)
    part = g2.switching_aware_partition(g, 4, g2.PartitionerParams(seed=scale + 2))
    plan = g2.build_partition_plan(g, part.labels, 4)
    model = g2.create_model(F, C, num_layers=L, hidden_dim=H, seed=scale + 3, aggregation_mode=mode)
    return g, ds, plan, model


CASES = [
    # (scale, deg, F, C, L, H, mode, directed, f32)
    (11, 12, 32, 40, 3, 32, "mean_self_loop", False, True),    # papers-like: AF last layer
    (11, 12, 32, 7, 2, 16, "mean_self_loop", False, True),     # transform-first last layer
    (11, 12, 32, 40, 3, 32, "symmetric_norm", False, False),   # sym, f64 features (staged)
    (10, 16, 30, 9, 2, 24, "symmetric_norm", True, True),      # directed graph, F % 4 != 0
]


@pytest.mark.parametrize("cache", ["none", "part"])
@pytest.mark.parametrize("case", CASES)
def test_streaming_matches_resident_and_oracle(case, cache):
    scale, deg, F, C, L, H, mode, directed, f32 = case
    g, ds, plan, model = _setup(scale, deg, F, C, L, H, mode, directed, f32)
    epochs, lr = 2, 0.05
    ref = TrainSession(ds, plan, model)
    m_ref, tr_ref = ref.train(epochs, lr, use_graph=False)
    # no HBM feature cache (every pass streams), or the first chunks cached
    xb = 0 if cache == "none" else 900 * 4 * ((F + 3) // 4 * 4)
    ss = StreamSession(ds, plan, model, chunk_rows=300, x_cache_bytes=xb)
    assert ss.engine.cache_rows == (0 if cache == "none" else 900)
    assert ss.sg.symmetric == (not directed)
    assert len(ss.sg.chunks) > 3 and any(s.n_segs for s in ss.sg.fwd_chunks)
    m_st, tr_st = ss.train(epochs, lr)
    for (_, l1, a1), (_, l2, a2) in zip(tr_st, tr_ref):
        assert abs(l1 - l2) <= 1e-5 * abs(l2)
        assert abs(a1 - a2) <= 2.0 / ds.train_mask.sum()
    topos = oplan.build_plan(g.src_ptr, g.dst_idx, plan.labels, 4)
    W, grads, tr_or = gcn.train_partitioned(np.asarray(ds.features, np.float64), ds.labels,
                                            ds.train_mask, topos, model.weights, epochs, lr, mode=mode)
    for i in range(L):
        assert rel_l2(m_st.weights[i], m_ref.weights[i]) < 1e-5
        assert rel_l2(m_st.weight_grads[i], m_ref.weight_grads[i]) < 1e-5
        assert rel_l2(m_st.weights[i], W[i]) < 1e-4
    for (_, l1, _), (_, l2, _) in zip(tr_st, tr_or):
        assert abs(l1 - l2) <= 1e-4 * abs(l2)


@pytest.mark.parametrize("case", [CASES[0], CASES[2]])
@pytest.mark.parametrize("cache", ["none", "part"])
def test_streaming_features_kept_in_layer_buffer(monkeypatch, cache, case):
    """The hidden-layer regather streams the features into the consumed
    layer buffer and computes A_1 = act((A_hat X) W_0) from them; the
    layer-0 backward and the next epoch's layer-0 transform read the same
    rows there: one host pass per epoch instead of three, results within
    the streamed-vs-resident tolerance of the transform-first regather."""
    scale, deg, F, C, L, H, mode, directed, f32 = case
    g, ds, plan, model = _setup(scale, deg, F, C, L, H, mode, directed, f32)
    xb = 0 if cache == "none" else 900 * 4 * F
    runs = {}
    for on in ("1", "0"):
        monkeypatch.setenv("GRD_STREAM_STASH", on)
        ss = StreamSession(ds, plan, model, chunk_rows=300, x_cache_bytes=xb)
        assert ss.engine.stash_on == (on == "1")
        m, tr = ss.train(3, 0.05)
        runs[on] = (m, tr, ss.engine.h2d_bytes, ss)
    (m1, tr1, b1, ss1), (m0, tr0, b0, _) = runs["1"], runs["0"]
    for (_, l1, _), (_, l0, _) in zip(tr1, tr0):
        assert abs(l1 - l0) <= 1e-5 * abs(l0)
    for i in range(L):
        assert rel_l2(m1.weights[i], m0.weights[i]) < 1e-5
        assert rel_l2(m1.weight_grads[i], m0.weight_grads[i]) < 1e-5
    streamed = (g.num_vertices - ss1.engine.cache_rows) * F * 4
    # off: 3 passes every epoch; on: 2 in the first epoch, then 1
    assert b0 - b1 == 5 * streamed
    assert ss1.engine._xbuf is not None
    ss1.reset(ds, model)            # re-binding the features drops the kept rows
    assert ss1.engine._xbuf is None
    m2, tr2 = ss1.train(1, 0.05)
    assert abs(tr2[0][1] - tr1[0][1]) <= 1e-5 * abs(tr1[0][1])


def test_streaming_deep_hidden_layers_on_host():
    """L = 4: A_2 goes to pinned host memory in forward and streams back."""
    g, ds, plan, model = _setup(11, 12, 32, 48, 4, 32, "mean_self_loop")
    ref = TrainSession(ds, plan, model)
    m_ref, tr_ref = ref.train(2, 0.05, use_graph=False)
    ss = StreamSession(ds, plan, model, chunk_rows=500, x_cache_bytes=0)
    assert 2 in ss.engine.host_acts
    m_st, tr_st = ss.train(2, 0.05)
    for (_, l1, _), (_, l2, _) in zip(tr_st, tr_ref):
        assert abs(l1 - l2) <= 1e-5 * abs(l2)
    for i in range(4):
        assert rel_l2(m_st.weights[i], m_ref.weights[i]) < 1e-5


def test_partitioned_train_selects_streaming(monkeypatch):
    """GRD_ENGINE=stream routes the public API through the streaming engine
    (the automatic choice makes it when the resident working set exceeds
    the free HBM)."""
    g, ds, plan, model = _setup(10, 8, 16, 5, 2, 8, "mean_self_loop")
    monkeypatch.setenv("GRD_ENGINE", "stream")
    m1, tr1, _ = g2.partitioned_train(ds, plan, model, epochs=1, lr=0.05)
    assert any(isinstance(v, StreamSession) for v in plan.device_cache.values())
    monkeypatch.setenv("GRD_ENGINE", "resident")
    plan2 = g2.build_partition_plan(g, plan.labels, 4)
    m2, tr2, _ = g2.partitioned_train(ds, plan2, model, epochs=1, lr=0.05)
    assert abs(tr1[0][1] - tr2[0][1]) <= 1e-5 * abs(tr2[0][1])
    for a, b in zip(m1.weights, m2.weights):
        assert rel_l2(a, b) < 1e-5


def test_streaming_session_rebinds_features(monkeypatch):
    """A second call on the same plan with other features refills the HBM
    feature cache (no stale rows)."""
    g, ds, plan, model = _setup(10, 8, 16, 5, 2, 8, "mean_self_loop")
    monkeypatch.setenv("GRD_ENGINE", "stream")
    g2.partitioned_train(ds, plan, model, epochs=1, lr=0.05)
    ds2 = g2.LabeledDataset(graph=g, features=(ds.features * 0.5).astype(np.float32),
                            labels=ds.labels, train_mask=ds.train_mask)
    m1, tr1, _ = g2.partitioned_train(ds2, plan, model, epochs=1, lr=0.05)
    sess = [v for v in plan.device_cache.values() if isinstance(v, StreamSession)][0]
    assert sess.engine.cache_rows == g.num_vertices      # fully cached
    ref = TrainSession(ds2, plan, model)
    m2, tr2 = ref.train(1, 0.05, use_graph=False)
    assert abs(tr1[0][1] - tr2[0][1]) <= 1e-5 * abs(tr2[0][1])
    for a, b in zip(m1.weights, m2.weights):
        assert rel_l2(a, b) < 1e-5


@pytest.mark.parametrize("host_rows", [0, 700])
def test_streaming_from_nvme_tier(tmp_path, host_rows):
    """Features kept in their GRIN file (load_dataset(mmap_features=True)):
    HBM cache (first 600 rows) -> pinned host cache window -> direct reads
    from the file through the bounce-buffer ring.  Same epoch as the
    resident engine on the in-memory features."""
    from paper_2605_11517_b200.tiers import FileRows
    g, ds, plan, model = _setup(11, 12, 32, 40, 3, 32, "mean_self_loop")
    ds.save(tmp_path)
    mm = g2.load_dataset(tmp_path, mmap_features=True)
    ref = TrainSession(ds, plan, model)
    m_ref, tr_ref = ref.train(2, 0.05, use_graph=False)
    ss = StreamSession(mm, plan, model, chunk_rows=300, x_cache_bytes=600 * 32 * 4,
                       host_cache_bytes=host_rows * 32 * 4)
    src = ss.engine.x_src
    assert isinstance(src, FileRows)
    assert (src.host_lo, src.host_hi) == (600, 600 + host_rows)
    m_st, tr_st = ss.train(2, 0.05)
    # pass 1 reads every non-HBM-cached row from the file; later passes only
    # the rows outside both caches (3 passes over X in 2 epochs: the layer-1
    # regather leaves the rows in a layer buffer for the layer-0 backward and
    # the next epoch's forward)
    V, rb = g.num_vertices, 32 * 4
    outside = V - 600 - host_rows
    assert src.storage_bytes >= rb * ((V - 600) + 2 * outside)
    assert src.storage_bytes < rb * ((V - 600) + 3 * outside) + 2 * (1 << 20)
    for (_, l1, _), (_, l2, _) in zip(tr_st, tr_ref):
        assert abs(l1 - l2) <= 1e-5 * abs(l2)
    for i in range(3):
        assert rel_l2(m_st.weights[i], m_ref.weights[i]) < 1e-5


SAGE_CASES = [
    # (scale, deg, F, C, L, H, directed, chunk_rows)
    (11, 12, 48, 7, 3, 32, False, 300),     # configs[4]-like: every layer transform-first
    (11, 12, 40, 5, 2, 24, True, 256),      # directed graph: separate backward CSR
    (10, 16, 64, 9, 4, 32, False, 200),     # L = 4: A_2 kept on the host and streamed back
]


@pytest.mark.parametrize("case", SAGE_CASES)
def test_streaming_sage_matches_resident_and_oracle(case):
    """GraphSAGE-mean through the streaming engine: same epoch as the
    resident layer-wise engine (1e-5) and the builder oracle (1e-4)."""
    from oracle import sage_gat
    scale, deg, F, C, L, H, directed, rows = case
    g, ds, plan, model = _setup(scale, deg, F, C, L, H, "sage_mean", directed)
    epochs, lr = 2, 0.05
    ref = TrainSession(ds, plan, model)
    m_ref, tr_ref = ref.train(epochs, lr, use_graph=False)
    ss = StreamSession(ds, plan, model, chunk_rows=rows, x_cache_bytes=3 * rows * 4 * F)
    assert ss.engine.sage and ss.engine.cache_rows == 3 * rows
    assert any(s.n_segs for s in ss.sg.fwd_chunks)
    if L > 3:
        assert 2 in ss.engine.host_acts
    m_st, tr_st = ss.train(epochs, lr)
    for (_, l1, a1), (_, l2, a2) in zip(tr_st, tr_ref):
        assert abs(l1 - l2) <= 1e-5 * abs(l2)
        assert abs(a1 - a2) <= 2.0 / ds.train_mask.sum()
    W, tr_or = sage_gat.train_sage(np.asarray(ds.features, np.float64), ds.labels, ds.train_mask,
                                   g.src_ptr, g.dst_idx, model.weights, epochs, lr)[::2]
    for i in range(L):
        assert rel_l2(m_st.weights[i], m_ref.weights[i]) < 1e-5
        assert rel_l2(m_st.weight_grads[i], m_ref.weight_grads[i]) < 1e-5
        assert rel_l2(m_st.weights[i], W[i]) < 1e-4
    for (_, l1, _), (_, l2, _) in zip(tr_st, tr_or):
        assert abs(l1 - l2) <= 1e-4 * abs(l2)


def test_streaming_sage_from_nvme_tier(tmp_path):
    """configs[4]'s path in small: GraphSAGE with the features in their GRIN
    file behind HBM and host caches, read with direct I/O."""
    from paper_2605_11517_b200.tiers import FileRows
    g, ds, plan, model = _setup(11, 12, 64, 6, 3, 32, "sage_mean")
    ds.save(tmp_path)
    mm = g2.load_dataset(tmp_path, mmap_features=True)
    ref = TrainSession(ds, plan, model)
    m_ref, tr_ref = ref.train(2, 0.05, use_graph=False)
    ss = StreamSession(mm, plan, model, chunk_rows=300, x_cache_bytes=600 * 64 * 4,
                       host_cache_bytes=300 * 64 * 4)
    assert isinstance(ss.engine.x_src, FileRows)
    m_st, tr_st = ss.train(2, 0.05)
    assert ss.engine.x_src.storage_bytes > 0
    for (_, l1, _), (_, l2, _) in zip(tr_st, tr_ref):
        assert abs(l1 - l2) <= 1e-5 * abs(l2)
    for i in range(3):
        assert rel_l2(m_st.weights[i], m_ref.weights[i]) < 1e-5


GAT_CASES = [
    # (scale, deg, F, C, L, H, heads, directed, chunk rows)
    (11, 12, 48, 7, 3, 32, 4, False, 300),    # configs[2]-like, 3 layers
    (11, 12, 40, 5, 2, 16, 2, True, 256),     # directed graph: separate out-CSR for the pull
    (10, 16, 64, 9, 4, 32, 4, False, 200),    # L = 4: A_2 kept on the host and streamed back
]


@pytest.mark.parametrize("case", GAT_CASES)
def test_streaming_gat_matches_resident_and_oracle(case):
    """GAT through the streaming engine (four layer-height buffers, the
    features streamed, hidden layers regathered in the backward): same
    epoch as the resident layer-wise engine (1e-5) and the builder oracle
    (1e-4), with a partial HBM feature cache and split heavy rows."""
    from oracle import sage_gat
    scale, deg, F, C, L, H, heads, directed, rows = case
    g, ds, plan, _ = _setup(scale, deg, F, C, L, H, "gat", directed)
    model = g2.create_model(F, C, num_layers=L, hidden_dim=H, seed=scale + 3, aggregation_mode="gat",
                            heads=heads)
    epochs, lr = 2, 0.05
    ref = TrainSession(ds, plan, model)
    m_ref, tr_ref = ref.train(epochs, lr, use_graph=False)
    ss = StreamSession(ds, plan, model, chunk_rows=rows, x_cache_bytes=3 * rows * 4 * F)
    assert ss.engine.gat and ss.engine.cache_rows == 3 * rows
    assert any(s.n_segs for s in ss.sg.fwd_chunks)
    if L > 3:
        assert 2 in ss.engine.host_acts
    m_st, tr_st = ss.train(epochs, lr)
    for (_, l1, a1), (_, l2, a2) in zip(tr_st, tr_ref):
        assert abs(l1 - l2) <= 1e-5 * abs(l2)
        assert abs(a1 - a2) <= 2.0 / ds.train_mask.sum()
    W, grads, tr_or = sage_gat.train_gat(np.asarray(ds.features, np.float64), ds.labels,
                                         ds.train_mask, g.src_ptr, g.dst_idx, model.weights, heads,
                                         epochs, lr)
    for i in range(L):
        assert rel_l2(m_st.weights[i], m_ref.weights[i]) < 1e-5
        assert rel_l2(m_st.weight_grads[i], m_ref.weight_grads[i]) < 1e-5
        assert rel_l2(m_st.weights[i], W[i]) < 1e-4
    for (_, l1, _), (_, l2, _) in zip(tr_st, tr_or):
        assert abs(l1 - l2) <= 1e-4 * abs(l2)


def test_partitioned_train_streams_gat(monkeypatch):
    """GRD_ENGINE=stream routes a GAT model to the streaming engine."""
    g, ds, plan, _ = _setup(10, 8, 16, 4, 2, 8, "gat")
    model = g2.create_model(16, 4, num_layers=2, hidden_dim=8, seed=3, aggregation_mode="gat", heads=2)
    monkeypatch.setenv("GRD_ENGINE", "stream")
    plan.device_cache.clear()
    st, tst, _ = g2.partitioned_train(ds, plan, model, epochs=1, lr=0.05)
    assert isinstance(g2.training.session_for(ds, plan, model), StreamSession)
    monkeypatch.setenv("GRD_ENGINE", "resident")
    plan.device_cache.clear()
    rs, trs, _ = g2.partitioned_train(ds, plan, model, epochs=1, lr=0.05)
    assert abs(tst[0][1] - trs[0][1]) <= 1e-5 * abs(trs[0][1])
    for a, b in zip(st.weights, rs.weights):
        assert rel_l2(a, b) < 1e-5
    plan.device_cache.clear()
