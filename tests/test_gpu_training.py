"""End-to-end parity of the GPU training path with the reference.

Float tolerance (north star): per-tensor L2-relative error <= 1e-4 for
weights, weight gradients and per-partition grad_GA after the stated epochs;
loss relative <= 1e-4.  Reference values come from tests/golden (generated
by the reference itself) and from the pinned oracle.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from conftest import rel_l2, small_case_inputs  # noqa: E402
from oracle import gcn, plan as oplan  # noqa: E402
import paper_2605_11517_b200 as g2  # noqa: E402

TOL = 1e-4


def _plan(inp):
    return g2.build_partition_plan(inp.graph, inp.labels, inp.P)


@pytest.mark.parametrize("name", ["mean", "sym", "rownorm", "dropout", "widen"])
def test_partitioned_train_matches_golden(small_golden, name):
    case = small_golden[name]
    inp = small_case_inputs(case)
    trained, trace, ledger = g2.partitioned_train(inp.dataset, _plan(inp), inp.model,
                                                  epochs=inp.epochs, lr=0.05)
    assert ledger is None
    want = case["trace"]
    for (e, l, a), row in zip(trace, want):
        assert e == int(row[0])
        assert abs(l - row[1]) <= TOL * abs(row[1])
        assert abs(a - row[2]) <= 2.0 / inp.dataset.train_mask.sum() + 1e-12
    for i in range(inp.L):
        assert rel_l2(trained.weights[i], case[f"w_final_{i}"]) < TOL
        assert rel_l2(trained.weight_grads[i], case[f"wgrad_final_{i}"]) < TOL


@pytest.mark.parametrize("name", ["mean", "sym", "rownorm", "widen"])
def test_per_partition_grads_match_golden(small_golden, name):
    case = small_golden[name]
    inp = small_case_inputs(case)
    seen = {}

    def probe(epoch, layer, pid, gga, gw):
        if epoch == 0:
            seen[(layer, pid)] = (gga, gw)

    g2.partitioned_train(inp.dataset, _plan(inp), inp.model, epochs=1, lr=0.05, grad_probe=probe)
    assert len(seen) == inp.L * inp.P
    for (layer, pid), (gga, gw) in seen.items():
        ref_ga, ref_w = case[f"grad_ga_{layer}_{pid}"], case[f"grad_w_{layer}_{pid}"]
        assert gga.shape == ref_ga.shape and gw.shape == ref_w.shape
        assert rel_l2(gga, ref_ga) < TOL
        assert rel_l2(gw, ref_w) < TOL


@pytest.mark.slow
def test_config1_one_epoch_matches_reference(config1_golden):
    gold = config1_golden
    g = g2.generate_kronecker(17, 8, seed=0)
    ds = g2.make_random_dataset(g, feature_dim=128, num_classes=10, seed=1)
    res = g2.switching_aware_partition(g, 8, g2.PartitionerParams(seed=2))
    np.testing.assert_array_equal(res.labels, gold["sa_labels"].astype(np.int32))
    plan = g2.build_partition_plan(g, res.labels, 8)
    model = g2.create_model(128, 10, num_layers=2, hidden_dim=64, seed=3)
    trained, trace, _ = g2.partitioned_train(ds, plan, model, epochs=1, lr=0.01)
    assert abs(trace[0][1] - float(gold["loss"])) <= TOL * abs(float(gold["loss"]))
    assert abs(trace[0][2] - float(gold["acc"])) <= 3.0 / ds.train_mask.sum()
    for i in range(2):
        assert rel_l2(trained.weights[i], gold[f"w_final_{i}"]) < TOL
        assert rel_l2(trained.weight_grads[i], gold[f"wgrad_{i}"]) < TOL


def test_layer_forward_kats():
    # reference test_training.py:99-117
    g = g2.build_csr([], 1)
    plan = g2.build_partition_plan(g, np.zeros(1, dtype=np.int32), 1)
    eye = g2.ModelState(weights=[np.eye(2), np.eye(2)], weight_grads=[np.zeros((2, 2))] * 2)
    out = g2.layer_forward(0, np.array([[-1.0, 2.0]]), plan.topologies[0], eye)
    np.testing.assert_array_equal(out, [[0.0, 2.0]])
    g = g2.build_csr([(1, 0), (2, 0)], 3)
    plan = g2.build_partition_plan(g, np.zeros(3, dtype=np.int32), 1)
    one = g2.ModelState(weights=[np.array([[1.0]])], weight_grads=[np.zeros((1, 1))])
    out = g2.layer_forward(0, np.array([[1.0], [2.0], [4.0]]), plan.topologies[0], one)
    assert out[0, 0] == pytest.approx(7.0 / 3.0, rel=1e-7)
    out = g2.layer_forward(0, np.array([[-9.0], [0.0], [0.0]]), plan.topologies[0], one)
    assert out[0, 0] == pytest.approx(-3.0, rel=1e-7)
    with pytest.raises(ValueError):
        g2.layer_forward(0, np.zeros((2, 1)), plan.topologies[0], one)
    with pytest.raises(ValueError):
        g2.layer_forward(0, np.zeros((3, 5)), plan.topologies[0], one)


def test_backward_hand_chain_rule_path3():
    # reference test_training.py:152-165 with oracles.path3_linear_backward
    g = g2.build_csr([(0, 1), (1, 2), (1, 0), (2, 1)], 3)
    plan = g2.build_partition_plan(g, np.zeros(3, dtype=np.int32), 1)
    x = np.array([[1.0, 2.0], [3.0, 5.0], [0.5, -1.0]])
    w = np.array([[1.0, 0.5], [-0.25, 2.0]])
    dz = np.array([[0.1, -0.2], [0.3, 0.7], [-1.0, 0.4]])
    model = g2.ModelState(weights=[w], weight_grads=[np.zeros_like(w)])
    a_out = g2.layer_forward(0, x, plan.topologies[0], model)
    grad_ga, grad_w = g2.regather_backward(0, 0, a_out, dz, x, plan, model)
    glob = g2.scatter_accumulate(grad_ga, plan.gather_maps[0], np.zeros((3, 2)))
    h = np.stack([(x[0] + x[1]) / 2, (x[0] + x[1] + x[2]) / 3, (x[1] + x[2]) / 2])
    dh = dz @ w.T
    want_gx = np.stack([dh[0] / 2 + dh[1] / 3, dh[0] / 2 + dh[1] / 3 + dh[2] / 2, dh[1] / 3 + dh[2] / 2])
    np.testing.assert_allclose(glob, want_gx, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(grad_w, h.T @ dz, rtol=1e-6, atol=1e-7)
    with pytest.raises(ValueError):
        g2.regather_backward(0, 0, a_out, dz, x[:2], plan, model)


def test_scatter_accumulate_kats():
    glob = np.zeros((3, 2))
    g2.scatter_accumulate(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([0, 1]), glob)
    g2.scatter_accumulate(np.array([[10.0, 20.0], [30.0, 40.0]]), np.array([1, 2]), glob)
    np.testing.assert_array_equal(glob, [[1.0, 2.0], [13.0, 24.0], [30.0, 40.0]])


def _kron_setup(scale=8, deg=8, P=6, L=3, H=8, seed=4, mode="mean_self_loop"):
    g = g2.generate_kronecker(scale, deg, seed=0)
    ds = g2.make_random_dataset(g, feature_dim=6, num_classes=3, seed=1)
    labels = g2.random_partition(g.num_vertices, P, seed=8)
    plan = g2.build_partition_plan(g, labels, P)
    model = g2.create_model(6, 3, num_layers=L, hidden_dim=H, seed=seed, aggregation_mode=mode)
    return ds, plan, model


def test_shuffled_schedule_is_bitwise_identical():
    ds, plan, model = _kron_setup()
    rng = np.random.default_rng(19)
    m_a, t_a, _ = g2.partitioned_train(ds, plan, model, epochs=3, lr=0.01,
                                       partition_order=lambda l, ph: list(range(6)))
    m_b, t_b, _ = g2.partitioned_train(ds, plan, model, epochs=3, lr=0.01,
                                       partition_order=lambda l, ph: list(rng.permutation(6)))
    assert t_a == t_b
    assert all(np.array_equal(a, b) for a, b in zip(m_a.weights, m_b.weights))


def test_regather_equals_snapshot_bitwise():
    ds, plan, model = _kron_setup(P=4)

    def run(snap):
        seen = {}
        g2.partitioned_train(ds, plan, model, epochs=2, lr=0.01, use_snapshots=snap,
                             grad_probe=lambda e, l, p, gga, gw: seen.__setitem__((e, l, p), gga))
        return seen

    a, b = run(False), run(True)
    assert a.keys() == b.keys()
    assert all(np.array_equal(a[k], b[k]) for k in a)


def test_reruns_are_bitwise_identical_and_model_untouched():
    ds, plan, model = _kron_setup()
    before = [w.copy() for w in model.weights]
    m_a, t_a, _ = g2.partitioned_train(ds, plan, model, epochs=3, lr=0.01)
    m_b, t_b, _ = g2.partitioned_train(ds, plan, model, epochs=3, lr=0.01)
    assert t_a == t_b
    assert all(np.array_equal(a, b) for a, b in zip(m_a.weights, m_b.weights))
    assert all(np.array_equal(a, b) for a, b in zip(model.weights, before))


@pytest.mark.parametrize("mode", ["mean_self_loop", "symmetric_norm"])
def test_layerwise_and_partitionwise_engines_agree(mode):
    ds, plan, model = _kron_setup(scale=9, mode=mode)
    m_a, t_a, _ = g2.partitioned_train(ds, plan, model, epochs=4, lr=0.05)
    m_b, t_b, _ = g2.partitioned_train(ds, plan, model, epochs=4, lr=0.05,
                                       partition_order=lambda l, ph: range(plan.num_partitions))
    for (_, la, _), (_, lb, _) in zip(t_a, t_b):
        assert abs(la - lb) <= TOL * abs(lb)
    for a, b in zip(m_a.weights, m_b.weights):
        assert rel_l2(a, b) < TOL


def test_partitioned_vs_monolithic_and_compute_gradients():
    ds, plan, model = _kron_setup(scale=9)
    topos = oplan.build_plan(ds.graph.src_ptr, ds.graph.dst_idx,
                             np.zeros(ds.graph.num_vertices, dtype=np.int32), 1)
    W, grads, trace = gcn.train_partitioned(ds.features, ds.labels, ds.train_mask, topos,
                                            model.weights, 5, 0.05)
    m_ref, t_ref = g2.reference_train(ds, model, epochs=5, lr=0.05)
    m_par, t_par, _ = g2.partitioned_train(ds, plan, model, epochs=5, lr=0.05)
    for (_, lo, _), (_, lr_, _), (_, lp, _) in zip(trace, t_ref, t_par):
        assert abs(lr_ - lo) <= TOL * abs(lo)
        assert abs(lp - lo) <= TOL * abs(lo)
    for w, a, b in zip(W, m_ref.weights, m_par.weights):
        assert rel_l2(a, w) < TOL and rel_l2(b, w) < TOL
    loss, acc, gw = g2.compute_gradients(ds, model)
    _, g_ref, tr = gcn.train_partitioned(ds.features, ds.labels, ds.train_mask, topos,
                                         model.weights, 1, 0.0)
    assert abs(loss - tr[0][1]) <= TOL * abs(tr[0][1])
    for a, b in zip(gw, g_ref):
        assert rel_l2(a, b) < TOL


def test_nonfinite_loss_raises_and_epochs_zero():
    ds, plan, model = _kron_setup()
    bad = g2.create_model(6, 3, num_layers=3, hidden_dim=8, seed=3)
    for w in bad.weights:
        w[:] = 1e30
    with pytest.raises(ValueError):
        g2.partitioned_train(ds, plan, bad, epochs=1, lr=0.01)
    trained, trace, _ = g2.partitioned_train(ds, plan, model, epochs=0, lr=0.01)
    assert trace == []
    assert all(np.array_equal(a, b) for a, b in zip(trained.weights, model.weights))


def test_hierarchy_hooks_called_in_reference_order():
    ds, plan, model = _kron_setup(P=3, L=2)
    calls = []

    class Hooks:
        ledger = "ledger"

        def __getattr__(self, name):
            if name == "partition_order":
                return lambda layer, phase: [2, 0, 1]
            return lambda *a: calls.append((name,) + a)

    _, _, ledger = g2.partitioned_train(ds, plan, model, epochs=1, lr=0.01, hierarchy=Hooks())
    assert ledger == "ledger"
    want = [("begin_epoch",)]
    for layer in range(2):
        want += [("forward_partition", layer, p) for p in (2, 0, 1)] + [("end_forward_layer", layer)]
    want.append(("loss_stage",))
    for layer in (1, 0):
        want += [("backward_partition", layer, p) for p in (2, 0, 1)] + [("end_backward_layer", layer)]
    want.append(("end_epoch",))
    assert calls == want
