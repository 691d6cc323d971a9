"""Pin the CPU oracle (oracle/) to golden vectors produced by the reference."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import rel_l2, small_case_inputs
from oracle import gcn, graph as ograph, partition as opart, plan as oplan


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", ["mean", "sym", "rownorm", "dropout", "widen"])
def test_oracle_training_matches_reference(small_golden, name):
    case = small_golden[name]
    inp = small_case_inputs(case)
    g = inp.graph
    assert _digest(g.src_ptr, g.dst_idx) == str(case["graph_digest"])
    topos = oplan.build_plan(g.src_ptr, g.dst_idx, inp.labels, inp.P)
    for i, w in enumerate(inp.model.weights):
        np.testing.assert_array_equal(w, case[f"w_init_{i}"])
    seen = {}

    def probe(epoch, layer, pid, gga, gw):
        if epoch == 0:
            seen[(layer, pid)] = (gga, gw)

    W, grads, trace = gcn.train_partitioned(
        inp.dataset.features, inp.dataset.labels, inp.dataset.train_mask, topos, inp.model.weights,
        inp.epochs, 0.05, mode=inp.mode, row_normalize=inp.rownorm, dropout_rate=inp.dropout,
        dropout_seed=inp.model.dropout_seed, probe=probe)
    np.testing.assert_allclose(np.array(trace), case["trace"], rtol=1e-12, atol=1e-14)
    for i in range(inp.L):
        np.testing.assert_allclose(W[i], case[f"w_final_{i}"], rtol=1e-11, atol=1e-13)
        np.testing.assert_allclose(grads[i], case[f"wgrad_final_{i}"], rtol=1e-10, atol=1e-13)
    for (layer, pid), (gga, gw) in seen.items():
        assert rel_l2(gga, case[f"grad_ga_{layer}_{pid}"]) < 1e-12
        assert rel_l2(gw, case[f"grad_w_{layer}_{pid}"]) < 1e-12


def test_oracle_generator_and_partitioner_small(small_golden):
    case = small_golden["mean"]
    scale, deg = int(case["spec"][0]), int(case["spec"][1])
    ptr, dst = ograph.kronecker(scale, deg, seed=scale)
    assert _digest(ptr, dst) == str(case["graph_digest"])
    np.testing.assert_array_equal(opart.random_labels(ptr.size - 1, 4, scale + 2), case["labels"])


@pytest.mark.slow
def test_oracle_config1(config1_golden):
    """Config 1 end to end in the oracle: partitioner labels, plan digests and
    one epoch of partitioned training against the reference's values."""
    from paper_2605_11517_b200 import generate_kronecker, make_random_dataset, create_model
    gold = config1_golden
    g = generate_kronecker(17, 8, seed=0)
    assert _digest(g.src_ptr, g.dst_idx) == str(gold["graph_digest"])
    ds = make_random_dataset(g, feature_dim=128, num_classes=10, seed=1)
    assert _digest(ds.features) == str(gold["features_digest"])
    assert _digest(ds.labels, ds.train_mask) == str(gold["labels_digest"])
    labels = gold["sa_labels"].astype(np.int32)
    topos = oplan.build_plan(g.src_ptr, g.dst_idx, labels, 8)
    for q, t in enumerate(topos):
        assert _digest(t.targets, t.gather_map, t.tgt_ptr, t.src_pos, t.edge_local_target,
                       t.self_pos, t.target_indeg, t.gather_indeg) == str(gold[f"plan_digest_{q}"])
    model = create_model(128, 10, num_layers=2, hidden_dim=64, seed=3)
    W, grads, trace = gcn.train_partitioned(ds.features, ds.labels, ds.train_mask, topos,
                                            model.weights, 1, 0.01)
    assert trace[0][1] == pytest.approx(float(gold["loss"]), rel=1e-12)
    assert trace[0][2] == float(gold["acc"])
    for i in range(2):
        np.testing.assert_allclose(W[i], gold[f"w_final_{i}"], rtol=1e-10, atol=1e-14)
        assert rel_l2(grads[i], gold[f"wgrad_{i}"]) < 1e-10
