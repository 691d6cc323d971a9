"""Generate golden fixtures from the reference package itself.

Runs only in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Outputs (committed, small):
  small_cases.npz  per-(layer, partition) tensors, traces and weights of the
                   reference's partitioned_train on 256-512-vertex Kronecker
                   graphs (mean / symmetric / row-normalised / dropout)
  config1.npz      BASELINE config 1 (generate_kronecker(17, 8, 0), F=128,
                   C=10, L=2, H=64, P=8 switching-aware labels, lr 0.01):
                   graph + plan digests, partitioner result, and the
                   1-epoch loss / accuracy / weights / weight gradients
"""

from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from grinder.dataset import make_random_dataset  # noqa: E402
from grinder.graph import generate_kronecker  # noqa: E402
from grinder.model import create_model  # noqa: E402
from grinder.partition import PartitionerParams, random_partition, switching_aware_partition  # noqa: E402
from grinder.plan import build_partition_plan  # noqa: E402
from grinder.training import partitioned_train  # noqa: E402

OUT = Path(__file__).resolve().parent


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


SMALL = {
    # name: (scale, deg, F, C, P, layers, hidden, mode, rownorm, dropout, epochs)
    "mean": (8, 8, 6, 3, 4, 3, 8, "mean_self_loop", False, 0.0, 3),
    "sym": (9, 8, 6, 3, 8, 3, 8, "symmetric_norm", False, 0.0, 3),
    "rownorm": (8, 6, 6, 3, 4, 2, 6, "mean_self_loop", True, 0.0, 2),
    "dropout": (8, 8, 6, 3, 1, 2, 6, "mean_self_loop", False, 0.3, 2),
    "widen": (8, 8, 4, 3, 4, 2, 12, "symmetric_norm", False, 0.0, 2),
}


def small_cases() -> dict:
    out = {}
    for name, (scale, deg, F, C, P, L, H, mode, rn, dr, epochs) in SMALL.items():
        g = generate_kronecker(scale, deg, seed=scale)
        ds = make_random_dataset(g, feature_dim=F, num_classes=C, seed=scale + 1)
        labels = random_partition(g.num_vertices, P, seed=scale + 2)
        plan = build_partition_plan(g, labels, P)
        model = create_model(F, C, num_layers=L, hidden_dim=H, seed=scale + 3,
                             aggregation_mode=mode, row_normalize=rn, dropout_rate=dr)
        seen = {}

        def probe(epoch, layer, pid, grad_ga, grad_w):
            if epoch == 0:
                seen[(layer, pid)] = (grad_ga.copy(), grad_w.copy())

        trained, trace, _ = partitioned_train(ds, plan, model, epochs=epochs, lr=0.05,
                                              grad_probe=probe)
        p = f"{name}/"
        out[p + "spec"] = np.array([scale, deg, F, C, P, L, H, int(rn), epochs], dtype=np.int64)
        out[p + "mode"] = np.array(mode)
        out[p + "dropout"] = np.array(dr)
        out[p + "labels"] = labels
        out[p + "trace"] = np.array([[e, l, a] for e, l, a in trace], dtype=np.float64)
        for i, w in enumerate(model.weights):
            out[p + f"w_init_{i}"] = w
        for i, w in enumerate(trained.weights):
            out[p + f"w_final_{i}"] = w
            out[p + f"wgrad_final_{i}"] = trained.weight_grads[i]
        for (layer, pid), (gga, gw) in seen.items():
            out[p + f"grad_ga_{layer}_{pid}"] = gga
            out[p + f"grad_w_{layer}_{pid}"] = gw
        out[p + "graph_digest"] = np.array(digest(g.src_ptr, g.dst_idx))
    return out


def config1() -> dict:
    t0 = time.time()
    g = generate_kronecker(17, 8, seed=0)
    ds = make_random_dataset(g, feature_dim=128, num_classes=10, seed=1)
    res = switching_aware_partition(g, 8, PartitionerParams(seed=2))
    plan = build_partition_plan(g, res.labels, 8)
    model = create_model(128, 10, num_layers=2, hidden_dim=64, seed=3)
    print(f"config1 preprocessing {time.time() - t0:.1f}s", flush=True)
    t0 = time.time()
    trained, trace, _ = partitioned_train(ds, plan, model, epochs=1, lr=0.01)
    print(f"config1 reference epoch {time.time() - t0:.1f}s", flush=True)
    out = {
        "graph_digest": np.array(digest(g.src_ptr, g.dst_idx)),
        "num_edges": np.array(g.num_edges),
        "features_digest": np.array(digest(ds.features)),
        "labels_digest": np.array(digest(ds.labels, ds.train_mask)),
        "sa_labels": res.labels.astype(np.int8),
        "sa_objective_trace": np.array(res.objective_trace),
        "sa_initial_objective": np.array(res.initial_objective),
        "sa_iterations": np.array(res.iterations),
        "sa_converged": np.array(res.converged),
        "sa_max_sizes": np.array(res.max_size_per_iteration),
        "loss": np.array(trace[0][1]),
        "acc": np.array(trace[0][2]),
    }
    for q, t in enumerate(plan.topologies):
        out[f"plan_digest_{q}"] = np.array(digest(t.targets, t.gather_map, t.tgt_ptr, t.src_pos,
                                                  t.edge_local_target, t.self_pos, t.target_indeg,
                                                  t.gather_indeg))
    for i, w in enumerate(trained.weights):
        out[f"w_final_{i}"] = w
        out[f"wgrad_{i}"] = trained.weight_grads[i]
    return out


def main() -> None:
    np.savez_compressed(OUT / "small_cases.npz", **small_cases())
    np.savez_compressed(OUT / "config1.npz", **config1())
    for f in ("small_cases.npz", "config1.npz"):
        print(f, (OUT / f).stat().st_size, "bytes")


if __name__ == "__main__" and not {"--ledger", "--ledger4", "--papers", "--products"} & set(sys.argv):
    main()


def ledger_cases() -> dict:
    """Ledgers of the reference's simulate_epoch (GRINNDER) for the tier
    manager's parity test: host capacities that keep whole layers, force
    per-partition slabs, or force page-granular vertex reads; bypass on/off."""
    import json
    from grinder.hierarchy import HierarchyConfig
    from grinder.simulate import ledger_summary, simulate_epoch
    g = generate_kronecker(7, 6, seed=3)
    labels = random_partition(g.num_vertices, 4, seed=1)
    plan = build_partition_plan(g, labels, 4)
    dims = [6, 5, 5, 3]
    out = {"labels": labels, "graph_digest": np.array(digest(g.src_ptr, g.dst_idx))}
    n = g.num_vertices
    cases = {
        "layer_lru": dict(host_capacity=3 * n * 6 * 4, bytes_per_value=4),
        "partition_lru": dict(host_capacity=n * 6 * 4 // 2, bytes_per_value=4),
        "vertex": dict(host_capacity=64, bytes_per_value=4, page_size=64),
        "no_bypass": dict(host_capacity=3 * n * 6 * 8, bytes_per_value=8),
        "tight": dict(host_capacity=n * 6 * 8 + 100, bytes_per_value=8),
    }
    if FP32_LEDGERS:
        # every case at 4 bytes per value: what an executing (fp32) session
        # moves, so its recorded ledger is compared with the reference's
        cases["no_bypass"] = dict(host_capacity=3 * n * 6 * 4, bytes_per_value=4)
        cases["tight"] = dict(host_capacity=n * 6 * 4 + 100, bytes_per_value=4)
        cases["tiny_pages"] = dict(host_capacity=0, bytes_per_value=4, page_size=16)
    for name, kw in cases.items():
        bypass = name != "no_bypass"
        from grinder.hierarchy import PolicySpec
        pol = PolicySpec("GRINNDER", bypass_enabled=bypass)
        led = simulate_epoch(plan, dims, pol, HierarchyConfig(**kw), epochs=2)
        out[f"{name}/events"] = np.array(json.dumps(led.events))
        out[f"{name}/summary"] = np.array(json.dumps(ledger_summary(led), sort_keys=True))
        out[f"{name}/stage_table"] = np.array(json.dumps(led.stage_table(1), sort_keys=True))
        out[f"{name}/config"] = np.array(json.dumps(kw, sort_keys=True))
    return out


FP32_LEDGERS = "--ledger4" in sys.argv

if __name__ == "__main__" and "--ledger" in sys.argv:
    np.savez_compressed(OUT / "ledger_cases.npz", **ledger_cases())
if __name__ == "__main__" and "--ledger4" in sys.argv:
    np.savez_compressed(OUT / "ledger_cases_fp32.npz", **ledger_cases())


def _integer_artifacts(g, ds, res, plan) -> dict:
    out = {
        "graph_digest": np.array(digest(g.src_ptr, g.dst_idx)),
        "num_vertices": np.array(g.num_vertices),
        "num_edges": np.array(g.num_edges),
        "sa_labels_digest": np.array(digest(res.labels)),
        "sa_sizes": np.bincount(res.labels, minlength=plan.num_partitions).astype(np.int64),
        "sa_objective_trace": np.array(res.objective_trace),
        "sa_initial_objective": np.array(res.initial_objective),
        "sa_iterations": np.array(res.iterations),
        "sa_converged": np.array(res.converged),
        "sa_max_sizes": np.array(res.max_size_per_iteration),
        "gather_rows": np.array([t.gather_map.size for t in plan.topologies], dtype=np.int64),
    }
    if ds is not None:
        out["features_digest"] = np.array(digest(ds.features))
        out["labels_digest"] = np.array(digest(ds.labels, ds.train_mask))
    for q, t in enumerate(plan.topologies):
        out[f"plan_digest_{q}"] = np.array(digest(t.targets, t.gather_map, t.tgt_ptr, t.src_pos,
                                                  t.edge_local_target, t.self_pos, t.target_indeg,
                                                  t.gather_indeg))
    return out


def papers_small() -> dict:
    """configs[3]'s model (3-layer GCN, F=H=128, C=172, P=16 switching-aware,
    CLI seeds 0/1/2/3, lr 0.01) on the largest papers-shaped (average degree
    12) Kronecker graph the reference finishes here: generate_kronecker(22, 12)."""
    scale, deg, F, C, L, H, P = PAPERS_SHAPE
    t0 = time.time()
    g = generate_kronecker(scale, deg, seed=0)
    print(f"papers generate {time.time() - t0:.1f}s", flush=True)
    ds = make_random_dataset(g, feature_dim=F, num_classes=C, seed=1)
    t0 = time.time()
    res = switching_aware_partition(g, P, PartitionerParams(seed=2))
    print(f"papers partition {time.time() - t0:.1f}s", flush=True)
    t0 = time.time()
    plan = build_partition_plan(g, res.labels, P)
    print(f"papers plan {time.time() - t0:.1f}s", flush=True)
    model = create_model(F, C, num_layers=L, hidden_dim=H, seed=3)
    out = _integer_artifacts(g, ds, res, plan)
    del g
    t0 = time.time()
    trained, trace, _ = partitioned_train(ds, plan, model, epochs=1, lr=0.01)
    print(f"papers reference epoch {time.time() - t0:.1f}s", flush=True)
    out["spec"] = np.array(PAPERS_SHAPE, dtype=np.int64)
    out["loss"] = np.array(trace[0][1])
    out["acc"] = np.array(trace[0][2])
    for i, w in enumerate(trained.weights):
        out[f"w_final_{i}"] = w
        out[f"wgrad_{i}"] = trained.weight_grads[i]
    return out


def products_integers() -> dict:
    """configs[1]/[2]'s graph generate_kronecker(21, 30, 0) with P=8
    switching-aware partitions (seed 2) and its plan: integer artefacts only
    (the reference has no GraphSAGE / GAT to train)."""
    t0 = time.time()
    g = generate_kronecker(21, 30, seed=0)
    print(f"products generate {time.time() - t0:.1f}s", flush=True)
    t0 = time.time()
    res = switching_aware_partition(g, 8, PartitionerParams(seed=2))
    print(f"products partition {time.time() - t0:.1f}s", flush=True)
    t0 = time.time()
    plan = build_partition_plan(g, res.labels, 8)
    print(f"products plan {time.time() - t0:.1f}s", flush=True)
    return _integer_artifacts(g, None, res, plan)


# (scale, avg degree, F, C, layers, hidden, partitions)
PAPERS_SHAPE = (22, 12, 128, 172, 3, 128, 16)

if __name__ == "__main__" and "--papers" in sys.argv:
    np.savez_compressed(OUT / "papers_s22.npz", **papers_small())
if __name__ == "__main__" and "--products" in sys.argv:
    np.savez_compressed(OUT / "products_s21.npz", **products_integers())
