"""Per-layer weight-gradient error of one GraphSAGE / GAT epoch at the
BASELINE widths against the float64 oracle, for the package under the
given root (to bisect a regression).  Usage:
  python tools/debug_widths.py ROOT MODE [KEY=VAL ...]   (env knobs)"""
import os
import sys

root, mode = sys.argv[1], sys.argv[2]
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    os.environ[k] = v
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.abspath(root))
import numpy as np  # noqa: E402

import paper_2605_11517_b200 as g2  # noqa: E402
from oracle import sage_gat  # noqa: E402

assert g2.__file__.startswith(os.path.abspath(root)), g2.__file__


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


scale = int(os.environ.get("SCALE", "14"))
g = g2.generate_kronecker(scale, 30, seed=scale)
F = int(os.environ.get("F", "100"))
H = int(os.environ.get("H", "256"))
ds = g2.make_random_dataset(g, feature_dim=F, num_classes=47, seed=scale + 1)
part = g2.switching_aware_partition(g, 8, g2.PartitionerParams(seed=scale + 2))
plan = g2.build_partition_plan(g, part.labels, 8)
model = g2.create_model(F, 47, num_layers=3, hidden_dim=H, seed=scale + 3, aggregation_mode=mode)
trained, trace, _ = g2.partitioned_train(ds, plan, model, epochs=1, lr=0.01)
if mode in ("mean_self_loop", "symmetric_norm"):
    from oracle import gcn
    W, grads, ref = gcn.train_partitioned(ds.features, ds.labels, ds.train_mask, plan.topologies,
                                          model.weights, 1, 0.01, mode=mode)
elif mode == "gat":
    W, grads, ref = sage_gat.train_gat(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                       model.weights, 4, 1, 0.01)
else:
    W, grads, ref = sage_gat.train_sage(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                        model.weights, 1, 0.01)
print(root, mode, sys.argv[3:], "loss", abs(trace[0][1] - ref[0][1]) / abs(ref[0][1]),
      "dW", [round(rel(a, b), 7) for a, b in zip(trained.weight_grads, grads)])
if mode == "sage_mean":
    for l, (a, b) in enumerate(zip(trained.weight_grads, grads)):
        h = a.shape[1] // 2
        print(f"  layer {l}: root {rel(a[:, :h], b[:, :h]):.3e}  nbr {rel(a[:, h:], b[:, h:]):.3e}  "
              f"|root| {np.linalg.norm(b[:, :h]):.3e} |nbr| {np.linalg.norm(b[:, h:]):.3e}")
