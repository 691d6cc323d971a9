"""Weight-gradient error against float64 under the GEMM precision knobs:
the papers-shaped golden case (reference float64) and GraphSAGE at the
products widths (builder oracle).  Usage: KEY=VAL env, prints one line."""
import os
import sys

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np  # noqa: E402

import paper_2605_11517_b200 as g2  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


case = sys.argv[1]
tag = " ".join(f"{k}={os.environ.get(k, '-')}" for k in ("GRD_GEMM_KCHUNK", "GRD_WGRAD_FRESH", "GRD_GEMM_KSPLIT_TB"))
if case == "papers":
    z = dict(np.load("tests/golden/papers_s22.npz"))
    scale, deg, F, C, L, H, P = [int(x) for x in z["spec"]]
    g = g2.generate_kronecker(scale, deg, seed=0, device="cuda")
    labels = g2.switching_aware_partition(g, P, g2.PartitionerParams(seed=2)).labels
    plan = g2.build_partition_plan(g, labels, P, device="cuda")
    ds = g2.make_random_dataset(g, feature_dim=F, num_classes=C, seed=1, feature_dtype=np.float32)
    model = g2.create_model(F, C, num_layers=L, hidden_dim=H, seed=3)
    tr, trace, _ = g2.partitioned_train(ds, plan, model, 1, 0.01)
    print(case, tag, [f"{rel(d, z[f'wgrad_{i}']):.2e}" for i, d in enumerate(tr.weight_grads)])
else:
    from oracle import sage_gat
    g = g2.generate_kronecker(14, 30, seed=14)
    ds = g2.make_random_dataset(g, feature_dim=100, num_classes=47, seed=15)
    plan = g2.build_partition_plan(g, g2.switching_aware_partition(g, 8, g2.PartitionerParams(seed=16)).labels, 8)
    model = g2.create_model(100, 47, num_layers=3, hidden_dim=256, seed=17, aggregation_mode="sage_mean")
    tr, trace, _ = g2.partitioned_train(ds, plan, model, 1, 0.01)
    _, grads, _ = sage_gat.train_sage(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx,
                                      model.weights, 1, 0.01)
    print(case, tag, [f"{rel(a, b):.2e}" for a, b in zip(tr.weight_grads, grads)])
