import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from conftest import rel_l2
from oracle import sage_gat
import paper_2605_11517_b200 as g2
for (F, H, C, L) in [(6, 12, 3, 3), (16, 8, 5, 2)]:
    g = g2.generate_kronecker(9, 8, seed=9)
    ds = g2.make_random_dataset(g, feature_dim=F, num_classes=C, seed=10)
    part = g2.switching_aware_partition(g, 4, g2.PartitionerParams(seed=11))
    plan = g2.build_partition_plan(g, part.labels, 4)
    model = g2.create_model(F, C, num_layers=L, hidden_dim=H, seed=12, aggregation_mode="sage_mean")
    for ep in (1, 3):
        trained, trace, _ = g2.partitioned_train(ds, plan, model, epochs=ep, lr=0.05)
        W, grads, ref = sage_gat.train_sage(ds.features, ds.labels, ds.train_mask, g.src_ptr, g.dst_idx, model.weights, ep, 0.05)
        print(F, H, C, L, "epochs", ep, "loss", trace[-1][1], ref[-1][1])
        for i, (a, b) in enumerate(zip(trained.weight_grads, grads)):
            print("  layer", i, "grad rel", rel_l2(a, b), "norm", np.linalg.norm(b), "W rel", rel_l2(trained.weights[i], W[i]),
                  "root", rel_l2(a[:, :b.shape[1]//2], b[:, :b.shape[1]//2]), "nbr", rel_l2(a[:, b.shape[1]//2:], b[:, b.shape[1]//2:]))
