import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from conftest import rel_l2
from oracle import sage_gat
import paper_2605_11517_b200 as g2
from paper_2605_11517_b200.training import TrainSession
for mode in ("sage_mean", "mean_self_loop"):
    g = g2.generate_kronecker(9, 8, seed=9)
    ds = g2.make_random_dataset(g, feature_dim=6, num_classes=3, seed=10)
    part = g2.switching_aware_partition(g, 4, g2.PartitionerParams(seed=11))
    plan = g2.build_partition_plan(g, part.labels, 4)
    model = g2.create_model(6, 3, num_layers=3, hidden_dim=12, seed=12, aggregation_mode=mode)
    runs = {}
    for tag, ep, graph in [("fresh1", 1, True), ("cached1", 1, True), ("cached3", 3, True), ("cached1b", 1, True)]:
        m, t, _ = g2.partitioned_train(ds, plan, model, epochs=ep, lr=0.05)
        runs[tag] = (m, t)
    for tag, ug in [("nograph1", False), ("graph1", True)]:
        s = TrainSession(ds, plan, model)
        m, t = s.train(1, 0.05, use_graph=ug)
        runs[tag] = (m, t)
    base = runs["fresh1"][0]
    for tag, (m, t) in runs.items():
        print(mode, tag, t[-1][1], [f"{rel_l2(a, b):.2e}" for a, b in zip(m.weight_grads, base.weight_grads)])
