"""Epoch of the executing SSO manager on a papers-shaped graph (configs[3]'s
model) for host-tier capacities that keep whole layers, force partition
slabs, or force page-granular vertex reads: wall time per epoch, ledger
bytes per link, the manager's storage-tier traffic.
Usage: python tools/sso_probe.py [SCALE] [PARTITIONS] [EPOCHS]"""
import json
import sys
import tempfile
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_11517_b200 as g2  # noqa: E402
from paper_2605_11517_b200.hierarchy import HierarchyConfig, TierSession, ledger_summary  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
P = int(sys.argv[2]) if len(sys.argv) > 2 else 16
epochs = int(sys.argv[3]) if len(sys.argv) > 3 else 2
spec = dict(bench.WORKLOADS["papers_gcn"], scale=scale, deg=12, P=P, feature_dtype="float32")
g, ds, plan, model, prep = bench.build_workload(spec)
V, E, L = g.num_vertices, g.num_edges, model.num_layers
layer = V * 128 * 4
out = {"graph": f"generate_kronecker({scale}, 12): {V} V / {E} E, P = {P}", "runs": {}}
resident, rtrace, _ = g2.partitioned_train(ds, plan, model, 1, 0.01)
for name, cap in (("layer_lru", 3 * layer), ("partition_lru", layer // 2), ("vertex", 0)):
    with tempfile.TemporaryDirectory(dir=bench.os.environ.get("GRD_TIER_DIR")) as d:
        cfg = HierarchyConfig(host_capacity=cap, bytes_per_value=4)
        sess = TierSession(plan, model.dims, "GRINNDER", cfg, directory=d)
        t0 = time.perf_counter()
        trained, trace, ledger = g2.partitioned_train(ds, plan, model, epochs, 0.01, hierarchy=sess)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / epochs
        summ = ledger_summary(ledger)
        wall = {k: round(v / epochs, 3) for k, v in sorted(sess.wall.items(), key=lambda kv: -kv[1])}
        out["runs"][name] = {"host_wall_s_per_epoch": wall,
            "granularity": sess.granularity, "s_per_epoch": round(dt, 3),
            "edges_per_s": round(L * E / dt, 1),
            "loss_vs_resident": abs(trace[0][1] - rtrace[0][1]) / rtrace[0][1],
            "GB_per_epoch": {k: round(v["total"] / epochs / 1e9, 3) for k, v in summ["links"].items()},
            "cache_hit_rate": summ["cache"]["hit_rate"], "peak_residency_GB": {
                k: round(v / 1e9, 3) for k, v in summ["peak_residency"].items()}}
        sess.close()
        print(name, json.dumps(out["runs"][name]), flush=True)
print(json.dumps(out))
