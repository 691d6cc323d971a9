"""Aggregation micro-benchmark at the products shape (2.1 M V / 62.9 M E),
the aggregation calls of the bench epochs: GCN mean (self loop), SAGE mean
(no self, root add) forward, scaled transposed pulls, GAT weighted forward /
permuted pull; A/B over GRD_AGG_ASYNC in one process, L2 flushed between
launches.  Prints ms per case and variant."""
import os, sys, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2605_11517_b200 as g2
from paper_2605_11517_b200 import ops
from paper_2605_11517_b200.engine import DeviceGraph
g = g2.generate_kronecker(21, 30, seed=0)
part = g2.switching_aware_partition(g, 8, g2.PartitionerParams(seed=2))
plan = g2.build_partition_plan(g, part.labels, 8)
dev = 'cuda'
dg = DeviceGraph(g, plan, dev)
n, E = g.num_vertices, g.num_edges
flush = torch.zeros(128 * 1024 * 1024, device=dev)
def timeit(fn, reps=8):
    fn(); torch.cuda.synchronize()
    t = 0.0
    for _ in range(reps):
        flush.add_(1.0)
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        t += s.elapsed_time(e)
    return t / reps
env = os.environ.get("AGG_BENCH_ENV", "GRD_AGG_ASYNC")
widths = [int(w) for w in os.environ.get("AGG_BENCH_WIDTHS", "100,256").split(",")]
variants = sys.argv[1:] or ["0", "1"]
res = {}
inv_deg = dg.scale("inv_deg")
for w in widths:
    y = torch.randn(n, ops.ld_of(w), device=dev); out = ops.zeros_rows(n, w, dev)
    addy = torch.randn(n, ops.ld_of(w), device=dev)
    cases = {
        "gcn_fwd": (dg.fwd, dict(post_div_deg=True)),
        "sage_fwd": (dg.fwd, dict(post_div_deg=2, no_self=True, add_y=addy)),
        "sage_pull_scaled": (dg.bwd, dict(src_scale=inv_deg, no_self=True)),
        "gcn_pull": (dg.bwd, {}),
    }
    for name, (spec, kw) in cases.items():
        for v in variants:
            os.environ[env] = v
            res[f"{name}_{w}_v{v}"] = round(timeit(lambda: ops.agg_sum(spec, y, out, w, **kw)), 3)
print(json.dumps(res))
