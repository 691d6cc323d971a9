"""Aggregation micro-benchmark at the products shape (2.1 M V / 62.9 M E):
plain mean sums at widths 47/100/256 (forward in-CSR and transposed pull)
and the GAT weighted forward / permuted pull at 4 x 64, L2 flushed between
launches.  Prints ms and algorithmic GB/s per case."""
import sys, json
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
def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    t = 0.0
    for _ in range(reps):
        flush.add_(1.0)
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        t += s.elapsed_time(e)
    return t / reps
res = {}
for w in (47, 100, 256):
    y = torch.randn(n, ops.ld_of(w), device=dev); out = ops.zeros_rows(n, w, dev)
    for name, spec, kw in (("fwd", dg.fwd, dict(post_div_deg=True)), ("pull", dg.bwd, {})):
        ms = timeit(lambda: ops.agg_sum(spec, y, out, w, **kw))
        gb = (8 * (n + 1) + 4 * E + 4 * w * (E + n) + 4 * w * n) / 1e9
        res[f"mean_{name}_{w}"] = dict(ms=round(ms, 3), GBs=round(gb / ms * 1e3, 1))
H, dhp = 4, 64
hdp = H * dhp
y = torch.randn(n, hdp, device=dev); out = ops.zeros_rows(n, hdp, dev)
alpha = torch.rand(E * H, device=dev); aself = torch.rand(n * H, device=dev)
perm = dg.out_to_in_perm()
ms = timeit(lambda: ops.agg_sum(dg.fwd, y, out, hdp, edge_w=alpha, self_w=aself, heads=H, head_ld=dhp))
gb = (8 * (n + 1) + 4 * E + 4 * hdp * (E + 2 * n) + 16 * (E + n)) / 1e9
res["gat_fwd_256"] = dict(ms=round(ms, 3), GBs=round(gb / ms * 1e3, 1))
ms = timeit(lambda: ops.agg_sum(dg.bwd, y, out, hdp, edge_w=alpha, edge_w_perm=perm, self_w=aself, heads=H,
                                head_ld=dhp))
res["gat_pull_256"] = dict(ms=round(ms, 3), GBs=round((gb + 4 * E) / ms * 1e3, 1))
print(json.dumps(res))
