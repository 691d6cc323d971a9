"""One 256-wide and one 48-wide aggregation of the products graph (for ncu)."""
import sys
sys.path.insert(0, '.')
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_11517_b200 import ops  # noqa: E402
from paper_2605_11517_b200.engine import DeviceGraph  # noqa: E402

g, ds, plan, model, _ = bench.build_workload(bench.WORKLOADS["products_sage"])
dg = DeviceGraph(g, plan, "cuda")
n = g.num_vertices
for w in (256, 48):
    y = torch.randn(n, w, device="cuda")
    out = torch.zeros(n, w, device="cuda")
    for _ in range(2):
        ops.agg_sum(dg.fwd, y, out, w, post_div_deg=2, no_self=True, relu=True)
torch.cuda.synchronize()
