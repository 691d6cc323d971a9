import sys
sys.path.insert(0, '.')
import torch
import bench
from paper_2605_11517_b200 import ops
from paper_2605_11517_b200.engine import DeviceGraph
g, ds, plan, model, _ = bench.build_workload(bench.WORKLOADS["products_sage"])
dg = DeviceGraph(g, plan, "cuda")
n = g.num_vertices
Y = torch.randn(n, 96, device="cuda")
Yn = Y[:, 48:].contiguous()
Yr = Y[:, :48].contiguous()
out = torch.zeros(n, 48, device="cuda")
flush = torch.zeros(128 * 1024 * 1024, device="cuda")
def t(fn):
    ts = []
    for _ in range(7):
        flush.add_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return sorted(ts)[3]
print("strided Y_n + add_y strided", t(lambda: ops.agg_sum(dg.fwd, Y[:, 48:], out, 47, post_div_deg=2, no_self=True, add_y=Y[:, :48])))
print("dense Y_n + add_y dense", t(lambda: ops.agg_sum(dg.fwd, Yn, out, 47, post_div_deg=2, no_self=True, add_y=Yr)))
print("dense Y_n, no add_y", t(lambda: ops.agg_sum(dg.fwd, Yn, out, 47, post_div_deg=2, no_self=True)))
print("strided Y_n, no add_y", t(lambda: ops.agg_sum(dg.fwd, Y[:, 48:], out, 47, post_div_deg=2, no_self=True)))
print("bwd dense", t(lambda: ops.agg_sum(dg.bwd, Yn, out, 47, no_self=True)))
