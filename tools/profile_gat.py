"""Driver for `ncu --set full` of the GAT kernels at the products shape:
one edge softmax, one forward weighted aggregation, one edge backward and
one transposed (permuted-weight) pull, hdp = 4 x 64."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2605_11517_b200 as g2
from paper_2605_11517_b200 import ops
from paper_2605_11517_b200.engine import DeviceGraph
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 21
g = g2.generate_kronecker(scale, 30, seed=0)
plan = g2.build_partition_plan(g, g2.random_partition(g.num_vertices, 8, 1), 8)
dev = 'cuda'
dg = DeviceGraph(g, plan, dev)
n, H, dhp = g.num_vertices, 4, 64
hdp = H * dhp
ld_ext = ops.ld_of(hdp + 2 * H)
pext = torch.randn(n, ld_ext, device=dev)
E = dg.fwd.nnz
alpha = torch.zeros(E * H, device=dev); aself = torch.zeros(n * H, device=dev)
st = ops.zeros_rows(n, 2 * H, dev)
ops.gat_pack_scores(pext, n, H, dhp, st)
ops.gat_softmax(dg.fwd, pext, H, dhp, alpha, aself, st=st)
O = ops.zeros_rows(n, hdp, dev)
ops.agg_sum(dg.fwd, pext[:, :hdp], O, hdp, edge_w=alpha, self_w=aself, heads=H, head_ld=dhp, relu=True)
go = torch.randn(n, hdp, device=dev)
delta = torch.zeros_like(alpha); dself = torch.zeros_like(aself)
gext = ops.zeros_rows(n, ld_ext, dev)
ops.gat_softmax_bwd(dg.fwd, pext, H, dhp, alpha, aself, go, O, delta, dself, gext)
perm = dg.out_to_in_perm()
ops.agg_sum(dg.bwd, go, gext[:, :hdp], hdp, edge_w=alpha, edge_w_perm=perm, self_w=aself, heads=H, head_ld=dhp)
ops.gat_src_grad(dg.bwd, H, dhp, perm, delta, dself, gext)
torch.cuda.synchronize()
print("ok", n, E, dg.fwd.n_heavy, dg.fwd.n_segs)
# the fused pull backward (default path): row dots, the pull, the target sums
cdot = torch.zeros(n * H, device=dev)
ops.gat_row_dots(go, O, n, H, dhp, cdot)
ops.gat_pull_bwd(dg.bwd, pext, H, dhp, perm, alpha, aself, go, cdot, delta, dself, gext, st=st)
ops.gat_dst_grad(dg.fwd, H, dhp, delta, dself, gext)
torch.cuda.synchronize()
print("fused ok")
