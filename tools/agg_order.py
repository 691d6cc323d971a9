"""Does the row processing order of the 256-wide aggregation matter?  Same
graph / sums, rows in (a) the plan's partition order, (b) vertex order,
(c) random order, (d) descending degree."""
import sys
sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_11517_b200 import ops  # noqa: E402
from paper_2605_11517_b200.ops import AggSpec  # noqa: E402

spec = bench.WORKLOADS["products_sage"]
g, ds, plan, model, _ = bench.build_workload(spec)
n = g.num_vertices
f = plan.flat
dev = "cuda"
in_deg = np.diff(f.in_ptr)          # per perm row
deg_v = np.empty(n, np.int64)
deg_v[f.perm] = in_deg
import os  # noqa: E402
W = int(os.environ.get("AGG_ORDER_WIDTH", "256"))
y = torch.randn(n, W, device=dev)
out = torch.zeros(n, W, device=dev)
flush = torch.zeros(128 * 1024 * 1024, device=dev)


def spec_for(order):
    # rows = vertices in `order`; edges of each row in the plan's order
    rows_perm = np.empty(n, np.int64)
    rows_perm[f.perm] = np.arange(n)
    pr = rows_perm[order]                      # plan row of each new row
    cnt = in_deg[pr]
    ptr = np.zeros(n + 1, np.int64)
    np.cumsum(cnt, out=ptr[1:])
    starts = f.in_ptr[pr]
    idx = np.concatenate([f.in_src[s:s + c] for s, c in zip(starts, cnt)]) if n < 0 else None
    # vectorised gather of edge ranges
    rep = np.repeat(starts - ptr[:-1], cnt)
    idx = f.in_src[np.arange(ptr[-1]) + rep]
    sp = AggSpec.build(ptr, idx, dev, out_idx=order.astype(np.int32))
    sp.partial(W)
    return sp


def timeit(sp, reps=10):
    ts = []
    for _ in range(reps):
        flush.add_(1.0)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        ops.agg_sum(sp, y, out, W, post_div_deg=2, no_self=True, relu=True)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return sorted(ts)[len(ts) // 2]


rng = np.random.default_rng(0)
lg = np.floor(np.log2(np.maximum(deg_v, 1))).astype(np.int64)
rank = np.empty(n, np.int64)
rank[f.perm] = np.arange(n)
orders = {"plan (partition) order": f.perm.astype(np.int64), "vertex order": np.arange(n),
          "random order": rng.permutation(n), "descending degree": np.argsort(-deg_v, kind="stable"),
          "ascending degree": np.argsort(deg_v, kind="stable"),
          "log2-degree buckets desc, plan order inside": np.lexsort((rank, -lg)),
          "log2-degree buckets desc, vertex order inside": np.lexsort((np.arange(n), -lg)),
          "partition-major, descending degree inside": np.lexsort((-deg_v, plan.labels if hasattr(plan, "labels") else rank * 8 // n))}
ref = None
for name, order in orders.items():
    sp = spec_for(order)
    ms = timeit(sp)
    r = out.clone()
    if ref is None:
        ref = r
    print(f"{name:24s} {ms:7.3f} ms  identical={torch.equal(r, ref)}")
