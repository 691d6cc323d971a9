"""Eager (per-launch Python + ctypes) vs CUDA-graph-replayed epoch: the host
overhead the sharded (N > 1, eager) engine pays per epoch."""
import sys
import time
sys.path.insert(0, '.')
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_11517_b200.training import session_for  # noqa: E402

g, ds, plan, model, _ = bench.build_workload(bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "products_sage"])
sess = session_for(ds, plan, model)
for _ in range(3):
    sess.run_epoch(0, 0.01, use_graph=False)
    sess.run_epoch(0, 0.01)
torch.cuda.synchronize()
for mode in ("graph", "eager"):
    t0 = time.perf_counter()
    cpu = 0.0
    for _ in range(10):
        c0 = time.perf_counter()
        sess.run_epoch(0, 0.01, use_graph=(mode == "graph"))
        cpu += time.perf_counter() - c0
    torch.cuda.synchronize()
    print(f"{mode}: {(time.perf_counter() - t0) / 10 * 1e3:.2f} ms/epoch wall, host enqueue {cpu / 10 * 1e3:.2f} ms")
