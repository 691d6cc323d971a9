"""Aggregation launches of the streaming engine at the papers shape (one
full-graph 128-wide mean aggregation over generate_kronecker(SCALE, 12) in
vertex order, the transposed pull with a source scale), ms and DRAM-side
GB/s of the streaming model; run once per GRD_AGG_* setting (the launcher
reads its knobs once per process).  Usage: python tools/agg_papers.py [SCALE]"""
import json
import os
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_11517_b200 as g2  # noqa: E402
from paper_2605_11517_b200 import ops  # noqa: E402
from paper_2605_11517_b200.stream import StreamGraph  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = g2.generate_kronecker(scale, 12, seed=0, device="cuda")
torch.cuda.empty_cache()
sg = StreamGraph(g, torch.device("cuda"), 1 << 20, 128)
n, E = g.num_vertices, g.num_edges
y = torch.randn(n, 128, device="cuda")
out = torch.zeros(n, 128, device="cuda")
flush = torch.zeros(128 * 1024 * 1024, device="cuda")
s_inv = sg.scale("inv_deg1")


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.add_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


res = {"knobs": {k: v for k, v in os.environ.items() if k.startswith("GRD_AGG")}, "V": n, "E": E}
for name, kw in (("mean_fwd", dict(post_div_deg=True, relu=True)),
                 ("pull_scaled", dict(src_scale=s_inv))):
    ms = timeit(lambda: ops.agg_sum(sg.fwd, y, out, 128, **kw))
    model_bytes = 8 * (n + 1) + 4 * E + 512 * (E + n) + 512 * n
    res[name] = {"ms": round(ms, 3), "model_GBs": round(model_bytes / ms / 1e6, 1)}
print(json.dumps(res))
