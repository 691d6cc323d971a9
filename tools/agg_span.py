"""Address-span probe of the 128-wide aggregation: the same graph and the
same gathered values, with the source rows ldy = 128 / 256 / 512 / 1024
floats apart (same lines touched, 1-8x the pages): a per-edge cost that
grows with the span is address-translation (TLB) bound, not DRAM bound.
Usage: python tools/agg_span.py [SCALE]"""
import json
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_2605_11517_b200 as g2  # noqa: E402
from paper_2605_11517_b200 import ops  # noqa: E402
from paper_2605_11517_b200.stream import StreamGraph  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = g2.generate_kronecker(scale, 12, seed=0, device="cuda")
torch.cuda.empty_cache()
sg = StreamGraph(g, torch.device("cuda"), 1 << 20, 128)
n, E = g.num_vertices, g.num_edges
out = torch.zeros(n, 128, device="cuda")
flush = torch.zeros(128 * 1024 * 1024, device="cuda")


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


res = {"V": n, "E": E}
for ld in (128, 256, 512, 1024):
    if n * ld * 4 > 80e9:
        break
    big = torch.randn(n, ld, device="cuda")
    y = big[:, :128]
    ms = timeit(lambda: ops.agg_sum(sg.fwd, y, out, 128, post_div_deg=True, relu=True))
    res[f"ld{ld}"] = {"ms": round(ms, 3), "span_GB": round(n * ld * 4 / 1e9, 1)}
    print(json.dumps(res), flush=True)
    del big, y
    torch.cuda.empty_cache()
