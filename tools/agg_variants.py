"""Aggregation variants at the papers / products shapes: times (ms, L2
flushed) and a digest of every output, so runs under different GRD_AGG_*
settings (read once per process) can be compared for speed and bitwise
equality.  Usage: GRD_AGG_BULK=1 python tools/agg_variants.py [SCALE]"""
import hashlib
import json
import os
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
flush = torch.zeros(128 * 1024 * 1024, device="cuda")
gen = torch.Generator(device="cuda").manual_seed(1)
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


def digest(t):
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:16]


res = {"knobs": {k: v for k, v in os.environ.items() if k.startswith("GRD_AGG")}, "V": n, "E": E}
heads = 4
ew = torch.rand(E * heads, device="cuda", generator=gen)
sw = torch.rand(n * heads, device="cuda", generator=gen)
for w in (128, 100, 256):
    y = torch.randn(n, ops.ld_of(w), device="cuda", generator=gen)
    out = torch.zeros(n, ops.ld_of(w), device="cuda")
    cases = [("mean", dict(post_div_deg=True, relu=True)), ("scaled", dict(src_scale=s_inv))]
    if w == 256:
        cases.append(("gat", dict(edge_w=ew, self_w=sw, heads=heads, head_ld=64)))
    for name, kw in cases:
        ms = timeit(lambda: ops.agg_sum(sg.fwd, y, out, w, **kw))
        out.zero_()
        ops.agg_sum(sg.fwd, y, out, w, **kw)
        rows = E + n
        res[f"{name}{w}"] = {"ms": round(ms, 3), "rows_GBs": round(rows * 4 * w / ms / 1e6, 1),
                             "digest": digest(out)}
    del y, out
    torch.cuda.empty_cache()
print(json.dumps(res))
