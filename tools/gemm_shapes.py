"""Per-launch time of the GEMM shapes an epoch runs, against the HBM time
of their compulsory bytes (A + B + C once): papers_full (chunked 1 M-row
transforms at 128 wide, the 172-class logits and their transposed
product, the whole-layer 134 M-row transform, the weight gradients) and
products (2.1 M rows x 256).  Usage: python tools/gemm_shapes.py [papers|products]"""
import json
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_2605_11517_b200 import ops  # noqa: E402

dev = 'cuda'
peak = json.load(open('MEASURED_PEAKS.json'))['hbm_gbs'] if __import__('os').path.exists('MEASURED_PEAKS.json') else 6553.0


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


which = sys.argv[1] if len(sys.argv) > 1 else "papers"
shapes = {
    "papers": [(1 << 20, 128, 128, 0), (1 << 20, 172, 128, 0), (1 << 20, 128, 172, 1),
               (1 << 24, 128, 128, 0)],
    "products": [(2097152, 512, 100, 0), (2097152, 256, 256, 0), (2097152, 47, 256, 0),
                 (2097152, 256, 47, 1)],
}[which]
wg = {"papers": [(128, 128, 1 << 20), (128, 172, 1 << 20)],
      "products": [(256, 256, 2097152), (100, 512, 2097152)]}[which]
res = {}
for m, n, k, tb in shapes:
    a = ops.zeros_rows(m, k, dev)
    a[:, :k].uniform_(-0.5, 0.5)
    b = ops.zeros_rows(n if tb else k, k if tb else n, dev)
    b.uniform_(-0.5, 0.5)
    c = ops.zeros_rows(m, n, dev)
    ms = timeit(lambda: ops.gemm(a, b, c, m, n, k, trans_b=bool(tb)))
    byt = 4 * (m * ops.ld_of(k) + m * ops.ld_of(n))
    res[f"gemm {m}x{n}x{k} tb{tb}"] = dict(ms=round(ms, 4), GBs=round(byt / ms / 1e6, 1),
                                           frac=round(byt / ms / 1e6 / peak, 3),
                                           tflops=round(2 * m * n * k / ms / 1e9, 1))
    del a, b, c
for m, n, k in wg:
    a = ops.zeros_rows(k, m, dev)
    a.uniform_(-0.5, 0.5)
    b = ops.zeros_rows(k, n, dev)
    b.uniform_(-0.5, 0.5)
    dw = torch.zeros(m, ops.ld_of(n), device=dev)
    ms = timeit(lambda: ops.wgrad_sgd(a, b, dw, m, n, k))
    byt = 4 * k * (ops.ld_of(m) + ops.ld_of(n))
    res[f"wgrad {m}x{n} K={k}"] = dict(ms=round(ms, 4), GBs=round(byt / ms / 1e6, 1),
                                       frac=round(byt / ms / 1e6 / peak, 3))
    del a, b, dw
print(json.dumps(res, indent=1))
