"""Forward / input-gradient GEMM: accuracy against float64 and time per shape
for the current GRD_GEMM_PREC (bf16x3 default, tf32x3).  Run once per
setting:  GRD_GEMM_PREC=tf32x3 python tools/gemm_prec.py"""
import json
import os
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_2605_11517_b200 import ops  # noqa: E402

dev = 'cuda'


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def padded(x):
    t = ops.zeros_rows(x.shape[0], x.shape[1], dev)
    t[:, : x.shape[1]] = x
    return t


res = {"prec": os.environ.get("GRD_GEMM_PREC", "bf16x3")}
torch.manual_seed(0)
SHAPES = [(1000, 47, 13, 0), (777, 100, 300, 1), (4096, 256, 256, 0),
          (2097152, 256, 100, 0), (2097152, 512, 256, 0), (2097152, 96, 256, 0),
          (2097152, 256, 512, 1), (2097152, 100, 256, 1), (4194304, 512, 1024, 0)]
for (m, n, k, tb) in SHAPES:
    a = padded(torch.rand(m, k, device=dev) - 0.5)
    b = padded((torch.rand(n, k, device=dev) - 0.5) if tb else (torch.rand(k, n, device=dev) - 0.5))
    c = ops.zeros_rows(m, n, dev)
    fn = lambda: ops.gemm(a, b, c, m, n, k, trans_b=bool(tb))  # noqa: E731
    ms = timeit(fn, reps=5 if m > 100000 else 20)
    r = min(m, 65536)
    bb = b[:, :k].double().T if tb else b[:, :n].double()
    ref = a[:r, :k].double() @ bb
    err = float((c[:r, :n].double() - ref).norm() / ref.norm())
    res[f"{m}x{n}x{k} tb{tb}"] = dict(ms=round(ms, 4), rel_err=err,
                                      tflops=round(2 * m * n * k / ms / 1e9, 1),
                                      GBs=round(4 * (m * k + m * n) / ms / 1e6, 1))
print(json.dumps(res, indent=1))

# weight-gradient GEMMs (split-K, MN-major operands), always 3xTF32
wg = {}
for (m, n, k) in [(256, 512, 2097152), (100, 256, 2097152), (256, 96, 2097152), (1024, 512, 1048576)]:
    a = torch.rand(k, (m + 3) // 4 * 4, device=dev) - 0.5
    b = torch.rand(k, (n + 3) // 4 * 4, device=dev) - 0.5
    dw = torch.zeros(m, (n + 3) // 4 * 4, device=dev)
    ms = timeit(lambda: ops.wgrad_sgd(a, b, dw, m, n, k), reps=5)
    r = min(k, 262144)
    ops.wgrad_sgd(a[:r], b[:r], dw, m, n, r)
    ref = a[:r, :m].double().T @ b[:r, :n].double()
    err = float((dw[:, :n].double() - ref).norm() / ref.norm())
    wg[f"wgrad {m}x{n} K={k}"] = dict(ms=round(ms, 4), rel_err=err,
                                     GBs=round(4 * k * (m + n) / ms / 1e6, 1))
print(json.dumps(wg, indent=1))
