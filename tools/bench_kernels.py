"""Micro-benchmark of individual kernels (GEMM shapes of the GNN layers, aggregation)."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2605_11517_b200 import ops

dev = 'cuda'
def timeit(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

res = {}
for (m, n, k, ta, tb) in [(131072, 64, 128, 0, 0), (2097152, 256, 256, 0, 0), (2097152, 512, 256, 0, 0),
                          (2097152, 256, 100, 0, 0), (2097152, 100, 256, 0, 1), (2097152, 47, 256, 0, 0)]:
    a = torch.randn((k, m) if ta else (m, k), device=dev)
    b = torch.randn((n, k) if tb else (k, n), device=dev)
    c = torch.empty((m, (n + 3) // 4 * 4), device=dev)
    a = ops.zeros_rows(a.shape[0], a.shape[1], dev).copy_(torch.nn.functional.pad(a, (0, (-a.shape[1]) % 4)))
    b = ops.zeros_rows(b.shape[0], b.shape[1], dev).copy_(torch.nn.functional.pad(b, (0, (-b.shape[1]) % 4)))
    ms = timeit(lambda: ops.gemm(a, b, c, m, n, k, trans_a=bool(ta), trans_b=bool(tb)))
    ref = (a[:, :k].double() @ (b[:, :k].double().T if tb else b[:, :n].double())) if m <= 131072 else None
    err = None
    if ref is not None:
        err = float((c[:, :n].double() - ref).norm() / ref.norm())
    gb = 4 * (m * k + k * n + m * n) / 1e9
    res[f"gemm {m}x{n}x{k} ta{ta} tb{tb}"] = dict(ms=round(ms, 4), tflops=round(2 * m * n * k / ms / 1e9, 1),
                                                   GBs=round(gb / ms * 1e3, 1), rel_err=err)
for (m, n, k) in [(128, 64, 131072), (256, 256, 2097152), (100, 256, 2097152)]:
    a = torch.randn(k, (m + 3) // 4 * 4, device=dev); b = torch.randn(k, (n + 3) // 4 * 4, device=dev)
    dw = torch.zeros(m, (n + 3) // 4 * 4, device=dev)
    ms = timeit(lambda: ops.wgrad_sgd(a, b, dw, m, n, k))
    ref = a[:, :m].double().T @ b[:, :n].double()
    err = float((dw[:, :n].double() - ref).norm() / ref.norm())
    res[f"wgrad {m}x{n} K={k}"] = dict(ms=round(ms, 4), tflops=round(2 * m * n * k / ms / 1e9, 1),
                                       GBs=round(4 * k * (m + n) / ms / 1e6, 1), rel_err=err)
print(json.dumps(res, indent=1))
