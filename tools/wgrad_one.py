import sys, json
sys.path.insert(0, '.')
import torch
from paper_2605_11517_b200 import ops
dev='cuda'
def timeit(fn, reps=20):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
out = {}
for m, n, k in [(128, 128, 1 << 20), (128, 172, 1 << 20), (256, 256, 2097152)]:
    a = ops.zeros_rows(k, m, dev); a.uniform_(-0.5, 0.5)
    b = ops.zeros_rows(k, n, dev); b.uniform_(-0.5, 0.5)
    dw = torch.zeros(m, ops.ld_of(n), device=dev)
    out[f"{m}x{n}"] = round(timeit(lambda: ops.wgrad_sgd(a, b, dw, m, n, k)), 4)
print(json.dumps(out))
