"""Host-link probe: DMA H2D / D2H bandwidth from pinned memory and the
GPU-initiated (zero-copy) row gather from pinned host memory."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2605_11517_b200 import ops
dev = 'cuda'
V, d = 16_777_216, 128
host = torch.empty((V, d), dtype=torch.float32).pin_memory()
host.normal_()
dbuf = torch.empty((V // 2, d), device=dev)
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    s = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - s) / reps
n = V // 2
tt = t(lambda: dbuf.copy_(host[:n], non_blocking=True))
print(f"H2D DMA {n*d*4/tt/1e9:.1f} GB/s")
tt = t(lambda: host[:n].copy_(dbuf, non_blocking=True))
print(f"D2H DMA {n*d*4/tt/1e9:.1f} GB/s")
for name, idx in (("sequential", torch.arange(n, dtype=torch.int32, device=dev)),
                  ("random", torch.randint(0, V, (n,), dtype=torch.int32, device=dev))):
    tt = t(lambda: ops.gather_rows(host, idx, dbuf, d))
    print(f"zero-copy gather {name} 512B rows: {n*d*4/tt/1e9:.1f} GB/s")
for w in (32, 64):
    idx = torch.randint(0, V, (n,), dtype=torch.int32, device=dev)
    tt = t(lambda: ops.gather_rows(host, idx, dbuf, w))
    print(f"zero-copy gather random {w*4}B of 512B rows: {n*w*4/tt/1e9:.1f} GB/s")
