import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2605_11517_b200 import ops
m, n, k = 128, 32, 32
a = torch.arange(k * m, dtype=torch.float32, device='cuda').reshape(k, m) + 1   # A^T storage, a[k][m] = k*m+m+1
b = torch.arange(k * n, dtype=torch.float32, device='cuda').reshape(k, n) + 1
dw = torch.zeros(m, n, device='cuda')
ops.wgrad_sgd(a, b, dw, m, n, k)
torch.cuda.synchronize()
raw = np.fromfile('gpurun_out/dbg_stage.bin', dtype=np.float32)
print("A region first 64 floats:", raw[:64])
print("A region nonzero count (16KB):", np.count_nonzero(raw[:4096]))
print("B region (after 2*16KB) first 64:", raw[8192:8192+64])
print("B nonzero:", np.count_nonzero(raw[8192:8192+1024]))
ref = a.double().T @ b.double()
print("rel", float((dw.double()-ref).norm()/ref.norm()))
