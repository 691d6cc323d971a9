"""Tiny driver for `ncu --set full`: one forward GEMM, one weight-gradient
GEMM and one aggregation of the products-shaped workload's sizes."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2605_11517_b200 import ops
dev = 'cuda'
m, k, n = 2097152, 256, 512
a = torch.randn(m, k, device=dev); b = torch.randn(k, n, device=dev); c = torch.empty(m, n, device=dev)
ops.gemm(a, b, c, m, n, k)
dw = torch.zeros(256, 256, device=dev); h = torch.randn(m, 256, device=dev)
ops.wgrad_sgd(a, h, dw, 256, 256, m)
torch.cuda.synchronize()
