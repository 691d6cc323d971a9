import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2605_11517_b200 import ops
torch.manual_seed(0)
m, n, k = 256, 64, 64
a = torch.randn(k, m, device='cuda')   # A^T storage
b = torch.randn(k, n, device='cuda')
c = torch.zeros(m, n, device='cuda')
ops.gemm(a, b, c, m, n, k, trans_a=True)
ref = a.double().T @ b.double()
print(os.environ.get("GRD_MN_NATIVE"), "rel", float((c.double() - ref).norm() / ref.norm()), "cnorm", float(c.norm()))
# block structure probe: which output rows are right
err_rows = ((c.double() - ref).norm(dim=1) / ref.norm(dim=1)).cpu().numpy()
print("rows ok:", np.flatnonzero(err_rows < 1e-4)[:40])
# try with A = K-contig, B = MN-major via wgrad api
dw = torch.zeros(m, n, device='cuda')
ops.wgrad_sgd(a, b, dw, m, n, k)
print("wgrad rel", float((dw.double() - ref).norm() / ref.norm()))
