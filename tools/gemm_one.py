"""One forward GEMM launch of a given shape (for ncu): M N K [trans_b]."""
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_2605_11517_b200 import ops  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
tb = len(sys.argv) > 4 and sys.argv[4] == "1"
dev = "cuda"
a = ops.zeros_rows(m, k, dev)
a[:, :k] = torch.rand(m, k, device=dev) - 0.5
b = ops.zeros_rows(n if tb else k, k if tb else n, dev)
b.uniform_(-0.5, 0.5)
c = ops.zeros_rows(m, n, dev)
for _ in range(3):
    ops.gemm(a, b, c, m, n, k, trans_b=tb)
torch.cuda.synchronize()
