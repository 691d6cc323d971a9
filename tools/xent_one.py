"""softmax_xent launch time at the papers chunk shape (1 M rows x 172 classes)."""
import sys
sys.path.insert(0, '.')
import torch  # noqa: E402
from paper_2605_11517_b200 import ops  # noqa: E402
n, c = 1 << 20, 172
lg = ops.zeros_rows(n, c, 'cuda'); lg[:, :c].normal_(0, 3)
lab = torch.randint(0, c, (n,), dtype=torch.int32, device='cuda')
mask = (torch.rand(n, device='cuda') < 0.5).to(torch.uint8)
g = ops.zeros_rows(n, c, 'cuda')
st = torch.zeros(4, dtype=torch.float64, device='cuda')
part = ops.loss_partials(n, 'cuda')
f = lambda: ops.softmax_xent(lg, n, c, lab, mask, int(mask.sum()), g, st, part)
for _ in range(5): f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50): f()
b.record(); torch.cuda.synchronize()
print(f"softmax_xent 1M x 172: {a.elapsed_time(b) / 50:.4f} ms")
