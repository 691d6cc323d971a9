"""L2-relative error of the tensor-core GEMM / weight-gradient against
float64 at the GraphSAGE layer shapes (debugging aid)."""
import sys

sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_2605_11517_b200 import ops  # noqa: E402

dev = 'cuda'
torch.manual_seed(0)


def rel(a, b):
    return float((a - b).norm() / b.norm())


def mat(r, c, scale=1.0):
    t = ops.zeros_rows(r, c, dev)
    t[:, :c] = (torch.rand(r, c, device=dev) - 0.5) * scale
    return t


for V in (512, 2048, 16384):
    for (n, k, tb, relu) in [(256, 512, 1, True), (256, 96, 1, True), (512, 256, 0, False),
                             (96, 256, 0, False), (256, 200, 0, True), (200, 256, 1, False)]:
        a = mat(V, k)
        b = mat(n, k) if tb else mat(k, n)
        ref_t = mat(V, n) if relu else None
        c = ops.zeros_rows(V, n, dev)
        ops.gemm(a, b, c, V, n, k, trans_b=bool(tb), relu_ref=ref_t)
        A = a[:, :k].double()
        B = (b[:, :k].double().T if tb else b[:, :n].double())
        R = A @ B
        if relu:
            R = R * (ref_t[:, :n] > 0).double()
        print(f"V={V} gemm n={n} k={k} tb={tb} relu={relu}: {rel(c[:, :n].double(), R):.2e}")
    for (m, n) in [(200, 256), (256, 512), (256, 96)]:
        a = mat(V, m)
        b = mat(V, n)
        dw = torch.zeros(m, ops.ld_of(n), device=dev)
        ops.wgrad_sgd(a, b, dw, m, n, V)
        R = a[:, :m].double().T @ b[:, :n].double()
        print(f"V={V} wgrad {m}x{n}: {rel(dw[:, :n].double(), R):.2e}")
