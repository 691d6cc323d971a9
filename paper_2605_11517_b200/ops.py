"""Thin launch wrappers over the C ABI for torch CUDA tensors.

Every function launches one of the library's sm_100a kernels on torch's
current stream; no torch compute op is used on the training path.  Dense
device matrices are fp32, row-major, with ``ld = round_up(width, 4)`` and
zero padding columns (see include/grinder_b200.h).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

__all__ = ["AggSpec", "agg_sum", "gather_rows", "gemm", "ld_of", "mask_scale_rows",
           "mul_rows", "rownorm_bwd", "rownorm_fwd", "scatter_add_rows", "softmax_xent",
           "stream_ptr", "wgrad_sgd", "zeros_rows"]

HEAVY_THRESHOLD = 128   # rows above this degree are split ...
SEGMENT_EDGES = 128     # ... into segments of this many edges


class Recorder:
    """Launch accounting for the benchmark: counts this library's kernel
    launches and, when ``timing`` is on, brackets each op with CUDA events on
    the launching stream together with its algorithmic bytes / flops."""

    def __init__(self):
        self.launches = 0
        self.calls = 0
        self.timing = False
        self.records: list = []

    def reset(self) -> None:
        self.launches = 0
        self.records = []


RECORDER = Recorder()


# GRD_NVTX=1: every op is an NVTX range "<op>#<n>" (n counts op calls), so
# `ncu --nvtx --print-nvtx-rename kernel` attributes each CUDA kernel to the
# op invocation that launched it (tools/dram_traffic.py)
_NVTX = os.environ.get("GRD_NVTX", "0") == "1"


def _launch(name: str, nlaunch: int, nbytes: float, flops: float, fn) -> None:
    RECORDER.launches += nlaunch
    if _NVTX:
        RECORDER.calls += 1
        torch.cuda.nvtx.range_push(f"{name}#{RECORDER.calls}")
        try:
            _launch_inner(name, nbytes, flops, fn)
        finally:
            torch.cuda.nvtx.range_pop()
        return
    _launch_inner(name, nbytes, flops, fn)


def _launch_inner(name: str, nbytes: float, flops: float, fn) -> None:
    if not RECORDER.timing:
        fn()
        return
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record()
    fn()
    end.record()
    RECORDER.records.append((name, float(nbytes), float(flops), start, end))


def ld_of(width: int) -> int:
    return (int(width) + 3) // 4 * 4


def zeros_rows(rows: int, width: int, device) -> torch.Tensor:
    """Zero-initialised [rows, ld_of(width)] fp32 matrix (padding stays 0)."""
    return torch.zeros((int(rows), ld_of(width)), dtype=torch.float32, device=device)


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def _p(t) -> int | None:
    return None if t is None else t.data_ptr()


def _ld(t: torch.Tensor) -> int:
    return int(t.stride(0))


SMALL_EDGES = 3   # grd_gat_args.n_small: rows the GAT softmax runs at 4 lanes per row
MID_EDGES = 15    # grd_gat_args.n_mid: at 16 lanes per row


def _small_tail(deg: np.ndarray, limit: int) -> int:
    """Length of the trailing run of rows with <= limit edges (the
    low-degree tail of the degree-sorted device CSRs)."""
    big = np.flatnonzero(deg > limit)
    return int(deg.size - (big[-1] + 1 if big.size else 0))


@dataclass
class AggSpec:
    """A static CSR over which rows are sum-aggregated, uploaded once, with
    its deterministic heavy-row segmentation (include/grinder_b200.h K2)."""

    n_rows: int
    row_ptr: torch.Tensor            # int64 [n_rows+1]
    idx: torch.Tensor                # int32 [nnz]
    out_idx: torch.Tensor | None     # int32 [n_rows]
    self_idx: torch.Tensor | None    # int32 [n_rows]
    heavy_rows: torch.Tensor | None
    heavy_seg_ptr: torch.Tensor | None
    seg_heavy: torch.Tensor | None
    heavy_counter: torch.Tensor | None
    n_heavy: int
    n_segs: int
    nnz: int
    _partial: torch.Tensor | None = None
    n_small: int = 0                 # trailing rows with <= SMALL_EDGES edges
    n_mid: int = 0                   # rows before them with <= MID_EDGES edges

    @classmethod
    def build(cls, row_ptr: np.ndarray, idx: np.ndarray, device, out_idx=None, self_idx=None,
              heavy_threshold: int = HEAVY_THRESHOLD, seg_len: int = SEGMENT_EDGES) -> "AggSpec":
        row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        n = row_ptr.size - 1
        deg = np.diff(row_ptr)
        heavy = np.flatnonzero(deg > heavy_threshold).astype(np.int32)
        nseg = (deg[heavy] + seg_len - 1) // seg_len
        seg_ptr = np.zeros(heavy.size + 1, dtype=np.int64)
        np.cumsum(nseg, out=seg_ptr[1:])
        seg_heavy = np.repeat(np.arange(heavy.size, dtype=np.int32), nseg)

        def up(a, dt):
            if a is None:
                return None
            return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(device)

        has_heavy = heavy.size > 0
        return cls(
            n_rows=n, row_ptr=up(row_ptr, np.int64), idx=up(idx, np.int32),
            out_idx=up(out_idx, np.int32), self_idx=up(self_idx, np.int32),
            heavy_rows=up(heavy, np.int32) if has_heavy else None,
            heavy_seg_ptr=up(seg_ptr, np.int64) if has_heavy else None,
            seg_heavy=up(seg_heavy, np.int32) if has_heavy else None,
            heavy_counter=torch.zeros(16 * max(heavy.size, 1), dtype=torch.int32, device=device)
            if has_heavy else None,
            n_heavy=int(heavy.size), n_segs=int(seg_heavy.size), nnz=int(row_ptr[-1]),
            n_small=_small_tail(deg, SMALL_EDGES),
            n_mid=_small_tail(deg, MID_EDGES) - _small_tail(deg, SMALL_EDGES),
        )

    def partial(self, width: int) -> torch.Tensor | None:
        if self.n_segs == 0:
            return None
        need = self.n_segs * ld_of(width)
        if self._partial is None or self._partial.numel() < need:
            self._partial = torch.empty(need, dtype=torch.float32, device=self.row_ptr.device)
        return self._partial


def agg_sum(spec: AggSpec, y: torch.Tensor, out: torch.Tensor, width: int, *,
            src_scale=None, post_scale=None, post_div_deg=False, relu=False,
            mask_ref=None, no_self=False, add_y=None, edge_w=None, edge_w_perm=None,
            self_w=None, heads=1, head_ld=4) -> None:
    """out[o] = act(post(sum_e y[idx_e] (+ y[self])) + add_y[o]); post_div_deg:
    False/0 none, True/1 divide by deg+1, 2 divide by deg (GraphSAGE mean)."""
    a = _lib.GrdAggArgs()
    a.n_rows = spec.n_rows
    a.row_ptr = _p(spec.row_ptr)
    a.idx = _p(spec.idx)
    a.out_idx = _p(spec.out_idx)
    a.self_idx = _p(spec.self_idx)
    a.y = _p(y)
    a.ldy = _ld(y)
    a.src_scale = _p(src_scale)
    a.post_scale = _p(post_scale)
    a.post_div_deg = int(post_div_deg)
    a.relu = int(bool(relu))
    a.out = _p(out)
    a.ldo = _ld(out)
    a.width = int(width)
    a.heavy_threshold = HEAVY_THRESHOLD if spec.n_segs else 0
    a.n_heavy = spec.n_heavy
    a.heavy_rows = _p(spec.heavy_rows)
    a.heavy_seg_ptr = _p(spec.heavy_seg_ptr)
    a.seg_heavy = _p(spec.seg_heavy)
    a.n_segs = spec.n_segs
    a.seg_len = SEGMENT_EDGES
    a.seg_partial = _p(spec.partial(width))
    a.heavy_counter = _p(spec.heavy_counter)
    a.mask_ref = _p(mask_ref)
    a.ld_mask_ref = _ld(mask_ref) if mask_ref is not None else 0
    a.no_self = int(bool(no_self))
    a.add_y = _p(add_y)
    a.ld_add_y = _ld(add_y) if add_y is not None else 0
    a.edge_w = _p(edge_w)
    a.edge_w_perm = _p(edge_w_perm)
    a.self_w = _p(self_w)
    a.heads = int(heads)
    a.head_ld = int(head_ld)
    R, E, w = spec.n_rows, spec.nnz, int(width)
    nbytes = 8 * (R + 1) + 4 * E + 4 * w * (E + R * (not no_self)) + 4 * w * R
    nbytes += 4 * w * R * (add_y is not None) + 4 * int(heads) * (E + R) * (edge_w is not None)
    nbytes += 4 * R * ((spec.out_idx is not None) + (spec.self_idx is not None)
                       + (post_scale is not None))
    nbytes += 4 * (E + R) * (src_scale is not None) + 4 * w * R * (mask_ref is not None)
    _launch("agg_sum", 1, nbytes, 2.0 * w * (E + R),
            lambda: _lib.check(_lib.lib().grd_agg_sum(ctypes.byref(a), stream_ptr()), "agg_sum"))


# K chunk of one tensor-core accumulation (GRD_GEMM_KCHUNK; 0 = whole K).
# tcgen05's fused accumulation truncates, so the 3xTF32 error grows with the
# number of MMAs summed into one accumulator (~2e-6 relative at K = 128,
# ~4e-6 at K = 512 on random data) and is biased; gradients that sum many
# cancelling terms amplify it (GraphSAGE at F = 100 / H = 256: 1.4e-3 on
# layer 0's weight gradient).  K deeper than _KMAX (192: the GraphSAGE
# K = 200 case needs the split, the papers K = 172 product does not,
# tools/prec_matrix.py) is split into 128-deep chunks whose partials the
# epilogue adds to C with round-to-nearest fp32 adds (its accumulate path);
# the row scale / element multiply / ReLU apply with the last chunk.  (An
# in-kernel variant, GRD_GEMM_KCH, measured slower.)  Weight gradients
# (trans_a) use in-kernel fresh accumulators instead (GRD_WGRAD_FRESH).
_KCHUNK = int(os.environ.get("GRD_GEMM_KCHUNK", "128"))
_KMAX = int(os.environ.get("GRD_GEMM_KMAX", "192"))
# Input-gradient GEMMs (A @ W^T) stay whole (GRD_GEMM_KSPLIT_TB=1 splits
# them too): the GraphSAGE K = 512 input gradient unsplit leaves every weight
# gradient's error where it was (6.0e-5 / 2.8e-5 / 7.8e-6 at the products
# widths; tools/prec_matrix.py) and saves three read-modify-write passes
# over its 2.1 GB output: products_sage GEMM 15.7 -> 12.1 ms per epoch.
_KSPLIT_TB = os.environ.get("GRD_GEMM_KSPLIT_TB", "0") != "0"


def gemm(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor, m: int, n: int, k: int, *,
         trans_a=False, trans_b=False, row_scale=None, elem_mul=None, relu_ref=None,
         relu_out=False, accumulate=False, c2=None, split=0) -> None:
    """c[:m,:n] (=|+=) epi(opA(a) @ opB(b)) over the first k of the inner dim;
    with c2, columns >= split land in c2[:, col - split] instead."""
    k = int(k)
    if _KCHUNK and k > max(_KCHUNK, _KMAX) and not trans_a and c2 is None and (_KSPLIT_TB or not trans_b):
        starts = list(range(0, k, _KCHUNK))
        for i, k0 in enumerate(starts):
            k1 = min(k, k0 + _KCHUNK)
            last = i == len(starts) - 1
            _gemm_once(a[:, k0:], b[:, k0:] if trans_b else b[k0:], c, m, n, k1 - k0,
                       trans_b=trans_b, row_scale=row_scale if last else None,
                       elem_mul=elem_mul if last else None, relu_ref=relu_ref if last else None,
                       relu_out=relu_out and last, accumulate=accumulate or i > 0)
        return
    _gemm_once(a, b, c, m, n, k, trans_a=trans_a, trans_b=trans_b, row_scale=row_scale,
               elem_mul=elem_mul, relu_ref=relu_ref, relu_out=relu_out, accumulate=accumulate,
               c2=c2, split=split)


def _gemm_once(a, b, c, m, n, k, *, trans_a=False, trans_b=False, row_scale=None, elem_mul=None,
               relu_ref=None, relu_out=False, accumulate=False, c2=None, split=0) -> None:
    g = _lib.GrdGemmArgs()
    g.m, g.n, g.k = int(m), int(n), int(k)
    g.a, g.lda, g.trans_a = _p(a), _ld(a), int(bool(trans_a))
    g.b, g.ldb, g.trans_b = _p(b), _ld(b), int(bool(trans_b))
    g.c, g.ldc = _p(c), _ld(c)
    g.row_scale = _p(row_scale)
    g.elem_mul = _p(elem_mul)
    g.ld_elem_mul = _ld(elem_mul) if elem_mul is not None else 0
    g.relu_ref = _p(relu_ref)
    g.ld_relu_ref = _ld(relu_ref) if relu_ref is not None else 0
    g.relu_out = int(bool(relu_out))
    g.accumulate = int(bool(accumulate))
    g.c2 = _p(c2)
    g.ldc2 = _ld(c2) if c2 is not None else 0
    g.split = int(split) if c2 is not None else 0
    m, n, k = int(m), int(n), int(k)
    need = int(_lib.lib().grd_gemm_workspace(n, k))
    ws = _workspace(("pack", c.device), need)
    g.workspace = _p(ws)
    g.workspace_elems = ws.numel()
    nbytes = 4 * (m * k + k * n + m * n) + 4 * m * (row_scale is not None)
    nbytes += 4 * m * n * ((elem_mul is not None) + (relu_ref is not None) + bool(accumulate))
    _launch("gemm", 2, nbytes, 2.0 * m * n * k,
            lambda: _lib.check(_lib.lib().grd_gemm(ctypes.byref(g), stream_ptr()), "gemm"))


_WS: dict = {}


def _workspace(key, elems: int) -> torch.Tensor:
    """Scratch buffers of the library (grown on demand, reused; allocated
    before CUDA-graph capture by the engine's warm-up epoch)."""
    if not isinstance(key, tuple):
        key = ("wgrad", key)
    device = key[1]
    ws = _WS.get((key[0], str(device)))
    if ws is None or ws.numel() < elems:
        ws = torch.empty(max(elems, 1), dtype=torch.float32, device=device)
        _WS[(key[0], str(device))] = ws
    return ws


def wgrad_sgd(a: torch.Tensor, b: torch.Tensor, dw: torch.Tensor, m: int, n: int, k: int, *,
              accumulate=False, w: torch.Tensor | None = None, lr: float = 0.0) -> None:
    """dw[:m,:n] (=|+=) a[:k,:m]^T @ b[:k,:n]; then w -= lr*dw if w given."""
    L = _lib.lib()
    need = int(L.grd_wgrad_workspace(m, n, k))
    ws = _workspace(dw.device, need)
    nbytes = 4 * (k * m + k * n + m * n) + 8 * m * n * (w is not None) + 4 * m * n * bool(accumulate)
    _launch("wgrad_sgd", 2, nbytes, 2.0 * m * n * k, lambda: _lib.check(L.grd_wgrad_sgd(
        int(m), int(n), int(k), _p(a), _ld(a), _p(b), _ld(b), _p(dw), _ld(dw),
        int(bool(accumulate)), _p(w), _ld(w) if w is not None else 0, float(lr), _p(ws),
        ws.numel(), stream_ptr()), "wgrad_sgd"))


def gather_rows(src: torch.Tensor, idx: torch.Tensor, dst: torch.Tensor, width: int) -> None:
    n = idx.numel()
    _launch("gather_rows", 1, 4 * n + 8 * n * int(width), 0, lambda: _lib.check(
        _lib.lib().grd_gather_rows(_p(src), _ld(src), _p(idx), n, int(width), _p(dst), _ld(dst),
                                   stream_ptr()), "gather_rows"))


def scatter_add_rows(src: torch.Tensor, idx: torch.Tensor, dst: torch.Tensor, width: int) -> None:
    n = idx.numel()
    _launch("scatter_add_rows", 1, 4 * n + 12 * n * int(width), n * int(width), lambda: _lib.check(
        _lib.lib().grd_scatter_add_rows(_p(src), _ld(src), _p(idx), n, int(width), _p(dst), _ld(dst),
                                        stream_ptr()), "scatter_add_rows"))


def mul_rows(x: torch.Tensor, m: torch.Tensor, y: torch.Tensor, n_rows: int, width: int) -> None:
    _launch("mul_rows", 1, 12 * int(n_rows) * int(width), int(n_rows) * int(width), lambda: _lib.check(
        _lib.lib().grd_mul_rows(_p(x), _ld(x), _p(m), _ld(m), int(n_rows), int(width), _p(y), _ld(y),
                                stream_ptr()), "mul_rows"))


def mask_scale_rows(x: torch.Tensor, y: torch.Tensor, n_rows: int, width: int, *, ref=None,
                    row_scale=None) -> None:
    _launch("mask_scale_rows", 1, 12 * int(n_rows) * int(width), int(n_rows) * int(width),
            lambda: _lib.check(_lib.lib().grd_mask_scale_rows(
                _p(x), _ld(x), _p(ref), _ld(ref) if ref is not None else 0, _p(row_scale),
                int(n_rows), int(width), _p(y), _ld(y), stream_ptr()), "mask_scale_rows"))


def rownorm_fwd(pre: torch.Tensor, out: torch.Tensor, n_rows: int, width: int, relu: bool,
                out_idx=None) -> None:
    _launch("rownorm_fwd", 1, 8 * int(n_rows) * int(width), 3 * int(n_rows) * int(width),
            lambda: _lib.check(_lib.lib().grd_rownorm_fwd(
                _p(pre), _ld(pre), int(n_rows), int(width), int(relu), _p(out_idx), _p(out), _ld(out),
                stream_ptr()), "rownorm_fwd"))


def rownorm_bwd(pre: torch.Tensor, grad_y: torch.Tensor, grad_pre: torch.Tensor, n_rows: int,
                width: int, *, a_out=None, row_scale=None) -> None:
    _launch("rownorm_bwd", 1, 16 * int(n_rows) * int(width), 8 * int(n_rows) * int(width),
            lambda: _lib.check(_lib.lib().grd_rownorm_bwd(
                _p(pre), _ld(pre), _p(grad_y), _ld(grad_y), _p(a_out),
                _ld(a_out) if a_out is not None else 0, int(n_rows), int(width), _p(row_scale),
                _p(grad_pre), _ld(grad_pre), stream_ptr()), "rownorm_bwd"))


def softmax_xent(logits: torch.Tensor, n_rows: int, n_classes: int, labels: torch.Tensor,
                 mask: torch.Tensor, mask_count: int, grad: torch.Tensor, stats: torch.Tensor,
                 partials: torch.Tensor, grad_scale=None, grad2=None, grad2_scale=None) -> None:
    """stats (float64 cuda[4]) <- {loss, accuracy, loss_sum, correct};
    optionally grad2 = grad * grad2_scale (per row) as well."""
    n, c = int(n_rows), int(n_classes)
    nbytes = 8 * n * c + 9 * n + 4 * n * (grad_scale is not None)
    nbytes += (4 * n * c + 4 * n) * (grad2 is not None)
    _launch("softmax_xent", 2, nbytes, 6.0 * n * c, lambda: _lib.check(_lib.lib().grd_softmax_xent2(
        _p(logits), _ld(logits), n, c, _p(labels), _p(mask), int(mask_count), _p(grad), _ld(grad),
        _p(grad_scale), _p(grad2), _ld(grad2) if grad2 is not None else 0, _p(grad2_scale),
        _p(partials), _p(stats), stream_ptr()), "softmax_xent"))


def loss_partials(n_rows: int, device) -> torch.Tensor:
    return torch.empty(int(_lib.lib().grd_loss_partials(int(n_rows))), dtype=torch.float64,
                       device=device)


# ---------------------------------------------------------------- GAT ops --
def _gat_args(spec: AggSpec, p_ext, heads, dhp, **kw):
    a = _lib.GrdGatArgs()
    a.n_rows = spec.n_rows
    a.row_ptr = _p(spec.row_ptr)
    a.idx = _p(spec.idx)
    a.out_idx = _p(spec.out_idx)
    a.p_ext = _p(p_ext)
    a.ld_ext = _ld(p_ext)
    a.heads, a.dhp, a.hdp = int(heads), int(dhp), int(heads) * int(dhp)
    a.slope = 0.2
    a.heavy_threshold = HEAVY_THRESHOLD
    a.seg_len = SEGMENT_EDGES
    a.n_heavy = spec.n_heavy
    a.heavy_rows = _p(spec.heavy_rows)
    a.heavy_seg_ptr = _p(spec.heavy_seg_ptr)
    a.seg_heavy = _p(spec.seg_heavy)
    a.n_segs = spec.n_segs
    a.seg_scratch = _p(spec.partial(2 * int(heads)))
    a.n_small = spec.n_small
    a.n_mid = spec.n_mid
    for k, v in kw.items():
        if k.startswith("ld_"):
            setattr(a, k, int(v))
        else:
            setattr(a, k, _p(v))
    return a


def gat_pack_scores(p_ext, n_rows, heads, dhp, st) -> None:
    """st[:, 0:2H] = [s | t] columns of P_ext (compact score table)."""
    H = int(heads)
    _launch("gat_params", 1, 4 * int(n_rows) * 4 * H, 0, lambda: _lib.check(_lib.lib().grd_gat_pack_scores(
        _p(p_ext), _ld(p_ext), int(n_rows), H, H * int(dhp), _p(st), _ld(st), stream_ptr()),
        "gat_pack_scores"))


def gat_softmax(spec, p_ext, heads, dhp, alpha, alpha_self, st=None) -> None:
    """alpha = edge softmax of LeakyReLU(s_u + t_v) over in(v) + self loop
    (scores from the compact table ``st`` when given)."""
    kw = {} if st is None else dict(st=st, ld_st=_ld(st))
    a = _gat_args(spec, p_ext, heads, dhp, alpha=alpha, alpha_self=alpha_self, **kw)
    E, R = spec.nnz, spec.n_rows
    # idx + s_u sector per edge, t_v per row, alpha written
    nbytes = 8 * (R + 1) + 4 * E + 4 * heads * (E + R) * 2 + 4 * heads * R
    launches = 1 + (spec.n_mid > 0) + (spec.n_small > 0) + 2 * (spec.n_segs > 0)
    _launch("gat_softmax", launches, nbytes, 8.0 * heads * (E + R),
            lambda: _lib.check(_lib.lib().grd_gat_softmax(ctypes.byref(a), stream_ptr()), "gat_softmax"))


def gat_softmax_bwd(spec, p_ext, heads, dhp, alpha, alpha_self, grad_o, o_fwd, delta, delta_self,
                    grad_ext) -> None:
    """Per-edge score gradients delta and the target-score gradient dt."""
    a = _gat_args(spec, p_ext, heads, dhp, alpha=alpha, alpha_self=alpha_self, grad_o=grad_o,
                  ld_go=_ld(grad_o), o_fwd=o_fwd, ld_o=_ld(o_fwd), delta=delta,
                  delta_self=delta_self, grad_ext=grad_ext, ld_gext=_ld(grad_ext))
    E, R, hdp = spec.nnz, spec.n_rows, heads * dhp
    # P_u row per edge (+ self), gO and O rows per target, alpha/s read, delta written
    nbytes = 8 * (R + 1) + 4 * E + 4 * hdp * (E + 3 * R) + 3 * 4 * heads * (E + R)
    _launch("gat_softmax_bwd", 1 + (spec.n_heavy > 0), nbytes, 2.0 * hdp * (E + 2 * R),
            lambda: _lib.check(_lib.lib().grd_gat_softmax_bwd(ctypes.byref(a), stream_ptr()),
                               "gat_softmax_bwd"))


def gat_src_grad(spec, heads, dhp, edge_perm, delta, delta_self, grad_ext) -> None:
    a = _gat_args(spec, grad_ext, heads, dhp, edge_perm=edge_perm, delta=delta, delta_self=delta_self,
                  grad_ext=grad_ext, ld_gext=_ld(grad_ext))
    E, R = spec.nnz, spec.n_rows
    _launch("gat_src_grad", 1 + (spec.n_mid > 0) + (spec.n_small > 0) + (spec.n_heavy > 0), 8 * E + 4 * heads * (E + 2 * R), heads * E,
            lambda: _lib.check(_lib.lib().grd_gat_src_grad(ctypes.byref(a), stream_ptr()),
                               "gat_src_grad"))


def gat_row_dots(g, o, n_rows, heads, dhp, c) -> None:
    """c[r, h] = gO_r,h . O_r,h (the softmax backward's per-target term)."""
    _launch("gat_row_dots", 1, 8 * int(n_rows) * int(heads) * int(dhp) + 4 * int(n_rows) * int(heads),
            2.0 * int(n_rows) * int(heads) * int(dhp),
            lambda: _lib.check(_lib.lib().grd_gat_row_dots(
                _p(g), _ld(g), _p(o), _ld(o), int(n_rows), int(heads), int(dhp), _p(c), stream_ptr()),
                "gat_row_dots"))


def gat_pull_bwd(spec, p_ext, heads, dhp, edge_perm, alpha, alpha_self, grad_o, c_dot, delta,
                 delta_self, grad_ext, alpha_t=None, st=None) -> None:
    """Fused GAT backward over the transposed pull: dP, ds and the per-edge
    score gradients delta from one gather of gO_v per edge."""
    H = int(heads)
    hdp = H * int(dhp)
    kw = {} if st is None else dict(st=st, ld_st=_ld(st))
    a = _gat_args(spec, p_ext, heads, dhp, edge_perm=edge_perm, alpha=alpha, alpha_self=alpha_self,
                  grad_o=grad_o, ld_go=_ld(grad_o), c_dot=c_dot, delta=delta, delta_self=delta_self,
                  grad_ext=grad_ext, ld_gext=_ld(grad_ext), alpha_t=alpha_t,
                  seg_wide=spec.partial(hdp + H), **kw)
    E, R = spec.nnz, spec.n_rows
    # per edge: idx + perm, the gO_v row, alpha / t / c / delta per head;
    # per row: own P and gO rows, dP + ds written
    nbytes = 8 * (R + 1) + 8 * E + 4 * hdp * (E + 3 * R) + 4 * H * (4 * E + 3 * R)
    _launch("gat_pull_bwd", 1 + (spec.n_heavy > 0), nbytes, 4.0 * hdp * (E + R),
            lambda: _lib.check(_lib.lib().grd_gat_pull_bwd(ctypes.byref(a), stream_ptr()),
                               "gat_pull_bwd"))


def gat_dst_grad(spec, heads, dhp, delta, delta_self, grad_ext) -> None:
    """dt_v = sum of delta over v's in-edges (+ the self term), forward CSR order."""
    a = _gat_args(spec, grad_ext, heads, dhp, delta=delta, delta_self=delta_self,
                  grad_ext=grad_ext, ld_gext=_ld(grad_ext))
    E, R = spec.nnz, spec.n_rows
    _launch("gat_dst_grad", 1 + (spec.n_mid > 0) + (spec.n_small > 0) + (spec.n_heavy > 0),
            8 * R + 4 * heads * (E + 2 * R), heads * E,
            lambda: _lib.check(_lib.lib().grd_gat_dst_grad(ctypes.byref(a), stream_ptr()),
                               "gat_dst_grad"))


def gat_build_wext(w, att, d_in, heads, dh, dhp, wext) -> None:
    _launch("gat_params", 1, 0, 0, lambda: _lib.check(_lib.lib().grd_gat_build_wext(
        _p(w), _ld(w), _p(att), int(d_in), int(heads), int(dh), int(dhp), _p(wext), _ld(wext),
        stream_ptr()), "gat_build_wext"))


def gat_param_grads(dwext, w, att, d_in, heads, dh, dhp, dw, datt, lr) -> None:
    _launch("gat_params", 3, 0, 0, lambda: _lib.check(_lib.lib().grd_gat_param_grads(
        _p(dwext), _ld(dwext), _p(w), _ld(w), _p(att), int(d_in), int(heads), int(dh), int(dhp),
        _p(dw), _p(datt), float(lr), stream_ptr()), "gat_param_grads"))


def head_mean(o, n_rows, heads, dh, dhp, out, backward=False) -> None:
    _launch("head_mean", 1, 4 * n_rows * heads * dhp * 2, n_rows * heads * dhp,
            lambda: _lib.check(_lib.lib().grd_head_mean(
                _p(o), _ld(o), int(n_rows), int(heads), int(dh), int(dhp), _p(out), _ld(out),
                int(bool(backward)), stream_ptr()), "head_mean"))
