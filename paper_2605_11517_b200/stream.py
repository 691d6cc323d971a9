"""Layer-streaming engine: the partition-wise GCN epoch for graphs whose
layers do not all fit in HBM (BASELINE configs[3], ogbn-papers100M-shaped:
134 M vertices x 128 features = 68.7 GB per fp32 layer, against 180 GB of
HBM per B200).

The HBM-resident engine (engine.LayerwiseEngine) keeps every layer, its
gradient and three scratch layers in HBM.  Here HBM holds only what the
aggregation must gather at random — the whole graph (one CSR when the graph
is symmetric) and TWO whole-height layer buffers — and everything that is
only ever read or written row-sequentially streams through HBM in row
chunks:

* the features X stay in the host tier (the dataset's own fp32 array,
  page-locked in place) and are streamed H2D in row chunks on a copy stream,
  double-buffered against the chunk GEMMs, wherever a layer needs them
  (forward transform, the layer-1 regather, the layer-0 weight gradient);
* the hidden layer A_1 is *regathered* in backward — recomputed from the
  streamed X as act(A_hat (X W_0)) chunk by chunk — instead of being kept
  (the reference's regather-based backward, training.py:113-114, applied
  to the one layer that does not fit); deeper hidden layers (L > 3) go to
  pinned host memory at forward time and stream back;
* the last layer, the loss and the last layer's backward are ONE chunked
  pass (aggregate, transform, softmax-CE, weight gradient, input gradient),
  so the logits and their gradient are never materialised whole.

The association per layer is the LayerwiseEngine's (transform-first when
d_out <= d_in: aggregation at the narrow width and no forward recompute);
every kernel is the same sm_100a kernel with the same epilogue fusions, so
results equal the resident engine's up to fp32 summation order (split-K
chunks of the weight gradients).  Chunks are contiguous vertex ranges;
aggregation over a chunk is a view of the whole CSR (row-pointer slice,
shared edge array, global self rows), so nothing is copied per chunk.

GraphSAGE-mean layers (configs[4]: IGB-shaped, 1024 features) stream the
same way with the pair Y = X [W_root | W_nbr] in the layer buffer:
out = act(Y_root + mean_in(Y_nbr)) (the root add fused into the
aggregation epilogue), and in backward the gradient buffer holds
[gp | mean_in^T gp] so the weight gradient and the input gradient are one
GEMM each per chunk (engine.LayerwiseEngine._forward_sage/_backward_sage).

GAT layers (configs[2]'s model) stream with four layer-height buffers —
[P | s | t] of the layer at hand, the layer input / upstream gradient, the
last layer's per-head aggregate then every layer's d[P | s | t], and a
regathered hidden input — plus the attention and its gradient per edge:
the forward transform streams the features, the loss runs per chunk, each
layer's backward is the fused pull backward (engine.LayerwiseEngine), and
hidden layers regather their input (layer 1 from the streamed features
through layer 0, deeper layers from pinned host memory) and recompute
their attention.

Supported: GCN layers (mean_self_loop / symmetric_norm) without row
normalisation or dropout, L >= 2, hidden layers transform-first
(d_{l+1} <= d_l for l < L-1); the last layer either way.  GraphSAGE-mean:
every layer transform-first (the last one included).  GAT: any L >= 2 (one
device).
"""

from __future__ import annotations

import os
import weakref

import numpy as np
import torch

from . import _lib, ops
from .engine import _degree_scale, _LayerCfg, _Weights
from .ops import HEAVY_THRESHOLD, SEGMENT_EDGES, AggSpec, ld_of
from .tiers import FileRows, HostRows, file_backing

__all__ = ["StreamGraph", "StreamingEngine", "streaming_supported", "register_host"]


def streaming_supported(model) -> str | None:
    """None if the streaming engine can train ``model``, else the reason."""
    if model.kind not in ("gcn", "sage", "gat"):
        return "the streaming engine trains GCN, GraphSAGE-mean and GAT layers"
    if model.row_normalize or model.dropout_rate:
        return "the streaming engine trains without row normalisation / dropout"
    dims = model.dims
    L = len(dims) - 1
    if L < 2:
        return "the streaming engine needs at least two layers"
    if model.kind == "gat":
        return None                 # every layer transforms first ([P | s | t] = A W_ext)
    last = L if model.kind == "sage" else L - 1
    if any(dims[l + 1] > dims[l] for l in range(last)):
        return ("GraphSAGE layers must all be transform-first (d_out <= d_in)"
                if model.kind == "sage" else "hidden layers must be transform-first (d_out <= d_in)")
    return None


_REGISTERED: dict[int, int] = {}


def _unregister(ptr: int) -> None:
    if _REGISTERED.pop(ptr, None) is not None:
        torch._C._cudart.cudaHostUnregister(ptr)


def register_host(t: torch.Tensor, owner=None) -> torch.Tensor:
    """Page-lock a CPU tensor's memory in place (cudaHostRegister), so chunk
    copies from it are true async DMA without a staging copy.  The
    registration is dropped when ``owner`` (the numpy array that owns the
    memory) is collected, before its memory is freed."""
    ptr, nbytes = t.data_ptr(), t.numel() * t.element_size()
    if ptr in _REGISTERED and _REGISTERED[ptr] >= nbytes:
        return t
    if t.is_pinned():
        return t
    if owner is None:
        raise ValueError("register_host needs the owner of the memory")
    rc = torch._C._cudart.cudaHostRegister(ptr, nbytes, 0)
    if int(rc) != 0:
        raise RuntimeError(f"cudaHostRegister of {nbytes} bytes failed ({int(rc)})")
    _REGISTERED[ptr] = nbytes
    weakref.finalize(owner, _unregister, ptr)
    return t


def _chunk_ranges(n: int, rows: int) -> list[tuple[int, int]]:
    return [(r0, min(r0 + rows, n)) for r0 in range(0, n, rows)]


def _chunk_spec(parent: AggSpec, host_ptr: np.ndarray, r0: int, r1: int,
                self_ids: torch.Tensor) -> AggSpec:
    """Rows [r0, r1) of ``parent`` as a spec of their own: a view of the
    parent's row pointers and edges, output rows 0..r1-r0, self rows (and
    thus sources) global, heavy rows re-segmented locally."""
    sub = host_ptr[r0:r1 + 1]
    deg = np.diff(sub)
    heavy = np.flatnonzero(deg > HEAVY_THRESHOLD).astype(np.int32)
    nseg = (deg[heavy] + SEGMENT_EDGES - 1) // SEGMENT_EDGES
    seg_ptr = np.zeros(heavy.size + 1, dtype=np.int64)
    np.cumsum(nseg, out=seg_ptr[1:])
    seg_heavy = np.repeat(np.arange(heavy.size, dtype=np.int32), nseg)
    dev = parent.row_ptr.device
    has = heavy.size > 0
    spec = AggSpec(
        n_rows=r1 - r0, row_ptr=parent.row_ptr[r0:r1 + 1], idx=parent.idx, out_idx=None,
        self_idx=self_ids[r0:r1],
        heavy_rows=torch.from_numpy(heavy).to(dev) if has else None,
        heavy_seg_ptr=torch.from_numpy(seg_ptr).to(dev) if has else None,
        seg_heavy=torch.from_numpy(seg_heavy).to(dev) if has else None,
        heavy_counter=torch.zeros(16 * max(heavy.size, 1), dtype=torch.int32, device=dev)
        if has else None,
        n_heavy=int(heavy.size), n_segs=int(seg_heavy.size), nnz=int(sub[-1] - sub[0]))
    spec._partial = parent._partial      # same stream, sequential: one scratch
    return spec


def _pull_perm(sg) -> torch.Tensor:
    """For every edge of the out-CSR (the GAT pull: row u, neighbour v) its
    position in the forward in-CSR (row v, neighbour u), plus one padding
    element — device sorts of the (source, target) keys (setup only)."""
    dev = sg.device
    V = sg.num_vertices

    def keys(spec, row_is_source: bool):
        ptr = spec.row_ptr
        rows = torch.repeat_interleave(torch.arange(spec.n_rows, device=dev, dtype=torch.int64),
                                       ptr[1:] - ptr[:-1])
        cols = spec.idx[: spec.nnz].to(torch.int64)
        return rows * V + cols if row_is_source else cols * V + rows

    k_in = keys(sg.fwd, False)            # (source, target) of every forward edge
    order = torch.argsort(k_in)
    k_sorted = k_in[order]
    del k_in
    k_out = keys(sg.bwd, True)
    pos = order[torch.searchsorted(k_sorted, k_out)]
    if not torch.equal(k_sorted[torch.searchsorted(k_sorted, k_out)], k_out):
        raise RuntimeError("the out-CSR and the in-CSR hold different edges")
    return torch.cat([pos.to(torch.int32), torch.zeros(1, dtype=torch.int32, device=dev)])


class StreamGraph:
    """The graph on the device for the streaming engine, in vertex order:
    forward in-CSR (the transpose of the graph's CSR, sources ascending),
    the out-CSR for the transposed pull (the same arrays when the graph is
    symmetric), per-chunk views of both, and degree scales."""

    def __init__(self, graph, device, chunk_rows: int, max_width: int, threads: int = 0):
        n, m = graph.num_vertices, graph.num_edges
        L = _lib.lib()
        src_ptr = np.ascontiguousarray(graph.src_ptr, dtype=np.int64)
        dst_idx = np.ascontiguousarray(graph.dst_idx, dtype=np.int32)
        t_ptr = np.empty(n + 1, dtype=np.int64)
        t_idx = np.empty(max(m, 1), dtype=np.int32)
        _lib.check(L.grd_csr_transpose(n, _lib.ptr(src_ptr), _lib.ptr(dst_idx), n, _lib.ptr(t_ptr),
                                       _lib.ptr(t_idx)), "csr_transpose")
        t_idx = t_idx[:m]
        eq = np.zeros(1, dtype=np.int32)
        _lib.check(L.grd_csr_same_rows(n, _lib.ptr(src_ptr), _lib.ptr(dst_idx), _lib.ptr(t_ptr),
                                       _lib.ptr(t_idx), int(threads), _lib.ptr(eq)), "csr_same_rows")
        self.symmetric = bool(eq[0])
        self.device = device
        self.num_vertices, self.num_edges = n, m
        self.fwd = AggSpec.build(t_ptr, t_idx, device)
        self.fwd.partial(max_width)
        if self.symmetric:
            self.bwd, bwd_ptr = self.fwd, t_ptr
        else:
            self.bwd, bwd_ptr = AggSpec.build(src_ptr, dst_idx, device), src_ptr
            self.bwd.partial(max_width)
        del t_idx
        self.self_ids = torch.arange(n, dtype=torch.int32, device=device)
        self.chunks = _chunk_ranges(n, int(chunk_rows))
        self.fwd_chunks = [_chunk_spec(self.fwd, t_ptr, r0, r1, self.self_ids) for r0, r1 in self.chunks]
        self.bwd_chunks = self.fwd_chunks if self.symmetric else \
            [_chunk_spec(self.bwd, bwd_ptr, r0, r1, self.self_ids) for r0, r1 in self.chunks]
        self._deg = np.diff(t_ptr).astype(np.float64)
        self._scales: dict[str, torch.Tensor] = {}
        self.n_rows = self.n_local = n      # rows computed / buffer rows
        self.comm = None

    def exchange(self, buf: torch.Tensor, width: int) -> None:
        """One device holds every row: nothing to exchange."""

    def gat_pull(self):
        """(pull spec, its edges' positions in the forward CSR) of GAT's
        transposed pull: the in-CSR's transpose."""
        if getattr(self, "_gat_pull", None) is None:
            self._gat_pull = (self.bwd, _pull_perm(self))
        return self._gat_pull

    def reverse_add(self, buf: torch.Tensor, width: int) -> None:
        """One device: no halo partial sums to return."""

    def scale(self, name: str | None) -> torch.Tensor | None:
        if name is None:
            return None
        t = self._scales.get(name)
        if t is None:
            t = torch.from_numpy(_degree_scale(name, self._deg).astype(np.float32)).to(self.device)
            self._scales[name] = t
        return t


class ShardStreamGraph:
    """One rank's shard for the streaming engine (distributed.py): rows the
    rank computes are its owned vertices, the layer buffers hold
    [owned | halo] rows (engine.ShardDeviceGraph's layout), and every
    aggregation is preceded by one halo exchange of its input (NCCL
    all-to-all, received in place into the halo block).  Chunks run over
    the owned rows; features are needed for owned rows only — the first
    layer's halo rows travel as P0 = X W0."""

    def __init__(self, graph, plan, shard, comm, device, chunk_rows: int, max_width: int):
        from .engine import ShardDeviceGraph
        dg = ShardDeviceGraph(graph, plan, shard, comm, device)
        self.dg, self.comm, self.device, self.shard = dg, comm, device, shard
        self.num_vertices = plan.num_vertices
        self.num_edges = int(shard.in_ptr[-1])
        self.n_rows, self.n_local = shard.n_own, shard.n_local
        self.symmetric = False
        self.fwd, self.bwd = dg.fwd, dg.bwd
        self.fwd.partial(max_width)
        self.bwd.partial(max_width)
        self.self_ids = torch.arange(max(self.n_local, 1), dtype=torch.int32, device=device)
        self.chunks = _chunk_ranges(self.n_rows, int(chunk_rows))
        in_ptr = np.ascontiguousarray(shard.in_ptr, dtype=np.int64)
        out_ptr = np.ascontiguousarray(shard.out_ptr, dtype=np.int64)
        self.fwd_chunks = [_chunk_spec(self.fwd, in_ptr, r0, r1, self.self_ids) for r0, r1 in self.chunks]
        self.bwd_chunks = [_chunk_spec(self.bwd, out_ptr, r0, r1, self.self_ids)
                           for r0, r1 in self.chunks]

    def exchange(self, buf: torch.Tensor, width: int) -> None:
        self.dg.exchange(buf, width)

    def gat_pull(self):
        """GAT's transposed pull over the local in-CSR's transpose (every
        local source row, owned targets only; engine.ShardDeviceGraph)."""
        return self.dg.gat_pull()

    def reverse_add(self, buf: torch.Tensor, width: int) -> None:
        """Halo rows' partial sums back to their owners (engine.ShardDeviceGraph)."""
        self.dg.reverse_add(buf, width)

    def scale(self, name: str | None) -> torch.Tensor | None:
        return self.dg.scale(name)


def _rows(t: torch.Tensor | None, r0: int, r1: int) -> torch.Tensor | None:
    return None if t is None else t[r0:r1]


class StreamingEngine:
    """One GCN epoch with host-resident features (module docstring)."""

    def __init__(self, sg: StreamGraph, model, features, labels: np.ndarray,
                 train_mask: np.ndarray, x_cache_bytes: int | None = None,
                 mask_count: int | None = None):
        why = streaming_supported(model)
        if why is not None:
            raise NotImplementedError(why)
        dev = sg.device
        self.sg, self.device, self.model = sg, dev, model
        self.dims = model.dims
        self.L = model.num_layers
        self.V = sg.n_rows          # rows this engine computes (owned rows when sharded)
        self.NL = sg.n_local        # rows of the layer buffers (owned + halo when sharded)
        self.comm = sg.comm
        if self.comm is not None and self.L > 3:
            raise NotImplementedError("the sharded streaming engine trains models of <= 3 layers")
        self.mode = model.aggregation_mode
        self.cfg = [_LayerCfg(l, self.dims, self.mode, False, l == self.L - 1, model.heads)
                    for l in range(self.L)]
        self.wts = _Weights(model, dev)
        F = self.dims[0]
        self.labels = torch.from_numpy(np.asarray(labels, dtype=np.int32)).to(dev)
        self.mask = torch.from_numpy(np.asarray(train_mask, dtype=np.uint8)).to(dev)
        # sharded: the global count (each rank holds its owned rows' mask)
        self.mask_count = int(np.count_nonzero(train_mask)) if mask_count is None else int(mask_count)
        if self.mask_count == 0:
            raise ValueError("loss mask selects no vertices")
        last = self.cfg[-1]
        self.sage = model.kind == "sage"
        hid = max(ld_of(d) for d in self.dims[1:self.L])
        width = max(hid, last.ld_out if last.transform_first else 0)
        if self.sage:
            # layer buffers hold the pair Y = [Y_root | Y_nbr] in forward and
            # [gp | mean^T gp] in backward: twice a layer's output width
            width = max([hid] + [2 * c.ld_out for c in self.cfg])
        self.gat = model.kind == "gat"
        if self.gat:
            self._gat_buffers(sg, model, hid)
            width = self.ext_w
        # two whole-height layer buffers (zeroed once: pad columns stay 0)
        self.buf = [ops.zeros_rows(self.NL, width, dev),
                    ops.zeros_rows(self.NL, hid if self.gat else width, dev)]
        # transform-first last layer: its scaled logit gradient G' is pulled
        # whole, so it needs a third (narrow) buffer; GraphSAGE keeps
        # [G | mean^T G] there
        gw = 2 * last.ld_out if self.sage else last.d_out
        self.gbuf = ops.zeros_rows(self.NL, gw, dev) if (last.transform_first and not self.gat) else None
        # deeper hidden layers (l >= 2) kept in pinned host memory
        hw = hid if (self.sage or self.gat) else width
        self.host_acts = {l: torch.zeros((self.V, hw), dtype=torch.float32, pin_memory=True)
                          for l in range(2, self.L - 1)}
        cr = max(r1 - r0 for r0, r1 in sg.chunks)
        self.chunk_rows = cr
        maxw = max(ld_of(d) for d in self.dims)
        # streamed host rows (features, or a deeper hidden layer kept on the host)
        xw = max([ld_of(F)] + [t.shape[1] for t in self.host_acts.values()])
        # GCN whose feature rows fit a layer buffer row: every feature pass
        # lands in a layer buffer (epoch()), so the two chunk buffers of
        # streamed rows are never used — their HBM goes to the feature cache
        self.stash_on = (os.environ.get("GRD_STREAM_STASH", "1") != "0"
                         and all(ld_of(d) == d for d in self.dims[1:]))
        self.x_in_buf = (self.stash_on and not (self.sage or self.gat) and not self.host_acts
                         and self.buf[0].shape[1] == ld_of(F) == self.buf[1].shape[1])
        self._xc_elems = cr * xw
        self.xc = None if self.x_in_buf else \
            [torch.zeros(cr * xw, dtype=torch.float32, device=dev) for _ in range(2)]
        self.ac = ops.zeros_rows(cr, maxw, dev)                       # regathered hidden rows
        self.nc = ops.zeros_rows(cr, maxw, dev)                       # aggregate / pull rows
        self.lc = ops.zeros_rows(cr, last.d_out, dev)                 # logits
        self.gc = ops.zeros_rows(cr, last.d_out, dev)                 # logit gradient
        # input-gradient rows: not needed when every GCN input gradient is
        # written in place over its H rows (_gemm_rowwise)
        need_dc = self.sage or self.gat or not all(self._gemm_rowwise(self.cfg[l])
                                                  for l in range(1, self.L))
        self.dc = ops.zeros_rows(cr, maxw, dev) if need_dc else None
        self.copy_stream = torch.cuda.Stream(dev)
        self._ready = [torch.cuda.Event() for _ in range(2)]
        self._free = [torch.cuda.Event() for _ in range(2)]
        self.n_chunks = len(sg.chunks)
        self.stats_all = torch.zeros((self.n_chunks, 4), dtype=torch.float64, device=dev)
        self.stats = torch.zeros(4, dtype=torch.float64, device=dev)
        self.partials = ops.loss_partials(cr, dev)
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        # HBM cache of the leading feature rows (X never changes within a
        # call): whatever HBM is left after the working set, in whole chunks
        self._cache_ready = torch.cuda.Event()
        row_bytes = 4 * ld_of(F)
        if x_cache_bytes is None:
            # blocks torch's caching allocator holds but does not use (e.g.
            # left by the GPU plan builder) are available to the cache too
            free, _ = torch.cuda.mem_get_info(dev)
            free += torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
            # margin for the lazily allocated scratch (heavy-row partials,
            # GEMM / weight-gradient workspaces): GRD_STREAM_MARGIN_GB
            margin = float(os.environ.get("GRD_STREAM_MARGIN_GB", "1.5"))
            x_cache_bytes = max(0, free - int(margin * 2**30))
        rows = min(self.V, int(x_cache_bytes) // row_bytes)
        rows = max([r1 for _, r1 in sg.chunks if r1 <= rows], default=0)
        self.cache_rows = rows
        self.x_cache = torch.empty((rows, ld_of(F)), dtype=torch.float32, device=dev) if rows else None
        self.set_features(features)

    # ------------------------------------------------------------ helpers --
    def _scale(self, c) -> torch.Tensor | None:
        return self.sg.scale("s") if c.sym else None

    def _pre_scale(self, l: int) -> torch.Tensor | None:
        """Scale the producer of dA_{l+1} applies for a transform-first
        consumer layer l (LayerwiseEngine._consumer_epilogue)."""
        c = self.cfg[l]
        return self.sg.scale(c.pre_scale) if c.transform_first else None

    def _combine(self, sym: bool, consumer_scale):
        if consumer_scale is None:
            return self.sg.scale("s") if sym else None
        if not sym:
            return consumer_scale
        return self.sg.scale("inv_deg1")

    def _stream(self, src, fn, stash_to: torch.Tensor | None = None,
                stash_from: torch.Tensor | None = None) -> None:
        """For every row chunk: fn(rows, r0, r1) on the compute stream, the
        rows coming from the HBM feature cache when cached, else by H2D from
        the row source (tiers.py: host memory or the NVMe tier file) on the
        copy stream into one of two device buffers.  A buffer's copy waits
        only for that buffer's last use, so the first transfers of a pass
        overlap whatever compute precedes it.

        ``stash_to``: a free whole-height layer buffer that receives every
        row (streamed chunks land in their own rows instead of the chunk
        buffers; cached chunks are copied from the HBM cache) and keeps
        them.  ``stash_from``: such a buffer filled earlier — every row is
        read in place, no transfer.  ``fn`` may be None (fill only)."""
        if stash_from is not None:
            for r0, r1 in self.sg.chunks:
                if fn is not None:
                    fn(stash_from[r0:r1, :src.width], r0, r1)
            return
        cur = torch.cuda.current_stream(self.device)
        cs = self.copy_stream
        width = src.width
        cached = src is self.x_src and self.x_cache is not None
        fill = cached and not self.x_cache_valid
        if fill or stash_to is not None:
            cs.wait_stream(cur)            # earlier readers of the cache / stash buffer are done
        hits = self.cache_rows if cached and not fill else 0
        src.begin_pass([(r0, r1) for r0, r1 in self.sg.chunks if r1 > hits])
        try:
            nb = 0
            for r0, r1 in self._pass_order(hits):
                n = r1 - r0
                if r1 <= hits:
                    x = self.x_cache[r0:r1]
                    if stash_to is not None:
                        x = stash_to[r0:r1, :width]
                        x.copy_(self.x_cache[r0:r1])
                    if fn is not None:
                        fn(x, r0, r1)
                    continue
                to_cache = cached and r1 <= self.cache_rows
                if to_cache:                    # first pass fills the HBM cache
                    dst, ready, free = self.x_cache[r0:r1], self._cache_ready, None
                elif stash_to is not None:      # rows kept in the layer buffer
                    dst, ready, free = stash_to[r0:r1, :width], torch.cuda.Event(), None
                else:
                    if self.xc is None:         # first use outside a layer buffer
                        self.xc = [torch.zeros(self._xc_elems, dtype=torch.float32, device=self.device)
                                   for _ in range(2)]
                    b = nb & 1
                    nb += 1
                    dst = self.xc[b][: n * width].view(n, width)
                    ready, free = self._ready[b], self._free[b]
                with torch.cuda.stream(cs):
                    if free is not None:
                        cs.wait_event(free)
                    view, token = src.acquire(r0, r1)
                    dst.copy_(view, non_blocking=True)
                    ready.record(cs)
                    done = torch.cuda.Event()
                    done.record(cs)
                src.release(token, done)
                cur.wait_event(ready)
                if to_cache and stash_to is not None:
                    stash_to[r0:r1, :width].copy_(dst)
                    dst = stash_to[r0:r1, :width]
                if fn is not None:
                    fn(dst, r0, r1)
                if free is not None:
                    free.record(cur)
                self.h2d_bytes += n * width * 4
        finally:
            src.end_pass()
        if cached:
            self.x_cache_valid = True

    def _pass_order(self, hits: int) -> list:
        """Chunk order of one pass: the streamed chunks (rows >= hits) in
        order, with the HBM-cached chunks spread evenly between them, so the
        host link always has a transfer queued while cached chunks compute
        (``GRD_STREAM_INTERLEAVE=0``: cached chunks first)."""
        chunks = self.sg.chunks
        cached = [c for c in chunks if c[1] <= hits]
        streamed = [c for c in chunks if c[1] > hits]
        if not cached or not streamed or os.environ.get("GRD_STREAM_INTERLEAVE", "1") == "0":
            return cached + streamed
        out, j = [], 0
        for i, c in enumerate(streamed):
            out.append(c)
            upto = (i + 1) * len(cached) // len(streamed)
            out.extend(cached[j:upto])
            j = upto
        return out + cached[j:]

    def set_features(self, src) -> None:
        """Re-bind the feature rows (the HBM cache refills on the next pass)."""
        if src.n_rows != self.V or src.width != ld_of(self.dims[0]):
            raise ValueError("feature rows must be [V, round_up(F, 4)]")
        src.configure(self.cache_rows)
        self.x_src = src
        self.x_cache_valid = False
        self._xbuf = None

    def _to_host(self, src: torch.Tensor, host: torch.Tensor) -> None:
        """D2H of a whole layer in row chunks on the copy stream."""
        cur = torch.cuda.current_stream(self.device)
        self.copy_stream.wait_stream(cur)
        with torch.cuda.stream(self.copy_stream):
            for r0, r1 in self.sg.chunks:
                host[r0:r1].copy_(src[r0:r1, : host.shape[1]], non_blocking=True)
        cur.wait_stream(self.copy_stream)
        self.d2h_bytes += host.numel() * 4

    # -------------------------------------------------------------- epoch --
    def epoch(self, lr: float) -> None:
        if self.sage:
            self._epoch_sage(lr)
            return
        if self.gat:
            self._epoch_gat(lr)
            return
        sg, cfg, L, V = self.sg, self.cfg, self.L, self.V
        W, dW = self.wts.w, self.wts.dw
        for dw in dW:
            dw.zero_()
        B = list(self.buf)                  # B[1] holds the current layer input
        xb, self._xbuf = self._xbuf, None
        if xb is not None:
            # the last epoch's backward left every feature row in layer
            # buffer xb: P_0 goes to the other buffer, A_1 over the rows
            B = [self.buf[1] if xb is self.buf[0] else self.buf[0], xb]
        # ---- forward of the hidden (transform-first) layers ----
        for l in range(L - 1):
            c = cfg[l]
            s = self._scale(c)
            P = B[0][:, : c.ld_out]
            if l == 0:
                self._stream(self.x_src, lambda x, r0, r1: ops.gemm(
                    x, W[0], P[r0:r1], r1 - r0, c.d_out, c.d_in, row_scale=_rows(s, r0, r1)),
                    stash_from=xb,
                    # first epoch: the streamed rows land in B[1], which A_1 then overwrites
                    stash_to=B[1] if (xb is None and self.x_in_buf and self._x_fits(B[1])) else None)
            else:
                ops.gemm(B[1][:, : c.ld_in], W[l], P, V, c.d_out, c.d_in, row_scale=s)
            sg.exchange(P, c.d_out)                               # halo rows of P
            ops.agg_sum(sg.fwd, P, B[1][:, : c.ld_out], c.d_out, post_div_deg=not c.sym,
                        post_scale=s, relu=True)
            if l + 1 in self.host_acts:
                self._to_host(B[1], self.host_acts[l + 1])
        # ---- last layer + loss + last layer backward, one chunked pass ----
        self._last_layer(B)
        # ---- backward of the hidden layers: B[1] = dA_{l+1} (pre-scaled) ----
        for l in reversed(range(L - 1)):
            c = cfg[l]
            s = self._scale(c)
            D = B[1][:, : c.ld_out]
            if l == 0:
                self._backward_first(D, s, B[0])
                break
            H = B[0][:, : c.ld_out]
            sg.exchange(D, c.d_out)
            ops.agg_sum(sg.bwd, D, H, c.d_out, post_scale=s)            # H = A_hat^T D
            ref_scale = self._pre_scale(l - 1)
            if l == 1 and self._x_fits(B[1]):
                # regather A_1 = act((A_hat X) W_0) chunk by chunk from the
                # feature rows themselves, streamed into the consumed buffer
                # of D (one host pass; the rows stay there for the layer-0
                # backward and the next epoch's forward)
                c0 = cfg[0]
                s0 = self._scale(c0)
                X = B[1][:, : c0.ld_in]
                self._stream(self.x_src, None, stash_to=B[1])
                sg.exchange(X, c0.d_in)
                for (r0, r1), spec in zip(sg.chunks, sg.fwd_chunks):
                    n = r1 - r0
                    N = self.nc[:n, : c0.ld_in]
                    ops.agg_sum(spec, X, N, c0.d_in, src_scale=s0, post_div_deg=not c0.sym,
                                post_scale=_rows(s0, r0, r1))
                    a = self.ac[:n, : c.ld_in]
                    ops.gemm(N, W[0], a, n, c0.d_out, c0.d_in, relu_out=True)
                    self._hidden_grad(l, a, H, B[0], r0, r1, ref_scale)
                self._xbuf = B[1]
            elif l == 1:
                # regather A_1 = act(A_hat (X W_0)) chunk by chunk from P_0
                c0 = cfg[0]
                s0 = self._scale(c0)
                P0 = B[1][:, : c0.ld_out]
                self._stream(self.x_src, lambda x, r0, r1: ops.gemm(
                    x, W[0], P0[r0:r1], r1 - r0, c0.d_out, c0.d_in, row_scale=_rows(s0, r0, r1)))
                sg.exchange(P0, c0.d_out)
                for (r0, r1), spec in zip(sg.chunks, sg.fwd_chunks):
                    n = r1 - r0
                    a = self.ac[:n, : c.ld_in]
                    ops.agg_sum(spec, P0, a, c0.d_out, post_div_deg=not c0.sym,
                                post_scale=_rows(s0, r0, r1), relu=True)
                    self._hidden_grad(l, a, H, B[0], r0, r1, ref_scale)
            else:
                def step(a, r0, r1):
                    self._hidden_grad(l, a, H, B[0], r0, r1, ref_scale)
                self._stream(HostRows(self.host_acts[l]), step)
            B[0], B[1] = B[1], B[0]
        if self.comm is not None:      # every layer's weight gradient in one all-reduce
            self.comm.all_reduce_sum(self.wts.grad_bucket)
            self.stats.copy_(self.stats_all.sum(dim=0))
            self.comm.all_reduce_sum(self.stats)
        # ---- SGD (training.py:352-354) ----
        for w, dw in zip(W, dW):
            ops.wgrad_sgd(w, w, dw, dw.shape[0], dw.shape[1], 0, accumulate=True, w=w, lr=lr)

    def _hidden_grad(self, l: int, a: torch.Tensor, H: torch.Tensor, out: torch.Tensor, r0: int,
                     r1: int, ref_scale) -> None:
        """Rows [r0, r1) of a transform-first layer's backward given its input
        rows a: dW_l += a^T H, dA_l = relu'(a) (H W_l^T) * pre-scale(l-1),
        written over the (consumed) rows of ``out``, the buffer holding H."""
        c = self.cfg[l]
        n = r1 - r0
        Hc = H[r0:r1]
        ops.wgrad_sgd(a, Hc, self.wts.dw[l], c.d_in, c.d_out, n, accumulate=True)
        if out.data_ptr() == H.data_ptr() and self._gemm_rowwise(c):
            # dA_l rows written straight over the H rows they are computed
            # from: one N tile and no K split, so every CTA has loaded its
            # rows' whole K extent before its epilogue stores them
            ops.gemm(Hc, self.wts.w[l], out[r0:r1, : c.ld_in], n, c.d_in, c.d_out, trans_b=True,
                     row_scale=_rows(ref_scale, r0, r1), relu_ref=a)
            return
        if self.dc is None:
            self.dc = ops.zeros_rows(self.chunk_rows, max(ld_of(d) for d in self.dims), self.device)
        d = self.dc[:n, : c.ld_in]
        ops.gemm(Hc, self.wts.w[l], d, n, c.d_in, c.d_out, trans_b=True,
                 row_scale=_rows(ref_scale, r0, r1), relu_ref=a)
        # dA_l rows replace the (consumed) H rows: row copy kernel (K1, identity rows)
        ops.gather_rows(d, self.sg.self_ids[:n], out[r0:r1], c.ld_in)

    @staticmethod
    def _gemm_rowwise(c) -> bool:
        """Whether the input-gradient GEMM ``H W^T`` (n = d_in, k = d_out)
        runs as one N tile without a K split (ops.gemm / grd_gemm_tc.cu
        pick_bn), so it may overwrite its own A rows."""
        bn_max = int(os.environ.get("GRD_GEMM_BN_MAX", "256"))
        return (os.environ.get("GRD_STREAM_INPLACE", "1") != "0" and c.ld_in <= min(bn_max, 128)
                and not ops._KSPLIT_TB)

    def _x_fits(self, buf: torch.Tensor) -> bool:
        """Whether the feature rows can live in layer buffer ``buf`` (same
        row width, so every chunk is one contiguous block)."""
        return (self.stash_on and buf.shape[1] == self.x_src.width and buf.shape[0] >= self.V
                and buf.is_contiguous())

    def _backward_first(self, D: torch.Tensor, s, free: torch.Tensor) -> None:
        """Layer 0: dW_0 = X^T (A_hat^T D), chunk by chunk with X streamed.

        ``free`` is the other layer buffer, unused until the next epoch: the
        streamed feature rows are copied into its rows instead of the chunk
        buffers, so the next epoch's layer-0 transform reads them from HBM
        instead of over the host link again (GRD_STREAM_STASH=0: off)."""
        c = self.cfg[0]
        stash_from = stash_to = None
        if self._xbuf is free:          # the hidden layer-1 regather left X here
            stash_from = free
        elif self._x_fits(free):
            stash_to = free
        specs = self.sg.bwd_chunks

        spec_of = {r0: sp for (r0, _), sp in zip(self.sg.chunks, specs)}
        self.sg.exchange(D, c.d_out)

        def step(x, r0, r1):
            n = r1 - r0
            h = self.nc[:n, : c.ld_out]
            ops.agg_sum(spec_of[r0], D, h, c.d_out, post_scale=_rows(s, r0, r1))
            ops.wgrad_sgd(x, h, self.wts.dw[0], c.d_in, c.d_out, n, accumulate=True)
        self._stream(self.x_src, step, stash_to=stash_to, stash_from=stash_from)
        self._xbuf = free if (stash_to is not None or stash_from is not None) else None

    def _last_layer(self, B: list) -> None:
        """Forward, loss and backward of the last layer in one chunked pass;
        leaves dA_{L-1} (masked, pre-scaled for layer L-2) in B[1]."""
        sg, L = self.sg, self.L
        l = L - 1
        c = self.cfg[l]
        W, dW = self.wts.w[l], self.wts.dw[l]
        s = self._scale(c)
        A = B[1][:, : c.ld_in]
        C = c.d_out
        prev_ref_scale = self._pre_scale(l - 1)
        if not c.transform_first:
            # N = A_hat A (regathered per chunk), logits = N W; gn = (G W^T) * pre_scale
            Q = B[0][:, : c.ld_in]
            sg.exchange(A, c.d_in)
            for i, ((r0, r1), spec) in enumerate(zip(sg.chunks, sg.fwd_chunks)):
                n = r1 - r0
                N = self.nc[:n, : c.ld_in]
                ops.agg_sum(spec, A, N, c.d_in, src_scale=s, post_div_deg=not c.sym,
                            post_scale=_rows(s, r0, r1))
                lg = self.lc[:n]
                ops.gemm(N, W, lg, n, C, c.d_in)
                g = self.gc[:n]
                ops.softmax_xent(lg, n, C, self.labels[r0:r1], self.mask[r0:r1], self.mask_count,
                                 g, self.stats_all[i], self.partials)
                ops.wgrad_sgd(N, g, dW, c.d_in, C, n, accumulate=True)
                ops.gemm(g, W, Q[r0:r1], n, c.d_in, C, trans_b=True,
                         row_scale=_rows(self.sg.scale(c.pre_scale), r0, r1))
            post = self._combine(c.sym, prev_ref_scale)
            # dA_{L-1} = relu'(A) (A_hat^T Q) * post, in place over A
            sg.exchange(Q, c.d_in)
            ops.agg_sum(sg.bwd, Q, A, c.d_in, post_scale=post, mask_ref=A)
            return
        # transform-first: P = A W (whole), logits rows = act-free A_hat P
        P = B[0][:, : c.ld_out]
        ops.gemm(A, W, P, self.V, C, c.d_in, row_scale=s)
        sg.exchange(P, C)
        G = self.gbuf
        pre = self.sg.scale(c.pre_scale)
        for i, ((r0, r1), spec) in enumerate(zip(sg.chunks, sg.fwd_chunks)):
            n = r1 - r0
            lg = self.lc[:n]
            ops.agg_sum(spec, P, lg, C, post_div_deg=not c.sym, post_scale=_rows(s, r0, r1))
            ops.softmax_xent(lg, n, C, self.labels[r0:r1], self.mask[r0:r1], self.mask_count,
                             G[r0:r1], self.stats_all[i], self.partials, grad_scale=pre[r0:r1])
        H = B[0][:, : c.ld_out]
        sg.exchange(G, C)
        ops.agg_sum(sg.bwd, G, H, C, post_scale=s)                  # H = A_hat^T G'
        for r0, r1 in sg.chunks:
            self._hidden_grad(l, A[r0:r1], H, B[0], r0, r1, prev_ref_scale)
        B[0], B[1] = B[1], B[0]   # dA_{L-1} now in the buffer that held H

    # ------------------------------------------------- GraphSAGE-mean --
    # Buffer roles for the whole epoch: B1 holds layer inputs A_l (forward)
    # and the regathered pair Y_0 (backward); B0 holds the pair Y_l in
    # forward and [gp_l | mean^T gp_l] in backward.
    def _sage_layer_out(self, spec, Y: torch.Tensor, out: torch.Tensor, c, r0: int | None = None,
                        r1: int | None = None, relu: bool = True) -> None:
        """out = act(Y_root + mean_in(Y_nbr)) over the rows of ``spec``
        (all rows, or the chunk [r0, r1) with chunk-local output rows).  The
        caller has filled Y_nbr's halo rows (sharded: _sage_halo)."""
        lo = c.ld_out
        root = Y[:, :lo] if r0 is None else Y[r0:r1, :lo]
        ops.agg_sum(spec, Y[:, lo: 2 * lo], out, c.d_out, post_div_deg=2, no_self=True,
                    add_y=root, relu=relu)

    def _sage_halo(self, Y: torch.Tensor, c) -> None:
        """Halo rows of the neighbour half Y_nbr (sharded; one device: no-op)."""
        lo = c.ld_out
        self.sg.exchange(Y[:, lo: 2 * lo], c.d_out)

    def _sage_pull(self, G: torch.Tensor, c) -> None:
        """G[:, lo:2lo] = mean_in^T G[:, :lo] (pull over out-edges, 1/deg_v;
        sharded: gp's halo rows first, the graph is symmetric)."""
        lo = c.ld_out
        self.sg.exchange(G[:, :lo], c.d_out)
        ops.agg_sum(self.sg.bwd, G[:, :lo], G[:, lo: 2 * lo], c.d_out,
                    src_scale=self.sg.scale("inv_deg"), no_self=True)

    def _sage_grad(self, l: int, a: torch.Tensor, G: torch.Tensor, r0: int, r1: int) -> None:
        """Rows [r0, r1) of layer l's backward given its input rows a:
        dW_l += a^T [gp | H]; dA_l = relu'(a) ([gp | H] [W_root | W_nbr]^T),
        written over the (consumed) rows of B0 (layer-wise _backward_sage)."""
        c = self.cfg[l]
        n = r1 - r0
        gc = G[r0:r1, : 2 * c.ld_out]
        ops.wgrad_sgd(a, gc, self.wts.dw[l], c.d_in, 2 * c.ld_out, n, accumulate=True)
        if l > 0:
            d = self.dc[:n, : c.ld_in]
            ops.gemm(gc, self.wts.w[l], d, n, c.d_in, 2 * c.ld_out, trans_b=True, relu_ref=a)
            ops.gather_rows(d, self.sg.self_ids[:n], self.buf[0][r0:r1], c.ld_in)

    def _epoch_sage(self, lr: float) -> None:
        sg, cfg, L, V = self.sg, self.cfg, self.L, self.V
        W, dW = self.wts.w, self.wts.dw
        for dw in dW:
            dw.zero_()
        B0, B1 = self.buf
        # ---- forward of the hidden layers: Y_l -> B0, A_{l+1} -> B1 ----
        for l in range(L - 1):
            c = cfg[l]
            Y = B0[:, : 2 * c.ld_out]
            if l == 0:
                self._stream(self.x_src, lambda x, r0, r1: ops.gemm(
                    x, W[0], Y[r0:r1], r1 - r0, 2 * c.ld_out, c.d_in))
            else:
                ops.gemm(B1[:, : c.ld_in], W[l], Y, V, 2 * c.ld_out, c.d_in)
            self._sage_halo(Y, c)
            self._sage_layer_out(sg.fwd, Y, B1[:, : c.ld_out], c)
            if l + 1 in self.host_acts:
                self._to_host(B1, self.host_acts[l + 1])
        # ---- last layer, loss and its backward in one chunked pass ----
        l = L - 1
        c = cfg[l]
        A = B1[:, : c.ld_in]
        Y = B0[:, : 2 * c.ld_out]
        ops.gemm(A, W[l], Y, V, 2 * c.ld_out, c.d_in)
        self._sage_halo(Y, c)
        G = self.gbuf
        C = c.d_out
        for i, ((r0, r1), spec) in enumerate(zip(sg.chunks, sg.fwd_chunks)):
            n = r1 - r0
            lg = self.lc[:n]
            self._sage_layer_out(spec, Y, lg, c, r0, r1, relu=False)
            ops.softmax_xent(lg, n, C, self.labels[r0:r1], self.mask[r0:r1], self.mask_count,
                             G[r0:r1, : c.ld_out], self.stats_all[i], self.partials)
        self._sage_pull(G, c)
        for r0, r1 in sg.chunks:
            self._sage_grad(l, A[r0:r1], G, r0, r1)
        # ---- hidden layers: gp_l in B0[:, :lo] ----
        for l in reversed(range(L - 1)):
            c = cfg[l]
            self._sage_pull(B0, c)
            if l == 0:
                self._stream(self.x_src, lambda x, r0, r1: ops.wgrad_sgd(
                    x, B0[r0:r1, : 2 * c.ld_out], dW[0], c.d_in, 2 * c.ld_out, r1 - r0,
                    accumulate=True))
            elif l == 1:
                # regather A_1 = relu(Y0_root + mean(Y0_nbr)) chunk by chunk
                c0 = cfg[0]
                Y0 = B1[:, : 2 * c0.ld_out]
                self._stream(self.x_src, lambda x, r0, r1: ops.gemm(
                    x, W[0], Y0[r0:r1], r1 - r0, 2 * c0.ld_out, c0.d_in))
                self._sage_halo(Y0, c0)
                for (r0, r1), spec in zip(sg.chunks, sg.fwd_chunks):
                    a = self.ac[: r1 - r0, : c.ld_in]
                    self._sage_layer_out(spec, Y0, a, c0, r0, r1)
                    self._sage_grad(l, a, B0, r0, r1)
            else:
                self._stream(HostRows(self.host_acts[l]),
                             lambda a, r0, r1, _l=l: self._sage_grad(_l, a, B0, r0, r1))
        if self.comm is not None:      # every layer's weight gradient in one all-reduce
            self.comm.all_reduce_sum(self.wts.grad_bucket)
            self.stats.copy_(self.stats_all.sum(dim=0))
            self.comm.all_reduce_sum(self.stats)
        # ---- SGD (training.py:352-354) ----
        for w, dw in zip(W, dW):
            ops.wgrad_sgd(w, w, dw, dw.shape[0], dw.shape[1], 0, accumulate=True, w=w, lr=lr)

    # ------------------------------------------------------------------ GAT --
    # Buffers: B0 [P | s | t] of the layer at hand; B1 the layer input A_l in
    # forward and the upstream gradient gO in backward; B2 the last layer's
    # per-head aggregate O, then every layer's dL/d[P | s | t]; B3 the last
    # layer's gO, then the regathered input A_l of a hidden layer.  Per edge:
    # attention and score gradients (E x heads each).  The backward of a
    # hidden layer regathers A_l (layer 1: from the streamed features, layer
    # 0's transform, softmax and aggregation; deeper: from pinned host
    # memory) and recomputes its [P | s | t] and attention — the
    # reference's regather, applied to the layer that does not fit.
    def _gat_buffers(self, sg, model, hid: int) -> None:
        dev = self.device
        H = model.heads
        cl = self.cfg[-1]
        self.ext_w = max(c.ld_ext for c in self.cfg)
        E = sg.fwd.nnz
        self.gbuf2 = ops.zeros_rows(self.NL, max(self.ext_w, cl.hdp), dev)
        self.gbuf3 = ops.zeros_rows(self.NL, max(hid, cl.hdp), dev)
        self.alpha = torch.zeros(max(E * H, 1), dtype=torch.float32, device=dev)
        self.delta = torch.zeros_like(self.alpha)
        self.alpha_self = torch.zeros(max(self.NL * H, 1), dtype=torch.float32, device=dev)
        self.delta_self = torch.zeros_like(self.alpha_self)
        self.cdot = torch.zeros_like(self.alpha_self)
        self.st = ops.zeros_rows(self.NL, 2 * H, dev)
        self.pull, self.edge_perm = sg.gat_pull()

    def _gat_transform(self, l: int, src, P: torch.Tensor) -> None:
        """[P | s | t] = A_l W_ext -> P (src: a device matrix, or the streamed
        feature rows for layer 0), then the edge softmax of layer l."""
        c, wt = self.cfg[l], self.wts
        d_in, dh, dhp = wt.shape[l]
        ops.gat_build_wext(wt.w[l], wt.att[l], d_in, c.heads, dh, dhp, wt.wext[l])
        if isinstance(src, torch.Tensor):
            ops.gemm(src[:, : c.ld_in], wt.wext[l], P, self.V, c.n_ext, c.d_in)
        else:
            self._stream(src, lambda x, r0, r1: ops.gemm(x, wt.wext[l], P[r0:r1], r1 - r0, c.n_ext,
                                                         c.d_in))
        self.sg.exchange(P, c.n_ext)                      # halo rows of [P | s | t]
        ops.gat_pack_scores(P, self.NL, c.heads, c.dhp, self.st)
        ops.gat_softmax(self.sg.fwd, P, c.heads, c.dhp, self.alpha, self.alpha_self, st=self.st)

    def _gat_aggregate(self, l: int, P: torch.Tensor, out: torch.Tensor) -> None:
        c = self.cfg[l]
        ops.agg_sum(self.sg.fwd, P[:, : c.hdp], out, c.hdp, edge_w=self.alpha, self_w=self.alpha_self,
                    heads=c.heads, head_ld=c.dhp, relu=not c.last)

    def _gat_backward(self, l: int, P: torch.Tensor, gO: torch.Tensor, G: torch.Tensor) -> None:
        """dL/d[P | s | t] of layer l into G (engine.LayerwiseEngine's fused
        pull backward; c = gO . O is in self.cdot)."""
        c = self.cfg[l]
        if self.NL > self.V:
            # sharded: halo rows carry no gradient of their own (no self term);
            # their rows of G collect partial sums for their owners
            gO[self.V:].zero_()
            self.cdot[self.V * c.heads:].zero_()
        ops.gat_pull_bwd(self.pull, P, c.heads, c.dhp, self.edge_perm, self.alpha,
                         self.alpha_self, gO, self.cdot, self.delta, self.delta_self, G, st=self.st)
        ops.gat_dst_grad(self.sg.fwd, c.heads, c.dhp, self.delta, self.delta_self, G)
        self.sg.reverse_add(G, c.hdp + c.heads)

    def _gat_input_grad(self, l: int, G: torch.Tensor, A: torch.Tensor, out: torch.Tensor) -> None:
        """Per chunk: gO_{l-1} = relu'(A_l) (G W_ext^T) and c_{l-1} = gO . A_l
        (A_l = relu(O_{l-1}), the lower layer's output), written to ``out``
        (which may be A's own buffer: each chunk is read before it is
        overwritten)."""
        c = self.cfg[l]
        cp = self.cfg[l - 1]
        for r0, r1 in self.sg.chunks:
            n = r1 - r0
            d = self.dc[:n, : c.ld_in]
            ops.gemm(G[r0:r1, : c.ld_ext], self.wts.wext[l], d, n, c.d_in, c.n_ext, trans_b=True,
                     relu_ref=A[r0:r1])
            ops.gat_row_dots(d, A[r0:r1], n, cp.heads, cp.dhp, self.cdot[r0 * cp.heads:])
            ops.gather_rows(d, self.sg.self_ids[:n], out[r0:r1], c.ld_in)

    def _epoch_gat(self, lr: float) -> None:
        cfg, L, V = self.cfg, self.L, self.V
        wt = self.wts
        for dw in wt.dwext:
            dw.zero_()
        B0, B1 = self.buf
        B2, B3 = self.gbuf2, self.gbuf3
        # ---- forward ----
        for l in range(L - 1):
            c = cfg[l]
            P = B0[:, : c.ld_ext]
            self._gat_transform(l, self.x_src if l == 0 else B1, P)
            self._gat_aggregate(l, P, B1[:, : c.hdp])            # A_{l+1} over A_l
            if l + 1 in self.host_acts:
                self._to_host(B1, self.host_acts[l + 1])
        l = L - 1
        c = cfg[l]
        P = B0[:, : c.ld_ext]
        self._gat_transform(l, self.x_src if l == 0 else B1, P)
        O = B2[:, : c.hdp]
        self._gat_aggregate(l, P, O)
        # loss per chunk: logits = mean over heads, gO = dL/dlogits / heads
        C = c.d_out
        for i, (r0, r1) in enumerate(self.sg.chunks):
            n = r1 - r0
            lg = self.lc[:n]
            ops.head_mean(O[r0:r1], n, c.heads, c.dh, c.dhp, lg)
            g = self.gc[:n]
            ops.softmax_xent(lg, n, C, self.labels[r0:r1], self.mask[r0:r1], self.mask_count, g,
                             self.stats_all[i], self.partials)
            ops.head_mean(g, n, c.heads, c.dh, c.dhp, B3[r0:r1, : c.hdp], backward=True)
        ops.gat_row_dots(B3[:, : c.hdp], O, V, c.heads, c.dhp, self.cdot)
        # ---- backward of the last layer: its [P | s | t], attention, input in place ----
        G = B2[:, : c.ld_ext]
        self._gat_backward(l, P, B3[:, : c.hdp], G)
        if l == 0:
            self._stream(self.x_src, lambda x, r0, r1: ops.wgrad_sgd(
                x, G[r0:r1], wt.dwext[0], c.d_in, c.n_ext, r1 - r0, accumulate=True))
        else:
            A = B1[:, : c.ld_in]
            ops.wgrad_sgd(A, G, wt.dwext[l], c.d_in, c.n_ext, V)
            self._gat_input_grad(l, G, A, B1)                       # gO_{L-2} over A_{L-1}
        # ---- hidden layers: gO_l in B1 ----
        for l in reversed(range(L - 1)):
            c = cfg[l]
            P = B0[:, : c.ld_ext]
            if l == 0:
                self._gat_transform(0, self.x_src, P)
            else:
                A = B3[:, : c.ld_in]
                if l == 1:            # regather A_1 from the streamed features
                    P0 = B0[:, : cfg[0].ld_ext]
                    self._gat_transform(0, self.x_src, P0)
                    self._gat_aggregate(0, P0, A)
                else:
                    self._stream(HostRows(self.host_acts[l]),
                                 lambda a, r0, r1, _A=A: ops.gather_rows(
                                     a, self.sg.self_ids[: r1 - r0], _A[r0:r1], _A.shape[1]))
                self._gat_transform(l, A, P)
            G = B2[:, : c.ld_ext]
            self._gat_backward(l, P, B1[:, : c.hdp], G)
            if l == 0:
                self._stream(self.x_src, lambda x, r0, r1: ops.wgrad_sgd(
                    x, G[r0:r1], wt.dwext[0], c.d_in, c.n_ext, r1 - r0, accumulate=True))
            else:
                ops.wgrad_sgd(A, G, wt.dwext[l], c.d_in, c.n_ext, V)
                self._gat_input_grad(l, G, A, B1)
        if self.comm is not None:      # every layer's dW_ext in one all-reduce
            self.comm.all_reduce_sum(wt.grad_bucket)
            self.stats.copy_(self.stats_all.sum(dim=0))
            self.comm.all_reduce_sum(self.stats)
        # ---- SGD: dW, datt from dW_ext ----
        for l in range(L):
            c = cfg[l]
            d_in, dh, dhp = wt.shape[l]
            ops.gat_param_grads(wt.dwext[l], wt.w[l], wt.att[l], d_in, c.heads, dh, dhp, wt.dw[l],
                                wt.datt[l], lr)

    def read_stats(self) -> tuple[float, float]:
        """(loss, accuracy) of the last epoch: per-chunk sums added in chunk
        order on the host (float64); sharded: the ranks' sums all-reduced at
        the end of the epoch."""
        if self.comm is not None:
            st = self.stats.cpu().numpy()
            return float(st[2]) / self.mask_count, float(st[3]) / self.mask_count
        s = self.stats_all.cpu().numpy()
        loss = float(np.sum(s[:, 2])) / self.mask_count
        acc = float(np.sum(s[:, 3])) / self.mask_count
        self.stats.copy_(torch.tensor([loss, acc, s[:, 2].sum(), s[:, 3].sum()], dtype=torch.float64))
        return loss, acc


# --------------------------------------------------------------------------
# when to stream, and the session partitioned_train drives
# --------------------------------------------------------------------------
def resident_bytes(num_vertices: int, num_edges: int, model) -> int:
    """HBM the layer-wise resident engine needs (engine.LayerwiseEngine):
    forward + backward CSRs, every layer, three scratch layers of the widest
    width, heavy-row scratch, degree scales."""
    V, E = int(num_vertices), int(num_edges)
    lds = [ld_of(d) for d in model.dims]
    wide = max(lds) * (2 if model.kind == "sage" else 1)
    if model.kind == "gat":
        wide = max(wide, model.heads * max(lds) + 2 * model.heads + 4)
    graph = 2 * (8 * (V + 1) + 4 * E) + 4 * V
    layers = 4 * V * (sum(lds) + 3 * wide)
    scratch = 4 * E * max(lds) // 64 + 16 * V
    edge_state = 8 * E * model.heads if model.kind == "gat" else 0
    return graph + layers + scratch + edge_state


def streaming_bytes(num_vertices: int, num_edges: int, model, chunk_rows: int,
                    symmetric: bool = True) -> int:
    """HBM the streaming engine needs (StreamingEngine)."""
    V, E = int(num_vertices), int(num_edges)
    lds = [ld_of(d) for d in model.dims]
    width = max(lds[1:-1] + ([lds[-1]] if lds[-1] <= lds[-2] else []))
    gw = lds[-1]
    if model.kind == "sage":
        width = max([width] + [2 * x for x in lds[1:]])
        gw = 2 * lds[-1]
    graph = (1 if symmetric else 2) * (8 * (V + 1) + 4 * E) + 4 * V
    layers = 2 * 4 * V * width + (4 * V * gw if lds[-1] <= lds[-2] else 0)
    if model.kind == "gat":
        # B0 / B2 [P | s | t], B1 / B3 a layer (heads x padded head width),
        # attention + score gradients per edge and the pull's permutation
        H = model.heads
        hdp = max(H * ld_of(d // H) for d in model.dims[1:-1]) if len(model.dims) > 2 else 0
        hdp = max(hdp, H * lds[-1])
        ext = ld_of(hdp + 2 * H)
        layers = 4 * V * (2 * ext + 2 * hdp) + 8 * E * H + 4 * E + 16 * V * H
    chunks = 4 * int(chunk_rows) * (2 * max(lds) + 3 * max(lds) + 2 * lds[-1])
    return graph + layers + chunks + 4 * E * max(lds) // 64 + 16 * V


DEFAULT_CHUNK_ROWS = int(os.environ.get("GRD_CHUNK_ROWS", str(1 << 20)))


def feature_rows(dataset, chunk_rows: int = DEFAULT_CHUNK_ROWS, host_cache_bytes: int | None = None):
    """The dataset's features as a row source (tiers.py) of fp32
    [V, round_up(F, 4)] rows:

    * features memory-mapped from a GRIN feature file (``load_dataset(...,
      mmap_features=True)``) stay in that file — the NVMe tier — with a
      pinned host-cache window of ``host_cache_bytes`` (default: host memory
      available less 16 GiB; GRD_HOST_CACHE_GB overrides);
    * fp32 features with F % 4 == 0 in memory are page-locked in place;
    * anything else is converted once into a padded pinned copy."""
    feats = dataset.features
    f = feats.shape[1]
    backing = file_backing(feats) if feats.dtype == np.float32 else None
    if backing is not None and f % 4 == 0:
        src = getattr(dataset, "_file_rows", None)
        if src is None or (src.path, src.data_offset) != backing:
            if host_cache_bytes is None:
                env = os.environ.get("GRD_HOST_CACHE_GB")
                if env:
                    host_cache_bytes = int(float(env) * 2**30)
                else:
                    import psutil
                    host_cache_bytes = max(0, psutil.virtual_memory().available - (16 << 30))
            src = FileRows(backing[0], backing[1], feats.shape[0], f, chunk_rows,
                           host_cache_bytes=host_cache_bytes)
            dataset._file_rows = src
        return src
    if feats.dtype == np.float32 and feats.flags.c_contiguous and f % 4 == 0:
        root = feats
        while isinstance(root.base, np.ndarray):
            root = root.base
        return HostRows(register_host(torch.from_numpy(feats), owner=root))
    stage = getattr(dataset, "_stream_stage", None)
    if stage is None or tuple(stage.shape) != (feats.shape[0], ld_of(f)):
        stage = torch.zeros((feats.shape[0], ld_of(f)), dtype=torch.float32, pin_memory=True)
        dataset._stream_stage = stage
    np.copyto(stage.numpy()[:, :f], feats, casting="same_kind")
    return HostRows(stage)


class StreamSession:
    """Device session (training.TrainSession's interface) over the
    streaming engine: graph upload cached on the plan, features streamed
    from the host on every epoch."""

    layerwise = True

    def __init__(self, dataset, plan, model, chunk_rows: int = DEFAULT_CHUNK_ROWS,
                 x_cache_bytes: int | None = None, host_cache_bytes: int | None = None,
                 comm=None, shard=None, owned_features: torch.Tensor | None = None):
        """``comm``: this process is one rank of a sharded run (distributed.
        Communicator): the rank streams its owned rows only; ``shard`` (a
        ShardPlan, default build_shard_plan) and ``owned_features`` (page-
        locked [n_own, round_up(F, 4)] rows in the shard's owned order,
        default gathered from ``dataset.features``) let a caller that never
        materialises the whole feature matrix supply them."""
        from .model import copy_model
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.comm = comm
        maxw = max(ld_of(d) for d in model.dims)
        if comm is None:
            key = ("stream_graph", str(self.dev), int(chunk_rows))
            sg = plan.device_cache.get(key)
            if sg is None:
                sg = StreamGraph(dataset.graph, self.dev, chunk_rows, maxw)
                plan.device_cache[key] = sg
            src = feature_rows(dataset, chunk_rows, host_cache_bytes)
            labels, mask, count = dataset.labels, dataset.train_mask, None
        else:
            key = ("stream_shard", comm.rank, comm.world, str(self.dev), int(chunk_rows))
            sg = plan.device_cache.get(key)
            if sg is None:
                if shard is None:
                    from .distributed import build_shard_plan
                    shard = build_shard_plan(dataset.graph, plan, comm.rank, comm.world, comm)
                sg = ShardStreamGraph(dataset.graph, plan, shard, comm, self.dev, chunk_rows, maxw)
                plan.device_cache[key] = sg
            owned = sg.shard.owned
            if owned_features is None:
                f = dataset.features.shape[1]
                owned_features = torch.zeros((owned.size, ld_of(f)), dtype=torch.float32,
                                             pin_memory=True)
                np.copyto(owned_features.numpy()[:, :f], dataset.features[owned], casting="same_kind")
            src = HostRows(owned_features)
            labels = np.asarray(dataset.labels)[owned]
            mask = np.asarray(dataset.train_mask)[owned]
            count = int(np.count_nonzero(dataset.train_mask))
        self.sg = sg
        self.dg = sg
        self.model = copy_model(model)
        self.dataset = dataset
        if x_cache_bytes is None and os.environ.get("GRD_X_CACHE_GB"):
            x_cache_bytes = int(float(os.environ["GRD_X_CACHE_GB"]) * 2**30)
        self.engine = StreamingEngine(sg, self.model, src, labels, mask, x_cache_bytes=x_cache_bytes,
                                      mask_count=count)

    def reset(self, dataset, model) -> int:
        from .model import copy_model
        eng = self.engine
        if self.comm is not None:
            raise NotImplementedError("a sharded streaming session is bound to its dataset")
        eng.set_features(feature_rows(dataset, self.sg.chunks[0][1] if self.sg.chunks else 1))
        from .training import pinned_rows
        eng.labels.copy_(pinned_rows(dataset, "labels", np.asarray(dataset.labels), torch.int32),
                         non_blocking=True)
        eng.mask.copy_(pinned_rows(dataset, "mask", np.asarray(dataset.train_mask), torch.uint8),
                       non_blocking=True)
        eng.mask_count = int(np.count_nonzero(dataset.train_mask))
        self.model = copy_model(model)
        eng.model = self.model
        eng.wts.load(self.model)
        self.dataset = dataset
        return eng.labels.numel() * 4 + eng.mask.numel() + sum(w.size * 4 for w in self.model.weights)

    def run_epoch(self, epoch: int, lr: float, use_graph: bool = True) -> None:
        self.engine.epoch(lr)

    def read_stats(self) -> tuple[float, float]:
        return self.engine.read_stats()

    def train(self, epochs: int, lr: float, **_):
        trace = []
        for epoch in range(epochs):
            self.engine.epoch(lr)
            loss, acc = self.read_stats()
            if not np.isfinite(loss):
                raise ValueError(f"non-finite loss {loss} at epoch {epoch}; "
                                 f"reduce the learning rate or check the inputs")
            trace.append((epoch, loss, acc))
        self.engine.wts.export(self.model)
        return self.model, trace
