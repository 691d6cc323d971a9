"""Structured storage offloading (SSO): partition-wise training whose layer
activations live in the host tier, not in HBM (the tier
contract is hierarchy.py's GRINNDER session).

The device holds only what one (layer, partition) step needs: the gathered
block GA_p, the partition's outputs / gradient slices and the weights.
Host tier: every layer ``A^l`` and the two live gradient layers in
page-locked memory, rows in *partition order* (``plan.flat.perm``) so a
partition's targets are one contiguous slab.

B200-first data movement:

* **regather = a GPU-initiated gather from host memory.**  The pinned host
  layers are mapped into the device address space (UVA), so GA_p is
  gathered by the row-gather kernel (K1) reading the host rows directly over
  the host link, straight into HBM: no CPU gather pass, no staging copy.
* a partition's output slab goes back with one D2H on a copy stream, and the
  backward reads the stored output / upstream-gradient slabs in place
  (zero-copy) inside the mask kernel;
* input gradients: each partition's grad_GA is copied into pinned staging
  and accumulated into the host gradient layer by an ordered native
  scatter-add in ascending partition id (training.py:339-346) on a worker
  thread that trails the GPU, so results equal the HBM-resident engines'
  whatever order the tier session schedules (a 3-buffer ring when the
  order is ascending, else one block per partition).

Every hook of the attached ``TierSession`` fires at its stage in the
reference's order, so the ledger of a real run is event-for-event the
simulated one (test_simulate.py:479-493 pins the same property).
"""

from __future__ import annotations

import os
import threading

import numpy as np
import torch

from . import _lib, ops
from .engine import DevicePartition, LayerOps
from .ops import ld_of

__all__ = ["OffloadedTrainer"]


def _pinned(rows: int, width: int, zero: bool = False) -> torch.Tensor:
    """Page-locked [rows, ld(width)] allocated in place (no pageable staging)."""
    t = torch.empty((int(rows), ld_of(width)), dtype=torch.float32, pin_memory=True)
    if zero:
        t.zero_()
    return t


class _OrderedScatter:
    """Accumulates per-partition input gradients into the host gradient layer
    in ascending partition id, as their D2H copies complete."""

    def __init__(self, trainer, layer: int, width: int):
        self.t, self.width = trainer, width
        self.ready = {}
        self.cv = threading.Condition()
        self.next = 0
        self.error = None
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def submit(self, pid: int, event: torch.cuda.Event, buf: torch.Tensor) -> None:
        with self.cv:
            self.ready[pid] = (event, buf)
            self.cv.notify_all()

    def wait_done(self, pid: int) -> None:
        """Block until partitions 0..pid are accumulated (their buffers free)."""
        with self.cv:
            while self.next <= pid and self.error is None:
                self.cv.wait()

    def _run(self) -> None:
        t = self.t
        try:
            while self.next < t.P:
                with self.cv:
                    while self.next not in self.ready:
                        self.cv.wait()
                    ev, buf = self.ready.pop(self.next)
                ev.synchronize()
                g = t.gpos[self.next]
                _lib.check(_lib.lib().grd_host_scatter_add_rows(
                    buf.data_ptr(), buf.stride(0), g.ctypes.data, g.size, self.width,
                    t.grad_prev.data_ptr(), t.grad_prev.stride(0), t.threads), "host_scatter_add_rows")
                with self.cv:
                    self.next += 1
                    self.cv.notify_all()
        except BaseException as exc:   # surfaced by join()
            with self.cv:
                self.error = exc
                self.cv.notify_all()

    def join(self) -> None:
        self.thread.join()
        if self.error is not None:
            raise self.error


class OffloadedTrainer:
    """GCN partition-wise training with host-resident layers (module docstring)."""

    def __init__(self, dataset, plan, model, session, device, threads: int | None = None):
        if model.kind != "gcn" or model.row_normalize or model.dropout_rate:
            raise NotImplementedError("the offloaded path trains GCN layers without "
                                      "row normalisation / dropout")
        self.plan, self.session, self.device = plan, session, device
        self.threads = threads or (os.cpu_count() or 1)
        f = plan.flat
        self.P = plan.num_partitions
        self.V = plan.num_vertices
        self.part_ptr = f.part_ptr
        rank = np.empty(self.V, dtype=np.int64)
        rank[f.perm] = np.arange(self.V)
        self.perm = f.perm.astype(np.int64)
        # gather rows of each partition as positions in partition order
        self.gpos = [rank[f.gather_map[f.gather_ptr[q]:f.gather_ptr[q + 1]]] for q in range(self.P)]
        self.gpos_dev = [torch.from_numpy(g.astype(np.int32)).to(device) for g in self.gpos]
        self.parts = [DevicePartition.from_plan(plan, q, device) for q in range(self.P)]
        self.lops = LayerOps(model, device)
        self.model = model
        self.dims = model.dims
        self.L = model.num_layers
        maxw = max(self.dims)
        # host tier: A^0..A^L and two gradient layers, partition order
        # (every row of A^1.. is written by a D2H of a full-ld output block
        # before it is read; A^0's pad columns are zeroed here)
        self.layers = [_pinned(self.V, d) for d in self.dims]
        feats = dataset.features32()
        x0 = self.layers[0]
        if x0.shape[1] != self.dims[0]:
            x0[:, self.dims[0]:].zero_()
        x0[:, : self.dims[0]].copy_(torch.from_numpy(feats[self.perm]))
        self.grad_cur = _pinned(self.V, maxw, zero=True)
        self.grad_prev = _pinned(self.V, maxw, zero=True)
        # grad_GA staging (hidden widths only: layer 0 has no input gradient):
        # a ring of kRing pinned buffers when a layer's backward visits the
        # partitions in ascending order (the scatter trails by < kRing), else a
        # pool holding every partition's block (allocated on first need)
        self.gptr = np.zeros(self.P + 1, dtype=np.int64)
        np.cumsum([g.size for g in self.gpos], out=self.gptr[1:])
        self.hid_ld = ld_of(max(self.dims[1:-1], default=1))
        gmax = max((g.size for g in self.gpos), default=1)
        self.ring = [torch.empty(gmax * self.hid_ld, dtype=torch.float32, pin_memory=True)
                     for _ in range(self.kRing)] if self.L > 1 else []
        self.ga_pool = None
        self.labels = torch.from_numpy(np.asarray(dataset.labels, dtype=np.int32)[self.perm]).to(device)
        self.mask = torch.from_numpy(np.asarray(dataset.train_mask, dtype=np.uint8)[self.perm]).to(device)
        self.mask_count = int(np.count_nonzero(dataset.train_mask))
        self.copy_stream = torch.cuda.Stream(device)
        self.stats = torch.zeros(4, dtype=torch.float64, device=device)
        self.partials = ops.loss_partials(self.V, device)
        self.bytes_h2d = 0
        self.bytes_d2h = 0

    kRing = 3

    def _ga_buffer(self, pid: int, width: int, ascending: bool, scatter) -> torch.Tensor:
        ld, rows = ld_of(width), int(self.gpos[pid].size)
        if ascending:
            if pid >= self.kRing:
                scatter.wait_done(pid - self.kRing)
            return self.ring[pid % self.kRing][: rows * ld].view(rows, ld)
        if self.ga_pool is None:
            self.ga_pool = torch.empty(int(self.gptr[-1]) * self.hid_ld, dtype=torch.float32,
                                       pin_memory=True)
        a = int(self.gptr[pid]) * ld
        return self.ga_pool[a: a + rows * ld].view(rows, ld)

    def _slab(self, host: torch.Tensor, pid: int) -> torch.Tensor:
        r0, r1 = int(self.part_ptr[pid]), int(self.part_ptr[pid + 1])
        return host[r0:r1]

    def _regather(self, layer: int, pid: int) -> torch.Tensor:
        """GA_p gathered by the device straight from the host layer (UVA)."""
        width = self.dims[layer]
        idx = self.gpos_dev[pid]
        ga = ops.zeros_rows(idx.numel(), width, self.device)
        ops.gather_rows(self.layers[layer], idx, ga, width)
        self.bytes_h2d += idx.numel() * ld_of(width) * 4
        return ga

    def _to_host(self, src: torch.Tensor, dst: torch.Tensor) -> torch.cuda.Event:
        """Async D2H on the copy stream after the producing kernels."""
        done = torch.cuda.Event()
        done.record()
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_event(done)
            dst.copy_(src[:, : dst.shape[1]], non_blocking=True)
            src.record_stream(self.copy_stream)
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        self.bytes_d2h += dst.numel() * 4
        return ev

    # -- one epoch ----------------------------------------------------------
    def epoch(self, epoch: int, lr: float, order_of, grad_probe=None, to_host=None) -> None:
        hs = self.session
        hs.begin_epoch()
        dev = self.device
        for l in range(self.L):
            for pid in order_of(l, "forward"):
                out = self.lops.layer_forward(l, self._regather(l, pid), self.parts[pid])
                self._to_host(out, self._slab(self.layers[l + 1], pid))
                hs.forward_partition(l, pid)
            self.copy_stream.synchronize()              # A^{l+1} complete on the host
            hs.end_forward_layer(l)
        # loss over the logits, read in place from the host tier
        C = self.dims[-1]
        grad = ops.zeros_rows(self.V, C, dev)
        ops.softmax_xent(self.layers[-1], self.V, C, self.labels, self.mask, self.mask_count, grad,
                         self.stats, self.partials)
        self.bytes_h2d += self.layers[-1].numel() * 4
        self._to_host(grad, self.grad_cur[:, : grad.shape[1]]).synchronize()
        loss = float(self.stats[0].item())
        if not np.isfinite(loss):
            raise ValueError(f"non-finite loss {loss} at epoch {epoch}; "
                             f"reduce the learning rate or check the inputs")
        hs.loss_stage()
        wts = self.lops.wts
        for dw in wts.dw:
            dw.zero_()
        for l in reversed(range(self.L)):
            d_in, d_out = self.dims[l], self.dims[l + 1]
            grad_w = {}
            probes = {}
            scatter = None
            if l > 0:
                self.grad_prev.zero_()
                scatter = _OrderedScatter(self, l, d_in)
            order = list(order_of(l, "backward"))
            ascending = order == list(range(self.P))
            try:
                for pid in order:
                    part = self.parts[pid]
                    # stored output (ReLU mask) and upstream gradient: read in place
                    a_out = self._slab(self.layers[l + 1], pid)
                    g = self._slab(self.grad_cur, pid)[:, : ld_of(d_out)]
                    self.bytes_h2d += (a_out.numel() + g.numel()) * 4
                    gga, gw = self.lops.backward_from_ga(l, self._regather(l, pid), a_out, g, part)
                    grad_w[pid] = gw
                    if grad_probe is not None:
                        probes[pid] = gga
                    if scatter is not None:
                        buf = self._ga_buffer(pid, d_in, ascending, scatter)
                        scatter.submit(pid, self._to_host(gga, buf), buf)
                    hs.backward_partition(l, pid)
            finally:
                if scatter is not None:
                    scatter.join()
            for pid in range(self.P):                    # ascending partition id
                if grad_probe is not None:
                    grad_probe(epoch, l, pid, to_host(probes[pid], d_in), to_host(grad_w[pid], d_out, d_in))
                self._add(wts.dw[l], grad_w[pid])
            hs.end_backward_layer(l)
            self.grad_cur, self.grad_prev = self.grad_prev, self.grad_cur
        for w, dw in zip(wts.w, wts.dw):
            ops.wgrad_sgd(w, w, dw, dw.shape[0], dw.shape[1], 0, accumulate=True, w=w, lr=lr)
        hs.end_epoch()

    _eye: dict = {}

    def _add(self, dst: torch.Tensor, src: torch.Tensor) -> None:
        rows = src.shape[0]
        idx = self._eye.get((rows, str(self.device)))
        if idx is None:
            idx = torch.arange(rows, dtype=torch.int32, device=self.device)
            self._eye[(rows, str(self.device))] = idx
        ops.scatter_add_rows(src, idx, dst, src.shape[1])

    def read_stats(self) -> tuple[float, float]:
        s = self.stats.cpu().numpy()
        return float(s[0]), float(s[1])
