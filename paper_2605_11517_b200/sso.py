"""Partition-wise training through the SSO manager: the
layers, their gradients and the topology live in the storage tier, the
host tier caches input layers, and the device holds one (layer, partition)
stage at a time (hierarchy.TierSession executes every move).

Per layer the trainer walks the manager's schedule with a one-stage
lookahead: while partition p's kernels run on the compute stream, the CPU
reads p+1's topology record and cache misses from storage and the copy
stream uploads p+1's gathered rows; then p's outputs come down (D2H on the
copy stream) and go to storage.  The hook order, and hence the ledger, is
the reference's (training.py:283-357): stage-in of p+1 follows p's cache
refresh, and each transfer is recorded against the stage it serves.

Input gradients of a layer accumulate in the manager's reserved host buffer
in ascending partition id whatever the schedule (training.py:339-346), so
results equal the HBM-resident engines' up to fp32 rounding and are
invariant to the partition order.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib, ops
from .engine import LayerOps

__all__ = ["OffloadedTrainer"]


class _AscendingAccumulator:
    """Adds per-partition input-gradient blocks into the host buffer in
    ascending partition id, as soon as every lower id has been added."""

    def __init__(self, session, P: int, width: int):
        self.s, self.P, self.width = session, P, width
        self.pending: dict = {}
        self.next = 0
        self.threads = os.cpu_count() or 1

    def __call__(self, pid: int, rows) -> None:
        self.pending[pid] = rows
        while self.next in self.pending:
            q = self.next
            block = self.pending.pop(q)
            f = self.s.plan.flat
            gmap = f.gather_map[f.gather_ptr[q]:f.gather_ptr[q + 1]].astype(np.int64)
            acc = self.s.host.grad_acc
            if gmap.size and block is not None:
                _lib.check(_lib.lib().grd_host_scatter_add_rows(
                    block.data_ptr(), self.width, gmap.ctypes.data, gmap.size, self.width,
                    acc.data_ptr(), acc.stride(0), self.threads), "host_scatter_add_rows")
            self.next += 1

    def finish(self) -> None:
        if self.pending or self.next != self.P:
            raise RuntimeError("backward visited a partition twice or skipped one")


class OffloadedTrainer:
    """Partition-wise training (GCN, GraphSAGE, GAT layers) whose data lives
    in the SSO tiers."""

    def __init__(self, dataset, plan, model, session, device):
        if model.row_normalize or model.dropout_rate:
            raise NotImplementedError("the offloaded path trains GCN, GraphSAGE and GAT layers "
                                      "without row normalisation / dropout")
        if list(session.dims) != list(model.dims):
            raise ValueError(f"tier session dims {session.dims} != model dims {model.dims}")
        self.s, self.plan, self.device = session, plan, device
        session.bind(dataset.features32(), device)
        self.lops = LayerOps(model, device)
        self.dims = model.dims
        self.L = model.num_layers
        self.P = plan.num_partitions
        self.V = plan.num_vertices
        self.labels = torch.from_numpy(np.asarray(dataset.labels, dtype=np.int32)).to(device)
        self.mask = torch.from_numpy(np.asarray(dataset.train_mask, dtype=np.uint8)).to(device)
        self.mask_count = int(np.count_nonzero(dataset.train_mask))
        if self.mask_count == 0:
            raise ValueError("loss mask selects no vertices")
        self.stats = torch.zeros(4, dtype=torch.float64, device=device)
        self.partials = ops.loss_partials(self.V, device)

    def _wait(self, slot) -> None:
        torch.cuda.current_stream(self.device).wait_event(slot.ready)

    def _done(self) -> torch.cuda.Event:
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        return ev

    def _loss(self, logits: torch.Tensor) -> torch.Tensor:
        C = self.dims[-1]
        grad = ops.zeros_rows(self.V, C, self.device)
        ops.softmax_xent(logits, self.V, C, self.labels, self.mask, self.mask_count, grad,
                         self.stats, self.partials)
        return grad

    def epoch(self, epoch: int, lr: float, order_of, grad_probe=None, to_host=None) -> None:
        s = self.s
        s.begin_epoch()
        for l in range(self.L):
            order = list(order_of(l, "forward"))
            prev = None                      # (slot, out, done) awaiting its store
            for pid in order:
                slot = s.open_forward(l, pid)    # overlaps the previous stage's kernels
                self._wait(slot)
                out = self.lops.layer_forward(l, slot.ga, slot.part)
                s.touch_output(slot)
                cur = (slot, out, self._done())
                if prev is not None:
                    s.close_forward(*prev)
                prev = cur
            if prev is not None:
                s.close_forward(*prev)
            s.end_forward_layer(l)
        s.run_loss(self._loss)
        loss = float(self.stats[0].item())
        if not np.isfinite(loss):
            raise ValueError(f"non-finite loss {loss} at epoch {epoch}; "
                             f"reduce the learning rate or check the inputs")
        lops = self.lops
        for l in range(self.L):
            lops.grad_sink(l).zero_()
        for l in reversed(range(self.L)):
            d_in, d_out = self.dims[l], self.dims[l + 1]
            acc = _AscendingAccumulator(s, self.P, d_in) if l > 0 else None
            grad_w, probes = {}, {}
            prev = None
            for pid in order_of(l, "backward"):
                slot = s.open_backward(l, pid)
                self._wait(slot)
                a_out = slot.a_out if slot.a_out is not None else slot.grad
                gga, gw = self.lops.backward_from_ga(l, slot.ga, a_out, slot.grad, slot.part)
                grad_w[pid] = gw
                if grad_probe is not None:
                    probes[pid] = gga
                cur = (slot, gga, self._done(), acc)
                if prev is not None:
                    s.close_backward(*prev)
                prev = cur
            if prev is not None:
                s.close_backward(*prev)
            if acc is not None:
                acc.finish()
            for pid in range(self.P):                    # ascending partition id
                if grad_probe is not None:
                    grad_probe(epoch, l, pid, to_host(probes[pid], d_in),
                               self.lops.grad_w_host(l, grad_w[pid], to_host))
                self._add(lops.grad_sink(l), grad_w[pid])
            s.end_backward_layer(l)
        lops.sgd(lr)
        s.end_epoch()

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
