"""Structured storage offloading (SSO): partition-wise training whose layer
activations live in the host tier, not in HBM (the tier
contract is hierarchy.py's GRINNDER session).

The device holds only what one (layer, partition) step needs: the gathered
block GA_p, the partition's outputs / gradient slices and the weights.
Host tier: every layer ``A^l`` and the two live gradient layers in
page-locked memory, rows in *partition order* (``plan.flat.perm``) so a
partition's targets are one contiguous slab (outputs go back with a single
D2H, output slices come up with a single H2D) while its gather rows are
regathered by a native OpenMP gather (``grd_host_gather_rows``).  Two
staging slots double-buffer the next partition's regather + H2D on a copy
stream while the current one computes (the reference's 2-partition staging
buffer, hierarchy.py:457-463).  Input gradients accumulate in the host
write-back buffer by an ordered native scatter-add in ascending partition id
(training.py:339-346), so results equal the HBM-resident engines'.

Every hook of the attached ``TierSession`` fires at its stage in the
reference's order, so the ledger of a real run is event-for-event the
simulated one (test_simulate.py:479-493 pins the same property).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import _lib, ops
from .engine import DevicePartition, LayerOps
from .ops import ld_of

__all__ = ["OffloadedTrainer"]


def _pinned(rows: int, width: int) -> torch.Tensor:
    return torch.zeros((int(rows), ld_of(width)), dtype=torch.float32).pin_memory()


class _Slot:
    """One staging slot: pinned host block + device block + ready event."""

    def __init__(self, rows: int, width: int, device):
        self.host = _pinned(rows, width)
        self.dev = torch.zeros((int(rows), ld_of(width)), dtype=torch.float32, device=device)
        self.ready = torch.cuda.Event()
        self.pid = None


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
        self.parts = [DevicePartition.from_plan(plan, q, device) for q in range(self.P)]
        self.lops = LayerOps(model, device)
        self.model = model
        self.dims = model.dims
        self.L = model.num_layers
        maxw = max(self.dims)
        # host tier: A^0..A^L and two gradient layers, partition order
        self.layers = [_pinned(self.V, d) for d in self.dims]
        feats = dataset.features32()
        self.layers[0][:, : self.dims[0]].copy_(torch.from_numpy(feats[self.perm]))
        self.grad_cur = _pinned(self.V, maxw)
        self.grad_prev = _pinned(self.V, maxw)
        self.labels = torch.from_numpy(np.asarray(dataset.labels, dtype=np.int32)[self.perm]).to(device)
        self.mask = torch.from_numpy(np.asarray(dataset.train_mask, dtype=np.uint8)[self.perm]).to(device)
        self.mask_count = int(np.count_nonzero(dataset.train_mask))
        gmax = max((g.size for g in self.gpos), default=1)
        self.slots = [_Slot(max(gmax, 1), maxw, device) for _ in range(2)]
        self.copy_stream = torch.cuda.Stream(device)
        self.pool = ThreadPoolExecutor(max_workers=1)
        self.stats = torch.zeros(4, dtype=torch.float64, device=device)
        self.partials = ops.loss_partials(self.V, device)
        self.bytes_h2d = 0
        self.bytes_d2h = 0

    # -- staging ----------------------------------------------------------
    def _fill(self, slot: _Slot, layer: int, pid: int) -> None:
        """Host regather of GA_p into the slot, then async H2D on the copy stream."""
        width = self.dims[layer]
        g = self.gpos[pid]
        src = self.layers[layer]
        _lib.check(_lib.lib().grd_host_gather_rows(
            src.data_ptr(), src.stride(0), g.ctypes.data, g.size, width, slot.host.data_ptr(),
            slot.host.stride(0), self.threads), "host_gather_rows")
        with torch.cuda.stream(self.copy_stream):
            ld = slot.host.stride(0)
            slot.dev[: g.size].copy_(slot.host[: g.size], non_blocking=True)
            slot.ready.record(self.copy_stream)
        self.bytes_h2d += g.size * ld * 4
        slot.pid = pid

    def _staged(self, layer: int, order: list[int]):
        """Yield (pid, device GA block) with the next partition prefetched."""
        if not order:
            return
        fut = self.pool.submit(self._fill, self.slots[0], layer, order[0])
        for i, pid in enumerate(order):
            fut.result()
            slot = self.slots[i % 2]
            nxt = None
            if i + 1 < len(order):
                # the other slot's previous block must be consumed first
                other = self.slots[(i + 1) % 2]
                torch.cuda.current_stream().synchronize()
                nxt = self.pool.submit(self._fill, other, layer, order[i + 1])
            torch.cuda.current_stream().wait_event(slot.ready)
            yield pid, slot.dev[: self.gpos[pid].size]
            fut = nxt

    def _slab(self, host: torch.Tensor, pid: int, width: int) -> torch.Tensor:
        r0, r1 = int(self.part_ptr[pid]), int(self.part_ptr[pid + 1])
        return host[r0:r1]

    # -- one epoch ----------------------------------------------------------
    def epoch(self, epoch: int, lr: float, order_of, grad_probe=None, to_host=None) -> None:
        hs = self.session
        hs.begin_epoch()
        dev = self.device
        for l in range(self.L):
            d_out = self.dims[l + 1]
            for pid, ga in self._staged(l, list(order_of(l, "forward"))):
                out = self.lops.layer_forward(l, ga, self.parts[pid])
                dst = self._slab(self.layers[l + 1], pid, d_out)
                dst.copy_(out[:, : dst.shape[1]], non_blocking=True)
                self.bytes_d2h += out.numel() * 4
                hs.forward_partition(l, pid)
            torch.cuda.current_stream().synchronize()   # A^{l+1} complete on the host
            hs.end_forward_layer(l)
        # loss over the logits streamed up once
        C = self.dims[-1]
        logits = self.layers[-1].to(dev, non_blocking=True)
        grad = ops.zeros_rows(self.V, C, dev)
        ops.softmax_xent(logits, self.V, C, self.labels, self.mask, self.mask_count, grad, self.stats,
                         self.partials)
        self.grad_cur[:, : grad.shape[1]].copy_(grad)
        self.bytes_h2d += logits.numel() * 4
        self.bytes_d2h += grad.numel() * 4
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
            results = {}
            for pid, ga in self._staged(l, list(order_of(l, "backward"))):
                part = self.parts[pid]
                a_out = self._slab(self.layers[l + 1], pid, d_out).to(dev, non_blocking=True)
                g = self._slab(self.grad_cur, pid, d_out)[:, : ld_of(d_out)].to(dev, non_blocking=True)
                self.bytes_h2d += (a_out.numel() + g.numel()) * 4
                gga, gw = self.lops.backward_from_ga(l, ga, a_out, g, part)
                host_ga = torch.empty(gga.shape, dtype=torch.float32).pin_memory()
                host_ga.copy_(gga, non_blocking=True)
                self.bytes_d2h += gga.numel() * 4
                results[pid] = (host_ga, gga, gw)
                hs.backward_partition(l, pid)
            torch.cuda.current_stream().synchronize()
            if l > 0:
                self.grad_prev.zero_()
            for pid in range(self.P):                    # ascending partition id
                host_ga, gga, gw = results[pid]
                if grad_probe is not None:
                    grad_probe(epoch, l, pid, to_host(gga, d_in), to_host(gw, d_out, d_in))
                self._add(wts.dw[l], gw)
                if l > 0:
                    g = self.gpos[pid]
                    _lib.check(_lib.lib().grd_host_scatter_add_rows(
                        host_ga.data_ptr(), host_ga.stride(0), g.ctypes.data, g.size, d_in,
                        self.grad_prev.data_ptr(), self.grad_prev.stride(0), self.threads),
                        "host_scatter_add_rows")
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
