"""Public training API (reference: grinder/training.py), executed on the GPU.

Same names, signatures, return values and ValueError behaviour as the
reference:

* ``partitioned_train(dataset, plan, model, epochs, lr, hierarchy=None,
  use_snapshots=False, grad_probe=None, partition_order=None)``
  -> ``(ModelState, [(epoch, loss, acc)], ledger)`` (training.py:259-358)
* ``layer_forward`` / ``regather_backward`` / ``scatter_accumulate`` — the
  per-(layer, partition) operators (training.py:86-175)
* ``reference_train`` / ``compute_gradients`` — the monolithic (P = 1)
  execution (training.py:193-256)

Inputs may be the reference's numpy arrays; everything computes in fp32 on
the device through libgrinder_b200.so (no CPU fallback).  Without observers
(``grad_probe``, ``use_snapshots``, ``hierarchy``) the fused layer-wide
engine runs and each epoch is replayed from a captured CUDA graph; with
observers the literal per-partition schedule runs so every hook and probe
sees per-partition tensors in the reference's order.
"""

from __future__ import annotations

import os

from pathlib import Path

import numpy as np
import torch

from . import ops
from .dataset import LabeledDataset
from .engine import (DeviceGraph, DevicePartition, LayerOps, LayerwiseEngine, PartitionEngine,
                     ShardDeviceGraph)
from .model import ModelState, copy_model
from .plan import PartitionPlan, PartitionTopology, build_partition_plan

__all__ = [
    "compute_gradients",
    "layer_forward",
    "partitioned_train",
    "reference_train",
    "regather_backward",
    "scatter_accumulate",
    "trace_to_csv",
    "write_trace_csv",
    "TrainSession",
    "pinned_features",
    "session_for",
]


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2605_11517_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(mat: np.ndarray, dev, width: int | None = None) -> torch.Tensor:
    mat = np.asarray(mat)
    rows, cols = mat.shape
    t = ops.zeros_rows(rows, cols if width is None else width, dev)
    t[:, :cols] = torch.from_numpy(np.ascontiguousarray(mat, dtype=np.float32)).to(dev)
    return t


def _to_host(t: torch.Tensor, cols: int, rows: int | None = None) -> np.ndarray:
    r = t.shape[0] if rows is None else rows
    return t[:r, :cols].double().cpu().numpy()


# --------------------------------------------------------------------------
# per-(layer, partition) operators
# --------------------------------------------------------------------------
def layer_forward(layer: int, input_rows: np.ndarray, topology: PartitionTopology,
                  model: ModelState) -> np.ndarray:
    """One layer over one partition: gathered rows in, target rows out."""
    weight = model.weights[layer]
    if input_rows.ndim != 2 or input_rows.shape[0] != topology.gather_map.size:
        raise ValueError(f"input has {input_rows.shape[0]} rows, gather map needs "
                         f"{topology.gather_map.size}")
    if input_rows.shape[1] != weight.shape[0]:
        raise ValueError(f"input width {input_rows.shape[1]} != layer {layer} input dim "
                         f"{weight.shape[0]}")
    dev = _device()
    lops = LayerOps(model, dev)
    part = DevicePartition.from_topology(topology, dev)
    out = lops.layer_forward(layer, _to_dev(input_rows, dev), part)
    return _to_host(out, model.dims[layer + 1])


def regather_backward(layer: int, partition: int, A_out: np.ndarray, grad_out: np.ndarray,
                      cached_A_in: np.ndarray, plan: PartitionPlan, model: ModelState
                      ) -> tuple[np.ndarray, np.ndarray]:
    """Backward of one (layer, partition) from inputs regathered out of the
    resident layer activations (training.py:146-163)."""
    topo = plan.topologies[partition]
    if cached_A_in is None or cached_A_in.shape[0] < plan.num_vertices:
        raise ValueError(f"partition {partition} input activations are not resident; the "
                         f"hierarchy must load them before backward")
    if A_out.shape[0] != topo.targets.size or grad_out.shape != A_out.shape:
        raise ValueError("output rows must match the partition's target count")
    dev = _device()
    lops = LayerOps(model, dev)
    part = DevicePartition.from_topology(topo, dev)
    d_in, d_out = model.dims[layer], model.dims[layer + 1]
    a_in = _to_dev(cached_A_in, dev)
    ga = ops.zeros_rows(part.num_gather, d_in, dev)
    ops.gather_rows(a_in, part.gather_map, ga, d_in)
    grad_ga, grad_w = lops.backward_from_ga(layer, ga, _to_dev(A_out, dev), _to_dev(grad_out, dev),
                                            part)
    return _to_host(grad_ga, d_in), lops.grad_w_host(layer, grad_w, _to_host)


def scatter_accumulate(grad_GA: np.ndarray, gather_map: np.ndarray,
                       global_grad: np.ndarray) -> np.ndarray:
    """global_grad[gather_map] += grad_GA in place (training.py:166-175)."""
    dev = _device()
    width = global_grad.shape[1]
    g = _to_dev(global_grad, dev)
    idx = torch.from_numpy(np.asarray(gather_map, dtype=np.int32)).to(dev)
    ops.scatter_add_rows(_to_dev(grad_GA, dev), idx, g, width)
    global_grad[...] = _to_host(g, width)
    return global_grad


# --------------------------------------------------------------------------
# sessions: device-resident state reused across calls
# --------------------------------------------------------------------------
class TrainSession:
    """Device-resident training state for one (dataset, plan, model config).

    Uploads the plan once (cached on the plan object), keeps activations,
    gradients and fp32 weights in HBM, and replays the fused epoch from a
    CUDA graph.  ``partitioned_train`` uses one internally; benchmarks and
    multi-epoch drivers can hold one explicitly.
    """

    def __init__(self, dataset: LabeledDataset, plan: PartitionPlan, model: ModelState,
                 layerwise: bool = True, comm=None):
        if plan.num_vertices != dataset.graph.num_vertices:
            raise ValueError("plan was built for a different graph")
        self.dev = _device()
        self.comm = comm
        if comm is None:
            key = ("device_graph", str(self.dev))
            dg = plan.device_cache.get(key)
            if dg is None:
                dg = DeviceGraph(dataset.graph, plan, self.dev)
                plan.device_cache[key] = dg
        else:
            if not layerwise:
                raise NotImplementedError("per-partition observers run on one device")
            from .distributed import build_shard_plan
            key = ("shard", comm.rank, comm.world, str(self.dev))
            dg = plan.device_cache.get(key)
            if dg is None:
                shard = build_shard_plan(dataset.graph, plan, comm.rank, comm.world, comm)
                dg = ShardDeviceGraph(dataset.graph, plan, shard, comm, self.dev)
                plan.device_cache[key] = dg
        self.dg = dg
        self.model = copy_model(model)
        self.dataset = dataset
        F = dataset.feature_dim
        if layerwise and model.kind == "sage" and model.dims[1] > model.dims[0]:
            # room for mean(X) beside X (engine: one [X | mean(X)] GEMM in layer 0)
            buf = torch.zeros((dg.n_local, 2 * ops.ld_of(F)), dtype=torch.float32, device=self.dev)
            features = buf[:, : ops.ld_of(F)]
        else:
            features = ops.zeros_rows(dg.n_local, F, self.dev)
        cls = LayerwiseEngine if layerwise else PartitionEngine
        own = slice(None) if comm is None else dg.shard.owned
        self.engine = cls(dg, self.model, features, np.asarray(dataset.labels)[own],
                          np.asarray(dataset.train_mask)[own],
                          mask_count=int(np.count_nonzero(dataset.train_mask)))
        self.upload_features(dataset)
        self.layerwise = layerwise
        self._graph = None
        self._graph_lr = None
        self.stats_host = torch.zeros(4, dtype=torch.float64).pin_memory()

    def signature(self) -> tuple:
        m = self.model
        return (tuple(m.dims), m.aggregation_mode, m.heads, m.row_normalize, m.dropout_rate,
                m.dropout_seed, self.layerwise)

    def upload_features(self, dataset: LabeledDataset) -> int:
        """H2D of the features (this device's rows) from pinned host memory;
        returns bytes moved."""
        src = pinned_features(dataset)
        if self.comm is not None:
            src = src[torch.from_numpy(self.dg.shard.local_ids)]
        dst = self.engine.acts[0]
        f = src.shape[1]
        if dst.shape[1] == f:
            dst.copy_(src, non_blocking=True)
        else:
            dst[:, :f].copy_(src, non_blocking=True)
        return src.numel() * 4

    def reset(self, dataset: LabeledDataset, model: ModelState) -> int:
        """Re-bind the session to (dataset, model): uploads features, labels,
        mask and weights into the existing buffers (a captured CUDA graph
        stays valid).  Returns the H2D bytes."""
        eng = self.engine
        moved = self.upload_features(dataset)
        own = slice(None) if self.comm is None else self.dg.shard.owned
        lab, msk = np.asarray(dataset.labels)[own], np.asarray(dataset.train_mask)[own]
        eng.labels.copy_(pinned_rows(dataset, "labels", lab, torch.int32), non_blocking=True)
        eng.mask.copy_(pinned_rows(dataset, "mask", msk, torch.uint8), non_blocking=True)
        count = int(np.count_nonzero(dataset.train_mask))
        if count != eng.mask_count:
            # the loss kernel takes 1/|mask| by value: a captured epoch graph
            # holds the old count, so it is re-captured on the next epoch
            eng.mask_count = count
            self._graph = None
        if count == 0:
            raise ValueError("train_mask selects no vertices")
        self.model = copy_model(model)
        eng.wts.load(self.model)
        self.dataset = dataset
        moved += eng.labels.numel() * 4 + eng.mask.numel()
        moved += sum(w.size * 4 for w in self.model.weights)
        return moved

    def _capture(self, lr: float) -> None:
        eng = self.engine
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            # warm-up outside capture so lazily built scale arrays / heavy-row
            # scratch exist before the graph records their addresses
            params = eng.wts.params()
            snap = [w.clone() for w in params]
            eng.epoch(lr)
            for w, s in zip(params, snap):
                w.copy_(s)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        # no garbage collection while capturing (a finalizer's CUDA call, e.g.
        # cudaHostUnregister of a collected array, would invalidate the
        # capture), and other threads' CUDA calls do not count against it
        import gc
        gc_was = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                eng.epoch(lr)
        finally:
            if gc_was:
                gc.enable()
        self._graph, self._graph_lr = g, lr

    def run_epoch(self, epoch: int, lr: float, use_graph: bool = True) -> None:
        """Enqueue one fused epoch (loss stats land in engine.stats)."""
        eng = self.engine
        if self.comm is not None:
            use_graph = False   # collectives stay outside CUDA graphs
        if eng.dropout_rate > 0.0:
            eng.set_dropout(epoch)
            use_graph = False   # fresh masks every epoch
        if not use_graph:
            eng.epoch(lr)
            return
        if self._graph is None or self._graph_lr != lr:
            self._capture(lr)
        self._graph.replay()

    def read_stats(self) -> tuple[float, float]:
        self.stats_host.copy_(self.engine.stats)
        s = self.stats_host.numpy()
        return float(s[0]), float(s[1])

    def train(self, epochs: int, lr: float, hierarchy=None, use_snapshots=False, grad_probe=None,
              partition_order=None, use_graph: bool = True):
        P = self.dg.num_partitions

        def order_of(layer: int, phase: str) -> list[int]:
            if partition_order is not None:
                return list(partition_order(layer, phase))
            if hierarchy is not None:
                return list(hierarchy.partition_order(layer, phase))
            return list(range(P))

        trace = []
        for epoch in range(epochs):
            if self.layerwise:
                self.run_epoch(epoch, lr, use_graph=use_graph)
                loss, acc = self.read_stats()
                if not np.isfinite(loss):
                    raise ValueError(f"non-finite loss {loss} at epoch {epoch}; "
                                     f"reduce the learning rate or check the inputs")
            else:
                eng = self.engine
                eng.set_dropout(epoch)
                eng.epoch(epoch, lr, order_of, hierarchy=hierarchy, use_snapshots=use_snapshots,
                          grad_probe=grad_probe, to_host=_to_host)
                loss, acc = self.read_stats()
            trace.append((epoch, loss, acc))
        self.engine.wts.export(self.model)
        return self.model, trace


def partitioned_train(dataset: LabeledDataset, plan: PartitionPlan, model: ModelState, epochs: int,
                      lr: float, hierarchy=None, use_snapshots: bool = False, grad_probe=None,
                      partition_order=None):
    """Partition-wise training with on-demand input regathering
    (training.py:259-358).  Returns (model, trace, ledger)."""
    if plan.num_vertices != dataset.graph.num_vertices:
        raise ValueError("plan was built for a different graph")
    observed = hierarchy is not None or use_snapshots or grad_probe is not None \
        or partition_order is not None
    from .hierarchy import TierSession
    if isinstance(hierarchy, TierSession) and hierarchy.execute:
        if use_snapshots:
            raise NotImplementedError("the offloaded path regathers; snapshots stay in HBM only")
        return _offloaded_train(dataset, plan, model, epochs, lr, hierarchy, grad_probe,
                                partition_order)
    session = session_for(dataset, plan, model, layerwise=not observed)
    trained, trace = session.train(epochs, lr, hierarchy=hierarchy, use_snapshots=use_snapshots,
                                   grad_probe=grad_probe, partition_order=partition_order)
    if epochs == 0:
        trained = copy_model(model)
    return trained, trace, getattr(hierarchy, "ledger", None)


def pinned_rows(dataset: LabeledDataset, name: str, values: np.ndarray, dtype) -> torch.Tensor:
    """``values`` converted to ``dtype`` in a page-locked staging buffer kept
    on the dataset (refilled every call), so its H2D copy is a true async
    DMA instead of a pageable copy."""
    key = "_pinned_" + name
    stage = getattr(dataset, key, None)
    if stage is None or stage.numel() != values.size or stage.dtype != dtype:
        stage = torch.empty(values.size, dtype=dtype).pin_memory()
        setattr(dataset, key, stage)
    np.copyto(stage.numpy(), values, casting="unsafe")
    return stage


def pinned_features(dataset: LabeledDataset) -> torch.Tensor:
    """Host fp32 features to upload.  fp32 features are used in place (a
    page-locked array gives a true async H2D); f64 features are converted
    on every call into a page-locked staging buffer kept on the dataset, so
    in-place edits of ``dataset.features`` are always seen."""
    feats = dataset.features
    if feats.dtype == np.float32 and feats.flags.c_contiguous:
        return torch.from_numpy(feats)
    stage = getattr(dataset, "_pinned", None)
    if stage is None or tuple(stage.shape) != tuple(feats.shape):
        stage = torch.empty(feats.shape, dtype=torch.float32).pin_memory()
        dataset._pinned = stage
    np.copyto(stage.numpy(), feats, casting="same_kind")
    return stage


def _communicator():
    """A Communicator when this process is one rank of a multi-rank job."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        from .distributed import Communicator
        return Communicator()
    return None


def session_for(dataset: LabeledDataset, plan: PartitionPlan, model: ModelState,
                layerwise: bool = True) -> TrainSession:
    """A device session for (dataset, plan, model config), reused across
    calls: the plan upload, buffers and the captured epoch graph persist on
    the plan (``plan.device_cache``); inputs are re-uploaded every call.
    Inside an initialised torch.distributed job with several ranks the
    session is this rank's shard of the partitions (distributed.py)."""
    comm = _communicator()
    key = ("session", tuple(model.dims), model.aggregation_mode, model.heads, model.row_normalize,
           model.dropout_rate, model.dropout_seed, layerwise, comm is not None)
    sess = plan.device_cache.get(key)
    # the engine choice is made once per (plan, model config): a later call
    # must not re-decide against the HBM the cached session itself holds
    forced = os.environ.get("GRD_ENGINE", "")
    if sess is not None and forced in ("stream", "resident"):
        from .stream import StreamSession
        if isinstance(sess, StreamSession) != (forced == "stream"):
            del plan.device_cache[key]      # release it before building the other engine
            sess = None
            import gc
            gc.collect()
            torch.cuda.empty_cache()
    if sess is None:
        stream = layerwise and _use_streaming(dataset, model, comm)
        if stream:
            from .stream import StreamSession
            sess = StreamSession(dataset, plan, model, comm=comm)
        else:
            sess = TrainSession(dataset, plan, model, layerwise=layerwise, comm=comm)
        plan.device_cache[key] = sess
    else:
        if plan.num_vertices != dataset.graph.num_vertices:
            raise ValueError("plan was built for a different graph")
        sess.reset(dataset, model)
    return sess


def _use_streaming(dataset: LabeledDataset, model: ModelState, comm=None) -> bool:
    """Stream the layers through HBM (stream.py) when the resident engine's
    working set does not fit the device; GRD_ENGINE=stream|resident forces.
    Sharded: a rank's rows are its owned vertices plus their halo (about
    three times V / world on the papers-shaped graphs)."""
    import os
    from .stream import resident_bytes, streaming_supported
    forced = os.environ.get("GRD_ENGINE", "")
    if forced in ("stream", "resident"):
        if forced == "stream" and streaming_supported(model) is not None:
            raise NotImplementedError(streaming_supported(model))
        return forced == "stream"
    if streaming_supported(model) is not None or (comm is not None and model.num_layers > 3):
        return False
    free, _ = torch.cuda.mem_get_info()
    avail = free + torch.cuda.memory_reserved() - torch.cuda.memory_allocated()
    g = dataset.graph
    rows = g.num_vertices if comm is None else min(g.num_vertices, 3 * g.num_vertices // comm.world)
    edges = g.num_edges if comm is None else g.num_edges // comm.world
    return resident_bytes(rows, edges, model) > 0.9 * avail


def _offloaded_train(dataset, plan, model, epochs, lr, hierarchy, grad_probe, partition_order):
    """Structured storage offloading: layers live in the host tier (sso.py)."""
    from .sso import OffloadedTrainer
    trained = copy_model(model)
    if epochs == 0:
        return trained, [], hierarchy.ledger
    trainer = OffloadedTrainer(dataset, plan, trained, hierarchy, _device())

    def order_of(layer: int, phase: str) -> list[int]:
        if partition_order is not None:
            return list(partition_order(layer, phase))
        return list(hierarchy.partition_order(layer, phase))

    trace = []
    for epoch in range(epochs):
        trainer.epoch(epoch, lr, order_of, grad_probe=grad_probe, to_host=_to_host)
        loss, acc = trainer.read_stats()
        trace.append((epoch, loss, acc))
    trainer.lops.wts.export(trained)
    return trained, trace, hierarchy.ledger


def _whole_graph_plan(dataset: LabeledDataset) -> PartitionPlan:
    n = dataset.graph.num_vertices
    return build_partition_plan(dataset.graph, np.zeros(n, dtype=np.int32), 1)


def reference_train(dataset: LabeledDataset, model: ModelState, epochs: int, lr: float):
    """Whole-graph training (training.py:193-206): the P = 1 plan."""
    trained, trace, _ = partitioned_train(dataset, _whole_graph_plan(dataset), model, epochs, lr)
    return trained, trace


def compute_gradients(dataset: LabeledDataset, model: ModelState):
    """Monolithic loss, train accuracy and per-layer weight gradients
    (training.py:231-236), without updating the weights."""
    session = TrainSession(dataset, _whole_graph_plan(dataset), model)
    trained, trace = session.train(1, 0.0, use_graph=False)
    _, loss, acc = trace[0]
    return loss, acc, trained.weight_grads


def trace_to_csv(trace: list[tuple[int, float, float]]) -> str:
    rows = ["epoch,loss,train_acc"] + [f"{e},{l!r},{a!r}" for e, l, a in trace]
    return "\n".join(rows) + "\n"


def write_trace_csv(path: str | Path, trace: list[tuple[int, float, float]]) -> None:
    Path(path).write_text(trace_to_csv(trace))
