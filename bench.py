"""Benchmark of the partition-wise full-graph training step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

A step is one full-graph training epoch (forward over every partition, loss,
regather backward, SGD) of the named synthetic workload.  The default is
``papers_full``: configs[3] at full size (3-layer GCN, F=H=128, C=172 on a
134 M-vertex / 1.61 B-edge papers-shaped Kronecker graph, 16 switching-aware
partitions), the north-star target.  Prints ONE JSON line (rank 0).  Metric
(BASELINE.json): aggregated edges/s = L*|E| per epoch over all GPUs, plus
epoch time; ``roofline`` is the dominant kernel's DRAM-side HBM fraction
(ncu DRAM bytes per launch over the live launch time) with the SURVEY 8(d)
per-edge streaming-model figure beside it; ``engines`` times the other
engines (kept-state / regather layer-wise, per-partition with the K1 gather,
streaming) on the largest papers-shaped instance the reference itself
trained for the golden fixtures.

--impl reference times the reference algorithm's CPU implementation — the
float64 numpy restatement in oracle/ (pinned to the reference's golden
vectors; the reference package itself is not installed on the GPU box) —
on the host cores, on a bounded sample of the same workload built by the
oracle alone (oracle/workload.py: no product code, no native library).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# name -> synthetic workload (BASELINE.json configs; seeds follow the
# reference CLI: graph S, dataset S+1, partitioner S+2, model S+3; lr 0.01)
WORKLOADS = {
    "config1": dict(
        desc="configs[0]: 2-layer GCN hidden 64, generate_kronecker(17, 8): 131,072 V / "
             "1,048,576 E, 128 feats, 10 classes, 8 switching-aware partitions",
        scale=17, deg=8, F=128, C=10, L=2, H=64, P=8, mode="mean_self_loop",
    ref_sample=dict(scale=15, deg=8)),
}
WORKLOADS["products_sage"] = dict(
    desc="configs[1]: 3-layer GraphSAGE-mean hidden 256, ogbn-products-shaped "
         "generate_kronecker(21, 30): 2,097,152 V / 62,914,560 E, 100 feats, 47 classes, "
         "8 switching-aware partitions",
    scale=21, deg=30, F=100, C=47, L=3, H=256, P=8, mode="sage_mean",
    cpu_sample=dict(scale=18, deg=30), ref_sample=dict(scale=17, deg=30))
WORKLOADS["products_gat"] = dict(
    desc="configs[2]: 3-layer GAT (4 heads x 64 concat, mean on the last layer) on the "
         "ogbn-products-shaped generate_kronecker(21, 30): 2,097,152 V / 62,914,560 E, "
         "100 feats, 47 classes, 8 switching-aware partitions",
    scale=21, deg=30, F=100, C=47, L=3, H=256, P=8, mode="gat", heads=4,
    cpu_sample=dict(scale=16, deg=30), ref_sample=dict(scale=15, deg=30))
WORKLOADS["papers_gcn"] = dict(
    desc="configs[3] shape at 1/3.3 size (HBM-resident on one B200): 3-layer GCN hidden 128, "
         "ogbn-papers100M-shaped generate_kronecker(25, 14): 33,554,432 V / 469,762,048 E "
         "(papers100M average degree), 128 feats, 172 classes, 16 switching-aware partitions",
    scale=25, deg=14, F=128, C=172, L=3, H=128, P=16, mode="mean_self_loop",
    cpu_sample=dict(scale=16, deg=14), ref_sample=dict(scale=15, deg=14))
WORKLOADS["papers_full"] = dict(
    desc="configs[3] at full size: 3-layer GCN hidden 128 on an ogbn-papers100M-shaped "
         "generate_kronecker(27, 12): 134,217,728 V / 1,610,612,736 E (1.6 B edges, papers "
         "average degree), 128 feats, 172 classes, 16 switching-aware partitions; the layers do "
         "not fit HBM, so the streaming engine keeps two layer buffers + the graph in HBM and "
         "streams the host-resident features (stream.py)",
    scale=27, deg=12, F=128, C=172, L=3, H=128, P=16, mode="mean_self_loop",
    feature_dtype="float32", host_gb=150, cpu_sample=dict(scale=16, deg=12),
    ref_sample=dict(scale=15, deg=12), sharded_stream=True)
WORKLOADS["papers_s22"] = dict(
    desc="configs[3]'s model on the papers-shaped golden instance generate_kronecker(22, 12): "
         "4,194,304 V / 50,331,648 E, 128 feats, 172 classes, 16 switching-aware partitions "
         "(the reference itself trained it for tests/golden/papers_s22.npz); at N > 1 it runs "
         "papers_full's sharded layer-streaming path at a size one GPU can host twice",
    scale=22, deg=12, F=128, C=172, L=3, H=128, P=16, mode="mean_self_loop",
    feature_dtype="float32", cpu_sample=dict(scale=16, deg=12), ref_sample=dict(scale=15, deg=12),
    sharded_stream=True)
WORKLOADS["igb_nvme"] = dict(
    desc="configs[4] model and tiers at 1/24 of its size: 3-layer GraphSAGE-mean hidden 256 on "
         "IGB-shaped 1024-wide features, generate_kronecker(22, 12) (4,194,304 V / 50,331,648 E), "
         "19 classes, 8 partitions; the 17.2 GB feature file stays on the box's disk "
         "(load_dataset(mmap_features=True)) behind a 4 GiB HBM cache and a 4 GiB pinned host "
         "cache, the rest read per pass with direct I/O (tiers.py, streaming engine)",
    scale=22, deg=12, F=1024, C=19, L=3, H=256, P=8, mode="sage_mean",
    feature_dtype="float32", tier="nvme", x_cache_gb=4, host_cache_gb=4,
    cpu_sample=dict(scale=14, deg=12))
DEFAULT_WORKLOAD = "papers_full"
LR = 0.01
SEED = 0


def rank_info():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def _cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def build_workload(spec):
    import paper_2605_11517_b200 as g2
    t0 = time.perf_counter()
    gpu_gen = spec["scale"] >= 20 and _cuda_ok()
    if gpu_gen:   # bit-identical to the host generator (tests/test_gpu_generate.py)
        import torch
        g = g2.generate_kronecker(spec["scale"], spec["deg"], seed=SEED, device="cuda")
        torch.cuda.empty_cache()
    else:
        g = g2.generate_kronecker(spec["scale"], spec["deg"], seed=SEED)
    t_gen = time.perf_counter() - t0
    ds = g2.make_random_dataset(g, feature_dim=spec["F"], num_classes=spec["C"], seed=SEED + 1,
                                feature_dtype=np.dtype(spec.get("feature_dtype", "float64")))
    t1 = time.perf_counter()
    # GPU partitioner when the GPU generator ran: bit-identical labels, trace
    # and iteration count (tests/test_gpu_partition.py, reference digests in
    # tests/test_gpu_golden_scale.py)
    part = g2.switching_aware_partition(g, spec["P"], g2.PartitionerParams(seed=SEED + 2),
                                        device="cuda" if gpu_gen else None)
    t_part = time.perf_counter() - t1
    t2 = time.perf_counter()
    # bit-identical to the host plan (tests/test_gpu_plan.py)
    plan = g2.build_partition_plan(g, part.labels, spec["P"], device="cuda" if gpu_gen else None)
    t_plan = time.perf_counter() - t2
    if gpu_gen:
        import torch
        torch.cuda.empty_cache()    # the plan builder's sort scratch
    model = g2.create_model(spec["F"], spec["C"], num_layers=spec["L"], hidden_dim=spec["H"],
                            seed=SEED + 3, aggregation_mode=spec["mode"],
                            heads=spec.get("heads", 4))
    prep = {"generate_s": round(t_gen, 3), "generator": "gpu" if gpu_gen else "host", "partition_s": round(t_part, 3),
            "partitioner": "gpu" if gpu_gen else "host", "plan_s": round(t_plan, 3), "partitioner_iterations": part.iterations}
    return g, ds, plan, model, prep


class ClockSampler:
    """NVML sampling of SM clock / throttle reasons while the timed region runs."""

    REASONS = {
        "hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4,
    }

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = None
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(index).uuid)
                self.h = pynvml.nvmlDeviceGetHandleByUUID(
                    uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(0 if pynvml.nvmlDeviceGetCount() == 1 else index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML missing
            self.nv = None
        self.active = False
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        while not self._stop.is_set():
            if self.nv is not None and self.active:
                try:
                    mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                    util = self.nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                    getr = getattr(self.nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                        self.nv.nvmlDeviceGetCurrentClocksThrottleReasons
                    mask = getr(self.h)
                    self.samples.append((mhz, util))
                    for name, bit in self.REASONS.items():
                        if mask & bit:
                            self.reasons.add(name)
                except Exception:
                    pass
            time.sleep(0.002)

    def summary(self):
        self._stop.set()
        loaded = [m for m, u in self.samples if u > 0] or [m for m, _ in self.samples]
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1671.0)), "measured"
    return 6650.0, 1590.0, "fallback"


def flush_l2(buf):
    buf.add_(1.0)   # 512 MiB write evicts the 126 MB L2 between timed steps


# the papers-shaped instance the reference itself trained for the golden
# fixtures (tests/golden/papers_s22.npz): configs[3]'s model on
# generate_kronecker(22, 12)
ENGINE_SPEC = dict(desc="configs[3]'s model (3-layer GCN, F=H=128, C=172, P=16) on "
                        "generate_kronecker(22, 12): 4,194,304 V / 50,331,648 E",
                   scale=22, deg=12, F=128, C=172, L=3, H=128, P=16, mode="mean_self_loop",
                   feature_dtype="float32")


def engine_table(reps: int = 3):
    """Epoch time of each engine on ENGINE_SPEC, so every subsystem of the
    north star is timed: the layer-wise engine keeping the forward state
    (the default when HBM allows), the same engine regathering in the
    backward (GRD_KEEP_AGG=0: the reference's regather schedule), the
    per-partition engine (K1 gather of GA_p per (layer, partition),
    regather backward, scatter — the schedule observers see) and the
    layer-streaming engine (stream.py).  CUDA events on the current stream,
    L2 flushed before every epoch."""
    import gc
    import torch
    from paper_2605_11517_b200.stream import StreamSession
    from paper_2605_11517_b200.training import TrainSession
    g, ds, plan, model, _ = build_workload(ENGINE_SPEC)
    edges = ENGINE_SPEC["L"] * g.num_edges
    flush = torch.zeros(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
    out = {"workload": ENGINE_SPEC["desc"], "reps": reps,
           "hbm_allocated_GB_before": round(torch.cuda.memory_allocated() / 2**30, 2)}

    def timed(run):
        for w in range(2):
            run(w)
        ms = []
        for k in range(reps):
            flush_l2(flush)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            run(k)
            e.record()
            torch.cuda.synchronize()
            ms.append(s.elapsed_time(e))
        return min(ms)

    def record(name, ms, loss, note):
        out[name] = {"ms_per_epoch": round(ms, 3), "edges_per_s": round(edges / (ms * 1e-3), 1),
                     "loss": loss, "note": note}

    prev = os.environ.get("GRD_KEEP_AGG")
    for name, keep, note in (("layerwise_kept", "1", "HBM-resident layer-wise, forward "
                              "aggregates kept for the weight gradient"),
                             ("layerwise_regather", "0", "HBM-resident layer-wise, backward "
                              "regathers (GRD_KEEP_AGG=0)")):
        os.environ["GRD_KEEP_AGG"] = keep
        sess = TrainSession(ds, plan, model)
        ms = timed(lambda k: sess.run_epoch(k, LR))
        record(name, ms, sess.read_stats()[0], note)
        del sess
        gc.collect()
    if prev is None:
        os.environ.pop("GRD_KEEP_AGG", None)
    else:
        os.environ["GRD_KEEP_AGG"] = prev
    sess = TrainSession(ds, plan, model, layerwise=False)
    ms = timed(lambda k: sess.train(1, LR, use_graph=False))
    record("per_partition", ms, sess.read_stats()[0],
           "per-(layer, partition) schedule: K1 gather of GA_p, aggregate, transform; "
           "regather backward; ascending-pid scatter (eager, includes the weight export)")
    del sess
    gc.collect()
    sess = StreamSession(ds, plan, model)
    ms = timed(lambda k: sess.run_epoch(k, LR))
    record("streaming", ms, sess.read_stats()[0], "layer-streaming engine (stream.py), "
           "features in the HBM cache")
    del sess, flush
    plan.device_cache.clear()
    gc.collect()
    torch.cuda.empty_cache()
    return out


def run_ours(args, spec, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2605_11517_b200 as g2
    from paper_2605_11517_b200 import ops
    from paper_2605_11517_b200.training import session_for

    # GRD_BENCH_BACKEND=gloo lets the multi-rank path run with every rank on
    # one GPU (a functional check of this script's N > 1 logic on a 1-GPU
    # box); production runs use NCCL with one GPU per rank
    backend = os.environ.get("GRD_BENCH_BACKEND", "nccl")
    gpu = local_rank if backend == "nccl" else local_rank % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1 and spec.get("sharded_stream"):
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        return run_sharded_stream(args, spec, rank, world, dev, backend)
    need = spec.get("host_gb")
    if need:
        import psutil
        have = psutil.virtual_memory().available / 2**30
        if have < need:
            raise SystemExit(f"workload {args.workload} needs ~{need} GiB of host memory, "
                             f"{have:.0f} GiB available")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    g, ds, plan, model, prep = build_workload(spec)
    L, E = spec["L"], g.num_edges
    if spec.get("tier") == "nvme":
        # the features go to a GRIN feature file on the box's disk and are
        # trained from there (memory-mapped, read with direct I/O)
        import tempfile
        tier_dir = Path(os.environ.get("GRD_TIER_DIR", tempfile.gettempdir())) / f"grd_{args.workload}"
        t0 = time.perf_counter()
        ds.save(tier_dir)
        ds = g2.load_dataset(tier_dir, mmap_features=True)
        prep["tier_file_write_s"] = round(time.perf_counter() - t0, 3)
        os.environ["GRD_ENGINE"] = "stream"
        os.environ["GRD_X_CACHE_GB"] = str(spec["x_cache_gb"])
        os.environ["GRD_HOST_CACHE_GB"] = str(spec["host_cache_gb"])
    # the session partitioned_train itself uses (cached on the plan): the
    # e2e leg below re-binds the same device buffers instead of a second copy
    sess = session_for(ds, plan, model)
    flush = torch.zeros(128 * 1024 * 1024, dtype=torch.float32, device=dev)

    # ---- instrumented epoch: per-kernel CUDA-event timing + launch count --
    sess.run_epoch(0, LR, use_graph=False)
    torch.cuda.synchronize()
    ops.RECORDER.reset()
    ops.RECORDER.timing = True
    flush_l2(flush)
    h2d0 = getattr(sess.engine, "h2d_bytes", 0)
    st0 = getattr(getattr(sess.engine, "x_src", None), "storage_bytes", 0)
    sess.engine.epoch(LR)
    torch.cuda.synchronize()
    stream_bytes = getattr(sess.engine, "h2d_bytes", 0) - h2d0
    storage_bytes = getattr(getattr(sess.engine, "x_src", None), "storage_bytes", 0) - st0
    ops.RECORDER.timing = False
    launches_per_epoch = ops.RECORDER.launches
    per_kernel = {}
    for name, nbytes, flops, s, e in ops.RECORDER.records:
        k = per_kernel.setdefault(name, {"ms": 0.0, "bytes": 0.0, "flops": 0.0, "launches": 0})
        k["ms"] += s.elapsed_time(e)
        k["bytes"] += nbytes
        k["flops"] += flops
        k["launches"] += 1
    ops.RECORDER.reset()

    # ---- timed region: K graph-replayed epochs, L2 flushed between steps --
    for w in range(args.warmup):
        flush_l2(flush)
        sess.run_epoch(w, LR)
    torch.cuda.synchronize()
    clocks = ClockSampler(gpu)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.active = True
    events = []
    for k in range(args.steps):
        flush_l2(flush)
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        sess.run_epoch(args.warmup + k, LR)
        e.record()
        events.append((s, e))
    torch.cuda.synchronize()
    clocks.active = False
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in events]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    loss, acc = sess.read_stats()

    # ---- e2e: public API, host buffers, H2D/D2H inside the timed region --
    if ds.features.dtype == np.float32:
        ds_e2e = ds          # fp32 host array, page-locked in place by the engine
    else:
        f32 = torch.empty(ds.features.shape, dtype=torch.float32).pin_memory()
        f32.numpy()[...] = ds.features
        ds_e2e = g2.LabeledDataset(graph=ds.graph, features=f32.numpy(), labels=ds.labels,
                                   train_mask=ds.train_mask)
    for _ in range(max(1, args.warmup)):
        g2.partitioned_train(ds_e2e, plan, model, epochs=1, lr=LR)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    x0 = getattr(sess.engine, "h2d_bytes", 0)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        trained, trace, _ = g2.partitioned_train(ds_e2e, plan, model, epochs=1, lr=LR)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.steps
    e2e_x_bytes = (getattr(sess.engine, "h2d_bytes", 0) - x0) / args.steps
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = ds.features.size * 4 + ds.labels.size * 4 + ds.train_mask.size + \
        sum(w.size * 4 for w in model.weights)
    streaming = hasattr(sess.engine, "x_src")
    if streaming:   # features: what the engine actually moved per e2e epoch
        h2d += e2e_x_bytes - ds.features.size * 4
    d2h = sum(w.size * 8 * 2 for w in model.weights) + 32

    clock = clocks.summary()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None

    hbm_peak, tf_peak, peak_kind = load_peaks()
    dom = max(per_kernel, key=lambda n: per_kernel[n]["ms"])
    epoch_ms_instr = sum(k["ms"] for k in per_kernel.values())

    traffic = json.loads((ROOT / "profiles" / "traffic.json").read_text()) \
        if (ROOT / "profiles" / "traffic.json").exists() else {}
    tr = traffic.get(args.workload, {})

    def roof(name):
        """HBM roofline of one kernel: DRAM bytes per launch (one ncu capture
        of this workload, profiles/traffic.json) over the live average launch
        time; the SURVEY 8(d) per-edge streaming model (no cache reuse
        credited, so it can exceed the peak when hub rows hit L2) beside it."""
        k = per_kernel[name]
        per_launch_s = k["ms"] * 1e-3 / k["launches"]
        model_gbs = k["bytes"] / k["launches"] / per_launch_s / 1e9
        r = {"kernel": name, "bound": "hbm", "peak": hbm_peak, "unit": "GB/s",
             "peak_source": f"{peak_kind} (MEASURED_PEAKS.json copy bandwidth, burst)",
             "launches_per_epoch": k["launches"], "ms_per_epoch": round(k["ms"], 4),
             "share_of_kernel_time": round(k["ms"] / epoch_ms_instr, 4),
             "share_of_epoch": round(k["ms"] / ms_per_step, 4),
             "algorithmic_bytes_per_launch": int(k["bytes"] / k["launches"]),
             "streaming_model_GBs": round(model_gbs, 1),
             "streaming_model_frac": round(model_gbs / hbm_peak, 4)}
        if name in tr:
            dram = float(tr[name])
            gbs = dram / per_launch_s / 1e9
            r.update(achieved=round(gbs, 1), frac=round(gbs / hbm_peak, 4), traffic=int(dram),
                     frac_nominal_8TBs=round(gbs / 8000.0, 4),
                     basis="ncu dram__bytes_read.sum + dram__bytes_write.sum per launch "
                           f"({tr.get('_source', 'profiles/traffic.json')}) / live launch time")
        else:
            r.update(achieved=round(model_gbs, 1), frac=round(model_gbs / hbm_peak, 4),
                     frac_nominal_8TBs=round(model_gbs / 8000.0, 4),
                     traffic=None, basis="streaming model (no ncu DRAM capture of this workload)")
        return r

    roofline = roof(dom)
    agg_roof = roof("agg_sum") if "agg_sum" in per_kernel else None
    edges_per_epoch = L * E
    # strong scaling: the N ranks together train ONE epoch of the whole graph,
    # so the job processes L*|E| edges per step whatever N is
    value = edges_per_epoch / (ms_per_step * 1e-3)
    out = {
        "metric": "aggregated edges/s (L*|E| per full-graph training epoch)",
        "value": round(value, 1),
        "unit": "edges/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "epoch_s": round(ms_per_step * 1e-3, 7),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (bit-exact reference generator / dataset / partitioner; random-init weights)",
        "config": {
            "workload": args.workload, "desc": spec["desc"], "num_vertices": g.num_vertices,
            "num_edges": E, "layers": L, "hidden": spec["H"], "features": spec["F"],
            "classes": spec["C"], "partitions": spec["P"], "aggregation": spec["mode"],
            "parallelism": "single" if world == 1 else
            f"partition-parallel x{world} (halo all-to-all + grad all-reduce over {backend.upper()})",
            "l2": "flushed (512 MiB write) before every timed step", "lr": LR,
            "preprocess": prep, "loss_last_step": loss, "acc_last_step": acc,
            "storage_read_bytes_per_epoch": storage_bytes if streaming else None,
            "engine": f"streaming: {sess.engine.cache_rows} of {g.num_vertices} feature rows "
                      f"cached in HBM; {sess.engine.x_src.describe()}; {stream_bytes / 1e9:.1f} GB "
                      "over the host link per epoch (inside value; the layer-1 regather streams the "
                      "feature rows into the consumed layer buffer, where the layer-0 backward "
                      "and the next epoch's layer-0 transform read them; e2e re-binds the "
                      "features every call, so it refills the HBM cache and streams twice)" if streaming else
                      "HBM-resident layer-wise (inputs resident before the timed region)",
        },
        "e2e": {"value": round(edges_per_epoch / e2e_s, 1), "unit": "edges/s",
                "s_per_step": round(e2e_s, 6), "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "api": "paper_2605_11517_b200.partitioned_train(..., epochs=1) with pinned host features"},
        "roofline": roofline,
        "agg_roofline": agg_roof,
        "kernels": {n: {"ms_per_epoch": round(k["ms"], 4), "launches": k["launches"],
                        "GB_per_epoch": round(k["bytes"] / 1e9, 4),
                        "GFLOP_per_epoch": round(k["flops"] / 1e9, 4)}
                    for n, k in sorted(per_kernel.items(), key=lambda kv: -kv[1]["ms"])},
        "clocks": clock,
        "gpu_launches": launches_per_epoch * args.steps,
    }
    if world == 1 and not args.no_engines:
        # after the headline measurement, with its buffers released, so the
        # table's own allocations cannot shrink the headline's HBM cache
        del sess
        plan.device_cache.clear()
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        out["engines"] = engine_table()
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(spec)
    if world > 1:
        dist.destroy_process_group()
    return out


def run_sharded_stream(args, spec, rank, world, dev, backend):
    """configs[3] on N ranks: the shard-aware layer-streaming engine.  No
    rank holds the whole feature matrix or the whole partition plan: rank 0
    partitions and broadcasts the labels, every rank generates the graph on
    its GPU, builds its shard from the labels (lean_shard_plan), generates
    its owned feature rows on the device (bit-exact with the dataset's
    PCG64 stream) into page-locked host memory and streams them; halo rows
    of every aggregation's input travel by all-to-all, weight gradients by
    one all-reduce."""
    import torch
    import torch.distributed as dist
    import paper_2605_11517_b200 as g2
    from types import SimpleNamespace
    from paper_2605_11517_b200 import ops
    from paper_2605_11517_b200.dataset import random_feature_rows, random_labels_mask
    from paper_2605_11517_b200.distributed import Communicator, LabelPlan, lean_shard_plan
    from paper_2605_11517_b200.stream import StreamSession
    t0 = time.perf_counter()
    g = g2.generate_kronecker(spec["scale"], spec["deg"], seed=SEED, device=dev)
    torch.cuda.empty_cache()
    t_gen = time.perf_counter() - t0
    n = g.num_vertices
    lab = torch.empty(n, dtype=torch.int32, device=dev if backend == "nccl" else "cpu")
    t1 = time.perf_counter()
    if rank == 0:
        part = g2.switching_aware_partition(g, spec["P"], g2.PartitionerParams(seed=SEED + 2),
                                            device=dev)
        lab.copy_(torch.from_numpy(part.labels.astype(np.int32)))
    dist.broadcast(lab, 0)
    labels = lab.cpu().numpy()
    del lab
    t_part = time.perf_counter() - t1
    t2 = time.perf_counter()
    comm = Communicator()
    lplan = LabelPlan(g, labels, spec["P"])
    shard = lean_shard_plan(g, lplan, rank, world, comm)
    dev_rows = random_feature_rows(spec["F"], SEED + 1, rows=shard.owned, device=dev)
    owned = torch.empty(dev_rows.shape, dtype=torch.float32, pin_memory=True)
    owned.copy_(dev_rows)
    del dev_rows
    torch.cuda.empty_cache()
    labels_all, mask_all = random_labels_mask(n, spec["F"], spec["C"], SEED + 1)
    t_shard = time.perf_counter() - t2
    ds = SimpleNamespace(graph=g, labels=labels_all, train_mask=mask_all, features=None)
    model = g2.create_model(spec["F"], spec["C"], num_layers=spec["L"], hidden_dim=spec["H"],
                            seed=SEED + 3, aggregation_mode=spec["mode"])
    # this rank's HBM: what the other ranks sharing a GPU (gloo checks) leave
    cache = None
    if backend != "nccl":
        free, _ = torch.cuda.mem_get_info(dev)
        cache = max(0, free // world - (4 << 30))
    sess = StreamSession(ds, lplan, model, comm=comm, shard=shard, owned_features=owned,
                         x_cache_bytes=cache)
    eng = sess.engine
    L, E = spec["L"], g.num_edges
    flush = torch.zeros(128 * 1024 * 1024, dtype=torch.float32, device=dev)
    sess.run_epoch(0, LR)
    torch.cuda.synchronize()
    ops.RECORDER.reset()
    ops.RECORDER.timing = True
    flush_l2(flush)
    eng.epoch(LR)
    torch.cuda.synchronize()
    ops.RECORDER.timing = False
    launches = ops.RECORDER.launches
    per_kernel = {}
    for name, nbytes, flops, s0, e0 in ops.RECORDER.records:
        k = per_kernel.setdefault(name, {"ms": 0.0, "bytes": 0.0, "launches": 0})
        k["ms"] += s0.elapsed_time(e0)
        k["bytes"] += nbytes
        k["launches"] += 1
    ops.RECORDER.reset()
    for w in range(args.warmup):
        flush_l2(flush)
        sess.run_epoch(w, LR)
    torch.cuda.synchronize()
    clocks = ClockSampler(torch.cuda.current_device())
    dist.barrier()
    torch.cuda.synchronize()
    clocks.active = True
    events = []
    for k in range(args.steps):
        flush_l2(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sess.run_epoch(args.warmup + k, LR)
        b.record()
        events.append((a, b))
    torch.cuda.synchronize()
    clocks.active = False
    dist.barrier()
    tot = torch.tensor([sum(a.elapsed_time(b) for a, b in events)], device=dev if backend == "nccl" else "cpu")
    dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms = float(tot.item()) / args.steps
    loss, acc = sess.read_stats()
    # e2e: an epoch with the owned features streamed from page-locked host
    # memory inside it plus the trained weights' download, wall clock
    dist.barrier()
    h0 = eng.h2d_bytes
    t0 = time.perf_counter()
    for _ in range(args.steps):
        # features re-bound every step (as partitioned_train does): the HBM
        # cache and the stashed rows are refilled from the host inside it
        eng.set_features(eng.x_src)
        sess.run_epoch(0, LR)
        eng.wts.export(sess.model)
    torch.cuda.synchronize()
    e2e = (time.perf_counter() - t0) / args.steps
    h2d = (eng.h2d_bytes - h0) / args.steps
    et = torch.tensor([e2e], device=dev if backend == "nccl" else "cpu")
    dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e = float(et.item())
    clock = clocks.summary()
    if rank != 0:
        dist.destroy_process_group()
        return None
    hbm_peak, _, peak_kind = load_peaks()
    dom = max(per_kernel, key=lambda k: per_kernel[k]["ms"])
    kd = per_kernel[dom]
    model_gbs = kd["bytes"] / (kd["ms"] * 1e-3) / 1e9
    value = L * E / (ms * 1e-3)
    out = {
        "metric": "aggregated edges/s (L*|E| per full-graph training epoch)",
        "value": round(value, 1), "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "epoch_s": round(ms * 1e-3, 7),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (bit-exact reference generator / dataset / partitioner; random-init "
                "weights; each rank generates its own feature rows)",
        "config": {"workload": args.workload, "desc": spec["desc"], "num_vertices": n,
                   "num_edges": E, "layers": L, "hidden": spec["H"], "features": spec["F"],
                   "classes": spec["C"], "partitions": spec["P"], "aggregation": spec["mode"],
                   "parallelism": f"partition-parallel x{world}, sharded layer-streaming engine "
                                  f"(halo all-to-all + one weight-gradient all-reduce over "
                                  f"{backend.upper()})",
                   "l2": "flushed (512 MiB write) before every timed step", "lr": LR,
                   "preprocess": {"generate_s": round(t_gen, 3), "partition_s": round(t_part, 3),
                                  "shard_and_rows_s": round(t_shard, 3)},
                   "rank0_rows": {"owned": shard.n_own, "halo": int(shard.halo.size),
                                  "hbm_cached_feature_rows": eng.cache_rows},
                   "loss_last_step": loss, "acc_last_step": acc},
        "e2e": {"value": round(L * E / e2e, 1), "unit": "edges/s", "s_per_step": round(e2e, 6),
                "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(sum(w.size * 8 * 2 for w in model.weights)),
                "api": "sharded StreamSession epoch (the engine partitioned_train dispatches to) "
                       "with page-locked host feature rows, weights downloaded every step"},
        "roofline": sharded_roof(args.workload, dom, model_gbs, hbm_peak, peak_kind),
        "kernels": {k: {"ms_per_epoch": round(v["ms"], 3), "launches": v["launches"]}
                    for k, v in per_kernel.items()},
        "clocks": clock, "gpu_launches": launches * args.steps,
    }
    dist.destroy_process_group()
    return out


def sharded_roof(workload, dom, model_gbs, hbm_peak, peak_kind):
    """Roofline of the sharded run's dominant kernel (rank 0).  ncu cannot
    capture a multi-rank command, so the DRAM side is estimated: the
    streaming-model rate times the kernel's DRAM / streaming-model byte
    ratio measured at N = 1 on the same workload (profiles/traffic.json
    over the N = 1 bench line's algorithmic bytes per launch)."""
    r = {"kernel": dom, "bound": "hbm", "peak": hbm_peak, "unit": "GB/s", "peak_source": peak_kind,
         "streaming_model_GBs": round(model_gbs, 1),
         "streaming_model_frac": round(model_gbs / hbm_peak, 4)}
    ratio = None
    try:
        tr = json.loads((ROOT / "profiles" / "traffic.json").read_text()).get(workload, {})
        line = json.loads((ROOT / "profiles" / f"r02_bench_{workload}.json").read_text())
        for key in ("roofline", "agg_roofline"):
            rf = line.get(key) or {}
            if rf.get("kernel") == dom and dom in tr and rf.get("algorithmic_bytes_per_launch"):
                ratio = float(tr[dom]) / float(rf["algorithmic_bytes_per_launch"])
                break
    except (OSError, ValueError):
        ratio = None
    if ratio is None:
        r.update(achieved=round(model_gbs, 1), frac=round(model_gbs / hbm_peak, 4),
                 frac_nominal_8TBs=round(model_gbs / 8000.0, 4), traffic=None,
                 basis="streaming model (rank 0; no ncu capture of the sharded run)")
    else:
        gbs = model_gbs * ratio
        r.update(achieved=round(gbs, 1), frac=round(gbs / hbm_peak, 4),
                 frac_nominal_8TBs=round(gbs / 8000.0, 4), traffic=None, dram_per_model_byte=round(ratio, 4),
                 basis="rank 0's streaming-model rate x the DRAM / model byte ratio ncu measured "
                       "for this kernel at N = 1 (profiles/traffic.json, profiles/r02_bench_"
                       f"{workload}.json)")
    return r


def oracle_sample(spec, key):
    """The bounded CPU sample of the workload, built by the oracle alone
    (oracle/workload.py): the same model on generate_kronecker(scale, deg)
    of the same average degree, or the workload itself when it is small."""
    from oracle import workload
    smp = spec.get(key) or spec.get("cpu_sample") or dict(scale=spec["scale"], deg=spec["deg"])
    s = workload.build(smp["scale"], smp["deg"], spec["F"], spec["C"], spec["L"], spec["H"],
                       spec["P"], mode=spec["mode"], heads=spec.get("heads", 4), seed=SEED)
    whole = smp["scale"] == spec["scale"] and smp["deg"] == spec["deg"]
    what = (f"generate_kronecker({smp['scale']}, {smp['deg']}) ({s.num_vertices} V / "
            f"{s.num_edges} E){' (the whole workload)' if whole else ', same model'}")
    return s, what


def _oracle_name(spec):
    return ("oracle/sage_gat.py (torch float64 CPU, builder-defined layer)"
            if spec["mode"] in ("sage_mean", "gat") else
            "oracle/gcn.py (float64 numpy restatement of the reference's partitioned_train, "
            "pinned to its golden vectors)")


def cpu_baseline(spec):
    from oracle import workload
    s, what = oracle_sample(spec, "cpu_sample")
    secs = workload.epoch_seconds(s, LR)
    return {"value": round(spec["L"] * s.num_edges / secs, 1), "unit": "edges/s",
            "cores": os.cpu_count(), "kind": "port",
            "sample": f"one epoch of {what} in {_oracle_name(spec)}, all host threads "
                      f"(OpenBLAS; numpy gathers / reduceat single-threaded): {secs:.2f} s"}


def run_reference(args, spec, rank, world):
    """The reference arm: the pinned CPU restatement of the reference's
    path on the box's host cores; rank 0 only (the others exit 0)."""
    if rank != 0:
        return None
    from oracle import workload
    s, what = oracle_sample(spec, "ref_sample")
    for _ in range(args.warmup):
        workload.epoch_seconds(s, LR)
    times = [workload.epoch_seconds(s, LR) for _ in range(args.steps)]
    secs = sum(times) / len(times)
    value = spec["L"] * s.num_edges / secs
    return {
        "impl": "reference",
        "metric": "aggregated edges/s (L*|E| per full-graph training epoch)",
        "value": round(value, 1), "unit": "edges/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(secs * 1e3, 3), "epoch_s": round(secs, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (oracle-built: reference generator / dataset / partitioner / plan "
                "restated)",
        "config": {"workload": args.workload, "desc": spec["desc"], "sample": what,
                   "sample_num_edges": s.num_edges, "sample_build_s": round(s.build_s, 2),
                   "implementation": _oracle_name(spec)},
        "cpu_baseline": {"value": round(value, 1), "unit": "edges/s", "cores": os.cpu_count(),
                         "kind": "port", "sample": f"one epoch of {what} per step"},
        "e2e": {"value": round(value, 1), "unit": "edges/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-engines", action="store_true",
                    help="skip the per-engine epoch table (ENGINE_SPEC)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    rank, world, local_rank = rank_info()
    if world > 1 and os.environ.get("OMP_NUM_THREADS") == "1":
        # torchrun pins every rank to one OpenMP thread; the native
        # preprocessing (generator, partitioner, plan) gets its share of cores
        os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or 1) // world))
    spec = WORKLOADS[args.workload]
    if args.impl == "reference":
        out = run_reference(args, spec, rank, world)
    else:
        out = run_ours(args, spec, rank, world, local_rank)
    if out is not None and rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
