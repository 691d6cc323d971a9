"""Host-tier (SSO) epoch probe at a papers-shaped scale: trainer set-up time,
epoch wall time, host-gather time, H2D/D2H bytes.
Usage: python tools/sso_probe.py SCALE PARTITIONS"""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2605_11517_b200.hierarchy import HierarchyConfig, TierSession
from paper_2605_11517_b200.sso import OffloadedTrainer
from paper_2605_11517_b200.model import copy_model
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
P = int(sys.argv[2]) if len(sys.argv) > 2 else 16
spec = dict(bench.WORKLOADS["papers_gcn"], scale=scale, P=P)
t0 = time.perf_counter()
g, ds, plan, model, prep = bench.build_workload(spec)
print("prep", prep, "build", round(time.perf_counter() - t0, 1), "V", g.num_vertices, "E", g.num_edges, flush=True)
cfg = HierarchyConfig(gpu_capacity=64 << 30, host_capacity=180 << 30, bytes_per_value=4)
sess = TierSession(plan, model.dims, "GRINNDER", cfg, aggregation_mode=model.aggregation_mode)
t0 = time.perf_counter()
tr = OffloadedTrainer(ds, plan, copy_model(model), sess, torch.device("cuda"))
torch.cuda.synchronize()
print("trainer init s", round(time.perf_counter() - t0, 2), flush=True)
order = lambda l, ph: list(sess.partition_order(l, ph))
for ep in range(3):
    h0, d0 = tr.bytes_h2d, tr.bytes_d2h
    torch.cuda.synchronize(); t0 = time.perf_counter()
    tr.epoch(ep, 0.01, order)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    L, E = model.num_layers, g.num_edges
    print(f"epoch {ep}: {dt:.3f} s  edges/s {L*E/dt/1e9:.3f} G  "
          f"H2D {(tr.bytes_h2d-h0)/1e9:.2f} GB  D2H {(tr.bytes_d2h-d0)/1e9:.2f} GB  loss {tr.read_stats()[0]:.5f}",
          flush=True)
