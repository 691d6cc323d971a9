"""One eager training epoch of a bench workload inside cudaProfilerStart/Stop,
for `ncu --profile-from-start off --set full` (per-kernel DRAM traffic of the
epoch the bench times).  Usage: python tools/profile_epoch.py [workload]"""
import sys
sys.path.insert(0, '.')
import torch
import bench
from paper_2605_11517_b200.training import session_for
name = sys.argv[1] if len(sys.argv) > 1 else bench.DEFAULT_WORKLOAD
g, ds, plan, model, _ = bench.build_workload(bench.WORKLOADS[name])
sess = session_for(ds, plan, model)
sess.run_epoch(0, bench.LR, use_graph=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
sess.engine.epoch(bench.LR)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", name)
