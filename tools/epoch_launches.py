"""Per-launch CUDA-event times of one instrumented epoch of a bench workload
(the bench's own RECORDER): name, algorithmic bytes, ms, GB/s per launch."""
import sys
sys.path.insert(0, '.')
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_11517_b200 import ops  # noqa: E402
from paper_2605_11517_b200.training import session_for  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else bench.DEFAULT_WORKLOAD
g, ds, plan, model, _ = bench.build_workload(bench.WORKLOADS[name])
sess = session_for(ds, plan, model)
flush = torch.zeros(128 * 1024 * 1024, device="cuda")
for _ in range(2):
    sess.run_epoch(0, bench.LR, use_graph=False)
torch.cuda.synchronize()
ops.RECORDER.reset()
ops.RECORDER.timing = True
flush.add_(1.0)
sess.engine.epoch(bench.LR)
torch.cuda.synchronize()
tot = 0.0
for i, (k, nbytes, flops, s, e) in enumerate(ops.RECORDER.records):
    ms = s.elapsed_time(e)
    tot += ms
    print(f"{i:3d} {k:16s} {nbytes / 1e9:8.3f} GB {ms:8.3f} ms {nbytes / ms / 1e6:8.1f} GB/s {flops / ms / 1e9:8.1f} TF/s")
print(f"total {tot:.3f} ms")
