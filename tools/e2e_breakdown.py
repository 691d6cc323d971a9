"""Where the end-to-end partitioned_train call spends its time beyond the
device epoch (products workload): session reset (H2D of features, labels,
mask, weights), the epoch, the export of weights / gradients."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_11517_b200 as g2  # noqa: E402
from paper_2605_11517_b200.training import session_for  # noqa: E402

spec = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else bench.DEFAULT_WORKLOAD]
g, ds, plan, model, _ = bench.build_workload(spec)
f32 = torch.empty(ds.features.shape, dtype=torch.float32).pin_memory()
f32.numpy()[...] = ds.features
ds = g2.LabeledDataset(graph=ds.graph, features=f32.numpy(), labels=ds.labels, train_mask=ds.train_mask)
for _ in range(3):
    g2.partitioned_train(ds, plan, model, epochs=1, lr=0.01)
torch.cuda.synchronize()


def t(fn, reps=5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


sess = session_for(ds, plan, model)
print("full partitioned_train  %.2f ms" % t(lambda: g2.partitioned_train(ds, plan, model, epochs=1, lr=0.01)))
print("session_for (reset)     %.2f ms" % t(lambda: session_for(ds, plan, model)))
print("  upload_features       %.2f ms" % t(lambda: sess.upload_features(ds)))
eng = sess.engine
print("  labels+mask copy      %.2f ms" % t(lambda: (
    eng.labels.copy_(torch.from_numpy(np.asarray(ds.labels, dtype=np.int32))),
    eng.mask.copy_(torch.from_numpy(np.asarray(ds.train_mask, dtype=np.uint8))))))
print("run_epoch (graph)       %.2f ms" % t(lambda: sess.run_epoch(0, 0.01)))
print("read_stats              %.2f ms" % t(lambda: sess.read_stats()))
print("export weights          %.2f ms" % t(lambda: eng.wts.export(sess.model)))
