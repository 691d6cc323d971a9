"""Phase times of the GPU switching-aware partitioner at a given scale:
python tools/partition_profile.py SCALE DEG P"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2605_11517_b200 as g2
from paper_2605_11517_b200 import partition as pm

scale, deg, P = (int(x) for x in sys.argv[1:4])
g = g2.generate_kronecker(scale, deg, seed=0, device="cuda")
torch.cuda.empty_cache()
acc = {}
orig_rel = pm._relocate_sorted


def timed_rel(*a, **k):
    torch.cuda.synchronize(); t = time.perf_counter()
    orig_rel(*a, **k)
    torch.cuda.synchronize(); acc["relocate"] = acc.get("relocate", 0) + time.perf_counter() - t


pm._relocate_sorted = timed_rel
L = pm._lib.lib()
orig_an, orig_sum = L.grd_sa_analyze, L.grd_sum_sequential


class Wrap:
    def __getattr__(self, n):
        return getattr(L, n)

    def grd_sa_analyze(self, *a):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = orig_an(*a)
        torch.cuda.synchronize(); acc["analyze_kernel"] = acc.get("analyze_kernel", 0) + time.perf_counter() - t
        return r

    def grd_sum_sequential(self, *a):
        t = time.perf_counter()
        r = orig_sum(*a)
        acc["host_sum"] = acc.get("host_sum", 0) + time.perf_counter() - t
        return r


pm._lib.lib = lambda: Wrap()
t0 = time.perf_counter()
res = g2.switching_aware_partition(g, P, g2.PartitionerParams(seed=2), device="cuda")
tot = time.perf_counter() - t0
print({"total_s": round(tot, 2), "iterations": res.iterations, **{k: round(v, 2) for k, v in acc.items()}})
