#!/bin/bash
# GEMM / wgrad kernel tests and the default bench under each cluster size.
mkdir -p gpurun_out
for c in 1 2 4; do
  GRD_GEMM_CLUSTER=$c timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm or wgrad" > gpurun_out/gemm_c$c.txt 2>&1
  echo "cluster $c rc=$?" >> gpurun_out/gemm_c$c.txt
  GRD_GEMM_CLUSTER=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
done
