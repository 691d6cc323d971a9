#!/bin/bash
# default bench under each GEMM N-tile cap (stages follow from shared memory)
mkdir -p gpurun_out
for bn in 256 128 64; do
  for c in 1 2; do
    GRD_GEMM_CLUSTER=$c GRD_GEMM_BN_MAX=$bn timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_bn${bn}_c$c.json 2> gpurun_out/bench_bn${bn}_c$c.err
  done
done
