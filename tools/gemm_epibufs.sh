#!/bin/bash
# GEMM shape timings with one / two TMA-store staging tiles per epilogue warp.
mkdir -p gpurun_out
for w in papers products; do
  for E in 1 2 3; do
    echo "== $w epibufs=$E"
    GRD_GEMM_EPI_BUFS=$E timeout 300 python tools/gemm_shapes.py $w
  done
done > gpurun_out/gemm_epibufs.txt 2>&1
echo "matrix rc=$?"
