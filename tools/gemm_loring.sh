#!/bin/bash
# GEMM shape timings of the papers / products epochs for every lo-ring depth
# (GRD_GEMM_LORING) with and without the TMA-store epilogue.
mkdir -p gpurun_out
for w in papers products; do
  for L in 0 1 2 3; do
    for T in 1 0; do
      echo "== $w loring=$L tma=$T"
      GRD_GEMM_LORING=$L GRD_GEMM_TMA_STORE=$T timeout 300 python tools/gemm_shapes.py $w
    done
  done
done > gpurun_out/gemm_loring.txt 2>&1
echo "matrix rc=$?"
