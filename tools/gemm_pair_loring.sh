#!/bin/bash
# Papers / products GEMM shapes: CTA pairs (GRD_GEMM_PAIR 1 / 2) x lo-ring depth.
mkdir -p gpurun_out
for w in papers products; do
  for P in 1 2; do
    for L in 0 1 2 3; do
      echo "== $w pair=$P loring=$L"
      GRD_GEMM_PAIR=$P GRD_GEMM_LORING=$L timeout 300 python tools/gemm_shapes.py $w
    done
  done
done > gpurun_out/gemm_pair_loring.txt 2>&1
echo "matrix rc=$?"
