#!/bin/bash
# GEMM / weight-gradient shapes of the papers_full epoch: per-launch times
# against their compulsory HBM bytes (default and without the TMA-store
# staging tiles), then one full ncu capture of the chunked forward transform
# and of the 128x128 weight gradient.
mkdir -p gpurun_out
python tools/gemm_shapes.py papers > gpurun_out/gemm_shapes_papers.json 2>&1; echo "shapes rc=$?"
GRD_GEMM_TMA_STORE=0 python tools/gemm_shapes.py papers > gpurun_out/gemm_shapes_papers_notma.json 2>&1; echo "shapes notma rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -s 2 -c 1 \
  -o gpurun_out/ncu_gemm_fwd128 -f python tools/gemm_one.py 1048576 128 128 > gpurun_out/ncu_gemm_fwd128.log 2>&1; echo "ncu fwd rc=$?"
if [ -n "$WGRAD" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -s 5 -c 1 \
  -o gpurun_out/ncu_wgrad128 -f python tools/wgrad_one.py > gpurun_out/ncu_wgrad128.log 2>&1; echo "ncu wgrad rc=$?"
fi
