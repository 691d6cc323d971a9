#!/bin/bash
# ncu --set full of one 128-wide aggregation launch of the streaming engine
# (the headline's dominant kernel) on the papers-shaped graph at 1/4 size
# (generate_kronecker(25, 14), GRD_ENGINE=stream), plus its raw CSV export.
mkdir -p gpurun_out
GRD_ENGINE=stream timeout 1500 ncu --set full --clock-control none --import-source on \
    --profile-from-start off -k regex:agg_async --launch-skip 20 --launch-count 1 \
    -o gpurun_out/agg_papers -f python tools/profile_epoch.py papers_gcn > gpurun_out/ncu_agg.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/agg_papers.ncu-rep --page raw --csv > gpurun_out/agg_papers_raw.csv 2>/dev/null
ncu -i gpurun_out/agg_papers.ncu-rep --page details --csv > gpurun_out/agg_papers_details.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:gemm_tf32x3 --launch-skip 3 --launch-count 1 \
    -o gpurun_out/gemm_papers -f python tools/gemm_one.py 1048576 128 128 > gpurun_out/ncu_gemm.log 2>&1
echo "ncu gemm rc=$?"
ncu -i gpurun_out/gemm_papers.ncu-rep --page details --csv > gpurun_out/gemm_papers_details.csv 2>/dev/null
