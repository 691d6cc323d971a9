#!/bin/bash
# Per-op DRAM traffic (ncu, NVTX-attributed) of every bench workload, merged
# into gpurun_out/traffic.json, then each workload's bench line re-measured
# so its roofline divides those bytes by the live per-call time.
mkdir -p gpurun_out
cp profiles/traffic.json gpurun_out/traffic.json
for W in ${WORKLOADS:-products_sage products_gat papers_gcn config1}; do
  GRD_NVTX=1 timeout 900 ncu --nvtx --print-nvtx-rename kernel --profile-from-start off \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/dram_$W.csv python tools/profile_epoch.py $W > gpurun_out/ncu_dram_$W.log 2>&1
  echo "ncu $W rc=$?"
  python tools/dram_traffic.py gpurun_out/dram_$W.csv $W gpurun_out/traffic.json > gpurun_out/dram_$W.txt
done
cp gpurun_out/traffic.json profiles/traffic.json
for W in ${WORKLOADS:-products_sage products_gat papers_gcn config1}; do
  timeout 900 python bench.py --workload $W --steps 20 --warmup 5 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
  echo "bench $W rc=$?"
done
