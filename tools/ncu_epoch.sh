#!/bin/bash
# ncu --set full capture of one products_sage epoch (current kernels) plus the
# launch list of the bench command; exports raw CSV for tools/ncu_summary.py.
W=${1:-products_sage}
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o gpurun_out/epoch_$W -f python tools/profile_epoch.py $W > gpurun_out/ncu_epoch_$W.log 2>&1
ncu -i gpurun_out/epoch_$W.ncu-rep --page raw --csv > gpurun_out/epoch_$W.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline \
    > /dev/null 2>&1
ls -la gpurun_out/
