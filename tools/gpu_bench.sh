#!/bin/bash
# One GPU call: bench line + kernel launch list + ncu full capture of the top kernel.
set -x
W=${WORKLOAD:-config1}
python bench.py --workload $W --steps 20 --warmup 3 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
