#!/bin/bash
# compute-sanitizer passes over the kernel-level GPU tests (small shapes):
# memcheck on every kernel family, racecheck / synccheck on the aggregation
# (heavy-row ticket combine) and GAT kernels.  Logs to gpurun_out/.
mkdir -p gpurun_out
CS=compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?"
timeout 1500 $CS --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "agg_sum or gat" > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?"
timeout 1500 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "agg_sum or gat" > gpurun_out/sanitize_synccheck.log 2>&1; echo "synccheck rc=$?"
