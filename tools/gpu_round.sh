#!/bin/bash
# One GPU-box pass: -m gpu tests, the default bench line, the per-op DRAM
# traffic capture of the default workload, and the reference arm.
W=${W:-papers_full}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total --format=csv > gpurun_out/smi.txt; free -g >> gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/pytest.log
fi
timeout 1800 python bench.py --workload $W --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench_$W.err
if [ -z "$SKIP_NCU" ]; then
  GRD_NVTX=1 timeout 1500 ncu --nvtx --print-nvtx-rename kernel --profile-from-start off \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/dram_$W.csv python tools/profile_epoch.py $W > gpurun_out/ncu_dram_$W.log 2>&1
  echo "ncu rc=$?"
  # merge into the committed table (other workloads' entries stay)
  [ -f gpurun_out/traffic.json ] || cp profiles/traffic.json gpurun_out/traffic.json
  python tools/dram_traffic.py gpurun_out/dram_$W.csv $W gpurun_out/traffic.json
fi
if [ -z "$SKIP_REF" ]; then
  timeout 900 python bench.py --impl reference --workload $W --steps 20 --warmup 5 > gpurun_out/ref_$W.json 2> gpurun_out/ref_$W.err; echo "ref rc=$?"
fi
