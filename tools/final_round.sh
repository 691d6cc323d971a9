#!/bin/bash
# Round-end pass on one B200: every -m gpu test, smoke(), the default bench
# line (papers_full) with its per-op DRAM capture and the reference arm, and
# the ncu launch list of the default bench command.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_final.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"
SKIP_TESTS=1 bash tools/gpu_round.sh
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_papers_full.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-engines \
  > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
python tools/summarize_launches.py gpurun_out/launches_papers_full.csv gpurun_out/launches_papers_full.json \
  > gpurun_out/launches_papers_full.txt 2>&1; head -12 gpurun_out/launches_papers_full.txt
