#!/bin/bash
# Every bench workload once (round-end refresh of profiles/r01_bench_*.json).
mkdir -p gpurun_out
for W in config1 products_gat papers_gcn igb_nvme papers_full; do
  S=5; [ "$W" = papers_full ] && S=3; [ "$W" = igb_nvme ] && S=3
  timeout 1500 python bench.py --workload $W --steps $S --warmup 3 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
  echo "$W rc=$?"
  python - "$W" <<'PY'
import json, sys
w = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/bench_{w}.json"))
    print(w, d["ms_per_step"], "ms", d["value"], "edges/s e2e", d["e2e"]["value"], d["config"]["preprocess"])
except Exception as e:
    print(w, "failed", e)
PY
done
