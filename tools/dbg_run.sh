cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
GRD_TIER_DIR=/tmp timeout 1200 python tools/sso_probe.py 22 16 2 > gpurun_out/sso_probe.log 2>&1; echo "sso rc=$?"; grep -v "^{" gpurun_out/sso_probe.log | tail -3
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_papers_full.json 2> gpurun_out/bench_papers_full.err; echo "bench rc=$?"
timeout 900 python bench.py --workload products_sage --steps 20 --warmup 5 --no-engines > gpurun_out/bench_products_sage.json 2>&1; echo "products rc=$?"
