cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_papers_full.json 2> gpurun_out/bench_papers_full.err; echo "papers rc=$?"
timeout 900 python bench.py --workload products_sage --steps 20 --warmup 5 --no-engines > gpurun_out/bench_products_sage.json 2> gpurun_out/bench_products_sage.err; echo "products rc=$?"
GRD_GEMM_KCHUNK=0 timeout 900 python bench.py --workload products_sage --steps 20 --warmup 5 --no-engines --no-cpu-baseline > gpurun_out/bench_products_sage_nochunk.json 2>&1; echo "products nochunk rc=$?"
timeout 300 python tools/gemm_shapes.py products
