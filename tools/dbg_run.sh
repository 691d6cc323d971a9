cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sso.py -q -x 2>&1 | tail -5
for t in 1 0; do echo "TMA_STORE=$t"; GRD_GEMM_TMA_STORE=$t timeout 300 python tools/gemm_shapes.py papers | python -c "import json,sys; d=json.load(sys.stdin); [print(k, v['ms'], v.get('frac')) for k,v in d.items()]"; GRD_GEMM_TMA_STORE=$t timeout 300 python tools/gemm_shapes.py products | python -c "import json,sys; d=json.load(sys.stdin); [print(k, v['ms'], v.get('frac')) for k,v in d.items()]"; done
GRD_TIER_DIR=/tmp timeout 1200 python tools/sso_probe.py 22 16 2 2>&1 | grep -v "^{" | tail -4
timeout 1500 python bench.py --steps 5 --warmup 3 --no-engines --no-cpu-baseline > gpurun_out/bench_pf.json 2>&1; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_pf.json')); print(d['ms_per_step'], d['config']['engine'][:80], {k: v['ms_per_epoch'] for k, v in d['kernels'].items()})"
