cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -3
timeout 300 python tools/gemm_prec_shapes.py 2>&1 | grep -E "16384"
timeout 300 python tools/prec_matrix.py sage 2>&1 | tail -1
timeout 300 python tools/prec_matrix.py papers 2>&1 | tail -1
timeout 300 python tools/gemm_shapes.py products | python -c "import json,sys; d=json.load(sys.stdin); [print(k, v['ms'], v.get('frac')) for k,v in d.items()]"
timeout 900 python bench.py --workload products_sage --steps 10 --warmup 3 --no-engines --no-cpu-baseline > gpurun_out/bench_ps.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/bench_ps.json')); print('products', d['ms_per_step'], {k: v['ms_per_epoch'] for k, v in d['kernels'].items()})"
