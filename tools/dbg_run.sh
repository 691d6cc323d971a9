cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_models.py tests/test_gpu_golden_scale.py -q -x 2>&1 | tail -3
timeout 300 python tools/prec_matrix.py sage 2>&1 | tail -1
timeout 1800 python bench.py --steps 20 --warmup 5 --no-engines --no-cpu-baseline > gpurun_out/bench_papers_full.json 2> gpurun_out/bench_papers_full.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_papers_full.json')); print(d['ms_per_step'], {k: v['ms_per_epoch'] for k, v in d['kernels'].items()})"
bash tools/ncu_agg.sh
