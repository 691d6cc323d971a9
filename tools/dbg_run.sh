cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_models.py tests/test_gpu_sso.py tests/test_gpu_training.py -q -x 2>&1 | tail -3
for d in 4 6 8 3; do GRD_AGG_ASYNC_DEPTH=$d timeout 300 python tools/agg_papers.py 25 2>&1 | tail -1; done
GRD_AGG_ASYNC=0 timeout 300 python tools/agg_papers.py 25 2>&1 | tail -1
