cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15
