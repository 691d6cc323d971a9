cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
timeout 300 python tools/debug_widths.py . sage_mean 2>&1 | tail -4
timeout 300 python tools/debug_widths.py . gat 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
