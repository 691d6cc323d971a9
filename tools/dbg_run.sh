cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
GRD_TIER_DIR=/tmp timeout 1200 python tools/sso_probe.py 22 16 1 2>&1 | grep -v "^{" | tail -4
timeout 300 python tools/gemm_shapes.py papers | python -c "import json,sys; d=json.load(sys.stdin); [print(k, v['ms'], v.get('frac')) for k,v in d.items()]"
