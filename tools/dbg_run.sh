cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
bash tools/sanitize.sh
GRD_TIER_DIR=/tmp timeout 1500 python tools/sso_probe.py 22 16 2 > gpurun_out/sso_probe.log 2>&1; echo "sso rc=$?"
