cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sso.py tests/test_gpu_kernels.py -q -x 2>&1 | tail -3
timeout 300 python tools/debug_widths.py . sage_mean GRD_GEMM_PREC=bf16x3 2>&1 | tail -4
GRD_TIER_DIR=/tmp timeout 1200 python tools/sso_probe.py 22 16 2 > gpurun_out/sso_probe.log 2>&1; echo "sso rc=$?"; grep -v "^{" gpurun_out/sso_probe.log | cut -c1-400
