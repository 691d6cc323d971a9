cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sso.py tests/test_gpu_kernels.py -q -x 2>&1 | tail -3
timeout 300 python tools/debug_widths.py . sage_mean GRD_GEMM_PREC=bf16x3 2>&1 | tail -4
