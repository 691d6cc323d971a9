cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; exec > gpurun_out/dbg.log 2>&1
for kc in 200 160 100; do
  GRD_GEMM_KCHUNK=$kc timeout 300 python tools/prec_matrix.py sage 2>&1 | tail -1
done
