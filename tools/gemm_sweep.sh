for bn in 256 128; do echo "BN_MAX=$bn"; GRD_GEMM_BN_MAX=$bn timeout 120 python tools/bench_kernels.py; done
