// Internal launcher of the tcgen05 3xTF32 GEMM (grd_gemm_tc.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

struct GrdTcGemm {
    int64_t m, n, k;
    const float* a; int64_t lda; int trans_a;   // A stored M x K, or K x M if trans_a
    const float* b; int64_t ldb; int trans_b;   // B stored K x N, or N x K if trans_b
    float* c; int64_t ldc;
    const float* row_scale;
    const float* elem_mul; int64_t ld_elem_mul;
    const float* relu_ref; int64_t ld_relu_ref;
    int relu_out;
    int accumulate;
    int k_splits;        // > 1: split-K, partial tiles to `partial` ([splits][m][round_up(n,4)])
    int64_t k_chunk;     // multiple of 32
    float* partial;
    const float* b_packed;   // opB pre-split by grd_tc_pack_b (then b/ldb/trans_b unused)
    int bf16;                // bf16x3 split (row-major A, packed B); else 3xTF32
    float* c2; int64_t ldc2; // columns >= split (> 0) go to c2 (plain stores only)
    int64_t split;
};

cudaError_t grd_tc_gemm(const GrdTcGemm& g, cudaStream_t st);
// elements needed to pack opB (n x k) into hi/lo tensor-core tiles
int64_t grd_tc_pack_elems(int64_t n, int64_t k);
cudaError_t grd_tc_pack_b(const float* b, int64_t ldb, int trans_b, int64_t n, int64_t k, float* out,
                          cudaStream_t st, int bf16);
// 1 when forward / input-gradient GEMMs use the bf16x3 split (GRD_GEMM_PREC)
int grd_tc_bf16x3();
