// Switching-aware partitioner, device analysis pass (partition.py:140-200;
// the host version is Analyzer::run in grd_host.cpp).
//
// One warp per vertex, grid-stride over vertices.  The warp counts its
// out-neighbours' partitions in a per-warp shared-memory histogram (the
// neighbour labels are read straight through dst_idx, so no per-iteration
// dst_part array is materialised), lane 0 evaluates the vertex's f64
// objective term with the host's operation order ((1 + share) - penalty,
// IEEE division), and the warp picks the top-`depth` partitions by (count
// desc, id asc) with one shuffle argmax per slot.  The f64 objective itself
// is summed sequentially in vertex order on the host (grd_sum_sequential),
// which is what keeps the convergence decisions bit-identical to the
// reference's numba loop.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/grinder_b200.h"
#include "grd_common.h"

using namespace grd;

namespace {

constexpr int kWarps = 8;               // warps per block
constexpr int kMaxParts = 1024;         // per-warp histogram capacity

__global__ void __launch_bounds__(kWarps * 32)
sa_analyze_kernel(int64_t n, const int64_t* __restrict__ src_ptr, const int32_t* __restrict__ dst_idx,
                  const int32_t* __restrict__ labels, const int64_t* __restrict__ sizes, int32_t p,
                  int32_t depth, double denom, double* __restrict__ terms, int32_t* __restrict__ prefs,
                  unsigned long long* __restrict__ num_candidates) {
    extern __shared__ int32_t hist_all[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    int32_t* hist = hist_all + warp * p;
    const int64_t warps_total = int64_t(gridDim.x) * kWarps;
    unsigned long long cand = 0;
    for (int64_t v = int64_t(blockIdx.x) * kWarps + warp; v < n; v += warps_total) {
        for (int c = lane; c < p; c += 32) hist[c] = 0;
        __syncwarp();
        const int64_t b = src_ptr[v], e = src_ptr[v + 1];
        for (int64_t j = b + lane; j < e; j += 32) atomicAdd(&hist[labels[dst_idx[j]]], 1);
        __syncwarp();
        const int32_t own = labels[v];
        const int64_t deg = e - b;
        if (lane == 0) {
            const double penalty = static_cast<double>(sizes[own]) / denom;
            if (deg > 0) {
                const double share = static_cast<double>(hist[own]) / static_cast<double>(deg);
                terms[v] = __dadd_rn(__dadd_rn(1.0, share), -penalty);
            } else {
                terms[v] = __dadd_rn(1.0, -penalty);
            }
        }
        // top `depth` partitions by (count desc, id asc) among the touched ones
        int32_t prev_count = 0x7fffffff, prev_id = -1;
        int32_t first = p;
        int32_t s = 0;
        for (; s < depth; ++s) {
            int32_t best = p, best_count = 0;
            for (int c = lane; c < p; c += 32) {
                const int32_t cc = hist[c];
                if (cc == 0) continue;
                if (cc > prev_count || (cc == prev_count && c <= prev_id)) continue;
                if (best == p || cc > best_count || (cc == best_count && c < best)) {
                    best = c;
                    best_count = cc;
                }
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                const int32_t ob = __shfl_xor_sync(0xffffffffu, best, off);
                const int32_t oc = __shfl_xor_sync(0xffffffffu, best_count, off);
                if (ob != p && (best == p || oc > best_count || (oc == best_count && ob < best))) {
                    best = ob;
                    best_count = oc;
                }
            }
            if (best == p) break;
            if (s == 0) first = best;
            if (lane == 0) prefs[int64_t(s) * n + v] = best;
            prev_count = best_count;
            prev_id = best;
        }
        // a vertex whose favourite is its own partition is not a candidate:
        // every slot carries the sentinel p (as do unused slots)
        const bool candidate = first != p && first != own;
        if (lane == 0) {
            const int32_t from = candidate ? s : 0;
            for (int32_t t = from; t < depth; ++t) prefs[int64_t(t) * n + v] = p;
            cand += candidate ? 1ull : 0ull;
        }
        __syncwarp();
    }
    if (lane == 0 && cand) atomicAdd(num_candidates, cand);
}

}  // namespace

extern "C" int grd_sa_analyze(int64_t num_vertices, const int64_t* src_ptr, const int32_t* dst_idx,
                              const int32_t* labels, const int64_t* sizes, int32_t num_partitions,
                              int32_t group_depth, double denom, double* terms, int32_t* prefs,
                              unsigned long long* num_candidates, void* stream) {
    clear_error();
    if (num_partitions < 2 || num_partitions > kMaxParts)
        return fail(kErrArg, "sa_analyze: num_partitions must be in [2, %d]", kMaxParts);
    if (group_depth < 1) return fail(kErrArg, "sa_analyze: group_depth must be >= 1");
    if (num_vertices <= 0) return 0;
    if (!src_ptr || !dst_idx || !labels || !sizes || !terms || !prefs || !num_candidates)
        return fail(kErrArg, "sa_analyze: null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int sms = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = size_t(kWarps) * num_partitions * sizeof(int32_t);
    const int64_t want = (num_vertices + kWarps - 1) / kWarps;
    const int grid = static_cast<int>(want < int64_t(sms) * 16 ? want : int64_t(sms) * 16);
    sa_analyze_kernel<<<grid, kWarps * 32, smem, st>>>(num_vertices, src_ptr, dst_idx, labels, sizes,
                                                      num_partitions, group_depth, denom, terms, prefs,
                                                      num_candidates);
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return fail(static_cast<int>(err), "sa_analyze: %s", cudaGetErrorString(err));
    return 0;
}
