// sm_100a device kernels of the partition-wise GCN training step and their
// extern "C" launchers (include/grinder_b200.h).
//
//   K1  gather_rows        training.py:301,330   acts[layer][gather_map]
//   K2  agg_sum            training.py:38-65     neighbour sum + self, normalise
//   K8  agg_sum (pull)     training.py:130-143   transposed aggregation
//   K9  scatter_add_rows   training.py:166-175   global_grad[gather_map] += grad_GA
//   K3/K6/K7 gemm          training.py:76,128-129 dense transform / dgrad
//   K6  wgrad_sgd          training.py:128,343,352-354 split-K dW + SGD
//   K4  softmax_xent       model.py:102-129      masked softmax-CE + accuracy
//
// Every reduction runs in a fixed order (no float atomics), so results are
// bitwise reproducible and independent of partition schedule.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "../../include/grinder_b200.h"
#include "grd_common.h"
#include "grd_gemm_tc.h"

using namespace grd;

namespace {

constexpr int kWarp = 32;
constexpr int kMaxAggChunks = 16;   // heavy_counter holds n_heavy x 16 slots

inline int launch_status(const char* what) {
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return fail(static_cast<int>(err), "%s: %s", what, cudaGetErrorString(err));
    return 0;
}

__device__ __forceinline__ float4 f4_fma(float s, const float4 v, float4 a) {
    a.x = fmaf(s, v.x, a.x);
    a.y = fmaf(s, v.y, a.y);
    a.z = fmaf(s, v.z, a.z);
    a.w = fmaf(s, v.w, a.w);
    return a;
}
__device__ __forceinline__ float4 f4_add(float4 a, const float4 b) {
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    return a;
}
__device__ __forceinline__ float4 f4_shfl_xor(float4 v, int off) {
    v.x = __shfl_xor_sync(0xffffffffu, v.x, off);
    v.y = __shfl_xor_sync(0xffffffffu, v.y, off);
    v.z = __shfl_xor_sync(0xffffffffu, v.z, off);
    v.w = __shfl_xor_sync(0xffffffffu, v.w, off);
    return v;
}
__device__ __forceinline__ float4 ld_nc_f4(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
}

// ------------------------------------------------------------------- K2 --
// The warp is split into NG = 32/LPR lane groups of LPR lanes; each lane of a
// group holds NV float4 column chunks of a row (width <= 4*LPR*NV).
//  * light rows (degree <= heavy_threshold): one row per lane GROUP, so a
//    warp keeps NG rows in flight; each group walks its own edge list with
//    U row loads issued before they are summed (sequential per row).
//  * heavy-row segments: one segment per WARP, the NG groups splitting its
//    edges, combined by a fixed-order butterfly; the last segment of a row
//    to finish sums the segment partials in segment order (deterministic).
template <int LPR, int NV>
__device__ __forceinline__ void load_row(const float* row, int sub, int w4, float4 (&v)[NV]) {
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        const int q = sub + c * LPR;
        v[c] = q < w4 ? ld_nc_f4(row + 4 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// acc += sum over edges e = beg + first, beg + first + stride, ... < end
// Edge weight of chunk c: per-source scale, or (WE) the per-edge per-head
// weight edge_w[e, head(c)] (GAT attention), e optionally permuted.
template <int NV, bool WE>
__device__ __forceinline__ void edge_weights(const grd_agg_args& a, int64_t e, int32_t j,
                                             const int (&hd)[NV], float (&w)[NV]) {
    if constexpr (WE) {
        const int64_t eid = a.edge_w_perm ? a.edge_w_perm[e] : e;
        const float* we = a.edge_w + eid * a.heads;
#pragma unroll
        for (int c = 0; c < NV; ++c) w[c] = __ldg(we + hd[c]);
    } else {
        const float s = a.src_scale ? __ldg(a.src_scale + j) : 1.0f;
#pragma unroll
        for (int c = 0; c < NV; ++c) w[c] = s;
    }
}

template <int LPR, int NV, int U, bool WE>
__device__ __forceinline__ void agg_edges(const grd_agg_args& a, int64_t beg, int64_t end, int stride,
                                          int sub, int w4, const int (&hd)[NV], float4 (&acc)[NV]) {
    const float* __restrict__ y = a.y;
    const int32_t* __restrict__ idx = a.idx;
    int64_t e = beg;
    for (; e + int64_t(U - 1) * stride < end; e += int64_t(U) * stride) {
        int32_t j[U];
#pragma unroll
        for (int u = 0; u < U; ++u) j[u] = __ldg(idx + e + int64_t(u) * stride);
        float4 v[U][NV];
        float s[U][NV];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            edge_weights<NV, WE>(a, e + int64_t(u) * stride, j[u], hd, s[u]);
            load_row<LPR, NV>(y + int64_t(j[u]) * a.ldy, sub, w4, v[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int c = 0; c < NV; ++c) acc[c] = f4_fma(s[u][c], v[u][c], acc[c]);
    }
    for (; e < end; e += stride) {
        const int32_t jj = __ldg(idx + e);
        float s[NV];
        edge_weights<NV, WE>(a, e, jj, hd, s);
        float4 v[NV];
        load_row<LPR, NV>(y + int64_t(jj) * a.ldy, sub, w4, v);
#pragma unroll
        for (int c = 0; c < NV; ++c) acc[c] = f4_fma(s[c], v[c], acc[c]);
    }
}

// self term, post-scale, activation, mask, store — by the LPR lanes of a group
template <int LPR, int NV, bool WE>
__device__ __forceinline__ void agg_finish(const grd_agg_args& a, int64_t r, int64_t deg, int sub,
                                           int w4, const int (&hd)[NV], float4 (&acc)[NV],
                                           bool add_self = true) {
    const int32_t orow = a.out_idx ? a.out_idx[r] : static_cast<int32_t>(r);
    const int32_t srow = (a.no_self || !add_self) ? -1 : (a.self_idx ? a.self_idx[r] : orow);
    if (srow >= 0) {
        float s[NV];
        if constexpr (WE) {
#pragma unroll
            for (int c = 0; c < NV; ++c) s[c] = a.self_w[int64_t(orow) * a.heads + hd[c]];
        } else {
            const float sc = a.src_scale ? a.src_scale[srow] : 1.0f;
#pragma unroll
            for (int c = 0; c < NV; ++c) s[c] = sc;
        }
        float4 v[NV];
        load_row<LPR, NV>(a.y + int64_t(srow) * a.ldy, sub, w4, v);
#pragma unroll
        for (int c = 0; c < NV; ++c) acc[c] = f4_fma(s[c], v[c], acc[c]);
    }
    const float div = static_cast<float>(a.post_div_deg == 2 ? deg : deg + 1);
    const bool do_div = a.post_div_deg == 1 || (a.post_div_deg == 2 && deg > 0);
    const float ps = a.post_scale ? a.post_scale[orow] : 1.0f;
    float* out = a.out + int64_t(orow) * a.ldo;
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        const int q = sub + c * LPR;
        if (q >= w4) continue;
        float4 v = acc[c];
        if (do_div) { v.x /= div; v.y /= div; v.z /= div; v.w /= div; }
        if (a.post_scale) { v.x *= ps; v.y *= ps; v.z *= ps; v.w *= ps; }
        if (a.add_y) v = f4_add(v, ld_nc_f4(a.add_y + int64_t(orow) * a.ld_add_y + 4 * q));
        if (a.relu) {
            v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f);
            v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
        }
        if (a.mask_ref) {
            const float4 m = ld_nc_f4(a.mask_ref + int64_t(orow) * a.ld_mask_ref + 4 * q);
            if (!(m.x > 0.f)) v.x = 0.f;
            if (!(m.y > 0.f)) v.y = 0.f;
            if (!(m.z > 0.f)) v.z = 0.f;
            if (!(m.w > 0.f)) v.w = 0.f;
        }
        *reinterpret_cast<float4*>(out + 4 * q) = v;
    }
}

// A heavy-row segment's partial (held by lanes < LPR) goes to seg_partial;
// the last segment of the row to arrive sums the partials in segment order
// and finishes the row (deterministic).
template <int LPR, int NV, bool WE>
__device__ __forceinline__ void heavy_tail(const grd_agg_args& a, int64_t s, int lane, int sub, int w4, int ldp,
                                           const int (&hd)[NV], float4 (&acc)[NV]) {
    const int32_t h = a.seg_heavy[s];
    const int64_t r = a.heavy_rows[h];
    const int64_t seg0 = a.heavy_seg_ptr[h], nseg = a.heavy_seg_ptr[h + 1] - seg0;
    const int64_t rb = a.row_ptr[r], re = a.row_ptr[r + 1];
    if (lane < LPR) {
        float* part = a.seg_partial + s * ldp;
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            const int q = sub + c * LPR;
            if (q < w4) __stcg(reinterpret_cast<float4*>(part + 4 * q), acc[c]);
        }
    }
    __threadfence();
    __syncwarp();
    int ticket = 0;
    if (lane == 0) ticket = atomicAdd(a.heavy_counter + h, 1);
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
    if (ticket != nseg - 1) return;
    // Last segment to finish: combine partials in segment order.
    __threadfence();
    if (lane >= LPR) return;
#pragma unroll
    for (int c = 0; c < NV; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t t = 0; t < nseg; ++t) {
        const float* part = a.seg_partial + (seg0 + t) * ldp;
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            const int q = sub + c * LPR;
            if (q < w4) acc[c] = f4_add(acc[c], __ldcg(reinterpret_cast<const float4*>(part + 4 * q)));
        }
    }
    agg_finish<LPR, NV, WE>(a, r, re - rb, sub, w4, hd, acc);
    if (lane == 0) a.heavy_counter[h] = 0;
}

// Column chunking: blockIdx.y selects a chunk of `chunk_cols` columns.  Blocks
// run chunk-major, so at any time the SMs gather one column slice of the rows
// of the partitions currently in flight, which keeps that slice of the
// gathered set L2-resident (the partition order of the rows is the locality).
template <int LPR, int NV, int U, bool WE>
__global__ void __launch_bounds__(256, (WE && LPR == 32 && NV <= 2) ? 4 : 0) agg_sum_kernel(const grd_agg_args a_in, int64_t light_warps,
                                                      int chunk_cols) {
    constexpr int NG = kWarp / LPR;
    grd_agg_args a = a_in;
    const int col0 = static_cast<int>(blockIdx.y) * chunk_cols;
    const int ldp = 4 * ((a_in.width + 3) / 4);   // partial row stride (full width)
    a.width = min(chunk_cols, a_in.width - col0);
    a.y += col0;
    a.out += col0;
    if (a.add_y) a.add_y += col0;
    if (a.mask_ref) a.mask_ref += col0;
    if (a.seg_partial) a.seg_partial += col0;
    if (a.heavy_counter) a.heavy_counter += blockIdx.y * a.n_heavy;
    const int lane = threadIdx.x & (kWarp - 1);
    const int g = lane / LPR;
    const int sub = lane % LPR;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const int w4 = (a.width + 3) / 4;
    float4 acc[NV];
    int hd[NV];                           // head of each column chunk (WE)
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        hd[c] = WE ? min((col0 + 4 * (sub + c * LPR)) / a.head_ld, a.heads - 1) : 0;
    }

    if (warp < light_warps) {
        const int64_t r = warp * NG + g;
        if (r >= a.n_rows) return;
        const int64_t beg = a.row_ptr[r], end = a.row_ptr[r + 1];
        if (a.heavy_threshold > 0 && end - beg > a.heavy_threshold) return;  // segmented
        agg_edges<LPR, NV, U, WE>(a, beg, end, 1, sub, w4, hd, acc);
        agg_finish<LPR, NV, WE>(a, r, end - beg, sub, w4, hd, acc);
        return;
    }
    const int64_t s = warp - light_warps;
    if (s >= a.n_segs) return;
    const int32_t h = a.seg_heavy[s];
    const int64_t r = a.heavy_rows[h];
    const int64_t seg0 = a.heavy_seg_ptr[h], nseg = a.heavy_seg_ptr[h + 1] - seg0;
    const int64_t rb = a.row_ptr[r], re = a.row_ptr[r + 1];
    const int64_t beg = rb + (s - seg0) * a.seg_len;
    const int64_t end = min(beg + int64_t(a.seg_len), re);
    agg_edges<LPR, NV, U, WE>(a, beg + g, end, NG, sub, w4, hd, acc);
#pragma unroll
    for (int off = kWarp / 2; off >= LPR; off >>= 1)
#pragma unroll
        for (int c = 0; c < NV; ++c) acc[c] = f4_add(acc[c], f4_shfl_xor(acc[c], off));
    heavy_tail<LPR, NV, WE>(a, s, lane, sub, w4, ldp, hd, acc);
}

// ---------------------------------------------------- K2 staged variant --
// Rows of 17..64 float4 chunks (one row per warp, LPR = 32): each lane
// streams its NV 16-byte chunks of the next K-1 neighbour rows into a private
// shared-memory ring with cp.async, so loads in flight hold no registers and
// a warp keeps K rows in flight (the register-staged kernel above keeps 4-8).
// A row's weight (src_scale, or the GAT per-head edge weight) rides along as
// a 4-byte cp.async into a parallel ring; each lane reads back only what it
// copied, so wait_group alone orders the ring (no warp barrier).  The light
// row's self term is the last item of its stream.  Source ids come from a
// 32-edge index window loaded one window ahead.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(unsigned dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async4(unsigned dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

constexpr int kAsyncWarps = 4;   // warps per block of the staged kernel

// MODE: 0 unweighted, 1 source-scaled (src_scale[j]), 2 GAT per-edge
// per-head weights (edge_w[perm(e), head(chunk)], self_w for the self item),
// each lane copying the NV weights of its own chunks.
template <int NV, int G, int K, int MODE>
__global__ void __launch_bounds__(kAsyncWarps * 32) agg_async_kernel(const grd_agg_args a, int64_t light_warps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr bool SCALED = MODE == 1;
    constexpr bool WE = MODE == 2;
    constexpr int kSlots = G * K;                     // rows in flight per warp
    constexpr int kWN = WE ? NV : (SCALED ? 1 : 0);   // weights per slot and lane
    const int lane = threadIdx.x & (kWarp - 1);
    const int wib = threadIdx.x / kWarp;
    float4* ring = reinterpret_cast<float4*>(smem_raw) + size_t(wib) * kSlots * NV * kWarp;
    float* wring = reinterpret_cast<float*>(reinterpret_cast<float4*>(smem_raw) +
                                            size_t(kAsyncWarps) * kSlots * NV * kWarp) +
                   size_t(wib) * kSlots * kWN * kWarp;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const int w4 = (a.width + 3) / 4;
    const int ldp = 4 * w4;
    int hd[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) hd[c] = WE ? min((4 * (lane + c * kWarp)) / a.head_ld, a.heads - 1) : 0;

    int64_t r, beg, end, seg = -1;
    if (warp < light_warps) {
        r = warp;
        if (r >= a.n_rows) return;
        beg = a.row_ptr[r];
        end = a.row_ptr[r + 1];
        if (a.heavy_threshold > 0 && end - beg > a.heavy_threshold) return;  // segmented
    } else {
        seg = warp - light_warps;
        if (seg >= a.n_segs) return;
        const int32_t h = a.seg_heavy[seg];
        r = a.heavy_rows[h];
        beg = a.row_ptr[r] + (seg - a.heavy_seg_ptr[h]) * a.seg_len;
        end = min(beg + int64_t(a.seg_len), a.row_ptr[r + 1]);
    }
    const int32_t orow = a.out_idx ? a.out_idx[r] : static_cast<int32_t>(r);
    const int32_t srow = (seg >= 0 || a.no_self) ? -1 : (a.self_idx ? a.self_idx[r] : orow);
    const int64_t ne = end - beg;
    const int64_t n = ne + (srow >= 0 ? 1 : 0);

    auto window = [&](int64_t m) -> int32_t {
        const int64_t i = m * kWarp + lane;
        return i < ne ? __ldg(a.idx + beg + i) : srow;
    };
    // SCALED: the windows' per-source scales, gathered one window ahead too;
    // WE: the windows' weight rows (edge ids through edge_w_perm)
    auto scales = [&](int64_t m, int32_t j) -> float {
        if constexpr (SCALED) return j >= 0 ? __ldg(a.src_scale + j) : 0.f;
        if constexpr (WE) {
            const int64_t i = m * kWarp + lane;
            if (!a.edge_w_perm) return __int_as_float(static_cast<int>(i));
            return __int_as_float(i < ne ? __ldg(a.edge_w_perm + beg + i) : 0);
        }
        return 0.f;
    };
    int32_t wa = window(0), wb = n > kWarp ? window(1) : 0;
    float sa = scales(0, wa), sb = n > kWarp ? scales(1, wb) : 0.f;
    int64_t ma = 0;
    // group g = rows 4g .. 4g+G-1 (G divides 32: a group never straddles a window)
    auto issue = [&](int64_t g) {
        const int64_t p0 = g * G;
        if (p0 < n) {
            const int64_t m = p0 >> 5;
            if (m != ma) {
                wa = wb;
                sa = sb;
                ma = m;
                if ((m + 1) * kWarp < n) {
                    wb = window(m + 1);
                    sb = scales(m + 1, wb);
                }
            }
            const int slot0 = static_cast<int>(g % K) * G;
#pragma unroll
            for (int u = 0; u < G; ++u) {
                const int64_t p = p0 + u;
                const int32_t j = __shfl_sync(0xffffffffu, wa, static_cast<int>(p & (kWarp - 1)));
                const float sv = (SCALED || WE) ? __shfl_sync(0xffffffffu, sa, static_cast<int>(p & (kWarp - 1))) : 0.f;
                if (p < n) {
                    const float* row = a.y + int64_t(j) * a.ldy;
#pragma unroll
                    for (int c = 0; c < NV; ++c) {
                        const int q = lane + c * kWarp;
                        if (q < w4) cp_async16(smem_u32(ring + ((slot0 + u) * NV + c) * kWarp + lane), row + 4 * q);
                    }
                    if constexpr (SCALED)   // after the row copies: the scale load may still be in flight
                        wring[(slot0 + u) * kWarp + lane] = sv;
                    if constexpr (WE) {
                        const float* wrow = p < ne ? a.edge_w + (a.edge_w_perm ? int64_t(__float_as_int(sv)) : beg + p) * a.heads
                                                   : a.self_w + int64_t(orow) * a.heads;
#pragma unroll
                        for (int c = 0; c < NV; ++c)
                            cp_async4(smem_u32(wring + ((slot0 + u) * NV + c) * kWarp + lane), wrow + hd[c]);
                    }
                }
            }
        }
        cp_commit();
    };

#pragma unroll
    for (int g = 0; g < K - 1; ++g) issue(g);
    float4 acc[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t ng = (n + G - 1) / G;
    for (int64_t g = 0; g < ng; ++g) {
        issue(g + K - 1);
        cp_wait<K - 1>();
        const int slot0 = static_cast<int>(g % K) * G;
#pragma unroll
        for (int u = 0; u < G; ++u) {
            if (g * G + u >= n) break;
#pragma unroll
            for (int c = 0; c < NV; ++c) {
                const float w = WE ? wring[((slot0 + u) * NV + c) * kWarp + lane]
                                   : (SCALED ? wring[(slot0 + u) * kWarp + lane] : 1.f);
                acc[c] = f4_fma(w, ring[((slot0 + u) * NV + c) * kWarp + lane], acc[c]);
            }
        }
    }
    cp_wait<0>();
    if (seg < 0) {
        agg_finish<32, NV, WE>(a, r, ne, lane, w4, hd, acc, /*add_self=*/false);
        return;
    }
    heavy_tail<32, NV, WE>(a, seg, lane, lane, w4, ldp, hd, acc);
}

template <int NV, int G, int K, int MODE>
int launch_async_t(const grd_agg_args& a, cudaStream_t st) {
    const int64_t warps = a.n_rows + a.n_segs;
    if (warps == 0) return 0;
    const int wn = MODE == 2 ? NV : (MODE == 1 ? 1 : 0);
    const size_t smem = size_t(kAsyncWarps) * G * K * kWarp * (16 * NV + 4 * wn);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(agg_async_kernel<NV, G, K, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        attr = true;
    }
    const int64_t blocks = (warps + kAsyncWarps - 1) / kAsyncWarps;
    agg_async_kernel<NV, G, K, MODE><<<static_cast<unsigned>(blocks), kAsyncWarps * kWarp, smem, st>>>(a, a.n_rows);
    return launch_status("agg_sum(staged)");
}

template <int NV, int G, int K>
int launch_async(const grd_agg_args& a, cudaStream_t st) {
    if (a.edge_w) return launch_async_t<NV, G, K, 2>(a, st);
    if (a.src_scale) return launch_async_t<NV, G, K, 1>(a, st);
    return launch_async_t<NV, G, K, 0>(a, st);
}

template <int LPR, int NV, int U, bool WE>
int launch_agg_t(const grd_agg_args& a, int chunk_cols, cudaStream_t st) {
    constexpr int NG = kWarp / LPR;
    const int64_t light_warps = (a.n_rows + NG - 1) / NG;
    const int64_t warps = light_warps + a.n_segs;
    if (warps == 0) return 0;
    const int64_t blocks = (warps * kWarp + 255) / 256;
    const unsigned chunks = static_cast<unsigned>((a.width + chunk_cols - 1) / chunk_cols);
    agg_sum_kernel<LPR, NV, U, WE><<<dim3(static_cast<unsigned>(blocks), chunks), 256, 0, st>>>(a, light_warps,
                                                                                               chunk_cols);
    return launch_status("agg_sum");
}

template <int LPR, int NV, int U>
int launch_agg(const grd_agg_args& a, int chunk_cols, cudaStream_t st) {
    if (a.edge_w) return launch_agg_t<LPR, NV, U, true>(a, chunk_cols, st);
    return launch_agg_t<LPR, NV, U, false>(a, chunk_cols, st);
}

int agg_chunk_cols(int width) {
    static int cfg = -1;
    if (cfg < 0) {
        const char* e = getenv("GRD_AGG_CHUNK");
        cfg = e ? atoi(e) : 0;   // measured: chunking does not pay on B200 (L2 already absorbs reuse)
    }
    if (cfg <= 0 || width <= cfg) return (width + 3) / 4 * 4;
    return (cfg + 3) / 4 * 4;
}

// ------------------------------------------------------------ K1 / K9 --
// LPR lanes per row (rows of w4 <= LPR chunks: a narrow row, e.g. GAT's
// 16-byte per-edge attention rows, no longer idles 31 lanes of a warp)
template <bool kAdd, int LPR>
__global__ void __launch_bounds__(256) row_copy_kernel(const float* __restrict__ src, int64_t lds,
                                                       const int32_t* __restrict__ idx, int64_t n_rows,
                                                       int w4, float* __restrict__ dst, int64_t ldd) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int sub = static_cast<int>(t & (LPR - 1));
    const int64_t r = t / LPR;
    if (r >= n_rows) return;
    const int32_t j = idx[r];
    if (kAdd) {
        const float* s = src + r * lds;
        float* d = dst + int64_t(j) * ldd;
        for (int q = sub; q < w4; q += LPR) {
            float4 v = *reinterpret_cast<float4*>(d + 4 * q);
            v = f4_add(v, ld_nc_f4(s + 4 * q));
            *reinterpret_cast<float4*>(d + 4 * q) = v;
        }
    } else {
        const float* s = src + int64_t(j) * lds;
        float* d = dst + r * ldd;
        for (int q = sub; q < w4; q += LPR)
            *reinterpret_cast<float4*>(d + 4 * q) = ld_nc_f4(s + 4 * q);
    }
}

template <bool kAdd>
void launch_row_copy(const float* src, int64_t lds, const int32_t* idx, int64_t n_rows, int w4, float* dst,
                     int64_t ldd, cudaStream_t st) {
#define GRD_ROW_COPY(L)                                                                              \
    row_copy_kernel<kAdd, L><<<static_cast<unsigned>((n_rows * L + 255) / 256), 256, 0, st>>>(src, lds, idx, n_rows, w4, dst, ldd)
    if (w4 <= 1) GRD_ROW_COPY(1);
    else if (w4 <= 2) GRD_ROW_COPY(2);
    else if (w4 <= 4) GRD_ROW_COPY(4);
    else if (w4 <= 8) GRD_ROW_COPY(8);
    else if (w4 <= 16) GRD_ROW_COPY(16);
    else GRD_ROW_COPY(32);
#undef GRD_ROW_COPY
}

// ----------------------------------------------------------- K6 reduce --
// Split-K partials of the tensor-core weight gradient are summed here in a
// fixed order (no float atomics), fused with the SGD step.
__global__ void wgrad_reduce_kernel(int64_t m, int64_t n, int64_t splits, int64_t ldp, const float* ws,
                                    float* dw, int64_t lddw, int accumulate, float* w, int64_t ldw,
                                    float lr) {
    // warp per output element: lane z sums splits z, z+32, ...; fixed butterfly
    const int lane = threadIdx.x & (kWarp - 1);
    const int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    if (i >= m * n) return;
    float s = 0.f;
    const int64_t r = i / n, c = i % n;
    for (int64_t z = lane; z < splits; z += kWarp) s += __ldcg(ws + (z * m + r) * ldp + c);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane != 0) return;
    if (accumulate) s += dw[r * lddw + c];
    dw[r * lddw + c] = s;
    if (w) w[r * ldw + c] -= lr * s;
}

int64_t wgrad_splits(int64_t m, int64_t n, int64_t k) {
    const int64_t bn = n >= 256 ? 256 : (n + 31) / 32 * 32;   // MN-major B tile width
    const int64_t tiles = ((m + 127) / 128) * ((n + bn - 1) / bn);
    // >= one wave of CTAs, and K chunks of <= 8192 rows so each fp32 TMEM
    // accumulation stays short (partials are then reduced in a fixed tree)
    int64_t splits = (148 + tiles - 1) / tiles;
    const int64_t min_splits = (k + 8191) / 8192;
    if (splits < min_splits) splits = min_splits;
    const int64_t max_splits = (k + 1023) / 1024;
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
    return splits;
}

// -------------------------------------------------------------------- K4 --
constexpr int kLossBlocks = 1184;  // 148 SMs x 8
constexpr int kXentRegCols = 256;  // rows up to this many classes reduce in registers

__global__ void __launch_bounds__(256) xent_kernel(const float* __restrict__ logits, int64_t ldl,
                                                   int64_t n_rows, int c, const int32_t* __restrict__ labels,
                                                   const uint8_t* __restrict__ mask, float inv_count,
                                                   float* __restrict__ grad, int64_t ldg,
                                                   const float* __restrict__ gscale, double* partials,
                                                   float* __restrict__ grad2, int64_t ldg2,
                                                   const float* __restrict__ g2scale) {
    const int lane = threadIdx.x & (kWarp - 1);
    const int warp = threadIdx.x / kWarp;
    const int c4 = (c + 3) / 4 * 4;
    double loss_acc = 0.0;
    double correct = 0.0;
    const int64_t nwarps = int64_t(gridDim.x) * (blockDim.x / kWarp);
    if (c <= 2 * kWarp) {
        // <= 64 classes: the row lives in two registers per lane, each exp is
        // computed once, and the next row's logits / label / mask are loaded
        // while this one reduces (same arithmetic as the general loop below,
        // so the same bits)
        int64_t r = int64_t(blockIdx.x) * (blockDim.x / kWarp) + warp;
        auto load = [&](int64_t rr, float& a, float& b, int& yy, bool& mm) {
            const float* row = logits + rr * ldl;
            a = lane < c ? row[lane] : -INFINITY;
            b = lane + kWarp < c ? row[lane + kWarp] : -INFINITY;
            yy = labels[rr];
            mm = mask[rr] != 0;
        };
        float v0 = 0.f, v1 = 0.f;
        int y = 0;
        bool on = false;
        if (r < n_rows) load(r, v0, v1, y, on);
        for (; r < n_rows; r += nwarps) {
            float n0 = 0.f, n1 = 0.f;
            int ny = 0;
            bool non = false;
            if (r + nwarps < n_rows) load(r + nwarps, n0, n1, ny, non);
            float* grow = grad + r * ldg;
            float* grow2 = grad2 ? grad2 + r * ldg2 : nullptr;
            const float s2 = grad2 ? g2scale[r] : 0.f;
            if (lane < c4 - c) {
                grow[c + lane] = 0.f;
                if (grow2) grow2[c + lane] = 0.f;
            }
            if (!on) {
                if (lane < c) grow[lane] = 0.f;
                if (lane + kWarp < c) grow[lane + kWarp] = 0.f;
                if (grow2) {
                    if (lane < c) grow2[lane] = 0.f;
                    if (lane + kWarp < c) grow2[lane + kWarp] = 0.f;
                }
            } else {
                float mx = v0;
                int arg = lane < c ? lane : 0x7fffffff;
                if (v1 > mx) { mx = v1; arg = lane + kWarp; }
                for (int off = 16; off > 0; off >>= 1) {
                    const float om = __shfl_xor_sync(0xffffffffu, mx, off);
                    const int oa = __shfl_xor_sync(0xffffffffu, arg, off);
                    if (om > mx || (om == mx && oa < arg)) { mx = om; arg = oa; }
                }
                const float e0 = lane < c ? expf(v0 - mx) : 0.f;
                const float e1 = lane + kWarp < c ? expf(v1 - mx) : 0.f;
                float sum = e0 + e1;
                if (!(lane + kWarp < c)) sum = e0;
                // the general loop adds j = lane first, then j = lane + 32
                for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
                const float scale = gscale ? gscale[r] : 1.0f;
                const float inv_sum = 1.0f / sum;   // one division per row, not per class
                if (lane < c) {
                    float pr = e0 * inv_sum;
                    if (lane == y) pr -= 1.0f;
                    const float gv = pr * inv_count * scale;
                    grow[lane] = gv;
                    if (grow2) grow2[lane] = gv * s2;     // the pull's source scale, pre-applied
                }
                if (lane + kWarp < c) {
                    float pr = e1 * inv_sum;
                    if (lane + kWarp == y) pr -= 1.0f;
                    const float gv = pr * inv_count * scale;
                    grow[lane + kWarp] = gv;
                    if (grow2) grow2[lane + kWarp] = gv * s2;
                }
                const float ey = __shfl_sync(0xffffffffu, y < kWarp ? e0 : e1, y & (kWarp - 1));
                if (lane == 0) {
                    loss_acc -= static_cast<double>(logf(ey / sum));
                    correct += (arg == y) ? 1.0 : 0.0;
                }
            }
            v0 = n0; v1 = n1; y = ny; on = non;
        }
        r = n_rows;   // fall through to the block reduction
    }
    if (c > 2 * kWarp && c <= kXentRegCols) {
        // 65..256 classes: the row lives in registers (up to 8 per lane, j =
        // lane + 32 k), the next row is loaded while this one reduces; the
        // same per-lane orders as the general loop below (max / argmax and
        // the exp sum over ascending j, then the butterfly): the same bits
        constexpr int NV = kXentRegCols / kWarp;
        int64_t r = int64_t(blockIdx.x) * (blockDim.x / kWarp) + warp;
        float v[NV], nv[NV];
        int y = 0, ny = 0;
        bool on = false, non = false;
        auto load = [&](int64_t rr, float (&x)[NV], int& yy, bool& mm) {
            const float* row = logits + rr * ldl;
#pragma unroll
            for (int k = 0; k < NV; ++k) x[k] = lane + k * kWarp < c ? row[lane + k * kWarp] : -INFINITY;
            yy = labels[rr];
            mm = mask[rr] != 0;
        };
        if (r < n_rows) load(r, v, y, on);
        for (; r < n_rows; r += nwarps) {
            if (r + nwarps < n_rows) load(r + nwarps, nv, ny, non);
            float* grow = grad + r * ldg;
            float* grow2 = grad2 ? grad2 + r * ldg2 : nullptr;
            const float s2 = grad2 ? g2scale[r] : 0.f;
            if (lane < c4 - c) {
                grow[c + lane] = 0.f;
                if (grow2) grow2[c + lane] = 0.f;
            }
            if (!on) {
#pragma unroll
                for (int k = 0; k < NV; ++k) {
                    const int j = lane + k * kWarp;
                    if (j < c) {
                        grow[j] = 0.f;
                        if (grow2) grow2[j] = 0.f;
                    }
                }
            } else {
                float mx = -INFINITY;
                int arg = 0x7fffffff;
#pragma unroll
                for (int k = 0; k < NV; ++k) {
                    const int j = lane + k * kWarp;
                    if (j < c && (v[k] > mx || (v[k] == mx && j < arg))) { mx = v[k]; arg = j; }
                }
                for (int off = 16; off > 0; off >>= 1) {
                    const float om = __shfl_xor_sync(0xffffffffu, mx, off);
                    const int oa = __shfl_xor_sync(0xffffffffu, arg, off);
                    if (om > mx || (om == mx && oa < arg)) { mx = om; arg = oa; }
                }
                float e[NV];
                float sum = 0.f;
#pragma unroll
                for (int k = 0; k < NV; ++k) {
                    e[k] = lane + k * kWarp < c ? expf(v[k] - mx) : 0.f;
                    if (lane + k * kWarp < c) sum += e[k];
                }
                for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
                const float scale = gscale ? gscale[r] : 1.0f;
                const float inv_sum = 1.0f / sum;   // one division per row, not per class
                float ey = 0.f;
#pragma unroll
                for (int k = 0; k < NV; ++k) {
                    const int j = lane + k * kWarp;
                    if (j < c) {
                        float pr = e[k] * inv_sum;
                        if (j == y) { pr -= 1.0f; ey = e[k]; }
                        const float gv = pr * inv_count * scale;
                        grow[j] = gv;
                        if (grow2) grow2[j] = gv * s2;
                    }
                }
                ey = __shfl_sync(0xffffffffu, ey, y & (kWarp - 1));
                if (lane == 0) {
                    loss_acc -= static_cast<double>(logf(ey / sum));
                    correct += (arg == y) ? 1.0 : 0.0;
                }
            }
#pragma unroll
            for (int k = 0; k < NV; ++k) v[k] = nv[k];
            y = ny;
            on = non;
        }
    }
    for (int64_t r = c <= kXentRegCols ? n_rows : int64_t(blockIdx.x) * (blockDim.x / kWarp) + warp; r < n_rows;
         r += nwarps) {
        const float* row = logits + r * ldl;
        float* grow = grad + r * ldg;
        float* grow2 = grad2 ? grad2 + r * ldg2 : nullptr;
        const float s2 = grad2 ? g2scale[r] : 0.f;
        // padding columns [c, round_up(c, 4)) are part of the 16-byte rows the
        // aggregation kernels read: keep them zero
        if (lane < c4 - c) {
            grow[c + lane] = 0.f;
            if (grow2) grow2[c + lane] = 0.f;
        }
        if (!mask[r]) {
            for (int j = lane; j < c; j += kWarp) {
                grow[j] = 0.f;
                if (grow2) grow2[j] = 0.f;
            }
            continue;
        }
        // max and first argmax (np.argmax semantics)
        float mx = -INFINITY;
        int arg = 0x7fffffff;
        for (int j = lane; j < c; j += kWarp) {
            const float v = row[j];
            if (v > mx || (v == mx && j < arg)) { mx = v; arg = j; }
        }
        for (int off = 16; off > 0; off >>= 1) {
            const float om = __shfl_xor_sync(0xffffffffu, mx, off);
            const int oa = __shfl_xor_sync(0xffffffffu, arg, off);
            if (om > mx || (om == mx && oa < arg)) { mx = om; arg = oa; }
        }
        float sum = 0.f;
        for (int j = lane; j < c; j += kWarp) sum += expf(row[j] - mx);
        for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
        const int y = labels[r];
        const float scale = gscale ? gscale[r] : 1.0f;
        const float inv_sum = 1.0f / sum;
        for (int j = lane; j < c; j += kWarp) {
            float p = expf(row[j] - mx) * inv_sum;
            if (j == y) p -= 1.0f;
            const float gv = p * inv_count * scale;
            grow[j] = gv;
            if (grow2) grow2[j] = gv * s2;
        }
        if (lane == 0) {
            const float py = expf(row[y] - mx) / sum;
            loss_acc -= static_cast<double>(logf(py));
            correct += (arg == y) ? 1.0 : 0.0;
        }
    }
    __shared__ double sl[8], sc[8];
    if (lane == 0) { sl[warp] = loss_acc; sc[warp] = correct; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x / kWarp); ++w) { a += sl[w]; b += sc[w]; }
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = b;
    }
}

// One block of 1024 threads: strided partial sums, then a fixed-order tree.
__global__ void __launch_bounds__(1024) xent_finalize_kernel(const double* partials, int nblocks,
                                                             double count, double* stats) {
    __shared__ double sa[1024], sb[1024];
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < nblocks; i += blockDim.x) { a += partials[2 * i]; b += partials[2 * i + 1]; }
    sa[threadIdx.x] = a;
    sb[threadIdx.x] = b;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) { sa[threadIdx.x] += sa[threadIdx.x + w]; sb[threadIdx.x] += sb[threadIdx.x + w]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        stats[0] = sa[0] / count;
        stats[1] = sb[0] / count;
        stats[2] = sa[0];
        stats[3] = sb[0];
    }
}

// ------------------------------------------------------------ helpers --
__global__ void mul_rows_kernel(const float* x, int64_t ldx, const float* m, int64_t ldm, int64_t n_rows,
                                int width, float* y, int64_t ldy) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_rows * width) return;
    const int64_t r = i / width, c = i % width;
    y[r * ldy + c] = x[r * ldx + c] * m[r * ldm + c];
}

__global__ void mask_scale_rows_kernel(const float* x, int64_t ldx, const float* ref, int64_t ldref,
                                       const float* row_scale, int64_t n_rows, int width, float* y,
                                       int64_t ldy) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_rows * width) return;
    const int64_t r = i / width, c = i % width;
    float v = x[r * ldx + c];
    if (ref && !(ref[r * ldref + c] > 0.f)) v = 0.f;
    if (row_scale) v *= row_scale[r];
    y[r * ldy + c] = v;
}

__global__ void rownorm_fwd_kernel(const float* pre, int64_t ld, int64_t n_rows, int width, int relu,
                                   const int32_t* out_idx, float* out, int64_t ldo) {
    const int lane = threadIdx.x & (kWarp - 1);
    const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    if (r >= n_rows) return;
    const float* p = pre + r * ld;
    float ss = 0.f;
    for (int j = lane; j < width; j += kWarp) ss = fmaf(p[j], p[j], ss);
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    const float nrm = sqrtf(ss);
    float* o = out + int64_t(out_idx ? out_idx[r] : r) * ldo;
    for (int j = lane; j < width; j += kWarp) {
        float v = nrm > 0.f ? p[j] / nrm : 0.f;
        if (relu) v = fmaxf(v, 0.f);
        o[j] = v;
    }
}

__global__ void rownorm_bwd_kernel(const float* pre, int64_t ldp, const float* gy, int64_t ldg,
                                   const float* a_out, int64_t lda, int64_t n_rows, int width,
                                   const float* row_scale, float* gp, int64_t ldgp) {
    const int lane = threadIdx.x & (kWarp - 1);
    const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    if (r >= n_rows) return;
    const float* p = pre + r * ldp;
    const float* g = gy + r * ldg;
    const float* ao = a_out ? a_out + r * lda : nullptr;
    float ss = 0.f;
    for (int j = lane; j < width; j += kWarp) ss = fmaf(p[j], p[j], ss);
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    const float nrm = sqrtf(ss);
    float inner = 0.f;
    for (int j = lane; j < width; j += kWarp) {
        const float u = nrm > 0.f ? p[j] / nrm : 0.f;
        const float gj = (ao && !(ao[j] > 0.f)) ? 0.f : g[j];
        inner = fmaf(u, gj, inner);
    }
    for (int off = 16; off > 0; off >>= 1) inner += __shfl_xor_sync(0xffffffffu, inner, off);
    const float rs = row_scale ? row_scale[r] : 1.0f;
    float* o = gp + r * ldgp;
    for (int j = lane; j < width; j += kWarp) {
        const float u = nrm > 0.f ? p[j] / nrm : 0.f;
        const float gj = (ao && !(ao[j] > 0.f)) ? 0.f : g[j];
        const float v = nrm > 0.f ? (gj - u * inner) / nrm : 0.f;
        o[j] = v * rs;
    }
}

inline unsigned blocks_for(int64_t threads, int per_block = 256) {
    return static_cast<unsigned>((threads + per_block - 1) / per_block);
}

}  // namespace

// =====================================================================
// extern "C" launchers
// =====================================================================
extern "C" int grd_device_sm_count(int32_t* sm_count) {
    clear_error();
    int dev = 0, v = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return fail(static_cast<int>(e), "sm count: %s", cudaGetErrorString(e));
    *sm_count = v;
    return 0;
}

extern "C" int grd_gather_rows(const float* src, int64_t ld_src, const int32_t* idx, int64_t n_rows,
                               int32_t width, float* dst, int64_t ld_dst, void* stream) {
    clear_error();
    if (n_rows == 0) return 0;
    if (!src || !idx || !dst || width <= 0 || ld_src % 4 || ld_dst % 4)
        return fail(kErrArg, "gather_rows: bad arguments");
    launch_row_copy<false>(src, ld_src, idx, n_rows, (width + 3) / 4, dst, ld_dst, static_cast<cudaStream_t>(stream));
    return launch_status("gather_rows");
}

// Strided 2-D copy between any two of {device, page-locked host} memory
// (cudaMemcpyDefault under UVA): `rows` rows of `width_bytes`, pitches in
// bytes.  The SSO tiers keep rows unpadded (d values) while device matrices
// are padded to ld = round_up(d, 4); the copy engine moves exactly
// rows * width_bytes over the host link, the pitch change is free.
extern "C" int grd_memcpy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch,
                            int64_t width_bytes, int64_t rows, void* stream) {
    clear_error();
    if (rows == 0 || width_bytes == 0) return 0;
    if (!dst || !src || width_bytes < 0 || rows < 0 || dpitch < width_bytes || spitch < width_bytes)
        return fail(kErrArg, "memcpy2d: bad arguments");
    const cudaError_t e = cudaMemcpy2DAsync(dst, static_cast<size_t>(dpitch), src, static_cast<size_t>(spitch),
                                            static_cast<size_t>(width_bytes), static_cast<size_t>(rows),
                                            cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fail(static_cast<int>(e), "memcpy2d: %s", cudaGetErrorString(e));
    return 0;
}

extern "C" int grd_scatter_add_rows(const float* src, int64_t ld_src, const int32_t* idx, int64_t n_rows,
                                    int32_t width, float* dst, int64_t ld_dst, void* stream) {
    clear_error();
    if (n_rows == 0) return 0;
    if (!src || !idx || !dst || width <= 0 || ld_src % 4 || ld_dst % 4)
        return fail(kErrArg, "scatter_add_rows: bad arguments");
    launch_row_copy<true>(src, ld_src, idx, n_rows, (width + 3) / 4, dst, ld_dst, static_cast<cudaStream_t>(stream));
    return launch_status("scatter_add_rows");
}

extern "C" int grd_agg_sum(const grd_agg_args* args, void* stream) {
    clear_error();
    if (!args) return fail(kErrArg, "agg_sum: null args");
    const grd_agg_args& a = *args;
    if (a.n_rows == 0 && a.width > 0) return 0;        // e.g. a rank that owns no rows
    if (a.n_rows < 0 || a.width <= 0 || a.width > 1024 || !a.row_ptr || !a.y || !a.out)
        return fail(kErrArg, "agg_sum: bad arguments (width %d)", a.width);
    if (a.ldy % 4 || a.ldo % 4 || (reinterpret_cast<uintptr_t>(a.y) & 15) ||
        (reinterpret_cast<uintptr_t>(a.out) & 15))
        return fail(kErrArg, "agg_sum: rows must be 16-byte aligned (ld %% 4 == 0)");
    if (a.n_segs > 0 && (!a.heavy_rows || !a.heavy_seg_ptr || !a.seg_heavy || !a.seg_partial ||
                         !a.heavy_counter || a.seg_len <= 0))
        return fail(kErrArg, "agg_sum: incomplete heavy-row split");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int cc = agg_chunk_cols(a.width);
    if (a.n_segs > 0 && (a.width + cc - 1) / cc > kMaxAggChunks)
        return fail(kErrArg, "agg_sum: too many column chunks");
    const int w4 = (cc + 3) / 4;
    // Unweighted rows of 17..64 chunks: the cp.async-staged kernel, 2 groups
    // of 2 rows in flight per warp (swept on B200 over 4..12 rows in flight and
    // group sizes 1..4: -12% at widths 100 and 256 against the register-
    // staged kernel; weighted rows stay on the latter, where staging the
    // per-edge weights costs more than it hides).  GRD_AGG_ASYNC=0 disables.
    const char* async_env = getenv("GRD_AGG_ASYNC");
    const int async_on = async_env ? atoi(async_env) : 1;
    // (scaled rows of <= 32 chunks measured faster on the register kernel)
    const char* mid_env = getenv("GRD_AGG_MID");
    const bool mid_override = mid_env && atoi(mid_env) > 0;
    if (async_on && !mid_override && !a.edge_w && cc >= a.width && w4 > (a.src_scale ? 32 : 16) && w4 <= 64) {
        // rows in flight per warp (GRD_AGG_ASYNC_DEPTH sweep hook: 4 default, 6, 8, 3x2)
        static int depth = -1;
        if (depth < 0) {
            const char* e = getenv("GRD_AGG_ASYNC_DEPTH");
            depth = e ? atoi(e) : 4;
        }
        if (w4 <= 32) {
            if (depth == 6) return launch_async<1, 2, 3>(a, st);
            if (depth == 8) return launch_async<1, 4, 2>(a, st);
            if (depth == 3) return launch_async<1, 1, 3>(a, st);
            return launch_async<1, 2, 2>(a, st);
        }
        return launch_async<2, 2, 2>(a, st);
    }
    // GAT weighted rows: staged variant opt-in (GRD_AGG_ASYNC_WE=1; parity-
    // green, but 157 vs 135 ms per products_gat epoch on B200: the NV 4-byte
    // weight copies per row cost more than the staging hides)
    const char* we_env = getenv("GRD_AGG_ASYNC_WE");
    if (a.edge_w && we_env && atoi(we_env) > 0 && cc >= a.width && w4 > 16 && w4 <= 64)
        return w4 <= 32 ? launch_async<1, 2, 2>(a, st) : launch_async<2, 2, 2>(a, st);
    // rows in flight per warp: 8 for the 17..32-chunk rows (measured +15% at
    // width 100), 4 above
    if (w4 <= 1) return launch_agg<1, 1, 4>(a, cc, st);
    if (w4 <= 2) return launch_agg<2, 1, 4>(a, cc, st);
    if (w4 <= 4) return launch_agg<4, 1, 4>(a, cc, st);
    if (w4 <= 8) return launch_agg<8, 1, 4>(a, cc, st);
    if (w4 <= 16) {
        // narrow rows: lane groups of LPR lanes with NV chunks each; swept on
        // B200 at the products shape (tools/agg_bench.py, GRD_AGG_NARROW):
        // 4 lanes x 3 chunks, 8 rows deep: -15..19% at widths 40/48 against
        // 16 lanes x 1 chunk; 8 x 2, 4 deep: -12% at width 64
        const char* nv_env = getenv("GRD_AGG_NARROW");
        const int nv = nv_env ? atoi(nv_env) : -1;
        switch (nv) {
            case 0: return launch_agg<16, 1, 4>(a, cc, st);
            case 1: return launch_agg<8, 2, 4>(a, cc, st);
            case 3: return launch_agg<4, 4, 4>(a, cc, st);
            case 4: return launch_agg<8, 2, 8>(a, cc, st);
            case 5: return launch_agg<4, 4, 2>(a, cc, st);
            default: break;
        }
        if (w4 <= 12) return launch_agg<4, 3, 8>(a, cc, st);
        return launch_agg<8, 2, 4>(a, cc, st);
    }
    if (w4 <= 64) {
        // mid widths: register variants against the staged kernel above
        const char* mv_env = getenv("GRD_AGG_MID");
        const int mv = mv_env ? atoi(mv_env) : 0;
        switch (mv) {
            case 1: if (w4 <= 32) return launch_agg<8, 4, 4>(a, cc, st); break;
            case 2: if (w4 <= 32) return launch_agg<16, 2, 4>(a, cc, st); break;
            case 3: return launch_agg<16, 4, 2>(a, cc, st);
            case 4: return launch_agg<8, 8, 2>(a, cc, st);
            case 5: if (w4 <= 32) return launch_agg<8, 4, 8>(a, cc, st); break;
            default: break;
        }
    }
    // scaled rows of 17..32 chunks (staged kernel off): 16 lanes x 2 chunks,
    // 4 deep (-7% at width 100 against one row per warp, 8 deep)
    if (w4 <= 32) return a.src_scale && !a.edge_w ? launch_agg<16, 2, 4>(a, cc, st)
                                                  : launch_agg<32, 1, 8>(a, cc, st);
    if (w4 <= 64) return launch_agg<32, 2, 4>(a, cc, st);
    if (w4 <= 128) return launch_agg<32, 4, 2>(a, cc, st);
    return launch_agg<32, 8, 1>(a, cc, st);
}

extern "C" int grd_gemm(const grd_gemm_args* args, void* stream) {
    clear_error();
    if (!args) return fail(kErrArg, "gemm: null args");
    const grd_gemm_args& g = *args;
    if (g.m < 0 || g.n < 0 || g.k < 0) return fail(kErrArg, "gemm: bad arguments");
    if (g.m == 0 || g.n == 0) return 0;                 // nothing to write
    if (!g.a || !g.b || !g.c) return fail(kErrArg, "gemm: bad arguments");
    GrdTcGemm t{};
    t.m = g.m; t.n = g.n; t.k = g.k;
    t.a = g.a; t.lda = g.lda; t.trans_a = g.trans_a;
    t.b = g.b; t.ldb = g.ldb; t.trans_b = g.trans_b;
    t.c = g.c; t.ldc = g.ldc;
    t.row_scale = g.row_scale;
    t.elem_mul = g.elem_mul; t.ld_elem_mul = g.ld_elem_mul;
    t.relu_ref = g.relu_ref; t.ld_relu_ref = g.ld_relu_ref;
    t.relu_out = g.relu_out; t.accumulate = g.accumulate;
    t.k_splits = 1;
    if (g.c2) {
        if (g.split <= 0 || g.split % 4 || g.ldc2 % 4 || g.accumulate || g.relu_ref || g.elem_mul ||
            (reinterpret_cast<uintptr_t>(g.c2) & 15))
            return fail(kErrArg, "gemm: split output needs split %% 4 == 0, aligned c2, no accumulate / "
                        "relu_ref / elem_mul");
        t.c2 = g.c2; t.ldc2 = g.ldc2; t.split = g.split;
    }
    if (g.lda % 4 || g.ldb % 4 || g.ldc % 4 || (reinterpret_cast<uintptr_t>(g.a) & 15) ||
        (reinterpret_cast<uintptr_t>(g.c) & 15))
        return fail(kErrArg, "gemm: leading dims must be multiples of 4 and rows 16-byte aligned");
    const int64_t need = grd_tc_pack_elems(g.n, g.k);
    if (!g.workspace || g.workspace_elems < need)
        return fail(kErrArg, "gemm: workspace needs %lld floats", (long long)need);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // opt-in bf16x3 serves plain products only (split outputs and
    // accumulating launches — the K-chunked ones — stay 3xTF32); the packed
    // operand's layout follows the same decision
    t.bf16 = !g.trans_a && !g.c2 && !g.accumulate && grd_tc_bf16x3();
    cudaError_t e = grd_tc_pack_b(g.b, g.ldb, g.trans_b, g.n, g.k, g.workspace, st, t.bf16);
    if (e == cudaSuccess) {
        t.b_packed = g.workspace;
        e = grd_tc_gemm(t, st);
    }
    if (e != cudaSuccess) return fail(static_cast<int>(e), "gemm: %s", cudaGetErrorString(e));
    return 0;
}

extern "C" int64_t grd_gemm_workspace(int64_t n, int64_t k) { return grd_tc_pack_elems(n, k); }

extern "C" int64_t grd_wgrad_workspace(int64_t m, int64_t n, int64_t k) {
    return wgrad_splits(m, n, k) * m * ((n + 3) / 4 * 4);
}

extern "C" int grd_wgrad_sgd(int64_t m, int64_t n, int64_t k, const float* a, int64_t lda, const float* b,
                             int64_t ldb, float* dw, int64_t lddw, int32_t accumulate, float* w, int64_t ldw,
                             float lr, float* workspace, int64_t workspace_elems, void* stream) {
    clear_error();
    if (m <= 0 || n <= 0 || k < 0 || (k > 0 && (!a || !b)) || !dw || !workspace)
        return fail(kErrArg, "wgrad: bad arguments");
    const int64_t splits = wgrad_splits(m, n, k);
    if (workspace_elems < splits * m * ((n + 3) / 4 * 4)) return fail(kErrArg, "wgrad: workspace too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (k > 0 && (lda % 4 || ldb % 4 || (reinterpret_cast<uintptr_t>(a) & 15) ||
                  (reinterpret_cast<uintptr_t>(b) & 15)))
        return fail(kErrArg, "wgrad: leading dims must be multiples of 4 and rows 16-byte aligned");
    const int64_t ldp = (n + 3) / 4 * 4;
    int64_t used = 1;
    if (k == 0) {
        cudaMemsetAsync(workspace, 0, sizeof(float) * m * ldp, st);
    } else {
        int64_t kchunk = (k + splits - 1) / splits;
        kchunk = (kchunk + 31) / 32 * 32;
        used = (k + kchunk - 1) / kchunk;
        GrdTcGemm t{};
        t.m = m; t.n = n; t.k = k;
        t.a = a; t.lda = lda; t.trans_a = 1;      // A^T: a stored K x M
        t.b = b; t.ldb = ldb; t.trans_b = 0;      // b stored K x N
        t.k_splits = static_cast<int>(used);
        t.k_chunk = kchunk;
        t.partial = workspace;
        const cudaError_t e = grd_tc_gemm(t, st);
        if (e != cudaSuccess) return fail(static_cast<int>(e), "wgrad: %s", cudaGetErrorString(e));
    }
    wgrad_reduce_kernel<<<blocks_for(m * n * kWarp), 256, 0, st>>>(m, n, used, ldp, workspace, dw, lddw,
                                                                    accumulate, w, ldw, lr);
    return launch_status("wgrad_reduce");
}

extern "C" int64_t grd_loss_partials(int64_t n_rows) {
    (void)n_rows;
    return 2 * kLossBlocks;
}

extern "C" int grd_softmax_xent(const float* logits, int64_t ld_logits, int64_t n_rows, int32_t n_classes,
                                const int32_t* labels, const uint8_t* mask, int64_t mask_count, float* grad,
                                int64_t ld_grad, const float* grad_scale, double* partials, double* stats_out,
                                void* stream) {
    return grd_softmax_xent2(logits, ld_logits, n_rows, n_classes, labels, mask, mask_count, grad, ld_grad,
                             grad_scale, nullptr, 0, nullptr, partials, stats_out, stream);
}

extern "C" int grd_softmax_xent2(const float* logits, int64_t ld_logits, int64_t n_rows, int32_t n_classes,
                                 const int32_t* labels, const uint8_t* mask, int64_t mask_count, float* grad,
                                 int64_t ld_grad, const float* grad_scale, float* grad2, int64_t ld_grad2,
                                 const float* grad2_scale, double* partials, double* stats_out, void* stream) {
    clear_error();
    if (grad2 && (!grad2_scale || ld_grad2 < n_classes)) return fail(kErrArg, "softmax_xent: grad2 needs its scale");
    if ((n_rows > 0 && (!logits || !labels || !mask || !grad)) || !partials || !stats_out || n_classes <= 0 ||
        n_rows < 0)
        return fail(kErrArg, "softmax_xent: bad arguments");
    if (mask_count <= 0) return fail(kErrArg, "loss mask selects no vertices");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const float inv = static_cast<float>(1.0 / static_cast<double>(mask_count));
    xent_kernel<<<kLossBlocks, 256, 0, st>>>(logits, ld_logits, n_rows, n_classes, labels, mask, inv, grad,
                                             ld_grad, grad_scale, partials, grad2, ld_grad2, grad2_scale);
    int rc = launch_status("softmax_xent");
    if (rc) return rc;
    xent_finalize_kernel<<<1, 1024, 0, st>>>(partials, kLossBlocks, static_cast<double>(mask_count), stats_out);
    return launch_status("softmax_xent_finalize");
}

extern "C" int grd_mul_rows(const float* x, int64_t ldx, const float* m, int64_t ldm, int64_t n_rows,
                            int32_t width, float* y, int64_t ldy, void* stream) {
    clear_error();
    if (n_rows == 0) return 0;
    if (!x || !m || !y) return fail(kErrArg, "mul_rows: bad arguments");
    mul_rows_kernel<<<blocks_for(n_rows * width), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        x, ldx, m, ldm, n_rows, width, y, ldy);
    return launch_status("mul_rows");
}

extern "C" int grd_mask_scale_rows(const float* x, int64_t ldx, const float* ref, int64_t ldref,
                                   const float* row_scale, int64_t n_rows, int32_t width, float* y,
                                   int64_t ldy, void* stream) {
    clear_error();
    if (n_rows == 0) return 0;
    if (!x || !y) return fail(kErrArg, "mask_scale_rows: bad arguments");
    mask_scale_rows_kernel<<<blocks_for(n_rows * width), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        x, ldx, ref, ldref, row_scale, n_rows, width, y, ldy);
    return launch_status("mask_scale_rows");
}

extern "C" int grd_rownorm_fwd(const float* pre, int64_t ld, int64_t n_rows, int32_t width, int32_t relu,
                               const int32_t* out_idx, float* out, int64_t ldo, void* stream) {
    clear_error();
    if (n_rows == 0) return 0;
    if (!pre || !out) return fail(kErrArg, "rownorm_fwd: bad arguments");
    rownorm_fwd_kernel<<<blocks_for(n_rows * kWarp), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        pre, ld, n_rows, width, relu, out_idx, out, ldo);
    return launch_status("rownorm_fwd");
}

extern "C" int grd_rownorm_bwd(const float* pre, int64_t ldp, const float* grad_y, int64_t ldg,
                               const float* a_out, int64_t lda, int64_t n_rows, int32_t width,
                               const float* row_scale, float* grad_pre, int64_t ldgp, void* stream) {
    clear_error();
    if (n_rows == 0) return 0;
    if (!pre || !grad_y || !grad_pre) return fail(kErrArg, "rownorm_bwd: bad arguments");
    rownorm_bwd_kernel<<<blocks_for(n_rows * kWarp), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        pre, ldp, grad_y, ldg, a_out, lda, n_rows, width, row_scale, grad_pre, ldgp);
    return launch_status("rownorm_bwd");
}
