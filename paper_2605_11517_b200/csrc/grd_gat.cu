// GAT layer kernels (builder-defined layer): edge
// softmax over in(v) U {v} per head, its backward, attention-score
// gradients and the parameter plumbing of the fused transform
//   P_ext = X [W | W a_src | W a_dst]      (one tcgen05 GEMM gives P, s, t)
// The weighted neighbour sums themselves (O_v = sum alpha_uv P_u and its
// transpose) run in grd_agg_sum with per-edge, per-head weights.
//
// Layout of P_ext rows (ld_ext floats): head h of P at [h*dhp, h*dhp + dh)
// (dhp = round_up(dh, 4), zero padded), s_h at hdp + h, t_h at hdp + H + h,
// hdp = H * dhp.  Per-edge arrays are [E][H] in the aggregation CSR's edge
// order; per-vertex arrays [V][H].
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "../../include/grinder_b200.h"
#include "grd_common.h"

using namespace grd;

namespace {

constexpr int kWarp = 32;
constexpr int kMaxHeads = 8;

__device__ __forceinline__ float lrelu(float z, float slope) { return z > 0.f ? z : z * slope; }
// (the aggregation kernel's float4 helpers: the fused pull must round alike)
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
__device__ __forceinline__ float lrelu_grad(float z, float slope) { return z > 0.f ? 1.f : slope; }

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

inline int launch_status(const char* what) {
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return fail(static_cast<int>(err), "%s: %s", what, cudaGetErrorString(err));
    return 0;
}

// ------------------------------------------------------------- work units --
// A CSR row is processed either whole (a "light" row: at most
// heavy_threshold edges, plus the self loop) or, when it is heavier, as
// seg_len-edge segments handled by separate warps (the self loop rides with
// segment 0) whose per-head partials a second, deterministic pass combines.
// Warp w < n_rows takes light row w (and skips it when heavy); warp
// n_rows + s takes segment s.  This keeps hub rows of the power-law graphs
// from serialising a whole launch behind one warp.
struct Unit {
    int64_t row, beg, end;   // CSR row and the edge range of this unit
    int64_t seg;             // segment index, -1 for a light row
    bool self;               // the unit carries the implicit self loop
};

__device__ __forceinline__ bool unit_of(const grd_gat_args& a, int64_t w, Unit& u) {
    if (w < a.n_rows) {
        const int64_t b = a.row_ptr[w], e = a.row_ptr[w + 1];
        if (e - b > a.heavy_threshold) return false;
        u = Unit{w, b, e, -1, true};
        return true;
    }
    const int64_t s = w - a.n_rows;
    if (s >= a.n_segs) return false;
    const int64_t hr = a.seg_heavy[s];
    const int64_t row = a.heavy_rows[hr];
    const int64_t k = s - a.heavy_seg_ptr[hr];
    const int64_t b = a.row_ptr[row] + k * a.seg_len;
    const int64_t e = min(b + int64_t(a.seg_len), a.row_ptr[row + 1]);
    u = Unit{row, b, e, s, k == 0};
    return true;
}

__device__ __forceinline__ int32_t vertex_of(const grd_gat_args& a, int64_t row) {
    return a.out_idx ? a.out_idx[row] : static_cast<int32_t>(row);
}

// (max, sum-of-exp) pair combine for the online softmax; empty = (-inf, 0).
__device__ __forceinline__ void lse_merge(float& m, float& d, float m2, float d2) {
    if (m2 == -INFINITY) return;
    if (m == -INFINITY) {
        m = m2;
        d = d2;
        return;
    }
    const float mm = fmaxf(m, m2);
    d = d * expf(m - mm) + d2 * expf(m2 - mm);
    m = mm;
}

constexpr int kItems = 5;   // ceil((128 edges + self loop) / 32) scores per lane

// ---------------------------------------------------------------- forward --
// Scores of source u for heads [0, HM): s_u (H values at column hdp),
// vectorised when the head count allows (rows are 16-byte aligned).
template <int HM>
__device__ __forceinline__ void load_heads(const float* p, int H, float (&out)[HM]) {
    if (HM % 4 == 0 && H == HM) {          // 16-byte aligned: hdp and H are multiples of 4
#pragma unroll
        for (int c = 0; c < HM / 4; ++c) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(p) + c);
            out[4 * c] = q.x;
            out[4 * c + 1] = q.y;
            out[4 * c + 2] = q.z;
            out[4 * c + 3] = q.w;
        }
        return;
    }
#pragma unroll
    for (int h = 0; h < HM; ++h) out[h] = h < H ? __ldg(p + h) : 0.f;
}

// Scores z = LeakyReLU(s_u + t_v) of one unit's (<= 129) items, kItems per
// lane (item lane + 32 it), -inf where absent; all loads issued up front.
template <int HM>
__device__ __forceinline__ void unit_scores(const grd_gat_args& a, const Unit& un, int32_t v, int lane,
                                            float (&z)[kItems][HM]) {
    const int H = a.heads;
    const int64_t ne = un.end - un.beg;
    const int64_t n = ne + (un.self ? 1 : 0);
    float tv[HM];
    load_heads<HM>(a.st ? a.st + int64_t(v) * a.ld_st + H : a.p_ext + int64_t(v) * a.ld_ext + a.hdp + H, H, tv);
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
        const int64_t i = lane + kWarp * it;
        if (it > 0 && kWarp * it >= n) {       // warp-uniform early exit
#pragma unroll
            for (int h = 0; h < HM; ++h) z[it][h] = -INFINITY;
            continue;
        }
        const int32_t u = i < ne ? a.idx[un.beg + i] : v;
        float su[HM];
        load_heads<HM>(a.st ? a.st + int64_t(u) * a.ld_st : a.p_ext + int64_t(u) * a.ld_ext + a.hdp, H, su);
#pragma unroll
        for (int h = 0; h < HM; ++h) z[it][h] = (i < n && h < H) ? lrelu(su[h] + tv[h], a.slope) : -INFINITY;
    }
}

template <int HM>
__device__ __forceinline__ void write_alpha(const grd_gat_args& a, const Unit& un, int32_t v, int lane,
                                            const float (&z)[kItems][HM], const float (&mx)[HM],
                                            const float (&inv)[HM]) {
    const int H = a.heads;
    const int64_t ne = un.end - un.beg;
    const int64_t n = ne + (un.self ? 1 : 0);
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
        const int64_t i = lane + kWarp * it;
        if (i >= n) continue;
        float* dst = i < ne ? a.alpha + (un.beg + i) * H : a.alpha_self + int64_t(v) * H;
#pragma unroll
        for (int h = 0; h < HM; ++h)
            if (h < H) dst[h] = __expf(z[it][h] - mx[h]) * inv[h];
    }
}

// light rows: z already holds exp(z - max) (computed once for the sum)
template <int HM>
__device__ __forceinline__ void write_alpha_e(const grd_gat_args& a, const Unit& un, int32_t v, int lane,
                                              const float (&e)[kItems][HM], const float (&inv)[HM]) {
    const int H = a.heads;
    const int64_t ne = un.end - un.beg;
    const int64_t n = ne + (un.self ? 1 : 0);
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
        const int64_t i = lane + kWarp * it;
        if (i >= n) continue;
        float* dst = i < ne ? a.alpha + (un.beg + i) * H : a.alpha_self + int64_t(v) * H;
#pragma unroll
        for (int h = 0; h < HM; ++h)
            if (h < H) dst[h] = e[it][h] * inv[h];
    }
}

// Pass 1, one warp per unit: the unit's scores stay in registers; a light
// row is normalised in place, a heavy segment leaves its per-head (max, sum
// exp) in seg_scratch[seg][2H].  HM = head count rounded up to 1, 2, 4 or 8
// (register arrays sized to it).
template <int HM>
__global__ void __launch_bounds__(256) gat_softmax_kernel(grd_gat_args a) {
    const int lane = threadIdx.x & (kWarp - 1);
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const int64_t nl = a.n_rows - a.n_small - a.n_mid;   // rows of this kernel; segments follow
    Unit un;
    if (!unit_of(a, w < nl ? w : a.n_rows + (w - nl), un)) return;
    const int H = a.heads;
    const int32_t v = vertex_of(a, un.row);
    const int64_t n = un.end - un.beg + (un.self ? 1 : 0);
    float z[kItems][HM], mx[HM], sm[HM];
    unit_scores<HM>(a, un, v, lane, z);
#pragma unroll
    for (int h = 0; h < HM; ++h) {
        mx[h] = z[0][h];
#pragma unroll
        for (int it = 1; it < kItems; ++it) mx[h] = fmaxf(mx[h], z[it][h]);
        mx[h] = warp_max(mx[h]);
        sm[h] = 0.f;
#pragma unroll
        for (int it = 0; it < kItems; ++it) {
            // exp once (fast ex2 path); z keeps it for the normalisation below
            const float e = (h < H && lane + kWarp * it < n) ? __expf(z[it][h] - mx[h]) : 0.f;
            z[it][h] = e;
            sm[h] += e;
        }
        sm[h] = warp_sum(sm[h]);
    }
    if (un.seg >= 0) {
        float* part = a.seg_scratch + un.seg * 2 * H;
#pragma unroll
        for (int h = 0; h < HM; ++h)
            if (h < H && lane == h) {
                part[h] = mx[h];
                part[H + h] = sm[h];
            }
        return;
    }
    float inv[HM];
#pragma unroll
    for (int h = 0; h < HM; ++h) inv[h] = 1.f / sm[h];
    write_alpha_e<HM>(a, un, v, lane, z, inv);
}

// The low-degree tail (the last n_small rows, <= 3 in-edges each: 66 % of
// the rows of the products-shaped Kronecker graph, 40 % with none) at
// kSmallLanes lanes per row, one item (edge or self loop) per lane: a warp
// per such row left 28+ lanes idle and made the launch warp-count bound.
// Rows longer than promised still come out right (items strided by
// kSmallLanes, online (max, sum) merge, scores recomputed).
constexpr int kSmallLanes = 4;
constexpr int kMidLanes = 16;   // the n_mid rows before them (<= 15 in-edges)

template <int HM>
__device__ __forceinline__ void small_scores(const grd_gat_args& a, int64_t b, int64_t ne, int32_t v,
                                             int64_t i, const float (&tv)[HM], float (&z)[HM]) {
    const int32_t u = i < ne ? a.idx[b + i] : v;
    float su[HM];
    load_heads<HM>(a.st ? a.st + int64_t(u) * a.ld_st : a.p_ext + int64_t(u) * a.ld_ext + a.hdp, a.heads, su);
#pragma unroll
    for (int h = 0; h < HM; ++h) z[h] = h < a.heads ? lrelu(su[h] + tv[h], a.slope) : -INFINITY;
}

template <int HM, int L>
__global__ void __launch_bounds__(256) gat_softmax_small_kernel(grd_gat_args a, int64_t r0, int64_t r1) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int sub = threadIdx.x & (L - 1);
    const int64_t row = r0 + t / L;
    const int H = a.heads;
    int64_t b = 0, ne = -1;
    int32_t v = 0;
    float tv[HM];
    if (row < r1) {
        b = a.row_ptr[row];
        ne = a.row_ptr[row + 1] - b;
        v = vertex_of(a, row);
        load_heads<HM>(a.st ? a.st + int64_t(v) * a.ld_st + H : a.p_ext + int64_t(v) * a.ld_ext + a.hdp + H, H, tv);
    }
    float z0[HM], mx[HM], sm[HM];
#pragma unroll
    for (int h = 0; h < HM; ++h) {
        z0[h] = -INFINITY;
        mx[h] = -INFINITY;
        sm[h] = 0.f;
    }
    for (int64_t i = sub; i <= ne; i += L) {   // items 0..ne-1 edges, ne the self loop
        float z[HM];
        small_scores<HM>(a, b, ne, v, i, tv, z);
#pragma unroll
        for (int h = 0; h < HM; ++h) {
            if (i == sub) z0[h] = z[h];
            lse_merge(mx[h], sm[h], z[h], 1.f);
        }
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1)
#pragma unroll
        for (int h = 0; h < HM; ++h) {
            const float m2 = __shfl_xor_sync(0xffffffffu, mx[h], o);
            const float d2 = __shfl_xor_sync(0xffffffffu, sm[h], o);
            lse_merge(mx[h], sm[h], m2, d2);
        }
    float inv[HM];
#pragma unroll
    for (int h = 0; h < HM; ++h) inv[h] = 1.f / sm[h];
    for (int64_t i = sub; i <= ne; i += L) {
        float z[HM];
        if (i == sub) {
#pragma unroll
            for (int h = 0; h < HM; ++h) z[h] = z0[h];
        } else {
            small_scores<HM>(a, b, ne, v, i, tv, z);
        }
        float* dst = i < ne ? a.alpha + (b + i) * H : a.alpha_self + int64_t(v) * H;
#pragma unroll
        for (int h = 0; h < HM; ++h)
            if (h < H) dst[h] = __expf(z[h] - mx[h]) * inv[h];
    }
}

// Pass 1b, one warp per heavy row: merge the row's segment partials in a
// fixed order (lane-strided, then a butterfly) into the first segment's slot.
// Once per row: every segment warp merging all of its row's partials was
// quadratic in the segment count of a hub row.
template <int HM>
__global__ void __launch_bounds__(256) gat_softmax_merge_kernel(grd_gat_args a) {
    const int lane = threadIdx.x & (kWarp - 1);
    const int64_t hr = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    if (hr >= a.n_heavy) return;
    const int H = a.heads;
    const int64_t s0 = a.heavy_seg_ptr[hr], s1 = a.heavy_seg_ptr[hr + 1];
    float mx[HM], sm[HM];
#pragma unroll
    for (int h = 0; h < HM; ++h) {
        mx[h] = -INFINITY;
        sm[h] = 0.f;
    }
    for (int64_t j = s0 + lane; j < s1; j += kWarp) {
        const float* part = a.seg_scratch + j * 2 * H;
#pragma unroll
        for (int h = 0; h < HM; ++h)
            if (h < H) lse_merge(mx[h], sm[h], part[h], part[H + h]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int h = 0; h < HM; ++h) {
            const float m2 = __shfl_xor_sync(0xffffffffu, mx[h], o);
            const float d2 = __shfl_xor_sync(0xffffffffu, sm[h], o);
            lse_merge(mx[h], sm[h], m2, d2);
        }
    __syncwarp();   // every lane has read the partials before lane h overwrites slot s0
    float* out = a.seg_scratch + s0 * 2 * H;
#pragma unroll
    for (int h = 0; h < HM; ++h)
        if (h < H && lane == h) {
            out[h] = mx[h];
            out[H + h] = sm[h];
        }
}

// Pass 2, one warp per heavy segment: merge the row's segment partials in a
// fixed order (every warp of the row gets bit-identical statistics), then
// normalise this segment's scores (recomputed, loads issued up front).
template <int HM>
__global__ void __launch_bounds__(256) gat_softmax_heavy_kernel(grd_gat_args a) {
    const int lane = threadIdx.x & (kWarp - 1);
    const int64_t s = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    Unit un;
    if (!unit_of(a, a.n_rows + s, un)) return;
    const int H = a.heads;
    const int32_t v = vertex_of(a, un.row);
    float z[kItems][HM];
    unit_scores<HM>(a, un, v, lane, z);
    // the row's merged statistics (gat_softmax_merge_kernel) sit in the slot
    // of its first segment
    const int64_t hr = a.seg_heavy[s];
    const float* stat = a.seg_scratch + a.heavy_seg_ptr[hr] * 2 * H;
    float mx[HM], sm[HM];
#pragma unroll
    for (int h = 0; h < HM; ++h) {
        mx[h] = h < H ? __ldg(stat + h) : -INFINITY;
        sm[h] = h < H ? __ldg(stat + H + h) : 1.f;
    }
    float inv[HM];
#pragma unroll
    for (int h = 0; h < HM; ++h) inv[h] = 1.f / sm[h];
    write_alpha<HM>(a, un, v, lane, z, mx, inv);
}

// --------------------------------------------------------------- backward --
// One warp per unit of target v, kU in-edges in flight:
//   dalpha_uv,h = gO_v,h . P_u,h                      (row gather of P_u)
//   c_v,h       = sum_u alpha_uv,h dalpha_uv,h = gO_v,h . O_v,h
//   delta_uv,h  = alpha_uv,h (dalpha_uv,h - c_v,h) lrelu'(s_u,h + t_v,h)
//   dt_v,h      = sum_u delta_uv,h                    (column hdp + H + h)
// c comes from the stored forward aggregate (o_fwd; with a ReLU-masked gO,
// relu(O) gives the same dot), so every edge is independent and one pass
// suffices.  Per-head dot products are reduced through shared memory.
constexpr int kU = 4;

// Per-lane partial dot products live in part[][j][.] with every head's cph
// chunks followed by one pad slot and rows kPartStride (= 4 mod 32) apart:
// the head sums then read 16 (edge, head) slots on distinct banks (the
// unpadded layout made them 6.6-way bank conflicts: 85 % of the kernel's
// shared-load wavefronts, ncu).
constexpr int kPartStride = 100;

template <int NV>
__global__ void __launch_bounds__(256) gat_edge_bwd_kernel(grd_gat_args a) {
    __shared__ float part[8][kU][kPartStride];
    __shared__ float cs[8][kMaxHeads];
    const int lane = threadIdx.x & (kWarp - 1);
    const int wib = threadIdx.x / kWarp;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    Unit un;
    if (!unit_of(a, w, un)) return;
    const int H = a.heads;
    const int q4 = a.hdp / 4;
    const int cph = a.dhp / 4;
    const int32_t v = vertex_of(a, un.row);
    const int hs = cph + 1;                    // padded head slot
    int pq[NV];                                // padded slot of chunk lane + 32 c
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        const int q = lane + c * kWarp;
        pq[c] = (q / cph) * hs + q % cph;
    }
    float4 g[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        const int q = lane + c * kWarp;
        float d = 0.f;
        g[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q < q4) {
            g[c] = *reinterpret_cast<const float4*>(a.grad_o + int64_t(v) * a.ld_go + 4 * q);
            const float4 o = *reinterpret_cast<const float4*>(a.o_fwd + int64_t(v) * a.ld_o + 4 * q);
            d = g[c].x * o.x + g[c].y * o.y + g[c].z * o.z + g[c].w * o.w;
        }
        if (q < q4) part[wib][0][pq[c]] = d;
    }
    __syncwarp();
    if (lane < H) {
        float c = 0.f;
        for (int k = 0; k < cph; ++k) c += part[wib][0][lane * hs + k];
        cs[wib][lane] = c;
    }
    __syncwarp();
    // lane L < kU*H owns (edge L / H of the batch, head L % H)
    const bool scal = lane < kU * H;
    const int my_h = lane % H, my_j = lane / H;
    const float c_my = cs[wib][my_h];
    const float t_my = a.p_ext[int64_t(v) * a.ld_ext + a.hdp + H + my_h];
    const int64_t ne = un.end - un.beg;
    const int64_t n = ne + (un.self ? 1 : 0);
    float dt = 0.f;
    for (int64_t i0 = 0; i0 < n; i0 += kU) {
        float4 p[kU][NV];
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            const int64_t i = i0 + j;
            const int32_t u = i < ne ? a.idx[un.beg + i] : v;
            const float* pu = a.p_ext + int64_t(u) * a.ld_ext;
#pragma unroll
            for (int c = 0; c < NV; ++c) {
                const int q = lane + c * kWarp;
                p[j][c] = (i < n && q < q4) ? __ldg(reinterpret_cast<const float4*>(pu + 4 * q))
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        const int64_t im = i0 + my_j;
        const bool mine = scal && im < n;
        float s_my = 0.f, al_my = 0.f;
        if (mine) {
            const int32_t u = im < ne ? a.idx[un.beg + im] : v;
            s_my = a.p_ext[int64_t(u) * a.ld_ext + a.hdp + my_h];   // beside the gathered P_u row
            al_my = im < ne ? a.alpha[(un.beg + im) * H + my_h] : a.alpha_self[int64_t(v) * H + my_h];
        }
#pragma unroll
        for (int j = 0; j < kU; ++j)
#pragma unroll
            for (int c = 0; c < NV; ++c)
                if (lane + c * kWarp < q4)
                    part[wib][j][pq[c]] = g[c].x * p[j][c].x + g[c].y * p[j][c].y +
                                          g[c].z * p[j][c].z + g[c].w * p[j][c].w;
        __syncwarp();
        if (mine) {
            float da = 0.f;
            for (int k = 0; k < cph; ++k) da += part[wib][my_j][my_h * hs + k];
            const float d = al_my * (da - c_my) * lrelu_grad(s_my + t_my, a.slope);
            if (im < ne)
                a.delta[(un.beg + im) * H + my_h] = d;
            else
                a.delta_self[int64_t(v) * H + my_h] = d;
            dt += d;
        }
        __syncwarp();
    }
    part[wib][0][lane] = scal ? dt : 0.f;
    __syncwarp();
    if (lane < H) {
        float t = 0.f;
        for (int j = 0; j < kU; ++j) t += part[wib][0][j * H + lane];
        if (un.seg < 0)
            a.grad_ext[int64_t(v) * a.ld_gext + a.hdp + H + lane] = t;
        else
            a.seg_scratch[un.seg * H + lane] = t;
    }
}

// Source score gradient ds_u,h = sum over u's out-edges of delta (edges
// addressed through the transposed CSR's permutation) + the self loop.
// L lanes per unit of the out-edge CSR: a warp (L = 32) for rows [r0, r1)
// and then every heavy segment, 16 / 4 lanes for the low-degree rows
// (AggSpec.n_mid / n_small, the same split as the edge softmax).
template <int L, int HM>
__global__ void __launch_bounds__(256) gat_src_grad_kernel(grd_gat_args a, int64_t r0, int64_t r1, int col0) {
    const int sub = threadIdx.x & (L - 1);
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / L;
    Unit un{0, 0, 0, -1, false};
    bool ok;
    if (w < r1 - r0)
        ok = unit_of(a, r0 + w, un);
    else
        ok = L == kWarp && unit_of(a, a.n_rows + (w - (r1 - r0)), un);
    if (L == kWarp && !ok) return;   // warp-uniform
    const int H = a.heads;
    float ds[HM];
#pragma unroll
    for (int h = 0; h < HM; ++h) ds[h] = 0.f;
    if (ok)
        for (int64_t i = un.beg + sub; i < un.end; i += L) {
            const float* de = a.delta + (a.edge_perm ? int64_t(a.edge_perm[i]) : i) * H;
#pragma unroll
            for (int h = 0; h < HM; ++h)
                if (h < H) ds[h] += de[h];
        }
#pragma unroll
    for (int h = 0; h < HM; ++h)
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) ds[h] += __shfl_xor_sync(0xffffffffu, ds[h], o);
    if (!ok) return;
    const int32_t r = vertex_of(a, un.row);
#pragma unroll
    for (int h = 0; h < HM; ++h) {
        if (h >= H || (h % L) != sub) continue;
        const float t = ds[h] + (un.self ? a.delta_self[int64_t(r) * H + h] : 0.f);
        if (un.seg < 0)
            a.grad_ext[int64_t(r) * a.ld_gext + col0 + h] = t;
        else
            a.seg_scratch[un.seg * H + h] = t;
    }
}

template <int HM>
void launch_src_grad(const grd_gat_args& a, cudaStream_t st, int col0) {
    const int64_t r_small = a.n_rows - a.n_small, r_mid = r_small - a.n_mid;
    const int64_t units = r_mid + a.n_segs;
    if (units > 0)
        gat_src_grad_kernel<kWarp, HM><<<static_cast<unsigned>((units * kWarp + 255) / 256), 256, 0, st>>>(a, 0, r_mid, col0);
    if (a.n_mid > 0)
        gat_src_grad_kernel<kMidLanes, HM><<<static_cast<unsigned>((a.n_mid * kMidLanes + 255) / 256), 256, 0, st>>>(
            a, r_mid, r_small, col0);
    if (a.n_small > 0)
        gat_src_grad_kernel<kSmallLanes, HM>
            <<<static_cast<unsigned>((a.n_small * kSmallLanes + 255) / 256), 256, 0, st>>>(a, r_small, a.n_rows, col0);
}

// Heavy rows of the two backward passes: one warp per heavy row sums its
// segments' per-head partials (fixed order) into grad_ext column col0 + h.
__global__ void __launch_bounds__(256) gat_heavy_sum_kernel(grd_gat_args a, int col0) {
    const int lane = threadIdx.x & (kWarp - 1);
    const int64_t hr = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    if (hr >= a.n_heavy) return;
    const int H = a.heads;
    const int64_t s0 = a.heavy_seg_ptr[hr], s1 = a.heavy_seg_ptr[hr + 1];
    float t[kMaxHeads];
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) t[h] = 0.f;
    for (int64_t j = s0 + lane; j < s1; j += kWarp)
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h)
            if (h < H) t[h] += a.seg_scratch[j * H + h];
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) t[h] = warp_sum(t[h]);
    const int32_t r = vertex_of(a, a.heavy_rows[hr]);
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h)
        if (h < H && lane == h) a.grad_ext[int64_t(r) * a.ld_gext + col0 + h] = t[h];
}

// W_ext = [W | W a_src | W a_dst]  (rows d_in, thread per (row, column))
__global__ void gat_build_wext_kernel(const float* w, int64_t ldw, const float* att, int64_t d_in, int H, int dh,
                                      int dhp, float* wext, int64_t ld_ext) {
    const int hdp = H * dhp;
    const int64_t cols = hdp + 2 * H;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= d_in * cols) return;
    const int64_t row = i / cols;
    const int col = static_cast<int>(i % cols);
    float v;
    if (col < hdp) {
        v = w[row * ldw + col];
    } else {
        const int k = col - hdp;                     // 0..2H-1
        const int h = k % H;
        const float* vec = att + (k / H) * H * dhp + h * dhp;    // a_src or a_dst row h
        float s = 0.f;
        for (int d = 0; d < dh; ++d) s = fmaf(w[row * ldw + h * dhp + d], vec[d], s);
        v = s;
    }
    wext[row * ld_ext + col] = v;
}

// dW = dW_ext[:, P] + dW_ext[:, s_h] a_src_h^T + dW_ext[:, t_h] a_dst_h^T;
// da_src_h = W_h^T dW_ext[:, s_h], da_dst_h likewise; then SGD on W and att.
__global__ void gat_param_grads_kernel(const float* dwext, int64_t ld_ext, float* w, int64_t ldw, float* att,
                                       int64_t d_in, int H, int dh, int dhp, float* dw, float* datt, float lr) {
    const int hdp = H * dhp;
    const int64_t nw = d_in * hdp;
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < nw) {
        const int64_t row = i / hdp;
        const int col = static_cast<int>(i % hdp);
        const int h = col / dhp, d = col % dhp;
        float g = 0.f;
        if (d < dh)
            g = dwext[row * ld_ext + col] + dwext[row * ld_ext + hdp + h] * att[h * dhp + d] +
                dwext[row * ld_ext + hdp + H + h] * att[H * dhp + h * dhp + d];
        dw[row * ldw + col] = g;
        return;
    }
    const int64_t j = i - nw;                    // attention vectors: 2 x H x dhp
    if (j >= 2 * H * dhp) return;
    const int which = static_cast<int>(j / (H * dhp));
    const int h = static_cast<int>((j % (H * dhp)) / dhp), d = static_cast<int>(j % dhp);
    float g = 0.f;
    if (d < dh)
        for (int64_t row = 0; row < d_in; ++row)
            g = fmaf(w[row * ldw + h * dhp + d], dwext[row * ld_ext + hdp + which * H + h], g);
    datt[j] = g;
}

__global__ void sgd_kernel(float* w, const float* g, int64_t n, float lr) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) w[i] -= lr * g[i];
}

// Last layer: out[v, j] = mean_h O[v, h*dhp + j]; backward spreads g/H.
__global__ void head_mean_kernel(const float* o, int64_t ldo, int64_t n_rows, int H, int dh, int dhp, float* out,
                                 int64_t ld_out, int backward) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_rows * dhp) return;
    const int64_t r = i / dhp;
    const int j = static_cast<int>(i % dhp);
    const float inv = 1.0f / static_cast<float>(H);
    if (!backward) {
        if (j >= dh) return;
        float s = 0.f;
        for (int h = 0; h < H; ++h) s += o[r * ldo + h * dhp + j];
        out[r * ld_out + j] = s * inv;
    } else {
        const float g = j < dh ? o[r * ldo + j] * inv : 0.f;   // o = dL/dlogits here
        for (int h = 0; h < H; ++h) out[r * ld_out + h * dhp + j] = g;
    }
}

unsigned warps_blocks(int64_t rows) { return static_cast<unsigned>((rows * kWarp + 255) / 256); }
unsigned blocks(int64_t n) { return static_cast<unsigned>((n + 255) / 256); }

unsigned unit_blocks(const grd_gat_args& a) { return warps_blocks(a.n_rows + a.n_segs); }

int check_units(const grd_gat_args* a, const char* what) {
    if (!a || a->heads < 1 || a->heads > kMaxHeads) return fail(kErrArg, "%s: heads must be 1..%d", what, kMaxHeads);
    if (a->heavy_threshold < 0 || a->heavy_threshold > 128 || a->seg_len < 1 || a->seg_len > 128)
        return fail(kErrArg, "%s: heavy_threshold and seg_len must be <= 128", what);
    if (a->n_segs > 0 && (!a->heavy_rows || !a->heavy_seg_ptr || !a->seg_heavy || !a->seg_scratch))
        return fail(kErrArg, "%s: heavy rows need their segmentation and seg_scratch", what);
    return 0;
}

// Per-edge sums of delta into a per-row column of grad_ext (col0 + h): over
// the pull CSR with edge_perm (ds_u, col0 = hdp) or over the forward CSR in
// its own edge order (dt_v, col0 = hdp + H, edge_perm null).
int edge_sums(const grd_gat_args& a, cudaStream_t st, int col0, const char* what) {
    const int H = a.heads;
    if (H == 1)
        launch_src_grad<1>(a, st, col0);
    else if (H == 2)
        launch_src_grad<2>(a, st, col0);
    else if (H <= 4)
        launch_src_grad<4>(a, st, col0);
    else
        launch_src_grad<8>(a, st, col0);
    int rc = launch_status(what);
    if (rc || a.n_heavy == 0) return rc;
    gat_heavy_sum_kernel<<<warps_blocks(a.n_heavy), 256, 0, st>>>(a, col0);
    return launch_status("gat_heavy_sum");
}

// ------------------------------------------------ fused pull backward --
// One warp per unit of the transposed pull (source u, its out-edges u -> v),
// kU out-edges per batch:
//   gO_v rows gathered ONCE per edge serve both the attention-score
//   gradient (dalpha_uv,h = gO_v,h . P_u,h against u's own P row, held in
//   registers) and dP_u += alpha_uv gO_v;
//   delta_uv,h = alpha (dalpha - c_v,h) lrelu'(s_u,h + t_v,h) is written at
//   the edge's forward position and summed into ds_u,h.
// The separate edge backward (grd_gat_softmax_bwd) gathered P_u once per
// in-edge of every target: the same row traffic again.  dP_u sums its
// edges in pull order with the self term last (heavy rows: each segment's
// edges in order, segment partials in segment order, then the self term) —
// a fixed order, deterministic run to run.  Per-head dot products are
// reduced through the same padded shared layout as the edge backward.
template <int NV, int MINB>
__global__ void __launch_bounds__(256, MINB) gat_pull_bwd_kernel(grd_gat_args a) {
    __shared__ float part[8][kU][kPartStride];
    __shared__ float alw[8][kU][kMaxHeads];
    const int lane = threadIdx.x & (kWarp - 1);
    const int wib = threadIdx.x / kWarp;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    Unit un;
    if (!unit_of(a, w, un)) return;
    const int H = a.heads;
    const int q4 = a.hdp / 4;
    const int cph = a.dhp / 4;
    const int hs = cph + 1;
    const int32_t u = vertex_of(a, un.row);
    const bool with_self = un.self && un.seg < 0;   // heavy rows: the self term after the segments
    int pq[NV], hc[NV];
    float4 pu[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        const int q = lane + c * kWarp;
        pq[c] = (q / cph) * hs + q % cph;
        hc[c] = min(q / cph, H - 1);
        pu[c] = q < q4 ? __ldg(reinterpret_cast<const float4*>(a.p_ext + int64_t(u) * a.ld_ext + 4 * q))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const bool scal = lane < kU * H;
    const int my_h = lane % H, my_j = lane / H;
    const float s_my = a.p_ext[int64_t(u) * a.ld_ext + a.hdp + my_h];
    const int64_t ne = un.end - un.beg;
    const int64_t n = ne + (with_self ? 1 : 0);
    float4 acc[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    float ds = 0.f;
    for (int64_t i0 = 0; i0 < n; i0 += kU) {
        float4 g[kU][NV];
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            const int64_t i = i0 + j;
            const int32_t v = i < ne ? a.idx[un.beg + i] : u;
            const float* gv = a.grad_o + int64_t(v) * a.ld_go;
#pragma unroll
            for (int c = 0; c < NV; ++c) {
                const int q = lane + c * kWarp;
                g[j][c] = (i < n && q < q4) ? __ldg(reinterpret_cast<const float4*>(gv + 4 * q))
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        const int64_t im = i0 + my_j;
        const bool mine = scal && im < n;
        float al = 0.f, tv = 0.f, cv = 0.f;
        int64_t ef = -1;
        if (mine) {
            int32_t v = u;
            if (im < ne) {
                const int64_t e = un.beg + im;
                v = a.idx[e];
                ef = a.edge_perm[e];
                al = a.alpha_t ? a.alpha_t[e * H + my_h] : a.alpha[ef * H + my_h];
            } else {
                al = a.alpha_self[int64_t(u) * H + my_h];
            }
            tv = a.st ? a.st[int64_t(v) * a.ld_st + H + my_h] : a.p_ext[int64_t(v) * a.ld_ext + a.hdp + H + my_h];
            cv = a.c_dot[int64_t(v) * H + my_h];
            alw[wib][my_j][my_h] = al;
        }
#pragma unroll
        for (int j = 0; j < kU; ++j)
#pragma unroll
            for (int c = 0; c < NV; ++c)
                if (lane + c * kWarp < q4)
                    part[wib][j][pq[c]] = g[j][c].x * pu[c].x + g[j][c].y * pu[c].y + g[j][c].z * pu[c].z +
                                          g[j][c].w * pu[c].w;
        __syncwarp();
        if (mine) {
            float da = 0.f;
            for (int k = 0; k < cph; ++k) da += part[wib][my_j][my_h * hs + k];
            const float d = al * (da - cv) * lrelu_grad(s_my + tv, a.slope);
            if (im < ne)
                a.delta[ef * H + my_h] = d;
            else
                a.delta_self[int64_t(u) * H + my_h] = d;
            ds += d;
        }
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            if (i0 + j >= n) break;
#pragma unroll
            for (int c = 0; c < NV; ++c) acc[c] = f4_fma(alw[wib][j][hc[c]], g[j][c], acc[c]);
        }
        __syncwarp();
    }
    part[wib][0][lane] = scal ? ds : 0.f;
    __syncwarp();
    float dsh = 0.f;
    if (lane < H)
        for (int j = 0; j < kU; ++j) dsh += part[wib][0][j * H + lane];
    const int ldw = (a.hdp + H + 3) / 4 * 4;
    float* dst = un.seg < 0 ? a.grad_ext + int64_t(u) * a.ld_gext : a.seg_wide + un.seg * ldw;
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        const int q = lane + c * kWarp;
        if (q < q4) *reinterpret_cast<float4*>(dst + 4 * q) = acc[c];
    }
    if (lane < H) dst[a.hdp + lane] = dsh;
}

// Heavy pull rows: one warp per row sums its segments' dP / ds partials in
// segment order, then adds the self term (alpha_self gO_u, and delta_self
// from u's own rows) exactly as the unfused pull's finish does.
template <int NV>
__global__ void __launch_bounds__(256) gat_pull_heavy_kernel(grd_gat_args a) {
    __shared__ float part[8][kPartStride];
    const int lane = threadIdx.x & (kWarp - 1);
    const int wib = threadIdx.x / kWarp;
    const int64_t hr = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    if (hr >= a.n_heavy) return;
    const int H = a.heads;
    const int q4 = a.hdp / 4;
    const int cph = a.dhp / 4;
    const int hs = cph + 1;
    const int ldw = (a.hdp + H + 3) / 4 * 4;
    const int32_t u = vertex_of(a, a.heavy_rows[hr]);
    const int64_t s0 = a.heavy_seg_ptr[hr], s1 = a.heavy_seg_ptr[hr + 1];
    float4 acc[NV], gu[NV], pu[NV];
    int hc[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        const int q = lane + c * kWarp;
        hc[c] = min(q / cph, H - 1);
        acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        gu[c] = pu[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q < q4) {
            for (int64_t s = s0; s < s1; ++s)
                acc[c] = f4_add(acc[c], *reinterpret_cast<const float4*>(a.seg_wide + s * ldw + 4 * q));
            gu[c] = *reinterpret_cast<const float4*>(a.grad_o + int64_t(u) * a.ld_go + 4 * q);
            pu[c] = *reinterpret_cast<const float4*>(a.p_ext + int64_t(u) * a.ld_ext + 4 * q);
            part[wib][(q / cph) * hs + q % cph] = gu[c].x * pu[c].x + gu[c].y * pu[c].y + gu[c].z * pu[c].z +
                                                  gu[c].w * pu[c].w;
        }
    }
    __syncwarp();
    float ds = 0.f, d = 0.f;
    if (lane < H) {
        for (int64_t s = s0; s < s1; ++s) ds += a.seg_wide[s * ldw + a.hdp + lane];
        float da = 0.f;
        for (int k = 0; k < cph; ++k) da += part[wib][lane * hs + k];
        const float al = a.alpha_self[int64_t(u) * H + lane];
        const float tu = a.st ? a.st[int64_t(u) * a.ld_st + H + lane] : a.p_ext[int64_t(u) * a.ld_ext + a.hdp + H + lane];
        const float su = a.p_ext[int64_t(u) * a.ld_ext + a.hdp + lane];
        d = al * (da - a.c_dot[int64_t(u) * H + lane]) * lrelu_grad(su + tu, a.slope);
        a.delta_self[int64_t(u) * H + lane] = d;
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < NV; ++c) {
        const int q = lane + c * kWarp;
        const float al = a.alpha_self[int64_t(u) * H + hc[c]];
        if (q < q4)
            *reinterpret_cast<float4*>(a.grad_ext + int64_t(u) * a.ld_gext + 4 * q) = f4_fma(al, gu[c], acc[c]);
    }
    if (lane < H) a.grad_ext[int64_t(u) * a.ld_gext + a.hdp + lane] = ds + d;
}

// c[r, h] = gO_r,h . O_r,h, 16-byte chunks summed in order (thread per (row, head))
__global__ void gat_row_dots_kernel(const float* __restrict__ g, int64_t ldg, const float* __restrict__ o,
                                    int64_t ldo, int64_t n_rows, int H, int dhp, float* __restrict__ c) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_rows * H) return;
    const int64_t r = i / H;
    const int h = static_cast<int>(i % H);
    const float4* gr = reinterpret_cast<const float4*>(g + r * ldg + h * dhp);
    const float4* orow = reinterpret_cast<const float4*>(o + r * ldo + h * dhp);
    float s = 0.f;
    for (int k = 0; k < dhp / 4; ++k) {
        const float4 x = __ldg(gr + k), y = __ldg(orow + k);
        s += x.x * y.x + x.y * y.y + x.z * y.z + x.w * y.w;
    }
    c[i] = s;
}

}  // namespace

extern "C" int grd_gat_softmax(const grd_gat_args* args, void* stream) {
    clear_error();
    if (int rc = check_units(args, "gat_softmax")) return rc;
    if (args->n_rows == 0) return 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int H = args->heads;
    if (args->n_small < 0 || args->n_mid < 0 || args->n_small + args->n_mid > args->n_rows)
        return fail(kErrArg, "gat_softmax: n_small %lld + n_mid %lld outside [0, n_rows]",
                    (long long)args->n_small, (long long)args->n_mid);
    const int64_t r_mid = args->n_rows - args->n_small - args->n_mid, r_small = args->n_rows - args->n_small;
    const unsigned nb = warps_blocks(r_mid + args->n_segs);
    if (nb > 0) {
        if (H == 1)
            gat_softmax_kernel<1><<<nb, 256, 0, st>>>(*args);
        else if (H == 2)
            gat_softmax_kernel<2><<<nb, 256, 0, st>>>(*args);
        else if (H <= 4)
            gat_softmax_kernel<4><<<nb, 256, 0, st>>>(*args);
        else
            gat_softmax_kernel<8><<<nb, 256, 0, st>>>(*args);
    }
    if (args->n_mid > 0) {
        const unsigned sb = static_cast<unsigned>((args->n_mid * kMidLanes + 255) / 256);
        if (H == 1)
            gat_softmax_small_kernel<1, kMidLanes><<<sb, 256, 0, st>>>(*args, r_mid, r_small);
        else if (H == 2)
            gat_softmax_small_kernel<2, kMidLanes><<<sb, 256, 0, st>>>(*args, r_mid, r_small);
        else if (H <= 4)
            gat_softmax_small_kernel<4, kMidLanes><<<sb, 256, 0, st>>>(*args, r_mid, r_small);
        else
            gat_softmax_small_kernel<8, kMidLanes><<<sb, 256, 0, st>>>(*args, r_mid, r_small);
    }
    if (args->n_small > 0) {
        const unsigned sb = static_cast<unsigned>((args->n_small * kSmallLanes + 255) / 256);
        const int64_t r1 = args->n_rows;
        if (H == 1)
            gat_softmax_small_kernel<1, kSmallLanes><<<sb, 256, 0, st>>>(*args, r_small, r1);
        else if (H == 2)
            gat_softmax_small_kernel<2, kSmallLanes><<<sb, 256, 0, st>>>(*args, r_small, r1);
        else if (H <= 4)
            gat_softmax_small_kernel<4, kSmallLanes><<<sb, 256, 0, st>>>(*args, r_small, r1);
        else
            gat_softmax_small_kernel<8, kSmallLanes><<<sb, 256, 0, st>>>(*args, r_small, r1);
    }
    int rc = launch_status("gat_softmax");
    if (rc || args->n_segs == 0) return rc;
    if (H == 1)
        gat_softmax_merge_kernel<1><<<warps_blocks(args->n_heavy), 256, 0, st>>>(*args);
    else if (H == 2)
        gat_softmax_merge_kernel<2><<<warps_blocks(args->n_heavy), 256, 0, st>>>(*args);
    else if (H <= 4)
        gat_softmax_merge_kernel<4><<<warps_blocks(args->n_heavy), 256, 0, st>>>(*args);
    else
        gat_softmax_merge_kernel<8><<<warps_blocks(args->n_heavy), 256, 0, st>>>(*args);
    if ((rc = launch_status("gat_softmax_merge"))) return rc;
    if (H == 1)
        gat_softmax_heavy_kernel<1><<<warps_blocks(args->n_segs), 256, 0, st>>>(*args);
    else if (H == 2)
        gat_softmax_heavy_kernel<2><<<warps_blocks(args->n_segs), 256, 0, st>>>(*args);
    else if (H <= 4)
        gat_softmax_heavy_kernel<4><<<warps_blocks(args->n_segs), 256, 0, st>>>(*args);
    else
        gat_softmax_heavy_kernel<8><<<warps_blocks(args->n_segs), 256, 0, st>>>(*args);
    return launch_status("gat_softmax_heavy");
}

extern "C" int grd_gat_softmax_bwd(const grd_gat_args* args, void* stream) {
    clear_error();
    if (int rc = check_units(args, "gat_softmax_bwd")) return rc;
    if (args->n_rows == 0) return 0;
    if (args->hdp > 256 || args->hdp % 4 || args->dhp % 4 || !args->grad_o || !args->o_fwd ||
        args->ld_go % 4 || args->ld_o % 4 || args->ld_ext % 4)
        return fail(kErrArg, "gat_softmax_bwd: hdp <= 256, 16-byte aligned rows, grad_o and o_fwd required");
    if (args->n_rows == 0) return 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (args->hdp <= 128)
        gat_edge_bwd_kernel<1><<<unit_blocks(*args), 256, 0, st>>>(*args);
    else
        gat_edge_bwd_kernel<2><<<unit_blocks(*args), 256, 0, st>>>(*args);
    int rc = launch_status("gat_edge_bwd");
    if (rc || args->n_heavy == 0) return rc;
    gat_heavy_sum_kernel<<<warps_blocks(args->n_heavy), 256, 0, st>>>(*args, args->hdp + args->heads);
    return launch_status("gat_heavy_sum");
}

extern "C" int grd_gat_src_grad(const grd_gat_args* args, void* stream) {
    clear_error();
    if (int rc = check_units(args, "gat_src_grad")) return rc;
    if (args->n_rows == 0) return 0;
    if (!args->edge_perm) return fail(kErrArg, "gat_src_grad: needs edge_perm");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (args->n_small < 0 || args->n_mid < 0 || args->n_small + args->n_mid > args->n_rows)
        return fail(kErrArg, "gat_src_grad: bad n_small / n_mid");
    return edge_sums(*args, st, args->hdp, "gat_src_grad");
}

__global__ void gat_pack_scores_kernel(const float* __restrict__ p_ext, int64_t ld_ext, int64_t n_rows, int H,
                                       int hdp, float* __restrict__ st, int64_t ld_st) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int w = 2 * H;
    if (i >= n_rows * w) return;
    const int64_t r = i / w;
    const int c = static_cast<int>(i % w);
    st[r * ld_st + c] = p_ext[r * ld_ext + hdp + c];
}

extern "C" int grd_gat_pack_scores(const float* p_ext, int64_t ld_ext, int64_t n_rows, int32_t heads, int32_t hdp,
                                   float* st, int64_t ld_st, void* stream) {
    clear_error();
    if (n_rows == 0) return 0;
    if (!p_ext || !st || heads < 1 || heads > kMaxHeads || ld_st < 2 * heads || n_rows < 0)
        return fail(kErrArg, "gat_pack_scores: bad arguments");
    const int64_t n = n_rows * 2 * heads;
    gat_pack_scores_kernel<<<blocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(p_ext, ld_ext, n_rows, heads,
                                                                                      hdp, st, ld_st);
    return launch_status("gat_pack_scores");
}

extern "C" int grd_gat_build_wext(const float* w, int64_t ldw, const float* att, int64_t d_in, int32_t heads,
                                  int32_t dh, int32_t dhp, float* wext, int64_t ld_ext, void* stream) {
    clear_error();
    const int64_t n = d_in * (int64_t(heads) * dhp + 2 * heads);
    gat_build_wext_kernel<<<blocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(w, ldw, att, d_in, heads, dh,
                                                                                    dhp, wext, ld_ext);
    return launch_status("gat_build_wext");
}

extern "C" int grd_gat_param_grads(const float* dwext, int64_t ld_ext, float* w, int64_t ldw, float* att,
                                   int64_t d_in, int32_t heads, int32_t dh, int32_t dhp, float* dw, float* datt,
                                   float lr, void* stream) {
    clear_error();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t n = d_in * int64_t(heads) * dhp + 2 * int64_t(heads) * dhp;
    gat_param_grads_kernel<<<blocks(n), 256, 0, st>>>(dwext, ld_ext, w, ldw, att, d_in, heads, dh, dhp, dw, datt,
                                                      lr);
    int rc = launch_status("gat_param_grads");
    if (rc || lr == 0.f) return rc;
    const int64_t nw = d_in * ldw, na = 2 * int64_t(heads) * dhp;
    sgd_kernel<<<blocks(nw), 256, 0, st>>>(w, dw, nw, lr);
    sgd_kernel<<<blocks(na), 256, 0, st>>>(att, datt, na, lr);
    return launch_status("gat_sgd");
}

extern "C" int grd_head_mean(const float* o, int64_t ldo, int64_t n_rows, int32_t heads, int32_t dh, int32_t dhp,
                             float* out, int64_t ld_out, int32_t backward, void* stream) {
    clear_error();
    if (n_rows == 0) return 0;
    head_mean_kernel<<<blocks(n_rows * dhp), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        o, ldo, n_rows, heads, dh, dhp, out, ld_out, backward);
    return launch_status("head_mean");
}

extern "C" int grd_gat_pull_bwd(const grd_gat_args* args, void* stream) {
    clear_error();
    if (int rc = check_units(args, "gat_pull_bwd")) return rc;
    if (args->n_rows == 0) return 0;
    if (args->hdp > 256 || args->hdp % 4 || args->dhp % 4 || !args->grad_o || !args->c_dot || !args->edge_perm ||
        !args->alpha || !args->alpha_self || !args->delta || !args->delta_self || !args->grad_ext ||
        args->ld_go % 4 || args->ld_ext % 4 || args->ld_gext % 4)
        return fail(kErrArg, "gat_pull_bwd: hdp <= 256, 16-byte aligned rows, all operands required");
    if (args->n_segs > 0 && !args->seg_wide) return fail(kErrArg, "gat_pull_bwd: heavy rows need seg_wide");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // resident blocks per SM the register budget is capped for
    // (GRD_GAT_PULL_MINB sweep hook; products_gat, hdp 256: 2 -> 123
    // registers, 17.7 ms per launch; 3 -> 80 (32 B spill), 15.8 ms; 4 -> 64,
    // 20.7 ms; hdp <= 128 fits 64 registers without spilling)
    static int minb = -1;
    if (minb < 0) {
        const char* e = getenv("GRD_GAT_PULL_MINB");
        minb = e ? atoi(e) : 3;
    }
    const unsigned nb = unit_blocks(*args);
    if (args->hdp <= 128) {
        if (minb >= 3) gat_pull_bwd_kernel<1, 4><<<nb, 256, 0, st>>>(*args);
        else gat_pull_bwd_kernel<1, 2><<<nb, 256, 0, st>>>(*args);
    } else {
        if (minb >= 4) gat_pull_bwd_kernel<2, 4><<<nb, 256, 0, st>>>(*args);
        else if (minb == 3) gat_pull_bwd_kernel<2, 3><<<nb, 256, 0, st>>>(*args);
        else gat_pull_bwd_kernel<2, 2><<<nb, 256, 0, st>>>(*args);
    }
    int rc = launch_status("gat_pull_bwd");
    if (rc || args->n_heavy == 0) return rc;
    if (args->hdp <= 128)
        gat_pull_heavy_kernel<1><<<warps_blocks(args->n_heavy), 256, 0, st>>>(*args);
    else
        gat_pull_heavy_kernel<2><<<warps_blocks(args->n_heavy), 256, 0, st>>>(*args);
    return launch_status("gat_pull_heavy");
}

extern "C" int grd_gat_dst_grad(const grd_gat_args* args, void* stream) {
    clear_error();
    if (int rc = check_units(args, "gat_dst_grad")) return rc;
    if (args->n_rows == 0) return 0;
    if (args->n_small < 0 || args->n_mid < 0 || args->n_small + args->n_mid > args->n_rows)
        return fail(kErrArg, "gat_dst_grad: bad n_small / n_mid");
    grd_gat_args a = *args;
    a.edge_perm = nullptr;   // the forward CSR's own edge order
    return edge_sums(a, static_cast<cudaStream_t>(stream), a.hdp + a.heads, "gat_dst_grad");
}

extern "C" int grd_gat_row_dots(const float* g, int64_t ld_g, const float* o, int64_t ld_o, int64_t n_rows,
                                int32_t heads, int32_t dhp, float* c, void* stream) {
    clear_error();
    if (n_rows == 0) return 0;
    if (!g || !o || !c || heads < 1 || dhp % 4 || ld_g % 4 || ld_o % 4)
        return fail(kErrArg, "gat_row_dots: bad arguments");
    gat_row_dots_kernel<<<blocks(n_rows * heads), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        g, ld_g, o, ld_o, n_rows, heads, dhp, c);
    return launch_status("gat_row_dots");
}
