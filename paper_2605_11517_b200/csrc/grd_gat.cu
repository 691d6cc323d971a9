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

#include "../../include/grinder_b200.h"
#include "grd_common.h"

using namespace grd;

namespace {

constexpr int kWarp = 32;
constexpr int kMaxHeads = 8;

__device__ __forceinline__ float lrelu(float z, float slope) { return z > 0.f ? z : z * slope; }
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

// ---------------------------------------------------------------- forward --
// Warp per target row; lanes stride over the row's edges (self loop last).
// Three passes over H scalars per edge: max, sum of exp, normalised alpha.
__global__ void __launch_bounds__(256) gat_softmax_kernel(grd_gat_args a) {
    const int lane = threadIdx.x & (kWarp - 1);
    const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    if (r >= a.n_rows) return;
    const int H = a.heads;
    const int64_t beg = a.row_ptr[r], end = a.row_ptr[r + 1];
    const int32_t v = a.out_idx ? a.out_idx[r] : static_cast<int32_t>(r);
    const float* sv = a.p_ext + int64_t(v) * a.ld_ext + a.hdp;     // s_v (self), then t_v
    const int64_t n = end - beg + 1;                                // + self loop
    float mx[kMaxHeads], sm[kMaxHeads], tv[kMaxHeads];
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) {
        mx[h] = -INFINITY;
        sm[h] = 0.f;
        tv[h] = h < H ? sv[H + h] : 0.f;
    }
    auto src_of = [&](int64_t i) -> int32_t { return i < end - beg ? a.idx[beg + i] : v; };
    for (int64_t i = lane; i < n; i += kWarp) {
        const float* su = a.p_ext + int64_t(src_of(i)) * a.ld_ext + a.hdp;
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h)
            if (h < H) mx[h] = fmaxf(mx[h], lrelu(su[h] + tv[h], a.slope));
    }
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) mx[h] = warp_max(mx[h]);
    for (int64_t i = lane; i < n; i += kWarp) {
        const float* su = a.p_ext + int64_t(src_of(i)) * a.ld_ext + a.hdp;
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h)
            if (h < H) sm[h] += expf(lrelu(su[h] + tv[h], a.slope) - mx[h]);
    }
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) sm[h] = warp_sum(sm[h]);
    for (int64_t i = lane; i < n; i += kWarp) {
        const float* su = a.p_ext + int64_t(src_of(i)) * a.ld_ext + a.hdp;
        float* dst = i < end - beg ? a.alpha + (beg + i) * H : a.alpha_self + int64_t(v) * H;
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h)
            if (h < H) dst[h] = expf(lrelu(su[h] + tv[h], a.slope) - mx[h]) / sm[h];
    }
}

// --------------------------------------------------------------- backward --
// dalpha_uv,h = gO_h[v] . P_h[u] for every in-edge (and the self loop).
// Warp per target row: gO row in registers, one neighbour row per step,
// per-head dot products combined through shared memory.
__global__ void __launch_bounds__(256) gat_edge_dot_kernel(grd_gat_args a) {
    __shared__ float part[8][64];
    const int lane = threadIdx.x & (kWarp - 1);
    const int wib = threadIdx.x / kWarp;
    const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    if (r >= a.n_rows) return;
    const int H = a.heads;
    const int q4 = a.hdp / 4;               // float4 chunks per row (<= 64)
    const int per_head = a.dhp / 4;
    const int64_t beg = a.row_ptr[r], end = a.row_ptr[r + 1];
    const int32_t v = a.out_idx ? a.out_idx[r] : static_cast<int32_t>(r);
    float4 g[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const int q = lane + c * kWarp;
        g[c] = q < q4 ? *reinterpret_cast<const float4*>(a.grad_o + int64_t(v) * a.ld_go + 4 * q)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int64_t i = 0; i <= end - beg; ++i) {
        const int32_t u = i < end - beg ? a.idx[beg + i] : v;
        const float* pu = a.p_ext + int64_t(u) * a.ld_ext;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int q = lane + c * kWarp;
            float d = 0.f;
            if (q < q4) {
                const float4 p = __ldg(reinterpret_cast<const float4*>(pu + 4 * q));
                d = g[c].x * p.x + g[c].y * p.y + g[c].z * p.z + g[c].w * p.w;
            }
            part[wib][q] = d;
        }
        __syncwarp();
        if (lane < H) {
            float s = 0.f;
            for (int k = 0; k < per_head; ++k) s += part[wib][lane * per_head + k];
            float* dst = i < end - beg ? a.dalpha + (beg + i) * H : a.dalpha_self + int64_t(v) * H;
            dst[lane] = s;
        }
        __syncwarp();
    }
}

// delta_uv,h = alpha (dalpha - sum_u' alpha dalpha) * lrelu'(z); the target
// score gradient dt_v,h = sum_u delta_uv,h lands in column hdp+H+h of grad_ext.
__global__ void __launch_bounds__(256) gat_softmax_bwd_kernel(grd_gat_args a) {
    const int lane = threadIdx.x & (kWarp - 1);
    const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    if (r >= a.n_rows) return;
    const int H = a.heads;
    const int64_t beg = a.row_ptr[r], end = a.row_ptr[r + 1];
    const int32_t v = a.out_idx ? a.out_idx[r] : static_cast<int32_t>(r);
    const int64_t n = end - beg + 1;
    const float* tvp = a.p_ext + int64_t(v) * a.ld_ext + a.hdp + H;
    float c[kMaxHeads], dt[kMaxHeads], tv[kMaxHeads];
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) {
        c[h] = 0.f;
        dt[h] = 0.f;
        tv[h] = h < H ? tvp[h] : 0.f;
    }
    for (int64_t i = lane; i < n; i += kWarp) {
        const float* al = i < end - beg ? a.alpha + (beg + i) * H : a.alpha_self + int64_t(v) * H;
        const float* da = i < end - beg ? a.dalpha + (beg + i) * H : a.dalpha_self + int64_t(v) * H;
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h)
            if (h < H) c[h] = fmaf(al[h], da[h], c[h]);
    }
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) c[h] = warp_sum(c[h]);
    for (int64_t i = lane; i < n; i += kWarp) {
        const bool self = i == end - beg;
        const int32_t u = self ? v : a.idx[beg + i];
        const float* su = a.p_ext + int64_t(u) * a.ld_ext + a.hdp;
        const float* al = self ? a.alpha_self + int64_t(v) * H : a.alpha + (beg + i) * H;
        const float* da = self ? a.dalpha_self + int64_t(v) * H : a.dalpha + (beg + i) * H;
        float* de = self ? a.delta_self + int64_t(v) * H : a.delta + (beg + i) * H;
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) {
            if (h >= H) continue;
            const float d = al[h] * (da[h] - c[h]) * lrelu_grad(su[h] + tv[h], a.slope);
            de[h] = d;
            dt[h] += d;
        }
    }
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) dt[h] = warp_sum(dt[h]);
    if (lane < H) a.grad_ext[int64_t(v) * a.ld_gext + a.hdp + H + lane] = dt[lane];
}

// Source score gradient ds_u,h = sum over u's out-edges of delta (edges
// addressed through the transposed CSR's permutation) + the self loop.
__global__ void __launch_bounds__(256) gat_src_grad_kernel(grd_gat_args a) {
    const int lane = threadIdx.x & (kWarp - 1);
    const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    if (r >= a.n_rows) return;
    const int H = a.heads;
    const int64_t beg = a.row_ptr[r], end = a.row_ptr[r + 1];
    float ds[kMaxHeads];
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) ds[h] = 0.f;
    for (int64_t i = beg + lane; i < end; i += kWarp) {
        const float* de = a.delta + int64_t(a.edge_perm[i]) * H;
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h)
            if (h < H) ds[h] += de[h];
    }
#pragma unroll
    for (int h = 0; h < kMaxHeads; ++h) ds[h] = warp_sum(ds[h]);
    if (lane < H)
        a.grad_ext[r * a.ld_gext + a.hdp + lane] = ds[lane] + a.delta_self[r * H + lane];
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

}  // namespace

extern "C" int grd_gat_softmax(const grd_gat_args* args, void* stream) {
    clear_error();
    if (!args || args->heads < 1 || args->heads > kMaxHeads) return fail(kErrArg, "gat_softmax: bad heads");
    if (args->n_rows == 0) return 0;
    gat_softmax_kernel<<<warps_blocks(args->n_rows), 256, 0, static_cast<cudaStream_t>(stream)>>>(*args);
    return launch_status("gat_softmax");
}

extern "C" int grd_gat_softmax_bwd(const grd_gat_args* args, void* stream) {
    clear_error();
    if (!args || args->heads < 1 || args->heads > kMaxHeads || args->hdp > 256 || args->hdp % 4)
        return fail(kErrArg, "gat_softmax_bwd: bad shape");
    if (args->n_rows == 0) return 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    gat_edge_dot_kernel<<<warps_blocks(args->n_rows), 256, 0, st>>>(*args);
    int rc = launch_status("gat_edge_dot");
    if (rc) return rc;
    gat_softmax_bwd_kernel<<<warps_blocks(args->n_rows), 256, 0, st>>>(*args);
    return launch_status("gat_softmax_bwd");
}

extern "C" int grd_gat_src_grad(const grd_gat_args* args, void* stream) {
    clear_error();
    if (!args || !args->edge_perm) return fail(kErrArg, "gat_src_grad: needs edge_perm");
    if (args->n_rows == 0) return 0;
    gat_src_grad_kernel<<<warps_blocks(args->n_rows), 256, 0, static_cast<cudaStream_t>(stream)>>>(*args);
    return launch_status("gat_src_grad");
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
