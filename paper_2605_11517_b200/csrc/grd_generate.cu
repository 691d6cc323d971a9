// GPU Kronecker/RMAT pair generator (graph.py:158-209 generate_kronecker):
// the vertex pairs of one round, bit-exact with numpy's PCG64 stream.
//
// numpy draws the round level by level: element i of level k is stream
// position k * batch + i (relative to the round's start), i.e. the output
// after k * batch + i + 1 LCG steps.  Each thread owns kChunk consecutive
// elements: it jumps once (O(log i0)) to its first position of level 0,
// draws its kChunk values by plain steps, and reaches the next level by the
// constant jump A^batch (precomputed on the host), accumulating the pairs'
// bits in registers.  Output: the canonical key lo * n + hi, or -1 for a
// self loop (removed by the caller, which also deduplicates in
// first-occurrence order and builds the CSR).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/grinder_b200.h"
#include "grd_common.h"

using namespace grd;

namespace {

using u128 = unsigned __int128;
constexpr int kChunk = 16;

struct PcgArgs {
    u128 state, inc;          // stream state at the round's start, increment
    u128 jump_mul, jump_add;  // state -> jump_mul * state + jump_add == batch steps
    double c0, c1, c2, c3;    // cumulative initiator
};

__device__ __forceinline__ u128 pcg_mult() {
    return (static_cast<u128>(0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;
}

__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
    const uint64_t hi = static_cast<uint64_t>(s >> 64);
    const uint64_t lo = static_cast<uint64_t>(s);
    const unsigned rot = static_cast<unsigned>(s >> 122);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

// state after `delta` LCG steps
__device__ __forceinline__ u128 advance(u128 state, u128 inc, uint64_t delta) {
    u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

__global__ void __launch_bounds__(256) kron_keys_kernel(int scale, int64_t batch, PcgArgs a, int64_t* keys) {
    const int64_t i0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * kChunk;
    if (i0 >= batch) return;
    const int cnt = static_cast<int>(batch - i0 < kChunk ? batch - i0 : kChunk);
    const u128 mult = pcg_mult();
    u128 s = advance(a.state, a.inc, static_cast<uint64_t>(i0));   // before element i0, level 0
    uint32_t src[kChunk], dst[kChunk];
#pragma unroll
    for (int j = 0; j < kChunk; ++j) src[j] = dst[j] = 0;
    for (int level = 0; level < scale; ++level) {
        u128 st = s;
#pragma unroll
        for (int j = 0; j < kChunk; ++j) {
            if (j < cnt) {
                st = st * mult + a.inc;
                const double r = static_cast<double>(xsl_rr(st) >> 11) * (1.0 / 9007199254740992.0);
                // np.searchsorted(cum, r, side="right") = #{cum <= r}
                const uint32_t q = (a.c0 <= r) + (a.c1 <= r) + (a.c2 <= r) + (a.c3 <= r);
                src[j] = (src[j] << 1) | (q >> 1);
                dst[j] = (dst[j] << 1) | (q & 1u);
            }
        }
        s = a.jump_mul * s + a.jump_add;          // same element, next level
    }
    const int64_t n = int64_t{1} << scale;
#pragma unroll
    for (int j = 0; j < kChunk; ++j) {
        if (j >= cnt) break;
        const int64_t lo = src[j] < dst[j] ? src[j] : dst[j];
        const int64_t hi = src[j] < dst[j] ? dst[j] : src[j];
        keys[i0 + j] = lo == hi ? -1 : lo * n + hi;
    }
}

// Feature rows of make_random_dataset (dataset.py:75-98): the matrix is
// the first draws of the dataset's PCG64 stream, numpy's random(dtype=
// float32) = (next_uint32 >> 8) * 2^-24, next_uint32 taking the low half of
// a 64-bit output first and its high half next, then - 0.5.  Value k of the
// row-major [V, F] matrix is half k % 2 of output k / 2.  One thread per
// requested row: a log-time jump to its first output, then plain steps.
__global__ void __launch_bounds__(256) feature_rows_kernel(u128 state, u128 inc, const int64_t* rows,
                                                           int64_t row0, int64_t n_rows, int F, float* out,
                                                           int64_t ldo) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_rows) return;
    const int64_t r = rows ? rows[i] : row0 + i;
    const uint64_t k0 = static_cast<uint64_t>(r) * static_cast<uint64_t>(F);
    const u128 mult = pcg_mult();
    u128 s = advance(state, inc, k0 >> 1);          // before output k0 / 2
    float* dst = out + i * ldo;
    uint64_t cur = 0;
    bool have = false;
    if (k0 & 1) {                                    // the row starts with a high half
        s = s * mult + inc;
        cur = xsl_rr(s);
        have = true;
    }
    for (int j = 0; j < F; ++j) {
        uint32_t u;
        if (have) {
            u = static_cast<uint32_t>(cur >> 32);
            have = false;
        } else {
            s = s * mult + inc;
            cur = xsl_rr(s);
            u = static_cast<uint32_t>(cur & 0xffffffffu);
            have = true;
        }
        dst[j] = static_cast<float>(u >> 8) * (1.0f / 16777216.0f) - 0.5f;
    }
}

}  // namespace

extern "C" int grd_feature_rows(const uint64_t* pcg_words, const int64_t* rows, int64_t row0,
                                int64_t n_rows, int32_t feature_dim, float* out, int64_t ld_out,
                                void* stream) {
    clear_error();
    if (n_rows == 0) return 0;
    if (!pcg_words || n_rows < 0 || feature_dim <= 0 || !out || ld_out < feature_dim || (!rows && row0 < 0))
        return fail(kErrArg, "feature_rows: bad arguments");
    const u128 state = (static_cast<u128>(pcg_words[0]) << 64) | pcg_words[1];
    const u128 inc = (static_cast<u128>(pcg_words[2]) << 64) | pcg_words[3];
    const int64_t blocks = (n_rows + 255) / 256;
    feature_rows_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        state, inc, rows, row0, n_rows, feature_dim, out, ld_out);
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return fail(static_cast<int>(err), "feature_rows: %s", cudaGetErrorString(err));
    return 0;
}

extern "C" int grd_kronecker_keys(int32_t scale, int64_t batch, const uint64_t* pcg_words, const double* cum,
                                  int64_t* keys, void* stream) {
    clear_error();
    if (scale < 4 || scale > 30) return fail(kErrArg, "kronecker_keys: scale must be in [4, 30]");
    if (batch < 0 || !pcg_words || !cum || (batch > 0 && !keys)) return fail(kErrArg, "kronecker_keys: bad arguments");
    if (batch == 0) return 0;
    PcgArgs a;
    a.state = (static_cast<u128>(pcg_words[0]) << 64) | pcg_words[1];
    a.inc = (static_cast<u128>(pcg_words[2]) << 64) | pcg_words[3];
    a.jump_mul = (static_cast<u128>(pcg_words[4]) << 64) | pcg_words[5];
    a.jump_add = (static_cast<u128>(pcg_words[6]) << 64) | pcg_words[7];
    a.c0 = cum[0];
    a.c1 = cum[1];
    a.c2 = cum[2];
    a.c3 = cum[3];
    const int64_t threads = (batch + kChunk - 1) / kChunk;
    const int64_t blocks = (threads + 255) / 256;
    if (blocks > 0x7fffffffLL) return fail(kErrArg, "kronecker_keys: batch too large");
    kron_keys_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(scale, batch, a,
                                                                                                    keys);
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return fail(static_cast<int>(err), "kronecker_keys: %s", cudaGetErrorString(err));
    return 0;
}
