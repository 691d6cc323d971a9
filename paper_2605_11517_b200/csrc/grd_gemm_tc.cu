// Dense fp32 GEMM on the 5th-generation tensor cores (tcgen05, sm_100a) with
// the 3xTF32 split, for the GNN dense transforms (training.py:76,128-129):
//   C = epi(opA(A) opB(B)) at fp32-grade accuracy.  An opt-in bf16x3 split
// for the forward / input-gradient GEMMs is below (gemm_bf16x3_ws).
//
// 3xTF32:  A = Ah + Al, B = Bh + Bl, Ah = A & 0xffffe000 (exact TF32),
//          Al = A - Ah;  C ~= Al*Bh + Ah*Bl + Ah*Bh  (kind::tf32 MMAs,
//          fp32 accumulation in TMEM; the dropped Al*Bl is ~2^-22 relative).
//
// Warp-specialised persistent kernel (14 warps):
//   warp 0     producer: TMA tensor copies of raw A (and, for the weight
//              gradient, raw B) into a ring of shared-memory stages; the
//              weight operand of forward/dgrad GEMMs is pre-split into hi/lo
//              K-major tiles by a small pack kernel and arrives by one 1-D
//              bulk copy per stage;
//   warp 1     MMA issuer: one elected thread, 12 tcgen05.mma per 32-deep K
//              block, tcgen05.commit releases the stage / publishes a tile;
//   warps 2-9  converters: split each raw stage into hi (in place) and lo;
//   warps 10-13 epilogue: tcgen05.ld of the double-buffered TMEM accumulator,
//              fused row-scale / element-multiply / ReLU-mask / ReLU /
//              accumulate, 128-byte row stores (or split-K partial tiles).
// Clusters of C = 1, 2 or 4 CTAs along M share the weight operand: each CTA of
// a cluster fetches 1/C of every B stage and multicasts it into all C CTAs'
// shared memory (TMA / bulk-copy .multicast::cluster), and the MMA issuer's
// stage-release commit arrives on the empty barrier of every CTA of the
// cluster, so a stage is refilled only when all C consumers are done with it.
// This divides the L2->SM traffic of the (re-read per M tile) B operand by C.
// Shared-memory tiles use the canonical 128-byte swizzled layouts: K-major
// SWIZZLE_128B for row-major activations (TMA box 32 K x 128 rows) and, for
// the weight-gradient operands whose rows run along K, MN-major
// SWIZZLE_128B_BASE32B (TMA SWIZZLE_128B_ATOM_32B boxes of 32 MN x 32 K),
// the only MN-major layout the tf32 MMA accepts.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "grd_gemm_tc.h"

namespace grd_tc {

constexpr int kBM = 128;
constexpr int kBK = 32;
constexpr int kWarps = 14;
constexpr int kThreads = kWarps * 32;
constexpr int kConvWarp0 = 2;
constexpr int kConvWarps = 4;
constexpr int kConvThreads = kConvWarps * 32;
constexpr int kEpiWarp0 = kConvWarp0 + kConvWarps;
constexpr int kEpiWarps = 8;            // two per TMEM lane quarter (column halves)
constexpr int kEpiThreads = kEpiWarps * 32;
static_assert(kEpiWarp0 + kEpiWarps == kWarps, "warp roles");

enum OpMode : int {
    kKMajorTma = 0,     // raw, K-contiguous rows, one TMA box (32 x rows)
    kMNMajorTma = 1,    // raw, rows contiguous along MN: TMA boxes (32 MN x 32 K rows)
                        // in the SW128_32B-atom layout the tf32 MMA reads MN-major
    kPacked = 2,        // pre-split hi/lo K-major tiles, one bulk copy
};

struct Params {
    int64_t m, n, k;
    int bn;
    int a_mode, b_mode;
    const float* b_packed;          // kPacked: [ntile][kblock][hi|lo][bn x 32]
    int64_t kchunk;                 // split-K chunk (multiple of 32)
    int splits;
    int stages;
    int b_resident;                 // packed B loaded once per CTA and kept in shared memory
    int cluster;                    // CTAs per cluster along M (1, 2, 4)
    int pair;                       // 1: cluster of 2 = a cta_group::2 pair (M = 256)
    float* c; int64_t ldc;
    const float* row_scale;
    const float* elem_mul; int64_t ld_elem_mul;
    const float* relu_ref; int64_t ld_relu_ref;
    int relu_out;
    int accumulate;
    float* partial; int64_t ld_partial;   // split-K: [z][m][ld_partial]
    float* c2; int64_t ldc2; int64_t split;   // columns >= split (> 0) go to c2
    int tma_store;                  // epilogue chunks leave through shared memory by TMA
    int kch;                        // K blocks per TMEM accumulation (0: the whole K)
    int hi_raw;                     // 1: the raw fp32 tile is the hi operand (the MMA reads
                                    // only its tf32 bits), the converter writes lo alone
    int lo_slots;                   // > 0: lo tiles live in their own ring of this many slots
                                    // (a stage then carries raw operands only: deeper ring)
    int epi_bufs;                   // TMA-store staging tiles per epilogue warp (1 or 2)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Shared-memory matrix descriptor, version 1.  layout: 2 = SWIZZLE_128B
// (K-major here), 1 = SWIZZLE_128B_BASE32B (the MN-major tf32 layout).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2u) {
    uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1u) << 46;
    d |= static_cast<uint64_t>(layout) << 61;
    return d;
}

// kind::tf32, D fp32, M = 128, N = bn; a/b major: 0 = K, 1 = MN.
__device__ __forceinline__ uint32_t make_idesc(int bn, int a_mn, int b_mn, int m = kBM) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
           (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(bn >> 3) << 17) |
           (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred done;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                       uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_2d_mc(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                          uint64_t* bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void bulk_copy_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
// arrive on the barrier at the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// CTA-pair (cta_group::2) MMA: issued by the even CTA; A rows 0-127 / 128-255
// and B rows [0, N/2) / [N/2, N) come from the two CTAs' shared memory at the
// same offsets; each CTA's TMEM receives its 128 rows x N.
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float4 hi4(float4 v) {
    v.x = __uint_as_float(__float_as_uint(v.x) & 0xffffe000u);
    v.y = __uint_as_float(__float_as_uint(v.y) & 0xffffe000u);
    v.z = __uint_as_float(__float_as_uint(v.z) & 0xffffe000u);
    v.w = __uint_as_float(__float_as_uint(v.w) & 0xffffe000u);
    return v;
}

// Split a raw tile in place: hi over raw, lo into `lo` (same swizzled layout,
// elementwise).  Shared-space 128-bit accesses, 4 loads in flight per thread.
__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
}
__device__ __forceinline__ void split_tile(uint8_t* raw, uint8_t* lo, uint32_t bytes, int ctid, int nthr,
                                           bool write_hi = true) {
    const uint32_t r0 = smem_u32(raw), l0 = smem_u32(lo);
    const uint32_t n16 = bytes / 16;
    uint32_t i = ctid;
    for (; i + 3u * nthr < n16; i += 4u * nthr) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = lds128(r0 + (i + u * nthr) * 16u);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float4 h = hi4(v[u]);
            if (write_hi) sts128(r0 + (i + u * nthr) * 16u, h);
            sts128(l0 + (i + u * nthr) * 16u, make_float4(v[u].x - h.x, v[u].y - h.y, v[u].z - h.z, v[u].w - h.w));
        }
    }
    for (; i < n16; i += nthr) {
        const float4 v = lds128(r0 + i * 16u);
        const float4 h = hi4(v);
        if (write_hi) sts128(r0 + i * 16u, h);
        sts128(l0 + i * 16u, make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w));
    }
}


// Epilogue of one 32-row x 32-column accumulator chunk (one warp): tcgen05.ld
// gives lane l row l; lane l applies the fused epilogue to its row's 32
// columns and stores them (8 x 16 B).  Staging the chunk through shared
// memory for row-contiguous stores was measured 30-50 % slower end to end
// on the store-heavy shapes (tools/gemm_prec.py), so the stores stay per row.
// The chunk's epilogue operands (C when accumulating, the ReLU reference)
// are loaded before the accumulator is waited for / read from TMEM, so the
// loads are in flight meanwhile (-12 % GEMM time).
struct EpiIn {
    float4 o[8], e[8];
};

__device__ __forceinline__ void epi_prefetch(const Params& p, int64_t row, int64_t col0, EpiIn& in,
                                             bool accumulate) {
    const int64_t n_pad = (p.n + 3) / 4 * 4;
    const bool live = row < p.m && col0 < n_pad && !p.partial;
    const float* crow = p.c + row * p.ldc + col0;
#pragma unroll
    for (int j4 = 0; j4 < 8; ++j4) {
        const int64_t n = col0 + 4 * j4;
        const bool ok = live && n < n_pad;
        in.o[j4] = (ok && accumulate) ? *reinterpret_cast<const float4*>(crow + 4 * j4)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
        in.e[j4] = (ok && p.relu_ref) ? __ldg(reinterpret_cast<const float4*>(p.relu_ref + row * p.ld_relu_ref + n))
                                      : make_float4(1.f, 1.f, 1.f, 1.f);
    }
}

template <bool kSplit>
__device__ __forceinline__ void epi_store_direct(const Params& p, const float (&v)[32], int64_t row, int64_t col0,
                                                 int z, const EpiIn& in) {
    if (row >= p.m) return;
    const int64_t n_pad = (p.n + 3) / 4 * 4;
    if (p.partial) {
        float* out = p.partial + (int64_t(z) * p.m + row) * p.ld_partial + col0;
#pragma unroll
        for (int j = 0; j < 32; j += 4)
            if (col0 + j < n_pad) *reinterpret_cast<float4*>(out + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        return;
    }
    const float rs = p.row_scale ? p.row_scale[row] : 1.0f;
    float* crow = p.c + row * p.ldc + col0;
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
        const int64_t n = col0 + j;
        if (n >= n_pad) continue;
        // columns >= split go to the second destination (host-checked: no
        // accumulate / relu_ref / elem_mul operands with a split output)
        float* dst = (kSplit && p.split > 0 && n >= p.split) ? p.c2 + row * p.ldc2 + (n - p.split) : crow + j;
        float4 x = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        const float4 oo = in.o[j / 4];
        x.x += oo.x; x.y += oo.y; x.z += oo.z; x.w += oo.w;
        if (p.row_scale) { x.x *= rs; x.y *= rs; x.z *= rs; x.w *= rs; }
        if (p.elem_mul) {
            const float4 m = *reinterpret_cast<const float4*>(p.elem_mul + row * p.ld_elem_mul + n);
            x.x *= m.x; x.y *= m.y; x.z *= m.z; x.w *= m.w;
        }
        const float4 ee = in.e[j / 4];
        if (!(ee.x > 0.f)) x.x = 0.f;
        if (!(ee.y > 0.f)) x.y = 0.f;
        if (!(ee.z > 0.f)) x.z = 0.f;
        if (!(ee.w > 0.f)) x.w = 0.f;
        if (p.relu_out) {
            x.x = fmaxf(x.x, 0.f); x.y = fmaxf(x.y, 0.f); x.z = fmaxf(x.z, 0.f); x.w = fmaxf(x.w, 0.f);
        }
        *reinterpret_cast<float4*>(dst) = x;
    }
}

// TMA-store epilogue: a warp's 32-row x 32-column chunk is written to its
// 4 KB shared staging tile in the 128-byte-swizzled layout the tensor map
// names (the 16-byte column group j of row r sits at group j ^ (r & 7), so a
// warp's row-per-lane float4 stores spread over all banks) and one lane
// issues the bulk tensor store.  The global writes are whole 128-byte row
// segments issued by the TMA engine instead of 32 scattered 16-byte stores
// per instruction.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void epi_stage_tma(const Params& p, const float (&v)[32], int64_t row, int64_t col0,
                                              const EpiIn& in, uint8_t* stage, int lane) {
    const float rs = (p.row_scale && row < p.m) ? p.row_scale[row] : 1.0f;
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
        float4 x = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        const float4 oo = in.o[j / 4];
        x.x += oo.x; x.y += oo.y; x.z += oo.z; x.w += oo.w;
        if (p.row_scale) { x.x *= rs; x.y *= rs; x.z *= rs; x.w *= rs; }
        if (p.elem_mul && row < p.m && col0 + j < (p.n + 3) / 4 * 4) {
            const float4 m = *reinterpret_cast<const float4*>(p.elem_mul + row * p.ld_elem_mul + col0 + j);
            x.x *= m.x; x.y *= m.y; x.z *= m.z; x.w *= m.w;
        }
        const float4 ee = in.e[j / 4];
        if (!(ee.x > 0.f)) x.x = 0.f;
        if (!(ee.y > 0.f)) x.y = 0.f;
        if (!(ee.z > 0.f)) x.z = 0.f;
        if (!(ee.w > 0.f)) x.w = 0.f;
        if (p.relu_out) {
            x.x = fmaxf(x.x, 0.f); x.y = fmaxf(x.y, 0.f); x.z = fmaxf(x.z, 0.f); x.w = fmaxf(x.w, 0.f);
        }
        const uint32_t grp = static_cast<uint32_t>(j >> 2) ^ static_cast<uint32_t>(lane & 7);
        *reinterpret_cast<float4*>(stage + lane * 128 + grp * 16) = x;
    }
}

// A K chunk's partial sum (not the tile's last chunk): C = C_so_far + acc,
// no epilogue operators yet; the next chunk reads it back (same thread,
// same addresses, the tile hot in L2).
__device__ __forceinline__ void epi_store_raw(const Params& p, const float (&v)[32], int64_t row, int64_t col0,
                                              const EpiIn& in) {
    if (row >= p.m) return;
    const int64_t n_pad = (p.n + 3) / 4 * 4;
    float* crow = p.c + row * p.ldc + col0;
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
        if (col0 + j >= n_pad) continue;
        const float4 oo = in.o[j / 4];
        *reinterpret_cast<float4*>(crow + j) =
            make_float4(v[j] + oo.x, v[j + 1] + oo.y, v[j + 2] + oo.z, v[j + 3] + oo.w);
    }
}

// Epilogue warps' loop over the tiles of this CTA (both kernels): TMEM
// accumulator `acc` of the i-th tile with K work, drained chunk by chunk.
template <bool kPair, bool kSplit, class TileFn>
__device__ __forceinline__ void epilogue_loop(const Params& p, uint32_t tmem, uint64_t* tfull, uint64_t* tempty,
                                              int warp, int lane, int64_t t0, int64_t tstep,
                                              int64_t ntiles, TileFn tile_of,
                                              const CUtensorMap* map_c = nullptr, uint8_t* stage = nullptr) {
    const bool tma = !kSplit && p.tma_store && stage != nullptr;
    // two staging tiles per warp: a chunk is staged while the previous
    // chunk's bulk store still reads the other tile
    const int ebufs = p.epi_bufs > 1 ? 2 : 1;
    int eb = 0;
    const int q = warp & 3;                               // TMEM lane quarter
    const int half = (warp - kEpiWarp0) >> 2;             // which interleaved column chunks
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    const int bn = p.bn;
    const int64_t nkb = (p.k + kBK - 1) / kBK;
    // K chunks accumulated separately (p.kch): each chunk's TMEM partial is
    // added to C with round-to-nearest fp32 adds, the epilogue operators
    // apply with the last chunk (kSplit / split-K tiles: one chunk)
    const int nch = (!kSplit && p.kch > 0 && !p.partial) ? static_cast<int>((nkb + p.kch - 1) / p.kch) : 1;
    int64_t i = 0;
    for (int64_t t = t0; t < ntiles; t += tstep) {
        int64_t m0, n0;
        int z;
        bool has_k;
        tile_of(t, m0, n0, z, has_k);
        const int64_t row0 = m0 + q * 32;
        const int64_t n_pad = (p.n + 3) / 4 * 4;
        const int chunks = has_k ? nch : 1;
        for (int ch = 0; ch < chunks; ++ch) {
            const bool last = ch == chunks - 1;
            const int acc = static_cast<int>(i & 1);
            bool waited = false;
            for (int c0 = 32 * half; c0 < bn; c0 += 64) {
                EpiIn in;
                epi_prefetch(p, row0 + lane, n0 + c0, in, ch > 0 || p.accumulate);
                if (has_k && !waited) {
                    mbar_wait(tfull + acc, static_cast<uint32_t>((i / 2) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    waited = true;
                }
                float v[32];
                if (has_k) {
                    tmem_ld32(tmem + lane_base + static_cast<uint32_t>(acc * bn + c0), v);
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = 0.f;
                }
                if (row0 >= p.m || n0 + c0 >= n_pad) continue;   // warp-uniform
                if (!last) {
                    epi_store_raw(p, v, row0 + lane, n0 + c0, in);
                    continue;
                }
                if (tma && chunks == 1) {
                    uint8_t* sb = stage + eb * 4096;
                    // the staging tile's last store (ebufs chunks ago) has read it
                    if (lane == 0) {
                        if (ebufs > 1) tma_store_wait_read1();
                        else tma_store_wait_read();
                    }
                    __syncwarp();
                    epi_stage_tma(p, v, row0 + lane, n0 + c0, in, sb, lane);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0)
                        tma_store_2d(map_c, sb, static_cast<int32_t>(n0 + c0), static_cast<int32_t>(row0));
                    eb = (eb + 1) % ebufs;
                    continue;
                }
                epi_store_direct<kSplit>(p, v, row0 + lane, n0 + c0, z, in);
            }
            if (has_k) {
                // a warp without columns in this tile (bn <= 32) still waits for
                // the accumulator before releasing it: no arrival may run ahead
                // into the buffer's next phase
                if (!waited) mbar_wait(tfull + acc, static_cast<uint32_t>((i / 2) & 1));
                asm volatile("tcgen05.fence::before_thread_sync;");
                if (kPair) mbar_arrive_cluster(tempty + acc, 0);
                else mbar_arrive(tempty + acc);
                ++i;
            }
        }
    }
    if (tma && lane == 0) tma_store_wait_all();
}

// Split-K partial tiles with fresh accumulators (kFresh): the MMA issuer
// starts a new TMEM accumulator for every 32-deep K block, and these warps
// add the K blocks' partials in registers with round-to-nearest fp32 adds.
// The tensor cores' fused accumulation truncates (measured: the 3xTF32
// error grows linearly with the number of MMAs accumulated, ~4e-6 relative
// at 192 and ~8e-6 at 168-3072 accumulation steps); a weight gradient sums
// 10^4..10^6 rows whose terms largely cancel, which amplifies that bias to
// 1e-3 (GraphSAGE layer 0 at F = 100, H = 256).  12 MMAs per accumulator
// keep it at the per-product rounding.  bn <= 128: two 32-column chunks of
// running sums per thread.
template <bool kPair, class TileFn, class KbFn>
__device__ __forceinline__ void epilogue_fresh(const Params& p, uint32_t tmem, uint64_t* tfull, uint64_t* tempty,
                                               int warp, int lane, int64_t t0, int64_t tstep, int64_t ntiles,
                                               TileFn tile_of, KbFn kblocks) {
    const int q = warp & 3;
    const int half = (warp - kEpiWarp0) >> 2;
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    const int bn = p.bn;
    int64_t g = 0;                                  // accumulator uses (K blocks) so far
    for (int64_t t = t0; t < ntiles; t += tstep) {
        int64_t m0, n0;
        int z;
        bool has_k;
        tile_of(t, m0, n0, z, has_k);
        const int64_t nkb = kblocks(z);
        float run[2][32];
#pragma unroll
        for (int ci = 0; ci < 2; ++ci)
#pragma unroll
            for (int j = 0; j < 32; ++j) run[ci][j] = 0.f;
        for (int64_t kb = 0; kb < nkb; ++kb, ++g) {
            const int acc = static_cast<int>(g & 1);
            mbar_wait(tfull + acc, static_cast<uint32_t>((g / 2) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
            for (int ci = 0; ci < 2; ++ci) {
                const int c0 = 32 * half + 64 * ci;
                if (c0 >= bn) continue;
                float v[32];
                tmem_ld32(tmem + lane_base + static_cast<uint32_t>(acc * bn + c0), v);
#pragma unroll
                for (int j = 0; j < 32; ++j) run[ci][j] += v[j];
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            if (kPair) mbar_arrive_cluster(tempty + acc, 0);
            else mbar_arrive(tempty + acc);
        }
        const int64_t row0 = m0 + q * 32;
        const int64_t n_pad = (p.n + 3) / 4 * 4;
        EpiIn in;
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
            in.o[j4] = make_float4(0.f, 0.f, 0.f, 0.f);
            in.e[j4] = make_float4(1.f, 1.f, 1.f, 1.f);
        }
#pragma unroll
        for (int ci = 0; ci < 2; ++ci) {
            const int c0 = 32 * half + 64 * ci;
            if (c0 >= bn || row0 >= p.m || n0 + c0 >= n_pad) continue;
            epi_store_direct<false>(p, run[ci], row0 + lane, n0 + c0, z, in);
        }
    }
}

// kPair: a kernel containing cta_group::2 instructions must be launched in
// clusters of 2, so the CTA-pair variant is its own instantiation.
template <bool kPair, bool kSplit, bool kFresh = false>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tf32x3_ws(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               const __grid_constant__ CUtensorMap map_c, const Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int bn = p.bn;
    const int S = p.stages;
    constexpr bool pair = kPair;
    const int bnl = pair ? bn / 2 : bn;                      // B rows staged by this CTA
    const uint32_t a_bytes = kBM * 128u;
    const uint32_t b_bytes = static_cast<uint32_t>(bnl) * 128u;
    // stage: A hi | A lo | B hi | B lo   (A raw lands in A hi and is split in place)
    // B-resident mode (small packed weight, one N tile, no split-K): stages
    // carry A only, and this CTA's B hi|lo tiles of every K block sit after
    // the ring for the whole launch — loaded once instead of once per M tile.
    // lo ring (p.lo_slots > 0): a stage carries the raw operands only
    // (A raw | B raw, or B's packed hi|lo) and the converters write the lo
    // tiles into a separate ring of lo_slots slots, released by the MMAs that
    // read them; a lo tile lives only between its stage's conversion and
    // MMAs, so the same shared memory holds a raw ring twice as deep — the
    // loads in flight per SM are what bounds these HBM-streaming shapes.
    const bool bres = p.b_resident != 0;
    const bool lring = p.lo_slots > 0;
    const int SL = lring ? p.lo_slots : 0;
    const bool b_conv = p.b_mode != kPacked;                // B split by the converters
    const int64_t nkb_b = (p.k + kBK - 1) / kBK;
    const uint32_t stage_bytes = lring ? a_bytes + (bres ? 0u : (b_conv ? b_bytes : 2u * b_bytes))
                                       : (bres ? 2u * a_bytes : 2u * (a_bytes + b_bytes));
    const uint32_t lo_bytes = a_bytes + (b_conv ? b_bytes : 0u);
    uint8_t* lo_ring = smem + S * stage_bytes;
    const uint32_t b_off = lring ? a_bytes : 2u * a_bytes;  // B's offset inside a stage
    uint8_t* bres_smem = lo_ring + SL * lo_bytes;
    const uint32_t bres_bytes = bres ? static_cast<uint32_t>(nkb_b) * 2u * b_bytes : 0u;
    // TMA-store staging: 4 KB per epilogue warp, 1024-byte aligned (swizzle atoms)
    uint8_t* epi_stage = smem + ((static_cast<uint32_t>(bres_smem - smem) + bres_bytes + 1023u) & ~1023u);
    const uint32_t epi_bytes = p.tma_store ? static_cast<uint32_t>(kEpiWarps * p.epi_bufs) * 4096u : 0u;
    uint64_t* bars = reinterpret_cast<uint64_t*>(p.tma_store ? epi_stage + epi_bytes : bres_smem + bres_bytes);
    uint64_t* full = bars;             // [S]
    uint64_t* conv = bars + S;         // [S]
    uint64_t* empty = bars + 2 * S;    // [S]
    uint64_t* tfull = bars + 3 * S;    // [2]
    uint64_t* tempty = bars + 3 * S + 2;   // [2]
    uint64_t* bready = bars + 3 * S + 4;   // [1] resident B landed
    uint64_t* lofree = bars + 3 * S + 5;   // [SL] lo slot consumed by its MMAs
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 5 + SL);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int C = p.cluster;
    const int crank = C > 1 ? static_cast<int>(cluster_rank()) : 0;
    const uint16_t cmask = static_cast<uint16_t>((1u << C) - 1u);
    const int64_t mt = (p.m + kBM - 1) / kBM;
    const int64_t mg = (mt + C - 1) / C;            // M groups of C tiles (one per CTA)
    const int64_t nt = (p.n + bn - 1) / bn;
    const int64_t ntiles = mg * nt * p.splits;      // cluster work items
    const int64_t cid = blockIdx.x / C, ncl = gridDim.x / C;
    const int64_t nkb_full = (p.kchunk + kBK - 1) / kBK;
    uint32_t tmem_cols = 32;
    while (tmem_cols < static_cast<uint32_t>(2 * bn)) tmem_cols <<= 1;

    if (warp == 0) {
        if constexpr (kPair) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(tmem_cols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(tmem_cols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    if (threadIdx.x == 32) {
        // pair: the even CTA's conv / tempty barriers collect both CTAs'
        // converters / epilogue threads; its commits arrive on both CTAs'
        // empty / tfull barriers
        const uint32_t nc = pair ? 2u : 1u;
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(conv + s, kConvThreads * nc);
            mbar_init(empty + s, pair ? 1u : static_cast<uint32_t>(C));
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, kEpiThreads * nc);
        }
        mbar_init(bready, 1);
        for (int l = 0; l < SL; ++l) mbar_init(lofree + l, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)));
        if (p.b_mode != kPacked) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)));
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (C > 1) cluster_sync();     // peers' barriers exist before any multicast
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    auto kblocks_of = [&](int z) -> int64_t {
        const int64_t k0 = int64_t(z) * p.kchunk;
        const int64_t k1 = min(k0 + p.kchunk, p.k);
        return k1 > k0 ? (k1 - k0 + kBK - 1) / kBK : 0;
    };

    if (warp == 0) {
        // ------------------------------------------------ TMA producer --
        if (lane == 0) {
            if (bres) {
                // this CTA's B rows (pair: its half) of every K block, once
                mbar_expect_tx(bready, bres_bytes);
                for (int64_t kb = 0; kb < nkb_b; ++kb) {
                    const float* src = p.b_packed + kb * (2 * int64_t(bn) * kBK) + int64_t(crank) * bnl * kBK;
                    uint8_t* dst = bres_smem + kb * 2 * b_bytes;
                    bulk_copy(dst, src, b_bytes, bready);
                    bulk_copy(dst + b_bytes, src + int64_t(bn) * kBK, b_bytes, bready);
                }
            }
            uint64_t g = 0;
            for (int64_t t = cid; t < ntiles; t += ncl) {
                const int z = static_cast<int>(t / (mg * nt));
                const int64_t r = t % (mg * nt);
                const int64_t m0 = ((r / nt) * C + crank) * kBM, ntile = r % nt, n0 = ntile * bn;
                const int64_t nkb = kblocks_of(z);
                for (int64_t kb = 0; kb < nkb; ++kb, ++g) {
                    const int s = static_cast<int>(g % S);
                    if (g >= static_cast<uint64_t>(S)) mbar_wait(empty + s, static_cast<uint32_t>((g / S - 1) & 1));
                    uint8_t* st = smem + s * stage_bytes;
                    const int64_t k0 = int64_t(z) * p.kchunk + kb * kBK;
                    uint32_t bytes = a_bytes;
                    if (!bres) bytes += (p.b_mode == kPacked) ? 2u * b_bytes : b_bytes;
                    mbar_expect_tx(full + s, bytes);
                    if (p.a_mode == kKMajorTma) {
                        tma_2d(st, &map_a, static_cast<int32_t>(k0), static_cast<int32_t>(m0), full + s);
                    } else {
                        for (int j = 0; j < kBM / 32; ++j)
                            tma_2d(st + j * 4096, &map_a, static_cast<int32_t>(m0 + 32 * j),
                                   static_cast<int32_t>(k0), full + s);
                    }
                    if (bres) continue;
                    uint8_t* bdst = st + b_off;
                    if (pair) {
                        // this CTA's half of the B tile: rows [crank * bnl, +bnl)
                        const int64_t nb0 = n0 + crank * bnl;
                        if (p.b_mode == kPacked) {
                            const int64_t nkb_all = (p.k + kBK - 1) / kBK;
                            const float* src = p.b_packed + (ntile * nkb_all + k0 / kBK) * (2 * int64_t(bn) * kBK);
                            bulk_copy(bdst, src + int64_t(crank) * bnl * kBK, b_bytes, full + s);
                            bulk_copy(bdst + b_bytes, src + int64_t(bn) * kBK + int64_t(crank) * bnl * kBK, b_bytes,
                                      full + s);
                        } else if (p.b_mode == kKMajorTma) {
                            tma_2d(bdst, &map_b, static_cast<int32_t>(k0), static_cast<int32_t>(nb0), full + s);
                        } else {
                            for (int j = 0; j < bnl / 32; ++j)
                                tma_2d(bdst + j * 4096, &map_b, static_cast<int32_t>(nb0 + 32 * j),
                                       static_cast<int32_t>(k0), full + s);
                        }
                    } else if (p.b_mode == kPacked) {
                        const int64_t kbg = (k0 / kBK);
                        const int64_t nkb_all = (p.k + kBK - 1) / kBK;
                        const float* src = p.b_packed + (ntile * nkb_all + kbg) * (2 * int64_t(bn) * kBK);
                        if (C == 1) {
                            bulk_copy(bdst, src, 2u * b_bytes, full + s);
                        } else {   // this CTA's 1/C slice of the hi|lo tile, into every CTA
                            const uint32_t slice = 2u * b_bytes / static_cast<uint32_t>(C);
                            bulk_copy_mc(bdst + crank * slice, reinterpret_cast<const uint8_t*>(src) + crank * slice,
                                         slice, full + s, cmask);
                        }
                    } else if (p.b_mode == kKMajorTma) {
                        tma_2d(bdst, &map_b, static_cast<int32_t>(k0), static_cast<int32_t>(n0), full + s);
                    } else {
                        for (int j = 0; j < bn / 32; ++j) {
                            if (C == 1)
                                tma_2d(bdst + j * 4096, &map_b, static_cast<int32_t>(n0 + 32 * j),
                                       static_cast<int32_t>(k0), full + s);
                            else if (j % C == crank)
                                tma_2d_mc(bdst + j * 4096, &map_b, static_cast<int32_t>(n0 + 32 * j),
                                          static_cast<int32_t>(k0), full + s, cmask);
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------- MMA issuer --
        if (lane == 0 && (!pair || crank == 0)) {
            // K-major: SW128, advance 32 B per 8-deep MMA inside the 128 B row.
            // MN-major: SW128_32B atoms of 32 MN x 4 K rows, LBO = 4 KB between
            // 32-wide MN atoms, SBO = 512 B between 4-row K groups, advance
            // 1024 B (8 K rows) per MMA.
            const int a_mn = p.a_mode == kMNMajorTma;
            const int b_mn = p.b_mode == kMNMajorTma;
            const uint32_t idesc = make_idesc(bn, a_mn, b_mn, pair ? 2 * kBM : kBM);
            const uint32_t a_step = a_mn ? 1024u : 32u, b_step = b_mn ? 1024u : 32u;
            const uint32_t a_lbo = a_mn ? 4096u : 16u, b_lbo = b_mn ? 4096u : 16u;
            const uint32_t a_sbo = a_mn ? 512u : 1024u, b_sbo = b_mn ? 512u : 1024u;
            const uint32_t a_lay = a_mn ? 1u : 2u, b_lay = b_mn ? 1u : 2u;
            uint64_t g = 0;
            int64_t i = 0;   // tiles with K work (empty split-K tiles are skipped)
            int64_t fresh = 0;   // kFresh: accumulators started so far
            if (bres) {
                mbar_wait(bready, 0u);
                asm volatile("tcgen05.fence::after_thread_sync;");
            }
            for (int64_t t = cid; t < ntiles; t += ncl) {
                const int z = static_cast<int>(t / (mg * nt));
                const int64_t nkb = kblocks_of(z);
                if (nkb == 0) continue;
                int acc = static_cast<int>(i & 1);
                if (!kFresh) {
                    if (i >= 2) mbar_wait(tempty + acc, static_cast<uint32_t>((i / 2 - 1) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;");
                }
                uint32_t tacc = tmem + static_cast<uint32_t>(acc * bn);
                const int64_t kch = (!kFresh && p.kch > 0 && !p.partial) ? p.kch : 0;
                for (int64_t kb = 0; kb < nkb; ++kb, ++g) {
                    if (kch && kb > 0 && kb % kch == 0) {
                        // next K chunk: publish this one, move to the other accumulator
                        if constexpr (kPair) mma_commit_pair(tfull + acc);
                        else mma_commit(tfull + acc);
                        ++i;
                        acc = static_cast<int>(i & 1);
                        if (i >= 2) mbar_wait(tempty + acc, static_cast<uint32_t>((i / 2 - 1) & 1));
                        asm volatile("tcgen05.fence::after_thread_sync;");
                        tacc = tmem + static_cast<uint32_t>(acc * bn);
                    }
                    if constexpr (kFresh) {
                        // a fresh accumulator per K block (epilogue_fresh sums them)
                        acc = static_cast<int>(fresh & 1);
                        if (fresh >= 2) mbar_wait(tempty + acc, static_cast<uint32_t>((fresh / 2 - 1) & 1));
                        asm volatile("tcgen05.fence::after_thread_sync;");
                        tacc = tmem + static_cast<uint32_t>(acc * bn);
                    }
                    const int s = static_cast<int>(g % S);
                    mbar_wait(conv + s, static_cast<uint32_t>((g / S) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    uint8_t* st = smem + s * stage_bytes;
                    const int slot = lring ? static_cast<int>(g % SL) : 0;
                    uint8_t* lo = lring ? lo_ring + slot * lo_bytes : st + a_bytes;
                    const uint32_t ah = smem_u32(st), al = smem_u32(lo);
                    const uint8_t* bst = bres ? bres_smem + kb * 2 * b_bytes : st + b_off;
                    const uint32_t bh = smem_u32(bst);
                    const uint32_t bl = smem_u32((lring && b_conv) ? lo + a_bytes : bst + b_bytes);
#pragma unroll
                    for (int kk = 0; kk < kBK / 8; ++kk) {
                        const uint64_t dah = make_desc(ah + kk * a_step, a_lbo, a_sbo, a_lay);
                        const uint64_t dal = make_desc(al + kk * a_step, a_lbo, a_sbo, a_lay);
                        const uint64_t dbh = make_desc(bh + kk * b_step, b_lbo, b_sbo, b_lay);
                        const uint64_t dbl = make_desc(bl + kk * b_step, b_lbo, b_sbo, b_lay);
                        const uint32_t keep = (kk > 0 || (!kFresh && (kch ? kb % kch : kb) > 0)) ? 1u : 0u;
                        if constexpr (kPair) {
                            mma_tf32_pair(tacc, dal, dbh, idesc, keep);
                            mma_tf32_pair(tacc, dah, dbl, idesc, 1u);
                            mma_tf32_pair(tacc, dah, dbh, idesc, 1u);
                        } else {
                            mma_tf32(tacc, dal, dbh, idesc, keep);
                            mma_tf32(tacc, dah, dbl, idesc, 1u);
                            mma_tf32(tacc, dah, dbh, idesc, 1u);
                        }
                    }
                    if constexpr (kPair) mma_commit_pair(empty + s);   // both CTAs' stage s
                    else if (C == 1) mma_commit(empty + s);
                    else mma_commit_mc(empty + s, cmask);   // release the stage in every CTA
                    if (lring) {                            // and the lo slot (each CTA its own)
                        if constexpr (kPair) mma_commit_pair(lofree + slot);
                        else mma_commit(lofree + slot);
                    }
                    if constexpr (kFresh) {
                        if constexpr (kPair) mma_commit_pair(tfull + acc);
                        else mma_commit(tfull + acc);
                        ++fresh;
                    }
                }
                if constexpr (!kFresh) {
                    if constexpr (kPair) mma_commit_pair(tfull + acc);   // both CTAs' accumulators
                    else mma_commit(tfull + acc);
                }
                ++i;
            }
        }
    } else if (warp < kEpiWarp0) {
        // -------------------------------------------------- converters --
        const int ctid = threadIdx.x - kConvWarp0 * 32;
        uint64_t g = 0;
        for (int64_t t = cid; t < ntiles; t += ncl) {
            const int z = static_cast<int>(t / (mg * nt));
            const int64_t nkb = kblocks_of(z);
            for (int64_t kb = 0; kb < nkb; ++kb, ++g) {
                const int s = static_cast<int>(g % S);
                mbar_wait(full + s, static_cast<uint32_t>((g / S) & 1));
                uint8_t* st = smem + s * stage_bytes;
                uint8_t* lo = st + a_bytes;
                if (lring) {
                    const int slot = static_cast<int>(g % SL);
                    if (g >= static_cast<uint64_t>(SL))
                        mbar_wait(lofree + slot, static_cast<uint32_t>((g / SL - 1) & 1));
                    lo = lo_ring + slot * lo_bytes;
                }
                split_tile(st, lo, a_bytes, ctid, kConvThreads, !p.hi_raw);
                uint8_t* bh = st + b_off;
                if (b_conv) split_tile(bh, lring ? lo + a_bytes : bh + b_bytes, b_bytes, ctid, kConvThreads, !p.hi_raw);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (pair) mbar_arrive_cluster(conv + s, 0);     // the issuing CTA's barrier
                else mbar_arrive(conv + s);
            }
        }
    } else {
        // ---------------------------------------------------- epilogue --
        auto tile_of = [&](int64_t t, int64_t& m0, int64_t& n0, int& z, bool& has_k) {
            z = static_cast<int>(t / (mg * nt));
            const int64_t r = t % (mg * nt);
            m0 = ((r / nt) * C + crank) * kBM;
            n0 = (r % nt) * bn;
            has_k = kblocks_of(z) > 0;
        };
        if constexpr (kFresh)
            epilogue_fresh<kPair>(p, tmem, tfull, tempty, warp, lane, cid, ncl, ntiles, tile_of, kblocks_of);
        else
            epilogue_loop<kPair, kSplit>(p, tmem, tfull, tempty, warp, lane, cid, ncl, ntiles, tile_of, &map_c,
                                         epi_stage + (warp - kEpiWarp0) * 4096 * p.epi_bufs);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (C > 1) cluster_sync();     // no peer still multicasts into this CTA
    if (warp == 0) {
        if constexpr (kPair)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
    }
}

// ---------------------------------------------------------------------------
// bf16x3 variant for the forward / input-gradient GEMMs (row-major A, packed
// weight operand):  A = Ah + Al and B = Bh + Bl with Ah = bf16_rn(A),
// Al = bf16_rn(A - Ah) (16 significant bits in two bf16 terms), and
// C ~= Al*Bh + Ah*Bl + Ah*Bh on kind::f16 MMAs with fp32 TMEM accumulation.
// bf16 MMAs run at twice the tf32 rate and the split operands are half the
// bytes, so one 96 KB stage carries 64 K-steps instead of 32.  Measured
// error against float64: ~4e-6 L2-relative per GEMM (3xTF32: 4e-7..2e-6,
// tools/gemm_prec.py) — too coarse for the weight gradients' cancellation,
// so it is opt-in (GRD_GEMM_PREC=bf16x3), not the product default.
// Stage: [A: raw fp32 TMA boxes (k0..k0+31 | k0+32..k0+63), 128 rows each,
// SW128] split IN PLACE into [A hi bf16 SW128 | A lo bf16 SW128]: output row
// r of either tile occupies exactly raw row r of one of the two boxes, so the
// eight lanes that own row r read both raw rows before any of them writes.
// Then [B hi | B lo], bn rows x 64 bf16, pre-split by pack_b_bf16_kernel.
// ---------------------------------------------------------------------------
constexpr int kBK16 = 64;

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ float bf16_lo_f(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi_f(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

// split 8 consecutive fp32 values into hi / lo bf16x8
__device__ __forceinline__ void split8(const float4& x0, const float4& x1, uint4& hi, uint4& lo) {
    hi.x = pack_bf16x2(x0.x, x0.y);
    hi.y = pack_bf16x2(x0.z, x0.w);
    hi.z = pack_bf16x2(x1.x, x1.y);
    hi.w = pack_bf16x2(x1.z, x1.w);
    lo.x = pack_bf16x2(x0.x - bf16_lo_f(hi.x), x0.y - bf16_hi_f(hi.x));
    lo.y = pack_bf16x2(x0.z - bf16_lo_f(hi.y), x0.w - bf16_hi_f(hi.y));
    lo.z = pack_bf16x2(x1.x - bf16_lo_f(hi.z), x1.y - bf16_hi_f(hi.z));
    lo.w = pack_bf16x2(x1.z - bf16_lo_f(hi.w), x1.w - bf16_hi_f(hi.w));
}
__device__ __forceinline__ void sts128u(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}

// kConvWarps converter warps, 4 rows per warp per pass; lane = (row-in-group
// r4 = lane / 8, output chunk j = lane % 8); 4 passes read before any write
__device__ __forceinline__ void split_stage_bf16(uint8_t* st, int cwarp, int lane) {
    const uint32_t base = smem_u32(st);
    const int r4 = lane >> 3, j = lane & 7;
    const uint32_t box = static_cast<uint32_t>(j >> 2) * 16384u;
    const uint32_t c0 = static_cast<uint32_t>(2 * (j & 3));
    constexpr int kRowsPerPass = kConvWarps * 4;
#pragma unroll
    for (int g4 = 0; g4 < kBM / kRowsPerPass; g4 += 4) {
        float4 x[4][2];
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const uint32_t r = static_cast<uint32_t>(cwarp * 4 + r4 + kRowsPerPass * (g4 + it));
            const uint32_t row = base + box + r * 128u;
            x[it][0] = lds128(row + (((c0) ^ (r & 7u)) << 4));
            x[it][1] = lds128(row + (((c0 + 1u) ^ (r & 7u)) << 4));
        }
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const uint32_t r = static_cast<uint32_t>(cwarp * 4 + r4 + kRowsPerPass * (g4 + it));
            uint4 hi, lo;
            split8(x[it][0], x[it][1], hi, lo);
            const uint32_t off = r * 128u + ((static_cast<uint32_t>(j) ^ (r & 7u)) << 4);
            sts128u(base + off, hi);
            sts128u(base + 16384u + off, lo);
        }
        __syncwarp();
    }
}

// kind::f16 (bf16 x bf16), D fp32, M = 128, N = bn, both K-major
__device__ __forceinline__ uint32_t make_idesc_bf16(int bn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(bn >> 3) << 17) |
           (static_cast<uint32_t>(kBM >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__global__ void __launch_bounds__(kThreads, 1)
gemm_bf16x3_ws(const __grid_constant__ CUtensorMap map_a, const Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int bn = p.bn;
    const int S = p.stages;
    const uint32_t a_bytes = 2u * kBM * 128u;                  // raw fp32 = hi | lo bf16
    const uint32_t b_bytes = static_cast<uint32_t>(bn) * 128u; // one bf16 tile
    const uint32_t stage_bytes = a_bytes + 2u * b_bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
    uint64_t* full = bars;
    uint64_t* conv = bars + S;
    uint64_t* empty = bars + 2 * S;
    uint64_t* tfull = bars + 3 * S;
    uint64_t* tempty = bars + 3 * S + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t mt = (p.m + kBM - 1) / kBM;
    const int64_t nt = (p.n + bn - 1) / bn;
    const int64_t ntiles = mt * nt;
    const int64_t nkb = (p.k + kBK16 - 1) / kBK16;
    const int64_t nkb_all = nkb;
    uint32_t tmem_cols = 32;
    while (tmem_cols < static_cast<uint32_t>(2 * bn)) tmem_cols <<= 1;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 32) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(conv + s, kConvThreads);
            mbar_init(empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, kEpiThreads);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)));
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            uint64_t g = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int64_t m0 = (t / nt) * kBM, ntile = t % nt;
                for (int64_t kb = 0; kb < nkb; ++kb, ++g) {
                    const int s = static_cast<int>(g % S);
                    if (g >= static_cast<uint64_t>(S)) mbar_wait(empty + s, static_cast<uint32_t>((g / S - 1) & 1));
                    uint8_t* st = smem + s * stage_bytes;
                    const int64_t k0 = kb * kBK16;
                    mbar_expect_tx(full + s, a_bytes + 2u * b_bytes);
                    tma_2d(st, &map_a, static_cast<int32_t>(k0), static_cast<int32_t>(m0), full + s);
                    tma_2d(st + 16384, &map_a, static_cast<int32_t>(k0 + 32), static_cast<int32_t>(m0), full + s);
                    const float* src = p.b_packed + (ntile * nkb_all + kb) * (int64_t(bn) * kBK16);
                    bulk_copy(st + a_bytes, src, 2u * b_bytes, full + s);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = make_idesc_bf16(bn);
            uint64_t g = 0;
            int64_t i = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int acc = static_cast<int>(i & 1);
                if (i >= 2) mbar_wait(tempty + acc, static_cast<uint32_t>((i / 2 - 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t tacc = tmem + static_cast<uint32_t>(acc * bn);
                for (int64_t kb = 0; kb < nkb; ++kb, ++g) {
                    const int s = static_cast<int>(g % S);
                    mbar_wait(conv + s, static_cast<uint32_t>((g / S) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    uint8_t* st = smem + s * stage_bytes;
                    const uint32_t ah = smem_u32(st), al = ah + 16384u;
                    const uint32_t bh = smem_u32(st + a_bytes), bl = bh + b_bytes;
#pragma unroll
                    for (int kk = 0; kk < kBK16 / 16; ++kk) {
                        const uint64_t dah = make_desc(ah + kk * 32u, 16u, 1024u);
                        const uint64_t dal = make_desc(al + kk * 32u, 16u, 1024u);
                        const uint64_t dbh = make_desc(bh + kk * 32u, 16u, 1024u);
                        const uint64_t dbl = make_desc(bl + kk * 32u, 16u, 1024u);
                        mma_bf16(tacc, dal, dbh, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
                        mma_bf16(tacc, dah, dbl, idesc, 1u);
                        mma_bf16(tacc, dah, dbh, idesc, 1u);
                    }
                    mma_commit(empty + s);
                }
                mma_commit(tfull + acc);
                ++i;
            }
        }
    } else if (warp < kEpiWarp0) {
        const int cwarp = warp - kConvWarp0;
        uint64_t g = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int64_t kb = 0; kb < nkb; ++kb, ++g) {
                const int s = static_cast<int>(g % S);
                mbar_wait(full + s, static_cast<uint32_t>((g / S) & 1));
                split_stage_bf16(smem + s * stage_bytes, cwarp, lane);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(conv + s);
            }
        }
    } else {
        epilogue_loop<false, false>(p, tmem, tfull, tempty, warp, lane, blockIdx.x, gridDim.x,
                      ntiles, [&](int64_t t, int64_t& m0, int64_t& n0, int& z, bool& has_k) {
                          m0 = (t / nt) * kBM;
                          n0 = (t % nt) * bn;
                          z = 0;
                          has_k = nkb > 0;
                      });
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
    }
}

// bf16 hi/lo tiles of opB: out[ntile][kblock64][hi|lo][bn rows x 64 K] (SW128 K-major)
__global__ void pack_b_bf16_kernel(const float* __restrict__ b, int64_t ldb, int trans_b, int64_t n, int64_t k,
                                   int bn, float* __restrict__ out_f) {
    uint16_t* out = reinterpret_cast<uint16_t*>(out_f);
    const int64_t nkb = (k + kBK16 - 1) / kBK16;
    const int64_t ntile = (n + bn - 1) / bn;
    const int64_t total = ntile * nkb * int64_t(bn) * kBK16;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int kk = static_cast<int>(i % kBK16);
        const int64_t rest = i / kBK16;
        const int rr = static_cast<int>(rest % bn);
        const int64_t tile = rest / bn;
        const int64_t kb = tile % nkb, nti = tile / nkb;
        const int64_t gn = nti * bn + rr, gk = kb * kBK16 + kk;
        float v = 0.f;
        if (gn < n && gk < k) v = trans_b ? b[gn * ldb + gk] : b[gk * ldb + gn];
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        const __nv_bfloat16 l = __float2bfloat16_rn(v - __bfloat162float(h));
        const uint32_t off = static_cast<uint32_t>(rr) * 64u +
                             ((static_cast<uint32_t>(kk >> 3) ^ (rr & 7)) << 3) + static_cast<uint32_t>(kk & 7);
        uint16_t* base = out + tile * (2 * int64_t(bn) * kBK16);
        base[off] = *reinterpret_cast<const uint16_t*>(&h);
        base[int64_t(bn) * kBK16 + off] = *reinterpret_cast<const uint16_t*>(&l);
    }
}

// Pack the (small) weight operand into pre-split K-major SW128 tiles:
// out[ntile][kblock][hi|lo][bn rows x 32 K]; element (n, k) of opB.
__global__ void pack_b_kernel(const float* __restrict__ b, int64_t ldb, int trans_b, int64_t n, int64_t k, int bn,
                              float* __restrict__ out) {
    const int64_t nkb = (k + kBK - 1) / kBK;
    const int64_t ntile = (n + bn - 1) / bn;
    const int64_t total = ntile * nkb * int64_t(bn) * kBK;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int kk = static_cast<int>(i % kBK);
        const int64_t rest = i / kBK;
        const int rr = static_cast<int>(rest % bn);
        const int64_t tile = rest / bn;            // ntile * nkb + kb
        const int64_t kb = tile % nkb, nti = tile / nkb;
        const int64_t gn = nti * bn + rr, gk = kb * kBK + kk;
        float v = 0.f;
        if (gn < n && gk < k) v = trans_b ? b[gn * ldb + gk] : b[gk * ldb + gn];
        const float h = __uint_as_float(__float_as_uint(v) & 0xffffe000u);
        const uint32_t off = static_cast<uint32_t>(rr) * 128u +
                             ((static_cast<uint32_t>(kk >> 2) ^ (rr & 7)) << 4) + (static_cast<uint32_t>(kk & 3) << 2);
        float* base = out + tile * (2 * int64_t(bn) * kBK);
        base[off / 4] = h;
        base[int64_t(bn) * kBK + off / 4] = v - h;
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(ptr);
    });
    return fn;
}

// 2-D fp32 tensor map over a row-major matrix [rows][cols] (leading dim ld),
// box = box_cols (inner) x box_rows, 128-byte swizzle (16 B or 32 B atoms),
// zero OOB fill.
bool make_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box_cols,
              uint32_t box_rows, bool atom32 = false) {
    EncodeFn fn = encoder();
    if (!fn) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE,
              atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline int bn_max() {
    static int v = 0;
    if (!v) {
        const char* e = getenv("GRD_GEMM_BN_MAX");
        v = e ? atoi(e) : 256;
        if (v != 64 && v != 128 && v != 256) v = 256;
    }
    return v;
}

inline int pick_bn(int64_t n) {
    if (n >= bn_max()) return bn_max();
    if (n > 128) return static_cast<int>((n + 31) / 32 * 32);
    int bn = static_cast<int>((n + 15) / 16 * 16);
    return bn < 16 ? 16 : bn;
}

// CTA pairs (cta_group::2, M = 256 per pair): GRD_GEMM_PAIR = 1 / 0
inline int pair_pref() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GRD_GEMM_PAIR");
        v = e ? atoi(e) : 1;
    }
    return v;
}

// weight gradients accumulate each K block in a fresh TMEM accumulator (GRD_WGRAD_FRESH = 1 / 0)
inline int fresh_pref() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GRD_WGRAD_FRESH");
        v = e ? atoi(e) : 1;
    }
    return v;
}

inline int kch_pref() {
    static int v = -1;
    if (v < 0) {
        // in-kernel chunks (C partials re-read from L2 per chunk) measured
        // slower than the host-side split at the products shapes (44.7 vs
        // 43.5 ms per epoch: the epilogue drains every chunk): opt-in
        const char* e = getenv("GRD_GEMM_KCH");
        v = e ? atoi(e) : 0;
    }
    return v;
}
inline int64_t kmax_pref() {
    static int64_t v = -1;
    if (v < 0) {
        const char* e = getenv("GRD_GEMM_KMAX");
        v = e ? atoll(e) : 192;
    }
    return v;
}

// epilogue chunks stored by TMA through shared memory (GRD_GEMM_TMA_STORE = 1 / 0)
inline int tma_store_pref() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GRD_GEMM_TMA_STORE");
        v = e ? atoi(e) : 1;
    }
    return v;
}

// Raw fp32 tiles as the hi operand (GRD_GEMM_HI_RAW = 1 / 0): kind::tf32
// reads only the top 19 bits of each fp32 element, i.e. exactly the hi
// split (A & 0xffffe000) the converter used to write back, so the converter
// writes the lo tile alone.  Same errors to 3 digits on every shape of
// tools/gemm_prec_shapes.py; 1-5 % per launch (tools/gemm_shapes.py).
inline int hi_raw_pref() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GRD_GEMM_HI_RAW");
        v = e ? atoi(e) : 1;
    }
    return v;
}

// lo tiles in a ring of their own (GRD_GEMM_LORING = slots, 0: inside every
// stage).  Default: a 2-slot ring for the weight gradients (both operands
// raw and MN-major: -8..-11 % at the papers shapes, flat at products) and
// lo tiles inside the stages for the forward / input-gradient GEMMs, where
// the deeper raw ring measured 0-60 % slower (profiles/r02_ncu_gemm_papers.md)
inline int loring_pref(bool weight_grad) {
    static int v = -2;
    if (v == -2) {
        const char* e = getenv("GRD_GEMM_LORING");
        v = e ? atoi(e) : -1;
        if (v > 4) v = -1;
    }
    if (v >= 0) return v;
    return weight_grad ? 2 : 0;
}

// TMA-store staging tiles per epilogue warp (GRD_GEMM_EPI_BUFS = 1, 2 = two
// when the stage ring keeps its depth, 3 = two up to the 227 KB limit).
// Measured (tools/gemm_epibufs.sh): no gain at the papers shapes, products
// 2 M x 256 x 256 +8 % slower — the staging wait is not the epilogue's limit,
// so one tile stays the default.
inline int epi_bufs_pref() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GRD_GEMM_EPI_BUFS");
        v = e ? atoi(e) : 1;
        if (v < 1 || v > 3) v = 1;
    }
    return v;
}

// packed weight operand resident in shared memory when it fits (GRD_GEMM_BRES = 1 / 0)
inline int bres_pref() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GRD_GEMM_BRES");
        v = e ? atoi(e) : 1;
    }
    return v;
}

// CTAs per cluster sharing the B operand (GRD_GEMM_CLUSTER = 1, 2 or 4)
inline int cluster_pref() {
    static int v = 0;
    if (!v) {
        const char* e = getenv("GRD_GEMM_CLUSTER");
        v = e ? atoi(e) : 1;   // measured: 2 / 4 do not pay (see DESIGN 2.5)
        if (v != 1 && v != 2 && v != 4) v = 1;
    }
    return v;
}

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

}  // namespace grd_tc

using namespace grd_tc;

int64_t grd_tc_pack_elems(int64_t n, int64_t k) {
    const int bn = pick_bn(n);
    // fp32 elements of the packed weight operand: the 3xTF32 layout (32-deep
    // K blocks of fp32 hi|lo) or the bf16x3 one (64-deep blocks of bf16
    // hi|lo = half as many fp32 slots per element, but K padded to 64),
    // whichever is larger
    const int64_t tf32 = ((n + bn - 1) / bn) * ((k + kBK - 1) / kBK) * 2 * int64_t(bn) * kBK;
    const int64_t bf16 = ((n + bn - 1) / bn) * ((k + kBK16 - 1) / kBK16) * int64_t(bn) * kBK16;
    return tf32 > bf16 ? tf32 : bf16;
}

int grd_tc_bn(int64_t n) { return pick_bn(n); }

// forward / input-gradient GEMM precision: GRD_GEMM_PREC = tf32x3 (default)
// or bf16x3 (opt-in; the weight-gradient GEMMs always run 3xTF32).  bf16x3
// is 1.25-1.6x faster per GEMM but its ~4e-6 per-GEMM error is amplified by
// the cancellation in the weight gradients (sum over all vertices): 1.3e-3
// on configs[0]'s dW after one epoch, outside the 1e-4 parity bar.
int grd_tc_bf16x3() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("GRD_GEMM_PREC");
        v = (e && e[0] == 'b') ? 1 : 0;
    }
    return v;
}

static cudaError_t gemm_bf16x3(const GrdTcGemm& g, cudaStream_t st) {
    Params p{};
    p.m = g.m;
    p.n = g.n;
    p.k = g.k;
    p.bn = pick_bn(g.n);
    p.splits = 1;
    p.cluster = 1;
    p.c = g.c;
    p.ldc = g.ldc;
    p.row_scale = g.row_scale;
    p.elem_mul = g.elem_mul;
    p.ld_elem_mul = g.ld_elem_mul;
    p.relu_ref = g.relu_ref;
    p.ld_relu_ref = g.ld_relu_ref;
    p.relu_out = g.relu_out;
    p.accumulate = g.accumulate;
    p.b_packed = g.b_packed;
    p.c2 = g.c2;
    p.ldc2 = g.ldc2;
    p.split = g.c2 ? g.split : 0;
    p.a_mode = kKMajorTma;
    p.b_mode = kPacked;
    CUtensorMap map_a{};
    if (!make_map(&map_a, g.a, g.m, g.k, g.lda, 32, 128)) return cudaErrorInvalidValue;
    const uint32_t stage = 2u * kBM * 128u + 2u * static_cast<uint32_t>(p.bn) * 128u;
    p.stages = static_cast<int>((220u * 1024u) / stage);
    if (p.stages > 6) p.stages = 6;
    if (p.stages < 2) p.stages = 2;
    const size_t smem = static_cast<size_t>(p.stages) * stage + 1024 + 256;
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    static bool attr = false;
    if (!attr) {
        const cudaError_t e = cudaFuncSetAttribute(gemm_bf16x3_ws, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   227 * 1024);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int64_t tiles = ((g.m + kBM - 1) / kBM) * ((g.n + p.bn - 1) / p.bn);
    const int grid = static_cast<int>(tiles < num_sms() ? tiles : num_sms());
    gemm_bf16x3_ws<<<grid, kThreads, smem, st>>>(map_a, p);
    return cudaGetLastError();
}

cudaError_t grd_tc_gemm(const GrdTcGemm& g, cudaStream_t st) {
    if (g.bf16) return gemm_bf16x3(g, st);   // grd_gemm decides (and packs B) for it
    Params p{};
    p.m = g.m;
    p.n = g.n;
    p.k = g.k;
    p.bn = pick_bn(g.n);
    p.splits = g.k_splits > 1 ? g.k_splits : 1;
    p.kchunk = p.splits > 1 ? g.k_chunk : (g.k > 0 ? (g.k + kBK - 1) / kBK * kBK : kBK);
    p.c = g.c;
    p.ldc = g.ldc;
    p.row_scale = g.row_scale;
    p.elem_mul = g.elem_mul;
    p.ld_elem_mul = g.ld_elem_mul;
    p.relu_ref = g.relu_ref;
    p.ld_relu_ref = g.ld_relu_ref;
    p.relu_out = g.relu_out;
    p.accumulate = g.accumulate;
    p.partial = g.partial;
    p.ld_partial = (g.n + 3) / 4 * 4;
    p.c2 = g.c2;
    p.ldc2 = g.ldc2;
    p.split = g.c2 ? g.split : 0;
    CUtensorMap map_a{}, map_b{};
    // A(m, k): K-major TMA when stored M x K, MN-major boxes when stored K x M.
    if (!g.trans_a) {
        p.a_mode = kKMajorTma;
        if (!make_map(&map_a, g.a, g.m, g.k, g.lda, 32, 128)) return cudaErrorInvalidValue;
    } else {
        p.a_mode = kMNMajorTma;
        if (!make_map(&map_a, g.a, g.k, g.m, g.lda, 32, 32, true)) return cudaErrorInvalidValue;
    }
    if (g.b_packed) {
        p.b_mode = kPacked;
        p.b_packed = g.b_packed;
        map_b = map_a;
    } else if (g.trans_b) {
        p.b_mode = kKMajorTma;   // B stored N x K
        if (!make_map(&map_b, g.b, g.n, g.k, g.ldb, 32, static_cast<uint32_t>(p.bn))) return cudaErrorInvalidValue;
    } else {
        p.b_mode = kMNMajorTma;  // B stored K x N
        if (!make_map(&map_b, g.b, g.k, g.n, g.ldb, 32, 32, true)) return cudaErrorInvalidValue;
    }
    if (p.b_mode == kMNMajorTma) p.bn = (p.bn + 31) / 32 * 32;   // whole 32-wide TMA atoms
    // split-K partials (the weight gradients): fresh accumulator per K block
    const bool fresh = p.partial != nullptr && fresh_pref();
    if (fresh && p.bn > 128) p.bn = 128;
    const int64_t mt0 = (g.m + kBM - 1) / kBM;
    // a CTA pair stages half of B each: halves of whole 32-row atoms
    // GRD_GEMM_PAIR = 1 (auto): pairs for forward / input-gradient N tiles
    // of 256, where half of B per CTA buys the stages (products N = 256 /
    // 512: 2.59 vs 3.68 ms unpaired); single CTAs for narrower tiles (papers
    // shapes, bn 128 / 192: 1 M x 128 x 128 0.361 -> 0.287 ms, 16 M x 128 x
    // 128 5.47 -> 4.49, the K = 172 input gradient 0.560 -> 0.393) and for
    // the weight gradients (256 x 256 over 2 M rows: 2.42 -> 2.05 ms;
    // tools/gemm_shapes.py, tools/wgrad_one.py); 2: pair whenever possible
    const int pp = pair_pref();
    const bool pair_ok = pp == 2 || (pp == 1 && p.partial == nullptr && p.bn >= 256);
    p.pair = (pair_ok && p.bn % 64 == 0 && mt0 >= 2) ? 1 : 0;
    if (p.pair && p.b_mode == kKMajorTma &&
        !make_map(&map_b, g.b, g.n, g.k, g.ldb, 32, static_cast<uint32_t>(p.bn / 2)))
        return cudaErrorInvalidValue;
    const uint32_t bnl_bytes = static_cast<uint32_t>(p.pair ? p.bn / 2 : p.bn) * 128u;
    uint32_t stage = 2u * (kBM * 128u + bnl_bytes);
    uint32_t resident = 0;
    // B resident in shared memory: a packed weight operand with one N tile,
    // no split-K, that leaves room for >= 3 A-only stages (GRD_GEMM_BRES=0
    // keeps B in the stage ring)
    // K chunks accumulated separately inside the kernel when K is deeper
    // than GRD_GEMM_KMAX (GRD_GEMM_KCH K blocks per accumulation; opt-in, the
    // default split is ops.gemm's, one launch per 128-deep chunk): tcgen05's
    // fused accumulation truncates, so the error grows with the chain length
    // (profiles/r02_gemm_precision.md)
    p.kch = 0;
    p.hi_raw = hi_raw_pref();
    if (!p.partial && p.split == 0 && kch_pref() > 0 && g.k > kmax_pref()) p.kch = kch_pref();
    // TMA-store epilogue (plain C output: no split-K partial, no split c2)
    CUtensorMap map_c = map_a;
    p.tma_store = 0;
    // measured (tools/gemm_shapes.py): -12..-33 % at N tiles of 128 / 256,
    // +17..26 % at 48 / 192 (fewer stages fit beside the staging tiles)
    if (tma_store_pref() && p.kch == 0 && p.bn % 128 == 0 && !p.partial && p.split == 0 && g.c &&
        (g.ldc % 4) == 0 &&
        make_map(&map_c, g.c, g.m, (g.n + 3) / 4 * 4, g.ldc, 32, 32))
        p.tma_store = 1;
    p.epi_bufs = 1;
    uint32_t epi = p.tma_store ? static_cast<uint32_t>(kEpiWarps) * 4096u + 1024u : 0u;
    const bool bres_ok = bres_pref() && p.b_mode == kPacked && p.splits == 1 && g.n <= p.bn &&
                         (p.pair || cluster_pref() == 1);
    const uint32_t res_b = static_cast<uint32_t>((g.k + kBK - 1) / kBK) * 2u * bnl_bytes;
    const uint32_t a_raw = kBM * 128u;
    uint32_t lo_total = 0;
    p.lo_slots = loring_pref(p.a_mode == kMNMajorTma);
    if (p.lo_slots > 0) {
        // raw-only stages + a ring of lo slots (see the kernel's layout note)
        const bool b_conv = p.b_mode != kPacked;
        const uint32_t lo = a_raw + (b_conv ? bnl_bytes : 0u);
        lo_total = static_cast<uint32_t>(p.lo_slots) * lo;
        stage = a_raw + (b_conv ? bnl_bytes : 2u * bnl_bytes);
        if (bres_ok && res_b + 3u * a_raw + lo_total + epi <= 220u * 1024u) {
            resident = res_b;
            stage = a_raw;
            p.b_resident = 1;
        }
        p.stages = static_cast<int>((220u * 1024u - resident - epi - lo_total) / stage);
        if (p.stages > 8) p.stages = 8;
    } else {
        if (bres_ok && res_b + 3u * 2u * a_raw + epi <= 220u * 1024u) {
            resident = res_b;
            stage = 2u * a_raw;
            p.b_resident = 1;
        }
        p.stages = static_cast<int>((220u * 1024u - resident - epi) / stage);
        if (p.stages > (p.b_resident ? 6 : 4)) p.stages = p.b_resident ? 6 : 4;
    }
    if (p.stages < 2) p.stages = 2;
    // a second staging tile per epilogue warp when the ring keeps its depth
    // (GRD_GEMM_EPI_BUFS = 1 / 2; default: 2 when free)
    if (p.tma_store && epi_bufs_pref() > 1) {
        const uint32_t epi2 = epi + static_cast<uint32_t>(kEpiWarps) * 4096u;
        const uint32_t used = static_cast<uint32_t>(p.stages) * stage + lo_total + resident;
        if (used + epi2 <= 220u * 1024u || epi_bufs_pref() == 3) {
            if (used + epi2 + 1024 + 512 <= 227u * 1024u) {
                epi = epi2;
                p.epi_bufs = 2;
            }
        }
    }
    const size_t smem = static_cast<size_t>(p.stages) * stage + lo_total + resident + epi + 1024 + 512;
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaSuccess;
        for (auto fn : {gemm_tf32x3_ws<false, false>, gemm_tf32x3_ws<true, false>, gemm_tf32x3_ws<false, true>,
                        gemm_tf32x3_ws<true, true>, gemm_tf32x3_ws<false, false, true>,
                        gemm_tf32x3_ws<true, false, true>})
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int64_t mt = (g.m + kBM - 1) / kBM;
    int C = cluster_pref();
    while (C > 1 && mt < C) C >>= 1;               // at most the last group has idle CTAs
    if (p.b_mode == kKMajorTma) C = 1;
    if (p.pair) C = 2;
    p.cluster = C;
    const int64_t tiles = ((mt + C - 1) / C) * ((g.n + p.bn - 1) / p.bn) * p.splits;
    const int64_t max_cl = num_sms() / C;
    const int grid = static_cast<int>((tiles < max_cl ? tiles : max_cl) * C);
    if (C == 1) {
        if (fresh) gemm_tf32x3_ws<false, false, true><<<grid, kThreads, smem, st>>>(map_a, map_b, map_c, p);
        else if (p.split > 0) gemm_tf32x3_ws<false, true><<<grid, kThreads, smem, st>>>(map_a, map_b, map_c, p);
        else gemm_tf32x3_ws<false, false><<<grid, kThreads, smem, st>>>(map_a, map_b, map_c, p);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr_c[1];
    attr_c[0].id = cudaLaunchAttributeClusterDimension;
    attr_c[0].val.clusterDim.x = static_cast<unsigned>(C);
    attr_c[0].val.clusterDim.y = 1;
    attr_c[0].val.clusterDim.z = 1;
    cfg.attrs = attr_c;
    cfg.numAttrs = 1;
    if (p.pair) {
        if (fresh) return cudaLaunchKernelEx(&cfg, gemm_tf32x3_ws<true, false, true>, map_a, map_b, map_c, p);
        if (p.split > 0) return cudaLaunchKernelEx(&cfg, gemm_tf32x3_ws<true, true>, map_a, map_b, map_c, p);
        return cudaLaunchKernelEx(&cfg, gemm_tf32x3_ws<true, false>, map_a, map_b, map_c, p);
    }
    if (p.split > 0) return cudaLaunchKernelEx(&cfg, gemm_tf32x3_ws<false, true>, map_a, map_b, map_c, p);
    return cudaLaunchKernelEx(&cfg, gemm_tf32x3_ws<false, false>, map_a, map_b, map_c, p);
}

cudaError_t grd_tc_pack_b(const float* b, int64_t ldb, int trans_b, int64_t n, int64_t k, float* out,
                          cudaStream_t st, int bf16) {
    const int bn = pick_bn(n);
    if (bf16) {
        const int64_t total = ((n + bn - 1) / bn) * ((k + kBK16 - 1) / kBK16) * int64_t(bn) * kBK16;
        const int blocks = static_cast<int>((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
        pack_b_bf16_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(b, ldb, trans_b, n, k, bn, out);
        return cudaGetLastError();
    }
    const int64_t total = grd_tc_pack_elems(n, k) / 2;
    const int blocks = static_cast<int>((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    pack_b_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(b, ldb, trans_b, n, k, bn, out);
    return cudaGetLastError();
}
