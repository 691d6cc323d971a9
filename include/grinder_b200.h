/*
 * grinder_b200.h — C ABI of the B200-native partition-wise GNN training step.
 *
 * This is the drop-in boundary for the hot path named by BASELINE.json's
 * north_star: GriNNder's partition-wise full-graph training step
 * (reference package `grinder`, /root/reference/pkg/src/grinder).  The
 * reference has no FFI — its boundary is the Python API in training.py,
 * plan.py and partition.py — so every entry point below names the Python
 * function it replaces.  The Python package `paper_2605_11517_b200`
 * binds these with ctypes and keeps the reference's
 * function names, argument meaning and ValueError behaviour.
 *
 * Conventions
 *   - Plain C types only: pointers, int32/int64 sizes and leading
 *     dimensions, and the CUDA stream passed as `void*` (a cudaStream_t).
 *   - Return value: 0 = ok, < 0 = argument error, > 0 = cudaError_t.
 *     grd_last_error() returns a thread-local message for the last failure.
 *   - Ownership: the caller allocates every buffer (device buffers come from
 *     torch's caching allocator); the library never frees caller memory.
 *     Opaque handles (grd_plan_*) own host memory until *_destroy.
 *   - Device calls are asynchronous on the given stream and re-entrant; the
 *     caller synchronises.  All reductions use fixed orders: no float
 *     atomics, so every result is bitwise reproducible run to run.
 *   - Dense row-major fp32 matrices carry a leading dimension (ld, elements);
 *     activation buffers are padded to ld = round_up(width, 4) with zero
 *     padding columns so rows are 16-byte aligned for 128-bit accesses.
 */
#ifndef GRINDER_B200_H
#define GRINDER_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GRD_ABI_VERSION 1

int grd_abi_version(void);
const char* grd_last_error(void);
/* Number of SMs of the current device (for grid sizing by the host side). */
int grd_device_sm_count(int32_t* sm_count);

/* ------------------------------------------------------------------------
 * Host-side preprocessing (runs on CPU cores; no GPU needed).
 * --------------------------------------------------------------------- */

/* Symmetric Kronecker/RMAT graph, bit-exact with
 * graph.py:158-209 generate_kronecker(scale, avg_degree, seed).
 * `pcg_state` = {state_hi, state_lo, inc_hi, inc_lo} of
 * numpy.random.PCG64(seed) (the stream numpy would draw from) and `cum` the
 * f64 cumulative initiator np.cumsum((0.57,0.19,0.19,0.05)).  Writes CSR
 * src_ptr[2^scale + 1] and dst_idx[<= dst_capacity]; *num_edges_out gets |E|. */
int grd_kronecker_generate(int32_t scale, int64_t avg_degree,
                           const uint64_t* pcg_state, const double* cum,
                           int64_t* src_ptr, int32_t* dst_idx,
                           int64_t dst_capacity, int64_t* num_edges_out,
                           int32_t num_threads);
/* GPU variant of one generator round (graph.py:158-209): the `batch` vertex
 * pairs of the round as canonical keys lo * 2^scale + hi (-1 for a self
 * loop) into device memory `keys`.  pcg_words = {state_hi, state_lo, inc_hi,
 * inc_lo} of the PCG64 stream at the round's start, then {mul_hi, mul_lo,
 * add_hi, add_lo} of the LCG jump by `batch` steps; cum = the cumulative
 * initiator (host arrays).  Deduplication / CSR build are the caller's
 * (graph.generate_kronecker(..., device="cuda")). */
int grd_kronecker_keys(int32_t scale, int64_t batch, const uint64_t* pcg_words,
                       const double* cum, int64_t* keys, void* stream);

/* Rows of make_random_dataset's feature matrix (dataset.py:75-98) on the
 * device, bit-exact with numpy: out[i, :F] = features[rows[i]] (rows NULL:
 * the contiguous rows row0 .. row0 + n_rows - 1), pcg_words = {state_hi,
 * state_lo, inc_hi, inc_lo} of PCG64(seed).  Lets each rank of a sharded
 * run create only its own rows. */
int grd_feature_rows(const uint64_t* pcg_words, const int64_t* rows, int64_t row0,
                     int64_t n_rows, int32_t feature_dim, float* out, int64_t ld_out,
                     void* stream);

/* Switching-aware partitioner, bit-exact with partition.py:254-321
 * switching_aware_partition (its numba kernels _analyze_kernel :140-200 and
 * _relocate_kernel :203-251).  `labels` holds random_partition()'s labels on
 * entry (partition.py:103-111, drawn by numpy on the host) and the final
 * labels on exit.  objective_trace needs max_iters slots, max_size_trace
 * max_iters + 1. */
typedef struct grd_partitioner_params {
    double alpha_balance;
    double beta;
    double epsilon;
    int32_t patience;
    int32_t group_depth;
    int32_t max_iters;
    int32_t reserved;
} grd_partitioner_params;

int grd_sa_partition(int64_t num_vertices, const int64_t* src_ptr,
                     const int32_t* dst_idx, int32_t num_partitions,
                     const grd_partitioner_params* params, int32_t* labels,
                     double* objective_trace, int64_t* max_size_trace,
                     double* initial_objective, int32_t* iterations,
                     int32_t* converged, int32_t num_threads);

/* Device analysis pass of the switching-aware partitioner (partition.py:
 * 140-200 _analyze_kernel; GPU variant of the analysis inside
 * grd_sa_partition): for every vertex v of the device CSR, with `labels`
 * and the partition `sizes` (int64[p]) of the current iteration, writes its
 * f64 objective term terms[v] = (1 + share_own) - sizes[own] / denom and its
 * preference slots prefs[s * n + v] (s < group_depth; the top partitions of
 * its out-neighbours by (count desc, id asc), all slots = p when the top one
 * is its own partition or it has no neighbours), and adds the number of
 * candidates (top partition != own) to *num_candidates (device u64).  The
 * caller sums `terms` sequentially in vertex order (grd_sum_sequential) and
 * relocates (partition.switching_aware_partition(..., device="cuda")).
 * 2 <= num_partitions <= 1024.  All pointers are device memory. */
int grd_sa_analyze(int64_t num_vertices, const int64_t* src_ptr, const int32_t* dst_idx,
                   const int32_t* labels, const int64_t* sizes, int32_t num_partitions,
                   int32_t group_depth, double denom, double* terms, int32_t* prefs,
                   unsigned long long* num_candidates, void* stream);

/* Left-to-right f64 sum of x[0..n) (the reference's sequential objective
 * loop, partition.py:190-199), host memory. */
int grd_sum_sequential(const double* x, int64_t n, double* out);

/* Partition plan, bit-exact with plan.py:75-136 build_partition_plan.
 * Layout (concatenated over partitions in ascending id):
 *   part_ptr[P+1]        offsets of each partition's targets in perm
 *   perm[V]              targets of partition 0 ascending, then 1, ...
 *   in_ptr[V+1]          edge offsets per perm row (== concatenated tgt_ptr)
 *   in_src[E]            global source vertex of each edge
 *   in_src_pos[E]        its gather-map position (== src_pos)
 *   gather_ptr[P+1]      offsets of each partition's gather map
 *   gather_map[sum G]    gather maps, each sorted by (owner, vertex id)
 *   self_pos[V]          gather position of each target (perm order)
 *   in_degree[V]         global in-degree per vertex
 * Edges of one target are ordered by ascending gather position. */
typedef struct grd_plan grd_plan;
int grd_plan_create(int64_t num_vertices, const int64_t* src_ptr,
                    const int32_t* dst_idx, const int32_t* labels,
                    int32_t num_partitions, int32_t num_threads,
                    grd_plan** plan_out);
int grd_plan_sizes(const grd_plan* plan, int64_t* num_edges,
                   int64_t* gather_total);
int grd_plan_export(const grd_plan* plan, int64_t* part_ptr, int32_t* perm,
                    int64_t* in_ptr, int32_t* in_src, int32_t* in_src_pos,
                    int64_t* gather_ptr, int32_t* gather_map,
                    int32_t* self_pos, int32_t* in_degree);
void grd_plan_destroy(grd_plan* plan);

/* Host-tier row movement for the structured-storage-offloading (SSO) path
 * (hierarchy.py:549-583 charges these bytes):
 *   gather      dst[i,:] = src[idx[i],:]     (regather of GA_p from the host cache)
 *   scatter-add dst[idx[i],:] += src[i,:]   (host gradient write-back buffer;
 *                                            idx duplicate-free, training.py:166-175)
 * OpenMP over rows; row-major fp32 with leading dimensions. */
/* Stable CSR transpose (counting sort): col_ptr[n_cols+1], col_rows[nnz] =
 * for each column the referencing rows in ascending order (the edge order of
 * np.add.at in a partition's transposed aggregation, training.py:141). */
int grd_csr_transpose(int64_t n_rows, const int64_t* row_ptr, const int32_t* idx,
                      int64_t n_cols, int64_t* col_ptr, int32_t* col_rows);
/* Row-set equality: *equal_out = 1 iff sorted(row r of A) == row r of B
 * for every r (B rows ascending).  With B = grd_csr_transpose(A) this tests
 * that the graph is symmetric (the reference's generators are,
 * graph.py:158-209), so the streaming engine keeps one CSR in HBM for both
 * aggregation directions. */
int grd_csr_same_rows(int64_t n_rows, const int64_t* ptr_a, const int32_t* idx_a,
                      const int64_t* ptr_b, const int32_t* idx_b,
                      int32_t num_threads, int32_t* equal_out);
int grd_host_gather_rows(const float* src, int64_t ld_src, const int64_t* idx,
                         int64_t n_rows, int32_t width, float* dst,
                         int64_t ld_dst, int32_t num_threads);
int grd_host_scatter_add_rows(const float* src, int64_t ld_src,
                              const int64_t* idx, int64_t n_rows,
                              int32_t width, float* dst, int64_t ld_dst,
                              int32_t num_threads);

/* Storage tier (SSO, the ledger's gpu_storage /
 * host_storage links, hierarchy.py:519-583): page-cache-bypassing (O_DIRECT)
 * file I/O between tier files and page-locked host buffers, split into
 * 8 MiB requests served by num_threads threads.  offset, nbytes and the
 * buffer address must be multiples of grd_direct_alignment() (4096).
 * grd_direct_open reports in *direct_out whether O_DIRECT is in effect (a
 * filesystem without it falls back to buffered I/O).  Reads past the end of
 * the file return zeros. */
int64_t grd_direct_alignment(void);
int grd_direct_open(const char* path, int32_t writable, int64_t size, int32_t* fd_out,
                    int32_t* direct_out);
int grd_direct_close(int32_t fd);
int grd_direct_read(int32_t fd, int64_t offset, int64_t nbytes, void* dst, int32_t num_threads);
int grd_direct_write(int32_t fd, int64_t offset, int64_t nbytes, const void* src,
                     int32_t num_threads);

/* Row-run I/O of the SSO manager's tier files (hierarchy.py): run i is
 * records [first[i], first[i] + count[i]) of `record` bytes at file offset
 * first[i] * record, packed back to back in buf; write != 0 writes buf to
 * the file, else reads (past the end of the file reads zeros).  Buffered
 * pread / pwrite spread over num_threads threads by bytes. */
int grd_file_runs(int32_t fd, int32_t write, int64_t record, const int64_t* first,
                  const int64_t* count, int64_t nruns, void* buf, int32_t num_threads);
/* The same row runs between a packed buffer and a memory-mapped tier file
 * at `base` (memcpy into / out of the page cache, OpenMP over runs). */
int grd_mem_runs(void* base, int32_t write, int64_t record, const int64_t* first,
                 const int64_t* count, int64_t nruns, void* buf, int32_t num_threads);

/* ------------------------------------------------------------------------
 * Device kernels (sm_100a).  All take `stream` = cudaStream_t.
 * --------------------------------------------------------------------- */

/* K1 — row gather: dst[i,:] = src[idx[i],:]  (training.py:301,330
 * `acts[layer][topo.gather_map]`). */
int grd_gather_rows(const float* src, int64_t ld_src, const int32_t* idx,
                    int64_t n_rows, int32_t width, float* dst, int64_t ld_dst,
                    void* stream);

/* Strided 2-D copy (cudaMemcpy2DAsync, cudaMemcpyDefault) between device
 * and/or page-locked host memory: `rows` rows of `width_bytes` bytes, row
 * pitches in bytes.  The SSO tiers keep unpadded rows; device matrices are
 * padded — the host link moves exactly rows * width_bytes. */
int grd_memcpy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch,
                 int64_t width_bytes, int64_t rows, void* stream);

/* K9 — row scatter-add: dst[idx[i],:] += src[i,:] (training.py:166-175
 * scatter_accumulate; idx is duplicate-free). */
int grd_scatter_add_rows(const float* src, int64_t ld_src,
                         const int32_t* idx, int64_t n_rows, int32_t width,
                         float* dst, int64_t ld_dst, void* stream);

/* K2/K8 — CSR sum-aggregation (SpMM pull), one warp per row:
 *   s   = sum_{e in [row_ptr[r], row_ptr[r+1])} src_scale[idx[e]] * Y[idx[e],:]
 *       + src_scale[self] * Y[self,:]            (self = self_idx[r] or out row)
 *   out[out_row,:] = act( post(s) )
 * post: divide by (row degree + 1) (mean, training.py:61-65) and/or multiply
 * by post_scale[out_row] (symmetric norm).  Rows whose degree exceeds
 * heavy_threshold are split into fixed segments (heavy_* arrays) whose
 * partials are combined in segment order by the last finishing warp, so the
 * result is deterministic.  Forward aggregation (training.py:48-58), its
 * backward recompute (:113-114) and the transposed aggregation (:130-143,
 * pulled over a CSC/CSR of the opposite direction) all map onto this. */
typedef struct grd_agg_args {
    int64_t n_rows;
    const int64_t* row_ptr;
    const int32_t* idx;
    const int32_t* out_idx;    /* nullable: output row of row r (else r)  */
    const int32_t* self_idx;   /* nullable: self row (else out row); <0 none */
    const float* y;
    int64_t ldy;
    const float* src_scale;    /* nullable: per-Y-row multiplier           */
    const float* post_scale;   /* nullable: per-output-row multiplier      */
    int32_t post_div_deg;      /* 1: divide by (degree + 1) (mean with self loop);
                                  2: divide by degree (mean over neighbours; 0 if none) */
    int32_t relu;
    float* out;
    int64_t ldo;
    int32_t width;
    int32_t heavy_threshold;   /* <= 0: no splitting                       */
    int64_t n_heavy;
    const int32_t* heavy_rows;     /* [n_heavy] row indices                */
    const int64_t* heavy_seg_ptr;  /* [n_heavy+1] segment offsets          */
    const int32_t* seg_heavy;      /* [n_segs] owning heavy index          */
    int64_t n_segs;
    int32_t seg_len;               /* edges per segment                    */
    int32_t no_self;               /* 1: no implicit self term             */
    float* seg_partial;            /* [n_segs * round_up(width,4)] scratch */
    int32_t* heavy_counter;        /* [16 * n_heavy] zero on entry, zero on exit
                                      (one slot per heavy row and column chunk) */
    const float* mask_ref;         /* nullable: out = mask_ref[out_row,:] > 0 ? out : 0 */
    int64_t ld_mask_ref;
    const float* add_y;            /* nullable: add_y[out_row,:] added after post-scaling,
                                      before the activation (GraphSAGE root term) */
    int64_t ld_add_y;
    const float* edge_w;           /* nullable: per-edge, per-head weights [E, heads]
                                      replacing src_scale (GAT attention) */
    const int32_t* edge_w_perm;    /* nullable: weight row of edge e is edge_w_perm[e] */
    const float* self_w;           /* self-term weights [out rows, heads] (with edge_w) */
    int32_t heads;
    int32_t head_ld;               /* columns per head (multiple of 4) */
} grd_agg_args;

/* GAT edge softmax (builder-defined layer).  Rows are
 * aggregation targets (row_ptr/idx = in-edges, out_idx = vertex of a row);
 * p_ext rows hold [P (heads x dhp) | s (heads) | t (heads)].
 *   grd_gat_softmax:     alpha[e,h] = softmax over in(v) U {v} of
 *                        LeakyReLU(s_u + t_v); self loop in alpha_self[v,h]
 *   grd_gat_softmax_bwd: delta = alpha (gO_h[v].P_h[u] - gO_h[v].O_h[v])
 *                        lrelu'(z) per edge; dt_v = sum delta -> grad_ext
 *                        column hdp + H + h
 *   grd_gat_src_grad:    rows = sources over out-edges (edge_perm maps to the
 *                        in-edge order): ds_u = sum delta (+ self) -> grad_ext
 *                        column hdp + h
 * Rows above heavy_threshold (<= 128) edges are processed as seg_len-edge
 * segments by separate warps, combined in a fixed order (deterministic);
 * the segmentation is the same as grd_agg_args'. */
typedef struct grd_gat_args {
    int64_t n_rows;
    const int64_t* row_ptr;
    const int32_t* idx;
    const int32_t* out_idx;
    const int32_t* edge_perm;
    int32_t heavy_threshold;       /* light rows: at most this many edges (<= 128) */
    int32_t seg_len;               /* edges per heavy-row segment (<= 128) */
    int64_t n_heavy;
    const int32_t* heavy_rows;     /* [n_heavy] */
    const int64_t* heavy_seg_ptr;  /* [n_heavy+1] */
    const int32_t* seg_heavy;      /* [n_segs] */
    int64_t n_segs;
    float* seg_scratch;            /* [n_segs * 2 * heads] when n_segs > 0 */
    const float* p_ext;
    int64_t ld_ext;
    int32_t heads;                 /* 1..8 */
    int32_t hdp;                   /* heads * dhp (<= 256 for the backward) */
    int32_t dhp;                   /* padded per-head width, multiple of 4 */
    float slope;                   /* LeakyReLU negative slope (0.2) */
    float* alpha;
    float* alpha_self;
    const float* grad_o;           /* dL/dO [rows, hdp] (ld_go) */
    int64_t ld_go;
    const float* o_fwd;            /* forward aggregate O (relu(O) when grad_o is
                                      ReLU-masked) [rows, hdp] (ld_o) */
    int64_t ld_o;
    float* delta;
    float* delta_self;
    float* grad_ext;               /* dL/dP_ext: s and t columns written here */
    int64_t ld_gext;
    const float* st;               /* optional compact scores [rows, ld_st] for
                                      grd_gat_softmax: s_u in columns 0..H-1, t_v in H..2H-1
                                      (grd_gat_pack_scores); null: p_ext's s / t columns.
                                      The backward reads s_u beside the P_u row it gathers. */
    int64_t ld_st;
    int64_t n_small;               /* grd_gat_softmax, grd_gat_src_grad: the last n_small rows have at most
                                      3 in-edges each (caller's guarantee, e.g. the
                                      low-degree tail of a degree-sorted CSR; 0 = none):
                                      4 lanes per row instead of a warp */
    int64_t n_mid;                 /* the n_mid rows before those have at most 15
                                      in-edges each: 16 lanes per row (0 = none) */
    const float* c_dot;            /* grd_gat_pull_bwd: c[v, h] = gO_v,h . O_v,h
                                      (grd_gat_row_dots) [rows, heads] */
    const float* alpha_t;          /* grd_gat_pull_bwd, nullable: attention already
                                      in the pull's edge order [E, heads] */
    float* seg_wide;               /* grd_gat_pull_bwd: heavy-segment partials
                                      [n_segs, round_up(hdp + heads, 4)] */
} grd_gat_args;
int grd_gat_softmax(const grd_gat_args* args, void* stream);
int grd_gat_softmax_bwd(const grd_gat_args* args, void* stream);
int grd_gat_src_grad(const grd_gat_args* args, void* stream);
/* Fused GAT backward over the transposed pull (rows = sources u, idx = the
 * out-neighbours v, edge_perm = each pull edge's forward position):
 *   dalpha_uv,h = gO_v,h . P_u,h          (gO_v gathered once per edge)
 *   delta_uv,h  = alpha (dalpha - c_v,h) lrelu'(s_u,h + t_v,h)  -> delta[fwd e]
 *   dP_u        = sum_v alpha_uv gO_v + alpha_self gO_u         -> grad_ext[u, 0:hdp]
 *   ds_u,h      = sum_v delta_uv,h + delta_self_u,h             -> grad_ext[u, hdp + h]
 * replacing grd_gat_softmax_bwd's P_u row gather per in-edge.  The target
 * score gradients dt_v = sum over in-edges of delta follow from
 * grd_gat_dst_grad over the forward CSR. */
int grd_gat_pull_bwd(const grd_gat_args* args, void* stream);
/* dt_v,h = sum_{e in row v} delta[e, h] + delta_self[v, h] over the forward
 * CSR (edges in its own order) -> grad_ext[v, hdp + heads + h]. */
int grd_gat_dst_grad(const grd_gat_args* args, void* stream);
/* c[r, h] = sum_{d < dhp} g[r, h dhp + d] o[r, h dhp + d] (16-byte chunks in
 * order), the per-head gO . O of every row. */
int grd_gat_row_dots(const float* g, int64_t ld_g, const float* o, int64_t ld_o, int64_t n_rows,
                     int32_t heads, int32_t dhp, float* c, void* stream);
/* st[r, 0:2H] = p_ext[r, hdp : hdp + 2H]: the per-vertex attention scores as
 * one 32-byte row each (H = 4), so the edge-softmax's per-edge score gathers
 * hit a table that stays in L2 instead of one line of a wide P_ext row each. */
int grd_gat_pack_scores(const float* p_ext, int64_t ld_ext, int64_t n_rows, int32_t heads,
                        int32_t hdp, float* st, int64_t ld_st, void* stream);
/* W_ext = [W | W a_src | W a_dst] (att = [a_src; a_dst], each heads x dhp). */
int grd_gat_build_wext(const float* w, int64_t ldw, const float* att, int64_t d_in,
                       int32_t heads, int32_t dh, int32_t dhp, float* wext,
                       int64_t ld_ext, void* stream);
/* dW, datt from dW_ext, then W -= lr dW, att -= lr datt (lr = 0: no step). */
int grd_gat_param_grads(const float* dwext, int64_t ld_ext, float* w, int64_t ldw,
                        float* att, int64_t d_in, int32_t heads, int32_t dh,
                        int32_t dhp, float* dw, float* datt, float lr, void* stream);
/* Last GAT layer: out = mean over heads (backward = 1: spread dL/dout / heads). */
int grd_head_mean(const float* o, int64_t ldo, int64_t n_rows, int32_t heads,
                  int32_t dh, int32_t dhp, float* out, int64_t ld_out,
                  int32_t backward, void* stream);
int grd_agg_sum(const grd_agg_args* args, void* stream);

/* K3/K6/K7 — dense fp32 GEMM on tcgen05 tensor cores, 3xTF32 split
 * (fp32-grade accuracy), with fused epilogue (training.py:76,128-129):
 *   C[m,n] = epi( sum_k opA(A)[m,k] * opB(B)[k,n] )
 * transA: A stored K x M (lda);  transB: B stored N x K (ldb).  B (the
 * weight operand) is pre-split into `workspace`, which needs
 * grd_gemm_workspace(n, k) floats.  Leading dimensions must be multiples of
 * 4 and matrices 16-byte aligned (TMA).
 * epi: v = acc (+ C if accumulate); v *= row_scale[m]; v *= elem_mul[m,n];
 * v = relu_ref[m,n]>0 ? v : 0; relu_out: max(v,0); C = v.  Epilogue
 * pointers are nullable; columns up to round_up(n,4) are written. */
typedef struct grd_gemm_args {
    int64_t m, n, k;
    const float* a; int64_t lda; int32_t trans_a;
    int32_t trans_b;
    const float* b; int64_t ldb;
    float* c; int64_t ldc;
    const float* row_scale;
    const float* elem_mul; int64_t ld_elem_mul;
    const float* relu_ref; int64_t ld_relu_ref;
    int32_t relu_out;          /* apply max(acc, 0) */
    int32_t accumulate;
    float* workspace;          /* >= grd_gemm_workspace(n, k) floats */
    int64_t workspace_elems;
    float* c2; int64_t ldc2;   /* optional: columns >= split go to c2[:, col - split] */
    int64_t split;             /* (multiple of 4; not with accumulate / relu_ref / elem_mul) */
} grd_gemm_args;
int64_t grd_gemm_workspace(int64_t n, int64_t k);
int grd_gemm(const grd_gemm_args* args, void* stream);

/* K6 — weight gradient  dW = A^T B  with K = number of rows (long), as a
 * deterministic split-K: fixed row chunks write partials to `workspace`
 * ([splits, M, N]), then one ordered reduction writes dW (or adds to it when
 * `accumulate`, the ascending-pid sum of training.py:343) and, if w is
 * non-null, applies the SGD step W -= lr * dW (training.py:352-354).
 * workspace_elems must be >= grd_wgrad_workspace(m, n, k). */
int64_t grd_wgrad_workspace(int64_t m, int64_t n, int64_t k);
int grd_wgrad_sgd(int64_t m, int64_t n, int64_t k, const float* a,
                  int64_t lda, const float* b, int64_t ldb, float* dw,
                  int64_t lddw, int32_t accumulate, float* w, int64_t ldw,
                  float lr, float* workspace, int64_t workspace_elems,
                  void* stream);

/* K4 — masked softmax cross-entropy (model.py:102-129): per masked row,
 * loss -= log softmax(logits)[label]; grad = (softmax - onehot) / count *
 * grad_scale[row] (grad_scale nullable); unmasked rows get zero gradient and
 * the padding columns [n_classes, round_up(n_classes,4)) are zeroed.
 * stats_out (device, 4 doubles): {loss, accuracy, loss_sum, correct}.
 * `partials` needs grd_loss_partials(n_rows) doubles of scratch. */
int64_t grd_loss_partials(int64_t n_rows);
int grd_softmax_xent(const float* logits, int64_t ld_logits, int64_t n_rows,
                     int32_t n_classes, const int32_t* labels,
                     const uint8_t* mask, int64_t mask_count,
                     float* grad, int64_t ld_grad, const float* grad_scale,
                     double* partials, double* stats_out, void* stream);
/* grd_softmax_xent that also writes grad2[r, :] = grad[r, :] * grad2_scale[r]
 * (e.g. GraphSAGE's 1/deg source scale of the following transposed pull,
 * applied once per row instead of once per edge). */
int grd_softmax_xent2(const float* logits, int64_t ld_logits, int64_t n_rows,
                      int32_t n_classes, const int32_t* labels, const uint8_t* mask,
                      int64_t mask_count, float* grad, int64_t ld_grad,
                      const float* grad_scale, float* grad2, int64_t ld_grad2,
                      const float* grad2_scale, double* partials, double* stats_out,
                      void* stream);

/* Elementwise helpers. */
/* y[i,:] = x[i,:] * m[i,:]  (dropout, training.py:178-185,297). */
int grd_mul_rows(const float* x, int64_t ldx, const float* m, int64_t ldm,
                 int64_t n_rows, int32_t width, float* y, int64_t ldy,
                 void* stream);
/* y[i,:] = (ref[i,:] > 0 ? x[i,:] : 0) * row_scale[i]  (ReLU derivative
 * mask and degree scale, training.py:115-118,130-139); ref/row_scale
 * nullable; in-place allowed. */
int grd_mask_scale_rows(const float* x, int64_t ldx, const float* ref,
                        int64_t ldref, const float* row_scale, int64_t n_rows,
                        int32_t width, float* y, int64_t ldy, void* stream);
/* Row-L2 normalisation forward / backward (training.py:75-80,119-127). */
int grd_rownorm_fwd(const float* pre, int64_t ld, int64_t n_rows,
                    int32_t width, int32_t relu, const int32_t* out_idx,
                    float* out, int64_t ldo, void* stream);
int grd_rownorm_bwd(const float* pre, int64_t ldp, const float* grad_y,
                    int64_t ldg, const float* a_out, int64_t lda,
                    int64_t n_rows, int32_t width, const float* row_scale,
                    float* grad_pre, int64_t ldgp, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GRINDER_B200_H */
