// Host-side preprocessing for the partition-wise training step:
//   * the Kronecker/RMAT generator, reproducing numpy's PCG64 stream
//     (graph.py:158-209 generate_kronecker),
//   * the switching-aware partitioner (partition.py:140-321),
//   * the partition plan (plan.py:75-136 build_partition_plan).
// All three are integer/byte work on CPU cores: results are bit-exact with
// the reference for identical inputs, and independent of the thread count.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <vector>

#include "../../include/grinder_b200.h"
#include "grd_common.h"

namespace grd {

std::string& last_error_slot() {
    thread_local std::string slot;
    return slot;
}

namespace {

// ---------------------------------------------------------------- PCG64 --
// numpy's default bit generator: 128-bit LCG, XSL-RR 64-bit output, and
// random() = (next64 >> 11) * 2^-53 (numpy/random/src/pcg64).
using u128 = unsigned __int128;

const u128 kPcgMult = (static_cast<u128>(0x2360ED051FC65DA4ULL) << 64) |
                      0x4385DF649FCCF645ULL;

struct Pcg64 {
    u128 state;
    u128 inc;

    inline uint64_t next64() {
        state = state * kPcgMult + inc;
        const uint64_t hi = static_cast<uint64_t>(state >> 64);
        const uint64_t lo = static_cast<uint64_t>(state);
        const unsigned rot = static_cast<unsigned>(state >> 122);
        const uint64_t x = hi ^ lo;
        return (x >> rot) | (x << ((64u - rot) & 63u));
    }
    inline double next_double() {
        return static_cast<double>(next64() >> 11) * (1.0 / 9007199254740992.0);
    }
    // Jump the LCG ahead by `delta` steps (O(log delta)).
    void advance(uint64_t delta) {
        u128 cur_mult = kPcgMult, cur_plus = inc;
        u128 acc_mult = 1, acc_plus = 0;
        while (delta > 0) {
            if (delta & 1) {
                acc_mult *= cur_mult;
                acc_plus = acc_plus * cur_mult + cur_plus;
            }
            cur_plus = (cur_mult + 1) * cur_plus;
            cur_mult *= cur_mult;
            delta >>= 1;
        }
        state = acc_mult * state + acc_plus;
    }
};

// Open-addressing set of non-negative int64 keys (first-occurrence dedup).
class KeySet {
  public:
    explicit KeySet(int64_t expected) {
        uint64_t cap = 1024;
        while (cap < static_cast<uint64_t>(expected) * 2) cap <<= 1;
        slots_.assign(cap, -1);
        mask_ = cap - 1;
    }
    // Returns true if the key was newly inserted.
    bool insert(int64_t key) {
        uint64_t h = static_cast<uint64_t>(key);
        h ^= h >> 33; h *= 0xff51afd7ed558ccdULL; h ^= h >> 33;
        h *= 0xc4ceb9fe1a85ec53ULL; h ^= h >> 33;
        uint64_t i = h & mask_;
        while (true) {
            const int64_t s = slots_[i];
            if (s == key) return false;
            if (s < 0) { slots_[i] = key; ++size_; maybe_grow(); return true; }
            i = (i + 1) & mask_;
        }
    }
    int64_t size() const { return size_; }

  private:
    void maybe_grow() {
        if (static_cast<uint64_t>(size_) * 2 <= mask_ + 1) return;
        std::vector<int64_t> old;
        old.swap(slots_);
        slots_.assign(old.size() * 2, -1);
        mask_ = slots_.size() - 1;
        size_ = 0;
        for (int64_t k : old) if (k >= 0) insert(k);
    }
    std::vector<int64_t> slots_;
    uint64_t mask_ = 0;
    int64_t size_ = 0;
};

int threads_or_default(int32_t t) { return t > 0 ? t : omp_get_max_threads(); }

}  // namespace
}  // namespace grd

using namespace grd;

extern "C" int grd_abi_version(void) { return GRD_ABI_VERSION; }

extern "C" const char* grd_last_error(void) { return last_error_slot().c_str(); }

// --------------------------------------------------------------------------
// Kronecker generator (graph.py:158-209).  Each round draws `batch` vertex
// pairs by `scale` recursive quadrant picks; numpy draws level by level, so
// element i of level k is stream position base + k*batch + i.  Threads take
// contiguous element ranges and jump the LCG to their first position.
// --------------------------------------------------------------------------
extern "C" int grd_kronecker_generate(int32_t scale, int64_t avg_degree,
                                      const uint64_t* pcg_state, const double* cum,
                                      int64_t* src_ptr, int32_t* dst_idx,
                                      int64_t dst_capacity, int64_t* num_edges_out,
                                      int32_t num_threads) {
    clear_error();
    if (scale < 4 || scale > 30) return fail(kErrArg, "scale must be in [4, 30]");
    if (avg_degree < 1) return fail(kErrArg, "avg_degree must be positive");
    if (!pcg_state || !cum || !src_ptr || !dst_idx || !num_edges_out)
        return fail(kErrArg, "null argument");
    const int64_t n = int64_t{1} << scale;
    const int64_t target = (avg_degree * n) / 2;
    const int nt = threads_or_default(num_threads);

    Pcg64 base;
    base.state = (static_cast<u128>(pcg_state[0]) << 64) | pcg_state[1];
    base.inc = (static_cast<u128>(pcg_state[2]) << 64) | pcg_state[3];
    const double c0 = cum[0], c1 = cum[1], c2 = cum[2], c3 = cum[3];

    KeySet seen(target);
    std::vector<int64_t> keys;  // first-occurrence unique keys, <= target
    keys.reserve(static_cast<size_t>(target));
    std::vector<int64_t> src, dst;
    bool done = false;
    for (int round = 0; round < 64 && !done; ++round) {
        const int64_t remaining = target - seen.size();
        if (remaining <= 0) break;
        const int64_t batch = std::max<int64_t>(4 * remaining, 1024);
        src.assign(static_cast<size_t>(batch), 0);
        dst.assign(static_cast<size_t>(batch), 0);
#pragma omp parallel num_threads(nt)
        {
            const int tid = omp_get_thread_num();
            const int nth = omp_get_num_threads();
            const int64_t i0 = batch * tid / nth;
            const int64_t i1 = batch * (tid + 1) / nth;
            for (int level = 0; level < scale && i0 < i1; ++level) {
                Pcg64 rng = base;
                rng.advance(static_cast<uint64_t>(level) * batch + i0);
                for (int64_t i = i0; i < i1; ++i) {
                    const double r = rng.next_double();
                    // np.searchsorted(cum, r, side="right") = #{cum <= r}
                    const int64_t q = (c0 <= r) + (c1 <= r) + (c2 <= r) + (c3 <= r);
                    src[i] = (src[i] << 1) | (q >> 1);
                    dst[i] = (dst[i] << 1) | (q & 1);
                }
            }
        }
        base.advance(static_cast<uint64_t>(scale) * batch);
        // np.unique over everything collected decides whether to continue;
        // scanning in draw order until `target` uniques are seen is
        // equivalent, and also yields the first-occurrence survivors.
        for (int64_t i = 0; i < batch; ++i) {
            const int64_t lo = std::min(src[i], dst[i]);
            const int64_t hi = std::max(src[i], dst[i]);
            if (lo == hi) continue;
            const int64_t key = lo * n + hi;
            if (seen.insert(key)) {
                keys.push_back(key);
                if (static_cast<int64_t>(keys.size()) == target) { done = true; break; }
            }
        }
    }
    src.clear(); src.shrink_to_fit();
    dst.clear(); dst.shrink_to_fit();

    // _csr_from_pairs(concat(lo, hi), concat(hi, lo)): each source keeps its
    // edges in appearance order: first the (lo -> hi) edges, then (hi -> lo).
    const int64_t m = static_cast<int64_t>(keys.size());
    if (2 * m > dst_capacity) return fail(kErrArg, "dst_capacity %lld < %lld",
                                          (long long)dst_capacity, (long long)(2 * m));
    std::vector<int64_t> cursor(static_cast<size_t>(n) + 1, 0);
    for (int64_t k : keys) { ++cursor[k / n + 1]; ++cursor[k % n + 1]; }
    for (int64_t v = 0; v < n; ++v) cursor[v + 1] += cursor[v];
    std::memcpy(src_ptr, cursor.data(), sizeof(int64_t) * (n + 1));
    for (int64_t k : keys) dst_idx[cursor[k / n]++] = static_cast<int32_t>(k % n);
    for (int64_t k : keys) dst_idx[cursor[k % n]++] = static_cast<int32_t>(k / n);
    *num_edges_out = 2 * m;
    return 0;
}

// --------------------------------------------------------------------------
// Switching-aware partitioner (partition.py:254-321).
// --------------------------------------------------------------------------
namespace {

struct Analyzer {
    int64_t n;
    const int64_t* src_ptr;
    int32_t p;
    int32_t depth;
    int nt;
    std::vector<double> terms;

    // One pass of _analyze_kernel (partition.py:140-200).  Per-vertex work is
    // parallel; the f64 objective is summed sequentially in vertex order so
    // the convergence test sees the same bits as the reference.
    double run(const int32_t* dst_part, const int32_t* labels,
               const int64_t* sizes, double denom, int32_t* prefs,
               int64_t* num_candidates) {
        terms.resize(static_cast<size_t>(n));
        int64_t cand = 0;
#pragma omp parallel num_threads(nt) reduction(+ : cand)
        {
            std::vector<int64_t> counts(static_cast<size_t>(p), 0);
            std::vector<int32_t> touched(static_cast<size_t>(p));
#pragma omp for schedule(dynamic, 4096)
            for (int64_t v = 0; v < n; ++v) {
                const int64_t b = src_ptr[v], e = src_ptr[v + 1];
                const int64_t deg = e - b;
                int32_t k = 0;
                for (int64_t j = b; j < e; ++j) {
                    const int32_t c = dst_part[j];
                    if (counts[c] == 0) touched[k++] = c;
                    ++counts[c];
                }
                const int32_t own = labels[v];
                const double penalty = static_cast<double>(sizes[own]) / denom;
                if (deg > 0) {
                    const double share = static_cast<double>(counts[own]) /
                                         static_cast<double>(deg);
                    terms[v] = (1.0 + share) - penalty;
                } else {
                    terms[v] = 1.0 - penalty;
                }
                for (int32_t s = 0; s < depth; ++s) prefs[int64_t(s) * n + v] = p;
                if (k > 0) {
                    // Ranked by (count desc, id asc), top `depth` slots.
                    int64_t prev_count = int64_t{1} << 62;
                    int32_t prev_id = -1;
                    const int32_t top = depth < k ? depth : k;
                    for (int32_t s = 0; s < top; ++s) {
                        int32_t best = -1;
                        int64_t best_count = 0;
                        for (int32_t t = 0; t < k; ++t) {
                            const int32_t c = touched[t];
                            const int64_t cc = counts[c];
                            if (cc > prev_count || (cc == prev_count && c <= prev_id)) continue;
                            if (best == -1 || cc > best_count || (cc == best_count && c < best)) {
                                best = c;
                                best_count = cc;
                            }
                        }
                        if (best == -1) break;
                        prefs[int64_t(s) * n + v] = best;
                        prev_count = best_count;
                        prev_id = best;
                    }
                    if (prefs[v] == own) {
                        for (int32_t s = 0; s < depth; ++s) prefs[int64_t(s) * n + v] = p;
                    } else {
                        ++cand;
                    }
                }
                for (int32_t t = 0; t < k; ++t) counts[touched[t]] = 0;
            }
        }
        double objective = 0.0;
        for (int64_t v = 0; v < n; ++v) objective += terms[v];
        *num_candidates = cand;
        return objective;
    }
};

// np.lexsort(prefs[::-1]) restricted to candidates (all non-candidates carry
// the sentinel and sort last; the relocation loop stops there).  LSD radix
// over the slots with stable counting sorts = lexicographic, ties by id.
void candidate_order(int64_t n, int32_t p, int32_t depth, const int32_t* prefs,
                     std::vector<int64_t>& order, std::vector<int64_t>& tmp,
                     std::vector<int64_t>& bucket) {
    order.clear();
    for (int64_t v = 0; v < n; ++v)
        if (prefs[v] != p) order.push_back(v);
    tmp.resize(order.size());
    bucket.assign(static_cast<size_t>(p) + 2, 0);
    for (int32_t s = depth - 1; s >= 0; --s) {
        const int32_t* key = prefs + int64_t(s) * n;
        std::fill(bucket.begin(), bucket.end(), 0);
        for (int64_t v : order) ++bucket[key[v] + 1];
        for (int32_t b = 0; b <= p; ++b) bucket[b + 1] += bucket[b];
        for (int64_t v : order) tmp[bucket[key[v]]++] = v;
        order.swap(tmp);
    }
}

// _relocate_kernel (partition.py:203-251).
void relocate(const std::vector<int64_t>& order, int64_t n, int32_t p,
              int32_t depth, const int32_t* prefs, int32_t* labels,
              const int64_t* sizes, int64_t cap_limit) {
    const int64_t total = static_cast<int64_t>(order.size());
    auto same_tail = [&](int64_t a, int64_t b) {
        for (int32_t s = 1; s < depth; ++s)
            if (prefs[int64_t(s) * n + a] != prefs[int64_t(s) * n + b]) return false;
        return true;
    };
    int64_t i = 0;
    while (i < total) {
        const int32_t target = prefs[order[i]];
        if (target >= p) break;
        int64_t block_end = i;
        while (block_end < total && prefs[order[block_end]] == target) ++block_end;
        int64_t best_start = i, best_len = 0, run_start = i;
        for (int64_t j = i + 1; j <= block_end; ++j) {
            const bool same = j < block_end && same_tail(order[j], order[run_start]);
            if (!same) {
                const int64_t run_len = j - run_start;
                if (run_len > best_len) { best_len = run_len; best_start = run_start; }
                run_start = j;
            }
        }
        int64_t capacity = cap_limit - sizes[target];
        if (capacity < 0) capacity = 0;
        const int64_t take = best_len < capacity ? best_len : capacity;
        for (int64_t t = best_start; t < best_start + take; ++t) labels[order[t]] = target;
        i = block_end;
    }
}

}  // namespace

extern "C" int grd_sa_partition(int64_t num_vertices, const int64_t* src_ptr,
                                const int32_t* dst_idx, int32_t num_partitions,
                                const grd_partitioner_params* params, int32_t* labels,
                                double* objective_trace, int64_t* max_size_trace,
                                double* initial_objective, int32_t* iterations,
                                int32_t* converged, int32_t num_threads) {
    clear_error();
    if (num_partitions < 2) return fail(kErrArg, "num_partitions must be >= 2 here");
    if (!params || !src_ptr || !labels || !objective_trace || !max_size_trace ||
        !initial_objective || !iterations || !converged)
        return fail(kErrArg, "null argument");
    if (params->group_depth < 2 || params->max_iters < 1 || params->patience < 1)
        return fail(kErrArg, "invalid partitioner params");
    const int64_t n = num_vertices;
    const int32_t p = num_partitions;
    const int64_t m = src_ptr[n];
    const int nt = threads_or_default(num_threads);
    for (int64_t v = 0; v < n; ++v)
        if (labels[v] < 0 || labels[v] >= p) return fail(kErrArg, "initial label out of range");

    // Python float arithmetic of partition.py:272,281.
    const double denom = params->alpha_balance * static_cast<double>(n) / static_cast<double>(p);
    const int64_t cap_limit = static_cast<int64_t>(
        std::floor(params->beta * static_cast<double>(n) / static_cast<double>(p) + 1e-9));
    const int32_t depth = params->group_depth;

    std::vector<int32_t> dst_part(static_cast<size_t>(m));
    std::vector<int64_t> sizes(static_cast<size_t>(p), 0);
    std::vector<int32_t> prefs(static_cast<size_t>(depth) * n);
    auto refresh = [&]() {
        std::fill(sizes.begin(), sizes.end(), 0);
        for (int64_t v = 0; v < n; ++v) ++sizes[labels[v]];
#pragma omp parallel for num_threads(nt) schedule(static)
        for (int64_t j = 0; j < m; ++j) dst_part[j] = labels[dst_idx[j]];
    };
    auto max_size = [&]() { return *std::max_element(sizes.begin(), sizes.end()); };

    Analyzer an{n, src_ptr, p, depth, nt, {}};
    refresh();
    int64_t num_candidates = 0;
    double obj_prev = an.run(dst_part.data(), labels, sizes.data(), denom, prefs.data(),
                             &num_candidates);
    *initial_objective = obj_prev;
    int32_t n_trace = 0;
    max_size_trace[0] = max_size();
    bool conv = false;
    bool broke = false;
    int32_t iters = 0, streak = 0;
    std::vector<int64_t> order, tmp, bucket;
    for (int32_t it = 0; it < params->max_iters; ++it) {
        if (num_candidates == 0) { conv = true; broke = true; break; }
        candidate_order(n, p, depth, prefs.data(), order, tmp, bucket);
        relocate(order, n, p, depth, prefs.data(), labels, sizes.data(), cap_limit);
        ++iters;
        refresh();
        const double obj_cur = an.run(dst_part.data(), labels, sizes.data(), denom,
                                      prefs.data(), &num_candidates);
        objective_trace[n_trace++] = obj_cur;
        max_size_trace[n_trace] = max_size();
        double rel;
        if (obj_prev != 0.0) rel = (obj_cur - obj_prev) / std::fabs(obj_prev);
        else rel = obj_cur == 0.0 ? 0.0 : std::numeric_limits<double>::infinity();
        if (rel < params->epsilon) {
            ++streak;
            if (streak >= params->patience) { conv = true; broke = true; obj_prev = obj_cur; break; }
        } else {
            streak = 0;
        }
        obj_prev = obj_cur;
    }
    if (!broke) conv = num_candidates == 0;
    *iterations = iters;
    *converged = conv ? 1 : 0;
    return 0;
}

extern "C" int grd_sum_sequential(const double* x, int64_t n, double* out) {
    clear_error();
    if (!out || (n > 0 && !x)) return fail(kErrArg, "sum_sequential: null argument");
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += x[i];
    *out = acc;
    return 0;
}

// --------------------------------------------------------------------------
// Partition plan (plan.py:75-136).  The (owner, id) order of every gather
// map is the global "perm" order (targets of partition 0 ascending, then 1,
// ...), so ranks in perm order are the sort key throughout.
// --------------------------------------------------------------------------
struct grd_plan {
    int64_t V = 0, E = 0;
    int32_t P = 0;
    std::vector<int64_t> part_ptr, in_ptr, gather_ptr;
    std::vector<int32_t> perm, in_src, in_src_pos, gather_map, self_pos, in_degree;
};

extern "C" int grd_plan_create(int64_t num_vertices, const int64_t* src_ptr,
                               const int32_t* dst_idx, const int32_t* labels,
                               int32_t num_partitions, int32_t num_threads,
                               grd_plan** plan_out) {
    clear_error();
    if (!src_ptr || !labels || !plan_out) return fail(kErrArg, "null argument");
    if (num_partitions < 1) return fail(kErrArg, "num_partitions must be >= 1");
    const int64_t n = num_vertices;
    const int32_t P = num_partitions;
    const int nt = threads_or_default(num_threads);
    for (int64_t v = 0; v < n; ++v)
        if (labels[v] < 0 || labels[v] >= P)
            return fail(kErrArg, "labels out of range for num_partitions");
    std::unique_ptr<grd_plan> pl(new grd_plan);
    pl->V = n;
    pl->P = P;
    const int64_t m = src_ptr[n];
    pl->E = m;

    pl->in_degree.assign(static_cast<size_t>(n), 0);
    for (int64_t j = 0; j < m; ++j) ++pl->in_degree[dst_idx[j]];

    // perm / rank: partition blocks, ascending vertex id inside.
    pl->part_ptr.assign(static_cast<size_t>(P) + 1, 0);
    for (int64_t v = 0; v < n; ++v) ++pl->part_ptr[labels[v] + 1];
    for (int32_t q = 0; q < P; ++q) pl->part_ptr[q + 1] += pl->part_ptr[q];
    pl->perm.resize(static_cast<size_t>(n));
    std::vector<int32_t> rank(static_cast<size_t>(n));
    {
        std::vector<int64_t> cur(pl->part_ptr.begin(), pl->part_ptr.end() - 1);
        for (int64_t v = 0; v < n; ++v) {
            const int64_t r = cur[labels[v]]++;
            pl->perm[r] = static_cast<int32_t>(v);
            rank[v] = static_cast<int32_t>(r);
        }
    }
    // In-edge lists per perm row, each sorted by the source's rank: visit
    // sources in rank order and append to their destinations.
    pl->in_ptr.assign(static_cast<size_t>(n) + 1, 0);
    for (int64_t r = 0; r < n; ++r) pl->in_ptr[r + 1] = pl->in_ptr[r] + pl->in_degree[pl->perm[r]];
    pl->in_src.resize(static_cast<size_t>(m));
    pl->in_src_pos.resize(static_cast<size_t>(m));
    {
        std::vector<int64_t> cur(pl->in_ptr.begin(), pl->in_ptr.end() - 1);
        for (int64_t r = 0; r < n; ++r) {
            const int32_t u = pl->perm[r];
            for (int64_t j = src_ptr[u]; j < src_ptr[u + 1]; ++j)
                pl->in_src[cur[rank[dst_idx[j]]]++] = u;
        }
    }
    // Per partition: gather map = targets U in-sources, ordered by rank.
    std::vector<std::vector<int32_t>> gathers(static_cast<size_t>(P));
    pl->self_pos.resize(static_cast<size_t>(n));
#pragma omp parallel for num_threads(nt) schedule(dynamic, 1)
    for (int32_t q = 0; q < P; ++q) {
        const int64_t r0 = pl->part_ptr[q], r1 = pl->part_ptr[q + 1];
        const int64_t e0 = pl->in_ptr[r0], e1 = pl->in_ptr[r1];
        std::vector<int32_t> ranks;
        ranks.reserve(static_cast<size_t>((r1 - r0) + (e1 - e0)));
        for (int64_t r = r0; r < r1; ++r) ranks.push_back(static_cast<int32_t>(r));
        for (int64_t e = e0; e < e1; ++e) ranks.push_back(rank[pl->in_src[e]]);
        std::sort(ranks.begin(), ranks.end());
        ranks.erase(std::unique(ranks.begin(), ranks.end()), ranks.end());
        for (int64_t e = e0; e < e1; ++e) {
            const int32_t rk = rank[pl->in_src[e]];
            pl->in_src_pos[e] = static_cast<int32_t>(
                std::lower_bound(ranks.begin(), ranks.end(), rk) - ranks.begin());
        }
        for (int64_t r = r0; r < r1; ++r)
            pl->self_pos[r] = static_cast<int32_t>(
                std::lower_bound(ranks.begin(), ranks.end(), static_cast<int32_t>(r)) -
                ranks.begin());
        for (auto& rk : ranks) rk = pl->perm[rk];  // rank -> vertex id
        gathers[q].swap(ranks);
    }
    pl->gather_ptr.assign(static_cast<size_t>(P) + 1, 0);
    for (int32_t q = 0; q < P; ++q)
        pl->gather_ptr[q + 1] = pl->gather_ptr[q] + static_cast<int64_t>(gathers[q].size());
    pl->gather_map.resize(static_cast<size_t>(pl->gather_ptr[P]));
    for (int32_t q = 0; q < P; ++q) {
        std::copy(gathers[q].begin(), gathers[q].end(), pl->gather_map.begin() + pl->gather_ptr[q]);
        std::vector<int32_t>().swap(gathers[q]);
    }
    *plan_out = pl.release();
    return 0;
}

extern "C" int grd_plan_sizes(const grd_plan* plan, int64_t* num_edges, int64_t* gather_total) {
    clear_error();
    if (!plan || !num_edges || !gather_total) return fail(kErrArg, "null argument");
    *num_edges = plan->E;
    *gather_total = plan->gather_ptr.back();
    return 0;
}

extern "C" int grd_plan_export(const grd_plan* plan, int64_t* part_ptr, int32_t* perm,
                               int64_t* in_ptr, int32_t* in_src, int32_t* in_src_pos,
                               int64_t* gather_ptr, int32_t* gather_map,
                               int32_t* self_pos, int32_t* in_degree) {
    clear_error();
    if (!plan) return fail(kErrArg, "null plan");
    auto put = [](auto* dst, const auto& src) {
        if (dst && !src.empty()) std::memcpy(dst, src.data(), sizeof(src[0]) * src.size());
    };
    put(part_ptr, plan->part_ptr);
    put(perm, plan->perm);
    put(in_ptr, plan->in_ptr);
    put(in_src, plan->in_src);
    put(in_src_pos, plan->in_src_pos);
    put(gather_ptr, plan->gather_ptr);
    put(gather_map, plan->gather_map);
    put(self_pos, plan->self_pos);
    put(in_degree, plan->in_degree);
    return 0;
}

extern "C" void grd_plan_destroy(grd_plan* plan) { delete plan; }

// --------------------------------------------------------------------------
// Stable CSR transpose (counting sort): for every column c, the rows that
// reference it in ascending row order -- the order np.argsort(idx, "stable")
// yields, i.e. np.add.at's edge order of a partition's transposed
// aggregation (training.py:141).
// --------------------------------------------------------------------------
extern "C" int grd_csr_transpose(int64_t n_rows, const int64_t* row_ptr, const int32_t* idx, int64_t n_cols,
                                 int64_t* col_ptr, int32_t* col_rows) {
    clear_error();
    if (n_rows < 0 || n_cols < 0 || !row_ptr || !col_ptr || (row_ptr[n_rows] > 0 && (!idx || !col_rows)))
        return fail(kErrArg, "csr_transpose: bad arguments");
    const int64_t nnz = row_ptr[n_rows];
    std::vector<int64_t> fill(static_cast<size_t>(n_cols) + 1, 0);
    for (int64_t e = 0; e < nnz; ++e) {
        const int32_t c = idx[e];
        if (c < 0 || c >= n_cols) return fail(kErrArg, "csr_transpose: column %d out of range", c);
        ++fill[static_cast<size_t>(c) + 1];
    }
    for (int64_t c = 0; c < n_cols; ++c) fill[c + 1] += fill[c];
    std::copy(fill.begin(), fill.end(), col_ptr);
    for (int64_t r = 0; r < n_rows; ++r)
        for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) col_rows[fill[idx[e]]++] = static_cast<int32_t>(r);
    return 0;
}

// Row-set equality of two CSRs with the same row count: row r of A, sorted,
// equals row r of B (B's rows ascending, e.g. a grd_csr_transpose result).
// A graph whose transpose has the same rows is symmetric, so one CSR serves
// both the forward in-edge aggregation and the transposed pull.
extern "C" int grd_csr_same_rows(int64_t n_rows, const int64_t* ptr_a, const int32_t* idx_a,
                                 const int64_t* ptr_b, const int32_t* idx_b, int32_t num_threads,
                                 int32_t* equal_out) {
    clear_error();
    if (n_rows < 0 || !ptr_a || !ptr_b || !equal_out) return fail(kErrArg, "csr_same_rows: bad arguments");
    *equal_out = 0;
    if (ptr_a[n_rows] != ptr_b[n_rows]) return 0;
    for (int64_t r = 0; r <= n_rows; ++r)
        if (ptr_a[r] != ptr_b[r]) return 0;
    const int nt = threads_or_default(num_threads);
    int64_t bad = 0;
#pragma omp parallel num_threads(nt) reduction(+ : bad)
    {
        std::vector<int32_t> row;
#pragma omp for schedule(dynamic, 8192)
        for (int64_t r = 0; r < n_rows; ++r) {
            if (bad) continue;
            const int64_t b = ptr_a[r], e = ptr_a[r + 1];
            row.assign(idx_a + b, idx_a + e);
            std::sort(row.begin(), row.end());
            if (!std::equal(row.begin(), row.end(), idx_b + b)) ++bad;
        }
    }
    *equal_out = bad == 0 ? 1 : 0;
    return 0;
}

// --------------------------------------------------------------------------
// Host-tier row gather / scatter-add for the SSO path.
// --------------------------------------------------------------------------
extern "C" int grd_host_gather_rows(const float* src, int64_t ld_src, const int64_t* idx, int64_t n_rows,
                                    int32_t width, float* dst, int64_t ld_dst, int32_t num_threads) {
    clear_error();
    if (n_rows == 0) return 0;
    if (!src || !idx || !dst || width <= 0 || ld_src < width || ld_dst < width)
        return fail(kErrArg, "host_gather_rows: bad arguments");
    const int nt = threads_or_default(num_threads);
#pragma omp parallel for num_threads(nt) schedule(static, 256)
    for (int64_t i = 0; i < n_rows; ++i)
        std::memcpy(dst + i * ld_dst, src + idx[i] * ld_src, sizeof(float) * static_cast<size_t>(width));
    return 0;
}

extern "C" int grd_host_scatter_add_rows(const float* src, int64_t ld_src, const int64_t* idx, int64_t n_rows,
                                         int32_t width, float* dst, int64_t ld_dst, int32_t num_threads) {
    clear_error();
    if (n_rows == 0) return 0;
    if (!src || !idx || !dst || width <= 0 || ld_src < width || ld_dst < width)
        return fail(kErrArg, "host_scatter_add_rows: bad arguments");
    const int nt = threads_or_default(num_threads);
#pragma omp parallel for num_threads(nt) schedule(static, 256)
    for (int64_t i = 0; i < n_rows; ++i) {
        float* d = dst + idx[i] * ld_dst;
        const float* s = src + i * ld_src;
        for (int32_t j = 0; j < width; ++j) d[j] += s[j];
    }
    return 0;
}
