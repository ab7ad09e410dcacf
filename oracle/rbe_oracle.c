/*
 * rbe_oracle.c -- CPU restatement of the reference's exhaustive RBE retrieval
 * hot path.  TEST INFRASTRUCTURE ONLY: this file is the checker used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.  Nothing in
 * the product package (paper_1802_06466_b200/) links, loads or calls it.
 *
 * Parity pin: tests/test_oracle.py checks every function here against
 *   (1) the SPEC.md known-answer tests (tests/golden/spec_kats.json), and
 *   (2) the reference's own sources compiled unmodified into
 *       oracle/_ref/librbe_ref.so (oracle/Makefile), on seeded inputs, and
 *   (3) golden search fixtures produced by that compiled reference
 *       (tests/golden/search_cases.json, made by tests/golden/make_golden.py).
 *
 * Every function cites the reference file:line it restates (paths relative to
 * the reference's proj/ directory).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define RBO_GAMMA 0x9e3779b97f4a7c15ull

/* splitmix64 finaliser; src/bench.cpp:15-21 (state += gamma; mix(state)).
 * Counter form: value #j of a stream seeded with `seed` is mix(seed+(j+1)*gamma). */
uint64_t rbo_splitmix64_at(uint64_t seed, uint64_t j) {
    uint64_t z = seed + (j + 1) * RBO_GAMMA;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static uint64_t pad_mask(uint32_t dim) {
    return (dim % 64 == 0) ? ~0ull : ((1ull << (dim % 64)) - 1);
}

/* Synthetic corpus: plane-major stream over the GLOBAL doc
 * index (src/bench.cpp:98-105): word w of plane t of global doc i is stream
 * value j = (t*N + i)*wpp + w; the last word of every doc plane is pad-masked
 * (src/bench.cpp:96).  Global doc i -> partition i % P, slot i / P
 * (src/index.cpp:53).  Fills one partition's plane blocks [kp][count*wpp]. */
void rbo_gen_partition_planes(uint64_t seed, uint64_t n_total, uint32_t dim, uint32_t kp,
                              uint32_t n_partitions, uint32_t partition,
                              uint64_t count, uint64_t* planes) {
    const uint64_t wpp = (dim + 63) / 64;
    const uint64_t pm = pad_mask(dim);
    for (uint32_t t = 0; t < kp; ++t) {
        uint64_t* block = planes + (uint64_t)t * count * wpp;
        for (uint64_t s = 0; s < count; ++s) {
            const uint64_t i = s * n_partitions + partition;
            for (uint64_t w = 0; w < wpp; ++w) {
                uint64_t v = rbo_splitmix64_at(seed, ((uint64_t)t * n_total + i) * wpp + w);
                if (w + 1 == wpp) v &= pm;
                block[s * wpp + w] = v;
            }
        }
    }
}

/* Same for the slots [begin, end) only (parallel callers; planes laid out for `count`). */
void rbo_gen_partition_planes_range(uint64_t seed, uint64_t n_total, uint32_t dim, uint32_t kp,
                                    uint32_t n_partitions, uint32_t partition, uint64_t count,
                                    uint64_t begin, uint64_t end, uint64_t* planes) {
    const uint64_t wpp = (dim + 63) / 64;
    const uint64_t pm = pad_mask(dim);
    for (uint32_t t = 0; t < kp; ++t) {
        uint64_t* block = planes + (uint64_t)t * count * wpp;
        for (uint64_t s = begin; s < end; ++s) {
            const uint64_t i = s * n_partitions + partition;
            for (uint64_t w = 0; w < wpp; ++w) {
                uint64_t v = rbo_splitmix64_at(seed, ((uint64_t)t * n_total + i) * wpp + w);
                if (w + 1 == wpp) v &= pm;
                block[s * wpp + w] = v;
            }
        }
    }
}

/* Query q, plane s, word w = stream value (q*qp + s)*wpp + w, pad-masked. */
void rbo_gen_queries(uint64_t seed, uint32_t n_queries, uint32_t dim, uint32_t qp, uint64_t* out) {
    const uint64_t wpp = (dim + 63) / 64;
    const uint64_t pm = pad_mask(dim);
    for (uint64_t j = 0; j < (uint64_t)n_queries * qp * wpp; ++j) {
        uint64_t v = rbo_splitmix64_at(seed, j);
        if ((j + 1) % wpp == 0) v &= pm;
        out[j] = v;
    }
}

/* binary_dot_words, include/rbe/binary_vector.hpp:33-40: dim - 2*sum popcount(x^y);
 * no pad masking (pad bits are zero by convention only). */
int64_t rbo_binary_dot_words(const uint64_t* x, const uint64_t* y, uint64_t nwords, uint32_t dim) {
    uint64_t mismatched = 0;
    for (uint64_t i = 0; i < nwords; ++i) mismatched += (uint64_t)__builtin_popcountll(x[i] ^ y[i]);
    return (int64_t)dim - 2 * (int64_t)mismatched;
}

/* combine_plane_dots, src/embedding.cpp:38-58: Horner over weight levels
 * l = s + t; returns the exact scaled integer accumulator in *acc_out and the
 * double ldexp(acc, -L) (L = qp + kp - 2), or double(sum) unweighted. */
double rbo_combine_plane_dots(const int64_t* dots, uint32_t qp, uint32_t kp, int residual_weights,
                              int64_t* acc_out) {
    if (!residual_weights) {
        int64_t sum = 0;
        for (uint32_t i = 0; i < qp * kp; ++i) sum += dots[i];
        if (acc_out) *acc_out = sum;
        return (double)sum;
    }
    const uint32_t levels = qp + kp - 2;
    int64_t acc = 0;
    for (uint32_t l = 0; l <= levels; ++l) {
        acc <<= (l > 0 ? 1 : 0);
        const uint32_t s_lo = l >= kp ? l - kp + 1 : 0;
        const uint32_t s_hi = l < qp ? l : qp - 1;
        for (uint32_t s = s_lo; s <= s_hi; ++s) acc += dots[s * kp + (l - s)];
    }
    if (acc_out) *acc_out = acc;
    return ldexp((double)acc, -(int)levels);
}

/* make_embedding magnitude, src/embedding.cpp:7-36: refined_vector in double
 * (plane t weighs 2^-t with residual weights, 1 otherwise), sum of squares in
 * dimension order, correctly rounded sqrt.  `plane_stride` is the distance in
 * u64 words between consecutive planes of this embedding. */
double rbo_magnitude(const uint64_t* planes, uint64_t plane_stride, uint32_t dim, uint32_t n_planes,
                     int residual_weights) {
    double sq = 0.0;
    for (uint32_t i = 0; i < dim; ++i) {
        double x = 0.0;
        for (uint32_t t = 0; t < n_planes; ++t) {
            const double w = residual_weights ? ldexp(1.0, -(int)t) : 1.0;
            const int bit = (int)((planes[(uint64_t)t * plane_stride + i / 64] >> (i % 64)) & 1u);
            x += bit ? w : -w;
        }
        sq += x * x;
    }
    return sqrt(sq);
}

/* Per-partition magnitudes as the index stores them: float(magnitude)
 * (src/index.cpp:58-66). */
void rbo_partition_magnitudes(const uint64_t* planes, uint64_t count, uint32_t dim, uint32_t kp,
                              int residual_weights, float* mags) {
    const uint64_t wpp = (dim + 63) / 64;
    for (uint64_t s = 0; s < count; ++s)
        mags[s] = (float)rbo_magnitude(planes + s * wpp, count * wpp, dim, kp, residual_weights);
}

/* Same for the slots [begin, end) of a partition of `count` docs (parallel callers). */
void rbo_partition_magnitudes_range(const uint64_t* planes, uint64_t count, uint64_t begin, uint64_t end,
                                    uint32_t dim, uint32_t kp, int residual_weights, float* mags) {
    const uint64_t wpp = (dim + 63) / 64;
    for (uint64_t s = begin; s < end; ++s)
        mags[s] = (float)rbo_magnitude(planes + s * wpp, count * wpp, dim, kp, residual_weights);
}

/* thread_assignment, src/search.cpp:10-26.  Returns the number of slots written. */
uint32_t rbo_thread_assignment(uint32_t blocks, uint32_t tpb, uint32_t ipt, uint64_t count,
                               uint32_t block, uint32_t thread, uint64_t* out) {
    (void)blocks;
    uint32_t n = 0;
    uint64_t z = (uint64_t)block * tpb * ipt + thread;
    for (uint32_t i = 0; i < ipt; ++i, z += tpb)
        if (z < count) out[n++] = z;
    return n;
}

typedef struct {
    double score;
    int64_t acc;
    uint64_t slot;
} rbo_cand;

typedef struct {
    double score;
    uint64_t id;
    uint32_t partition;
    int64_t acc;
} rbo_entry;

/* BoundedQueue::insert, src/search.cpp:32-48: keeps the best `cap` by
 * (score desc, slot asc); a full queue admits only a strictly greater score;
 * equal scores go after existing ones (upper_bound). */
static void queue_insert(rbo_cand* q, uint32_t* size, uint32_t cap, double score, int64_t acc,
                         uint64_t slot) {
    if (*size == cap) {
        if (score <= q[*size - 1].score) return;
        --*size;
    }
    uint32_t pos = 0;
    while (pos < *size && !(score > q[pos].score)) ++pos;
    memmove(q + pos + 1, q + pos, (size_t)(*size - pos) * sizeof(rbo_cand));
    q[pos].score = score;
    q[pos].acc = acc;
    q[pos].slot = slot;
    ++*size;
}

/* entry_less, src/search.cpp:50-53: (score desc, id asc). */
static int entry_cmp(const void* a, const void* b) {
    const rbo_entry* x = (const rbo_entry*)a;
    const rbo_entry* y = (const rbo_entry*)b;
    if (x->score != y->score) return x->score > y->score ? -1 : 1;
    return x->id < y->id ? -1 : (x->id > y->id ? 1 : 0);
}

/* local_select + global_select for one partition (src/search.cpp:57-128).
 * planes: [kp][count*wpp]; query: [qp][wpp].  Writes <= n entries sorted by
 * (score desc, id asc) to out and returns their number; *scored += count.
 * Returns -1 on the reference's invalid_argument preconditions
 * (src/search.cpp:62-71, 80-82). */
int64_t rbo_partition_select(const uint64_t* query, uint32_t qp, uint32_t dim, uint32_t kp,
                             int residual_weights, const uint64_t* planes, const float* mags,
                             const uint64_t* ids, uint64_t count, uint32_t partition,
                             uint32_t blocks, uint32_t tpb, uint32_t ipt, uint32_t queue_length,
                             uint64_t n, rbo_entry* out, uint64_t* scored) {
    if (queue_length == 0) return -1;
    if ((uint64_t)blocks * tpb * ipt < count) return -1;
    if (qp * kp > 64) return -1;
    const uint64_t wpp = (dim + 63) / 64;
    const uint64_t n_threads = (uint64_t)blocks * tpb;
    const uint32_t cap = queue_length;
    rbo_cand* qbuf = (rbo_cand*)malloc(sizeof(rbo_cand) * (size_t)cap);
    uint64_t n_surv_cap = 1024, n_surv = 0;
    rbo_entry* surv = (rbo_entry*)malloc(sizeof(rbo_entry) * n_surv_cap);
    int64_t dots[64];
    uint64_t sc = 0;
    for (uint64_t th = 0; th < n_threads; ++th) {
        const uint64_t x = th / tpb, y = th % tpb;
        uint32_t size = 0;
        uint64_t z = x * tpb * ipt + y;
        for (uint32_t i = 0; i < ipt; ++i, z += tpb) {
            if (z >= count) continue;
            for (uint32_t s = 0; s < qp; ++s)
                for (uint32_t t = 0; t < kp; ++t)
                    dots[s * kp + t] = rbo_binary_dot_words(query + (uint64_t)s * wpp,
                                                            planes + (uint64_t)t * count * wpp + z * wpp,
                                                            wpp, dim);
            int64_t acc;
            const double score = rbo_combine_plane_dots(dots, qp, kp, residual_weights, &acc) /
                                 (double)mags[z];
            queue_insert(qbuf, &size, cap, score, acc, z);
            ++sc;
        }
        for (uint32_t k = 0; k < size; ++k) {
            if (n_surv == n_surv_cap) {
                n_surv_cap *= 2;
                surv = (rbo_entry*)realloc(surv, sizeof(rbo_entry) * n_surv_cap);
            }
            surv[n_surv].score = qbuf[k].score;
            surv[n_surv].id = ids[qbuf[k].slot];
            surv[n_surv].partition = partition;
            surv[n_surv].acc = qbuf[k].acc;
            ++n_surv;
        }
    }
    qsort(surv, (size_t)n_surv, sizeof(rbo_entry), entry_cmp);
    const uint64_t m = n_surv < n ? n_surv : n;
    memcpy(out, surv, (size_t)m * sizeof(rbo_entry));
    free(surv);
    free(qbuf);
    if (scored) *scored += sc;
    return (int64_t)m;
}

/* Cross-partition merge, src/search.cpp:160-167: concatenate per-partition
 * top-n, sort by entry_less, truncate to n.  In-place over `entries`. */
uint64_t rbo_merge(rbo_entry* entries, uint64_t total, uint64_t n) {
    qsort(entries, (size_t)total, sizeof(rbo_entry), entry_cmp);
    return total < n ? total : n;
}

/* search, src/search.cpp:130-168, for a partitioned index given as arrays of
 * per-partition pointers.  out must hold P*n entries (scratch); returns the
 * number of merged entries (<= n) at the front of out, or -1 on error. */
int64_t rbo_search(const uint64_t* query, uint32_t qp, uint32_t dim, uint32_t kp, int residual_weights,
                   uint32_t n_partitions, const uint64_t* const* planes, const float* const* mags,
                   const uint64_t* const* ids, const uint64_t* counts, uint32_t blocks, uint32_t tpb,
                   uint32_t ipt, uint32_t queue_length, uint64_t n, rbo_entry* out,
                   uint64_t* scored) {
    uint64_t total_keywords = 0;
    for (uint32_t p = 0; p < n_partitions; ++p) total_keywords += counts[p];
    if (n_partitions == 0 || total_keywords == 0) return -1;
    uint64_t total = 0;
    for (uint32_t p = 0; p < n_partitions; ++p) {
        const int64_t m = rbo_partition_select(query, qp, dim, kp, residual_weights, planes[p], mags[p],
                                               ids[p], counts[p], p, blocks, tpb, ipt, queue_length,
                                               n, out + total, scored);
        if (m < 0) return -1;
        total += (uint64_t)m;
    }
    return (int64_t)rbo_merge(out, total, n);
}
