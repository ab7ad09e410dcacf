// ref_shim.cpp -- a C ABI over the REFERENCE's own hot-path sources, compiled
// unmodified from /root/reference/proj/src into oracle/_ref/librbe_ref.so by
// oracle/Makefile.  TEST INFRASTRUCTURE ONLY: used by tests/ to pin the C
// restatement (oracle/rbe_oracle.c) and by bench.py as the reference CPU arm /
// cpu_baseline.  This file contains no retrieval logic of its own: every result
// comes from rbe::search / rbe::local_select / rbe::global_select /
// rbe::binary_dot / rbe::make_embedding / rbe::save_index / rbe::load_index.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "rbe/bench.hpp"
#include "rbe/binary_vector.hpp"
#include "rbe/embedding.hpp"
#include "rbe/index.hpp"
#include "rbe/analysis.hpp"
#include "rbe/search.hpp"

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

// 1 = invalid_argument, 2 = out_of_range, 3 = runtime_error/other
#define REF_TRY(...)                                               \
    try {                                                          \
        __VA_ARGS__;                                                    \
        return 0;                                                  \
    } catch (const std::invalid_argument& e) { return fail(e, 1); } \
    catch (const std::out_of_range& e) { return fail(e, 2); }       \
    catch (const std::exception& e) { return fail(e, 3); }

rbe::RbeEmbedding make_query(const uint64_t* words, uint32_t qp, uint32_t dim) {
    const size_t wpp = rbe::PackedBinaryVector::words_for(dim);
    std::vector<rbe::PackedBinaryVector> planes(qp);
    for (uint32_t s = 0; s < qp; ++s) {
        planes[s].dim = dim;
        planes[s].words.assign(words + s * wpp, words + (s + 1) * wpp);
    }
    rbe::RbeEmbedding e;
    e.planes = std::move(planes);  // search never reads the query magnitude
    return e;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// --- index handle: a real rbe::KeywordIndex whose public vectors are filled
// directly (Partition fields are public, index.hpp:16-21).
void* ref_index_new(uint32_t dim, uint32_t kp, int residual_weights, uint32_t n_partitions) {
    auto* idx = new rbe::KeywordIndex();
    idx->dim = dim;
    idx->keyword_planes = kp;
    idx->residual_weights = residual_weights != 0;
    idx->partitions.resize(n_partitions);
    return idx;
}

void ref_index_free(void* h) { delete static_cast<rbe::KeywordIndex*>(h); }

// planes: [kp][count*wpp] u64, mags: f32[count], ids: u64[count]
int ref_index_set_partition(void* h, uint32_t p, uint64_t count, const uint64_t* planes,
                            const float* mags, const uint64_t* ids) {
    REF_TRY({
        auto* idx = static_cast<rbe::KeywordIndex*>(h);
        rbe::Partition& part = idx->partitions.at(p);
        const size_t wpp = idx->words_per_plane();
        part.count = count;
        part.plane_blocks.assign(idx->keyword_planes, {});
        for (uint32_t t = 0; t < idx->keyword_planes; ++t)
            part.plane_blocks[t].assign(planes + t * count * wpp, planes + (t + 1) * count * wpp);
        part.magnitudes.assign(mags, mags + count);
        part.ids.assign(ids, ids + count);
    })
}

// Build through the reference's IndexBuilder (index.cpp:36-78): embeddings
// given as [N][kp][wpp] words, ids[N]; magnitudes recomputed (embedding carries 0).
void* ref_index_build(uint32_t dim, uint32_t kp, int residual_weights, uint32_t n_partitions,
                      uint64_t n_docs, const uint64_t* words, const uint64_t* ids, int* status) {
    try {
        const size_t wpp = rbe::PackedBinaryVector::words_for(dim);
        rbe::IndexBuilder builder(n_partitions, residual_weights != 0);
        for (uint64_t i = 0; i < n_docs; ++i) {
            rbe::RbeEmbedding e;
            e.planes.resize(kp);
            for (uint32_t t = 0; t < kp; ++t) {
                e.planes[t].dim = dim;
                const uint64_t* src = words + (i * kp + t) * wpp;
                e.planes[t].words.assign(src, src + wpp);
            }
            e.magnitude = 0.0;
            builder.add(ids[i], e);
        }
        auto* idx = new rbe::KeywordIndex(builder.finish());
        *status = 0;
        return idx;
    } catch (const std::invalid_argument& e) {
        *status = fail(e, 1);
    } catch (const std::exception& e) {
        *status = fail(e, 3);
    }
    return nullptr;
}

uint64_t ref_index_count(void* h, uint32_t p) {
    return static_cast<rbe::KeywordIndex*>(h)->partitions.at(p).count;
}

int ref_index_get_partition(void* h, uint32_t p, uint64_t* planes, float* mags, uint64_t* ids) {
    REF_TRY({
        auto* idx = static_cast<rbe::KeywordIndex*>(h);
        const rbe::Partition& part = idx->partitions.at(p);
        const size_t wpp = idx->words_per_plane();
        for (uint32_t t = 0; t < idx->keyword_planes; ++t)
            std::memcpy(planes + t * part.count * wpp, part.plane_blocks[t].data(),
                        part.count * wpp * 8);
        std::memcpy(mags, part.magnitudes.data(), part.count * 4);
        std::memcpy(ids, part.ids.data(), part.count * 8);
    })
}

int ref_save_index(void* h, const char* path) {
    REF_TRY(rbe::save_index(*static_cast<rbe::KeywordIndex*>(h), path))
}

void* ref_load_index(const char* path, int* status, uint32_t* dim, uint32_t* kp, int* rw,
                     uint32_t* n_partitions) {
    try {
        auto* idx = new rbe::KeywordIndex(rbe::load_index(path));
        *dim = idx->dim;
        *kp = idx->keyword_planes;
        *rw = idx->residual_weights ? 1 : 0;
        *n_partitions = uint32_t(idx->partitions.size());
        *status = 0;
        return idx;
    } catch (const std::exception& e) {
        *status = fail(e, 3);
    }
    return nullptr;
}

// rbe::search (search.cpp:130-168) for Q queries [Q][qp][wpp].  n_threads > 1
// runs the query-parallel harness of BASELINE.md §3 mode 2 (each std::thread
// calls rbe::search on its own slice of queries; the index is shared const).
// Output per query q at [q*n, q*n + out_count[q]).
int ref_search_batch(void* h, const uint64_t* queries, uint32_t n_queries, uint32_t qp,
                     uint32_t blocks, uint32_t tpb, uint32_t ipt, uint32_t queue_length, uint64_t n,
                     double* scores, uint64_t* ids, uint32_t* parts, uint64_t* out_count,
                     uint64_t* scored, uint32_t n_threads) {
    auto* idx = static_cast<rbe::KeywordIndex*>(h);
    rbe::ScanGeometry g;
    g.blocks = blocks;
    g.threads_per_block = tpb;
    g.items_per_thread = ipt;
    g.queue_length = queue_length;
    const size_t wpp = rbe::PackedBinaryVector::words_for(idx->dim);
    std::vector<int> status(std::max<uint32_t>(n_threads, 1), 0);
    std::vector<std::string> errs(status.size());
    std::vector<uint64_t> sc(status.size(), 0);
    auto worker = [&](uint32_t w) {
        try {
            rbe::SearchStats stats;
            for (uint32_t q = w; q < n_queries; q += uint32_t(status.size())) {
                rbe::RbeEmbedding e = make_query(queries + size_t(q) * qp * wpp, qp, idx->dim);
                rbe::SelectionResult r = rbe::search(e, *idx, g, n, &stats);
                out_count[q] = r.entries.size();
                for (size_t k = 0; k < r.entries.size(); ++k) {
                    scores[q * n + k] = r.entries[k].score;
                    ids[q * n + k] = r.entries[k].id;
                    parts[q * n + k] = r.entries[k].partition;
                }
            }
            sc[w] = stats.scored;
        } catch (const std::invalid_argument& e) {
            status[w] = 1;
            errs[w] = e.what();
        } catch (const std::out_of_range& e) {
            status[w] = 2;
            errs[w] = e.what();
        } catch (const std::exception& e) {
            status[w] = 3;
            errs[w] = e.what();
        }
    };
    if (status.size() == 1) {
        worker(0);
    } else {
        std::vector<std::thread> ts;
        for (uint32_t w = 0; w < status.size(); ++w) ts.emplace_back(worker, w);
        for (auto& t : ts) t.join();
    }
    uint64_t total = 0;
    for (size_t w = 0; w < status.size(); ++w) {
        total += sc[w];
        if (status[w] != 0) {
            g_err = errs[w];
            return status[w];
        }
    }
    if (scored) *scored = total;
    return 0;
}

// rbe::local_select + rbe::global_select for one partition (search.cpp:57-128).
int ref_partition_select(void* h, const uint64_t* query, uint32_t qp, uint32_t p, uint32_t blocks,
                         uint32_t tpb, uint32_t ipt, uint32_t queue_length, uint64_t n,
                         double* scores, uint64_t* ids, uint32_t* parts, uint64_t* out_count,
                         uint64_t* n_survivors) {
    REF_TRY({
        auto* idx = static_cast<rbe::KeywordIndex*>(h);
        rbe::ScanGeometry g{blocks, tpb, ipt, queue_length};
        rbe::RbeEmbedding e = make_query(query, qp, idx->dim);
        auto lists = rbe::local_select(e, *idx, p, g);
        uint64_t ns = 0;
        for (auto& l : lists) ns += l.size();
        if (n_survivors) *n_survivors = ns;
        rbe::SelectionResult r = rbe::global_select(lists, idx->partitions.at(p), p, n);
        *out_count = r.entries.size();
        for (size_t k = 0; k < r.entries.size(); ++k) {
            scores[k] = r.entries[k].score;
            ids[k] = r.entries[k].id;
            parts[k] = r.entries[k].partition;
        }
    })
}

// rbe::local_select alone (search.cpp:57-113): the per-thread candidate lists,
// flattened to [threads][ql] (ql = the caller's stride) with counts[threads].
int ref_local_select(void* h, const uint64_t* query, uint32_t qp, uint32_t p, uint32_t blocks, uint32_t tpb,
                     uint32_t ipt, uint32_t queue_length, uint32_t ql, double* scores, uint64_t* slots,
                     uint32_t* counts, uint64_t* scored) {
    REF_TRY({
        auto* idx = static_cast<rbe::KeywordIndex*>(h);
        rbe::ScanGeometry g{blocks, tpb, ipt, queue_length};
        rbe::RbeEmbedding e = make_query(query, qp, idx->dim);
        rbe::SearchStats st;
        auto lists = rbe::local_select(e, *idx, p, g, &st);
        for (size_t t = 0; t < lists.size(); ++t) {
            if (lists[t].size() > ql) throw std::logic_error("ref_local_select: list longer than the stride");
            counts[t] = uint32_t(lists[t].size());
            for (size_t k = 0; k < lists[t].size(); ++k) {
                scores[t * ql + k] = lists[t][k].score;
                slots[t * ql + k] = lists[t][k].slot;
            }
        }
        if (scored) *scored = st.scored;
    })
}

// Leaf functions (binary_vector.hpp:33-43, embedding.cpp:7-90, search.cpp:10-26).
int ref_pack(const int* values, uint32_t n, uint64_t* words, uint32_t* dim) {
    REF_TRY({
        rbe::PackedBinaryVector v = rbe::pack(std::span<const int>(values, n));
        *dim = v.dim;
        std::memcpy(words, v.words.data(), v.words.size() * 8);
    })
}

int ref_binary_dot(const uint64_t* x, uint32_t xdim, const uint64_t* y, uint32_t ydim, int64_t* out) {
    REF_TRY({
        rbe::PackedBinaryVector a, b;
        a.dim = xdim;
        b.dim = ydim;
        a.words.assign(x, x + rbe::PackedBinaryVector::words_for(xdim));
        b.words.assign(y, y + rbe::PackedBinaryVector::words_for(ydim));
        *out = rbe::binary_dot(a, b);
    })
}

double ref_combine_plane_dots(const int64_t* dots, uint32_t qp, uint32_t kp, int rw) {
    return rbe::combine_plane_dots(dots, qp, kp, rw != 0);
}

// words: [n_planes][wpp]
int ref_make_embedding(const uint64_t* words, uint32_t n_planes, uint32_t dim, int rw, double* magnitude) {
    REF_TRY({
        const size_t wpp = rbe::PackedBinaryVector::words_for(dim);
        std::vector<rbe::PackedBinaryVector> planes(n_planes);
        for (uint32_t t = 0; t < n_planes; ++t) {
            planes[t].dim = dim;
            planes[t].words.assign(words + t * wpp, words + (t + 1) * wpp);
        }
        *magnitude = rbe::make_embedding(std::move(planes), rw != 0).magnitude;
    })
}

int ref_rbe_score(const uint64_t* qwords, uint32_t qp, const uint64_t* kwords, uint32_t kp, uint32_t dim,
                  int rw, int normalize, double* out) {
    REF_TRY({
        const size_t wpp = rbe::PackedBinaryVector::words_for(dim);
        auto mk = [&](const uint64_t* w, uint32_t np) {
            std::vector<rbe::PackedBinaryVector> planes(np);
            for (uint32_t t = 0; t < np; ++t) {
                planes[t].dim = dim;
                planes[t].words.assign(w + t * wpp, w + (t + 1) * wpp);
            }
            return rbe::make_embedding(std::move(planes), rw != 0);
        };
        rbe::SimilarityConfig cfg;
        cfg.query_planes = qp;
        cfg.keyword_planes = kp;
        cfg.residual_weights = rw != 0;
        cfg.normalize_query = normalize != 0;
        *out = rbe::rbe_score(mk(qwords, qp), mk(kwords, kp), cfg);
    })
}

int ref_thread_assignment(uint32_t blocks, uint32_t tpb, uint32_t ipt, uint32_t queue_length,
                          uint64_t count, uint32_t block, uint32_t thread, uint64_t* out,
                          uint32_t* n_out) {
    REF_TRY({
        rbe::ScanGeometry g{blocks, tpb, ipt, queue_length};
        auto v = rbe::thread_assignment(g, count, block, thread);
        *n_out = uint32_t(v.size());
        std::copy(v.begin(), v.end(), out);
    })
}

int ref_scan_benchmark(uint64_t count, uint32_t dim, uint32_t qp, uint32_t kp, uint32_t repeats,
                       uint64_t seed, double* binary_tput, double* float_tput) {
    REF_TRY({
        rbe::BenchResult r = rbe::run_scan_benchmark(count, dim, qp, kp, repeats, seed, true, true);
        *binary_tput = r.binary_throughput;
        *float_tput = r.float_throughput;
    })
}

// Appendix A selection-miss model (src/analysis.cpp:143-184): predicted recall@N of the
// length-1-queue scan of C candidates with I items per thread.
int ref_expected_recall(uint64_t C, uint64_t N, uint64_t I, double* recall, double* misses) {
    REF_TRY({
        const rbe::RecallPrediction r = rbe::expected_recall(C, N, I);
        *recall = r.expected_recall;
        *misses = r.expected_misses;
    })
}

// Monte Carlo of the same model (src/analysis.cpp:99-141): frequency of L = 0 misses.
int ref_simulate_miss_zero(uint64_t C, uint64_t N, uint64_t I, uint32_t queue_length, uint64_t trials, uint64_t seed,
                           double* p_zero) {
    REF_TRY({
        const auto f = rbe::simulate_miss(C, N, I, queue_length, trials, seed);
        auto it = f.find(0);
        *p_zero = it == f.end() ? 0.0 : it->second;
    })
}

}  // extern "C"
