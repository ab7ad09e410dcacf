// rbe/search.hpp -- exhaustive top-N retrieval (drop-in for the reference's
// include/rbe/search.hpp:12-70).  rbe::search runs on B200s through the C ABI
// of include/rbe_cuda.h; there is no CPU scan.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "rbe/index.hpp"

struct rbe_cuda_index;

namespace rbe {

/// Algorithm-1 geometry: thread y of block x scans z = x*T_b*I + y + i*T_b.
struct ScanGeometry {
    uint32_t blocks = 1;
    uint32_t threads_per_block = 256;
    uint32_t items_per_thread = 256;
    uint32_t queue_length = 1;

    uint64_t capacity() const { return uint64_t(blocks) * threads_per_block * items_per_thread; }
};

std::vector<uint64_t> thread_assignment(const ScanGeometry& geometry, uint64_t partition_count, uint32_t block,
                                        uint32_t thread);

struct Candidate {
    double score = 0.0;
    uint64_t slot = 0;
};

// Layout-identical to the reference's SelectionEntry (search.hpp:34-38).  The exact
// integer accumulator behind a score (score = ldexp(acc, -L) / magnitude) is returned
// separately (DeviceIndex::search_words' `accs`).
struct SelectionEntry {
    double score = 0.0;
    uint64_t id = 0;
    uint32_t partition = 0;
};

struct SelectionResult {
    std::vector<SelectionEntry> entries;
};

struct SearchStats {
    uint64_t scored = 0;          // similarity evaluations (== Q * keywords)
    uint32_t variant = 0;         // RBE_VARIANT_* of the last batch
    uint64_t candidates = 0;      // TENSOR: pairs past the threshold filter
    uint64_t survivors = 0;       // per-logical-thread survivors selected from
    double device_ms = 0.0;       // device time of the last batch
};

enum class ScanVariant : uint32_t { Auto = 0, Exact = 1, Tensor = 2 };

/// Ingest statistics of DeviceIndex::from_rbei.
struct LoadStats {
    uint64_t file_bytes = 0;  // partition bytes read from the file
    double seconds = 0.0;     // wall time (all devices)
};

/// The HBM-resident index: partition p lives on devices[p % devices.size()].
class DeviceIndex {
public:
    DeviceIndex(const KeywordIndex& index, std::vector<int> devices = {0});
    /// Synthetic corpus generated on the device(s); only the
    /// partitions whose p % world == rank are materialised (multi-process use).
    static DeviceIndex synthetic(uint32_t dim, uint32_t keyword_planes, bool residual_weights, uint64_t n_docs,
                                 uint32_t partitions, uint64_t seed, std::vector<int> devices = {0},
                                 uint32_t rank = 0, uint32_t world = 1);
    /// RBEI v1 file straight into HBM: the reference's load_index
    /// (src/index.cpp:170-208) plus the upload in one streamed pass -- pread by host
    /// threads into page-locked staging, copy, re-pack on the device.  Partition p goes to
    /// devices[p % devices.size()]; the devices are loaded concurrently.  Same errors as
    /// load_index (std::runtime_error); magnitudes must be finite and > 0.
    static DeviceIndex from_rbei(const std::string& path, std::vector<int> devices = {0}, uint32_t io_threads = 0,
                                 LoadStats* stats = nullptr);
    /// RBEE bulk embeddings built into an index on the device(s): the
    /// reference's `rbe build` loop (EmbeddingReader + IndexBuilder, src/embedding_io.cpp:48-95,
    /// src/index.cpp:36-78) with the records streamed to HBM, scattered round-robin into the
    /// partitions and their magnitudes recomputed on the device where not > 0.  Partition p on
    /// devices[p % devices.size()]; same errors as the reference.
    static DeviceIndex build_rbee(const std::string& path, uint32_t partitions, std::vector<int> devices = {0},
                                  uint32_t io_threads = 0, LoadStats* stats = nullptr);
    /// Write the index as an RBEI v1 file (byte-identical to save_index of the same
    /// KeywordIndex), one partition at a time from the device.
    void save_index(const std::string& path) const;
    ~DeviceIndex();
    DeviceIndex(DeviceIndex&&) noexcept;
    DeviceIndex& operator=(DeviceIndex&&) noexcept;

    uint32_t dim() const { return dim_; }
    uint32_t keyword_planes() const { return kp_; }
    bool residual_weights() const { return rw_; }
    uint32_t partition_count() const { return partitions_; }
    uint64_t total_keywords() const { return total_; }
    uint64_t max_partition_count() const { return max_count_; }
    uint64_t device_bytes() const;
    uint64_t scan_bytes() const;  // algorithmic bytes one batch reads
    const std::vector<int>& devices() const { return devices_; }
    /// Copy local partition back in the reference layout (tests).
    Partition download_partition(uint32_t partition) const;

    /// Raw batched call: queries [Q][qp][wpp] words -> per-query results; `accs` (optional)
    /// receives each entry's exact integer accumulator, parallel to the entries.
    std::vector<SelectionResult> search_words(std::span<const uint64_t> query_words, uint32_t n_queries,
                                              uint32_t query_planes, const ScanGeometry& geometry, uint64_t n,
                                              SearchStats* stats = nullptr, ScanVariant variant = ScanVariant::Auto,
                                              uint32_t probe_tiles = 0,
                                              std::vector<std::vector<int64_t>>* accs = nullptr) const;
    /// Same, writing into caller-owned [Q][n] arrays (counts[Q] valid entries per query);
    /// stats may be null (then the batch runs with a single host synchronisation).
    void search_words_into(std::span<const uint64_t> query_words, uint32_t n_queries, uint32_t query_planes,
                           const ScanGeometry& geometry, uint64_t n, double* scores, uint64_t* ids,
                           uint32_t* partitions, int64_t* accs, uint64_t* counts, SearchStats* stats = nullptr,
                           ScanVariant variant = ScanVariant::Auto, uint32_t probe_tiles = 0) const;
    rbe_cuda_index* handle(size_t i) const { return handles_.at(i).get(); }
    size_t handle_count() const { return handles_.size(); }
    /// (handle index, local slot) of a resident global partition; throws out_of_range otherwise.
    std::pair<size_t, uint32_t> locate(uint32_t partition) const;
    uint64_t partition_size(uint32_t partition) const;

private:
    DeviceIndex() = default;
    struct Deleter {
        void operator()(rbe_cuda_index* p) const;
    };
    std::vector<std::unique_ptr<rbe_cuda_index, Deleter>> handles_;
    std::vector<int> devices_;
    uint32_t dim_ = 0, kp_ = 1, partitions_ = 0;
    bool rw_ = true;
    uint64_t total_ = 0, max_count_ = 0;
    // global partition -> (handle, local slot) or handle -1 when not resident
    std::vector<int> part_handle_;
    std::vector<uint32_t> part_local_;
    std::vector<uint64_t> part_count_;
};

/// local_select (reference search.hpp:53-57) on the device: the per-logical-thread
/// candidate lists of one partition, indexed by block * threads_per_block + thread, each
/// ordered by (score desc, slot asc).  The KeywordIndex overload uploads that partition
/// for the call.
std::vector<std::vector<Candidate>> local_select(const RbeEmbedding& query, const DeviceIndex& index,
                                                 uint32_t partition, const ScanGeometry& geometry,
                                                 SearchStats* stats = nullptr);
std::vector<std::vector<Candidate>> local_select(const RbeEmbedding& query, const KeywordIndex& index,
                                                 uint32_t partition, const ScanGeometry& geometry,
                                                 SearchStats* stats = nullptr);

/// global_select (reference search.hpp:61-63): the best n of one partition's surviving
/// candidates under (score desc, id asc), selected on the device.
SelectionResult global_select(const std::vector<std::vector<Candidate>>& per_thread, const Partition& partition,
                              uint32_t partition_ordinal, uint64_t n);

/// rbe::search on the device store.
SelectionResult search(const RbeEmbedding& query, const DeviceIndex& index, const ScanGeometry& geometry, uint64_t n,
                       SearchStats* stats = nullptr);
/// Drop-in signature: uploads `index` to device 0 for the call (build a
/// DeviceIndex once to amortise the upload).
SelectionResult search(const RbeEmbedding& query, const KeywordIndex& index, const ScanGeometry& geometry, uint64_t n,
                       SearchStats* stats = nullptr);
/// One pass over the store for a whole batch of queries.
std::vector<SelectionResult> search_batch(std::span<const RbeEmbedding> queries, const DeviceIndex& index,
                                          const ScanGeometry& geometry, uint64_t n, SearchStats* stats = nullptr);

}  // namespace rbe
