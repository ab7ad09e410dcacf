// scan_tensor.h -- the TENSOR scan variant (scan_tensor.cu): int8 tensor-core
// scoring of every (query, doc) pair, a conservative per-query threshold from
// a probe pass, and exact (FP64) per-logical-thread selection of the few
// pairs that pass it.  See DESIGN.md §4.
#pragma once

#include <string>
#include <vector>

#include "../../include/rbe_cuda.h"
#include "internal.h"

namespace rbe_dev {

struct TensorScanPlan {
    uint32_t Q = 0, qp = 0;
    uint64_t n = 0;
    uint32_t probe_tiles = 0;
    uint32_t ptop = 4;                // probe values kept per (query, strip)
    uint64_t n_strips = 0;            // strips (128 or 256 logical threads of one block)
    std::vector<uint64_t> prefix;     // strips per local partition, cumulative [n_parts + 1]
    uint64_t surv_cap = 0;            // per-query survivor capacity (<= 1 per logical thread)
    bool lossless = false;            // queue_length >= items_per_thread: survivors are all docs >= theta
    size_t query_bytes = 0, probe_bytes = 0, threshold_bytes = 0, state_bytes = 0;
};

bool tensor_supported(const Shape& s, uint32_t qp, const rbe_scan_geometry& g, uint32_t Q, std::string* why);
TensorScanPlan plan_tensor_scan(const Shape& s, uint32_t qp, const rbe_scan_geometry& g, uint32_t Q,
                                const std::vector<uint64_t>& counts, uint64_t n, uint32_t probe_tiles,
                                uint64_t min_cap = 0);
// returns the number of kernels launched
uint32_t run_tensor_scan(const TensorScanPlan& plan, const ScanArgs& a, const Shape& s, const uint64_t* d_queries,
                         void* d_qtensor, void* d_probe, void* d_thresholds, void* d_state,
                         unsigned long long* d_candidates, cudaStream_t st);

}  // namespace rbe_dev
