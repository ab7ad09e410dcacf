// capi.cu -- implementation of include/rbe_cuda.h: the device index (HBM
// store) and the batched search orchestration (query upload, scan kernel,
// device selection, result download).  No CPU fallback: every compute entry
// point fails with RBE_CUDA_ERUNTIME when CUDA is unusable.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rbe_cuda.h"
#include "internal.h"
#include "scan_tensor.h"

using namespace rbe_dev;

namespace {

thread_local std::string g_last_error;

struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct OutOfRange : std::out_of_range {
    using std::out_of_range::out_of_range;
};

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return RBE_CUDA_OK;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return RBE_CUDA_EINVAL;
    } catch (const std::out_of_range& e) {
        g_last_error = e.what();
        return RBE_CUDA_ERANGE;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return RBE_CUDA_ERUNTIME;
    } catch (...) {
        g_last_error = "unknown error";
        return RBE_CUDA_ERUNTIME;
    }
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(size_t b) {
        if (b <= bytes) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        if (b == 0) return;
        RBE_CK(cudaMalloc(&p, b));
        bytes = b;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

uint64_t round_up(uint64_t x, uint64_t m) { return (x + m - 1) / m * m; }

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        RBE_CK(cudaGetDevice(&prev));
        if (prev != dev) RBE_CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

struct rbe_cuda_index {
    int device = 0;
    Shape shape;
    PlanePerm perm{};
    struct Local {
        uint32_t ordinal;
        uint64_t count, count_pad;
        uint32_t* planes;
        float* mags;
        uint64_t* ids;
    };
    std::vector<Local> parts;
    void* store = nullptr;
    size_t store_bytes = 0;
    PartDesc* d_parts = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[4] = {};
    std::mutex mu;
    // per-batch scratch, grown on demand
    DevBuf queries, qperm, qtensor, surv, surv_count, counters, queue_scratch, sel_scratch, out, probe, thresholds, soa;
    bool mag_range_ok = false;   // cached magnitude range (tensor threshold bins)
    float mag_lo = 0.0f, mag_hi = 0.0f;
    Result* host_out = nullptr;  // pinned staging for the D2H of results
    size_t host_out_cap = 0;
    void ensure_host_out(size_t n) {
        if (n <= host_out_cap) return;
        if (host_out) cudaFreeHost(host_out);
        host_out = nullptr;
        host_out_cap = 0;
        RBE_CK(cudaMallocHost(&host_out, n * sizeof(Result)));
        host_out_cap = n;
    }

    ~rbe_cuda_index() {
        cudaSetDevice(device);
        for (DevBuf* b : {&queries, &qperm, &qtensor, &surv, &surv_count, &counters, &queue_scratch, &sel_scratch, &out,
                          &probe, &thresholds, &soa})
            b->release();
        if (d_parts) cudaFree(d_parts);
        if (store) cudaFree(store);
        if (host_out) cudaFreeHost(host_out);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace {

// true if p points into page-locked host memory (cudaMallocHost / cudaHostRegister)
bool pinned_host(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

void check_device_usable(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw CudaError(std::string("no usable CUDA device (") + cudaGetErrorString(e) +
                        "); the RBE search path has no CPU fallback");
    if (device < 0 || device >= n) throw InvalidArgument("rbe_cuda: device ordinal out of range");
    cudaDeviceProp prop;
    RBE_CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        throw CudaError("rbe_cuda: kernels are compiled for sm_100a (B200); device " + std::to_string(device) +
                        " is sm_" + std::to_string(prop.major) + std::to_string(prop.minor));
}

// Reference-order argument checks of search / local_select (search.cpp:62-71, 80-82, 133-135).
void validate_search(const rbe_cuda_index* ix, uint32_t qp, const rbe_scan_geometry* g) {
    uint64_t total = 0;
    for (auto& p : ix->parts) total += p.count;
    if (ix->parts.empty() || total == 0) throw InvalidArgument("search: empty index");
    if (qp == 0) throw InvalidArgument("local_select: query dimension mismatch");
    if (g->queue_length == 0) throw InvalidArgument("local_select: queue_length must be positive");
    const uint64_t capacity = uint64_t(g->blocks) * g->threads_per_block * g->items_per_thread;
    for (auto& p : ix->parts)
        if (capacity < p.count) throw InvalidArgument("local_select: geometry does not cover partition");
    if (uint64_t(qp) * ix->shape.kp > 64) throw InvalidArgument("local_select: too many planes");
}

struct BatchResult {
    rbe_search_stats stats{};
};

// Runs one batch with queries already on the device (ix->queries) and leaves
// rbe_result[Q][n] in ix->out.  Returns stats.
// sync = false (tensor variant only): the whole batch is enqueued on `st` with no host
// synchronisation (no stats; the consistency flag is checked by the next synchronous call).
void run_batch(rbe_cuda_index* ix, cudaStream_t st, uint32_t Q, uint32_t qp, const rbe_scan_geometry* g, uint64_t n,
               const rbe_search_options* opt, rbe_search_stats* st_out, bool sync = true) {
    const Shape& s = ix->shape;
    ScanArgs a;
    a.parts = ix->d_parts;
    a.n_parts = uint32_t(ix->parts.size());
    a.blocks = g->blocks;
    a.tpb = g->threads_per_block;
    a.ipt = g->items_per_thread;
    a.ql = g->queue_length;
    a.Q = Q;
    a.qp = qp;

    uint32_t variant = opt ? opt->variant : RBE_VARIANT_AUTO;
    const uint32_t probe_tiles = opt && opt->probe_tiles ? opt->probe_tiles : 0;
    std::string why;
    const bool tensor_ok = tensor_supported(s, qp, *g, Q, &why);
    if (variant == RBE_VARIANT_TENSOR && !tensor_ok)
        throw InvalidArgument("search: tensor variant unsupported for this shape: " + why);
    if (variant == RBE_VARIANT_AUTO) variant = tensor_ok ? RBE_VARIANT_TENSOR : RBE_VARIANT_EXACT;
    if (variant != RBE_VARIANT_TENSOR) sync = true;  // the exact kernel may need its overflow retry

    rbe_search_stats stats{};
    stats.variant = variant;
    ix->counters.ensure(64);
    unsigned long long* d_scored = ix->counters.as<unsigned long long>();
    unsigned int* d_overflow = reinterpret_cast<unsigned int*>(d_scored + 2);
    unsigned int* d_error = d_overflow + 1;
    unsigned long long* d_cands = d_scored + 4;
    a.scored = d_scored;
    a.overflow = d_overflow;
    a.error = d_error;
    if (variant == RBE_VARIANT_TENSOR && !ix->mag_range_ok) {
        // one-time (per index contents) magnitude range for the threshold bins
        uint32_t* d_rng = reinterpret_cast<uint32_t*>(d_scored + 6);
        const uint32_t init[2] = {0xffffffffu, 0u};
        RBE_CK(cudaMemcpyAsync(d_rng, init, 8, cudaMemcpyHostToDevice, st));
        for (auto& p : ix->parts) launch_mag_range(p.mags, p.count, d_rng, st);
        uint32_t rng[2];
        RBE_CK(cudaMemcpyAsync(rng, d_rng, 8, cudaMemcpyDeviceToHost, st));
        RBE_CK(cudaStreamSynchronize(st));
        std::memcpy(&ix->mag_lo, &rng[0], 4);
        std::memcpy(&ix->mag_hi, &rng[1], 4);
        ix->mag_range_ok = true;
    }
    a.mag_lo = ix->mag_lo;
    a.mag_hi = ix->mag_hi;

    RBE_CK(cudaEventRecord(ix->ev[0], st));
    for (int attempt = 0; attempt < 2; ++attempt) {
        RBE_CK(cudaMemsetAsync(ix->counters.p, 0, 64, st));
        ix->surv_count.ensure(sizeof(unsigned long long) * Q);
        RBE_CK(cudaMemsetAsync(ix->surv_count.p, 0, sizeof(unsigned long long) * Q, st));
        a.surv_count = ix->surv_count.as<unsigned long long>();
        if (variant == RBE_VARIANT_EXACT) {
            const uint64_t ql_eff = std::min<uint64_t>(a.ql, a.ipt);
            const uint64_t threads = uint64_t(a.blocks) * a.tpb;
            uint64_t cap = 0;
            for (auto& p : ix->parts) cap += std::min<uint64_t>(p.count, threads * ql_eff);
            a.surv_cap = std::max<uint64_t>(cap, 1);
            ix->surv.ensure(sizeof(Result) * a.surv_cap * Q);
            a.surv = ix->surv.as<Result>();
            ix->qperm.ensure(sizeof(uint32_t) * size_t(Q) * s.kp * qp * s.w32);
            launch_prepare_queries_exact(ix->queries.as<uint64_t>(), ix->qperm.as<uint32_t>(), Q, qp, s, ix->perm, st);
            const size_t qs = exact_queue_scratch_bytes(a);
            ix->queue_scratch.ensure(qs);
            RBE_CK(cudaEventRecord(ix->ev[1], st));
            launch_scan_exact(a, s, ix->qperm.as<uint32_t>(), qs ? ix->queue_scratch.p : nullptr, st);
            RBE_CK(cudaEventRecord(ix->ev[2], st));
            stats.launches += 2;
        } else {
            std::vector<uint64_t> counts;
            for (auto& p : ix->parts) counts.push_back(p.count);
            TensorScanPlan plan = plan_tensor_scan(s, qp, *g, Q, counts, n, probe_tiles);
            a.surv_cap = plan.surv_cap;
            ix->surv.ensure(sizeof(Result) * a.surv_cap * Q);
            a.surv = ix->surv.as<Result>();
            ix->qtensor.ensure(plan.query_bytes);
            ix->probe.ensure(plan.probe_bytes);
            ix->thresholds.ensure(plan.threshold_bytes);
            ix->queue_scratch.ensure(plan.state_bytes);
            RBE_CK(cudaEventRecord(ix->ev[1], st));
            stats.launches += run_tensor_scan(plan, a, s, ix->queries.as<uint64_t>(), ix->qtensor.p, ix->probe.p,
                                              ix->thresholds.p, ix->queue_scratch.p, d_cands, st);
            RBE_CK(cudaEventRecord(ix->ev[2], st));
        }
        if (!sync) break;  // the tensor kernel never sets the overflow flag
        unsigned int flags[2] = {0, 0};
        RBE_CK(cudaMemcpyAsync(flags, d_overflow, sizeof(flags), cudaMemcpyDeviceToHost, st));
        RBE_CK(cudaStreamSynchronize(st));
        if (flags[1]) throw std::logic_error("tensor scan: accumulator recovery failed (internal error)");
        const unsigned int overflow = flags[0];
        if (!overflow) break;
        if (variant == RBE_VARIANT_EXACT) throw std::logic_error("exact scan overflowed its survivor list");
        // candidate/survivor buffer overflow in the tensor kernel: redo exactly.
        variant = RBE_VARIANT_EXACT;
        stats.variant = variant;
        stats.fallback = 1;
    }
    const size_t ss = select_scratch_bytes(Q, a.surv_cap, n);
    ix->sel_scratch.ensure(ss);
    ix->out.ensure(sizeof(Result) * size_t(Q) * n);
    launch_select_topn(a.surv, a.surv_count, a.surv_cap, Q, n, ix->out.as<Result>(), ix->sel_scratch.p, ss, st);
    stats.launches += 1;
    RBE_CK(cudaEventRecord(ix->ev[3], st));
    if (!sync) {
        if (st_out) *st_out = stats;
        return;
    }
    unsigned long long host_counters[8];
    RBE_CK(cudaMemcpyAsync(host_counters, ix->counters.p, 64, cudaMemcpyDeviceToHost, st));
    std::vector<unsigned long long> sc(Q);
    RBE_CK(cudaMemcpyAsync(sc.data(), ix->surv_count.p, sizeof(unsigned long long) * Q, cudaMemcpyDeviceToHost, st));
    RBE_CK(cudaStreamSynchronize(st));
    stats.scored = host_counters[0];
    stats.candidates = host_counters[4];
    for (auto c : sc) stats.survivors += std::min<uint64_t>(c, a.surv_cap);
    float ms = 0;
    RBE_CK(cudaEventElapsedTime(&ms, ix->ev[1], ix->ev[2]));
    stats.scan_ms = ms;
    RBE_CK(cudaEventElapsedTime(&ms, ix->ev[0], ix->ev[3]));
    stats.total_ms = ms;
    if (st_out) *st_out = stats;
}

__global__ void gather_lists_kernel(const Result* in, uint32_t n_lists, uint32_t Q, uint64_t n, Result* out,
                                    unsigned long long* counts) {
    const uint64_t total = uint64_t(n_lists) * Q * n;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total; e += uint64_t(gridDim.x) * blockDim.x) {
        const Result r = in[e];
        if (!r.valid) continue;
        const uint32_t q = uint32_t((e / n) % Q);
        const unsigned long long pos = atomicAdd(counts + q, 1ull);
        out[uint64_t(q) * n_lists * n + pos] = r;
    }
}

}  // namespace

extern "C" {

const char* rbe_cuda_last_error(void) { return g_last_error.c_str(); }

const char* rbe_cuda_version(void) { return "rbe_cuda 0.1 sm_100a"; }

int rbe_cuda_index_create(const rbe_index_shape* shape, uint32_t n_partitions, const uint32_t* ordinals,
                          const uint64_t* counts, int device, rbe_cuda_index** out) {
    return guarded([&] {
        if (!shape || !out || (n_partitions && (!ordinals || !counts))) throw InvalidArgument("rbe_cuda_index_create: null argument");
        if (shape->dim == 0) throw InvalidArgument("rbe_cuda_index_create: dim must be positive");
        if (shape->keyword_planes == 0 || shape->keyword_planes > uint32_t(kMaxPlanes))
            throw InvalidArgument("rbe_cuda_index_create: keyword_planes must be in [1, 64]");
        check_device_usable(device);
        DeviceGuard dg(device);
        auto ix = std::make_unique<rbe_cuda_index>();
        ix->device = device;
        ix->shape.dim = shape->dim;
        ix->shape.kp = shape->keyword_planes;
        ix->shape.rw = shape->residual_weights ? 1 : 0;
        ix->shape.wpp = (shape->dim + 63) / 64;
        ix->shape.w32 = 2 * ix->shape.wpp;
        ix->perm = derive_plane_permutation(ix->shape.kp, ix->shape.rw != 0);
        // layout: per partition planes [kp][count_pad][w32] u32 | mags [count_pad] f32 | ids [count] u64
        size_t off = 0;
        std::vector<size_t> offs;
        for (uint32_t i = 0; i < n_partitions; ++i) {
            const uint64_t cp = round_up(counts[i], 512) + 512;
            offs.push_back(off);
            off += round_up(size_t(ix->shape.kp) * cp * ix->shape.w32 * 4, 256);
            off += round_up(cp * 4, 256);
            off += round_up(std::max<uint64_t>(counts[i], 1) * 8, 256);
        }
        ix->store_bytes = off;
        if (off) RBE_CK(cudaMalloc(&ix->store, off));
        std::vector<PartDesc> descs;
        RBE_CK(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
        for (auto& e : ix->ev) RBE_CK(cudaEventCreate(&e));
        for (uint32_t i = 0; i < n_partitions; ++i) {
            rbe_cuda_index::Local L;
            L.ordinal = ordinals[i];
            L.count = counts[i];
            L.count_pad = round_up(counts[i], 512) + 512;
            char* base = static_cast<char*>(ix->store) + offs[i];
            L.planes = reinterpret_cast<uint32_t*>(base);
            base += round_up(size_t(ix->shape.kp) * L.count_pad * ix->shape.w32 * 4, 256);
            L.mags = reinterpret_cast<float*>(base);
            base += round_up(L.count_pad * 4, 256);
            L.ids = reinterpret_cast<uint64_t*>(base);
            RBE_CK(cudaMemsetAsync(L.planes, 0, size_t(ix->shape.kp) * L.count_pad * ix->shape.w32 * 4, ix->stream));
            launch_fill_f32(L.mags, L.count_pad, 1.0f, ix->stream);
            ix->parts.push_back(L);
            PartDesc d{L.planes, L.mags, L.ids, L.count, L.count_pad, L.ordinal, 0};
            descs.push_back(d);
        }
        if (!descs.empty()) {
            RBE_CK(cudaMalloc(&ix->d_parts, sizeof(PartDesc) * descs.size()));
            RBE_CK(cudaMemcpyAsync(ix->d_parts, descs.data(), sizeof(PartDesc) * descs.size(), cudaMemcpyHostToDevice,
                                   ix->stream));
        }
        RBE_CK(cudaStreamSynchronize(ix->stream));
        *out = ix.release();
    });
}

int rbe_cuda_index_upload_partition(rbe_cuda_index* ix, uint32_t i, const uint64_t* planes, const float* mags,
                                    const uint64_t* ids) {
    return guarded([&] {
        if (!ix) throw InvalidArgument("rbe_cuda_index_upload_partition: null index");
        std::lock_guard<std::mutex> lk(ix->mu);
        if (i >= ix->parts.size()) throw OutOfRange("rbe_cuda_index_upload_partition: partition out of range");
        DeviceGuard dg(ix->device);
        auto& L = ix->parts[i];
        if (L.count == 0) return;
        if (!planes || !mags || !ids) throw InvalidArgument("rbe_cuda_index_upload_partition: null buffer");
        const Shape& s = ix->shape;
        const size_t nat_bytes = size_t(s.kp) * L.count * s.wpp * 8;
        DevBuf tmp;
        tmp.ensure(nat_bytes + 64);
        RBE_CK(cudaMemcpyAsync(tmp.p, planes, nat_bytes, cudaMemcpyHostToDevice, ix->stream));
        launch_repack_planes(tmp.as<uint64_t>(), L.planes, L.count, L.count_pad, s, ix->perm, ix->stream);
        ix->mag_range_ok = false;
        RBE_CK(cudaMemcpyAsync(L.mags, mags, L.count * 4, cudaMemcpyHostToDevice, ix->stream));
        RBE_CK(cudaMemcpyAsync(L.ids, ids, L.count * 8, cudaMemcpyHostToDevice, ix->stream));
        ix->counters.ensure(64);
        RBE_CK(cudaMemsetAsync(ix->counters.p, 0, 4, ix->stream));
        launch_validate_mags(L.mags, L.count, ix->counters.as<uint32_t>(), ix->stream);
        uint32_t bad = 0;
        RBE_CK(cudaMemcpyAsync(&bad, ix->counters.p, 4, cudaMemcpyDeviceToHost, ix->stream));
        RBE_CK(cudaStreamSynchronize(ix->stream));
        tmp.release();
        if (bad) throw InvalidArgument("rbe_cuda_index_upload_partition: keyword magnitudes must be finite and > 0");
    });
}

int rbe_cuda_index_fill_synthetic(rbe_cuda_index* ix, uint64_t seed, uint64_t n_total, uint32_t n_parts_total) {
    return guarded([&] {
        if (!ix) throw InvalidArgument("rbe_cuda_index_fill_synthetic: null index");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        if (n_parts_total == 0) throw InvalidArgument("rbe_cuda_index_fill_synthetic: need at least one partition");
        ix->mag_range_ok = false;
        for (auto& L : ix->parts) {
            if (L.ordinal >= n_parts_total) throw InvalidArgument("rbe_cuda_index_fill_synthetic: ordinal >= partitions");
            const uint64_t expect = L.ordinal < n_total ? (n_total - L.ordinal + n_parts_total - 1) / n_parts_total : 0;
            if (expect != L.count)
                throw InvalidArgument("rbe_cuda_index_fill_synthetic: partition count does not match round-robin split");
            launch_fill_synthetic(L.planes, L.mags, L.ids, L.count, L.count_pad, L.ordinal, n_parts_total, n_total, seed,
                                  ix->shape, ix->perm, ix->stream);
        }
        RBE_CK(cudaStreamSynchronize(ix->stream));
    });
}

int rbe_cuda_index_download_partition(const rbe_cuda_index* cix, uint32_t i, uint64_t* planes, float* mags,
                                      uint64_t* ids) {
    return guarded([&] {
        rbe_cuda_index* ix = const_cast<rbe_cuda_index*>(cix);
        if (!ix) throw InvalidArgument("rbe_cuda_index_download_partition: null index");
        std::lock_guard<std::mutex> lk(ix->mu);
        if (i >= ix->parts.size()) throw OutOfRange("rbe_cuda_index_download_partition: partition out of range");
        DeviceGuard dg(ix->device);
        auto& L = ix->parts[i];
        if (L.count == 0) return;
        const Shape& s = ix->shape;
        const size_t nat_bytes = size_t(s.kp) * L.count * s.wpp * 8;
        DevBuf tmp;
        tmp.ensure(nat_bytes);
        launch_unpack_planes(L.planes, tmp.as<uint64_t>(), L.count, L.count_pad, s, ix->perm, ix->stream);
        if (planes) RBE_CK(cudaMemcpyAsync(planes, tmp.p, nat_bytes, cudaMemcpyDeviceToHost, ix->stream));
        if (mags) RBE_CK(cudaMemcpyAsync(mags, L.mags, L.count * 4, cudaMemcpyDeviceToHost, ix->stream));
        if (ids) RBE_CK(cudaMemcpyAsync(ids, L.ids, L.count * 8, cudaMemcpyDeviceToHost, ix->stream));
        RBE_CK(cudaStreamSynchronize(ix->stream));
    });
}

int rbe_cuda_index_destroy(rbe_cuda_index* ix) {
    return guarded([&] { delete ix; });
}

int rbe_cuda_index_bytes(const rbe_cuda_index* ix, uint64_t* device_bytes, uint64_t* scan_bytes) {
    return guarded([&] {
        if (!ix) throw InvalidArgument("rbe_cuda_index_bytes: null index");
        uint64_t docs = 0;
        for (auto& L : ix->parts) docs += L.count;
        if (device_bytes) *device_bytes = ix->store_bytes;
        if (scan_bytes) *scan_bytes = docs * (uint64_t(ix->shape.kp) * ix->shape.wpp * 8 + 4);
    });
}

int rbe_cuda_search_device(rbe_cuda_index* ix, const uint64_t* d_query_words, uint32_t n_queries, uint32_t query_planes,
                           const rbe_scan_geometry* geometry, uint64_t n, const rbe_search_options* options,
                           rbe_result* d_out, void* stream, rbe_search_stats* stats) {
    return guarded([&] {
        if (!ix || !geometry) throw InvalidArgument("rbe_cuda_search_device: null argument");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        validate_search(ix, query_planes, geometry);
        if (n_queries == 0 || n == 0) return;
        if (!d_query_words || !d_out) throw InvalidArgument("rbe_cuda_search_device: null buffer");
        // all work is issued on the caller's stream when given (so its events
        // bracket exactly this batch), else on the index's own stream
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ix->stream;
        const size_t qbytes = size_t(n_queries) * query_planes * ix->shape.wpp * 8;
        ix->queries.ensure(qbytes);
        RBE_CK(cudaMemcpyAsync(ix->queries.p, d_query_words, qbytes, cudaMemcpyDeviceToDevice, st));
        run_batch(ix, st, n_queries, query_planes, geometry, n, options, stats, stats != nullptr);
        RBE_CK(cudaMemcpyAsync(d_out, ix->out.p, sizeof(Result) * n_queries * n, cudaMemcpyDeviceToDevice, st));
        if (stats) RBE_CK(cudaStreamSynchronize(st));
    });
}

int rbe_cuda_search(rbe_cuda_index* ix, const uint64_t* query_words, uint32_t n_queries, uint32_t query_planes,
                    const rbe_scan_geometry* geometry, uint64_t n, const rbe_search_options* options, double* scores,
                    uint64_t* ids, uint32_t* partitions, int64_t* accs, uint64_t* counts, rbe_search_stats* stats) {
    return guarded([&] {
        if (!ix || !geometry) throw InvalidArgument("rbe_cuda_search: null argument");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        validate_search(ix, query_planes, geometry);
        if (n_queries == 0) return;
        if (n == 0) {
            if (counts) std::fill(counts, counts + n_queries, 0);
            if (stats) *stats = rbe_search_stats{};
            return;
        }
        if (!query_words || !scores || !ids || !partitions || !counts)
            throw InvalidArgument("rbe_cuda_search: null buffer");
        const size_t qbytes = size_t(n_queries) * query_planes * ix->shape.wpp * 8;
        ix->queries.ensure(qbytes);
        RBE_CK(cudaMemcpyAsync(ix->queries.p, query_words, qbytes, cudaMemcpyHostToDevice, ix->stream));
        // without stats the batch runs with a single host synchronisation (after the D2H below)
        run_batch(ix, ix->stream, n_queries, query_planes, geometry, n, options, stats, stats != nullptr);
        const size_t ne = size_t(n_queries) * n;
        if (pinned_host(scores) && pinned_host(ids) && pinned_host(partitions) && pinned_host(counts) &&
            (!accs || pinned_host(accs))) {
            // caller buffers in pinned host memory: convert to their layout on the device and DMA
            // straight into them (no staging, no host scatter)
            const size_t b8 = ne * 8, b4 = ne * 4;
            ix->soa.ensure(3 * b8 + b4 + size_t(n_queries) * 8 + 256);
            uint8_t* base = static_cast<uint8_t*>(ix->soa.p);
            double* dS = reinterpret_cast<double*>(base);
            uint64_t* dI = reinterpret_cast<uint64_t*>(base + b8);
            int64_t* dA = reinterpret_cast<int64_t*>(base + 2 * b8);
            uint64_t* dC = reinterpret_cast<uint64_t*>(base + 3 * b8);
            uint32_t* dP = reinterpret_cast<uint32_t*>(base + 3 * b8 + size_t(n_queries) * 8);
            launch_results_to_soa(ix->out.as<Result>(), n_queries, n, dS, dI, dP, accs ? dA : nullptr, dC, ix->stream);
            RBE_CK(cudaMemcpyAsync(scores, dS, b8, cudaMemcpyDeviceToHost, ix->stream));
            RBE_CK(cudaMemcpyAsync(ids, dI, b8, cudaMemcpyDeviceToHost, ix->stream));
            RBE_CK(cudaMemcpyAsync(partitions, dP, b4, cudaMemcpyDeviceToHost, ix->stream));
            if (accs) RBE_CK(cudaMemcpyAsync(accs, dA, b8, cudaMemcpyDeviceToHost, ix->stream));
            RBE_CK(cudaMemcpyAsync(counts, dC, size_t(n_queries) * 8, cudaMemcpyDeviceToHost, ix->stream));
            RBE_CK(cudaStreamSynchronize(ix->stream));
            return;
        }
        // pageable caller buffers: the same device-side conversion, one D2H into pinned staging,
        // then contiguous copies (no per-record scatter on the host)
        const size_t b8 = ne * 8, b4 = ne * 4;
        ix->soa.ensure(3 * b8 + b4 + size_t(n_queries) * 8 + 256);
        uint8_t* base = static_cast<uint8_t*>(ix->soa.p);
        double* dS = reinterpret_cast<double*>(base);
        uint64_t* dI = reinterpret_cast<uint64_t*>(base + b8);
        int64_t* dA = reinterpret_cast<int64_t*>(base + 2 * b8);
        uint64_t* dC = reinterpret_cast<uint64_t*>(base + 3 * b8);
        uint32_t* dP = reinterpret_cast<uint32_t*>(base + 3 * b8 + size_t(n_queries) * 8);
        launch_results_to_soa(ix->out.as<Result>(), n_queries, n, dS, dI, dP, accs ? dA : nullptr, dC, ix->stream);
        const size_t total = 3 * b8 + b4 + size_t(n_queries) * 8;
        ix->ensure_host_out((total + sizeof(Result) - 1) / sizeof(Result));
        uint8_t* h = reinterpret_cast<uint8_t*>(ix->host_out);
        RBE_CK(cudaMemcpyAsync(h, base, total, cudaMemcpyDeviceToHost, ix->stream));
        RBE_CK(cudaStreamSynchronize(ix->stream));
        std::memcpy(scores, h, b8);
        std::memcpy(ids, h + b8, b8);
        if (accs) std::memcpy(accs, h + 2 * b8, b8);
        std::memcpy(counts, h + 3 * b8, size_t(n_queries) * 8);
        std::memcpy(partitions, h + 3 * b8 + size_t(n_queries) * 8, b4);
    });
}

int rbe_cuda_host_alloc(size_t bytes, void** out) {
    return guarded([&] {
        if (!out) throw InvalidArgument("rbe_cuda_host_alloc: null output");
        *out = nullptr;
        if (bytes == 0) return;
        RBE_CK(cudaMallocHost(out, bytes));
    });
}

int rbe_cuda_host_free(void* p) {
    return guarded([&] {
        if (p) RBE_CK(cudaFreeHost(p));
    });
}

int rbe_cuda_index_last_batch_ms(rbe_cuda_index* ix, double* scan_ms, double* total_ms) {
    return guarded([&] {
        if (!ix) throw InvalidArgument("rbe_cuda_index_last_batch_ms: null index");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        RBE_CK(cudaEventSynchronize(ix->ev[3]));
        float ms = 0;
        RBE_CK(cudaEventElapsedTime(&ms, ix->ev[1], ix->ev[2]));
        if (scan_ms) *scan_ms = ms;
        RBE_CK(cudaEventElapsedTime(&ms, ix->ev[0], ix->ev[3]));
        if (total_ms) *total_ms = ms;
    });
}

int rbe_cuda_merge_device(int device, const rbe_result* d_in, uint32_t n_lists, uint32_t n_queries, uint64_t n,
                          rbe_result* d_out, void* stream) {
    return guarded([&] {
        check_device_usable(device);
        DeviceGuard dg(device);
        if (n_queries == 0 || n == 0) return;
        if (!d_in || !d_out) throw InvalidArgument("rbe_cuda_merge_device: null buffer");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const uint64_t cap = uint64_t(n_lists) * n;
        DevBuf tmp, cnt, scr;
        tmp.ensure(sizeof(Result) * cap * n_queries);
        cnt.ensure(sizeof(unsigned long long) * n_queries);
        RBE_CK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * n_queries, st));
        const uint64_t total = cap * n_queries;
        gather_lists_kernel<<<unsigned(std::min<uint64_t>((total + 255) / 256, 65535)), 256, 0, st>>>(
            reinterpret_cast<const Result*>(d_in), n_lists, n_queries, n, tmp.as<Result>(),
            cnt.as<unsigned long long>());
        RBE_CK(cudaGetLastError());
        const size_t ss = select_scratch_bytes(n_queries, cap, n);
        scr.ensure(ss);
        launch_select_topn(tmp.as<Result>(), cnt.as<unsigned long long>(), cap, n_queries, n,
                           reinterpret_cast<Result*>(d_out), scr.p, ss, st);
        RBE_CK(cudaStreamSynchronize(st));
    });
}

int rbe_cuda_search_multi(rbe_cuda_index* const* handles, uint32_t n_handles, const uint64_t* query_words,
                          uint32_t n_queries, uint32_t query_planes, const rbe_scan_geometry* geometry, uint64_t n,
                          const rbe_search_options* options, double* scores, uint64_t* ids, uint32_t* partitions,
                          int64_t* accs, uint64_t* counts, rbe_search_stats* stats) {
    if (n_handles == 1)
        return rbe_cuda_search(handles[0], query_words, n_queries, query_planes, geometry, n, options, scores, ids,
                               partitions, accs, counts, stats);
    return guarded([&] {
        if (!handles || n_handles == 0 || !geometry) throw InvalidArgument("rbe_cuda_search_multi: null argument");
        for (uint32_t h = 0; h < n_handles; ++h) {
            std::lock_guard<std::mutex> lk(handles[h]->mu);
            validate_search(handles[h], query_planes, geometry);
        }
        if (n_queries == 0) return;
        if (n == 0) {
            if (counts) std::fill(counts, counts + n_queries, 0);
            return;
        }
        const int root = handles[0]->device;
        const size_t cells = size_t(n_queries) * n;
        const size_t list_bytes = sizeof(Result) * cells;
        const size_t qbytes = size_t(n_queries) * query_planes * handles[0]->shape.wpp * 8;
        rbe_search_stats total{};
        std::vector<DevBuf> dq(n_handles), dres(n_handles);
        DevBuf gathered, merged;
        for (uint32_t h = 0; h < n_handles; ++h) {
            DeviceGuard dg(handles[h]->device);
            dq[h].ensure(qbytes);
            dres[h].ensure(list_bytes);
            RBE_CK(cudaMemcpy(dq[h].p, query_words, qbytes, cudaMemcpyHostToDevice));
            rbe_search_stats st{};
            const int rc = rbe_cuda_search_device(handles[h], dq[h].as<uint64_t>(), n_queries, query_planes, geometry,
                                                  n, options, dres[h].as<rbe_result>(), nullptr, &st);
            if (rc != RBE_CUDA_OK) {
                if (rc == RBE_CUDA_EINVAL) throw InvalidArgument(g_last_error);
                if (rc == RBE_CUDA_ERANGE) throw OutOfRange(g_last_error);
                throw CudaError(g_last_error);
            }
            total.scored += st.scored;
            total.candidates += st.candidates;
            total.survivors += st.survivors;
            total.variant = st.variant;
            total.fallback |= st.fallback;
            total.launches += st.launches;
            total.scan_ms = std::max(total.scan_ms, st.scan_ms);
            total.total_ms = std::max(total.total_ms, st.total_ms);
        }
        DeviceGuard dg(root);
        gathered.ensure(list_bytes * n_handles);
        merged.ensure(list_bytes);
        for (uint32_t h = 0; h < n_handles; ++h)
            RBE_CK(cudaMemcpyPeer(static_cast<char*>(gathered.p) + h * list_bytes, root, dres[h].p, handles[h]->device,
                                  list_bytes));
        const int rc = rbe_cuda_merge_device(root, gathered.as<rbe_result>(), n_handles, n_queries, n,
                                             merged.as<rbe_result>(), nullptr);
        if (rc != RBE_CUDA_OK) throw CudaError(g_last_error);
        std::vector<Result> host(cells);
        RBE_CK(cudaMemcpy(host.data(), merged.p, list_bytes, cudaMemcpyDeviceToHost));
        for (uint32_t q = 0; q < n_queries; ++q) {
            uint64_t c = 0;
            for (uint64_t k = 0; k < n; ++k) {
                const Result& r = host[size_t(q) * n + k];
                if (!r.valid) break;
                const size_t o = size_t(q) * n + k;
                scores[o] = r.score;
                ids[o] = r.id;
                partitions[o] = r.partition;
                if (accs) accs[o] = r.acc;
                ++c;
            }
            counts[q] = c;
        }
        for (uint32_t h = 0; h < n_handles; ++h) {
            DeviceGuard g2(handles[h]->device);
            dq[h].release();
            dres[h].release();
        }
        gathered.release();
        merged.release();
        if (stats) *stats = total;
    });
}

}  // extern "C"
