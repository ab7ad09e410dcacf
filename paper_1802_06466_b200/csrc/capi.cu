// capi.cu -- implementation of include/rbe_cuda.h: the device index (HBM
// store) and the batched search orchestration (query upload, scan kernel,
// device selection, result download).  No CPU fallback: every compute entry
// point fails with RBE_CUDA_ERUNTIME when CUDA is unusable.
//
// Concurrency and lifetime rules (include/rbe_cuda.h):
//  * every device buffer is owned (DevBuf frees itself) and per-batch scratch is
//    grown on demand, never allocated per call in steady state;
//  * a batch may be issued on any stream; each index records an event at the end
//    of its last batch and the next batch's stream waits on it before touching
//    the index's scratch, so batches on different streams never overlap;
//  * the tensor kernel's internal-consistency flag is sticky: it is never cleared
//    per batch, and the next synchronous call on the index (rbe_cuda_search,
//    search_device with stats, last_batch_ms, search_multi) reports it.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nvtx3/nvToolsExt.h>
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sort.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <thread>
#include <array>
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

// Owned device allocation, grown on demand (cudaFree synchronises the device,
// so growing never races with in-flight work that used the old buffer).
class DevBuf {
public:
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
        o.p = nullptr;
        o.bytes = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            bytes = o.bytes;
            o.p = nullptr;
            o.bytes = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void ensure(size_t b) {
        if (b <= bytes) return;
        release();
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
    void* p = nullptr;
    size_t bytes = 0;
};

uint64_t round_up(uint64_t x, uint64_t m) { return (x + m - 1) / m * m; }

// NVTX range for the host-side phases (batch enqueue, scan plan, selection, ingest), so a
// profiler timeline attributes launches to the phase that issued them
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

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

// Device usability, checked once per device (cudaGetDeviceProperties is slow).
constexpr int kMaxDevices = 64;
void check_device_usable(int device) {
    static std::once_flag count_once;
    static int n_devices = 0;
    static cudaError_t count_err = cudaSuccess;
    std::call_once(count_once, [] { count_err = cudaGetDeviceCount(&n_devices); });
    if (count_err != cudaSuccess || n_devices == 0)
        throw CudaError(std::string("no usable CUDA device (") + cudaGetErrorString(count_err) +
                        "); the RBE search path has no CPU fallback");
    if (device < 0 || device >= n_devices || device >= kMaxDevices)
        throw InvalidArgument("rbe_cuda: device ordinal out of range");
    static std::mutex mu;
    static std::array<int, kMaxDevices> major{};  // 0 = not yet queried
    std::lock_guard<std::mutex> lk(mu);
    if (major[device] == 0) {
        cudaDeviceProp prop;
        RBE_CK(cudaGetDeviceProperties(&prop, device));
        major[device] = prop.major * 100 + prop.minor;
    }
    if (major[device] / 100 != 10)
        throw CudaError("rbe_cuda: kernels are compiled for sm_100a (B200); device " + std::to_string(device) +
                        " is sm_" + std::to_string(major[device]));
}

// Stream-ordered exclusive use of a set of scratch buffers: the stream of the next
// user waits for the end of the previous user's work when it ran on another stream.
struct StreamOrder {
    cudaEvent_t done = nullptr;
    cudaStream_t last = nullptr;
    bool used = false;
    void acquire(cudaStream_t st) {
        if (used && last != st) RBE_CK(cudaStreamWaitEvent(st, done, 0));
    }
    void release(cudaStream_t st) {
        RBE_CK(cudaEventRecord(done, st));
        last = st;
        used = true;
    }
};

// Per-device context for the calls that take a device ordinal rather than an
// index (merge, select): persistent scratch, its own stream, stream ordering.
// Never destroyed (process lifetime): freeing at static destruction would race
// with the CUDA runtime's own teardown.
struct DeviceCtx {
    std::mutex mu;
    cudaStream_t stream = nullptr;
    StreamOrder order;
    DevBuf tmp, cnt, scr, io;
};
DeviceCtx& device_ctx(int device) {
    static std::mutex mu;
    static std::array<DeviceCtx*, kMaxDevices> ctx{};
    std::lock_guard<std::mutex> lk(mu);
    if (!ctx[device]) {
        DeviceGuard dg(device);
        auto* c = new DeviceCtx();
        RBE_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        RBE_CK(cudaEventCreateWithFlags(&c->order.done, cudaEventDisableTiming));
        ctx[device] = c;
    }
    return *ctx[device];
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

// Enqueue the merge of n_lists result lists per query (in = [n_lists][Q][n]) into
// out = [Q][n] on stream st, with the scratch buffers given (no host synchronisation).
void enqueue_merge(const Result* d_in, uint32_t n_lists, uint32_t Q, uint64_t n, Result* d_out, DevBuf& tmp,
                   DevBuf& cnt, DevBuf& scr, cudaStream_t st) {
    const uint64_t cap = uint64_t(n_lists) * n;
    tmp.ensure(sizeof(Result) * cap * Q);
    cnt.ensure(sizeof(unsigned long long) * Q);
    RBE_CK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * Q, st));
    const uint64_t total = cap * Q;
    gather_lists_kernel<<<unsigned(std::min<uint64_t>((total + 255) / 256, 65535)), 256, 0, st>>>(
        d_in, n_lists, Q, n, tmp.as<Result>(), cnt.as<unsigned long long>());
    RBE_CK(cudaGetLastError());
    const size_t ss = select_scratch_bytes(Q, cap, n);
    scr.ensure(ss);
    launch_select_topn(tmp.as<Result>(), cnt.as<unsigned long long>(), cap, Q, n, d_out, scr.p, ss, st);
}

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
    uint64_t total = 0;  // documents held by this handle
    DevBuf store;
    DevBuf d_parts;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[4] = {};  // batch start, scan start, scan end, batch end (timing)
    StreamOrder order;       // scratch ownership across streams
    std::mutex mu;
    // per-batch scratch, grown on demand
    DevBuf queries, qperm, qtensor, surv, surv_count, counters, queue_scratch, sel_scratch, out, probe, thresholds, soa;
    // multi-handle search, on the root handle: the gathered lists, the merged list, merge scratch
    DevBuf gathered, merged, mtmp, mcnt, mscr;
    DevBuf sticky;               // u32 internal-consistency flag, cleared only when reported
    bool mag_range_ok = false;   // cached magnitude range (tensor threshold bins)
    float mag_lo = 0.0f, mag_hi = 0.0f;
    uint8_t* host_out = nullptr;  // page-locked staging for result D2H (+ flags)
    size_t host_out_cap = 0;
    void ensure_host_out(size_t bytes) {
        if (bytes <= host_out_cap) return;
        if (host_out) cudaFreeHost(host_out);
        host_out = nullptr;
        host_out_cap = 0;
        RBE_CK(cudaMallocHost(&host_out, bytes));
        host_out_cap = bytes;
    }

    ~rbe_cuda_index() {
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        if (host_out) cudaFreeHost(host_out);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (order.done) cudaEventDestroy(order.done);
        if (stream) cudaStreamDestroy(stream);
        // DevBuf members free themselves (device already current)
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

// Reference-order argument checks of local_select (search.cpp:62-71, 80-82) for one handle;
// the empty-index check of search (search.cpp:133-135) is done over all handles by the caller.
void validate_shape(const rbe_cuda_index* ix, uint32_t qp, const rbe_scan_geometry* g) {
    if (qp == 0) throw InvalidArgument("local_select: query dimension mismatch");
    if (g->queue_length == 0) throw InvalidArgument("local_select: queue_length must be positive");
    const uint64_t capacity = uint64_t(g->blocks) * g->threads_per_block * g->items_per_thread;
    for (auto& p : ix->parts)
        if (capacity < p.count) throw InvalidArgument("local_select: geometry does not cover partition");
    if (uint64_t(qp) * ix->shape.kp > 64) throw InvalidArgument("local_select: too many planes");
}
void validate_search(const rbe_cuda_index* ix, uint32_t qp, const rbe_scan_geometry* g) {
    if (ix->parts.empty() || ix->total == 0) throw InvalidArgument("search: empty index");
    validate_shape(ix, qp, g);
}

// Reports (and clears) the sticky internal-consistency flag; `flag` is its value as read
// back by the caller's synchronous copy.
void report_sticky(rbe_cuda_index* ix, uint32_t flag) {
    if (!flag) return;
    RBE_CK(cudaMemsetAsync(ix->sticky.p, 0, 4, ix->stream));
    RBE_CK(cudaStreamSynchronize(ix->stream));
    throw std::logic_error("tensor scan: accumulator recovery failed (internal error)");
}
void check_sticky_sync(rbe_cuda_index* ix, cudaStream_t st) {
    uint32_t* h = reinterpret_cast<uint32_t*>(ix->host_out);
    RBE_CK(cudaMemcpyAsync(h, ix->sticky.p, 4, cudaMemcpyDeviceToHost, st));
    RBE_CK(cudaStreamSynchronize(st));
    report_sticky(ix, *h);
}

struct Pending {
    rbe_search_stats stats{};
    uint64_t surv_cap = 0;
    uint32_t Q = 0;
};

// Enqueue one batch with the queries already on the device (ix->queries); leaves
// rbe_result[Q][n] in ix->out.  The tensor variant never synchronises here; the
// exact variant does (its survivor-overflow retry).  The caller holds ix->mu, has
// acquired ix->order on st and releases it afterwards.
Pending enqueue_batch(rbe_cuda_index* ix, cudaStream_t st, uint32_t Q, uint32_t qp, const rbe_scan_geometry* g,
                      uint64_t n, const rbe_search_options* opt) {
    NvtxRange nvtx("rbe_cuda.batch");
    const Shape& s = ix->shape;
    ScanArgs a;
    a.parts = ix->d_parts.as<PartDesc>();
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

    Pending pd;
    pd.Q = Q;
    pd.stats.variant = variant;
    ix->counters.ensure(64);
    unsigned long long* d_scored = ix->counters.as<unsigned long long>();
    unsigned int* d_overflow = reinterpret_cast<unsigned int*>(d_scored + 2);
    unsigned long long* d_cands = d_scored + 4;
    a.scored = d_scored;
    a.overflow = d_overflow;
    a.error = ix->sticky.as<unsigned int>();
    if (variant == RBE_VARIANT_TENSOR && !ix->mag_range_ok) {
        // one-time (per index contents) magnitude range for the threshold bins
        uint32_t* d_rng = reinterpret_cast<uint32_t*>(d_scored + 6);
        const uint32_t init[2] = {0xffffffffu, 0u};
        RBE_CK(cudaMemcpyAsync(d_rng, init, 8, cudaMemcpyHostToDevice, st));
        for (auto& p : ix->parts) launch_mag_range(p.mags, p.count, d_rng, st);
        uint32_t* rng = reinterpret_cast<uint32_t*>(ix->host_out);
        RBE_CK(cudaMemcpyAsync(rng, d_rng, 8, cudaMemcpyDeviceToHost, st));
        RBE_CK(cudaStreamSynchronize(st));
        std::memcpy(&ix->mag_lo, &rng[0], 4);
        std::memcpy(&ix->mag_hi, &rng[1], 4);
        ix->mag_range_ok = true;
    }
    a.mag_lo = ix->mag_lo;
    a.mag_hi = ix->mag_hi;

    RBE_CK(cudaEventRecord(ix->ev[0], st));
    uint64_t lossless_cap = 0;
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
            pd.stats.launches += 2;
            // survivor-list overflow cannot happen by construction (cap = every per-thread
            // survivor); checked anyway, synchronously
            uint32_t* h = reinterpret_cast<uint32_t*>(ix->host_out);
            RBE_CK(cudaMemcpyAsync(h, d_overflow, 4, cudaMemcpyDeviceToHost, st));
            RBE_CK(cudaStreamSynchronize(st));
            if (*h) throw std::logic_error("exact scan overflowed its survivor list");
            break;
        }
        std::vector<uint64_t> counts;
        for (auto& p : ix->parts) counts.push_back(p.count);
        TensorScanPlan plan = plan_tensor_scan(s, qp, *g, Q, counts, n, probe_tiles, lossless_cap);
        a.surv_cap = plan.surv_cap;
        ix->surv.ensure(sizeof(Result) * a.surv_cap * Q);
        a.surv = ix->surv.as<Result>();
        ix->qtensor.ensure(plan.query_bytes);
        ix->probe.ensure(plan.probe_bytes);
        ix->thresholds.ensure(plan.threshold_bytes);
        ix->queue_scratch.ensure(plan.state_bytes);
        RBE_CK(cudaEventRecord(ix->ev[1], st));
        pd.stats.launches += run_tensor_scan(plan, a, s, ix->queries.as<uint64_t>(), ix->qtensor.p, ix->probe.p,
                                             ix->thresholds.p, ix->queue_scratch.p, d_cands, st);
        RBE_CK(cudaEventRecord(ix->ev[2], st));
        // queue_length 1: at most one survivor per logical thread, never overflows.  Lossless
        // geometry: every document >= theta survives; a bounded list, re-run once with the exact
        // size if a query overflowed it (synchronous, this case only)
        if (plan.lossless) {
            unsigned long long* h = reinterpret_cast<unsigned long long*>(ix->host_out);
            ix->ensure_host_out(sizeof(unsigned long long) * Q);
            h = reinterpret_cast<unsigned long long*>(ix->host_out);
            RBE_CK(cudaMemcpyAsync(h, a.surv_count, sizeof(unsigned long long) * Q, cudaMemcpyDeviceToHost, st));
            RBE_CK(cudaStreamSynchronize(st));
            const unsigned long long mx = *std::max_element(h, h + Q);
            if (mx > plan.surv_cap && attempt == 0) {
                lossless_cap = mx;
                continue;
            }
            if (mx > plan.surv_cap) throw std::logic_error("tensor scan overflowed its survivor list twice");
        }
        break;
    }
    const size_t ss = select_scratch_bytes(Q, a.surv_cap, n);
    ix->sel_scratch.ensure(ss);
    ix->out.ensure(sizeof(Result) * size_t(Q) * n);
    {
        NvtxRange nvtx_sel("rbe_cuda.select");
        launch_select_topn(a.surv, a.surv_count, a.surv_cap, Q, n, ix->out.as<Result>(), ix->sel_scratch.p, ss, st);
    }
    pd.stats.launches += 1;
    RBE_CK(cudaEventRecord(ix->ev[3], st));
    pd.surv_cap = a.surv_cap;
    return pd;
}

// Wait for an enqueued batch, read its counters and the sticky flag (reported as an
// error), and fill the stats.
void finish_batch(rbe_cuda_index* ix, cudaStream_t st, const Pending& pd, rbe_search_stats* st_out) {
    const uint32_t Q = pd.Q;
    ix->ensure_host_out(64 + 8 + sizeof(unsigned long long) * Q);
    unsigned long long* hc = reinterpret_cast<unsigned long long*>(ix->host_out);
    uint32_t* hflag = reinterpret_cast<uint32_t*>(hc + 8);
    unsigned long long* hs = hc + 9;
    RBE_CK(cudaMemcpyAsync(hc, ix->counters.p, 64, cudaMemcpyDeviceToHost, st));
    RBE_CK(cudaMemcpyAsync(hflag, ix->sticky.p, 4, cudaMemcpyDeviceToHost, st));
    RBE_CK(cudaMemcpyAsync(hs, ix->surv_count.p, sizeof(unsigned long long) * Q, cudaMemcpyDeviceToHost, st));
    RBE_CK(cudaStreamSynchronize(st));
    report_sticky(ix, *hflag);
    if (!st_out) return;
    rbe_search_stats stats = pd.stats;
    stats.scored = hc[0];
    stats.candidates = hc[4];
    for (uint32_t q = 0; q < Q; ++q) stats.survivors += std::min<uint64_t>(hs[q], pd.surv_cap);
    float ms = 0;
    RBE_CK(cudaEventElapsedTime(&ms, ix->ev[1], ix->ev[2]));
    stats.scan_ms = ms;
    RBE_CK(cudaEventElapsedTime(&ms, ix->ev[0], ix->ev[3]));
    stats.total_ms = ms;
    *st_out = stats;
}

struct HostOut {
    double* scores;
    uint64_t* ids;
    uint32_t* partitions;
    int64_t* accs;
    uint64_t* counts;
};

// Device result records [Q][n] on ix's device -> the caller's host arrays (one
// device-side conversion to their layout, then DMA straight into page-locked arrays
// or one staged copy for pageable ones), the sticky flag read back with them.
void deliver(rbe_cuda_index* ix, const Result* d_res, uint32_t Q, uint64_t n, const HostOut& o, cudaStream_t st) {
    const size_t ne = size_t(Q) * n;
    const size_t b8 = ne * 8, b4 = ne * 4;
    ix->soa.ensure(3 * b8 + b4 + size_t(Q) * 8 + 256);
    uint8_t* base = static_cast<uint8_t*>(ix->soa.p);
    double* dS = reinterpret_cast<double*>(base);
    uint64_t* dI = reinterpret_cast<uint64_t*>(base + b8);
    int64_t* dA = reinterpret_cast<int64_t*>(base + 2 * b8);
    uint64_t* dC = reinterpret_cast<uint64_t*>(base + 3 * b8);
    uint32_t* dP = reinterpret_cast<uint32_t*>(base + 3 * b8 + size_t(Q) * 8);
    launch_results_to_soa(d_res, Q, n, dS, dI, dP, o.accs ? dA : nullptr, dC, st);
    const bool pinned = pinned_host(o.scores) && pinned_host(o.ids) && pinned_host(o.partitions) &&
                        pinned_host(o.counts) && (!o.accs || pinned_host(o.accs));
    const size_t total = 3 * b8 + b4 + size_t(Q) * 8;
    ix->ensure_host_out(16 + (pinned ? 0 : total));
    uint32_t* hflag = reinterpret_cast<uint32_t*>(ix->host_out);
    uint8_t* h = ix->host_out + 16;
    if (pinned) {
        RBE_CK(cudaMemcpyAsync(o.scores, dS, b8, cudaMemcpyDeviceToHost, st));
        RBE_CK(cudaMemcpyAsync(o.ids, dI, b8, cudaMemcpyDeviceToHost, st));
        RBE_CK(cudaMemcpyAsync(o.partitions, dP, b4, cudaMemcpyDeviceToHost, st));
        if (o.accs) RBE_CK(cudaMemcpyAsync(o.accs, dA, b8, cudaMemcpyDeviceToHost, st));
        RBE_CK(cudaMemcpyAsync(o.counts, dC, size_t(Q) * 8, cudaMemcpyDeviceToHost, st));
    } else {
        RBE_CK(cudaMemcpyAsync(h, base, total, cudaMemcpyDeviceToHost, st));
    }
    RBE_CK(cudaMemcpyAsync(hflag, ix->sticky.p, 4, cudaMemcpyDeviceToHost, st));
    RBE_CK(cudaStreamSynchronize(st));
    report_sticky(ix, *hflag);
    if (!pinned) {
        std::memcpy(o.scores, h, b8);
        std::memcpy(o.ids, h + b8, b8);
        if (o.accs) std::memcpy(o.accs, h + 2 * b8, b8);
        std::memcpy(o.counts, h + 3 * b8, size_t(Q) * 8);
        std::memcpy(o.partitions, h + 3 * b8 + size_t(Q) * 8, b4);
    }
}

void rethrow_status(int rc) {
    if (rc == RBE_CUDA_OK) return;
    if (rc == RBE_CUDA_EINVAL) throw InvalidArgument(g_last_error);
    if (rc == RBE_CUDA_ERANGE) throw OutOfRange(g_last_error);
    throw CudaError(g_last_error);
}

}  // namespace

namespace {

// ---------------------------------------------------------------- ingest
// One partition in the reference's natural layout (Partition::plane_blocks [kp][count][wpp]
// u64, magnitudes f32, ids u64; index.hpp:16-21) streamed into HBM in chunks of documents:
// the host fills a page-locked staging buffer per chunk (from memory or from an RBEI file, with
// several host threads), the chunk's plane words are copied to a device staging buffer and
// re-packed into the store layout by the device, magnitudes and ids are copied in place.  Two
// staging buffers alternate, so the host fill of chunk c + 1 overlaps the copies and the repack
// of chunk c.
struct ChunkSource {
    virtual ~ChunkSource() = default;
    // write docs [z0, z0 + n): plane words [kp][n][wpp], then n f32 magnitudes, then n u64 ids
    virtual void fill(uint8_t* dst, uint64_t z0, uint64_t n) = 0;
};

// run `pieces` (byte-range copies) on up to `threads` host threads
struct Piece {
    uint8_t* dst;
    uint64_t off;  // file offset, or source address for memory copies
    size_t len;
};
template <typename F>
void run_pieces(std::vector<Piece>& pieces, uint32_t threads, F&& copy) {
    std::vector<Piece> split;
    constexpr size_t kPiece = size_t(8) << 20;
    for (const Piece& pc : pieces)
        for (size_t o = 0; o < pc.len; o += kPiece)
            split.push_back(Piece{pc.dst + o, pc.off + o, std::min(kPiece, pc.len - o)});
    const uint32_t T = std::max<uint32_t>(1, std::min<uint32_t>(threads, uint32_t(split.size())));
    if (T == 1) {
        for (const Piece& pc : split) copy(pc);
        return;
    }
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(T);
    for (uint32_t t = 0; t < T; ++t)
        pool.emplace_back([&, t] {
            try {
                for (size_t k = t; k < split.size(); k += T) copy(split[k]);
            } catch (...) {
                errs[t] = std::current_exception();
            }
        });
    for (auto& th : pool) th.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

std::vector<Piece> chunk_pieces(uint8_t* dst, uint64_t planes0, uint64_t mags0, uint64_t ids0, uint64_t count,
                                uint32_t kp, uint32_t wpp, uint64_t z0, uint64_t n) {
    std::vector<Piece> v;
    for (uint32_t t = 0; t < kp; ++t)
        v.push_back(Piece{dst + size_t(t) * n * wpp * 8, planes0 + (uint64_t(t) * count + z0) * wpp * 8, size_t(n) * wpp * 8});
    uint8_t* m = dst + size_t(kp) * n * wpp * 8;
    v.push_back(Piece{m, mags0 + z0 * 4, size_t(n) * 4});
    v.push_back(Piece{m + n * 4, ids0 + z0 * 8, size_t(n) * 8});
    return v;
}

struct MemorySource : ChunkSource {
    const uint64_t* planes;
    const float* mags;
    const uint64_t* ids;
    uint64_t count;
    uint32_t kp, wpp, threads;
    void fill(uint8_t* dst, uint64_t z0, uint64_t n) override {
        auto pcs = chunk_pieces(dst, uint64_t(uintptr_t(planes)), uint64_t(uintptr_t(mags)), uint64_t(uintptr_t(ids)),
                                count, kp, wpp, z0, n);
        run_pieces(pcs, threads, [](const Piece& pc) {
            std::memcpy(pc.dst, reinterpret_cast<const void*>(uintptr_t(pc.off)), pc.len);
        });
    }
};

struct FileSource : ChunkSource {
    int fd = -1;
    std::string path;
    uint64_t planes0, mags0, ids0, count;
    uint32_t kp, wpp, threads;
    uint64_t* bytes_read = nullptr;
    void fill(uint8_t* dst, uint64_t z0, uint64_t n) override {
        auto pcs = chunk_pieces(dst, planes0, mags0, ids0, count, kp, wpp, z0, n);
        run_pieces(pcs, threads, [&](const Piece& pc) {
            size_t done = 0;
            while (done < pc.len) {
                const ssize_t r = ::pread(fd, pc.dst + done, pc.len - done, off_t(pc.off + done));
                if (r < 0 && errno == EINTR) continue;
                if (r <= 0) throw std::runtime_error("truncated index file: " + path);
                done += size_t(r);
            }
        });
        for (const Piece& pc : pcs) *bytes_read += pc.len;
    }
};

void stream_partition(rbe_cuda_index* ix, uint32_t i, ChunkSource& src) {
    NvtxRange nvtx("rbe_cuda.ingest_partition");
    auto& L = ix->parts[i];
    if (L.count == 0) return;
    const Shape& s = ix->shape;
    cudaStream_t st = ix->stream;
    const size_t plane_doc = size_t(s.kp) * s.wpp * 8, per_doc = plane_doc + 12;
    const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(L.count, (size_t(64) << 20) / per_doc));
    struct Host {
        uint8_t* p = nullptr;
        ~Host() {
            if (p) cudaFreeHost(p);
        }
    } host[2];
    DevBuf dnat[2];
    cudaEvent_t ev[2] = {nullptr, nullptr};
    struct Events {
        cudaEvent_t* e;
        ~Events() {
            for (int k = 0; k < 2; ++k)
                if (e[k]) cudaEventDestroy(e[k]);
        }
    } ev_guard{ev};
    for (int k = 0; k < 2; ++k) {
        RBE_CK(cudaMallocHost(&host[k].p, chunk * per_doc));
        dnat[k].ensure(chunk * plane_doc);
        RBE_CK(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
    }
    ix->order.acquire(st);
    uint64_t c = 0;
    for (uint64_t z0 = 0; z0 < L.count; z0 += chunk, ++c) {
        const int k = int(c & 1);
        const uint64_t n = std::min(chunk, L.count - z0);
        if (c >= 2) RBE_CK(cudaEventSynchronize(ev[k]));  // staging k free again
        src.fill(host[k].p, z0, n);
        RBE_CK(cudaMemcpyAsync(dnat[k].p, host[k].p, n * plane_doc, cudaMemcpyHostToDevice, st));
        RBE_CK(cudaMemcpyAsync(L.mags + z0, host[k].p + n * plane_doc, n * 4, cudaMemcpyHostToDevice, st));
        RBE_CK(cudaMemcpyAsync(L.ids + z0, host[k].p + n * plane_doc + n * 4, n * 8, cudaMemcpyHostToDevice, st));
        // chunk [z0, z0 + n) of the store: plane t of doc z lives at (t count_pad + z) w32
        launch_repack_planes(dnat[k].as<uint64_t>(), L.planes + z0 * s.w32, n, L.count_pad, s, ix->perm, st);
        RBE_CK(cudaEventRecord(ev[k], st));
    }
    ix->mag_range_ok = false;
    ix->counters.ensure(64);
    RBE_CK(cudaMemsetAsync(ix->counters.p, 0, 4, st));
    launch_validate_mags(L.mags, L.count, ix->counters.as<uint32_t>(), st);
    uint32_t* bad = reinterpret_cast<uint32_t*>(ix->host_out);
    RBE_CK(cudaMemcpyAsync(bad, ix->counters.p, 4, cudaMemcpyDeviceToHost, st));
    ix->order.release(st);
    RBE_CK(cudaStreamSynchronize(st));
    if (*bad) throw InvalidArgument("keyword magnitudes must be finite and > 0");
}

// RBEE v1 bulk embeddings header ("RBEE", u32 version, dim, plane count, rw; then fixed-width
// records of u64 id, plane words, f32 magnitude), read as the reference's EmbeddingReader does
// (src/embedding_io.cpp:48-77), with the same errors
struct RbeeHeader {
    rbe_index_shape shape{};
    uint64_t count = 0;
    uint64_t record_bytes = 0;
};
constexpr uint64_t kRbeeHeaderBytes = 4 + 4 * 4;

RbeeHeader read_rbee_header(const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("cannot open embeddings file: " + path);
    struct Closer {
        FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "RBEE", 4) != 0)
        throw std::runtime_error("not an RBEE embeddings file: " + path);
    uint32_t h[4] = {0, 0, 0, 0};
    const size_t got = std::fread(h, 4, 4, f);
    if (got < 1 || h[0] != 1) throw std::runtime_error("unsupported embeddings version");
    RbeeHeader r;
    r.shape.dim = got >= 2 ? h[1] : 0;
    r.shape.keyword_planes = got >= 3 ? h[2] : 0;
    r.shape.residual_weights = got >= 4 && h[3] != 0;
    if (r.shape.dim == 0 || r.shape.keyword_planes == 0) throw std::runtime_error("embeddings file has empty shape: " + path);
    struct stat sb;
    if (::stat(path.c_str(), &sb) != 0) throw std::runtime_error("cannot open embeddings file: " + path);
    const uint64_t size = uint64_t(sb.st_size);
    const uint64_t wpp = (uint64_t(r.shape.dim) + 63) / 64;
    r.record_bytes = 8 + uint64_t(r.shape.keyword_planes) * wpp * 8 + 4;
    if (size < kRbeeHeaderBytes || (size - kRbeeHeaderBytes) % r.record_bytes != 0)
        throw std::runtime_error("embeddings file has truncated records: " + path);
    r.count = (size - kRbeeHeaderBytes) / r.record_bytes;
    return r;
}

// ascending sort of u64 keys on the device (build-time validation only; thrust's radix sort)
void sort_u64(uint64_t* d, uint64_t n, cudaStream_t st) {
    thrust::sort(thrust::cuda::par.on(st), thrust::device_ptr<uint64_t>(d), thrust::device_ptr<uint64_t>(d) + n);
}

uint32_t default_io_threads() { return std::max(1u, std::min(16u, std::thread::hardware_concurrency())); }

// RBEI v1 header ("RBEI", u32 version, dim, kp, rw, P, u64 count[P]), read the
// way the reference's load_index reads it (src/index.cpp:170-189), with the same errors
struct RbeiHeader {
    rbe_index_shape shape{};
    std::vector<uint64_t> counts;
    uint64_t data_offset = 0;  // first byte of partition 0
    uint64_t file_bytes = 0;
};

RbeiHeader read_rbei_header(const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("cannot open index: " + path);
    struct Closer {
        FILE* f;
        ~Closer() { std::fclose(f); }
    } closer{f};
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "RBEI", 4) != 0)
        throw std::runtime_error("not an RBEI index file: " + path);
    uint32_t h[5];
    if (std::fread(h, 4, 5, f) != 5) throw std::runtime_error("truncated index file: " + path);
    if (h[0] != 1) throw std::runtime_error("unsupported index version");
    RbeiHeader r;
    r.shape.dim = h[1];
    r.shape.keyword_planes = h[2];
    r.shape.residual_weights = h[3] != 0;
    r.counts.resize(h[4]);
    if (h[4] && std::fread(r.counts.data(), 8, h[4], f) != h[4]) throw std::runtime_error("truncated index file: " + path);
    r.data_offset = 4 + 5 * 4 + uint64_t(h[4]) * 8;
    struct stat sb;
    if (::stat(path.c_str(), &sb) != 0) throw std::runtime_error("cannot open index: " + path);
    r.file_bytes = uint64_t(sb.st_size);
    const uint64_t wpp = (uint64_t(r.shape.dim) + 63) / 64;
    uint64_t end = r.data_offset;
    for (uint64_t c : r.counts) end += c * (uint64_t(r.shape.keyword_planes) * wpp * 8 + 12);
    if (end > r.file_bytes) throw std::runtime_error("truncated index file: " + path);
    return r;
}

}  // namespace

extern "C" {

const char* rbe_cuda_last_error(void) { return g_last_error.c_str(); }

const char* rbe_cuda_version(void) { return "rbe_cuda 0.2 sm_100a"; }

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
        ix->store.ensure(off);
        RBE_CK(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
        for (auto& e : ix->ev) RBE_CK(cudaEventCreate(&e));
        RBE_CK(cudaEventCreateWithFlags(&ix->order.done, cudaEventDisableTiming));
        ix->ensure_host_out(4096);
        ix->sticky.ensure(4);
        RBE_CK(cudaMemsetAsync(ix->sticky.p, 0, 4, ix->stream));
        std::vector<PartDesc> descs;
        for (uint32_t i = 0; i < n_partitions; ++i) {
            rbe_cuda_index::Local L;
            L.ordinal = ordinals[i];
            L.count = counts[i];
            L.count_pad = round_up(counts[i], 512) + 512;
            char* base = static_cast<char*>(ix->store.p) + offs[i];
            L.planes = reinterpret_cast<uint32_t*>(base);
            base += round_up(size_t(ix->shape.kp) * L.count_pad * ix->shape.w32 * 4, 256);
            L.mags = reinterpret_cast<float*>(base);
            base += round_up(L.count_pad * 4, 256);
            L.ids = reinterpret_cast<uint64_t*>(base);
            RBE_CK(cudaMemsetAsync(L.planes, 0, size_t(ix->shape.kp) * L.count_pad * ix->shape.w32 * 4, ix->stream));
            launch_fill_f32(L.mags, L.count_pad, 1.0f, ix->stream);
            ix->parts.push_back(L);
            ix->total += L.count;
            PartDesc d{L.planes, L.mags, L.ids, L.count, L.count_pad, L.ordinal, 0};
            descs.push_back(d);
        }
        if (!descs.empty()) {
            ix->d_parts.ensure(sizeof(PartDesc) * descs.size());
            RBE_CK(cudaMemcpyAsync(ix->d_parts.p, descs.data(), sizeof(PartDesc) * descs.size(), cudaMemcpyHostToDevice,
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
        MemorySource src;
        src.planes = planes;
        src.mags = mags;
        src.ids = ids;
        src.count = L.count;
        src.kp = ix->shape.kp;
        src.wpp = ix->shape.wpp;
        src.threads = default_io_threads();
        try {
            stream_partition(ix, i, src);
        } catch (const InvalidArgument& e) {
            throw InvalidArgument(std::string("rbe_cuda_index_upload_partition: ") + e.what());
        }
    });
}

int rbe_cuda_rbei_header(const char* path, rbe_index_shape* shape, uint32_t* n_partitions, uint64_t* counts,
                         uint32_t counts_cap) {
    return guarded([&] {
        if (!path || !shape || !n_partitions) throw InvalidArgument("rbe_cuda_rbei_header: null argument");
        const RbeiHeader h = read_rbei_header(path);
        *shape = h.shape;
        *n_partitions = uint32_t(h.counts.size());
        if (counts)
            for (uint32_t p = 0; p < std::min<uint32_t>(counts_cap, uint32_t(h.counts.size())); ++p) counts[p] = h.counts[p];
    });
}

int rbe_cuda_rbee_header(const char* path, rbe_index_shape* shape, uint64_t* count) {
    return guarded([&] {
        if (!path || !shape || !count) throw InvalidArgument("rbe_cuda_rbee_header: null argument");
        const RbeeHeader h = read_rbee_header(path);
        *shape = h.shape;
        *count = h.count;
    });
}

int rbe_cuda_index_build_rbee(const char* path, uint32_t n_partitions_total, const uint32_t* partitions,
                              uint32_t n_partitions, int device, uint32_t io_threads, rbe_cuda_index** out,
                              rbe_load_stats* stats) {
    return guarded([&] {
        if (!path || !out || (n_partitions && !partitions)) throw InvalidArgument("rbe_cuda_index_build_rbee: null argument");
        if (n_partitions_total == 0) throw InvalidArgument("IndexBuilder: need at least one partition");
        const auto t0 = std::chrono::steady_clock::now();
        const RbeeHeader h = read_rbee_header(path);
        const uint32_t P = n_partitions_total;
        std::vector<uint32_t> sel;
        if (n_partitions) sel.assign(partitions, partitions + n_partitions);
        else
            for (uint32_t p = 0; p < P; ++p) sel.push_back(p);
        std::vector<int32_t> local(P, -1);
        std::vector<uint64_t> counts;
        for (uint32_t i = 0; i < sel.size(); ++i) {
            if (sel[i] >= P) throw OutOfRange("rbe_cuda_index_build_rbee: partition out of range");
            local[sel[i]] = int32_t(i);
            counts.push_back(sel[i] < h.count ? (h.count - sel[i] + P - 1) / P : 0);  // record k -> k % P
        }
        rbe_cuda_index* raw = nullptr;
        const int rc = rbe_cuda_index_create(&h.shape, uint32_t(sel.size()), sel.data(), counts.data(), device, &raw);
        if (rc != RBE_CUDA_OK) {
            const std::string msg = g_last_error;
            if (rc == RBE_CUDA_EINVAL) throw InvalidArgument(msg);
            if (rc == RBE_CUDA_ERANGE) throw OutOfRange(msg);
            throw std::runtime_error(msg);
        }
        std::unique_ptr<rbe_cuda_index> ix(raw);
        const int fd = ::open(path, O_RDONLY);
        if (fd < 0) throw std::runtime_error("cannot open embeddings file: " + std::string(path));
        struct Fd {
            int fd;
            ~Fd() { ::close(fd); }
        } fd_guard{fd};
        ::posix_fadvise(fd, 0, 0, POSIX_FADV_SEQUENTIAL);
        DeviceGuard dg(device);
        std::lock_guard<std::mutex> lk(ix->mu);
        cudaStream_t st = ix->stream;
        const uint32_t threads = io_threads ? io_threads : default_io_threads();
        // records streamed in 64 MB chunks: pread -> page-locked staging -> device -> scatter kernel
        const uint64_t chunk = std::max<uint64_t>(1, (uint64_t(64) << 20) / h.record_bytes);
        struct Host {
            uint8_t* p = nullptr;
            ~Host() {
                if (p) cudaFreeHost(p);
            }
        } host[2];
        DevBuf drec[2], dlocal, dbad;
        cudaEvent_t ev[2] = {nullptr, nullptr};
        struct Events {
            cudaEvent_t* e;
            ~Events() {
                for (int k = 0; k < 2; ++k)
                    if (e[k]) cudaEventDestroy(e[k]);
            }
        } ev_guard{ev};
        const uint64_t nchunk = std::min(chunk, std::max<uint64_t>(h.count, 1));
        for (int k = 0; k < 2; ++k) {
            RBE_CK(cudaMallocHost(&host[k].p, nchunk * h.record_bytes));
            drec[k].ensure(nchunk * h.record_bytes);
            RBE_CK(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
        }
        dlocal.ensure(sizeof(int32_t) * P);
        dbad.ensure(16);  // [0] zero magnitudes, [1] non-finite magnitudes, [2] duplicate ids
        RBE_CK(cudaMemcpyAsync(dlocal.p, local.data(), sizeof(int32_t) * P, cudaMemcpyHostToDevice, st));
        RBE_CK(cudaMemsetAsync(dbad.p, 0, 16, st));
        uint64_t bytes = 0, c = 0;
        for (uint64_t r0 = 0; r0 < h.count; r0 += chunk, ++c) {
            const int k = int(c & 1);
            const uint64_t n = std::min(chunk, h.count - r0);
            if (c >= 2) RBE_CK(cudaEventSynchronize(ev[k]));
            std::vector<Piece> pcs{Piece{host[k].p, kRbeeHeaderBytes + r0 * h.record_bytes, size_t(n * h.record_bytes)}};
            const std::string pth(path);
            run_pieces(pcs, threads, [&](const Piece& pc) {
                size_t done = 0;
                while (done < pc.len) {
                    const ssize_t r = ::pread(fd, pc.dst + done, pc.len - done, off_t(pc.off + done));
                    if (r < 0 && errno == EINTR) continue;
                    if (r <= 0) throw std::runtime_error("truncated embeddings record");
                    done += size_t(r);
                }
            });
            bytes += n * h.record_bytes;
            RBE_CK(cudaMemcpyAsync(drec[k].p, host[k].p, n * h.record_bytes, cudaMemcpyHostToDevice, st));
            launch_rbee_scatter(drec[k].as<uint32_t>(), r0, n, P, dlocal.as<int32_t>(), ix->d_parts.as<PartDesc>(),
                                ix->shape, ix->perm, dbad.as<uint32_t>(), st);
            RBE_CK(cudaEventRecord(ev[k], st));
        }
        // IndexBuilder::finish: duplicate ids (within this handle; across handles the caller merges)
        uint64_t total = 0;
        for (auto& L : ix->parts) total += L.count;
        uint32_t* h_flags = reinterpret_cast<uint32_t*>(ix->host_out);
        if (total > 1) {
            DevBuf sorted;
            sorted.ensure(total * 8);
            uint64_t off = 0;
            for (auto& L : ix->parts) {
                RBE_CK(cudaMemcpyAsync(sorted.as<uint64_t>() + off, L.ids, L.count * 8, cudaMemcpyDeviceToDevice, st));
                off += L.count;
            }
            sort_u64(sorted.as<uint64_t>(), total, st);
            launch_count_adjacent_equal(sorted.as<uint64_t>(), total, dbad.as<uint32_t>() + 2, st);
        }
        RBE_CK(cudaMemcpyAsync(h_flags, dbad.p, 12, cudaMemcpyDeviceToHost, st));
        RBE_CK(cudaStreamSynchronize(st));
        ix->mag_range_ok = false;
        if (h_flags[0]) throw InvalidArgument("IndexBuilder: keyword has zero magnitude");
        if (h_flags[1]) throw InvalidArgument("rbe_cuda_index_build_rbee: keyword magnitudes must be finite and > 0");
        if (h_flags[2]) throw InvalidArgument("IndexBuilder: duplicate keyword id");
        if (stats) {
            stats->file_bytes_read = bytes;
            stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        *out = ix.release();
    });
}

int rbe_cuda_index_sorted_ids(const rbe_cuda_index* cix, uint64_t* ids) {
    return guarded([&] {
        rbe_cuda_index* ix = const_cast<rbe_cuda_index*>(cix);
        if (!ix || !ids) throw InvalidArgument("rbe_cuda_index_sorted_ids: null argument");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        uint64_t total = 0;
        for (auto& L : ix->parts) total += L.count;
        if (!total) return;
        cudaStream_t st = ix->stream;
        ix->order.acquire(st);
        DevBuf sorted;
        sorted.ensure(total * 8);
        uint64_t off = 0;
        for (auto& L : ix->parts) {
            RBE_CK(cudaMemcpyAsync(sorted.as<uint64_t>() + off, L.ids, L.count * 8, cudaMemcpyDeviceToDevice, st));
            off += L.count;
        }
        sort_u64(sorted.as<uint64_t>(), total, st);
        RBE_CK(cudaMemcpyAsync(ids, sorted.p, total * 8, cudaMemcpyDeviceToHost, st));
        ix->order.release(st);
        RBE_CK(cudaStreamSynchronize(st));
    });
}

int rbe_cuda_index_open_rbei(const char* path, const uint32_t* partitions, uint32_t n_partitions, int device,
                             uint32_t io_threads, rbe_cuda_index** out, rbe_load_stats* stats) {
    return guarded([&] {
        if (!path || !out || (n_partitions && !partitions)) throw InvalidArgument("rbe_cuda_index_open_rbei: null argument");
        const auto t0 = std::chrono::steady_clock::now();
        const RbeiHeader h = read_rbei_header(path);
        std::vector<uint32_t> sel;
        if (n_partitions) sel.assign(partitions, partitions + n_partitions);
        else
            for (uint32_t p = 0; p < h.counts.size(); ++p) sel.push_back(p);
        std::vector<uint64_t> counts;
        for (uint32_t p : sel) {
            if (p >= h.counts.size()) throw OutOfRange("rbe_cuda_index_open_rbei: partition out of range");
            counts.push_back(h.counts[p]);
        }
        rbe_cuda_index* raw = nullptr;
        const int rc = rbe_cuda_index_create(&h.shape, uint32_t(sel.size()), sel.data(), counts.data(), device, &raw);
        if (rc != RBE_CUDA_OK) {
            const std::string msg = g_last_error;
            if (rc == RBE_CUDA_EINVAL) throw InvalidArgument(msg);
            if (rc == RBE_CUDA_ERANGE) throw OutOfRange(msg);
            throw std::runtime_error(msg);
        }
        std::unique_ptr<rbe_cuda_index> ix(raw);
        const int fd = ::open(path, O_RDONLY);
        if (fd < 0) throw std::runtime_error("cannot open index: " + std::string(path));
        struct Fd {
            int fd;
            ~Fd() { ::close(fd); }
        } fd_guard{fd};
        ::posix_fadvise(fd, 0, 0, POSIX_FADV_SEQUENTIAL);
        // partition byte offsets in the file (partitions are stored back to back)
        const uint64_t wpp = ix->shape.wpp, kp = ix->shape.kp;
        std::vector<uint64_t> poff(h.counts.size() + 1, h.data_offset);
        for (size_t p = 0; p < h.counts.size(); ++p) poff[p + 1] = poff[p] + h.counts[p] * (kp * wpp * 8 + 12);
        uint64_t bytes = 0;
        DeviceGuard dg(device);
        std::lock_guard<std::mutex> lk(ix->mu);
        for (size_t i = 0; i < sel.size(); ++i) {
            FileSource src;
            src.fd = fd;
            src.path = path;
            src.count = h.counts[sel[i]];
            src.planes0 = poff[sel[i]];
            src.mags0 = src.planes0 + src.count * kp * wpp * 8;
            src.ids0 = src.mags0 + src.count * 4;
            src.kp = uint32_t(kp);
            src.wpp = uint32_t(wpp);
            src.threads = io_threads ? io_threads : default_io_threads();
            src.bytes_read = &bytes;
            try {
                stream_partition(ix.get(), uint32_t(i), src);
            } catch (const InvalidArgument& e) {
                throw InvalidArgument(std::string("rbe_cuda_index_open_rbei: ") + e.what());
            }
        }
        if (stats) {
            stats->file_bytes_read = bytes;
            stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        *out = ix.release();
    });
}

int rbe_cuda_index_fill_synthetic(rbe_cuda_index* ix, uint64_t seed, uint64_t n_total, uint32_t n_parts_total) {
    return guarded([&] {
        if (!ix) throw InvalidArgument("rbe_cuda_index_fill_synthetic: null index");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        if (n_parts_total == 0) throw InvalidArgument("rbe_cuda_index_fill_synthetic: need at least one partition");
        cudaStream_t st = ix->stream;
        ix->order.acquire(st);
        ix->mag_range_ok = false;
        for (auto& L : ix->parts) {
            if (L.ordinal >= n_parts_total) throw InvalidArgument("rbe_cuda_index_fill_synthetic: ordinal >= partitions");
            const uint64_t expect = L.ordinal < n_total ? (n_total - L.ordinal + n_parts_total - 1) / n_parts_total : 0;
            if (expect != L.count)
                throw InvalidArgument("rbe_cuda_index_fill_synthetic: partition count does not match round-robin split");
            launch_fill_synthetic(L.planes, L.mags, L.ids, L.count, L.count_pad, L.ordinal, n_parts_total, n_total, seed,
                                  ix->shape, ix->perm, st);
        }
        ix->order.release(st);
        RBE_CK(cudaStreamSynchronize(st));
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
        cudaStream_t st = ix->stream;
        ix->order.acquire(st);
        const size_t nat_bytes = size_t(s.kp) * L.count * s.wpp * 8;
        DevBuf tmp;
        tmp.ensure(nat_bytes);
        launch_unpack_planes(L.planes, tmp.as<uint64_t>(), L.count, L.count_pad, s, ix->perm, st);
        if (planes) RBE_CK(cudaMemcpyAsync(planes, tmp.p, nat_bytes, cudaMemcpyDeviceToHost, st));
        if (mags) RBE_CK(cudaMemcpyAsync(mags, L.mags, L.count * 4, cudaMemcpyDeviceToHost, st));
        if (ids) RBE_CK(cudaMemcpyAsync(ids, L.ids, L.count * 8, cudaMemcpyDeviceToHost, st));
        ix->order.release(st);
        RBE_CK(cudaStreamSynchronize(st));
    });
}

int rbe_cuda_index_destroy(rbe_cuda_index* ix) {
    return guarded([&] { delete ix; });
}

int rbe_cuda_index_bytes(const rbe_cuda_index* ix, uint64_t* device_bytes, uint64_t* scan_bytes) {
    return guarded([&] {
        if (!ix) throw InvalidArgument("rbe_cuda_index_bytes: null index");
        if (device_bytes) *device_bytes = ix->store.bytes;
        if (scan_bytes) *scan_bytes = ix->total * (uint64_t(ix->shape.kp) * ix->shape.wpp * 8 + 4);
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
        ix->order.acquire(st);
        const size_t qbytes = size_t(n_queries) * query_planes * ix->shape.wpp * 8;
        ix->queries.ensure(qbytes);
        RBE_CK(cudaMemcpyAsync(ix->queries.p, d_query_words, qbytes, cudaMemcpyDeviceToDevice, st));
        const Pending pd = enqueue_batch(ix, st, n_queries, query_planes, geometry, n, options);
        RBE_CK(cudaMemcpyAsync(d_out, ix->out.p, sizeof(Result) * n_queries * n, cudaMemcpyDeviceToDevice, st));
        ix->order.release(st);
        if (stats) finish_batch(ix, st, pd, stats);
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
        cudaStream_t st = ix->stream;
        ix->order.acquire(st);
        const size_t qbytes = size_t(n_queries) * query_planes * ix->shape.wpp * 8;
        ix->queries.ensure(qbytes);
        RBE_CK(cudaMemcpyAsync(ix->queries.p, query_words, qbytes, cudaMemcpyHostToDevice, st));
        const Pending pd = enqueue_batch(ix, st, n_queries, query_planes, geometry, n, options);
        // without stats the batch runs with a single host synchronisation (inside deliver)
        deliver(ix, ix->out.as<Result>(), n_queries, n, HostOut{scores, ids, partitions, accs, counts}, st);
        ix->order.release(st);
        if (stats) finish_batch(ix, st, pd, stats);
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
        // surface an accumulator-recovery failure of any batch enqueued without stats
        check_sticky_sync(ix, ix->stream);
        float ms = 0;
        RBE_CK(cudaEventElapsedTime(&ms, ix->ev[1], ix->ev[2]));
        if (scan_ms) *scan_ms = ms;
        RBE_CK(cudaEventElapsedTime(&ms, ix->ev[0], ix->ev[3]));
        if (total_ms) *total_ms = ms;
    });
}

int rbe_cuda_index_check(rbe_cuda_index* ix) {
    return guarded([&] {
        if (!ix) throw InvalidArgument("rbe_cuda_index_check: null index");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        if (ix->order.used) RBE_CK(cudaEventSynchronize(ix->order.done));
        check_sticky_sync(ix, ix->stream);
    });
}

int rbe_cuda_index_inject_error(rbe_cuda_index* ix) {
    return guarded([&] {
        if (!ix) throw InvalidArgument("rbe_cuda_index_inject_error: null index");
        std::lock_guard<std::mutex> lk(ix->mu);
        DeviceGuard dg(ix->device);
        const uint32_t one = 1;
        RBE_CK(cudaMemcpyAsync(ix->sticky.p, &one, 4, cudaMemcpyHostToDevice, ix->stream));
        RBE_CK(cudaStreamSynchronize(ix->stream));
    });
}

int rbe_cuda_merge_device(int device, const rbe_result* d_in, uint32_t n_lists, uint32_t n_queries, uint64_t n,
                          rbe_result* d_out, void* stream) {
    return guarded([&] {
        check_device_usable(device);
        if (n_queries == 0 || n == 0) return;
        if (!d_in || !d_out) throw InvalidArgument("rbe_cuda_merge_device: null buffer");
        if (n_lists == 0) throw InvalidArgument("rbe_cuda_merge_device: need at least one list");
        DeviceCtx& c = device_ctx(device);
        std::lock_guard<std::mutex> lk(c.mu);
        DeviceGuard dg(device);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c.stream;
        c.order.acquire(st);
        enqueue_merge(reinterpret_cast<const Result*>(d_in), n_lists, n_queries, n, reinterpret_cast<Result*>(d_out),
                      c.tmp, c.cnt, c.scr, st);
        c.order.release(st);
    });
}

int rbe_cuda_select_topn(int device, const double* scores, const uint64_t* ids, uint64_t count, uint32_t partition,
                         uint64_t n, double* out_scores, uint64_t* out_ids, uint64_t* out_count) {
    return guarded([&] {
        check_device_usable(device);
        if (!out_count) throw InvalidArgument("rbe_cuda_select_topn: null output");
        *out_count = 0;
        if (n == 0 || count == 0) return;
        if (!scores || !ids || !out_scores || !out_ids) throw InvalidArgument("rbe_cuda_select_topn: null buffer");
        DeviceCtx& c = device_ctx(device);
        std::lock_guard<std::mutex> lk(c.mu);
        DeviceGuard dg(device);
        cudaStream_t st = c.stream;
        c.order.acquire(st);
        std::vector<Result> recs(count);
        for (uint64_t i = 0; i < count; ++i) recs[i] = Result{scores[i], ids[i], 0, partition, 1u};
        const uint64_t m = std::min<uint64_t>(n, count);
        c.io.ensure(sizeof(Result) * (count + m) + sizeof(unsigned long long));
        Result* d_in = c.io.as<Result>();
        Result* d_out = d_in + count;
        unsigned long long* d_cnt = reinterpret_cast<unsigned long long*>(d_out + m);
        const unsigned long long cnt = count;
        RBE_CK(cudaMemcpyAsync(d_in, recs.data(), sizeof(Result) * count, cudaMemcpyHostToDevice, st));
        RBE_CK(cudaMemcpyAsync(d_cnt, &cnt, sizeof(cnt), cudaMemcpyHostToDevice, st));
        const size_t ss = select_scratch_bytes(1, count, m);
        c.scr.ensure(ss);
        launch_select_topn(d_in, d_cnt, count, 1, m, d_out, c.scr.p, ss, st);
        std::vector<Result> res(m);
        RBE_CK(cudaMemcpyAsync(res.data(), d_out, sizeof(Result) * m, cudaMemcpyDeviceToHost, st));
        c.order.release(st);
        RBE_CK(cudaStreamSynchronize(st));
        uint64_t k = 0;
        for (; k < m && res[k].valid; ++k) {
            out_scores[k] = res[k].score;
            out_ids[k] = res[k].id;
        }
        *out_count = k;
    });
}

int rbe_cuda_local_select(rbe_cuda_index* ix, uint32_t i, const uint64_t* query_words, uint32_t query_planes,
                          const rbe_scan_geometry* geometry, double* scores, uint64_t* slots, uint32_t* counts,
                          uint64_t* scored) {
    return guarded([&] {
        if (!ix || !geometry) throw InvalidArgument("rbe_cuda_local_select: null argument");
        std::lock_guard<std::mutex> lk(ix->mu);
        if (i >= ix->parts.size()) throw OutOfRange("rbe_cuda_local_select: partition out of range");
        DeviceGuard dg(ix->device);
        if (query_planes == 0) throw InvalidArgument("local_select: query dimension mismatch");
        if (geometry->queue_length == 0) throw InvalidArgument("local_select: queue_length must be positive");
        const auto& L = ix->parts[i];
        if (uint64_t(geometry->blocks) * geometry->threads_per_block * geometry->items_per_thread < L.count)
            throw InvalidArgument("local_select: geometry does not cover partition");
        if (uint64_t(query_planes) * ix->shape.kp > 64) throw InvalidArgument("local_select: too many planes");
        if (!query_words || !scores || !slots || !counts) throw InvalidArgument("rbe_cuda_local_select: null buffer");
        const Shape& s = ix->shape;
        cudaStream_t st = ix->stream;
        ix->order.acquire(st);
        ScanArgs a;
        a.parts = ix->d_parts.as<PartDesc>() + i;
        a.n_parts = 1;
        a.blocks = geometry->blocks;
        a.tpb = geometry->threads_per_block;
        a.ipt = geometry->items_per_thread;
        a.ql = geometry->queue_length;
        a.Q = 1;
        a.qp = query_planes;
        const uint64_t threads = uint64_t(a.blocks) * a.tpb;
        const uint64_t ql_eff = std::min<uint64_t>(a.ql, a.ipt);
        const size_t qbytes = size_t(query_planes) * s.wpp * 8;
        ix->queries.ensure(qbytes);
        RBE_CK(cudaMemcpyAsync(ix->queries.p, query_words, qbytes, cudaMemcpyHostToDevice, st));
        ix->counters.ensure(64);
        RBE_CK(cudaMemsetAsync(ix->counters.p, 0, 64, st));
        a.scored = ix->counters.as<unsigned long long>();
        a.overflow = reinterpret_cast<unsigned int*>(a.scored + 2);
        a.error = ix->sticky.as<unsigned int>();
        const size_t lbytes = threads * ql_eff * 16 + threads * 4;
        ix->surv.ensure(lbytes + 256);
        a.list_scores = ix->surv.as<double>();
        a.list_slots = reinterpret_cast<uint64_t*>(a.list_scores + threads * ql_eff);
        a.list_counts = reinterpret_cast<uint32_t*>(a.list_slots + threads * ql_eff);
        ix->qperm.ensure(sizeof(uint32_t) * size_t(s.kp) * query_planes * s.w32);
        launch_prepare_queries_exact(ix->queries.as<uint64_t>(), ix->qperm.as<uint32_t>(), 1, query_planes, s, ix->perm,
                                     st);
        const size_t qs = exact_queue_scratch_bytes(a);
        ix->queue_scratch.ensure(qs);
        launch_scan_exact(a, s, ix->qperm.as<uint32_t>(), qs ? ix->queue_scratch.p : nullptr, st);
        RBE_CK(cudaMemcpyAsync(scores, a.list_scores, threads * ql_eff * 8, cudaMemcpyDeviceToHost, st));
        RBE_CK(cudaMemcpyAsync(slots, a.list_slots, threads * ql_eff * 8, cudaMemcpyDeviceToHost, st));
        RBE_CK(cudaMemcpyAsync(counts, a.list_counts, threads * 4, cudaMemcpyDeviceToHost, st));
        unsigned long long* hsc = reinterpret_cast<unsigned long long*>(ix->host_out);
        RBE_CK(cudaMemcpyAsync(hsc, a.scored, 8, cudaMemcpyDeviceToHost, st));
        ix->order.release(st);
        RBE_CK(cudaStreamSynchronize(st));
        if (scored) *scored = *hsc;
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
        // lock every handle for the whole call, in address order (no lock-order inversion)
        std::vector<rbe_cuda_index*> order(handles, handles + n_handles);
        for (auto* h : order)
            if (!h) throw InvalidArgument("rbe_cuda_search_multi: null handle");
        std::sort(order.begin(), order.end());
        if (std::adjacent_find(order.begin(), order.end()) != order.end())
            throw InvalidArgument("rbe_cuda_search_multi: a handle appears twice");
        std::vector<std::unique_lock<std::mutex>> locks;
        for (auto* h : order) locks.emplace_back(h->mu);
        // the reference rejects only an index whose total is empty (search.cpp:133-135);
        // handles without documents take no part in the scan
        uint64_t total = 0;
        for (uint32_t h = 0; h < n_handles; ++h) total += handles[h]->total;
        if (total == 0) throw InvalidArgument("search: empty index");
        std::vector<rbe_cuda_index*> act;
        for (uint32_t h = 0; h < n_handles; ++h) {
            validate_shape(handles[h], query_planes, geometry);
            if (handles[h]->total) act.push_back(handles[h]);
        }
        if (n_queries == 0) return;
        if (n == 0) {
            if (counts) std::fill(counts, counts + n_queries, 0);
            if (stats) *stats = rbe_search_stats{};
            return;
        }
        if (!query_words || !scores || !ids || !partitions || !counts)
            throw InvalidArgument("rbe_cuda_search_multi: null buffer");
        const size_t cells = size_t(n_queries) * n;
        const size_t list_bytes = sizeof(Result) * cells;
        const size_t qbytes = size_t(n_queries) * query_planes * act[0]->shape.wpp * 8;
        // 1. every device scans its partitions, concurrently: all batches are enqueued on
        //    their handle's own stream before anything waits
        std::vector<Pending> pend(act.size());
        for (size_t h = 0; h < act.size(); ++h) {
            rbe_cuda_index* ix = act[h];
            DeviceGuard dg(ix->device);
            cudaStream_t st = ix->stream;
            ix->order.acquire(st);
            ix->queries.ensure(qbytes);
            RBE_CK(cudaMemcpyAsync(ix->queries.p, query_words, qbytes, cudaMemcpyHostToDevice, st));
            pend[h] = enqueue_batch(ix, st, n_queries, query_planes, geometry, n, options);
            ix->order.release(st);  // records the end of this handle's batch
        }
        // 2. the root gathers the lists peer-to-peer (after each handle's batch event) and merges
        rbe_cuda_index* root = act[0];
        const Result* merged_list = nullptr;
        {
            DeviceGuard dg(root->device);
            cudaStream_t st = root->stream;
            root->gathered.ensure(list_bytes * act.size());
            root->merged.ensure(list_bytes);
            for (size_t h = 0; h < act.size(); ++h) {
                char* dst = static_cast<char*>(root->gathered.p) + h * list_bytes;
                if (h) RBE_CK(cudaStreamWaitEvent(st, act[h]->order.done, 0));
                RBE_CK(cudaMemcpyPeerAsync(dst, root->device, act[h]->out.p, act[h]->device, list_bytes, st));
            }
            if (act.size() > 1) {
                enqueue_merge(root->gathered.as<Result>(), uint32_t(act.size()), n_queries, n, root->merged.as<Result>(),
                              root->mtmp, root->mcnt, root->mscr, st);
                merged_list = root->merged.as<Result>();
            } else {
                merged_list = root->gathered.as<Result>();
            }
            deliver(root, merged_list, n_queries, n, HostOut{scores, ids, partitions, accs, counts}, st);
            root->order.release(st);  // root's scratch was used on its stream after its batch
        }
        // 3. the other handles: their batches are complete (the root waited on them); read
        //    their sticky flags (and stats)
        rbe_search_stats tot{};
        for (size_t h = 0; h < act.size(); ++h) {
            rbe_cuda_index* ix = act[h];
            DeviceGuard dg(ix->device);
            rbe_search_stats s{};
            finish_batch(ix, ix->stream, pend[h], &s);
            tot.scored += s.scored;
            tot.candidates += s.candidates;
            tot.survivors += s.survivors;
            tot.variant = s.variant;
            tot.fallback |= s.fallback;
            tot.launches += s.launches;
            tot.scan_ms = std::max(tot.scan_ms, s.scan_ms);
            tot.total_ms = std::max(tot.total_ms, s.total_ms);
        }
        if (act.size() > 1) tot.launches += 2;  // gather + merge select on the root
        if (stats) *stats = tot;
    });
}

}  // extern "C"
