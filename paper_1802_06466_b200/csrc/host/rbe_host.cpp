// rbe_host.cpp -- the host side of the drop-in rbe:: API (include/rbe/*.hpp).
// Index building, RBEI I/O and the small single-pair helpers are host code as
// in the reference (src/binary_vector.cpp, src/embedding.cpp, src/index.cpp);
// every retrieval (search, search_batch) goes through the C ABI of
// include/rbe_cuda.h onto the B200.  Error types and messages follow the
// reference so callers (and the Python layer) see the same exceptions.
#include <algorithm>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>

#include "rbe/binary_vector.hpp"
#include "rbe/embedding.hpp"
#include "rbe/index.hpp"
#include "rbe/search.hpp"
#include "rbe_cuda.h"

namespace rbe {

// ------------------------------------------------------------ binary vectors
PackedBinaryVector pack(std::span<const int> values) {
    if (values.empty()) throw std::invalid_argument("pack: empty input");
    PackedBinaryVector v;
    v.dim = uint32_t(values.size());
    v.words.resize(PackedBinaryVector::words_for(v.dim));
    for (size_t i = 0; i < values.size(); ++i) {
        const int x = values[i];
        if (x != 1 && x != -1) throw std::invalid_argument("pack: values must be -1 or +1");
        v.words[i >> 6] |= uint64_t(x == 1) << (i & 63);
    }
    return v;
}

std::vector<int> unpack(const PackedBinaryVector& v) {
    std::vector<int> out;
    out.reserve(v.dim);
    for (uint32_t i = 0; i < v.dim; ++i) out.push_back(((v.words[i >> 6] >> (i & 63)) & 1u) ? 1 : -1);
    return out;
}

int64_t binary_dot(const PackedBinaryVector& x, const PackedBinaryVector& y) {
    if (x.dim != y.dim) throw std::invalid_argument("binary_dot: dimension mismatch");
    return binary_dot_words(x.words.data(), y.words.data(), x.words.size(), x.dim);
}

// ------------------------------------------------------------ embeddings
std::vector<double> refined_vector(const RbeEmbedding& e, bool residual_weights) {
    if (e.planes.empty()) throw std::invalid_argument("refined_vector: embedding has no planes");
    const uint32_t dim = e.planes[0].dim;
    std::vector<double> r(dim, 0.0);
    double w = 1.0;
    for (const PackedBinaryVector& p : e.planes) {
        if (p.dim != dim) throw std::invalid_argument("refined_vector: plane dim mismatch");
        for (uint32_t i = 0; i < dim; ++i) r[i] += ((p.words[i >> 6] >> (i & 63)) & 1u) ? w : -w;
        if (residual_weights) w *= 0.5;  // exact: 2^-t
    }
    return r;
}

RbeEmbedding make_embedding(std::vector<PackedBinaryVector> planes, bool residual_weights) {
    RbeEmbedding e;
    e.planes = std::move(planes);
    double sq = 0.0;
    for (double x : refined_vector(e, residual_weights)) sq += x * x;
    e.magnitude = std::sqrt(sq);
    return e;
}

int64_t combine_plane_dots_scaled(const int64_t* dots, uint32_t qp, uint32_t kp, bool residual_weights) {
    // two's-complement (mod 2^64) arithmetic, like the reference's shifts
    uint64_t acc = 0;
    if (!residual_weights) {
        for (uint32_t i = 0; i < qp * kp; ++i) acc += uint64_t(dots[i]);
        return int64_t(acc);
    }
    // pair (s, t) carries 2^(L - s - t), L = qp + kp - 2: identical to the
    // Horner-over-levels integer of the reference (exact integer arithmetic).
    const uint32_t L = qp + kp - 2;
    for (uint32_t s = 0; s < qp; ++s)
        for (uint32_t t = 0; t < kp; ++t) acc += uint64_t(dots[s * kp + t]) << (L - s - t);
    return int64_t(acc);
}

double combine_plane_dots(const int64_t* dots, uint32_t qp, uint32_t kp, bool residual_weights) {
    const int64_t acc = combine_plane_dots_scaled(dots, qp, kp, residual_weights);
    return residual_weights ? std::ldexp(double(acc), -int(qp + kp - 2)) : double(acc);
}

double rbe_score(const RbeEmbedding& q, const RbeEmbedding& k, const SimilarityConfig& cfg) {
    if (q.planes.size() != cfg.query_planes || k.planes.size() != cfg.keyword_planes)
        throw std::invalid_argument("rbe_score: plane count does not match config");
    if (q.dim() != k.dim()) throw std::invalid_argument("rbe_score: dimension mismatch");
    if (!(k.magnitude > 0.0)) throw std::invalid_argument("rbe_score: zero keyword magnitude");
    if (cfg.query_planes * cfg.keyword_planes > 64) throw std::invalid_argument("rbe_score: too many planes");
    std::vector<int64_t> dots(size_t(cfg.query_planes) * cfg.keyword_planes);
    for (uint32_t s = 0; s < cfg.query_planes; ++s)
        for (uint32_t t = 0; t < cfg.keyword_planes; ++t)
            dots[s * cfg.keyword_planes + t] = binary_dot(q.planes[s], k.planes[t]);
    double score = combine_plane_dots(dots.data(), cfg.query_planes, cfg.keyword_planes, cfg.residual_weights) /
                   k.magnitude;
    if (cfg.normalize_query) {
        if (!(q.magnitude > 0.0)) throw std::invalid_argument("rbe_score: zero query magnitude");
        score /= q.magnitude;
    }
    return score;
}

// ------------------------------------------------------------ keyword index
uint64_t KeywordIndex::total_keywords() const {
    uint64_t n = 0;
    for (const Partition& p : partitions) n += p.count;
    return n;
}

uint64_t KeywordIndex::plane_bytes_per_keyword() const { return uint64_t(keyword_planes) * words_per_plane() * 8; }

uint64_t KeywordIndex::plane_payload_bytes() const {
    uint64_t b = 0;
    for (const Partition& p : partitions)
        for (const auto& blk : p.plane_blocks) b += blk.size() * sizeof(uint64_t);
    return b;
}

IndexBuilder::IndexBuilder(uint32_t partition_count, bool residual_weights) {
    if (partition_count == 0) throw std::invalid_argument("IndexBuilder: need at least one partition");
    index_.residual_weights = residual_weights;
    index_.partitions.resize(partition_count);
}

void IndexBuilder::add(uint64_t id, const RbeEmbedding& embedding) {
    if (embedding.planes.empty()) throw std::invalid_argument("IndexBuilder: embedding has no planes");
    if (added_ == 0) {
        index_.dim = embedding.dim();
        index_.keyword_planes = uint32_t(embedding.planes.size());
        for (Partition& p : index_.partitions) p.plane_blocks.resize(index_.keyword_planes);
    } else if (embedding.dim() != index_.dim || embedding.planes.size() != index_.keyword_planes) {
        throw std::invalid_argument("IndexBuilder: inconsistent dim or plane count in stream");
    }
    ids_.push_back(id);
    Partition& part = index_.partitions[added_ % index_.partitions.size()];
    for (uint32_t t = 0; t < index_.keyword_planes; ++t) {
        const auto& w = embedding.planes[t].words;
        part.plane_blocks[t].insert(part.plane_blocks[t].end(), w.begin(), w.end());
    }
    double mag = embedding.magnitude;
    if (!(mag > 0.0)) mag = make_embedding(embedding.planes, index_.residual_weights).magnitude;
    if (!(mag > 0.0)) throw std::invalid_argument("IndexBuilder: keyword has zero magnitude");
    part.magnitudes.push_back(float(mag));
    part.ids.push_back(id);
    ++part.count;
    ++added_;
}

KeywordIndex IndexBuilder::finish() {
    std::vector<uint64_t> sorted = ids_;
    std::sort(sorted.begin(), sorted.end());
    if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
        throw std::invalid_argument("IndexBuilder: duplicate keyword id");
    return std::move(index_);
}

KeywordIndex build_index(std::span<const std::pair<uint64_t, RbeEmbedding>> embeddings, uint32_t partition_count,
                         bool residual_weights) {
    IndexBuilder b(partition_count, residual_weights);
    for (const auto& [id, e] : embeddings) b.add(id, e);
    return b.finish();
}

RbeEmbedding index_entry(const KeywordIndex& index, uint32_t partition, uint64_t slot) {
    const Partition& p = index.partitions.at(partition);
    if (slot >= p.count) throw std::out_of_range("index_entry: slot out of range");
    const size_t wpp = index.words_per_plane();
    std::vector<PackedBinaryVector> planes(index.keyword_planes);
    for (uint32_t t = 0; t < index.keyword_planes; ++t) {
        planes[t].dim = index.dim;
        const uint64_t* src = p.plane_blocks[t].data() + slot * wpp;
        planes[t].words.assign(src, src + wpp);
    }
    RbeEmbedding e = make_embedding(std::move(planes), index.residual_weights);
    e.magnitude = double(p.magnitudes[slot]);
    return e;
}

// RBEI v1: "RBEI", u32 version, u32 dim, u32 kp, u32 rw, u32 P, u64 count[P],
// then per partition: plane blocks (u64 LE), f32 magnitudes, u64 ids.  The
// host is little-endian (x86-64 / aarch64), so blocks move with bulk I/O.
static_assert(std::endian::native == std::endian::little, "RBEI bulk I/O assumes a little-endian host");

namespace {
constexpr char kMagic[4] = {'R', 'B', 'E', 'I'};
constexpr uint32_t kVersion = 1;

template <typename T>
void put(std::ofstream& f, const T* p, size_t n) {
    f.write(reinterpret_cast<const char*>(p), std::streamsize(n * sizeof(T)));
}
template <typename T>
void get(std::ifstream& f, T* p, size_t n) {
    f.read(reinterpret_cast<char*>(p), std::streamsize(n * sizeof(T)));
}
}  // namespace

void save_index(const KeywordIndex& index, const std::filesystem::path& path) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open index for writing: " + path.string());
    f.write(kMagic, 4);
    const uint32_t hdr[5] = {kVersion, index.dim, index.keyword_planes, index.residual_weights ? 1u : 0u,
                             uint32_t(index.partitions.size())};
    put(f, hdr, 5);
    for (const Partition& p : index.partitions) put(f, &p.count, 1);
    for (const Partition& p : index.partitions) {
        for (const auto& blk : p.plane_blocks) put(f, blk.data(), blk.size());
        put(f, p.magnitudes.data(), p.magnitudes.size());
        put(f, p.ids.data(), p.ids.size());
    }
    if (!f) throw std::runtime_error("failed writing index: " + path.string());
}

KeywordIndex load_index(const std::filesystem::path& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open index: " + path.string());
    char magic[4];
    f.read(magic, 4);
    if (!f || std::memcmp(magic, kMagic, 4) != 0) throw std::runtime_error("not an RBEI index file: " + path.string());
    uint32_t version = 0;
    get(f, &version, 1);
    if (version != kVersion) throw std::runtime_error("unsupported index version");
    uint32_t hdr[4] = {};
    get(f, hdr, 4);
    KeywordIndex index;
    index.dim = hdr[0];
    index.keyword_planes = hdr[1];
    index.residual_weights = hdr[2] != 0;
    index.partitions.resize(hdr[3]);
    for (Partition& p : index.partitions) get(f, &p.count, 1);
    const size_t wpp = index.words_per_plane();
    for (Partition& p : index.partitions) {
        if (!f) break;
        p.plane_blocks.assign(index.keyword_planes, {});
        for (auto& blk : p.plane_blocks) {
            blk.resize(p.count * wpp);
            get(f, blk.data(), blk.size());
        }
        p.magnitudes.resize(p.count);
        get(f, p.magnitudes.data(), p.count);
        p.ids.resize(p.count);
        get(f, p.ids.data(), p.count);
    }
    if (!f) throw std::runtime_error("truncated index file: " + path.string());
    return index;
}

// ------------------------------------------------------------ search
std::vector<uint64_t> thread_assignment(const ScanGeometry& g, uint64_t count, uint32_t block, uint32_t thread) {
    if (block >= g.blocks || thread >= g.threads_per_block)
        throw std::invalid_argument("thread_assignment: block or thread out of range");
    std::vector<uint64_t> items;
    const uint64_t base = uint64_t(block) * g.threads_per_block * g.items_per_thread + thread;
    for (uint32_t i = 0; i < g.items_per_thread; ++i) {
        const uint64_t z = base + uint64_t(i) * g.threads_per_block;
        if (z < count) items.push_back(z);
    }
    return items;
}

namespace {

[[noreturn]] void raise(int status) {
    const std::string msg = rbe_cuda_last_error();
    if (status == RBE_CUDA_EINVAL) throw std::invalid_argument(msg);
    if (status == RBE_CUDA_ERANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
}

void ck(int status) {
    if (status != RBE_CUDA_OK) raise(status);
}

}  // namespace

void DeviceIndex::Deleter::operator()(rbe_cuda_index* p) const { rbe_cuda_index_destroy(p); }

DeviceIndex::~DeviceIndex() = default;
DeviceIndex::DeviceIndex(DeviceIndex&&) noexcept = default;
DeviceIndex& DeviceIndex::operator=(DeviceIndex&&) noexcept = default;

DeviceIndex::DeviceIndex(const KeywordIndex& index, std::vector<int> devices) {
    if (devices.empty()) throw std::invalid_argument("DeviceIndex: need at least one device");
    devices_ = devices;
    dim_ = index.dim;
    kp_ = index.keyword_planes;
    rw_ = index.residual_weights;
    partitions_ = uint32_t(index.partitions.size());
    const rbe_index_shape shape{index.dim, index.keyword_planes, index.residual_weights ? 1u : 0u};
    const size_t wpp = index.words_per_plane();
    for (size_t d = 0; d < devices.size(); ++d) {
        std::vector<uint32_t> ords;
        std::vector<uint64_t> counts;
        for (uint32_t p = uint32_t(d); p < partitions_; p += uint32_t(devices.size())) {
            ords.push_back(p);
            counts.push_back(index.partitions[p].count);
        }
        rbe_cuda_index* h = nullptr;
        ck(rbe_cuda_index_create(&shape, uint32_t(ords.size()), ords.data(), counts.data(), devices[d], &h));
        handles_.emplace_back(h);
        part_handle_.resize(partitions_, -1);
        part_local_.resize(partitions_, 0);
        part_count_.resize(partitions_, 0);
        for (size_t i = 0; i < ords.size(); ++i) {
            part_handle_[ords[i]] = int(d);
            part_local_[ords[i]] = uint32_t(i);
            part_count_[ords[i]] = counts[i];
        }
        for (size_t i = 0; i < ords.size(); ++i) {
            const Partition& part = index.partitions[ords[i]];
            if (part.count == 0) continue;
            if (part.plane_blocks.size() != kp_ || part.magnitudes.size() != part.count || part.ids.size() != part.count)
                throw std::invalid_argument("DeviceIndex: partition arrays inconsistent with count");
            std::vector<uint64_t> planes;
            planes.reserve(size_t(kp_) * part.count * wpp);
            for (const auto& blk : part.plane_blocks) {
                if (blk.size() != part.count * wpp)
                    throw std::invalid_argument("DeviceIndex: plane block size inconsistent with count");
                planes.insert(planes.end(), blk.begin(), blk.end());
            }
            ck(rbe_cuda_index_upload_partition(h, uint32_t(i), planes.data(), part.magnitudes.data(), part.ids.data()));
        }
        for (uint64_t c : counts) {
            total_ += c;
            max_count_ = std::max(max_count_, c);
        }
    }
}

DeviceIndex DeviceIndex::synthetic(uint32_t dim, uint32_t kp, bool rw, uint64_t n_docs, uint32_t partitions,
                                   uint64_t seed, std::vector<int> devices, uint32_t rank, uint32_t world) {
    if (partitions == 0) throw std::invalid_argument("IndexBuilder: need at least one partition");
    if (devices.empty() || world == 0 || rank >= world) throw std::invalid_argument("DeviceIndex: bad device layout");
    DeviceIndex ix;
    ix.devices_ = devices;
    ix.dim_ = dim;
    ix.kp_ = kp;
    ix.rw_ = rw;
    ix.partitions_ = partitions;
    const rbe_index_shape shape{dim, kp, rw ? 1u : 0u};
    const uint32_t G = uint32_t(devices.size()) * world;
    for (size_t d = 0; d < devices.size(); ++d) {
        const uint32_t slot = rank * uint32_t(devices.size()) + uint32_t(d);
        std::vector<uint32_t> ords;
        std::vector<uint64_t> counts;
        for (uint32_t p = slot; p < partitions; p += G) {
            ords.push_back(p);
            counts.push_back(p < n_docs ? (n_docs - p + partitions - 1) / partitions : 0);
        }
        rbe_cuda_index* h = nullptr;
        ck(rbe_cuda_index_create(&shape, uint32_t(ords.size()), ords.data(), counts.data(), devices[d], &h));
        ix.handles_.emplace_back(h);
        ix.part_handle_.resize(partitions, -1);
        ix.part_local_.resize(partitions, 0);
        ix.part_count_.resize(partitions, 0);
        for (size_t i = 0; i < ords.size(); ++i) {
            ix.part_handle_[ords[i]] = int(d);
            ix.part_local_[ords[i]] = uint32_t(i);
            ix.part_count_[ords[i]] = counts[i];
        }
        ck(rbe_cuda_index_fill_synthetic(h, seed, n_docs, partitions));
        for (uint64_t c : counts) {
            ix.total_ += c;
            ix.max_count_ = std::max(ix.max_count_, c);
        }
    }
    return ix;
}

DeviceIndex DeviceIndex::from_rbei(const std::string& path, std::vector<int> devices, uint32_t io_threads,
                                   LoadStats* stats) {
    if (devices.empty()) throw std::invalid_argument("DeviceIndex: need at least one device");
    const auto t0 = std::chrono::steady_clock::now();
    rbe_index_shape shape{};
    uint32_t P = 0;
    ck(rbe_cuda_rbei_header(path.c_str(), &shape, &P, nullptr, 0));
    std::vector<uint64_t> counts(P);
    ck(rbe_cuda_rbei_header(path.c_str(), &shape, &P, counts.data(), P));
    DeviceIndex ix;
    ix.devices_ = devices;
    ix.dim_ = shape.dim;
    ix.kp_ = shape.keyword_planes;
    ix.rw_ = shape.residual_weights != 0;
    ix.partitions_ = P;
    ix.part_handle_.assign(P, -1);
    ix.part_local_.assign(P, 0);
    ix.part_count_.assign(P, 0);
    const size_t G = devices.size();
    std::vector<std::vector<uint32_t>> ords(G);
    for (uint32_t p = 0; p < P; ++p) ords[p % G].push_back(p);
    // one loader thread per device; the host threads reading the file are split among them
    const uint32_t per_dev = io_threads ? std::max<uint32_t>(1, io_threads / uint32_t(G))
                                        : std::max<uint32_t>(1, std::min<uint32_t>(16, std::thread::hardware_concurrency()) /
                                                                    uint32_t(G));
    std::vector<rbe_cuda_index*> raw(G, nullptr);
    std::vector<rbe_load_stats> st(G, rbe_load_stats{0, 0.0});
    std::vector<int> rc(G, RBE_CUDA_OK);
    std::vector<std::string> err(G);
    std::vector<std::thread> pool;
    for (size_t d = 0; d < G; ++d)
        pool.emplace_back([&, d] {
            // a device without partitions gets an empty handle (n = 0 would mean "all partitions")
            rc[d] = ords[d].empty()
                        ? rbe_cuda_index_create(&shape, 0, nullptr, nullptr, devices[d], &raw[d])
                        : rbe_cuda_index_open_rbei(path.c_str(), ords[d].data(), uint32_t(ords[d].size()), devices[d],
                                                   per_dev, &raw[d], &st[d]);
            if (rc[d] != RBE_CUDA_OK) err[d] = rbe_cuda_last_error();
        });
    for (auto& t : pool) t.join();
    for (size_t d = 0; d < G; ++d) ix.handles_.emplace_back(raw[d]);  // owned (destroyed on error too)
    for (size_t d = 0; d < G; ++d)
        if (rc[d] != RBE_CUDA_OK) {
            if (rc[d] == RBE_CUDA_EINVAL) throw std::invalid_argument(err[d]);
            if (rc[d] == RBE_CUDA_ERANGE) throw std::out_of_range(err[d]);
            throw std::runtime_error(err[d]);
        }
    uint64_t bytes = 0;
    for (size_t d = 0; d < G; ++d) {
        bytes += st[d].file_bytes_read;
        for (size_t i = 0; i < ords[d].size(); ++i) {
            const uint32_t p = ords[d][i];
            ix.part_handle_[p] = int(d);
            ix.part_local_[p] = uint32_t(i);
            ix.part_count_[p] = counts[p];
            ix.total_ += counts[p];
            ix.max_count_ = std::max(ix.max_count_, counts[p]);
        }
    }
    if (stats) {
        stats->file_bytes = bytes;
        stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    return ix;
}

DeviceIndex DeviceIndex::build_rbee(const std::string& path, uint32_t partitions, std::vector<int> devices,
                                    uint32_t io_threads, LoadStats* stats) {
    if (devices.empty()) throw std::invalid_argument("DeviceIndex: need at least one device");
    if (partitions == 0) throw std::invalid_argument("IndexBuilder: need at least one partition");
    const auto t0 = std::chrono::steady_clock::now();
    rbe_index_shape shape{};
    uint64_t n = 0;
    ck(rbe_cuda_rbee_header(path.c_str(), &shape, &n));
    DeviceIndex ix;
    ix.devices_ = devices;
    ix.dim_ = shape.dim;
    ix.kp_ = shape.keyword_planes;
    ix.rw_ = shape.residual_weights != 0;
    ix.partitions_ = partitions;
    ix.part_handle_.assign(partitions, -1);
    ix.part_local_.assign(partitions, 0);
    ix.part_count_.assign(partitions, 0);
    const size_t G = devices.size();
    std::vector<std::vector<uint32_t>> ords(G);
    for (uint32_t p = 0; p < partitions; ++p) ords[p % G].push_back(p);
    const uint32_t per_dev = std::max<uint32_t>(
        1, (io_threads ? io_threads : std::min<uint32_t>(16, std::thread::hardware_concurrency())) / uint32_t(G));
    std::vector<rbe_cuda_index*> raw(G, nullptr);
    std::vector<rbe_load_stats> st(G, rbe_load_stats{0, 0.0});
    std::vector<int> rc(G, RBE_CUDA_OK);
    std::vector<std::string> err(G);
    std::vector<std::thread> pool;
    for (size_t d = 0; d < G; ++d)
        pool.emplace_back([&, d] {
            rc[d] = ords[d].empty()
                        ? rbe_cuda_index_create(&shape, 0, nullptr, nullptr, devices[d], &raw[d])
                        : rbe_cuda_index_build_rbee(path.c_str(), partitions, ords[d].data(), uint32_t(ords[d].size()),
                                                    devices[d], per_dev, &raw[d], &st[d]);
            if (rc[d] != RBE_CUDA_OK) err[d] = rbe_cuda_last_error();
        });
    for (auto& t : pool) t.join();
    for (size_t d = 0; d < G; ++d) ix.handles_.emplace_back(raw[d]);
    for (size_t d = 0; d < G; ++d)
        if (rc[d] != RBE_CUDA_OK) {
            if (rc[d] == RBE_CUDA_EINVAL) throw std::invalid_argument(err[d]);
            if (rc[d] == RBE_CUDA_ERANGE) throw std::out_of_range(err[d]);
            throw std::runtime_error(err[d]);
        }
    uint64_t bytes = 0;
    std::vector<uint64_t> held(G, 0);
    for (size_t d = 0; d < G; ++d) {
        bytes = std::max<uint64_t>(bytes, st[d].file_bytes_read);
        for (size_t i = 0; i < ords[d].size(); ++i) {
            const uint32_t p = ords[d][i];
            const uint64_t c = p < n ? (n - p + partitions - 1) / partitions : 0;
            ix.part_handle_[p] = int(d);
            ix.part_local_[p] = uint32_t(i);
            ix.part_count_[p] = c;
            ix.total_ += c;
            ix.max_count_ = std::max(ix.max_count_, c);
            held[d] += c;
        }
    }
    // IndexBuilder::finish across handles: each handle checked its own ids; merge the sorted lists
    size_t with_ids = 0;
    for (uint64_t h : held) with_ids += h ? 1 : 0;
    if (with_ids > 1) {
        std::vector<uint64_t> all;
        all.reserve(ix.total_);
        for (size_t d = 0; d < G; ++d) {
            if (!held[d]) continue;
            std::vector<uint64_t> ids(held[d]);
            ck(rbe_cuda_index_sorted_ids(ix.handles_[d].get(), ids.data()));
            const size_t mid = all.size();
            all.insert(all.end(), ids.begin(), ids.end());
            std::inplace_merge(all.begin(), all.begin() + mid, all.end());
        }
        if (std::adjacent_find(all.begin(), all.end()) != all.end())
            throw std::invalid_argument("IndexBuilder: duplicate keyword id");
    }
    if (stats) {
        stats->file_bytes = bytes;
        stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    return ix;
}

void DeviceIndex::save_index(const std::string& path) const {
    for (int h : part_handle_)
        if (h < 0) throw std::out_of_range("save_index: not every partition is resident in this process");
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open index for writing: " + path);
    auto u32 = [&](uint32_t v) { out.write(reinterpret_cast<const char*>(&v), 4); };
    out.write("RBEI", 4);
    u32(1);
    u32(dim_);
    u32(kp_);
    u32(rw_ ? 1 : 0);
    u32(partitions_);
    for (uint32_t p = 0; p < partitions_; ++p) out.write(reinterpret_cast<const char*>(&part_count_[p]), 8);
    for (uint32_t p = 0; p < partitions_; ++p) {
        const Partition part = download_partition(p);
        for (const auto& blk : part.plane_blocks)
            out.write(reinterpret_cast<const char*>(blk.data()), std::streamsize(blk.size() * 8));
        out.write(reinterpret_cast<const char*>(part.magnitudes.data()), std::streamsize(part.count * 4));
        out.write(reinterpret_cast<const char*>(part.ids.data()), std::streamsize(part.count * 8));
    }
    if (!out) throw std::runtime_error("failed writing index: " + path);
}

uint64_t DeviceIndex::device_bytes() const {
    uint64_t t = 0;
    for (auto& h : handles_) {
        uint64_t b = 0;
        ck(rbe_cuda_index_bytes(h.get(), &b, nullptr));
        t += b;
    }
    return t;
}

uint64_t DeviceIndex::scan_bytes() const {
    uint64_t t = 0;
    for (auto& h : handles_) {
        uint64_t b = 0;
        ck(rbe_cuda_index_bytes(h.get(), nullptr, &b));
        t += b;
    }
    return t;
}

Partition DeviceIndex::download_partition(uint32_t partition) const {
    if (partition >= partitions_) throw std::out_of_range("download_partition: partition out of range");
    const int h = part_handle_[partition];
    if (h < 0) throw std::out_of_range("download_partition: partition not resident in this process");
    Partition p;
    p.count = part_count_[partition];
    const size_t wpp = PackedBinaryVector::words_for(dim_);
    std::vector<uint64_t> planes(size_t(kp_) * p.count * wpp);
    p.magnitudes.resize(p.count);
    p.ids.resize(p.count);
    ck(rbe_cuda_index_download_partition(handles_[h].get(), part_local_[partition], planes.data(), p.magnitudes.data(),
                                         p.ids.data()));
    p.plane_blocks.resize(kp_);
    for (uint32_t t = 0; t < kp_; ++t)
        p.plane_blocks[t].assign(planes.begin() + t * p.count * wpp, planes.begin() + (t + 1) * p.count * wpp);
    return p;
}

std::pair<size_t, uint32_t> DeviceIndex::locate(uint32_t partition) const {
    if (partition >= partitions_) throw std::out_of_range("partition out of range");
    const int h = part_handle_[partition];
    if (h < 0) throw std::out_of_range("partition not resident in this process");
    return {size_t(h), part_local_[partition]};
}

uint64_t DeviceIndex::partition_size(uint32_t partition) const {
    if (partition >= partitions_) throw std::out_of_range("partition out of range");
    return part_count_[partition];
}

std::vector<SelectionResult> DeviceIndex::search_words(std::span<const uint64_t> query_words, uint32_t n_queries,
                                                       uint32_t query_planes, const ScanGeometry& g, uint64_t n,
                                                       SearchStats* stats, ScanVariant variant, uint32_t probe_tiles,
                                                       std::vector<std::vector<int64_t>>* acc_out) const {
    const size_t wpp = PackedBinaryVector::words_for(dim_);
    if (query_words.size() != size_t(n_queries) * query_planes * wpp)
        throw std::invalid_argument("search: query buffer size does not match (Q, planes, dim)");
    const rbe_scan_geometry geo{g.blocks, g.threads_per_block, g.items_per_thread, g.queue_length};
    rbe_search_options opt{};
    opt.variant = uint32_t(variant);
    opt.probe_tiles = probe_tiles;
    const size_t cells = size_t(n_queries) * size_t(n);
    std::vector<SelectionResult> out(n_queries);
    std::vector<double> scores(cells);
    std::vector<uint64_t> ids(cells), counts(n_queries);
    std::vector<uint32_t> parts(cells);
    std::vector<int64_t> accs(cells);
    rbe_search_stats st{};
    std::vector<rbe_cuda_index*> hs;
    for (auto& h : handles_) hs.push_back(h.get());
    // one device: rbe_cuda_search; several devices in this process: each scans
    // its partitions, lists are copied peer-to-peer and merged on the first
    // device (rbe_cuda_search_multi).
    ck(rbe_cuda_search_multi(hs.data(), uint32_t(hs.size()), query_words.data(), n_queries, query_planes, &geo, n,
                             &opt, scores.data(), ids.data(), parts.data(), accs.data(), counts.data(), &st));
    if (acc_out) acc_out->assign(n_queries, {});
    for (uint32_t q = 0; q < n_queries; ++q) {
        auto& e = out[q].entries;
        e.resize(counts[q]);
        for (uint64_t k = 0; k < counts[q]; ++k) {
            const size_t o = size_t(q) * n + k;
            e[k] = SelectionEntry{scores[o], ids[o], parts[o]};
        }
        if (acc_out) (*acc_out)[q].assign(accs.begin() + size_t(q) * n, accs.begin() + size_t(q) * n + counts[q]);
    }
    if (stats) {
        stats->scored += st.scored;
        stats->variant = st.variant;
        stats->candidates += st.candidates;
        stats->survivors += st.survivors;
        stats->device_ms += st.total_ms;
    }
    return out;
}

void DeviceIndex::search_words_into(std::span<const uint64_t> query_words, uint32_t n_queries, uint32_t query_planes,
                                    const ScanGeometry& g, uint64_t n, double* scores, uint64_t* ids,
                                    uint32_t* partitions, int64_t* accs, uint64_t* counts, SearchStats* stats,
                                    ScanVariant variant, uint32_t probe_tiles) const {
    const size_t wpp = PackedBinaryVector::words_for(dim_);
    if (query_words.size() != size_t(n_queries) * query_planes * wpp)
        throw std::invalid_argument("search: query buffer size does not match (Q, planes, dim)");
    const rbe_scan_geometry geo{g.blocks, g.threads_per_block, g.items_per_thread, g.queue_length};
    rbe_search_options opt{};
    opt.variant = uint32_t(variant);
    opt.probe_tiles = probe_tiles;
    rbe_search_stats st{};
    std::vector<rbe_cuda_index*> hs;
    for (auto& h : handles_) hs.push_back(h.get());
    ck(rbe_cuda_search_multi(hs.data(), uint32_t(hs.size()), query_words.data(), n_queries, query_planes, &geo, n,
                             &opt, scores, ids, partitions, accs, counts, stats ? &st : nullptr));
    if (stats) {
        stats->scored += st.scored;
        stats->variant = st.variant;
        stats->candidates += st.candidates;
        stats->survivors += st.survivors;
        stats->device_ms += st.total_ms;
    }
}

namespace {

void check_query(const RbeEmbedding& q, uint32_t dim) {
    if (q.dim() != dim) throw std::invalid_argument("local_select: query dimension mismatch");
    for (const auto& p : q.planes)
        if (p.dim != dim || p.words.size() != PackedBinaryVector::words_for(dim))
            throw std::invalid_argument("local_select: query dimension mismatch");
}

std::vector<uint64_t> flatten(std::span<const RbeEmbedding> qs, uint32_t dim, uint32_t* qp) {
    std::vector<uint64_t> w;
    *qp = qs.empty() ? 1 : uint32_t(qs[0].planes.size());
    for (const RbeEmbedding& q : qs) {
        check_query(q, dim);
        if (q.planes.size() != *qp)
            throw std::invalid_argument("search_batch: all queries of a batch need the same plane count");
        for (const auto& p : q.planes) w.insert(w.end(), p.words.begin(), p.words.end());
    }
    return w;
}

}  // namespace

std::vector<std::vector<Candidate>> local_select(const RbeEmbedding& query, const DeviceIndex& index,
                                                 uint32_t partition, const ScanGeometry& geometry,
                                                 SearchStats* stats) {
    check_query(query, index.dim());
    const auto [h, local] = index.locate(partition);
    if (geometry.queue_length == 0) throw std::invalid_argument("local_select: queue_length must be positive");
    const uint64_t threads = uint64_t(geometry.blocks) * geometry.threads_per_block;
    const uint64_t ql = std::min<uint64_t>(geometry.queue_length, geometry.items_per_thread);
    std::vector<uint64_t> words;
    for (const auto& p : query.planes) words.insert(words.end(), p.words.begin(), p.words.end());
    std::vector<double> scores(threads * ql);
    std::vector<uint64_t> slots(threads * ql);
    std::vector<uint32_t> counts(threads);
    uint64_t scored = 0;
    const rbe_scan_geometry geo{geometry.blocks, geometry.threads_per_block, geometry.items_per_thread,
                                geometry.queue_length};
    ck(rbe_cuda_local_select(index.handle(h), local, words.data(), uint32_t(query.planes.size()), &geo,
                             scores.data(), slots.data(), counts.data(), &scored));
    std::vector<std::vector<Candidate>> lists(threads);
    for (uint64_t t = 0; t < threads; ++t) {
        lists[t].reserve(geometry.queue_length);
        for (uint32_t k = 0; k < counts[t]; ++k) lists[t].push_back(Candidate{scores[t * ql + k], slots[t * ql + k]});
    }
    if (stats) stats->scored += scored;
    return lists;
}

std::vector<std::vector<Candidate>> local_select(const RbeEmbedding& query, const KeywordIndex& index,
                                                 uint32_t partition, const ScanGeometry& geometry,
                                                 SearchStats* stats) {
    check_query(query, index.dim);
    if (geometry.queue_length == 0) throw std::invalid_argument("local_select: queue_length must be positive");
    const Partition& part = index.partitions.at(partition);
    if (geometry.capacity() < part.count) throw std::invalid_argument("local_select: geometry does not cover partition");
    // a one-partition device copy of just this partition (ordinal kept)
    KeywordIndex one;
    one.dim = index.dim;
    one.keyword_planes = index.keyword_planes;
    one.residual_weights = index.residual_weights;
    one.partitions.push_back(part);
    DeviceIndex dev(one, {0});
    return local_select(query, dev, 0, geometry, stats);
}

SelectionResult global_select(const std::vector<std::vector<Candidate>>& per_thread, const Partition& partition,
                              uint32_t partition_ordinal, uint64_t n) {
    std::vector<double> scores;
    std::vector<uint64_t> ids;
    for (const auto& list : per_thread)
        for (const Candidate& c : list) {
            scores.push_back(c.score);
            ids.push_back(partition.ids.at(c.slot));  // slot -> id (search.cpp:121-122)
        }
    SelectionResult r;
    if (scores.empty() || n == 0) return r;
    const uint64_t m = std::min<uint64_t>(n, scores.size());
    std::vector<double> os(m);
    std::vector<uint64_t> oi(m);
    uint64_t got = 0;
    ck(rbe_cuda_select_topn(0, scores.data(), ids.data(), scores.size(), partition_ordinal, n, os.data(), oi.data(),
                            &got));
    r.entries.resize(got);
    for (uint64_t k = 0; k < got; ++k) r.entries[k] = SelectionEntry{os[k], oi[k], partition_ordinal};
    return r;
}

std::vector<SelectionResult> search_batch(std::span<const RbeEmbedding> queries, const DeviceIndex& index,
                                          const ScanGeometry& geometry, uint64_t n, SearchStats* stats) {
    if (index.total_keywords() == 0) throw std::invalid_argument("search: empty index");
    uint32_t qp = 1;
    const std::vector<uint64_t> w = flatten(queries, index.dim(), &qp);
    return index.search_words(w, uint32_t(queries.size()), qp, geometry, n, stats);
}

SelectionResult search(const RbeEmbedding& query, const DeviceIndex& index, const ScanGeometry& geometry, uint64_t n,
                       SearchStats* stats) {
    if (index.total_keywords() == 0) throw std::invalid_argument("search: empty index");
    return search_batch(std::span<const RbeEmbedding>(&query, 1), index, geometry, n, stats).at(0);
}

namespace {

// The drop-in search(query, KeywordIndex, ...) keeps the device copy of the last
// index it saw, so a reference-style loop of per-query calls uploads once.  The
// KeywordIndex is immutable after build; the key is its shape plus
// the address, size and first/last words of every array, so a rebuilt or resized
// index is re-uploaded.
std::vector<uint64_t> fingerprint(const KeywordIndex& k) {
    std::vector<uint64_t> f{k.dim, k.keyword_planes, k.residual_weights ? 1u : 0u, k.partitions.size()};
    auto add = [&](const void* p, size_t n, uint64_t first, uint64_t last) {
        f.push_back(reinterpret_cast<uintptr_t>(p));
        f.push_back(n);
        f.push_back(first);
        f.push_back(last);
    };
    for (const Partition& p : k.partitions) {
        f.push_back(p.count);
        for (const auto& b : p.plane_blocks) add(b.data(), b.size(), b.empty() ? 0 : b.front(), b.empty() ? 0 : b.back());
        add(p.magnitudes.data(), p.magnitudes.size(), 0, 0);
        add(p.ids.data(), p.ids.size(), p.ids.empty() ? 0 : p.ids.front(), p.ids.empty() ? 0 : p.ids.back());
    }
    return f;
}

struct DropInCache {
    std::mutex mu;
    std::vector<uint64_t> key;
    std::shared_ptr<DeviceIndex> dev;
};
DropInCache& drop_in_cache() {
    static DropInCache* c = new DropInCache();  // process lifetime (no teardown-order races)
    return *c;
}

}  // namespace

SelectionResult search(const RbeEmbedding& query, const KeywordIndex& index, const ScanGeometry& geometry, uint64_t n,
                       SearchStats* stats) {
    if (index.partitions.empty() || index.total_keywords() == 0) throw std::invalid_argument("search: empty index");
    check_query(query, index.dim);
    std::shared_ptr<DeviceIndex> dev;
    {
        DropInCache& c = drop_in_cache();
        std::lock_guard<std::mutex> lk(c.mu);
        std::vector<uint64_t> key = fingerprint(index);
        if (!c.dev || c.key != key) {
            c.dev.reset();
            c.dev = std::make_shared<DeviceIndex>(index, std::vector<int>{0});
            c.key = std::move(key);
        }
        dev = c.dev;
    }
    return search(query, *dev, geometry, n, stats);
}

}  // namespace rbe
