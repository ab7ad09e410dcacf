// bindings.cpp -- pybind11 module paper_1802_06466_b200._core, the drop-in for
// the reference's rbe._core retrieval surface (bindings/rbe_module.cpp:22-55,
// 157-205): same names, arguments, return shapes and exception types
// (invalid_argument -> ValueError, out_of_range -> IndexError,
// runtime_error -> RuntimeError).  Additions: DeviceIndex (HBM-resident
// store), search_batch, numpy batch entry points and the device-pointer
// calls used by the multi-GPU (torch.distributed) path.
#include <pybind11/numpy.h>
#include <pybind11/operators.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>
#include <pybind11/stl/filesystem.h>

#include <cstring>

#include "rbe/index.hpp"
#include "rbe/search.hpp"
#include "rbe_cuda.h"

namespace py = pybind11;
using namespace rbe;

namespace {

void ck(int status) {
    if (status == RBE_CUDA_OK) return;
    const std::string msg = rbe_cuda_last_error();
    if (status == RBE_CUDA_EINVAL) throw std::invalid_argument(msg);
    if (status == RBE_CUDA_ERANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
}

py::list to_tuples(const SelectionResult& r) {
    py::list out;
    for (const SelectionEntry& e : r.entries) out.append(py::make_tuple(e.score, e.id, e.partition));
    return out;
}

py::dict stats_dict(const SearchStats& s) {
    py::dict d;
    d["scored"] = s.scored;
    d["variant"] = s.variant == RBE_VARIANT_TENSOR ? "tensor" : (s.variant == RBE_VARIANT_EXACT ? "exact" : "auto");
    d["candidates"] = s.candidates;
    d["survivors"] = s.survivors;
    d["device_ms"] = s.device_ms;
    return d;
}

ScanVariant parse_variant(const std::string& v) {
    if (v == "auto") return ScanVariant::Auto;
    if (v == "exact") return ScanVariant::Exact;
    if (v == "tensor") return ScanVariant::Tensor;
    throw std::invalid_argument("variant must be 'auto', 'exact' or 'tensor'");
}

std::shared_ptr<DeviceIndex> device_of(py::object index) {
    if (py::isinstance<DeviceIndex>(index)) return index.cast<std::shared_ptr<DeviceIndex>>();
    // KeywordIndex: immutable from Python, so its device copy is cached on the
    // object (first search uploads it to device 0).
    if (py::hasattr(index, "_device_cache")) return index.attr("_device_cache").cast<std::shared_ptr<DeviceIndex>>();
    const KeywordIndex& k = index.cast<const KeywordIndex&>();
    if (k.partitions.empty() || k.total_keywords() == 0) throw std::invalid_argument("search: empty index");
    std::shared_ptr<DeviceIndex> d;
    {
        py::gil_scoped_release nogil;
        d = std::make_shared<DeviceIndex>(k, std::vector<int>{0});
    }
    index.attr("_device_cache") = py::cast(d);
    return d;
}

}  // namespace

PYBIND11_MODULE(_core, m) {
    m.doc() = "B200-native exhaustive RBE retrieval (drop-in for rbe._core's search path)";

    // --- binary vectors and similarity (host helpers, as in the reference)
    py::class_<PackedBinaryVector>(m, "PackedBinaryVector")
        .def_readonly("dim", &PackedBinaryVector::dim)
        .def_readonly("words", &PackedBinaryVector::words)
        .def(py::self == py::self)
        .def("__repr__",
             [](const PackedBinaryVector& v) { return "<PackedBinaryVector dim=" + std::to_string(v.dim) + ">"; });
    m.def("pack", [](const std::vector<int>& values) { return pack(values); }, py::arg("values"));
    m.def("unpack", &unpack, py::arg("vector"));
    m.def("binary_dot", &binary_dot, py::arg("x"), py::arg("y"));

    py::class_<RbeEmbedding>(m, "RbeEmbedding")
        .def_readonly("planes", &RbeEmbedding::planes)
        .def_readonly("magnitude", &RbeEmbedding::magnitude)
        .def_property_readonly("dim", &RbeEmbedding::dim);
    m.def("make_embedding", &make_embedding, py::arg("planes"), py::arg("residual_weights") = true);
    m.def("refined_vector", &refined_vector, py::arg("embedding"), py::arg("residual_weights") = true);

    py::class_<SimilarityConfig>(m, "SimilarityConfig")
        .def(py::init<>())
        .def_readwrite("query_planes", &SimilarityConfig::query_planes)
        .def_readwrite("keyword_planes", &SimilarityConfig::keyword_planes)
        .def_readwrite("residual_weights", &SimilarityConfig::residual_weights)
        .def_readwrite("normalize_query", &SimilarityConfig::normalize_query);
    m.def("rbe_score", &rbe_score, py::arg("query"), py::arg("keyword"), py::arg("config"));

    // --- index
    py::class_<KeywordIndex>(m, "KeywordIndex", py::dynamic_attr())
        .def_readonly("dim", &KeywordIndex::dim)
        .def_readonly("keyword_planes", &KeywordIndex::keyword_planes)
        .def_readonly("residual_weights", &KeywordIndex::residual_weights)
        .def_property_readonly("total_keywords", &KeywordIndex::total_keywords)
        .def_property_readonly("plane_bytes_per_keyword", &KeywordIndex::plane_bytes_per_keyword)
        .def_property_readonly("plane_payload_bytes", &KeywordIndex::plane_payload_bytes)
        .def_property_readonly("partition_count", [](const KeywordIndex& k) { return k.partitions.size(); })
        .def("partition_arrays",
             [](const KeywordIndex& k, uint32_t p) {
                 const Partition& part = k.partitions.at(p);
                 const size_t wpp = k.words_per_plane();
                 py::array_t<uint64_t> planes({size_t(k.keyword_planes), size_t(part.count * wpp)});
                 if (part.count)
                     for (uint32_t t = 0; t < k.keyword_planes; ++t)
                         std::memcpy(planes.mutable_data(t, 0), part.plane_blocks[t].data(), part.count * wpp * 8);
                 py::array_t<float> mags(part.count);
                 std::memcpy(mags.mutable_data(), part.magnitudes.data(), part.count * 4);
                 py::array_t<uint64_t> ids(part.count);
                 std::memcpy(ids.mutable_data(), part.ids.data(), part.count * 8);
                 return py::make_tuple(planes, mags, ids);
             },
             py::arg("partition"), "(planes[kp][count*wpp] u64, magnitudes f32, ids u64) of one partition");

    m.def(
        "build_index",
        [](const std::vector<std::pair<uint64_t, RbeEmbedding>>& embeddings, uint32_t partitions, bool rw) {
            return build_index(embeddings, partitions, rw);
        },
        py::arg("embeddings"), py::arg("partitions") = 1, py::arg("residual_weights") = true);
    m.def(
        "index_from_arrays",
        [](uint32_t dim, uint32_t kp, bool rw, py::list parts) {
            KeywordIndex k;
            k.dim = dim;
            k.keyword_planes = kp;
            k.residual_weights = rw;
            const size_t wpp = k.words_per_plane();
            for (py::handle h : parts) {
                auto t = h.cast<py::tuple>();
                auto planes = t[0].cast<py::array_t<uint64_t, py::array::c_style | py::array::forcecast>>();
                auto mags = t[1].cast<py::array_t<float, py::array::c_style | py::array::forcecast>>();
                auto ids = t[2].cast<py::array_t<uint64_t, py::array::c_style | py::array::forcecast>>();
                Partition p;
                p.count = uint64_t(ids.size());
                if (size_t(planes.size()) != size_t(kp) * p.count * wpp || size_t(mags.size()) != p.count)
                    throw std::invalid_argument("index_from_arrays: array sizes do not match (kp, count, dim)");
                p.plane_blocks.resize(kp);
                for (uint32_t t2 = 0; t2 < kp; ++t2)
                    p.plane_blocks[t2].assign(planes.data() + t2 * p.count * wpp, planes.data() + (t2 + 1) * p.count * wpp);
                p.magnitudes.assign(mags.data(), mags.data() + p.count);
                p.ids.assign(ids.data(), ids.data() + p.count);
                k.partitions.push_back(std::move(p));
            }
            return k;
        },
        py::arg("dim"), py::arg("keyword_planes"), py::arg("residual_weights"), py::arg("partitions"),
        "KeywordIndex from reference-layout arrays [(planes[kp][count*wpp] u64, magnitudes f32, ids u64)]");
    m.def("save_index", &save_index, py::arg("index"), py::arg("path"));
    m.def("load_index", &load_index, py::arg("path"));
    m.def(
        "index_entry", [](const KeywordIndex& k, uint32_t p, uint64_t slot) { return index_entry(k, p, slot); },
        py::arg("index"), py::arg("partition"), py::arg("slot"));

    py::class_<ScanGeometry>(m, "ScanGeometry")
        .def(py::init<>())
        .def_readwrite("blocks", &ScanGeometry::blocks)
        .def_readwrite("threads_per_block", &ScanGeometry::threads_per_block)
        .def_readwrite("items_per_thread", &ScanGeometry::items_per_thread)
        .def_readwrite("queue_length", &ScanGeometry::queue_length)
        .def_property_readonly("capacity", &ScanGeometry::capacity);
    m.def("thread_assignment", &thread_assignment, py::arg("geometry"), py::arg("partition_count"), py::arg("block"),
          py::arg("thread"));

    py::class_<SearchStats>(m, "SearchStats")
        .def(py::init<>())
        .def_readonly("scored", &SearchStats::scored)
        .def_readonly("candidates", &SearchStats::candidates)
        .def_readonly("survivors", &SearchStats::survivors)
        .def_readonly("device_ms", &SearchStats::device_ms);

    // --- the device store
    m.def(
        "rbei_header",
        [](const std::string& path) {
            rbe_index_shape shape{};
            uint32_t P = 0;
            if (rbe_cuda_rbei_header(path.c_str(), &shape, &P, nullptr, 0) != RBE_CUDA_OK)
                throw std::runtime_error(rbe_cuda_last_error());
            std::vector<uint64_t> counts(P);
            if (rbe_cuda_rbei_header(path.c_str(), &shape, &P, counts.data(), P) != RBE_CUDA_OK)
                throw std::runtime_error(rbe_cuda_last_error());
            py::dict d;
            d["dim"] = shape.dim;
            d["keyword_planes"] = shape.keyword_planes;
            d["residual_weights"] = shape.residual_weights != 0;
            d["counts"] = counts;
            return d;
        },
        py::arg("path"), "RBEI v1 header (host only): shape and partition sizes");
    m.def(
        "rbee_header",
        [](const std::string& path) {
            rbe_index_shape shape{};
            uint64_t n = 0;
            if (rbe_cuda_rbee_header(path.c_str(), &shape, &n) != RBE_CUDA_OK) throw std::runtime_error(rbe_cuda_last_error());
            py::dict d;
            d["dim"] = shape.dim;
            d["plane_count"] = shape.keyword_planes;
            d["residual_weights"] = shape.residual_weights != 0;
            d["count"] = n;
            return d;
        },
        py::arg("path"), "RBEE v1 header (host only): shape and record count");
    py::class_<DeviceIndex, std::shared_ptr<DeviceIndex>>(m, "DeviceIndex", py::dynamic_attr())
        .def(py::init([](const KeywordIndex& k, std::vector<int> devices) {
                 py::gil_scoped_release nogil;
                 return std::make_shared<DeviceIndex>(k, std::move(devices));
             }),
             py::arg("index"), py::arg("devices") = std::vector<int>{0})
        .def_static(
            "synthetic",
            [](uint32_t dim, uint32_t kp, bool rw, uint64_t n_docs, uint32_t partitions, uint64_t seed,
               std::vector<int> devices, uint32_t rank, uint32_t world) {
                py::gil_scoped_release nogil;
                return std::make_shared<DeviceIndex>(
                    DeviceIndex::synthetic(dim, kp, rw, n_docs, partitions, seed, std::move(devices), rank, world));
            },
            py::arg("dim"), py::arg("keyword_planes"), py::arg("residual_weights"), py::arg("n_docs"),
            py::arg("partitions") = 1, py::arg("seed") = 0xD0C5, py::arg("devices") = std::vector<int>{0},
            py::arg("rank") = 0, py::arg("world") = 1)
        .def_static(
            "from_rbei",
            [](const std::string& path, std::vector<int> devices, uint32_t io_threads) {
                LoadStats st;
                std::shared_ptr<DeviceIndex> ix;
                {
                    py::gil_scoped_release nogil;
                    ix = std::make_shared<DeviceIndex>(DeviceIndex::from_rbei(path, std::move(devices), io_threads, &st));
                }
                py::object o = py::cast(ix);
                py::dict d;
                d["file_bytes"] = st.file_bytes;
                d["seconds"] = st.seconds;
                d["gb_per_s"] = st.seconds > 0 ? double(st.file_bytes) / st.seconds / 1e9 : 0.0;
                o.attr("load_stats") = d;
                return o;
            },
            py::arg("path"), py::arg("devices") = std::vector<int>{0}, py::arg("io_threads") = 0,
            "RBEI file straight into HBM (load_index + upload in one streamed pass); sets .load_stats")
        .def_static(
            "build_rbee",
            [](const std::string& path, uint32_t partitions, std::vector<int> devices, uint32_t io_threads) {
                LoadStats st;
                std::shared_ptr<DeviceIndex> ix;
                {
                    py::gil_scoped_release nogil;
                    ix = std::make_shared<DeviceIndex>(
                        DeviceIndex::build_rbee(path, partitions, std::move(devices), io_threads, &st));
                }
                py::object o = py::cast(ix);
                py::dict d;
                d["file_bytes"] = st.file_bytes;
                d["seconds"] = st.seconds;
                d["gb_per_s"] = st.seconds > 0 ? double(st.file_bytes) / st.seconds / 1e9 : 0.0;
                o.attr("load_stats") = d;
                return o;
            },
            py::arg("path"), py::arg("partitions") = 1, py::arg("devices") = std::vector<int>{0},
            py::arg("io_threads") = 0,
            "RBEE bulk embeddings built into an index on the device (rbe build); sets .load_stats")
        .def(
            "save_index",
            [](const DeviceIndex& d, const std::string& path) {
                py::gil_scoped_release nogil;
                d.save_index(path);
            },
            py::arg("path"))
        .def_property_readonly("dim", &DeviceIndex::dim)
        .def_property_readonly("keyword_planes", &DeviceIndex::keyword_planes)
        .def_property_readonly("residual_weights", &DeviceIndex::residual_weights)
        .def_property_readonly("partition_count", &DeviceIndex::partition_count)
        .def_property_readonly("total_keywords", &DeviceIndex::total_keywords)
        .def_property_readonly("max_partition_count", &DeviceIndex::max_partition_count)
        .def_property_readonly("device_bytes", &DeviceIndex::device_bytes)
        .def_property_readonly("scan_bytes", &DeviceIndex::scan_bytes)
        .def_property_readonly("devices", &DeviceIndex::devices)
        .def("handle", [](const DeviceIndex& d, size_t i) { return reinterpret_cast<uintptr_t>(d.handle(i)); },
             py::arg("i") = 0)
        .def("partition_size", &DeviceIndex::partition_size, py::arg("partition"))
        .def("download_partition",
             [](const DeviceIndex& d, uint32_t p) {
                 Partition part;
                 {
                     py::gil_scoped_release nogil;
                     part = d.download_partition(p);
                 }
                 const size_t wpp = PackedBinaryVector::words_for(d.dim());
                 py::array_t<uint64_t> planes({size_t(d.keyword_planes()), size_t(part.count * wpp)});
                 if (part.count)
                     for (uint32_t t = 0; t < d.keyword_planes(); ++t)
                         std::memcpy(planes.mutable_data(t, 0), part.plane_blocks[t].data(), part.count * wpp * 8);
                 py::array_t<float> mags(part.count);
                 std::memcpy(mags.mutable_data(), part.magnitudes.data(), part.count * 4);
                 py::array_t<uint64_t> ids(part.count);
                 std::memcpy(ids.mutable_data(), part.ids.data(), part.count * 8);
                 return py::make_tuple(planes, mags, ids);
             },
             py::arg("partition"))
        .def(
            "search_words",
            [](const DeviceIndex& d, py::array_t<uint64_t, py::array::c_style | py::array::forcecast> words,
               const ScanGeometry& g, uint64_t n, const std::string& variant, uint32_t probe_tiles, bool with_stats,
               py::object out) {
                if (words.ndim() != 3) throw std::invalid_argument("search_words: words must be [Q][planes][wpp]");
                const uint32_t Q = uint32_t(words.shape(0)), qp = uint32_t(words.shape(1));
                const ScanVariant v = parse_variant(variant);
                // results land directly in the returned arrays (entries past counts[q] are zero); with
                // out=(scores, ids, partitions, accs, counts) the caller's arrays are reused (a serving
                // loop then writes warm pages instead of faulting in fresh ones every batch)
                using F = py::array;
                py::array_t<double, F::c_style> scores;
                py::array_t<uint64_t, F::c_style> ids;
                py::array_t<uint32_t, F::c_style> parts;
                py::array_t<int64_t, F::c_style> accs;
                py::array_t<uint64_t, F::c_style> counts;
                if (out.is_none()) {
                    scores = py::array_t<double, F::c_style>({size_t(Q), size_t(n)});
                    ids = py::array_t<uint64_t, F::c_style>({size_t(Q), size_t(n)});
                    parts = py::array_t<uint32_t, F::c_style>({size_t(Q), size_t(n)});
                    accs = py::array_t<int64_t, F::c_style>({size_t(Q), size_t(n)});
                    counts = py::array_t<uint64_t, F::c_style>(Q);
                } else {
                    py::tuple t = out.cast<py::tuple>();
                    if (t.size() != 5) throw std::invalid_argument("search_words: out must be (scores, ids, partitions, accs, counts)");
                    auto take = [&](auto& dst, size_t k, size_t want) {
                        using A = std::decay_t<decltype(dst)>;
                        if (!A::check_(t[k])) throw std::invalid_argument("search_words: out array has the wrong dtype or layout");
                        dst = t[k].cast<A>();
                        if (size_t(dst.size()) != want || !dst.writeable())
                            throw std::invalid_argument("search_words: out array has the wrong size or is read-only");
                    };
                    take(scores, 0, size_t(Q) * n);
                    take(ids, 1, size_t(Q) * n);
                    take(parts, 2, size_t(Q) * n);
                    take(accs, 3, size_t(Q) * n);
                    take(counts, 4, size_t(Q));
                }
                SearchStats st;
                {
                    double* S = scores.mutable_data();
                    uint64_t* I = ids.mutable_data();
                    uint32_t* P = parts.mutable_data();
                    int64_t* A = accs.mutable_data();
                    uint64_t* C = counts.mutable_data();
                    py::gil_scoped_release nogil;
                    d.search_words_into(std::span<const uint64_t>(words.data(), size_t(words.size())), Q, qp, g, n,
                                        S, I, P, A, C, with_stats ? &st : nullptr, v, probe_tiles);
                    for (uint32_t q = 0; q < Q; ++q) {
                        const size_t o = size_t(q) * n;
                        for (uint64_t k = C[q]; k < n; ++k) {
                            S[o + k] = 0.0;
                            I[o + k] = 0;
                            P[o + k] = 0;
                            A[o + k] = 0;
                        }
                    }
                }
                return py::make_tuple(scores, ids, parts, accs, counts, stats_dict(st));
            },
            py::arg("words"), py::arg("geometry"), py::arg("n"), py::arg("variant") = "auto",
            py::arg("probe_tiles") = 0, py::arg("with_stats") = true, py::arg("out") = py::none(),
            "Batched search over raw query words [Q][planes][wpp] -> (scores, ids, partitions, accs, counts, stats)");

    // --- search (drop-in) and batch
    m.def(
        "search",
        [](const RbeEmbedding& query, py::object index, const ScanGeometry& g, uint64_t n) {
            if (py::isinstance<KeywordIndex>(index)) {
                const KeywordIndex& k = index.cast<const KeywordIndex&>();
                if (k.partitions.empty() || k.total_keywords() == 0) throw std::invalid_argument("search: empty index");
                if (query.dim() != k.dim) throw std::invalid_argument("local_select: query dimension mismatch");
            }
            std::shared_ptr<DeviceIndex> d = device_of(index);
            SelectionResult r;
            {
                py::gil_scoped_release nogil;
                r = search(query, *d, g, n);
            }
            return to_tuples(r);
        },
        py::arg("query"), py::arg("index"), py::arg("geometry"), py::arg("n"),
        "Returns [(score, id, partition)] ordered by (score desc, id asc)");
    m.def(
        "search_batch",
        [](const std::vector<RbeEmbedding>& queries, py::object index, const ScanGeometry& g, uint64_t n) {
            std::shared_ptr<DeviceIndex> d = device_of(index);
            std::vector<SelectionResult> r;
            {
                py::gil_scoped_release nogil;
                r = search_batch(queries, *d, g, n);
            }
            py::list out;
            for (auto& x : r) out.append(to_tuples(x));
            return out;
        },
        py::arg("queries"), py::arg("index"), py::arg("geometry"), py::arg("n"));

    // --- device-pointer entry points (torch.distributed multi-GPU path)
    m.def(
        "search_device",
        [](uintptr_t handle, uintptr_t d_words, uint32_t Q, uint32_t qp, const ScanGeometry& g, uint64_t n,
           uintptr_t d_out, uintptr_t stream, const std::string& variant, bool with_stats) {
            const rbe_scan_geometry geo{g.blocks, g.threads_per_block, g.items_per_thread, g.queue_length};
            rbe_search_options opt{};
            opt.variant = uint32_t(parse_variant(variant));
            rbe_search_stats st{};
            int status;
            {
                py::gil_scoped_release nogil;
                status = rbe_cuda_search_device(reinterpret_cast<rbe_cuda_index*>(handle),
                                                reinterpret_cast<const uint64_t*>(d_words), Q, qp, &geo, n, &opt,
                                                reinterpret_cast<rbe_result*>(d_out),
                                                reinterpret_cast<void*>(stream), with_stats ? &st : nullptr);
            }
            ck(status);
            py::dict d;
            d["scored"] = st.scored;
            d["variant"] = st.variant == RBE_VARIANT_TENSOR ? "tensor" : "exact";
            d["candidates"] = st.candidates;
            d["survivors"] = st.survivors;
            d["scan_ms"] = st.scan_ms;
            d["total_ms"] = st.total_ms;
            d["launches"] = st.launches;
            d["fallback"] = st.fallback;
            return d;
        },
        py::arg("handle"), py::arg("d_words"), py::arg("n_queries"), py::arg("query_planes"), py::arg("geometry"),
        py::arg("n"), py::arg("d_out"), py::arg("stream") = 0, py::arg("variant") = "auto",
        py::arg("with_stats") = true);
    m.def(
        "last_batch_ms",
        [](uintptr_t handle) {
            double scan = 0, total = 0;
            int status;
            {
                py::gil_scoped_release nogil;
                status = rbe_cuda_index_last_batch_ms(reinterpret_cast<rbe_cuda_index*>(handle), &scan, &total);
            }
            ck(status);
            return py::make_tuple(scan, total);
        },
        py::arg("handle"));
    m.def(
        "merge_device",
        [](int device, uintptr_t d_in, uint32_t n_lists, uint32_t Q, uint64_t n, uintptr_t d_out, uintptr_t stream) {
            int status;
            {
                py::gil_scoped_release nogil;
                status = rbe_cuda_merge_device(device, reinterpret_cast<const rbe_result*>(d_in), n_lists, Q, n,
                                               reinterpret_cast<rbe_result*>(d_out), reinterpret_cast<void*>(stream));
            }
            ck(status);
        },
        py::arg("device"), py::arg("d_in"), py::arg("n_lists"), py::arg("n_queries"), py::arg("n"), py::arg("d_out"),
        py::arg("stream") = 0);
    // --- local_select / global_select on the device (reference search.hpp:53-63)
    m.def(
        "local_select_arrays",
        [](const DeviceIndex& d, py::array_t<uint64_t, py::array::c_style | py::array::forcecast> words,
           uint32_t partition, const ScanGeometry& g) {
            if (words.ndim() != 2) throw std::invalid_argument("local_select: words must be [planes][wpp]");
            const auto [h, local] = d.locate(partition);
            const uint64_t threads = uint64_t(g.blocks) * g.threads_per_block;
            const uint64_t ql = std::min<uint64_t>(g.queue_length, g.items_per_thread);
            py::array_t<double> scores({size_t(threads), size_t(ql)});
            py::array_t<uint64_t> slots({size_t(threads), size_t(ql)});
            py::array_t<uint32_t> counts(threads);
            uint64_t scored = 0;
            const rbe_scan_geometry geo{g.blocks, g.threads_per_block, g.items_per_thread, g.queue_length};
            int status;
            {
                double* S = scores.mutable_data();
                uint64_t* Z = slots.mutable_data();
                uint32_t* C = counts.mutable_data();
                py::gil_scoped_release nogil;
                status = rbe_cuda_local_select(d.handle(h), local, words.data(), uint32_t(words.shape(0)), &geo, S, Z,
                                               C, &scored);
            }
            ck(status);
            return py::make_tuple(scores, slots, counts, scored);
        },
        py::arg("index"), py::arg("words"), py::arg("partition"), py::arg("geometry"),
        "local_select on the device -> (scores[threads][ql], slots[threads][ql], counts[threads], scored)");
    m.def(
        "local_select",
        [](const RbeEmbedding& query, py::object index, uint32_t partition, const ScanGeometry& g) {
            std::vector<std::vector<Candidate>> lists;
            if (py::isinstance<DeviceIndex>(index)) {
                const DeviceIndex& d = index.cast<const DeviceIndex&>();
                py::gil_scoped_release nogil;
                lists = local_select(query, d, partition, g);
            } else {
                const KeywordIndex& k = index.cast<const KeywordIndex&>();
                py::gil_scoped_release nogil;
                lists = local_select(query, k, partition, g);
            }
            py::list out;
            for (const auto& l : lists) {
                py::list row;
                for (const Candidate& c : l) row.append(py::make_tuple(c.score, c.slot));
                out.append(row);
            }
            return out;
        },
        py::arg("query"), py::arg("index"), py::arg("partition"), py::arg("geometry"),
        "Per-logical-thread [(score, slot)] lists of one partition (reference local_select)");
    m.def(
        "select_topn",
        [](py::array_t<double, py::array::c_style | py::array::forcecast> scores,
           py::array_t<uint64_t, py::array::c_style | py::array::forcecast> ids, uint32_t partition, uint64_t n,
           int device) {
            if (scores.size() != ids.size()) throw std::invalid_argument("select_topn: scores and ids differ in size");
            const uint64_t m = std::min<uint64_t>(n, uint64_t(scores.size()));
            py::array_t<double> os(m);
            py::array_t<uint64_t> oi(m);
            uint64_t got = 0;
            int status;
            {
                double* S = os.mutable_data();
                uint64_t* I = oi.mutable_data();
                py::gil_scoped_release nogil;
                status = rbe_cuda_select_topn(device, scores.data(), ids.data(), uint64_t(scores.size()), partition, n,
                                              S, I, &got);
            }
            ck(status);
            return py::make_tuple(os[py::slice(0, got, 1)], oi[py::slice(0, got, 1)]);
        },
        py::arg("scores"), py::arg("ids"), py::arg("partition"), py::arg("n"), py::arg("device") = 0,
        "global_select's selection on the device: top n (score desc, id asc) -> (scores, ids)");
    m.def(
        "index_check",
        [](uintptr_t handle) {
            int status;
            {
                py::gil_scoped_release nogil;
                status = rbe_cuda_index_check(reinterpret_cast<rbe_cuda_index*>(handle));
            }
            ck(status);
        },
        py::arg("handle"));
    m.def(
        "index_inject_error", [](uintptr_t handle) { ck(rbe_cuda_index_inject_error(reinterpret_cast<rbe_cuda_index*>(handle))); },
        py::arg("handle"), "test hook: set the index's sticky internal-consistency flag");
    m.attr("RESULT_RECORD_BYTES") = sizeof(rbe_result);
    m.def("version", [] { return std::string(rbe_cuda_version()); });
}
