// cli.cpp -- `rbe-cuda`, the command-line caller of the B200 path: the
// reference CLI's `build` and `query` subcommands (tools/rbe_main.cpp:103-211) over the
// HBM-resident index.
//
//   rbe-cuda build --embeddings E.rbee --output I.rbei [--partitions P] [--devices 0,1,..]
//       RBEE -> index built on the device(s) -> RBEI; prints the reference's stats line.
//   rbe-cuda query --index I.rbei --queries Q.rbee [--n 10] [--blocks 0] [--threads-per-block 256]
//                  [--items-per-thread 256] [--queue-length 1] [--batch-size 64]
//                  [--devices 0,1,..] [--output F]
//       RBEI -> HBM once (DeviceIndex::from_rbei), then the queries in batches through
//       search_batch (one pass over the store per batch).  Output lines are the reference's
//       "query\tid\tscore" (%zu\t%llu\t%.9g); stderr gets the reference's latency line
//       (per query) plus the per-batch mean / p50 / p99 and queries/s.
//
// Queries are read as RBEE records (pre-computed query embeddings; record ids are ignored and
// queries are numbered by position, as the reference numbers --batch lines): the text encoder
// (embed_text, model.cpp) stays outside the GPU path (SURVEY.md §8(f) note).
// Exit codes as the reference: 2 for usage errors and std::invalid_argument, 1 otherwise
// (rbe_main.cpp:440-458).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "rbe/search.hpp"
#include "rbe_cuda.h"

namespace {

constexpr int kExitUsage = 2;
constexpr int kExitRuntime = 1;

struct Usage : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

const char* kHelp =
    "rbe-cuda: exhaustive RBE retrieval on B200\n"
    "  build --embeddings FILE.rbee --output FILE.rbei [--partitions P] [--devices 0,1,...]\n"
    "  query --index FILE.rbei --queries FILE.rbee [--n 10] [--blocks 0] [--threads-per-block 256]\n"
    "        [--items-per-thread 256] [--queue-length 1] [--batch-size 64] [--devices 0,...] [--output FILE]\n";

struct Args {
    std::map<std::string, std::string> kv;
    std::string get(const std::string& k, const std::string& def = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? def : it->second;
    }
    uint64_t num(const std::string& k, uint64_t def, bool positive) const {
        auto it = kv.find(k);
        if (it == kv.end()) return def;
        char* end = nullptr;
        const unsigned long long v = std::strtoull(it->second.c_str(), &end, 10);
        if (!end || *end || it->second.empty() || it->second[0] == '-' || (positive && v == 0))
            throw Usage("--" + k + ": expected a " + std::string(positive ? "positive" : "non-negative") + " integer");
        return v;
    }
    std::vector<int> devices() const {
        std::vector<int> d;
        std::string s = get("devices", "0");
        size_t pos = 0;
        while (pos <= s.size()) {
            const size_t c = s.find(',', pos);
            const std::string tok = s.substr(pos, c == std::string::npos ? std::string::npos : c - pos);
            if (tok.empty()) throw Usage("--devices: expected a comma-separated list of device ordinals");
            d.push_back(std::atoi(tok.c_str()));
            if (c == std::string::npos) break;
            pos = c + 1;
        }
        return d;
    }
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& allowed) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0) throw Usage("unexpected argument: " + k);
        k = k.substr(2);
        if (std::find(allowed.begin(), allowed.end(), k) == allowed.end()) throw Usage("unknown option: --" + k);
        if (i + 1 >= argc) throw Usage("--" + k + " needs a value");
        a.kv[k] = argv[++i];
    }
    return a;
}

// RBEE records -> query embeddings (embedding_io.cpp:79-95 record layout)
std::vector<rbe::RbeEmbedding> read_queries(const std::string& path) {
    rbe_index_shape shape{};
    uint64_t n = 0;
    if (rbe_cuda_rbee_header(path.c_str(), &shape, &n) != RBE_CUDA_OK) throw std::runtime_error(rbe_cuda_last_error());
    const size_t wpp = (shape.dim + 63) / 64;
    std::ifstream in(path, std::ios::binary);
    in.seekg(20);
    std::vector<rbe::RbeEmbedding> qs(n);
    std::vector<uint64_t> words(shape.keyword_planes * wpp);
    for (uint64_t k = 0; k < n; ++k) {
        uint64_t id;
        float mag;
        in.read(reinterpret_cast<char*>(&id), 8);
        in.read(reinterpret_cast<char*>(words.data()), std::streamsize(words.size() * 8));
        in.read(reinterpret_cast<char*>(&mag), 4);
        if (!in) throw std::runtime_error("truncated embeddings record");
        for (uint32_t t = 0; t < shape.keyword_planes; ++t) {
            rbe::PackedBinaryVector v;
            v.dim = shape.dim;
            v.words.assign(words.begin() + t * wpp, words.begin() + (t + 1) * wpp);
            qs[k].planes.push_back(std::move(v));
        }
        qs[k].magnitude = mag;
    }
    return qs;
}

int run_build(const Args& a) {
    const std::string emb = a.get("embeddings"), out = a.get("output");
    if (emb.empty() || out.empty()) throw Usage("build: --embeddings and --output are required");
    const uint32_t P = uint32_t(a.num("partitions", 1, true));
    rbe::LoadStats st;
    const rbe::DeviceIndex ix = rbe::DeviceIndex::build_rbee(emb, P, a.devices(), 0, &st);
    ix.save_index(out);
    const uint64_t per_kw = uint64_t(ix.keyword_planes()) * ((ix.dim() + 63) / 64) * 8;
    std::printf("keywords=%llu partitions=%u plane_bytes_per_keyword=%llu plane_payload_bytes=%llu\n",
                (unsigned long long)ix.total_keywords(), P, (unsigned long long)per_kw,
                (unsigned long long)(per_kw * ix.total_keywords()));
    std::fprintf(stderr, "build_seconds=%.3f embeddings_gb_per_s=%.2f\n", st.seconds,
                 st.seconds > 0 ? double(st.file_bytes) / st.seconds / 1e9 : 0.0);
    return 0;
}

int run_query(const Args& a) {
    const std::string index_path = a.get("index"), qpath = a.get("queries");
    if (index_path.empty() || qpath.empty()) throw Usage("query: --index and --queries are required");
    const uint64_t n = a.num("n", 10, true);
    rbe::ScanGeometry g;
    g.threads_per_block = uint32_t(a.num("threads-per-block", 256, true));
    g.items_per_thread = uint32_t(a.num("items-per-thread", 256, true));
    g.queue_length = uint32_t(a.num("queue-length", 1, true));
    const uint64_t blocks = a.num("blocks", 0, false);
    const uint64_t batch = a.num("batch-size", 64, true);
    rbe::LoadStats ls;
    const rbe::DeviceIndex ix = rbe::DeviceIndex::from_rbei(index_path, a.devices(), 0, &ls);
    if (ix.total_keywords() == 0) throw std::runtime_error("index is empty");
    const uint64_t per_block = uint64_t(g.threads_per_block) * g.items_per_thread;
    g.blocks = blocks ? uint32_t(blocks) : uint32_t((ix.max_partition_count() + per_block - 1) / per_block);
    const std::vector<rbe::RbeEmbedding> qs = read_queries(qpath);

    std::ofstream file_out;
    if (!a.get("output").empty()) {
        file_out.open(a.get("output"));
        if (!file_out) throw std::runtime_error("cannot open output file: " + a.get("output"));
    }
    std::ostream& out = a.get("output").empty() ? std::cout : file_out;
    std::vector<double> batch_ms, query_ms;
    char buf[96];
    for (size_t q0 = 0; q0 < qs.size(); q0 += batch) {
        const size_t nb = std::min<size_t>(batch, qs.size() - q0);
        const auto t0 = std::chrono::steady_clock::now();
        const std::vector<rbe::SelectionResult> res =
            rbe::search_batch(std::span<const rbe::RbeEmbedding>(qs.data() + q0, nb), ix, g, n);
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        batch_ms.push_back(ms);
        for (size_t k = 0; k < nb; ++k) query_ms.push_back(ms);  // every query of a batch waits for the batch
        for (size_t k = 0; k < nb; ++k)
            for (const rbe::SelectionEntry& e : res[k].entries) {
                std::snprintf(buf, sizeof(buf), "%zu\t%llu\t%.9g\n", q0 + k, (unsigned long long)e.id, e.score);
                out << buf;
            }
    }
    auto stats = [](std::vector<double> v, double& mean, double& p50, double& p99) {
        std::sort(v.begin(), v.end());
        mean = 0;
        for (double x : v) mean += x;
        mean /= double(v.size());
        p50 = v[size_t(std::ceil(0.50 * double(v.size()))) - 1];
        p99 = v[size_t(std::ceil(0.99 * double(v.size()))) - 1];
    };
    if (!query_ms.empty()) {
        double mean, p50, p99;
        stats(query_ms, mean, p50, p99);
        std::fprintf(stderr, "queries=%zu latency_mean_ms=%.3f latency_p99_ms=%.3f\n", query_ms.size(), mean, p99);
        double total = 0;
        for (double x : batch_ms) total += x;
        stats(batch_ms, mean, p50, p99);
        std::fprintf(stderr,
                     "batches=%zu batch_size=%llu batch_latency_mean_ms=%.3f batch_latency_p50_ms=%.3f "
                     "batch_latency_p99_ms=%.3f queries_per_s=%.1f index_load_seconds=%.3f index_load_gb_per_s=%.2f\n",
                     batch_ms.size(), (unsigned long long)batch, mean, p50, p99,
                     double(query_ms.size()) / (total / 1e3), ls.seconds,
                     ls.seconds > 0 ? double(ls.file_bytes) / ls.seconds / 1e9 : 0.0);
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2 || !std::strcmp(argv[1], "--help") || !std::strcmp(argv[1], "-h")) {
        std::fputs(kHelp, argc < 2 ? stderr : stdout);
        return argc < 2 ? kExitUsage : 0;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "build") return run_build(parse(argc, argv, 2, {"embeddings", "output", "partitions", "devices"}));
        if (cmd == "query")
            return run_query(parse(argc, argv, 2,
                                   {"index", "queries", "n", "blocks", "threads-per-block", "items-per-thread",
                                    "queue-length", "batch-size", "devices", "output"}));
        throw Usage("unknown subcommand: " + cmd);
    } catch (const Usage& e) {
        std::fprintf(stderr, "%s\n%s", e.what(), kHelp);
        return kExitUsage;
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kExitUsage;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kExitRuntime;
    }
}
