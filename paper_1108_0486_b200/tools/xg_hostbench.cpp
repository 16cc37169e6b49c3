// xg_hostbench -- the reference's two host-side throughput methods run over
// the GPU drop-in (include/xg/gpu.hpp), as a C++ user of the reference would
// call it:
//
//   measure_throughput (proj/src/bench.cpp:67-93): per-word pulls through the
//     virtual WordSource::next() of xg::gpu::XorgensSource (next_word served
//     inline from double-buffered pinned device refills); each trial = `count`
//     words in 20 chunks, the best chunk rate on thread CPU time; one warm-up
//     trial discarded (bench.cpp:19-53).  The wall-clock rate of the same
//     trials is reported beside it (thread CPU time does not see blocking).
//   measure_ensemble_throughput (bench.cpp:95-112): steady_clock around
//     xg::gpu::BlockEnsemble::generate(count / blocks) -- the reference's
//     vector<vector<uint64_t>> result, allocated and filled -- then every word
//     folded into the sink.
//
// usage: xg_hostbench [words_count=1e8] [trials=5] [blocks=16384] [ens_count=2^30]
// prints one JSON object.
#include <time.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include "xg/gpu.hpp"

namespace {

// The reference's consumer interface (proj/include/xg/stream.hpp:17-22).
class WordSource {
public:
    virtual ~WordSource() = default;
    virtual std::uint64_t next() = 0;
    virtual unsigned word_bits() const = 0;
};

double thread_cpu_seconds() {
    timespec ts;
    clock_gettime(CLOCK_THREAD_CPUTIME_ID, &ts);
    return static_cast<double>(ts.tv_sec) + static_cast<double>(ts.tv_nsec) * 1e-9;
}

struct Report {
    std::vector<double> rate;
    double mean = 0, min = 0, max = 0, cv = 0;
};

Report run_trials(unsigned trials, const std::function<double()>& trial) {
    trial();  // warm-up, discarded (bench.cpp:29)
    Report r;
    for (unsigned t = 0; t < trials; ++t) r.rate.push_back(trial());
    double sum = 0;
    r.min = r.max = r.rate.front();
    for (double v : r.rate) {
        sum += v;
        r.min = std::min(r.min, v);
        r.max = std::max(r.max, v);
    }
    r.mean = sum / trials;
    double var = 0;
    for (double v : r.rate) var += (v - r.mean) * (v - r.mean);
    r.cv = std::sqrt(var / trials) / r.mean;
    return r;
}

std::string json(const Report& r) {
    char b[256];
    std::snprintf(b, sizeof b, "{\"mean\": %.6g, \"min\": %.6g, \"max\": %.6g, \"cv\": %.4g}", r.mean,
                  r.min, r.max, r.cv);
    return b;
}

}  // namespace

int main(int argc, char** argv) {
    const std::uint64_t count = argc > 1 ? std::strtoull(argv[1], nullptr, 0) : 100000000ull;
    const unsigned trials = argc > 2 ? static_cast<unsigned>(std::atoi(argv[2])) : 5u;
    const unsigned blocks = argc > 3 ? static_cast<unsigned>(std::atoi(argv[3])) : 16384u;
    const std::uint64_t ens_count = argc > 4 ? std::strtoull(argv[4], nullptr, 0) : (1ull << 30);
    const auto p = xg::gpu::xorgensgp32_params();

    // measure_throughput over the drop-in WordSource (bench.cpp:67-93)
    xg::gpu::XorgensSource<WordSource> src(p, 1);
    WordSource& source = src;
    std::uint64_t sink = 0;
    double wall_sum = 0;
    constexpr unsigned chunks = 20;
    auto trial = [&]() -> double {
        const std::uint64_t chunk_size = count / chunks;
        double best = 0.0;
        std::uint64_t produced = 0;
        const auto w0 = std::chrono::steady_clock::now();
        for (unsigned c = 0; c < chunks; ++c) {
            const std::uint64_t n = (c == chunks - 1) ? count - produced : chunk_size;
            const double start = thread_cpu_seconds();
            for (std::uint64_t i = 0; i < n; ++i) sink ^= source.next();
            const double elapsed = thread_cpu_seconds() - start;
            produced += n;
            if (elapsed > 0.0) best = std::max(best, static_cast<double>(n) / elapsed);
        }
        const std::chrono::duration<double> dw = std::chrono::steady_clock::now() - w0;
        wall_sum += static_cast<double>(count) / dw.count();
        return best;
    };
    const Report src_rep = run_trials(trials, trial);
    const double src_wall = wall_sum / (trials + 1);

    // measure_ensemble_throughput over the drop-in BlockEnsemble (bench.cpp:95-112)
    xg::gpu::BlockEnsemble ens(p, 1, blocks, 63);
    const std::size_t per_block = ens_count / blocks;
    const std::uint64_t total = static_cast<std::uint64_t>(per_block) * blocks;
    auto etrial = [&]() -> double {
        const auto start = std::chrono::steady_clock::now();
        auto out = ens.generate(per_block);
        const std::chrono::duration<double> elapsed = std::chrono::steady_clock::now() - start;
        for (const auto& b : out)
            for (std::uint64_t w : b) sink ^= w;
        return static_cast<double>(total) / elapsed.count();
    };
    const Report ens_rep = run_trials(trials, etrial);

    // The host-side ceiling of that result type: the same allocation
    // (blocks x reserve(per_block)) and the same u32 -> uint64 appends from a
    // resident 256 MiB u32 source, on the same threads, with no GPU, no PCIe
    // and no generator -- what building vector<vector<uint64_t>> costs on
    // this host by itself.
    const unsigned nthr = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::uint32_t> srcbuf(std::min<std::uint64_t>(total, 1ull << 26), 0x9e3779b9u);
    auto htrial = [&]() -> double {
        const auto start = std::chrono::steady_clock::now();
        std::vector<std::vector<std::uint64_t>> out(blocks);
        std::vector<std::thread> pool;
        for (unsigned id = 0; id < nthr; ++id)
            pool.emplace_back([&, id] {
                for (unsigned i = id; i < blocks; i += nthr) {
                    out[i].reserve(per_block);
                    const std::uint32_t* src =
                        srcbuf.data() + (static_cast<std::uint64_t>(i) * per_block) % (srcbuf.size() - per_block + 1);
                    out[i].insert(out[i].end(), src, src + per_block);
                }
            });
        for (auto& th : pool) th.join();
        const std::chrono::duration<double> elapsed = std::chrono::steady_clock::now() - start;
        for (const auto& b : out) sink ^= b.back();
        return static_cast<double>(total) / elapsed.count();
    };
    const Report host_rep = run_trials(trials, htrial);

    std::printf("{\"measure_throughput\": {\"api\": \"xg::gpu::XorgensSource<WordSource>::next "
                "(virtual, next_word inline from pinned refills)\", \"count\": %llu, \"trials\": %u, "
                "\"rn_per_s\": %s, \"wall_rn_per_s\": %.6g}, "
                "\"measure_ensemble_throughput\": {\"api\": \"xg::gpu::BlockEnsemble::generate -> "
                "vector<vector<uint64_t>>\", \"blocks\": %u, \"per_block\": %zu, \"trials\": %u, "
                "\"rn_per_s\": %s, \"bytes_per_word_host\": 8}, "
                "\"host_result_ceiling\": {\"what\": \"the same vector<vector<uint64_t>> built from a "
                "resident u32 buffer on %u threads, no GPU\", \"rn_per_s\": %s}, \"sink\": %llu}\n",
                static_cast<unsigned long long>(count), trials, json(src_rep).c_str(), src_wall, blocks,
                per_block, trials, json(ens_rep).c_str(), nthr, json(host_rep).c_str(),
                static_cast<unsigned long long>(sink));
    return 0;
}
