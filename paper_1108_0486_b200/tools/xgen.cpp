// xgen (GPU backend): the reference CLI's `gen`, `bench` and `params`
// subcommands (proj/tools/xgen.cpp) over libxg_gpu.so.  Same flags, output
// formats and exit codes, so golden files and scripts written against the
// reference keep working:
//
//   0 success, 64 unknown generator, 65 lanes or blocks out of range,
//   66 I/O error, 67 invalid arguments   (proj/tools/xgen.cpp:4-8,26-32)
//
// Generators: every xorgens id of the reference registry
// (proj/src/registry.cpp:27-42): xorgensgp32, xorgens-raw (linear part only),
// tiny:r2w8, tiny:r2w16, tiny:r4w16 and their tiny-raw: forms.  `test` (the
// statistical battery, xgen.cpp:132-191) runs the GPU battery of the Python
// host layer over the same library: this binary execs
// `python3 -m paper_1108_0486_b200.xgen_test` with the subcommand's arguments
// (exit codes 0 / 2 suspect / 3 fail as the reference).  The CPU baselines
// (xorwow, mt19937) are not part of the GPU backend: 64.
#include <cuda_runtime.h>

#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include <unistd.h>

#include "xg_gpu.h"

namespace {

constexpr int exit_ok = 0;
constexpr int exit_unknown_generator = 64;
constexpr int exit_lane_range = 65;
constexpr int exit_io = 66;
constexpr int exit_bad_args = 67;

struct Gen {
    std::string id;
    bool weyl;
    xg_params_t p;
    const char* note;
};

bool find_generator(const std::string& id, Gen* g) {
    struct Row { const char* id; bool weyl; xg_params_t (*params)(); const char* note; };
    static const Row rows[] = {  // proj/src/registry.cpp:27-42
        {"xorgensgp32", true, xg_params_xorgensgp32, "nominal; primitivity not re-verified"},
        {"xorgens-raw", false, xg_params_xorgensgp32, "linear part only (Weyl ablated); nominal"},
        {"tiny:r2w8", true, xg_params_tiny_r2w8,
         "exact: (2^16-1)*2^8 = 16776960, verified by exhaustive iteration"},
        {"tiny:r2w16", true, xg_params_tiny_r2w16, "linear period 2^32-1 verified by matrix-order search"},
        {"tiny:r4w16", true, xg_params_tiny_r4w16, "linear period 2^64-1 verified by matrix-order search"},
        {"tiny-raw:r2w8", false, xg_params_tiny_r2w8, "exact: 2^16-1 = 65535, verified by exhaustive iteration"},
        {"tiny-raw:r2w16", false, xg_params_tiny_r2w16, "exact: 2^32-1, verified by matrix-order search"},
        {"tiny-raw:r4w16", false, xg_params_tiny_r4w16, "exact: 2^64-1, verified by matrix-order search"},
    };
    for (const Row& r : rows)
        if (id == r.id) {
            *g = {id, r.weyl, r.params(), r.note};
            return true;
        }
    return false;
}

struct Args {
    std::string cmd, generator = "xorgensgp32", format = "hex", output;
    uint64_t seed = 0, count = 0;
    bool have_count = false, as_json = false;
    unsigned blocks = 1, lanes = 1, trials = 5;
    std::string positional;
};

bool parse_u64(const char* s, uint64_t* v) {
    char* end = nullptr;
    errno = 0;
    unsigned long long x = std::strtoull(s, &end, 0);
    if (errno || !end || *end || s[0] == '-') return false;
    *v = x;
    return true;
}

int parse(int argc, char** argv, Args* a) {
    if (argc < 2) return exit_bad_args;
    a->cmd = argv[1];
    for (int i = 2; i < argc; ++i) {
        std::string k = argv[i];
        auto need = [&](uint64_t* v) {
            return i + 1 < argc && parse_u64(argv[++i], v);
        };
        uint64_t v = 0;
        if (k == "--generator" || k == "-g") {
            if (i + 1 >= argc) return exit_bad_args;
            a->generator = argv[++i];
        } else if (k == "--seed") {
            if (!need(&a->seed)) return exit_bad_args;
        } else if (k == "--count") {
            if (!need(&a->count)) return exit_bad_args;
            a->have_count = true;
        } else if (k == "--format") {
            if (i + 1 >= argc) return exit_bad_args;
            a->format = argv[++i];
            if (a->format != "raw-le" && a->format != "hex" && a->format != "u32-lines")
                return exit_bad_args;
        } else if (k == "--output" || k == "-o") {
            if (i + 1 >= argc) return exit_bad_args;
            a->output = argv[++i];
        } else if (k == "--blocks") {
            if (!need(&v) || v > 0xffffffffull) return exit_bad_args;
            a->blocks = static_cast<unsigned>(v);
        } else if (k == "--lanes") {
            if (!need(&v) || v > 0xffffffffull) return exit_bad_args;
            a->lanes = static_cast<unsigned>(v);
        } else if (k == "--trials") {
            if (!need(&v) || v > 1000) return exit_bad_args;
            a->trials = static_cast<unsigned>(v);
        } else if (k == "--json") {
            a->as_json = true;
        } else if (!k.empty() && k[0] != '-' && a->positional.empty()) {
            a->positional = k;
        } else {
            return exit_bad_args;
        }
    }
    return exit_ok;
}

// proj/tools/xgen.cpp:51-66: raw-le = w/8 little-endian bytes per word, hex
// = w/4 digits, u32-lines = decimal.
void emit(std::ostream& out, const uint64_t* w, size_t n, unsigned bits, const std::string& format) {
    std::string buf;
    if (format == "raw-le") {
        buf.resize(n * (bits / 8));
        char* d = buf.data();
        for (size_t i = 0; i < n; ++i)
            for (unsigned b = 0; b < bits / 8; ++b) *d++ = static_cast<char>((w[i] >> (8 * b)) & 0xff);
    } else {
        buf.reserve(n * 21);
        char tmp[32];
        for (size_t i = 0; i < n; ++i) {
            int len = format == "hex"
                          ? std::snprintf(tmp, sizeof tmp, "%0*llx\n", static_cast<int>(bits / 4),
                                          static_cast<unsigned long long>(w[i]))
                          : std::snprintf(tmp, sizeof tmp, "%llu\n", static_cast<unsigned long long>(w[i]));
            buf.append(tmp, static_cast<size_t>(len));
        }
    }
    out.write(buf.data(), static_cast<std::streamsize>(buf.size()));
}

int fail(const char* msg, int code) {
    std::cerr << "xgen: " << msg << "\n";
    return code;
}

// Fills `per` words for the handle's `n` streams into host memory as uint64
// (block-major), continuing the streams.  The raw (Weyl-ablated) generators
// are 32-bit-or-narrower, so their u32 words are widened here.
int fill_host(xg_ensemble_t h, bool weyl, uint64_t per, uint32_t n, uint64_t* dev,
              uint64_t* host) {
    const size_t cnt = static_cast<size_t>(n) * per;
    if (weyl) {
        int rc = xg_fill_words(h, per, dev, nullptr);
        if (rc) return rc;
        return cudaMemcpy(host, dev, cnt * 8, cudaMemcpyDeviceToHost) == cudaSuccess ? XG_OK : XG_ECUDA;
    }
    uint32_t* d32 = reinterpret_cast<uint32_t*>(dev);
    int rc = xg_fill_raw_u32(h, per, d32, nullptr);
    if (rc) return rc;
    uint32_t* h32 = reinterpret_cast<uint32_t*>(host) + cnt;  // upper half of the buffer
    if (cudaMemcpy(h32, d32, cnt * 4, cudaMemcpyDeviceToHost) != cudaSuccess) return XG_ECUDA;
    for (size_t i = 0; i < cnt; ++i) host[i] = h32[i];
    return XG_OK;
}

int cmd_gen(const Args& a) {
    Gen g;
    if (!find_generator(a.generator, &g))
        return fail(("unknown generator: " + a.generator).c_str(), exit_unknown_generator);
    if (!a.have_count) return fail("--count is required", exit_bad_args);
    const xg_params_t p = g.p;
    const unsigned blocks = std::max(1u, a.blocks);
    const unsigned lanes = std::max(1u, a.lanes);
    if (a.blocks > 1 || a.lanes > 1) {
        if (!g.weyl) return fail("--blocks/--lanes apply only to xorgens generators", exit_bad_args);
        if (a.count % blocks != 0) return fail("--count must be divisible by --blocks", exit_bad_args);
        // BlockEnsemble(params, seed, blocks, lanes) throws out_of_range for
        // lanes == 0 (proj/src/parallel.cpp:90-91) -> exit 65 (xgen.cpp:99-101)
        if (a.lanes == 0) return fail("lane count must be at least 1", exit_lane_range);
    }
    if (lanes > xg_lane_bound(&p)) return fail("lane count exceeds min(s, r - s)", exit_lane_range);

    std::ofstream file;
    std::ostream* out = &std::cout;
    if (!a.output.empty() && a.output != "-") {
        file.open(a.output, std::ios::binary);
        if (!file) return fail(("cannot open output file: " + a.output).c_str(), exit_io);
        out = &file;
    }
    const uint64_t per_block = a.count / blocks;
    if (per_block == 0) return exit_ok;

    // Block-major output: blocks are produced in groups whose whole per-block
    // output fits a 256 MiB staging buffer; a single block longer than that is
    // produced in continuation chunks.
    constexpr uint64_t kStageWords = 1ull << 25;
    const uint64_t chunk = std::min<uint64_t>(per_block, kStageWords);
    const uint32_t group = static_cast<uint32_t>(
        std::max<uint64_t>(1, std::min<uint64_t>(blocks, kStageWords / chunk)));
    uint64_t* dev = nullptr;
    if (cudaMalloc(&dev, static_cast<size_t>(group) * chunk * 8) != cudaSuccess)
        return fail("device allocation failed", exit_io);
    std::vector<uint64_t> host(static_cast<size_t>(group) * chunk);
    int rc = exit_ok;
    for (uint32_t b0 = 0; b0 < blocks && rc == exit_ok; b0 += group) {
        const uint32_t n = std::min(group, blocks - b0);
        xg_ensemble_t h = nullptr;
        int e = xg_ensemble_create(&p, a.seed, b0, n, lanes, 0, nullptr, &h);
        if (e == XG_ERANGE) { rc = fail("lane count exceeds min(s, r - s)", exit_lane_range); break; }
        if (e) { rc = fail(xg_strerror(e), exit_io); break; }
        if (chunk == per_block) {
            e = fill_host(h, g.weyl, per_block, n, dev, host.data());
            if (e) rc = fail(xg_strerror(e), exit_io);
            else emit(*out, host.data(), static_cast<size_t>(n) * per_block, p.w, a.format);
        } else {  // n == 1
            for (uint64_t done = 0; done < per_block && rc == exit_ok; done += chunk) {
                const uint64_t m = std::min(chunk, per_block - done);
                e = fill_host(h, g.weyl, m, 1, dev, host.data());
                if (e) rc = fail(xg_strerror(e), exit_io);
                else emit(*out, host.data(), m, p.w, a.format);
            }
        }
        xg_ensemble_destroy(h);
    }
    cudaFree(dev);
    out->flush();
    if (rc == exit_ok && !*out) return fail("write error", exit_io);
    return rc;
}

// Device-timed RN/s of the fill (CUDA events), one warm-up trial discarded,
// mean/min/max/cv over `trials` like ThroughputReport (proj/src/bench.cpp:19-53).
int cmd_bench(const Args& a) {
    Gen g;
    if (!find_generator(a.generator, &g))
        return fail(("unknown generator: " + a.generator).c_str(), exit_unknown_generator);
    const xg_params_t p = g.p;
    if (p.w != 32) return fail("bench measures the 32-bit generators", exit_bad_args);
    const uint64_t count = a.have_count ? a.count : 100000000ull;
    if (count < 1000000) return fail("throughput trials need count >= 1e6", exit_bad_args);
    if (a.trials < 3) return fail("throughput needs >= 3 trials", exit_bad_args);
    const unsigned blocks = std::max(1u, a.blocks);
    const uint64_t per = count / blocks;
    if (per == 0) return fail("--count must be at least --blocks", exit_bad_args);
    xg_ensemble_t h = nullptr;
    int e = xg_ensemble_create(&p, 0, 0, blocks, xg_lane_bound(&p), 0, nullptr, &h);
    if (e == XG_ERANGE) return fail("blocks out of range", exit_lane_range);
    if (e) return fail(xg_strerror(e), exit_io);
    uint32_t* dev = nullptr;
    if (cudaMalloc(&dev, static_cast<size_t>(blocks) * per * 4) != cudaSuccess) {
        xg_ensemble_destroy(h);
        return fail("device allocation failed", exit_io);
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    std::vector<double> rates;
    uint32_t sink = 0;
    for (unsigned t = 0; t <= a.trials; ++t) {
        cudaEventRecord(e0);
        e = g.weyl ? xg_fill_u32(h, per, dev, nullptr) : xg_fill_raw_u32(h, per, dev, nullptr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        if (e) break;
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        uint32_t last = 0;
        cudaMemcpy(&last, dev + blocks * per - 1, 4, cudaMemcpyDeviceToHost);
        sink ^= last;
        if (t > 0) rates.push_back(static_cast<double>(blocks * per) / (ms * 1e-3));
    }
    cudaFree(dev);
    xg_ensemble_destroy(h);
    if (e) return fail(xg_strerror(e), exit_io);
    double sum = 0, mn = rates[0], mx = rates[0];
    for (double r : rates) { sum += r; mn = std::min(mn, r); mx = std::max(mx, r); }
    const double mean = sum / rates.size();
    double var = 0;
    for (double r : rates) var += (r - mean) * (r - mean);
    const double cv = std::sqrt(var / rates.size()) / mean;
    const std::string id = a.generator + (blocks > 1 ? " x" + std::to_string(blocks) : "");
    if (a.as_json) {
        std::printf("{\"generator\": \"%s\", \"count_per_trial\": %" PRIu64 ", \"trials\": %u, "
                    "\"rn_per_s\": [", id.c_str(), blocks * per, a.trials);
        for (size_t i = 0; i < rates.size(); ++i) std::printf(i ? ", %.6e" : "%.6e", rates[i]);
        std::printf("], \"mean\": %.6e, \"min\": %.6e, \"max\": %.6e, \"cv\": %.6f, \"sink\": %u, "
                    "\"timing\": \"device (CUDA events)\"}\n", mean, mn, mx, cv, sink);
    } else {
        std::printf("%s: mean %.3e RN/s (min %.3e, max %.3e, cv %.2f%%, sink %08x)\n", id.c_str(),
                    mean, mn, mx, 100.0 * cv, sink);
    }
    return exit_ok;
}

// proj/tools/xgen.cpp:236-261
int cmd_params(const Args& a) {
    const std::string id = a.positional.empty() ? a.generator : a.positional;
    Gen g;
    if (!find_generator(id, &g))
        return fail(("unknown generator: " + id).c_str(), exit_unknown_generator);
    const xg_params_t p = g.p;
    std::cout << "generator:    " << id << "\n"
              << "r,s:          " << p.r << "," << p.s << "\n"
              << "a,b,c,d:      " << p.a << "," << p.b << "," << p.c << "," << p.d << "\n"
              << "word bits:    " << p.w << "\n";
    if (g.weyl)
        std::cout << "gamma:        " << p.gamma << "\n"
                  << "omega:        " << p.omega << "\n";
    std::cout << "lane bound:   " << xg_lane_bound(&p) << "\n"
              << "state words:  " << p.r + 1 << "\n"
              << "period:       "
              << (g.weyl ? "~2^" + std::to_string(p.r * p.w + p.w)
                         : "2^" + std::to_string(p.r * p.w) + "-1")
              << "\n"
              << "period note:  " << g.note << "\n"
              << "backend:      " << xg_build_info() << "\n";
    return exit_ok;
}

}  // namespace

// `xgen test ...`: exec the GPU battery CLI (paper_1108_0486_b200/xgen_test.py)
// with the repository root (three levels above this binary) on PYTHONPATH.
int exec_test(int argc, char** argv) {
    char self[PATH_MAX];
    const ssize_t n = readlink("/proc/self/exe", self, sizeof self - 1);
    if (n <= 0) return fail("cannot locate the xgen binary", exit_io);
    self[n] = 0;
    std::string root(self);
    for (int up = 0; up < 3; ++up) root = root.substr(0, root.find_last_of('/'));
    const char* old = getenv("PYTHONPATH");
    const std::string pp = old && *old ? root + ":" + old : root;
    setenv("PYTHONPATH", pp.c_str(), 1);
    std::vector<char*> args;
    static char py[] = "python3", m[] = "-m", mod[] = "paper_1108_0486_b200.xgen_test";
    args.push_back(py);
    args.push_back(m);
    args.push_back(mod);
    for (int i = 2; i < argc; ++i) args.push_back(argv[i]);
    args.push_back(nullptr);
    execvp(py, args.data());
    return fail("cannot run python3 for the battery", exit_io);
}

int main(int argc, char** argv) {
    if (argc >= 2 && std::strcmp(argv[1], "test") == 0) return exec_test(argc, argv);
    Args a;
    if (int rc = parse(argc, argv, &a)) {
        std::cerr << "usage: xgen gen|test|bench|params [options]  (GPU backend)\n";
        return rc;
    }
    if (a.cmd == "gen") return cmd_gen(a);
    if (a.cmd == "bench") return cmd_bench(a);
    if (a.cmd == "params") {
        if (a.positional.empty()) return fail("params needs a generator id", exit_bad_args);
        return cmd_params(a);
    }
    return fail(("unknown subcommand: " + a.cmd).c_str(), exit_bad_args);
}
