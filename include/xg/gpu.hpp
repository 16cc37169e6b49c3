// xg/gpu.hpp -- header-only C++ mirror of the reference xg API over the C ABI
// (include/xg_gpu.h, libxg_gpu.so).  For C++ users of the reference library:
// the same class names, signatures, argument meaning and exception types, in
// namespace xg::gpu, so switching is a namespace change.
//
//   reference (proj/include/xg/...)              this header
//   xg::BlockEnsemble(params, seed, blocks, lanes) xg::gpu::BlockEnsemble(...)
//   BlockEnsemble::generate(per_block, workers)    same signature, same
//                                                  vector<vector<uint64_t>> result
//   xg::XorgensState(params, seed).next_word()     xg::gpu::XorgensState(...)
//   XorgensState::from_raw / logical_buffer /      same
//     weyl_value
//   xg::batch_step(state, lanes)                   xg::gpu::batch_step
//   std::out_of_range / ParamValidationError /     same exception classes
//     std::invalid_argument
//
// `Params` is any struct with the GeneratorParams fields (r, s, a, b, c, d, w,
// omega, gamma), so an xg::GeneratorParams can be passed as is.
#pragma once

#include <cstdint>
#include <algorithm>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "xg_gpu.h"

namespace xg {
namespace gpu {

class ParamValidationError : public std::invalid_argument {
public:
    explicit ParamValidationError(int code)
        : std::invalid_argument(xg_strerror(code)), code_(code - 1) {}
    int code() const noexcept { return code_; }  // ParamError ordinal

private:
    int code_;
};

class CudaError : public std::runtime_error {
public:
    explicit CudaError(int code) : std::runtime_error(xg_strerror(code)), code_(code) {}
    int code() const noexcept { return code_; }

private:
    int code_;
};

inline void check(int rc) {
    if (rc == XG_OK) return;
    if (rc >= 1 && rc <= 6) throw ParamValidationError(rc);
    if (rc == XG_ERANGE) throw std::out_of_range(xg_strerror(rc));
    if (rc == XG_EINVAL || rc == XG_EUNSUPPORTED) throw std::invalid_argument(xg_strerror(rc));
    throw CudaError(rc);
}

template <class Params>
inline xg_params_t to_c(const Params& p) {
    xg_params_t c;
    c.r = p.r; c.s = p.s; c.a = p.a; c.b = p.b; c.c = p.c; c.d = p.d; c.w = p.w;
    c.omega = p.omega;
    c.gamma = p.gamma;
    return c;
}

inline xg_params_t xorgensgp32_params() { return xg_params_xorgensgp32(); }

template <class Params>
inline unsigned lane_bound(const Params& p) {
    const xg_params_t c = to_c(p);
    return xg_lane_bound(&c);
}

class BlockEnsemble {
public:
    template <class Params>
    BlockEnsemble(const Params& params, std::uint64_t base_seed, unsigned num_blocks,
                  unsigned lanes, std::uint64_t first_stream = 0, int device = 0,
                  xg_stream_t stream = nullptr)
        : base_seed_(base_seed), lanes_(lanes), r_(params.r), w_(params.w) {
        const xg_params_t c = to_c(params);
        check(xg_ensemble_create(&c, base_seed, first_stream, num_blocks, lanes, device, stream,
                                 &h_));
        n_ = num_blocks;
    }
    BlockEnsemble(const BlockEnsemble&) = delete;
    BlockEnsemble& operator=(const BlockEnsemble&) = delete;
    BlockEnsemble(BlockEnsemble&& o) noexcept { *this = std::move(o); }
    BlockEnsemble& operator=(BlockEnsemble&& o) noexcept {
        std::swap(h_, o.h_);
        std::swap(nc_, o.nc_);
        n_ = o.n_;
        base_seed_ = o.base_seed_;
        lanes_ = o.lanes_;
        r_ = o.r_;
        w_ = o.w_;
        return *this;
    }
    ~BlockEnsemble() {
        if (h_) xg_ensemble_destroy(h_);
    }

    // proj/include/xg/parallel.hpp:46-47: block-major, continues every block.
    // The rows are reserved by the host threads (no page is touched) and
    // filled tile by tile straight from pinned staging by
    // xg_generate_host_tiles: words cross PCIe once, as u32, and each block's
    // vector<uint64_t> is appended to in one pass (insert widens u32 ->
    // uint64) while the device generates and copies the next tile.
    // `workers` = host threads (0: hardware_concurrency), as the reference's
    // workers (parallel.cpp:115-116); the output never depends on it.
    std::vector<std::vector<std::uint64_t>> generate(std::size_t per_block,
                                                     unsigned workers = 0) {
        std::vector<std::vector<std::uint64_t>> out(n_);
        if (!per_block) return out;
        const xg_ensemble_t hh = h();
        unsigned t = workers ? workers : std::max(1u, std::thread::hardware_concurrency());
        t = std::min(t, 32u);
        {
            const unsigned ta = std::min<unsigned>(t, std::max(1u, n_));
            std::vector<std::thread> pool;
            for (unsigned id = 0; id < ta; ++id)
                pool.emplace_back([&, id] {
                    for (unsigned i = id; i < n_; i += ta) out[i].reserve(per_block);
                });
            for (auto& th : pool) th.join();
        }
        check(xg_generate_host_tiles(hh, per_block, &append_tile, &out, t, nullptr));
        return out;
    }

    // Device-buffer fills (asynchronous on `stream`).
    void fill_u32(std::uint64_t per_block, std::uint32_t* dev, xg_stream_t s = nullptr) {
        check(xg_fill_u32(h(), per_block, dev, s));
    }
    void fill_u64(std::uint64_t per_block, std::uint64_t* dev, xg_stream_t s = nullptr) {
        check(xg_fill_u64(h(), per_block, dev, s));
    }
    void fill_f32(std::uint64_t per_block, float* dev, xg_stream_t s = nullptr) {
        check(xg_fill_f32(h(), per_block, dev, s));
    }
    void fill_f64(std::uint64_t per_block, double* dev, xg_stream_t s = nullptr) {
        check(xg_fill_f64(h(), per_block, dev, s));
    }
    void mc_pi(std::uint64_t samples, std::uint64_t* dev_hits, xg_stream_t s = nullptr) {
        check(xg_mc_pi(h(), samples, dev_hits, s));
    }
    // Fused matrix_rank_test counting (proj/src/stattests/tests.cpp:93-109):
    // adds the (rank 32, 31, <= 30) bins to dev_counts[0..2].
    void rank_test(std::uint64_t matrices, std::uint64_t* dev_counts, xg_stream_t s = nullptr) {
        check(xg_rank_test(h(), matrices, dev_counts, s));
    }
    // linear_complexity_test's per-block Berlekamp-Massey (tests.cpp:128-178):
    // adds the histogram of complexities to dev_hist[0..block_length].
    void linear_complexity_test(unsigned block_length, std::uint64_t blocks, std::uint64_t* dev_hist,
                                xg_stream_t s = nullptr) {
        check(xg_linear_complexity_test(h(), block_length, blocks, dev_hist, s));
    }

    unsigned num_blocks() const noexcept { return n_; }
    unsigned lanes() const noexcept { return lanes_; }
    unsigned word_bits() const noexcept { return w_; }
    std::uint64_t base_seed() const noexcept { return base_seed_; }

    std::pair<std::vector<std::uint64_t>, std::uint64_t> block_state(unsigned i) const {
        std::vector<std::uint64_t> buf(r_);
        std::uint64_t w = 0;
        check(xg_state_export(h(), i, buf.data(), &w));
        return {buf, w};
    }
    void set_block_state(unsigned i, const std::vector<std::uint64_t>& buf, std::uint64_t weyl) {
        if (buf.size() != r_) throw std::invalid_argument("buffer size must equal r");
        check(xg_state_import(h(), i, buf.data(), weyl));
    }
    // Whole-ensemble checkpoint: r window words per block (oldest first) + weyl.
    void export_state(std::vector<std::uint32_t>& window, std::vector<std::uint32_t>& weyl) const {
        window.resize(static_cast<std::size_t>(n_) * r_);
        weyl.resize(n_);
        check(xg_state_export_all(h(), window.data(), weyl.data()));
    }
    void import_state(const std::vector<std::uint32_t>& window, const std::vector<std::uint32_t>& weyl) {
        if (window.size() != static_cast<std::size_t>(n_) * r_ || weyl.size() != n_)
            throw std::invalid_argument("checkpoint size differs from the ensemble");
        check(xg_state_import_all(h(), window.data(), weyl.data()));
    }
    // The C handle, after handing back any next_word words cached here.
    xg_ensemble_t handle() const { return h(); }

protected:
    BlockEnsemble() = default;
    // next_word cache (XorgensState): a view of pinned refill words
    // (xg_next_view); unread ones are returned before any other call.
    struct NextCache {
        const std::uint64_t* p = nullptr;
        std::uint64_t pos = 0, n = 0;
    };
    mutable NextCache nc_;
    void give_back() const {
        if (nc_.n) {
            check(xg_next_return(h_, nc_.n - nc_.pos));
            nc_ = NextCache{};
        }
    }
    xg_ensemble_t h() const {
        give_back();
        return h_;
    }
    // xg_tile_fn of generate(): part `part` of `parts` appends rows
    // stream0 + part, + parts, ... of the tile (a stream's tiles arrive in
    // word order, one thread per row).
    static void append_tile(void* ctx, std::uint64_t stream0, std::uint64_t, std::uint64_t streams,
                            std::uint64_t words, const void* tile, unsigned elem_bytes, unsigned part,
                            unsigned parts) {
        auto& out = *static_cast<std::vector<std::vector<std::uint64_t>>*>(ctx);
        for (std::uint64_t i = part; i < streams; i += parts) {
            auto& row = out[stream0 + i];
            if (elem_bytes == 4) {
                const auto* src = static_cast<const std::uint32_t*>(tile) + i * words;
                row.insert(row.end(), src, src + words);
            } else {
                const auto* src = static_cast<const std::uint64_t*>(tile) + i * words;
                row.insert(row.end(), src, src + words);
            }
        }
    }
    xg_ensemble_t h_ = nullptr;
    unsigned n_ = 0;
    std::uint64_t base_seed_ = 0;
    unsigned lanes_ = 0;
    unsigned r_ = 0;
    unsigned w_ = 32;
};

// One serial stream (proj/include/xg/xorgens.hpp:20-96), served from device refills.
class XorgensState : public BlockEnsemble {
public:
    template <class Params>
    XorgensState(const Params& params, std::uint64_t seed, int device = 0)
        : BlockEnsemble(params, seed, 1u, lane_bound(params), 0, device) {}

    template <class Params>
    static XorgensState from_raw(const Params& params, const std::vector<std::uint64_t>& buffer,
                                 std::uint64_t weyl, int device = 0) {
        if (buffer.size() != params.r) throw std::invalid_argument("buffer size must equal r");
        const xg_params_t c = to_c(params);
        XorgensState st;
        check(xg_ensemble_create_from_raw(&c, 1, buffer.data(), &weyl, device, nullptr, &st.h_));
        st.n_ = 1;
        st.r_ = params.r;
        st.w_ = params.w;
        st.lanes_ = lane_bound(params);
        return st;
    }

    // Inline on the hot path: one load from the pinned refill slot.
    std::uint64_t next_word() {
        if (nc_.pos == nc_.n) refill();
        return nc_.p[nc_.pos++];
    }
    std::uint64_t next_u64() {
        if (w_ == 64) return next_word();
        const std::uint64_t lo = next_word();
        return lo | (next_word() << 32);
    }
    std::vector<std::uint64_t> logical_buffer() const { return block_state(0).first; }
    std::uint64_t weyl_value() const { return block_state(0).second; }

private:
    XorgensState() = default;
    void refill() {
        nc_ = NextCache{};
        check(xg_next_view(h_, &nc_.p, &nc_.n));
    }
};

// proj/src/parallel.cpp:8-42
inline std::vector<std::uint64_t> batch_step(XorgensState& st, unsigned lanes) {
    if (lanes == 0 || lanes > st.lanes()) throw std::out_of_range("lane count exceeds min(s, r - s)");
    std::vector<std::uint64_t> out(lanes);
    for (auto& v : out) v = st.next_word();
    return out;
}

// XorgensSource (proj/include/xg/stream.hpp:25-35) over device refills.
// Templated on the consumer's WordSource base so this header needs no
// reference header: `xg::gpu::XorgensSource<xg::WordSource> src(params, seed)`
// plugs into anything that takes an `xg::WordSource&` (the battery, bench).
template <class WordSourceBase>
class XorgensSource final : public WordSourceBase {
public:
    template <class Params>
    XorgensSource(const Params& params, std::uint64_t seed, int device = 0)
        : state_(params, seed, device) {}
    std::uint64_t next() override { return state_.next_word(); }
    unsigned word_bits() const override { return state_.word_bits(); }
    XorgensState& state() noexcept { return state_; }

private:
    XorgensState state_;
};

}  // namespace gpu
}  // namespace xg
