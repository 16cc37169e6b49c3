/*
 * xg_gpu.h -- C ABI of the B200-native xorgensGP generator (libxg_gpu.so).
 *
 * A drop-in for the reference CPU library's generation path.  Each entry point
 * names the reference interface it replaces (paths relative to the reference
 * tree).  Plain C types only: no C++, no CUDA or torch headers are needed to
 * call it.  `xg_stream_t` is ABI-identical to `cudaStream_t`
 * (`struct CUstream_st*`); NULL means the legacy default stream.
 *
 * All generation calls are asynchronous on the caller's stream and write to
 * caller-owned device memory, except xg_generate_host / xg_next_* /
 * xg_state_export / xg_state_import, which synchronise.
 *
 * Error model (no exceptions cross the ABI):
 *   XG_OK                    success
 *   1..6                     1 + ParamError ordinal, same check order as
 *                            xg::check_params (proj/src/params.cpp:22-37)
 *   XG_ERANGE                std::out_of_range in the reference (lanes outside
 *                            [1, lane_bound], zero streams, stream index)
 *   XG_EINVAL                std::invalid_argument (NULL / misaligned buffer,
 *                            size overflow, wrong handle kind)
 *   XG_EUNSUPPORTED          the call is not defined for these parameters: the
 *                            u64/f32/f64/MC conventions and whole-ensemble
 *                            checkpoints need the w = 32, r = 128,
 *                            lane_bound >= 32 kernels; 32-bit outputs need
 *                            w <= 32; r > 16384 is not supported
 *   XG_ECUDA / XG_ENOMEM     CUDA runtime failure / device allocation failure
 */
#ifndef XG_GPU_H
#define XG_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* xg_stream_t;
typedef struct xg_ensemble* xg_ensemble_t;

enum {
    XG_OK = 0,
    XG_EPARAM_BAD_WORD_SIZE = 1,       /* ParamError::bad_word_size */
    XG_EPARAM_S_OUT_OF_RANGE = 2,      /* ParamError::s_out_of_range */
    XG_EPARAM_GCD_NOT_ONE = 3,         /* ParamError::gcd_not_one */
    XG_EPARAM_SHIFT_OUT_OF_RANGE = 4,  /* ParamError::shift_out_of_range */
    XG_EPARAM_GAMMA_OUT_OF_RANGE = 5,  /* ParamError::gamma_out_of_range */
    XG_EPARAM_EVEN_WEYL_INCREMENT = 6, /* ParamError::even_weyl_increment */
    XG_ERANGE = 16,
    XG_EINVAL = 17,
    XG_EUNSUPPORTED = 18,
    XG_ECUDA = 19,
    XG_ENOMEM = 20
};

/* GeneratorParams, same field order and meaning
 * (proj/include/xg/params.hpp:17-29). */
typedef struct {
    unsigned r, s, a, b, c, d, w;
    uint64_t omega;
    unsigned gamma;
} xg_params_t;

/* ---- parameters (host only, no GPU needed) ------------------------------ */

/* check_params (proj/include/xg/params.hpp:52, proj/src/params.cpp:22-37):
 * XG_OK or 1 + ParamError. */
int xg_params_check(const xg_params_t* p);
/* to_string(ParamError) (proj/src/params.cpp:7-18) and the ABI codes. */
const char* xg_strerror(int code);
/* lane_bound (proj/include/xg/params.hpp:59-61): min(s, r - s). */
unsigned xg_lane_bound(const xg_params_t* p);
/* recommended_weyl_increment (proj/src/params.cpp:53-62); 0 for a bad w
 * (the reference throws ParamValidationError(bad_word_size)). */
uint64_t xg_recommended_weyl_increment(unsigned w);
/* default_output_shift (proj/include/xg/params.hpp:77). */
unsigned xg_default_output_shift(unsigned w);
/* Shipped sets (proj/src/params.cpp:83-86). */
xg_params_t xg_params_xorgensgp32(void);
xg_params_t xg_params_tiny_r2w8(void);
xg_params_t xg_params_tiny_r2w16(void);
xg_params_t xg_params_tiny_r4w16(void);
/* XG_OK when the GPU can generate `p` (every valid set with r <= 16384), else
 * the check_params code or XG_EUNSUPPORTED. */
int xg_gpu_supported(const xg_params_t* p);
/* 1 when `p` runs on the register-window kernels (w = 32, r = 128,
 * lane_bound >= 32: xorgensgp32 and every set shaped like it), 0 when it runs
 * on the general-parameter kernels (correct for any valid set, not tuned). */
int xg_fast_path(const xg_params_t* p);

/* ---- ensembles ----------------------------------------------------------- */

/* BlockEnsemble(params, base_seed, num_blocks, lanes)
 * (proj/include/xg/parallel.hpp:35-40, proj/src/parallel.cpp:84-95) plus the
 * seeding constructor XorgensState(params, seed) (proj/src/xorgens.cpp:19-32)
 * for every block, run on the device.  Stream g of the handle is seeded with
 * base_seed + first_stream + g (uint64 wrap); first_stream lets a multi-GPU
 * job give each device a disjoint slice of one global ensemble.  `lanes` is
 * validated like the reference (XG_ERANGE unless 1 <= lanes <= lane_bound);
 * the output never depends on it. */
int xg_ensemble_create(const xg_params_t* p, uint64_t base_seed, uint64_t first_stream,
                       uint32_t num_streams, unsigned lanes, int device, xg_stream_t stream,
                       xg_ensemble_t* out);
/* XorgensState::from_raw (proj/include/xg/xorgens.hpp:33-35,
 * proj/src/xorgens.cpp:34-38) for num_streams streams: buffers holds
 * num_streams * r words, each stream's r most recent values oldest first;
 * words are masked to w bits, no warm-up, no zero check. */
int xg_ensemble_create_from_raw(const xg_params_t* p, uint32_t num_streams,
                                const uint64_t* buffers, const uint64_t* weyls, int device,
                                xg_stream_t stream, xg_ensemble_t* out);
int xg_ensemble_destroy(xg_ensemble_t h);
/* num_blocks() / base_seed() / lanes() (proj/include/xg/parallel.hpp:49-51). */
int xg_ensemble_info(xg_ensemble_t h, uint32_t* num_streams, uint64_t* base_seed,
                     uint64_t* first_stream, unsigned* lanes, int* device);

/* ---- generation (device buffers, asynchronous) --------------------------- */

/* Calls on one stream of >= 2^20 words, or on 2 .. 700 streams of >= 2^18
 * words each, of a register-window set (w = 32, r = 128, lane_bound >= 32) are
 * generated as up
 * to 1024 segments in parallel, their start states computed by GF(2)
 * jump-ahead (csrc/xg_jump.cuh): the same words, at ensemble speed instead of
 * one warp per stream.  The first such call per parameter set and segment
 * length builds the jump tables on the calling stream and synchronises it
 * (tens of ms); capture such calls into CUDA graphs only after a first
 * eager call. */

/* BlockEnsemble::generate(per_block) (proj/src/parallel.cpp:97-135):
 * dev_out[g * per_stream + k] = word k of stream g, continuing each stream
 * from the handle's state (a second call continues where the first stopped).
 * Byte-identical to `xgen gen --format raw-le --blocks`
 * (proj/tools/xgen.cpp:51-57,94-98). */
int xg_fill_u32(xg_ensemble_t h, uint64_t per_stream, uint32_t* dev_out, xg_stream_t stream);
/* Every word as a uint64 (the w-bit value zero-extended): exactly the element
 * type and layout of BlockEnsemble::generate()'s result
 * (proj/include/xg/parallel.hpp:46-47).  Works for every parameter set,
 * including w = 64. */
int xg_fill_words(xg_ensemble_t h, uint64_t per_stream, uint64_t* dev_out, xg_stream_t stream);
/* Two consecutive words per value, lo = first: value = w[2k] | w[2k+1] << 32
 * (the raw-le stream read as little-endian uint64).  Not in the reference. */
int xg_fill_u64(xg_ensemble_t h, uint64_t per_stream, uint64_t* dev_out, xg_stream_t stream);
/* The Weyl-ablated linear stream: RawXorgens::next() = step_linear()
 * (proj/include/xg/baselines.hpp:60-71, registry id "xorgens-raw",
 * proj/src/registry.cpp:29-30) -- same seeding, output x_i, and the Weyl
 * accumulator is left unchanged.  Same layout as xg_fill_u32. */
int xg_fill_raw_u32(xg_ensemble_t h, uint64_t per_stream, uint32_t* dev_out, xg_stream_t stream);
/* Uniform [0,1): f32 = (word >> 8) * 2^-24, one word per value.  Exact. */
int xg_fill_f32(xg_ensemble_t h, uint64_t per_stream, float* dev_out, xg_stream_t stream);
/* Uniform [0,1): f64 = (u64 >> 11) * 2^-53 with u64 as in xg_fill_u64. Exact. */
int xg_fill_f64(xg_ensemble_t h, uint64_t per_stream, double* dev_out, xg_stream_t stream);
/* Fused in-register Monte Carlo pi.  samples_per_stream must be a multiple
 * of 32 (XG_EINVAL otherwise): each stream supplies 2*samples_per_stream words,
 * sample m being the consecutive pair (w[2m], w[2m+1]) -- the pair one lane
 * of the pair-lane kernel holds after a double step, so no word moves between
 * lanes.  Each word read as a signed 32-bit coordinate in
 * [-2^31, 2^31); hit iff x^2 + y^2 < 2^62 (exact integer test, the unit disc
 * in the square [-1, 1)^2, P(hit) = pi/4).  The hit count over all streams is ADDED to
 * *dev_hits (a device uint64).  No HBM traffic. */
int xg_mc_pi(xg_ensemble_t h, uint64_t samples_per_stream, uint64_t* dev_hits,
             xg_stream_t stream);

/* Fused GF(2) matrix-rank test -- the reference's matrix_rank_test
 * (proj/src/stattests/tests.cpp:81-126, M = 32) run inside the generator:
 * each stream supplies 32*matrices_per_stream words continuing its stream,
 * every 32 consecutive words are one 32 x 32 matrix (row i = word i, bits MSB
 * first as BitSource reads them, proj/include/xg/stream.hpp:95-112), and the
 * ranks are binned (32, 31, <= 30) and ADDED to dev_counts[0..2] (device
 * uint64[3]).  The chi-square statistic and p-value follow on the host from
 * the counts.  No HBM traffic.  w = 32 sets with r - s < 64 (the pair-lane
 * kernel); XG_EUNSUPPORTED otherwise.  Replaces tests.cpp:81-126 (the
 * counting loop; rank: proj/src/stattests/gf2.cpp:8-33). */
int xg_rank_test(xg_ensemble_t h, uint64_t matrices_per_stream, uint64_t* dev_counts,
                 xg_stream_t stream);

/* Linear complexity test (the reference's linear_complexity_test,
 * proj/src/stattests/tests.cpp:128-178): each stream supplies
 * ceil(block_length * blocks_per_stream / 32) words continuing its stream,
 * read as a BitSource reads them (MSB first), cut into blocks of block_length
 * bits; the Berlekamp-Massey linear complexity L of every block
 * (proj/src/stattests/gf2.cpp:62-110) is histogrammed: dev_hist[L] += 1
 * (device uint64[block_length + 1]).  The reference's bins, chi-square and
 * p-value follow on the host from the histogram.  1 <= block_length <= 2^18
 * (XG_EINVAL otherwise; blocks up to 1023 bits keep the polynomials in
 * registers, longer ones in shared memory); w = 32 sets (XG_EUNSUPPORTED
 * otherwise). */
int xg_linear_complexity_test(xg_ensemble_t h, unsigned block_length, uint64_t blocks_per_stream,
                              uint64_t* dev_hist, xg_stream_t stream);

/* Berlekamp-Massey (proj/src/stattests/gf2.cpp:62-110) of `count` device
 * bit sequences of nbits bits each (1 <= nbits <= 2^18), sequence q starting
 * at word q * stride_words, bits MSB first (bit i = bit 31 - i % 32 of word
 * i / 32): dev_L[q] = its linear complexity.  One warp per sequence. */
int xg_berlekamp_massey(const uint32_t* dev_seqs, uint64_t nbits, uint32_t count,
                        uint64_t stride_words, uint32_t* dev_L, xg_stream_t stream);
/* matrix_rank_test's counting loop (tests.cpp:93-109) over a device word
 * buffer: matrix k = words [32k, 32k+32), row i = word i (bits MSB first);
 * dev_counts[0..2] += matrices of rank 32, 31, <= 30.  For any word source
 * (file words, the raw stream, sets xg_rank_test does not take). */
int xg_rank_words(const uint32_t* dev_words, uint64_t matrices, uint64_t* dev_counts,
                  xg_stream_t stream);
/* linear_complexity_test's per-block Berlekamp-Massey (tests.cpp:128-178)
 * over a device word buffer read MSB first: `blocks` blocks of block_length
 * bits (<= 2^18) from bit 0; dev_hist[L] += 1 per block (XG_EINVAL if the
 * buffer holds fewer than block_length * blocks bits). */
int xg_lc_words(const uint32_t* dev_words, uint64_t nwords, unsigned block_length, uint64_t blocks,
                uint64_t* dev_hist, xg_stream_t stream);
/* w-bit words (w = 8, 16, 32; each in the low bits of a uint32, e.g. a fill of
 * a tiny set) -> the bit stream BitSource reads (w bits per word, MSB first,
 * proj/include/xg/stream.hpp:95-110) packed into ceil(n w / 32) uint32 words,
 * the input for the counting calls below; left_align = 1: n words, each
 * shifted to the top of its 32 bits (birthday spacings' draws). */
int xg_pack_words(const uint32_t* dev_in, uint64_t n, unsigned w, int left_align, uint32_t* dev_out,
                  xg_stream_t stream);
/* Counting loops of monobit and runs_test (proj/src/stattests/tests.cpp:33-79)
 * over the first nbits bits of a device word buffer read MSB first (as
 * BitSource reads 32-bit words): dev_out2[0] += ones, dev_out2[1] +=
 * adjacent-bit transitions (runs = 1 + transitions). */
int xg_bits_ones_runs(const uint32_t* dev_words, uint64_t nbits, uint64_t* dev_out2,
                      xg_stream_t stream);
/* Birthday spacings (tests.cpp:175-212) over `rounds` consecutive groups of
 * n_draws device words: each round sorts the words' top t_bits bits and their
 * n_draws - 1 spacings and counts equal neighbours; *dev_dup += the total.
 * 2 <= n_draws <= 8192, 1 <= t_bits <= 32 (XG_EINVAL otherwise). */
int xg_birthday_duplicates(const uint32_t* dev_words, uint32_t n_draws, uint32_t rounds,
                           unsigned t_bits, uint64_t* dev_dup, xg_stream_t stream);
/* The handle-less calls above (Berlekamp-Massey, ones/runs, birthday) and
 * xg_digest_u32 run on the device that owns their input pointer, whatever
 * device is current (XG_EINVAL for a host or unregistered pointer). */

/* Row digests for parity checks: for each row r of a (rows x per_row)
 * row-major buffer of 32-bit elements e_k, dev_xor[r] = xor of e_k,
 * dev_sum[r] = sum e_k, dev_wsum[r] = sum e_k * (k + 1) (mod 2^64).  Floats
 * are digested through their bit patterns (f64 rows as 2 * per_row u32
 * halves).  Golden digests of the reference's streams in the same form:
 * tests/golden/full_size.json. */
int xg_digest_u32(const uint32_t* dev_words, uint64_t rows, uint64_t per_row, uint32_t* dev_xor,
                  uint64_t* dev_sum, uint64_t* dev_wsum, xg_stream_t stream);
/* Advance every stream by `words` without storing (discard).  On a
 * one-stream handle of a register-window set, words >= 2^20 jump: O(log words)
 * GF(2) products by cached powers of the transition matrix, no generation. */
int xg_skip(xg_ensemble_t h, uint64_t words, xg_stream_t stream);

/* ---- host-facing calls (synchronise) -------------------------------------- */

/* BlockEnsemble::generate into HOST memory: same layout as xg_fill_u32,
 * generated in stream chunks and copied device->host with the copies
 * overlapping generation.  host_out should be pinned for full speed. */
int xg_generate_host(xg_ensemble_t h, uint64_t per_stream, uint32_t* host_out,
                     xg_stream_t stream);
/* Uniform f32 / f64 values (DESIGN.md section 3 conventions) into host
 * memory, block-major like xg_generate_host, fused conversion on the device;
 * w = 32 register-window sets (XG_EUNSUPPORTED otherwise). */
int xg_generate_host_f32(xg_ensemble_t h, uint64_t per_stream, float* host_out, xg_stream_t stream);
int xg_generate_host_f64(xg_ensemble_t h, uint64_t per_stream, double* host_out, xg_stream_t stream);
/* BlockEnsemble::generate into the reference's own result layout: rows[g]
 * points at per_stream uint64 elements for stream g (e.g. the data() of
 * vector<uint64_t> per block).  Words cross PCIe as u32 (w <= 32) through
 * pinned staging and are widened into the rows by host threads while the next
 * tile is generated and copied. */
int xg_generate_host_rows(xg_ensemble_t h, uint64_t per_stream, uint64_t* const* rows,
                          xg_stream_t stream);
/* generate() handed to the caller tile by tile, straight from pinned
 * staging: for each tile (streams [stream0, stream0 + streams), words
 * [word0, word0 + words) of each, row-major, elements of elem_bytes = 4 for
 * w <= 32 else 8), fn is called once on each of `parts` host threads (part =
 * 0 .. parts-1, threads = 0: hardware_concurrency up to 32) and may split the
 * tile between them; the next tile is generated and copied meanwhile.  A
 * stream's tiles arrive in word order, so fn can append (what
 * xg::gpu::BlockEnsemble::generate does: vector<uint64_t>::insert into
 * reserved rows, one pass over host memory). */
typedef void (*xg_tile_fn)(void* ctx, uint64_t stream0, uint64_t word0, uint64_t streams,
                           uint64_t words, const void* tile, unsigned elem_bytes, unsigned part,
                           unsigned parts);
int xg_generate_host_tiles(xg_ensemble_t h, uint64_t per_stream, xg_tile_fn fn, void* ctx,
                           unsigned threads, xg_stream_t stream);
/* The same with every word in the reference's uint64 container -- exactly
 * the element type of generate()'s result; any w, including 64. */
int xg_generate_host_words(xg_ensemble_t h, uint64_t per_stream, uint64_t* host_out,
                           xg_stream_t stream);
/* XorgensState::next_word (proj/include/xg/xorgens.hpp:58-62) on a
 * one-stream handle: the w-bit word in a uint64, served from device-generated
 * refills; interleaving with fills / exports keeps the exact serial stream.
 * Refills are double-buffered: two pinned slots of 2^16 words, the next one
 * generated and copied on a private stream while this one is served. */
int xg_next_word(xg_ensemble_t h, uint64_t* out);
/* Zero-copy batch form of next_word (what xg::gpu::XorgensState inlines):
 * *words points at the next *count unserved words of the stream in pinned host
 * memory, each in a uint64 as next_word returns it, valid until the next call
 * on the handle.  The words count as served; words the caller did not use
 * are handed back with xg_next_return(h, unread) before any other call, so
 * the next word / fill / export continues right after the last word used. */
int xg_next_view(xg_ensemble_t h, const uint64_t** words, uint64_t* count);
int xg_next_return(xg_ensemble_t h, uint64_t unread);
/* next_word as uint32 (w <= 32). */
int xg_next_u32(xg_ensemble_t h, uint32_t* out);
/* w = 32: two words, lo = first; w = 64: one word. */
int xg_next_u64(xg_ensemble_t h, uint64_t* out);
/* logical_buffer() + weyl_value() of stream `index`
 * (proj/include/xg/xorgens.hpp:72-76): r words oldest first. */
int xg_state_export(xg_ensemble_t h, uint32_t index, uint64_t* buffer, uint64_t* weyl);
/* Replace stream `index` with from_raw(params, buffer, weyl). */
int xg_state_import(xg_ensemble_t h, uint32_t index, const uint64_t* buffer, uint64_t weyl);

/* Checkpoint / resume of a whole ensemble: the device
 * state of every stream, host_window[g*r + i] = logical_buffer()[i] of stream
 * g (oldest first) and host_weyl[g] = weyl_value(), as 32-bit words (w = 32).
 * Importing into an ensemble with the same parameters and stream count
 * resumes every stream exactly. */
int xg_state_export_all(xg_ensemble_t h, uint32_t* host_window, uint32_t* host_weyl);
int xg_state_import_all(xg_ensemble_t h, const uint32_t* host_window, const uint32_t* host_weyl);

/* ---- jump-ahead support (host only, no GPU) ------------------------------ */

/* The minimal polynomial m(x) of a register-window set's one-word transition
 * over GF(2) -- the polynomial the jump-ahead path reduces x^n by
 * (csrc/xg_jump.cuh): Berlekamp-Massey over the raw stream, degree 4096
 * required and checked.  coeffs64[k / 64] bit k % 64 = coefficient of x^k for
 * k < 4096 (64 words; the x^4096 term is implied).  XG_EUNSUPPORTED for the
 * general-parameter sets or a degree below 4096 (jumps then use powers of
 * the transition matrix). */
int xg_jump_minpoly(const xg_params_t* p, uint64_t* coeffs64);

/* ---- multi-GPU partitioner (host only) ----------------------------------- */

/* Contiguous, balanced split of global streams [0, total) over `world`
 * devices: rank k gets [floor(k*total/world), floor((k+1)*total/world)).
 * Mirrors the block striping of proj/src/parallel.cpp:115-134 lifted to
 * devices; the union of all ranks' fills is the single-device fill. */
int xg_partition(uint64_t total_streams, uint32_t world, uint32_t rank, uint64_t* first,
                 uint32_t* count);

/* Launch bookkeeping: number of kernels this library has launched since load
 * (bench.py reports it as gpu_launches). */
uint64_t xg_kernel_launches(void);
const char* xg_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* XG_GPU_H */
