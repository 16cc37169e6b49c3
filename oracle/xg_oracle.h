/*
 * xg_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C) of the reference xorgens / xorgensGP generation
 * path, used as the parity checker for the CUDA path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  Nothing in paper_1108_0486_b200/ links or calls it.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * the reference tree, proj/...).  Parity of the restatement itself is pinned by
 * tests/test_oracle.py against the reference's own known-answer vectors
 * (proj/tests/test_xorgens.cpp:163-173, proj/tests/golden/gen_gp32_seed42_count4.hex)
 * and against oracle/_ref (the reference sources compiled unmodified).
 *
 * Conversions (u64 / f32 / f64 / Monte Carlo) do not exist in the reference;
 * they are the conventions defined in DESIGN.md section 3 and are restated here
 * exactly as the kernels implement them.
 */
#ifndef XG_ORACLE_H
#define XG_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XGO_MAX_R 1024u

/* proj/include/xg/params.hpp:17-29 (same field order) */
typedef struct {
    unsigned r, s, a, b, c, d, w;
    uint64_t omega;
    unsigned gamma;
} xgo_params;

/* proj/include/xg/xorgens.hpp:90-95: params, mask, circular buffer, idx, weyl */
typedef struct {
    xgo_params p;
    uint64_t mask;
    uint64_t x[XGO_MAX_R];
    unsigned idx;
    uint64_t weyl;
} xgo_state;

/* 0 = valid, else 1 + ParamError ordinal (proj/include/xg/params.hpp:31-38). */
int xgo_check_params(const xgo_params* p);
unsigned xgo_lane_bound(const xgo_params* p);
uint64_t xgo_recommended_weyl_increment(unsigned w); /* 0 when w is invalid */
xgo_params xgo_xorgensgp32_params(void);
xgo_params xgo_tiny_r2w8_params(void);
xgo_params xgo_tiny_r2w16_params(void);
xgo_params xgo_tiny_r4w16_params(void);

uint64_t xgo_splitmix64(uint64_t* state);

/* Serial generator.  Return 0 on success, else an oracle error (<0) or 1+ParamError. */
int xgo_seed(xgo_state* st, const xgo_params* p, uint64_t seed);
int xgo_from_raw(xgo_state* st, const xgo_params* p, const uint64_t* buffer, uint64_t weyl);
uint64_t xgo_step_linear(xgo_state* st);
uint64_t xgo_weyl_next(xgo_state* st);
uint64_t xgo_next_word(xgo_state* st);
void xgo_logical_buffer(const xgo_state* st, uint64_t* out);
uint64_t xgo_weyl_value(const xgo_state* st);
size_t xgo_state_size(void);

/* Lane batching: -1 when lanes is out of range (std::out_of_range). */
int xgo_batch_step(xgo_state* st, unsigned lanes, uint64_t* out);
int xgo_unsynchronized_batch(xgo_state* st, unsigned lanes, uint64_t* out);

/* Words 0..n-1 of stream `seed`, as 32-bit values (w <= 32). */
int xgo_stream_u32(const xgo_params* p, uint64_t seed, uint64_t n, uint32_t* out);

/* Block ensemble over an array of states (proj/src/parallel.cpp:84-135).
 * states[g] is seeded with base_seed + first_stream + g (uint64 wrap).  */
int xgo_ensemble_seed(xgo_state* states, const xgo_params* p, uint64_t base_seed,
                      uint64_t first_stream, uint32_t num_streams, int threads);
/* Block-major fill, continuing each state: out[g*per_stream + k]. */
int xgo_ensemble_fill_u32(xgo_state* states, uint32_t num_streams, uint64_t per_stream,
                          uint32_t* out, int threads);
/* Words in the reference's uint64 container (any w). */
int xgo_ensemble_fill_words(xgo_state* states, uint32_t num_streams, uint64_t per_stream,
                            uint64_t* out, int threads);
/* Weyl-ablated linear stream (RawXorgens, proj/include/xg/baselines.hpp:60-71). */
int xgo_ensemble_fill_raw_u32(xgo_state* states, uint32_t num_streams, uint64_t per_stream,
                              uint32_t* out, int threads);
int xgo_ensemble_fill_f32(xgo_state* states, uint32_t num_streams, uint64_t per_stream,
                          float* out, int threads);
int xgo_ensemble_fill_f64(xgo_state* states, uint32_t num_streams, uint64_t per_stream,
                          double* out, int threads);
/* Monte Carlo pi: per-stream hit counts over samples_per_stream samples
 * (a multiple of 32; sample m is the consecutive pair (w[2m], w[2m+1])). */
int xgo_ensemble_mc_pi(xgo_state* states, uint32_t num_streams, uint64_t samples_per_stream,
                       uint64_t* hits_per_stream, int threads);
/* Matrix-rank bins (rank 32, 31, <= 30) of the next matrices_per_stream
 * 32 x 32 matrices of each stream (32 words each), 3 counts per stream. */
int xgo_ensemble_rank_counts(xgo_state* states, uint32_t num_streams, uint64_t matrices_per_stream,
                             uint64_t* counts3_per_stream, int threads);
unsigned xgo_gf2_rank32(const uint32_t* rows);
/* Per-stream checksums of the next n words (continuing): xor and
 * sum_k word_k*(k+1) mod 2^64. */
int xgo_ensemble_checksums(xgo_state* states, uint32_t num_streams, uint64_t n,
                           uint32_t* xor_out, uint64_t* wsum_out, int threads);

/* Conventions. */
float xgo_u32_to_f32(uint32_t u);
double xgo_u32pair_to_f64(uint32_t lo, uint32_t hi);
uint64_t xgo_u32pair_to_u64(uint32_t lo, uint32_t hi);
int xgo_mc_hit(uint32_t x, uint32_t y);

#ifdef __cplusplus
}
#endif
#endif
