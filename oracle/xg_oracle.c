/*
 * xg_oracle.c -- TEST INFRASTRUCTURE ONLY (see xg_oracle.h).
 *
 * Plain-C restatement of the reference CPU xorgens path.  Each function names
 * the reference lines it follows; paths are relative to the reference tree.
 * Never linked into the product library.
 */
#include "xg_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- parameters: proj/src/params.cpp ---------------------------------- */

static unsigned gcd_u(unsigned a, unsigned b) {
    while (b) {
        unsigned t = a % b;
        a = b;
        b = t;
    }
    return a;
}

/* proj/src/params.cpp:22-37 -- same check order, codes = 1 + ParamError
 * ordinal (proj/include/xg/params.hpp:31-38). */
int xgo_check_params(const xgo_params* p) {
    if (p->w != 8 && p->w != 16 && p->w != 32 && p->w != 64) return 1;
    if (p->s == 0 || p->s >= p->r) return 2;
    if (gcd_u(p->r, p->s) != 1) return 3;
    const unsigned sh[4] = {p->a, p->b, p->c, p->d};
    for (int i = 0; i < 4; ++i)
        if (sh[i] == 0 || sh[i] >= p->w) return 4;
    if (p->gamma == 0 || p->gamma >= p->w) return 5;
    if ((p->omega & 1u) == 0) return 6;
    return 0;
}

/* proj/include/xg/params.hpp:59-61 */
unsigned xgo_lane_bound(const xgo_params* p) {
    return p->s < p->r - p->s ? p->s : p->r - p->s;
}

/* proj/src/params.cpp:53-62 */
uint64_t xgo_recommended_weyl_increment(unsigned w) {
    switch (w) {
    case 8: return 159u;
    case 16: return 40503u;
    case 32: return UINT64_C(2654435769);
    case 64: return UINT64_C(11400714819323198485);
    default: return 0;
    }
}

/* proj/src/params.cpp:66-79 (default gamma = w/2, proj/include/xg/params.hpp:77) */
static xgo_params make_params(unsigned r, unsigned s, unsigned a, unsigned b, unsigned c,
                              unsigned d, unsigned w) {
    xgo_params p;
    p.r = r; p.s = s; p.a = a; p.b = b; p.c = c; p.d = d; p.w = w;
    p.omega = xgo_recommended_weyl_increment(w);
    p.gamma = w / 2;
    return p;
}

/* proj/src/params.cpp:83-86 */
xgo_params xgo_xorgensgp32_params(void) { return make_params(128, 65, 15, 14, 12, 17, 32); }
xgo_params xgo_tiny_r2w8_params(void) { return make_params(2, 1, 1, 1, 5, 7, 8); }
xgo_params xgo_tiny_r2w16_params(void) { return make_params(2, 1, 1, 1, 6, 11, 16); }
xgo_params xgo_tiny_r4w16_params(void) { return make_params(4, 3, 1, 2, 5, 8, 16); }

/* ---- serial generator: proj/include/xg/xorgens.hpp, proj/src/xorgens.cpp */

/* proj/include/xg/mix.hpp:9-14 */
uint64_t xgo_splitmix64(uint64_t* state) {
    uint64_t z = (*state += UINT64_C(0x9e3779b97f4a7c15));
    z = (z ^ (z >> 30)) * UINT64_C(0xbf58476d1ce4e5b9);
    z = (z ^ (z >> 27)) * UINT64_C(0x94d049bb133111eb);
    return z ^ (z >> 31);
}

/* proj/include/xg/params.hpp:26-28 */
static uint64_t mask_of(unsigned w) {
    return w >= 64 ? ~UINT64_C(0) : ((UINT64_C(1) << w) - 1);
}

/* proj/include/xg/xorgens.hpp:13-18 */
static inline uint64_t xorshift_transform(uint64_t x, unsigned l, unsigned r, uint64_t mask) {
    uint64_t t = (x ^ (x << l)) & mask;
    return t ^ (t >> r);
}

static int state_init(xgo_state* st, const xgo_params* p) {
    int e = xgo_check_params(p);
    if (e) return e;
    if (p->r > XGO_MAX_R) return -2;
    memset(st, 0, sizeof(*st));
    st->p = *p;
    st->mask = mask_of(p->w);
    return 0;
}

/* proj/src/xorgens.cpp:19-32: r SplitMix draws into the buffer, one for the
 * Weyl accumulator, zero guard, then 4r discarded outputs. */
int xgo_seed(xgo_state* st, const xgo_params* p, uint64_t seed) {
    int e = state_init(st, p);
    if (e) return e;
    uint64_t mix = seed;
    int any_nonzero = 0;
    for (unsigned i = 0; i < p->r; ++i) {
        st->x[i] = xgo_splitmix64(&mix) & st->mask;
        any_nonzero |= st->x[i] != 0;
    }
    st->weyl = xgo_splitmix64(&mix) & st->mask;
    if (!any_nonzero) st->x[0] = UINT64_C(0x9e3779b97f4a7c15) & st->mask;
    for (unsigned i = 0; i < 4 * p->r; ++i) xgo_next_word(st);
    return 0;
}

/* proj/src/xorgens.cpp:9-17,34-38: masked copy, idx = 0, no warm-up. */
int xgo_from_raw(xgo_state* st, const xgo_params* p, const uint64_t* buffer, uint64_t weyl) {
    int e = state_init(st, p);
    if (e) return e;
    for (unsigned i = 0; i < p->r; ++i) st->x[i] = buffer[i] & st->mask;
    st->weyl = weyl & st->mask;
    return 0;
}

/* proj/include/xg/xorgens.hpp:39-47 */
uint64_t xgo_step_linear(xgo_state* st) {
    const xgo_params* p = &st->p;
    uint64_t t = xorshift_transform(st->x[st->idx], p->a, p->b, st->mask);
    unsigned tap = st->idx + (p->r - p->s);
    if (tap >= p->r) tap -= p->r;
    uint64_t v = t ^ xorshift_transform(st->x[tap], p->c, p->d, st->mask);
    st->x[st->idx] = v;
    if (++st->idx == p->r) st->idx = 0;
    return v;
}

/* proj/include/xg/xorgens.hpp:50-53 */
uint64_t xgo_weyl_next(xgo_state* st) {
    st->weyl = (st->weyl + st->p.omega) & st->mask;
    return st->weyl;
}

/* proj/include/xg/xorgens.hpp:58-62 */
uint64_t xgo_next_word(xgo_state* st) {
    uint64_t v = xgo_step_linear(st);
    uint64_t wk = xgo_weyl_next(st);
    return ((wk ^ (wk >> st->p.gamma)) + v) & st->mask;
}

/* proj/src/xorgens.cpp:40-46 */
void xgo_logical_buffer(const xgo_state* st, uint64_t* out) {
    for (unsigned i = 0; i < st->p.r; ++i) out[i] = st->x[(st->idx + i) % st->p.r];
}

/* proj/include/xg/xorgens.hpp:76 */
uint64_t xgo_weyl_value(const xgo_state* st) { return st->weyl; }

size_t xgo_state_size(void) { return sizeof(xgo_state); }

/* ---- lane batching: proj/src/parallel.cpp ------------------------------ */

/* proj/src/parallel.cpp:8-42: gather from the pre-batch buffer, then commit
 * and add the Weyl term in sequence order. */
int xgo_batch_step(xgo_state* st, unsigned lanes, uint64_t* out) {
    const xgo_params* p = &st->p;
    if (lanes == 0 || lanes > xgo_lane_bound(p)) return -1;
    const unsigned r = p->r, back_s = p->r - p->s, idx = st->idx;
    uint64_t fresh[XGO_MAX_R];
    for (unsigned l = 0; l < lanes; ++l) {
        unsigned pos_r = idx + l;
        if (pos_r >= r) pos_r -= r;
        unsigned pos_s = idx + l + back_s;
        while (pos_s >= r) pos_s -= r;
        fresh[l] = xorshift_transform(st->x[pos_r], p->a, p->b, st->mask) ^
                   xorshift_transform(st->x[pos_s], p->c, p->d, st->mask);
    }
    uint64_t weyl = st->weyl;
    for (unsigned l = 0; l < lanes; ++l) {
        unsigned pos = idx + l;
        if (pos >= r) pos -= r;
        st->x[pos] = fresh[l];
        weyl = (weyl + p->omega) & st->mask;
        out[l] = ((weyl ^ (weyl >> p->gamma)) + fresh[l]) & st->mask;
    }
    st->idx = (idx + lanes) % r; /* advance_raw, proj/include/xg/xorgens.hpp:84-87 */
    st->weyl = weyl;
    return 0;
}

/* proj/src/parallel.cpp:44-76: the racy in-place schedule (negative test). */
int xgo_unsynchronized_batch(xgo_state* st, unsigned lanes, uint64_t* out) {
    const xgo_params* p = &st->p;
    if (lanes == 0 || lanes > p->r) return -1;
    const unsigned r = p->r, back_s = p->r - p->s, idx = st->idx;
    uint64_t fresh[XGO_MAX_R];
    for (unsigned l = lanes; l-- > 0;) {
        unsigned pos_r = idx + l;
        if (pos_r >= r) pos_r -= r;
        unsigned pos_s = idx + l + back_s;
        while (pos_s >= r) pos_s -= r;
        fresh[l] = xorshift_transform(st->x[pos_r], p->a, p->b, st->mask) ^
                   xorshift_transform(st->x[pos_s], p->c, p->d, st->mask);
        st->x[pos_r] = fresh[l];
    }
    uint64_t weyl = st->weyl;
    for (unsigned l = 0; l < lanes; ++l) {
        weyl = (weyl + p->omega) & st->mask;
        out[l] = ((weyl ^ (weyl >> p->gamma)) + fresh[l]) & st->mask;
    }
    st->idx = (idx + lanes) % r;
    st->weyl = weyl;
    return 0;
}

int xgo_stream_u32(const xgo_params* p, uint64_t seed, uint64_t n, uint32_t* out) {
    xgo_state* st = (xgo_state*)malloc(sizeof(xgo_state));
    if (!st) return -3;
    int e = xgo_seed(st, p, seed);
    if (!e)
        for (uint64_t k = 0; k < n; ++k) out[k] = (uint32_t)xgo_next_word(st);
    free(st);
    return e;
}

/* ---- conventions (not in the reference) ----------- */

float xgo_u32_to_f32(uint32_t u) { return (float)(u >> 8) * 0x1.0p-24f; }

uint64_t xgo_u32pair_to_u64(uint32_t lo, uint32_t hi) {
    return (uint64_t)lo | ((uint64_t)hi << 32);
}

double xgo_u32pair_to_f64(uint32_t lo, uint32_t hi) {
    return (double)(xgo_u32pair_to_u64(lo, hi) >> 11) * 0x1.0p-53;
}

/* Words read as signed 32-bit coordinates in [-2^31, 2^31): hit iff the
 * point lies inside the disc x^2 + y^2 < 2^62 (exact; sum <= 2^63). */
int xgo_mc_hit(uint32_t x, uint32_t y) {
    int64_t xs = (int32_t)x, ys = (int32_t)y;
    uint64_t q = (uint64_t)(xs * xs) + (uint64_t)(ys * ys);
    return q < (UINT64_C(1) << 62);
}

/* ---- GF(2) rank: proj/src/stattests/gf2.cpp:8-33 ------------------------- */

/* Rank of a 32 x 32 GF(2) matrix given as 32 row words -- the reference's
 * row-by-row elimination: each row is reduced by the established pivots
 * (in the order they were found), then its lowest set column (bit index,
 * gf2.cpp:24-29 scans col = 0 upwards) becomes a new pivot. */
unsigned xgo_gf2_rank32(const uint32_t* rows_in) {
    uint32_t rows[32];
    unsigned pcol[32], prow[32], npiv = 0;
    for (int i = 0; i < 32; ++i) rows[i] = rows_in[i];
    for (unsigned i = 0; i < 32; ++i) {
        for (unsigned k = 0; k < npiv; ++k)
            if ((rows[i] >> pcol[k]) & 1u) rows[i] ^= rows[prow[k]];
        for (unsigned col = 0; col < 32; ++col) {
            if ((rows[i] >> col) & 1u) {
                pcol[npiv] = col;
                prow[npiv] = i;
                ++npiv;
                break;
            }
        }
    }
    return npiv;
}

/* ---- block ensemble: proj/src/parallel.cpp:84-135 ----------------------- */

typedef struct {
    int kind;
    xgo_state* states;
    uint32_t num_streams;
    uint64_t n;
    void* out;
    void* out2;
    const xgo_params* p;
    uint64_t base_seed;
    int rc;
    uint32_t t, used;
} job_t;

enum { J_SEED, J_U32, J_F32, J_F64, J_MC, J_SUM, J_RAW, J_WORDS, J_RANK };

static void run_one(job_t* j, uint32_t g) {
    xgo_state* st = &j->states[g];
    switch (j->kind) {
    case J_SEED: {
        int e = xgo_seed(st, j->p, j->base_seed + (uint64_t)g);
        if (e) j->rc = e;
        break;
    }
    case J_U32: {
        uint32_t* o = (uint32_t*)j->out + (size_t)g * j->n;
        for (uint64_t k = 0; k < j->n; ++k) o[k] = (uint32_t)xgo_next_word(st);
        break;
    }
    case J_WORDS: {
        /* next_word() values in their uint64 container (BlockEnsemble::generate) */
        uint64_t* o = (uint64_t*)j->out + (size_t)g * j->n;
        for (uint64_t k = 0; k < j->n; ++k) o[k] = xgo_next_word(st);
        break;
    }
    case J_RAW: {
        /* RawXorgens::next() = step_linear(), proj/include/xg/baselines.hpp:65 */
        uint32_t* o = (uint32_t*)j->out + (size_t)g * j->n;
        for (uint64_t k = 0; k < j->n; ++k) o[k] = (uint32_t)xgo_step_linear(st);
        break;
    }
    case J_F32: {
        float* o = (float*)j->out + (size_t)g * j->n;
        for (uint64_t k = 0; k < j->n; ++k) o[k] = xgo_u32_to_f32((uint32_t)xgo_next_word(st));
        break;
    }
    case J_F64: {
        double* o = (double*)j->out + (size_t)g * j->n;
        for (uint64_t k = 0; k < j->n; ++k) {
            uint32_t lo = (uint32_t)xgo_next_word(st);
            uint32_t hi = (uint32_t)xgo_next_word(st);
            o[k] = xgo_u32pair_to_f64(lo, hi);
        }
        break;
    }
    case J_MC: {
        /* sample m is the consecutive word pair
         * (w[2m], w[2m+1]); samples_per_stream is a multiple of 32. */
        uint64_t hits = 0;
        for (uint64_t k = 0; k < j->n; ++k) {
            uint32_t x = (uint32_t)xgo_next_word(st);
            uint32_t y = (uint32_t)xgo_next_word(st);
            hits += (uint64_t)xgo_mc_hit(x, y);
        }
        ((uint64_t*)j->out)[g] = hits;
        break;
    }
    case J_RANK: {
        /* matrix_rank_test's counting loop (proj/src/stattests/tests.cpp:93-109),
         * M = 32: matrix k = the next 32 words, row i = word i (bits MSB first
         * as BitSource reads them, proj/include/xg/stream.hpp:99-106, so the
         * row value IS the word).  out = 3 bins per stream. */
        uint64_t* o = (uint64_t*)j->out + (size_t)g * 3;
        uint32_t rows[32];
        o[0] = o[1] = o[2] = 0;
        for (uint64_t k = 0; k < j->n; ++k) {
            for (int i = 0; i < 32; ++i) rows[i] = (uint32_t)xgo_next_word(st);
            unsigned r = xgo_gf2_rank32(rows);
            if (r == 32) ++o[0];
            else if (r == 31) ++o[1];
            else ++o[2];
        }
        break;
    }
    case J_SUM: {
        uint32_t x = 0;
        uint64_t s = 0;
        for (uint64_t k = 0; k < j->n; ++k) {
            uint32_t v = (uint32_t)xgo_next_word(st);
            x ^= v;
            s += (uint64_t)v * (k + 1);
        }
        ((uint32_t*)j->out)[g] = x;
        ((uint64_t*)j->out2)[g] = s;
        break;
    }
    }
}

static void* worker(void* arg) {
    job_t* j = (job_t*)arg;
    for (uint32_t g = j->t; g < j->num_streams; g += j->used) run_one(j, g);
    return NULL;
}

/* Blocks striped over threads exactly like proj/src/parallel.cpp:115-134;
 * results are schedule independent. */
static int run_jobs(job_t proto, int threads) {
    if (threads <= 0) threads = 1;
    uint32_t used = (uint32_t)threads < proto.num_streams ? (uint32_t)threads : proto.num_streams;
    if (used <= 1) {
        proto.t = 0;
        proto.used = 1;
        worker(&proto);
        return proto.rc;
    }
    job_t* jobs = (job_t*)calloc(used, sizeof(job_t));
    pthread_t* tids = (pthread_t*)calloc(used, sizeof(pthread_t));
    if (!jobs || !tids) {
        free(jobs);
        free(tids);
        return -3;
    }
    for (uint32_t t = 0; t < used; ++t) {
        jobs[t] = proto;
        jobs[t].t = t;
        jobs[t].used = used;
        pthread_create(&tids[t], NULL, worker, &jobs[t]);
    }
    int rc = 0;
    for (uint32_t t = 0; t < used; ++t) {
        pthread_join(tids[t], NULL);
        if (jobs[t].rc) rc = jobs[t].rc;
    }
    free(jobs);
    free(tids);
    return rc;
}

/* proj/src/parallel.cpp:84-95: block i <- XorgensState(params, base_seed + i). */
int xgo_ensemble_seed(xgo_state* states, const xgo_params* p, uint64_t base_seed,
                      uint64_t first_stream, uint32_t num_streams, int threads) {
    job_t j;
    memset(&j, 0, sizeof j);
    j.kind = J_SEED;
    j.states = states;
    j.num_streams = num_streams;
    j.p = p;
    j.base_seed = base_seed + first_stream;
    return run_jobs(j, threads);
}

static int fill(int kind, xgo_state* states, uint32_t num_streams, uint64_t n, void* out,
                void* out2, int threads) {
    job_t j;
    memset(&j, 0, sizeof j);
    j.kind = kind;
    j.states = states;
    j.num_streams = num_streams;
    j.n = n;
    j.out = out;
    j.out2 = out2;
    return run_jobs(j, threads);
}

/* proj/src/parallel.cpp:97-135 (block-major, continues each block's state). */
int xgo_ensemble_fill_u32(xgo_state* states, uint32_t num_streams, uint64_t per_stream,
                          uint32_t* out, int threads) {
    return fill(J_U32, states, num_streams, per_stream, out, NULL, threads);
}
int xgo_ensemble_fill_words(xgo_state* states, uint32_t num_streams, uint64_t per_stream,
                             uint64_t* out, int threads) {
    return fill(J_WORDS, states, num_streams, per_stream, out, NULL, threads);
}
int xgo_ensemble_fill_raw_u32(xgo_state* states, uint32_t num_streams, uint64_t per_stream,
                              uint32_t* out, int threads) {
    return fill(J_RAW, states, num_streams, per_stream, out, NULL, threads);
}
int xgo_ensemble_fill_f32(xgo_state* states, uint32_t num_streams, uint64_t per_stream,
                          float* out, int threads) {
    return fill(J_F32, states, num_streams, per_stream, out, NULL, threads);
}
int xgo_ensemble_fill_f64(xgo_state* states, uint32_t num_streams, uint64_t per_stream,
                          double* out, int threads) {
    return fill(J_F64, states, num_streams, per_stream, out, NULL, threads);
}
int xgo_ensemble_mc_pi(xgo_state* states, uint32_t num_streams, uint64_t samples_per_stream,
                       uint64_t* hits_per_stream, int threads) {
    if (samples_per_stream % 32 != 0) return -1;
    return fill(J_MC, states, num_streams, samples_per_stream, hits_per_stream, NULL, threads);
}
int xgo_ensemble_rank_counts(xgo_state* states, uint32_t num_streams, uint64_t matrices_per_stream,
                             uint64_t* counts3_per_stream, int threads) {
    return fill(J_RANK, states, num_streams, matrices_per_stream, counts3_per_stream, NULL, threads);
}
int xgo_ensemble_checksums(xgo_state* states, uint32_t num_streams, uint64_t n,
                           uint32_t* xor_out, uint64_t* wsum_out, int threads) {
    return fill(J_SUM, states, num_streams, n, xor_out, wsum_out, threads);
}
