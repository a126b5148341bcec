/*
 * chunklab_oracle.h -- CPU restatement of the COREY hot path (TEST INFRASTRUCTURE).
 *
 * This is the parity oracle, not the product.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * path (paper_2604_10597_b200/, include/) never links or calls anything here.
 *
 * Every function restates one function of the reference C++ headers at
 * /root/reference/proj/include/chunklab (cited per function), in plain C99 so
 * it compiles with gcc alone.  Build with -ffp-contract=off and without
 * -march=native: the reference's bits depend on FMA contraction being off
 * (SURVEY.md finding 3).
 *
 * Parity pinning: the restatement is checked bit-for-bit against
 *   (1) the known-answer vectors of SURVEY.md Appendix B (derived from the
 *       reference itself), committed under tests/golden/, and
 *   (2) the reference headers compiled in place into oracle/_ref/ (see
 *       oracle/Makefile, oracle/ref_shim.cpp) whenever /root/reference exists.
 * The Mamba-1 extension (softplus(delta+bias) pre-transform, SiLU(z) gate) has
 * no counterpart in the reference; its recurrence core reduces exactly onto
 * scan_sequential (checked in tests/test_oracle.py), the two elementwise ops
 * are "parity unpinned".
 */
#ifndef CHUNKLAB_ORACLE_H
#define CHUNKLAB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes (messages mirror the reference's invalid_input strings) ---- */
enum {
  OR_OK = 0,
  OR_NO_SAMPLES = 1,          /* "no samples"                     entropy.hpp:101-138 */
  OR_NON_FINITE = 2,          /* "non-finite input"               entropy.hpp:42, scan.hpp:70-72 */
  OR_DEGENERATE_SPEC = 3,     /* "degenerate spec"                entropy.hpp:56-62 */
  OR_EPSILON = 4,             /* "epsilon must be positive" */
  OR_STRIDE = 5,              /* "stride must be >= 1" */
  OR_FIXED_RANGE = 6,         /* "fixed range requires lo < hi" */
  OR_BOUNDS = 7,              /* "invalid chunk bounds"           chunk.hpp:34-40 */
  OR_HREF = 8,                /* "h_ref must be positive" */
  OR_SIGNAL = 9,              /* "signal must be >= 0"            chunk.hpp:72 */
  OR_SHAPE = 10,              /* "shape mismatch"                 scan.hpp:54-69 */
  OR_CHUNK = 11,              /* "chunk must be >= 1"             scan.hpp:127 */
  OR_MISSING_SEQ_LEN = 12,    /* "missing feature: seq_len"       chunk.hpp:197-201 */
  OR_MISSING_ENTROPY = 13,    /* "missing feature: full_entropy / sampled_entropy" */
  OR_BUCKETS = 14,            /* "bucket_set must be ..." */
  OR_POLICY = 15              /* other policy validation failures */
};
const char* or_error_string(int code);

/* ---- RNG: mt19937_64 + the reference's explicit transforms (rng.hpp:16-93) ---- */
typedef struct {
  uint64_t mt[312];
  int idx;
  double spare;
  int has_spare;
} or_rng;

void or_rng_seed(or_rng* r, uint64_t seed);
uint64_t or_rng_next_u64(or_rng* r);
double or_rng_uniform(or_rng* r);                       /* rng.hpp:23-25 */
double or_rng_uniform_range(or_rng* r, double lo, double hi);
uint64_t or_rng_index(or_rng* r, uint64_t n);           /* rng.hpp:31-40 */
double or_rng_normal(or_rng* r);                        /* rng.hpp:44-59 */
double or_rng_laplace(or_rng* r, double scale);         /* rng.hpp:62-66 */
double or_rng_student_t(or_rng* r, int dof);            /* rng.hpp:69-77 */
uint64_t or_derive_seed(uint64_t seed, uint64_t tag);   /* rng.hpp:87-93 */

/* ---- synthetic activations (synthetic.hpp:29-64) ---- */
enum { OR_DIST_UNIFORM = 0, OR_DIST_NORMAL = 1, OR_DIST_LAPLACE = 2, OR_DIST_SPARSE = 3 };
int or_generate_activations(int dist, double laplace_scale, double nonzero_fraction,
                            uint64_t seed, size_t n, double* out);

/* ---- histogram + entropy (entropy.hpp:87-174) ---- */
enum { OR_RANGE_DYNAMIC = 0, OR_RANGE_FIXED = 1 };
typedef struct {
  int bin_count;
  double epsilon;
  int range_mode;
  double fixed_lo, fixed_hi;
  uint64_t sample_stride;
} or_hist_spec;

int or_validate_spec(const or_hist_spec* s);                       /* entropy.hpp:56-62 */
int or_bin_index(double v, double lo, double hi, int k);           /* entropy.hpp:87-94 */
/* counts[k] (uint64), masses[k]; lo/hi/n out.  Span version, entropy.hpp:101-138. */
int or_compute_histogram(const double* values, size_t n_values, const or_hist_spec* spec,
                         uint64_t* counts, double* masses, double* lo, double* hi,
                         uint64_t* sample_count);
/* entropy.hpp:149-164 */
int or_estimate_entropy(const double* masses, int k, double epsilon, double* raw_nats,
                        double* normalized);

/* token_entropy (entropy.hpp:180-210): values as (channels, length), length contiguous;
 * per position t the slice values[c*length + t], c = 0..channels-1, through
 * compute_histogram + estimate_entropy; raw entropies averaged in position order.
 * The whole tensor is validated first (validate_tensor: every value finite). */
int or_token_entropy(const double* values, size_t channels, size_t length,
                     const or_hist_spec* spec, double* raw_nats, double* normalized,
                     uint64_t* sample_count);

/* ---- chunk rule + scheduler family (chunk.hpp) ---- */
int or_log2_exact(uint64_t v);                                     /* common.hpp:25-32 */
double or_round_half_up(double x);                                 /* common.hpp:35 */
int or_validate_bounds(int c_min, int c_max);                      /* chunk.hpp:34-40 */
/* chunk.hpp:68-89 */
int or_select_chunk(double signal_nats, int c_min, int c_max, double h_ref_nats, int* chunk,
                    double* r);
int or_snap_to_buckets(int chunk, const int* buckets, int n_buckets); /* chunk.hpp:206-218 */
uint64_t or_kernel_calls(uint64_t seq_len, uint64_t chunk);           /* chunk.hpp:92-95 */

enum {
  OR_POL_STATIC = 0,
  OR_POL_MIDPOINT = 1,
  OR_POL_FULL_HIST = 2,
  OR_POL_SAMPLED_HIST = 3,
  OR_POL_LEARNED_TABLE = 4,
  OR_POL_GUARDED = 5
};
typedef struct {
  int kind;
  int static_chunk;
  /* guarded: the inner policy is described by the inner_* fields */
  int inner_kind;
  int inner_static_chunk;
  int safe_chunk;
  int min_delta_buckets;
  /* learned table */
  uint64_t threshold_tokens;
  int short_chunk, long_chunk;
  /* bucket set */
  int n_buckets;
  int buckets[16];
} or_policy;

typedef struct {
  int has_full_entropy;
  double full_entropy_nats;
  int has_sampled_entropy;
  double sampled_entropy_nats;
  int has_seq_len;
  uint64_t seq_len;
} or_features;

/* Scheduler::decide for the on-device subset (chunk.hpp:256-368).
 * source_code: 0 static, 1 midpoint, 2 full_histogram, 3 sampled_histogram,
 * 4 learned_table, +16 = guarded[inner], 32 = guarded[fallback]. */
int or_schedule(const or_policy* p, const or_features* f, int c_min, int c_max,
                double h_ref_nats, int* chunk, double* r, double* signal, int* source_code);

/* ---- reference recurrence (scan.hpp:77-136), fp64 ---- */
typedef struct {
  size_t channels, state_dim, seq_len;
  const double *a, *b, *c, *d, *x;
  size_t a_len, b_len, c_len, d_len, x_len;
} or_scan_params;

int or_scan_chunked(const or_scan_params* p, const double* h0 /* may be NULL */,
                    size_t chunk /* 0 = sequential */, double* y, double* h_out);
/* random_scan_params (scan.hpp:140-163): fills a,b,c,d,x (caller-allocated). */
void or_random_scan_params(uint64_t seed, size_t channels, size_t state_dim, size_t seq_len,
                           int time_varying, double* a, double* b, double* c, double* d,
                           double* x);

/* ---- Mamba-1 selective scan, fp64 (extension; see header comment) ----
 * u, delta, z, y: (batch, dim, L); A: (dim, N); Bm, Cm: (batch, N, L);
 * Dv, delta_bias: (dim) or NULL; h0/h_last: (batch, dim, N) or NULL.
 * Rows [row_begin, row_end) of the (batch*dim) flattening are computed
 * (independent, so a row subset is exact for those rows). */
int or_mamba1_scan_rows(const double* u, const double* delta, const double* A, const double* Bm,
                        const double* Cm, const double* Dv, const double* z,
                        const double* delta_bias, int delta_softplus, size_t batch, size_t dim,
                        size_t N, size_t L, size_t row_begin, size_t row_end, const double* h0,
                        double* y, double* h_last);
/* Same, float inputs widened to double per element (bench CPU baseline). */
int or_mamba1_scan_rows_f32(const float* u, const float* delta, const float* A, const float* Bm,
                            const float* Cm, const float* Dv, const float* z,
                            const float* delta_bias, int delta_softplus, size_t batch,
                            size_t dim, size_t N, size_t L, size_t row_begin, size_t row_end,
                            double* y, double* h_last);
/* Histogram over float values widened to double (entropy.hpp:101-138 on io.hpp f32 ingestion). */
int or_compute_histogram_f32(const float* values, size_t n_values, const or_hist_spec* spec,
                             uint64_t* counts, double* lo, double* hi, uint64_t* sample_count);

/* FNV-1a 64 over bytes (fixtures.hpp:160-167), used for golden digests. */
uint64_t or_fnv1a64(const void* data, size_t n_bytes);

#ifdef __cplusplus
}
#endif
#endif
