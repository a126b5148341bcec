/*
 * chunklab_oracle.c -- CPU restatement of the COREY hot path (TEST INFRASTRUCTURE ONLY).
 * See chunklab_oracle.h for scope and pinning.  Compile: -O2 -ffp-contract=off.
 * Citations are to /root/reference/proj/include/chunklab/<file>:<line>.
 */
#include "chunklab_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

const char* or_error_string(int code) {
  switch (code) {
    case OR_OK: return "ok";
    case OR_NO_SAMPLES: return "no samples";
    case OR_NON_FINITE: return "non-finite input";
    case OR_DEGENERATE_SPEC: return "degenerate spec";
    case OR_EPSILON: return "epsilon must be positive";
    case OR_STRIDE: return "stride must be >= 1";
    case OR_FIXED_RANGE: return "fixed range requires lo < hi";
    case OR_BOUNDS: return "invalid chunk bounds";
    case OR_HREF: return "h_ref must be positive";
    case OR_SIGNAL: return "signal must be >= 0";
    case OR_SHAPE: return "shape mismatch";
    case OR_CHUNK: return "chunk must be >= 1";
    case OR_MISSING_SEQ_LEN: return "missing feature: seq_len";
    case OR_MISSING_ENTROPY: return "missing feature: full_entropy";
    case OR_BUCKETS: return "bucket_set must be strictly increasing powers of two";
    default: return "invalid policy";
  }
}

/* ------------------------------------------------------------------------- */
/* mt19937_64 (the raw generator behind chunklab::Rng, rng.hpp:16).  Standard  */
/* parameters; the distribution transforms below follow rng.hpp:23-77.        */
/* ------------------------------------------------------------------------- */
#define MT_N 312
#define MT_M 156

void or_rng_seed(or_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
  r->spare = 0.0;
  r->has_spare = 0;
}

static void mt_refill(or_rng* r) {
  static const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  static const uint64_t mag = 0xB5026F5AA96619E9ULL;
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= mag;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->idx = 0;
}

uint64_t or_rng_next_u64(or_rng* r) {
  if (r->idx >= MT_N) mt_refill(r);
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:23-25: 53 random bits scaled by 2^-53. */
double or_rng_uniform(or_rng* r) { return (double)(or_rng_next_u64(r) >> 11) * 0x1.0p-53; }

double or_rng_uniform_range(or_rng* r, double lo, double hi) {
  return lo + (hi - lo) * or_rng_uniform(r);
}

/* rng.hpp:31-40: rejection sampling on the raw word. */
uint64_t or_rng_index(or_rng* r, uint64_t n) {
  const uint64_t span = n;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % span;
  uint64_t v;
  do {
    v = or_rng_next_u64(r);
  } while (v >= limit);
  return v % span;
}

/* rng.hpp:44-59: Marsaglia polar, spare cached. */
double or_rng_normal(or_rng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u, v, s;
  do {
    u = 2.0 * or_rng_uniform(r) - 1.0;
    v = 2.0 * or_rng_uniform(r) - 1.0;
    s = u * u + v * v;
  } while (s >= 1.0 || s == 0.0);
  const double m = sqrt(-2.0 * log(s) / s);
  r->spare = v * m;
  r->has_spare = 1;
  return u * m;
}

/* rng.hpp:62-66: inverse CDF. */
double or_rng_laplace(or_rng* r, double scale) {
  const double u = or_rng_uniform(r) - 0.5;
  const double sign = u < 0.0 ? -1.0 : 1.0;
  return -scale * sign * log(1.0 - 2.0 * fabs(u));
}

/* rng.hpp:69-77 */
double or_rng_student_t(or_rng* r, int dof) {
  const double z = or_rng_normal(r);
  double chi2 = 0.0;
  for (int i = 0; i < dof; ++i) {
    const double g = or_rng_normal(r);
    chi2 += g * g;
  }
  return z / sqrt(chi2 / (double)dof);
}

/* rng.hpp:87-93: splitmix64 finalizer. */
uint64_t or_derive_seed(uint64_t seed, uint64_t tag) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (tag + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* synthetic.hpp:29-64 */
int or_generate_activations(int dist, double laplace_scale, double nonzero_fraction,
                            uint64_t seed, size_t n, double* out) {
  or_rng values;
  or_rng_seed(&values, seed);
  switch (dist) {
    case OR_DIST_UNIFORM:
      for (size_t i = 0; i < n; ++i) out[i] = or_rng_uniform(&values);
      break;
    case OR_DIST_NORMAL:
      for (size_t i = 0; i < n; ++i) out[i] = or_rng_normal(&values);
      break;
    case OR_DIST_LAPLACE:
      if (!(laplace_scale > 0.0)) return OR_POLICY;
      for (size_t i = 0; i < n; ++i) out[i] = or_rng_laplace(&values, laplace_scale);
      break;
    case OR_DIST_SPARSE: {
      if (!(nonzero_fraction > 0.0 && nonzero_fraction <= 1.0)) return OR_POLICY;
      or_rng mask;
      or_rng_seed(&mask, or_derive_seed(seed, 0x5ba7));
      for (size_t i = 0; i < n; ++i)
        out[i] = or_rng_uniform(&mask) < nonzero_fraction ? or_rng_normal(&values) : 0.0;
      break;
    }
    default:
      return OR_POLICY;
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* histogram + entropy                                                        */
/* ------------------------------------------------------------------------- */

/* entropy.hpp:56-62 */
int or_validate_spec(const or_hist_spec* s) {
  if (s->bin_count < 2) return OR_DEGENERATE_SPEC;
  if (!(s->epsilon > 0.0)) return OR_EPSILON;
  if (s->sample_stride < 1) return OR_STRIDE;
  if (s->range_mode == OR_RANGE_FIXED && !(s->fixed_lo < s->fixed_hi)) return OR_FIXED_RANGE;
  return OR_OK;
}

/* entropy.hpp:87-94: floor((v-lo)/(hi-lo)*K) in fp64, clamped to [0, K-1]. */
int or_bin_index(double v, double lo, double hi, int k) {
  const double width = hi - lo;
  if (!(width > 0.0)) return 0;
  int idx = (int)floor((v - lo) / width * k);
  if (idx < 0) idx = 0;
  if (idx >= k) idx = k - 1;
  return idx;
}

/* entropy.hpp:101-138.  Two passes: strided min/max + finite check, then
 * strided binning.  Counts are returned alongside the masses. */
int or_compute_histogram(const double* values, size_t n_values, const or_hist_spec* spec,
                         uint64_t* counts, double* masses, double* lo_out, double* hi_out,
                         uint64_t* sample_count) {
  int rc = or_validate_spec(spec);
  if (rc) return rc;
  const size_t stride = (size_t)spec->sample_stride;
  size_t n = 0;
  double lo = INFINITY, hi = -INFINITY;
  for (size_t i = 0; i < n_values; i += stride) {
    const double v = values[i];
    if (!isfinite(v)) return OR_NON_FINITE;
    /* std::min(lo, v) returns lo unless v < lo; std::max(hi, v) returns hi unless hi < v. */
    if (v < lo) lo = v;
    if (hi < v) hi = v;
    ++n;
  }
  if (n == 0) return OR_NO_SAMPLES;
  if (spec->range_mode == OR_RANGE_FIXED) {
    lo = spec->fixed_lo;
    hi = spec->fixed_hi;
  }
  const int k = spec->bin_count;
  memset(counts, 0, sizeof(uint64_t) * (size_t)k);
  for (size_t i = 0; i < n_values; i += stride) ++counts[or_bin_index(values[i], lo, hi, k)];
  if (masses) {
    const double inv_n = 1.0 / (double)n;
    for (int b = 0; b < k; ++b) masses[b] = (double)counts[b] * inv_n;
  }
  *lo_out = lo;
  *hi_out = hi;
  *sample_count = n;
  return OR_OK;
}

int or_token_entropy(const double* values, size_t channels, size_t length,
                     const or_hist_spec* spec, double* raw_nats, double* normalized,
                     uint64_t* sample_count) {
  /* entropy.hpp:182-186: validate_tensor, validate_spec; the caller passes the shape */
  for (size_t i = 0; i < channels * length; ++i)
    if (!isfinite(values[i])) return OR_NON_FINITE;
  int rc = or_validate_spec(spec);
  if (rc) return rc;
  const int k = spec->bin_count;
  double* slice = (double*)malloc(sizeof(double) * (channels ? channels : 1));
  uint64_t* counts = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)k);
  double* masses = (double*)malloc(sizeof(double) * (size_t)k);
  double raw_sum = 0.0;
  uint64_t samples = 0;
  for (size_t t = 0; t < length && rc == OR_OK; ++t) {
    for (size_t c = 0; c < channels; ++c) slice[c] = values[c * length + t];
    double lo, hi, raw, norm;
    uint64_t n;
    rc = or_compute_histogram(slice, channels, spec, counts, masses, &lo, &hi, &n);
    if (rc == OR_OK) rc = or_estimate_entropy(masses, k, spec->epsilon, &raw, &norm);
    if (rc == OR_OK) {
      raw_sum += raw;
      samples += n;
    }
  }
  free(slice);
  free(counts);
  free(masses);
  if (rc) return rc;
  *raw_nats = raw_sum / (double)length;
  *normalized = *raw_nats / log((double)k);
  *sample_count = samples;
  return OR_OK;
}

int or_compute_histogram_f32(const float* values, size_t n_values, const or_hist_spec* spec,
                             uint64_t* counts, double* lo_out, double* hi_out,
                             uint64_t* sample_count) {
  int rc = or_validate_spec(spec);
  if (rc) return rc;
  const size_t stride = (size_t)spec->sample_stride;
  size_t n = 0;
  double lo = INFINITY, hi = -INFINITY;
  for (size_t i = 0; i < n_values; i += stride) {
    const double v = (double)values[i];
    if (!isfinite(v)) return OR_NON_FINITE;
    if (v < lo) lo = v;
    if (hi < v) hi = v;
    ++n;
  }
  if (n == 0) return OR_NO_SAMPLES;
  if (spec->range_mode == OR_RANGE_FIXED) {
    lo = spec->fixed_lo;
    hi = spec->fixed_hi;
  }
  const int k = spec->bin_count;
  memset(counts, 0, sizeof(uint64_t) * (size_t)k);
  for (size_t i = 0; i < n_values; i += stride)
    ++counts[or_bin_index((double)values[i], lo, hi, k)];
  *lo_out = lo;
  *hi_out = hi;
  *sample_count = n;
  return OR_OK;
}

/* entropy.hpp:149-164: raw = -sum_{p>0} p*log(p+eps) in bin order. */
int or_estimate_entropy(const double* masses, int k, double epsilon, double* raw_nats,
                        double* normalized) {
  if (k < 2) return OR_DEGENERATE_SPEC;
  if (!(epsilon > 0.0)) return OR_EPSILON;
  double raw = 0.0;
  for (int i = 0; i < k; ++i) {
    const double p = masses[i];
    if (p > 0.0) raw -= p * log(p + epsilon);
  }
  *raw_nats = raw;
  *normalized = raw / log((double)k);
  return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* chunk rule + scheduler                                                     */
/* ------------------------------------------------------------------------- */
static int is_pow2(uint64_t v) { return v != 0 && (v & (v - 1)) == 0; }

int or_log2_exact(uint64_t v) {
  int e = 0;
  while (v > 1) {
    v >>= 1;
    ++e;
  }
  return e;
}

double or_round_half_up(double x) { return floor(x + 0.5); }

int or_validate_bounds(int c_min, int c_max) {
  if (c_min <= 0 || c_max <= 0 || !is_pow2((uint64_t)c_min) || !is_pow2((uint64_t)c_max) ||
      c_min > c_max)
    return OR_BOUNDS;
  return OR_OK;
}

/* chunk.hpp:68-89 */
int or_select_chunk(double signal_nats, int c_min, int c_max, double h_ref_nats, int* chunk,
                    double* r_out) {
  int rc = or_validate_bounds(c_min, c_max);
  if (rc) return rc;
  if (!(h_ref_nats > 0.0)) return OR_HREF;
  if (!(signal_nats >= 0.0)) return OR_SIGNAL;
  double r = signal_nats / h_ref_nats;
  if (r > 1.0) r = 1.0; /* std::min(x, 1.0) */
  const double target = (double)c_min + r * (double)(c_max - c_min);
  const double exponent = or_round_half_up(log2(target));
  const double pow2 = exp2(exponent);
  int c = (int)pow2;
  if (c < c_min) c = c_min;
  if (c > c_max) c = c_max;
  *chunk = c;
  *r_out = r;
  return OR_OK;
}

/* chunk.hpp:206-218: nearest bucket by |log2| distance, ties toward larger. */
int or_snap_to_buckets(int chunk, const int* buckets, int n_buckets) {
  int best = buckets[0];
  double best_dist = INFINITY;
  const double lc = log2((double)chunk);
  for (int i = 0; i < n_buckets; ++i) {
    const int b = buckets[i];
    const double dist = fabs(log2((double)b) - lc);
    if (dist < best_dist || (dist == best_dist && b > best)) {
      best = b;
      best_dist = dist;
    }
  }
  return best;
}

uint64_t or_kernel_calls(uint64_t seq_len, uint64_t chunk) {
  if (seq_len == 0 || chunk == 0) return 0;
  return (seq_len + chunk - 1) / chunk;
}

static int member(const or_policy* p, int c) {
  for (int i = 0; i < p->n_buckets; ++i)
    if (p->buckets[i] == c) return 1;
  return 0;
}

/* chunk.hpp:149-181 restricted to the device policy subset. */
static int validate_policy(const or_policy* p) {
  if (p->n_buckets < 1 || p->n_buckets > 16) return OR_BUCKETS;
  int prev = 0;
  for (int i = 0; i < p->n_buckets; ++i) {
    const int b = p->buckets[i];
    if (b <= 0 || !is_pow2((uint64_t)b) || b <= prev) return OR_BUCKETS;
    prev = b;
  }
  if (p->kind == OR_POL_STATIC && !member(p, p->static_chunk)) return OR_POLICY;
  if (p->kind == OR_POL_LEARNED_TABLE && (!member(p, p->short_chunk) || !member(p, p->long_chunk)))
    return OR_POLICY;
  if (p->kind == OR_POL_GUARDED) {
    if (!member(p, p->safe_chunk) || p->min_delta_buckets < 0) return OR_POLICY;
    if (p->inner_kind == OR_POL_STATIC && !member(p, p->inner_static_chunk)) return OR_POLICY;
    if (p->inner_kind == OR_POL_GUARDED) return OR_POLICY;
  }
  return OR_OK;
}

static int decide_simple(const or_policy* p, int kind, int static_chunk, const or_features* f,
                         int c_min, int c_max, double h_ref, int* chunk, double* r,
                         double* signal, int* source) {
  int rc;
  *r = 0.0;
  *signal = 0.0;
  switch (kind) {
    case OR_POL_STATIC: /* chunk.hpp:281-283 */
      *chunk = static_chunk;
      *source = 0;
      return OR_OK;
    case OR_POL_MIDPOINT: { /* chunk.hpp:285-291 */
      const int n = p->n_buckets;
      int idx = (n + 1) / 2;
      if (idx > n - 1) idx = n - 1;
      *chunk = p->buckets[idx];
      *source = 1;
      return OR_OK;
    }
    case OR_POL_FULL_HIST:    /* chunk.hpp:298-302 */
    case OR_POL_SAMPLED_HIST: { /* chunk.hpp:304-309 */
      const int full = kind == OR_POL_FULL_HIST;
      if (full ? !f->has_full_entropy : !f->has_sampled_entropy) return OR_MISSING_ENTROPY;
      const double s = full ? f->full_entropy_nats : f->sampled_entropy_nats;
      int c;
      rc = or_select_chunk(s, c_min, c_max, h_ref, &c, r);
      if (rc) return rc;
      *chunk = or_snap_to_buckets(c, p->buckets, p->n_buckets);
      *signal = s;
      *source = full ? 2 : 3;
      return OR_OK;
    }
    case OR_POL_LEARNED_TABLE: /* chunk.hpp:360-368, strict < */
      if (!f->has_seq_len) return OR_MISSING_SEQ_LEN;
      *chunk = f->seq_len < p->threshold_tokens ? p->short_chunk : p->long_chunk;
      *signal = (double)f->seq_len;
      *source = 4;
      return OR_OK;
    default:
      return OR_POLICY;
  }
}

int or_schedule(const or_policy* p, const or_features* f, int c_min, int c_max,
                double h_ref_nats, int* chunk, double* r, double* signal, int* source_code) {
  int rc = validate_policy(p);
  if (rc) return rc;
  rc = or_validate_bounds(c_min, c_max);
  if (rc) return rc;
  if (p->kind != OR_POL_GUARDED)
    return decide_simple(p, p->kind, p->static_chunk, f, c_min, c_max, h_ref_nats, chunk, r,
                         signal, source_code);
  /* chunk.hpp:344-358 */
  int inner_chunk, inner_src;
  rc = decide_simple(p, p->inner_kind, p->inner_static_chunk, f, c_min, c_max, h_ref_nats,
                     &inner_chunk, r, signal, &inner_src);
  if (rc) return rc;
  int delta = or_log2_exact((uint64_t)inner_chunk) - or_log2_exact((uint64_t)p->safe_chunk);
  if (delta < 0) delta = -delta;
  if (delta >= p->min_delta_buckets) {
    *chunk = inner_chunk;
    *source_code = 16 + inner_src;
  } else {
    *chunk = p->safe_chunk;
    *source_code = 32;
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* reference recurrence, scan.hpp:77-136                                      */
/* ------------------------------------------------------------------------- */
static int validate_scan(const or_scan_params* p) {
  if (p->channels == 0 || p->state_dim == 0 || p->seq_len == 0) return OR_SHAPE;
  const size_t cs = p->channels * p->state_dim;
  if (p->a_len != cs && p->a_len != p->seq_len * cs) return OR_SHAPE;
  if (p->b_len != p->state_dim && p->b_len != p->seq_len * p->state_dim) return OR_SHAPE;
  if (p->c_len != p->state_dim && p->c_len != p->seq_len * p->state_dim) return OR_SHAPE;
  if (p->d_len != p->channels) return OR_SHAPE;
  if (p->x_len != p->channels * p->seq_len) return OR_SHAPE;
  const double* arrs[5] = {p->a, p->b, p->c, p->d, p->x};
  const size_t lens[5] = {p->a_len, p->b_len, p->c_len, p->d_len, p->x_len};
  for (int k = 0; k < 5; ++k)
    for (size_t i = 0; i < lens[k]; ++i)
      if (!isfinite(arrs[k][i])) return OR_NON_FINITE;
  return OR_OK;
}

/* scan.hpp:77-100: t outer, channel middle, state inner. */
static void scan_window(const or_scan_params* p, size_t t0, size_t t1, double* h, double* y) {
  const size_t n = p->state_dim, ch = p->channels, L = p->seq_len;
  const int at = p->a_len == L * ch * n;
  const int bt = p->b_len == L * n;
  const int ct = p->c_len == L * n;
  for (size_t t = t0; t < t1; ++t) {
    const double* a_t = at ? p->a + t * ch * n : p->a;
    const double* b_t = bt ? p->b + t * n : p->b;
    const double* c_t = ct ? p->c + t * n : p->c;
    for (size_t c = 0; c < ch; ++c) {
      const double x_ct = p->x[c * L + t];
      double* h_c = h + c * n;
      const double* a_ct = a_t + c * n;
      double out = 0.0;
      for (size_t s = 0; s < n; ++s) {
        h_c[s] = a_ct[s] * h_c[s] + b_t[s] * x_ct;
        out += c_t[s] * h_c[s];
      }
      y[c * L + t] = out + p->d[c] * x_ct;
    }
  }
}

int or_scan_chunked(const or_scan_params* p, const double* h0, size_t chunk, double* y,
                    double* h_out) {
  int rc = validate_scan(p);
  if (rc) return rc;
  const size_t cs = p->channels * p->state_dim;
  if (h0) {
    for (size_t i = 0; i < cs; ++i)
      if (!isfinite(h0[i])) return OR_NON_FINITE;
    memcpy(h_out, h0, cs * sizeof(double));
  } else {
    memset(h_out, 0, cs * sizeof(double));
  }
  const size_t L = p->seq_len;
  if (chunk == 0) chunk = L;
  for (size_t t = 0; t < L; t += chunk) {
    const size_t t1 = t + chunk < L ? t + chunk : L;
    scan_window(p, t, t1, h_out, y);
  }
  return OR_OK;
}

/* scan.hpp:140-163 */
void or_random_scan_params(uint64_t seed, size_t channels, size_t state_dim, size_t seq_len,
                           int time_varying, double* a, double* b, double* c, double* d,
                           double* x) {
  or_rng rng;
  or_rng_seed(&rng, seed);
  const size_t a_n = time_varying ? seq_len * channels * state_dim : channels * state_dim;
  const size_t bc_n = time_varying ? seq_len * state_dim : state_dim;
  for (size_t i = 0; i < a_n; ++i) a[i] = or_rng_uniform_range(&rng, 0.5, 0.995);
  for (size_t i = 0; i < bc_n; ++i) b[i] = or_rng_normal(&rng);
  for (size_t i = 0; i < bc_n; ++i) c[i] = or_rng_normal(&rng) / sqrt((double)state_dim);
  for (size_t i = 0; i < channels; ++i) d[i] = 0.1 * or_rng_normal(&rng);
  for (size_t i = 0; i < channels * seq_len; ++i) x[i] = or_rng_normal(&rng);
}

/* ------------------------------------------------------------------------- */
/* Mamba-1 selective scan (extension).  Per (b, c): delta' = softplus(delta +  */
/* bias) (mamba_ssm convention: identity above 20), x = delta'*u,             */
/* h_s = exp(delta'*A[c,s])*h_s + B[b,s,t]*x ; out += C[b,s,t]*h_s (state      */
/* order, scan.hpp:97-98), y = out + D[c]*u, y *= z*sigmoid(z).               */
/* Rows are independent, so the channel loop can be outermost without         */
/* changing any per-row operation order.                                      */
/* ------------------------------------------------------------------------- */
static inline double softplus64(double v) { return v <= 20.0 ? log1p(exp(v)) : v; }
static inline double silu64(double v) { return v / (1.0 + exp(-v)); }

#define MAMBA_ROW_BODY(LOAD)                                                              \
  for (size_t row = row_begin; row < row_end; ++row) {                                    \
    const size_t bb = row / dim, c = row % dim;                                           \
    const size_t base = row * L;                                                          \
    double h[64];                                                                         \
    for (size_t s = 0; s < N; ++s) h[s] = 0.0;                                            \
    const double bias = delta_bias ? (double)LOAD(delta_bias, c) : 0.0;                   \
    const double dskip = Dv ? (double)LOAD(Dv, c) : 0.0;                                  \
    for (size_t t = 0; t < L; ++t) {                                                      \
      const double uu = (double)LOAD(u, base + t);                                        \
      double dt = (double)LOAD(delta, base + t) + bias;                                   \
      if (delta_softplus) dt = softplus64(dt);                                            \
      const double xx = dt * uu;                                                          \
      double out = 0.0;                                                                   \
      for (size_t s = 0; s < N; ++s) {                                                    \
        const double a = exp(dt * (double)LOAD(A, c * N + s));                            \
        const double bv = (double)LOAD(Bm, (bb * N + s) * L + t);                         \
        const double cv = (double)LOAD(Cm, (bb * N + s) * L + t);                         \
        h[s] = a * h[s] + bv * xx;                                                        \
        out += cv * h[s];                                                                 \
      }                                                                                   \
      double yy = out + dskip * uu;                                                       \
      if (z) yy = yy * silu64((double)LOAD(z, base + t));                                 \
      y[(row - row_begin) * L + t] = yy;                                                  \
    }                                                                                     \
    if (h_last)                                                                           \
      for (size_t s = 0; s < N; ++s) h_last[(row - row_begin) * N + s] = h[s];           \
  }

#define LOAD_PLAIN(arr, i) ((arr)[(i)])

int or_mamba1_scan_rows(const double* u, const double* delta, const double* A, const double* Bm,
                        const double* Cm, const double* Dv, const double* z,
                        const double* delta_bias, int delta_softplus, size_t batch, size_t dim,
                        size_t N, size_t L, size_t row_begin, size_t row_end, const double* h0,
                        double* y, double* h_last) {
  if (N == 0 || N > 64 || L == 0 || dim == 0 || batch == 0) return OR_SHAPE;
  if (row_end > batch * dim || row_begin > row_end) return OR_SHAPE;
  if (h0) {
    /* initial state variant (scan.hpp:102-109 semantics) */
    for (size_t row = row_begin; row < row_end; ++row) {
      const size_t bb = row / dim, c = row % dim, base = row * L;
      double h[64];
      for (size_t s = 0; s < N; ++s) h[s] = h0[row * N + s];
      const double bias = delta_bias ? delta_bias[c] : 0.0;
      const double dskip = Dv ? Dv[c] : 0.0;
      for (size_t t = 0; t < L; ++t) {
        const double uu = u[base + t];
        double dt = delta[base + t] + bias;
        if (delta_softplus) dt = softplus64(dt);
        const double xx = dt * uu;
        double out = 0.0;
        for (size_t s = 0; s < N; ++s) {
          const double a = exp(dt * A[c * N + s]);
          h[s] = a * h[s] + Bm[(bb * N + s) * L + t] * xx;
          out += Cm[(bb * N + s) * L + t] * h[s];
        }
        double yy = out + dskip * uu;
        if (z) yy = yy * silu64(z[base + t]);
        y[(row - row_begin) * L + t] = yy;
      }
      if (h_last)
        for (size_t s = 0; s < N; ++s) h_last[(row - row_begin) * N + s] = h[s];
    }
    return OR_OK;
  }
  MAMBA_ROW_BODY(LOAD_PLAIN)
  return OR_OK;
}

int or_mamba1_scan_rows_f32(const float* u, const float* delta, const float* A, const float* Bm,
                            const float* Cm, const float* Dv, const float* z,
                            const float* delta_bias, int delta_softplus, size_t batch,
                            size_t dim, size_t N, size_t L, size_t row_begin, size_t row_end,
                            double* y, double* h_last) {
  if (N == 0 || N > 64 || L == 0 || dim == 0 || batch == 0) return OR_SHAPE;
  if (row_end > batch * dim || row_begin > row_end) return OR_SHAPE;
  MAMBA_ROW_BODY(LOAD_PLAIN)
  return OR_OK;
}

uint64_t or_fnv1a64(const void* data, size_t n_bytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ULL;
  for (size_t i = 0; i < n_bytes; ++i) {
    h ^= (uint64_t)p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}
