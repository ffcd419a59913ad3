/*
 * sgmv_oracle.c -- CPU ORACLE (test infrastructure only; see sgmv_oracle.h).
 *
 * Plain-C restatement of the reference's SGMV path.  Every function cites the
 * reference file:line it restates (paths relative to /root/reference/proj).
 * Compile with -ffp-contract=off: the fp64 sums must round exactly like the
 * reference's Release build (x86-64 -O3 emits no FMA there).
 */
#include "sgmv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EINVAL (-1)

/* ------------------------------------------------------------------------ */
/* mt19937_64 (the engine behind lorasim::Rng, workload.hpp:41).  The engine's
 * sequence is fixed by the C++ standard ([rand.predef]); restated here.      */
/* ------------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ull
#define MT_LOWER 0x000000007FFFFFFFull

size_t orc_rng_size(void) { return sizeof(orc_rng); }

void orc_rng_seed(orc_rng* g, uint64_t seed) {
  g->mt[0] = seed;
  for (uint32_t i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + i;
  g->mti = MT_N;
}

static void mt_twist(orc_rng* g) {
  for (uint32_t i = 0; i < MT_N; ++i) {
    const uint64_t x = (g->mt[i] & MT_UPPER) | (g->mt[(i + 1) % MT_N] & MT_LOWER);
    uint64_t xa = x >> 1;
    if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
    g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ xa;
  }
  g->mti = 0;
}

uint64_t orc_rng_next(orc_rng* g) {
  if (g->mti >= MT_N) mt_twist(g);
  uint64_t x = g->mt[g->mti++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}

/* workload.hpp:20 */
double orc_rng_uniform01(orc_rng* g) { return (double)(orc_rng_next(g) >> 11) * 0x1.0p-53; }

/* workload.cpp:16-24: rejection sampling against the largest multiple of n */
int orc_rng_uniform_index(orc_rng* g, uint64_t n, uint64_t* out) {
  if (n == 0) return ORC_EINVAL;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t x;
  do {
    x = orc_rng_next(g);
  } while (x >= limit);
  *out = x % n;
  return 0;
}

/* workload.cpp:26-29 */
int orc_rng_uniform_int(orc_rng* g, int lo, int hi, int* out) {
  if (hi < lo) return ORC_EINVAL;
  uint64_t k;
  orc_rng_uniform_index(g, (uint64_t)(hi - lo) + 1, &k);
  *out = lo + (int)k;
  return 0;
}

/* workload.cpp:31-36: std::upper_bound over the cumulative weights */
size_t orc_rng_discrete(orc_rng* g, const double* cumulative, size_t n, double total) {
  const double u = orc_rng_uniform01(g) * total;
  size_t lo = 0, hi = n; /* first index with cumulative[i] > u */
  while (lo < hi) {
    const size_t mid = lo + (hi - lo) / 2;
    if (u < cumulative[mid]) hi = mid; else lo = mid + 1;
  }
  if (lo == n) return n - 1;
  return lo;
}

/* experiments.cpp:14-18, test_sgmv.cpp:21-25 */
void orc_rng_fill_pm1(orc_rng* g, double* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = orc_rng_uniform01(g) * 2.0 - 1.0;
}

/* workload.hpp:33-38: Fisher-Yates from the end */
void orc_rng_shuffle_i64(orc_rng* g, int64_t* v, size_t n) {
  for (size_t i = n; i > 1; --i) {
    uint64_t j;
    orc_rng_uniform_index(g, (uint64_t)i, &j);
    const int64_t t = v[i - 1];
    v[i - 1] = v[j];
    v[j] = t;
  }
}

/* workload.cpp:38-44: splitmix64 finalizer */
uint64_t orc_derive_seed(uint64_t seed, uint64_t stream) {
  uint64_t z = seed + 0x9E3779B97F4A7C15ull * (stream + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* workload.cpp:92-104 */
int orc_model_count_for(int n, int popularity) {
  if (n <= 0) return 0;
  switch (popularity) {
    case ORC_DISTINCT: return n;
    case ORC_IDENTICAL: return 1;
    case ORC_UNIFORM:
    case ORC_SKEWED: return (int)ceil(sqrt((double)n));
  }
  return 0;
}

/* workload.cpp:106-143 */
int orc_assign_models(int n, int popularity, double alpha, uint64_t seed, int64_t* out) {
  if (n < 0) return ORC_EINVAL;
  if (n == 0) return 0;
  for (int i = 0; i < n; ++i) out[i] = 0;
  orc_rng g;
  orc_rng_seed(&g, seed);
  switch (popularity) {
    case ORC_DISTINCT:
      for (int i = 0; i < n; ++i) out[i] = i;
      break;
    case ORC_IDENTICAL:
      break;
    case ORC_UNIFORM: {
      const int m = orc_model_count_for(n, popularity);
      for (int i = 0; i < n; ++i) out[i] = i % m;
      orc_rng_shuffle_i64(&g, out, (size_t)n);
      break;
    }
    case ORC_SKEWED: {
      if (alpha <= 1.0) return ORC_EINVAL;
      const int m = orc_model_count_for(n, popularity);
      double* cumulative = (double*)malloc(sizeof(double) * (size_t)m);
      double total = 0.0, w = 1.0;
      for (int i = 0; i < m; ++i) {
        total += w;
        cumulative[i] = total;
        w /= alpha;
      }
      for (int i = 0; i < n; ++i) out[i] = (int64_t)orc_rng_discrete(&g, cumulative, (size_t)m, total);
      free(cumulative);
      break;
    }
    default:
      return ORC_EINVAL;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* SGMV operators                                                            */
/* ------------------------------------------------------------------------ */

/* sgmv.cpp:31-38 (Segments ctor invariants) */
int orc_check_segments(const size_t* bounds, size_t nseg) {
  if (bounds[0] != 0) return ORC_EINVAL;
  for (size_t i = 1; i <= nseg; ++i)
    if (bounds[i] <= bounds[i - 1]) return ORC_EINVAL;
  return 0;
}

/* sgmv.cpp:105-119: seg -> row -> k -> d, ascending d, overwrite */
int orc_sgmv_shrink(const double* x, size_t h_in, const size_t* bounds, size_t nseg,
                    const double* A, size_t rank, double* v) {
  if (orc_check_segments(bounds, nseg)) return ORC_EINVAL;
  for (size_t s = 0; s < nseg; ++s) {
    const double* a = A + s * h_in * rank;
    for (size_t j = bounds[s]; j < bounds[s + 1]; ++j) {
      for (size_t k = 0; k < rank; ++k) {
        double acc = 0.0;
        for (size_t d = 0; d < h_in; ++d) acc += x[j * h_in + d] * a[d * rank + k];
        v[j * rank + k] = acc;
      }
    }
  }
  return 0;
}

/* sgmv.cpp:121-136: seg -> row -> c -> k, ascending k, overwrite */
int orc_sgmv_expand(const double* v, size_t rank, const size_t* bounds, size_t nseg,
                    const double* B, size_t h_out, double* y) {
  if (orc_check_segments(bounds, nseg)) return ORC_EINVAL;
  for (size_t s = 0; s < nseg; ++s) {
    const double* b = B + s * rank * h_out;
    for (size_t j = bounds[s]; j < bounds[s + 1]; ++j) {
      for (size_t c = 0; c < h_out; ++c) {
        double acc = 0.0;
        for (size_t k = 0; k < rank; ++k) acc += v[j * rank + k] * b[k * h_out + c];
        y[j * h_out + c] = acc;
      }
    }
  }
  return 0;
}

/* sgmv.cpp:138-141: expand(shrink(batch)); empty batch returns 0x0 */
int orc_lora_addon(const double* x, size_t h_in, const size_t* bounds, size_t nseg,
                   const double* A, const double* B, size_t rank, size_t h_out, double* y) {
  if (nseg == 0) return 0;
  const size_t rows = bounds[nseg];
  double* v = (double*)malloc(sizeof(double) * (rows * rank != 0 ? rows * rank : 1));
  int st = orc_sgmv_shrink(x, h_in, bounds, nseg, A, rank, v);
  if (!st) st = orc_sgmv_expand(v, rank, bounds, nseg, B, h_out, y);
  free(v);
  return st;
}

/* sgmv.cpp:9-19: i -> k -> j accumulation */
static void matmul(const double* a, size_t m, size_t kdim, const double* b, size_t n, double* out) {
  for (size_t i = 0; i < m * n; ++i) out[i] = 0.0;
  for (size_t i = 0; i < m; ++i)
    for (size_t k = 0; k < kdim; ++k) {
      const double aik = a[i * kdim + k];
      for (size_t j = 0; j < n; ++j) out[i * n + j] += aik * b[k * n + j];
    }
}

/* sgmv.cpp:143-155: x*w + lora_addon */
int orc_dense_projection(const double* x, size_t h_in, const size_t* bounds, size_t nseg,
                         const double* A, const double* B, size_t rank, size_t h_out,
                         const double* w, double* y) {
  const size_t rows = nseg ? bounds[nseg] : 0;
  if (rows == 0) return 0;
  matmul(x, rows, h_in, w, h_out, y);
  double* addon = (double*)malloc(sizeof(double) * rows * h_out);
  int st = orc_lora_addon(x, h_in, bounds, nseg, A, B, rank, h_out, addon);
  if (!st)
    for (size_t i = 0; i < rows * h_out; ++i) y[i] += addon[i];
  free(addon);
  return st;
}

/* sgmv.cpp:157-184: per-row tmp = x*A accumulated d-major, then tmp*B */
int orc_lora_loop_oracle(const double* x, size_t h_in, const size_t* bounds, size_t nseg,
                         const double* A, const double* B, size_t rank, size_t h_out,
                         double* y) {
  if (nseg == 0) return 0;
  if (orc_check_segments(bounds, nseg)) return ORC_EINVAL;
  double* tmp = (double*)malloc(sizeof(double) * rank);
  for (size_t s = 0; s < nseg; ++s) {
    const double* a = A + s * h_in * rank;
    const double* b = B + s * rank * h_out;
    for (size_t j = bounds[s]; j < bounds[s + 1]; ++j) {
      for (size_t k = 0; k < rank; ++k) tmp[k] = 0.0;
      for (size_t d = 0; d < h_in; ++d) {
        const double xd = x[j * h_in + d];
        for (size_t k = 0; k < rank; ++k) tmp[k] += xd * a[d * rank + k];
      }
      for (size_t c = 0; c < h_out; ++c) {
        double acc = 0.0;
        for (size_t k = 0; k < rank; ++k) acc += tmp[k] * b[k * h_out + c];
        y[j * h_out + c] = acc;
      }
    }
  }
  free(tmp);
  return 0;
}

/* sgmv.cpp:186-217: gather per-row adapter, then row-wise products (k -> d) */
int orc_gather_bmm_oracle(const double* x, size_t h_in, const size_t* bounds, size_t nseg,
                          const double* A, const double* B, size_t rank, size_t h_out,
                          double* y) {
  if (nseg == 0) return 0;
  if (orc_check_segments(bounds, nseg)) return ORC_EINVAL;
  const size_t rows = bounds[nseg];
  size_t* row_seg = (size_t*)malloc(sizeof(size_t) * rows);
  for (size_t s = 0; s < nseg; ++s)
    for (size_t j = bounds[s]; j < bounds[s + 1]; ++j) row_seg[j] = s;
  double* v = (double*)malloc(sizeof(double) * rank);
  for (size_t j = 0; j < rows; ++j) {
    const double* a = A + row_seg[j] * h_in * rank;
    const double* b = B + row_seg[j] * rank * h_out;
    for (size_t k = 0; k < rank; ++k) {
      v[k] = 0.0;
      for (size_t d = 0; d < h_in; ++d) v[k] += x[j * h_in + d] * a[d * rank + k];
    }
    for (size_t c = 0; c < h_out; ++c) {
      double acc = 0.0;
      for (size_t k = 0; k < rank; ++k) acc += v[k] * b[k * h_out + c];
      y[j * h_out + c] = acc;
    }
  }
  free(v);
  free(row_seg);
  return 0;
}

/* sgmv.cpp:21-29 */
double orc_max_abs_diff(const double* a, const double* b, size_t n) {
  double worst = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double d = fabs(a[i] - b[i]);
    if (d > worst) worst = d;
  }
  return worst;
}

/* ------------------------------------------------------------------------ */
/* verify_sgmv trial generation: experiments.cpp:35-76                        */
/* ------------------------------------------------------------------------ */
int orc_verify_next_trial(orc_rng* g, int trial, size_t* h_in_out, size_t* h_out_out,
                          size_t* rank_out, size_t* rows_out, size_t* nseg_out, size_t* bounds,
                          int64_t* seg_ids, double* x, double* A, double* B) {
  static const size_t dims[] = {8, 64, 128};
  static const size_t ranks[] = {8, 16, 32, 64};
  const int pop = trial % 4; /* experiments.cpp:20-31 */
  uint64_t k;
  orc_rng_uniform_index(g, 3, &k);
  const size_t h_in = dims[k];
  orc_rng_uniform_index(g, 3, &k);
  const size_t h_out = dims[k];
  size_t fitting[4], nfit = 0;
  for (int i = 0; i < 4; ++i)
    if (ranks[i] <= (h_in < h_out ? h_in : h_out)) fitting[nfit++] = ranks[i];
  orc_rng_uniform_index(g, nfit, &k);
  const size_t rank = fitting[k];
  const int max_rows = pop == ORC_DISTINCT ? 8 : 64;
  int rows;
  orc_rng_uniform_int(g, 1, max_rows, &rows);
  int64_t assignment[64];
  orc_assign_models(rows, pop, 1.5, orc_rng_next(g), assignment);

  /* std::map<LoraId, vector<int>>: ascending id, members in original order */
  int64_t ids[64];
  size_t nids = 0;
  for (int i = 0; i < rows; ++i) {
    size_t p = 0;
    while (p < nids && ids[p] != assignment[i]) ++p;
    if (p == nids) ids[nids++] = assignment[i];
  }
  for (size_t i = 1; i < nids; ++i) /* insertion sort ascending */
    for (size_t j = i; j > 0 && ids[j - 1] > ids[j]; --j) {
      const int64_t t = ids[j];
      ids[j] = ids[j - 1];
      ids[j - 1] = t;
    }
  bounds[0] = 0;
  size_t cursor = 0;
  for (size_t s = 0; s < nids; ++s) {
    size_t members = 0;
    for (int i = 0; i < rows; ++i) members += assignment[i] == ids[s];
    /* g++ evaluates emplace_back's arguments right to left: B, then A. */
    orc_rng_fill_pm1(g, B + s * rank * h_out, rank * h_out);
    orc_rng_fill_pm1(g, A + s * h_in * rank, h_in * rank);
    for (size_t m = 0; m < members; ++m) {
      orc_rng_fill_pm1(g, x + cursor * h_in, h_in);
      ++cursor;
    }
    bounds[s + 1] = cursor;
    seg_ids[s] = ids[s];
  }
  *h_in_out = h_in;
  *h_out_out = h_out;
  *rank_out = rank;
  *rows_out = (size_t)rows;
  *nseg_out = nids;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Cost model: cost_model.cpp:8-40, 55-61                                     */
/* ------------------------------------------------------------------------ */
double orc_sgmv_flop(int64_t n, int64_t rows, int64_t h_in, int64_t h_out) {
  (void)n;
  return 2.0 * (double)rows * (double)h_in * (double)h_out;
}

double orc_sgmv_io_bytes(int64_t n, int64_t rows, int64_t h_in, int64_t h_out, int elem_bytes) {
  const double r = (double)rows;
  const double weights = (double)n * (double)h_in * (double)h_out;
  return (r * ((double)h_in + (double)h_out) + weights) * (double)elem_bytes;
}

double orc_arithmetic_intensity(int64_t n, int64_t rows, int64_t h_in, int64_t h_out,
                                int elem_bytes) {
  const double io = orc_sgmv_io_bytes(n, rows, h_in, h_out, elem_bytes);
  if (io <= 0.0) return NAN;
  return orc_sgmv_flop(n, rows, h_in, h_out) / io;
}

double orc_sgmv_latency(int64_t n, int64_t rows, int64_t h_in, int64_t h_out, double peak_flops,
                        double mem_bw, double kernel_overhead, int elem_bytes) {
  const double c = orc_sgmv_flop(n, rows, h_in, h_out) / peak_flops;
  const double m = orc_sgmv_io_bytes(n, rows, h_in, h_out, elem_bytes) / mem_bw;
  double t = c > m ? c : m;
  return t > kernel_overhead ? t : kernel_overhead;
}

double orc_gather_bmm_extra_elements(int64_t n, int64_t rows, int64_t h_in, int64_t h_out) {
  (void)n;
  return 2.0 * (double)rows * (double)h_in * (double)h_out;
}

double orc_adapter_pair_io_bytes(double rows, double models, double h, double r, int elem_bytes) {
  return 2.0 * (rows * (h + r) + models * h * r) * (double)elem_bytes;
}

double orc_adapter_pair_flop(double rows, double h, double r) { return 4.0 * rows * h * r; }

/* ------------------------------------------------------------------------ */
/* plan_batch segment construction, MultiLora mode: simulator.cpp:267-310     */
/* ------------------------------------------------------------------------ */
int orc_plan_segments(size_t nreq, const int64_t* req_lora, const uint8_t* req_prefill_done,
                      const int32_t* req_prompt, int64_t* prefill, int64_t* decodes,
                      size_t* n_decodes, size_t* bounds, int64_t* seg_loras, size_t* nseg) {
  *prefill = -1;
  for (size_t i = 0; i < nreq; ++i)
    if (!req_prefill_done[i]) { *prefill = (int64_t)i; break; }
  /* distinct decode loras, ascending */
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (nreq ? nreq : 1));
  size_t norder = 0;
  for (size_t i = 0; i < nreq; ++i) {
    if (!req_prefill_done[i]) continue;
    size_t p = 0;
    while (p < norder && order[p] != req_lora[i]) ++p;
    if (p == norder) order[norder++] = req_lora[i];
  }
  for (size_t i = 1; i < norder; ++i)
    for (size_t j = i; j > 0 && order[j - 1] > order[j]; --j) {
      const int64_t t = order[j];
      order[j] = order[j - 1];
      order[j - 1] = t;
    }
  /* the prefill's adapter group first (simulator.cpp:280-287) */
  if (*prefill >= 0) {
    const int64_t pl = req_lora[*prefill];
    for (size_t p = 0; p < norder; ++p)
      if (order[p] == pl) {
        for (size_t q = p; q > 0; --q) order[q] = order[q - 1];
        order[0] = pl;
        break;
      }
  }
  size_t acc = 0, ns = 0, nd = 0;
  bounds[0] = 0;
#define PUSH_ROWS(lora, nrows)                                     \
  do {                                                             \
    acc += (nrows);                                                \
    if (ns > 0 && seg_loras[ns - 1] == (lora)) {                   \
      bounds[ns] = acc;                                            \
    } else {                                                       \
      seg_loras[ns] = (lora);                                      \
      bounds[++ns] = acc;                                          \
    }                                                              \
  } while (0)
  if (*prefill >= 0) PUSH_ROWS(req_lora[*prefill], (size_t)req_prompt[*prefill]);
  for (size_t p = 0; p < norder; ++p) {
    size_t members = 0;
    for (size_t i = 0; i < nreq; ++i)
      if (req_prefill_done[i] && req_lora[i] == order[p]) {
        decodes[nd++] = (int64_t)i;
        ++members;
      }
    PUSH_ROWS(order[p], members);
  }
#undef PUSH_ROWS
  *n_decodes = nd;
  *nseg = ns;
  free(order);
  return 0;
}
