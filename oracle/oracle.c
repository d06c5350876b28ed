/*
 * TEST INFRASTRUCTURE ONLY — CPU parity oracle. See oracle.h for what is
 * pinned (metadata, against oracle/_ref) and what is parity-unpinned (layer
 * arithmetic, restated from the paper's equations).
 */
#include "oracle.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* metadata restatement                                                      */
/* ------------------------------------------------------------------------ */

/* R:proj/src/placement.cpp:52-68 — ePerGPU = ceil(E/n); split i = smallest
 * nid in (last, N] with row_ptr[nid] >= min(row_ptr[last] + ePerGPU, E);
 * N when last == N. Linear scan like R:proj/tests/test_util.hpp:31-53. */
void orc_split_points(uint64_t n, const uint64_t* row_ptr, uint32_t num_gpus,
                      uint64_t* out) {
  const uint64_t e = row_ptr[n];
  const uint64_t per = (e + num_gpus - 1) / num_gpus;
  uint64_t last = 0;
  for (uint32_t i = 0; i + 1 < num_gpus; ++i) {
    uint64_t nid = n;
    if (last < n) {
      uint64_t target = row_ptr[last] + per;
      if (target > e) target = e;
      for (uint64_t c = last + 1; c <= n; ++c)
        if (row_ptr[c] >= target) {
          nid = c;
          break;
        }
    }
    out[i] = nid;
    last = nid;
  }
}

/* R:proj/src/placement.cpp:86-104 */
void orc_placement(uint64_t n, const uint64_t* row_ptr, uint32_t num_gpus,
                   int mode, uint64_t* ranges) {
  if (mode == 0) {
    const uint64_t per = (n + num_gpus - 1) / num_gpus;
    for (uint32_t i = 0; i < num_gpus; ++i) {
      uint64_t lb = (uint64_t)i * per, ub = (uint64_t)(i + 1) * per;
      ranges[2 * i] = lb < n ? lb : n;
      ranges[2 * i + 1] = ub < n ? ub : n;
    }
    return;
  }
  uint64_t* pts = (uint64_t*)malloc(sizeof(uint64_t) * (num_gpus + 1));
  orc_split_points(n, row_ptr, num_gpus, pts);
  uint64_t lb = 0;
  for (uint32_t i = 0; i < num_gpus; ++i) {
    uint64_t ub = (i + 1 < num_gpus) ? pts[i] : n;
    ranges[2 * i] = lb;
    ranges[2 * i + 1] = ub;
    lb = ub;
  }
  free(pts);
}

/* R:proj/src/placement.cpp:108-119 — first range whose ub is past id. */
void orc_translate(uint32_t num_gpus, const uint64_t* ranges, uint64_t id,
                   uint32_t* gpu, uint64_t* off) {
  for (uint32_t g = 0; g < num_gpus; ++g)
    if (id < ranges[2 * g + 1]) {
      *gpu = g;
      *off = id - ranges[2 * g];
      return;
    }
  *gpu = num_gpus;
  *off = 0;
}

/* R:proj/src/workload.cpp:26-58 (ownership split, order kept) and 60-82
 * (ceil(deg/ps) slices per row of each kind). chunk = (lb, ub) of `gpu`. */
void orc_partition_counts(uint64_t n, const uint64_t* row_ptr,
                          const uint64_t* col, uint32_t num_gpus,
                          const uint64_t* ranges, const uint64_t* chunk,
                          uint32_t gpu, uint32_t ps, uint64_t* counts) {
  (void)n;
  uint64_t lp = 0, rp = 0, le = 0, re = 0;
  for (uint64_t v = chunk[0]; v < chunk[1]; ++v) {
    uint64_t nl = 0, nr = 0;
    for (uint64_t k = row_ptr[v]; k < row_ptr[v + 1]; ++k) {
      uint32_t g;
      uint64_t off;
      orc_translate(num_gpus, ranges, col[k], &g, &off);
      if (g == gpu)
        ++nl;
      else
        ++nr;
    }
    lp += (nl + ps - 1) / ps;
    rp += (nr + ps - 1) / ps;
    le += nl;
    re += nr;
  }
  counts[0] = lp;
  counts[1] = rp;
  counts[2] = le;
  counts[3] = re;
}

/* R:proj/src/workload.cpp:103-124 */
uint32_t orc_warp_tasks(uint64_t n_local, uint64_t n_remote, uint32_t dist,
                        uint64_t w, uint8_t* kinds, uint32_t* idx) {
  uint32_t k = 0;
  const uint64_t b = w * dist;
  for (uint64_t i = b; i < b + dist && i < n_local; ++i) {
    kinds[k] = 0;
    idx[k++] = (uint32_t)i;
  }
  for (uint64_t i = b; i < b + dist && i < n_remote; ++i) {
    kinds[k] = 1;
    idx[k++] = (uint32_t)i;
  }
  return k;
}

/* ------------------------------------------------------------------------ */
/* layer forward                                                             */
/* ------------------------------------------------------------------------ */

static void set_threads(int threads) {
  if (threads > 0) omp_set_num_threads(threads);
}

static double* inv_sqrt_deg(uint64_t n, const uint64_t* row_ptr) {
  double* s = (double*)malloc(sizeof(double) * (n ? n : 1));
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < (int64_t)n; ++v)
    s[v] = 1.0 / sqrt((double)(row_ptr[v + 1] - row_ptr[v]) + 1.0);
  return s;
}

#define RELU(x) ((x) > 0 ? (x) : 0)

/* Aggregate (R:PAPER.md:33-38): a_v = self_scale*h_v + Σ_{u∈N(v)} h_u. */
#define DEFINE_AGG(NAME, ACC)                                                  \
  static void NAME(uint64_t n, const uint64_t* row_ptr, const uint64_t* col,   \
                   const float* x, uint32_t d, double self_scale,             \
                   const double* isd, int relu_in, uint64_t lo, uint64_t hi,  \
                   float* out) {                                              \
    (void)n;                                                                  \
    _Pragma("omp parallel")                                                   \
    {                                                                          \
      ACC* acc = (ACC*)malloc(sizeof(ACC) * (d ? d : 1));                     \
      _Pragma("omp for schedule(dynamic, 256)")                               \
      for (int64_t vv = (int64_t)lo; vv < (int64_t)hi; ++vv) {                \
        const uint64_t v = (uint64_t)vv;                                       \
        const ACC sv = isd ? (ACC)isd[v] : (ACC)1;                            \
        for (uint32_t j = 0; j < d; ++j) {                                    \
          ACC h = (ACC)x[v * d + j];                                          \
          if (relu_in) h = RELU(h);                                           \
          acc[j] = (ACC)self_scale * h * sv;                                  \
        }                                                                     \
        for (uint64_t k = row_ptr[v]; k < row_ptr[v + 1]; ++k) {              \
          const uint64_t u = col[k];                                          \
          const ACC su = isd ? (ACC)isd[u] : (ACC)1;                          \
          const float* xu = x + u * d;                                        \
          if (relu_in)                                                        \
            for (uint32_t j = 0; j < d; ++j) acc[j] += RELU((ACC)xu[j]) * su; \
          else                                                                \
            for (uint32_t j = 0; j < d; ++j) acc[j] += (ACC)xu[j] * su;       \
        }                                                                     \
        for (uint32_t j = 0; j < d; ++j)                                      \
          out[(v - lo) * d + j] = (float)(acc[j] * sv);                       \
      }                                                                        \
      free(acc);                                                              \
    }                                                                          \
  }

DEFINE_AGG(agg_f64, double)
DEFINE_AGG(agg_f32, float)

void orc_aggregate(int acc64, int threads, uint64_t n, const uint64_t* row_ptr,
                   const uint64_t* col, const float* x, uint32_t d,
                   double self_scale, int norm, int relu_in, uint64_t row_lo,
                   uint64_t row_hi, float* out) {
  set_threads(threads);
  double* isd = norm ? inv_sqrt_deg(n, row_ptr) : NULL;
  if (acc64)
    agg_f64(n, row_ptr, col, x, d, self_scale, isd, relu_in, row_lo, row_hi,
            out);
  else
    agg_f32(n, row_ptr, col, x, d, self_scale, isd, relu_in, row_lo, row_hi,
            out);
  free(isd);
}

/* Update (R:PAPER.md:38-40, "a fully-connected NN layer"). */
#define DEFINE_DENSE(NAME, ACC)                                                \
  static void NAME(uint64_t n, const float* x, uint32_t k, const float* w,    \
                   const float* b, uint32_t m, int act, float* y) {           \
    _Pragma("omp parallel")                                                   \
    {                                                                          \
      ACC* acc = (ACC*)malloc(sizeof(ACC) * (m ? m : 1));                     \
      _Pragma("omp for schedule(static)")                                     \
      for (int64_t r = 0; r < (int64_t)n; ++r) {                              \
        for (uint32_t j = 0; j < m; ++j) acc[j] = b ? (ACC)b[j] : (ACC)0;     \
        const float* xr = x + (uint64_t)r * k;                                \
        for (uint32_t i = 0; i < k; ++i) {                                    \
          const ACC xi = (ACC)xr[i];                                          \
          const float* wi = w + (uint64_t)i * m;                              \
          for (uint32_t j = 0; j < m; ++j) acc[j] += xi * (ACC)wi[j];         \
        }                                                                     \
        float* yr = y + (uint64_t)r * m;                                      \
        if (act == 1) {                                                       \
          for (uint32_t j = 0; j < m; ++j) yr[j] = (float)RELU(acc[j]);       \
        } else if (act == 2) {                                                \
          ACC mx = acc[0];                                                    \
          for (uint32_t j = 1; j < m; ++j) mx = acc[j] > mx ? acc[j] : mx;    \
          ACC s = 0;                                                          \
          for (uint32_t j = 0; j < m; ++j) {                                  \
            acc[j] = (ACC)exp((double)(acc[j] - mx));                         \
            s += acc[j];                                                      \
          }                                                                   \
          for (uint32_t j = 0; j < m; ++j) yr[j] = (float)(acc[j] / s);       \
        } else {                                                              \
          for (uint32_t j = 0; j < m; ++j) yr[j] = (float)acc[j];             \
        }                                                                     \
      }                                                                        \
      free(acc);                                                              \
    }                                                                          \
  }

DEFINE_DENSE(dense_f64, double)
DEFINE_DENSE(dense_f32, float)

void orc_dense(int acc64, int threads, uint64_t n, const float* x, uint32_t k,
               const float* w, const float* b, uint32_t m, int act, float* y) {
  set_threads(threads);
  if (acc64)
    dense_f64(n, x, k, w, b, m, act, y);
  else
    dense_f32(n, x, k, w, b, m, act, y);
}

static void softmax_rows(int threads, uint64_t n, uint32_t m, const float* in,
                         float* out) {
  set_threads(threads);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < (int64_t)n; ++r) {
    const float* a = in + (uint64_t)r * m;
    float* o = out + (uint64_t)r * m;
    double mx = a[0], s = 0;
    for (uint32_t j = 1; j < m; ++j) mx = a[j] > mx ? a[j] : mx;
    for (uint32_t j = 0; j < m; ++j) s += exp((double)a[j] - mx);
    for (uint32_t j = 0; j < m; ++j) o[j] = (float)(exp((double)a[j] - mx) / s);
  }
}

/* Z = softmax(Â ReLU(Â X W1) W2) (R:PAPER.md:504-508). Â X W1 is evaluated
 * as Â (X W1) (associativity; exact in real arithmetic) and the second layer
 * as (Â H) W2, aggregating at min(in, out) width — the same association the
 * product uses, stated here so the fp64 oracle and the GPU round the same
 * terms. */
void orc_gcn2_forward(int acc64, int threads, uint64_t n,
                      const uint64_t* row_ptr, const uint64_t* col,
                      const float* x, uint32_t d, const float* w1,
                      uint32_t hidden, const float* w2, uint32_t classes,
                      int norm, float* h1, float* logits, float* z) {
  float* y1 = (float*)malloc(sizeof(float) * n * hidden + 4);
  float* a1 = (float*)malloc(sizeof(float) * n * hidden + 4);
  float* lg = logits ? logits : (float*)malloc(sizeof(float) * n * classes + 4);
  orc_dense(acc64, threads, n, x, d, w1, NULL, hidden, 0, y1);
  orc_aggregate(acc64, threads, n, row_ptr, col, y1, hidden, 1.0, norm, 0, 0,
                n, a1);
  /* layer 2: aggregate ReLU(a1) at width `hidden`, then W2. */
  orc_aggregate(acc64, threads, n, row_ptr, col, a1, hidden, 1.0, norm, 1, 0,
                n, y1);
  if (h1) {
    set_threads(threads);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)(n * hidden); ++i) h1[i] = RELU(a1[i]);
  }
  orc_dense(acc64, threads, n, y1, hidden, w2, NULL, classes, 0, lg);
  if (z) softmax_rows(threads, n, classes, lg, z);
  if (!logits) free(lg);
  free(y1);
  free(a1);
}

void orc_gin_forward(int acc64, int threads, uint64_t n,
                     const uint64_t* row_ptr, const uint64_t* col,
                     const float* x, uint32_t layers, const uint32_t* dims,
                     uint32_t hidden, const float* w1, const float* b1,
                     const float* w2, const float* b2, double eps,
                     float* logits, float* z) {
  uint32_t maxd = hidden;
  for (uint32_t l = 0; l <= layers; ++l) maxd = dims[l] > maxd ? dims[l] : maxd;
  float* h = (float*)malloc(sizeof(float) * n * maxd + 4);
  float* a = (float*)malloc(sizeof(float) * n * maxd + 4);
  float* t = (float*)malloc(sizeof(float) * n * hidden + 4);
  memcpy(h, x, sizeof(float) * n * dims[0]);
  size_t ow1 = 0, ob1 = 0, ow2 = 0, ob2 = 0;
  for (uint32_t l = 0; l < layers; ++l) {
    const uint32_t din = dims[l], dout = dims[l + 1];
    orc_aggregate(acc64, threads, n, row_ptr, col, h, din, 1.0 + eps, 0, 0, 0,
                  n, a);
    orc_dense(acc64, threads, n, a, din, w1 + ow1, b1 + ob1, hidden, 1, t);
    const int last = (l + 1 == layers);
    orc_dense(acc64, threads, n, t, hidden, w2 + ow2, b2 + ob2, dout,
              last ? 0 : 1, h);
    ow1 += (size_t)din * hidden;
    ob1 += hidden;
    ow2 += (size_t)hidden * dout;
    ob2 += dout;
  }
  const uint32_t c = dims[layers];
  if (logits) memcpy(logits, h, sizeof(float) * n * c);
  if (z) softmax_rows(threads, n, c, h, z);
  free(h);
  free(a);
  free(t);
}

/* ------------------------------------------------------------------------ */
/* synthetic inputs for bench.py's reference arm (no product code on it)     */
/* ------------------------------------------------------------------------ */

/* SplitMix64 (R:proj/include/pipeshard/rng.hpp:26-54). */
static uint64_t sm_next(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t sm_below(uint64_t* s, uint64_t n) {
  const uint64_t reject_from = ~0ull - (~0ull % n);
  uint64_t v;
  do v = sm_next(s);
  while (v >= reject_from);
  return v % n;
}
static double sm_unit(uint64_t* s) { return (double)(sm_next(s) >> 11) * 0x1.0p-53; }

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}
static void sort_rows(uint64_t n, const uint64_t* row_ptr, uint64_t* col) {
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < (int64_t)n; ++v)
    qsort(col + row_ptr[v], row_ptr[v + 1] - row_ptr[v], sizeof(uint64_t), cmp_u64);
}

/* R:proj/src/graph.cpp:139-176 — per node one degree draw (uniform: floor(d)
 * + Bernoulli(frac); powerlaw: Pareto alpha 1.6 clipped to [1, N-1]), then
 * that many uniform neighbors, one stream; rows sorted, duplicates kept.
 * Returns E; fills row_ptr[n+1] / col[E] only when col != NULL. */
uint64_t orc_gen_synthetic(int kind, uint64_t n, double avg, uint64_t seed,
                           uint64_t* row_ptr, uint64_t* col) {
  uint64_t s = seed, e = 0;
  const uint64_t whole = (uint64_t)avg;
  const double frac = avg - (double)whole;
  const double alpha = 1.6;
  double x_min = avg * (alpha - 1.0) / alpha;
  if (x_min < 0.5) x_min = 0.5;
  const double neg_inv_alpha = -1.0 / alpha;
  const double cap = n == 1 ? 1.0 : (double)(n - 1);
  const double hi = cap > 1.0 ? cap : 1.0;
  if (row_ptr) row_ptr[0] = 0;
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t deg;
    if (kind == 0) {
      deg = whole + (sm_unit(&s) < frac ? 1 : 0);
    } else {
      const double u = sm_unit(&s);
      double x = floor(x_min * pow(1.0 - u, neg_inv_alpha));
      if (x < 1.0) x = 1.0;
      if (x > hi) x = hi;
      deg = (uint64_t)x;
    }
    for (uint64_t k = 0; k < deg; ++k) {
      const uint64_t c = sm_below(&s, n);
      if (col) col[e] = c;
      ++e;
    }
    if (row_ptr) row_ptr[v + 1] = e;
  }
  if (col && row_ptr) sort_rows(n, row_ptr, col);
  return e;
}

/* RMAT edge stream of the product's generator (csrc/host/graph.cpp gen_rmat;
 * not a reference algorithm — a locality-bearing input): blocks
 * of 65536 edges, block b seeded seed ^ (0xD1B54A32D192ED03 * (b + 1)); per
 * edge scale quadrant draws (a, b, c, 1-a-b-c), out-of-range pairs redrawn.
 * CSR row = source, rows sorted, duplicates kept. row_ptr[n+1], col[m]. */
void orc_gen_rmat(uint64_t n, uint64_t m, uint64_t seed, double a, double b, double c,
                  uint64_t* row_ptr, uint64_t* col) {
  unsigned scale = 0;
  while (n > 1 && (1ull << scale) < n) ++scale;
  const double ab = a + b, abc = a + b + c;
  const uint64_t kBlock = 1u << 16, blocks = (m + kBlock - 1) / kBlock;
  uint64_t* src = (uint64_t*)malloc(sizeof(uint64_t) * (m ? m : 1));
  uint64_t* dst = (uint64_t*)malloc(sizeof(uint64_t) * (m ? m : 1));
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t blk = 0; blk < (int64_t)blocks; ++blk) {
    uint64_t s = seed ^ (0xD1B54A32D192ED03ull * (uint64_t)(blk + 1));
    const uint64_t lo = (uint64_t)blk * kBlock, hi = lo + kBlock < m ? lo + kBlock : m;
    for (uint64_t i = lo; i < hi; ++i) {
      uint64_t u, v;
      do {
        u = v = 0;
        for (unsigned l = 0; l < scale; ++l) {
          const double r = sm_unit(&s);
          const unsigned q = r < a ? 0u : r < ab ? 1u : r < abc ? 2u : 3u;
          u = (u << 1) | (q >> 1);
          v = (v << 1) | (q & 1u);
        }
      } while (u >= n || v >= n);
      src[i] = u;
      dst[i] = v;
    }
  }
  memset(row_ptr, 0, sizeof(uint64_t) * (n + 1));
  for (uint64_t i = 0; i < m; ++i) ++row_ptr[src[i] + 1];
  for (uint64_t v = 0; v < n; ++v) row_ptr[v + 1] += row_ptr[v];
  uint64_t* cur = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  memcpy(cur, row_ptr, sizeof(uint64_t) * n);
  for (uint64_t i = 0; i < m; ++i) col[cur[src[i]]++] = dst[i];
  free(cur);
  free(src);
  free(dst);
  sort_rows(n, row_ptr, col);
}
