/* CPU restatement of the synthetic-world generators -- TEST INFRASTRUCTURE.
 *
 * Builds, on the host cores, the same synthetic BASELINE worlds the device
 * builds (paper_2207_14696_b200/csrc/fg_data.cu, synth.py): the planted-
 * partition power-law CSR graph, the planted labels, the row-addressable
 * feature matrix and its SQ payload (the reference's continuous MSB-first
 * stream, sq.py:114-129 + bitpack.py:17-36).  Used only by
 *   - bench.py --impl reference / cpu_baseline: the CPU reference arm's
 *     world, built without the product library (libfgb200.so is never
 *     loaded by that process);
 *   - tests/: bit-identity of this world with the device world.
 * Every float operation is an IEEE-rounded add/mul/fma/div/sqrt in the same
 * order as fg_detmath.cuh (compiled with -ffp-contract=off), so the results
 * are bit-identical to the device generators.
 *
 * Speed (the reference arm builds papers100M-shape worlds: 1.6e9 edges,
 * 1.4e10 feature values): the generators run over fixed-size batches in
 * separate simple loops that the compiler vectorises (the deterministic
 * functions are branch-free), the position -> node Feistel bijection is
 * tabulated once per graph, the per-class constants of the power law and the
 * class means of the features are computed once.
 *
 * Build: oracle/Makefile (gcc -O3 -ffp-contract=off -pthread), output
 * oracle/_build/libfgoracle[_v4].so (generic x86-64-v3 and AVX-512 builds).
 * Loops run on a small pthread pool (the image has no libgomp); FGO_THREADS
 * overrides the thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#include <time.h>
#include <unistd.h>

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ---------------------------------------------------------- thread pool */
typedef void (*range_fn)(int64_t lo, int64_t hi, void* ctx);
typedef struct {
  int64_t n, chunk;
  int64_t next;
  range_fn fn;
  void* ctx;
} ParJob;

static int fgo_threads(void) {
  const char* e = getenv("FGO_THREADS");
  long v = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
  return v > 0 ? (int)(v > 256 ? 256 : v) : 1;
}

static void* par_worker(void* arg) {
  ParJob* j = (ParJob*)arg;
  for (;;) {
    const int64_t lo = __atomic_fetch_add(&j->next, j->chunk, __ATOMIC_RELAXED);
    if (lo >= j->n) break;
    j->fn(lo, lo + j->chunk < j->n ? lo + j->chunk : j->n, j->ctx);
  }
  return NULL;
}

/* fn over [0, n) in dynamically scheduled chunks on every host thread */
static void par_for(int64_t n, int64_t chunk, range_fn fn, void* ctx) {
  if (n <= 0) return;
  ParJob j = {n, chunk > 0 ? chunk : 1, 0, fn, ctx};
  int T = fgo_threads();
  if ((int64_t)T > (n + j.chunk - 1) / j.chunk) T = (int)((n + j.chunk - 1) / j.chunk);
  pthread_t th[256];
  int started = 0;
  for (int t = 1; t < T; ++t)
    if (pthread_create(&th[started], NULL, par_worker, &j) == 0) ++started;
  par_worker(&j);
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------ hashing */
static inline uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint64_t dbits(double x) { uint64_t b; memcpy(&b, &x, 8); return b; }
static inline double bitsd(uint64_t b) { double x; memcpy(&x, &b, 8); return x; }

/* ------------------------------------------ deterministic float64 math */
/* fg_detmath.cuh det::log2 (branch-free form of the same operations) */
static inline double det_log2(double x) {
  const uint64_t b = dbits(x);
  const int64_t e0 = (int64_t)((b >> 52) & 0x7FF) - 1023;
  const double m0 = bitsd((b & 0xFFFFFFFFFFFFFull) | (1023ull << 52));
  const int big = m0 > 0x1.6a09e667f3bcdp+0;
  const double m = big ? m0 * 0.5 : m0;
  const int64_t e = e0 + big;
  const double s = (m - 1.0) / (m + 1.0);
  const double s2 = s * s;
  double p = 0x1.47ae147ae147bp-5;
  p = fma(p, s2, 0x1.642c8590b2164p-5);
  p = fma(p, s2, 0x1.8618618618618p-5);
  p = fma(p, s2, 0x1.af286bca1af28p-5);
  p = fma(p, s2, 0x1.e1e1e1e1e1e1ep-5);
  p = fma(p, s2, 0x1.1111111111111p-4);
  p = fma(p, s2, 0x1.3b13b13b13b14p-4);
  p = fma(p, s2, 0x1.745d1745d1746p-4);
  p = fma(p, s2, 0x1.c71c71c71c71cp-4);
  p = fma(p, s2, 0x1.2492492492492p-3);
  p = fma(p, s2, 0x1.999999999999ap-3);
  p = fma(p, s2, 0x1.5555555555555p-2);
  p = fma(p, s2, 1.0);
  const double ln_m = (2.0 * s) * p;
  return fma(ln_m, 0x1.71547652b82fep+0, (double)e);
}

/* det::exp2 */
static inline double det_exp2(double y) {
  const double k = floor(y + 0.5);
  const double t = (y - k) * 0x1.62e42fefa39efp-1;
  double p = 0x1.93974a8c07c9dp-37;
  p = fma(p, t, 0x1.6124613a86d09p-33);
  p = fma(p, t, 0x1.1eed8eff8d898p-29);
  p = fma(p, t, 0x1.ae64567f544e4p-26);
  p = fma(p, t, 0x1.27e4fb7789f5cp-22);
  p = fma(p, t, 0x1.71de3a556c734p-19);
  p = fma(p, t, 0x1.a01a01a01a01ap-16);
  p = fma(p, t, 0x1.a01a01a01a01ap-13);
  p = fma(p, t, 0x1.6c16c16c16c17p-10);
  p = fma(p, t, 0x1.1111111111111p-7);
  p = fma(p, t, 0x1.5555555555555p-5);
  p = fma(p, t, 0x1.5555555555555p-3);
  p = fma(p, t, 0.5);
  p = fma(p, t, 1.0);
  p = fma(p, t, 1.0);
  const double scale = bitsd((uint64_t)((int64_t)k + 1023) << 52);
  return p * scale;
}

static inline double det_pow(double base, double e) { return det_exp2(e * det_log2(base)); }

/* det::cos_turns: cos(2 pi t), t in [0, 1) */
static inline double det_cos_turns(double t) {
  const double q = floor(t * 4.0);
  const double th = (t - q * 0.25) * 0x1.921fb54442d18p+2;
  const double t2 = th * th;
  double c = 0x1.0ce396db7f853p-70;
  c = fma(c, -t2, 0x1.e542ba4020225p-62);
  c = fma(c, -t2, 0x1.6827863b97d97p-53);
  c = fma(c, -t2, 0x1.ae7f3e733b81fp-45);
  c = fma(c, -t2, 0x1.93974a8c07c9dp-37);
  c = fma(c, -t2, 0x1.1eed8eff8d898p-29);
  c = fma(c, -t2, 0x1.27e4fb7789f5cp-22);
  c = fma(c, -t2, 0x1.a01a01a01a01ap-16);
  c = fma(c, -t2, 0x1.6c16c16c16c17p-10);
  c = fma(c, -t2, 0x1.5555555555555p-5);
  c = fma(c, -t2, 0.5);
  c = fma(c, -t2, 1.0);
  double s = 0x1.71b8ef6dcf572p-66;
  s = fma(s, -t2, 0x1.2f49b46814157p-57);
  s = fma(s, -t2, 0x1.952c77030ad4ap-49);
  s = fma(s, -t2, 0x1.ae7f3e733b81fp-41);
  s = fma(s, -t2, 0x1.6124613a86d09p-33);
  s = fma(s, -t2, 0x1.ae64567f544e4p-26);
  s = fma(s, -t2, 0x1.71de3a556c734p-19);
  s = fma(s, -t2, 0x1.a01a01a01a01ap-13);
  s = fma(s, -t2, 0x1.1111111111111p-7);
  s = fma(s, -t2, 0x1.5555555555555p-3);
  s = fma(s, -t2, 1.0);
  s = s * th;
  const double r01 = q == 0.0 ? c : -s;
  const double r23 = q == 2.0 ? -c : s;
  return q < 2.0 ? r01 : r23;
}

/* ------------------------------------------------------------ features */
/* fg_data.cu: elem_key / gauss / k_synth */
static inline uint64_t elem_key(uint64_t seed, int64_t i, int64_t j) {
  return splitmix64(seed ^ splitmix64((uint64_t)i * 0x100000001B3ull + (uint64_t)j));
}

static inline float gauss1(uint64_t key) {
  const uint64_t h = splitmix64(key);
  const double u1 = (double)(int64_t)((h >> 40) + 1u) * 0x1p-24;
  const double u2 = (double)(int64_t)(h & 0xFFFFFFu) * 0x1p-24;
  const double ln_u1 = det_log2(u1) * 0x1.62e42fefa39efp-1;
  return (float)(sqrt(-2.0 * ln_u1) * det_cos_turns(u2));
}

#define FB 256 /* feature batch (elements) */

/* z[t] = gauss(key[t]) for a batch: staged loops the compiler vectorises */
static void gauss_batch(const uint64_t* restrict key, int m, float* restrict z) {
  double u1[FB], u2[FB], l[FB], c[FB];
  for (int t = 0; t < m; ++t) {
    const uint64_t h = splitmix64(key[t]);
    u1[t] = (double)(int64_t)((h >> 40) + 1u) * 0x1p-24;
    u2[t] = (double)(int64_t)(h & 0xFFFFFFu) * 0x1p-24;
  }
  for (int t = 0; t < m; ++t) l[t] = det_log2(u1[t]) * 0x1.62e42fefa39efp-1;
  for (int t = 0; t < m; ++t) c[t] = det_cos_turns(u2[t]);
  for (int t = 0; t < m; ++t) z[t] = (float)(sqrt(-2.0 * l[t]) * c[t]);
}

/* Per-column constants of kinds 2 / 3 (the shared direction, the class
 * means): table[c * d + j] = gauss(elem_key(seed ^ K, c, j)). */
typedef struct {
  int kind;
  uint64_t seed;
  int64_t d;
  const int32_t* labels;
  float* table; /* kind 2: [d], kind 3: [classes][d] */
} FeatGen;

static float* column_table(int kind, uint64_t seed, int64_t d, int64_t classes) {
  if (kind != 2 && kind != 3) return NULL;
  const int64_t rows = kind == 2 ? 1 : classes;
  float* t = (float*)malloc(sizeof(float) * (size_t)(rows * d));
  if (!t) return NULL;
  for (int64_t c = 0; c < rows; ++c)
    for (int64_t j = 0; j < d; ++j)
      t[c * d + j] = kind == 2 ? gauss1(elem_key(seed ^ 0xC0FFEEull, -1, j))
                               : gauss1(elem_key(seed ^ 0xC1A55ull, c, j));
  return t;
}

/* out[0 .. d) = row i of the matrix (k_synth) */
static void feature_row(const FeatGen* g, int64_t i, float* restrict out) {
  uint64_t key[FB];
  float z[FB];
  for (int64_t j0 = 0; j0 < g->d; j0 += FB) {
    const int m = (int)(g->d - j0 < FB ? g->d - j0 : FB);
    for (int t = 0; t < m; ++t) key[t] = elem_key(g->seed, i, j0 + t);
    gauss_batch(key, m, z);
    float* o = out + j0;
    switch (g->kind) {
      case 0:
        for (int t = 0; t < m; ++t) o[t] = z[t];
        break;
      case 1: {
        double ex[FB];
        for (int t = 0; t < m; ++t) ex[t] = det_exp2((double)z[t] * 0x1.71547652b82fep+0);
        for (int t = 0; t < m; ++t) {
          const uint64_t sgn = splitmix64(elem_key(g->seed ^ 0x5151ull, i, j0 + t));
          const float mag = (float)ex[t];
          o[t] = (sgn & 1) ? mag : -mag;
        }
        break;
      }
      case 2: {
        const float* s = g->table + j0;
        for (int t = 0; t < m; ++t) {
          const float a = 0.9486833f * s[t], b = 0.31622777f * z[t];
          o[t] = a + b;
        }
        break;
      }
      default: {
        const float* mu = g->table + (int64_t)(g->labels ? g->labels[i] : 0) * g->d + j0;
        for (int t = 0; t < m; ++t) {
          const float a = 0.6f * mu[t], b = 0.8f * z[t];
          o[t] = a + b;
        }
        break;
      }
    }
  }
}

static int64_t max_label(const int32_t* labels, int64_t n) {
  int64_t c = 0;
  for (int64_t i = 0; i < n; ++i) c = labels[i] > c ? labels[i] : c;
  return c + 1;
}

typedef struct {
  const FeatGen* g;
  int64_t row0;
  const int64_t* row_ids;
  float* out;
} SynthCtx;

static void synth_rows(int64_t lo, int64_t hi, void* p) {
  const SynthCtx* c = (const SynthCtx*)p;
  for (int64_t r = lo; r < hi; ++r)
    feature_row(c->g, c->row_ids ? c->row_ids[r] : c->row0 + r, c->out + r * c->g->d);
}

/* rows [row0, row0+rows) (row_ids == NULL) or the listed rows, row-major.
 * `classes` bounds the labels of kind 3 (<= 0: derived from the rows). */
int fgo_synth_features(int kind, uint64_t seed, int64_t row0, const int64_t* row_ids,
                       int64_t rows, int64_t d, const int32_t* labels, int64_t classes,
                       float* out) {
  if (kind < 0 || kind > 3 || rows < 0 || d < 1 || (kind == 3 && !labels)) return 1;
  if (rows == 0) return 0;
  if (kind == 3 && classes <= 0) {
    classes = 0;
    for (int64_t r = 0; r < rows; ++r) {
      const int64_t c = labels[row_ids ? row_ids[r] : row0 + r] + 1;
      classes = c > classes ? c : classes;
    }
  }
  FeatGen g = {kind, seed, d, labels, column_table(kind, seed, d, classes)};
  if ((kind == 2 || kind == 3) && !g.table) return 3;
  SynthCtx c = {&g, row0, row_ids, out};
  par_for(rows, 64, synth_rows, &c);
  free(g.table);
  return 0;
}

/* ----------------------------------------------------------- SQ payload */
/* quantize_sq of rows [0, n) through the reference's bucket thresholds
 * thr[0 .. half-2] (the smallest float |x| whose sq.py:120-127 offset
 * reaches j, found with the reference's formula on the host): code =
 * half + #{t_j <= |x|} for x >= 0 (-0.0 included), half - 1 - # otherwise;
 * k = 1: x >= 0.  Packed MSB-first as one continuous stream
 * (bitpack.py:17-36); 8-row groups start on a byte.  Also counts the
 * zero elements met. */
typedef struct {
  const FeatGen* g;
  int k;
  int64_t n;
  const float* thr;
  uint8_t* payload;
  int64_t zeros;
} EncCtx;

static void sq_encode_groups(int64_t g0, int64_t g1, void* p) {
  EncCtx* x = (EncCtx*)p;
  const int k = x->k, half = 1 << (k - 1);
  const int64_t n = x->n, d = x->g->d, row_bits = d * k;
  float* row = (float*)malloc(sizeof(float) * (size_t)d);
  uint8_t* code = (uint8_t*)malloc((size_t)d);
  int64_t zeros = 0;
  for (int64_t g = g0; g < g1; ++g) {
    const int64_t r1 = 8 * g + 8 < n ? 8 * g + 8 : n;
    uint32_t acc = 0;
    int nacc = 0;
    int64_t byte = g * row_bits; /* 8 rows * row_bits / 8 */
    for (int64_t i = 8 * g; i < r1; ++i) {
      feature_row(x->g, i, row);
      for (int64_t j = 0; j < d; ++j) {
        const float v = row[j];
        const float a = fabsf(v);
        int c = 0;
        for (int t = 0; t < half - 1; ++t) c += x->thr[t] <= a;
        const int neg = v < 0.0f; /* -0.0 counts as >= 0 */
        zeros += v == 0.0f;
        code[j] = (uint8_t)(k == 1 ? (neg ? 0 : 1) : (neg ? half - 1 - c : half + c));
      }
      for (int64_t j = 0; j < d; ++j) {
        acc = (acc << k) | code[j];
        nacc += k;
        if (nacc >= 8) {
          x->payload[byte++] = (uint8_t)(acc >> (nacc - 8));
          nacc -= 8;
        }
      }
    }
    if (nacc) x->payload[byte] = (uint8_t)(acc << (8 - nacc));
  }
  free(row);
  free(code);
  __atomic_fetch_add(&x->zeros, zeros, __ATOMIC_RELAXED);
}

/* returns the number of zero elements met (>= 0), or < 0 on error */
int64_t fgo_sq_encode_stream(int kind, uint64_t seed, int64_t n, int64_t d, const int32_t* labels,
                             int64_t classes, int k, const float* thr, uint8_t* payload) {
  if (k < 1 || k > 8 || (kind == 3 && !labels)) return -1;
  memset(payload, 0, (size_t)((n * d * k + 7) / 8));
  if (kind == 3 && classes <= 0) classes = max_label(labels, n);
  FeatGen g = {kind, seed, d, labels, column_table(kind, seed, d, classes)};
  EncCtx x = {&g, k, n, thr, payload, 0};
  par_for((n + 7) / 8, 64, sq_encode_groups, &x);
  free(g.table);
  return x.zeros;
}

/* Values at flat positions pos[0 .. m) (sorted) of the n x d matrix: the
 * linspace-strided fit sample of sq.py:104-106, its nonzero ranks mapped to
 * positions with the zero list of fgo_find_zeros. */
typedef struct {
  const FeatGen* g;
  const int64_t* pos;
  int64_t m;
  float* out;
} PosCtx;

static void values_rows(int64_t lo, int64_t hi, void* p) {
  const PosCtx* x = (const PosCtx*)p;
  const int64_t d = x->g->d;
  float* row = (float*)malloc(sizeof(float) * (size_t)d);
  /* [lo, hi) indexes pos[]; consecutive positions of one row share it */
  int64_t cur = -1;
  for (int64_t q = lo; q < hi; ++q) {
    const int64_t i = x->pos[q] / d;
    if (i != cur) {
      feature_row(x->g, i, row);
      cur = i;
    }
    x->out[q] = row[x->pos[q] - i * d];
  }
  free(row);
}

int fgo_values_at(int kind, uint64_t seed, int64_t d, const int32_t* labels, int64_t classes,
                  const int64_t* pos, int64_t m, float* out) {
  if (kind == 3 && classes <= 0) return 1;
  FeatGen g = {kind, seed, d, labels, column_table(kind, seed, d, classes)};
  PosCtx x = {&g, pos, m, out};
  par_for(m, 4096, values_rows, &x);
  free(g.table);
  return 0;
}

/* Flat positions of the zero elements of rows [0, n) (fit_sq's
 * `flat[flat != 0]`, sq.py:99, needs them to map the linspace sample's
 * nonzero ranks back to positions).  Writes at most cap positions (unsorted
 * across row chunks) and returns the total count. */
typedef struct {
  const FeatGen* g;
  int64_t* pos;
  int64_t cap, count;
} ZeroCtx;

static void zero_rows(int64_t lo, int64_t hi, void* p) {
  ZeroCtx* x = (ZeroCtx*)p;
  const int64_t d = x->g->d;
  float* row = (float*)malloc(sizeof(float) * (size_t)d);
  for (int64_t i = lo; i < hi; ++i) {
    feature_row(x->g, i, row);
    for (int64_t j = 0; j < d; ++j)
      if (row[j] == 0.0f) {
        const int64_t slot = __atomic_fetch_add(&x->count, 1, __ATOMIC_RELAXED);
        if (slot < x->cap) x->pos[slot] = i * d + j;
      }
  }
  free(row);
}

int64_t fgo_find_zeros(int kind, uint64_t seed, int64_t n, int64_t d, const int32_t* labels,
                       int64_t classes, int64_t* pos, int64_t cap) {
  if (kind == 3 && classes <= 0) return -1;
  FeatGen g = {kind, seed, d, labels, column_table(kind, seed, d, classes)};
  ZeroCtx x = {&g, pos, cap, 0};
  par_for(n, 256, zero_rows, &x);
  free(g.table);
  return x.count;
}

/* --------------------------------------------------------------- graphs */
/* fg_data.cu: GraphGen / feistel / powerlaw_rank / gen_edge */
typedef struct {
  uint64_t seed;
  int64_t n, classes;
  double alpha, homophily;
  int bits;
  /* derived once: class sizes q / q+1, their power-law (hi - 1) and 1/a1 */
  int64_t q, r;
  double him1[2], inv_a1;
  const int32_t* perm; /* position -> node id (the Feistel bijection) */
} GraphGen;

static inline int64_t feistel(int64_t x, const GraphGen* g) {
  const int half = g->bits / 2;
  const uint64_t mask = (1ull << half) - 1;
  uint64_t y = (uint64_t)x;
  for (int walk = 0; walk < 512; ++walk) {
    uint64_t lo = y & mask, hi = y >> half;
    for (int r = 0; r < 4; ++r) {
      const uint64_t f = splitmix64(lo ^ (g->seed * 0x9E3779B97F4A7C15ull + r)) & mask;
      const uint64_t t = hi ^ f;
      hi = lo;
      lo = t;
    }
    y = (hi << half) | lo;
    if ((int64_t)y < g->n) return (int64_t)y;
  }
  return x;
}

static void make_gen(GraphGen* g, uint64_t seed, int64_t n, int64_t classes, double alpha,
                     double homophily) {
  memset(g, 0, sizeof(*g));
  g->seed = seed;
  g->n = n;
  g->classes = classes;
  g->alpha = alpha;
  g->homophily = homophily;
  g->bits = 2;
  while ((1ll << g->bits) < n) g->bits += 2;
  g->q = n / classes;
  g->r = n % classes;
  /* powerlaw_rank: hi = pow(size + 1, 1 - alpha) depends on the size only */
  const double a1 = 1.0 - alpha;
  for (int b = 0; b < 2; ++b) g->him1[b] = det_pow((double)(g->q + b) + 1.0, a1) - 1.0;
  g->inv_a1 = 1.0 / a1;
}

typedef struct {
  GraphGen* g;
  int32_t* perm;
} PermCtx;

static void perm_fill(int64_t lo, int64_t hi, void* p) {
  PermCtx* c = (PermCtx*)p;
  for (int64_t i = lo; i < hi; ++i) c->perm[i] = (int32_t)feistel(i, c->g);
}

#define EB 512 /* edge batch */

/* endpoints (node ids) of undirected edges e0 .. e0+m-1 (gen_edge) */
static void gen_edges(const GraphGen* g, int64_t e0, int m, int64_t* restrict a,
                      int64_t* restrict b) {
  double uu[EB], uv[EB], hu[EB], hv[EB];
  int64_t su[EB], sv[EB], stu[EB], stv[EB];
  const int64_t q = g->q, r = g->r, C = g->classes;
  for (int t = 0; t < m; ++t) {
    const uint64_t h0 = splitmix64(g->seed ^ splitmix64((uint64_t)(e0 + t) * 4 + 1));
    const uint64_t h1 = splitmix64(h0 + 0x51ED27ull);
    const uint64_t h2 = splitmix64(h1 + 0xA11CEull);
    const uint64_t h3 = splitmix64(h2 + 0xB0Bull);
    const double d0 = ((double)(int64_t)(h0 >> 11) + 0.5) * 0x1p-53;
    const double d1 = ((double)(int64_t)(h1 >> 11) + 0.5) * 0x1p-53;
    const double d2 = ((double)(int64_t)(h2 >> 11) + 0.5) * 0x1p-53;
    const double d3 = ((double)(int64_t)(h3 >> 11) + 0.5) * 0x1p-53;
    const double d3x = ((double)(int64_t)((h3 ^ 0x5A5Aull) >> 11) + 0.5) * 0x1p-53;
    const int64_t cu = (int64_t)(d0 * (double)C);
    const int64_t cw = (int64_t)(d3x * (double)C);
    const int64_t cv = d2 < g->homophily ? cu : cw;
    su[t] = cu < r;  /* size = q + (c < r) */
    sv[t] = cv < r;
    stu[t] = cu * q + (cu < r ? cu : r);
    stv[t] = cv * q + (cv < r ? cv : r);
    uu[t] = d1;
    uv[t] = d3;
  }
  for (int t = 0; t < m; ++t) {
    hu[t] = su[t] ? g->him1[1] : g->him1[0];
    hv[t] = sv[t] ? g->him1[1] : g->him1[0];
  }
  double xu[EB], xv[EB];
  const double inv_a1 = g->inv_a1;
  for (int t = 0; t < m; ++t) xu[t] = det_pow(fma(uu[t], hu[t], 1.0), inv_a1);
  for (int t = 0; t < m; ++t) xv[t] = det_pow(fma(uv[t], hv[t], 1.0), inv_a1);
  for (int t = 0; t < m; ++t) {
    const int64_t szu = q + su[t], szv = q + sv[t];
    int64_t ru = (int64_t)xu[t] - 1, rv = (int64_t)xv[t] - 1;
    ru = ru < 0 ? 0 : (ru >= szu ? szu - 1 : ru);
    rv = rv < 0 ? 0 : (rv >= szv ? szv - 1 : rv);
    a[t] = g->perm[stu[t] + ru];
    b[t] = g->perm[stv[t] + rv];
  }
}

typedef struct {
  const GraphGen* g;
  uint32_t* degrees;
  int64_t* off;
  int64_t* cur;
  int32_t* col;
} GraphCtx;

static void edge_degrees(int64_t lo, int64_t hi, void* p) {
  const GraphCtx* c = (const GraphCtx*)p;
  int64_t a[EB], b[EB];
  for (int64_t e = lo; e < hi; e += EB) {
    const int m = (int)(hi - e < EB ? hi - e : EB);
    gen_edges(c->g, e, m, a, b);
    for (int t = 0; t < m; ++t) {
      if (a[t] == b[t]) continue;
      __atomic_fetch_add(c->degrees + a[t], 1u, __ATOMIC_RELAXED);
      __atomic_fetch_add(c->degrees + b[t], 1u, __ATOMIC_RELAXED);
    }
  }
}

static void edge_emit(int64_t lo, int64_t hi, void* p) {
  const GraphCtx* c = (const GraphCtx*)p;
  int64_t a[EB], b[EB];
  for (int64_t e = lo; e < hi; e += EB) {
    const int m = (int)(hi - e < EB ? hi - e : EB);
    gen_edges(c->g, e, m, a, b);
    for (int t = 0; t < m; ++t) {
      if (a[t] == b[t]) continue;
      c->col[__atomic_fetch_add(c->cur + a[t], 1, __ATOMIC_RELAXED)] = (int32_t)b[t];
      c->col[__atomic_fetch_add(c->cur + b[t], 1, __ATOMIC_RELAXED)] = (int32_t)a[t];
    }
  }
}

static void rows_init(int64_t lo, int64_t hi, void* p) {
  const GraphCtx* c = (const GraphCtx*)p;
  for (int64_t i = lo; i < hi; ++i) {
    c->col[c->off[i]] = (int32_t)i; /* self loop */
    c->cur[i] = c->off[i] + 1;
  }
}

static void insertion_i32(int32_t* v, int64_t m) {
  for (int64_t i = 1; i < m; ++i) {
    const int32_t x = v[i];
    int64_t j = i - 1;
    while (j >= 0 && v[j] > x) {
      v[j + 1] = v[j];
      --j;
    }
    v[j + 1] = x;
  }
}

/* in-place quicksort (median of three, insertion sort below 32, smaller
 * side first so the explicit stack stays O(log m)) */
static void sort_i32(int32_t* v, int64_t m) {
  int64_t stack[128];
  int sp = 0;
  int64_t lo = 0, hi = m - 1;
  for (;;) {
    while (hi - lo >= 32) {
      const int64_t mid = lo + (hi - lo) / 2;
      int32_t a = v[lo], b = v[mid], c = v[hi];
      const int32_t piv = a < b ? (b < c ? b : (a < c ? c : a)) : (a < c ? a : (b < c ? c : b));
      int64_t i = lo, j = hi;
      while (i <= j) {
        while (v[i] < piv) ++i;
        while (v[j] > piv) --j;
        if (i <= j) {
          const int32_t t = v[i];
          v[i] = v[j];
          v[j] = t;
          ++i;
          --j;
        }
      }
      if (j - lo < hi - i) {
        stack[sp++] = i;
        stack[sp++] = hi;
        hi = j;
      } else {
        stack[sp++] = lo;
        stack[sp++] = j;
        lo = i;
      }
    }
    insertion_i32(v + lo, hi - lo + 1);
    if (!sp) break;
    hi = stack[--sp];
    lo = stack[--sp];
  }
}

static void rows_sort_dedup(int64_t lo, int64_t hi, void* p) {
  const GraphCtx* c = (const GraphCtx*)p;
  for (int64_t i = lo; i < hi; ++i) {
    int32_t* r = c->col + c->off[i];
    const int64_t m = c->off[i + 1] - c->off[i];
    sort_i32(r, m);
    int64_t u = 0;
    for (int64_t t = 0; t < m; ++t)
      if (t == 0 || r[t] != r[t - 1]) r[u++] = r[t];
    c->cur[i] = u;
  }
}

/* The graph generator's state: the Feistel table is built here, once. */
void* fgo_graph_open(uint64_t seed, int64_t n, int64_t classes, double alpha,
                     double homophily) {
  if (n < 2 || classes < 1 || n >= (1ll << 31)) return NULL;
  GraphGen* g = (GraphGen*)malloc(sizeof(GraphGen));
  int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  if (!g || !perm) {
    free(g);
    free(perm);
    return NULL;
  }
  make_gen(g, seed, n, classes, alpha, homophily);
  PermCtx pc = {g, perm};
  par_for(n, 1 << 16, perm_fill, &pc);
  g->perm = perm;
  return g;
}

void fgo_graph_close(void* h) {
  GraphGen* g = (GraphGen*)h;
  if (!g) return;
  free((void*)g->perm);
  free(g);
}

/* degrees[n] = endpoint counts of the non-self edges (duplicates included),
 * fg_graph_degrees; returns sum(degrees) + n (raw entries incl. self loops) */
int64_t fgo_graph_degrees(void* h, int64_t num_edges, uint32_t* degrees) {
  GraphGen* g = (GraphGen*)h;
  memset(degrees, 0, sizeof(uint32_t) * (size_t)g->n);
  GraphCtx c = {g, degrees, NULL, NULL, NULL};
  par_for(num_edges, 1 << 15, edge_degrees, &c);
  int64_t total = g->n;
  for (int64_t i = 0; i < g->n; ++i) total += degrees[i];
  return total;
}

/* The symmetric, self-looped, sorted, duplicate-free CSR (synth.
 * generate_graph); col has room for the raw entry count fgo_graph_degrees
 * returned.  Writes off[n+1] and col[0 .. nnz), returns nnz. */
int64_t fgo_graph_build(void* h, int64_t num_edges, const uint32_t* degrees, int64_t* off,
                        int32_t* col) {
  GraphGen* g = (GraphGen*)h;
  const int64_t n = g->n;
  off[0] = 0;
  for (int64_t i = 0; i < n; ++i) off[i + 1] = off[i] + (int64_t)degrees[i] + 1;
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  if (!cur) return -1;
  GraphCtx c = {g, (uint32_t*)degrees, off, cur, col};
  const int verbose = getenv("FGO_VERBOSE") != NULL;
  double t0 = now_s();
  par_for(n, 1 << 16, rows_init, &c);
  par_for(num_edges, 1 << 15, edge_emit, &c);
  double t1 = now_s();
  par_for(n, 4096, rows_sort_dedup, &c); /* unique count into cur[i] */
  double t2 = now_s();
  /* compact: rows move left only, so a sequential pass is safe */
  int64_t pos = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t src = off[i];
    off[i] = pos;
    if (src != pos) memmove(col + pos, col + src, sizeof(int32_t) * (size_t)cur[i]);
    pos += cur[i];
  }
  off[n] = pos;
  free(cur);
  if (verbose)
    fprintf(stderr, "[fgoracle] emit %.2f s, sort+dedup %.2f s, compact %.2f s\n", t1 - t0,
            t2 - t1, now_s() - t2);
  return pos;
}

/* fg_graph_labels: planted class of each node (class of position p ->
 * node perm[p]) */
typedef struct {
  const GraphGen* g;
  int32_t* labels;
} LabelCtx;

static void node_labels(int64_t lo, int64_t hi, void* p) {
  const LabelCtx* c = (const LabelCtx*)p;
  const int64_t q = c->g->q, r = c->g->r;
  const int64_t big = r * (q + 1);
  for (int64_t pos = lo; pos < hi; ++pos) {
    const int64_t cl = pos < big ? pos / (q + 1) : r + (pos - big) / q;
    c->labels[c->g->perm[pos]] = (int32_t)cl;
  }
}

int fgo_graph_labels(void* h, int32_t* labels) {
  LabelCtx c = {(GraphGen*)h, labels};
  par_for(((GraphGen*)h)->n, 1 << 16, node_labels, &c);
  return 0;
}

int fgo_num_threads(void) { return fgo_threads(); }
