// Deterministic, row-addressable synthetic feature generation on the device
// (SURVEY.md §8d): element (i, j) is a pure function of (seed, i, j), so the
// oracle can regenerate any row subset and configs whose raw matrix cannot be
// held (MAG240M-shape, 750 GB fp32) are produced chunk by chunk and
// compressed on the fly.  Distributions follow the reference's
// generate_features kinds (pkg/src/featgrind/graphstore.py:291-324), plus a
// class-conditional kind with planted labels for the trainer.
#include "fg_common.cuh"
#include "fg_detmath.cuh"

namespace fg {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Box-Muller from two 24-bit uniforms of one 64-bit hash, in float64 with the
// deterministic elementary functions (fg_detmath.cuh), rounded once to float:
// the same bits as the C restatement (oracle/fgoracle.c).
__device__ __forceinline__ float gauss(uint64_t key) {
  const uint64_t h = splitmix64(key);
  const double u1 = (double)((uint32_t)(h >> 40) + 1u) * 0x1p-24;  // (0, 1]
  const double u2 = (double)(uint32_t)(h & 0xFFFFFFu) * 0x1p-24;   // [0, 1)
  const double ln_u1 = det::mul(det::log2(u1), 0x1.62e42fefa39efp-1);
  return __double2float_rn(det::mul(__dsqrt_rn(det::mul(-2.0, ln_u1)), det::cos_turns(u2)));
}

__device__ __forceinline__ uint64_t elem_key(uint64_t seed, int64_t i, int64_t j) {
  return splitmix64(seed ^ splitmix64((uint64_t)i * 0x100000001B3ull + (uint64_t)j));
}

__global__ void k_synth(int kind, uint64_t seed, int64_t row0, const int64_t* __restrict__ row_ids,
                        int64_t rows, int64_t d, const int32_t* __restrict__ labels,
                        int num_classes, float* __restrict__ out) {
  const int64_t total = rows * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / d, j = t - r * d;
    const int64_t i = row_ids ? row_ids[r] : row0 + r;
    const float z = gauss(elem_key(seed, i, j));
    float v;
    switch (kind) {
      case 0:  // normal
        v = z;
        break;
      case 1: {  // lognormal magnitude, random sign
        const uint64_t sgn = splitmix64(elem_key(seed ^ 0x5151ull, i, j));
        const float mag = __double2float_rn(det::exp2(det::mul((double)z, 0x1.71547652b82fep+0)));
        v = (sgn & 1) ? mag : -mag;
        break;
      }
      case 2: {  // correlated: shared direction + per-row noise (weight 0.9)
        const float s = gauss(elem_key(seed ^ 0xC0FFEEull, -1, j));
        v = __fadd_rn(__fmul_rn(0.9486833f, s), __fmul_rn(0.31622777f, z));
        break;
      }
      default: {  // class-conditional: mean direction of the planted label
        const int c = labels ? labels[i] : 0;
        const float m = gauss(elem_key(seed ^ 0xC1A55ull, c, j));
        v = __fadd_rn(__fmul_rn(0.6f, m), __fmul_rn(0.8f, z));
        break;
      }
    }
    out[t] = v;
  }
}

}  // namespace fg

using namespace fg;

extern "C" int fg_synth_features(int kind, uint64_t seed, int64_t row0, int64_t rows, int64_t d,
                                 const int32_t* labels, int num_classes, float* out, void* s) {
  FG_CHECK_ARG(kind >= 0 && kind <= 3, "fg_synth_features: kind must be 0..3");
  FG_CHECK_ARG(kind != 3 || labels != nullptr, "class-conditional kind needs labels");
  FG_CHECK_ARG(rows >= 0 && d >= 1, "fg_synth_features: bad shape");
  if (rows == 0) return FG_OK;
  k_synth<<<grid_for(rows * d, 256), 256, 0, as_stream(s)>>>(kind, seed, row0, nullptr, rows, d,
                                                             labels, num_classes, out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_synth_feature_rows(int kind, uint64_t seed, const int64_t* row_ids,
                                     int64_t rows, int64_t d, const int32_t* labels,
                                     int num_classes, float* out, void* s) {
  FG_CHECK_ARG(kind >= 0 && kind <= 3, "fg_synth_feature_rows: kind must be 0..3");
  FG_CHECK_ARG(kind != 3 || labels != nullptr, "class-conditional kind needs labels");
  FG_CHECK_ARG(rows >= 0 && d >= 1 && (rows == 0 || row_ids), "fg_synth_feature_rows: bad shape");
  if (rows == 0) return FG_OK;
  k_synth<<<grid_for(rows * d, 256), 256, 0, as_stream(s)>>>(kind, seed, 0, row_ids, rows, d,
                                                             labels, num_classes, out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

// ---------------------------------------------------- synthetic graphs
// Degree-corrected planted partition at any scale: node
// positions are grouped by class (C equal blocks); position -> node id is a
// fixed Feistel bijection (hubs spread over the id space).  Edge e is a pure
// function of (seed, e): endpoint ranks follow a continuous power law
// w(rank) ~ (rank+1)^-alpha inside a class (closed-form inverse CDF); the
// second endpoint stays in the first's class with probability `homophily`.
// The CSR is built in node-range chunks: every chunk regenerates all edges
// and keeps the directed entries whose source falls in the chunk, so memory
// is bounded by the chunk, not the graph.
namespace fg {

struct GraphGen {
  uint64_t seed;
  int64_t n;
  int64_t classes;
  double alpha;
  double homophily;
  int bits;  // Feistel domain bits (even)
};

__device__ __forceinline__ double u01(uint64_t h) {
  return det::mul(det::add((double)(h >> 11), 0.5), 0x1p-53);  // (0, 1)
}

__device__ __forceinline__ int64_t feistel(int64_t x, const GraphGen& g) {
  const int half = g.bits / 2;
  const uint64_t mask = (1ull << half) - 1;
  uint64_t y = (uint64_t)x;
  for (int walk = 0; walk < 512; ++walk) {
    uint64_t lo = y & mask, hi = y >> half;
    for (int r = 0; r < 4; ++r) {
      const uint64_t f = splitmix64(lo ^ (g.seed * 0x9E3779B97F4A7C15ull + r)) & mask;
      const uint64_t t = hi ^ f;
      hi = lo;
      lo = t;
    }
    y = (hi << half) | lo;
    if ((int64_t)y < g.n) return (int64_t)y;
  }
  return x;  // unreachable in practice (domain <= 4n)
}

__device__ __forceinline__ int64_t class_size(const GraphGen& g, int64_t c) {
  return g.n / g.classes + (c < g.n % g.classes ? 1 : 0);
}
__device__ __forceinline__ int64_t class_start(const GraphGen& g, int64_t c) {
  const int64_t q = g.n / g.classes, r = g.n % g.classes;
  return c * q + (c < r ? c : r);
}

__device__ __forceinline__ int64_t powerlaw_rank(double u, int64_t size, double alpha) {
  // continuous inverse CDF of x^-alpha on [1, size+1)
  // (deterministic pow: the same bits as oracle/fgoracle.c)
  const double a1 = det::sub(1.0, alpha);
  const double hi = det::pow(det::add((double)size, 1.0), a1);
  const double x = det::pow(det::fma(u, det::sub(hi, 1.0), 1.0), det::div(1.0, a1));
  int64_t r = (int64_t)x - 1;
  return r < 0 ? 0 : (r >= size ? size - 1 : r);
}

// endpoints (node ids) of undirected edge e
__device__ __forceinline__ void gen_edge(const GraphGen& g, int64_t e, int64_t& a, int64_t& b) {
  const uint64_t h0 = splitmix64(g.seed ^ splitmix64((uint64_t)e * 4 + 1));
  const uint64_t h1 = splitmix64(h0 + 0x51ED27ull);
  const uint64_t h2 = splitmix64(h1 + 0xA11CEull);
  const uint64_t h3 = splitmix64(h2 + 0xB0Bull);
  const int64_t cu = (int64_t)det::mul(u01(h0), (double)g.classes);
  const int64_t su = class_size(g, cu);
  const int64_t pu = class_start(g, cu) + powerlaw_rank(u01(h1), su, g.alpha);
  const int64_t cv =
      u01(h2) < g.homophily ? cu : (int64_t)det::mul(u01(h3 ^ 0x5A5Aull), (double)g.classes);
  const int64_t sv = class_size(g, cv);
  const int64_t pv = class_start(g, cv) + powerlaw_rank(u01(h3), sv, g.alpha);
  a = feistel(pu, g);
  b = feistel(pv, g);
}

__global__ void k_edge_degree(GraphGen g, int64_t E, unsigned int* __restrict__ deg) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a, b;
    gen_edge(g, e, a, b);
    if (a == b) continue;
    atomicAdd(deg + a, 1u);
    atomicAdd(deg + b, 1u);
  }
}

__global__ void k_edge_emit(GraphGen g, int64_t E, int64_t lo, int64_t hi,
                            unsigned long long* __restrict__ cursor, int64_t cap,
                            int64_t* __restrict__ keys) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a, b;
    gen_edge(g, e, a, b);
    if (a == b) continue;
    if (a >= lo && a < hi) {
      const unsigned long long s = atomicAdd(cursor, 1ull);
      if ((int64_t)s < cap) keys[s] = (a - lo) * g.n + b;
    }
    if (b >= lo && b < hi) {
      const unsigned long long s = atomicAdd(cursor, 1ull);
      if ((int64_t)s < cap) keys[s] = (b - lo) * g.n + a;
    }
  }
}

__global__ void k_node_labels(GraphGen g, int32_t* __restrict__ labels) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < g.n;
       p += (int64_t)gridDim.x * blockDim.x) {
    // class of position p
    const int64_t q = g.n / g.classes, r = g.n % g.classes;
    const int64_t big = r * (q + 1);
    const int64_t c = p < big ? p / (q + 1) : r + (p - big) / q;
    labels[feistel(p, g)] = (int32_t)c;
  }
}

inline GraphGen make_gen(uint64_t seed, int64_t n, int64_t classes, double alpha,
                         double homophily) {
  GraphGen g{seed, n, classes, alpha, homophily, 2};
  while ((1ll << g.bits) < n) g.bits += 2;
  return g;
}

}  // namespace fg

extern "C" int fg_graph_degrees(uint64_t seed, int64_t n, int64_t classes, double alpha,
                                double homophily, int64_t num_edges, uint32_t* degrees,
                                void* s) {
  FG_CHECK_ARG(n >= 2 && classes >= 1 && alpha > 0 && alpha != 1.0, "fg_graph_degrees: bad args");
  const GraphGen g = make_gen(seed, n, classes, alpha, homophily);
  k_edge_degree<<<grid_for(num_edges, 256, 16), 256, 0, as_stream(s)>>>(g, num_edges, degrees);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_graph_emit(uint64_t seed, int64_t n, int64_t classes, double alpha,
                             double homophily, int64_t num_edges, int64_t lo, int64_t hi,
                             unsigned long long* cursor, int64_t cap, int64_t* keys, void* s) {
  FG_CHECK_ARG(lo >= 0 && hi <= n && lo < hi, "fg_graph_emit: bad node range");
  FG_CHECK_ARG((double)(hi - lo) * (double)n < 9.2e18, "fg_graph_emit: key overflow");
  const GraphGen g = make_gen(seed, n, classes, alpha, homophily);
  k_edge_emit<<<grid_for(num_edges, 256, 16), 256, 0, as_stream(s)>>>(g, num_edges, lo, hi,
                                                                      cursor, cap, keys);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_graph_labels(uint64_t seed, int64_t n, int64_t classes, int32_t* labels,
                               void* s) {
  const GraphGen g = make_gen(seed, n, classes, 0.5, 0.0);
  k_node_labels<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(g, labels);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

// ------------------------------------------------ CSR self-loop census
// Number of nodes whose (sorted) row holds the node itself: binary search per
// row.  load_graph's self-loop flag check (graphstore.py:421-425) without the
// nnz-sized row expansion.
namespace fg {
__global__ void k_csr_self_loops(const int64_t* __restrict__ off, const int32_t* __restrict__ col,
                                 int64_t n, unsigned long long* __restrict__ count) {
  unsigned long long mine = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = off[i], hi = off[i + 1];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (col[mid] < i) lo = mid + 1; else hi = mid;
    }
    mine += (lo < off[i + 1] && col[lo] == i) ? 1ull : 0ull;
  }
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(count, mine);
}
}  // namespace fg

extern "C" int fg_csr_self_loops(const int64_t* row_offsets, const int32_t* col_indices, int64_t n,
                                 unsigned long long* count, void* s) {
  FG_CHECK_ARG(n >= 0 && count != nullptr, "fg_csr_self_loops: bad args");
  FG_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(unsigned long long), as_stream(s)));
  if (n == 0) return FG_OK;
  k_csr_self_loops<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(row_offsets, col_indices, n, count);
  FG_LAUNCH_CHECK();
  return FG_OK;
}
