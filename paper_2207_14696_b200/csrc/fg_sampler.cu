// GPU neighbour sampler that reproduces the reference sampler draw for draw.
//
// Reference: pkg/src/featgrind/pipeline.py:185-222 (sample_batches).  Within
// a batch the reference walks layers, and within a layer the sorted node list,
// calling numpy Generator.choice(nbrs, f, replace=False) on ONE serial PCG64
// stream.  For deg > f, choice consumes exactly 2f-1 32-bit draws (Floyd: f
// Lemire draws on [0, j], then f-1 tail-shuffle draws) unless a Lemire draw is
// rejected (probability (2^32 mod (j+1)) / 2^32).  So node i's first draw sits
// at stream offset sum_{i'<i} draws(i'), a prefix sum; each thread jumps its
// own PCG64 cursor there (128-bit LCG jump table) and runs Floyd serially.
// A node whose Lemire draw was rejected consumed extra draws: every later node
// of the layer is then redone with the corrected offset by a cooperative
// fix-up kernel (rare: ~f*deg/2^32 per node).  Deterministic, no float math.
//
// np.unique over node ids (< n) is done with a bitmap: mark, popcount
// prefix, ordered emit (ascending ids), rank lookup, clear.
#include <cooperative_groups.h>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "fg_common.cuh"
#include "fg_pcg64.cuh"

namespace cg = cooperative_groups;

namespace fg {

constexpr int kSampThreads = 256;
constexpr int kLocalF = 32;           // fanouts up to this use a local index buffer
constexpr int64_t kNoBad = INT64_MAX;

struct LayerWs {
  int64_t* block_sums;  // [2 * nb] (picks, draws) per block
  int64_t* block_offs;  // [2 * nb]
  int64_t* draw_off;    // [N] nominal stream offset per node
  uint32_t* used;       // [N] draws actually consumed
  int64_t* scal;        // [8]: 0 total picks, 1 total draws, 2 bad slot 0, 3 bad slot 1, 4 delta
};

inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

inline LayerWs carve(void* ws, int64_t N) {
  const int64_t nb = ceil_div(N > 0 ? N : 1, kSampThreads);
  char* p = (char*)ws;
  LayerWs w;
  w.block_sums = (int64_t*)p; p += align256(2 * nb * 8);
  w.block_offs = (int64_t*)p; p += align256(2 * nb * 8);
  w.draw_off = (int64_t*)p; p += align256(N * 8);
  w.used = (uint32_t*)p; p += align256(N * 4);
  w.scal = (int64_t*)p; p += align256(8 * 8);
  return w;
}

inline int64_t layer_ws_bytes(int64_t N) {
  const int64_t nb = ceil_div(N > 0 ? N : 1, kSampThreads);
  return 2 * align256(2 * nb * 8) + align256(N * 8) + align256(N * 4) + align256(64);
}

__device__ __forceinline__ void node_counts(const int64_t* __restrict__ off,
                                            const int32_t* __restrict__ nodes, int64_t i,
                                            int64_t live, int f, int64_t& deg, int64_t& cnt,
                                            int64_t& draws) {
  deg = cnt = draws = 0;
  if (i < live) {
    const int32_t u = nodes[i];
    deg = off[u + 1] - off[u];
    cnt = deg < f ? deg : f;
    draws = deg > f ? 2 * (int64_t)f - 1 : 0;
  }
}

// Floyd + tail shuffle for one node (numpy Generator.choice, replace=False,
// the pop <= 10000 or f <= pop // 50 branch).  Returns draws consumed.
__device__ uint32_t sample_node(const int64_t* __restrict__ off, const int32_t* __restrict__ col,
                                int32_t u, int f, const uint64_t* __restrict__ rng, uint64_t q,
                                int32_t* __restrict__ out, uint32_t* __restrict__ bitmap) {
  const int64_t b = off[u];
  const int64_t deg = off[u + 1] - b;
  if (deg <= f) {
    for (int64_t t = 0; t < deg; ++t) {
      const int32_t v = col[b + t];
      out[t] = v;
      if (bitmap) atomicOr(bitmap + (v >> 5), 1u << (v & 31));
    }
    return 0;
  }
  PcgCursor c = rng_cursor_at(rng, q);
  uint32_t used = 0;
  uint32_t local[kLocalF];
  uint32_t* idx = f <= kLocalF ? local : reinterpret_cast<uint32_t*>(out);
  for (int t = 0; t < f; ++t) {
    const uint32_t j = (uint32_t)(deg - f + t);
    uint32_t v = c.lemire(j, used);
    for (int s = 0; s < t; ++s)
      if (idx[s] == v) { v = j; break; }
    idx[t] = v;
  }
  for (int i = f - 1; i >= 1; --i) {
    const uint32_t j = c.lemire((uint32_t)i, used);
    const uint32_t tmp = idx[i];
    idx[i] = idx[j];
    idx[j] = tmp;
  }
  for (int t = 0; t < f; ++t) {
    const int32_t v = col[b + idx[t]];
    out[t] = v;
    if (bitmap) atomicOr(bitmap + (v >> 5), 1u << (v & 31));
  }
  return used;
}

__global__ void __launch_bounds__(kSampThreads)
k_layer_count(const int64_t* __restrict__ off, const int32_t* __restrict__ nodes,
              const int64_t* __restrict__ nlive, int64_t N, int f, LayerWs ws,
              int32_t* err_flag) {
  using BR = cub::BlockReduce<int64_t, kSampThreads>;
  __shared__ typename BR::TempStorage tmp;
  const int64_t i = blockIdx.x * (int64_t)kSampThreads + threadIdx.x;
  const int64_t live = min64(*nlive, N);
  int64_t deg, cnt, draws;
  node_counts(off, nodes, i, live, f, deg, cnt, draws);
  if (deg > 10000 && f > deg / 50) atomicExch(err_flag, FG_EUSAGE);  // numpy's FY branch
  const int64_t sp = BR(tmp).Sum(cnt);
  __syncthreads();
  const int64_t sd = BR(tmp).Sum(draws);
  if (threadIdx.x == 0) {
    ws.block_sums[2 * blockIdx.x] = sp;
    ws.block_sums[2 * blockIdx.x + 1] = sd;
  }
}

// single block: exclusive scan of per-block (picks, draws)
__global__ void __launch_bounds__(1024)
k_layer_scan(int64_t nb, LayerWs ws, int64_t* __restrict__ num_picks, int64_t max_picks,
             int32_t* err_flag) {
  using BS = cub::BlockScan<int64_t, 1024>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int64_t carry[2];
  if (threadIdx.x == 0) carry[0] = carry[1] = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t i = base + threadIdx.x;
    for (int k = 0; k < 2; ++k) {
      const int64_t v = i < nb ? ws.block_sums[2 * i + k] : 0;
      int64_t ex, agg;
      BS(tmp).ExclusiveSum(v, ex, agg);
      __syncthreads();
      if (i < nb) ws.block_offs[2 * i + k] = ex + carry[k];
      __syncthreads();
      if (threadIdx.x == 0) carry[k] += agg;
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    ws.scal[0] = carry[0];
    ws.scal[1] = carry[1];
    ws.scal[2] = kNoBad;
    ws.scal[3] = kNoBad;
    ws.scal[4] = 0;
    *num_picks = carry[0];
    if (carry[0] > max_picks) atomicExch(err_flag, FG_EUSAGE);
  }
}

__global__ void __launch_bounds__(kSampThreads)
k_layer_sample(const int64_t* __restrict__ off, const int32_t* __restrict__ col,
               const int32_t* __restrict__ nodes, const int64_t* __restrict__ nlive, int64_t N,
               int f, const uint64_t* __restrict__ rng, LayerWs ws, int32_t* __restrict__ indptr,
               int32_t* __restrict__ picks, int64_t max_picks, uint32_t* __restrict__ bitmap) {
  using BS = cub::BlockScan<int64_t, kSampThreads>;
  __shared__ typename BS::TempStorage tmp;
  const int64_t i = blockIdx.x * (int64_t)kSampThreads + threadIdx.x;
  const int64_t live = min64(*nlive, N);
  int64_t deg, cnt, draws;
  node_counts(off, nodes, i, live, f, deg, cnt, draws);
  int64_t pick_off, draw_off;
  BS(tmp).ExclusiveSum(cnt, pick_off);
  __syncthreads();
  BS(tmp).ExclusiveSum(draws, draw_off);
  pick_off += ws.block_offs[2 * blockIdx.x];
  draw_off += ws.block_offs[2 * blockIdx.x + 1];
  if (i < N) indptr[i] = (int32_t)pick_off;
  if (i == N - 1) indptr[N] = (int32_t)(pick_off + cnt);
  if (i >= live || pick_off + cnt > max_picks) return;
  ws.draw_off[i] = draw_off;
  const uint32_t used = sample_node(off, col, nodes[i], f, rng, (uint64_t)draw_off,
                                    picks + pick_off, bitmap);
  ws.used[i] = used;
  if ((int64_t)used != draws) atomicMin((long long*)&ws.scal[2], (long long)i);
}

// Cooperative fix-up + stream advance.  Every block reads the first rejecting
// node; in the common case there is none and only the stream advance runs.
__global__ void __launch_bounds__(kSampThreads)
k_layer_fixup(const int64_t* __restrict__ off, const int32_t* __restrict__ col,
              const int32_t* __restrict__ nodes, const int64_t* __restrict__ nlive, int64_t N,
              int f, uint64_t* __restrict__ rng, LayerWs ws, const int32_t* __restrict__ indptr,
              int32_t* __restrict__ picks, uint32_t* __restrict__ bitmap, int64_t n_nodes_graph) {
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
  volatile int64_t* scal = ws.scal;
  int64_t cur = scal[2];
  int64_t delta = 0;
  if (cur != kNoBad) {
    cg::grid_group grid = cg::this_grid();
    const int64_t live = min64(*nlive, N);
    int rd = 2;
    while (cur != kNoBad) {
      const int64_t nominal = 2 * (int64_t)f - 1;
      delta += (int64_t)ws.used[cur] - nominal;
      const int wr = rd == 2 ? 3 : 2;
      for (int64_t i = cur + 1 + gtid; i < live; i += gsize) {
        const int32_t u = nodes[i];
        const int64_t deg = off[u + 1] - off[u];
        if (deg <= f) continue;  // no draws: picks unaffected by the stream
        const uint32_t used = sample_node(off, col, u, f, rng, (uint64_t)(ws.draw_off[i] + delta),
                                          picks + indptr[i], nullptr);
        ws.used[i] = used;
        if ((int64_t)used != nominal) atomicMin((long long*)&ws.scal[wr], (long long)i);
      }
      grid.sync();
      cur = scal[wr];
      grid.sync();
      if (gtid == 0) scal[rd] = kNoBad;
      grid.sync();
      rd = wr;
    }
    // picks changed after the first rejection: rebuild this layer's marks
    if (bitmap) {
      const int64_t words = (n_nodes_graph + 31) >> 5;
      for (int64_t w = gtid; w < words; w += gsize) bitmap[w] = 0;
      grid.sync();
      const int64_t total = scal[0];
      for (int64_t e = gtid; e < total; e += gsize) {
        const int32_t v = picks[e];
        atomicOr(bitmap + (v >> 5), 1u << (v & 31));
      }
    }
    if (gtid == 0) scal[4] = delta;
  }
  if (gtid == 0) {
    const uint64_t T = (uint64_t)(scal[1] + delta);
    PcgCursor c = rng_cursor_at(rng, T);
    rng[RNG_STATE] = c.s.lo;
    rng[RNG_STATE + 1] = c.s.hi;
    rng[RNG_HAS32] = c.have ? 1 : 0;
    rng[RNG_BUF] = c.hi;
    rng[RNG_LAST] = T;
  }
}

// ------------------------------------------------------------- bitmap
constexpr int kBmThreads = 256;
constexpr int kBmWords = 8;  // words per thread
constexpr int64_t kBmPerBlock = (int64_t)kBmThreads * kBmWords;

__global__ void k_mark32(const int32_t* __restrict__ ids, const int64_t* __restrict__ cnt,
                         int64_t max_count, uint32_t* __restrict__ bm) {
  const int64_t live = min64(*cnt, max_count);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < live;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = ids[i];
    atomicOr(bm + (v >> 5), 1u << (v & 31));
  }
}
__global__ void k_mark64(const int64_t* __restrict__ ids, const int64_t* __restrict__ cnt,
                         int64_t max_count, uint32_t* __restrict__ bm) {
  const int64_t live = min64(*cnt, max_count);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < live;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = ids[i];
    atomicOr(bm + (v >> 5), 1u << (v & 31));
  }
}

__global__ void __launch_bounds__(kBmThreads)
k_bm_count(const uint32_t* __restrict__ bm, int64_t words, int64_t* __restrict__ bsum) {
  using BR = cub::BlockReduce<int64_t, kBmThreads>;
  __shared__ typename BR::TempStorage tmp;
  const int64_t w0 = blockIdx.x * kBmPerBlock + threadIdx.x * (int64_t)kBmWords;
  int64_t c = 0;
#pragma unroll
  for (int k = 0; k < kBmWords; ++k)
    if (w0 + k < words) c += __popc(bm[w0 + k]);
  const int64_t s = BR(tmp).Sum(c);
  if (threadIdx.x == 0) bsum[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024)
k_bm_scan(int64_t nb, const int64_t* __restrict__ bsum, int64_t* __restrict__ boff,
          int64_t* __restrict__ out_count) {
  using BS = cub::BlockScan<int64_t, 1024>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < nb ? bsum[i] : 0;
    int64_t ex, agg;
    BS(tmp).ExclusiveSum(v, ex, agg);
    if (i < nb) boff[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) *out_count = carry;
}

__global__ void __launch_bounds__(kBmThreads)
k_bm_emit(const uint32_t* __restrict__ bm, int64_t words, const int64_t* __restrict__ boff,
          int32_t* __restrict__ out, int64_t max_out, int32_t* __restrict__ wprefix) {
  using BS = cub::BlockScan<int64_t, kBmThreads>;
  __shared__ typename BS::TempStorage tmp;
  const int64_t w0 = blockIdx.x * kBmPerBlock + threadIdx.x * (int64_t)kBmWords;
  uint32_t wv[kBmWords];
  int64_t c = 0;
#pragma unroll
  for (int k = 0; k < kBmWords; ++k) {
    wv[k] = (w0 + k < words) ? bm[w0 + k] : 0u;
    c += __popc(wv[k]);
  }
  int64_t pos;
  BS(tmp).ExclusiveSum(c, pos);
  pos += boff[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kBmWords; ++k) {
    if (w0 + k >= words) break;
    if (wprefix) wprefix[w0 + k] = (int32_t)pos;
    uint32_t x = wv[k];
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      if (pos < max_out) out[pos] = (int32_t)(((w0 + k) << 5) + b);
      ++pos;
    }
  }
}

__global__ void k_bm_rank(const int32_t* __restrict__ ids, const int64_t* __restrict__ cnt,
                          int64_t max_count, const uint32_t* __restrict__ bm,
                          const int32_t* __restrict__ wprefix, int32_t* __restrict__ rank) {
  const int64_t live = min64(*cnt, max_count);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < live;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = ids[i];
    const uint32_t w = bm[v >> 5];
    rank[i] = wprefix[v >> 5] + __popc(w & ((1u << (v & 31)) - 1u));
  }
}

__global__ void k_bm_clear(const int32_t* __restrict__ ids, const int64_t* __restrict__ cnt,
                           int64_t max_count, uint32_t* __restrict__ bm) {
  const int64_t live = min64(*cnt, max_count);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < live;
       i += (int64_t)gridDim.x * blockDim.x)
    bm[ids[i] >> 5] = 0u;
}

}  // namespace fg

using namespace fg;

extern "C" {

int64_t fg_sample_workspace_bytes(int64_t max_nodes) { return layer_ws_bytes(max_nodes); }

int fg_sample_layer(const int64_t* row_offsets, const int32_t* col_indices, int64_t n,
                    const int32_t* nodes, const int64_t* num_nodes_dev, int64_t max_nodes,
                    int fanout, uint64_t* rng_dev, int32_t* indptr, int32_t* picks,
                    int64_t max_picks, int64_t* num_picks_dev, uint32_t* bitmap, void* ws,
                    int64_t ws_bytes, int32_t* err_flag, void* s) {
  FG_CHECK_ARG(fanout >= 1, "fanouts must be >= 1");
  FG_CHECK_ARG(fanout <= 200,
               "fanout %d > 200 can reach numpy's partial Fisher-Yates choice branch "
               "(deg > 10000 and f > deg // 50), which this sampler does not emulate",
               fanout);
  FG_CHECK_ARG(max_nodes >= 1 && n >= 1, "fg_sample_layer: empty layer capacity");
  FG_CHECK_ARG(ws_bytes >= layer_ws_bytes(max_nodes), "fg_sample_layer: workspace too small");
  FG_CHECK_ARG(max_picks < INT32_MAX, "fg_sample_layer: picks must fit int32 offsets");
  FG_CHECK_ARG(row_offsets && col_indices && nodes && num_nodes_dev && rng_dev && indptr &&
                   picks && num_picks_dev && err_flag,
               "fg_sample_layer: null argument");
  cudaStream_t st = as_stream(s);
  LayerWs w = carve(ws, max_nodes);
  const int64_t nb = ceil_div(max_nodes, kSampThreads);
  k_layer_count<<<(unsigned)nb, kSampThreads, 0, st>>>(row_offsets, nodes, num_nodes_dev,
                                                       max_nodes, fanout, w, err_flag);
  FG_LAUNCH_CHECK();
  k_layer_scan<<<1, 1024, 0, st>>>(nb, w, num_picks_dev, max_picks, err_flag);
  FG_LAUNCH_CHECK();
  k_layer_sample<<<(unsigned)nb, kSampThreads, 0, st>>>(row_offsets, col_indices, nodes,
                                                        num_nodes_dev, max_nodes, fanout, rng_dev,
                                                        w, indptr, picks, max_picks, bitmap);
  FG_LAUNCH_CHECK();
  // cooperative fix-up: grid sized to be co-resident
  static thread_local int coop_blocks = 0;
  if (coop_blocks == 0) {
    int per_sm = 0;
    FG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_layer_fixup,
                                                              kSampThreads, 0));
    coop_blocks = sm_count() * (per_sm < 2 ? (per_sm < 1 ? 1 : per_sm) : 2);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(coop_blocks);
  cfg.blockDim = dim3(kSampThreads);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  FG_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_layer_fixup, row_offsets, col_indices, nodes,
                                 num_nodes_dev, max_nodes, fanout, rng_dev, w,
                                 (const int32_t*)indptr, picks, bitmap, n));
  count_launch();
  return FG_OK;
}

int64_t fg_bitmap_workspace_bytes(int64_t n) {
  const int64_t words = (n + 31) / 32;
  const int64_t nb = ceil_div(words > 0 ? words : 1, kBmPerBlock);
  return 2 * align256(nb * 8);
}

int fg_bitmap_mark(const int32_t* ids, const int64_t* cnt, int64_t max_count, uint32_t* bm,
                   void* s) {
  if (max_count == 0) return FG_OK;
  k_mark32<<<grid_for(max_count, 256), 256, 0, as_stream(s)>>>(ids, cnt, max_count, bm);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_bitmap_mark64(const int64_t* ids, const int64_t* cnt, int64_t max_count, uint32_t* bm,
                     void* s) {
  if (max_count == 0) return FG_OK;
  k_mark64<<<grid_for(max_count, 256), 256, 0, as_stream(s)>>>(ids, cnt, max_count, bm);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_bitmap_compact(uint32_t* bm, int64_t n, int32_t* out_ids, int64_t max_out,
                      int64_t* out_count, int32_t* wprefix, void* ws, int64_t ws_bytes, void* s) {
  FG_CHECK_ARG(n >= 1 && n < INT32_MAX, "fg_bitmap_compact: n must be in [1, 2^31)");
  FG_CHECK_ARG(ws_bytes >= fg_bitmap_workspace_bytes(n), "fg_bitmap_compact: workspace too small");
  cudaStream_t st = as_stream(s);
  const int64_t words = (n + 31) / 32;
  const int64_t nb = ceil_div(words, kBmPerBlock);
  int64_t* bsum = (int64_t*)ws;
  int64_t* boff = (int64_t*)((char*)ws + align256(nb * 8));
  k_bm_count<<<(unsigned)nb, kBmThreads, 0, st>>>(bm, words, bsum);
  FG_LAUNCH_CHECK();
  k_bm_scan<<<1, 1024, 0, st>>>(nb, bsum, boff, out_count);
  FG_LAUNCH_CHECK();
  k_bm_emit<<<(unsigned)nb, kBmThreads, 0, st>>>(bm, words, boff, out_ids, max_out, wprefix);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_bitmap_rank(const int32_t* ids, const int64_t* cnt, int64_t max_count, const uint32_t* bm,
                   const int32_t* wprefix, int32_t* rank, void* s) {
  if (max_count == 0) return FG_OK;
  k_bm_rank<<<grid_for(max_count, 256), 256, 0, as_stream(s)>>>(ids, cnt, max_count, bm, wprefix,
                                                                rank);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_bitmap_clear(const int32_t* ids, const int64_t* cnt, int64_t max_count, uint32_t* bm,
                    void* s) {
  if (max_count == 0) return FG_OK;
  k_bm_clear<<<grid_for(max_count, 256), 256, 0, as_stream(s)>>>(ids, cnt, max_count, bm);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

}  // extern "C"
