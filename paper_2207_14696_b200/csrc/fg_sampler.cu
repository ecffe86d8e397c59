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
// The prefix sum is single-pass (decoupled look-back, fg_scan.cuh) inside the
// sampling kernel itself.  A node whose Lemire draw was rejected consumed
// extra draws: every later node of the layer is then redone with the
// corrected offset by the CTA that finishes last (rare: ~f*deg/2^32 per
// node), which also advances the stream.  Deterministic, no float math.
//
// np.unique over node ids (< n) is done with a bitmap: mark, popcount
// prefix, ordered emit (ascending ids), rank lookup, clear.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/block/block_radix_sort.cuh>

#include <stdlib.h>

#include "fg_common.cuh"
#include "fg_pcg64.cuh"
#include "fg_scan.cuh"

namespace fg {

constexpr int kSampThreads = 256;
constexpr int kLocalF = 32;           // fanouts up to this use a local index buffer

// Layer workspace.  The head (counters + scalars + look-back status) is
// zeroed by one memset per layer.
struct LayerWs {
  unsigned int* ctr;    // [0] tile ticket, [1] prefix done, [2] sample done, [3] fix-up done
  int64_t* scal;        // [0] total picks, [1] total draws, [2] bad key, [3] delta,
                        // [4] bad key of the parallel fix-up pass
  unsigned long long* status;  // [nb] look-back status words
  int64_t* draw_off;    // [N] nominal stream offset per node
  uint32_t* used;       // [N] draws actually consumed
  int64_t head_bytes;   // bytes to zero per layer
};

inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

// look-back tiles of the prefix kernel (256 nodes each)
inline int64_t layer_tiles(int64_t N) { return ceil_div(N > 0 ? N : 1, kSampThreads); }

inline LayerWs carve(void* ws, int64_t N) {
  const int64_t nb = layer_tiles(N);
  char* p = (char*)ws;
  LayerWs w;
  w.ctr = (unsigned int*)p;
  w.scal = (int64_t*)(p + 64);
  w.status = (unsigned long long*)(p + 128);
  w.head_bytes = align256(128 + nb * 8);
  p += w.head_bytes;
  w.draw_off = (int64_t*)p; p += align256(N * 8);
  w.used = (uint32_t*)p;
  return w;
}

inline int64_t layer_ws_bytes(int64_t N) {
  const int64_t nb = layer_tiles(N);
  return align256(128 + nb * 8) + align256(N * 8) + align256(N * 4);
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

// packed per-node (picks, draws): draws in bits 30..61, picks in bits 0..29
constexpr int kPickBits = 30;
constexpr unsigned long long kPickMask = (1ull << kPickBits) - 1;

// Run by the CTA that finishes last: totals, rejection fix-up, stream
// advance.  (All other CTAs' writes are visible: scan_last_block fenced.)
__device__ void layer_finish(const int64_t* __restrict__ off, const int32_t* __restrict__ col,
                             const int32_t* __restrict__ nodes, int64_t live, int f,
                             uint64_t* __restrict__ rng, LayerWs ws,
                             const int32_t* __restrict__ indptr, int32_t* __restrict__ picks,
                             int64_t max_picks, int64_t* __restrict__ num_picks,
                             int32_t* __restrict__ err_flag, int64_t* s_bad_slot,
                             int64_t delta0 = 0) {
  int64_t& s_bad = *s_bad_slot;
  const int64_t tot_draws = ws.scal[1];  // from the prefix kernel
  if (threadIdx.x == 0) s_bad = *(volatile int64_t*)&ws.scal[2];
  __syncthreads();
  int64_t bad = s_bad;
  int64_t delta = delta0;
  const int64_t nominal = 2 * (int64_t)f - 1;
  while (bad != 0) {
    const int64_t b = INT64_MAX - bad;
    delta += (int64_t)ws.used[b] - nominal;
    __syncthreads();
    if (threadIdx.x == 0) *(volatile int64_t*)&ws.scal[2] = 0;
    __syncthreads();
    for (int64_t k = b + 1 + threadIdx.x; k < live; k += blockDim.x) {
      const int32_t u = nodes[k];
      if (off[u + 1] - off[u] <= f) continue;  // no draws: unaffected
      const uint32_t used = sample_node(off, col, u, f, rng, (uint64_t)(ws.draw_off[k] + delta),
                                        picks + indptr[k], nullptr);
      ws.used[k] = used;
      if ((int64_t)used != nominal) atomicMax((long long*)&ws.scal[2], (long long)(INT64_MAX - k));
    }
    __threadfence_block();
    __syncthreads();
    if (threadIdx.x == 0) s_bad = *(volatile int64_t*)&ws.scal[2];
    __syncthreads();
    bad = s_bad;
  }
  if (threadIdx.x == 0) {
    ws.scal[3] = delta;
    const uint64_t T = (uint64_t)(tot_draws + delta);
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

// Two-level bitmap: level 0 = one bit per node (words0 words, a multiple of
// 32), level 1 = one bit per level-0 word (at bm + words0), set by the
// marker that turned the word non-zero.  Compaction walks level 1 and reads
// only non-empty level-0 words (MAG240M-shape: 1 MB instead of 30 MB per
// unique, and the word-prefix table is written only where ranks are asked).
inline int64_t bm_words0(int64_t n) { return ((n + 31) / 32 + 31) / 32 * 32; }

__device__ __forceinline__ void bm_mark(uint32_t* __restrict__ bm, int64_t words0, int64_t v) {
  const int64_t w = v >> 5;
  const uint32_t old = atomicOr(bm + w, 1u << (v & 31));
  if (old == 0u) atomicOr(bm + words0 + (w >> 5), 1u << (w & 31));
}

__global__ void k_mark32(const int32_t* __restrict__ ids, const int64_t* __restrict__ cnt,
                         int64_t max_count, uint32_t* __restrict__ bm, int64_t words0) {
  const int64_t live = min64(*cnt, max_count);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < live;
       i += (int64_t)gridDim.x * blockDim.x)
    bm_mark(bm, words0, ids[i]);
}
__global__ void k_mark64(const int64_t* __restrict__ ids, const int64_t* __restrict__ cnt,
                         int64_t max_count, uint32_t* __restrict__ bm, int64_t words0) {
  const int64_t live = min64(*cnt, max_count);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < live;
       i += (int64_t)gridDim.x * blockDim.x)
    bm_mark(bm, words0, ids[i]);
}


// Kernel 1 of a layer: per-node (picks, draws) counts and their exclusive
// prefix in one pass (look-back); writes indptr and each node's stream
// offset; the last CTA writes the totals.
// Register-resident Floyd + tail shuffle for a compile-time fanout F <= 16
// (same draws and results as sample_node; no local-memory index buffer).
template <int F>
__device__ __forceinline__ uint32_t sample_node_reg(const int64_t* __restrict__ off,
                                                    const int32_t* __restrict__ col, int32_t u,
                                                    const uint64_t* blk, uint64_t q,
                                                    int32_t* __restrict__ out) {
  const int64_t b = off[u];
  const int64_t deg = off[u + 1] - b;
  if (deg <= F) {
    for (int64_t t = 0; t < deg; ++t) out[t] = col[b + t];
    return 0;
  }
  PcgCursor c = rng_cursor_at(blk, q);
  uint32_t used = 0;
  uint32_t idx[F];
#pragma unroll
  for (int t = 0; t < F; ++t) {
    const uint32_t j = (uint32_t)(deg - F + t);
    const uint32_t v = c.lemire(j, used);
    bool dup = false;
#pragma unroll
    for (int s2 = 0; s2 < t; ++s2) dup |= idx[s2] == v;
    idx[t] = dup ? j : v;
  }
#pragma unroll
  for (int i = F - 1; i >= 1; --i) {
    const uint32_t j = c.lemire((uint32_t)i, used);
    uint32_t vj = idx[0];
#pragma unroll
    for (int s2 = 1; s2 < i; ++s2) vj = (uint32_t)s2 == j ? idx[s2] : vj;
    vj = j == (uint32_t)i ? idx[i] : vj;
#pragma unroll
    for (int s2 = 0; s2 < i; ++s2) idx[s2] = (uint32_t)s2 == j ? idx[i] : idx[s2];
    idx[i] = vj;
  }
#pragma unroll
  for (int t = 0; t < F; ++t) out[t] = col[b + idx[t]];
  return used;
}

__global__ void __launch_bounds__(kSampThreads)
k_layer_prefix(const int64_t* __restrict__ off, const int32_t* __restrict__ nodes,
               const int64_t* __restrict__ nlive, int64_t N, int f, LayerWs ws,
               int32_t* __restrict__ indptr, int64_t max_picks, int64_t* __restrict__ num_picks,
               int32_t* __restrict__ err_flag, unsigned int ntiles) {
  using BS = cub::BlockScan<unsigned long long, kSampThreads>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ unsigned int s_u32;
  __shared__ unsigned long long s_u64;
  const ScanState sc{ws.status, ws.ctr, ws.ctr + 1};
  const unsigned int tile = scan_take_tile(sc, &s_u32);
  const int64_t i = (int64_t)tile * kSampThreads + threadIdx.x;
  const int64_t live = min64(*nlive, N);
  int64_t deg, cnt, draws;
  node_counts(off, nodes, i, live, f, deg, cnt, draws);
  if (deg > 10000 && f > deg / 50) atomicExch(err_flag, FG_EUSAGE);  // numpy's FY branch
  const unsigned long long mine = ((unsigned long long)draws << kPickBits) | (unsigned long long)cnt;
  unsigned long long excl, agg;
  BS(tmp).ExclusiveSum(mine, excl, agg);
  const unsigned long long prefix = scan_tile_prefix(sc, tile, agg, &s_u64);
  const int64_t pick_off = (int64_t)((prefix & kPickMask) + (excl & kPickMask));
  const int64_t draw_off = (int64_t)((prefix >> kPickBits) + (excl >> kPickBits));
  if (i < N) indptr[i] = (int32_t)pick_off;
  if (i == N - 1) indptr[N] = (int32_t)(pick_off + cnt);
  if (i < live) ws.draw_off[i] = draw_off;
  if (scan_last_block(sc, ntiles, &s_u32) && threadIdx.x == 0) {
    const unsigned long long total = ws.status[ntiles - 1] & kScanValMask;
    const int64_t tot_picks = (int64_t)(total & kPickMask);
    *num_picks = tot_picks;
    ws.scal[0] = tot_picks;
    ws.scal[1] = (int64_t)(total >> kPickBits);
    if (tot_picks > max_picks) atomicExch(err_flag, FG_EUSAGE);
  }
}

// Last CTA of the sampling kernel (done ticket ctr[2]): fix-up + advance.
__device__ __forceinline__ bool sample_last_block(LayerWs ws, unsigned int nblocks,
                                                  unsigned int* slot) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) *slot = atomicAdd(ws.ctr + 2, 1u) == nblocks - 1 ? 1u : 0u;
  __syncthreads();
  const bool last = *slot != 0;
  if (last) __threadfence();
  return last;
}

// Kernel 2, thread per node (large layers): serial numpy-exact sampling;
// F > 0 selects the register-resident variant for that fanout.  The PCG64
// block (state + jump table) is read from shared memory.
template <int F>
__global__ void __launch_bounds__(kSampThreads)
k_layer_sample(const int64_t* __restrict__ off, const int32_t* __restrict__ col,
               const int32_t* __restrict__ nodes, const int64_t* __restrict__ nlive, int64_t N,
               int f, uint64_t* __restrict__ rng, LayerWs ws, const int32_t* __restrict__ indptr,
               int32_t* __restrict__ picks, int64_t max_picks, int64_t* __restrict__ num_picks,
               int32_t* __restrict__ err_flag) {
  __shared__ unsigned int s_u32;
  __shared__ int64_t s_bad;
  __shared__ uint64_t s_blk[FG_RNG_WORDS];
  for (int k = threadIdx.x; k < FG_RNG_WORDS; k += blockDim.x) s_blk[k] = rng[k];
  __syncthreads();
  const int64_t live = min64(*nlive, N);
  const int64_t i = blockIdx.x * (int64_t)kSampThreads + threadIdx.x;
  if (i < live) {
    const int32_t u = nodes[i];
    const int64_t deg = off[u + 1] - off[u];
    const int32_t po = indptr[i];
    const int64_t draws = deg > f ? 2 * (int64_t)f - 1 : 0;
    if (po + min64(deg, f) <= max_picks) {
      const uint32_t used =
          F > 0 ? sample_node_reg<(F > 0 ? F : 1)>(off, col, u, s_blk, (uint64_t)ws.draw_off[i],
                                                   picks + po)
                : sample_node(off, col, u, f, s_blk, (uint64_t)ws.draw_off[i], picks + po,
                              nullptr);
      ws.used[i] = used;
      if ((int64_t)used != draws) atomicMax((long long*)&ws.scal[2], (long long)(INT64_MAX - i));
    }
  }
  if (!sample_last_block(ws, gridDim.x, &s_u32)) return;
  // a rejection leaves the layer to k_layer_fixup (parallel re-sample of the
  // later nodes); otherwise finish here (advance the stream)
  if (*(volatile int64_t*)&ws.scal[2] != 0) return;
  layer_finish(off, col, nodes, live, f, rng, ws, indptr, picks, max_picks, num_picks, err_flag,
               &s_bad);
}

// Kernel 2 (D = 2f-1 <= G): a group of G lanes owns one node.  Lane t
// computes the node's t-th 32-bit draw directly (the group leader jumps the
// PCG64 cursor to the node's stream offset; lanes step <= 16 outputs further
// through the jump table), every Lemire draw is evaluated in parallel, then
// Floyd's duplicate rule and the tail shuffle run as f and f-1 shuffle
// steps.  If any draw of the node would be rejected by Lemire the leader
// redoes the node serially (exact numpy consumption; the layer fix-up then
// shifts later nodes).
template <int G>
__global__ void __launch_bounds__(kSampThreads)
k_layer_sample_group(const int64_t* __restrict__ off, const int32_t* __restrict__ col,
                     const int32_t* __restrict__ nodes, const int64_t* __restrict__ nlive,
                     int64_t N, int f, uint64_t* __restrict__ rng, LayerWs ws,
                     const int32_t* __restrict__ indptr, int32_t* __restrict__ picks,
                     int64_t max_picks, int64_t* __restrict__ num_picks,
                     int32_t* __restrict__ err_flag) {
  constexpr int NPB = kSampThreads / G;
  __shared__ unsigned int s_u32;
  __shared__ int64_t s_bad;
  __shared__ uint64_t s_blk[FG_RNG_WORDS];  // PCG64 state + jump table
  for (int k = threadIdx.x; k < FG_RNG_WORDS; k += blockDim.x) s_blk[k] = rng[k];
  __syncthreads();
  const uint64_t* s_tab = s_blk + RNG_TABLE;  // entries for 1, 2, 4, 8, 16 steps
  const int gl = threadIdx.x % G;
  const int64_t i = blockIdx.x * (int64_t)NPB + threadIdx.x / G;
  const unsigned int gmask =
      G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
  const int64_t live = min64(*nlive, N);
  if (i < live) {
    const int32_t u = nodes[i];
    const int64_t b = off[u];
    const int64_t deg = off[u + 1] - b;
    const int32_t po = indptr[i];
    const int64_t draw_off = ws.draw_off[i];
    int32_t* out = picks + po;
    uint32_t used = 0;
    if (po + min64(deg, f) <= max_picks) {
      if (deg <= f) {
        for (int64_t t = gl; t < deg; t += G) out[t] = col[b + t];
      } else {
        uint64_t s_lo = 0, s_hi = 0;
        uint32_t have = 0, hbuf = 0;
        if (gl == 0) {
          const PcgCursor c0 = rng_cursor_at(s_blk, (uint64_t)draw_off);
          s_lo = c0.s.lo; s_hi = c0.s.hi; have = c0.have; hbuf = c0.hi;
        }
        s_lo = __shfl_sync(gmask, s_lo, 0, G);
        s_hi = __shfl_sync(gmask, s_hi, 0, G);
        have = __shfl_sync(gmask, have, 0, G);
        hbuf = __shfl_sync(gmask, hbuf, 0, G);
        const int D = 2 * f - 1;
        uint32_t res = 0;
        bool rej = false;
        if (gl < D) {
          uint32_t val;
          if (have && gl == 0) {
            val = hbuf;
          } else {
            const uint32_t q = have ? gl - 1 : gl;
            const uint32_t k = (q >> 1) + 1;  // outputs to step (<= 16)
            u128 st = make_u128(s_hi, s_lo);
#pragma unroll
            for (int bit = 0; bit < 5; ++bit) {
              if (k & (1u << bit)) {
                const uint64_t* e = s_tab + 4 * bit;
                st = muladd128(make_u128(e[1], e[0]), st, make_u128(e[3], e[2]));
              }
            }
            const uint64_t o = xsl_rr(st);
            val = (q & 1) ? (uint32_t)(o >> 32) : (uint32_t)o;
          }
          // Floyd step t < f draws on [0, deg-f+t]; shuffle draw t >= f on [0, 2f-1-t]
          const uint32_t r = gl < f ? (uint32_t)(deg - f + gl) : (uint32_t)(2 * f - 1 - gl);
          const uint32_t span = r + 1u;
          const uint64_t m = (uint64_t)val * span;
          const uint32_t low = (uint32_t)m;
          if (low < span) rej = low < (0xFFFFFFFFu - r) % span;
          res = (uint32_t)(m >> 32);
        }
        if (__any_sync(gmask, rej)) {
          if (gl == 0) used = sample_node(off, col, u, f, rng, (uint64_t)draw_off, out, nullptr);
        } else {
          uint32_t sel = res;  // lane t < f: t-th Floyd choice
          for (int t = 0; t < f; ++t) {
            const uint32_t vt = __shfl_sync(gmask, res, t, G);
            const unsigned int hit = __ballot_sync(gmask, gl < t && sel == vt) & gmask;
            if (gl == t && hit) sel = (uint32_t)(deg - f + t);
          }
          for (int ii = f - 1; ii >= 1; --ii) {  // tail shuffle
            const uint32_t j = __shfl_sync(gmask, res, 2 * f - 1 - ii, G);
            const uint32_t a = __shfl_sync(gmask, sel, ii, G);
            const uint32_t bj = __shfl_sync(gmask, sel, (int)j, G);
            if (gl == ii) sel = bj;
            if (gl == (int)j) sel = a;
          }
          if (gl < f) out[gl] = col[b + sel];
          used = (uint32_t)D;
        }
        if (gl == 0) {
          ws.used[i] = used;
          if ((int64_t)used != D) atomicMax((long long*)&ws.scal[2], (long long)(INT64_MAX - i));
        }
      }
    }
  }
  if (!sample_last_block(ws, gridDim.x, &s_u32)) return;
  // a rejection leaves the layer to k_layer_fixup (parallel re-sample of the
  // later nodes); otherwise finish here (advance the stream)
  if (*(volatile int64_t*)&ws.scal[2] != 0) return;
  layer_finish(off, col, nodes, live, f, rng, ws, indptr, picks, max_picks, num_picks, err_flag,
               &s_bad);
}

// Kernel 3 (no-op unless the sampling kernel saw a Lemire rejection): the
// first rejecting node b consumed delta extra draws, so every later node's
// draws start delta further into the stream.  All of them are re-sampled in
// parallel (thread per node) at the corrected offsets; a rejection among
// them (rare squared) is handled by the last CTA's serial loop
// (layer_finish), which also advances the stream.
__global__ void __launch_bounds__(kSampThreads)
k_layer_fixup(const int64_t* __restrict__ off, const int32_t* __restrict__ col,
              const int32_t* __restrict__ nodes, const int64_t* __restrict__ nlive, int64_t N,
              int f, uint64_t* __restrict__ rng, LayerWs ws, const int32_t* __restrict__ indptr,
              int32_t* __restrict__ picks, int64_t max_picks, int64_t* __restrict__ num_picks,
              int32_t* __restrict__ err_flag) {
  const int64_t bad = ws.scal[2];
  if (bad == 0) return;  // uniform across the grid: nothing to redo
  __shared__ unsigned int s_u32;
  __shared__ int64_t s_bad;
  __shared__ uint64_t s_blk[FG_RNG_WORDS];
  for (int k = threadIdx.x; k < FG_RNG_WORDS; k += blockDim.x) s_blk[k] = rng[k];
  __syncthreads();
  const int64_t live = min64(*nlive, N);
  const int64_t b = INT64_MAX - bad;
  const int64_t nominal = 2 * (int64_t)f - 1;
  const int64_t delta = (int64_t)ws.used[b] - nominal;
  for (int64_t i = b + 1 + blockIdx.x * (int64_t)kSampThreads + threadIdx.x; i < live;
       i += (int64_t)gridDim.x * kSampThreads) {
    const int32_t u = nodes[i];
    const int64_t deg = off[u + 1] - off[u];
    const int32_t po = indptr[i];
    if (deg > f && po + f <= max_picks) {
      const uint32_t used = sample_node(off, col, u, f, s_blk,
                                        (uint64_t)(ws.draw_off[i] + delta), picks + po, nullptr);
      ws.used[i] = used;
      if ((int64_t)used != nominal) atomicMax((long long*)&ws.scal[4], (long long)(INT64_MAX - i));
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_u32 = atomicAdd(ws.ctr + 3, 1u) == gridDim.x - 1 ? 1u : 0u;
  __syncthreads();
  if (!s_u32) return;
  __threadfence();
  // the serial loop continues from the pass's first rejection (if any) with
  // the shift accumulated so far
  if (threadIdx.x == 0) ws.scal[2] = *(volatile int64_t*)&ws.scal[4];
  __syncthreads();
  layer_finish(off, col, nodes, live, f, rng, ws, indptr, picks, max_picks, num_picks, err_flag,
               &s_bad, delta);
}

// Single-pass compaction over level 1: thread per kBmIpt consecutive quarters
// of level-1 words (8 level-0 words = 256 node ids each); popcounts of its
// non-empty words, block scan, decoupled look-back prefix, ordered emit of
// the set bits (ascending ids) and the word prefix of every non-empty level-0
// word.  IPT = 8 for large bitmaps (round 2: a papers100M-shape bitmap, 111 M
// ids, is 212 tiles instead of 1.7 K, one wave with a short look-back chain),
// 1 below ~10 M ids (products-shape: 1 item per thread keeps ~40 CTAs busy).
constexpr int kBmIpt = 8;
inline int bm_ipt(int64_t words0) {
  static const int env = [] {  // FG_BM_IPT: force 1 / 2 / 4 / 8 / 16 items per thread
    const char* e = getenv("FG_BM_IPT");
    return e ? atoi(e) : 0;
  }();
  if (env == 1 || env == 2 || env == 4 || env == 8 || env == 16) return env;
  return words0 / 32 * 4 >= 148ll * kBmThreads * 8 ? kBmIpt : 1;
}
template <int IPT>
__global__ void __launch_bounds__(kBmThreads)
k_bm_compact(const uint32_t* __restrict__ bm, int64_t words0, unsigned long long* status,
             unsigned int* ctr, int32_t* __restrict__ out, int64_t max_out,
             int64_t* __restrict__ out_count, int32_t* __restrict__ wprefix, unsigned int ntiles) {
  using BS = cub::BlockScan<unsigned long long, kBmThreads>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ unsigned int s_u32;
  __shared__ unsigned long long s_u64;
  const ScanState sc{status, ctr, ctr + 1};
  const unsigned int tile = scan_take_tile(sc, &s_u32);
  // items = (level-1 word j, quarter qq), kBmIpt consecutive per thread:
  // level-0 words 32j + 8qq .. +7
  const int64_t l1w = words0 / 32;
  const int64_t item0 = ((int64_t)tile * kBmThreads + threadIdx.x) * IPT;
  uint32_t l1[IPT];
  unsigned long long c = 0;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int64_t item = item0 + i;
    const int64_t j = item >> 2;
    l1[i] = j < l1w ? (__ldg(bm + words0 + j) >> (8 * (int)(item & 3))) & 0xFFu : 0u;
    const int64_t wbase = j * 32 + 8 * (item & 3);
    for (uint32_t x = l1[i]; x; x &= x - 1) c += __popc(__ldg(bm + wbase + (__ffs(x) - 1)));
  }
  unsigned long long excl, agg;
  BS(tmp).ExclusiveSum(c, excl, agg);
  const unsigned long long prefix = scan_tile_prefix(sc, tile, agg, &s_u64);
  int64_t pos = (int64_t)(prefix + excl);
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int64_t item = item0 + i;
    const int64_t wbase = (item >> 2) * 32 + 8 * (item & 3);
    for (uint32_t x = l1[i]; x; x &= x - 1) {
      const int64_t w = wbase + (__ffs(x) - 1);
      uint32_t bits = __ldg(bm + w);
      if (wprefix) wprefix[w] = (int32_t)pos;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        if (pos < max_out) out[pos] = (int32_t)((w << 5) + b);
        ++pos;
      }
    }
  }
  if (scan_last_block(sc, ntiles, &s_u32) && threadIdx.x == 0)
    *out_count = (int64_t)(status[ntiles - 1] & kScanValMask);
}

// Seed layer (pipeline.py:203 np.sort of the batch's permutation slice): one
// CTA radix-sorts the <= 4096 seed ids in shared memory (cub::BlockRadixSort
// over the id bits) instead of marking, compacting and clearing the whole
// n-bit bitmap (three kernels, ~25 us at papers100M-shape for 1024 ids).
// Duplicates are kept, as np.sort keeps them.
template <int IPT>
__global__ void __launch_bounds__(1024)
k_sort_ids(const int64_t* __restrict__ ids, const int64_t* __restrict__ cnt, int64_t cap,
           int32_t* __restrict__ out, int64_t* __restrict__ out_cnt, int end_bit) {
  using BRS = cub::BlockRadixSort<uint32_t, 1024, IPT>;
  __shared__ typename BRS::TempStorage tmp;
  const int64_t live = min64(*cnt, cap);
  uint32_t k[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int64_t j = (int64_t)threadIdx.x * IPT + i;
    k[i] = j < live ? (uint32_t)ids[j] : 0xFFFFFFFFu;
  }
  // pads (0xFFFFFFFF) sort after every id: their low end_bit bits are the
  // maximum and the sort is stable (pads come last in the input)
  BRS(tmp).Sort(k, 0, end_bit);
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int64_t j = (int64_t)threadIdx.x * IPT + i;
    if (j < live) out[j] = (int32_t)k[i];
  }
  if (threadIdx.x == 0) *out_cnt = live;
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
                           int64_t max_count, uint32_t* __restrict__ bm, int64_t words0) {
  const int64_t live = min64(*cnt, max_count);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < live;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = ids[i] >> 5;
    bm[w] = 0u;
    bm[words0 + (w >> 5)] = 0u;
  }
}

}  // namespace fg

using namespace fg;

// Grid of the sampler's grid-stride helper kernels (mark / rank / clear):
// FG_SAMPLER_PER_SM CTAs per SM (default 8).  Fewer CTAs leave more SM slots
// to the training kernels the sampler overlaps with.
static int sampler_grid(int64_t items) {
  static const int per_sm = [] {
    const char* e = getenv("FG_SAMPLER_PER_SM");
    const int v = e ? atoi(e) : 8;
    return v > 0 ? v : 8;
  }();
  return grid_for(items, 256, per_sm);
}

extern "C" {

int64_t fg_sample_workspace_bytes(int64_t max_nodes) { return layer_ws_bytes(max_nodes); }

int fg_sample_layer(const int64_t* row_offsets, const int32_t* col_indices, int64_t n,
                    const int32_t* nodes, const int64_t* num_nodes_dev, int64_t max_nodes,
                    int fanout, uint64_t* rng_dev, int32_t* indptr, int32_t* picks,
                    int64_t max_picks, int64_t* num_picks_dev, uint32_t* bitmap, void* ws,
                    int64_t ws_bytes, int32_t* err_flag, void* s) {
  FG_CHECK_ARG(fanout >= 1, "fanouts must be >= 1");
  // (numpy's partial Fisher-Yates branch, deg > 10000 and f > deg // 50, is
  // flagged per node by k_layer_prefix: any fanout is accepted up front)
  FG_CHECK_ARG(max_nodes >= 1 && n >= 1, "fg_sample_layer: empty layer capacity");
  FG_CHECK_ARG(ws_bytes >= layer_ws_bytes(max_nodes), "fg_sample_layer: workspace too small");
  FG_CHECK_ARG(max_picks < INT32_MAX && max_picks < (1ll << kPickBits),
               "fg_sample_layer: picks must fit int32 offsets");
  FG_CHECK_ARG(row_offsets && col_indices && nodes && num_nodes_dev && rng_dev && indptr &&
                   picks && num_picks_dev && err_flag,
               "fg_sample_layer: null argument");
  cudaStream_t st = as_stream(s);
  LayerWs w = carve(ws, max_nodes);
  FG_CUDA_TRY(cudaMemsetAsync(ws, 0, w.head_bytes, st));
  const int64_t nt = ceil_div(max_nodes, kSampThreads);
  k_layer_prefix<<<(unsigned)nt, kSampThreads, 0, st>>>(row_offsets, nodes, num_nodes_dev,
                                                        max_nodes, fanout, w, indptr, max_picks,
                                                        num_picks_dev, err_flag, (unsigned)nt);
  FG_LAUNCH_CHECK();
  const int D = 2 * fanout - 1;
  // tiny layer (the seeds): G lanes per node (parallel draws).  Above
  // FG_SAMPLE_GROUP_MAX nodes (default 2048) thread-per-node: G x fewer warps,
  // which measured faster once sampling overlaps training (15 K-node layer:
  // sample chain 155 -> 147 us, pipelined step 302 -> 288 us).
  static const int64_t group_max = [] {
    const char* e = getenv("FG_SAMPLE_GROUP_MAX");
    return e ? (int64_t)atoll(e) : (int64_t)2048;
  }();
  if (D <= 32 && max_nodes <= group_max) {
    const int G = D <= 16 ? 16 : 32;
    const int64_t nb = ceil_div(max_nodes, kSampThreads / G);
    if (G == 16)
      k_layer_sample_group<16><<<(unsigned)nb, kSampThreads, 0, st>>>(
          row_offsets, col_indices, nodes, num_nodes_dev, max_nodes, fanout, rng_dev, w, indptr,
          picks, max_picks, num_picks_dev, err_flag);
    else
      k_layer_sample_group<32><<<(unsigned)nb, kSampThreads, 0, st>>>(
          row_offsets, col_indices, nodes, num_nodes_dev, max_nodes, fanout, rng_dev, w, indptr,
          picks, max_picks, num_picks_dev, err_flag);
  } else {
#define FG_SAMPLE_F(F)                                                                     \
  k_layer_sample<F><<<(unsigned)nt, kSampThreads, 0, st>>>(                               \
      row_offsets, col_indices, nodes, num_nodes_dev, max_nodes, fanout, rng_dev, w, indptr, \
      picks, max_picks, num_picks_dev, err_flag)
    switch (fanout) {
      case 1: FG_SAMPLE_F(1); break;
      case 2: FG_SAMPLE_F(2); break;
      case 3: FG_SAMPLE_F(3); break;
      case 4: FG_SAMPLE_F(4); break;
      case 5: FG_SAMPLE_F(5); break;
      case 6: FG_SAMPLE_F(6); break;
      case 8: FG_SAMPLE_F(8); break;
      case 10: FG_SAMPLE_F(10); break;
      case 12: FG_SAMPLE_F(12); break;
      case 15: FG_SAMPLE_F(15); break;
      case 16: FG_SAMPLE_F(16); break;
      default: FG_SAMPLE_F(0); break;
    }
#undef FG_SAMPLE_F
  }
  FG_LAUNCH_CHECK();
  // grid-stride over the nodes after the first rejection: a few CTAs per SM
  // (the common no-rejection case is one flag read per CTA; a capacity-sized
  // grid of immediately-exiting CTAs cost ~9 us per MAG-scale layer)
  const unsigned fix_grid = (unsigned)min64(nt, (int64_t)sm_count() * 4);
  k_layer_fixup<<<fix_grid, kSampThreads, 0, st>>>(row_offsets, col_indices, nodes,
                                                       num_nodes_dev, max_nodes, fanout, rng_dev, w,
                                                       indptr, picks, max_picks, num_picks_dev,
                                                       err_flag);
  FG_LAUNCH_CHECK();
  if (bitmap) {  // next layer's unique set: mark after any fix-up rewrote picks
    k_mark32<<<sampler_grid(max_picks), 256, 0, st>>>(picks, num_picks_dev, max_picks, bitmap,
                                                       bm_words0(n));
    FG_LAUNCH_CHECK();
  }
  return FG_OK;
}

int64_t fg_bitmap_words(int64_t n) { return bm_words0(n) + bm_words0(n) / 32; }

int64_t fg_bitmap_workspace_bytes(int64_t n) {
  const int64_t l1w = bm_words0(n > 0 ? n : 1) / 32;
  const int64_t nb = ceil_div(4 * l1w, (int64_t)kBmThreads);  // IPT = 1 upper bound
  return align256(64 + nb * 8);
}

int fg_bitmap_mark(const int32_t* ids, const int64_t* cnt, int64_t max_count, uint32_t* bm,
                   int64_t n, void* s) {
  if (max_count == 0) return FG_OK;
  k_mark32<<<sampler_grid(max_count), 256, 0, as_stream(s)>>>(ids, cnt, max_count, bm,
                                                               bm_words0(n));
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_bitmap_mark64(const int64_t* ids, const int64_t* cnt, int64_t max_count, uint32_t* bm,
                     int64_t n, void* s) {
  if (max_count == 0) return FG_OK;
  k_mark64<<<sampler_grid(max_count), 256, 0, as_stream(s)>>>(ids, cnt, max_count, bm,
                                                               bm_words0(n));
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_bitmap_compact(uint32_t* bm, int64_t n, int32_t* out_ids, int64_t max_out,
                      int64_t* out_count, int32_t* wprefix, void* ws, int64_t ws_bytes, void* s) {
  FG_CHECK_ARG(n >= 1 && n < INT32_MAX, "fg_bitmap_compact: n must be in [1, 2^31)");
  FG_CHECK_ARG(ws_bytes >= fg_bitmap_workspace_bytes(n), "fg_bitmap_compact: workspace too small");
  cudaStream_t st = as_stream(s);
  const int64_t words0 = bm_words0(n);
  const int ipt = bm_ipt(words0);
  const int64_t nb = ceil_div(4 * (words0 / 32), (int64_t)kBmThreads * ipt);
  unsigned int* ctr = (unsigned int*)ws;
  unsigned long long* status = (unsigned long long*)((char*)ws + 64);
  FG_CUDA_TRY(cudaMemsetAsync(ws, 0, 64 + nb * 8, st));
  auto kern = ipt == 16 ? k_bm_compact<16> : ipt == 8 ? k_bm_compact<8> : ipt == 4 ? k_bm_compact<4>
            : ipt == 2 ? k_bm_compact<2> : k_bm_compact<1>;
  kern<<<(unsigned)nb, kBmThreads, 0, st>>>(bm, words0, status, ctr, out_ids, max_out, out_count,
                                            wprefix, (unsigned)nb);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_sort_ids(const int64_t* ids, const int64_t* cnt, int64_t cap, int32_t* out,
                int64_t* out_cnt, int64_t n, void* s) {
  FG_CHECK_ARG(cap >= 0 && cap <= 4096, "fg_sort_ids: at most 4096 ids");
  FG_CHECK_ARG(n >= 1 && n < INT32_MAX, "fg_sort_ids: n must be in [1, 2^31)");
  if (cap == 0) return FG_OK;
  cudaStream_t st = as_stream(s);
  const int ipt = (int)ceil_div(cap, 1024);
  int end_bit = 1;
  while (end_bit < 32 && (1ll << end_bit) < n) ++end_bit;  // ids < n <= 2^end_bit
  switch (ipt) {
    case 1: k_sort_ids<1><<<1, 1024, 0, st>>>(ids, cnt, cap, out, out_cnt, end_bit); break;
    case 2: k_sort_ids<2><<<1, 1024, 0, st>>>(ids, cnt, cap, out, out_cnt, end_bit); break;
    case 3: k_sort_ids<3><<<1, 1024, 0, st>>>(ids, cnt, cap, out, out_cnt, end_bit); break;
    default: k_sort_ids<4><<<1, 1024, 0, st>>>(ids, cnt, cap, out, out_cnt, end_bit); break;
  }
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_bitmap_rank(const int32_t* ids, const int64_t* cnt, int64_t max_count, const uint32_t* bm,
                   const int32_t* wprefix, int32_t* rank, void* s) {
  if (max_count == 0) return FG_OK;
  k_bm_rank<<<sampler_grid(max_count), 256, 0, as_stream(s)>>>(ids, cnt, max_count, bm, wprefix,
                                                                rank);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_bitmap_clear(const int32_t* ids, const int64_t* cnt, int64_t max_count, uint32_t* bm,
                    int64_t n, void* s) {
  if (max_count == 0) return FG_OK;
  k_bm_clear<<<sampler_grid(max_count), 256, 0, as_stream(s)>>>(ids, cnt, max_count, bm,
                                                                  bm_words0(n));
  FG_LAUNCH_CHECK();
  return FG_OK;
}

}  // extern "C"
