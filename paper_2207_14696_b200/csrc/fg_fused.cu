// Fused gather -> decode -> mean over a sampled block (the north-star hot path).
//
// Semantics: out[v] = (1/cnt_v) * sum over the sampled picks u of v of
// decode(u), the row-stochastic mean D̂⁻¹Â of pkg/src/featgrind/factors.py:
// 108-114 restricted to the sampled block; decode(u) is exactly
// dequantize_sq (sq.py:132-153) or decode_vq (vq.py:330-344).  Decoded rows
// exist only in registers: HBM sees the packed code rows and the aggregate.
//
// Roofline: HBM-bound.  Algorithmic bytes per launch
//   E * (row_bytes + 4) + N_dst * (4 + d * out_bytes)
//
// Structure (v2, after ncu showed v1 issue-bound at 70 % issue / 6 % DRAM):
//  * persistent CTAs walk tiles of kTD destinations; the tile's indptr slice
//    and source ids are staged in shared memory with coalesced loads;
//  * VQ 8-bit codes: one thread owns a destination and G = 32/W consecutive
//    parts, so each pick costs ONE aligned G-byte load of its code row, G
//    shared-memory codebook lookups and G*W/2 packed FADD2s; all U picks'
//    loads of an unrolled batch are issued before any lookup;
//  * SQ: one thread owns 16 codes of a destination row (one 2k-byte load per
//    pick), LUT replicated 32x across banks (conflict-free), FADD2 sums;
//  * mean via one reciprocal per destination, vector stores, and only live
//    destinations are written (rows past the live count keep their previous,
//    finite contents; callers zero the buffer once at allocation);
//  * `out_ld` lets the caller pad rows (e.g. d=100 -> 112) so the following
//    bf16 GEMM sees 16-element-aligned K.
#include <algorithm>
#include <stdlib.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <type_traits>

#include "fg_common.cuh"

namespace fg {

constexpr int kTD = 128;     // destinations per tile
constexpr int kSrcCap = kTD * 8;   // staged src ids per tile (fanout <= 8 fully staged)

__device__ __forceinline__ int64_t live_dst(const int64_t* p, int64_t cap) {
  const int64_t v = *p;
  return v < cap ? v : cap;
}

typedef unsigned long long u64;

// packed fp32 pair add (sm_100 FADD2); identical rounding to two FADDs
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) {
  u64 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// packed fp32 pair fma (sm_100 FFMA2): a * b + c per lane of the pair
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
// acc += x (mean) or acc += w * x (edge-weighted sum; w2 = (w, w))
template <bool WT>
__device__ __forceinline__ u64 acc2(u64 acc, u64 x, u64 w2) {
  if constexpr (WT) return ffma2(x, w2, acc);
  else return fadd2(acc, x);
}
__device__ __forceinline__ u64 bcast2(float w) {
  const u64 b = __float_as_uint(w);
  return (b << 32) | b;
}
__device__ __forceinline__ u64 pack2(float x, float y) {
  return ((u64)__float_as_uint(y) << 32) | __float_as_uint(x);
}
__device__ __forceinline__ float lo2(u64 v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi2(u64 v) { return __uint_as_float((uint32_t)(v >> 32)); }

// 32-byte (one full L2 sector) global store: STG.E.256 on sm_100.  The fused
// kernels' threads own 32-64 B output runs; 16-byte stores from lanes 32-64 B
// apart are half-sector writes (ncu, v4 MAG240M: 9.2 M store sectors for
// 148 MB of output = 2x), one 256-bit store per sector is not.
__device__ __forceinline__ void stg256(void* p, const uint32_t* w) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]),
                 "r"(w[6]), "r"(w[7]) : "memory");
}
__device__ __forceinline__ bool aligned32(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 31) == 0;
}

// Store n (multiple of 2) consecutive outputs v[0..n) * inv at p; uses 32-,
// 16- or 8-byte vector stores when `vec` (caller guarantees 16-B alignment;
// 32-B runs are used when the address is 32-B aligned).
template <int N>
__device__ __forceinline__ void store_scaled(float* p, const u64* acc, float inv, bool vec) {
  if (vec && N % 8 == 0 && aligned32(p)) {
#pragma unroll
    for (int i = 0; i < N / 8; ++i) {
      uint32_t w[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        w[2 * j] = __float_as_uint(lo2(acc[4 * i + j]) * inv);
        w[2 * j + 1] = __float_as_uint(hi2(acc[4 * i + j]) * inv);
      }
      stg256(p + 8 * i, w);
    }
  } else if (vec && N % 4 == 0) {
#pragma unroll
    for (int i = 0; i < N / 4; ++i)
      reinterpret_cast<float4*>(p)[i] =
          make_float4(lo2(acc[2 * i]) * inv, hi2(acc[2 * i]) * inv, lo2(acc[2 * i + 1]) * inv,
                      hi2(acc[2 * i + 1]) * inv);
  } else {
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      p[2 * i] = lo2(acc[i]) * inv;
      p[2 * i + 1] = hi2(acc[i]) * inv;
    }
  }
}
template <int N>
__device__ __forceinline__ void store_scaled(__nv_bfloat16* p, const u64* acc, float inv,
                                             bool vec) {
  uint32_t w[N / 2];
#pragma unroll
  for (int i = 0; i < N / 2; ++i) {
    const __nv_bfloat162 b = __floats2bfloat162_rn(lo2(acc[i]) * inv, hi2(acc[i]) * inv);
    w[i] = *reinterpret_cast<const uint32_t*>(&b);
  }
  if (vec && N % 16 == 0 && aligned32(p)) {
#pragma unroll
    for (int i = 0; i < N / 16; ++i) stg256(p + 16 * i, w + 8 * i);
  } else if (vec && N % 8 == 0) {
#pragma unroll
    for (int i = 0; i < N / 8; ++i)
      reinterpret_cast<uint4*>(p)[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
  } else {
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      p[2 * i] = __float2bfloat16_rn(lo2(acc[i]) * inv);
      p[2 * i + 1] = __float2bfloat16_rn(hi2(acc[i]) * inv);
    }
  }
}

// ------------------------------------------------------- tile pipeline
// Each persistent CTA walks tiles tile0, tile0+G, ... of kTD destinations.
// Two smem buffers hold (indptr slice, src ids).  While tile t is computed,
// the src ids of tile t+G (whose indptr slice is already in smem) and the
// indptr slice of tile t+2G are loaded into registers, then stored after the
// compute phase: the staging round trips overlap the code-row loads.
constexpr int kThreads = 512;

template <int NT>
struct Stage {
  static constexpr int kPer = kSrcCap / NT;
  int32_t ip;                 // one indptr entry (threads 0..kTD)
  int32_t src[kPer];          // src ids e0 + threadIdx.x + k*NT
};

template <int NT>
__device__ __forceinline__ void stage_load_ip(const int32_t* __restrict__ indptr, int64_t tile,
                                              int64_t max_dst, Stage<NT>& st) {
  for (int t = threadIdx.x; t <= kTD; t += NT)  // NT may be < kTD + 1
    if (t == (int)threadIdx.x) st.ip = __ldg(indptr + min64(tile * kTD + t, max_dst));
}
template <int NT>
__device__ __forceinline__ void stage_store_ip(int32_t* s_ip, const Stage<NT>& st,
                                               const int32_t* __restrict__ indptr, int64_t tile,
                                               int64_t max_dst) {
  if ((int)threadIdx.x <= kTD) s_ip[threadIdx.x] = st.ip;
  // entries past the thread count (NT <= kTD) are loaded directly
  for (int t = threadIdx.x + NT; t <= kTD; t += NT)
    s_ip[t] = __ldg(indptr + min64(tile * kTD + t, max_dst));
}
template <int NT>
__device__ __forceinline__ void stage_load_src(const int32_t* __restrict__ src, const int32_t* s_ip,
                                               Stage<NT>& st) {
  const int32_t e0 = s_ip[0], cnt = s_ip[kTD] - e0;
  if (cnt > kSrcCap) return;  // compute falls back to global src loads
#pragma unroll
  for (int k = 0; k < Stage<NT>::kPer; ++k) {
    const int t = threadIdx.x + k * NT;
    if (t < cnt) st.src[k] = __ldg(src + e0 + t);
  }
}
// pf_rows (optional): also prefetch each staged source's code row into L2,
// so the next tile's row loads hit L2 instead of DRAM
template <int NT>
__device__ __forceinline__ void stage_store_src(int32_t* s_src, const int32_t* s_ip,
                                                const Stage<NT>& st,
                                                const uint8_t* pf_rows = nullptr,
                                                int64_t pf_stride = 0) {
  const int32_t cnt = s_ip[kTD] - s_ip[0];
  if (cnt > kSrcCap) return;
#pragma unroll
  for (int k = 0; k < Stage<NT>::kPer; ++k) {
    const int t = threadIdx.x + k * NT;
    if (t < cnt) {
      s_src[t] = st.src[k];
      if (pf_rows)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pf_rows + (int64_t)st.src[k] * pf_stride));
    }
  }
}

// Drives the pipeline; `compute(tile, s_ip, s_src)` processes one tile.
template <int NT = kThreads, typename F>
__device__ __forceinline__ void tile_pipeline(const int32_t* __restrict__ indptr,
                                              const int32_t* __restrict__ src, int64_t max_dst,
                                              int64_t ntiles, int32_t* s_ip0, int32_t* s_ip1,
                                              int32_t* s_src0, int32_t* s_src1, F&& compute,
                                              int64_t tile0 = -1, int64_t step = -1,
                                              const uint8_t* pf_rows = nullptr,
                                              int64_t pf_stride = 0) {
  // default: CTA b walks tiles b, b + grid, ...; part-sliced kernels pass
  // their own (first tile, stride) so one slice's CTAs cover every tile
  if (step < 0) step = gridDim.x;
  int64_t tile = tile0 < 0 ? (int64_t)blockIdx.x : tile0;
  Stage<NT> st, st2;
  // prologue: buffer 0 <- (ip, src) of tile; buffer 1 <- ip of tile+step
  stage_load_ip<NT>(indptr, tile, max_dst, st);
  stage_store_ip<NT>(s_ip0, st, indptr, tile, max_dst);
  __syncthreads();
  stage_load_src<NT>(src, s_ip0, st);
  if (tile + step < ntiles) stage_load_ip<NT>(indptr, tile + step, max_dst, st2);
  stage_store_src<NT>(s_src0, s_ip0, st, pf_rows, pf_stride);
  if (tile + step < ntiles) stage_store_ip<NT>(s_ip1, st2, indptr, tile + step, max_dst);
  __syncthreads();
  bool odd = false;
  for (; tile < ntiles; tile += step) {
    int32_t* ip_c = odd ? s_ip1 : s_ip0;
    int32_t* ip_n = odd ? s_ip0 : s_ip1;
    int32_t* src_c = odd ? s_src1 : s_src0;
    int32_t* src_n = odd ? s_src0 : s_src1;
    const bool has_n = tile + step < ntiles, has_nn = tile + 2 * step < ntiles;
    if (has_n) stage_load_src<NT>(src, ip_n, st);
    if (has_nn) stage_load_ip<NT>(indptr, tile + 2 * step, max_dst, st2);
    compute(tile, ip_c, src_c);
    __syncthreads();
    if (has_n) stage_store_src<NT>(src_n, ip_n, st, pf_rows, pf_stride);
    if (has_nn) stage_store_ip<NT>(ip_c, st2, indptr, tile + 2 * step, max_dst);
    __syncthreads();
    odd = !odd;
  }
}

// bf16x2 (low, high) -> packed fp32 pair (low in bits 0..31)
__device__ __forceinline__ u64 bf16x2_to_f32x2(uint32_t w) {
  return ((u64)(w & 0xFFFF0000u) << 32) | (u64)(w << 16);
}
__device__ __forceinline__ uint2 lds64(const void* p) {
  uint2 r;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return r;
}
// one 16-byte shared-memory load (keeps the compiler from splitting it)
__device__ __forceinline__ float4 lds128(const float* p) {
  float4 r;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return r;
}

// --------------------------------------------- bulk async smem fill (TMA)
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// Thread 0 launches cp.async.bulk copies of `bytes` (multiple of 16) from
// global to shared, completing on `mbar`; everyone later waits with
// bulk_wait.  The copy runs on the TMA engine while threads stage tiles.
__device__ __forceinline__ void bulk_fill(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* mbar) {
  if (threadIdx.x == 0) {
    const uint32_t mb = smem_addr(mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes));
    const uint32_t chunk = 32768;
    for (uint32_t off = 0; off < bytes; off += chunk) {
      const uint32_t n = bytes - off < chunk ? bytes - off : chunk;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(smem_addr((char*)dst + off)), "l"((const char*)src + off), "r"(n), "r"(mb)
          : "memory");
    }
  }
}
__device__ __forceinline__ void bulk_wait(uint64_t* mbar) {
  const uint32_t mb = smem_addr(mbar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(mb) : "memory");
  }
}

// ------------------------------------------------------------------- SQ
template <int K>
__device__ __forceinline__ void load_chunk(const uint8_t* p, uint64_t& w0, uint64_t& w1) {
  constexpr int CB = 2 * K;
  w0 = w1 = 0;
  if constexpr (CB == 16) {
    const uint4 q = ldg_stream16(p);
    w0 = ((uint64_t)q.y << 32) | q.x;
    w1 = ((uint64_t)q.w << 32) | q.z;
  } else if constexpr (CB == 8) {
    const uint2 q = ldg_stream8(p);
    w0 = ((uint64_t)q.y << 32) | q.x;
  } else if constexpr (CB == 4) {
    w0 = ldg_stream4(p);
  } else if constexpr (CB == 2) {
    w0 = __ldg(reinterpret_cast<const uint16_t*>(p));
  } else {
#pragma unroll
    for (int b = 0; b < CB; ++b) {
      const uint64_t byte = __ldg(p + b);
      if (b < 8) w0 |= byte << (8 * b); else w1 |= byte << (8 * (b - 8));
    }
  }
}

// Extracts the BW-bit field starting at bit j*K of the MSB-first chunk (BW = K
// for one code, 2K for the pair (code j, code j+1) with code j in the high bits).
template <int K, int BW = K>
__device__ __forceinline__ uint32_t sq_code(uint64_t w0, uint64_t w1, int j) {
  constexpr int Q = 1 << BW;
  const int bit = j * K;
  const int byte = bit >> 3;
  const int inb = bit & 7;
  const uint64_t word = byte < 8 ? w0 : w1;
  if (BW == 8 || inb + BW <= 8) {
    const uint32_t by = (uint32_t)(word >> (8 * (byte & 7))) & 0xFFu;
    return (by >> (8 - inb - BW)) & (Q - 1);
  }
  const int byte2 = byte + 1;
  const uint64_t word2 = byte2 < 8 ? w0 : w1;
  const uint32_t hi = (uint32_t)(word >> (8 * (byte & 7))) & 0xFFu;
  const uint32_t lo = (uint32_t)(word2 >> (8 * (byte2 & 7))) & 0xFFu;
  return (((hi << 8) | lo) >> (16 - inb - BW)) & (Q - 1);
}

template <int K, typename OT, bool WT>
__global__ void __launch_bounds__(kThreads, 2)
k_sq_mean(const uint8_t* __restrict__ rows, int64_t d, int64_t stride,
          const float* __restrict__ lut, const int32_t* __restrict__ indptr,
          const int32_t* __restrict__ src, const int64_t* __restrict__ ndst_dev,
          int64_t max_dst, OT* __restrict__ out, int64_t ld, const float* __restrict__ ew) {
  constexpr int Q = 1 << K;
  constexpr int CB = 2 * K;
  constexpr int U = K >= 5 ? 4 : 8;  // picks whose loads are issued together
  // k <= 4: one LDS.64 fetches the decoded PAIR (code j, code j+1) from a
  // 2^(2k)-entry table of float2, halving lookups and field extracts; the
  // pair lands in a u64 that feeds FADD2 directly.  Each table is replicated
  // per lane (entry * 32 + lane) so lookups are bank-conflict free.
  constexpr bool PAIR = 2 * K <= 8;
  constexpr int LW = PAIR ? (1 << (2 * K)) * 64 : Q * 32;  // table size in floats
  extern __shared__ float s_mem[];
  float* s_lut = s_mem;                                          // [Q][32]
  u64* s_lut2 = reinterpret_cast<u64*>(s_mem);                   // [Q*Q][32]
  int32_t* s_ip0 = reinterpret_cast<int32_t*>(s_mem + LW);       // [kTD + 1] x 2
  int32_t* s_ip1 = s_ip0 + kTD + 1;
  int32_t* s_src0 = s_ip1 + kTD + 1;                             // [kSrcCap] x 2
  int32_t* s_src1 = s_src0 + kSrcCap;
  const int lane = threadIdx.x & 31;
  const int64_t live = live_dst(ndst_dev, max_dst);
  const int64_t ntiles = (live + kTD - 1) / kTD;
  if ((int64_t)blockIdx.x >= ntiles) return;
  if constexpr (PAIR) {
    for (int i = threadIdx.x; i < Q * Q * 32; i += blockDim.x) {
      const int pv = i >> 5;
      s_lut2[i] = pack2(lut[pv >> K], lut[pv & (Q - 1)]);
    }
  } else {
    for (int i = threadIdx.x; i < Q * 32; i += blockDim.x) s_lut[i] = lut[i >> 5];
  }
  const int chunks = (int)((d + 15) >> 4);
  const bool vec_ok = (ld % 16) == 0;
  tile_pipeline(indptr, src, max_dst, ntiles, s_ip0, s_ip1, s_src0, s_src1,
                [&](int64_t tile, const int32_t* s_ip, const int32_t* s_src) {
    const int64_t v0 = tile * kTD;
    const int32_t e0 = s_ip[0];
    const bool staged = s_ip[kTD] - e0 <= kSrcCap;
    const int items = kTD * chunks;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int vl = it / chunks;
      const int c = it - vl * chunks;
      const int64_t v = v0 + vl;
      if (v >= live) break;
      u64 acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0ull;
      const int a = s_ip[vl] - e0;
      const int cnt = s_ip[vl + 1] - e0 - a;
      const int64_t boff = (int64_t)c * CB;
      for (int base = 0; base < cnt; base += U) {
        uint64_t w[U][2];
        u64 wt[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (base + u < cnt) {
            const int e = a + base + u;
            const int32_t sid = staged ? s_src[e] : __ldg(src + e0 + e);
            load_chunk<K>(rows + (int64_t)sid * stride + boff, w[u][0], w[u][1]);
            if constexpr (WT) wt[u] = bcast2(__ldg(ew + e0 + e));
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (base + u < cnt) {
#pragma unroll
            for (int j = 0; j < 16; j += 2) {
              if constexpr (PAIR) {
                const u64 x = s_lut2[sq_code<K, 2 * K>(w[u][0], w[u][1], j) * 32 + lane];
                acc[j / 2] = acc2<WT>(acc[j / 2], x, wt[u]);
              } else {
                const float x0 = s_lut[sq_code<K>(w[u][0], w[u][1], j) * 32 + lane];
                const float x1 = s_lut[sq_code<K>(w[u][0], w[u][1], j + 1) * 32 + lane];
                acc[j / 2] = acc2<WT>(acc[j / 2], pack2(x0, x1), wt[u]);
              }
            }
          }
        }
      }
      const float inv = WT ? 1.0f : (cnt ? 1.0f / (float)cnt : 0.0f);
      const int j0 = c * 16;
      OT* o = out + v * ld + j0;
      if (j0 + 16 <= d) {
        store_scaled<16>(o, acc, inv, vec_ok);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j0 + j < d) store_out(o + j, (j & 1 ? hi2(acc[j / 2]) : lo2(acc[j / 2])) * inv);
      }
    }
  });
}

// ---------------------------------------------------------- VQ (8-bit)
// Thread = (destination, group of G = 32/W parts): one aligned G-byte load of
// the code row per pick, G codebook lookups, G*W/2 FADD2s.
template <int G>
__device__ __forceinline__ void load_codes(const uint8_t* p, uint32_t* w) {
  if constexpr (G == 32) {
    const uint4 a = ldg_stream16(p), b = ldg_stream16(p + 16);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w; w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
  } else if constexpr (G == 16) {
    const uint4 a = ldg_stream16(p);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
  } else if constexpr (G == 8) {
    const uint2 a = ldg_stream8(p);
    w[0] = a.x; w[1] = a.y;
  } else if constexpr (G == 4) {
    w[0] = ldg_stream4(p);
  } else {
    w[0] = __ldg(reinterpret_cast<const uint16_t*>(p));
  }
}

// TT: codebook element type in shared memory.  float = exact fp32 decode;
// __nv_bfloat16 (bf16-output mode only) halves the shared-memory bytes per
// lookup, the kernel's binding resource for VQ; entries are rounded to bf16
// once (<= 2^-9 relative), accumulation stays fp32 (within the 1e-2 bf16
// tolerance of the north star).
template <int W, typename OT, bool SMEM, typename TT, bool WT = false>
__global__ void __launch_bounds__(kThreads, 2)
k_vq_mean8(const uint8_t* __restrict__ rows, int64_t d, int64_t stride,
           const TT* __restrict__ books, int length, int parts,
           const int32_t* __restrict__ indptr, const int32_t* __restrict__ src,
           const int64_t* __restrict__ ndst_dev, int64_t max_dst, OT* __restrict__ out,
           int64_t ld, const float* __restrict__ ew = nullptr) {
  constexpr int G = 32 / W;        // parts per thread
  constexpr int NW = (G + 3) / 4;  // 32-bit code words per load
  constexpr int U = 4;             // picks whose loads are issued together
  __shared__ __align__(8) uint64_t s_mbar;
  extern __shared__ float4 s_mem4[];
  const int64_t nbook = SMEM ? (int64_t)parts * length * W : 0;
  TT* s_book = reinterpret_cast<TT*>(s_mem4);
  const int64_t book_bytes16 = (nbook * (int64_t)sizeof(TT) + 15) & ~15ll;
  int32_t* s_ip0 = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(s_mem4) + book_bytes16);
  int32_t* s_ip1 = s_ip0 + kTD + 1;
  int32_t* s_src0 = s_ip1 + kTD + 1;
  int32_t* s_src1 = s_src0 + kSrcCap;
  const int64_t live = live_dst(ndst_dev, max_dst);
  const int64_t ntiles = (live + kTD - 1) / kTD;
  if ((int64_t)blockIdx.x >= ntiles) return;
  const TT* book = books;
  bool waited = !SMEM;
  if constexpr (SMEM) {
    // codebook -> smem on the TMA engine, overlapping the tile staging
    const uint32_t bytes = (uint32_t)(nbook * sizeof(TT)) & ~15u;
    bulk_fill(s_book, books, bytes, &s_mbar);
    for (int64_t i = bytes / sizeof(TT) + threadIdx.x; i < nbook; i += blockDim.x)
      s_book[i] = books[i];
    book = s_book;
  }
  const int groups = (parts + G - 1) / G;
  const bool vec_ok = (ld % 16) == 0;
  tile_pipeline(indptr, src, max_dst, ntiles, s_ip0, s_ip1, s_src0, s_src1,
                [&](int64_t tile, const int32_t* s_ip, const int32_t* s_src) {
    if (!waited) {
      bulk_wait(&s_mbar);
      waited = true;
    }
    const int64_t v0 = tile * kTD;
    const int32_t e0 = s_ip[0];
    const bool staged = s_ip[kTD] - e0 <= kSrcCap;
    const int items = kTD * groups;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int vl = it / groups;
      const int g = it - vl * groups;
      const int64_t v = v0 + vl;
      if (v >= live) break;
      const int p0 = g * G;
      const int np = min(G, parts - p0);
      u64 acc[G * W / 2];
#pragma unroll
      for (int j = 0; j < G * W / 2; ++j) acc[j] = 0ull;
      const int a = s_ip[vl] - e0;
      const int cnt = s_ip[vl + 1] - e0 - a;
      for (int base = 0; base < cnt; base += U) {
        uint32_t cw[U][NW];
        u64 wt[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (base + u < cnt) {
            const int e = a + base + u;
            const int32_t sid = staged ? s_src[e] : __ldg(src + e0 + e);
            load_codes<G>(rows + (int64_t)sid * stride + p0, cw[u]);
            if constexpr (WT) wt[u] = bcast2(__ldg(ew + e0 + e));
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (base + u < cnt) {
#pragma unroll
            for (int q = 0; q < G; ++q) {
              if (q < np) {
                const uint32_t code = (cw[u][q >> 2] >> (8 * (q & 3))) & 0xFFu;
                const TT* ent = book + ((int64_t)(p0 + q) * length + code) * W;
                if constexpr (!std::is_same<TT, float>::value && W >= 4) {
                  // bf16 entries: W/4 x 8-byte loads, widened to fp32 pairs
#pragma unroll
                  for (int j = 0; j < W; j += 4) {
                    const uint2 h = SMEM ? lds64(ent + j)
                                         : __ldg(reinterpret_cast<const uint2*>(ent + j));
                    acc[(q * W + j) / 2] = acc2<WT>(acc[(q * W + j) / 2], bf16x2_to_f32x2(h.x), wt[u]);
                    acc[(q * W + j) / 2 + 1] =
                        acc2<WT>(acc[(q * W + j) / 2 + 1], bf16x2_to_f32x2(h.y), wt[u]);
                  }
                } else if constexpr (W >= 4) {
#pragma unroll
                  for (int j = 0; j < W; j += 4) {
                    const float4 f = SMEM ? lds128(ent + j)
                                          : __ldg(reinterpret_cast<const float4*>(ent + j));
                    acc[(q * W + j) / 2] = acc2<WT>(acc[(q * W + j) / 2], pack2(f.x, f.y), wt[u]);
                    acc[(q * W + j) / 2 + 1] = acc2<WT>(acc[(q * W + j) / 2 + 1], pack2(f.z, f.w), wt[u]);
                  }
                } else if constexpr (W == 2) {
                  const float2 f = SMEM ? *reinterpret_cast<const float2*>(ent)
                                        : __ldg(reinterpret_cast<const float2*>(ent));
                  acc[q] = acc2<WT>(acc[q], pack2(f.x, f.y), wt[u]);
                } else {  // W == 1: pair adjacent parts
                  const float f = SMEM ? ent[0] : __ldg(ent);
                  acc[q / 2] = acc2<WT>(acc[q / 2], (q & 1) ? pack2(0.f, f) : pack2(f, 0.f), wt[u]);
                }
              }
            }
          }
        }
      }
      const float inv = WT ? 1.0f : (cnt ? 1.0f / (float)cnt : 0.0f);
      const int64_t col0 = (int64_t)p0 * W;
      OT* o = out + v * ld + col0;
      if (np == G && col0 + G * W <= d) {
        store_scaled<G * W>(o, acc, inv, vec_ok);
      } else {
#pragma unroll
        for (int j = 0; j < G * W; ++j)
          if (col0 + j < d && j < np * W)
            store_out(o + j, (j & 1 ? hi2(acc[j / 2]) : lo2(acc[j / 2])) * inv);
      }
    }
  });
  if (!waited) bulk_wait(&s_mbar);  // never leave with a copy in flight
}

// ------------------------------------------ VQ fast path (8-bit, bf16)
// Specialised for the training configuration: 8-bit codes, bf16 output, bf16
// codebooks in smem, W in {4, 8}.  v4 removed the per-lookup branches the
// ncu instruction mix was dominated by (IMAD/LOP3/ISETP/BSSY ~45 %): the pick
// count is dispatched once per item to a fully unrolled body, per-part smem
// base addresses are precomputed, a zero "part" absorbs the lanes of a
// partial last group, and every lookup is BFE + LEA + LDS + widen + FADD2.
// PR (diagnostic builds selected by FG_FUSED_PROBE, tools/fused_bench.py):
// bit 0 = no gather (sources from a 1024-row L2-resident set), bit 1 = no
// decode (codes added as numbers, no shared-memory lookups), bit 2 = no
// store (outputs kept only when impossible) -- to split the kernel's time
// between the random row gather, the codebook decode and the output stream.
template <int W, int G, int C, bool WT = false, int PR = 0>
__device__ __forceinline__ void vq_fast_body(const uint8_t* __restrict__ rows, int64_t stride,
                                             const int32_t* sids, uint32_t base0,
                                             uint32_t pstride, int p0, u64* acc,
                                             const u64* wt = nullptr) {
  constexpr int NB = G;  // code bytes per pick for this thread
  uint32_t cw[C][(NB + 3) / 4];
#pragma unroll
  for (int u = 0; u < C; ++u) load_codes<G>(rows + (int64_t)sids[u] * stride + p0, cw[u]);
#pragma unroll
  for (int u = 0; u < C; ++u) {
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const uint32_t code = (cw[u][q >> 2] >> (8 * (q & 3))) & 0xFFu;
      const uint32_t addr = base0 + q * pstride + code * (uint32_t)(W * 2);
      if constexpr ((PR & 2) != 0) {
        const float fc = (float)code;
        acc[q * (W / 2)] = fadd2(acc[q * (W / 2)], pack2(fc, fc));
      } else if constexpr (W == 4) {
        uint32_t x, y;
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(addr));
        const u64 wu = WT ? wt[u] : 0ull;
        acc[q * 2] = acc2<WT>(acc[q * 2], bf16x2_to_f32x2(x), wu);
        acc[q * 2 + 1] = acc2<WT>(acc[q * 2 + 1], bf16x2_to_f32x2(y), wu);
      } else {  // W == 8
        uint32_t x, y, z, w;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(addr));
        const u64 wu = WT ? wt[u] : 0ull;
        acc[q * 4] = acc2<WT>(acc[q * 4], bf16x2_to_f32x2(x), wu);
        acc[q * 4 + 1] = acc2<WT>(acc[q * 4 + 1], bf16x2_to_f32x2(y), wu);
        acc[q * 4 + 2] = acc2<WT>(acc[q * 4 + 2], bf16x2_to_f32x2(z), wu);
        acc[q * 4 + 3] = acc2<WT>(acc[q * 4 + 3], bf16x2_to_f32x2(w), wu);
      }
    }
  }
}

constexpr int kFastThreads = 256;  // 3 CTAs/SM -> 85 registers: 32 fp32 accumulators fit

template <int W, int G, bool WT = false, int PR = 0>
__global__ void __launch_bounds__(kFastThreads, 3)
k_vq_mean8_fast(const uint8_t* __restrict__ rows, int64_t d, int64_t stride,
                const __nv_bfloat16* __restrict__ books, int length, int parts,
                const int32_t* __restrict__ indptr, const int32_t* __restrict__ src,
                const int64_t* __restrict__ ndst_dev, int64_t max_dst,
                __nv_bfloat16* __restrict__ out, int64_t ld, int slice_parts, int nslices,
                const float* __restrict__ ew = nullptr, int pf = 0) {
  // G parts per thread: G * W = 32 fp32 accumulators.  Part slicing: when
  // the whole bf16 codebook does not fit the smem budget (MAG240M-shape:
  // 96 parts x 256 x 8 = 393 KB), CTA b serves parts [s*SP, s*SP+SP) of
  // every tile with s = b % nslices; the slices of one tile run on
  // neighbouring CTAs at the same time, so a code row's sectors are fetched
  // from DRAM once and the sibling slices hit L2.
  __shared__ __align__(8) uint64_t s_mbar;
  extern __shared__ float4 s_mem4[];
  const int slice = (int)(blockIdx.x % nslices);
  const int part_base = slice * slice_parts;
  const int lparts = min(slice_parts, parts - part_base);  // parts in this slice
  const int zp = (G - parts % G) % G;                      // zero parts after the last
  const int64_t nbook = (int64_t)lparts * length * W;      // bf16 elements
  const int64_t zero_part = (int64_t)zp * length * W;
  __nv_bfloat16* s_book = reinterpret_cast<__nv_bfloat16*>(s_mem4);
  const int64_t book_bytes16 = (((int64_t)slice_parts + zp) * length * W * 2 + 15) & ~15ll;
  int32_t* s_ip0 = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(s_mem4) + book_bytes16);
  int32_t* s_ip1 = s_ip0 + kTD + 1;
  int32_t* s_src0 = s_ip1 + kTD + 1;
  int32_t* s_src1 = s_src0 + kSrcCap;
  const int64_t live = live_dst(ndst_dev, max_dst);
  const int64_t ntiles = (live + kTD - 1) / kTD;
  const int64_t tile0 = blockIdx.x / nslices, tstep = gridDim.x / nslices;
  if (tile0 >= ntiles) return;
  const __nv_bfloat16* gbook = books + (int64_t)part_base * length * W;
  const uint32_t bytes = (uint32_t)(nbook * 2) & ~15u;
  bulk_fill(s_book, gbook, bytes, &s_mbar);
  for (int64_t i = bytes / 2 + threadIdx.x; i < nbook; i += blockDim.x) s_book[i] = gbook[i];
  for (int64_t i = threadIdx.x; i < zero_part; i += blockDim.x)
    s_book[nbook + i] = __float2bfloat16_rn(0.f);
  const uint32_t s_base = smem_addr(s_book);
  const int groups = (lparts + G - 1) / G;
  const bool vec_ok = (ld % 16) == 0;
  bool waited = false;
  tile_pipeline<kFastThreads>(indptr, src, max_dst, ntiles, s_ip0, s_ip1, s_src0, s_src1,
                [&](int64_t tile, const int32_t* s_ip, const int32_t* s_src) {
    if (!waited) {
      bulk_wait(&s_mbar);
      waited = true;
    }
    const int64_t v0 = tile * kTD;
    const int32_t e0 = s_ip[0];
    const bool staged = s_ip[kTD] - e0 <= kSrcCap;
    const int items = kTD * groups;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int vl = it / groups;
      const int g = it - vl * groups;
      const int64_t v = v0 + vl;
      if (v >= live) break;
      const int p0 = g * G;                  // slice-local part
      const int np = min(G, lparts - p0);
      // parts p0 .. p0+G-1; past the last part the table is zero padded
      const uint32_t pstride = (uint32_t)(length * W * 2);
      const uint32_t base0 = s_base + (uint32_t)p0 * pstride;
      const int pg = part_base + p0;         // global part (code byte, column)
      u64 acc[G * W / 2];
#pragma unroll
      for (int j = 0; j < G * W / 2; ++j) acc[j] = 0ull;
      const int a = s_ip[vl] - e0;
      const int cnt = s_ip[vl + 1] - e0 - a;
      for (int base = 0; base < cnt; base += 5) {  // batches of <= 5 picks
        const int cb = min(cnt - base, 5);
        int32_t sids[5];
        u64 wt[5];
        const int32_t* sp = staged ? s_src + a + base : src + e0 + a + base;  // tile-uniform
#pragma unroll
        for (int u = 0; u < 5; ++u)
          if (u < cb) {
            sids[u] = (PR & 1) ? (int32_t)((v * 5 + u) & 1023) : sp[u];
            if constexpr (WT) wt[u] = bcast2(__ldg(ew + e0 + a + base + u));
          }
        switch (cb) {
          case 1: vq_fast_body<W, G, 1, WT, PR>(rows, stride, sids, base0, pstride, pg, acc, wt); break;
          case 2: vq_fast_body<W, G, 2, WT, PR>(rows, stride, sids, base0, pstride, pg, acc, wt); break;
          case 3: vq_fast_body<W, G, 3, WT, PR>(rows, stride, sids, base0, pstride, pg, acc, wt); break;
          case 4: vq_fast_body<W, G, 4, WT, PR>(rows, stride, sids, base0, pstride, pg, acc, wt); break;
          default: vq_fast_body<W, G, 5, WT, PR>(rows, stride, sids, base0, pstride, pg, acc, wt); break;
        }
      }
      const float inv = WT ? 1.0f : (cnt ? 1.0f / (float)cnt : 0.0f);
      const int64_t col0 = (int64_t)pg * W;
      __nv_bfloat16* o = out + v * ld + col0;
      if ((PR & 4) && lo2(acc[0]) != -1234.5f) {
        // diagnostic: no store
      } else if (np == G && col0 + G * W <= d) {
        store_scaled<G * W>(o, acc, inv, vec_ok);
      } else {
#pragma unroll
        for (int j = 0; j < G * W; ++j)
          if (col0 + j < d) o[j] = __float2bfloat16_rn((j & 1 ? hi2(acc[j / 2]) : lo2(acc[j / 2])) * inv);
      }
    }
  }, tile0, tstep, pf ? rows + part_base : nullptr, stride);
  if (!waited) bulk_wait(&s_mbar);
}

// --------------------------------- VQ lane-per-part path (8-bit, bf16)
// v5 (round 2), for codebooks too large for one SM (MAG240M-shape: 96 parts x
// 256 x 8 bf16 = 393 KB).  The v4 kernel sliced parts 6 ways with 16 parts
// (16 B) per slice, so every slice CTA re-read its 16 B out of the row's
// 32-B sectors (ncu: DRAM read 2x the algorithmic bytes) and its random
// 16-B codebook lookups from 8 bank groups conflicted (~7.5 wavefronts per
// warp-wide lookup instead of 4).  Here:
//  * a slice is one 32-B SECTOR of the code row = 32 parts; CTA b serves
//    slice b % nslices of every tile, so each sector is read from DRAM by
//    exactly one CTA and no slice depends on L2 coincidences;
//  * a warp handles one destination at a time, lane = part: the pick's code
//    byte comes from a shared-memory copy of its sector and the lane's
//    lookup hits its own bank group -- part p's entries live at byte offset
//    (p % PPL) * EB of 128-B lines (PPL = 128 / EB parts per line), so the 8
//    (W = 8) or 16 (W = 4) lanes of one wavefront never share a bank:
//    the minimum 4 (2) wavefronts per warp lookup;
//  * the warp's bf16 output row segment (512 B for W = 8) is one coalesced
//    store per destination;
//  * cp.async pipeline over tiles of kTD destinations, one CTA per SM:
//    indptr slices 3 tiles ahead, source ids 2 ahead, code sectors 1 ahead
//    (smem rings of 4 / 3 / 2), so the random sector gathers of tile t+1
//    are in flight while tile t decodes; the codebook slice is filled by
//    per-entry cp.async into the interleaved layout.
// fp16x2 helpers (scaled fp16 codebooks, fg_codec_desc.table_h)
__device__ __forceinline__ uint32_t hadd2u(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ u64 h2_to_f32x2(uint32_t h) {
  float lo, hi;
  asm("{ .reg .b16 a, b; mov.b32 {a, b}, %2; cvt.f32.f16 %0, a; cvt.f32.f16 %1, b; }"
      : "=f"(lo), "=f"(hi) : "r"(h));
  return pack2(lo, hi);
}
constexpr int kLaneThreads = 1024;
constexpr int kLaneWarps = kLaneThreads / 32;

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// cp.async the indptr slice of `tile` (entries clamped at max_dst)
__device__ __forceinline__ void lane_issue_ip(int32_t* dst, const int32_t* __restrict__ indptr,
                                              int64_t tile, int64_t max_dst) {
  for (int t = threadIdx.x; t <= kTD; t += blockDim.x)
    cp_async4(dst + t, indptr + min64(tile * kTD + t, max_dst));
}
// cp.async the source ids of a tile whose indptr slice is in smem
__device__ __forceinline__ void lane_issue_src(int32_t* dst, const int32_t* s_ip,
                                               const int32_t* __restrict__ src) {
  const int32_t e0 = s_ip[0], cnt = s_ip[kTD] - e0;
  if (cnt > kSrcCap) return;  // compute reads them from global
  for (int t = threadIdx.x; t < cnt; t += blockDim.x) cp_async4(dst + t, src + e0 + t);
}
// cp.async the slice's 32-B code sector of every pick of a tile whose source
// ids are in smem (two 16-B copies per pick)
__device__ __forceinline__ void lane_issue_codes(uint8_t* dst, const int32_t* s_ip,
                                                 const int32_t* s_src,
                                                 const uint8_t* __restrict__ rows,
                                                 int64_t stride, int sector_off) {
  const int32_t cnt = s_ip[kTD] - s_ip[0];
  if (cnt > kSrcCap) return;
  for (int t = threadIdx.x; t < 2 * cnt; t += blockDim.x) {
    const int e = t >> 1, h = t & 1;
    cp_async16(dst + e * 32 + h * 16,
               rows + (int64_t)s_src[e] * stride + sector_off + h * 16);
  }
}

// fp16 lane body, C staged picks (compile-time count: no per-pick
// predication): C code bytes (lane-contiguous), C conflict-free 16/8-byte
// lookups, W/2 HADD2 each.  ncu of the generic loop: 84.5 M instructions for
// a MAG240M-shape launch, 71 % issue -- the per-destination predication and
// staged/global selects, not the lookups, were the cost.
template <int C, int W>
__device__ __forceinline__ void lane_f16_body(const uint8_t* cp, uint32_t lbase, uint32_t* h) {
  uint32_t code[C];
#pragma unroll
  for (int u = 0; u < C; ++u) code[u] = cp[u * 32];
#pragma unroll
  for (int u = 0; u < C; ++u) {  // the first pick initialises the sums
    const uint32_t addr = lbase + code[u] * 128u;
    if constexpr (W == 8) {
      uint32_t x, y, z, w;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(addr));
      if (u == 0) {
        h[0] = x; h[1] = y; h[2] = z; h[3] = w;
      } else {
        h[0] = hadd2u(h[0], x); h[1] = hadd2u(h[1], y);
        h[2] = hadd2u(h[2], z); h[3] = hadd2u(h[3], w);
      }
    } else {
      uint32_t x, y;
      asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(addr));
      if (u == 0) {
        h[0] = x; h[1] = y;
      } else {
        h[0] = hadd2u(h[0], x); h[1] = hadd2u(h[1], y);
      }
    }
  }
}
// 1/cnt for the <= 8-pick fast path (cnt = 0 -> 0)
__constant__ float kInvCnt[9] = {0.f, 1.f, 1.f / 2, 1.f / 3, 1.f / 4, 1.f / 5, 1.f / 6, 1.f / 7,
                                 1.f / 8};
template <int W>
__device__ __forceinline__ void lane_f16_chunk(const uint8_t* cp, int cb, uint32_t lbase,
                                               uint32_t* h) {
  if (cb == 5) {  // the fanout-5 input layer of every BASELINE config: one compare
    lane_f16_body<5, W>(cp, lbase, h);
    return;
  }
  switch (cb) {
    case 1: lane_f16_body<1, W>(cp, lbase, h); break;
    case 2: lane_f16_body<2, W>(cp, lbase, h); break;
    case 3: lane_f16_body<3, W>(cp, lbase, h); break;
    case 4: lane_f16_body<4, W>(cp, lbase, h); break;
    case 5: lane_f16_body<5, W>(cp, lbase, h); break;
    case 6: lane_f16_body<6, W>(cp, lbase, h); break;
    case 7: lane_f16_body<7, W>(cp, lbase, h); break;
    default: lane_f16_body<8, W>(cp, lbase, h); break;
  }
}

template <int W, bool WT, bool F16 = false, int NT = kLaneThreads>
__global__ void __launch_bounds__(NT, 1)
k_vq_mean8_lane(const uint8_t* __restrict__ rows, int64_t d, int64_t stride,
                const __nv_bfloat16* __restrict__ books, int length, int parts,
                const int32_t* __restrict__ indptr, const int32_t* __restrict__ src,
                const int64_t* __restrict__ ndst_dev, int64_t max_dst,
                __nv_bfloat16* __restrict__ out, int64_t ld, int nslices,
                const float* __restrict__ ew, const float* __restrict__ part_scale = nullptr) {
  constexpr int EB = W * 2;        // bytes per bf16 entry
  constexpr int PPL = 128 / EB;    // parts per 128-B line
  extern __shared__ __align__(128) uint8_t s_raw[];
  const int slice = (int)(blockIdx.x % nslices);
  const int64_t live = live_dst(ndst_dev, max_dst);
  const int64_t ntiles = (live + kTD - 1) / kTD;
  const int64_t tile0 = blockIdx.x / nslices, tstep = gridDim.x / nslices;
  if (tile0 >= ntiles) return;
  const int lparts = min(32, parts - slice * 32);
  // smem: codebook slice | 2 x code sectors | 3 x source ids | 4 x indptr
  uint8_t* const s_book = s_raw;
  uint8_t* const s_codes0 = s_book + (size_t)(32 / PPL) * length * 128;
  int32_t* const s_src0 = reinterpret_cast<int32_t*>(s_codes0 + 2 * kSrcCap * 32);
  int32_t* const s_ip0 = s_src0 + 3 * kSrcCap;
  auto IP = [&](int i) { return s_ip0 + i * (kTD + 4); };
  auto SRC = [&](int i) { return s_src0 + i * kSrcCap; };
  auto CODES = [&](int i) { return s_codes0 + i * (kSrcCap * 32); };
  // codebook slice -> interleaved smem lines (group 0, with the first tile's indptr)
  {
    const int nent = lparts * length;
    const __nv_bfloat16* g = books + (int64_t)slice * 32 * length * W;
    for (int c = threadIdx.x; c < nent; c += blockDim.x) {
      const int lp = c / length, e = c - lp * length;
      uint8_t* dst = s_book + ((lp / PPL) * length + e) * 128 + (lp % PPL) * EB;
      if constexpr (EB == 16) cp_async16(dst, g + (int64_t)c * W);
      else cp_async8(dst, g + (int64_t)c * W);
    }
  }
  const int sector_off = slice * 32;
  // prologue: ip(T0) | src(T0), ip(T1) | codes(T0), src(T1), ip(T2)
  lane_issue_ip(IP(0), indptr, tile0, max_dst);
  cp_commit();
  cp_wait_all();
  __syncthreads();
  lane_issue_src(SRC(0), IP(0), src);
  if (tile0 + tstep < ntiles) lane_issue_ip(IP(1), indptr, tile0 + tstep, max_dst);
  cp_commit();
  cp_wait_all();
  __syncthreads();
  lane_issue_codes(CODES(0), IP(0), SRC(0), rows, stride, sector_off);
  if (tile0 + tstep < ntiles) lane_issue_src(SRC(1), IP(1), src);
  if (tile0 + 2 * tstep < ntiles) lane_issue_ip(IP(2), indptr, tile0 + 2 * tstep, max_dst);
  cp_commit();
  cp_wait_all();
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool active = lane < lparts;
  const uint32_t lbase = smem_addr(s_book) + (uint32_t)((lane / PPL) * length * 128 +
                                                         (lane % PPL) * EB);
  const int64_t col0 = (int64_t)(slice * 32 + lane) * W;
  const bool full_part = col0 + W <= d;
  const bool vec_ok = (ld % 8) == 0;  // 16-B aligned bf16 row segments
  const float pscale = (F16 && active) ? __ldg(part_scale + slice * 32 + lane) : 1.0f;
  int k = 0;
  for (int64_t tile = tile0; tile < ntiles; tile += tstep, ++k) {
    // issue: codes(T_{k+1}), src(T_{k+2}), ip(T_{k+3})
    const int64_t t1 = tile + tstep, t2 = tile + 2 * tstep, t3 = tile + 3 * tstep;
    if (t1 < ntiles)
      lane_issue_codes(CODES((k + 1) & 1), IP((k + 1) & 3), SRC((k + 1) % 3), rows, stride,
                       sector_off);
    if (t2 < ntiles) lane_issue_src(SRC((k + 2) % 3), IP((k + 2) & 3), src);
    if (t3 < ntiles) lane_issue_ip(IP((k + 3) & 3), indptr, t3, max_dst);
    cp_commit();
    // compute tile T_k
    const int32_t* s_ip = IP(k & 3);
    const uint8_t* s_codes = CODES(k & 1);
    const int32_t e0 = s_ip[0];
    const bool staged = s_ip[kTD] - e0 <= kSrcCap;
    const int nv = (int)min64((int64_t)kTD, live - tile * kTD);  // live destinations of the tile
    for (int vl = warp; vl < nv; vl += (NT / 32)) {
      const int64_t v = tile * kTD + vl;
      const int a = s_ip[vl] - e0;
      const int cnt = s_ip[vl + 1] - e0 - a;
      if constexpr (F16 && W == 8 && NT > 512) {
        // fanout-5 input layer (every BASELINE config; 99.5 % of a MAG240M-
        // shape block's destinations): straight to the 5-pick body, no
        // dispatch, the first pick initialises the sums, constant 1/cnt
        if (staged && cnt == 5) {
          uint32_t h[W / 2];
          lane_f16_body<5, W>(s_codes + a * 32 + lane, lbase, h);
          if (active) {
            const float inv = 0.2f * pscale;
            uint32_t wv[W / 2];
#pragma unroll
            for (int j = 0; j < W / 2; ++j) {
              const u64 f = h2_to_f32x2(h[j]);
              const __nv_bfloat162 b2 = __floats2bfloat162_rn(lo2(f) * inv, hi2(f) * inv);
              wv[j] = *reinterpret_cast<const uint32_t*>(&b2);
            }
            __nv_bfloat16* o = out + v * ld + col0;
            if (full_part && vec_ok) {
              *reinterpret_cast<uint4*>(o) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
            } else {
#pragma unroll
              for (int j = 0; j < W; ++j)
                if (col0 + j < d)
                  o[j] = __ushort_as_bfloat16((unsigned short)(wv[j / 2] >> (16 * (j & 1))));
            }
          }
          continue;
        }
      }
      if constexpr (F16) {
        // bf16 row segment of destination vv from its fp16 sums
        auto emit = [&](int64_t vv, const uint32_t* h, float inv) {
          if (!active) return;
          uint32_t wv[W / 2];
#pragma unroll
          for (int j = 0; j < W / 2; ++j) {
            const u64 f = h2_to_f32x2(h[j]);
            const __nv_bfloat162 b2 = __floats2bfloat162_rn(lo2(f) * inv, hi2(f) * inv);
            wv[j] = *reinterpret_cast<const uint32_t*>(&b2);
          }
          __nv_bfloat16* o = out + vv * ld + col0;
          if (full_part && vec_ok) {
            if constexpr (W == 8)
              *reinterpret_cast<uint4*>(o) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
            else
              *reinterpret_cast<uint2*>(o) = make_uint2(wv[0], wv[1]);
          } else {
#pragma unroll
            for (int j = 0; j < W; ++j)
              if (col0 + j < d)
                o[j] = __ushort_as_bfloat16((unsigned short)(wv[j / 2] >> (16 * (j & 1))));
          }
        };
        // two 5-pick destinations of this warp (vl, vl + 32) in one pass:
        // the loop / dispatch / bookkeeping is shared, the bodies interleave.
        // W = 4, or any W at 512 threads (112 registers): products-shape
        // 30.9 -> 29.8 us; at W = 8 and 64 registers the doubled live
        // registers cost more than they save (MAG 74.1 -> 79.2 us).
        const int vl2 = vl + (NT / 32);
        if ((W == 4 || NT <= 512) && staged && cnt == 5 && vl2 < kTD && v + (NT / 32) < live) {
          const int a2 = s_ip[vl2] - e0;
          if (s_ip[vl2 + 1] - e0 - a2 == 5) {
            uint32_t h[W / 2], h2[W / 2];
            lane_f16_body<5, W>(s_codes + a * 32 + lane, lbase, h);
            lane_f16_body<5, W>(s_codes + a2 * 32 + lane, lbase, h2);
            const float inv = 0.2f * pscale;
            emit(v, h, inv);
            emit(v + (NT / 32), h2, inv);
            vl = vl2;  // the loop step moves past the partner
            continue;
          }
        }
        if (staged && cnt <= 8) {  // one HADD2 chunk, no fp32 pass
          uint32_t h[W / 2];
#pragma unroll
          for (int j = 0; j < W / 2; ++j) h[j] = 0u;
          if (cnt) lane_f16_chunk<W>(s_codes + a * 32 + lane, cnt, lbase, h);
          emit(v, h, kInvCnt[cnt] * pscale);
          continue;
        }
      }
      u64 acc[W / 2];
#pragma unroll
      for (int j = 0; j < W / 2; ++j) acc[j] = 0ull;
      for (int u0 = 0; u0 < cnt; u0 += 8) {
        const int cb = min(cnt - u0, 8);
        uint32_t code[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (u < cb) {
            const int e = a + u0 + u;
            code[u] = staged ? (uint32_t)s_codes[e * 32 + lane]
                             : (uint32_t)__ldg(rows + (int64_t)__ldg(src + e0 + e) * stride +
                                               sector_off + lane);
          }
        }
        if constexpr (F16) {  // fp16 entries, HADD2 over <= 8 picks, then fp32
          uint32_t h[W / 2];
#pragma unroll
          for (int j = 0; j < W / 2; ++j) h[j] = 0u;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (u < cb) {
              const uint32_t addr = lbase + code[u] * 128u;
              if constexpr (W == 8) {
                uint32_t x, y, z, w;
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(addr));
                h[0] = hadd2u(h[0], x); h[1] = hadd2u(h[1], y);
                h[2] = hadd2u(h[2], z); h[3] = hadd2u(h[3], w);
              } else {
                uint32_t x, y;
                asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(addr));
                h[0] = hadd2u(h[0], x); h[1] = hadd2u(h[1], y);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < W / 2; ++j) acc[j] = fadd2(acc[j], h2_to_f32x2(h[j]));
        } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (u < cb) {
            const uint32_t addr = lbase + code[u] * 128u;
            const u64 wu = WT ? bcast2(__ldg(ew + e0 + a + u0 + u)) : 0ull;
            if constexpr (W == 8) {
              uint32_t x, y, z, w;
              asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(addr));
              acc[0] = acc2<WT>(acc[0], bf16x2_to_f32x2(x), wu);
              acc[1] = acc2<WT>(acc[1], bf16x2_to_f32x2(y), wu);
              acc[2] = acc2<WT>(acc[2], bf16x2_to_f32x2(z), wu);
              acc[3] = acc2<WT>(acc[3], bf16x2_to_f32x2(w), wu);
            } else {
              uint32_t x, y;
              asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(addr));
              acc[0] = acc2<WT>(acc[0], bf16x2_to_f32x2(x), wu);
              acc[1] = acc2<WT>(acc[1], bf16x2_to_f32x2(y), wu);
            }
          }
        }
        }
      }
      if (active) {
        const float inv = (WT ? 1.0f : (cnt ? 1.0f / (float)cnt : 0.0f)) * pscale;
        __nv_bfloat16* o = out + v * ld + col0;
        if (full_part) {
          store_scaled<W>(o, acc, inv, vec_ok);
        } else {
#pragma unroll
          for (int j = 0; j < W; ++j)
            if (col0 + j < d)
              o[j] = __float2bfloat16_rn((j & 1 ? hi2(acc[j / 2]) : lo2(acc[j / 2])) * inv);
        }
      }
    }
    cp_wait_all();
    __syncthreads();
  }
}

// ------------------------------------ SQ lane-per-byte-group path (k in {4, 8}, bf16)
// Round 2, the lane kernel's structure for SQ rows whose code bytes are a
// multiple of 32 (papers100M-shape k=4 d=128: 64 B; arxiv-shape k=8 d=128:
// 128 B): a warp takes one destination at a time, lane l owns code bytes
// [l*NB, l*NB + NB) and the 8*NB/k outputs they decode to; whole code rows
// are staged one tile ahead by per-thread 16-byte cp.async (no TMA unit in
// the row path), the decode table is replicated per lane (k=4: decoded byte
// PAIRS, 8 B; k=8: 4 B: conflict-free), pick counts up to 8 run unpredicated
// bodies, and the destination's row is one coalesced store.
template <int RB>
__device__ __forceinline__ void sq_lane_issue_rows(uint8_t* dst, const int32_t* s_ip,
                                                   const int32_t* s_src,
                                                   const uint8_t* __restrict__ rows,
                                                   int64_t stride, int cap) {
  constexpr int CH = RB / 16;
  const int32_t cnt = s_ip[kTD] - s_ip[0];
  if (cnt > cap) return;
  for (int t = threadIdx.x; t < CH * cnt; t += blockDim.x) {
    const int e = t / CH, h = t - e * CH;
    cp_async16(dst + e * RB + h * 16, rows + (int64_t)s_src[e] * stride + h * 16);
  }
}

template <int K, int NB, int C>
__device__ __forceinline__ void sq_lane_body(const uint8_t* cp, uint32_t tb, u64* acc) {
  constexpr int RB = 32 * NB;
  uint32_t cw[C];
#pragma unroll
  for (int u = 0; u < C; ++u) {
    if constexpr (NB == 4) cw[u] = *reinterpret_cast<const uint32_t*>(cp + u * RB);
    else if constexpr (NB == 2) cw[u] = *reinterpret_cast<const uint16_t*>(cp + u * RB);
    else cw[u] = cp[u * RB];
  }
#pragma unroll
  for (int u = 0; u < C; ++u) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const uint32_t byte = (cw[u] >> (8 * b)) & 0xFFu;
      if constexpr (K == 4) {
        uint32_t x, y;
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(tb + byte * 256u));
        acc[b] = fadd2(acc[b], ((u64)y << 32) | x);
      } else if (b % 2 == 0) {
        const uint32_t b1 = (cw[u] >> (8 * (b + 1))) & 0xFFu;
        float f0, f1;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(f0) : "r"(tb + byte * 128u));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(f1) : "r"(tb + b1 * 128u));
        acc[b / 2] = fadd2(acc[b / 2], pack2(f0, f1));
      }
    }
  }
}

template <int K, int NB>
__global__ void __launch_bounds__(kLaneThreads, 1)
k_sq_mean_lane(const uint8_t* __restrict__ rows, int64_t stride, const float* __restrict__ lut,
               const int32_t* __restrict__ indptr, const int32_t* __restrict__ src,
               const int64_t* __restrict__ ndst_dev, int64_t max_dst,
               __nv_bfloat16* __restrict__ out, int64_t ld, int cap) {
  constexpr int RB = 32 * NB;        // code bytes per row
  constexpr int EPL = 8 * NB / K;    // outputs per lane
  constexpr int NA = EPL / 2;
  constexpr bool PAIR = K == 4;
  constexpr int LUTB = PAIR ? 256 * 32 * 8 : 256 * 32 * 4;
  extern __shared__ __align__(128) uint8_t s_raw[];
  const int64_t live = live_dst(ndst_dev, max_dst);
  const int64_t ntiles = (live + kTD - 1) / kTD;
  const int64_t tile0 = blockIdx.x, tstep = gridDim.x;
  if (tile0 >= ntiles) return;
  uint8_t* const s_lut = s_raw;
  uint8_t* const s_rows0 = s_raw + LUTB;                                  // [2][cap][RB]
  int32_t* const s_src0 = reinterpret_cast<int32_t*>(s_rows0 + 2 * (size_t)cap * RB);  // [3][cap]
  int32_t* const s_ip0 = s_src0 + 3 * cap;                                // [4][kTD + 4]
  auto IP = [&](int i) { return s_ip0 + i * (kTD + 4); };
  auto SRC = [&](int i) { return s_src0 + i * cap; };
  auto ROWS = [&](int i) { return s_rows0 + (size_t)i * cap * RB; };
  if constexpr (PAIR) {
    u64* t2 = reinterpret_cast<u64*>(s_lut);
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
      const int pv = i >> 5;
      t2[i] = pack2(__ldg(lut + (pv >> 4)), __ldg(lut + (pv & 15)));
    }
  } else {
    float* t1 = reinterpret_cast<float*>(s_lut);
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) t1[i] = __ldg(lut + (i >> 5));
  }
  auto issue_src = [&](int32_t* dst, const int32_t* ip) {
    const int32_t e0 = ip[0], c = ip[kTD] - e0;
    if (c > cap) return;
    for (int t = threadIdx.x; t < c; t += blockDim.x) cp_async4(dst + t, src + e0 + t);
  };
  lane_issue_ip(IP(0), indptr, tile0, max_dst);
  cp_commit();
  cp_wait_all();
  __syncthreads();
  issue_src(SRC(0), IP(0));
  if (tile0 + tstep < ntiles) lane_issue_ip(IP(1), indptr, tile0 + tstep, max_dst);
  cp_commit();
  cp_wait_all();
  __syncthreads();
  sq_lane_issue_rows<RB>(ROWS(0), IP(0), SRC(0), rows, stride, cap);
  if (tile0 + tstep < ntiles) issue_src(SRC(1), IP(1));
  if (tile0 + 2 * tstep < ntiles) lane_issue_ip(IP(2), indptr, tile0 + 2 * tstep, max_dst);
  cp_commit();
  cp_wait_all();
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t tb = smem_addr(s_lut) + (uint32_t)lane * (PAIR ? 8u : 4u);
  const bool vec_ok = (ld % 4) == 0;
  int k = 0;
  for (int64_t tile = tile0; tile < ntiles; tile += tstep, ++k) {
    const int64_t t1 = tile + tstep, t2 = tile + 2 * tstep, t3 = tile + 3 * tstep;
    if (t1 < ntiles) sq_lane_issue_rows<RB>(ROWS((k + 1) & 1), IP((k + 1) & 3), SRC((k + 1) % 3),
                                            rows, stride, cap);
    if (t2 < ntiles) issue_src(SRC((k + 2) % 3), IP((k + 2) & 3));
    if (t3 < ntiles) lane_issue_ip(IP((k + 3) & 3), indptr, t3, max_dst);
    cp_commit();
    const int32_t* s_ip = IP(k & 3);
    const uint8_t* s_rw = ROWS(k & 1);
    const int32_t e0 = s_ip[0];
    const bool staged = s_ip[kTD] - e0 <= cap;
    const int nv = (int)min64((int64_t)kTD, live - tile * kTD);  // live destinations of the tile
    for (int vl = warp; vl < nv; vl += kLaneWarps) {
      const int64_t v = tile * kTD + vl;
      const int a = s_ip[vl] - e0;
      const int cnt = s_ip[vl + 1] - e0 - a;
      u64 acc[NA];
#pragma unroll
      for (int j = 0; j < NA; ++j) acc[j] = 0ull;
      if (staged && cnt == 5) {  // fanout-5 input layer: no dispatch
        sq_lane_body<K, NB, 5>(s_rw + (size_t)a * RB + lane * NB, tb, acc);
      } else if (staged) {
        const uint8_t* cp = s_rw + (size_t)a * RB + lane * NB;
        int u0 = 0;
        for (; u0 + 8 <= cnt; u0 += 8) sq_lane_body<K, NB, 8>(cp + (size_t)u0 * RB, tb, acc);
        switch (cnt - u0) {
          case 1: sq_lane_body<K, NB, 1>(cp + (size_t)u0 * RB, tb, acc); break;
          case 2: sq_lane_body<K, NB, 2>(cp + (size_t)u0 * RB, tb, acc); break;
          case 3: sq_lane_body<K, NB, 3>(cp + (size_t)u0 * RB, tb, acc); break;
          case 4: sq_lane_body<K, NB, 4>(cp + (size_t)u0 * RB, tb, acc); break;
          case 5: sq_lane_body<K, NB, 5>(cp + (size_t)u0 * RB, tb, acc); break;
          case 6: sq_lane_body<K, NB, 6>(cp + (size_t)u0 * RB, tb, acc); break;
          case 7: sq_lane_body<K, NB, 7>(cp + (size_t)u0 * RB, tb, acc); break;
          default: break;
        }
      } else {  // tile larger than the staging buffer: codes from global
        for (int u = 0; u < cnt; ++u) {
          const uint8_t* rp = rows + (int64_t)__ldg(src + e0 + a + u) * stride + lane * NB;
          uint32_t tw = 0;
#pragma unroll
          for (int b = 0; b < NB; ++b) tw |= (uint32_t)__ldg(rp + b) << (8 * b);
          sq_lane_body<K, NB, 1>(reinterpret_cast<const uint8_t*>(&tw), tb, acc);
        }
      }
      const float inv = cnt ? (cnt <= 8 ? kInvCnt[cnt] : 1.0f / (float)cnt) : 0.0f;
      uint32_t w[NA];
#pragma unroll
      for (int j = 0; j < NA; ++j) {
        const __nv_bfloat162 b2 = __floats2bfloat162_rn(lo2(acc[j]) * inv, hi2(acc[j]) * inv);
        w[j] = *reinterpret_cast<const uint32_t*>(&b2);
      }
      __nv_bfloat16* o = out + v * ld + lane * EPL;
      if (vec_ok) {
        if constexpr (NA == 2) *reinterpret_cast<uint2*>(o) = make_uint2(w[0], w[1]);
        else if constexpr (NA == 4) *reinterpret_cast<uint4*>(o) = make_uint4(w[0], w[1], w[2], w[3]);
        else *reinterpret_cast<uint32_t*>(o) = w[0];
      } else {
#pragma unroll
        for (int j = 0; j < NA; ++j) {
          o[2 * j] = __ushort_as_bfloat16((unsigned short)(w[j] & 0xFFFFu));
          o[2 * j + 1] = __ushort_as_bfloat16((unsigned short)(w[j] >> 16));
        }
      }
    }
    cp_wait_all();
    __syncthreads();
  }
}

// SQ lane launch for bf16 output, mean, k in {4, 8}, d*k/8 a multiple of 32;
// false when not covered (FG_SQ_LANE=0 also disables it)
template <bool WT>
static bool launch_sq_lane(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                           const int64_t* ndst, int64_t max_dst, void* out, int64_t ld,
                           cudaStream_t st, int* rc) {
  if constexpr (WT) {
    return false;
  } else {
    static const int env = [] {
      const char* e = getenv("FG_SQ_LANE");
      return e ? atoi(e) : 1;
    }();
    const int K = c->bits;
    if (!env || !(K == 4 || K == 8) || (c->d * K) % 256 != 0 || c->elem_bits != 32) return false;
    const int RB = (int)(c->d * K / 8), NB = RB / 32;
    if (!(NB == 2 || NB == 4) || c->row_stride < RB || c->row_stride % 16 != 0) return false;
    const int lutb = K == 4 ? 256 * 32 * 8 : 256 * 32 * 4;
    const int tail = 4 * (kTD + 4) * 4;
    int cap = kSrcCap;
    while (cap > kTD && lutb + 2 * (int64_t)cap * RB + 3 * (int64_t)cap * 4 + tail > 220 * 1024)
      cap -= kTD;
    const int64_t smem = lutb + 2 * (int64_t)cap * RB + 3 * (int64_t)cap * 4 + tail;
    void (*kern)(const uint8_t*, int64_t, const float*, const int32_t*, const int32_t*,
                 const int64_t*, int64_t, __nv_bfloat16*, int64_t, int) =
        K == 4 ? (NB == 2 ? k_sq_mean_lane<4, 2> : k_sq_mean_lane<4, 4>)
               : (NB == 2 ? k_sq_mean_lane<8, 2> : k_sq_mean_lane<8, 4>);
    *rc = FG_OK;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
    if (err != cudaSuccess) {
      set_error("sq lane smem attribute: %s", cudaGetErrorString(err));
      *rc = FG_ECUDA;
      return true;
    }
    const int grid = (int)min64(ceil_div(max_dst, kTD), (int64_t)sm_count());
    kern<<<grid, kLaneThreads, smem, st>>>(c->rows, c->row_stride, (const float*)c->table, indptr,
                                           src, ndst, max_dst, (__nv_bfloat16*)out, ld, cap);
    count_launch();
    err = cudaGetLastError();
    if (err != cudaSuccess) {
      set_error("k_sq_mean_lane launch: %s", cudaGetErrorString(err));
      *rc = FG_ECUDA;
    }
    return true;
  }
}

// ------------------------------------------------- VQ (any code width)
template <int W, typename OT>
__global__ void __launch_bounds__(kThreads, 2)
k_vq_mean_bits(const uint8_t* __restrict__ rows, int64_t d, int64_t stride, int bits,
               const float* __restrict__ books, int length, int parts,
               const int32_t* __restrict__ indptr, const int32_t* __restrict__ src,
               const int64_t* __restrict__ ndst_dev, int64_t max_dst, OT* __restrict__ out,
               int64_t ld, const float* __restrict__ ew) {
  extern __shared__ int32_t s_stage[];
  int32_t* s_ip0 = s_stage;
  int32_t* s_ip1 = s_ip0 + kTD + 1;
  int32_t* s_src0 = s_ip1 + kTD + 1;
  int32_t* s_src1 = s_src0 + kSrcCap;
  const int64_t live = live_dst(ndst_dev, max_dst);
  const int64_t ntiles = (live + kTD - 1) / kTD;
  if ((int64_t)blockIdx.x >= ntiles) return;
  const uint32_t cmask = (1u << bits) - 1u;
  tile_pipeline(indptr, src, max_dst, ntiles, s_ip0, s_ip1, s_src0, s_src1,
                [&](int64_t tile, const int32_t* s_ip, const int32_t* s_src) {
    const int64_t v0 = tile * kTD;
    const int32_t e0 = s_ip[0];
    const bool staged = s_ip[kTD] - e0 <= kSrcCap;
    const int items = kTD * parts;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int vl = it / parts;
      const int p = it - vl * parts;
      const int64_t v = v0 + vl;
      if (v >= live) break;
      float acc[W];
#pragma unroll
      for (int j = 0; j < W; ++j) acc[j] = 0.f;
      const int a = s_ip[vl] - e0;
      const int cnt = s_ip[vl + 1] - e0 - a;
      const int64_t bit0 = (int64_t)p * bits;
      const int sh = (int)(bit0 & 7);
      for (int k = 0; k < cnt; ++k) {
        const int32_t sid = staged ? s_src[a + k] : __ldg(src + e0 + a + k);
        const uint8_t* rb = rows + (int64_t)sid * stride + (bit0 >> 3);
        uint32_t wv = (uint32_t)__ldg(rb) << 16;
        if (sh + bits > 8) wv |= (uint32_t)__ldg(rb + 1) << 8;
        if (sh + bits > 16) wv |= __ldg(rb + 2);
        const uint32_t code = (wv >> (24 - sh - bits)) & cmask;
        const float* ent = books + ((int64_t)p * length + code) * W;
        if (ew) {
          const float we = __ldg(ew + e0 + a + k);
#pragma unroll
          for (int j = 0; j < W; ++j) acc[j] = fmaf(we, __ldg(ent + j), acc[j]);
        } else {
#pragma unroll
          for (int j = 0; j < W; ++j) acc[j] += __ldg(ent + j);
        }
      }
      const float inv = ew ? 1.0f : (cnt ? 1.0f / (float)cnt : 0.0f);
      OT* o = out + v * ld + (int64_t)p * W;
#pragma unroll
      for (int j = 0; j < W; ++j)
        if ((int64_t)p * W + j < d) store_out(o + j, acc[j] * inv);
    }
  });
}

// ----------------------------------------- SQ mean, TMA row staging
// k_sq_mean spends most of its time waiting on its own row loads (ncu: long
// scoreboard stalls, DRAM 17 % busy): each thread has only `fanout` 8-byte
// loads in flight and issues them in bursts between compute phases.  Here the
// code rows of the NEXT tile are copied into shared memory by cp.async.bulk
// (one TMA copy per sampled edge, completing on a per-buffer mbarrier) while
// the current tile is decoded from shared memory, so the HBM gather runs in
// the background and needs no registers.  (Measured on papers100M-shape,
// k=4, 64 B rows: 38 us vs 41 us for the register kernel and 45 us for a
// per-thread 16 B LDGSTS variant; cp.async.bulk operands are warp-uniform,
// so per-lane rows issue through a 32-step ELECT loop.)  Pipeline depth per
// persistent CTA: indptr slices 3 tiles ahead (4-slot smem ring), src ids 2 ahead
// (registers), code rows 1 ahead (2 smem buffers).  A tile whose edges
// exceed the row buffer falls back to direct register loads.
constexpr int kBulkThreads = 512;
constexpr int kBulkRowCap = 1024;                          // rows per buffer, max
constexpr int kBulkSidPer = 4;  // src ids per thread (kBulkRowCap / kBulkThreads, or one gather4)
static_assert(kBulkSidPer * kBulkThreads >= kBulkRowCap, "row staging capacity");

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  const uint32_t mb = smem_addr(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(mb), "r"(parity) : "memory");
  }
}

// one 2K-byte chunk of 16 codes from shared memory (byte 0 in the low bits)
template <int K>
__device__ __forceinline__ void lds_chunk(const uint8_t* p, uint64_t& w0, uint64_t& w1) {
  constexpr int CB = 2 * K;
  const uint32_t a = smem_addr(p);
  w0 = w1 = 0;
  if constexpr (CB == 16) {
    uint32_t x, y, z, w;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a));
    w0 = ((uint64_t)y << 32) | x;
    w1 = ((uint64_t)w << 32) | z;
  } else if constexpr (CB == 8) {
    uint32_t x, y;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
    w0 = ((uint64_t)y << 32) | x;
  } else if constexpr (CB == 4) {
    uint32_t x;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x) : "r"(a));
    w0 = x;
  } else {  // CB even: 2-byte aligned halves
#pragma unroll
    for (int b = 0; b < CB; b += 2) {
      uint16_t h;
      asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(a + b));
      if (b < 8) w0 |= (uint64_t)h << (8 * b); else w1 |= (uint64_t)h << (8 * (b - 8));
    }
  }
}

template <int K, bool PAIR, bool WT = false>
__device__ __forceinline__ void sq_accumulate(u64 (&acc)[8], uint64_t w0, uint64_t w1,
                                              const float* s_lut, const u64* s_lut2, int lane,
                                              u64 wt = 0) {
#pragma unroll
  for (int j = 0; j < 16; j += 2) {
    if constexpr (PAIR) {
      acc[j / 2] = acc2<WT>(acc[j / 2], s_lut2[sq_code<K, 2 * K>(w0, w1, j) * 32 + lane], wt);
    } else {
      const float x0 = s_lut[sq_code<K>(w0, w1, j) * 32 + lane];
      const float x1 = s_lut[sq_code<K>(w0, w1, j + 1) * 32 + lane];
      acc[j / 2] = acc2<WT>(acc[j / 2], pack2(x0, x1), wt);
    }
  }
}

template <typename OT>
__device__ __forceinline__ void sq_store(OT* o, const u64 (&acc)[8], float inv, int j0, int64_t d,
                                         bool vec_ok) {
  if (j0 + 16 <= d) {
    store_scaled<16>(o, acc, inv, vec_ok);
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j0 + j < d) store_out(o + j, (j & 1 ? hi2(acc[j / 2]) : lo2(acc[j / 2])) * inv);
  }
}

// G4: rows staged by TMA tensor gathers (cp.async.bulk.tensor ... tile::gather4,
// sm_100): one instruction moves 4 code rows of 4 consecutive edges (row
// indices as coordinates), 4x fewer issue slots than per-row bulk copies,
// whose operands must be warp-uniform (a 32-step elect loop per warp).
template <int K, typename OT, bool WT, bool G4 = false, int PR = 0>
__global__ void __launch_bounds__(kBulkThreads, 1)
k_sq_mean_bulk(const uint8_t* __restrict__ rows, int64_t d, int64_t stride,
               const float* __restrict__ lut, const int32_t* __restrict__ indptr,
               const int32_t* __restrict__ src, const int64_t* __restrict__ ndst_dev,
               int64_t max_dst, OT* __restrict__ out, int64_t ld, int td, int row_cap, int rb,
               const float* __restrict__ ew, const __grid_constant__ CUtensorMap tmap) {
  constexpr int NT = kBulkThreads;
  constexpr int Q = 1 << K;
  constexpr bool PAIR = 2 * K <= 8;
  constexpr int LW = PAIR ? (1 << (2 * K)) * 64 : Q * 32;   // LUT floats
  constexpr int IPW = ((kTD + 1) * 4 + 3) & ~3;              // indptr ring ints
  extern __shared__ __align__(128) float s_mem[];
  float* s_lut = s_mem;
  u64* s_lut2 = reinterpret_cast<u64*>(s_mem);
  int32_t* s_ip = reinterpret_cast<int32_t*>(s_mem + LW);   // [4][kTD + 1]
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_ip + IPW);  // [2]
  // [2][buffer]: G4 packs rows in groups of 4 at a 128-byte-aligned group
  // pitch (tensor-copy destinations must be 128-byte aligned)
  uint8_t* s_rows = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(s_bar + 2) + 127) & ~static_cast<uintptr_t>(127));
  const int gstride = (4 * rb + 127) & ~127;
  const int64_t buf_bytes = G4 ? (int64_t)(row_cap >> 2) * gstride : (int64_t)row_cap * rb;
  auto rowp = [&](const uint8_t* base, int e) -> const uint8_t* {
    return G4 ? base + (int64_t)(e >> 2) * gstride + (e & 3) * rb : base + (int64_t)e * rb;
  };
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t live = live_dst(ndst_dev, max_dst);
  const int64_t ntiles = (live + td - 1) / td;
  if ((int64_t)blockIdx.x >= ntiles) return;
  const int64_t G = gridDim.x;
  if constexpr (PAIR) {
    for (int i = tid; i < Q * Q * 32; i += NT) {
      const int pv = i >> 5;
      s_lut2[i] = pack2(lut[pv >> K], lut[pv & (Q - 1)]);
    }
  } else {
    for (int i = tid; i < Q * 32; i += NT) s_lut[i] = lut[i >> 5];
  }
  if (tid == 0) {
    mbar_init(s_bar, 1);
    mbar_init(s_bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  const int chunks = (int)((d + 15) >> 4);
  const bool vec_ok = (ld % 16) == 0;
  auto tile_of = [&](int64_t k) { return (int64_t)blockIdx.x + k * G; };
  auto ip_slot = [&](int64_t k) { return s_ip + (int)(k & 3) * (kTD + 1); };
  auto load_ip = [&](int64_t tile) -> int32_t {
    return tid <= td ? __ldg(indptr + min64(tile * td + tid, live)) : 0;
  };
  auto store_ip = [&](int32_t* slot, int32_t v) { if (tid <= td) slot[tid] = v; };
  int32_t sid[kBulkSidPer];
  // G4: thread t owns edges 4t .. 4t+3 (one gather4); else edges t + j*NT
  auto edge_of = [&](int j) { return G4 ? 4 * tid + j : tid + j * NT; };
  auto load_sids = [&](const int32_t* ip) {
    const int32_t e0 = ip[0], ne = ip[td] - e0;
    if (ne > row_cap) return;
#pragma unroll
    for (int j = 0; j < kBulkSidPer; ++j) {
      const int e = edge_of(j);
      // G4 pads a partial last group with its last valid row (dummy copies
      // into buffer slack; never read)
      if (e < ne) sid[j] = (PR & 1) ? ((e0 + e) & 1023) : __ldg(src + e0 + e);
      else if (G4 && 4 * tid < ne) sid[j] = sid[j > 0 ? j - 1 : 0];
    }
  };
  auto issue_rows = [&](const int32_t* ip, int b) {
    const int32_t ne = ip[td] - ip[0];
    if (ne > row_cap) return;
    const uint32_t bar = smem_addr(s_bar + b);
    uint8_t* dst = s_rows + (int64_t)b * buf_bytes;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint32_t groups = G4 ? (uint32_t)((ne + 3) / 4) : 0u;
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                   ::"r"(bar), "r"((G4 ? groups * 4u : (uint32_t)ne) * (uint32_t)rb) : "memory");
    if constexpr (G4) {
      if ((uint32_t)tid < groups)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            ::"r"(smem_addr(dst + (int64_t)tid * gstride)),
              "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"(sid[0]), "r"(sid[1]),
              "r"(sid[2]), "r"(sid[3]), "r"(bar) : "memory");
    } else {
#pragma unroll
      for (int j = 0; j < kBulkSidPer; ++j) {
        const int e = tid + j * NT;
        if (e < ne)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
              ::"r"(smem_addr(dst + (int64_t)e * rb)), "l"(rows + (int64_t)sid[j] * stride),
                "r"(rb), "r"(bar) : "memory");
      }
    }
  };
  // prologue: indptr of tiles 0..2, rows of tile 0 in flight, src ids of tile 1
  {
    int32_t r[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) r[q] = tile_of(q) < ntiles ? load_ip(tile_of(q)) : 0;
#pragma unroll
    for (int q = 0; q < 3; ++q) if (tile_of(q) < ntiles) store_ip(ip_slot(q), r[q]);
  }
  __syncthreads();
  load_sids(ip_slot(0));
  issue_rows(ip_slot(0), 0);
  if (tile_of(1) < ntiles) load_sids(ip_slot(1));
  uint32_t phase = 0;
  for (int64_t k = 0; tile_of(k) < ntiles; ++k) {
    const int64_t tile = tile_of(k);
    const int b = (int)(k & 1);
    if (tile_of(k + 1) < ntiles) issue_rows(ip_slot(k + 1), b ^ 1);
    if (tile_of(k + 2) < ntiles) load_sids(ip_slot(k + 2));
    const bool has3 = tile_of(k + 3) < ntiles;
    int32_t ipr = 0;
    if (has3) ipr = load_ip(tile_of(k + 3));
    const int32_t* ip = ip_slot(k);
    const int32_t e0 = ip[0];
    const bool staged = ip[td] - e0 <= row_cap;
    if (staged) {
      mbar_wait_parity(s_bar + b, (phase >> b) & 1u);
      phase ^= 1u << b;
    }
    const uint8_t* rbuf = s_rows + (int64_t)b * buf_bytes;
    const int items = td * chunks;
    for (int it = tid; it < items; it += NT) {
      const int vl = it / chunks;
      const int c = it - vl * chunks;
      const int64_t v = tile * td + vl;
      if (v >= live) break;
      u64 acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0ull;
      const int a = ip[vl] - e0;
      const int cnt = ip[vl + 1] - e0 - a;
      if (staged) {
        const int coff = c * (2 * K);
        const float* ewp = WT ? ew + e0 + a : nullptr;
        int p = 0;
        for (; p + 4 <= cnt; p += 4) {
          uint64_t w[4][2];
          u64 wt[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            lds_chunk<K>(rowp(rbuf, a + p + u) + coff, w[u][0], w[u][1]);
            if constexpr (WT) wt[u] = bcast2(__ldg(ewp + p + u));
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if constexpr ((PR & 2) != 0) {
              acc[u] = fadd2(acc[u], w[u][0] ^ w[u][1]);
            } else {
              sq_accumulate<K, PAIR, WT>(acc, w[u][0], w[u][1], s_lut, s_lut2, lane,
                                         WT ? wt[u] : 0);
            }
          }
        }
        for (; p < cnt; ++p) {
          uint64_t w0, w1;
          lds_chunk<K>(rowp(rbuf, a + p) + coff, w0, w1);
          sq_accumulate<K, PAIR, WT>(acc, w0, w1, s_lut, s_lut2, lane,
                                     WT ? bcast2(__ldg(ewp + p)) : 0);
        }
      } else {
        const int64_t boff = (int64_t)c * (2 * K);
        for (int base = 0; base < cnt; base += 8) {
          uint64_t w[8][2];
          u64 wt[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (base + u < cnt) {
              load_chunk<K>(rows + (int64_t)__ldg(src + e0 + a + base + u) * stride + boff,
                            w[u][0], w[u][1]);
              if constexpr (WT) wt[u] = bcast2(__ldg(ew + e0 + a + base + u));
            }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (base + u < cnt)
              sq_accumulate<K, PAIR, WT>(acc, w[u][0], w[u][1], s_lut, s_lut2, lane,
                                         WT ? wt[u] : 0);
        }
      }
      const float inv = WT ? 1.0f : (cnt ? 1.0f / (float)cnt : 0.0f);
      if (!(PR & 4) || lo2(acc[0]) == -1234.5f)
        sq_store(out + v * ld + c * 16, acc, inv, c * 16, d, vec_ok);
    }
    // slot k+3 (= k-1 mod 4) was last read before the previous barrier; the
    // barrier below publishes it and retires row buffer b for tile k+2
    if (has3) store_ip(ip_slot(k + 3), ipr);
    __syncthreads();
  }
}

// 2-D uint8 tensor map over the code rows ([n][row_stride] bytes, box = the
// first rb bytes of one row) for the gather4 row staging; false when the
// driver entry point is unavailable (then per-row bulk copies are used).
static bool code_row_tensor_map(const fg_codec_desc* c, int rb, CUtensorMap* m) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  memset(m, 0, sizeof(*m));
  if (!encode || (reinterpret_cast<uintptr_t>(c->rows) & 15) || (c->row_stride & 15) || c->n < 1)
    return false;
  const cuuint64_t dims[2] = {(cuuint64_t)c->row_stride, (cuuint64_t)c->n};
  const cuuint64_t strides[1] = {(cuuint64_t)c->row_stride};
  const cuuint32_t box[2] = {(cuuint32_t)rb, 1u};
  const cuuint32_t estr[2] = {1u, 1u};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)c->rows, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// ------------------------------------------------------------ launchers
template <int K, typename OT, bool WT>
int launch_sq_w(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                const int64_t* ndst, int64_t max_dst, void* out, int64_t ld, cudaStream_t st,
                const float* ew) {
  if constexpr (std::is_same<OT, __nv_bfloat16>::value) {
    int rc = FG_OK;
    if (launch_sq_lane<WT>(c, indptr, src, ndst, max_dst, out, ld, st, &rc)) return rc;
  }
  // TMA-staged variant: needs a row buffer holding a tile of >= 32
  // destinations at fanout 8 next to the decode table
  {
    constexpr int kSmemBudget = 220 * 1024;
    const int lut_b = 2 * K <= 8 ? (1 << (2 * K)) * 32 * 8 : (1 << K) * 32 * 4;
    const int fixed = lut_b + ((((kTD + 1) * 4 + 3) & ~3) * 4) + 16;
    const int chunks = (int)((c->d + 15) / 16);
    const int rb = (chunks * 2 * K + 15) / 16 * 16;
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    const bool g4 = rb <= 256 && rb <= c->row_stride && code_row_tensor_map(c, rb, &tmap);
    const int gstride = (4 * rb + 127) & ~127;  // G4 group pitch (128-B aligned)
    int row_cap = g4 ? (kSmemBudget - fixed - 128) / (2 * gstride) * 4
                     : (kSmemBudget - fixed - 128) / (2 * rb);
    if (row_cap > kBulkRowCap) row_cap = kBulkRowCap;
    row_cap &= ~3;  // whole gather4 groups
    int td = kTD;
    while (td > 32 && td * 8 > row_cap) td /= 2;
    static const int bulk_env = [] {  // FG_SQ_BULK=0: register kernel (A/B)
      const char* e = getenv("FG_SQ_BULK");
      return e ? atoi(e) : 1;
    }();
    if (bulk_env && td * 8 <= row_cap && rb <= c->row_stride) {
      const int smem = fixed + 128 + 2 * (g4 ? (row_cap / 4) * gstride : row_cap * rb);
      const int grid = (int)min64(ceil_div(max_dst, td), (int64_t)sm_count());
      auto kern = g4 ? k_sq_mean_bulk<K, OT, WT, true> : k_sq_mean_bulk<K, OT, WT, false>;
      const int probe = [] {  // read per launch (diagnostic sweeps flip it in-process)  // diagnostics, see vq_fast_body
        const char* e = getenv("FG_FUSED_PROBE");
        return e ? atoi(e) : 0;
      }();
      if constexpr (!WT && K == 4) {
        if (g4 && probe) {
          switch (probe) {
            case 1: kern = k_sq_mean_bulk<K, OT, WT, true, 1>; break;
            case 2: kern = k_sq_mean_bulk<K, OT, WT, true, 2>; break;
            case 3: kern = k_sq_mean_bulk<K, OT, WT, true, 3>; break;
            case 4: kern = k_sq_mean_bulk<K, OT, WT, true, 4>; break;
            case 5: kern = k_sq_mean_bulk<K, OT, WT, true, 5>; break;
            case 6: kern = k_sq_mean_bulk<K, OT, WT, true, 6>; break;
            default: break;
          }
        }
      }
      FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kern<<<grid, kBulkThreads, smem, st>>>(c->rows, c->d, c->row_stride,
                                             (const float*)c->table, indptr, src, ndst, max_dst,
                                             (OT*)out, ld, td, row_cap, rb, ew, tmap);
      FG_LAUNCH_CHECK();
      return FG_OK;
    }
  }
  const int lut_bytes = 2 * K <= 8 ? (1 << (2 * K)) * 32 * 8 : (1 << K) * 32 * 4;
  const int smem = lut_bytes + 2 * (kTD + 1 + kSrcCap) * 4;
  auto kern = k_sq_mean<K, OT, WT>;
  FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = (int)min64(ceil_div(max_dst, kTD), (int64_t)sm_count() * 2);
  kern<<<grid, kThreads, smem, st>>>(c->rows, c->d, c->row_stride, (const float*)c->table,
                                     indptr, src, ndst, max_dst, (OT*)out, ld, ew);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

template <int K, typename OT>
int launch_sq(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
              const int64_t* ndst, int64_t max_dst, void* out, int64_t ld, cudaStream_t st,
              const float* ew) {
  return ew ? launch_sq_w<K, OT, true>(c, indptr, src, ndst, max_dst, out, ld, st, ew)
            : launch_sq_w<K, OT, false>(c, indptr, src, ndst, max_dst, out, ld, st, nullptr);
}

template <typename OT>
int dispatch_sq(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                const int64_t* ndst, int64_t max_dst, void* out, int64_t ld, cudaStream_t st,
                const float* ew) {
  switch (c->bits) {
    case 1: return launch_sq<1, OT>(c, indptr, src, ndst, max_dst, out, ld, st, ew);
    case 2: return launch_sq<2, OT>(c, indptr, src, ndst, max_dst, out, ld, st, ew);
    case 3: return launch_sq<3, OT>(c, indptr, src, ndst, max_dst, out, ld, st, ew);
    case 4: return launch_sq<4, OT>(c, indptr, src, ndst, max_dst, out, ld, st, ew);
    case 5: return launch_sq<5, OT>(c, indptr, src, ndst, max_dst, out, ld, st, ew);
    case 6: return launch_sq<6, OT>(c, indptr, src, ndst, max_dst, out, ld, st, ew);
    case 7: return launch_sq<7, OT>(c, indptr, src, ndst, max_dst, out, ld, st, ew);
    case 8: return launch_sq<8, OT>(c, indptr, src, ndst, max_dst, out, ld, st, ew);
  }
  set_error("bad SQ k %d", c->bits);
  return FG_EUSAGE;
}

template <int W, typename OT, bool WT>
int launch_vq_w(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                const int64_t* ndst, int64_t max_dst, void* out, int64_t ld, cudaStream_t st,
                const float* ew) {
  const int64_t book_bytes = (int64_t)c->num_parts * c->length * W * 4;
  const int64_t stage_bytes = 2 * (kTD + 1 + kSrcCap) * 4;
  const int64_t ntiles = ceil_div(max_dst, kTD);
  if (c->bits != 8) {
    auto kern = k_vq_mean_bits<W, OT>;
    const int grid = (int)min64(ntiles, (int64_t)sm_count() * 2);
    kern<<<grid, kThreads, stage_bytes, st>>>(c->rows, c->d, c->row_stride, c->bits,
                                         (const float*)c->table, c->length, c->num_parts, indptr,
                                         src, ndst, max_dst, (OT*)out, ld, ew);
    FG_LAUNCH_CHECK();
    return FG_OK;
  }
  // bf16 output may read the bf16 copy of the codebooks (half the smem bytes)
  const bool lp = std::is_same<OT, __nv_bfloat16>::value && c->table_lp != nullptr && W >= 4;
  if constexpr (std::is_same<OT, __nv_bfloat16>::value && (W == 4 || W == 8)) {
    // lane-per-part kernel (v5): sector slices of 32 parts, one CTA per SM.
    // Default whenever the fp16 copy of the codebook exists (scaled table_h,
    // HADD2 chunks) -- with the unpredicated C-pick bodies (lane_f16_body):
    // MAG240M-shape 125 (v4) -> 116.6 -> 76.9 us, products-shape 36.9 (v4)
    // -> 33.8 us.  With the bf16 table it was issue-bound (73 %) and tied v4,
    // so codecs without table_h stay on v4.
    // FG_VQ_LANE = 0 (off) | 1 (bf16 table) | 2 (fp16 table) forces a mode.
    static const int lane_force = [] {
      const char* e = getenv("FG_VQ_LANE");
      return e ? atoi(e) : -1;
    }();
    const int64_t v4_unsliced = (((int64_t)c->num_parts + (32 / W) - 1) / (32 / W) * (32 / W)) *
                                    c->length * W * 2 + stage_bytes;
    const bool has_h = !WT && c->table_h != nullptr && c->part_scale != nullptr;
    (void)v4_unsliced;
    const int lane_env = lane_force >= 0 ? lane_force : (has_h ? 2 : 0);
    const int64_t lane_smem = (int64_t)32 * c->length * W * 2 + 2 * kSrcCap * 32 +
                              3 * kSrcCap * 4 + 4 * (kTD + 4) * 4;
    if (lp && lane_env && c->row_stride % 32 == 0 && lane_smem <= 227 * 1024) {
      const int ns = (int)ceil_div(c->num_parts, 32);
      const bool f16 = !WT && c->table_h != nullptr && c->part_scale != nullptr && lane_env == 2;
      // fp16 tables: FG_VQ_LANE_NT=512 (112 registers, two 5-pick
      // destinations per warp pass) / 768 (80 registers) / 1024 (default).
      // Measured: MAG 71.2 / 71.1 / 71.2 us; products-shape kernel 28.7 vs
      // 29.9 us at 512 but the pipelined step 0.2408 vs 0.2381 ms (the
      // overlapped sampler), so 1024 everywhere
      static const int lane_nt_env = [] {
        const char* e = getenv("FG_VQ_LANE_NT");
        return e ? atoi(e) : 0;
      }();
      const int lane_nt = !f16 ? kLaneThreads : (lane_nt_env ? lane_nt_env : kLaneThreads);
      auto kern = !f16 ? k_vq_mean8_lane<W, WT, false>
                  : lane_nt == 512 ? k_vq_mean8_lane<W, false, true, 512>
                  : lane_nt == 768 ? k_vq_mean8_lane<W, false, true, 768>
                                   : k_vq_mean8_lane<W, false, true>;
      const int nthreads = (f16 && (lane_nt == 512 || lane_nt == 768)) ? lane_nt : kLaneThreads;
      FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)lane_smem));
      const int64_t per_slice = std::max<int64_t>(1, min64(ntiles, sm_count() / ns));
      kern<<<(int)(per_slice * ns), nthreads, lane_smem, st>>>(
          c->rows, c->d, c->row_stride,
          (const __nv_bfloat16*)(f16 ? c->table_h : c->table_lp), c->length,
          c->num_parts, indptr, src, ndst, max_dst, (__nv_bfloat16*)out, ld, ns, ew,
          c->part_scale);
      FG_LAUNCH_CHECK();
      return FG_OK;
    }
  }
  if constexpr (std::is_same<OT, __nv_bfloat16>::value && (W == 4 || W == 8)) {
    constexpr int GF = 32 / W;
    constexpr int64_t kFastSmem = 76 * 1024;  // three CTAs per SM (233 KB smem per SM)
    const int64_t part_bytes = (int64_t)c->length * W * 2;
    const int zp = (GF - c->num_parts % GF) % GF;
    // parts per slice: the whole codebook when it fits, else the largest
    // multiple of GF whose slice (+ zero pad + tile stage) fits
    int sp = c->num_parts;
    auto smem_for = [&](int s) {
      return ((((int64_t)s + zp) * part_bytes + 15) & ~15ll) + stage_bytes;
    };
    if (smem_for(sp) > kFastSmem) {
      sp = (int)((kFastSmem - stage_bytes) / part_bytes) - zp;
      sp = sp / GF * GF;
    }
    if (lp && sp >= GF) {
      const int ns = (int)ceil_div(c->num_parts, sp);
      const int64_t fast_smem = smem_for(sp);
      const int probe = [] {  // read per launch (diagnostic sweeps flip it in-process)
        const char* e = getenv("FG_FUSED_PROBE");
        return e ? atoi(e) : 0;
      }();
      auto kern = k_vq_mean8_fast<W, GF, WT>;
      if constexpr (!WT) {
        switch (probe) {
          case 1: kern = k_vq_mean8_fast<W, GF, WT, 1>; break;
          case 2: kern = k_vq_mean8_fast<W, GF, WT, 2>; break;
          case 3: kern = k_vq_mean8_fast<W, GF, WT, 3>; break;
          case 4: kern = k_vq_mean8_fast<W, GF, WT, 4>; break;
          case 5: kern = k_vq_mean8_fast<W, GF, WT, 5>; break;
          case 6: kern = k_vq_mean8_fast<W, GF, WT, 6>; break;
          default: break;
        }
      }
      FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)fast_smem));
      // grid: a multiple of the slice count, ~3 CTAs per SM in total
      // (FG_FUSED_CTA_PCT: percent of that, to leave room for overlapped work)
      static const int pct = [] {
        const char* e = getenv("FG_FUSED_CTA_PCT");
        const int v = e ? atoi(e) : 100;
        return v > 0 && v <= 100 ? v : 100;
      }();
      const int64_t per_slice = std::max<int64_t>(
          1, min64(ntiles, (int64_t)sm_count() * 3 * pct / 100 / ns));
      const int grid = (int)(per_slice * ns);
      // L2 prefetch of the next tile's code rows: unsliced codebooks only
      // (products 37.7 -> 37.0 us; with MAG's 6 part slices every slice CTA
      // would prefetch the same rows: 128 -> 181 us).  FG_FUSED_PREFETCH=0/1
      static const int pf_env = [] {
        const char* e = getenv("FG_FUSED_PREFETCH");
        return e ? atoi(e) : -1;
      }();
      const int pf = pf_env >= 0 ? pf_env : (ns == 1 ? 1 : 0);
      kern<<<grid, kFastThreads, fast_smem, st>>>(c->rows, c->d, c->row_stride,
                                              (const __nv_bfloat16*)c->table_lp, c->length,
                                              c->num_parts, indptr, src, ndst, max_dst,
                                              (__nv_bfloat16*)out, ld, sp, ns, ew, pf);
      FG_LAUNCH_CHECK();
      return FG_OK;
    }
  }
  const int64_t tab_bytes = lp ? book_bytes / 2 : book_bytes;
  const int64_t smem2 = ((tab_bytes + 15) & ~15ll) + stage_bytes;
  if (smem2 <= 220 * 1024) {
    const int per_sm = smem2 <= 110 * 1024 ? 2 : 1;
    const int grid = (int)min64(ntiles, (int64_t)sm_count() * per_sm);
    if (lp) {
      auto kern = k_vq_mean8<W, OT, true, __nv_bfloat16, WT>;
      FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem2));
      kern<<<grid, kThreads, smem2, st>>>(c->rows, c->d, c->row_stride,
                                          (const __nv_bfloat16*)c->table_lp, c->length,
                                          c->num_parts, indptr, src, ndst, max_dst, (OT*)out, ld, ew);
    } else {
      auto kern = k_vq_mean8<W, OT, true, float, WT>;
      FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem2));
      kern<<<grid, kThreads, smem2, st>>>(c->rows, c->d, c->row_stride, (const float*)c->table,
                                          c->length, c->num_parts, indptr, src, ndst, max_dst,
                                          (OT*)out, ld, ew);
    }
  } else {
    auto kern = k_vq_mean8<W, OT, false, float, WT>;
    const int grid = (int)min64(ntiles, (int64_t)sm_count() * 2);
    kern<<<grid, kThreads, stage_bytes, st>>>(c->rows, c->d, c->row_stride, (const float*)c->table,
                                         c->length, c->num_parts, indptr, src, ndst, max_dst,
                                         (OT*)out, ld, ew);
  }
  FG_LAUNCH_CHECK();
  return FG_OK;
}

template <int W, typename OT>
int launch_vq(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
              const int64_t* ndst, int64_t max_dst, void* out, int64_t ld, cudaStream_t st,
              const float* ew) {
  return ew ? launch_vq_w<W, OT, true>(c, indptr, src, ndst, max_dst, out, ld, st, ew)
            : launch_vq_w<W, OT, false>(c, indptr, src, ndst, max_dst, out, ld, st, nullptr);
}

template <typename OT>
int dispatch_vq(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                const int64_t* ndst, int64_t max_dst, void* out, int64_t ld, cudaStream_t st,
                const float* ew) {
  switch (c->width) {
    case 1: return launch_vq<1, OT>(c, indptr, src, ndst, max_dst, out, ld, st, ew);
    case 2: return launch_vq<2, OT>(c, indptr, src, ndst, max_dst, out, ld, st, ew);
    case 4: return launch_vq<4, OT>(c, indptr, src, ndst, max_dst, out, ld, st, ew);
    case 8: return launch_vq<8, OT>(c, indptr, src, ndst, max_dst, out, ld, st, ew);
    case 16: return launch_vq<16, OT>(c, indptr, src, ndst, max_dst, out, ld, st, ew);
  }
  set_error("fused VQ mean supports width in {1,2,4,8,16}, got %d", c->width);
  return FG_EUSAGE;
}

}  // namespace fg

using namespace fg;

static int gather_aggregate(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                            const float* edge_w, const int64_t* ndst, int64_t max_dst, void* out,
                            int64_t out_ld, int out_dtype, void* s) {
  FG_CHECK_ARG(c != nullptr && indptr != nullptr && ndst != nullptr, "null argument");
  FG_CHECK_ARG(c->elem_bits == 32, "fused aggregate needs a float32 decode table");
  FG_CHECK_ARG(out_dtype == FG_OUT_F32 || out_dtype == FG_OUT_BF16,
               "out dtype must be f32 or bf16");
  const int64_t ld = out_ld > 0 ? out_ld : c->d;
  FG_CHECK_ARG(ld >= c->d, "out_ld must be >= d");
  if (max_dst == 0) return FG_OK;
  cudaStream_t st = as_stream(s);
  if (c->kind == FG_CODEC_SQ) {
    FG_CHECK_ARG(c->row_stride % 16 == 0, "row stride must be a multiple of 16");
    FG_CHECK_ARG(c->row_stride >= ((c->d + 15) / 16) * 2 * c->bits,
                 "SQ row stride must cover ceil(d/16)*2k bytes (whole 16-code chunks)");
    return out_dtype == FG_OUT_F32
               ? dispatch_sq<float>(c, indptr, src, ndst, max_dst, out, ld, st, edge_w)
               : dispatch_sq<__nv_bfloat16>(c, indptr, src, ndst, max_dst, out, ld, st, edge_w);
  }
  if (c->kind == FG_CODEC_VQ) {
    FG_CHECK_ARG(c->bits >= 1 && c->bits <= 16, "bad VQ code bits");
    FG_CHECK_ARG(c->bits != 8 || c->row_stride >= ((c->num_parts + 31) / 32) * 32,
                 "8-bit VQ rows must be padded to 32 bytes");
    return out_dtype == FG_OUT_F32
               ? dispatch_vq<float>(c, indptr, src, ndst, max_dst, out, ld, st, edge_w)
               : dispatch_vq<__nv_bfloat16>(c, indptr, src, ndst, max_dst, out, ld, st, edge_w);
  }
  set_error("unknown codec kind %d", c->kind);
  return FG_EUSAGE;
}

extern "C" int fg_gather_dequant_mean(const fg_codec_desc* c, const int32_t* indptr,
                                      const int32_t* src, const int64_t* ndst, int64_t max_dst,
                                      void* out, int64_t out_ld, int out_dtype, void* s) {
  return gather_aggregate(c, indptr, src, nullptr, ndst, max_dst, out, out_ld, out_dtype, s);
}

extern "C" int fg_gather_dequant_wsum(const fg_codec_desc* c, const int32_t* indptr,
                                      const int32_t* src, const float* edge_w,
                                      const int64_t* ndst, int64_t max_dst, void* out,
                                      int64_t out_ld, int out_dtype, void* s) {
  FG_CHECK_ARG(edge_w != nullptr, "fg_gather_dequant_wsum: null edge weights");
  return gather_aggregate(c, indptr, src, edge_w, ndst, max_dst, out, out_ld, out_dtype, s);
}
