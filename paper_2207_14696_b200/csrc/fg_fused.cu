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
#include "fg_common.cuh"

namespace fg {

constexpr int kTD = 128;     // destinations per tile
constexpr int kSrcCap = kTD * 16;  // staged src ids per tile (fanout <= 16 fully staged)

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
__device__ __forceinline__ u64 pack2(float x, float y) {
  return ((u64)__float_as_uint(y) << 32) | __float_as_uint(x);
}
__device__ __forceinline__ float lo2(u64 v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float hi2(u64 v) { return __uint_as_float((uint32_t)(v >> 32)); }

// Store n (multiple of 2) consecutive outputs v[0..n) * inv at p; uses 16/8-byte
// vector stores when `vec` (caller guarantees alignment).
template <int N>
__device__ __forceinline__ void store_scaled(float* p, const u64* acc, float inv, bool vec) {
  if (vec && N % 4 == 0) {
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
  if (vec && N % 8 == 0) {
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

// Stage indptr[v0 .. v0+kTD] (clamped to max_dst) and the tile's src ids.
__device__ __forceinline__ void stage_tile(const int32_t* __restrict__ indptr,
                                           const int32_t* __restrict__ src, int64_t v0,
                                           int64_t max_dst, int32_t* s_ip, int32_t* s_src,
                                           int32_t& e0, int32_t& ecount) {
  for (int t = threadIdx.x; t <= kTD; t += blockDim.x) {
    const int64_t v = min64(v0 + t, max_dst);
    s_ip[t] = __ldg(indptr + v);
  }
  __syncthreads();
  e0 = s_ip[0];
  ecount = s_ip[kTD] - e0;
  if (ecount <= kSrcCap)
    for (int t = threadIdx.x; t < ecount; t += blockDim.x) s_src[t] = __ldg(src + e0 + t);
  __syncthreads();
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

template <int K>
__device__ __forceinline__ uint32_t sq_code(uint64_t w0, uint64_t w1, int j) {
  constexpr int Q = 1 << K;
  const int bit = j * K;
  const int byte = bit >> 3;
  const int inb = bit & 7;
  const uint64_t word = byte < 8 ? w0 : w1;
  if (K == 8 || inb + K <= 8) {
    const uint32_t by = (uint32_t)(word >> (8 * (byte & 7))) & 0xFFu;
    return (by >> (8 - inb - K)) & (Q - 1);
  }
  const int byte2 = byte + 1;
  const uint64_t word2 = byte2 < 8 ? w0 : w1;
  const uint32_t hi = (uint32_t)(word >> (8 * (byte & 7))) & 0xFFu;
  const uint32_t lo = (uint32_t)(word2 >> (8 * (byte2 & 7))) & 0xFFu;
  return (((hi << 8) | lo) >> (16 - inb - K)) & (Q - 1);
}

template <int K, typename OT>
__global__ void __launch_bounds__(512, 2)
k_sq_mean(const uint8_t* __restrict__ rows, int64_t d, int64_t stride,
          const float* __restrict__ lut, const int32_t* __restrict__ indptr,
          const int32_t* __restrict__ src, const int64_t* __restrict__ ndst_dev,
          int64_t max_dst, OT* __restrict__ out, int64_t ld) {
  constexpr int Q = 1 << K;
  constexpr int CB = 2 * K;
  constexpr int U = K >= 5 ? 4 : 8;  // picks whose loads are issued together
  extern __shared__ float s_mem[];
  float* s_lut = s_mem;                                        // [Q][32]
  int32_t* s_ip = reinterpret_cast<int32_t*>(s_mem + Q * 32);  // [kTD + 1]
  int32_t* s_src = s_ip + kTD + 1;                             // [kSrcCap]
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < Q * 32; i += blockDim.x) s_lut[i] = lut[i >> 5];
  const int64_t live = live_dst(ndst_dev, max_dst);
  const int chunks = (int)((d + 15) >> 4);
  const int64_t ntiles = (live + kTD - 1) / kTD;
  const bool vec_ok = (ld % 16) == 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t v0 = tile * kTD;
    int32_t e0, ecount;
    stage_tile(indptr, src, v0, max_dst, s_ip, s_src, e0, ecount);
    const bool staged = ecount <= kSrcCap;
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
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (base + u < cnt) {
            const int e = a + base + u;
            const int32_t sid = staged ? s_src[e] : __ldg(src + e0 + e);
            load_chunk<K>(rows + (int64_t)sid * stride + boff, w[u][0], w[u][1]);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (base + u < cnt) {
#pragma unroll
            for (int j = 0; j < 16; j += 2) {
              const float x0 = s_lut[sq_code<K>(w[u][0], w[u][1], j) * 32 + lane];
              const float x1 = s_lut[sq_code<K>(w[u][0], w[u][1], j + 1) * 32 + lane];
              acc[j / 2] = fadd2(acc[j / 2], pack2(x0, x1));
            }
          }
        }
      }
      const float inv = cnt ? 1.0f / (float)cnt : 0.0f;
      const int j0 = c * 16;
      OT* o = out + v * ld + j0;
      if (j0 + 16 <= d) {
        store_scaled<16>(o, acc, inv, vec_ok);
      } else {
        for (int j = 0; j < 16 && j0 + j < d; ++j)
          store_out(o + j, (j & 1 ? hi2(acc[j / 2]) : lo2(acc[j / 2])) * inv);
      }
    }
    __syncthreads();  // s_ip / s_src reused by the next tile
  }
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

template <int W, typename OT, bool SMEM>
__global__ void __launch_bounds__(512, 2)
k_vq_mean8(const uint8_t* __restrict__ rows, int64_t d, int64_t stride,
           const float* __restrict__ books, int length, int parts,
           const int32_t* __restrict__ indptr, const int32_t* __restrict__ src,
           const int64_t* __restrict__ ndst_dev, int64_t max_dst, OT* __restrict__ out,
           int64_t ld) {
  constexpr int G = 32 / W;        // parts per thread
  constexpr int NW = (G + 3) / 4;  // 32-bit code words per load
  constexpr int U = 4;             // picks whose loads are issued together
  extern __shared__ float4 s_mem4[];
  const int64_t nbook = SMEM ? (int64_t)parts * length * W : 0;
  float* s_book = reinterpret_cast<float*>(s_mem4);
  int32_t* s_ip = reinterpret_cast<int32_t*>(s_book + ((nbook + 3) & ~3ll));
  int32_t* s_src = s_ip + kTD + 1;
  const float* book = books;
  if constexpr (SMEM) {
    const float4* g4 = reinterpret_cast<const float4*>(books);
    for (int64_t i = threadIdx.x; i < nbook / 4; i += blockDim.x) s_mem4[i] = __ldg(g4 + i);
    for (int64_t i = (nbook & ~3ll) + threadIdx.x; i < nbook; i += blockDim.x)
      s_book[i] = __ldg(books + i);
    book = s_book;
  }
  const int64_t live = live_dst(ndst_dev, max_dst);
  const int groups = (parts + G - 1) / G;
  const int64_t ntiles = (live + kTD - 1) / kTD;
  const bool vec_ok = (ld % 16) == 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t v0 = tile * kTD;
    int32_t e0, ecount;
    stage_tile(indptr, src, v0, max_dst, s_ip, s_src, e0, ecount);
    const bool staged = ecount <= kSrcCap;
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
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (base + u < cnt) {
            const int e = a + base + u;
            const int32_t sid = staged ? s_src[e] : __ldg(src + e0 + e);
            load_codes<G>(rows + (int64_t)sid * stride + p0, cw[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (base + u < cnt) {
#pragma unroll
            for (int q = 0; q < G; ++q) {
              if (q < np) {
                const uint32_t code = (cw[u][q >> 2] >> (8 * (q & 3))) & 0xFFu;
                const float* ent = book + ((int64_t)(p0 + q) * length + code) * W;
                if constexpr (W >= 4) {
#pragma unroll
                  for (int j = 0; j < W; j += 4) {
                    const float4 f = SMEM ? *reinterpret_cast<const float4*>(ent + j)
                                          : __ldg(reinterpret_cast<const float4*>(ent + j));
                    acc[(q * W + j) / 2] = fadd2(acc[(q * W + j) / 2], pack2(f.x, f.y));
                    acc[(q * W + j) / 2 + 1] = fadd2(acc[(q * W + j) / 2 + 1], pack2(f.z, f.w));
                  }
                } else if constexpr (W == 2) {
                  const float2 f = SMEM ? *reinterpret_cast<const float2*>(ent)
                                        : __ldg(reinterpret_cast<const float2*>(ent));
                  acc[q] = fadd2(acc[q], pack2(f.x, f.y));
                } else {  // W == 1: pair adjacent parts
                  const float f = SMEM ? ent[0] : __ldg(ent);
                  acc[q / 2] = fadd2(acc[q / 2], (q & 1) ? pack2(0.f, f) : pack2(f, 0.f));
                }
              }
            }
          }
        }
      }
      const float inv = cnt ? 1.0f / (float)cnt : 0.0f;
      const int64_t col0 = (int64_t)p0 * W;
      OT* o = out + v * ld + col0;
      if (np == G && col0 + G * W <= d) {
        store_scaled<G * W>(o, acc, inv, vec_ok);
      } else {
        for (int j = 0; j < G * W && col0 + j < d; ++j)
          store_out(o + j, (j & 1 ? hi2(acc[j / 2]) : lo2(acc[j / 2])) * inv);
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------- VQ (any code width)
template <int W, typename OT>
__global__ void __launch_bounds__(512, 2)
k_vq_mean_bits(const uint8_t* __restrict__ rows, int64_t d, int64_t stride, int bits,
               const float* __restrict__ books, int length, int parts,
               const int32_t* __restrict__ indptr, const int32_t* __restrict__ src,
               const int64_t* __restrict__ ndst_dev, int64_t max_dst, OT* __restrict__ out,
               int64_t ld) {
  extern __shared__ int32_t s_stage[];
  int32_t* s_ip = s_stage;
  int32_t* s_src = s_ip + kTD + 1;
  const int64_t live = live_dst(ndst_dev, max_dst);
  const int64_t ntiles = (live + kTD - 1) / kTD;
  const uint32_t cmask = (1u << bits) - 1u;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t v0 = tile * kTD;
    int32_t e0, ecount;
    stage_tile(indptr, src, v0, max_dst, s_ip, s_src, e0, ecount);
    const bool staged = ecount <= kSrcCap;
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
#pragma unroll
        for (int j = 0; j < W; ++j) acc[j] += __ldg(ent + j);
      }
      const float inv = cnt ? 1.0f / (float)cnt : 0.0f;
      OT* o = out + v * ld + (int64_t)p * W;
      for (int j = 0; j < W && (int64_t)p * W + j < d; ++j) store_out(o + j, acc[j] * inv);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ launchers
template <int K, typename OT>
int launch_sq(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
              const int64_t* ndst, int64_t max_dst, void* out, int64_t ld, cudaStream_t st) {
  const int smem = (1 << K) * 32 * 4 + (kTD + 1 + kSrcCap) * 4;
  auto kern = k_sq_mean<K, OT>;
  FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = (int)min64(ceil_div(max_dst, kTD), (int64_t)sm_count() * 2);
  kern<<<grid, 512, smem, st>>>(c->rows, c->d, c->row_stride, (const float*)c->table, indptr,
                                src, ndst, max_dst, (OT*)out, ld);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

template <typename OT>
int dispatch_sq(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                const int64_t* ndst, int64_t max_dst, void* out, int64_t ld, cudaStream_t st) {
  switch (c->bits) {
    case 1: return launch_sq<1, OT>(c, indptr, src, ndst, max_dst, out, ld, st);
    case 2: return launch_sq<2, OT>(c, indptr, src, ndst, max_dst, out, ld, st);
    case 3: return launch_sq<3, OT>(c, indptr, src, ndst, max_dst, out, ld, st);
    case 4: return launch_sq<4, OT>(c, indptr, src, ndst, max_dst, out, ld, st);
    case 5: return launch_sq<5, OT>(c, indptr, src, ndst, max_dst, out, ld, st);
    case 6: return launch_sq<6, OT>(c, indptr, src, ndst, max_dst, out, ld, st);
    case 7: return launch_sq<7, OT>(c, indptr, src, ndst, max_dst, out, ld, st);
    case 8: return launch_sq<8, OT>(c, indptr, src, ndst, max_dst, out, ld, st);
  }
  set_error("bad SQ k %d", c->bits);
  return FG_EUSAGE;
}

template <int W, typename OT>
int launch_vq(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
              const int64_t* ndst, int64_t max_dst, void* out, int64_t ld, cudaStream_t st) {
  const int64_t book_bytes = (int64_t)c->num_parts * c->length * W * 4;
  const int64_t stage_bytes = (kTD + 1 + kSrcCap) * 4;
  const int64_t ntiles = ceil_div(max_dst, kTD);
  if (c->bits != 8) {
    auto kern = k_vq_mean_bits<W, OT>;
    const int grid = (int)min64(ntiles, (int64_t)sm_count() * 2);
    kern<<<grid, 512, stage_bytes, st>>>(c->rows, c->d, c->row_stride, c->bits,
                                         (const float*)c->table, c->length, c->num_parts, indptr,
                                         src, ndst, max_dst, (OT*)out, ld);
    FG_LAUNCH_CHECK();
    return FG_OK;
  }
  const int64_t smem2 = ((book_bytes + 15) & ~15ll) + stage_bytes;
  if (smem2 <= 110 * 1024 || smem2 <= 220 * 1024) {
    const int per_sm = smem2 <= 110 * 1024 ? 2 : 1;
    auto kern = k_vq_mean8<W, OT, true>;
    FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem2));
    const int grid = (int)min64(ntiles, (int64_t)sm_count() * per_sm);
    kern<<<grid, 512, smem2, st>>>(c->rows, c->d, c->row_stride, (const float*)c->table,
                                   c->length, c->num_parts, indptr, src, ndst, max_dst, (OT*)out,
                                   ld);
  } else {
    auto kern = k_vq_mean8<W, OT, false>;
    const int grid = (int)min64(ntiles, (int64_t)sm_count() * 2);
    kern<<<grid, 512, stage_bytes, st>>>(c->rows, c->d, c->row_stride, (const float*)c->table,
                                         c->length, c->num_parts, indptr, src, ndst, max_dst,
                                         (OT*)out, ld);
  }
  FG_LAUNCH_CHECK();
  return FG_OK;
}

template <typename OT>
int dispatch_vq(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                const int64_t* ndst, int64_t max_dst, void* out, int64_t ld, cudaStream_t st) {
  switch (c->width) {
    case 1: return launch_vq<1, OT>(c, indptr, src, ndst, max_dst, out, ld, st);
    case 2: return launch_vq<2, OT>(c, indptr, src, ndst, max_dst, out, ld, st);
    case 4: return launch_vq<4, OT>(c, indptr, src, ndst, max_dst, out, ld, st);
    case 8: return launch_vq<8, OT>(c, indptr, src, ndst, max_dst, out, ld, st);
    case 16: return launch_vq<16, OT>(c, indptr, src, ndst, max_dst, out, ld, st);
  }
  set_error("fused VQ mean supports width in {1,2,4,8,16}, got %d", c->width);
  return FG_EUSAGE;
}

}  // namespace fg

using namespace fg;

extern "C" int fg_gather_dequant_mean(const fg_codec_desc* c, const int32_t* indptr,
                                      const int32_t* src, const int64_t* ndst, int64_t max_dst,
                                      void* out, int64_t out_ld, int out_dtype, void* s) {
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
               ? dispatch_sq<float>(c, indptr, src, ndst, max_dst, out, ld, st)
               : dispatch_sq<__nv_bfloat16>(c, indptr, src, ndst, max_dst, out, ld, st);
  }
  if (c->kind == FG_CODEC_VQ) {
    FG_CHECK_ARG(c->bits >= 1 && c->bits <= 16, "bad VQ code bits");
    FG_CHECK_ARG(c->bits != 8 || c->row_stride >= ((c->num_parts + 31) / 32) * 32,
                 "8-bit VQ rows must be padded to 32 bytes");
    return out_dtype == FG_OUT_F32
               ? dispatch_vq<float>(c, indptr, src, ndst, max_dst, out, ld, st)
               : dispatch_vq<__nv_bfloat16>(c, indptr, src, ndst, max_dst, out, ld, st);
  }
  set_error("unknown codec kind %d", c->kind);
  return FG_EUSAGE;
}
