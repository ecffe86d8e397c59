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
// Latency structure.  A naive thread-per-(dst, part) loop walks the chain
// indptr -> src id -> code row -> lookup once per pick, which left the first
// version at 7 % of HBM peak.  Here a persistent CTA walks tiles of TD
// destinations: the tile's indptr slice and src ids are staged in shared
// memory with coalesced loads (two round trips for the whole tile), then every
// item thread issues ALL its code-row loads back to back (one round trip,
// up to 16 independent loads in flight per thread) before touching the decode
// tables.  Decode tables stay on chip:
//   SQ - 2^k-entry LUT replicated 32x across banks (conflict-free lookups);
//   VQ - the whole codebook in shared memory (two CTAs per SM fit 2x100 KB).
#include "fg_common.cuh"

namespace fg {

constexpr int kTD = 128;        // destinations per tile
constexpr int kMaxUnroll = 8;   // picks whose loads are issued together

__device__ __forceinline__ int64_t live_dst(const int64_t* p, int64_t cap) {
  const int64_t v = *p;
  return v < cap ? v : cap;
}

// Stage indptr[v0 .. v0+kTD] (clamped to max_dst) and the tile's src ids.
// Returns (e0, staged?) via references; s_src holds up to cap ids.
__device__ __forceinline__ void stage_tile(const int32_t* __restrict__ indptr,
                                           const int32_t* __restrict__ src, int64_t v0,
                                           int64_t max_dst, int32_t* s_ip, int32_t* s_src,
                                           int cap, int32_t& e0, int32_t& ecount) {
  for (int t = threadIdx.x; t <= kTD; t += blockDim.x) {
    const int64_t v = min64(v0 + t, max_dst);
    s_ip[t] = __ldg(indptr + v);
  }
  __syncthreads();
  e0 = s_ip[0];
  ecount = s_ip[kTD] - e0;
  if (ecount <= cap)
    for (int t = threadIdx.x; t < ecount; t += blockDim.x) s_src[t] = __ldg(src + e0 + t);
  __syncthreads();
}

// ------------------------------------------------------------------- SQ
// Item = (destination, 16-code chunk): 16*K bits = 2K bytes of each row.
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
__device__ __forceinline__ void sq_accumulate(uint64_t w0, uint64_t w1, const float* s_lut,
                                              int lane, float* acc) {
  constexpr int Q = 1 << K;
  // bytes little-endian in (w0, w1); codes MSB-first in the byte stream
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int bit = j * K;
    const int byte = bit >> 3;
    const int inb = bit & 7;
    const uint64_t word = byte < 8 ? w0 : w1;
    uint32_t q;
    if (K == 8 || inb + K <= 8) {
      const uint32_t by = (uint32_t)(word >> (8 * (byte & 7))) & 0xFFu;
      q = (by >> (8 - inb - K)) & (Q - 1);
    } else {
      const int byte2 = byte + 1;
      const uint64_t word2 = byte2 < 8 ? w0 : w1;
      const uint32_t hi = (uint32_t)(word >> (8 * (byte & 7))) & 0xFFu;
      const uint32_t lo = (uint32_t)(word2 >> (8 * (byte2 & 7))) & 0xFFu;
      q = (((hi << 8) | lo) >> (16 - inb - K)) & (Q - 1);
    }
    acc[j] += s_lut[q * 32 + lane];
  }
}

template <int K, typename OT>
__global__ void __launch_bounds__(512, 2)
k_sq_mean(const uint8_t* __restrict__ rows, int64_t d, int64_t stride,
          const float* __restrict__ lut, const int32_t* __restrict__ indptr,
          const int32_t* __restrict__ src, const int64_t* __restrict__ ndst_dev,
          int64_t max_dst, OT* __restrict__ out, int src_cap) {
  constexpr int Q = 1 << K;
  constexpr int CB = 2 * K;
  extern __shared__ float s_mem[];
  float* s_lut = s_mem;                                      // [Q][32]
  int32_t* s_ip = reinterpret_cast<int32_t*>(s_mem + Q * 32);  // [kTD + 1]
  int32_t* s_src = s_ip + kTD + 1;                           // [src_cap]
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < Q * 32; i += blockDim.x) s_lut[i] = lut[i >> 5];
  const int64_t live = live_dst(ndst_dev, max_dst);
  const int chunks = (int)((d + 15) >> 4);
  const int64_t ntiles = (max_dst + kTD - 1) / kTD;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t v0 = tile * kTD;
    int32_t e0, ecount;
    stage_tile(indptr, src, v0, max_dst, s_ip, s_src, src_cap, e0, ecount);
    const bool staged = ecount <= src_cap;
    const int items = kTD * chunks;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int vl = it / chunks;
      const int c = it - vl * chunks;
      const int64_t v = v0 + vl;
      if (v >= max_dst) break;
      float acc[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = 0.f;
      const int a = s_ip[vl] - e0, b = s_ip[vl + 1] - e0;
      const int cnt = v < live ? b - a : 0;
      const int64_t boff = (int64_t)c * CB;
      for (int base = 0; base < cnt; base += kMaxUnroll) {
        uint64_t w[kMaxUnroll][2];
#pragma unroll
        for (int u = 0; u < kMaxUnroll; ++u) {
          if (base + u < cnt) {
            const int e = a + base + u;
            const int32_t sid = staged ? s_src[e] : __ldg(src + e0 + e);
            load_chunk<K>(rows + (int64_t)sid * stride + boff, w[u][0], w[u][1]);
          }
        }
#pragma unroll
        for (int u = 0; u < kMaxUnroll; ++u)
          if (base + u < cnt) sq_accumulate<K>(w[u][0], w[u][1], s_lut, lane, acc);
      }
      const int j0 = c * 16;
      const int nval = (int)min64(16, d - j0);
      OT* o = out + v * d + j0;
      const float fc = (float)cnt;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < nval) store_out(o + j, cnt ? acc[j] / fc : 0.f);
    }
    __syncthreads();  // s_ip / s_src reused by the next tile
  }
}

// ------------------------------------------------------------------- VQ
// Item = (destination, part).  Codebook [P][L][W] fp32 in smem (SMEM) or
// read through L1/L2 (codebooks above the smem budget, e.g. L=2048).
template <int W, typename OT, bool SMEM>
__global__ void __launch_bounds__(1024, 2)
k_vq_mean(const uint8_t* __restrict__ rows, int64_t d, int64_t stride, int bits,
          const float* __restrict__ books, int length, int parts,
          const int32_t* __restrict__ indptr, const int32_t* __restrict__ src,
          const int64_t* __restrict__ ndst_dev, int64_t max_dst, OT* __restrict__ out,
          int src_cap) {
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
  const int64_t ntiles = (max_dst + kTD - 1) / kTD;
  const uint32_t cmask = (1u << bits) - 1u;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t v0 = tile * kTD;
    int32_t e0, ecount;
    stage_tile(indptr, src, v0, max_dst, s_ip, s_src, src_cap, e0, ecount);
    const bool staged = ecount <= src_cap;
    const int items = kTD * parts;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int vl = it / parts;
      const int p = it - vl * parts;
      const int64_t v = v0 + vl;
      if (v >= max_dst) break;
      float acc[W];
#pragma unroll
      for (int j = 0; j < W; ++j) acc[j] = 0.f;
      const int a = s_ip[vl] - e0, b = s_ip[vl + 1] - e0;
      const int cnt = v < live ? b - a : 0;
      const float* pb = book + (int64_t)p * length * W;
      const int64_t bit0 = (int64_t)p * bits;
      const int64_t byte0 = bit0 >> 3;
      const int sh = (int)(bit0 & 7);
      for (int base = 0; base < cnt; base += kMaxUnroll) {
        uint32_t code[kMaxUnroll];
#pragma unroll
        for (int u = 0; u < kMaxUnroll; ++u) {
          if (base + u < cnt) {
            const int e = a + base + u;
            const int32_t sid = staged ? s_src[e] : __ldg(src + e0 + e);
            const uint8_t* rb = rows + (int64_t)sid * stride + byte0;
            if (bits == 8) {
              code[u] = __ldg(rb);
            } else {
              uint32_t wv = (uint32_t)__ldg(rb) << 16;
              if (sh + bits > 8) wv |= (uint32_t)__ldg(rb + 1) << 8;
              if (sh + bits > 16) wv |= __ldg(rb + 2);
              code[u] = (wv >> (24 - sh - bits)) & cmask;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kMaxUnroll; ++u) {
          if (base + u < cnt) {
            const float* ent = pb + (int64_t)code[u] * W;
            if constexpr (W % 4 == 0) {
#pragma unroll
              for (int j = 0; j < W; j += 4) {
                const float4 q = SMEM ? *reinterpret_cast<const float4*>(ent + j)
                                      : __ldg(reinterpret_cast<const float4*>(ent + j));
                acc[j] += q.x; acc[j + 1] += q.y; acc[j + 2] += q.z; acc[j + 3] += q.w;
              }
            } else {
#pragma unroll
              for (int j = 0; j < W; ++j) acc[j] += ent[j];
            }
          }
        }
      }
      const int lo = p * W;
      const int wp = (int)min64(W, d - lo);
      OT* o = out + v * d + lo;
      const float fc = (float)cnt;
#pragma unroll
      for (int j = 0; j < W; ++j)
        if (j < wp) store_out(o + j, cnt ? acc[j] / fc : 0.f);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ launchers
constexpr int kSrcCap = kTD * 16;  // staged src ids per tile (fanout <= 16 fully staged)

template <int K, typename OT>
int launch_sq(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
              const int64_t* ndst, int64_t max_dst, void* out, cudaStream_t st) {
  const int smem = (1 << K) * 32 * 4 + (kTD + 1 + kSrcCap) * 4;
  auto kern = k_sq_mean<K, OT>;
  FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int64_t ntiles = ceil_div(max_dst, kTD);
  const int grid = (int)min64(ntiles, (int64_t)sm_count() * 2);
  kern<<<grid, 512, smem, st>>>(c->rows, c->d, c->row_stride, (const float*)c->table, indptr,
                                src, ndst, max_dst, (OT*)out, kSrcCap);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

template <typename OT>
int dispatch_sq(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                const int64_t* ndst, int64_t max_dst, void* out, cudaStream_t st) {
  switch (c->bits) {
    case 1: return launch_sq<1, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 2: return launch_sq<2, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 3: return launch_sq<3, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 4: return launch_sq<4, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 5: return launch_sq<5, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 6: return launch_sq<6, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 7: return launch_sq<7, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 8: return launch_sq<8, OT>(c, indptr, src, ndst, max_dst, out, st);
  }
  set_error("bad SQ k %d", c->bits);
  return FG_EUSAGE;
}

template <int W, typename OT>
int launch_vq(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
              const int64_t* ndst, int64_t max_dst, void* out, cudaStream_t st) {
  const int64_t book_bytes = (int64_t)c->num_parts * c->length * W * 4;
  const int64_t stage_bytes = (kTD + 1 + kSrcCap) * 4;
  const int64_t ntiles = ceil_div(max_dst, kTD);
  const bool in_smem = book_bytes + stage_bytes + 16 <= 110 * 1024;  // two CTAs per SM
  const bool in_smem1 = !in_smem && book_bytes + stage_bytes + 16 <= 220 * 1024;
  if (in_smem || in_smem1) {
    auto kern = k_vq_mean<W, OT, true>;
    const int smem = (int)(((book_bytes + 15) & ~15ll) + stage_bytes);
    FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int grid = (int)min64(ntiles, (int64_t)sm_count() * (in_smem ? 2 : 1));
    kern<<<grid, 1024, smem, st>>>(c->rows, c->d, c->row_stride, c->bits,
                                   (const float*)c->table, c->length, c->num_parts, indptr, src,
                                   ndst, max_dst, (OT*)out, kSrcCap);
  } else {
    auto kern = k_vq_mean<W, OT, false>;
    const int smem = (int)stage_bytes;
    FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int grid = (int)min64(ntiles, (int64_t)sm_count() * 2);
    kern<<<grid, 1024, smem, st>>>(c->rows, c->d, c->row_stride, c->bits,
                                   (const float*)c->table, c->length, c->num_parts, indptr, src,
                                   ndst, max_dst, (OT*)out, kSrcCap);
  }
  FG_LAUNCH_CHECK();
  return FG_OK;
}

template <typename OT>
int dispatch_vq(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                const int64_t* ndst, int64_t max_dst, void* out, cudaStream_t st) {
  switch (c->width) {
    case 1: return launch_vq<1, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 2: return launch_vq<2, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 4: return launch_vq<4, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 8: return launch_vq<8, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 16: return launch_vq<16, OT>(c, indptr, src, ndst, max_dst, out, st);
  }
  set_error("fused VQ mean supports width in {1,2,4,8,16}, got %d", c->width);
  return FG_EUSAGE;
}

}  // namespace fg

using namespace fg;

extern "C" int fg_gather_dequant_mean(const fg_codec_desc* c, const int32_t* indptr,
                                      const int32_t* src, const int64_t* ndst, int64_t max_dst,
                                      void* out, int out_dtype, void* s) {
  FG_CHECK_ARG(c != nullptr && indptr != nullptr && ndst != nullptr, "null argument");
  FG_CHECK_ARG(c->elem_bits == 32, "fused aggregate needs a float32 decode table");
  FG_CHECK_ARG(out_dtype == FG_OUT_F32 || out_dtype == FG_OUT_BF16,
               "out dtype must be f32 or bf16");
  if (max_dst == 0) return FG_OK;
  cudaStream_t st = as_stream(s);
  if (c->kind == FG_CODEC_SQ) {
    FG_CHECK_ARG(c->row_stride % 16 == 0, "row stride must be a multiple of 16");
    FG_CHECK_ARG(c->row_stride >= ((c->d + 15) / 16) * 2 * c->bits,
                 "SQ row stride must cover ceil(d/16)*2k bytes (whole 16-code chunks)");
    return out_dtype == FG_OUT_F32 ? dispatch_sq<float>(c, indptr, src, ndst, max_dst, out, st)
                                   : dispatch_sq<__nv_bfloat16>(c, indptr, src, ndst, max_dst,
                                                                out, st);
  }
  if (c->kind == FG_CODEC_VQ) {
    FG_CHECK_ARG(c->bits >= 1 && c->bits <= 16, "bad VQ code bits");
    return out_dtype == FG_OUT_F32 ? dispatch_vq<float>(c, indptr, src, ndst, max_dst, out, st)
                                   : dispatch_vq<__nv_bfloat16>(c, indptr, src, ndst, max_dst,
                                                                out, st);
  }
  set_error("unknown codec kind %d", c->kind);
  return FG_EUSAGE;
}
