// Fused gather -> decode -> mean kernels (the north-star hot path) and the
// hidden-layer block mean used by SAGE layers 2..L.
//
// Semantics: out[v] = (1/cnt_v) * sum over the sampled picks u of v of
// decode(u), the row-stochastic mean D̂⁻¹Â of pkg/src/featgrind/factors.py:
// 108-114 restricted to the sampled block; decode(u) is exactly
// dequantize_sq (sq.py:132-153) or decode_vq (vq.py:330-344).  Decoded rows
// exist only in registers: HBM sees the packed code rows and the aggregate.
//
// Roofline: HBM-bound.  Algorithmic bytes per launch
//   E * (row_bytes + 4) + N_dst * (4 + d * out_bytes)
// (E picks read one code row + one int32 source id; each destination reads
// one indptr entry and writes one output row).  Decode tables stay on chip:
//   SQ  - 2^k-entry LUT replicated 32x across banks (conflict-free lookups),
//   VQ  - the whole codebook in shared memory (one CTA per SM).
#include "fg_common.cuh"

namespace fg {

__device__ __forceinline__ int64_t live_count(const int64_t* p, int64_t cap) {
  const int64_t v = *p;
  return v < cap ? v : cap;
}

// ------------------------------------------------------------------- SQ
// Thread owns 16 consecutive codes (16*k bits = 2k bytes) of one destination
// row; CHUNK_BYTES = 2k.  LUT replicated per lane: s_lut[q * 32 + lane].
template <int K, typename OT>
__global__ void __launch_bounds__(256)
k_sq_mean(const uint8_t* __restrict__ rows, int64_t d, int64_t stride,
          const float* __restrict__ lut, const int32_t* __restrict__ indptr,
          const int32_t* __restrict__ src, const int64_t* __restrict__ ndst_dev,
          int64_t max_dst, OT* __restrict__ out) {
  constexpr int Q = 1 << K;
  constexpr int CB = 2 * K;  // chunk bytes
  extern __shared__ float s_lut[];  // [Q][32]
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < Q * 32; i += blockDim.x) s_lut[i] = lut[i >> 5];
  __syncthreads();
  const int64_t live = live_count(ndst_dev, max_dst);
  const int64_t chunks = (d + 15) >> 4;
  const int64_t total = max_dst * chunks;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / chunks;
    const int64_t c = t - v * chunks;
    const int64_t j0 = c * 16;
    const int nval = (int)min64(16, d - j0);
    float acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.f;
    int cnt = 0;
    if (v < live) {
      const int32_t e0 = indptr[v], e1 = indptr[v + 1];
      cnt = e1 - e0;
      const int64_t boff = c * CB;
      for (int32_t e = e0; e < e1; e += 4) {
        uint64_t w[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          w[u][0] = w[u][1] = 0;
          if (e + u < e1) {
            const uint8_t* p = rows + (int64_t)src[e + u] * stride + boff;
            if constexpr (CB == 16) {
              const uint4 q = ldg_stream16(p);
              w[u][0] = ((uint64_t)q.y << 32) | q.x;
              w[u][1] = ((uint64_t)q.w << 32) | q.z;
            } else if constexpr (CB == 8) {
              const uint2 q = ldg_stream8(p);
              w[u][0] = ((uint64_t)q.y << 32) | q.x;
            } else if constexpr (CB == 4) {
              w[u][0] = ldg_stream4(p);
            } else if constexpr (CB == 2) {
              w[u][0] = *reinterpret_cast<const uint16_t*>(p);
            } else {
#pragma unroll
              for (int b = 0; b < CB; ++b) {
                const uint64_t byte = p[b];
                if (b < 8) w[u][0] |= byte << (8 * b); else w[u][1] |= byte << (8 * (b - 8));
              }
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (e + u < e1) {
            // bytes are little-endian packed in w (byte b at bits 8b); codes
            // are MSB-first inside the byte stream.
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int bit = j * K;           // MSB-first bit offset
              const int byte = bit >> 3;
              const int inb = bit & 7;
              const uint64_t word = byte < 8 ? w[u][0] : w[u][1];
              const int bb = byte & 7;
              uint32_t q;
              if (K == 8 || (inb + K <= 8)) {
                const uint32_t by = (uint32_t)(word >> (8 * bb)) & 0xFFu;
                q = (by >> (8 - inb - K)) & (Q - 1);
              } else {  // straddles two bytes (K in {3,5,6,7})
                const int byte2 = byte + 1;
                const uint64_t word2 = byte2 < 8 ? w[u][0] : w[u][1];
                const uint32_t hi = (uint32_t)(word >> (8 * bb)) & 0xFFu;
                const uint32_t lo = (uint32_t)(word2 >> (8 * (byte2 & 7))) & 0xFFu;
                q = (((hi << 8) | lo) >> (16 - inb - K)) & (Q - 1);
              }
              acc[j] += s_lut[q * 32 + lane];
            }
          }
        }
      }
    }
    OT* o = out + v * d + j0;
    const float inv_cnt = cnt;  // exact small integer
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < nval) store_out(o + j, cnt ? acc[j] / inv_cnt : 0.f);
  }
}

// ------------------------------------------------------------------- VQ
// Thread per (destination, part).  Whole codebook [P][L][W] staged in smem.
template <int W, typename OT, bool SMEM>
__global__ void __launch_bounds__(1024)
k_vq_mean(const uint8_t* __restrict__ rows, int64_t d, int64_t stride, int bits,
          const float* __restrict__ books, int length, int parts,
          const int32_t* __restrict__ indptr, const int32_t* __restrict__ src,
          const int64_t* __restrict__ ndst_dev, int64_t max_dst, OT* __restrict__ out) {
  extern __shared__ float4 s_book4[];
  const float* book = books;
  if constexpr (SMEM) {
    const int64_t nf = (int64_t)parts * length * W;
    const float4* g4 = reinterpret_cast<const float4*>(books);
    for (int64_t i = threadIdx.x; i < nf / 4; i += blockDim.x) s_book4[i] = g4[i];
    for (int64_t i = (nf & ~3ll) + threadIdx.x; i < nf; i += blockDim.x)
      reinterpret_cast<float*>(s_book4)[i] = books[i];
    __syncthreads();
    book = reinterpret_cast<const float*>(s_book4);
  }
  const int64_t live = live_count(ndst_dev, max_dst);
  const int64_t total = max_dst * parts;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / parts;
    const int p = (int)(t - v * parts);
    float acc[W];
#pragma unroll
    for (int j = 0; j < W; ++j) acc[j] = 0.f;
    int cnt = 0;
    if (v < live) {
      const int32_t e0 = indptr[v], e1 = indptr[v + 1];
      cnt = e1 - e0;
      const float* pb = book + (int64_t)p * length * W;
      for (int32_t e = e0; e < e1; e += 4) {
        uint32_t code[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          code[u] = 0;
          if (e + u < e1) {
            const uint8_t* row = rows + (int64_t)src[e + u] * stride;
            if (bits == 8) {
              code[u] = __ldg(row + p);
            } else {
              const int64_t bit0 = (int64_t)p * bits;
              const uint8_t* b = row + (bit0 >> 3);
              const int sh = (int)(bit0 & 7);
              uint32_t wv = (uint32_t)__ldg(b) << 16;
              if (sh + bits > 8) wv |= (uint32_t)__ldg(b + 1) << 8;
              if (sh + bits > 16) wv |= __ldg(b + 2);
              code[u] = (wv >> (24 - sh - bits)) & ((1u << bits) - 1u);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (e + u < e1) {
            const float* ent = pb + (int64_t)code[u] * W;
            if constexpr (W % 4 == 0) {
#pragma unroll
              for (int j = 0; j < W; j += 4) {
                const float4 q = *reinterpret_cast<const float4*>(ent + j);
                acc[j] += q.x; acc[j + 1] += q.y; acc[j + 2] += q.z; acc[j + 3] += q.w;
              }
            } else {
#pragma unroll
              for (int j = 0; j < W; ++j) acc[j] += ent[j];
            }
          }
        }
      }
    }
    const int lo = p * W;
    const int wp = (int)min64(W, d - lo);
    OT* o = out + v * d + lo;
    const float fc = cnt;
#pragma unroll
    for (int j = 0; j < W; ++j)
      if (j < wp) store_out(o + j, cnt ? acc[j] / fc : 0.f);
  }
}

// --------------------------------------------------- hidden block mean
// bf16 [*, H] source rows addressed by local index; thread per 8 columns.
__device__ __forceinline__ void bf16x8_to_f32(const uint4 q, float* f) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ uint4 f32_to_bf16x8(const float* f) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 b = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    w[i] = *reinterpret_cast<const uint32_t*>(&b);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void __launch_bounds__(256)
k_block_mean_fwd(const uint16_t* __restrict__ h, int64_t H, const int32_t* __restrict__ indptr,
                 const int32_t* __restrict__ srcl, const int64_t* __restrict__ ndst_dev,
                 int64_t max_dst, uint16_t* __restrict__ out) {
  const int64_t live = live_count(ndst_dev, max_dst);
  const int64_t chunks = H >> 3;
  const int64_t total = max_dst * chunks;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / chunks, c = t - v * chunks;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int cnt = 0;
    if (v < live) {
      const int32_t e0 = indptr[v], e1 = indptr[v + 1];
      cnt = e1 - e0;
      for (int32_t e = e0; e < e1; e += 4) {
        uint4 q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (e + u < e1)
            q[u] = __ldg(reinterpret_cast<const uint4*>(h + (int64_t)srcl[e + u] * H) + c);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (e + u < e1) {
            float f[8];
            bf16x8_to_f32(q[u], f);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] += f[j];
          }
        }
      }
      if (cnt) {
        const float fc = cnt;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = acc[j] / fc;
      }
    }
    reinterpret_cast<uint4*>(out + v * H)[c] = f32_to_bf16x8(acc);
  }
}

__global__ void __launch_bounds__(256)
k_block_mean_bwd(const uint16_t* __restrict__ g, int64_t H, const int32_t* __restrict__ indptr,
                 const int32_t* __restrict__ srcl, const int64_t* __restrict__ ndst_dev,
                 int64_t max_dst, float* __restrict__ gsrc) {
  const int64_t live = live_count(ndst_dev, max_dst);
  const int64_t chunks = H >> 3;
  const int64_t total = live * chunks;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / chunks, c = t - v * chunks;
    const int32_t e0 = indptr[v], e1 = indptr[v + 1];
    if (e1 == e0) continue;
    float f[8];
    bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(g + v * H) + c), f);
    const float fc = e1 - e0;
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = f[j] / fc;
    for (int32_t e = e0; e < e1; ++e) {
      float4* dst = reinterpret_cast<float4*>(gsrc + (int64_t)srcl[e] * H + c * 8);
      atomicAdd(dst, make_float4(f[0], f[1], f[2], f[3]));
      atomicAdd(dst + 1, make_float4(f[4], f[5], f[6], f[7]));
    }
  }
}

__global__ void k_f32_to_bf16(const float* __restrict__ in, int64_t n8, uint16_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n8;
       t += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = reinterpret_cast<const float4*>(in)[2 * t];
    const float4 b = reinterpret_cast<const float4*>(in)[2 * t + 1];
    const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    reinterpret_cast<uint4*>(out)[t] = f32_to_bf16x8(f);
  }
}

template <int K, typename OT>
int launch_sq_mean(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                   const int64_t* ndst, int64_t max_dst, void* out, cudaStream_t st) {
  const int smem = (1 << K) * 32 * (int)sizeof(float);
  auto kern = k_sq_mean<K, OT>;
  if (smem > 48 * 1024)
    FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int64_t total = max_dst * ((c->d + 15) / 16);
  kern<<<grid_for(total, 256, 6), 256, smem, st>>>(c->rows, c->d, c->row_stride,
                                                   (const float*)c->table, indptr, src, ndst,
                                                   max_dst, (OT*)out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

template <typename OT>
int dispatch_sq_mean(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                     const int64_t* ndst, int64_t max_dst, void* out, cudaStream_t st) {
  switch (c->bits) {
    case 1: return launch_sq_mean<1, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 2: return launch_sq_mean<2, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 3: return launch_sq_mean<3, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 4: return launch_sq_mean<4, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 5: return launch_sq_mean<5, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 6: return launch_sq_mean<6, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 7: return launch_sq_mean<7, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 8: return launch_sq_mean<8, OT>(c, indptr, src, ndst, max_dst, out, st);
  }
  set_error("bad SQ k %d", c->bits);
  return FG_EUSAGE;
}

template <int W, typename OT>
int launch_vq_mean(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                   const int64_t* ndst, int64_t max_dst, void* out, cudaStream_t st) {
  const int64_t book_bytes = (int64_t)c->num_parts * c->length * W * sizeof(float);
  const int64_t total = max_dst * c->num_parts;
  if (book_bytes <= 200 * 1024) {
    auto kern = k_vq_mean<W, OT, true>;
    FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)book_bytes));
    const int threads = 1024;
    const int grid = (int)min64(ceil_div(total, threads), sm_count());
    kern<<<grid, threads, book_bytes, st>>>(c->rows, c->d, c->row_stride, c->bits,
                                            (const float*)c->table, c->length, c->num_parts,
                                            indptr, src, ndst, max_dst, (OT*)out);
  } else {
    auto kern = k_vq_mean<W, OT, false>;
    kern<<<grid_for(total, 256, 8), 256, 0, st>>>(c->rows, c->d, c->row_stride, c->bits,
                                                  (const float*)c->table, c->length, c->num_parts,
                                                  indptr, src, ndst, max_dst, (OT*)out);
  }
  FG_LAUNCH_CHECK();
  return FG_OK;
}

template <typename OT>
int dispatch_vq_mean(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                     const int64_t* ndst, int64_t max_dst, void* out, cudaStream_t st) {
  switch (c->width) {
    case 1: return launch_vq_mean<1, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 2: return launch_vq_mean<2, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 4: return launch_vq_mean<4, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 8: return launch_vq_mean<8, OT>(c, indptr, src, ndst, max_dst, out, st);
    case 16: return launch_vq_mean<16, OT>(c, indptr, src, ndst, max_dst, out, st);
  }
  set_error("fused VQ mean supports width in {1,2,4,8,16}, got %d", c->width);
  return FG_EUSAGE;
}

}  // namespace fg

using namespace fg;

extern "C" {

int fg_gather_dequant_mean(const fg_codec_desc* c, const int32_t* indptr, const int32_t* src,
                           const int64_t* ndst, int64_t max_dst, void* out, int out_dtype,
                           void* s) {
  FG_CHECK_ARG(c != nullptr && indptr != nullptr && ndst != nullptr, "null argument");
  FG_CHECK_ARG(c->elem_bits == 32, "fused aggregate needs a float32 decode table");
  FG_CHECK_ARG(out_dtype == FG_OUT_F32 || out_dtype == FG_OUT_BF16, "out dtype must be f32 or bf16");
  if (max_dst == 0) return FG_OK;
  cudaStream_t st = as_stream(s);
  if (c->kind == FG_CODEC_SQ) {
    FG_CHECK_ARG(c->row_stride % 16 == 0, "row stride must be a multiple of 16");
    FG_CHECK_ARG(c->row_stride >= ((c->d + 15) / 16) * 2 * c->bits,
                 "SQ row stride must cover ceil(d/16)*2k bytes (whole 16-code chunks)");
    return out_dtype == FG_OUT_F32
               ? dispatch_sq_mean<float>(c, indptr, src, ndst, max_dst, out, st)
               : dispatch_sq_mean<__nv_bfloat16>(c, indptr, src, ndst, max_dst, out, st);
  }
  if (c->kind == FG_CODEC_VQ) {
    FG_CHECK_ARG(c->bits >= 1 && c->bits <= 16, "bad VQ code bits");
    return out_dtype == FG_OUT_F32
               ? dispatch_vq_mean<float>(c, indptr, src, ndst, max_dst, out, st)
               : dispatch_vq_mean<__nv_bfloat16>(c, indptr, src, ndst, max_dst, out, st);
  }
  set_error("unknown codec kind %d", c->kind);
  return FG_EUSAGE;
}

int fg_block_mean_fwd(const uint16_t* h, int64_t H, const int32_t* indptr, const int32_t* srcl,
                      const int64_t* ndst, int64_t max_dst, uint16_t* out, void* s) {
  FG_CHECK_ARG(H % 8 == 0, "hidden dim must be a multiple of 8");
  if (max_dst == 0) return FG_OK;
  const int64_t total = max_dst * (H / 8);
  k_block_mean_fwd<<<grid_for(total, 256), 256, 0, as_stream(s)>>>(h, H, indptr, srcl, ndst,
                                                                   max_dst, out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_block_mean_bwd(const uint16_t* g, int64_t H, const int32_t* indptr, const int32_t* srcl,
                      const int64_t* ndst, int64_t max_dst, float* gsrc, void* s) {
  FG_CHECK_ARG(H % 8 == 0, "hidden dim must be a multiple of 8");
  if (max_dst == 0) return FG_OK;
  const int64_t total = max_dst * (H / 8);
  k_block_mean_bwd<<<grid_for(total, 256), 256, 0, as_stream(s)>>>(g, H, indptr, srcl, ndst,
                                                                   max_dst, gsrc);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_f32_to_bf16(const float* in, int64_t count, uint16_t* out, void* s) {
  FG_CHECK_ARG(count % 8 == 0, "count must be a multiple of 8");
  if (count == 0) return FG_OK;
  k_f32_to_bf16<<<grid_for(count / 8, 256), 256, 0, as_stream(s)>>>(in, count / 8, out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

}  // extern "C"
