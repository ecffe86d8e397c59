// Hidden-layer block mean used by SAGE layers 2..L (the fused layer-1
// gather-dequant-mean lives in fg_fused.cu).
//
// Semantics: out[v] = (1/cnt_v) * sum over picks e of v of h[local[e]], the
// row-stochastic mean of factors.py:108-114 over hidden rows; backward
// scatters grad/cnt with fp32 vector atomics.  HBM/L2 bound.
#include "fg_common.cuh"

namespace fg {

__device__ __forceinline__ int64_t live_count(const int64_t* p, int64_t cap) {
  const int64_t v = *p;
  return v < cap ? v : cap;
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

// RELU: apply max(0, .) to the source rows as they are loaded (the SAGE
// activation of the previous layer, fused so it never makes its own pass).
template <bool RELU>
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
            for (int j = 0; j < 8; ++j) acc[j] += RELU ? fmaxf(f[j], 0.f) : f[j];
          }
        }
      }
      if (cnt) {
        const float inv = 1.0f / (float)cnt;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] *= inv;
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

// fp32 gradient accumulator -> bf16; with `mask` (the pre-activation bf16
// rows) multiplies by relu'(x) = (x > 0), i.e. threshold_backward fused in.
__global__ void k_f32_to_bf16(const float* __restrict__ in, int64_t n8,
                              const uint16_t* __restrict__ mask, uint16_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n8;
       t += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = reinterpret_cast<const float4*>(in)[2 * t];
    const float4 b = reinterpret_cast<const float4*>(in)[2 * t + 1];
    float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    if (mask) {
      float m[8];
      bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(mask) + t), m);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = m[j] > 0.f ? f[j] : 0.f;
    }
    reinterpret_cast<uint4*>(out)[t] = f32_to_bf16x8(f);
  }
}

}  // namespace fg

using namespace fg;

extern "C" {

int fg_block_mean_fwd(const uint16_t* h, int64_t H, const int32_t* indptr, const int32_t* srcl,
                      const int64_t* ndst, int64_t max_dst, uint16_t* out, int relu_in,
                      void* s) {
  FG_CHECK_ARG(H % 8 == 0, "hidden dim must be a multiple of 8");
  if (max_dst == 0) return FG_OK;
  const int64_t total = max_dst * (H / 8);
  if (relu_in)
    k_block_mean_fwd<true><<<grid_for(total, 256), 256, 0, as_stream(s)>>>(h, H, indptr, srcl,
                                                                           ndst, max_dst, out);
  else
    k_block_mean_fwd<false><<<grid_for(total, 256), 256, 0, as_stream(s)>>>(h, H, indptr, srcl,
                                                                            ndst, max_dst, out);
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

int fg_f32_to_bf16(const float* in, int64_t count, const uint16_t* relu_mask, uint16_t* out,
                   void* s) {
  FG_CHECK_ARG(count % 8 == 0, "count must be a multiple of 8");
  if (count == 0) return FG_OK;
  k_f32_to_bf16<<<grid_for(count / 8, 256), 256, 0, as_stream(s)>>>(in, count / 8, relu_mask,
                                                                    out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

}  // extern "C"
