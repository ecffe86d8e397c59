// Hidden-layer block mean used by SAGE layers 2..L (the fused layer-1
// gather-dequant-mean lives in fg_fused.cu).
//
// Semantics: out[v] = (1/cnt_v) * sum over picks e of v of h[local[e]], the
// row-stochastic mean of factors.py:108-114 over hidden rows; backward
// scatters grad/cnt with fp32 vector atomics.  HBM/L2 bound.
#include "fg_common.cuh"
#include "fg_scan.cuh"

#include <cub/block/block_scan.cuh>

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
template <bool RELU, bool WT, bool MB = false>
__global__ void __launch_bounds__(256)
k_block_mean_fwd(const uint16_t* __restrict__ h, int64_t H, const int32_t* __restrict__ indptr,
                 const int32_t* __restrict__ srcl, const int64_t* __restrict__ ndst_dev,
                 int64_t max_dst, uint16_t* __restrict__ out, int64_t out_ld,
                 const float* __restrict__ ew, uint8_t* __restrict__ mbits = nullptr) {
  const int64_t live = live_count(ndst_dev, max_dst);
  const int64_t chunks = H >> 3;
  const int64_t ochunks = out_ld >> 3;  // out_ld = H, or H + 8 with a ones column
  const int64_t total = max_dst * ochunks;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / ochunks, c = t - v * ochunks;
    if (c >= chunks) {  // bias column chunk: [1, 0, ..., 0]
      reinterpret_cast<uint4*>(out + v * out_ld)[c] = make_uint4(0x3F80u, 0u, 0u, 0u);
      continue;
    }
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int cnt = 0;
    if (v < live) {
      const int32_t e0 = indptr[v], e1 = indptr[v + 1];
      cnt = e1 - e0;
      // 8 picks per batch: the src-id loads, then the 8 row loads, all in flight
      for (int32_t e = e0; e < e1; e += 8) {
        int32_t sl[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e + u < e1) sl[u] = srcl[e + u];
        uint4 q[8];
        float wgt[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e + u < e1) {
            q[u] = __ldg(reinterpret_cast<const uint4*>(h + (int64_t)sl[u] * H) + c);
            if constexpr (WT) wgt[u] = __ldg(ew + e + u);
          }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (e + u < e1) {
            float f[8];
            bf16x8_to_f32(q[u], f);
            if constexpr (MB) {  // the source's ReLU mask byte (bit t = feature 8c+t) for
              uint32_t b = 0;    // the backward's edge-tiled dW (fg_wgrad.cu, mask_kind 2)
#pragma unroll
              for (int j = 0; j < 8; ++j) b |= (f[j] > 0.f ? 1u : 0u) << j;
              mbits[(int64_t)sl[u] * chunks + c] = (uint8_t)b;
            }
            if constexpr (WT) {
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[j] = fmaf(wgt[u], RELU ? fmaxf(f[j], 0.f) : f[j], acc[j]);
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[j] += RELU ? fmaxf(f[j], 0.f) : f[j];
            }
          }
        }
      }
      if (cnt && !WT) {
        const float inv = 1.0f / (float)cnt;
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] *= inv;
      }
    }
    reinterpret_cast<uint4*>(out + v * out_ld)[c] = f32_to_bf16x8(acc);
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

int fg_block_mean_fwd_bits(const uint16_t* h, int64_t H, const int32_t* indptr,
                           const int32_t* srcl, const int64_t* ndst, int64_t max_dst,
                           uint16_t* out, int64_t out_ld, const float* edge_w,
                           uint8_t* relu_bits, void* s) {
  FG_CHECK_ARG(H % 8 == 0 && relu_bits != nullptr, "hidden dim must be a multiple of 8");
  if (out_ld == 0) out_ld = H;
  FG_CHECK_ARG(out_ld == H || out_ld == H + 8, "out_ld must be H or H + 8 (ones column)");
  if (max_dst == 0) return FG_OK;
  const int64_t total = max_dst * (out_ld / 8);
  const int grid = grid_for(total, 256);
  cudaStream_t st = as_stream(s);
  if (edge_w)
    k_block_mean_fwd<true, true, true><<<grid, 256, 0, st>>>(h, H, indptr, srcl, ndst, max_dst,
                                                              out, out_ld, edge_w, relu_bits);
  else
    k_block_mean_fwd<true, false, true><<<grid, 256, 0, st>>>(h, H, indptr, srcl, ndst, max_dst,
                                                               out, out_ld, nullptr, relu_bits);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_block_mean_fwd(const uint16_t* h, int64_t H, const int32_t* indptr, const int32_t* srcl,
                      const int64_t* ndst, int64_t max_dst, uint16_t* out, int64_t out_ld,
                      int relu_in, const float* edge_w, void* s) {
  FG_CHECK_ARG(H % 8 == 0, "hidden dim must be a multiple of 8");
  if (out_ld == 0) out_ld = H;
  FG_CHECK_ARG(out_ld == H || out_ld == H + 8, "out_ld must be H or H + 8 (ones column)");
  if (max_dst == 0) return FG_OK;
  const int64_t total = max_dst * (out_ld / 8);
  const int grid = grid_for(total, 256);
  cudaStream_t st = as_stream(s);
  if (relu_in && edge_w)
    k_block_mean_fwd<true, true><<<grid, 256, 0, st>>>(h, H, indptr, srcl, ndst, max_dst, out,
                                                        out_ld, edge_w);
  else if (relu_in)
    k_block_mean_fwd<true, false><<<grid, 256, 0, st>>>(h, H, indptr, srcl, ndst, max_dst, out,
                                                         out_ld, nullptr);
  else if (edge_w)
    k_block_mean_fwd<false, true><<<grid, 256, 0, st>>>(h, H, indptr, srcl, ndst, max_dst, out,
                                                         out_ld, edge_w);
  else
    k_block_mean_fwd<false, false><<<grid, 256, 0, st>>>(h, H, indptr, srcl, ndst, max_dst, out,
                                                          out_ld, nullptr);
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

// ------------------------------------------- gather-form (transposed) bwd
// The block's transpose (source rank -> incoming edges) lets the backward of
// the hidden block mean be a deterministic gather instead of fp32 atomics:
//   grad_src[r] = act'(h[r]) * sum_{e in in(r)} grad_out[dst(e)] / cnt(dst(e))
// summed in edge order.  Built per batch from unique 64-bit keys
// (rank << 32 | edge), so any sort yields the same order.
namespace fg {

// counting-sort transpose: histogram of source ranks, exclusive scan,
// placement through atomic cursors (list order within a source is
// scheduling-dependent; the backward sums a handful of terms per source).
__global__ void k_t_hist(const int32_t* __restrict__ local, const int64_t* __restrict__ ne_dev,
                         int64_t cap_e, int32_t* __restrict__ cnt) {
  const int64_t ne = min64(*ne_dev, cap_e);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + local[e], 1);
}

// exclusive scan of the per-source counts (single pass, look-back);
// writes t_indptr and the placement cursors
constexpr int kTsPer = 8;
__global__ void __launch_bounds__(256)
k_t_scan(int64_t n, const int32_t* __restrict__ cnt, int32_t* __restrict__ t_indptr,
         int32_t* __restrict__ cursor, unsigned long long* status, unsigned int* ctr,
         unsigned int ntiles) {
  using BS = cub::BlockScan<unsigned long long, 256>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ unsigned int s_u32;
  __shared__ unsigned long long s_u64;
  const ScanState sc{status, ctr, ctr + 1};
  const unsigned int tile = scan_take_tile(sc, &s_u32);
  const int64_t i0 = (int64_t)tile * 256 * kTsPer + threadIdx.x * (int64_t)kTsPer;
  int32_t v[kTsPer];
  unsigned long long c = 0;
#pragma unroll
  for (int k = 0; k < kTsPer; ++k) {
    v[k] = i0 + k < n ? cnt[i0 + k] : 0;
    c += (unsigned long long)v[k];
  }
  unsigned long long excl, agg;
  BS(tmp).ExclusiveSum(c, excl, agg);
  const unsigned long long prefix = scan_tile_prefix(sc, tile, agg, &s_u64);
  int32_t pos = (int32_t)(prefix + excl);
#pragma unroll
  for (int k = 0; k < kTsPer; ++k) {
    if (i0 + k < n) {
      t_indptr[i0 + k] = pos;
      cursor[i0 + k] = pos;
    }
    pos += v[k];
  }
  if (scan_last_block(sc, ntiles, &s_u32) && threadIdx.x == 0)
    t_indptr[n] = (int32_t)(status[ntiles - 1] & kScanValMask);
}

// place every edge; t_dst receives the dst of the edge (found from indptr)
__global__ void k_t_place(const int32_t* __restrict__ local, const int64_t* __restrict__ ne_dev,
                          int64_t cap_e, const int32_t* __restrict__ indptr,
                          const int64_t* __restrict__ nd_dev, int64_t max_dst,
                          int32_t* __restrict__ cursor, int32_t* __restrict__ t_dst,
                          float* __restrict__ t_w, int fmax, const float* __restrict__ ew,
                          int32_t* __restrict__ t_eid) {
  const int64_t nd = min64(*nd_dev, max_dst);
  // thread per (destination, pick slot k < fmax): picks of v are contiguous
  // in [indptr[v], indptr[v+1]) and number at most fmax
  const int64_t total = nd * fmax;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / fmax;
    const int k = (int)(t - v * fmax);
    const int32_t e0 = indptr[v], e1 = indptr[v + 1];
    const int32_t e = e0 + k;
    if (e >= e1) continue;
    const int32_t slot = atomicAdd(cursor + local[e], 1);
    t_dst[slot] = (int32_t)v;
    t_w[slot] = ew ? ew[e] : 1.0f / (float)(e1 - e0);
    if (t_eid) t_eid[slot] = e;
  }
}

// Thread per (group of R consecutive source rows, 8-byte chunk of 4
// columns).  Most sources have one or two transposed edges, so a thread per
// row is a three-deep dependent load chain (t_indptr -> t_dst -> g row) with
// nothing else in flight; R rows per thread issue R chains side by side
// (8-byte chunks keep the R-way state in registers at 3 CTAs/SM).
__device__ __forceinline__ void bf16x4_to_f32(const uint2 q, float* f) {
  f[0] = __uint_as_float(q.x << 16);
  f[1] = __uint_as_float(q.x & 0xFFFF0000u);
  f[2] = __uint_as_float(q.y << 16);
  f[3] = __uint_as_float(q.y & 0xFFFF0000u);
}
__device__ __forceinline__ uint2 f32_to_bf16x4(const float* f) {
  const __nv_bfloat162 a = __floats2bfloat162_rn(f[0], f[1]);
  const __nv_bfloat162 b = __floats2bfloat162_rn(f[2], f[3]);
  return make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
}

// RELU: 0 none, 1 mask = the forward's bf16 h rows (relu' = h > 0), 2 mask =
// packed ReLU bits (H/8 bytes per row, bit t of byte c = feature 8c + t, as
// fg_block_mean_fwd_bits / fg_input_block_mean_fwd write them)
template <int RELU, int R>
__global__ void __launch_bounds__(256, 3)
k_block_mean_bwd_t(const uint16_t* __restrict__ g, int64_t H, int64_t g_ld,
                   const int32_t* __restrict__ t_indptr,
                   const int32_t* __restrict__ t_dst, const float* __restrict__ t_w,
                   const int64_t* __restrict__ nsrc_dev, int64_t cap_src,
                   const uint16_t* __restrict__ mask, const uint8_t* __restrict__ mbits,
                   uint16_t* __restrict__ out) {
  const int64_t chunks = H >> 2;
  const int64_t ngroups = (cap_src + R - 1) / R;
  const int64_t total = ngroups * chunks;
  const int64_t live = live_count(nsrc_dev, cap_src);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rg = t / chunks, c = t - rg * chunks;
    const int64_t r0 = rg * R;
    int32_t i0[R], i1[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      i0[u] = i1[u] = 0;
      if (r0 + u < live) {
        i0[u] = t_indptr[r0 + u];
        i1[u] = t_indptr[r0 + u + 1];
      }
    }
    int32_t v[R];
    float w[R];
#pragma unroll
    for (int u = 0; u < R; ++u)
      if (i0[u] < i1[u]) { v[u] = t_dst[i0[u]]; w[u] = t_w[i0[u]]; }
    uint2 q[R], mq[R];
    uint32_t mb[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      mq[u] = make_uint2(0u, 0u);
      mb[u] = 0u;
      if (RELU == 1 && r0 + u < live) mq[u] = __ldg(reinterpret_cast<const uint2*>(mask + (r0 + u) * H) + c);
      if (RELU == 2 && r0 + u < live) mb[u] = __ldg(mbits + (r0 + u) * (H >> 3) + (c >> 1));
      if (i0[u] < i1[u]) q[u] = __ldg(reinterpret_cast<const uint2*>(g + (int64_t)v[u] * g_ld) + c);
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int64_t r = r0 + u;
      if (r >= cap_src) break;
      float acc[4] = {0, 0, 0, 0};
      if (i0[u] < i1[u]) {
        float f[4];
        bf16x4_to_f32(q[u], f);
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = f[j] * w[u];
      }
      // remaining transposed edges of this row (hub sources), 4 at a time
      for (int32_t i = i0[u] + 1; i < i1[u]; i += 4) {
        uint2 qq[4];
        float sc[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (i + k < i1[u]) {
            sc[k] = t_w[i + k];
            qq[k] = __ldg(reinterpret_cast<const uint2*>(g + (int64_t)t_dst[i + k] * g_ld) + c);
          }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (i + k < i1[u]) {
            float f[4];
            bf16x4_to_f32(qq[k], f);
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] = fmaf(f[j], sc[k], acc[j]);
          }
      }
      if (RELU == 1) {
        float m[4];
        bf16x4_to_f32(mq[u], m);
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = m[j] > 0.f ? acc[j] : 0.f;
      }
      if (RELU == 2) {
        const uint32_t nib = mb[u] >> ((c & 1) * 4);
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = (nib >> j) & 1u ? acc[j] : 0.f;
      }
      // padded source rows (r >= live) get a zero gradient
      reinterpret_cast<uint2*>(out + r * H)[c] = f32_to_bf16x4(acc);
    }
  }
}

// ----------------------------------------------------------- flat Adam
// torch.optim.Adam semantics (L2 weight decay folded into the gradient) over
// one flat fp32 parameter buffer; the step counter lives on the device so
// the update can sit inside a CUDA graph.  step[0] = steps taken, step[1] =
// block-completion counter: the last block to finish advances step[0] (no
// separate increment launch).  Optionally writes a bf16 shadow copy of the
// updated parameters (the next forward's GEMM operands: no cast kernels).
__global__ void k_adam(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                       float* __restrict__ v, int64_t n, int64_t* __restrict__ step,
                       float lr, float b1, float b2, float eps, float wd,
                       __nv_bfloat16* __restrict__ p_bf16) {
  const int64_t t = *(volatile int64_t*)step + 1;
  const float bc1 = 1.0f - powf(b1, (float)t);
  const float bc2 = 1.0f - powf(b2, (float)t);
  const float step_size = lr / bc1;
  const float bc2_sqrt = sqrtf(bc2);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float gi = g[i];
    if (wd != 0.f) gi += wd * p[i];
    const float mi = b1 * m[i] + (1.0f - b1) * gi;
    const float vi = b2 * v[i] + (1.0f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float pn = p[i] - step_size * mi / (sqrtf(vi) / bc2_sqrt + eps);
    p[i] = pn;
    if (p_bf16) p_bf16[i] = __float2bfloat16_rn(pn);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(step + 1);
    if (atomicAdd(ctr, 1ull) == gridDim.x - 1) {  // every block has read step[0]
      step[0] = t;
      *ctr = 0ull;
    }
  }
}

__global__ void k_to_bf16(const float* __restrict__ p, int64_t n, __nv_bfloat16* __restrict__ o) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    o[i] = __float2bfloat16_rn(p[i]);
}

}  // namespace fg

extern "C" int64_t fg_block_transpose_scratch_bytes(int64_t cap_src) {
  const int64_t nt = ceil_div(cap_src > 0 ? cap_src : 1, 256 * fg::kTsPer);
  return 2 * cap_src * 4 + 64 + nt * 8 + 256;
}

extern "C" int fg_block_transpose_ex(const int32_t* local, const int64_t* n_edges_dev,
                                     int64_t cap_e, const int32_t* indptr,
                                     const int64_t* n_dst_dev, int64_t max_dst, int max_per_dst,
                                     int64_t cap_src, int32_t* t_indptr, int32_t* t_dst,
                                     float* t_w, int32_t* t_eid, const float* edge_w,
                                     void* scratch, int64_t scratch_bytes, void* s) {
  FG_CHECK_ARG(max_per_dst >= 1, "fg_block_transpose: max_per_dst must be >= 1");
  FG_CHECK_ARG(cap_src >= 1, "fg_block_transpose: empty source capacity");
  FG_CHECK_ARG(scratch_bytes >= fg_block_transpose_scratch_bytes(cap_src),
               "fg_block_transpose: scratch too small");
  cudaStream_t st = as_stream(s);
  const int64_t nt = ceil_div(cap_src, 256 * fg::kTsPer);
  // layout: [ctr 64 B | status nt*8 | cnt cap_src | cursor cap_src]; one memset
  char* base = (char*)scratch;
  unsigned int* ctr = (unsigned int*)base;
  unsigned long long* status = (unsigned long long*)(base + 64);
  int32_t* cnt = (int32_t*)(base + 64 + nt * 8);
  int32_t* cursor = cnt + cap_src;
  FG_CUDA_TRY(cudaMemsetAsync(scratch, 0, 64 + nt * 8 + cap_src * 4, st));
  fg::k_t_hist<<<grid_for(cap_e, 256), 256, 0, st>>>(local, n_edges_dev, cap_e, cnt);
  FG_LAUNCH_CHECK();
  fg::k_t_scan<<<(unsigned)nt, 256, 0, st>>>(cap_src, cnt, t_indptr, cursor, status, ctr,
                                             (unsigned)nt);
  FG_LAUNCH_CHECK();
  fg::k_t_place<<<grid_for(max_dst * max_per_dst, 256), 256, 0, st>>>(
      local, n_edges_dev, cap_e, indptr, n_dst_dev, max_dst, cursor, t_dst, t_w, max_per_dst,
      edge_w, t_eid);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_block_transpose(const int32_t* local, const int64_t* n_edges_dev, int64_t cap_e,
                                  const int32_t* indptr, const int64_t* n_dst_dev,
                                  int64_t max_dst, int max_per_dst, int64_t cap_src,
                                  int32_t* t_indptr, int32_t* t_dst, float* t_w,
                                  const float* edge_w, void* scratch, int64_t scratch_bytes,
                                  void* s) {
  return fg_block_transpose_ex(local, n_edges_dev, cap_e, indptr, n_dst_dev, max_dst,
                               max_per_dst, cap_src, t_indptr, t_dst, t_w, nullptr, edge_w,
                               scratch, scratch_bytes, s);
}

static int block_mean_bwd_t(const uint16_t* g, int64_t H, int64_t g_ld, const int32_t* t_indptr,
                            const int32_t* t_dst, const float* t_w, const int64_t* n_src_dev,
                            int64_t cap_src, const uint16_t* relu_mask, const uint8_t* relu_bits,
                            uint16_t* out, void* s) {
  FG_CHECK_ARG(H % 8 == 0, "hidden dim must be a multiple of 8");
  if (g_ld == 0) g_ld = H;
  FG_CHECK_ARG(g_ld % 8 == 0 && g_ld >= H, "bad g_ld");
  if (cap_src == 0) return FG_OK;
  constexpr int R = 4;
  const int64_t total = (cap_src + R - 1) / R * (H / 4);
  if (relu_bits)
    fg::k_block_mean_bwd_t<2, R><<<grid_for(total, 256, 3), 256, 0, as_stream(s)>>>(
        g, H, g_ld, t_indptr, t_dst, t_w, n_src_dev, cap_src, nullptr, relu_bits, out);
  else if (relu_mask)
    fg::k_block_mean_bwd_t<1, R><<<grid_for(total, 256, 3), 256, 0, as_stream(s)>>>(
        g, H, g_ld, t_indptr, t_dst, t_w, n_src_dev, cap_src, relu_mask, nullptr, out);
  else
    fg::k_block_mean_bwd_t<0, R><<<grid_for(total, 256, 3), 256, 0, as_stream(s)>>>(
        g, H, g_ld, t_indptr, t_dst, t_w, n_src_dev, cap_src, nullptr, nullptr, out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_block_mean_bwd_t(const uint16_t* g, int64_t H, int64_t g_ld,
                                   const int32_t* t_indptr, const int32_t* t_dst,
                                   const float* t_w, const int64_t* n_src_dev, int64_t cap_src,
                                   const uint16_t* relu_mask, uint16_t* out, void* s) {
  return block_mean_bwd_t(g, H, g_ld, t_indptr, t_dst, t_w, n_src_dev, cap_src, relu_mask,
                          nullptr, out, s);
}

extern "C" int fg_block_mean_bwd_t_bits(const uint16_t* g, int64_t H, int64_t g_ld,
                                        const int32_t* t_indptr, const int32_t* t_dst,
                                        const float* t_w, const int64_t* n_src_dev,
                                        int64_t cap_src, const uint8_t* relu_bits,
                                        uint16_t* out, void* s) {
  FG_CHECK_ARG(relu_bits != nullptr, "relu_bits is required");
  return block_mean_bwd_t(g, H, g_ld, t_indptr, t_dst, t_w, n_src_dev, cap_src, nullptr,
                          relu_bits, out, s);
}

extern "C" int fg_adam_step(float* params, const float* grads, float* m, float* v, int64_t n,
                            int64_t* step_dev, float lr, float beta1, float beta2, float eps,
                            float weight_decay, uint16_t* params_bf16, void* s) {
  if (n == 0) return FG_OK;
  fg::k_adam<<<grid_for(n, 256, 4), 256, 0, as_stream(s)>>>(
      params, grads, m, v, n, step_dev, lr, beta1, beta2, eps, weight_decay,
      reinterpret_cast<__nv_bfloat16*>(params_bf16));
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_f32_to_bf16_plain(const float* in, int64_t n, uint16_t* out, void* s) {
  if (n == 0) return FG_OK;
  fg::k_to_bf16<<<grid_for(n, 256, 4), 256, 0, as_stream(s)>>>(
      in, n, reinterpret_cast<__nv_bfloat16*>(out));
  FG_LAUNCH_CHECK();
  return FG_OK;
}

// ------------------------------------------------ fused softmax + CE loss
// Rows r < n_valid (the live seeds) with label labels[node[r]]: loss = mean
// over valid rows of -log softmax(logits[r])[y]; grad = (softmax - onehot) /
// n_valid (0 for padded rows).  Warp per row, fp32 math, deterministic
// (per-row losses reduced by one CTA in row order).
namespace fg {
template <typename LT>
__global__ void k_softmax_ce(const LT* __restrict__ logits, int C, int64_t ld, int64_t rows,
                             const int64_t* __restrict__ nvalid_dev,
                             const int32_t* __restrict__ labels, const int32_t* __restrict__ node,
                             LT* __restrict__ grad, float* __restrict__ row_loss,
                             unsigned int* __restrict__ done, float* __restrict__ loss_out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nv = min64(*nvalid_dev, rows);
  const float inv_n = nv > 0 ? 1.0f / (float)nv : 0.0f;
  for (int64_t r = warp; r < rows; r += nwarps) {
    const LT* x = logits + r * ld;
    LT* gr = grad + r * ld;
    if (r >= nv) {
      for (int c = lane; c < ld; c += 32) gr[c] = (LT)0.f;
      if (lane == 0) row_loss[r] = 0.f;
      continue;
    }
    const int y = labels[node[r]];
    float mx = -INFINITY;
    for (int c = lane; c < C; c += 32) mx = fmaxf(mx, (float)x[c]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float se = 0.f;
    for (int c = lane; c < C; c += 32) se += __expf((float)x[c] - mx);
#pragma unroll
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const float lse = mx + __logf(se);
    for (int c = lane; c < C; c += 32) {
      const float p = __expf((float)x[c] - lse);
      gr[c] = (LT)((p - (c == y ? 1.f : 0.f)) * inv_n);
    }
    for (int c = C + lane; c < ld; c += 32) gr[c] = (LT)0.f;  // padded classes
    if (lane == 0) row_loss[r] = (lse - (float)x[y]) * inv_n;
  }
  // the last CTA to finish sums the per-row losses in row order
  // (deterministic) and re-arms the completion counter
  __shared__ bool last;
  __shared__ float part[256];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  float acc = 0.f;
  const int64_t per = (rows + blockDim.x - 1) / blockDim.x;
  const int64_t r0 = threadIdx.x * per, r1 = min64(rows, r0 + per);
  for (int64_t r = r0; r < r1; ++r) acc += *(volatile float*)(row_loss + r);
  part[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {  // fixed-shape tree (deterministic): 8 partials per lane, then xor
    float t = 0.f;
    for (int i = threadIdx.x; i < (int)blockDim.x; i += 32) t += part[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) {
      *loss_out = t;
      *done = 0u;
    }
  }
}

}  // namespace fg

extern "C" int fg_softmax_ce(const void* logits, int logits_bf16, int C, int64_t ld, int64_t rows,
                             const int64_t* n_valid_dev, const int32_t* labels,
                             const int32_t* row_node, void* grad, float* row_loss,
                             float* loss_out, unsigned int* counter, void* s) {
  FG_CHECK_ARG(C >= 1 && ld >= C && rows >= 1, "fg_softmax_ce: bad shape");
  FG_CHECK_ARG(counter != nullptr && loss_out != nullptr && row_loss != nullptr,
               "fg_softmax_ce: null argument");
  cudaStream_t st = as_stream(s);
  const int threads = 256;
  const int grid = (int)min64(ceil_div(rows * 32, threads), (int64_t)sm_count() * 8);
  if (logits_bf16)
    fg::k_softmax_ce<__nv_bfloat16><<<grid, threads, 0, st>>>(
        (const __nv_bfloat16*)logits, C, ld, rows, n_valid_dev, labels, row_node,
        (__nv_bfloat16*)grad, row_loss, counter, loss_out);
  else
    fg::k_softmax_ce<float><<<grid, threads, 0, st>>>((const float*)logits, C, ld, rows,
                                                      n_valid_dev, labels, row_node,
                                                      (float*)grad, row_loss, counter, loss_out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

// ------------------------------------------------- block edge weights
// Per-edge aggregation weights of a sampled block.  FG_AGG_MEAN: 1/cnt_v
// (the reference's row-stochastic mean, factors.py:108-114).  FG_AGG_GCN:
// Kipf's symmetric normalisation D^-1/2 A D^-1/2 over the full graph's
// degrees (self-loops included), estimated from the cnt_v sampled
// neighbours: w_e = (deg_v / cnt_v) / sqrt(deg_v deg_u) = sqrt(deg_v) /
// (cnt_v sqrt(deg_u)), so sum_e w_e x_u is unbiased for the full GCN sum.
namespace fg {
__global__ void k_edge_weights(int kind, const int64_t* __restrict__ off,
                               const int32_t* __restrict__ dst_nodes,
                               const int32_t* __restrict__ indptr,
                               const int32_t* __restrict__ src_nodes,
                               const int64_t* __restrict__ ndst_dev, int64_t max_dst,
                               float* __restrict__ w) {
  const int64_t live = min64(*ndst_dev, max_dst);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < live;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = indptr[v], b = indptr[v + 1];
    if (b == a) continue;
    const float inv = 1.0f / (float)(b - a);
    if (kind == FG_AGG_MEAN) {
      for (int32_t e = a; e < b; ++e) w[e] = inv;
    } else {
      const int32_t dv = dst_nodes[v];
      const float sv = sqrtf((float)(off[dv + 1] - off[dv])) * inv;
      for (int32_t e = a; e < b; ++e) {
        const int32_t u = src_nodes[e];
        w[e] = sv * rsqrtf((float)(off[u + 1] - off[u]));
      }
    }
  }
}
}  // namespace fg

extern "C" int fg_block_edge_weights(int kind, const int64_t* row_offsets,
                                     const int32_t* dst_nodes, const int32_t* indptr,
                                     const int32_t* src_nodes, const int64_t* n_dst_dev,
                                     int64_t max_dst, float* edge_w, void* s) {
  FG_CHECK_ARG(kind == FG_AGG_MEAN || kind == FG_AGG_GCN, "unknown aggregator kind %d", kind);
  FG_CHECK_ARG(indptr && n_dst_dev && edge_w, "fg_block_edge_weights: null argument");
  FG_CHECK_ARG(kind == FG_AGG_MEAN || (row_offsets && dst_nodes && src_nodes),
               "fg_block_edge_weights: GCN weights need the graph and node ids");
  if (max_dst == 0) return FG_OK;
  fg::k_edge_weights<<<grid_for(max_dst, 256), 256, 0, as_stream(s)>>>(
      kind, row_offsets, dst_nodes, indptr, src_nodes, n_dst_dev, max_dst, edge_w);
  FG_LAUNCH_CHECK();
  return FG_OK;
}
