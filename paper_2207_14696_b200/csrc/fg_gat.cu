// Graph-attention (GAT) edge kernels over sampled blocks — BASELINE config E's
// second aggregator variant (PAPER.md:259-261, 1048-1055 list GAT among the
// trained models; the reference itself has no model code).
//
// A block has destinations v (indptr over edges) and per-edge source rows
// local[e] (for the input layer the source of edge e is decoded row e).  Per
// head k, with projected source rows z and per-source scores
// el[u,k] = <z[u,k,:], a_l[k]>, er[u,k] = <z[u,k,:], a_r[k]>:
//   q[v,k]   = mean_{e in v} er[l_e, k]            (destination query, see below)
//   s[e,k]   = LeakyReLU(el[l_e, k] + q[v, k])
//   a[e,k]   = softmax over v's edges of s[., k]
//   out[v,k] = sum_e a[e,k] z[l_e, k, :]
// Standard GAT scores a destination with its own projected features; under the
// reference's block semantics (pipeline.py:203-221: a layer expands only the
// unique picks of the previous one) a destination that did not sample itself
// has no representation at the layer below, so its query is
// the mean of its sampled neighbours' er — computable for every destination.
//
// Forward: one thread per (destination, head).  Backward scatters into source
// rows with fp32 atomics (dz, d el, d er): the attention backward is not
// bitwise deterministic.
#include <algorithm>

#include "fg_common.cuh"

namespace fg {

__device__ __forceinline__ float leaky(float x, float s) { return x > 0.f ? x : s * x; }

// alpha[e, k], q[v, k]
__global__ void k_gat_softmax_fwd(const float* __restrict__ el, const float* __restrict__ er,
                                  int64_t ld, const int32_t* __restrict__ indptr,
                                  const int32_t* __restrict__ local, int64_t ndst_live_cap,
                                  const int64_t* __restrict__ ndst_dev, int heads, float slope,
                                  float* __restrict__ alpha, float* __restrict__ q) {
  const int64_t live = min64(*ndst_dev, ndst_live_cap);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < live * heads;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / heads;
    const int k = (int)(t - v * heads);
    const int32_t e0 = indptr[v], e1 = indptr[v + 1];
    if (e1 == e0) {
      q[t] = 0.f;
      continue;
    }
    float qs = 0.f;
    for (int32_t e = e0; e < e1; ++e) {
      const int64_t u = local ? local[e] : e;
      qs += er[u * ld + k];
    }
    const float qv = qs / (float)(e1 - e0);
    q[t] = qv;
    float mx = -INFINITY;
    for (int32_t e = e0; e < e1; ++e) {
      const int64_t u = local ? local[e] : e;
      mx = fmaxf(mx, leaky(el[u * ld + k] + qv, slope));
    }
    float den = 0.f;
    for (int32_t e = e0; e < e1; ++e) {
      const int64_t u = local ? local[e] : e;
      const float p = __expf(leaky(el[u * ld + k] + qv, slope) - mx);
      alpha[(int64_t)e * heads + k] = p;
      den += p;
    }
    const float inv = 1.f / den;
    for (int32_t e = e0; e < e1; ++e) alpha[(int64_t)e * heads + k] *= inv;
  }
}

// d el[u,k] += dpre_e ; d er[u,k] += (sum_e' dpre_e') / cnt_v
__global__ void k_gat_softmax_bwd(const float* __restrict__ el, int64_t ld,
                                  const float* __restrict__ q,
                                  const float* __restrict__ alpha, const float* __restrict__ dalpha,
                                  const int32_t* __restrict__ indptr,
                                  const int32_t* __restrict__ local, int64_t ndst_cap,
                                  const int64_t* __restrict__ ndst_dev, int heads, float slope,
                                  float* __restrict__ del, float* __restrict__ der) {
  const int64_t live = min64(*ndst_dev, ndst_cap);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < live * heads;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / heads;
    const int k = (int)(t - v * heads);
    const int32_t e0 = indptr[v], e1 = indptr[v + 1];
    if (e1 == e0) continue;
    float dot = 0.f;
    for (int32_t e = e0; e < e1; ++e)
      dot += alpha[(int64_t)e * heads + k] * dalpha[(int64_t)e * heads + k];
    const float qv = q[t];
    float dq = 0.f;
    for (int32_t e = e0; e < e1; ++e) {
      const int64_t u = local ? local[e] : e;
      const float a = alpha[(int64_t)e * heads + k];
      const float ds = a * (dalpha[(int64_t)e * heads + k] - dot);
      const float pre = el[u * ld + k] + qv;
      const float dpre = pre > 0.f ? ds : slope * ds;
      atomicAdd(del + u * ld + k, dpre);
      dq += dpre;
    }
    const float share = dq / (float)(e1 - e0);
    for (int32_t e = e0; e < e1; ++e) {
      const int64_t u = local ? local[e] : e;
      atomicAdd(der + u * ld + k, share);
    }
  }
}

__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float* f) {
  const uint4 q = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

// out[v, c*8 .. c*8+7] = sum_e alpha[e, head(c)] z[l_e, c*8 ..]; thread per
// (destination, 8-feature chunk); rows past the live count are zeroed.
__global__ void k_gat_agg_fwd(const __nv_bfloat16* __restrict__ z, int64_t hf, int heads,
                              const float* __restrict__ alpha, const int32_t* __restrict__ indptr,
                              const int32_t* __restrict__ local, int64_t max_dst,
                              const int64_t* __restrict__ ndst_dev, float* __restrict__ out) {
  const int64_t live = min64(*ndst_dev, max_dst);
  const int64_t chunks = hf >> 3;
  const int64_t F = hf / heads;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < max_dst * chunks;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / chunks, c = t - v * chunks;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (v < live) {
      const int k = (int)(c * 8 / F);
      for (int32_t e = indptr[v]; e < indptr[v + 1]; ++e) {
        const int64_t u = local ? local[e] : e;
        const float a = alpha[(int64_t)e * heads + k];
        float f[8];
        ld8(z + u * hf + c * 8, f);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = fmaf(a, f[j], acc[j]);
      }
    }
    float4* o = reinterpret_cast<float4*>(out + v * hf + c * 8);
    o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}

// dz[l_e] += alpha_e * dout_v ; dalpha[e, k] += <dout_v, z[l_e]> over head k
__global__ void k_gat_agg_bwd(const __nv_bfloat16* __restrict__ z, int64_t hf, int heads,
                              const float* __restrict__ alpha, const int32_t* __restrict__ indptr,
                              const int32_t* __restrict__ local, int64_t max_dst,
                              const int64_t* __restrict__ ndst_dev, const float* __restrict__ dout,
                              float* __restrict__ dz, float* __restrict__ dalpha) {
  const int64_t live = min64(*ndst_dev, max_dst);
  const int64_t chunks = hf >> 3;
  const int64_t F = hf / heads;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < live * chunks;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / chunks, c = t - v * chunks;
    const int k = (int)(c * 8 / F);
    const float4 d0 = reinterpret_cast<const float4*>(dout + v * hf + c * 8)[0];
    const float4 d1 = reinterpret_cast<const float4*>(dout + v * hf + c * 8)[1];
    const float g[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
    for (int32_t e = indptr[v]; e < indptr[v + 1]; ++e) {
      const int64_t u = local ? local[e] : e;
      const float a = alpha[(int64_t)e * heads + k];
      float f[8];
      ld8(z + u * hf + c * 8, f);
      float dp = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) dp = fmaf(g[j], f[j], dp);
      atomicAdd(dalpha + (int64_t)e * heads + k, dp);
      float4* dst = reinterpret_cast<float4*>(dz + u * hf + c * 8);
      atomicAdd(dst, make_float4(a * g[0], a * g[1], a * g[2], a * g[3]));
      atomicAdd(dst + 1, make_float4(a * g[4], a * g[5], a * g[6], a * g[7]));
    }
  }
}

}  // namespace fg

using namespace fg;

extern "C" int fg_gat_softmax_fwd(const float* el, const float* er, int64_t ld,
                                  const int32_t* indptr, const int32_t* local, int64_t max_dst,
                                  const int64_t* n_dst_dev, int heads, float slope, float* alpha,
                                  float* q, void* s) {
  FG_CHECK_ARG(el && er && indptr && n_dst_dev && alpha && q && heads >= 1, "null argument");
  if (ld == 0) ld = heads;
  FG_CHECK_ARG(ld >= heads, "fg_gat_softmax_fwd: ld < heads");
  if (max_dst == 0) return FG_OK;
  k_gat_softmax_fwd<<<grid_for(max_dst * heads, 256), 256, 0, as_stream(s)>>>(
      el, er, ld, indptr, local, max_dst, n_dst_dev, heads, slope, alpha, q);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_gat_softmax_bwd(const float* el, int64_t ld, const float* q,
                                  const float* alpha, const float* dalpha, const int32_t* indptr,
                                  const int32_t* local, int64_t max_dst,
                                  const int64_t* n_dst_dev, int heads, float slope, float* del,
                                  float* der, void* s) {
  FG_CHECK_ARG(el && q && alpha && dalpha && indptr && n_dst_dev && del && der, "null argument");
  if (ld == 0) ld = heads;
  FG_CHECK_ARG(ld >= heads, "fg_gat_softmax_bwd: ld < heads");
  if (max_dst == 0) return FG_OK;
  k_gat_softmax_bwd<<<grid_for(max_dst * heads, 256), 256, 0, as_stream(s)>>>(
      el, ld, q, alpha, dalpha, indptr, local, max_dst, n_dst_dev, heads, slope, del, der);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_gat_agg_fwd(const uint16_t* z, int64_t hf, int heads, const float* alpha,
                              const int32_t* indptr, const int32_t* local, int64_t max_dst,
                              const int64_t* n_dst_dev, float* out, void* s) {
  FG_CHECK_ARG(z && alpha && indptr && n_dst_dev && out, "null argument");
  FG_CHECK_ARG(hf % 8 == 0 && heads >= 1 && (hf / heads) % 8 == 0,
               "fg_gat_agg_fwd: per-head width must be a multiple of 8");
  if (max_dst == 0) return FG_OK;
  k_gat_agg_fwd<<<grid_for(max_dst * (hf / 8), 256), 256, 0, as_stream(s)>>>(
      reinterpret_cast<const __nv_bfloat16*>(z), hf, heads, alpha, indptr, local, max_dst,
      n_dst_dev, out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_gat_agg_bwd(const uint16_t* z, int64_t hf, int heads, const float* alpha,
                              const int32_t* indptr, const int32_t* local, int64_t max_dst,
                              const int64_t* n_dst_dev, const float* dout, float* dz,
                              float* dalpha, void* s) {
  FG_CHECK_ARG(z && alpha && indptr && n_dst_dev && dout && dz && dalpha, "null argument");
  FG_CHECK_ARG(hf % 8 == 0 && heads >= 1 && (hf / heads) % 8 == 0,
               "fg_gat_agg_bwd: per-head width must be a multiple of 8");
  if (max_dst == 0) return FG_OK;
  k_gat_agg_bwd<<<grid_for(max_dst * (hf / 8), 256), 256, 0, as_stream(s)>>>(
      reinterpret_cast<const __nv_bfloat16*>(z), hf, heads, alpha, indptr, local, max_dst,
      n_dst_dev, dout, dz, dalpha);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

// Input layer by linearity: sum_e alpha[e,k] (x_e W_k) = (sum_e alpha[e,k] x_e) W_k,
// so the attention-weighted aggregate is taken over the decoded input rows
// (one per pick, d columns) per head, and only N_dst x heads rows are
// projected -- no per-pick projection or per-pick gradient.
// out[v, k*d + j] = sum_{e in v} alpha[e, k] x[e, j]: block per 8
// destinations (warp per destination), lanes over the heads*d columns.
// dalpha[e, k] = <dout[v, k*d : (k+1)*d], x[e]>: warp per destination, one
// warp-wide dot per (edge, head).
namespace fg {
constexpr int kMaxHeads = 8;
__global__ void __launch_bounds__(256)
k_gat_xagg_fwd(const __nv_bfloat16* __restrict__ x, int d, int heads,
               const float* __restrict__ alpha, const int32_t* __restrict__ indptr,
               int64_t max_dst, const int64_t* __restrict__ ndst_dev, float* __restrict__ out) {
  // warp per destination; lane over input columns j; each x element is read
  // once and multiplied by every head's alpha
  const int64_t live = min64(*ndst_dev, max_dst);
  const int lane = threadIdx.x & 31;
  for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < max_dst;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    float* o = out + v * (int64_t)heads * d;
    const int32_t e0 = v < live ? indptr[v] : 0, e1 = v < live ? indptr[v + 1] : 0;
    for (int j = lane; j < d; j += 32) {
      float acc[kMaxHeads];
#pragma unroll
      for (int k = 0; k < kMaxHeads; ++k) acc[k] = 0.f;
      for (int32_t e = e0; e < e1; ++e) {
        const float xv = __bfloat162float(x[(int64_t)e * d + j]);
#pragma unroll
        for (int k = 0; k < kMaxHeads; ++k)
          if (k < heads) acc[k] = fmaf(__ldg(alpha + (int64_t)e * heads + k), xv, acc[k]);
      }
#pragma unroll
      for (int k = 0; k < kMaxHeads; ++k)
        if (k < heads) o[k * d + j] = acc[k];
    }
  }
}
__global__ void __launch_bounds__(256)
k_gat_xagg_bwd(const __nv_bfloat16* __restrict__ x, int d, int heads,
               const int32_t* __restrict__ indptr, int64_t max_dst,
               const int64_t* __restrict__ ndst_dev, const float* __restrict__ dout,
               float* __restrict__ dalpha) {
  // warp per destination; per edge the x row is read once and dotted with
  // every head's slice of dout (one butterfly per head)
  const int64_t live = min64(*ndst_dev, max_dst);
  const int lane = threadIdx.x & 31;
  for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < live;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t e0 = indptr[v], e1 = indptr[v + 1];
    const float* g = dout + v * (int64_t)heads * d;
    for (int32_t e = e0; e < e1; ++e) {
      const __nv_bfloat16* xr = x + (int64_t)e * d;
      float acc[kMaxHeads];
#pragma unroll
      for (int k = 0; k < kMaxHeads; ++k) acc[k] = 0.f;
      for (int j = lane; j < d; j += 32) {
        const float xv = __bfloat162float(xr[j]);
#pragma unroll
        for (int k = 0; k < kMaxHeads; ++k)
          if (k < heads) acc[k] = fmaf(g[k * d + j], xv, acc[k]);
      }
#pragma unroll
      for (int k = 0; k < kMaxHeads; ++k) {
        if (k < heads) {
          float a = acc[k];
#pragma unroll
          for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
          if (lane == 0) dalpha[(int64_t)e * heads + k] = a;
        }
      }
    }
  }
}
// ------------------------------------------------ input layer from codes
// Round 2: the GAT input layer reads the code rows of the last block's picks
// directly (no per-pick decoded bf16 matrix in HBM): every kernel below
// decodes the elements it needs in registers (SQ: LUT of the reference
// decodes; VQ 8-bit: codebook entry), exactly dequantize_sq / decode_vq
// (sq.py:132-153, vq.py:330-344).  kind 0 = rows already decoded (bf16, one
// row per pick, in pick order) for codecs outside that set.
struct GatCodes {
  int kind, bits, width, length;
  int64_t stride;       // bytes per row (kind 0: d * 2)
  const uint8_t* rows;  // code rows (kind 0: decoded bf16 rows)
  const float* table;   // SQ LUT / VQ fp32 codebooks [P][L][W]
  const int32_t* picks; // source node of each pick (unused for kind 0)
};
template <int KIND = -1>
__device__ __forceinline__ const uint8_t* gat_row(const GatCodes& c, int64_t e) {
  return (KIND == 0 || c.kind == 0) ? c.rows + e * c.stride
                                    : c.rows + (int64_t)__ldg(c.picks + e) * c.stride;
}
template <int KIND = -1>  // 0: decoded bf16 rows (compile-time), -1: runtime kind
__device__ __forceinline__ float gat_elem(const GatCodes& c, const uint8_t* row, int j) {
  if (KIND == 0 || c.kind == 0) {
    const uint16_t h = reinterpret_cast<const uint16_t*>(row)[j];
    return __uint_as_float((uint32_t)h << 16);
  }
  if (c.kind == FG_CODEC_SQ) {
    const int k = c.bits;
    if (k == 8) return __ldg(c.table + row[j]);
    const int64_t bit = (int64_t)j * k;
    const int b = (int)(bit >> 3), sh = (int)(bit & 7);
    uint32_t w = (uint32_t)row[b] << 8;
    if (sh + k > 8) w |= row[b + 1];
    return __ldg(c.table + ((w >> (16 - sh - k)) & ((1u << k) - 1u)));
  }
  const int p = j / c.width;  // VQ, 8-bit codes
  return __ldg(c.table + ((int64_t)p * c.length + row[p]) * c.width + (j - p * c.width));
}

// el[e, k] = <x_e, c[k]>, er[e, k] = <x_e, c[H + k]>: thread per pick, c in smem
__global__ void __launch_bounds__(256)
k_gat_code_scores(GatCodes cd, int d, int heads, const float* __restrict__ c,
                  const int64_t* __restrict__ ne_dev, int64_t e_cap, float* __restrict__ el,
                  float* __restrict__ er) {
  extern __shared__ float s_c[];  // [2H][d]
  for (int i = threadIdx.x; i < 2 * heads * d; i += blockDim.x) s_c[i] = c[i];
  __syncthreads();
  const int64_t ne = min64(*ne_dev, e_cap);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t* row = gat_row(cd, e);
    float acc[2 * kMaxHeads];
#pragma unroll
    for (int q = 0; q < 2 * kMaxHeads; ++q) acc[q] = 0.f;
    for (int j = 0; j < d; ++j) {
      const float x = gat_elem(cd, row, j);
#pragma unroll
      for (int q = 0; q < 2 * kMaxHeads; ++q)
        if (q < 2 * heads) acc[q] = fmaf(x, s_c[q * d + j], acc[q]);
    }
#pragma unroll
    for (int k = 0; k < kMaxHeads; ++k)
      if (k < heads) {
        el[e * heads + k] = acc[k];
        er[e * heads + k] = acc[heads + k];
      }
  }
}

// partial[b][q][j] = sum over block b's picks e of ds[e, q] x[e, j]
// (ds = [del | der], q < 2H): thread per column j, picks in fixed order
// (deterministic; the partials are summed in block order by the caller)
__global__ void k_gat_code_scores_bwd(GatCodes cd, int d, int heads,
                                      const float* __restrict__ del, const float* __restrict__ der,
                                      int64_t ld,
                                      const int64_t* __restrict__ ne_dev, int64_t e_cap,
                                      int64_t per_block, float* __restrict__ partial) {
  __shared__ float s_ds[32][2 * kMaxHeads];
  const int64_t ne = min64(*ne_dev, e_cap);
  const int64_t e_lo = blockIdx.x * per_block, e_hi = min64(ne, e_lo + per_block);
  float acc[2 * kMaxHeads];
#pragma unroll
  for (int q = 0; q < 2 * kMaxHeads; ++q) acc[q] = 0.f;
  for (int64_t e0 = e_lo; e0 < e_hi; e0 += 32) {
    const int nb = (int)min64(32, e_hi - e0);
    __syncthreads();
    for (int i = threadIdx.x; i < nb * 2 * heads; i += blockDim.x) {
      const int r = i / (2 * heads), q = i - r * 2 * heads;
      s_ds[r][q] = q < heads ? del[(e0 + r) * ld + q] : der[(e0 + r) * ld + q - heads];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      for (int r = 0; r < nb; ++r) {
        const float x = gat_elem(cd, gat_row(cd, e0 + r), j);
#pragma unroll
        for (int q = 0; q < 2 * kMaxHeads; ++q)
          if (q < 2 * heads) acc[q] = fmaf(s_ds[r][q], x, acc[q]);
      }
    }
  }
  // blockDim >= d: thread j owns column j
  const int j = threadIdx.x;
  if (j < d) {
#pragma unroll
    for (int q = 0; q < 2 * kMaxHeads; ++q)
      if (q < 2 * heads) partial[((int64_t)blockIdx.x * 2 * heads + q) * d + j] = acc[q];
  }
}

// A[v, k*d + j] = sum_{e in v} alpha[e, k] x[e, j] (bf16; rows past the live
// count zero): warp per destination, lane owns columns j = lane + 32 i
// (i < kXI, d <= 32 kXI), edges outer (each alpha and x element read once)
constexpr int kXI = 8;  // d <= 256
template <int HEADS, int XI, int KIND>
__global__ void __launch_bounds__(256)
k_gat_code_xagg_fwd(GatCodes cd, int d, const float* __restrict__ alpha,
                    const int32_t* __restrict__ indptr, int64_t max_dst,
                    const int64_t* __restrict__ ndst_dev, __nv_bfloat16* __restrict__ out,
                    int64_t out_ld) {
  constexpr int heads = HEADS;
  const int64_t live = min64(*ndst_dev, max_dst);
  const int lane = threadIdx.x & 31;
  for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < max_dst;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    __nv_bfloat16* o = out + v * out_ld;
    // columns past heads*d: [1, 0, ...] (the projection's bias row / the
    // weight gradient's bias column)
    for (int64_t j = (int64_t)heads * d + lane; j < out_ld; j += 32)
      o[j] = __float2bfloat16_rn(j == (int64_t)heads * d ? 1.f : 0.f);
    const int32_t e0 = v < live ? indptr[v] : 0, e1 = v < live ? indptr[v + 1] : 0;
    float acc[XI][HEADS];
#pragma unroll
    for (int i = 0; i < XI; ++i)
#pragma unroll
      for (int k = 0; k < HEADS; ++k) acc[i][k] = 0.f;
    for (int32_t e = e0; e < e1; ++e) {
      const uint8_t* row = gat_row<KIND>(cd, e);
      float al[HEADS];
#pragma unroll
      for (int k = 0; k < HEADS; ++k)
        al[k] = __ldg(alpha + (int64_t)e * heads + k);
#pragma unroll
      for (int i = 0; i < XI; ++i) {
        const int j = lane + 32 * i;
        if (j < d) {
          const float xv = gat_elem<KIND>(cd, row, j);
#pragma unroll
          for (int k = 0; k < HEADS; ++k)
            acc[i][k] = fmaf(al[k], xv, acc[i][k]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < HEADS; ++k)
#pragma unroll
        for (int i = 0; i < XI; ++i) {
          const int j = lane + 32 * i;
          if (j < d) o[k * d + j] = __float2bfloat16_rn(acc[i][k]);
        }
  }
}

// dalpha[e, k] = <dA[v, k*d : (k+1)*d], x_e>: warp per destination, dA[v]
// held in registers; B = 32/H edges at a time give 32 partial dots per lane,
// reduced across the warp by one 31-shuffle transpose-reduce (lane L ends
// with edge L/H, head L%H), then one coalesced 32-float store
template <int HEADS, int XI, int KIND>
__global__ void __launch_bounds__(256)
k_gat_code_xagg_bwd(GatCodes cd, int d, const int32_t* __restrict__ indptr,
                    int64_t max_dst, const int64_t* __restrict__ ndst_dev,
                    const __nv_bfloat16* __restrict__ dA, float* __restrict__ dalpha) {
  constexpr int heads = HEADS, B = 32 / HEADS;
  const int64_t live = min64(*ndst_dev, max_dst);
  const int lane = threadIdx.x & 31;
  for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < live;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t e0 = indptr[v], e1 = indptr[v + 1];
    const __nv_bfloat16* g = dA + v * (int64_t)heads * d;
    float gk[XI][HEADS];
#pragma unroll
    for (int i = 0; i < XI; ++i) {
      const int j = lane + 32 * i;
#pragma unroll
      for (int k = 0; k < HEADS; ++k)
        gk[i][k] = j < d ? __bfloat162float(g[k * d + j]) : 0.f;
    }
    for (int32_t eb = e0; eb < e1; eb += B) {
      float pv[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) pv[q] = 0.f;
#pragma unroll
      for (int b = 0; b < B; ++b) {
        if (eb + b < e1) {
          const uint8_t* row = gat_row<KIND>(cd, eb + b);
#pragma unroll
          for (int i = 0; i < XI; ++i) {
            const int j = lane + 32 * i;
            if (j < d) {
              const float xv = gat_elem<KIND>(cd, row, j);
#pragma unroll
              for (int k = 0; k < HEADS; ++k)
                pv[b * HEADS + k] = fmaf(gk[i][k], xv, pv[b * HEADS + k]);
            }
          }
        }
      }
      // transpose-reduce: lane L ends with the warp sum of pv[L]
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int q = 0; q < off; ++q) {
          const float send = upper ? pv[q] : pv[q + off];
          const float keep = upper ? pv[q + off] : pv[q];
          pv[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      const int eo = lane / heads;
      if (eb + eo < e1) dalpha[(int64_t)(eb + eo) * heads + (lane - eo * heads)] = pv[0];
    }
  }
}
}  // namespace fg

extern "C" int fg_gat_xagg_fwd(const uint16_t* x, int64_t d, int heads, const float* alpha,
                               const int32_t* indptr, int64_t max_dst, const int64_t* n_dst_dev,
                               float* out, void* s) {
  FG_CHECK_ARG(x && alpha && indptr && n_dst_dev && out && heads >= 1 && heads <= 8 && d >= 1,
               "fg_gat_xagg_fwd: bad argument (heads <= 8)");
  if (max_dst == 0) return FG_OK;
  fg::k_gat_xagg_fwd<<<grid_for(max_dst * 32, 256), 256, 0, as_stream(s)>>>(
      reinterpret_cast<const __nv_bfloat16*>(x), (int)d, heads, alpha, indptr, max_dst, n_dst_dev,
      out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_gat_xagg_bwd(const uint16_t* x, int64_t d, int heads, const int32_t* indptr,
                               int64_t max_dst, const int64_t* n_dst_dev, const float* dout,
                               float* dalpha, int64_t e_cap, void* s) {
  FG_CHECK_ARG(x && indptr && n_dst_dev && dout && dalpha && heads >= 1 && heads <= 8,
               "fg_gat_xagg_bwd: bad argument (heads <= 8)");
  if (max_dst == 0 || e_cap == 0) return FG_OK;
  fg::k_gat_xagg_bwd<<<grid_for(max_dst * 32, 256), 256, 0, as_stream(s)>>>(
      reinterpret_cast<const __nv_bfloat16*>(x), (int)d, heads, indptr, max_dst, n_dst_dev, dout,
      dalpha);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

// ------------------------------------------------ C ABI: input layer from codes
static fg::GatCodes gat_codes(const fg_codec_desc* c, const uint16_t* x_rows, int64_t d,
                              const int32_t* picks) {
  fg::GatCodes g{};
  if (x_rows) {
    g.kind = 0;
    g.rows = reinterpret_cast<const uint8_t*>(x_rows);
    g.stride = d * 2;
  } else {
    g.kind = c->kind;
    g.bits = c->bits;
    g.width = c->width;
    g.length = c->length;
    g.stride = c->row_stride;
    g.rows = c->rows;
    g.table = reinterpret_cast<const float*>(c->table);
  }
  g.picks = picks;
  return g;
}
static bool gat_codes_ok(const fg_codec_desc* c, const uint16_t* x_rows) {
  if (x_rows) return true;
  if (!c) return false;
  if (c->kind == FG_CODEC_SQ) return c->elem_bits == 32;
  return c->kind == FG_CODEC_VQ && c->bits == 8;
}

extern "C" int fg_gat_code_scores(const fg_codec_desc* codec, const uint16_t* x_rows,
                                  const int32_t* picks, const int64_t* n_picks_dev, int64_t e_cap,
                                  int64_t d, int heads, const float* c, float* el, float* er,
                                  void* s) {
  FG_CHECK_ARG(gat_codes_ok(codec, x_rows) && c && el && er && n_picks_dev && heads >= 1 &&
                   heads <= fg::kMaxHeads && d >= 1 && 2 * heads * d <= 12288,
               "fg_gat_code_scores: bad argument");
  if (e_cap == 0) return FG_OK;
  const fg::GatCodes g = gat_codes(codec, x_rows, d, picks);
  fg::k_gat_code_scores<<<grid_for(e_cap, 256), 256, (size_t)2 * heads * d * 4, as_stream(s)>>>(
      g, (int)d, heads, c, n_picks_dev, e_cap, el, er);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int64_t fg_gat_code_scores_bwd_blocks(int64_t e_cap) {
  return std::max<int64_t>(1, std::min<int64_t>(4 * sm_count(), ceil_div(e_cap, 512)));
}

extern "C" int fg_gat_code_scores_bwd(const fg_codec_desc* codec, const uint16_t* x_rows,
                                      const int32_t* picks, const int64_t* n_picks_dev,
                                      int64_t e_cap, int64_t d, int heads, const float* del,
                                      const float* der, int64_t ld, float* partial, void* s) {
  FG_CHECK_ARG(gat_codes_ok(codec, x_rows) && del && der && partial && n_picks_dev &&
                   heads >= 1 && heads <= fg::kMaxHeads && d >= 1 && d <= 1024,
               "fg_gat_code_scores_bwd: bad argument (d <= 1024)");
  if (ld == 0) ld = heads;
  FG_CHECK_ARG(ld >= heads, "fg_gat_code_scores_bwd: ld < heads");
  if (e_cap == 0) return FG_OK;
  const fg::GatCodes g = gat_codes(codec, x_rows, d, picks);
  const int64_t nb = fg_gat_code_scores_bwd_blocks(e_cap);
  const int64_t per = ceil_div(e_cap, nb);
  const int threads = (int)std::max<int64_t>(32, ceil_div(d, 32) * 32);
  fg::k_gat_code_scores_bwd<<<(unsigned)nb, threads, 0, as_stream(s)>>>(
      g, (int)d, heads, del, der, ld, n_picks_dev, e_cap, per, partial);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_gat_code_xagg_fwd(const fg_codec_desc* codec, const uint16_t* x_rows,
                                    const int32_t* picks, int64_t d, int heads,
                                    const float* alpha, const int32_t* indptr, int64_t max_dst,
                                    const int64_t* n_dst_dev, uint16_t* out, int64_t out_ld,
                                    void* s) {
  if (out_ld == 0) out_ld = heads * d;
  FG_CHECK_ARG(out_ld >= heads * d, "fg_gat_code_xagg_fwd: out_ld < heads * d");
  FG_CHECK_ARG(gat_codes_ok(codec, x_rows) && alpha && indptr && n_dst_dev && out &&
                   (heads == 1 || heads == 2 || heads == 4 || heads == 8) && d >= 1 &&
                   d <= 32 * fg::kXI,
               "fg_gat_code_xagg_fwd: bad argument (heads in {1,2,4,8}, d <= 256)");
  if (max_dst == 0) return FG_OK;
  const fg::GatCodes g = gat_codes(codec, x_rows, d, picks);
  auto* ob = reinterpret_cast<__nv_bfloat16*>(out);
  const dim3 grid(grid_for(max_dst * 32, 256));
  cudaStream_t st = as_stream(s);
#define FG_XAGG_FWD(H, XI)                                                                \
  do {                                                                                    \
    if (g.kind == 0)                                                                      \
      fg::k_gat_code_xagg_fwd<H, XI, 0><<<grid, 256, 0, st>>>(g, (int)d, alpha, indptr,   \
                                                              max_dst, n_dst_dev, ob,     \
                                                              out_ld);                    \
    else                                                                                  \
      fg::k_gat_code_xagg_fwd<H, XI, -1><<<grid, 256, 0, st>>>(g, (int)d, alpha, indptr,  \
                                                               max_dst, n_dst_dev, ob,    \
                                                               out_ld);                   \
  } while (0)
  const bool small = d <= 128;
  switch (heads) {
    case 1: if (small) FG_XAGG_FWD(1, 4); else FG_XAGG_FWD(1, 8); break;
    case 2: if (small) FG_XAGG_FWD(2, 4); else FG_XAGG_FWD(2, 8); break;
    case 4: if (small) FG_XAGG_FWD(4, 4); else FG_XAGG_FWD(4, 8); break;
    default: if (small) FG_XAGG_FWD(8, 4); else FG_XAGG_FWD(8, 8); break;
  }
#undef FG_XAGG_FWD
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_gat_code_xagg_bwd(const fg_codec_desc* codec, const uint16_t* x_rows,
                                    const int32_t* picks, int64_t d, int heads,
                                    const int32_t* indptr, int64_t max_dst,
                                    const int64_t* n_dst_dev, const uint16_t* dA, float* dalpha,
                                    void* s) {
  FG_CHECK_ARG(gat_codes_ok(codec, x_rows) && indptr && n_dst_dev && dA && dalpha &&
                   (heads == 1 || heads == 2 || heads == 4 || heads == 8) && d >= 1 &&
                   d <= 32 * fg::kXI,
               "fg_gat_code_xagg_bwd: bad argument (heads in {1,2,4,8}, d <= 256)");
  if (max_dst == 0) return FG_OK;
  const fg::GatCodes g = gat_codes(codec, x_rows, d, picks);
  const auto* dAb = reinterpret_cast<const __nv_bfloat16*>(dA);
  const dim3 grid(grid_for(max_dst * 32, 256));
  cudaStream_t st = as_stream(s);
#define FG_XAGG_BWD(H, XI)                                                                \
  do {                                                                                    \
    if (g.kind == 0)                                                                      \
      fg::k_gat_code_xagg_bwd<H, XI, 0><<<grid, 256, 0, st>>>(g, (int)d, indptr, max_dst,  \
                                                              n_dst_dev, dAb, dalpha);    \
    else                                                                                  \
      fg::k_gat_code_xagg_bwd<H, XI, -1><<<grid, 256, 0, st>>>(g, (int)d, indptr, max_dst, \
                                                               n_dst_dev, dAb, dalpha);   \
  } while (0)
  const bool small = d <= 128;
  switch (heads) {
    case 1: if (small) FG_XAGG_BWD(1, 4); else FG_XAGG_BWD(1, 8); break;
    case 2: if (small) FG_XAGG_BWD(2, 4); else FG_XAGG_BWD(2, 8); break;
    case 4: if (small) FG_XAGG_BWD(4, 4); else FG_XAGG_BWD(4, 8); break;
    default: if (small) FG_XAGG_BWD(8, 4); else FG_XAGG_BWD(8, 8); break;
  }
#undef FG_XAGG_BWD
  FG_LAUNCH_CHECK();
  return FG_OK;
}

// ------------------------------------------------ ELU between GAT layers
// forward: h = bf16(ELU(o + bias)) (o fp32 or bf16, row pitch ld_in; bias
// fp32 [cols] or NULL); backward: do = dh * ELU'(.) computed from the
// output h (1 where h > 0, h + 1 elsewhere), fp32 or bf16 out.  8 columns
// per thread (cols % 8 == 0).
namespace fg {
template <bool IN_F32>
__global__ void k_gat_elu_fwd(const void* __restrict__ in, int64_t ld_in,
                              const float* __restrict__ bias, int64_t rows, int64_t cols,
                              uint16_t* __restrict__ out) {
  const int64_t ch = cols >> 3;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * ch;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / ch, c = (t - r * ch) * 8;
    float f[8];
    if (IN_F32) {
      const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(in) + r * ld_in + c);
      const float4 a = p[0], b = p[1];
      f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
    } else {
      ld8(static_cast<const __nv_bfloat16*>(in) + r * ld_in + c, f);
    }
    if (bias) {
      const float4 a = reinterpret_cast<const float4*>(bias + c)[0];
      const float4 b = reinterpret_cast<const float4*>(bias + c)[1];
      f[0] += a.x; f[1] += a.y; f[2] += a.z; f[3] += a.w;
      f[4] += b.x; f[5] += b.y; f[6] += b.z; f[7] += b.w;
    }
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float x0 = f[2 * i] > 0.f ? f[2 * i] : __expf(f[2 * i]) - 1.f;
      const float x1 = f[2 * i + 1] > 0.f ? f[2 * i + 1] : __expf(f[2 * i + 1]) - 1.f;
      const __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
      w[i] = *reinterpret_cast<const uint32_t*>(&h);
    }
    reinterpret_cast<uint4*>(out + r * cols + c)[0] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}
template <bool OUT_F32>
__global__ void k_gat_elu_bwd(const __nv_bfloat16* __restrict__ dh,
                              const __nv_bfloat16* __restrict__ h, int64_t n8,
                              void* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n8;
       t += (int64_t)gridDim.x * blockDim.x) {
    float g[8], y[8];
    ld8(dh + t * 8, g);
    ld8(h + t * 8, y);
#pragma unroll
    for (int i = 0; i < 8; ++i) g[i] = y[i] > 0.f ? g[i] : g[i] * (y[i] + 1.f);
    if (OUT_F32) {
      float4* o = reinterpret_cast<float4*>(static_cast<float*>(out) + t * 8);
      o[0] = make_float4(g[0], g[1], g[2], g[3]);
      o[1] = make_float4(g[4], g[5], g[6], g[7]);
    } else {
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162 b = __floats2bfloat162_rn(g[2 * i], g[2 * i + 1]);
        w[i] = *reinterpret_cast<const uint32_t*>(&b);
      }
      reinterpret_cast<uint4*>(static_cast<uint16_t*>(out) + t * 8)[0] =
          make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}
}  // namespace fg

extern "C" int fg_gat_elu_fwd(const void* in, int in_f32, int64_t ld_in, const float* bias,
                              int64_t rows, int64_t cols, uint16_t* out, void* s) {
  FG_CHECK_ARG(in && out && cols % 8 == 0 && ld_in >= cols && ld_in % 8 == 0,
               "fg_gat_elu_fwd: bad argument (cols, ld_in multiples of 8)");
  FG_CHECK_ARG((uintptr_t)in % 16 == 0 && (uintptr_t)out % 16 == 0 &&
                   (uintptr_t)bias % 16 == 0, "fg_gat_elu_fwd: pointers must be 16-byte aligned");
  if (rows == 0) return FG_OK;
  const int64_t total = rows * (cols / 8);
  if (in_f32)
    fg::k_gat_elu_fwd<true><<<grid_for(total, 256), 256, 0, as_stream(s)>>>(
        in, ld_in, bias, rows, cols, out);
  else
    fg::k_gat_elu_fwd<false><<<grid_for(total, 256), 256, 0, as_stream(s)>>>(
        in, ld_in, bias, rows, cols, out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_gat_elu_bwd(const uint16_t* dh, const uint16_t* h, int64_t n, void* out,
                              int out_f32, void* s) {
  FG_CHECK_ARG(dh && h && out && n % 8 == 0, "fg_gat_elu_bwd: bad argument (n % 8)");
  FG_CHECK_ARG((uintptr_t)dh % 16 == 0 && (uintptr_t)h % 16 == 0 && (uintptr_t)out % 16 == 0,
               "fg_gat_elu_bwd: pointers must be 16-byte aligned");
  if (n == 0) return FG_OK;
  const auto* dhb = reinterpret_cast<const __nv_bfloat16*>(dh);
  const auto* hb = reinterpret_cast<const __nv_bfloat16*>(h);
  if (out_f32)
    fg::k_gat_elu_bwd<true><<<grid_for(n / 8, 256), 256, 0, as_stream(s)>>>(dhb, hb, n / 8, out);
  else
    fg::k_gat_elu_bwd<false><<<grid_for(n / 8, 256), 256, 0, as_stream(s)>>>(dhb, hb, n / 8, out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

// ------------------------------------------------ fused input-layer attention
// The input layer's sources are the decoded picks (row e = pick e, each pick
// belongs to exactly one destination), so a warp that owns destination v owns
// every row its attention touches.  Forward: per pick the 2H scores
// x_e . c[q] (one 9-shuffle transpose-reduce for 2H = 8), q = mean er, the
// per-head softmax of LeakyReLU(el + q), and A[v] = sum_e alpha x_e -- one
// pass over x instead of a score GEMM + softmax + aggregation (three).
// Backward: dalpha = <dA[v, head], x_e>, the softmax backward within the
// warp, and dc = sum_e [del | der]_e x_e accumulated in registers (per-CTA
// partials in fixed warp order; deterministic).
namespace fg {
// After tr_reduce<V>, lane L holds the warp total of pv[tr_index<V>(L)]
// (V a power of two <= 32): log2(V) halving exchanges at offsets 16, 8, ...,
// then a plain butterfly over the remaining offsets.
template <int V>
__device__ __forceinline__ float tr_reduce(float (&pv)[V], int lane) {
  int off = 16;
#pragma unroll
  for (int n = V; n > 1; n >>= 1, off >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const float send = upper ? pv[i] : pv[i + n / 2];
      const float keep = upper ? pv[i + n / 2] : pv[i];
      pv[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  float r = pv[0];
#pragma unroll
  for (; off >= 1; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
  return r;
}
template <int V>
__device__ __forceinline__ int tr_index(int lane) {
  int idx = 0, off = 16;
#pragma unroll
  for (int n = V; n > 1; n >>= 1, off >>= 1) idx = (idx << 1) | ((lane & off) ? 1 : 0);
  return idx;
}
template <int V>
__device__ __forceinline__ int tr_lane(int idx) {  // the lowest lane holding idx
  int lane = 0, off = 16, b = 0;
  for (int n = V; n > 2; n >>= 1) ++b;  // b = log2(V) - 1
#pragma unroll
  for (int n = V; n > 1; n >>= 1, off >>= 1, --b)
    if ((idx >> b) & 1) lane |= off;
  return lane;
}

// lane owns column pairs (2p, 2p+1), p = lane + 32 i (d even)
template <int XP>
__device__ __forceinline__ void load_row2(const __nv_bfloat16* __restrict__ xr, int d, int lane,
                                          float2 (&xv)[XP]) {
#pragma unroll
  for (int i = 0; i < XP; ++i) {
    const int j = 2 * (lane + 32 * i);
    xv[i] = j < d ? __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(xr + j))
                  : make_float2(0.f, 0.f);
  }
}

// Pick rows as the fused kernels read them: KIND 0 = decoded bf16 rows (row
// e = pick e, pitch d); KIND 1 = 8-bit SQ code rows read in place (row of
// node picks[e], decoded through the 256-entry LUT in shared memory): the
// picks' decoded matrix is never written.
struct IaSrc {
  const __nv_bfloat16* __restrict__ x;
  const uint8_t* __restrict__ rows;
  int64_t stride;
  const int32_t* __restrict__ picks;
  const float* lut;  // shared memory (KIND 1)
};
template <int XP, int KIND>
__device__ __forceinline__ void ia_load(const IaSrc& src, int64_t e, int d, int lane,
                                        float2 (&xv)[XP]) {
  if (KIND == 0) {
    load_row2<XP>(src.x + e * d, d, lane, xv);
  } else {
    const uint8_t* r = src.rows + (int64_t)__ldg(src.picks + e) * src.stride;
#pragma unroll
    for (int i = 0; i < XP; ++i) {
      const int j = 2 * (lane + 32 * i);
      if (j < d) {
        const uint32_t w = *reinterpret_cast<const uint16_t*>(r + j);
        xv[i] = make_float2(src.lut[w & 255u], src.lut[w >> 8]);
      } else {
        xv[i] = make_float2(0.f, 0.f);
      }
    }
  }
}

// Destinations with C <= kIaMaxP picks run a body specialised on C (rows,
// scores and attention in registers, no per-pick branches: the counts are
// warp-uniform, one switch per destination); larger ones take the general
// path through the scores / alpha / dalpha buffers.
constexpr int kIaMaxP = 6;

template <int HEADS, int XP, int KIND>
struct IaFwd {
  static constexpr int V = 2 * HEADS;
  IaSrc src;
  int d, lane, my;
  bool writer;
  float slope;
  float* __restrict__ sc;
  float* __restrict__ alpha;
  float2 cr[V][XP];

  __device__ __forceinline__ float scores(const float2 (&xv)[XP]) const {
    float pv[V];
#pragma unroll
    for (int s = 0; s < V; ++s) {
      float t = 0.f;
#pragma unroll
      for (int i = 0; i < XP; ++i) t = fmaf(xv[i].x, cr[s][i].x, fmaf(xv[i].y, cr[s][i].y, t));
      pv[s] = t;
    }
    return tr_reduce<V>(pv, lane);
  }
  __device__ __forceinline__ void accum(float2 (&acc)[XP][HEADS], const float (&al)[HEADS],
                                        const float2 (&xv)[XP]) const {
#pragma unroll
    for (int k = 0; k < HEADS; ++k)
#pragma unroll
      for (int i = 0; i < XP; ++i) {
        acc[i][k].x = fmaf(al[k], xv[i].x, acc[i][k].x);
        acc[i][k].y = fmaf(al[k], xv[i].y, acc[i][k].y);
      }
  }
  template <int C>
  __device__ __forceinline__ void body(int32_t e0, float* __restrict__ qv,
                                       float2 (&acc)[XP][HEADS]) const {
    // after the transpose-reduce lane L holds score my(L) of every pick: the
    // lanes with my = k < H run head k's softmax on their own registers
    // (one instruction per pick for all heads); the accumulation then takes
    // alpha[e][k] from a lane of head k (H shuffles per pick)
    float2 xr[C][XP];
    float rs[C];
#pragma unroll
    for (int e = 0; e < C; ++e) ia_load<XP, KIND>(src, e0 + e, d, lane, xr[e]);
    float qacc = 0.f;
#pragma unroll
    for (int e = 0; e < C; ++e) {
      rs[e] = scores(xr[e]);
      if (writer) sc[(int64_t)(e0 + e) * V + my] = rs[e];
      qacc += rs[e];
    }
    const int hk = my & (HEADS - 1);  // this lane's head (el lanes: my; er lanes: my - H)
    const float qk = __shfl_sync(0xffffffffu, qacc, tr_lane<V>(HEADS + hk)) * (1.f / C);
    if (writer && my < HEADS) qv[my] = qk;
    float mx = -INFINITY, den = 0.f;
#pragma unroll
    for (int e = 0; e < C; ++e) {
      rs[e] = leaky(rs[e] + qk, slope);
      mx = fmaxf(mx, rs[e]);
    }
#pragma unroll
    for (int e = 0; e < C; ++e) {
      rs[e] = __expf(rs[e] - mx);
      den += rs[e];
    }
    const float inv = 1.f / den;
#pragma unroll
    for (int e = 0; e < C; ++e) {
      rs[e] *= inv;  // alpha[e][hk] (meaningful on the el lanes)
      if (writer && my < HEADS) alpha[(int64_t)(e0 + e) * HEADS + my] = rs[e];
      float al[HEADS];
#pragma unroll
      for (int k = 0; k < HEADS; ++k) al[k] = __shfl_sync(0xffffffffu, rs[e], tr_lane<V>(k));
      accum(acc, al, xr[e]);
    }
  }
  // general path: scores through sc, rows re-read
  __device__ void general(int32_t e0, int32_t e1, float* __restrict__ qv,
                          float2 (&acc)[XP][HEADS]) const {
    float qacc = 0.f;
    for (int32_t e = e0; e < e1; ++e) {
      float2 xv[XP];
      ia_load<XP, KIND>(src, e, d, lane, xv);
      const float r = scores(xv);
      if (writer) sc[(int64_t)e * V + my] = r;
      if (my >= HEADS) qacc += r;
    }
    __syncwarp();
    const float rc = 1.f / (float)(e1 - e0);
    float qk[HEADS], mx[HEADS], inv[HEADS];
#pragma unroll
    for (int k = 0; k < HEADS; ++k) {
      qk[k] = __shfl_sync(0xffffffffu, qacc, tr_lane<V>(HEADS + k)) * rc;
      mx[k] = -INFINITY;
      inv[k] = 0.f;
      if (lane == k) qv[k] = qk[k];
    }
    for (int32_t e = e0; e < e1; ++e)
#pragma unroll
      for (int k = 0; k < HEADS; ++k)
        mx[k] = fmaxf(mx[k], leaky(sc[(int64_t)e * V + k] + qk[k], slope));
    for (int32_t e = e0; e < e1; ++e)
#pragma unroll
      for (int k = 0; k < HEADS; ++k)
        inv[k] += __expf(leaky(sc[(int64_t)e * V + k] + qk[k], slope) - mx[k]);
#pragma unroll
    for (int k = 0; k < HEADS; ++k) inv[k] = 1.f / inv[k];
    for (int32_t e = e0; e < e1; ++e) {
      float2 xv[XP];
      float al[HEADS];
      ia_load<XP, KIND>(src, e, d, lane, xv);
#pragma unroll
      for (int k = 0; k < HEADS; ++k) {
        al[k] = __expf(leaky(sc[(int64_t)e * V + k] + qk[k], slope) - mx[k]) * inv[k];
        if (lane == k) alpha[(int64_t)e * HEADS + k] = al[k];
      }
      accum(acc, al, xv);
    }
  }
};

template <int HEADS, int XP, int KIND>
__global__ void __launch_bounds__(256, 2)
k_gat_input_attn_fwd(IaSrc src, int d, const float* __restrict__ c,
                     const int32_t* __restrict__ indptr, int64_t max_dst, int64_t rows,
                     const int64_t* __restrict__ ndst_dev, float slope, float* __restrict__ sc,
                     float* __restrict__ alpha, float* __restrict__ q,
                     __nv_bfloat16* __restrict__ out, int64_t out_ld) {
  constexpr int V = 2 * HEADS;
  const int64_t live = min64(*ndst_dev, max_dst);
  __shared__ float s_lut[KIND ? 256 : 1];
  if (KIND) {
    for (int t = threadIdx.x; t < 256; t += blockDim.x) s_lut[t] = src.lut[t];
    __syncthreads();
    src.lut = s_lut;
  }
  IaFwd<HEADS, XP, KIND> f;
  f.src = src;
  f.d = d;
  f.lane = threadIdx.x & 31;
  f.my = tr_index<V>(f.lane);
  f.writer = (f.lane & (32 / V - 1)) == 0;
  f.slope = slope;
  f.sc = sc;
  f.alpha = alpha;
  const int lane = f.lane;
#pragma unroll
  for (int s = 0; s < V; ++s)
#pragma unroll
    for (int i = 0; i < XP; ++i) {
      const int j = 2 * (lane + 32 * i);
      f.cr[s][i] = j < d ? make_float2(__ldg(c + s * d + j), __ldg(c + s * d + j + 1))
                         : make_float2(0.f, 0.f);
    }
  for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < rows;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    __nv_bfloat16* o = out + v * out_ld;
    for (int64_t j = (int64_t)HEADS * d + lane; j < out_ld; j += 32)
      o[j] = __float2bfloat16_rn(j == (int64_t)HEADS * d ? 1.f : 0.f);
    const int32_t e0 = v < live ? indptr[v] : 0, e1 = v < live ? indptr[v + 1] : 0;
    float2 acc[XP][HEADS];
#pragma unroll
    for (int i = 0; i < XP; ++i)
#pragma unroll
      for (int k = 0; k < HEADS; ++k) acc[i][k] = make_float2(0.f, 0.f);
    float* qv = q + v * HEADS;
    switch (e1 - e0) {
      case 0: if (v < max_dst && lane < HEADS) qv[lane] = 0.f; break;
      case 1: f.template body<1>(e0, qv, acc); break;
      case 2: f.template body<2>(e0, qv, acc); break;
      case 3: f.template body<3>(e0, qv, acc); break;
      case 4: f.template body<4>(e0, qv, acc); break;
      case 5: f.template body<5>(e0, qv, acc); break;
      case 6: f.template body<6>(e0, qv, acc); break;
      default: f.general(e0, e1, qv, acc); break;
    }
#pragma unroll
    for (int k = 0; k < HEADS; ++k)
#pragma unroll
      for (int i = 0; i < XP; ++i) {
        const int j = 2 * (lane + 32 * i);
        if (j < d)
          *reinterpret_cast<__nv_bfloat162*>(o + k * d + j) =
              __floats2bfloat162_rn(acc[i][k].x, acc[i][k].y);
      }
  }
}

template <int HEADS, int XP, int KIND>
struct IaBwd {
  static constexpr int V = 2 * HEADS;
  IaSrc src;
  const float* __restrict__ sc;
  const float* __restrict__ alpha;
  float* __restrict__ dalpha;
  int d, lane, my;
  bool writer;
  float slope;
  float2 g[HEADS][XP];
  float2 dc[V][XP];

  __device__ __forceinline__ float dots(const float2 (&xv)[XP]) const {
    float pv[HEADS];
#pragma unroll
    for (int k = 0; k < HEADS; ++k) {
      float t = 0.f;
#pragma unroll
      for (int i = 0; i < XP; ++i) t = fmaf(g[k][i].x, xv[i].x, fmaf(g[k][i].y, xv[i].y, t));
      pv[k] = t;
    }
    return tr_reduce<HEADS>(pv, lane);
  }
  __device__ __forceinline__ void accum(const float2 (&xv)[XP], const float (&dl)[HEADS],
                                        const float (&sh)[HEADS]) {
#pragma unroll
    for (int k = 0; k < HEADS; ++k)
#pragma unroll
      for (int i = 0; i < XP; ++i) {
        dc[k][i].x = fmaf(dl[k], xv[i].x, dc[k][i].x);
        dc[k][i].y = fmaf(dl[k], xv[i].y, dc[k][i].y);
        dc[HEADS + k][i].x = fmaf(sh[k], xv[i].x, dc[HEADS + k][i].x);
        dc[HEADS + k][i].y = fmaf(sh[k], xv[i].y, dc[HEADS + k][i].y);
      }
  }
  template <int C>
  __device__ __forceinline__ void body(int32_t e0, const float (&qk)[HEADS]) {
    // after the transpose-reduce lane L holds dalpha[e][my(L)]: the softmax
    // backward of head my runs on that lane's registers; the accumulation
    // takes del[e][k] (and the er share) from a lane of head k
    float2 xr[C][XP];
    float da[C], al[C];
#pragma unroll
    for (int e = 0; e < C; ++e) ia_load<XP, KIND>(src, e0 + e, d, lane, xr[e]);
#pragma unroll
    for (int e = 0; e < C; ++e) al[e] = alpha[(int64_t)(e0 + e) * HEADS + my];
    float dot = 0.f;
#pragma unroll
    for (int e = 0; e < C; ++e) {
      da[e] = dots(xr[e]);
      dot = fmaf(al[e], da[e], dot);
    }
    float qm = qk[0];
#pragma unroll
    for (int k = 1; k < HEADS; ++k) qm = my == k ? qk[k] : qm;
    float shm = 0.f;
#pragma unroll
    for (int e = 0; e < C; ++e) {
      const float ds = al[e] * (da[e] - dot);
      da[e] = sc[(int64_t)(e0 + e) * V + my] + qm > 0.f ? ds : slope * ds;  // del[e][my]
      shm += da[e];
    }
    shm *= 1.f / C;
    float sh[HEADS];
#pragma unroll
    for (int k = 0; k < HEADS; ++k) sh[k] = __shfl_sync(0xffffffffu, shm, tr_lane<HEADS>(k));
#pragma unroll
    for (int e = 0; e < C; ++e) {
      float dl[HEADS];
#pragma unroll
      for (int k = 0; k < HEADS; ++k) dl[k] = __shfl_sync(0xffffffffu, da[e], tr_lane<HEADS>(k));
      accum(xr[e], dl, sh);
    }
  }
  __device__ void general(int32_t e0, int32_t e1, const float (&qk)[HEADS]) {
    float dot[HEADS], sh[HEADS];
#pragma unroll
    for (int k = 0; k < HEADS; ++k) dot[k] = sh[k] = 0.f;
    for (int32_t e = e0; e < e1; ++e) {  // dalpha[e, k] = <dA[v, k], x_e>
      float2 xv[XP];
      ia_load<XP, KIND>(src, e, d, lane, xv);
      const float r = dots(xv);
      if (writer) dalpha[(int64_t)e * HEADS + my] = r;
    }
    __syncwarp();
    for (int32_t e = e0; e < e1; ++e)
#pragma unroll
      for (int k = 0; k < HEADS; ++k)
        dot[k] = fmaf(alpha[(int64_t)e * HEADS + k], dalpha[(int64_t)e * HEADS + k], dot[k]);
    for (int32_t e = e0; e < e1; ++e)
#pragma unroll
      for (int k = 0; k < HEADS; ++k) {
        const float ds = alpha[(int64_t)e * HEADS + k] * (dalpha[(int64_t)e * HEADS + k] - dot[k]);
        sh[k] += sc[(int64_t)e * V + k] + qk[k] > 0.f ? ds : slope * ds;
      }
    const float rc = 1.f / (float)(e1 - e0);
#pragma unroll
    for (int k = 0; k < HEADS; ++k) sh[k] *= rc;
    for (int32_t e = e0; e < e1; ++e) {  // dc += [del | der]_e x_e
      float2 xv[XP];
      float dl[HEADS];
#pragma unroll
      for (int k = 0; k < HEADS; ++k) {
        const float ds = alpha[(int64_t)e * HEADS + k] * (dalpha[(int64_t)e * HEADS + k] - dot[k]);
        dl[k] = sc[(int64_t)e * V + k] + qk[k] > 0.f ? ds : slope * ds;
      }
      ia_load<XP, KIND>(src, e, d, lane, xv);
      accum(xv, dl, sh);
    }
  }
};

template <int HEADS, int XP, int KIND>
__global__ void __launch_bounds__(256, 2)
k_gat_input_attn_bwd(IaSrc src, int d, const float* __restrict__ sc,
                     const float* __restrict__ alpha, const float* __restrict__ q,
                     const __nv_bfloat16* __restrict__ dA, const int32_t* __restrict__ indptr,
                     int64_t max_dst, const int64_t* __restrict__ ndst_dev, float slope,
                     float* __restrict__ dalpha, float* __restrict__ partial) {
  constexpr int V = 2 * HEADS;
  extern __shared__ float s_dc[];  // [V][d]
  const int64_t live = min64(*ndst_dev, max_dst);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ float s_lut[KIND ? 256 : 1];
  if (KIND) {
    for (int t = threadIdx.x; t < 256; t += blockDim.x) s_lut[t] = src.lut[t];
    __syncthreads();
    src.lut = s_lut;
  }
  IaBwd<HEADS, XP, KIND> b;
  b.src = src;
  b.sc = sc;
  b.alpha = alpha;
  b.dalpha = dalpha;
  b.d = d;
  b.lane = lane;
  b.my = tr_index<HEADS>(lane);
  b.writer = (lane & (32 / HEADS - 1)) == 0;
  b.slope = slope;
#pragma unroll
  for (int s = 0; s < V; ++s)
#pragma unroll
    for (int i = 0; i < XP; ++i) b.dc[s][i] = make_float2(0.f, 0.f);
  for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < live;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t e0 = indptr[v], e1 = indptr[v + 1];
    if (e1 == e0) continue;
#pragma unroll
    for (int k = 0; k < HEADS; ++k)
#pragma unroll
      for (int i = 0; i < XP; ++i) {
        const int j = 2 * (lane + 32 * i);
        b.g[k][i] = j < d ? __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(
                                dA + (v * HEADS + k) * (int64_t)d + j))
                          : make_float2(0.f, 0.f);
      }
    float qk[HEADS];
#pragma unroll
    for (int k = 0; k < HEADS; ++k) qk[k] = q[v * HEADS + k];
    switch (e1 - e0) {
      case 1: b.template body<1>(e0, qk); break;
      case 2: b.template body<2>(e0, qk); break;
      case 3: b.template body<3>(e0, qk); break;
      case 4: b.template body<4>(e0, qk); break;
      case 5: b.template body<5>(e0, qk); break;
      case 6: b.template body<6>(e0, qk); break;
      default: b.general(e0, e1, qk); break;
    }
  }
  // CTA partial in fixed warp order
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    if (warp == w)
#pragma unroll
      for (int s = 0; s < V; ++s)
#pragma unroll
        for (int i = 0; i < XP; ++i) {
          const int j = 2 * (lane + 32 * i);
          if (j < d) {
            s_dc[s * d + j] = (w == 0 ? 0.f : s_dc[s * d + j]) + b.dc[s][i].x;
            s_dc[s * d + j + 1] = (w == 0 ? 0.f : s_dc[s * d + j + 1]) + b.dc[s][i].y;
          }
        }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < V * d; t += blockDim.x)
    partial[(int64_t)blockIdx.x * V * d + t] = s_dc[t];
}
}  // namespace fg

extern "C" int64_t fg_gat_input_attn_bwd_blocks(void) { return 2 * sm_count(); }

static bool ia_source(const fg_codec_desc* codec, const uint16_t* x_rows, const int32_t* picks,
                      int64_t d, fg::IaSrc& src, int& kind) {
  src = fg::IaSrc{};
  if (x_rows) {
    src.x = reinterpret_cast<const __nv_bfloat16*>(x_rows);
    kind = 0;
    return true;
  }
  if (!codec || !picks || codec->kind != FG_CODEC_SQ || codec->bits != 8 ||
      codec->elem_bits != 32 || codec->d != d || codec->row_stride % 2)
    return false;
  src.rows = codec->rows;
  src.stride = codec->row_stride;
  src.picks = picks;
  src.lut = static_cast<const float*>(codec->table);
  kind = 1;
  return true;
}

extern "C" int fg_gat_input_attn_fwd(const fg_codec_desc* codec, const uint16_t* x_rows,
                                     const int32_t* picks, int64_t d, int heads, const float* c,
                                     const int32_t* indptr, int64_t max_dst, int64_t rows,
                                     const int64_t* n_dst_dev, float slope, float* scores,
                                     float* alpha, float* q, uint16_t* out, int64_t out_ld,
                                     void* s) {
  fg::IaSrc src;
  int kind = 0;
  FG_CHECK_ARG(ia_source(codec, x_rows, picks, d, src, kind),
               "fg_gat_input_attn_fwd: x_rows, or an 8-bit SQ codec (fp32 LUT) + picks");
  FG_CHECK_ARG(c && indptr && n_dst_dev && scores && alpha && q && out && rows >= max_dst &&
                   (heads == 1 || heads == 2 || heads == 4 || heads == 8) && d >= 2 &&
                   d <= 256 && d % 2 == 0,
               "fg_gat_input_attn_fwd: bad argument (heads in {1,2,4,8}, even d <= 256)");
  if (out_ld == 0) out_ld = heads * d;
  FG_CHECK_ARG(out_ld >= heads * d, "fg_gat_input_attn_fwd: out_ld < heads * d");
  if (rows == 0) return FG_OK;
  auto* ob = reinterpret_cast<__nv_bfloat16*>(out);
  const dim3 grid(grid_for(rows * 32, 256));
  cudaStream_t st = as_stream(s);
#define FG_IA_FWD(H, XP)                                                                       \
  do {                                                                                         \
    if (kind)                                                                                  \
      fg::k_gat_input_attn_fwd<H, XP, 1><<<grid, 256, 0, st>>>(src, (int)d, c, indptr,         \
          max_dst, rows, n_dst_dev, slope, scores, alpha, q, ob, out_ld);                      \
    else                                                                                       \
      fg::k_gat_input_attn_fwd<H, XP, 0><<<grid, 256, 0, st>>>(src, (int)d, c, indptr,         \
          max_dst, rows, n_dst_dev, slope, scores, alpha, q, ob, out_ld);                      \
  } while (0)
  const bool small = d <= 128;
  switch (heads) {
    case 1: if (small) FG_IA_FWD(1, 2); else FG_IA_FWD(1, 4); break;
    case 2: if (small) FG_IA_FWD(2, 2); else FG_IA_FWD(2, 4); break;
    case 4: if (small) FG_IA_FWD(4, 2); else FG_IA_FWD(4, 4); break;
    default: if (small) FG_IA_FWD(8, 2); else FG_IA_FWD(8, 4); break;
  }
#undef FG_IA_FWD
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_gat_input_attn_bwd(const fg_codec_desc* codec, const uint16_t* x_rows,
                                     const int32_t* picks, int64_t d, int heads,
                                     const float* scores, const float* alpha, const float* q,
                                     const uint16_t* dA, const int32_t* indptr, int64_t max_dst,
                                     const int64_t* n_dst_dev, float slope, float* dalpha,
                                     float* partial, void* s) {
  fg::IaSrc src;
  int kind = 0;
  FG_CHECK_ARG(ia_source(codec, x_rows, picks, d, src, kind),
               "fg_gat_input_attn_bwd: x_rows, or an 8-bit SQ codec (fp32 LUT) + picks");
  FG_CHECK_ARG(scores && alpha && q && dA && indptr && n_dst_dev && dalpha && partial &&
                   (heads == 1 || heads == 2 || heads == 4 || heads == 8) && d >= 2 &&
                   d <= 256 && d % 2 == 0,
               "fg_gat_input_attn_bwd: bad argument (heads in {1,2,4,8}, even d <= 256)");
  const auto* gb = reinterpret_cast<const __nv_bfloat16*>(dA);
  const dim3 grid((unsigned)fg_gat_input_attn_bwd_blocks());
  const size_t smem = (size_t)2 * heads * d * sizeof(float);
  cudaStream_t st = as_stream(s);
#define FG_IA_BWD(H, XP)                                                                       \
  do {                                                                                         \
    if (kind)                                                                                  \
      fg::k_gat_input_attn_bwd<H, XP, 1><<<grid, 256, smem, st>>>(src, (int)d, scores, alpha, \
          q, gb, indptr, max_dst, n_dst_dev, slope, dalpha, partial);                          \
    else                                                                                       \
      fg::k_gat_input_attn_bwd<H, XP, 0><<<grid, 256, smem, st>>>(src, (int)d, scores, alpha, \
          q, gb, indptr, max_dst, n_dst_dev, slope, dalpha, partial);                          \
  } while (0)
  const bool small = d <= 128;
  switch (heads) {
    case 1: if (small) FG_IA_BWD(1, 2); else FG_IA_BWD(1, 4); break;
    case 2: if (small) FG_IA_BWD(2, 2); else FG_IA_BWD(2, 4); break;
    case 4: if (small) FG_IA_BWD(4, 2); else FG_IA_BWD(4, 4); break;
    default: if (small) FG_IA_BWD(8, 2); else FG_IA_BWD(8, 4); break;
  }
#undef FG_IA_BWD
  FG_LAUNCH_CHECK();
  return FG_OK;
}

// ------------------------------------------------ gather-form aggregation backward
// Over the block's transpose (per source row u its entries (v, e), from
// fg_block_transpose_ex): dz[u] = sum_entries alpha[e, head] dout[v] written
// once in bf16 (rows without entries or past the live count: zeros), and
// dalpha[e, k] = <dout[v, head k], z[u, head k]> written once per edge and
// head -- no zero fills, no float atomics, no fp32 dz.  Warp per source row,
// lane per 8-feature chunk (hf <= 256); the per-head dot is reduced over the
// head's G = hf/heads/8 lanes (heads == 1: the whole warp).
namespace fg {
__global__ void __launch_bounds__(256)
k_gat_agg_bwd_t(const __nv_bfloat16* __restrict__ z, int64_t hf, int heads,
                const float* __restrict__ alpha, const int32_t* __restrict__ t_indptr,
                const int32_t* __restrict__ t_dst, const int32_t* __restrict__ t_eid,
                const int64_t* __restrict__ nsrc_dev, int64_t cap_src,
                const float* __restrict__ dout, __nv_bfloat16* __restrict__ dz,
                float* __restrict__ dalpha) {
  const int64_t live = min64(*nsrc_dev, cap_src);
  const int lane = threadIdx.x & 31;
  const int chunks = (int)(hf >> 3);
  const int G = chunks / heads;
  const bool act = lane < chunks;
  const int k = act ? lane / G : 0;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < cap_src;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (u < live) {
      float zr[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (act) ld8(z + u * hf + lane * 8, zr);
      const int32_t s0 = t_indptr[u], s1 = t_indptr[u + 1];
      for (int32_t t = s0; t < s1; ++t) {
        const int32_t v = t_dst[t], e = t_eid[t];
        float p = 0.f;
        if (act) {
          const float4* gp = reinterpret_cast<const float4*>(dout + (int64_t)v * hf + lane * 8);
          const float4 g0 = gp[0], g1 = gp[1];
          const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
          const float a = alpha[(int64_t)e * heads + k];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            acc[j] = fmaf(a, g[j], acc[j]);
            p = fmaf(g[j], zr[j], p);
          }
        }
        if (heads == 1) {
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
        } else {
          for (int off = G >> 1; off >= 1; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
        }
        if (act && lane % G == 0) dalpha[(int64_t)e * heads + k] = p;
      }
    }
    if (act) {
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162 b = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
        w[i] = *reinterpret_cast<const uint32_t*>(&b);
      }
      reinterpret_cast<uint4*>(dz + u * hf + lane * 8)[0] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}
}  // namespace fg

extern "C" int fg_gat_agg_bwd_t_supported(int64_t hf, int heads) {
  if (hf % 8 || hf > 256 || heads < 1 || (hf / 8) % heads) return 0;
  const int64_t G = hf / 8 / heads;
  return heads == 1 || (G & (G - 1)) == 0;
}

extern "C" int fg_gat_agg_bwd_t(const uint16_t* z, int64_t hf, int heads, const float* alpha,
                                const int32_t* t_indptr, const int32_t* t_dst,
                                const int32_t* t_eid, const int64_t* n_src_dev, int64_t cap_src,
                                const float* dout, uint16_t* dz, float* dalpha, void* s) {
  FG_CHECK_ARG(z && alpha && t_indptr && t_dst && t_eid && n_src_dev && dout && dz && dalpha,
               "fg_gat_agg_bwd_t: null argument");
  FG_CHECK_ARG(fg_gat_agg_bwd_t_supported(hf, heads),
               "fg_gat_agg_bwd_t: hf <= 256, hf/8 lanes split evenly into power-of-2 heads");
  if (cap_src == 0) return FG_OK;
  fg::k_gat_agg_bwd_t<<<grid_for(cap_src * 32, 256), 256, 0, as_stream(s)>>>(
      reinterpret_cast<const __nv_bfloat16*>(z), hf, heads, alpha, t_indptr, t_dst, t_eid,
      n_src_dev, cap_src, dout, reinterpret_cast<__nv_bfloat16*>(dz), dalpha);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

// ------------------------------------------------ [a | b | 0] rows in bf16
// out[r] = bf16([a[r, :ac] | b[r, :bc] | 0 ...]) with row pitch out_ld (a
// multiple of 8): the GAT backward's [dz | ds] operand in one pass (a torch
// copy into the strided column slice runs the non-vectorised path).
namespace fg {
__global__ void k_cat_rows_bf16(const float* __restrict__ a, int64_t ac,
                                const float* __restrict__ b, int64_t bc, int64_t rows,
                                uint16_t* __restrict__ out, int64_t out_ld) {
  const int64_t ch = out_ld >> 3;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * ch;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / ch, c0 = (t - r * ch) * 8;
    float f[8];
    if (c0 + 8 <= ac && (ac & 3) == 0) {
      const float4* p = reinterpret_cast<const float4*>(a + r * ac + c0);
      const float4 x = p[0], y = p[1];
      f[0] = x.x; f[1] = x.y; f[2] = x.z; f[3] = x.w; f[4] = y.x; f[5] = y.y; f[6] = y.z; f[7] = y.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t c = c0 + j;
        f[j] = c < ac ? a[r * ac + c] : (c < ac + bc ? b[r * bc + (c - ac)] : 0.f);
      }
    }
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
      w[i] = *reinterpret_cast<const uint32_t*>(&h);
    }
    reinterpret_cast<uint4*>(out + r * out_ld + c0)[0] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}
}  // namespace fg

extern "C" int fg_cat_rows_bf16(const float* a, int64_t ac, const float* b, int64_t bc,
                                int64_t rows, uint16_t* out, int64_t out_ld, void* s) {
  FG_CHECK_ARG(a && out && out_ld % 8 == 0 && out_ld >= ac + bc && (bc == 0 || b),
               "fg_cat_rows_bf16: bad argument (out_ld % 8 == 0, >= ac + bc)");
  FG_CHECK_ARG((uintptr_t)out % 16 == 0 && (uintptr_t)a % 16 == 0,
               "fg_cat_rows_bf16: a / out must be 16-byte aligned");
  if (rows == 0) return FG_OK;
  fg::k_cat_rows_bf16<<<grid_for(rows * (out_ld / 8), 256), 256, 0, as_stream(s)>>>(
      a, ac, b, bc, rows, out, out_ld);
  FG_LAUNCH_CHECK();
  return FG_OK;
}
