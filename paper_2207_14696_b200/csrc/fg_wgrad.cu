// Fused block-mean backward + input-layer weight gradient on the 5th-gen
// tensor cores (tcgen05, accumulators in TMEM).
//
// The SAGE input layer computes h = X W^T (X: [cap_src, P] aggregated input
// features with a ones column, W: [H, P]) and the next block averages
// relu(h) over sampled neighbours.  Its backward is
//     dH[r]  = (h[r] > 0) * sum_{(r -> v) in block} w_rv g[v]     (rows r)
//     dW     = dH^T X                                              ([H, P])
// Done as two library calls (gather kernel writing dH, then a split-K GEMM)
// the ~1e5 x H activation gradient makes a round trip through HBM and the
// GEMM re-reads it: ~270 MB of traffic at products shape.  Here dH tiles are
// built in shared memory straight from the gather and fed to tcgen05.mma as
// the A operand; X tiles stream in by cp.async as the B operand; dW
// accumulates in TMEM across all tiles of a persistent CTA.  dH never
// exists in HBM.  Partial dW per CTA goes to a scratch slab that a second
// kernel reduces in fixed CTA order (deterministic).
//
// Operand layouts (no swizzle, "MN-major" canonical core-matrix layout: a
// core matrix is 8 K-rows x 16 bytes of 8 consecutive MN elements):
//   A = dH^T  [M = H features][K = 128 rows]: core (mb, kb) at (kb*H/8 + mb)*128
//   B = X     [K = 128 rows][N = P cols]:     core (nb, kb) at (kb*P/8 + nb)*128
// so K-adjacent cores are H/8*128 (A) / P/8*128 (B) bytes apart (LBO) and
// MN-adjacent cores 128 bytes apart (SBO).
//
// The reference has no trainer (the GraphSAGE model is
// new in this build); the aggregation being differentiated is its
// row-stochastic neighbour mean (reference/pkg/src/featgrind/factors.py:108-114).
// Numerics: dH is rounded to bf16 before the MMA (as the bf16 autograd path
// it replaces does), accumulation is fp32 in TMEM.
#include "fg_common.cuh"

namespace fg {

constexpr int kWgThreads = 512;
constexpr int kWgKT = 128;        // source rows per tile (MMA K extent)
constexpr int kWgEdgeCap = 2048;  // transposed edges staged per tile

__device__ __forceinline__ uint32_t wg_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory matrix descriptor, SWIZZLE_NONE, sm_100 version bits.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, both operands
// MN-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t umma_idesc_bf16_mn(int n) {
  return (1u << 4)                      // D format f32
       | (1u << 7)                      // A bf16
       | (1u << 10)                     // B bf16
       | (1u << 15)                     // A MN-major
       | (1u << 16)                     // B MN-major
       | ((uint32_t)(n >> 3) << 17)     // N / 8
       | ((uint32_t)(128 >> 4) << 24);  // M / 16
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void wg_bar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(wg_smem(bar)), "r"(count));
}
__device__ __forceinline__ void wg_bar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t mb = wg_smem(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(mb), "r"(parity) : "memory");
  }
}

__device__ __forceinline__ void bf16x8_f32(const uint4 q, float* f) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ uint4 f32_bf16x8(const float* f) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 b = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    w[i] = *reinterpret_cast<const uint32_t*>(&b);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// One persistent CTA per SM.  H in {128, 256}; P % 16 == 0, P <= 256;
// (H / 128) * P <= 512 TMEM columns.
__global__ void __launch_bounds__(kWgThreads, 1)
k_block_mean_wgrad(const uint16_t* __restrict__ g, int64_t g_ld,
                   const int32_t* __restrict__ t_indptr, const int32_t* __restrict__ t_dst,
                   const float* __restrict__ t_w, const int64_t* __restrict__ nsrc_dev,
                   int64_t cap_src, const uint16_t* __restrict__ hmask, int H,
                   const uint16_t* __restrict__ x, int P, float* __restrict__ partial,
                   uint32_t tmem_cols) {
  extern __shared__ __align__(1024) uint8_t wg_mem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int a_bytes = H * kWgKT * 2, b_bytes = kWgKT * P * 2;
  uint8_t* sA[2] = {wg_mem, wg_mem + a_bytes};
  uint8_t* sB[2] = {wg_mem + 2 * a_bytes, wg_mem + 2 * a_bytes + b_bytes};
  int32_t* s_ip = reinterpret_cast<int32_t*>(wg_mem + 2 * a_bytes + 2 * b_bytes);  // [KT + 1]
  int32_t* s_dst = s_ip + kWgKT + 4;                                                  // [EdgeCap]
  float* s_w = reinterpret_cast<float*>(s_dst + kWgEdgeCap);                         // [EdgeCap]
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_w + kWgEdgeCap);                  // [3]
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_bar + 3);

  const int64_t live = min64(*nsrc_dev, cap_src);
  const int64_t ntiles = (live + kWgKT - 1) / kWgKT;
  const int64_t G = gridDim.x;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(wg_smem(s_tmem)), "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    wg_bar_init(s_bar, 1);
    wg_bar_init(s_bar + 1, 1);
    wg_bar_init(s_bar + 2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *s_tmem;

  const int HB = H >> 3, PB = P >> 3;  // 16-byte chunks per row
  const uint32_t a_lbo = (uint32_t)HB * 128, b_lbo = (uint32_t)PB * 128;
  const uint32_t idesc = umma_idesc_bf16_mn(P);
  uint32_t phase = 0;
  int64_t k = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += G, ++k) {
    const int s = (int)(k & 1);
    if (k >= 2) {  // MMAs of tile k-2 have finished reading buffer s
      wg_bar_wait(s_bar + s, (phase >> s) & 1u);
      phase ^= 1u << s;
    }
    const int64_t r0 = tile * kWgKT;
    // ---- B = X tile by cp.async (rows past `live` read row 0 of a zero pad:
    // they are multiplied by zero dH rows, but must be finite -> zero-fill)
    {
      const uint32_t bbase = wg_smem(sB[s]);
      for (int i = tid; i < kWgKT * PB; i += kWgThreads) {
        const int rr = i & 7, q = i >> 3;
        const int nb = q % PB, kb = q / PB;
        const int r = kb * 8 + rr;
        const uint32_t dst = bbase + (uint32_t)((kb * PB + nb) * 128 + rr * 16);
        const int64_t gr = r0 + r;
        const int bytes = gr < live ? 16 : 0;  // src-size 0 -> zero fill
        const uint16_t* src = x + (gr < live ? gr : 0) * (int64_t)P + nb * 8;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                     ::"r"(dst), "l"(src), "r"(bytes) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // ---- transposed CSR slice of this tile
    if (tid <= kWgKT) s_ip[tid] = t_indptr[min64(r0 + tid, live)];
    __syncthreads();
    const int32_t ebase = s_ip[0];
    const int32_t ne = s_ip[kWgKT] - ebase;
    const bool staged = ne <= kWgEdgeCap;
    if (staged)
      for (int i = tid; i < ne; i += kWgThreads) {
        s_dst[i] = t_dst[ebase + i];
        s_w[i] = t_w[ebase + i];
      }
    __syncthreads();
    // ---- A = dH^T tile: item = (row r, 8-feature chunk c); a warp covers
    // 8 rows x 4 chunks so its 16-byte smem stores hit distinct banks
    {
      const uint32_t abase = wg_smem(sA[s]);
      const int groups = (kWgKT / 8) * (HB / 4);  // warp items per tile
      for (int wi = warp; wi < groups; wi += kWgThreads / 32) {
        const int rg = wi / (HB / 4), cg = wi - rg * (HB / 4);
        const int r = rg * 8 + (lane & 7);
        const int c = cg * 4 + (lane >> 3);
        const int64_t gr = r0 + r;
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (gr < live) {
          uint4 mq = make_uint4(0u, 0u, 0u, 0u);
          if (hmask) mq = __ldg(reinterpret_cast<const uint4*>(hmask + gr * H) + c);
          const int32_t e0 = s_ip[r] - ebase, e1 = s_ip[r + 1] - ebase;
          for (int32_t e = e0; e < e1; e += 2) {
            int32_t v0, v1 = 0;
            float w0, w1 = 0.f;
            if (staged) { v0 = s_dst[e]; w0 = s_w[e]; } else { v0 = t_dst[ebase + e]; w0 = t_w[ebase + e]; }
            const bool two = e + 1 < e1;
            if (two) {
              if (staged) { v1 = s_dst[e + 1]; w1 = s_w[e + 1]; }
              else { v1 = t_dst[ebase + e + 1]; w1 = t_w[ebase + e + 1]; }
            }
            const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(g + (int64_t)v0 * g_ld) + c);
            uint4 q1 = make_uint4(0u, 0u, 0u, 0u);
            if (two) q1 = __ldg(reinterpret_cast<const uint4*>(g + (int64_t)v1 * g_ld) + c);
            float f[8];
            bf16x8_f32(q0, f);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = fmaf(f[j], w0, acc[j]);
            if (two) {
              bf16x8_f32(q1, f);
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[j] = fmaf(f[j], w1, acc[j]);
            }
          }
          if (hmask) {
            float m[8];
            bf16x8_f32(mq, m);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = m[j] > 0.f ? acc[j] : 0.f;
          }
        }
        const uint4 o = f32_bf16x8(acc);
        const uint32_t dst = abase + (uint32_t)(((r >> 3) * HB + c) * 128 + (r & 7) * 16);
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};"
                     ::"r"(dst), "r"(o.x), "r"(o.y), "r"(o.z), "r"(o.w) : "memory");
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    // ---- MMA issue (one thread): dW[half] += A[half] . B over K = 128 rows
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t abase = wg_smem(sA[s]), bbase = wg_smem(sB[s]);
      for (int half = 0; half < H / 128; ++half) {
        for (int ks = 0; ks < kWgKT / 16; ++ks) {
          const uint64_t ad = umma_desc(abase + half * 16 * 128 + ks * 2 * a_lbo, a_lbo, 128);
          const uint64_t bd = umma_desc(bbase + ks * 2 * b_lbo, b_lbo, 128);
          umma_bf16(tmem + (uint32_t)(half * P), ad, bd, idesc, (k > 0 || ks > 0) ? 1u : 0u);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(wg_smem(s_bar + s)) : "memory");
    }
  }
  // ---- epilogue: wait for the last MMAs, TMEM -> registers -> partial slab
  const bool any = k > 0;
  if (any) {
    if (tid == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(wg_smem(s_bar + 2)) : "memory");
    wg_bar_wait(s_bar + 2, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  float* out = partial + (int64_t)blockIdx.x * H * P;
  // warp w reads TMEM lanes 32*(w%4).. of accumulator half (w/4) % (H/128);
  // the warpgroups split the columns
  const int wg = warp >> 2;                   // 4 warpgroups
  const int halves = H / 128;
  const int wg_per_half = 4 / halves;         // 2 (H=256) or 4 (H=128)
  const int half = wg / wg_per_half;
  const int part = wg % wg_per_half;
  const int row = half * 128 + (warp & 3) * 32 + lane;
  const int cols_per = (P / 16 + wg_per_half - 1) / wg_per_half * 16;
  const int c_lo = part * cols_per, c_hi = min(P, c_lo + cols_per);
  for (int c0 = c_lo; c0 < c_hi; c0 += 16) {
    uint32_t v[16];
    if (any) {
      const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(half * P + c0);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0u;
    }
    float4* o = reinterpret_cast<float4*>(out + (int64_t)row * P + c0);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      o[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                         __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
}

// dw[i] = sum_b partial[b][i] in CTA order (deterministic).
__global__ void k_wgrad_reduce(const float* __restrict__ partial, int nb, int64_t n,
                               float* __restrict__ dw) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < nb; ++b) s += partial[(int64_t)b * n + i];
    dw[i] = s;
  }
}

static int wgrad_smem_bytes(int H, int P) {
  return 2 * H * kWgKT * 2 + 2 * kWgKT * P * 2 + (kWgKT + 4) * 4 + kWgEdgeCap * 8 + 3 * 8 + 16;
}

}  // namespace fg

using namespace fg;

extern "C" int64_t fg_block_mean_wgrad_scratch_bytes(int64_t H, int64_t P) {
  return (int64_t)sm_count() * H * P * 4;
}

extern "C" int fg_block_mean_wgrad_supported(int64_t H, int64_t P) {
  if (!(H == 128 || H == 256)) return 0;
  if (P <= 0 || P % 16 != 0 || P > 256) return 0;
  if ((H / 128) * P > 512) return 0;
  return wgrad_smem_bytes((int)H, (int)P) <= 227 * 1024 ? 1 : 0;
}

extern "C" int fg_block_mean_wgrad(const uint16_t* g, int64_t g_ld, const int32_t* t_indptr,
                                   const int32_t* t_dst, const float* t_w,
                                   const int64_t* n_src_dev, int64_t cap_src,
                                   const uint16_t* h_mask, int64_t H, const uint16_t* x,
                                   int64_t P, float* dw, float* scratch, int64_t scratch_bytes,
                                   void* s) {
  FG_CHECK_ARG(fg_block_mean_wgrad_supported(H, P), "unsupported shape H=%lld P=%lld",
               (long long)H, (long long)P);
  FG_CHECK_ARG(g_ld >= H && g_ld % 8 == 0, "bad g_ld");
  const int nb = sm_count();
  FG_CHECK_ARG(scratch_bytes >= (int64_t)nb * H * P * 4, "scratch too small");
  const int smem = wgrad_smem_bytes((int)H, (int)P);
  FG_CUDA_TRY(cudaFuncSetAttribute(k_block_mean_wgrad, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   smem));
  uint32_t cols = 32;
  while (cols < (uint32_t)((H / 128) * P)) cols <<= 1;
  k_block_mean_wgrad<<<nb, kWgThreads, smem, as_stream(s)>>>(
      g, g_ld, t_indptr, t_dst, t_w, n_src_dev, cap_src, h_mask, (int)H, x, (int)P, scratch, cols);
  FG_LAUNCH_CHECK();
  const int64_t n = H * P;
  k_wgrad_reduce<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(scratch, nb, n, dw);
  FG_LAUNCH_CHECK();
  return FG_OK;
}
