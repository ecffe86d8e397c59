// Fused block-mean backward + input-layer weight gradient on the 5th-gen
// tensor cores (tcgen05, accumulators in TMEM).
//
// The SAGE input layer computes h = X W^T (X: [cap_src, P] aggregated input
// features with a ones column, W: [H, P]) and the next block averages
// relu(h) over sampled neighbours: a[v] = (1/cnt_v) sum_{e in v} relu(h[l_e]).
// Its weight gradient is
//     dW = sum_r dH[r]^T X[r],  dH[r] = relu'(h[r]) * sum_{e: l_e = r} g[v_e] / cnt_{v_e}
// and, because the ReLU mask is a per-row diagonal scaling, equally
//     dW = sum_e  A_e^T X[l_e],   A_e = bf16( relu'(h[l_e]) * g[v_e] / cnt_{v_e} )
// a GEMM whose K dimension is the block's sampled EDGES.  Tiling K by edges
// (128 per tile) gives every tile identical work -- no per-row edge loops,
// so hub sources (thousands of incoming edges) cannot stall a CTA -- and it
// needs no transposed CSR.  A tiles are built in shared memory from the
// gathers (two 16-byte loads per lane per edge, all in flight together) and
// fed to tcgen05.mma; X rows stream in by cp.async as B; dW accumulates in
// TMEM across the persistent CTA's tiles.  Neither dH nor the per-edge
// products ever reach HBM.  Per-CTA partials are reduced in fixed order
// (deterministic).
//
// Operand layouts (no swizzle, "MN-major" canonical core-matrix layout: a
// core matrix is 8 K-rows x 16 bytes of 8 consecutive MN elements):
//   A = [M = H features][K = 128 edges]: core (mb, kb) at (kb*H/8 + mb)*144
//     (cores padded to 144 B so per-lane core stores are bank-conflict free)
//   B = X [K = 128 edges][N = P cols]:   core (nb, kb) at (kb*P/8 + nb)*128
// so K-adjacent cores are H/8*144 (A) / P/8*128 (B) bytes apart (LBO) and
// MN-adjacent cores 144 (A) / 128 (B) bytes apart (SBO).
//
// The reference has no trainer (the GraphSAGE model is
// new in this build); the aggregation being differentiated is its
// row-stochastic neighbour mean (reference/pkg/src/featgrind/factors.py:108-114).
// Numerics: each edge term is rounded to bf16 before the MMA (the unfused
// bf16 autograd path rounds the per-row sums instead), accumulation is fp32
// in TMEM.
#include <stdlib.h>

#include "fg_common.cuh"

namespace fg {

constexpr int kWgThreads = 512;
constexpr int kWgKT = 128;        // edges per tile (MMA K extent)
constexpr int kWin = 256;         // indptr window per tile (dsts spanned by its edges)
constexpr int kCoreA = 144;       // A core-matrix pitch: 128 B + 16 B bank-rotation pad

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

// last v in [lo, hi) with indptr[v] <= e (indptr[lo] <= e): a 32-ary search
// by one warp, ~log32(n_dst) rounds of coalesced L2 loads.
__device__ __forceinline__ int64_t warp_find_dst(const int32_t* __restrict__ indptr, int64_t lo,
                                                 int64_t hi, int64_t e, int lane) {
  while (hi - lo > 1) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = lo + lane * step;
    const bool ok = p < hi && (int64_t)__ldg(indptr + p) <= e;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, ok);
    lo += (int64_t)(31 - __clz(m)) * step;
    hi = min64(hi, lo + step);
  }
  return lo;
}

// One persistent CTA per SM.  H in {128, 256}; P % 16 == 0, P <= 256;
// (H / 128) * P <= 512 TMEM columns.
__global__ void __launch_bounds__(kWgThreads, 1)
k_block_mean_wgrad(const uint16_t* __restrict__ g, int64_t g_ld,
                   const int32_t* __restrict__ indptr, const int64_t* __restrict__ ndst_dev,
                   int64_t max_dst, const int32_t* __restrict__ local,
                   const float* __restrict__ ew, const uint16_t* __restrict__ hmask,
                   const uint8_t* __restrict__ mbits, int H,
                   const uint16_t* __restrict__ x, int P, float* __restrict__ partial,
                   uint32_t tmem_cols) {
  extern __shared__ __align__(1024) uint8_t wg_mem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int a_bytes = (H / 8) * (kWgKT / 8) * kCoreA, b_bytes = kWgKT * P * 2;
  uint8_t* sA[2] = {wg_mem, wg_mem + a_bytes};
  uint8_t* sB[2] = {wg_mem + 2 * a_bytes, wg_mem + 2 * a_bytes + b_bytes};
  int32_t* s_l = reinterpret_cast<int32_t*>(wg_mem + 2 * a_bytes + 2 * b_bytes);  // [KT]
  int32_t* s_v = s_l + kWgKT;                                                     // [KT]
  float* s_w = reinterpret_cast<float*>(s_v + kWgKT);                             // [KT]
  int32_t* s_win = reinterpret_cast<int32_t*>(s_w + kWgKT);                       // [Win + 1]
  int64_t* s_vw = reinterpret_cast<int64_t*>(s_win + kWin + 1 + 1);               // [1] (8-B aligned)
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_vw + 1);                        // [3]
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_bar + 3);

  const int64_t live_dst = min64(*ndst_dev, max_dst);
  const int64_t nedges = live_dst > 0 ? (int64_t)indptr[live_dst] : 0;
  const int64_t ntiles = (nedges + kWgKT - 1) / kWgKT;
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
  const uint32_t a_lbo = (uint32_t)HB * kCoreA, b_lbo = (uint32_t)PB * 128;
  const uint32_t idesc = umma_idesc_bf16_mn(P);
  uint32_t phase = 0;
  int64_t k = 0;
  // CTA b owns the contiguous tile range [T*b/G, T*(b+1)/G), so the dst of
  // its edges only moves forward: each tile resolves v_e inside a window of
  // kWin+1 indptr entries starting at the dst of its first edge.  Warp 0
  // finds the next tile's window start and loads that window (registers)
  // while the current tile builds; every thread < 128 does the same for the
  // next tile's source ids.
  const int64_t t_lo = ntiles * blockIdx.x / G, t_hi = ntiles * (blockIdx.x + 1) / G;
  constexpr int kWinPer = (kWin + 1 + 31) / 32;
  int32_t pl = -1;
  int32_t pwin[kWinPer];
  int64_t pvw = 0;
  auto load_next = [&](int64_t tile, int64_t vw) {  // vw: dst of the tile's first edge
    if (tid < kWgKT) {
      const int64_t e = tile * kWgKT + tid;
      pl = e < nedges ? __ldg(local + e) : -1;
    }
    if (warp == 0) {
      pvw = vw;
#pragma unroll
      for (int u = 0; u < kWinPer; ++u) {
        const int64_t v = vw + lane + 32 * u;
        pwin[u] = v <= live_dst ? __ldg(indptr + v) : INT32_MAX;
      }
    }
  };
  if (t_lo < t_hi && warp == 0)
    load_next(t_lo, warp_find_dst(indptr, 0, live_dst, t_lo * kWgKT, lane));
  if (t_lo < t_hi && tid < kWgKT && warp != 0) load_next(t_lo, 0);
  for (int64_t tile = t_lo; tile < t_hi; ++tile, ++k) {
    const int s = (int)(k & 1);
    if (k >= 2) {  // MMAs of tile k-2 have finished reading buffer s
      wg_bar_wait(s_bar + s, (phase >> s) & 1u);
      phase ^= 1u << s;
    }
    if (tid < kWgKT) s_l[tid] = pl;
    if (warp == 0) {
#pragma unroll
      for (int u = 0; u < kWinPer; ++u)
        if (lane + 32 * u <= kWin) s_win[lane + 32 * u] = pwin[u];
      if (lane == 0) *s_vw = pvw;
    }
    __syncthreads();
    const int64_t vw = *s_vw;
    if (tile + 1 < t_hi) {
      // dst of the next tile's first edge: in this window unless dsts
      // without edges push it past the window (then a global search)
      const int64_t en = (tile + 1) * kWgKT;
      int64_t vn = 0;
      if (warp == 0) {
        if (en < (int64_t)s_win[kWin]) {
          int lo = 0, hi = kWin;  // last j with s_win[j] <= en
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if ((int64_t)s_win[mid] <= en) lo = mid; else hi = mid;
          }
          vn = vw + lo;
        } else {
          vn = warp_find_dst(indptr, vw, live_dst, en, lane);
        }
      }
      load_next(tile + 1, warp == 0 ? vn : 0);  // lands while this tile builds
    }
    // ---- B = X rows of the edges' sources by cp.async (dead slots zero-fill)
    {
      const uint32_t bbase = wg_smem(sB[s]);
      for (int i = tid; i < kWgKT * PB; i += kWgThreads) {
        const int rr = i & 7, q = i >> 3;
        const int nb = q % PB, kb = q / PB;
        const int r = kb * 8 + rr;
        const uint32_t dst = bbase + (uint32_t)((kb * PB + nb) * 128 + rr * 16);
        const int32_t l = s_l[r];
        const int bytes = l >= 0 ? 16 : 0;  // src-size 0 -> zero fill
        const uint16_t* src = x + (int64_t)(l >= 0 ? l : 0) * P + nb * 8;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                     ::"r"(dst), "l"(src), "r"(bytes) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // ---- A: warp -> core-matrix K group kb (8 edges); lane -> 8-feature
    // chunk (H = 256; for H = 128 half-warps take kb = 2w, 2w+1).  All 16
    // gathers of the group (g row of the dst, mask row of the source) are
    // issued before any is consumed.  The lane's 8 x 16 B result is one core
    // matrix; the 144-byte core pitch spreads a store wavefront over all banks.
    {
      const uint32_t abase = wg_smem(sA[s]);
      const int sub = lane / HB;
      const int c = lane - sub * HB;
      const int gpw = 32 / HB;
      for (int kb = warp * gpw + sub; kb < kWgKT / 8; kb += (kWgThreads / 32) * gpw) {
        if (c < 8) {  // resolve dst + weight of the group's 8 edges
          const int r = kb * 8 + c;
          const int64_t e = tile * kWgKT + r;
          int32_t v = 0;
          float wt = 0.f;
          if (s_l[r] >= 0) {
            int64_t vv;
            if (e < (int64_t)s_win[kWin]) {
              int lo = 0, hi = kWin;
              while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if ((int64_t)s_win[mid] <= e) lo = mid; else hi = mid;
              }
              vv = vw + lo;
              wt = ew ? __ldg(ew + e) : 1.0f / (float)(s_win[lo + 1] - s_win[lo]);
            } else {  // past the window (dsts without edges): serial search
              int64_t lo = vw, hi = live_dst;
              while (hi - lo > 1) {
                const int64_t mid = (lo + hi) >> 1;
                if ((int64_t)__ldg(indptr + mid) <= e) lo = mid; else hi = mid;
              }
              vv = lo;
              wt = ew ? __ldg(ew + e) : 1.0f / (float)(__ldg(indptr + lo + 1) - __ldg(indptr + lo));
            }
            v = (int32_t)vv;
          }
          s_v[r] = v;
          s_w[r] = wt;
        }
        __syncwarp();
        uint4 q[8];
        uint32_t mb[8];  // ReLU mask of the lane's 8 features (bit t = feature 8c+t)
        float w[8];
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          const int r = kb * 8 + rr;
          const int32_t l = s_l[r];
          w[rr] = s_w[r];
          q[rr] = make_uint4(0u, 0u, 0u, 0u);
          mb[rr] = 0xFFu;
          if (l >= 0) {
            q[rr] = __ldg(reinterpret_cast<const uint4*>(g + (int64_t)s_v[r] * g_ld) + c);
            if (mbits) {  // packed mask row: H/8 bytes, one per lane chunk
              mb[rr] = __ldg(mbits + (int64_t)l * HB + c);
            } else if (hmask) {
              float mm[8];
              bf16x8_f32(__ldg(reinterpret_cast<const uint4*>(hmask + (int64_t)l * H) + c), mm);
              uint32_t bits = 0;
#pragma unroll
              for (int t = 0; t < 8; ++t) bits |= (mm[t] > 0.f ? 1u : 0u) << t;
              mb[rr] = bits;
            }
          }
        }
        const uint32_t core = abase + (uint32_t)((kb * HB + c) * kCoreA);
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) {
          float f[8], o8[8];
          bf16x8_f32(q[rr], f);
#pragma unroll
          for (int t = 0; t < 8; ++t) o8[t] = (mb[rr] >> t) & 1u ? f[t] * w[rr] : 0.f;
          const uint4 o = f32_bf16x8(o8);
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};"
                       ::"r"(core + rr * 16), "r"(o.x), "r"(o.y), "r"(o.z), "r"(o.w) : "memory");
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    // ---- MMA issue (one thread): dW[half] += A[half] . B over K = 128 edges
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t abase = wg_smem(sA[s]), bbase = wg_smem(sB[s]);
      for (int half = 0; half < H / 128; ++half) {
        for (int ks = 0; ks < kWgKT / 16; ++ks) {
          const uint64_t ad = umma_desc(abase + half * 16 * kCoreA + ks * 2 * a_lbo, a_lbo, kCoreA);
          const uint64_t bd = umma_desc(bbase + ks * 2 * b_lbo, b_lbo, 128);
#ifndef FG_WGRAD_NO_MMA  // diagnostic build: everything but the tensor-core work
          umma_bf16(tmem + (uint32_t)(half * P), ad, bd, idesc, (k > 0 || ks > 0) ? 1u : 0u);
#endif
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

// dw[i] = sum_b partial[b][i] in CTA order (deterministic), two passes:
// segment j of kRedSeg sums partials [j*nb/S, (j+1)*nb/S) in order (float4
// columns, loads issued 8 ahead), then one pass sums the S segment results
// in order.  ~17 MB of partials (148 x 256 x 112 fp32) stream at HBM rate
// instead of one 148-deep dependent chain per output.
constexpr int kRedSeg = 8;

__global__ void k_wgrad_reduce_seg(const float4* __restrict__ partial, int nb, int64_t n4,
                                   float4* __restrict__ seg) {
  const int j = blockIdx.y;
  const int b0 = (int)((int64_t)nb * j / kRedSeg), b1 = (int)((int64_t)nb * (j + 1) / kRedSeg);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int b = b0;
    for (; b + 8 <= b1; b += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(partial + (int64_t)(b + u) * n4 + i);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
      }
    }
    for (; b < b1; ++b) {
      const float4 v = __ldcs(partial + (int64_t)b * n4 + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    seg[(int64_t)j * n4 + i] = acc;
  }
}

__global__ void k_wgrad_reduce_fin(const float4* __restrict__ seg, int64_t n4,
                                   float4* __restrict__ dw) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 acc = seg[i];
#pragma unroll
    for (int j = 1; j < kRedSeg; ++j) {
      const float4 v = seg[(int64_t)j * n4 + i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    dw[i] = acc;
  }
}

static int wgrad_smem_bytes(int H, int P) {
  return 2 * (H / 8) * (kWgKT / 8) * kCoreA + 2 * kWgKT * P * 2 + 3 * kWgKT * 4 +
         (kWin + 2) * 4 + 8 + 3 * 8 + 16;
}

}  // namespace fg

using namespace fg;

// scratch = [nb][H][P] fp32 partials | [kRedSeg][H][P] segment sums
extern "C" int64_t fg_block_mean_wgrad_scratch_bytes(int64_t H, int64_t P) {
  return ((int64_t)sm_count() + kRedSeg) * H * P * 4;
}

extern "C" int fg_block_mean_wgrad_supported(int64_t H, int64_t P) {
  if (!(H == 128 || H == 256)) return 0;
  if (P <= 0 || P % 16 != 0 || P > 256) return 0;
  if ((H / 128) * P > 512) return 0;
  return wgrad_smem_bytes((int)H, (int)P) <= 227 * 1024 ? 1 : 0;
}

extern "C" int fg_block_mean_wgrad(const uint16_t* g, int64_t g_ld, const int32_t* indptr,
                                   const int32_t* local, const int64_t* n_dst_dev,
                                   int64_t max_dst, const float* edge_w,
                                   const void* relu_mask, int mask_kind, int64_t H,
                                   const uint16_t* x, int64_t P, float* dw, float* scratch,
                                   int64_t scratch_bytes, void* s) {
  FG_CHECK_ARG(g != nullptr && indptr != nullptr && local != nullptr && n_dst_dev != nullptr &&
                   x != nullptr && dw != nullptr && scratch != nullptr,
               "null argument");
  FG_CHECK_ARG(fg_block_mean_wgrad_supported(H, P), "unsupported shape H=%lld P=%lld",
               (long long)H, (long long)P);
  FG_CHECK_ARG(g_ld >= H && g_ld % 8 == 0, "bad g_ld");
  // persistent CTAs on 3/4 of the SMs: the rest stay free for the sampler
  // kernels that overlap the training step on the side stream (products
  // step: 288 -> 276 us at 112 of 148 SMs; 96 is slower again).
  // Input pitch P > 128 (papers100M-shape, P = 144): 96 of 148 SMs
  // (pipelined step 0.2628 -> 0.2567 ms over three interleaved runs; 80:
  // 0.2577, 64: 0.263, 128: 0.266, 148: 0.295).  FG_WGRAD_CTAS overrides
  // (1 .. SM count).
  static const int nb_env = [] {
    const char* e = getenv("FG_WGRAD_CTAS");
    return e ? atoi(e) : 0;
  }();
  const int nb = nb_env > 0 && nb_env <= sm_count()
                     ? nb_env
                     : (P > 128 ? (sm_count() * 13) / 20 : (sm_count() * 3) / 4);
  FG_CHECK_ARG(scratch_bytes >= fg_block_mean_wgrad_scratch_bytes(H, P), "scratch too small");
  cudaStream_t st = as_stream(s);
  float* seg_f = scratch + (int64_t)nb * H * P;
  uint32_t cols = 32;
  while (cols < (uint32_t)((H / 128) * P)) cols <<= 1;
  const int smem = wgrad_smem_bytes((int)H, (int)P);
  FG_CUDA_TRY(cudaFuncSetAttribute(k_block_mean_wgrad, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   smem));
  k_block_mean_wgrad<<<nb, kWgThreads, smem, st>>>(g, g_ld, indptr, n_dst_dev, max_dst, local,
                                                   edge_w,
                                                   mask_kind == 1 ? (const uint16_t*)relu_mask
                                                                  : nullptr,
                                                   mask_kind == 2 ? (const uint8_t*)relu_mask
                                                                  : nullptr,
                                                   (int)H, x, (int)P, scratch,
                                                   cols);
  FG_LAUNCH_CHECK();
  const int64_t n4 = H * P / 4;  // P % 16 == 0
  float4* seg = reinterpret_cast<float4*>(seg_f);
  const dim3 rg((unsigned)((n4 + 255) / 256), kRedSeg);
  k_wgrad_reduce_seg<<<rg, 256, 0, st>>>(reinterpret_cast<const float4*>(scratch), nb, n4, seg);
  FG_LAUNCH_CHECK();
  k_wgrad_reduce_fin<<<(unsigned)((n4 + 255) / 256), 256, 0, st>>>(
      seg, n4, reinterpret_cast<float4*>(dw));
  FG_LAUNCH_CHECK();
  return FG_OK;
}

// ReLU mask bits of bf16 rows: out[r * H/8 + c] bit t = (h[r, 8c + t] > 0).
// One thread per 8-feature chunk (a 16-byte load, a byte store); run right
// after the GEMM that wrote h, while h is still in L2.
namespace fg {
__global__ void k_relu_bits(const uint16_t* __restrict__ h, int64_t rows, int64_t H,
                            uint8_t* __restrict__ out) {
  const int64_t chunks = rows * (H >> 3);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < chunks;
       i += (int64_t)gridDim.x * blockDim.x) {
    float f[8];
    bf16x8_f32(__ldg(reinterpret_cast<const uint4*>(h) + i), f);
    uint32_t b = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) b |= (f[t] > 0.f ? 1u : 0u) << t;
    out[i] = (uint8_t)b;
  }
}
}  // namespace fg

extern "C" int fg_relu_mask_bits(const uint16_t* h, int64_t rows, int64_t H, uint8_t* out,
                                 void* s) {
  FG_CHECK_ARG(H % 8 == 0, "fg_relu_mask_bits: H must be a multiple of 8");
  if (rows == 0) return FG_OK;
  fg::k_relu_bits<<<grid_for(rows * (H / 8), 256), 256, 0, as_stream(s)>>>(h, rows, H, out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}
