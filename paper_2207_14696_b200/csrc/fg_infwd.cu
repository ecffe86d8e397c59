// Fused SAGE input-layer projection + first hidden block mean (forward) on
// the 5th-gen tensor cores (tcgen05, accumulator in TMEM).
//
// The unfused forward is two HBM round trips over h0 = X W0^T
// ([cap_src, H] bf16, written by a GEMM, then gathered per edge by the block
// mean): a[v] = sum_{e in v} w_e relu(h0[l_e]).  Here the projection is done
// per EDGE instead of per source row -- the block's sources are almost all
// distinct (a source is picked by ~1.07 destinations at products scale), so
// the MMA work is the same -- and h0 never reaches HBM:
//
//   tile  = D = 128 / fanout consecutive destinations (<= 128 edges, CSR order)
//   A     = W0 [H][P], K-major, loaded into shared memory once per CTA
//   B     = X rows of the tile's edge sources, gathered by cp.async into a
//           K-major no-swizzle operand (row = edge, K = P input features)
//   D     = A B^T : [H features][128 edges] fp32 in TMEM (H/128 MMAs of M 128)
//   epilogue: thread = feature; along its TMEM columns (the tile's edges) it
//           applies ReLU, accumulates w_e-weighted sums per destination and
//           writes bf16 [a | 1 0 ... 0] (bias column); one warp ballot per
//           edge stores the source's ReLU mask bits (the backward's
//           fg_block_mean_wgrad mask_kind 2 input).
//
// The reference has no trainer; the aggregation is its
// row-stochastic neighbour mean (reference/pkg/src/featgrind/factors.py:108-114),
// or the GCN-normalised weights when edge_w is given.  Numerics: fp32
// accumulation of bf16 operands, h0 kept in fp32 (the unfused path rounds it
// to bf16 before the mean), bf16 output.
#include <stdlib.h>

#include "fg_common.cuh"

namespace fg {

constexpr int kIfThreads = 256;  // 8 warps: warp w reads TMEM lanes 32(w%4).., half w/4
constexpr int kIfRows = 128;     // edges per tile (MMA N) = features per MMA (M)

__device__ __forceinline__ uint32_t if_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t if_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // Blackwell descriptor version; SWIZZLE_NONE
  return d;
}
// kind::f16: D f32, A/B bf16, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t if_idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}
// K-major no-swizzle operand with PB core columns (8 bf16 each) along K:
// core (row/8, c) at ((row/8) * PB + c) * 128, row-in-core stride 16 B
__device__ __forceinline__ uint32_t if_off(int row, int c, int PB) {
  return (uint32_t)((((row >> 3) * PB + c) << 7) + ((row & 7) << 4));
}

// persistent CTAs over tiles of D destinations; H in {128, 256}, P % 16 == 0.
// The MMA is issued TRANSPOSED, D[feature][edge] = W0 . X^T (M = 128
// features per half, N = 128 edges), so a TMEM lane holds one feature of every
// edge of the tile: the per-destination sums are register adds along the
// lane's columns (edges of a destination are consecutive), with no staging or
// cross-thread reduction; a warp's ballot per edge gives that edge's source
// 32 ReLU mask bits.
struct Meta {
  int32_t l[kIfRows];      // edge source (-1: dead row)
  float w[kIfRows];        // edge weight (WT)
  int32_t j[kIfRows];      // edge -> destination in the tile
  int32_t ip[kIfRows + 2]; // tile indptr window [D + 1]
  float inv[kIfRows];      // flush scale per destination
  uint32_t fmask[4];       // bit t of word c: edge 32c+t ends its destination
  uint32_t emask[4];       // bit t of word c: destination 32c+t has no edges
};

template <bool WT>
__global__ void __launch_bounds__(kIfThreads)
k_input_block_mean_fwd(const uint16_t* __restrict__ x, int P, const uint16_t* __restrict__ w0,
                       int H, const int32_t* __restrict__ indptr,
                       const int32_t* __restrict__ local, const int64_t* __restrict__ ndst_dev,
                       int64_t max_dst, int D, const float* __restrict__ ew,
                       uint16_t* __restrict__ out, int64_t out_ld, uint8_t* __restrict__ mbits) {
  extern __shared__ __align__(1024) uint8_t if_mem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int PB = P >> 3, HB = H >> 3;
  uint8_t* sW = if_mem;                                   // W0: H x P bf16 (K-major)
  uint8_t* sX = sW + H * P * 2;                           // X rows: 128 x P bf16 (K-major)
  // per-tile metadata, double-buffered (tile k's epilogue reads set k&1
  // while tile k+1's is built in the other)
  Meta* meta = reinterpret_cast<Meta*>(sX + kIfRows * P * 2);  // [2]
  uint32_t* s_bits = reinterpret_cast<uint32_t*>(meta + 2);  // [8 warps][32] ballots
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_bits + 8 * 32);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_bar + 1);

  const int64_t live = min64(*ndst_dev, max_dst);
  // rows past the live destinations: zeros + the bias column, like fg_block_mean_fwd
  {
    const int64_t och = out_ld >> 3;
    for (int64_t i = (int64_t)blockIdx.x * kIfThreads + tid; i < (max_dst - live) * och;
         i += (int64_t)gridDim.x * kIfThreads) {
      const int64_t v = live + i / och, c = i - (i / och) * och;
      reinterpret_cast<uint4*>(out + v * out_ld)[c] =
          c < HB ? make_uint4(0u, 0u, 0u, 0u) : make_uint4(0x3F80u, 0u, 0u, 0u);
    }
  }
  const int64_t ntiles = (live + D - 1) / D;
  if ((int64_t)blockIdx.x >= ntiles) return;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(if_smem(s_tmem)), "r"((uint32_t)H));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(if_smem(s_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // W0 -> K-major operand, once
  for (int i = tid; i < H * PB; i += kIfThreads) {
    const int n = i / PB, c = i - n * PB;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                 ::"r"(if_smem(sW) + if_off(n, c, PB)), "l"(w0 + (int64_t)n * P + c * 8)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *s_tmem;
  const uint32_t idesc = if_idesc(kIfRows);  // M = 128 features, N = 128 edges
  const uint32_t lbo = 128, sbo = (uint32_t)PB * 128;
  const int halves = H >> 7;
  const int half = warp >> 2;                 // warps 4..7: features 128..255
  const bool epi = half < halves;
  const int fbase = half * 128 + (warp & 3) * 32;  // the warp's first feature
  const int f = fbase + lane;
  uint32_t phase = 0;

  // tile metadata: indptr window, then per-edge source / weight / dst / flush
  auto build_meta = [&](int64_t tile, Meta& m) {
    const int64_t v0 = tile * D;
    const int nd = (int)min64(D, live - v0);
    if (tid <= nd) m.ip[tid] = __ldg(indptr + v0 + tid);
    __syncthreads();
    const int32_t e0 = m.ip[0];
    const int ne = m.ip[nd] - e0;
    if (tid < kIfRows) {
      const int r = tid;
      int32_t l = -1, j = 0;
      bool last = false;
      if (r < ne) {
        l = __ldg(local + e0 + r);
        // destination of edge r: binary search over the tile's window
        int lo = 0, hi = nd;
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (m.ip[mid] - e0 <= r) lo = mid; else hi = mid;
        }
        j = lo;
        last = r + 1 == m.ip[j + 1] - e0;
        if (WT) m.w[r] = __ldg(ew + e0 + r);
      }
      m.l[r] = l;
      m.j[r] = j;
      const unsigned fm = __ballot_sync(0xFFFFFFFFu, last);
      if (lane == 0) m.fmask[warp] = fm;
      int cnt = 1;
      if (r < nd) {  // mean: scale the plain sum at the flush; weighted: sum as is
        cnt = m.ip[r + 1] - m.ip[r];
        m.inv[r] = WT ? 1.f : (cnt ? 1.0f / (float)cnt : 0.f);
      }
      const unsigned em = __ballot_sync(0xFFFFFFFFu, cnt == 0);
      if (lane == 0) m.emask[warp] = em;
    }
    __syncthreads();
  };
  // B = X rows of the edge sources by cp.async (dead rows zero-filled)
  auto gather = [&](const Meta& m) {
    for (unsigned i = tid; i < (unsigned)(kIfRows * PB); i += kIfThreads) {
      const unsigned r = i / (unsigned)PB, c = i - r * (unsigned)PB;
      const int32_t l = m.l[r];
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                   ::"r"(if_smem(sX) + if_off(r, c, PB)),
                     "l"(x + (int64_t)(l >= 0 ? l : 0) * P + c * 8), "r"(l >= 0 ? 16 : 0)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto issue_mma = [&]() {
    asm volatile("cp.async.wait_all;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // X staged; the previous epilogue's TMEM reads are done
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int hf = 0; hf < halves; ++hf) {
        for (int ks = 0; ks < PB / 2; ++ks) {  // K = 16 bf16 per MMA (2 core columns)
          const uint32_t off = (uint32_t)ks * 256;
          const uint64_t ad = if_desc(if_smem(sW) + (uint32_t)hf * 16 * sbo + off, lbo, sbo);
          const uint64_t bd = if_desc(if_smem(sX) + off, lbo, sbo);
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
              ::"r"(tmem + (uint32_t)hf * kIfRows), "l"(ad), "l"(bd), "r"(idesc),
                "r"(ks > 0 ? 1u : 0u));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(if_smem(s_bar)) : "memory");
    }
  };

  // pipeline: tile k+1's metadata is built while MMA k runs, its X rows are
  // gathered (into the operand MMA k has finished reading) while epilogue k
  // runs, and MMA k+1 is issued as soon as epilogue k has drained TMEM
  int64_t tile = blockIdx.x;
  int b = 0;
  build_meta(tile, meta[0]);
  gather(meta[0]);
  issue_mma();
  for (; tile < ntiles; tile += gridDim.x, b ^= 1) {
    const Meta& m = meta[b];
    const int64_t v0 = tile * D;
    const int nd = (int)min64(D, live - v0);
    const int ne = m.ip[nd] - m.ip[0];
    const bool more = tile + gridDim.x < ntiles;
    if (more) build_meta(tile + gridDim.x, meta[b ^ 1]);
    {
      const uint32_t mb = if_smem(s_bar);
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done) : "r"(mb), "r"(phase) : "memory");
      phase ^= 1u;
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (more) gather(meta[b ^ 1]);  // MMA k is done with sX
    if (epi) {
      uint16_t* orow = out + v0 * out_ld + f;
      float acc = 0.f;
      for (int c0 = 0; c0 < ne; c0 += 32) {
        uint32_t v[32];
        const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16) +
                            (uint32_t)(half * kIfRows + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
            "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
              "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
              "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
              "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const uint32_t fmask = m.fmask[c0 >> 5];  // bit t: edge c0+t ends its destination
        uint32_t* wbits = s_bits + warp * 32;
        // dead edges (c0+t >= ne) have zero-filled X rows: h = 0 adds nothing,
        // sets no mask bit and never flushes, so the loop needs no bounds test
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const float h = __uint_as_float(v[t]);
          const unsigned mk = __ballot_sync(0xFFFFFFFFu, h > 0.f);
          if (lane == 0) wbits[t] = mk;
          if (WT) acc = fmaf(fmaxf(h, 0.f), m.w[c0 + t], acc);
          else acc += fmaxf(h, 0.f);
          if ((fmask >> t) & 1u) {  // flush destination j (warp-uniform)
            const int j = m.j[c0 + t];
            orow[(int64_t)j * out_ld] = __bfloat16_as_ushort(__float2bfloat16_rn(acc * m.inv[j]));
            acc = 0.f;
          }
        }
        __syncwarp();
        if (c0 + lane < ne)  // edge c0+lane's 32 mask bits (bit t of byte c = feature 8c + t)
          *reinterpret_cast<uint32_t*>(mbits + (int64_t)m.l[c0 + lane] * HB + (fbase >> 3)) =
              wbits[lane];
        __syncwarp();
      }
      for (int q = 0; q * 32 < nd; ++q)  // destinations without edges
        for (uint32_t em = m.emask[q]; em; em &= em - 1)
          orow[(int64_t)(q * 32 + __ffs(em) - 1) * out_ld] = 0;
    }
    if (out_ld > H && tid < nd)  // bias column block [1, 0, ..., 0]
      reinterpret_cast<uint4*>(out + (v0 + tid) * out_ld + H)[0] = make_uint4(0x3F80u, 0u, 0u, 0u);
    if (more) issue_mma();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)H));
}

static int infwd_smem_bytes(int H, int P) {
  return H * P * 2 + kIfRows * P * 2 + 2 * (int)sizeof(Meta) + 8 * 32 * 4 + 8 + 16;
}

// ---------------------------------------------------------------- v2
// Warp-specialised version (round 2; ncu of v1 on the papers100M-shape step:
// 68.6 us, issue 27 %, 0.32 eligible warps, 1 CTA/SM at P = 144: every tile
// serialised metadata loads -> row gathers -> MMA -> epilogue behind block
// barriers).  One persistent CTA per SM, 10 warps:
//   warp 0   producer: tile metadata (indptr window, per-edge source /
//            destination / flush bits) and the cp.async gather of the edge
//            sources' X rows into a 3-stage ring (meta + B operand), each
//            lane's copies completing on the stage's `full` mbarrier
//            (cp.async.mbarrier.arrive.noinc);
//   warp 1   MMA issuer: D[acc] = W0 . X^T for 2 halves x P/16 K-steps into
//            one of TWO TMEM accumulators (2 x H columns), committed to
//            `acc_full`, so tile k+1's MMA runs under tile k's epilogue;
//   warps 2-9 epilogue (unchanged math): TMEM -> ReLU -> per-destination
//            sums -> bf16 rows + ReLU mask bits; they release the TMEM
//            accumulator (`acc_empty`) and the stage (`empty`).
constexpr int kIf2Threads = 576;  // producer, MMA issuer, 2 x 8 epilogue warps
constexpr int kIf2Stages = 3;

__device__ __forceinline__ void if_wait(const uint64_t* bar, uint32_t parity) {
  const uint32_t mb = if_smem(bar);
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(mb), "r"(parity) : "memory");
}
__device__ __forceinline__ void if_arrive(const uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(if_smem(bar)) : "memory");
}

template <bool WT>
__global__ void __launch_bounds__(kIf2Threads, 1)
k_input_block_mean_fwd2(const uint16_t* __restrict__ x, int P, const uint16_t* __restrict__ w0,
                        int H, const int32_t* __restrict__ indptr,
                        const int32_t* __restrict__ local, const int64_t* __restrict__ ndst_dev,
                        int64_t max_dst, int D, const float* __restrict__ ew,
                        uint16_t* __restrict__ out, int64_t out_ld, uint8_t* __restrict__ mbits) {
  extern __shared__ __align__(1024) uint8_t if_mem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int PB = P >> 3, HB = H >> 3;
  uint8_t* sW = if_mem;                                            // W0: H x P (K-major)
  uint8_t* sX0 = sW + H * P * 2;                                   // [stages] 128 x P
  Meta* meta = reinterpret_cast<Meta*>(sX0 + kIf2Stages * kIfRows * P * 2);  // [stages]
  uint32_t* s_bits = reinterpret_cast<uint32_t*>(meta + kIf2Stages);  // [16][32]
  uint64_t* s_full = reinterpret_cast<uint64_t*>(s_bits + 16 * 32);  // [stages]
  uint64_t* s_empty = s_full + kIf2Stages;                           // [stages]
  uint64_t* s_accf = s_empty + kIf2Stages;                           // [2]
  uint64_t* s_acce = s_accf + 2;                                     // [2]
  uint64_t* s_wbar = s_acce + 2;                                     // W0 loaded
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_wbar + 1);

  const int64_t live = min64(*ndst_dev, max_dst);
  {  // rows past the live destinations: zeros + the bias column
    const int64_t och = out_ld >> 3;
    for (int64_t i = (int64_t)blockIdx.x * kIf2Threads + tid; i < (max_dst - live) * och;
         i += (int64_t)gridDim.x * kIf2Threads) {
      const int64_t v = live + i / och, c = i - (i / och) * och;
      reinterpret_cast<uint4*>(out + v * out_ld)[c] =
          c < HB ? make_uint4(0u, 0u, 0u, 0u) : make_uint4(0x3F80u, 0u, 0u, 0u);
    }
  }
  const int64_t ntiles = (live + D - 1) / D;
  if ((int64_t)blockIdx.x >= ntiles) return;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(if_smem(s_tmem)), "r"((uint32_t)(2 * H)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < kIf2Stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 33;" ::"r"(if_smem(s_full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(if_smem(s_empty + s)));
    }
    for (int a = 0; a < 2; ++a) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(if_smem(s_accf + a)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(if_smem(s_acce + a)));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(if_smem(s_wbar)), "r"(kIf2Threads));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *s_tmem;
  // W0 -> K-major operand by everyone, completion on s_wbar (the MMA waits)
  for (int i = tid; i < H * PB; i += kIf2Threads) {
    const int n = i / PB, c = i - n * PB;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                 ::"r"(if_smem(sW) + if_off(n, c, PB)), "l"(w0 + (int64_t)n * P + c * 8)
                 : "memory");
  }
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(if_smem(s_wbar))
               : "memory");
  const int halves = H >> 7;
  const int64_t G = gridDim.x;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // software-pipelined: the indptr window of tile k+2 and the edge sources
    // of tile k+1 are loaded into registers while tile k's metadata and row
    // copies are issued (ncu of the unpipelined producer: 3 serial global
    // round trips per tile, the consumers spinning on `full`)
    constexpr int kIpq = (kIfRows + 31) / 32;  // indptr window entries per lane (D + 1 <= 128)
    auto nd_of = [&](int64_t t) { return (int)min64(D, live - t * D); };
    auto load_ip = [&](int64_t t, int32_t* r) {
      const int nd = nd_of(t);
#pragma unroll
      for (int q = 0; q < kIpq; ++q) {
        const int i = lane + 32 * q;
        r[q] = i <= nd ? __ldg(indptr + t * D + i) : 0;
      }
    };
    auto ip_at = [&](const int32_t* r, int i) {  // window entry i (uniform)
      int32_t v = 0;
#pragma unroll
      for (int q = 0; q < kIpq; ++q) {
        const int32_t x = __shfl_sync(0xFFFFFFFFu, r[q], i & 31);
        if ((i >> 5) == q) v = x;
      }
      return v;
    };
    auto load_l = [&](int64_t t, const int32_t* r, int32_t* lv) {
      const int32_t e0 = ip_at(r, 0), ne = ip_at(r, nd_of(t)) - e0;
#pragma unroll
      for (int q = 0; q < kIfRows / 32; ++q) {
        const int i = lane + 32 * q;
        lv[q] = i < ne ? __ldg(local + e0 + i) : -1;
      }
    };
    int32_t ip_c[kIpq], ip_n[kIpq], lv_c[kIfRows / 32];
    {
      const int64_t t0 = blockIdx.x;
      load_ip(t0, ip_c);
      load_l(t0, ip_c, lv_c);
      if (t0 + G < ntiles) load_ip(t0 + G, ip_n);
    }
    int k = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += G, ++k) {
      const int s = k % kIf2Stages, use = k / kIf2Stages;
      if (use > 0) if_wait(s_empty + s, (uint32_t)((use - 1) & 1));
      Meta& m = meta[s];
      const int nd = nd_of(tile);
#pragma unroll
      for (int q = 0; q < kIpq; ++q)
        if (lane + 32 * q <= nd) m.ip[lane + 32 * q] = ip_c[q];
      int32_t lv[kIfRows / 32];
#pragma unroll
      for (int q = 0; q < kIfRows / 32; ++q) lv[q] = lv_c[q];
      __syncwarp();
      const int32_t e0 = m.ip[0];
      const int ne = m.ip[nd] - e0;
      // next tiles' loads in flight while this tile is issued
      const bool has1 = tile + G < ntiles, has2 = tile + 2 * G < ntiles;
      if (has1) load_l(tile + G, ip_n, lv_c);
#pragma unroll
      for (int q = 0; q < kIpq; ++q) ip_c[q] = ip_n[q];
      if (has2) load_ip(tile + 2 * G, ip_n);
#pragma unroll
      for (int q = 0; q < kIfRows / 32; ++q) {
        const int r = lane + 32 * q;
        int j = 0;
        bool last = false;
        if (r < ne) {
          int lo = 0, hi = nd;
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (m.ip[mid] - e0 <= r) lo = mid; else hi = mid;
          }
          j = lo;
          last = r + 1 == m.ip[j + 1] - e0;
          if (WT) m.w[r] = __ldg(ew + e0 + r);
        }
        m.l[r] = lv[q];
        m.j[r] = j;
        const unsigned fm = __ballot_sync(0xFFFFFFFFu, last);
        if (lane == 0) m.fmask[q] = fm;
        int cnt = 1;
        if (r < nd) {
          cnt = m.ip[r + 1] - m.ip[r];
          m.inv[r] = WT ? 1.f : (cnt ? 1.0f / (float)cnt : 0.f);
        }
        const unsigned em = __ballot_sync(0xFFFFFFFFu, cnt == 0);
        if (lane == 0) m.emask[q] = em;
      }
      // B = X rows of the edge sources (dead rows zero-filled)
      const uint32_t xb = if_smem(sX0) + (uint32_t)(s * kIfRows * P * 2);
#pragma unroll
      for (int q = 0; q < kIfRows / 32; ++q) {
        const int r = lane + 32 * q;
        const int32_t l = lv[q];
        const uint16_t* rowp = x + (int64_t)(l >= 0 ? l : 0) * P;
        for (int c = 0; c < PB; ++c)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
                       ::"r"(xb + if_off(r, c, PB)), "l"(rowp + c * 8), "r"(l >= 0 ? 16 : 0)
                       : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(if_smem(s_full + s))
                   : "memory");
      __syncwarp();
      if (lane == 0) if_arrive(s_full + s);  // releases the metadata stores
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if_wait(s_wbar, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint32_t idesc = if_idesc(kIfRows);
    const uint32_t lbo = 128, sbo = (uint32_t)PB * 128;
    int k = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += G, ++k) {
      const int s = k % kIf2Stages, a = k & 1;
      if_wait(s_full + s, (uint32_t)((k / kIf2Stages) & 1));
      if (k >= 2) if_wait(s_acce + a, (uint32_t)(((k >> 1) - 1) & 1));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (lane == 0) {
        const uint32_t xb = if_smem(sX0) + (uint32_t)(s * kIfRows * P * 2);
        for (int hf = 0; hf < halves; ++hf) {
          for (int ks = 0; ks < PB / 2; ++ks) {
            const uint32_t off = (uint32_t)ks * 256;
            const uint64_t ad = if_desc(if_smem(sW) + (uint32_t)hf * 16 * sbo + off, lbo, sbo);
            const uint64_t bd = if_desc(xb + off, lbo, sbo);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                ::"r"(tmem + (uint32_t)(a * H + hf * kIfRows)), "l"(ad), "l"(bd), "r"(idesc),
                  "r"(ks > 0 ? 1u : 0u));
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(if_smem(s_accf + a)) : "memory");
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // two groups of 8 warps take alternate tiles (group g: tiles k = g mod 2,
    // TMEM accumulator g), so two epilogues run at once -- ncu: the per-edge
    // ReLU / ballot / running-sum chain of one 8-warp group bounded the
    // kernel (~4 us per tile)
    const int ew_all = warp - 2;              // 0..15
    const int grp = ew_all >> 3;
    const int ew_ = ew_all & 7;               // 0..7 within the group
    const int half = ew_ >> 2;                // warps 0-3 of a group: features 0..127
    const bool epi = half < halves;
    const int q4 = warp & 3;                  // TMEM lane quarter of this warp
    const int fbase = half * 128 + q4 * 32;
    const int f = fbase + lane;
    uint32_t* wbits = s_bits + ew_all * 32;
    int k = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += G, ++k) {
      if ((k & 1) != grp) continue;
      const int s = k % kIf2Stages, a = k & 1;
      if_wait(s_accf + a, (uint32_t)((k >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      const Meta& m = meta[s];
      const int64_t v0 = tile * D;
      const int nd = (int)min64(D, live - v0);
      const int ne = m.ip[nd] - m.ip[0];
      if (epi) {
        uint16_t* orow = out + v0 * out_ld + f;
        float acc = 0.f;
        for (int c0 = 0; c0 < ne; c0 += 32) {
          uint32_t v[32];
          const uint32_t ta = tmem + ((uint32_t)(q4 * 32) << 16) +
                              (uint32_t)(a * H + half * kIfRows + c0);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
              "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
                "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                "=r"(v[30]), "=r"(v[31])
              : "r"(ta));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          const uint32_t fmask = m.fmask[c0 >> 5];
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const float h = __uint_as_float(v[t]);
            const unsigned mk = __ballot_sync(0xFFFFFFFFu, h > 0.f);
            if (lane == 0) wbits[t] = mk;
            if (WT) acc = fmaf(fmaxf(h, 0.f), m.w[c0 + t], acc);
            else acc += fmaxf(h, 0.f);
            if ((fmask >> t) & 1u) {
              const int j = m.j[c0 + t];
              orow[(int64_t)j * out_ld] = __bfloat16_as_ushort(__float2bfloat16_rn(acc * m.inv[j]));
              acc = 0.f;
            }
          }
          __syncwarp();
          if (c0 + lane < ne)
            *reinterpret_cast<uint32_t*>(mbits + (int64_t)m.l[c0 + lane] * HB + (fbase >> 3)) =
                wbits[lane];
          __syncwarp();
        }
      }
      // TMEM accumulator a is drained: the MMA of tile k+2 may overwrite it
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) if_arrive(s_acce + a);
      if (epi) {
        uint16_t* orow = out + v0 * out_ld + f;
        for (int q = 0; q * 32 < nd; ++q)  // destinations without edges
          for (uint32_t em = m.emask[q]; em; em &= em - 1)
            orow[(int64_t)(q * 32 + __ffs(em) - 1) * out_ld] = 0;
      }
      if (out_ld > H && ew_ == 0)  // bias column block [1, 0, ..., 0] (the group's warp 0)
        for (int t = lane; t < nd; t += 32)
          reinterpret_cast<uint4*>(out + (v0 + t) * out_ld + H)[0] = make_uint4(0x3F80u, 0u, 0u, 0u);
      __syncwarp();
      if (lane == 0) if_arrive(s_empty + s);  // metadata + B stage free
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"((uint32_t)(2 * H)));
}

static int infwd2_smem_bytes(int H, int P) {
  return H * P * 2 + kIf2Stages * kIfRows * P * 2 + kIf2Stages * (int)sizeof(Meta) + 16 * 32 * 4 +
         (2 * kIf2Stages + 5) * 8 + 16;
}

}  // namespace fg

using namespace fg;

extern "C" int fg_input_block_mean_supported(int64_t H, int64_t P, int64_t fanout) {
  if (!(H == 128 || H == 256)) return 0;
  if (P <= 0 || P % 16 != 0 || P > 256) return 0;
  if (fanout < 1 || fanout > kIfRows) return 0;
  return infwd_smem_bytes((int)H, (int)P) <= 227 * 1024 ? 1 : 0;
}

extern "C" int fg_input_block_mean_fwd(const uint16_t* x, int64_t P, const uint16_t* w0,
                                       int64_t H, const int32_t* indptr, const int32_t* local,
                                       const int64_t* n_dst_dev, int64_t max_dst,
                                       int64_t fanout, const float* edge_w, uint16_t* out,
                                       int64_t out_ld, uint8_t* relu_bits, void* s) {
  FG_CHECK_ARG(x != nullptr && w0 != nullptr && indptr != nullptr && local != nullptr &&
                   n_dst_dev != nullptr && out != nullptr && relu_bits != nullptr,
               "null argument");
  FG_CHECK_ARG(fg_input_block_mean_supported(H, P, fanout),
               "unsupported shape H=%lld P=%lld fanout=%lld", (long long)H, (long long)P,
               (long long)fanout);
  if (out_ld == 0) out_ld = H;
  FG_CHECK_ARG(out_ld == H || out_ld == H + 8, "out_ld must be H or H + 8 (ones column)");
  if (max_dst == 0) return FG_OK;
  const int D = (int)min64(kIfRows / fanout, kIfRows - 1);
  // v2 (warp-specialised, two epilogue warp groups) where v1 fits only one
  // CTA per SM: papers100M-shape block (P = 144) 62.8 (v1) -> 44.5 us.  At
  // products shape (P = 112, v1 at 2 CTAs/SM) v2 is faster alone (46.5 vs
  // 48.5 us) but the step is slower (0.248 vs 0.238 ms: one 576-thread CTA
  // on every SM crowds out the overlapped sampler).  FG_INFWD_V2 = 0 / 1
  // forces v1 / v2.
  static const int v2_env = [] {
    const char* e = getenv("FG_INFWD_V2");
    return e ? atoi(e) : -1;
  }();
  const int smem2 = infwd2_smem_bytes((int)H, (int)P);
  int dev0 = 0, smem_sm0 = 0;
  FG_CUDA_TRY(cudaGetDevice(&dev0));
  FG_CUDA_TRY(cudaDeviceGetAttribute(&smem_sm0, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev0));
  const bool v1_single = smem_sm0 / (infwd_smem_bytes((int)H, (int)P) + 1024) < 2;
  const bool use_v2 = v2_env >= 0 ? v2_env != 0 : v1_single;
  if (use_v2 && smem2 <= 227 * 1024) {
    auto kern2 = edge_w ? k_input_block_mean_fwd2<true> : k_input_block_mean_fwd2<false>;
    FG_CUDA_TRY(cudaFuncSetAttribute(kern2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
    const int64_t tiles = (max_dst + D - 1) / D;
    const int grid = (int)max64(1, min64(tiles, (int64_t)sm_count()));
    kern2<<<grid, kIf2Threads, smem2, as_stream(s)>>>(
        x, (int)P, w0, (int)H, indptr, local, n_dst_dev, max_dst, D, edge_w, out, out_ld,
        relu_bits);
    FG_LAUNCH_CHECK();
    return FG_OK;
  }
  const int smem = infwd_smem_bytes((int)H, (int)P);
  auto kern = edge_w ? k_input_block_mean_fwd<true> : k_input_block_mean_fwd<false>;
  FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  // CTAs per SM: shared memory (1 KB reserved per CTA) and TMEM (H columns
  // each, 512 per SM) bound it; two co-resident CTAs overlap one's gathers
  // with the other's MMA + epilogue
  int dev = 0, smem_sm = 0;
  FG_CUDA_TRY(cudaGetDevice(&dev));
  FG_CUDA_TRY(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  int per_sm = smem_sm / (smem + 1024);
  per_sm = per_sm < 1 ? 1 : (per_sm > 512 / (int)H ? 512 / (int)H : per_sm);
  // s_ip holds D + 1 <= 128 entries
  const int64_t tiles = (max_dst + D - 1) / D;
  static const int ctas_env = [] {  // FG_INFWD_CTAS: grid override (tests, probes)
    const char* e = getenv("FG_INFWD_CTAS");
    return e ? atoi(e) : 0;
  }();
  const int64_t cap = ctas_env > 0 ? (int64_t)ctas_env : (int64_t)sm_count() * per_sm;
  const int grid = (int)max64(1, min64(tiles, cap));
  kern<<<grid, kIfThreads, smem, as_stream(s)>>>(
      x, (int)P, w0, (int)H, indptr, local, n_dst_dev, max_dst, D, edge_w, out, out_ld,
      relu_bits);
  FG_LAUNCH_CHECK();
  return FG_OK;
}
