// Codec fitting support on the device.
//
//  * fit_sq (pkg/src/featgrind/sq.py:84-111): the reference takes the
//    nonzeros in row-major order, subsamples them at the ranks
//    np.linspace(0, nnz-1, 10^7).astype(int64) when nnz > 10^7, then computes
//    np.quantile(log2|.|, [c, 1-c]).  log2 is monotone, so the quantiles only
//    need four order statistics of |x|; the device does the compaction /
//    strided gather and an exact radix select, the host applies numpy's own
//    log2 and quantile interpolation to those four values (bit-exact by
//    construction).
//  * fit_vq Lloyd assignment (vq.py:184-228): fp64 distances / similarities
//    ordered as the reference evaluates them.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "fg_common.cuh"

namespace fg {

constexpr int kNzThreads = 256;
constexpr int kNzPer = 16;
constexpr int64_t kNzChunk = (int64_t)kNzThreads * kNzPer;

__global__ void __launch_bounds__(kNzThreads)
k_nz_count(const float* __restrict__ x, int64_t count, int64_t* __restrict__ bcnt,
           unsigned long long* __restrict__ total) {
  using BR = cub::BlockReduce<int64_t, kNzThreads>;
  __shared__ typename BR::TempStorage tmp;
  const int64_t base = blockIdx.x * kNzChunk;
  int64_t c = 0;
#pragma unroll
  for (int k = 0; k < kNzPer; ++k) {
    const int64_t i = base + (int64_t)k * kNzThreads + threadIdx.x;
    if (i < count && x[i] != 0.0f) ++c;
  }
  const int64_t s = BR(tmp).Sum(c);
  if (threadIdx.x == 0) {
    if (bcnt) bcnt[blockIdx.x] = s;
    if (total) atomicAdd(total, (unsigned long long)s);
  }
}

__global__ void __launch_bounds__(1024)
k_nz_scan(int64_t nb, int64_t* __restrict__ b, int64_t base_rank) {
  using BS = cub::BlockScan<int64_t, 1024>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = base_rank;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < nb ? b[i] : 0;
    int64_t ex, agg;
    BS(tmp).ExclusiveSum(v, ex, agg);
    if (i < nb) b[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
}

// numpy linspace(0, nnz-1, cap) element i, truncated to int64.
__device__ __forceinline__ int64_t np_linspace_pick(int64_t i, int64_t cap, int64_t nnz,
                                                    double step) {
  if (i == cap - 1) return nnz - 1;
  return (int64_t)__dmul_rn((double)i, step);
}

__global__ void __launch_bounds__(kNzThreads)
k_nz_emit(const float* __restrict__ x, int64_t count, const int64_t* __restrict__ boff,
          int64_t nnz, int64_t cap, double step, float* __restrict__ out) {
  using BS = cub::BlockScan<int64_t, kNzThreads>;
  __shared__ typename BS::TempStorage tmp;
  // thread owns kNzPer consecutive elements so ranks follow row-major order
  const int64_t base = blockIdx.x * kNzChunk + (int64_t)threadIdx.x * kNzPer;
  float v[kNzPer];
  int64_t c = 0;
#pragma unroll
  for (int k = 0; k < kNzPer; ++k) {
    v[k] = (base + k < count) ? x[base + k] : 0.0f;
    c += v[k] != 0.0f;
  }
  int64_t r;
  BS(tmp).ExclusiveSum(c, r);
  r += boff[blockIdx.x];
  const bool all = nnz <= cap;
#pragma unroll
  for (int k = 0; k < kNzPer; ++k) {
    if (v[k] == 0.0f) continue;
    if (all) {
      out[r] = fabsf(v[k]);
    } else {
      int64_t i0 = (int64_t)((double)r / step) - 1;
      for (int64_t i = (i0 < 0 ? 0 : i0); i <= i0 + 3 && i < cap; ++i) {
        if (np_linspace_pick(i, cap, nnz, step) == r) { out[i] = fabsf(v[k]); break; }
      }
    }
    ++r;
  }
}

__global__ void k_hist_hi(const float* __restrict__ v, int64_t count, unsigned int* __restrict__ h) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(h + (__float_as_uint(v[i]) >> 16), 1u);
}

__global__ void k_hist_lo(const float* __restrict__ v, int64_t count, uint32_t hi_bin,
                          unsigned int* __restrict__ h) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t b = __float_as_uint(v[i]);
    if ((b >> 16) == hi_bin) atomicAdd(h + (b & 0xFFFFu), 1u);
  }
}

// Lloyd assignment: float64 points vs float64 centroids (vq.py:191-198).
__global__ void k_kmeans_assign(const double* __restrict__ pts, int64_t m, int w,
                                const double* __restrict__ cents, int k, int metric,
                                const double* __restrict__ cc, int32_t* __restrict__ assign,
                                double* __restrict__ cost);

}  // namespace fg

using namespace fg;

extern "C" {

int fg_gather_nonzero_sample_chunk(const float* x, int64_t count, int64_t rank_base,
                                   int64_t nnz, int64_t cap, float* out_abs, void* ws,
                                   int64_t ws_bytes, void* s);

int fg_count_nonzero(const float* x, int64_t count, unsigned long long* out_count, void* s) {
  FG_CHECK_ARG(out_count != nullptr, "fg_count_nonzero: null out");
  cudaStream_t st = as_stream(s);
  FG_CUDA_TRY(cudaMemsetAsync(out_count, 0, sizeof(unsigned long long), st));
  if (count == 0) return FG_OK;
  const int64_t nb = ceil_div(count, kNzChunk);
  k_nz_count<<<(unsigned)nb, kNzThreads, 0, st>>>(x, count, nullptr, out_count);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int64_t fg_nonzero_sample_workspace_bytes(int64_t count) {
  return (ceil_div(count > 0 ? count : 1, kNzChunk) * 8 + 255) & ~int64_t(255);
}

int fg_gather_nonzero_sample(const float* x, int64_t count, int64_t nnz, int64_t cap,
                             float* out_abs, void* ws, int64_t ws_bytes, void* s) {
  return fg_gather_nonzero_sample_chunk(x, count, 0, nnz, cap, out_abs, ws, ws_bytes, s);
}

int fg_gather_nonzero_sample_chunk(const float* x, int64_t count, int64_t rank_base,
                                   int64_t nnz, int64_t cap, float* out_abs, void* ws,
                                   int64_t ws_bytes, void* s) {
  FG_CHECK_ARG(cap >= 2 && nnz >= 0 && rank_base >= 0, "fg_gather_nonzero_sample: bad cap/nnz");
  FG_CHECK_ARG(ws_bytes >= fg_nonzero_sample_workspace_bytes(count), "workspace too small");
  if (count == 0 || nnz == 0) return FG_OK;
  cudaStream_t st = as_stream(s);
  const int64_t nb = ceil_div(count, kNzChunk);
  int64_t* b = (int64_t*)ws;
  k_nz_count<<<(unsigned)nb, kNzThreads, 0, st>>>(x, count, b, nullptr);
  FG_LAUNCH_CHECK();
  k_nz_scan<<<1, 1024, 0, st>>>(nb, b, rank_base);
  FG_LAUNCH_CHECK();
  // numpy: step = delta / div with delta = (nnz-1) - 0, div = cap - 1
  const double step = (double)(nnz - 1) / (double)(cap - 1);
  k_nz_emit<<<(unsigned)nb, kNzThreads, 0, st>>>(x, count, b, nnz, cap, step, out_abs);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int64_t fg_select_workspace_bytes(void) { return 65536 * 4; }

int fg_select_ranks(const float* vals, int64_t count, const int64_t* ranks, int num_ranks,
                    float* out_host, void* ws, int64_t ws_bytes, void* s) {
  FG_CHECK_ARG(ws_bytes >= fg_select_workspace_bytes(), "workspace too small");
  FG_CHECK_ARG(count >= 1, "fg_select_ranks: empty input");
  cudaStream_t st = as_stream(s);
  unsigned int* h = (unsigned int*)ws;
  static thread_local unsigned int hh[65536];
  FG_CUDA_TRY(cudaMemsetAsync(h, 0, 65536 * 4, st));
  k_hist_hi<<<grid_for(count, 256), 256, 0, st>>>(vals, count, h);
  FG_LAUNCH_CHECK();
  FG_CUDA_TRY(cudaMemcpyAsync(hh, h, 65536 * 4, cudaMemcpyDeviceToHost, st));
  FG_CUDA_TRY(cudaStreamSynchronize(st));
  for (int q = 0; q < num_ranks; ++q) {
    FG_CHECK_ARG(ranks[q] >= 0 && ranks[q] < count, "rank out of range");
    int64_t rem = ranks[q];
    uint32_t hb = 0;
    for (; hb < 65536; ++hb) {
      if (rem < (int64_t)hh[hb]) break;
      rem -= hh[hb];
    }
    static thread_local unsigned int hl[65536];
    FG_CUDA_TRY(cudaMemsetAsync(h, 0, 65536 * 4, st));
    k_hist_lo<<<grid_for(count, 256), 256, 0, st>>>(vals, count, hb, h);
    FG_LAUNCH_CHECK();
    FG_CUDA_TRY(cudaMemcpyAsync(hl, h, 65536 * 4, cudaMemcpyDeviceToHost, st));
    FG_CUDA_TRY(cudaStreamSynchronize(st));
    uint32_t lb = 0;
    for (; lb < 65536; ++lb) {
      if (rem < (int64_t)hl[lb]) break;
      rem -= hl[lb];
    }
    const uint32_t bits = (hb << 16) | lb;
    memcpy(out_host + q, &bits, 4);
  }
  return FG_OK;
}

}  // extern "C"

namespace fg {

__device__ __forceinline__ double pw_sumsq_short(const double* v, int n) {
  // numpy pairwise sum for n < 8 (sequential) and 8 <= n <= 128 (8 lanes)
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, __dmul_rn(v[i], v[i]));
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = __dmul_rn(v[j], v[j]);
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], __dmul_rn(v[i + j], v[i + j]));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, __dmul_rn(v[i], v[i]));
  return res;
}

__global__ void k_kmeans_cc(const double* __restrict__ cents, int k, int w, double* __restrict__ cc) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k; e += gridDim.x * blockDim.x)
    cc[e] = pw_sumsq_short(cents + (int64_t)e * w, w);
}

__global__ void k_kmeans_assign(const double* __restrict__ pts, int64_t m, int w,
                                const double* __restrict__ cents, int k, int metric,
                                const double* __restrict__ cc, int32_t* __restrict__ assign,
                                double* __restrict__ cost) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* p = pts + i * w;
    const double ss = metric == FG_METRIC_COSINE ? 0.0 : pw_sumsq_short(p, w);
    int best = 0;
    double bestv = 0.0;
    for (int e = 0; e < k; ++e) {
      const double* c = cents + (int64_t)e * w;
      double dot = __dmul_rn(p[0], c[0]);
      for (int j = 1; j < w; ++j) dot = __fma_rn(p[j], c[j], dot);
      if (metric == FG_METRIC_COSINE) {
        if (e == 0 || dot > bestv) { bestv = dot; best = e; }
      } else {
        double dd = __dadd_rn(__dadd_rn(ss, cc[e]), -__dmul_rn(2.0, dot));
        dd = dd > 0.0 ? dd : 0.0;
        if (e == 0 || dd < bestv) { bestv = dd; best = e; }
      }
    }
    assign[i] = best;
    cost[i] = metric == FG_METRIC_COSINE ? __dadd_rn(1.0, -bestv) : bestv;
  }
}

}  // namespace fg

extern "C" int fg_kmeans_assign(const double* pts, int64_t m, int w, const double* cents, int k,
                                int metric, int32_t* assign, double* cost, double* cc_scratch,
                                void* s) {
  FG_CHECK_ARG(w >= 1 && w <= 128 && k >= 1, "fg_kmeans_assign: bad shape");
  if (m == 0) return FG_OK;
  // the distance step on the tensor cores (screen + float64 recheck; same
  // assignment and exact cost) for the narrow parts k-means fits
  if (w <= 16) return fg_kmeans_assign_tc(pts, m, w, cents, k, metric, assign, cost, s);
  cudaStream_t st = as_stream(s);
  double* cc = nullptr;
  if (metric == FG_METRIC_EUCLIDEAN) {
    FG_CHECK_ARG(cc_scratch != nullptr, "euclidean assignment needs k doubles of scratch");
    cc = cc_scratch;  // (c*c).sum(axis=1) of the centroids
    k_kmeans_cc<<<grid_for(k, 256), 256, 0, st>>>(cents, k, w, cc);
    FG_LAUNCH_CHECK();
  }
  k_kmeans_assign<<<grid_for(m, 128, 16), 128, 0, st>>>(pts, m, w, cents, k, metric, cc, assign,
                                                        cost);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

// ------------------------------------------------ batched k-means++ seeding
// vq.py:166-181 for B independent jobs (every part x restart of fit_vq) at
// once, with no host round trip per centroid: the per-step uniforms
// u[b][c-1] = rng.random() are drawn up front from each job's own Generator
// (the same stream positions the reference consumes, as long as no job hits
// the degenerate `d2.sum() <= 0` branch, which is flagged on the device and
// redone on the host path).  Per step two kernels:
//   k_kpp_search: CTA per job -- total = sum of the block partials (fixed
//     order), target = u * total, the block whose running sum reaches the
//     target, then the first point inside it whose running sum reaches it
//     (np.searchsorted(np.cumsum(d2), target), clamped to m - 1); the point
//     becomes centroid c;
//   k_kpp_update: d2[i] = min(d2[i], ||x_i||^2 + ||c||^2 - 2 x_i.c) clamped at
//     0 (vq.py:154-156 expression order), per-block partial sums of the new d2.
// Float64 throughout; the running sums are blocked (not numpy's sequential
// cumsum), so picks can differ at exact prefix-sum boundaries (objective
// parity, tests/test_gpu_codecs.py).
constexpr int kKppBlock = 1024;

__global__ void __launch_bounds__(kKppBlock)
k_kpp_update(const double* __restrict__ pts, const double* __restrict__ xx,
             const int64_t* __restrict__ mrow, int64_t M, int w,
             const double* __restrict__ cents, int K, int c, double* __restrict__ d2,
             double* __restrict__ part, int64_t nblk, const int* __restrict__ flag) {
  const int64_t b = blockIdx.y;
  if (flag[b]) return;
  __shared__ double s_c[32];
  __shared__ double s_cc;
  __shared__ double s_red[kKppBlock / 32];
  const double* cb = cents + ((int64_t)b * K + c) * w;
  if (threadIdx.x < w) s_c[threadIdx.x] = cb[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    double cc = 0.0;
    for (int j = 0; j < w; ++j) cc += s_c[j] * s_c[j];
    s_cc = cc;
  }
  __syncthreads();
  const int64_t i = blockIdx.x * (int64_t)kKppBlock + threadIdx.x;
  double v = 0.0;
  if (i < mrow[b]) {
    const double* x = pts + (b * M + i) * w;
    double dot = 0.0;
    for (int j = 0; j < w; ++j) dot = fma(x[j], s_c[j], dot);
    const double dist = fmax(xx[b * M + i] + s_cc - 2.0 * dot, 0.0);
    double* dp = d2 + b * M + i;
    v = fmin(*dp, dist);
    *dp = v;
  }
  // fixed-order block sum (warp shuffles, then one warp)
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = s_red[threadIdx.x];
    for (int o = 16; o; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) part[b * nblk + blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024)
k_kpp_search(const double* __restrict__ pts, const int64_t* __restrict__ mrow, int64_t M, int w,
             const double* __restrict__ d2, const double* __restrict__ part, int64_t nblk,
             const double* __restrict__ u, int K, int c, double* __restrict__ cents,
             int* __restrict__ flag) {
  const int64_t b = blockIdx.x;
  if (flag[b]) return;
  __shared__ double s_tot, s_base;
  __shared__ int64_t s_blk;
  __shared__ double s_warp[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double* pb = part + b * nblk;
  // total in fixed order (one warp, strided partials then a shuffle tree)
  if (wid == 0) {
    double t = 0.0;
    for (int64_t j = lane; j < nblk; j += 32) t += pb[j];
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) s_tot = t;
  }
  __syncthreads();
  const double tot = s_tot;
  if (!(tot > 0.0)) {  // degenerate: the host redoes this job exactly
    if (tid == 0) flag[b] = 1;
    return;
  }
  const double target = u[b * (K - 1) + (c - 1)] * tot;
  // block containing the target: warp 0 scans the partials 32 at a time
  if (wid == 0) {
    double run = 0.0;
    int64_t found = nblk - 1;
    double base = 0.0;
    bool done = false;
    for (int64_t j0 = 0; j0 < nblk && !done; j0 += 32) {
      const int64_t j = j0 + lane;
      double v = j < nblk ? pb[j] : 0.0;
      double incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const double n = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += n;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, j < nblk && run + incl >= target);
      if (hit) {
        const int l = __ffs(hit) - 1;
        found = j0 + l;
        base = run + __shfl_sync(0xffffffffu, incl - v, l);
        done = true;
      } else {
        run += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (!done) base = run - (nblk ? pb[nblk - 1] : 0.0);  // clamp: last block
    if (lane == 0) {
      s_blk = found;
      s_base = base;
    }
  }
  __syncthreads();
  // inside the block: inclusive scan of its d2 values, first index >= target
  const int64_t i = s_blk * kKppBlock + tid;
  const double v = i < mrow[b] ? d2[b * M + i] : 0.0;
  double incl = v;
  for (int o = 1; o < 32; o <<= 1) {
    const double n = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += n;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    double t = s_warp[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const double n = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += n;
    }
    s_warp[lane] = t - s_warp[lane];  // exclusive warp offsets
  }
  __syncthreads();
  const double cum = s_base + s_warp[wid] + incl;
  __shared__ int64_t s_pick;
  if (tid == 0) s_pick = INT64_MAX;
  __syncthreads();
  if (i < mrow[b] && cum >= target) atomicMin((unsigned long long*)&s_pick, (unsigned long long)i);
  __syncthreads();
  int64_t pick = s_pick;
  if (pick == INT64_MAX) pick = mrow[b] - 1;  // searchsorted past the end -> clamp
  pick = pick < mrow[b] - 1 ? pick : mrow[b] - 1;
  if (tid < w) cents[((int64_t)b * K + c) * w + tid] = pts[(b * M + pick) * w + tid];
}

extern "C" int fg_kmeanspp_batched(const double* pts, const double* xx, const int64_t* mrow,
                                   int64_t B, int64_t M, int w, int K, const double* u,
                                   double* cents, double* d2, double* part, int* flag,
                                   void* s) {
  FG_CHECK_ARG(pts && xx && mrow && u && cents && d2 && part && flag && B >= 1 && M >= 1 &&
                   w >= 1 && w <= 32 && K >= 1,
               "fg_kmeanspp_batched: bad argument (width <= 32)");
  cudaStream_t st = as_stream(s);
  const int64_t nblk = ceil_div(M, kKppBlock);
  FG_CHECK_ARG(nblk <= 65535 * 1024ll, "fg_kmeanspp_batched: too many points");
  const dim3 ug((unsigned)nblk, (unsigned)B);
  // d2 = +inf before the first centroid: the first update sets d2 = dist(c0)
  k_kpp_update<<<ug, kKppBlock, 0, st>>>(pts, xx, mrow, M, w, cents, K, 0, d2, part, nblk, flag);
  FG_LAUNCH_CHECK();
  for (int c = 1; c < K; ++c) {
    k_kpp_search<<<(unsigned)B, 1024, 0, st>>>(pts, mrow, M, w, d2, part, nblk, u, K, c, cents,
                                                flag);
    FG_LAUNCH_CHECK();
    k_kpp_update<<<ug, kKppBlock, 0, st>>>(pts, xx, mrow, M, w, cents, K, c, d2, part, nblk,
                                            flag);
    FG_LAUNCH_CHECK();
  }
  return FG_OK;
}
