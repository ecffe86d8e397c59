// SQ / VQ codec kernels: layout conversion, encode, gather-decode.
//
// Reference counterparts (pkg/src/featgrind/):
//   bitpack.py:17-83  pack_codes / gather_bit_rows  -> fg_stream_to_rows / fg_rows_to_stream
//   sq.py:114-129     quantize_sq                   -> fg_sq_encode (threshold form)
//   sq.py:132-153     dequantize_sq(c, rows)        -> fg_sq_gather_dequant (LUT form)
//   vq.py:306-327     _assign_part / encode_vq      -> fg_vq_assign (fp64, numpy-ordered)
//   vq.py:330-344     decode_vq(c, rows)            -> fg_vq_gather_decode
// All of these are HBM-bound streaming / gather kernels except fg_vq_assign,
// which is FP64-ALU bound (K = width is tiny).
#include "fg_common.cuh"

namespace fg {

// ------------------------------------------------------------ bit layout

__global__ void k_stream_to_rows(const uint8_t* __restrict__ stream, int64_t stream_bytes,
                                 int64_t n, int64_t row_bits, uint8_t* __restrict__ rows,
                                 int64_t stride) {
  const int64_t total = n * stride;
  const int64_t row_bytes = (row_bits + 7) >> 3;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / stride, b = t - r * stride;
    uint8_t v = 0;
    if (b < row_bytes) {
      const int64_t g = r * row_bits + 8 * b;  // first source bit
      const int64_t byte = g >> 3;
      const int sh = (int)(g & 7);
      uint32_t w = (uint32_t)stream[byte] << 8;
      if (sh && byte + 1 < stream_bytes) w |= stream[byte + 1];
      v = (uint8_t)((w << sh) >> 8);
      const int64_t valid = row_bits - 8 * b;  // bits of this row in the byte
      if (valid < 8) v &= (uint8_t)(0xFF00u >> valid);
    }
    rows[t] = v;
  }
}

__global__ void k_rows_to_stream(const uint8_t* __restrict__ rows, int64_t n, int64_t row_bits,
                                 int64_t stride, uint8_t* __restrict__ stream,
                                 int64_t stream_bytes) {
  const int64_t total_bits = n * row_bits;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < stream_bytes;
       s += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    for (int t = 0; t < 8; ++t) {
      const int64_t g = 8 * s + t;
      uint32_t bit = 0;
      if (g < total_bits) {
        const int64_t r = g / row_bits, o = g - r * row_bits;
        bit = (rows[r * stride + (o >> 3)] >> (7 - (o & 7))) & 1u;
      }
      v = (v << 1) | bit;
    }
    stream[s] = (uint8_t)v;
  }
}

// ------------------------------------------------------------- SQ encode
// Thread per group of 8 consecutive elements of a row: 8 codes * k bits =
// exactly k bytes starting at byte g*k of the row (groups are byte aligned).
template <typename XT, typename TT>
__global__ void k_sq_encode(const XT* __restrict__ x, int64_t n, int64_t d, int k,
                            const TT* __restrict__ thr, uint8_t* __restrict__ rows,
                            int64_t stride) {
  __shared__ TT s_thr[128];
  const int half = 1 << (k - 1);
  for (int i = threadIdx.x; i < half - 1; i += blockDim.x) s_thr[i] = thr[i];
  __syncthreads();
  const int64_t groups = (d + 7) >> 3;
  const int64_t total = n * groups;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / groups, g = t - r * groups;
    const int64_t j0 = g * 8;
    const int cnt = (int)min64(8, d - j0);
    uint64_t acc = 0;  // 8*k <= 64 bits, MSB-first
    for (int e = 0; e < 8; ++e) {
      uint32_t code = 0;
      if (e < cnt) {
        const XT v = x[r * d + j0 + e];
        if (k == 1) {
          code = v >= (XT)0 ? 1u : 0u;  // sq.py:118; -0.0 >= 0 holds
        } else {
          const TT a = (TT)fabs((double)v);
          // offset = #thresholds <= |x| (monotone restatement of sq.py:120-127)
          int lo = 0, hi = half - 1;
          while (lo < hi) {  // first index with thr > a
            const int mid = (lo + hi) >> 1;
            if (s_thr[mid] <= a) lo = mid + 1; else hi = mid;
          }
          const int off = lo;
          code = v >= (XT)0 ? (uint32_t)(half + off) : (uint32_t)(half - 1 - off);
        }
      }
      acc = (acc << k) | code;
    }
    // acc holds 8*k bits right-aligned; emit k bytes MSB first
    uint8_t* dst = rows + r * stride + g * k;
    const int nbytes = (int)min64(k, ((d * k + 7) >> 3) - g * k);
    for (int b = 0; b < nbytes; ++b) dst[b] = (uint8_t)(acc >> (8 * (k - 1 - b)));
  }
}

// ------------------------------------------------- SQ gather dequantize
template <typename OT, typename LT>
__global__ void __launch_bounds__(256)
k_sq_gather(const uint8_t* __restrict__ rows, int64_t n, int64_t d, int k,
            int64_t stride, const LT* __restrict__ lut, const void* ids,
            int ids32, int64_t num_ids, OT* __restrict__ out,
            int32_t* err_flag) {
  // LUT replicated per lane (entry * 32 + lane): random codes never bank
  // conflict.  Thread per (row, 8 codes); the row id is loaded once per
  // group of lanes of the same row (L1 broadcast); 8 outputs are stored as
  // one 16-byte (bf16) / two 16-byte (fp32) vector when aligned.
  extern __shared__ __align__(16) unsigned char s_raw[];
  LT* s_lut = reinterpret_cast<LT*>(s_raw);
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (1 << k) * 32; i += blockDim.x) s_lut[i] = lut[i >> 5];
  __syncthreads();
  const int64_t groups = (d + 7) >> 3;
  const int64_t total = num_ids * groups;
  const uint32_t mask = (1u << k) - 1u;
  const bool vec = (d % 8) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  const bool vec8 = (d % 4) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;  // 8-B aligned groups
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i, g;
    if (total < (1ll << 31)) {  // 32-bit division (the 64-bit one dominated)
      const uint32_t t32 = (uint32_t)t, g32 = (uint32_t)groups;
      i = t32 / g32;
      g = t32 - (uint32_t)i * g32;
    } else {
      i = t / groups;
      g = t - i * groups;
    }
    const int64_t r = ids32 ? (int64_t)__ldg((const int32_t*)ids + i) : __ldg((const int64_t*)ids + i);
    if (r < 0 || r >= n) {
      if (g == 0) atomicExch(err_flag, FG_EDATA);
      continue;
    }
    const uint8_t* src = rows + r * stride + g * k;
    uint64_t acc = 0;
    if (k == 8) {
      acc = bswap64(*reinterpret_cast<const uint64_t*>(src));
    } else if (k == 4) {
      acc = bswap32(*reinterpret_cast<const uint32_t*>(src));
    } else if (k == 2) {
      acc = ((uint32_t)src[0] << 8) | src[1];
    } else {
      for (int b = 0; b < k; ++b) acc = (acc << 8) | src[b];
    }
    const int64_t j0 = g * 8;
    const int cnt = (int)min64(8, d - j0);
    OT* o = out + i * d + j0;
    LT v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t q = (uint32_t)(acc >> (k * (7 - e))) & mask;
      v[e] = s_lut[q * 32 + lane];
    }
    if (sizeof(OT) == 2 && vec8 && (cnt == 8 || cnt == 4)) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const __nv_bfloat162 b2 = __floats2bfloat162_rn((float)v[2 * e], (float)v[2 * e + 1]);
        w[e] = *reinterpret_cast<const uint32_t*>(&b2);
      }
      if (vec && cnt == 8) {
        *reinterpret_cast<uint4*>(o) = make_uint4(w[0], w[1], w[2], w[3]);
      } else {  // 8-byte aligned halves (d % 4 == 0, e.g. d = 100)
        reinterpret_cast<uint2*>(o)[0] = make_uint2(w[0], w[1]);
        if (cnt == 8) reinterpret_cast<uint2*>(o)[1] = make_uint2(w[2], w[3]);
      }
      continue;
    }
    if (vec && cnt == 8) {
      if constexpr (sizeof(OT) == 2) {
        continue;  // handled above
      } else if constexpr (sizeof(OT) == 4) {
        reinterpret_cast<float4*>(o)[0] = make_float4((float)v[0], (float)v[1], (float)v[2], (float)v[3]);
        reinterpret_cast<float4*>(o)[1] = make_float4((float)v[4], (float)v[5], (float)v[6], (float)v[7]);
        continue;
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (e < cnt) o[e] = cvt_out<OT>(v[e]);
  }
}


// ------------------------------------------------------ VQ gather decode
__device__ __forceinline__ uint32_t read_code(const uint8_t* row, int p, int bits) {
  if (bits == 8) return row[p];
  const int64_t bit0 = (int64_t)p * bits;
  const uint8_t* b = row + (bit0 >> 3);
  const int sh = (int)(bit0 & 7);
  // up to 16 + 7 bits -> 3 bytes
  uint32_t w = ((uint32_t)b[0] << 16);
  if (sh + bits > 8) w |= (uint32_t)b[1] << 8;
  if (sh + bits > 16) w |= b[2];
  return (w >> (24 - sh - bits)) & ((1u << bits) - 1u);
}

template <typename OT>
__global__ void k_vq_gather(const uint8_t* __restrict__ rows, int64_t n, int64_t d, int bits,
                            int64_t stride, const float* __restrict__ books, int width,
                            int length, int parts, const void* ids, int ids32,
                            int64_t num_ids, OT* __restrict__ out, int32_t* err_flag) {
  const int64_t total = num_ids * parts;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i;
    int p;
    if (total < (1ll << 31)) {  // 32-bit division
      i = (uint32_t)t / (uint32_t)parts;
      p = (int)((uint32_t)t - (uint32_t)i * (uint32_t)parts);
    } else {
      i = t / parts;
      p = (int)(t - i * parts);
    }
    const int64_t r = ids32 ? (int64_t)((const int32_t*)ids)[i] : ((const int64_t*)ids)[i];
    if (r < 0 || r >= n) {
      if (p == 0) atomicExch(err_flag, FG_EDATA);
      continue;
    }
    const uint32_t c = read_code(rows + r * stride, p, bits);
    if (c >= (uint32_t)length) { atomicExch(err_flag, FG_EDATA); continue; }
    const float* e = books + ((int64_t)p * length + c) * width;
    const int lo = p * width;
    const int wp = (int)min64(width, d - lo);
    OT* o = out + i * d + lo;
    if (wp == 4 && width == 4 && (d % 4) == 0 && sizeof(OT) == 4) {  // one 16-B copy
      *reinterpret_cast<float4*>(o) = __ldg(reinterpret_cast<const float4*>(e));
      continue;
    }
    for (int j = 0; j < wp; ++j) store_out(o + j, __ldg(e + j));
  }
}

// ------------------------------------------------------------ VQ assign
// numpy's pairwise add.reduce (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum) over the squares of a short vector, with explicit
// round-to-nearest intrinsics so nvcc cannot contract into FMAs.
__device__ double np_pairwise_sumsq(const double* v, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, __dmul_rn(v[i], v[i]));
    return r;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dmul_rn(v[j], v[j]);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], __dmul_rn(v[i + j], v[i + j]));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, __dmul_rn(v[i], v[i]));
    return res;
  }
  // n > 128: recursive halving (kept iterative-free for the small widths used;
  // widths > 128 are split the way numpy splits them)
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise_sumsq(v, n2), np_pairwise_sumsq(v + n2, n - n2));
}

// OpenBLAS dgemm inner product: FMA chain in k order from 0.
__device__ __forceinline__ double blas_dot(const double* a, const double* b, int n) {
  double acc = __dmul_rn(a[0], b[0]);
  for (int i = 1; i < n; ++i) acc = __fma_rn(a[i], b[i], acc);
  return acc;
}

constexpr int kMaxWidth = 64;

// Block = one part x a stripe of rows.  The part's codebook is staged in smem
// as float64 together with its squared norms (the (c*c).sum(axis=1) term),
// in tiles of `tile` entries when the whole part does not fit; the running
// best is carried across tiles with the same strict comparison, so the
// first-index tie rule is unchanged.
__device__ __forceinline__ void vq_write_code(uint8_t* rows, int64_t stride, int64_t r, int p,
                                              int bits, int best) {
  // `bits` bits at bit offset p*bits of the row; parts of a row are written
  // by different blocks, so OR big-endian word images atomically.
  const int64_t bit0 = (int64_t)p * bits;
  uint8_t* base = rows + r * stride;
  const int64_t w0 = bit0 >> 5;
  const int sh = (int)(bit0 & 31);
  const uint64_t span = (uint64_t)best << (64 - bits - sh);
  for (int wd = 0; wd < 2; ++wd) {
    const uint32_t be = (uint32_t)(span >> (32 * (1 - wd)));
    if (!be) continue;
    const int64_t wi = w0 + wd;
    if (wi * 4 >= stride) break;
    atomicOr(reinterpret_cast<unsigned int*>(base) + wi, bswap32(be));
  }
}

template <typename XT>
__global__ void k_vq_assign(const XT* __restrict__ x, int64_t n, int64_t d, int width,
                            int length, int parts, const float* __restrict__ books,
                            const int32_t* __restrict__ entries, int metric, int bits,
                            uint8_t* __restrict__ rows, int64_t stride,
                            int32_t* __restrict__ codes32, int tile) {
  extern __shared__ double s_book[];  // [tile][wp] then cc[tile]
  const int p = blockIdx.y;
  const int lo = p * width;
  const int wp = (int)min64(width, d - lo);
  const int L = entries[p];
  double* s_cc = s_book + (int64_t)tile * wp;
  const bool cosine = metric == FG_METRIC_COSINE;
  auto load_tile = [&](int t0) {
    const int cnt = min(tile, L - t0);
    for (int i = threadIdx.x; i < cnt * wp; i += blockDim.x) {
      const int e = i / wp, j = i - e * wp;
      s_book[i] = (double)books[((int64_t)p * length + t0 + e) * width + j];
    }
    __syncthreads();
    if (!cosine)
      for (int e = threadIdx.x; e < cnt; e += blockDim.x)
        s_cc[e] = np_pairwise_sumsq(s_book + e * wp, wp);
    __syncthreads();
  };
  const bool single = tile >= L;
  if (single) load_tile(0);
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += step) {
    const int64_t r = base + threadIdx.x;
    const bool active = r < n;
    double v[kMaxWidth];
    double ss = 0.0;
    bool live = active;  // cosine rows with zero norm keep code 0
    if (active) {
      for (int j = 0; j < wp; ++j) v[j] = (double)x[r * d + lo + j];
      ss = np_pairwise_sumsq(v, wp);
      if (cosine) {
        const double nrm = sqrt(ss);  // np.linalg.norm (vq.py:310)
        if (nrm > 0.0) {
          for (int j = 0; j < wp; ++j) v[j] = __ddiv_rn(v[j], nrm);
        } else {
          live = false;
        }
      }
    }
    int best = 0;
    double bestv = 0.0;
    for (int t0 = 0; t0 < L; t0 += tile) {
      if (!single) {
        __syncthreads();
        load_tile(t0);
      }
      if (live) {
        const int cnt = min(tile, L - t0);
        for (int e = 0; e < cnt; ++e) {
          const int ge = t0 + e;
          if (cosine) {
            const double sv = blas_dot(v, s_book + e * wp, wp);
            if (ge == 0 || sv > bestv) { bestv = sv; best = ge; }  // argmax: first maximum
          } else {
            // (xx + cc) - 2*dot, then max(., 0): vq.py:155-156
            double dd = __dadd_rn(__dadd_rn(ss, s_cc[e]),
                                  -__dmul_rn(2.0, blas_dot(v, s_book + e * wp, wp)));
            dd = dd > 0.0 ? dd : 0.0;
            if (ge == 0 || dd < bestv) { bestv = dd; best = ge; }  // argmin: first minimum
          }
        }
      }
    }
    if (active) {
      if (codes32) codes32[r * parts + p] = best;
      if (rows) vq_write_code(rows, stride, r, p, bits, best);
    }
  }
}

// ---------------------------------------- VQ assign on the tensor cores
// Screening GEMM + exact recheck.  For one codebook part (width w <= 16,
// entries N <= 256 per chunk) the scores S = X^ C^T of a 128-row tile are
// one tcgen05.mma chain (kind::tf32, M = 128, N = 256, K = 8 per MMA) into
// TMEM.  Operands are split 3xTF32 (x = xh + xl, c = ch + cl; D = xh.ch +
// xh.cl + xl.ch), so a score is within ~5e-6 * sum|x_i c_i| of the float64
// value.  Thread r of the epilogue (TMEM lane r = row r) reads its scores,
// finds the screening best and counts entries within a tolerance 20x that
// bound; with a single candidate (the common case) it is provably the float64
// argmin/argmax, otherwise the candidates are re-scored in float64 with the
// reference's exact operation order (blas_dot, np_pairwise_sumsq) and the
// first-index tie rule.  Codes are therefore bit-identical to the fp64 path
// (k_vq_assign above / vq.py:306-327).
constexpr int kTcRows = 128;
constexpr int kTcN = 256;
constexpr int kTcCand = 8;  // near-tie candidates re-scored exactly before a full rescoring

__device__ __forceinline__ uint32_t tc_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // Blackwell descriptor version; SWIZZLE_NONE
  return d;
}
// kind::tf32, D f32, A/B tf32 K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t tc_idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t mb = tc_smem(bar);
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(mb), "r"(parity) : "memory");
}
// tf32 split: hi = top 19 bits (truncation), lo = exact remainder
__device__ __forceinline__ void tf32_split(float v, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(v) & 0xFFFFE000u;
  lo = __float_as_uint(v - __uint_as_float(hi));
}
// byte offset of element (row, k) in a K-major no-swizzle operand whose K
// extent is KB core columns of 4 tf32: core (row/8, k/4) at
// ((row/8) * KB + k/4) * 128, row-in-core stride 16 B
__device__ __forceinline__ uint32_t tc_off(int row, int k, int KB) {
  return (uint32_t)((((row >> 3) * KB + (k >> 2)) << 7) + ((row & 7) << 4) + ((k & 3) << 2));
}

// KM (k-means / Lloyd assignment, vq.py:154-228 via fg_kmeans_assign): rows
// are float64 points already normalised by the caller, the "codebook" is the
// float64 centroid set (one part, `length` = k entries), and the exact
// float64 cost of the chosen centroid is written (cosine: 1 - dot).
template <typename XT, typename BT = float, bool KM = false>
__global__ void __launch_bounds__(kTcRows, 1)
k_vq_assign_tc(const XT* __restrict__ x, int64_t n, int64_t d, int width, int length, int parts,
               const BT* __restrict__ books, const int32_t* __restrict__ entries, int metric,
               int bits, uint8_t* __restrict__ rows, int64_t stride,
               int32_t* __restrict__ codes32, int KB, double* __restrict__ cost = nullptr) {
  // smem: A hi/lo [128 x 4KB floats], B hi/lo [256 x 4KB], cc [256], bar, tmem slot
  extern __shared__ __align__(128) uint8_t tc_mem[];
  const int a_bytes = kTcRows * KB * 16, b_bytes = kTcN * KB * 16;
  uint8_t* sAh = tc_mem;
  uint8_t* sAl = sAh + a_bytes;
  uint8_t* sBh = sAl + a_bytes;
  uint8_t* sBl = sBh + b_bytes;
  float* s_cc = reinterpret_cast<float*>(sBl + b_bytes);          // [256] fp32 |c|^2 (screen)
  double* s_ccd = reinterpret_cast<double*>(s_cc + kTcN);         // [256] fp64 |c|^2 (exact)
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_ccd + kTcN);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(s_bar + 1);
  float* s_cmax = reinterpret_cast<float*>(s_tmem + 1);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int p = blockIdx.y;
  const int lo = p * width;
  const int wp = (int)min64(width, d - lo);
  const int L = KM ? length : entries[p];
  const bool cosine = metric == FG_METRIC_COSINE;
  const BT* book = books + (int64_t)p * length * width;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(tc_smem(s_tmem)), "r"(kTcN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc_smem(s_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *s_tmem;
  const uint32_t idesc = tc_idesc_tf32(kTcN);
  uint32_t phase = 0;
  const int64_t ntiles = (n + kTcRows - 1) / kTcRows;
  const int nchunks = (L + kTcN - 1) / kTcN;
  int64_t tile = blockIdx.x;
  bool b_ready = false;
  // per-row state carried across chunks
  for (; tile < ntiles; tile += gridDim.x) {
    const int64_t r = tile * kTcRows + tid;
    const bool active = r < n;
    float xf[16];
    double ss = 0.0;
    bool live = active;
#pragma unroll
    for (int j = 0; j < 16; ++j) xf[j] = 0.f;
    if (active) {
      for (int j = 0; j < wp; ++j) {
        const double xv = (double)x[r * d + lo + j];
        xf[j] = (float)xv;
        ss = fma(xv, xv, ss);  // > 0 iff the sub-vector is non-zero (no fp64 underflow)
      }
      if (cosine && !KM) {
        if (ss > 0.0) {
          const float inv = (float)(1.0 / sqrt(ss));  // screening only: ~1e-7 relative
          for (int j = 0; j < wp; ++j) xf[j] *= inv;
        } else {
          live = false;
        }
      }
    }
    float xn1 = 0.f;  // sum |x_j| for the screening bound
    for (int j = 0; j < wp; ++j) xn1 += fabsf(xf[j]);
    // A row: split of the (normalised) row, zero padded to K = 4 * KB
    for (int k = 0; k < 4 * KB; ++k) {
      uint32_t h = 0, l = 0;
      if (live && k < wp) tf32_split(xf[k], h, l);
      *reinterpret_cast<uint32_t*>(sAh + tc_off(tid, k, KB)) = h;
      *reinterpret_cast<uint32_t*>(sAl + tc_off(tid, k, KB)) = l;
    }
    // screening best / runner-up over all chunks, and the largest tolerance
    float sb = 0.f, s2 = 0.f, tolmax = 0.f;
    int sbi = -1;
    bool has2 = false;
    int cand[kTcCand];
    int ncand = 0, prev_best = -1;
    bool prev_tie = false;
    for (int ch = 0; ch < nchunks; ++ch) {
      const int e0 = ch * kTcN;
      const int cnt = min(kTcN, L - e0);
      __syncthreads();  // previous chunk's epilogue done with B / TMEM
      // B: this chunk's entries (split) + their norms (once per CTA when the
      // codebook part is a single chunk)
      if (nchunks > 1 || !b_ready) {
      b_ready = true;
      for (int i = tid; i < kTcN * 4 * KB; i += kTcRows) {
        const int e = i / (4 * KB), k = i - e * (4 * KB);
        uint32_t h = 0, l = 0;
        if (e < cnt && k < wp) tf32_split(book[(int64_t)(e0 + e) * width + k], h, l);
        *reinterpret_cast<uint32_t*>(sBh + tc_off(e, k, KB)) = h;
        *reinterpret_cast<uint32_t*>(sBl + tc_off(e, k, KB)) = l;
      }
      float cm = 0.f;
      for (int e = tid; e < kTcN; e += kTcRows) {
        double cd = 0.0, c1 = 0.0;
        double cv[16];
        if (e < cnt) {
          for (int j = 0; j < wp; ++j) {
            cv[j] = (double)book[(int64_t)(e0 + e) * width + j];
            c1 = fmax(c1, fabs(cv[j]));
          }
          cd = np_pairwise_sumsq(cv, wp);
        }
        s_ccd[e] = cd;
        s_cc[e] = (float)cd;
        cm = fmaxf(cm, (float)c1);
      }
      // chunk max |c_j| (for the screening bound)
      for (int o = 16; o; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
      if ((tid & 31) == 0) s_cmax[warp] = cm;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t lbo = 128, sbo = (uint32_t)KB * 128;
        int acc = 0;
        for (int kk = 0; kk < KB; kk += 2) {  // K = 8 tf32 per MMA (2 core columns)
          const uint32_t off = (uint32_t)kk * 128;
          tc_mma(tmem, tc_desc(tc_smem(sAh) + off, lbo, sbo), tc_desc(tc_smem(sBh) + off, lbo, sbo),
                 idesc, acc);
          tc_mma(tmem, tc_desc(tc_smem(sAh) + off, lbo, sbo), tc_desc(tc_smem(sBl) + off, lbo, sbo),
                 idesc, 1u);
          tc_mma(tmem, tc_desc(tc_smem(sAl) + off, lbo, sbo), tc_desc(tc_smem(sBh) + off, lbo, sbo),
                 idesc, 1u);
          acc = 1;
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(tc_smem(s_bar)) : "memory");
      }
      tc_wait(s_bar, phase);
      phase ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;");
      const float cmax = fmaxf(fmaxf(s_cmax[0], s_cmax[1]), fmaxf(s_cmax[2], s_cmax[3]));
      // screening tolerance: 20x the 3xTF32 score error bound
      const float tol_dot = 1e-4f * xn1 * cmax + 1e-30f;
      const float ssf = (float)ss;
      const float tol = cosine ? tol_dot : 2.f * tol_dot + 1e-6f * (ssf + cmax * cmax * wp);
      tolmax = fmaxf(tolmax, tol);
      const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
      for (int c0 = 0; c0 < kTcN; c0 += 32) {  // warp-uniform (tcgen05.ld is collective)
        uint32_t q[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
            "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]),
              "=r"(q[7]), "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]),
              "=r"(q[13]), "=r"(q[14]), "=r"(q[15]), "=r"(q[16]), "=r"(q[17]), "=r"(q[18]),
              "=r"(q[19]), "=r"(q[20]), "=r"(q[21]), "=r"(q[22]), "=r"(q[23]), "=r"(q[24]),
              "=r"(q[25]), "=r"(q[26]), "=r"(q[27]), "=r"(q[28]), "=r"(q[29]), "=r"(q[30]),
              "=r"(q[31])
            : "r"(lane_base + (uint32_t)c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c0 >= cnt) continue;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int e = c0 + j;
          const float dot = __uint_as_float(q[j]);
          float sc = cosine ? dot : fmaxf(fmaf(-2.f, dot, ssf + s_cc[e]), 0.f);
          if (e >= cnt) sc = cosine ? -INFINITY : INFINITY;
          if (sbi < 0) { sb = sc; sbi = e0 + e; continue; }
          const bool better = cosine ? sc > sb : sc < sb;
          if (better) { s2 = sb; has2 = true; sb = sc; sbi = e0 + e; }
          else if (!has2 || (cosine ? sc > s2 : sc < s2)) { s2 = sc; has2 = true; }
        }
      }
      // near-tie rows of the warp: record this chunk's entries within tol of
      // the running best (a superset of those within tol of the final best)
      const bool tie = live && has2 && !(cosine ? s2 < sb - tolmax : s2 > sb + tolmax);
      if (tie && !prev_tie && prev_best >= 0) {
        // entries of earlier chunks were all below the then-best by more
        // than tol, so only that best itself can still be a candidate
        if (ncand < kTcCand) cand[ncand] = prev_best;
        ++ncand;
      }
      if (__any_sync(0xffffffffu, tie)) {
        for (int c0 = 0; c0 < kTcN; c0 += 32) {
          uint32_t q[32];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
              "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]),
                "=r"(q[7]), "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]),
                "=r"(q[13]), "=r"(q[14]), "=r"(q[15]), "=r"(q[16]), "=r"(q[17]), "=r"(q[18]),
                "=r"(q[19]), "=r"(q[20]), "=r"(q[21]), "=r"(q[22]), "=r"(q[23]), "=r"(q[24]),
                "=r"(q[25]), "=r"(q[26]), "=r"(q[27]), "=r"(q[28]), "=r"(q[29]), "=r"(q[30]),
                "=r"(q[31])
              : "r"(lane_base + (uint32_t)c0));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (!tie || c0 >= cnt) continue;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int e = c0 + j;
            if (e >= cnt) break;
            const float dot = __uint_as_float(q[j]);
            const float sc = cosine ? dot : fmaxf(fmaf(-2.f, dot, ssf + s_cc[e]), 0.f);
            if (cosine ? sc >= sb - tolmax : sc <= sb + tolmax) {
              if (ncand < kTcCand) cand[ncand] = e0 + e;
              ++ncand;
            }
          }
        }
      }
      if (!tie) ncand = 0;  // no near-tie so far: nothing but sbi can matter
      prev_tie = tie;
      prev_best = sbi;
      asm volatile("tcgen05.fence::before_thread_sync;");
    }
    int best = 0;
    if (live) {
      // the screening best is provably the float64 best unless the runner-up
      // is within 2x the error bound (tol is 20x); near-ties re-score every
      // entry in float64 with the reference's operation order (rare path)
      const bool alone = !has2 || (cosine ? s2 < sb - tolmax : s2 > sb + tolmax);
      double bestv = 0.0;
      if (alone && !KM) {
        best = sbi;
      } else {
        double v[16];
        for (int j = 0; j < wp; ++j) v[j] = (double)x[r * d + lo + j];
        const double ssx = np_pairwise_sumsq(v, wp);
        if (cosine && !KM) {
          const double nrm = sqrt(ssx);  // np.linalg.norm (vq.py:310)
          for (int j = 0; j < wp; ++j) v[j] = __ddiv_rn(v[j], nrm);
        }
        // k-means needs the exact cost of the chosen centroid even when the
        // screen resolved it alone
        const bool few = alone || ncand <= kTcCand;  // else every entry
        if (alone) { cand[0] = sbi; ncand = 1; }
        const int ne = few ? ncand : L;
        for (int i = 0; i < ne; ++i) {
          const int e = few ? cand[i] : i;
          double cvv[16];
          for (int j = 0; j < wp; ++j) cvv[j] = (double)book[(int64_t)e * width + j];
          const double dt = blas_dot(v, cvv, wp);
          double val = dt;
          if (!cosine) {
            val = __dadd_rn(__dadd_rn(ssx, np_pairwise_sumsq(cvv, wp)), -__dmul_rn(2.0, dt));
            val = val > 0.0 ? val : 0.0;
          }
          // candidates ascend, so strict improvement keeps the first index
          if (i == 0 || (cosine ? val > bestv : val < bestv)) { bestv = val; best = e; }
        }
      }
      if (KM && active) cost[r] = cosine ? __dadd_rn(1.0, -bestv) : bestv;
    }
    if (active) {
      const int code = live ? best : 0;
      if (codes32) codes32[KM ? r : r * parts + p] = code;
      if (!KM && rows) vq_write_code(rows, stride, r, p, bits, code);
    }
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcN));
}

}  // namespace fg

using namespace fg;

extern "C" {

int fg_stream_to_rows(const uint8_t* stream, int64_t stream_bytes, int64_t n, int64_t row_bits,
                      uint8_t* rows, int64_t row_stride, void* s) {
  FG_CHECK_ARG(n >= 0 && row_bits >= 1, "fg_stream_to_rows: bad shape");
  FG_CHECK_ARG(row_stride >= (row_bits + 7) / 8 && row_stride % 16 == 0,
               "fg_stream_to_rows: row_stride must be >= row bytes and a multiple of 16");
  FG_CHECK_ARG(stream_bytes >= (n * row_bits + 7) / 8, "fg_stream_to_rows: stream too short");
  if (n == 0) return FG_OK;
  const int64_t total = n * row_stride;
  k_stream_to_rows<<<grid_for(total, 256), 256, 0, as_stream(s)>>>(stream, stream_bytes, n,
                                                                   row_bits, rows, row_stride);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_rows_to_stream(const uint8_t* rows, int64_t n, int64_t row_bits, int64_t row_stride,
                      uint8_t* stream, int64_t stream_bytes, void* s) {
  FG_CHECK_ARG(n >= 0 && row_bits >= 1, "fg_rows_to_stream: bad shape");
  FG_CHECK_ARG(stream_bytes == (n * row_bits + 7) / 8, "fg_rows_to_stream: stream size mismatch");
  if (stream_bytes == 0) return FG_OK;
  k_rows_to_stream<<<grid_for(stream_bytes, 256), 256, 0, as_stream(s)>>>(rows, n, row_bits,
                                                                         row_stride, stream,
                                                                         stream_bytes);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_sq_encode(const void* x, int x_is_f64, int64_t n, int64_t d, int k, const float* thr,
                 const double* thr64, uint8_t* rows, int64_t stride, void* s) {
  FG_CHECK_ARG(k >= 1 && k <= 8, "k must be in [1, 8], got %d", k);
  FG_CHECK_ARG(n >= 0 && d >= 1, "fg_sq_encode: bad shape");
  FG_CHECK_ARG(stride >= (d * k + 7) / 8 && stride % 16 == 0, "fg_sq_encode: bad row_stride");
  FG_CHECK_ARG(k == 1 || (x_is_f64 ? thr64 != nullptr : thr != nullptr),
               "fg_sq_encode: thresholds required for k >= 2");
  if (n == 0) return FG_OK;
  FG_CUDA_TRY(cudaMemsetAsync(rows, 0, n * stride, as_stream(s)));
  const int64_t total = n * ((d + 7) / 8);
  const int grid = grid_for(total, 256);
  if (x_is_f64)
    k_sq_encode<double, double><<<grid, 256, 0, as_stream(s)>>>((const double*)x, n, d, k, thr64,
                                                                rows, stride);
  else
    k_sq_encode<float, float><<<grid, 256, 0, as_stream(s)>>>((const float*)x, n, d, k, thr, rows,
                                                              stride);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_sq_gather_dequant(const fg_codec_desc* c, const void* ids, int ids32, int64_t num_ids,
                         void* out, int out_dtype, int32_t* err_flag, void* s) {
  FG_CHECK_ARG(c && c->kind == FG_CODEC_SQ, "fg_sq_gather_dequant: not an SQ codec");
  FG_CHECK_ARG(c->bits >= 1 && c->bits <= 8, "fg_sq_gather_dequant: bad k");
  FG_CHECK_ARG(err_flag != nullptr, "fg_sq_gather_dequant: err_flag required");
  if (num_ids == 0) return FG_OK;
  const int64_t total = num_ids * ((c->d + 7) / 8);
  const int grid = grid_for(total, 256);
  cudaStream_t st = as_stream(s);
  static bool attrs = [] {  // replicated LUTs up to 64 KB (k = 8, float64)
    cudaFuncSetAttribute(k_sq_gather<double, double>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 32 * 8);
    cudaFuncSetAttribute(k_sq_gather<float, float>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 32 * 4);
    cudaFuncSetAttribute(k_sq_gather<__nv_bfloat16, float>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 32 * 4);
    return true;
  }();
  (void)attrs;
  if (c->elem_bits == 64) {
    FG_CHECK_ARG(out_dtype == FG_OUT_F64, "float64 codec decodes to float64");
    k_sq_gather<double, double><<<grid, 256, (1 << c->bits) * 32 * 8, st>>>(c->rows, c->n, c->d, c->bits, c->row_stride,
                                                      (const double*)c->table, ids, ids32, num_ids,
                                                      (double*)out, err_flag);
  } else if (out_dtype == FG_OUT_BF16) {
    k_sq_gather<__nv_bfloat16, float><<<grid, 256, (1 << c->bits) * 32 * 4, st>>>(c->rows, c->n, c->d, c->bits, c->row_stride,
                                                    (const float*)c->table, ids, ids32, num_ids,
                                                    (__nv_bfloat16*)out, err_flag);
  } else if (out_dtype == FG_OUT_F32) {
    k_sq_gather<float, float><<<grid, 256, (1 << c->bits) * 32 * 4, st>>>(c->rows, c->n, c->d, c->bits, c->row_stride,
                                                    (const float*)c->table, ids, ids32, num_ids,
                                                    (float*)out, err_flag);
  } else {
    FG_CHECK_ARG(false, "fg_sq_gather_dequant: unsupported out dtype %d", out_dtype);
  }
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_vq_gather_decode(const fg_codec_desc* c, const void* ids, int ids32, int64_t num_ids,
                        void* out, int out_dtype, int32_t* err_flag, void* s) {
  FG_CHECK_ARG(c && c->kind == FG_CODEC_VQ, "fg_vq_gather_decode: not a VQ codec");
  FG_CHECK_ARG(c->bits >= 1 && c->bits <= 16, "fg_vq_gather_decode: bad code bits");
  FG_CHECK_ARG(err_flag != nullptr, "fg_vq_gather_decode: err_flag required");
  if (num_ids == 0) return FG_OK;
  const int64_t total = num_ids * c->num_parts;
  const int grid = grid_for(total, 256);
  cudaStream_t st = as_stream(s);
  if (out_dtype == FG_OUT_F32)
    k_vq_gather<float><<<grid, 256, 0, st>>>(c->rows, c->n, c->d, c->bits, c->row_stride,
                                             (const float*)c->table, c->width, c->length,
                                             c->num_parts, ids, ids32, num_ids, (float*)out,
                                             err_flag);
  else if (out_dtype == FG_OUT_F64)
    k_vq_gather<double><<<grid, 256, 0, st>>>(c->rows, c->n, c->d, c->bits, c->row_stride,
                                              (const float*)c->table, c->width, c->length,
                                              c->num_parts, ids, ids32, num_ids, (double*)out,
                                              err_flag);
  else if (out_dtype == FG_OUT_BF16)
    k_vq_gather<__nv_bfloat16><<<grid, 256, 0, st>>>(c->rows, c->n, c->d, c->bits, c->row_stride,
                                                     (const float*)c->table, c->width, c->length,
                                                     c->num_parts, ids, ids32, num_ids,
                                                     (__nv_bfloat16*)out, err_flag);
  else
    FG_CHECK_ARG(false, "fg_vq_gather_decode: unsupported out dtype %d", out_dtype);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

static int vq_assign_impl(const void* x, int x_is_f64, int64_t n, int64_t d, int width,
                          int length, int parts, const float* books, const int32_t* entries,
                          int metric, int bits, uint8_t* rows, int64_t stride, int32_t* codes32,
                          void* s, bool allow_tc) {
  FG_CHECK_ARG(width >= 1 && width <= kMaxWidth, "fg_vq_assign: width must be in [1, %d]", kMaxWidth);
  FG_CHECK_ARG(parts == (int)((d + width - 1) / width), "fg_vq_assign: parts != ceil(d/width)");
  FG_CHECK_ARG(metric == FG_METRIC_COSINE || metric == FG_METRIC_EUCLIDEAN, "bad metric");
  FG_CHECK_ARG(rows == nullptr || (stride >= ((int64_t)parts * bits + 7) / 8 && stride % 16 == 0),
               "fg_vq_assign: bad row_stride");
  if (n == 0) return FG_OK;
  if (allow_tc && width <= 16) {  // tensor-core screen + exact recheck
    cudaStream_t st = as_stream(s);
    if (rows) FG_CUDA_TRY(cudaMemsetAsync(rows, 0, n * stride, st));
    const int KB = width <= 8 ? 2 : 4;
    const int64_t smem = 2 * (int64_t)kTcRows * KB * 16 + 2 * (int64_t)kTcN * KB * 16 +
                         kTcN * 4 + kTcN * 8 + 8 + 8 + 16;
    const int64_t ntiles = ceil_div(n, kTcRows);
    const int gx = (int)std::max<int64_t>(1, min64(ntiles, ceil_div(2 * sm_count(), parts)));
    dim3 grid(gx, parts);
    if (x_is_f64) {
      FG_CUDA_TRY(cudaFuncSetAttribute(k_vq_assign_tc<double>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_vq_assign_tc<double><<<grid, kTcRows, smem, st>>>((const double*)x, n, d, width, length,
                                                          parts, books, entries, metric, bits,
                                                          rows, stride, codes32, KB);
    } else {
      FG_CUDA_TRY(cudaFuncSetAttribute(k_vq_assign_tc<float>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_vq_assign_tc<float><<<grid, kTcRows, smem, st>>>((const float*)x, n, d, width, length,
                                                         parts, books, entries, metric, bits,
                                                         rows, stride, codes32, KB);
    }
    FG_LAUNCH_CHECK();
    return FG_OK;
  }
  const int64_t budget = 160 * 1024;  // bytes of smem for one codebook tile
  const int tile = (int)min64(length, budget / ((int64_t)(width + 1) * sizeof(double)));
  const int64_t smem = ((int64_t)tile * width + tile) * (int64_t)sizeof(double);
  cudaStream_t st = as_stream(s);
  if (rows) FG_CUDA_TRY(cudaMemsetAsync(rows, 0, n * stride, st));
  const int threads = 128;
  int gx = (int)min64(ceil_div(n, threads), (int64_t)sm_count() * 32 / parts + 1);
  dim3 grid(max(gx, 1), parts);
  if (x_is_f64) {
    FG_CUDA_TRY(cudaFuncSetAttribute(k_vq_assign<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_vq_assign<double><<<grid, threads, smem, st>>>((const double*)x, n, d, width, length, parts,
                                                     books, entries, metric, bits, rows, stride,
                                                     codes32, tile);
  } else {
    FG_CUDA_TRY(cudaFuncSetAttribute(k_vq_assign<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_vq_assign<float><<<grid, threads, smem, st>>>((const float*)x, n, d, width, length, parts,
                                                    books, entries, metric, bits, rows, stride,
                                                    codes32, tile);
  }
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_vq_assign(const void* x, int x_is_f64, int64_t n, int64_t d, int width, int length,
                 int parts, const float* books, const int32_t* entries, int metric, int bits,
                 uint8_t* rows, int64_t stride, int32_t* codes32, void* s) {
  return vq_assign_impl(x, x_is_f64, n, d, width, length, parts, books, entries, metric, bits,
                        rows, stride, codes32, s, true);
}

int fg_vq_assign_fp64(const void* x, int x_is_f64, int64_t n, int64_t d, int width, int length,
                      int parts, const float* books, const int32_t* entries, int metric, int bits,
                      uint8_t* rows, int64_t stride, int32_t* codes32, void* s) {
  return vq_assign_impl(x, x_is_f64, n, d, width, length, parts, books, entries, metric, bits,
                        rows, stride, codes32, s, false);
}

int fg_kmeans_assign_tc(const double* pts, int64_t m, int w, const double* cents, int k,
                        int metric, int32_t* assign, double* cost, void* s) {
  FG_CHECK_ARG(w >= 1 && w <= 16 && k >= 1, "fg_kmeans_assign_tc: width must be in [1, 16]");
  if (m == 0) return FG_OK;
  cudaStream_t st = as_stream(s);
  const int KB = w <= 8 ? 2 : 4;
  const int64_t smem = 2 * (int64_t)kTcRows * KB * 16 + 2 * (int64_t)kTcN * KB * 16 +
                       kTcN * 4 + kTcN * 8 + 8 + 8 + 16;
  const int gx = (int)min64(ceil_div(m, kTcRows), 2 * (int64_t)sm_count());
  auto kern = k_vq_assign_tc<double, double, true>;
  FG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<dim3(gx, 1), kTcRows, smem, st>>>(pts, m, w, w, k, 1, cents, nullptr, metric, 0, nullptr,
                                           0, assign, KB, cost);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

}  // extern "C"

// --------------------------------------------------- code layout (VQ)
namespace fg {
__global__ void k_codes_to_rows(const int32_t* __restrict__ codes, int64_t n, int parts, int bits,
                                uint8_t* __restrict__ rows, int64_t stride) {
  const int64_t row_bytes = ((int64_t)parts * bits + 7) >> 3;
  const int64_t total = n * stride;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / stride, b = t - r * stride;
    uint32_t v = 0;
    if (b < row_bytes) {
      // bits [8b, 8b+8) of the row: gather from the codes that cover them
      for (int k = 0; k < 8; ++k) {
        const int64_t g = 8 * b + k;
        uint32_t bit = 0;
        if (g < (int64_t)parts * bits) {
          const int p = (int)(g / bits), o = (int)(g - (int64_t)p * bits);
          bit = ((uint32_t)codes[r * parts + p] >> (bits - 1 - o)) & 1u;
        }
        v = (v << 1) | bit;
      }
    }
    rows[t] = (uint8_t)v;
  }
}

// Deterministic per-cluster sums in point order (np.bincount with weights,
// vq.py:159-164): `order` is a stable sort of points by cluster, `start`
// the first position of each cluster in it (k+1 entries).
__global__ void k_segment_sums(const double* __restrict__ pts, int64_t m, int w,
                               const int64_t* __restrict__ order, const int64_t* __restrict__ start,
                               int k, double* __restrict__ sums, double* __restrict__ counts) {
  const int64_t total = (int64_t)k * w;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t / w), j = (int)(t - (int64_t)c * w);
    double s = 0.0;
    for (int64_t i = start[c]; i < start[c + 1]; ++i) s = __dadd_rn(s, pts[order[i] * w + j]);
    sums[t] = s;
    if (j == 0) counts[c] = (double)(start[c + 1] - start[c]);
  }
}
}  // namespace fg

extern "C" int fg_codes_to_rows(const int32_t* codes, int64_t n, int parts, int bits,
                                uint8_t* rows, int64_t stride, void* s) {
  FG_CHECK_ARG(bits >= 1 && bits <= 16 && parts >= 1, "fg_codes_to_rows: bad shape");
  FG_CHECK_ARG(stride >= ((int64_t)parts * bits + 7) / 8 && stride % 16 == 0,
               "fg_codes_to_rows: bad row_stride");
  if (n == 0) return FG_OK;
  fg::k_codes_to_rows<<<grid_for(n * stride, 256), 256, 0, as_stream(s)>>>(codes, n, parts, bits,
                                                                           rows, stride);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

extern "C" int fg_segment_sums(const double* pts, int64_t m, int w, const int64_t* order,
                               const int64_t* start, int k, double* sums, double* counts,
                               void* s) {
  FG_CHECK_ARG(w >= 1 && k >= 1, "fg_segment_sums: bad shape");
  fg::k_segment_sums<<<grid_for((int64_t)k * w, 128, 16), 128, 0, as_stream(s)>>>(
      pts, m, w, order, start, k, sums, counts);
  FG_LAUNCH_CHECK();
  return FG_OK;
}
