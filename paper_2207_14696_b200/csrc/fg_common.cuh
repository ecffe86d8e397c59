// Shared helpers for the featgrind-b200 sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/featgrind_b200.h"

namespace fg {

// ---------------------------------------------------------------- errors
// Thread-local last-error text, surfaced through fg_last_error().  Entry
// points never throw across the C ABI; they return FG_OK / FG_EUSAGE /
// FG_EDATA / FG_ECUDA (mirroring the reference's exit codes 0/1/2,
// pkg/src/featgrind/cli.py:46-52 and errors.py:8-13).
void set_error(const char* fmt, ...);

#define FG_CHECK_ARG(cond, ...)                                   \
  do {                                                            \
    if (!(cond)) { ::fg::set_error(__VA_ARGS__); return FG_EUSAGE; } \
  } while (0)

#define FG_CUDA_TRY(expr)                                                    \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) {                                                 \
      ::fg::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                      __FILE__, __LINE__);                                   \
      return FG_ECUDA;                                                       \
    }                                                                        \
  } while (0)

// Every kernel launch of the library goes through FG_LAUNCH_CHECK, which
// also bumps a process-wide launch counter (fg_launch_count) so benchmarks
// can state how many of *our* kernels ran.
void count_launch();
#define FG_LAUNCH_CHECK()            \
  do {                               \
    ::fg::count_launch();            \
    FG_CUDA_TRY(cudaGetLastError()); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();  // cached multiprocessor count of the current device

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

// Grid for a grid-stride loop: enough CTAs to fill every SM `per_sm` times,
// never more than the work needs.
inline int grid_for(int64_t work_items, int threads, int per_sm = 8) {
  int64_t need = ceil_div(work_items > 0 ? work_items : 1, threads);
  int64_t cap = (int64_t)sm_count() * per_sm;
  return (int)(need < cap ? need : cap);
}

// Output element types for decode / aggregate kernels.
template <int OUT> struct OutT;
template <> struct OutT<FG_OUT_F32> { using T = float; };
template <> struct OutT<FG_OUT_BF16> { using T = __nv_bfloat16; };
template <> struct OutT<FG_OUT_F64> { using T = double; };

__device__ __forceinline__ void store_out(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_out(double* p, float v) { *p = (double)v; }
__device__ __forceinline__ void store_out(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

template <typename OT, typename VT>
__device__ __forceinline__ OT cvt_out(VT v) { return (OT)v; }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt_out<__nv_bfloat16, float>(float v) {
  return __float2bfloat16_rn(v);
}

// Streaming loads for read-once data (gathered code rows, index lists).
__device__ __forceinline__ uint4 ldg_stream16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg_stream8(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ldg_stream4(const void* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

// Byte-swap helpers: code rows are MSB-first bitstreams (bitpack.py:17-36),
// so the first byte in memory holds the most significant bits.
__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }
__device__ __forceinline__ uint64_t bswap64(uint64_t x) {
  uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  return ((uint64_t)bswap32(lo) << 32) | bswap32(hi);
}

}  // namespace fg
