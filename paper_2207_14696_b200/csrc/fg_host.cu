// Library plumbing: error text, device queries, and the host side of the
// PCG64 stream (seeded state import, epoch permutation).
#include <stdarg.h>

#include "fg_common.cuh"
#include "fg_pcg64.cuh"

namespace fg {

static thread_local char g_err[1024] = "";
static unsigned long long g_launches = 0;

void count_launch() { __atomic_fetch_add(&g_launches, 1ull, __ATOMIC_RELAXED); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int sm_count() {
  static thread_local int dev_cached = -1;
  static thread_local int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return sms;
  if (dev != dev_cached) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      sms = v;
    dev_cached = dev;
  }
  return sms;
}

}  // namespace fg

using namespace fg;

extern "C" {

const char* fg_last_error(void) { return g_err; }

int fg_version(void) { return 100; }

int64_t fg_launch_count(void) { return (int64_t)__atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int fg_set_l2_fetch_granularity(int bytes) {
  FG_CHECK_ARG(bytes == 0 || bytes == 32 || bytes == 64 || bytes == 128,
               "fg_set_l2_fetch_granularity: 32, 64 or 128 bytes (0 = query only)");
  if (bytes) FG_CUDA_TRY(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes));
  size_t v = 0;
  FG_CUDA_TRY(cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity));
  return (int)v == bytes || bytes == 0 ? FG_OK : FG_EUSAGE;
}

int fg_get_l2_fetch_granularity(int* out) {
  size_t v = 0;
  FG_CUDA_TRY(cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity));
  *out = (int)v;
  return FG_OK;
}

int fg_sm_count(int* out) {
  FG_CHECK_ARG(out != nullptr, "fg_sm_count: null out");
  *out = sm_count();
  return FG_OK;
}

int fg_rng_init(uint64_t* blk, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                uint64_t inc_lo, int has_uint32, uint32_t uinteger) {
  FG_CHECK_ARG(blk != nullptr, "fg_rng_init: null block");
  memset(blk, 0, sizeof(uint64_t) * FG_RNG_WORDS);
  blk[RNG_STATE] = state_lo;
  blk[RNG_STATE + 1] = state_hi;
  blk[RNG_INC] = inc_lo;
  blk[RNG_INC + 1] = inc_hi;
  blk[RNG_HAS32] = has_uint32 ? 1 : 0;
  blk[RNG_BUF] = uinteger;
  rng_build_table(blk);
  return FG_OK;
}

int fg_rng_read(const uint64_t* blk, uint64_t* state_hi, uint64_t* state_lo, int* has_uint32,
                uint32_t* uinteger) {
  FG_CHECK_ARG(blk && state_hi && state_lo && has_uint32 && uinteger, "fg_rng_read: null arg");
  *state_lo = blk[RNG_STATE];
  *state_hi = blk[RNG_STATE + 1];
  *has_uint32 = (int)blk[RNG_HAS32];
  *uinteger = (uint32_t)blk[RNG_BUF];
  return FG_OK;
}

// Generator.permutation on a 1-d int64 array == Fisher-Yates over the copy,
// i = n-1 .. 1, j = random_interval(i) (numpy _shuffle_raw).  Serial by
// construction (rejection counts are data dependent); one pass per epoch.
int fg_rng_permutation_host(uint64_t* blk, int64_t* ids, int64_t count) {
  FG_CHECK_ARG(blk != nullptr && (ids != nullptr || count == 0), "fg_rng_permutation_host: null arg");
  PcgCursor c;
  c.s = make_u128(blk[RNG_STATE + 1], blk[RNG_STATE]);
  c.inc = make_u128(blk[RNG_INC + 1], blk[RNG_INC]);
  c.have = blk[RNG_HAS32] != 0;
  c.hi = (uint32_t)blk[RNG_BUF];
  for (int64_t i = count - 1; i >= 1; --i) {
    int64_t j = (int64_t)c.interval((uint64_t)i);
    int64_t t = ids[i];
    ids[i] = ids[j];
    ids[j] = t;
  }
  blk[RNG_STATE] = c.s.lo;
  blk[RNG_STATE + 1] = c.s.hi;
  blk[RNG_HAS32] = c.have ? 1 : 0;
  blk[RNG_BUF] = c.hi;
  return FG_OK;
}

}  // extern "C"
