// Single-pass device-wide exclusive prefix (decoupled look-back, Merrill &
// Garland 2016) for kernels that both produce per-item counts and consume
// their global offsets in one launch (sampler layer, bitmap compaction).
//
// Tiles are numbered by an atomic ticket in arrival order, so a tile only
// ever waits on tiles whose CTAs are already running (no deadlock).  Each
// tile publishes a 64-bit status word: flag (2 bits) | value (62 bits);
// FLAG_AGG = the tile's own aggregate, FLAG_INC = inclusive prefix.  The
// status array and the ticket are zeroed by the launcher (memset node).
#pragma once
#include <stdint.h>

namespace fg {

constexpr unsigned long long kScanFlagAgg = 1ull << 62;
constexpr unsigned long long kScanFlagInc = 2ull << 62;
constexpr unsigned long long kScanValMask = (1ull << 62) - 1;

struct ScanState {
  unsigned long long* status;  // [num_tiles]
  unsigned int* ticket;        // tile ticket
  unsigned int* done;          // completion ticket (last-block detection)
};

// Thread 0 draws this CTA's tile index; broadcast through smem.
__device__ __forceinline__ unsigned int scan_take_tile(const ScanState& s, unsigned int* smem_slot) {
  if (threadIdx.x == 0) *smem_slot = atomicAdd(s.ticket, 1u);
  __syncthreads();
  return *smem_slot;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Returns the exclusive prefix of `tile` given its aggregate (values are
// non-negative sums of packed fields; must stay < 2^62).  All threads call;
// warp 0 performs a 32-wide parallel look-back over predecessor tiles.
__device__ __forceinline__ unsigned long long scan_tile_prefix(const ScanState& s, unsigned int tile,
                                                               unsigned long long agg,
                                                               unsigned long long* smem_slot) {
  if (threadIdx.x < 32) {
    volatile unsigned long long* st = s.status;
    const int lane = threadIdx.x;
    unsigned long long prefix = 0;
    if (tile == 0) {
      if (lane == 0) st[0] = kScanFlagInc | agg;
    } else {
      if (lane == 0) {
        st[tile] = kScanFlagAgg | agg;
        __threadfence();
      }
      __syncwarp();
      int64_t base = (int64_t)tile - 1;
      while (true) {
        const int64_t j = base - lane;
        unsigned long long w = kScanFlagInc;  // before tile 0: prefix 0
        if (j >= 0) w = st[j];
        while (__any_sync(0xffffffffu, (w >> 62) == 0)) {
          if ((w >> 62) == 0) w = st[j];
        }
        const unsigned int inc = __ballot_sync(0xffffffffu, (w >> 62) == 2);
        if (inc) {
          const int first = __ffs(inc) - 1;  // nearest predecessor with an inclusive prefix
          prefix += warp_sum_u64(lane <= first ? (w & kScanValMask) : 0ull);
          break;
        }
        prefix += warp_sum_u64(w & kScanValMask);
        base -= 32;
      }
      if (lane == 0) {
        __threadfence();
        st[tile] = kScanFlagInc | (prefix + agg);
      }
    }
    if (lane == 0) *smem_slot = prefix;
  }
  __syncthreads();
  return *smem_slot;
}

// True in every thread of the CTA that finishes last (after a
// __threadfence, so it sees all other CTAs' global writes).
__device__ __forceinline__ bool scan_last_block(const ScanState& s, unsigned int num_tiles,
                                                unsigned int* smem_slot) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) *smem_slot = atomicAdd(s.done, 1u) == num_tiles - 1 ? 1u : 0u;
  __syncthreads();
  const bool last = *smem_slot != 0;
  if (last) __threadfence();
  return last;
}

}  // namespace fg
