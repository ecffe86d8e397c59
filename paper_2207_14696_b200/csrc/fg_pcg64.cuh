// PCG64 (XSL-RR 128/64) as numpy's default_rng drives it, usable on host and
// device, plus the Lemire / masked-interval bounded draws numpy's Generator
// applies to its buffered 32-bit stream.  The reference reaches these through
// pipeline.py:199-216 (default_rng / permutation / choice); the algorithm is
// numpy 2.3.5's (random/_pcg64.pyx, src/distributions/distributions.c).
#pragma once
#include <stdint.h>

#include "../../include/featgrind_b200.h"

#ifdef __CUDACC__
#define FG_HD __host__ __device__ __forceinline__
#else
#define FG_HD inline
#endif

namespace fg {

struct u128 {
  uint64_t lo, hi;
};

FG_HD u128 make_u128(uint64_t hi, uint64_t lo) { u128 r; r.lo = lo; r.hi = hi; return r; }

FG_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// low 128 bits of a * b
FG_HD u128 mul128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo * b.lo;
  r.hi = mulhi64(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}

FG_HD u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1u : 0u);
  return r;
}

// a * s + c (mod 2^128)
FG_HD u128 muladd128(u128 a, u128 s, u128 c) { return add128(mul128(a, s), c); }

#define FG_PCG_MULT_HI 0x2360ED051FC65DA4ULL
#define FG_PCG_MULT_LO 0x4385DF649FCCF645ULL

FG_HD u128 pcg_mult() { return make_u128(FG_PCG_MULT_HI, FG_PCG_MULT_LO); }

FG_HD uint64_t xsl_rr(u128 s) {
  uint64_t v = s.hi ^ s.lo;
  unsigned rot = (unsigned)(s.hi >> 58);
  return (v >> rot) | (v << ((64u - rot) & 63u));
}

// RNG block layout (FG_RNG_WORDS uint64):
//  [0] state.lo [1] state.hi [2] inc.lo [3] inc.hi [4] has_uint32 [5] uinteger
//  [6] last-layer draw count (diagnostic) [7] reserved
//  [8 + 4*i .. 8 + 4*i + 3] : jump table entry i = (A.lo, A.hi, C.lo, C.hi)
//       such that advancing 2^i steps maps s -> A*s + C.
enum { RNG_STATE = 0, RNG_INC = 2, RNG_HAS32 = 4, RNG_BUF = 5, RNG_LAST = 6, RNG_TABLE = 8 };

// Stream cursor that reproduces numpy's pcg64_next32 buffering.
struct PcgCursor {
  u128 s;
  u128 inc;
  uint32_t hi;
  bool have;
  FG_HD uint64_t next64() {
    s = muladd128(s, pcg_mult(), inc);
    return xsl_rr(s);
  }
  FG_HD uint32_t next32() {
    if (have) { have = false; return hi; }
    uint64_t v = next64();
    have = true;
    hi = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  // numpy buffered_bounded_lemire_uint32: uniform on [0, r] for r < 2^32-1.
  // `used` counts 32-bit draws consumed (2f-1 per Floyd node unless a
  // rejection occurs).
  FG_HD uint32_t lemire(uint32_t r, uint32_t& used) {
    if (r == 0) return 0;
    if (r == 0xFFFFFFFFu) { used++; return next32(); }
    uint32_t span = r + 1u;
    uint64_t m = (uint64_t)next32() * span;
    used++;
    uint32_t low = (uint32_t)m;
    if (low < span) {
      uint32_t cut = (0xFFFFFFFFu - r) % span;
      while (low < cut) {
        m = (uint64_t)next32() * span;
        used++;
        low = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
  // numpy random_interval: masked rejection on [0, mx].
  FG_HD uint64_t interval(uint64_t mx) {
    if (mx == 0) return 0;
    uint64_t mask = mx;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
    if (mx <= 0xFFFFFFFFull) {
      for (;;) { uint64_t v = next32() & mask; if (v <= mx) return v; }
    }
    for (;;) { uint64_t v = next64() & mask; if (v <= mx) return v; }
  }
};

// Advance `s` by `steps` 64-bit outputs using the block's jump table.
FG_HD u128 rng_advance(const uint64_t* blk, u128 s, uint64_t steps) {
  int i = 0;
  while (steps) {
    if (steps & 1ull) {
      const uint64_t* e = blk + RNG_TABLE + 4 * i;
      s = muladd128(make_u128(e[1], e[0]), s, make_u128(e[3], e[2]));
    }
    steps >>= 1;
    ++i;
  }
  return s;
}

// Cursor positioned at 32-bit draw index q of the stream whose current
// position is stored in the block (state, has_uint32, uinteger).
FG_HD PcgCursor rng_cursor_at(const uint64_t* blk, uint64_t q) {
  PcgCursor c;
  c.s = make_u128(blk[RNG_STATE + 1], blk[RNG_STATE]);
  c.inc = make_u128(blk[RNG_INC + 1], blk[RNG_INC]);
  c.have = false;
  c.hi = (uint32_t)blk[RNG_BUF];
  if (blk[RNG_HAS32]) {
    if (q == 0) { c.have = true; return c; }
    q -= 1;
  }
  c.s = rng_advance(blk, c.s, q >> 1);
  if (q & 1ull) {
    uint64_t v = c.next64();
    c.have = true;
    c.hi = (uint32_t)(v >> 32);
  }
  return c;
}

// Host: fill jump table for the block's increment.
inline void rng_build_table(uint64_t* blk) {
  u128 a = pcg_mult();
  u128 c = make_u128(blk[RNG_INC + 1], blk[RNG_INC]);
  for (int i = 0; i < 64; ++i) {
    uint64_t* e = blk + RNG_TABLE + 4 * i;
    e[0] = a.lo; e[1] = a.hi; e[2] = c.lo; e[3] = c.hi;
    // 2^(i+1) steps: A' = A*A, C' = C*(A + 1)
    u128 one = make_u128(0, 1);
    c = mul128(c, add128(a, one));
    a = mul128(a, a);
  }
}

}  // namespace fg
