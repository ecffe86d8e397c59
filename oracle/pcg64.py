"""Pure-Python restatement of the numpy PCG64 stream as the reference uses it.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference sampler (pipeline.py:199-216) calls
``np.random.default_rng(seed)`` then ``rng.permutation(ids)`` and, per node,
``rng.choice(nbrs, fanout, replace=False)``.  Those live in numpy 2.3.5
(``numpy/random/_generator.pyx``, ``_pcg64.pyx``, ``distributions.c``), which
is not vendored in /root/reference.  Their published algorithms are:

* PCG64 (XSL-RR 128/64): ``state = state * MULT + inc`` (mod 2**128), output
  ``rotr64(hi ^ lo, hi >> 58)`` of the *new* state.
* 32-bit draws are buffered halves of 64-bit outputs: low half first, high
  half kept in ``uinteger`` with ``has_uint32`` set.
* ``choice(pop, f, replace=False)`` with ``pop <= 10000 or f <= pop // 50``:
  Floyd's algorithm for ``j = pop-f .. pop-1`` with a Lemire-32 bounded draw
  on ``[0, j]`` (value already chosen -> take ``j``), then a tail shuffle
  ``i = f-1 .. 1`` swapping ``idx[i]`` with ``idx[lemire(i)]``.
  Otherwise a partial Fisher-Yates over ``arange(pop)`` for
  ``i = pop-1 .. max(pop-f, 1)`` returning ``idx[pop-f:]`` (no extra shuffle).
* ``permutation(arr)``: Fisher-Yates for ``i = n-1 .. 1`` with the masked
  rejection draw ``random_interval(i)`` on 32-bit draws.

Verified draw-for-draw against numpy in tests/test_oracle.py (test_pcg_*).
"""

from __future__ import annotations

MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


def xsl_rr(state: int) -> int:
    hi, lo = state >> 64, state & MASK64
    v = hi ^ lo
    rot = hi >> 58
    return ((v >> rot) | (v << ((64 - rot) & 63))) & MASK64


class Pcg64Stream:
    """A PCG64 generator in the exact state layout numpy exposes."""

    def __init__(self, state: int, inc: int, has32: int = 0, buf: int = 0):
        self.state = state & MASK128
        self.inc = inc & MASK128
        self.has32 = int(bool(has32))
        self.buf = buf & 0xFFFFFFFF
        self.draws32 = 0  # diagnostic: 32-bit draws consumed

    @classmethod
    def from_numpy(cls, bitgen_state: dict) -> "Pcg64Stream":
        s = bitgen_state
        return cls(s["state"]["state"], s["state"]["inc"],
                   s["has_uint32"], s["uinteger"])

    @classmethod
    def seeded(cls, seed: int) -> "Pcg64Stream":
        import numpy as np  # numpy's SeedSequence seeding, then our stream
        return cls.from_numpy(np.random.default_rng(seed).bit_generator.state)

    def as_numpy_state(self) -> dict:
        return {"bit_generator": "PCG64",
                "state": {"state": self.state, "inc": self.inc},
                "has_uint32": self.has32, "uinteger": self.buf}

    def next64(self) -> int:
        self.state = (self.state * PCG_MULT + self.inc) & MASK128
        return xsl_rr(self.state)

    def next32(self) -> int:
        self.draws32 += 1
        if self.has32:
            self.has32 = 0
            return self.buf
        v = self.next64()
        self.has32, self.buf = 1, v >> 32
        return v & 0xFFFFFFFF

    def lemire32(self, r: int) -> int:
        """Uniform on [0, r] (numpy buffered_bounded_lemire_uint32)."""
        if r == 0:
            return 0
        if r == 0xFFFFFFFF:
            return self.next32()
        span = r + 1
        m = self.next32() * span
        low = m & 0xFFFFFFFF
        if low < span:
            cut = (0xFFFFFFFF - r) % span
            while low < cut:
                m = self.next32() * span
                low = m & 0xFFFFFFFF
        return m >> 32

    def interval(self, mx: int) -> int:
        """Uniform on [0, mx] by masked rejection (numpy random_interval)."""
        if mx == 0:
            return 0
        mask = mx
        for sh in (1, 2, 4, 8, 16, 32):
            mask |= mask >> sh
        if mx <= 0xFFFFFFFF:
            while True:
                v = self.next32() & mask
                if v <= mx:
                    return v
        while True:
            v = self.next64() & mask
            if v <= mx:
                return v

    # -- Generator-level operations -------------------------------------

    def choice_noreplace(self, pop: int, f: int) -> list[int]:
        """Index list numpy's ``choice(pop, f, replace=False)`` returns."""
        if pop > 10000 and f > pop // 50:
            # partial Fisher-Yates tail over arange(pop): track only moved slots
            moved: dict[int, int] = {}
            for i in range(pop - 1, max(pop - f, 1) - 1, -1):
                j = self.lemire32(i)
                vi, vj = moved.get(i, i), moved.get(j, j)
                moved[i], moved[j] = vj, vi
            return [moved.get(p, p) for p in range(pop - f, pop)]
        out: list[int] = []
        seen: set[int] = set()
        for j in range(pop - f, pop):
            v = self.lemire32(j)
            if v in seen:
                v = j
            seen.add(v)
            out.append(v)
        for i in range(f - 1, 0, -1):
            j = self.lemire32(i)
            out[i], out[j] = out[j], out[i]
        return out

    def permute(self, values) -> list:
        a = list(values)
        for i in range(len(a) - 1, 0, -1):
            j = self.interval(i)
            a[i], a[j] = a[j], a[i]
        return a


def advance_state(state: int, inc: int, steps: int) -> int:
    """LCG jump-ahead by ``steps`` 64-bit outputs (Brown's algorithm)."""
    acc_mult, acc_plus = 1, 0
    cur_mult, cur_plus = PCG_MULT, inc
    steps &= MASK128
    while steps:
        if steps & 1:
            acc_mult = (acc_mult * cur_mult) & MASK128
            acc_plus = (acc_plus * cur_mult + cur_plus) & MASK128
        cur_plus = ((cur_mult + 1) * cur_plus) & MASK128
        cur_mult = (cur_mult * cur_mult) & MASK128
        steps >>= 1
    return (acc_mult * state + acc_plus) & MASK128
