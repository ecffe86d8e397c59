// Deterministic, row-addressable synthetic feature generation on the device
// (SURVEY.md §8d): element (i, j) is a pure function of (seed, i, j), so the
// oracle can regenerate any row subset and configs whose raw matrix cannot be
// held (MAG240M-shape, 750 GB fp32) are produced chunk by chunk and
// compressed on the fly.  Distributions follow the reference's
// generate_features kinds (pkg/src/featgrind/graphstore.py:291-324), plus a
// class-conditional kind with planted labels for the trainer.
#include "fg_common.cuh"

namespace fg {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// two independent uniforms in (0, 1] from one 64-bit hash
__device__ __forceinline__ float gauss(uint64_t key) {
  const uint64_t h = splitmix64(key);
  const float u1 = ((uint32_t)(h >> 40) + 1u) * (1.0f / 16777216.0f);  // (0, 1]
  const float u2 = (uint32_t)(h & 0xFFFFFFu) * (1.0f / 16777216.0f);
  return sqrtf(-2.0f * __logf(u1)) * __cosf(6.2831853f * u2);
}

__device__ __forceinline__ uint64_t elem_key(uint64_t seed, int64_t i, int64_t j) {
  return splitmix64(seed ^ splitmix64((uint64_t)i * 0x100000001B3ull + (uint64_t)j));
}

__global__ void k_synth(int kind, uint64_t seed, int64_t row0, int64_t rows, int64_t d,
                        const int32_t* __restrict__ labels, int num_classes,
                        float* __restrict__ out) {
  const int64_t total = rows * d;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / d, j = t - r * d;
    const int64_t i = row0 + r;
    const float z = gauss(elem_key(seed, i, j));
    float v;
    switch (kind) {
      case 0:  // normal
        v = z;
        break;
      case 1: {  // lognormal magnitude, random sign
        const uint64_t sgn = splitmix64(elem_key(seed ^ 0x5151ull, i, j));
        v = __expf(z) * ((sgn & 1) ? 1.f : -1.f);
        break;
      }
      case 2: {  // correlated: shared direction + per-row noise (weight 0.9)
        const float s = gauss(elem_key(seed ^ 0xC0FFEEull, -1, j));
        v = 0.9486833f * s + 0.31622777f * z;
        break;
      }
      default: {  // class-conditional: mean direction of the planted label
        const int c = labels ? labels[i] : 0;
        const float m = gauss(elem_key(seed ^ 0xC1A55ull, c, j));
        v = 0.6f * m + 0.8f * z;
        break;
      }
    }
    out[t] = v;
  }
}

}  // namespace fg

using namespace fg;

extern "C" int fg_synth_features(int kind, uint64_t seed, int64_t row0, int64_t rows, int64_t d,
                                 const int32_t* labels, int num_classes, float* out, void* s) {
  FG_CHECK_ARG(kind >= 0 && kind <= 3, "fg_synth_features: kind must be 0..3");
  FG_CHECK_ARG(kind != 3 || labels != nullptr, "class-conditional kind needs labels");
  FG_CHECK_ARG(rows >= 0 && d >= 1, "fg_synth_features: bad shape");
  if (rows == 0) return FG_OK;
  k_synth<<<grid_for(rows * d, 256), 256, 0, as_stream(s)>>>(kind, seed, row0, rows, d, labels,
                                                             num_classes, out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}
