// MSB-first code bitstreams on the device (the reference's bitpack module):
//   bitpack.py:17-36  pack_codes       -> fg_bits_pack
//   bitpack.py:39-55  unpack_codes     -> fg_bits_unpack
//   bitpack.py:58-83  gather_bit_rows  -> fg_bit_rows_gather
// Stream layout: code i occupies bits [i*bits, (i+1)*bits), bit 0 of the
// stream is the MSB of byte 0; the final byte is zero-padded.  All three are
// HBM-bound and byte/bit parallel: one thread per output byte (pack) or per
// output element (unpack, gather), so every result byte is written exactly
// once (no atomics, deterministic).
#include "fg_common.cuh"

namespace fg {

// `bits` (1..32) bits starting at absolute stream bit `pos` (MSB first)
__device__ __forceinline__ uint64_t read_bits(const uint8_t* __restrict__ s, int64_t pos,
                                              int bits) {
  const int64_t b0 = pos >> 3;
  const int sh = (int)(pos & 7);
  const int need = (sh + bits + 7) >> 3;  // <= 5 bytes
  uint64_t w = 0;
  for (int i = 0; i < need; ++i) w = (w << 8) | s[b0 + i];
  return (w >> (need * 8 - sh - bits)) & ((1ull << bits) - 1);
}

__global__ void k_bits_pack(const int64_t* __restrict__ codes, int64_t count, int bits,
                            uint8_t* __restrict__ out, int64_t nbytes, int32_t* err) {
  const int64_t total_bits = count * bits;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nbytes;
       j += (int64_t)gridDim.x * blockDim.x) {
    uint32_t byte = 0;
    int64_t c_prev = -1;
    uint64_t v = 0;
    for (int k = 0; k < 8; ++k) {
      const int64_t p = 8 * j + k;
      if (p >= total_bits) break;
      const int64_t c = p / bits;
      if (c != c_prev) {
        const int64_t x = codes[c];
        // the thread holding the code's first bit reports an overflow once
        if ((x < 0 || (bits < 64 && (x >> bits) != 0)) && p == c * bits && err) atomicExch(err, 1);
        v = (uint64_t)x;
        c_prev = c;
      }
      const int within = (int)(p - c * bits);
      byte |= (uint32_t)((v >> (bits - 1 - within)) & 1u) << (7 - k);
    }
    out[j] = (uint8_t)byte;
  }
}

__global__ void k_bits_unpack(const uint8_t* __restrict__ s, int64_t start_bit, int64_t count,
                              int bits, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)read_bits(s, start_bit + i * bits, bits);
}

// out[r, j] = bit (rows[r] * row_bits + j) of the stream, as 0/1 bytes
__global__ void k_bit_rows_gather(const uint8_t* __restrict__ s, int64_t nbytes,
                                  int64_t row_bits, const int64_t* __restrict__ rows,
                                  int64_t nrows, uint8_t* __restrict__ out, int32_t* err) {
  const int64_t total = nrows * row_bits;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / row_bits, j = t - r * row_bits;
    const int64_t row = rows[r];
    uint8_t bit = 0;
    if (row < 0 || (row + 1) * row_bits > nbytes * 8) {
      if (j == 0 && err) atomicExch(err, 1);
    } else {
      const int64_t p = row * row_bits + j;
      bit = (s[p >> 3] >> (7 - (p & 7))) & 1;
    }
    out[t] = bit;
  }
}

}  // namespace fg

using namespace fg;

extern "C" {

int fg_bits_pack(const int64_t* codes, int64_t count, int bits, uint8_t* out, int32_t* err_flag,
                 void* s) {
  FG_CHECK_ARG(bits >= 1 && bits <= 32, "code width must be in [1, 32], got %d", bits);
  FG_CHECK_ARG(count >= 0, "fg_bits_pack: negative count");
  const int64_t nbytes = (count * bits + 7) / 8;
  if (nbytes == 0) return FG_OK;
  k_bits_pack<<<grid_for(nbytes, 256), 256, 0, as_stream(s)>>>(codes, count, bits, out, nbytes,
                                                                err_flag);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_bits_unpack(const uint8_t* stream, int64_t stream_bytes, int64_t start_bit, int64_t count,
                   int bits, int64_t* out, void* s) {
  FG_CHECK_ARG(bits >= 1 && bits <= 32, "code width must be in [1, 32], got %d", bits);
  FG_CHECK_ARG(count >= 0 && start_bit >= 0, "fg_bits_unpack: bad count / start");
  const int64_t need = start_bit + count * bits;
  if (need > stream_bytes * 8) {
    set_error("bitstream too short: need %lld bits, have %lld", (long long)need,
              (long long)(stream_bytes * 8));
    return FG_EDATA;
  }
  if (count == 0) return FG_OK;
  k_bits_unpack<<<grid_for(count, 256), 256, 0, as_stream(s)>>>(stream, start_bit, count, bits,
                                                                 out);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

int fg_bit_rows_gather(const uint8_t* stream, int64_t stream_bytes, int64_t row_bits,
                       const int64_t* rows, int64_t nrows, uint8_t* out, int32_t* err_flag,
                       void* s) {
  FG_CHECK_ARG(row_bits >= 1 && nrows >= 0, "fg_bit_rows_gather: bad shape");
  const int64_t total = nrows * row_bits;
  if (total == 0) return FG_OK;
  k_bit_rows_gather<<<grid_for(total, 256), 256, 0, as_stream(s)>>>(stream, stream_bytes,
                                                                     row_bits, rows, nrows, out,
                                                                     err_flag);
  FG_LAUNCH_CHECK();
  return FG_OK;
}

}  // extern "C"
