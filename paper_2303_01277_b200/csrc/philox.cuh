// Philox4x64-10 on sm_100a, bit-identical to numpy's np.random.Philox as
// consumed by halobit's RngStream (reference rngstream.py:26-39):
//   element i of a stream = philox4x64_10(ctr = {i/4 + 1, 0, 0, 0}, key)[i % 4]
//   uniform                = (word >> 11) * 2^-53
// The counter's high words are zero for every stream the halo path draws
// (< 2^66 elements), which removes one 64x64 product from round 1.
#pragma once
#include <cstdint>

namespace hb {

struct U64x4 { uint64_t w0, w1, w2, w3; };

__device__ __forceinline__ void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  lo = a * b;
  hi = __umul64hi(a, b);
}

// Full Philox4x64-10 block for counter {c0, 0, 0, 0}.
__device__ __forceinline__ U64x4 philox4x64_10(uint64_t c0, uint64_t k0, uint64_t k1) {
  constexpr uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  constexpr uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  uint64_t x0, x1, x2, x3, hi0, lo0, hi1, lo1;
  // round 1: x1 = x2 = x3 = 0  ->  mul(M1, x2) = 0
  mulhilo64(M0, c0, hi0, lo0);
  x0 = k0;            // hi1 ^ x1 ^ k0 with hi1 = x1 = 0
  x1 = 0;             // lo1
  x2 = hi0 ^ k1;      // hi0 ^ x3 ^ k1 with x3 = 0
  x3 = lo0;
#pragma unroll
  for (int r = 1; r < 10; ++r) {
    k0 += W0;
    k1 += W1;
    mulhilo64(M0, x0, hi0, lo0);
    mulhilo64(M1, x2, hi1, lo1);
    const uint64_t n0 = hi1 ^ x1 ^ k0;
    const uint64_t n2 = hi0 ^ x3 ^ k1;
    x1 = lo1;
    x3 = lo0;
    x0 = n0;
    x2 = n2;
  }
  return {x0, x1, x2, x3};
}

// Two independent blocks with interleaved rounds: doubles the ILP of the
// (latency-bound) 64-bit multiply chains.
__device__ __forceinline__ void philox4x64_10_x2(uint64_t ca, uint64_t cb, uint64_t k0, uint64_t k1,
                                                 U64x4& ra, U64x4& rb) {
  constexpr uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  constexpr uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  uint64_t a0, a1, a2, a3, b0, b1, b2, b3;
  uint64_t ah0, al0, ah1, al1, bh0, bl0, bh1, bl1;
  mulhilo64(M0, ca, ah0, al0);
  mulhilo64(M0, cb, bh0, bl0);
  a0 = k0; a1 = 0; a2 = ah0 ^ k1; a3 = al0;
  b0 = k0; b1 = 0; b2 = bh0 ^ k1; b3 = bl0;
#pragma unroll
  for (int r = 1; r < 10; ++r) {
    k0 += W0;
    k1 += W1;
    mulhilo64(M0, a0, ah0, al0);
    mulhilo64(M0, b0, bh0, bl0);
    mulhilo64(M1, a2, ah1, al1);
    mulhilo64(M1, b2, bh1, bl1);
    const uint64_t na0 = ah1 ^ a1 ^ k0, na2 = ah0 ^ a3 ^ k1;
    const uint64_t nb0 = bh1 ^ b1 ^ k0, nb2 = bh0 ^ b3 ^ k1;
    a1 = al1; a3 = al0; a0 = na0; a2 = na2;
    b1 = bl1; b3 = bl0; b0 = nb0; b2 = nb2;
  }
  ra = {a0, a1, a2, a3};
  rb = {b0, b1, b2, b3};
}

__device__ __forceinline__ double u53_to_double(uint64_t w) {
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ uint64_t pick(const U64x4& b, int s) {
  return s == 0 ? b.w0 : (s == 1 ? b.w1 : (s == 2 ? b.w2 : b.w3));
}

}  // namespace hb
