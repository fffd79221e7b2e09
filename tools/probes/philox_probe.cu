// Philox4x64-10 throughput probe (run on the B200): blocks/s for several
// implementations of the 64x64->128 multiply, full occupancy.
#include <cstdio>
#include <cstdint>
#include "../../paper_2303_01277_b200/csrc/philox.cuh"

__device__ __forceinline__ void mul_ptx(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  asm("mul.lo.u64 %0, %2, %3;\n\tmul.hi.u64 %1, %2, %3;" : "=l"(lo), "=l"(hi) : "l"(a), "l"(b));
}
// 32-bit decomposition with a known-constant multiplier (b = M).
__device__ __forceinline__ void mul_32(uint64_t a, uint64_t M, uint64_t& hi, uint64_t& lo) {
  const uint32_t al = (uint32_t)a, ah = (uint32_t)(a >> 32);
  const uint32_t ml = (uint32_t)M, mh = (uint32_t)(M >> 32);
  uint32_t p0l, p0h, p1l, p1h, p2l, p2h, p3l, p3h;
  p0l = al * ml; p0h = __umulhi(al, ml);
  p1l = al * mh; p1h = __umulhi(al, mh);
  p2l = ah * ml; p2h = __umulhi(ah, ml);
  p3l = ah * mh; p3h = __umulhi(ah, mh);
  uint32_t lo1, c1, hi0, hi1;
  asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, 0, 0;" : "=r"(lo1), "=r"(c1) : "r"(p0h), "r"(p1l));
  uint32_t lo1b, c2;
  asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;" : "=r"(lo1b), "=r"(c2) : "r"(lo1), "r"(p2l), "r"(c1));
  asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;" : "=r"(hi0), "=r"(hi1) : "r"(p1h), "r"(p2h), "r"(p3h));
  uint32_t h0, h1;
  asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, %5;" : "=r"(h0), "=r"(h1) : "r"(hi0), "r"(p3l), "r"(hi1), "r"(0));
  asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+r"(h0), "+r"(h1) : "r"(c2));
  lo = ((uint64_t)lo1b << 32) | p0l;
  hi = ((uint64_t)h1 << 32) | h0;
}

template <int V>
__device__ __forceinline__ void mul(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  if (V == 0) { lo = a * b; hi = __umul64hi(a, b); }
  else if (V == 1) mul_ptx(a, b, hi, lo);
  else mul_32(a, b, hi, lo);
}

template <int V>
__device__ __forceinline__ uint64_t philox_v(uint64_t c0, uint64_t k0, uint64_t k1) {
  constexpr uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  constexpr uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  uint64_t x0 = c0, x1 = 0, x2 = 0, x3 = 0, h0, l0, h1, l1;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += W0; k1 += W1; }
    mul<V>(x0, M0, h0, l0);
    mul<V>(x2, M1, h1, l1);
    const uint64_t n0 = h1 ^ x1 ^ k0, n2 = h0 ^ x3 ^ k1;
    x1 = l1; x3 = l0; x0 = n0; x2 = n2;
  }
  return x0 ^ x1 ^ x2 ^ x3;
}

template <int V>
__global__ void __launch_bounds__(256) kern(uint64_t* out, int iters, uint64_t k0, uint64_t k1) {
  uint64_t acc = 0;
  uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) acc ^= philox_v<V>(c + (uint64_t)i * 1000003ull, k0, k1);
  if (acc == 0x12345) out[0] = acc;
}

__global__ void __launch_bounds__(256) kern_ref(uint64_t* out, int iters, uint64_t k0, uint64_t k1) {
  uint64_t acc = 0;
  uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    hb::U64x4 u = hb::philox4x64_10(c + (uint64_t)i * 1000003ull, k0, k1);
    acc ^= u.w0 ^ u.w1 ^ u.w2 ^ u.w3;
  }
  if (acc == 0x12345) out[0] = acc;
}

int main() {
  uint64_t* out;
  cudaMalloc(&out, 8);
  const int blocks = 148 * 8, iters = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    launch();
    cudaEventRecord(a);
    for (int k = 0; k < 5; ++k) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double blocks_total = 5.0 * blocks * 256.0 * iters;
    printf("%-12s %.3f ms  %.1f G philox-blocks/s  = %.1f G uniforms/s\n", name, ms / 5,
           blocks_total / (ms / 1e3) / 1e9, 4 * blocks_total / (ms / 1e3) / 1e9);
  };
  run("hb", [&] { kern_ref<<<blocks, 256>>>(out, iters, 1, 2); });
  run("umul64hi", [&] { kern<0><<<blocks, 256>>>(out, iters, 1, 2); });
  run("ptx_mulhi", [&] { kern<1><<<blocks, 256>>>(out, iters, 1, 2); });
  run("mul32", [&] { kern<2><<<blocks, 256>>>(out, iters, 1, 2); });
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
