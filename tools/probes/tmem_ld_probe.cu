// TMEM -> register read throughput (tcgen05.ld) on one B200, to decide
// whether TMEM can stage the SpMM's gathered X rows instead of shared memory
// (the wide SpMM is bound by the L1TEX LSU pipe, 128 B/clk/SM).
// Each CTA (one per SM) allocates all 512 TMEM columns; W warps repeatedly load
// 32 lanes x NCOL columns (x NCOL 32-bit values per thread) from their lane
// quarter, U loads in flight per wait.  Prints bytes/clk/SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tmem_ld_probe tmem_ld_probe.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NCOL>
__device__ __forceinline__ void ld_tmem(uint32_t taddr, uint32_t (&r)[NCOL]);

template <>
__device__ __forceinline__ void ld_tmem<8>(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

template <int W, int U>
__global__ void __launch_bounds__(W * 32, 1) probe(uint32_t* out, int iters, unsigned long long* clk) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
  uint32_t acc = 0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) ld_tmem<8>(base + (uint32_t)(((it * U + u) * 8 + warp * 24) & 511), r[u]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc ^= r[u][k];
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) out[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int W, int U>
void run(uint32_t* out, unsigned long long* clk) {
  const int iters = 4096;
  probe<W, U><<<148, W * 32>>>(out, iters, clk);
  cudaDeviceSynchronize();
  probe<W, U><<<148, W * 32>>>(out, iters, clk);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < 148; ++i) cyc += (double)h[i] / 148;
  const double bytes = (double)W * iters * U * 32 * 8 * 4;   // per SM
  printf("warps %2d  loads in flight %d  %.1f B/clk/SM  (%s)\n", W, U, bytes / cyc,
         cudaGetErrorString(cudaGetLastError()));
}


// R reader warps (as above, 2 loads in flight) + 4 writer warps (one per lane
// quarter) storing 32x32b.x8 blocks; reports read and write B/clk/SM
template <int R, bool WRITE, bool READ>
__global__ void __launch_bounds__((R + 4) * 32, 1) mix(uint32_t* out, int iters, unsigned long long* clk) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
  uint32_t acc = threadIdx.x;
  unsigned long long t0 = clock64();
  if (warp < R) {
    if (READ)
    for (int it = 0; it < iters; ++it) {
      uint32_t r[2][8];
#pragma unroll
      for (int u = 0; u < 2; ++u) ld_tmem<8>(base + (uint32_t)(((it * 2 + u) * 8 + warp * 24) & 255), r[u]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= r[u][k];
    }
  } else if (WRITE) {
    // writers: columns 256..511, R/4 x fewer iterations' worth of bytes per warp
    for (int it = 0; it < iters; ++it) {
      const uint32_t a = base + 256 + (uint32_t)((it * 8) & 255);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a), "r"(acc), "r"(acc + 1),
                   "r"(acc + 2), "r"(acc + 3), "r"(acc + 4), "r"(acc + 5), "r"(acc + 6), "r"(acc + 7));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  unsigned long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) clk[blockIdx.x * 64 + warp] = t1 - t0;
  if (acc == 0x12345678u) out[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int R, bool WRITE, bool READ>
void runmix(uint32_t* out, unsigned long long* clk, int witers) {
  const int iters = 4096;
  mix<R, WRITE, READ><<<148, (R + 4) * 32>>>(out, READ ? iters : witers, clk);
  cudaDeviceSynchronize();
  mix<R, WRITE, READ><<<148, (R + 4) * 32>>>(out, READ ? iters : witers, clk);
  cudaError_t e = cudaDeviceSynchronize();
  static unsigned long long h[148 * 64];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double rc = 0, wc = 0;
  for (int b = 0; b < 148; ++b) {
    double mr = 0, mw = 0;
    for (int w = 0; w < R; ++w) mr = mr > h[b * 64 + w] ? mr : h[b * 64 + w];
    for (int w = R; w < R + 4; ++w) mw = mw > h[b * 64 + w] ? mw : h[b * 64 + w];
    rc += mr / 148; wc += mw / 148;
  }
  const int it_r = READ ? iters : 0, it_w = READ ? iters : witers;
  printf("readers %d write %d read %d: read %.1f B/clk/SM, write %.1f B/clk/SM (%s)\n", R, (int)WRITE, (int)READ,
         READ ? (double)R * it_r * 2 * 1024 / rc : 0.0, WRITE ? 4.0 * it_w * 1024 / wc : 0.0, cudaGetErrorString(e));
}

int main() {
  uint32_t* out;
  unsigned long long* clk;
  cudaMalloc(&out, 4);
  cudaMalloc(&clk, 148 * 64 * 8);
  run<4, 1>(out, clk);
  run<4, 4>(out, clk);
  run<8, 2>(out, clk);
  run<16, 1>(out, clk);
  run<16, 2>(out, clk);
  run<16, 4>(out, clk);
  run<32, 2>(out, clk);
  runmix<16, false, true>(out, clk, 0);
  runmix<16, true, false>(out, clk, 16384);
  runmix<16, true, true>(out, clk, 0);
  runmix<28, true, true>(out, clk, 0);
  return 0;
}
