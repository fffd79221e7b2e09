// tcgen05.cp .32x128b.warpx4 (smem -> all four TMEM lane quarters) as the
// staging path of a gathered-row SpMM: checks the layout (X row j of a 256-float
// window lands so that tcgen05.ld.32x32b.x8 at column 8j gives lane i the
// floats 4i..4i+3 and 128+4i..128+4i+3 of that row, in every lane quarter) and
// times the copy (smem bytes read per clock per SM).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tmem_cp_probe tmem_cp_probe.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

__device__ __forceinline__ void cp32(uint32_t taddr, uint64_t d) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(d));
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ROWS X rows of 256 floats in smem -> TMEM columns [0, 8 ROWS)
template <int ROWS>
__global__ void __launch_bounds__(128, 1) probe(int* bad, int iters, unsigned long long* clk, uint32_t lbo,
                                                uint32_t sbo) {
  extern __shared__ __align__(1024) float xs[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < ROWS * 256; i += blockDim.x) xs[i] = (float)(i / 256 * 1000 + i % 256);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t0 = tbase;
  const uint32_t sx = smem_u32(xs);
  unsigned long long c0 = clock64();
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll 4
      for (int j = 0; j < ROWS; ++j) {
        cp32(t0 + 8 * j, desc(sx + j * 1024, lbo, sbo));
        cp32(t0 + 8 * j + 4, desc(sx + j * 1024 + 512, lbo, sbo));
      }
      commit(&bar);
      mbar_wait(&bar, it & 1);
    }
  }
  __syncthreads();
  unsigned long long c1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = c1 - c0;
  mbar_wait(&bar, (iters - 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");
  int nbad = 0;
  for (int j = 0; j < ROWS; ++j) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(t0 + ((uint32_t)(32 * warp) << 16) + 8 * j));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int k = 0; k < 8; ++k) {
      const float want = (float)(j * 1000 + (k < 4 ? 4 * lane + k : 128 + 4 * lane + k - 4));
      if (__uint_as_float(r[k]) != want) {
        if (nbad == 0 && blockIdx.x == 0 && lane < 2)
          printf("warp %d lane %d row %d k %d got %.0f want %.0f\n", warp, lane, j, k, __uint_as_float(r[k]), want);
        ++nbad;
      }
    }
  }
  if (nbad) atomicAdd(bad, nbad);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t0));
}


template <int SHAPE>
__global__ void __launch_bounds__(128, 1) cp_rate(int iters, unsigned long long* clk) {
  extern __shared__ __align__(1024) float xs[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t0 = tbase, sx = smem_u32(xs);
  unsigned long long c0 = clock64();
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll 8
      for (int j = 0; j < 64; ++j) {
        if (SHAPE == 0) cp32(t0 + 8 * (j & 63), desc(sx + (j & 31) * 1024, 128, 128));
        if (SHAPE == 1) asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(t0 + 8 * (j & 63)), "l"(desc(sx + (j & 7) * 4096, 2048, 256)));
        if (SHAPE == 2) asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(t0 + 4 * (j & 127)), "l"(desc(sx + (j & 15) * 2048, 128, 256)));
      }
    }
    commit(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  unsigned long long c1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = c1 - c0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t0));
}

template <int SHAPE>
void rate(unsigned long long* clk, const char* name, double bytes_per_cp) {
  const int iters = 1000;
  cudaFuncSetAttribute(cp_rate<SHAPE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cp_rate<SHAPE><<<148, 128, 64 * 1024>>>(iters, clk);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < 148; ++i) cyc += (double)h[i] / 148;
  printf("%s: %.1f clk per cp, %.1f smem B/clk/SM (%s)\n", name, cyc / (64.0 * iters), bytes_per_cp * 64 * iters / cyc, cudaGetErrorString(e));
}

int main() {
  int* bad;
  unsigned long long* clk;
  cudaMalloc(&bad, 4);
  cudaMalloc(&clk, 148 * 8);
  const int iters = 2000;
  const uint32_t cfg[][2] = {{128, 128}, {512, 128}};
  for (auto& c : cfg) {
    cudaMemset(bad, 0, 4);
    cudaFuncSetAttribute(probe<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
    probe<32><<<148, 128, 32 * 1024>>>(bad, iters, clk, c[0], c[1]);
    cudaError_t e = cudaDeviceSynchronize();
    int hb = 0;
    unsigned long long h[148];
    cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < 148; ++i) cyc += (double)h[i] / 148;
    printf("lbo %u sbo %u: mismatches %d  smem read %.1f B/clk/SM  (%s)\n", c[0], c[1], hb,
           32.0 * 1024 * iters / cyc, cudaGetErrorString(e));
  }
  rate<0>(clk, "32x128b.warpx4", 512);
  rate<1>(clk, "128x256b", 4096);
  rate<2>(clk, "128x128b", 2048);
  return 0;
}
