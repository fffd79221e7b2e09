// L2 -> SM gather bandwidth for 512-byte rows (the d = 128 row-gather SpMM's
// traffic): warp LDG.128 gathers vs cp.async.bulk (TMA) row copies into a
// shared-memory ring, random rows of an L2-resident X (16 MB).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_bulk_gather_probe l2_bulk_gather_probe.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

// each warp: iters x 32 rows; lane group of 32 lanes reads one 512 B row per step (LDG.128)
template <int U>
__global__ void __launch_bounds__(1024, 1) ldg_gather(const float4* __restrict__ X, int nrows, int iters,
                                                      float* out) {
  const int lane = threadIdx.x & 31, gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t r = hash((uint32_t)(gw * iters * U + it * U + u)) % (uint32_t)nrows;
      v[u] = __ldg(X + (size_t)r * 32 + lane);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

// one producer thread per CTA issues 512 B bulk copies into a ring of SLOTS
// rows (BATCH rows per mbarrier); consumer warps sum the landed rows from smem
template <int SLOTS, int BATCH>
__global__ void __launch_bounds__(1024, 1) bulk_gather(const float4* __restrict__ X, int nrows, int rows_per_cta,
                                                       float* out, int consume) {
  extern __shared__ __align__(128) float4 ring[];
  constexpr int NB = SLOTS / BATCH;
  __shared__ __align__(8) uint64_t full[NB], empty[NB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[b])), "r"(nw - 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int nbatch = rows_per_cta / BATCH;
  if (warp == 0) {
    if (lane == 0) {
      for (int k = 0; k < nbatch; ++k) {
        const int b = k % NB;
        uint32_t ph = ((k / NB) & 1) ^ 1;
        asm volatile("{\n\t.reg .pred p;\n\tW0: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W0;\n\t}" ::"r"(smem_u32(&empty[b])), "r"(ph) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[b])), "r"(BATCH * 512) : "memory");
        for (int u = 0; u < BATCH; ++u) {
          const uint32_t r = hash((uint32_t)(blockIdx.x * rows_per_cta + k * BATCH + u)) % (uint32_t)nrows;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
                           smem_u32(ring + (b * BATCH + u) * 32)),
                       "l"(X + (size_t)r * 32), "r"(smem_u32(&full[b]))
                       : "memory");
        }
      }
    }
    return;
  }
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k = 0; k < nbatch; ++k) {
    const int b = k % NB;
    uint32_t ph = (k / NB) & 1;
    asm volatile("{\n\t.reg .pred p;\n\tW1: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W1;\n\t}" ::"r"(smem_u32(&full[b])), "r"(ph) : "memory");
    if (consume) {
      // consumer warp w sums rows w-1, w-1+(nw-1), ... of the batch
      for (int u = warp - 1; u < BATCH; u += nw - 1) {
        const float4 v = ring[(b * BATCH + u) * 32 + lane];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[b])) : "memory");
  }
  if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}

int main() {
  const int nrows = 16 * 1024 * 1024 / 512;           // 16 MB of 512-byte rows
  float4* X;
  float* out;
  cudaMalloc(&X, (size_t)nrows * 512);
  cudaMemset(X, 0, (size_t)nrows * 512);
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  auto report = [&](const char* name, double bytes, auto launch) {
    launch();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("%-34s %8.1f GB/s  (%s)\n", name, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  {
    const int iters = 256;
    report("ldg.128 gather, U=4", 148.0 * 32 * iters * 4 * 512,
           [&] { ldg_gather<4><<<148, 1024>>>(X, nrows, iters, out); });
    report("ldg.128 gather, U=8", 148.0 * 32 * (iters / 2) * 8 * 512,
           [&] { ldg_gather<8><<<148, 1024>>>(X, nrows, iters / 2, out); });
  }
  {
    const int rows_per_cta = 65536;
    const int smem = 256 * 512;
    cudaFuncSetAttribute(bulk_gather<256, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bulk_gather<256, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int consume = 0; consume < 2; ++consume) {
      report(consume ? "bulk 512B, 256 slots, b16, consume" : "bulk 512B, 256 slots, b16", 148.0 * rows_per_cta * 512,
             [&] { bulk_gather<256, 16><<<148, 512, smem>>>(X, nrows, rows_per_cta, out, consume); });
      report(consume ? "bulk 512B, 256 slots, b32, consume" : "bulk 512B, 256 slots, b32", 148.0 * rows_per_cta * 512,
             [&] { bulk_gather<256, 32><<<148, 512, smem>>>(X, nrows, rows_per_cta, out, consume); });
    }
  }
  return 0;
}
