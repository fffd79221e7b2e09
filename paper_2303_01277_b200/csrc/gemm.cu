// Dense combine GEMMs of the GNN layer on the 5th-gen tensor cores (tcgen05):
//   Z = P W            (trainer.py:294)   M = rows,   N = d_out, K = d_in
//   G = P^T m          (trainer.py:313)   M = d_in,   N = d_out, K = rows (split-K)
//   T = m W^T          (trainer.py:318-321)
// fp32 operands, fp32 accuracy through the 3xTF32 split: a = a_hi + a_lo
// (a_hi = tf32(a), a_lo = tf32(a - a_hi)); D += A_hi B_hi + A_hi B_lo + A_lo B_hi,
// accumulated in TMEM (fp32).  One elected thread issues tcgen05.mma; operands
// are staged (split on the fly) in shared memory in the K-major no-swizzle
// "interleaved" canonical layout; completion is tracked with tcgen05.commit on
// an mbarrier per stage; the epilogue reads TMEM with tcgen05.ld.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include "common.cuh"

namespace hb {

constexpr int kGM = 128;     // UMMA M (rows of the tile, = TMEM lanes)
constexpr int kGK = 32;      // K per stage (4 MMAs of K = 8)
constexpr int kGThreads = 128;

__device__ __forceinline__ uint32_t f2tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// K-major, SWIZZLE_NONE smem descriptor (version 1 for sm_100).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

// kind::tf32, D fp32, A/B tf32 K-major, M = 128, N = BN.
template <int BN>
__device__ __forceinline__ constexpr uint32_t make_idesc() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(kGM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Stage one operand tile (ROWS x kGK, logical [row][k]) into the interleaved
// K-major layout: byte(row, k) = (k/4)*(ROWS*16) + (row/8)*128 + (row%8)*16 + (k%4)*4.
// Element (row, k) of the operand lives at base + row*ld_r + k*ld_k.
template <int ROWS>
__device__ __forceinline__ void stage_tile(uint32_t* hi, uint32_t* lo, const float* __restrict__ base,
                                           int64_t ld_r, int64_t ld_k, int rows_valid, int k_valid) {
  const int tid = threadIdx.x;
  if (ld_k == 1) {
    // K contiguous: float4 along k
    for (int idx = tid; idx < ROWS * (kGK / 4); idx += kGThreads) {
      const int r = idx / (kGK / 4), c4 = idx % (kGK / 4);
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (r < rows_valid) {
        const float* p = base + (int64_t)r * ld_r + 4 * c4;
        if (4 * c4 + 3 < k_valid && ((((uintptr_t)p) & 15) == 0)) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(p));
          v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (4 * c4 + e < k_valid) v[e] = __ldg(p + e);
        }
      }
      const uint32_t off = (uint32_t)c4 * (ROWS * 4) + (uint32_t)(r >> 3) * 32 + (uint32_t)(r & 7) * 4;
      uint4 h, l;
      h.x = f2tf32(v[0]); l.x = f2tf32(v[0] - __uint_as_float(h.x));
      h.y = f2tf32(v[1]); l.y = f2tf32(v[1] - __uint_as_float(h.y));
      h.z = f2tf32(v[2]); l.z = f2tf32(v[2] - __uint_as_float(h.z));
      h.w = f2tf32(v[3]); l.w = f2tf32(v[3] - __uint_as_float(h.w));
      *reinterpret_cast<uint4*>(hi + off) = h;
      *reinterpret_cast<uint4*>(lo + off) = l;
    }
  } else {
    // rows contiguous (ld_r == 1) or generic: 4 consecutive rows per thread, one k
    for (int idx = tid; idx < (ROWS / 4) * kGK; idx += kGThreads) {
      const int k = idx / (ROWS / 4), r0 = 4 * (idx % (ROWS / 4));
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (k < k_valid) {
        const float* p = base + (int64_t)k * ld_k + (int64_t)r0 * ld_r;
        if (ld_r == 1 && r0 + 3 < rows_valid && ((((uintptr_t)p) & 15) == 0)) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(p));
          v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (r0 + e < rows_valid) v[e] = __ldg(p + (int64_t)e * ld_r);
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = r0 + e;
        const uint32_t off = (uint32_t)(k >> 2) * (ROWS * 4) + (uint32_t)(r >> 3) * 32 + (uint32_t)(r & 7) * 4 + (k & 3);
        const uint32_t h = f2tf32(v[e]);
        hi[off] = h;
        lo[off] = f2tf32(v[e] - __uint_as_float(h));
      }
    }
  }
}

// One CTA computes a kGM x BN tile of C over the K range [k_begin, k_end).
// C[m, n] = sum_k A[m, k] B[k, n]; A(m,k) = A + m*lda_m + k*lda_k, B(k,n) = B + k*ldb_k + n*ldb_n.
// Epilogue: out = acc (+ beta * C_old); if relu_out, also relu_out = max(out, 0).
// Split-K (gridDim.z > 1): the CTA writes its partial tile to ws[z] instead.
template <int BN>
__global__ void __launch_bounds__(kGThreads, 1)
gemm_tf32x3_kernel(int M, int N, int K, const float* __restrict__ A, int64_t lda_m, int64_t lda_k,
                   const float* __restrict__ B, int64_t ldb_k, int64_t ldb_n, float* __restrict__ C,
                   int64_t ldc, float beta, float* __restrict__ relu_out, int64_t ldr,
                   float* __restrict__ ws, int k_chunk) {
  extern __shared__ __align__(128) uint8_t gsm[];
  constexpr int A_WORDS = kGM * kGK, B_WORDS = BN * kGK;
  constexpr int STAGE_WORDS = 2 * A_WORDS + 2 * B_WORDS;
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tmem_base_s;
  uint32_t* smem = reinterpret_cast<uint32_t*>(gsm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kGM, n0 = blockIdx.y * BN;
  const int k_begin = blockIdx.z * k_chunk;
  const int k_end = min(K, k_begin + k_chunk);
  constexpr uint32_t TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;
  constexpr uint32_t idesc = make_idesc<BN>();
  uint32_t phase[2] = {0u, 0u};
  const int nk = (k_end - k_begin + kGK - 1) / kGK;

  for (int kt = 0; kt < nk; ++kt) {
    const int st = kt & 1;
    if (kt >= 2) {  // the MMAs that read this stage (issued at kt-2) must have finished
      mbar_wait(&bar[st], phase[st]);
      phase[st] ^= 1u;
    }
    uint32_t* sA_hi = smem + st * STAGE_WORDS;
    uint32_t* sA_lo = sA_hi + A_WORDS;
    uint32_t* sB_hi = sA_lo + A_WORDS;
    uint32_t* sB_lo = sB_hi + B_WORDS;
    const int k0 = k_begin + kt * kGK;
    const int kv = min(kGK, k_end - k0);
    stage_tile<kGM>(sA_hi, sA_lo, A + (int64_t)m0 * lda_m + (int64_t)k0 * lda_k, lda_m, lda_k, M - m0, kv);
    // B operand as [n][k]: element (n, k) = B + k*ldb_k + n*ldb_n
    stage_tile<BN>(sB_hi, sB_lo, B + (int64_t)k0 * ldb_k + (int64_t)n0 * ldb_n, ldb_n, ldb_k, N - n0, kv);
    fence_proxy_async_smem();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a_hi = smem_u32(sA_hi), a_lo = smem_u32(sA_lo);
      const uint32_t b_hi = smem_u32(sB_hi), b_lo = smem_u32(sB_lo);
      constexpr uint32_t LBO_A = kGM * 16, LBO_B = BN * 16;   // bytes between K chunks of 4
#pragma unroll
      for (int kk = 0; kk < kGK / 8; ++kk) {
        const uint32_t oa = (uint32_t)(2 * kk) * LBO_A, ob = (uint32_t)(2 * kk) * LBO_B;
        const uint64_t dah = make_desc(a_hi + oa, LBO_A, 128), dal = make_desc(a_lo + oa, LBO_A, 128);
        const uint64_t dbh = make_desc(b_hi + ob, LBO_B, 128), dbl = make_desc(b_lo + ob, LBO_B, 128);
        const uint32_t acc0 = (kt > 0 || kk > 0) ? 1u : 0u;
        mma_tf32(tmem, dah, dbh, idesc, acc0);
        mma_tf32(tmem, dah, dbl, idesc, 1u);
        mma_tf32(tmem, dal, dbh, idesc, 1u);
      }
      mma_commit(&bar[st]);
    }
    __syncwarp();
  }
  // wait for the last (up to two) outstanding commits
  for (int s = 0; s < 2; ++s) {
    const int uses = nk > s ? (nk - s + 1) / 2 : 0;   // commits issued on stage s
    const int waited = nk > s + 2 ? (nk - s - 2 + 1) / 2 : 0;
    if (uses > waited) mbar_wait(&bar[s], phase[s]);
  }
  asm volatile("tcgen05.fence::after_thread_sync;");

  // ---- epilogue: TMEM lane = row (warp w owns lanes 32w..32w+31), column = n --
  const int row = m0 + warp * 32 + lane;
  const bool split = gridDim.z > 1;
  float* crow = split ? ws + ((int64_t)blockIdx.z * M + row) * N : C + (int64_t)row * ldc;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 8) {
    uint32_t r[8];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
                 "tcgen05.wait::ld.sync.aligned;"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
    if (row < M) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int n = n0 + c0 + e;
        if (n < N) {
          float v = __uint_as_float(r[e]);
          if (!split) {
            if (beta != 0.f) v += beta * crow[n];
            crow[n] = v;
            if (relu_out) relu_out[(int64_t)row * ldr + n] = (v > 0.f || v != v) ? v : 0.f;
          } else {
            crow[n] = v;
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// Deterministic split-K reduction: C = sum_z ws[z] (+ beta C), fixed order.
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int M, int N, float* __restrict__ C,
                                     int64_t ldc, float beta) {
  const int64_t total = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int z = 0; z < splits; ++z) acc += ws[(int64_t)z * total + i];
    const int64_t m = i / N, n = i - m * N;
    float* c = C + m * ldc + n;
    *c = beta != 0.f ? acc + beta * *c : acc;
  }
}

template <int BN>
static cudaError_t launch_bn(int M, int N, int K, const float* A, int64_t lda_m, int64_t lda_k, const float* B,
                             int64_t ldb_k, int64_t ldb_n, float* C, int64_t ldc, float beta, float* relu_out,
                             int64_t ldr, float* ws, int64_t ws_floats, cudaStream_t st) {
  const size_t smem = (size_t)2 * (2 * kGM * kGK + 2 * BN * kGK) * 4;
  cudaFuncSetAttribute(gemm_tf32x3_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int gm = (M + kGM - 1) / kGM, gn = (N + BN - 1) / BN;
  int splits = 1;
  const int ctas = gm * gn;
  // split-K reduces into C without the ReLU copy: keep one split when a
  // ReLU output is requested
  if (ws != nullptr && relu_out == nullptr && ctas < num_sms() && K >= 4 * kGK) {
    splits = num_sms() / ctas;
    const int max_by_k = (K + 4 * kGK - 1) / (4 * kGK);
    if (splits > max_by_k) splits = max_by_k;
    const int64_t max_by_ws = ws_floats / ((int64_t)M * N);
    if (splits > max_by_ws) splits = (int)max_by_ws;
    if (splits < 1) splits = 1;
  }
  int k_chunk = (K + splits - 1) / splits;
  k_chunk = (k_chunk + kGK - 1) / kGK * kGK;
  splits = (K + k_chunk - 1) / k_chunk;
  if (splits < 1) splits = 1;
  dim3 grid(gm, gn, splits);
  gemm_tf32x3_kernel<BN><<<grid, kGThreads, smem, st>>>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta,
                                                         splits > 1 ? nullptr : relu_out, ldr,
                                                         splits > 1 ? ws : nullptr, k_chunk > 0 ? k_chunk : kGK);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (splits > 1) {
    int g = (int)(((int64_t)M * N + 255) / 256);
    if (g > num_sms() * 8) g = num_sms() * 8;
    splitk_reduce_kernel<<<g, 256, 0, st>>>(ws, splits, M, N, C, ldc, beta);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_gemm_tma(int, int, int, const float*, int64_t, int64_t, const float*, int64_t, int64_t, float*,
                            int64_t, float, float*, int64_t, float*, int64_t, cudaStream_t);

int g_gemm_path = 0;   // 0: TMA warp-specialised kernel when operands allow; 1: SIMT-staged kernel only
int g_gemm_ts = 0;     // 1: A split into TMEM (tcgen05.mma A-from-TMEM) kernel

cudaError_t launch_gemm_ts(int, int, int, const float*, int64_t, int64_t, const float*, int64_t, int64_t, float*,
                           int64_t, float, float*, int64_t, float*, int64_t, cudaStream_t);

cudaError_t launch_gemm_tf32x3(int M, int N, int K, const float* A, int64_t lda_m, int64_t lda_k, const float* B,
                               int64_t ldb_k, int64_t ldb_n, float* C, int64_t ldc, float beta, float* relu_out,
                               int64_t ldr, float* ws, int64_t ws_floats, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (K <= 0) return cudaErrorInvalidValue;
  if (C == nullptr)   // ReLU copy only: the A-in-TMEM kernel's TMA-store epilogue
    return launch_gemm_ts(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws, ws_floats, st);
  if (g_gemm_path == 0) {
    const cudaError_t e = launch_gemm_tma(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr,
                                          ws, ws_floats, st);
    if (e != cudaErrorNotSupported) return e;
  }
  if (N <= 32) return launch_bn<32>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws, ws_floats, st);
  if (N <= 64) return launch_bn<64>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws, ws_floats, st);
  if (N <= 128) return launch_bn<128>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws, ws_floats, st);
  // N > 128: 256-wide tiles over N
  return launch_bn<256>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws, ws_floats, st);
}

cudaError_t launch_gemm_ts_dual(int, int, int, const float*, int64_t, int64_t, const float*, int64_t, int64_t, int,
                                const float*, int64_t, int64_t, const float*, int64_t, int64_t, float*, int64_t, float,
                                float*, int64_t, float*, int64_t, cudaStream_t);

// C = A1 B1 + A2 B2 (+ beta C): one pass of the A-in-TMEM kernel over both K
// ranges when the operands allow (C written once, no read-back), otherwise
// two accumulating GEMMs.
cudaError_t launch_gemm2_tf32x3(int M, int N, int K1, const float* A1, int64_t lda1_m, int64_t lda1_k,
                                const float* B1, int64_t ldb1_k, int64_t ldb1_n, int K2, const float* A2,
                                int64_t lda2_m, int64_t lda2_k, const float* B2, int64_t ldb2_k, int64_t ldb2_n,
                                float* C, int64_t ldc, float beta, float* relu_out, int64_t ldr, float* ws,
                                int64_t ws_floats, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (K1 <= 0 || K2 <= 0) return cudaErrorInvalidValue;
  static const bool no_dual = getenv("HB_GEMM_NO_DUAL") != nullptr;
  if (C == nullptr && (no_dual || g_gemm_path != 0)) return cudaErrorNotSupported;
  if (!no_dual && g_gemm_path == 0) {
    const cudaError_t e = launch_gemm_ts_dual(M, N, K1, A1, lda1_m, lda1_k, B1, ldb1_k, ldb1_n, K2, A2, lda2_m,
                                              lda2_k, B2, ldb2_k, ldb2_n, C, ldc, beta, relu_out, ldr, ws, ws_floats,
                                              st);
    if (e != cudaErrorNotSupported || C == nullptr) return e;
  }
  cudaError_t e = launch_gemm_tf32x3(M, N, K1, A1, lda1_m, lda1_k, B1, ldb1_k, ldb1_n, C, ldc, beta, nullptr, 0, ws,
                                     ws_floats, st);
  if (e != cudaSuccess) return e;
  return launch_gemm_tf32x3(M, N, K2, A2, lda2_m, lda2_k, B2, ldb2_k, ldb2_n, C, ldc, 1.f, relu_out, ldr, ws,
                            ws_floats, st);
}

}  // namespace hb
