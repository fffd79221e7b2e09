// K5-K7 main path: persistent, warp-specialised tcgen05 GEMM with TMA-fed
// operands and the 3xTF32 split done in shared memory.
//
//   C[m, n] = sum_k A(m, k) B(k, n)  (+ beta C, optional fused ReLU copy)
//
// Shapes in the trainer (trainer.py:294, 313, 318-321):
//   Z = P W      A K-major (rows x d_in, ld), B MN-major (W, N contiguous)
//   G = P^T m    A MN-major (P^T), B MN-major (m); K = rows -> split-K
//   T = m W^T    A K-major, B K-major (W^T)
// Every operand is a row-major fp32 matrix with a 16-byte-multiple row
// stride, so TMA (cp.async.bulk.tensor, SWIZZLE_128B) stages any of them;
// the UMMA descriptors carry the K-major / MN-major choice.
//
// Warp roles (320 threads, one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer (one lane): A and B raw fp32 tiles -> stage s
//   warp 1      TMEM allocator + MMA issuer (one lane): 3 tcgen05.mma kind::tf32
//               per K=8 step (hi*hi + hi*lo + lo*hi), accumulators in TMEM,
//               double-buffered across tiles
//   warps 2-5   split: raw -> (hi = rna_tf32(x), lo = rna_tf32(x - hi)) in place
//               (elementwise, so it is layout-agnostic under the swizzle)
//   warps 6-9   epilogue: tcgen05.ld -> registers -> global (C or split-K
//               partial), overlapped with the next tile's main loop
// Barriers per stage: full (TMA tx bytes), conv (4 converter warps), empty
// (tcgen05.commit); per accumulator: tfull (commit), tempty (4 epilogue warps).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdlib>
#include "common.cuh"

namespace hb {
namespace gt {

constexpr int BM = 128;
constexpr int BK = 32;                    // fp32 per 128-byte swizzle row
constexpr int kThreads = 320;
constexpr int kConv0 = 2, kEpi0 = 6;      // first converter / epilogue warp

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE = 2 * (A_BYTES + B_BYTES);
  static constexpr int STAGES = BN == 256 ? 2 : (BN == 128 ? 3 : 4);
  static constexpr int SMEM = STAGES * STAGE + 1024;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
};

struct Params {
  int M, N, K;
  int a_mn, b_mn;          // 1 = MN-major operand
  int bsplit;              // 1: B arrives pre-split (hi / lo, K-major) via tmB / tmBl
  int mt, nt, splits, kb_per_split, nkb;
  float* C;
  int64_t ldc;
  float beta;
  float* relu_out;
  int64_t ldr;
  float* ws;               // split-K partials [splits][M][N]
};

__device__ __forceinline__ uint32_t rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// Swizzled smem descriptor (sm_100 version 1).  layout 2 = SWIZZLE_128B
// (K-major operands), layout 1 = SWIZZLE_128B_BASE32B (MN-major tf32 operands:
// the only MN-major layout UMMA accepts for 32-bit types; TMA produces it with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).
__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Tile t -> (m tile, n tile, split); n fastest so neighbouring CTAs share A.
__device__ __forceinline__ void tile_coords(const Params& p, int t, int& mi, int& ni, int& si) {
  ni = t % p.nt;
  mi = (t / p.nt) % p.mt;
  si = t / (p.nt * p.mt);
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmBl, Params p) {
  using C_ = Cfg<BN>;
  constexpr int S = C_::STAGES;
  extern __shared__ uint8_t smem_raw[];
  // aligned by pointer arithmetic on the __shared__ array (an integer round
  // trip would hide the address space and turn every access generic)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[S], conv[S], empty[S], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_s;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_tiles = p.mt * p.nt * p.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(C_::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mi, ni, si;
        tile_coords(p, t, mi, ni, si);
        const int kb0 = si * p.kb_per_split, kb1 = min(p.nkb, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % S;
          mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          uint8_t* st = smem + s * C_::STAGE;
          uint8_t* a_hi = st;
          uint8_t* b_hi = st + 2 * C_::A_BYTES;
          mbar_expect_tx(&full[s], C_::A_BYTES + (p.bsplit ? 2 : 1) * C_::B_BYTES);
          const int k0 = kb * BK;
          if (p.a_mn) {
#pragma unroll
            for (int j = 0; j < BM / 32; ++j) tma_2d(a_hi + j * 4096, &tmA, mi * BM + 32 * j, k0, &full[s]);
          } else {
            tma_2d(a_hi, &tmA, k0, mi * BM, &full[s]);
          }
          if (p.bsplit) {
            tma_2d(b_hi, &tmB, k0, ni * BN, &full[s]);
            tma_2d(b_hi + C_::B_BYTES, &tmBl, k0, ni * BN, &full[s]);
          } else if (p.b_mn) {
#pragma unroll
            for (int j = 0; j < BN / 32; ++j) tma_2d(b_hi + j * 4096, &tmB, ni * BN + 32 * j, k0, &full[s]);
          } else {
            tma_2d(b_hi, &tmB, k0, ni * BN, &full[s]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      // kind::tf32, fp32 accumulate, M = 128, N = BN, majors from the operands
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)p.a_mn << 15) |
                             ((uint32_t)p.b_mn << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      // K=8 step inside a stage: K-major +32 B within the 128-B swizzled row
      // (SBO = 1024 B between 8-row groups); MN-major +1024 B = 8 K-rows of
      // 128 B (BASE32B atoms of 4 K-rows: SBO = 512 B; LBO = 4096 B between
      // the 32-element MN blocks, one TMA box each).
      const uint32_t a_step = p.a_mn ? 1024u : 32u, b_step = p.b_mn ? 1024u : 32u;
      const uint32_t a_lbo = p.a_mn ? 4096u : 16u, b_lbo = p.b_mn ? 4096u : 16u;
      const uint32_t a_sbo = p.a_mn ? 512u : 1024u, b_sbo = p.b_mn ? 512u : 1024u;
      const uint32_t a_lay = p.a_mn ? 1u : 2u, b_lay = p.b_mn ? 1u : 2u;
      int it = 0, tc = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++tc) {
        int mi, ni, si;
        tile_coords(p, t, mi, ni, si);
        const int kb0 = si * p.kb_per_split, kb1 = min(p.nkb, kb0 + p.kb_per_split);
        const int acc = tc & 1;
        mbar_wait(&tempty[acc], ((tc >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d_tmem = tmem + (uint32_t)(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % S;
          mbar_wait(&conv[s], (it / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t st = smem_u32(smem + s * C_::STAGE);
          const uint32_t a_hi = st, a_lo = st + C_::A_BYTES;
          const uint32_t b_hi = st + 2 * C_::A_BYTES, b_lo = b_hi + C_::B_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t dah = sw_desc(a_hi + kk * a_step, a_lbo, a_sbo, a_lay);
            const uint64_t dal = sw_desc(a_lo + kk * a_step, a_lbo, a_sbo, a_lay);
            const uint64_t dbh = sw_desc(b_hi + kk * b_step, b_lbo, b_sbo, b_lay);
            const uint64_t dbl = sw_desc(b_lo + kk * b_step, b_lbo, b_sbo, b_lay);
            umma_tf32(d_tmem, dal, dbh, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
            umma_tf32(d_tmem, dah, dbl, idesc, 1u);
            umma_tf32(d_tmem, dah, dbh, idesc, 1u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp < kEpi0) {
    // ---------------- split: raw fp32 -> tf32 hi / lo ----------------
    const int ct = threadIdx.x - kConv0 * 32;
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int mi, ni, si;
      tile_coords(p, t, mi, ni, si);
      const int kb0 = si * p.kb_per_split, kb1 = min(p.nkb, kb0 + p.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = it % S;
        mbar_wait(&full[s], (it / S) & 1);
        uint8_t* st = smem + s * C_::STAGE;
        uint4* a_hi = reinterpret_cast<uint4*>(st);
        uint4* a_lo = reinterpret_cast<uint4*>(st + C_::A_BYTES);
        uint4* b_hi = reinterpret_cast<uint4*>(st + 2 * C_::A_BYTES);
        uint4* b_lo = reinterpret_cast<uint4*>(st + 2 * C_::A_BYTES + C_::B_BYTES);
#pragma unroll 4
        for (int i = ct; i < C_::A_BYTES / 16; i += 128) {
          const uint4 v = a_hi[i];
          uint4 h, l;
          h.x = rna_tf32(__uint_as_float(v.x)); l.x = rna_tf32(__uint_as_float(v.x) - __uint_as_float(h.x));
          h.y = rna_tf32(__uint_as_float(v.y)); l.y = rna_tf32(__uint_as_float(v.y) - __uint_as_float(h.y));
          h.z = rna_tf32(__uint_as_float(v.z)); l.z = rna_tf32(__uint_as_float(v.z) - __uint_as_float(h.z));
          h.w = rna_tf32(__uint_as_float(v.w)); l.w = rna_tf32(__uint_as_float(v.w) - __uint_as_float(h.w));
          a_hi[i] = h;
          a_lo[i] = l;
        }
#pragma unroll 4
        for (int i = ct; i < (p.bsplit ? 0 : C_::B_BYTES / 16); i += 128) {
          const uint4 v = b_hi[i];
          uint4 h, l;
          h.x = rna_tf32(__uint_as_float(v.x)); l.x = rna_tf32(__uint_as_float(v.x) - __uint_as_float(h.x));
          h.y = rna_tf32(__uint_as_float(v.y)); l.y = rna_tf32(__uint_as_float(v.y) - __uint_as_float(h.y));
          h.z = rna_tf32(__uint_as_float(v.z)); l.z = rna_tf32(__uint_as_float(v.z) - __uint_as_float(h.z));
          h.w = rna_tf32(__uint_as_float(v.w)); l.w = rna_tf32(__uint_as_float(v.w) - __uint_as_float(h.w));
          b_hi[i] = h;
          b_lo[i] = l;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[s]);
      }
    }
  } else {
    // ---------------- epilogue ----------------
    const int lg = warp & 3;                // TMEM lane group this warp may access
    int tc = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++tc) {
      int mi, ni, si;
      tile_coords(p, t, mi, ni, si);
      const int acc = tc & 1;
      mbar_wait(&tfull[acc], (tc >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int row = mi * BM + lg * 32 + lane;
      const int n0 = ni * BN;
      const int ncols = min(BN, p.N - n0);
      const bool split = p.splits > 1;
      float* crow = split ? p.ws + ((int64_t)si * p.M + row) * p.N : p.C + (int64_t)row * p.ldc;
      for (int c0 = 0; c0 < ncols; c0 += 32) {
        uint32_t r[32];
        const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * BN + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
              "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
              "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
              "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr)
            : "memory");
        if (row < p.M) {
          const int nb = n0 + c0;
          const int nv = min(32, p.N - nb);
          if (split) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (e < nv) crow[nb + e] = __uint_as_float(r[e]);
          } else {
            // all loads of the old C values first (no store can alias them in
            // between), then the stores; float4 wherever the row allows it
            float* rrow = p.relu_out ? p.relu_out + (int64_t)row * p.ldr + nb : nullptr;
            const bool cvec = ((p.ldc & 3) == 0) && ((((uintptr_t)(crow + nb)) & 15) == 0);
            const bool rvec = rrow && ((p.ldr & 3) == 0) && ((((uintptr_t)rrow) & 15) == 0);
            float v[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]);
            if (p.beta != 0.f) {
              float o[32];
#pragma unroll
              for (int e = 0; e < 32; e += 4) {
                if (cvec && e + 3 < nv) {
                  const float4 t = *reinterpret_cast<const float4*>(crow + nb + e);
                  o[e] = t.x; o[e + 1] = t.y; o[e + 2] = t.z; o[e + 3] = t.w;
                } else {
#pragma unroll
                  for (int u = 0; u < 4; ++u) o[e + u] = e + u < nv ? crow[nb + e + u] : 0.f;
                }
              }
#pragma unroll
              for (int e = 0; e < 32; ++e) v[e] += p.beta * o[e];
            }
#pragma unroll
            for (int e = 0; e < 32; e += 4) {
              if (cvec && e + 3 < nv) {
                *reinterpret_cast<float4*>(crow + nb + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
              } else {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  if (e + u < nv) crow[nb + e + u] = v[e + u];
              }
            }
            if (rrow) {
#pragma unroll
              for (int e = 0; e < 32; ++e) v[e] = (v[e] > 0.f || v[e] != v[e]) ? v[e] : 0.f;
#pragma unroll
              for (int e = 0; e < 32; e += 4) {
                if (rvec && e + 3 < nv) {
                  *reinterpret_cast<float4*>(rrow + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
                } else {
#pragma unroll
                  for (int u = 0; u < 4; ++u)
                    if (e + u < nv) rrow[e + u] = v[e + u];
                }
              }
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C_::TMEM_COLS));
  }
}

// B pre-split for the GEMMs whose B is a weight (Z = P W, T = m W^T): B is
// small and shared by every tile, so it is split once into K-major hi / lo
// arrays ([N][Kp], zero-padded) instead of in every CTA's converter warps.
// hi/lo[n * Kp + koff + k] = tf32 split of B[k, n] for k < kcnt (zero for k >= K)
__global__ void bsplit_kernel(const float* __restrict__ B, int64_t ldb_k, int64_t ldb_n, int K, int N, int kcnt,
                              int Kp, int koff, float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t total = (int64_t)N * kcnt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(i / kcnt), k = (int)(i - (int64_t)n * kcnt);
    const float x = k < K ? B[(int64_t)k * ldb_k + (int64_t)n * ldb_n] : 0.f;
    const uint32_t h = rna_tf32(x);
    const int64_t o = (int64_t)n * Kp + koff + k;
    hi[o] = __uint_as_float(h);
    lo[o] = __uint_as_float(rna_tf32(x - __uint_as_float(h)));
  }
}

// Deterministic split-K reduction (fixed order) + beta + optional ReLU copy.
__global__ void splitk_reduce2_kernel(const float* __restrict__ ws, int splits, int M, int N, float* __restrict__ C,
                                      int64_t ldc, float beta, float* __restrict__ relu_out, int64_t ldr) {
  const int64_t total = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int z = 0; z < splits; ++z) acc += ws[(int64_t)z * total + i];
    const int64_t m = i / N, n = i - m * N;
    float* c = C + m * ldc + n;
    const float v = beta != 0.f ? acc + beta * *c : acc;
    *c = v;
    if (relu_out) relu_out[m * ldr + n] = (v > 0.f || v != v) ? v : 0.f;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// 2-D fp32 tensor map: inner dim `inner` (contiguous), outer dim `outer` with
// row stride `ld` floats; box 32 x box_outer; SWIZZLE_128B.
static bool make_map(CUtensorMap* m, const float* base, int64_t inner, int64_t outer, int64_t ld, int box_outer,
                     bool mn_major) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {32u, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1u, 1u};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE,
            mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Operand (rows=MN extent, K extent) with element (mn, k) at base + mn*s_mn + k*s_k.
// TMA-eligible iff 16-byte aligned base and one unit stride with the other a
// multiple of 4 floats.
static bool tma_ok(const float* base, int64_t s_mn, int64_t s_k) {
  if (((uintptr_t)base) & 15) return false;
  if (s_k == 1) return s_mn % 4 == 0 && s_mn > 0;
  if (s_mn == 1) return s_k % 4 == 0 && s_k > 0;
  return false;
}

template <int BN>
static cudaError_t launch_bn(int M, int N, int K, const float* A, int64_t lda_m, int64_t lda_k, const float* B,
                             int64_t ldb_k, int64_t ldb_n, float* C, int64_t ldc, float beta, float* relu_out,
                             int64_t ldr, float* ws, int64_t ws_floats, cudaStream_t st) {
  using C_ = Cfg<BN>;
  Params p{};
  p.M = M; p.N = N; p.K = K;
  p.a_mn = lda_k == 1 ? 0 : 1;
  p.b_mn = ldb_k == 1 ? 0 : 1;
  CUtensorMap ta, tb;
  bool ok = p.a_mn ? make_map(&ta, A, M, K, lda_k, 32, true) : make_map(&ta, A, K, M, lda_m, BM, false);
  ok = ok && (p.b_mn ? make_map(&tb, B, N, K, ldb_k, 32, true) : make_map(&tb, B, K, N, ldb_n, BN, false));
  if (!ok) return cudaErrorNotSupported;
  p.mt = (M + BM - 1) / BM;
  p.nt = (N + BN - 1) / BN;
  p.nkb = (K + BK - 1) / BK;
  const int sms = num_sms();
  int splits = 1;
  const int tiles = p.mt * p.nt;
  if (ws != nullptr && tiles < sms && p.nkb >= 8) {
    splits = sms / tiles;
    if (splits > p.nkb / 4) splits = p.nkb / 4;
    const int64_t by_ws = ws_floats / ((int64_t)M * N);
    if (splits > by_ws) splits = (int)by_ws;
    if (splits < 1) splits = 1;
  }
  p.kb_per_split = (p.nkb + splits - 1) / splits;
  p.splits = (p.nkb + p.kb_per_split - 1) / p.kb_per_split;
  // weight-sized B with many tiles: split it once into the workspace
  CUtensorMap tbl = tb;
  const int Kp = (K + 3) & ~3;
  static const bool no_bsplit = getenv("HB_GEMM_NO_BSPLIT") != nullptr;
  if (!no_bsplit && p.splits == 1 && ws != nullptr && tiles >= 2 * sms && p.nkb >= 4 && (int64_t)N * K <= (1 << 20) &&
      2 * (int64_t)N * Kp <= ws_floats) {
    float* hi = ws;
    float* lo = ws + (int64_t)N * Kp;
    int g = (int)(((int64_t)N * Kp + 255) / 256);
    if (g > sms * 4) g = sms * 4;
    bsplit_kernel<<<g, 256, 0, st>>>(B, ldb_k, ldb_n, K, N, Kp, Kp, 0, hi, lo);
    if (make_map(&tb, hi, K, N, Kp, BN, false) && make_map(&tbl, lo, K, N, Kp, BN, false)) {
      p.bsplit = 1;
      p.b_mn = 0;
    } else {
      ok = make_map(&tb, B, p.b_mn ? N : K, p.b_mn ? K : N, p.b_mn ? ldb_k : ldb_n, p.b_mn ? 32 : BN, p.b_mn);
      if (!ok) return cudaErrorNotSupported;
    }
  }
  p.C = C; p.ldc = ldc; p.beta = beta; p.relu_out = p.splits > 1 ? nullptr : relu_out; p.ldr = ldr;
  p.ws = p.splits > 1 ? ws : nullptr;
  const int total = tiles * p.splits;
  const int grid = total < sms ? total : sms;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tma_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  gemm_tma_kernel<BN><<<grid, kThreads, C_::SMEM, st>>>(ta, tb, tbl, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.splits > 1) {
    int g = (int)(((int64_t)M * N + 255) / 256);
    if (g > sms * 8) g = sms * 8;
    splitk_reduce2_kernel<<<g, 256, 0, st>>>(ws, p.splits, M, N, C, ldc, beta, relu_out, ldr);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace gt

// host helpers shared with the A-in-TMEM kernels (gemm_ts.cu)
bool gemm_make_map(CUtensorMap* m, const float* base, int64_t inner, int64_t outer, int64_t ld, int box_outer,
                   bool mn_major) {
  return gt::make_map(m, base, inner, outer, ld, box_outer, mn_major);
}
cudaError_t gemm_bsplit_range(const float* B, int64_t ldb_k, int64_t ldb_n, int K, int N, int kcnt, int Kp, int koff,
                              float* hi, float* lo, cudaStream_t st) {
  int g = (int)(((int64_t)N * kcnt + 255) / 256);
  if (g > num_sms() * 4) g = num_sms() * 4;
  if (g < 1) g = 1;
  gt::bsplit_kernel<<<g, 256, 0, st>>>(B, ldb_k, ldb_n, K, N, kcnt, Kp, koff, hi, lo);
  return cudaGetLastError();
}
cudaError_t gemm_bsplit(const float* B, int64_t ldb_k, int64_t ldb_n, int K, int N, int Kp, float* hi, float* lo,
                        cudaStream_t st) {
  return gemm_bsplit_range(B, ldb_k, ldb_n, K, N, Kp, Kp, 0, hi, lo, st);
}
bool gemm_tma_ok(const float* base, int64_t s_mn, int64_t s_k) { return gt::tma_ok(base, s_mn, s_k); }
cudaError_t gemm_splitk_reduce(const float* ws, int splits, int M, int N, float* C, int64_t ldc, float beta,
                               float* relu_out, int64_t ldr, cudaStream_t st) {
  int g = (int)(((int64_t)M * N + 255) / 256);
  if (g > num_sms() * 8) g = num_sms() * 8;
  gt::splitk_reduce2_kernel<<<g, 256, 0, st>>>(ws, splits, M, N, C, ldc, beta, relu_out, ldr);
  return cudaGetLastError();
}
extern int g_gemm_ts;
extern int g_gemm_path;
cudaError_t launch_gemm_ts(int, int, int, const float*, int64_t, int64_t, const float*, int64_t, int64_t, float*,
                           int64_t, float, float*, int64_t, float*, int64_t, cudaStream_t);
cudaError_t launch_gemm_dw(int, int, int, const float*, int64_t, int64_t, const float*, int64_t, int64_t, float*,
                           int64_t, float, float*, int64_t, float*, int64_t, cudaStream_t);

// Returns cudaErrorNotSupported when an operand is not TMA-describable (the
// caller then uses the SIMT-staged kernel).
cudaError_t launch_gemm_tma(int M, int N, int K, const float* A, int64_t lda_m, int64_t lda_k, const float* B,
                            int64_t ldb_k, int64_t ldb_n, float* C, int64_t ldc, float beta, float* relu_out,
                            int64_t ldr, float* ws, int64_t ws_floats, cudaStream_t st) {
  if (!gt::tma_ok(A, lda_m, lda_k) || !gt::tma_ok(B, ldb_n, ldb_k)) return cudaErrorNotSupported;
  // A-in-TMEM kernel: default for tall GEMMs (many 128-row tiles, no split-K);
  // the long-K weight gradients (split-K) stay on the all-smem kernel, which
  // measured faster there
  static const int ts_env = getenv("HB_GEMM_TS") ? atoi(getenv("HB_GEMM_TS")) : -1;
  const bool tall = (int64_t)((M + 127) / 128) * ((N + 127) / 128) >= num_sms();
  const bool use_ts = ts_env >= 0 ? ts_env == 1 : (g_gemm_ts || (g_gemm_path == 0 && tall));
  if (use_ts) {
    const cudaError_t e = launch_gemm_ts(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws,
                                         ws_floats, st);
    if (e != cudaErrorNotSupported) return e;
  }
  // long-K weight gradients (few output tiles, split-K): A-in-TMEM kernel with
  // decoupled A / B rings
  static const int dw_env = getenv("HB_GEMM_DW") ? atoi(getenv("HB_GEMM_DW")) : 1;
  const int tiles128 = ((M + 127) / 128) * ((N + 127) / 128);
  if (dw_env && g_gemm_path == 0 && !g_gemm_ts && ws != nullptr && tiles128 < num_sms() &&
      (K + 31) / 32 >= 8) {
    const cudaError_t e = launch_gemm_dw(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws,
                                         ws_floats, st);
    if (e != cudaErrorNotSupported) return e;
  }
  static const int max_bn = getenv("HB_GEMM_BN") ? atoi(getenv("HB_GEMM_BN")) : 256;
  if (N <= 64 || max_bn == 64)
    return gt::launch_bn<64>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws, ws_floats, st);
  if (N <= 128 || max_bn == 128)
    return gt::launch_bn<128>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws, ws_floats, st);
  return gt::launch_bn<256>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws, ws_floats, st);
}

}  // namespace hb
