// K5-K7, CTA-pair variant: the tcgen05 3xTF32 GEMM of gemm_tma.cu on
// 256-row tiles computed by a cluster of two CTAs on two SMs
// (tcgen05.mma.cta_group::2, M = 256).  Each CTA stages its own 128 rows of
// A and HALF of the B tile (BN/2 columns); the pair's MMA reads both halves,
// so per SM the B bytes staged by TMA and read by the tensor core halve and
// a 3-stage ring fits next to the split (hi / lo) tiles.
//
// Roles per CTA as in gemm_tma.cu (TMA producer, MMA issuer, 4 converter
// warps, 4 epilogue warps); only CTA rank 0's MMA warp issues.  Cross-CTA
// synchronisation:
//   conv[s]   (rank 0)  8 arrivals: 4 local + 4 remote converter warps
//   empty[s]  (both)    tcgen05.commit multicast to both CTAs
//   tfull[a]  (both)    tcgen05.commit multicast to both CTAs
//   tempty[a] (rank 0)  8 arrivals: 4 local + 4 remote epilogue warps
// TMEM: tcgen05.alloc.cta_group::2, each CTA's accumulator holds its 128 rows.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdlib>
#include "common.cuh"

namespace hb {
namespace gt2 {

constexpr int BM = 128;                   // rows per CTA (256 per pair)
constexpr int BK = 32;
constexpr int kThreads = 320;
constexpr int kConv0 = 2, kEpi0 = 6;

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int BH_BYTES = (BN / 2) * BK * 4;     // this CTA's half of B
  static constexpr int STAGE = 2 * (A_BYTES + BH_BYTES);
  static constexpr int STAGES = BN == 256 ? 3 : 4;
  static constexpr int SMEM = STAGES * STAGE + 1024;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
};

struct Params {
  int M, N, K;
  int a_mn, b_mn;
  int bsplit;
  int mt2, nt, splits, kb_per_split, nkb;   // mt2: 256-row pair tiles
  float* C;
  int64_t ldc;
  float beta;
  float* relu_out;
  int64_t ldr;
  float* ws;
};

__device__ __forceinline__ uint32_t rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared::cluster address of `p` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

__device__ __forceinline__ void umma2_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// commit the issuing thread's MMAs to the barrier at `bar`'s offset in both CTAs
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

__device__ __forceinline__ void tile_coords(const Params& p, int t, int& mi, int& ni, int& si) {
  ni = t % p.nt;
  mi = (t / p.nt) % p.mt2;
  si = t / (p.nt * p.mt2);
}

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
gemm_tma2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
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
  const uint32_t rank = cluster_rank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int num_tiles = p.mt2 * p.nt * p.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 8);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(C_::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();                       // both CTAs' barriers initialised before any remote arrive
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    // ---------------- TMA producer (own A rows, own half of B) ----------------
    if (lane == 0) {
      int it = 0;
      for (int t = cid; t < num_tiles; t += ncl) {
        int mi, ni, si;
        tile_coords(p, t, mi, ni, si);
        const int kb0 = si * p.kb_per_split, kb1 = min(p.nkb, kb0 + p.kb_per_split);
        const int m0 = mi * 2 * BM + (int)rank * BM;
        const int nh0 = ni * BN + (int)rank * (BN / 2);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % S;
          mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          uint8_t* st = smem + s * C_::STAGE;
          uint8_t* a_hi = st;
          uint8_t* b_hi = st + 2 * C_::A_BYTES;
          mbar_expect_tx(&full[s], C_::A_BYTES + (p.bsplit ? 2 : 1) * C_::BH_BYTES);
          const int k0 = kb * BK;
          if (p.a_mn) {
#pragma unroll
            for (int j = 0; j < BM / 32; ++j) tma_2d(a_hi + j * 4096, &tmA, m0 + 32 * j, k0, &full[s]);
          } else {
            tma_2d(a_hi, &tmA, k0, m0, &full[s]);
          }
          if (p.bsplit) {
            tma_2d(b_hi, &tmB, k0, nh0, &full[s]);
            tma_2d(b_hi + C_::BH_BYTES, &tmBl, k0, nh0, &full[s]);
          } else if (p.b_mn) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_2d(b_hi + j * 4096, &tmB, nh0 + 32 * j, k0, &full[s]);
          } else {
            tma_2d(b_hi, &tmB, k0, nh0, &full[s]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (rank 0 only) ----------------
    if (rank == 0 && lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)p.a_mn << 15) |
                             ((uint32_t)p.b_mn << 16) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)((2 * BM) >> 4) << 24);
      const uint32_t a_step = p.a_mn ? 1024u : 32u, b_step = p.b_mn ? 1024u : 32u;
      const uint32_t a_lbo = p.a_mn ? 4096u : 16u, b_lbo = p.b_mn ? 4096u : 16u;
      const uint32_t a_sbo = p.a_mn ? 512u : 1024u, b_sbo = p.b_mn ? 512u : 1024u;
      const uint32_t a_lay = p.a_mn ? 1u : 2u, b_lay = p.b_mn ? 1u : 2u;
      int it = 0, tc = 0;
      for (int t = cid; t < num_tiles; t += ncl, ++tc) {
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
          const uint32_t b_hi = st + 2 * C_::A_BYTES, b_lo = b_hi + C_::BH_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t dah = sw_desc(a_hi + kk * a_step, a_lbo, a_sbo, a_lay);
            const uint64_t dal = sw_desc(a_lo + kk * a_step, a_lbo, a_sbo, a_lay);
            const uint64_t dbh = sw_desc(b_hi + kk * b_step, b_lbo, b_sbo, b_lay);
            const uint64_t dbl = sw_desc(b_lo + kk * b_step, b_lbo, b_sbo, b_lay);
            umma2_tf32(d_tmem, dal, dbh, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
            umma2_tf32(d_tmem, dah, dbl, idesc, 1u);
            umma2_tf32(d_tmem, dah, dbh, idesc, 1u);
          }
          umma2_commit_both(&empty[s]);
        }
        umma2_commit_both(&tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp < kEpi0) {
    // ---------------- split: raw fp32 -> tf32 hi / lo (own A rows, own B half) ----
    const int ct = threadIdx.x - kConv0 * 32;
    const uint32_t conv0 = rank == 0 ? 0u : mapa(&conv[0], 0);
    int it = 0;
    for (int t = cid; t < num_tiles; t += ncl) {
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
        uint4* b_lo = reinterpret_cast<uint4*>(st + 2 * C_::A_BYTES + C_::BH_BYTES);
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
        for (int i = ct; i < (p.bsplit ? 0 : C_::BH_BYTES / 16); i += 128) {
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
        if (lane == 0) {
          if (rank == 0) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&conv[s])) : "memory");
          } else {
            mbar_arrive_cluster(conv0 + (uint32_t)(s * sizeof(uint64_t)));
          }
        }
      }
    }
  } else {
    // ---------------- epilogue (own 128 rows) ----------------
    const int lg = warp & 3;
    const uint32_t tempty0 = rank == 0 ? 0u : mapa(&tempty[0], 0);
    int tc = 0;
    for (int t = cid; t < num_tiles; t += ncl, ++tc) {
      int mi, ni, si;
      tile_coords(p, t, mi, ni, si);
      const int acc = tc & 1;
      mbar_wait(&tfull[acc], (tc >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int row = mi * 2 * BM + (int)rank * BM + lg * 32 + lane;
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
                  const float4 t4 = *reinterpret_cast<const float4*>(crow + nb + e);
                  o[e] = t4.x; o[e + 1] = t4.y; o[e + 2] = t4.z; o[e + 3] = t4.w;
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
      if (lane == 0) {
        if (rank == 0) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[acc])) : "memory");
        } else {
          mbar_arrive_cluster(tempty0 + (uint32_t)(acc * sizeof(uint64_t)));
        }
      }
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();                       // the peer's MMAs into this CTA's TMEM are complete
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C_::TMEM_COLS));
  }
}

}  // namespace gt2

// Host side shared with gemm_tma.cu (tensor maps, B pre-split, split-K reduce).
bool gemm_make_map(CUtensorMap* m, const float* base, int64_t inner, int64_t outer, int64_t ld, int box_outer,
                   bool mn_major);
cudaError_t gemm_bsplit(const float* B, int64_t ldb_k, int64_t ldb_n, int K, int N, int Kp, float* hi, float* lo,
                        cudaStream_t st);
cudaError_t gemm_splitk_reduce(const float* ws, int splits, int M, int N, float* C, int64_t ldc, float beta,
                               float* relu_out, int64_t ldr, cudaStream_t st);

template <int BN>
static cudaError_t launch_pair_bn(int M, int N, int K, const float* A, int64_t lda_m, int64_t lda_k, const float* B,
                                  int64_t ldb_k, int64_t ldb_n, float* C, int64_t ldc, float beta, float* relu_out,
                                  int64_t ldr, float* ws, int64_t ws_floats, cudaStream_t st) {
  using C_ = gt2::Cfg<BN>;
  gt2::Params p{};
  p.M = M; p.N = N; p.K = K;
  p.a_mn = lda_k == 1 ? 0 : 1;
  p.b_mn = ldb_k == 1 ? 0 : 1;
  CUtensorMap ta, tb, tbl;
  bool ok = p.a_mn ? gemm_make_map(&ta, A, M, K, lda_k, 32, true) : gemm_make_map(&ta, A, K, M, lda_m, gt2::BM, false);
  if (!ok) return cudaErrorNotSupported;
  p.mt2 = (M + 2 * gt2::BM - 1) / (2 * gt2::BM);
  p.nt = (N + BN - 1) / BN;
  p.nkb = (K + gt2::BK - 1) / gt2::BK;
  const int pairs = num_sms() / 2;
  int splits = 1;
  const int tiles = p.mt2 * p.nt;
  if (ws != nullptr && tiles < pairs && p.nkb >= 8) {
    splits = pairs / tiles;
    if (splits > p.nkb / 4) splits = p.nkb / 4;
    const int64_t by_ws = ws_floats / ((int64_t)M * N);
    if (splits > by_ws) splits = (int)by_ws;
    if (splits < 1) splits = 1;
  }
  p.kb_per_split = (p.nkb + splits - 1) / splits;
  p.splits = (p.nkb + p.kb_per_split - 1) / p.kb_per_split;
  p.C = C; p.ldc = ldc; p.beta = beta; p.relu_out = p.splits > 1 ? nullptr : relu_out; p.ldr = ldr;
  p.ws = p.splits > 1 ? ws : nullptr;
  const int Kp = (K + 3) & ~3;
  static const bool no_bsplit = getenv("HB_GEMM_NO_BSPLIT") != nullptr;
  if (!no_bsplit && p.splits == 1 && ws != nullptr && tiles >= 2 * pairs && p.nkb >= 4 &&
      (int64_t)N * K <= (1 << 20) && 2 * (int64_t)N * Kp <= ws_floats) {
    float* hi = ws;
    float* lo = ws + (int64_t)N * Kp;
    cudaError_t e = gemm_bsplit(B, ldb_k, ldb_n, K, N, Kp, hi, lo, st);
    if (e != cudaSuccess) return e;
    if (!gemm_make_map(&tb, hi, K, N, Kp, BN / 2, false) || !gemm_make_map(&tbl, lo, K, N, Kp, BN / 2, false))
      return cudaErrorNotSupported;
    p.bsplit = 1;
    p.b_mn = 0;
  } else {
    ok = p.b_mn ? gemm_make_map(&tb, B, N, K, ldb_k, 32, true) : gemm_make_map(&tb, B, K, N, ldb_n, BN / 2, false);
    if (!ok) return cudaErrorNotSupported;
    tbl = tb;
  }
  const int total = tiles * p.splits;
  int grid = 2 * (total < pairs ? total : pairs);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gt2::gemm_tma2_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C_::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  gt2::gemm_tma2_kernel<BN><<<grid, gt2::kThreads, C_::SMEM, st>>>(ta, tb, tbl, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.splits > 1) e = gemm_splitk_reduce(ws, p.splits, M, N, C, ldc, beta, relu_out, ldr, st);
  return e;
}

// Returns cudaErrorNotSupported when the pair kernel does not apply (the
// caller then uses the single-CTA kernel).
cudaError_t launch_gemm_tma_pair(int M, int N, int K, const float* A, int64_t lda_m, int64_t lda_k, const float* B,
                                 int64_t ldb_k, int64_t ldb_n, float* C, int64_t ldc, float beta, float* relu_out,
                                 int64_t ldr, float* ws, int64_t ws_floats, cudaStream_t st) {
  if (N > 128 && N <= 256)
    return launch_pair_bn<256>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws, ws_floats,
                               st);
  return cudaErrorNotSupported;
}

}  // namespace hb
