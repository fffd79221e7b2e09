// K5-K7, A-from-TMEM variant of the tcgen05 3xTF32 GEMM (gemm_tma.cu).
//
// The converter warps split A into tf32 hi / lo in REGISTERS and store both
// halves straight into tensor memory (tcgen05.st); the MMAs then take A from
// TMEM (tcgen05.mma ... [d], [a_tmem], b_desc) and only B from shared memory.
// Compared with the all-smem kernel this removes the A hi/lo tiles from shared
// memory (32 KB per stage) and their smem write + tensor-core read traffic, so
// a BN=128 tile fits a 4-stage ring (48 KB per stage: raw A 16 KB + B hi/lo),
// and the stage ring hides the A load latency behind more MMAs in flight.
//
// TMEM columns (512): accumulators 2 x BN (double buffered across tiles), then
// S stages x 64 columns of A (32 hi + 32 lo; M = 128 rows = lanes, one tf32 per
// column).  Converter warp w owns TMEM lanes 32 (w % 4) .. +31 = its 32 rows of
// the A tile: K-major raw rows are read back from the SW128 TMA layout (8
// swizzled 16-byte chunks), MN-major ones from the SW128_BASE32B layout
// (column reads), which also transposes them into the K-major order TMEM A
// requires.
//
// The epilogue releases the accumulator after its last tcgen05.ld and writes
// C (and/or the ReLU copy) through swizzled smem chunks and TMA bulk stores.
// A dual GEMM C = A1 B1 + A2 B2 runs both K ranges through the same ring
// (tmA2 / tmB2 for k blocks >= nkb1).  gemm_dw_kernel (below) is the
// split-K weight-gradient variant with decoupled A / B rings.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdlib>
#include "common.cuh"

namespace hb {
namespace gts {

constexpr int BM = 128;
constexpr int BK = 32;
// warps: 0 TMA producer, 1 MMA issuer, 2-9 two groups of 4 converter warps,
// 10-13 epilogue.  The weight-gradient kernel runs both converter groups (group
// g takes the k blocks with it % 2 == g, so two blocks are split into TMEM at
// once); the tall kernel measured no faster that way and leaves group 1 idle.
constexpr int kThreads = 448;
constexpr int kConv0 = 2, kEpi0 = 10;

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;            // raw fp32 A tile
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE = A_BYTES + 2 * B_BYTES;     // raw A | B hi | B lo
  static constexpr int STAGES = BN == 128 ? 4 : 6;
  static constexpr int EPI_BYTES = 4 * 2 * 4096;          // 4 epilogue warps x 2 staging chunks (32 rows x 128 B)
  static constexpr int SMEM = STAGES * STAGE + EPI_BYTES + 1024;
  static constexpr uint32_t ACC_COLS = 2 * BN;
  static constexpr uint32_t TMEM_COLS = 512;
  static_assert(ACC_COLS + STAGES * 64 <= TMEM_COLS, "TMEM budget");
};

struct Params {
  int M, N, K;
  int a_mn, b_mn;
  int bsplit;
  int mt, nt, splits, kb_per_split, nkb;
  int nkb1;          // K blocks read from A1/B1; blocks nkb1.. come from A2/B2 (dual GEMM)
  int tma_store;     // epilogue writes C (and the ReLU copy) through TMA bulk stores
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

__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// One warp's 32 rows x 32 fp32 chunk -> SW128 staging (row = lane, 16-byte
// chunk c at c ^ (row & 7): conflict-free) -> TMA bulk store at (col, row0).
// The staging buffer is reused two stores later, so wait for <= 1 pending read.
__device__ __forceinline__ void stage_and_store(uint8_t* buf, const float (&v)[32], const CUtensorMap* map, int col,
                                                int row0, int lane) {
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
  __syncwarp();
  uint4* row = reinterpret_cast<uint4*>(buf + lane * 128);
#pragma unroll
  for (int c = 0; c < 8; ++c)
    row[c ^ (lane & 7)] = make_uint4(__float_as_uint(v[4 * c]), __float_as_uint(v[4 * c + 1]),
                                     __float_as_uint(v[4 * c + 2]), __float_as_uint(v[4 * c + 3]));
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) tma_store_2d(map, buf, col, row0);
}

__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

// D[tmem] (+)= A[tmem] * B[smem]
__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

#define HB_R32(a) a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], a[9], a[10], a[11], a[12], a[13], a[14], \
                  a[15], a[16], a[17], a[18], a[19], a[20], a[21], a[22], a[23], a[24], a[25], a[26], a[27], a[28], \
                  a[29], a[30], a[31]

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tile_coords(const Params& p, int t, int& mi, int& ni, int& si) {
  ni = t % p.nt;
  mi = (t / p.nt) % p.mt;
  si = t / (p.nt * p.mt);
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
gemm_ts_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmBl, const __grid_constant__ CUtensorMap tmA2,
               const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmC,
               const __grid_constant__ CUtensorMap tmR, Params p) {
  using C_ = Cfg<BN>;
  constexpr int S = C_::STAGES;
  extern __shared__ uint8_t smem_raw[];
  // aligned by pointer arithmetic on the __shared__ array (an integer round
  // trip would hide the address space and turn every access generic)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[S], conv[S], empty[S], tfull[2], tempty[2], cbar[4];
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
    for (int a = 0; a < 4; ++a) mbar_init(&cbar[a], 1);     // epilogue warps' C-chunk loads
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
    // ---------------- TMA producer: raw A + B (pre-split hi/lo or raw) ----------------
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
          uint8_t* a_raw = st;
          uint8_t* b_hi = st + C_::A_BYTES;
          mbar_expect_tx(&full[s], C_::A_BYTES + (p.bsplit ? 2 : 1) * C_::B_BYTES);
          const bool second = kb >= p.nkb1;               // dual GEMM: A2/B2 blocks follow A1/B1
          const CUtensorMap* ma = second ? &tmA2 : &tmA;
          const CUtensorMap* mb = second ? &tmB2 : &tmB;
          const int k0 = (second ? kb - p.nkb1 : kb) * BK;
          if (p.a_mn) {
#pragma unroll
            for (int j = 0; j < BM / 32; ++j) tma_2d(a_raw + j * 4096, ma, mi * BM + 32 * j, k0, &full[s]);
          } else {
            tma_2d(a_raw, ma, k0, mi * BM, &full[s]);
          }
          if (p.bsplit) {
            // pre-split workspace: A1 blocks at K kb*BK, A2 blocks right after nkb1*BK
            tma_2d(b_hi, &tmB, kb * BK, ni * BN, &full[s]);
            tma_2d(b_hi + C_::B_BYTES, &tmBl, kb * BK, ni * BN, &full[s]);
          } else if (p.b_mn) {
#pragma unroll
            for (int j = 0; j < BN / 32; ++j) tma_2d(b_hi + j * 4096, mb, ni * BN + 32 * j, k0, &full[s]);
          } else {
            tma_2d(b_hi, mb, k0, ni * BN, &full[s]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      // kind::tf32, fp32 accumulate, A from TMEM (K-major), B major from the operand
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)p.b_mn << 16) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      const uint32_t b_step = p.b_mn ? 1024u : 32u, b_lbo = p.b_mn ? 4096u : 16u;
      const uint32_t b_sbo = p.b_mn ? 512u : 1024u, b_lay = p.b_mn ? 1u : 2u;
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
          const uint32_t a_hi_t = tmem + C_::ACC_COLS + (uint32_t)(s * 64);
          const uint32_t a_lo_t = a_hi_t + 32;
          const uint32_t b_hi = smem_u32(smem + s * C_::STAGE + C_::A_BYTES), b_lo = b_hi + C_::B_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t dbh = sw_desc(b_hi + kk * b_step, b_lbo, b_sbo, b_lay);
            const uint64_t dbl = sw_desc(b_lo + kk * b_step, b_lbo, b_sbo, b_lay);
            umma_ts(d_tmem, a_lo_t + 8 * kk, dbh, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
            umma_ts(d_tmem, a_hi_t + 8 * kk, dbl, idesc, 1u);
            umma_ts(d_tmem, a_hi_t + 8 * kk, dbh, idesc, 1u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp < kEpi0) {
    // ---------------- split A into TMEM (and B in smem when raw) ----------------
    const int lg = warp & 3;                        // TMEM lanes 32*lg .. +31 = tile rows
    const int r = lg * 32 + lane;                   // this thread's A row within the tile
    const int ct = (threadIdx.x - kConv0 * 32) & 127;
    // the tall kernel measured no faster with two converter groups (the
    // weight-gradient kernel below is): group 1 idles here
    const int cg = (warp - kConv0) >> 2;
    int it = 0;
    for (int t = (cg == 0 ? blockIdx.x : num_tiles); t < num_tiles; t += gridDim.x) {
      int mi, ni, si;
      tile_coords(p, t, mi, ni, si);
      const int kb0 = si * p.kb_per_split, kb1 = min(p.nkb, kb0 + p.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = it % S;
        mbar_wait(&full[s], (it / S) & 1);
        const uint8_t* st = smem + s * C_::STAGE;
        float x[32];
        if (!p.a_mn) {
          // SW128 K-major: row r = 128 B, 16-byte chunk c stored at chunk c ^ (r & 7)
          const uint4* row = reinterpret_cast<const uint4*>(st + r * 128);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v = row[c ^ (r & 7)];
            x[4 * c] = __uint_as_float(v.x); x[4 * c + 1] = __uint_as_float(v.y);
            x[4 * c + 2] = __uint_as_float(v.z); x[4 * c + 3] = __uint_as_float(v.w);
          }
        } else {
          // SW128_BASE32B MN-major: box r / 32, K-row k = 128 B, 32-byte atoms
          // swizzled by Swizzle<2,5,2>: o ^ (((o >> 7) & 3) << 5)
          const uint8_t* box = st + (r >> 5) * 4096;
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const uint32_t o = (uint32_t)(k * 128 + (r & 31) * 4);
            x[k] = *reinterpret_cast<const float*>(box + (o ^ (((o >> 7) & 3u) << 5)));
          }
        }
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          hi[k] = rna_tf32(x[k]);
          lo[k] = rna_tf32(x[k] - __uint_as_float(hi[k]));
        }
        const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + C_::ACC_COLS + (uint32_t)(s * 64);
        tmem_st32(taddr, hi);
        tmem_st32(taddr + 32, lo);
        if (!p.bsplit) {
          uint4* b_hi = reinterpret_cast<uint4*>(smem + s * C_::STAGE + C_::A_BYTES);
          uint4* b_lo = reinterpret_cast<uint4*>(smem + s * C_::STAGE + C_::A_BYTES + C_::B_BYTES);
#pragma unroll 4
          for (int i = ct; i < C_::B_BYTES / 16; i += 128) {
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
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive_local(&conv[s]);
      }
    }
  } else {
    // ---------------- epilogue ----------------
    // TMEM -> registers (tcgen05.ld, 32 columns per step); the accumulator is
    // released to the MMA warp right after the tile's last load.  With
    // tma_store the chunk goes through a swizzled smem buffer and a TMA bulk
    // store (coalesced full-line writes, clipped at M / N by the tensor map);
    // otherwise (beta != 0, split-K workspace, unaligned C) per-row stores.
    const int lg = warp & 3;
    uint8_t* stg = smem + S * C_::STAGE + (warp - kEpi0) * (2 * 4096);
    int sb = 0;
    int tc = 0;
    uint32_t cph = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++tc) {
      int mi, ni, si;
      tile_coords(p, t, mi, ni, si);
      const int acc = tc & 1;
      mbar_wait(&tfull[acc], (tc >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int row0 = mi * BM + lg * 32;
      const int row = row0 + lane;
      const int n0 = ni * BN;
      const int ncols = min(BN, p.N - n0);
      const bool split = p.splits > 1;
      float* crow = split ? p.ws + ((int64_t)si * p.M + row) * p.N : p.C + (int64_t)row * p.ldc;
      for (int c0 = 0; c0 < ncols; c0 += 32) {
        uint32_t rr[32];
        const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * BN + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(rr[0]), "=r"(rr[1]), "=r"(rr[2]), "=r"(rr[3]), "=r"(rr[4]), "=r"(rr[5]), "=r"(rr[6]),
              "=r"(rr[7]), "=r"(rr[8]), "=r"(rr[9]), "=r"(rr[10]), "=r"(rr[11]), "=r"(rr[12]), "=r"(rr[13]),
              "=r"(rr[14]), "=r"(rr[15]), "=r"(rr[16]), "=r"(rr[17]), "=r"(rr[18]), "=r"(rr[19]), "=r"(rr[20]),
              "=r"(rr[21]), "=r"(rr[22]), "=r"(rr[23]), "=r"(rr[24]), "=r"(rr[25]), "=r"(rr[26]), "=r"(rr[27]),
              "=r"(rr[28]), "=r"(rr[29]), "=r"(rr[30]), "=r"(rr[31])
            : "r"(taddr)
            : "memory");
        if (c0 + 32 >= ncols) {
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mbar_arrive_local(&tempty[acc]);
        }
        float v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(rr[e]);
        if (p.tma_store) {
          if (p.beta != 0.f) {
            // accumulate: the C chunk arrives by TMA in the staging buffer's
            // swizzled layout (coalesced, rows beyond M zero-filled), is added
            // in registers, and the buffer is then reused for the store
            uint8_t* lb = stg + sb * 4096;
            if (lane == 0) {
              asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              mbar_expect_tx(&cbar[warp - kEpi0], 4096);
              tma_2d(lb, &tmC, n0 + c0, row0, &cbar[warp - kEpi0]);
            }
            mbar_wait(&cbar[warp - kEpi0], cph);
            cph ^= 1u;
            const uint4* lr = reinterpret_cast<const uint4*>(lb + lane * 128);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const uint4 q = lr[c ^ (lane & 7)];
              v[4 * c] += p.beta * __uint_as_float(q.x);
              v[4 * c + 1] += p.beta * __uint_as_float(q.y);
              v[4 * c + 2] += p.beta * __uint_as_float(q.z);
              v[4 * c + 3] += p.beta * __uint_as_float(q.w);
            }
            __syncwarp();
          }
          if (p.C) {
            stage_and_store(stg + sb * 4096, v, &tmC, n0 + c0, row0, lane);
            sb ^= 1;
          }
          if (p.relu_out) {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = (v[e] > 0.f || v[e] != v[e]) ? v[e] : 0.f;
            stage_and_store(stg + sb * 4096, v, &tmR, n0 + c0, row0, lane);
            sb ^= 1;
          }
          continue;
        }
        if (row < p.M) {
          const int nb = n0 + c0;
          const int nv = min(32, p.N - nb);
          if (split) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (e < nv) crow[nb + e] = v[e];
          } else {
            float* rrow = p.relu_out ? p.relu_out + (int64_t)row * p.ldr + nb : nullptr;
            const bool cvec = ((p.ldc & 3) == 0) && ((((uintptr_t)(crow + nb)) & 15) == 0);
            const bool rvec = rrow && ((p.ldr & 3) == 0) && ((((uintptr_t)rrow) & 15) == 0);
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
    }
    if (p.tma_store && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }

  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C_::TMEM_COLS));
  }
}


// ---------------------------------------------------------------------------
// Weight-gradient variant (G = P^T m: small M x N, K = rows, split-K): A in
// TMEM as above, but the raw A tiles have their own ring, released by the
// converter warps as soon as they hold the rows in registers, while B (raw
// fp32, split in place into hi | lo) sits in a separate ring released by the
// MMA commit.  Each split owns one output tile, so the accumulator is single
// (BN columns) and the freed TMEM holds CB A-slots; BN = 256 keeps B re-reads
// low.  The all-smem kernel keeps raw A/B and their hi/lo in one 2-stage ring
// and measured ~48 % tensor-pipe activity on these shapes (latency-bound).
template <int BN>
struct DwCfg {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int CB = BN == 256 ? 3 : 4;                 // B (+ TMEM A slot) stages
  static constexpr int RA = BN == 256 ? 2 : 4;                     // raw A stages
  static constexpr int SMEM = CB * 2 * B_BYTES + RA * A_BYTES + 1024;
  static constexpr uint32_t ACC = BN;
  static_assert(ACC + CB * 64 <= 512, "TMEM budget");
  static_assert(SMEM <= 227 * 1024, "smem budget");
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
gemm_dw_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, Params p) {
  using C_ = DwCfg<BN>;
  constexpr int CB = C_::CB, RA = C_::RA;
  extern __shared__ uint8_t smem_raw[];
  // aligned by pointer arithmetic on the __shared__ array (an integer round
  // trip would hide the address space and turn every access generic)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* bring = smem;                                   // CB x (B hi | B lo)
  uint8_t* aring = smem + CB * 2 * C_::B_BYTES;            // RA x raw A
  __shared__ __align__(8) uint64_t afull[RA], aempty[RA], bfull[CB], conv[CB], bempty[CB], tfull, tempty;
  __shared__ uint32_t tmem_base_s;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_tiles = p.mt * p.nt * p.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < RA; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 4);
    }
    for (int s = 0; s < CB; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&bempty[s], 1);
    }
    mbar_init(&tfull, 1);
    mbar_init(&tempty, 4);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(512));
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
          const int ra = it % RA, sb = it % CB;
          const int k0 = kb * BK;
          mbar_wait(&aempty[ra], ((it / RA) & 1) ^ 1);
          uint8_t* a_raw = aring + ra * C_::A_BYTES;
          mbar_expect_tx(&afull[ra], C_::A_BYTES);
          if (p.a_mn) {
#pragma unroll
            for (int j = 0; j < BM / 32; ++j) tma_2d(a_raw + j * 4096, &tmA, mi * BM + 32 * j, k0, &afull[ra]);
          } else {
            tma_2d(a_raw, &tmA, k0, mi * BM, &afull[ra]);
          }
          mbar_wait(&bempty[sb], ((it / CB) & 1) ^ 1);
          uint8_t* b_hi = bring + sb * 2 * C_::B_BYTES;
          mbar_expect_tx(&bfull[sb], C_::B_BYTES);
          if (p.b_mn) {
#pragma unroll
            for (int j = 0; j < BN / 32; ++j) tma_2d(b_hi + j * 4096, &tmB, ni * BN + 32 * j, k0, &bfull[sb]);
          } else {
            tma_2d(b_hi, &tmB, k0, ni * BN, &bfull[sb]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)p.b_mn << 16) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      const uint32_t b_step = p.b_mn ? 1024u : 32u, b_lbo = p.b_mn ? 4096u : 16u;
      const uint32_t b_sbo = p.b_mn ? 512u : 1024u, b_lay = p.b_mn ? 1u : 2u;
      int it = 0, tc = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++tc) {
        int mi, ni, si;
        tile_coords(p, t, mi, ni, si);
        const int kb0 = si * p.kb_per_split, kb1 = min(p.nkb, kb0 + p.kb_per_split);
        mbar_wait(&tempty, (tc & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int sb = it % CB;
          mbar_wait(&conv[sb], (it / CB) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t a_hi_t = tmem + C_::ACC + (uint32_t)(sb * 64);
          const uint32_t a_lo_t = a_hi_t + 32;
          const uint32_t b_hi = smem_u32(bring + sb * 2 * C_::B_BYTES), b_lo = b_hi + C_::B_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t dbh = sw_desc(b_hi + kk * b_step, b_lbo, b_sbo, b_lay);
            const uint64_t dbl = sw_desc(b_lo + kk * b_step, b_lbo, b_sbo, b_lay);
            umma_ts(tmem, a_lo_t + 8 * kk, dbh, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
            umma_ts(tmem, a_hi_t + 8 * kk, dbl, idesc, 1u);
            umma_ts(tmem, a_hi_t + 8 * kk, dbh, idesc, 1u);
          }
          umma_commit(&bempty[sb]);
        }
        umma_commit(&tfull);
      }
    }
    __syncwarp();
  } else if (warp < kEpi0) {
    // ---------------- converters: A -> TMEM hi/lo, B split in place ----------------
    const int lg = warp & 3;
    const int r = lg * 32 + lane;
    const int ct = (threadIdx.x - kConv0 * 32) & 127;
    // two converter groups alternate k blocks when both rings are even (each
    // barrier then always has the same group of waiters); otherwise group 1 idles
    constexpr bool kTwo = (CB % 2 == 0) && (RA % 2 == 0);
    const int cg = (warp - kConv0) >> 2;
    if (!kTwo && cg == 1) {
      // nothing to do
    } else {
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int mi, ni, si;
      tile_coords(p, t, mi, ni, si);
      const int kb0 = si * p.kb_per_split, kb1 = min(p.nkb, kb0 + p.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        if (kTwo && (it & 1) != cg) continue;
        const int ra = it % RA, sb = it % CB;
        mbar_wait(&afull[ra], (it / RA) & 1);
        const uint8_t* st = aring + ra * C_::A_BYTES;
        float x[32];
        if (!p.a_mn) {
          const uint4* row = reinterpret_cast<const uint4*>(st + r * 128);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 v = row[c ^ (r & 7)];
            x[4 * c] = __uint_as_float(v.x); x[4 * c + 1] = __uint_as_float(v.y);
            x[4 * c + 2] = __uint_as_float(v.z); x[4 * c + 3] = __uint_as_float(v.w);
          }
        } else {
          const uint8_t* box = st + (r >> 5) * 4096;
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const uint32_t o = (uint32_t)(k * 128 + (r & 31) * 4);
            x[k] = *reinterpret_cast<const float*>(box + (o ^ (((o >> 7) & 3u) << 5)));
          }
        }
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          hi[k] = rna_tf32(x[k]);
          lo[k] = rna_tf32(x[k] - __uint_as_float(hi[k]));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_local(&aempty[ra]);      // raw A consumed: the producer may refill it
        mbar_wait(&bfull[sb], (it / CB) & 1);                // also orders the TMEM slot's previous MMAs
        const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + C_::ACC + (uint32_t)(sb * 64);
        tmem_st32(taddr, hi);
        tmem_st32(taddr + 32, lo);
        uint4* b_hi = reinterpret_cast<uint4*>(bring + sb * 2 * C_::B_BYTES);
        uint4* b_lo = reinterpret_cast<uint4*>(bring + sb * 2 * C_::B_BYTES + C_::B_BYTES);
#pragma unroll 4
        for (int i = ct; i < C_::B_BYTES / 16; i += 128) {
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
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive_local(&conv[sb]);
      }
    }
    }
  } else {
    // ---------------- epilogue: split-K partial (or C with beta / ReLU) ----------------
    const int lg = warp & 3;
    int tc = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++tc) {
      int mi, ni, si;
      tile_coords(p, t, mi, ni, si);
      mbar_wait(&tfull, tc & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int row = mi * BM + lg * 32 + lane;
      const int n0 = ni * BN;
      const int ncols = min(BN, p.N - n0);
      const bool split = p.splits > 1;
      float* crow = split ? p.ws + ((int64_t)si * p.M + row) * p.N : p.C + (int64_t)row * p.ldc;
      for (int c0 = 0; c0 < ncols; c0 += 32) {
        uint32_t rr[32];
        const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(rr[0]), "=r"(rr[1]), "=r"(rr[2]), "=r"(rr[3]), "=r"(rr[4]), "=r"(rr[5]), "=r"(rr[6]),
              "=r"(rr[7]), "=r"(rr[8]), "=r"(rr[9]), "=r"(rr[10]), "=r"(rr[11]), "=r"(rr[12]), "=r"(rr[13]),
              "=r"(rr[14]), "=r"(rr[15]), "=r"(rr[16]), "=r"(rr[17]), "=r"(rr[18]), "=r"(rr[19]), "=r"(rr[20]),
              "=r"(rr[21]), "=r"(rr[22]), "=r"(rr[23]), "=r"(rr[24]), "=r"(rr[25]), "=r"(rr[26]), "=r"(rr[27]),
              "=r"(rr[28]), "=r"(rr[29]), "=r"(rr[30]), "=r"(rr[31])
            : "r"(taddr)
            : "memory");
        if (c0 + 32 >= ncols) {
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mbar_arrive_local(&tempty);
        }
        if (row >= p.M) continue;
        const int nb = n0 + c0;
        const int nv = min(32, p.N - nb);
        float v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(rr[e]);
        if (split) {
          const bool vec = ((p.N & 3) == 0);
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            if (vec && e + 3 < nv) {
              *reinterpret_cast<float4*>(crow + nb + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (e + u < nv) crow[nb + e + u] = v[e + u];
            }
          }
          continue;
        }
        float* rrow = p.relu_out ? p.relu_out + (int64_t)row * p.ldr + nb : nullptr;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          if (e < nv) {
            float o = v[e];
            if (p.beta != 0.f) o += p.beta * crow[nb + e];
            crow[nb + e] = o;
            if (rrow) rrow[e] = (o > 0.f || o != o) ? o : 0.f;
          }
        }
      }
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace gts

bool gemm_make_map(CUtensorMap* m, const float* base, int64_t inner, int64_t outer, int64_t ld, int box_outer,
                   bool mn_major);
bool gemm_tma_ok(const float* base, int64_t s_mn, int64_t s_k);
cudaError_t gemm_bsplit_range(const float* B, int64_t ldb_k, int64_t ldb_n, int K, int N, int kcnt, int Kp, int koff,
                              float* hi, float* lo, cudaStream_t st);
cudaError_t gemm_splitk_reduce(const float* ws, int splits, int M, int N, float* C, int64_t ldc, float beta,
                               float* relu_out, int64_t ldr, cudaStream_t st);

// C = A1 B1 (+ A2 B2) (+ beta C), optional ReLU copy.  K2 == 0: single GEMM.
// A operands are (M x K) with element (m, k) at A + m*lda_m + k*lda_k, B
// operands (K x N) at B + k*ldb_k + n*ldb_n; the two A (and the two raw B)
// operands must share their major order.
template <int BN>
static cudaError_t launch_ts_bn(int M, int N, int K1, const float* A1, int64_t lda1_m, int64_t lda1_k,
                                const float* B1, int64_t ldb1_k, int64_t ldb1_n, int K2, const float* A2,
                                int64_t lda2_m, int64_t lda2_k, const float* B2, int64_t ldb2_k, int64_t ldb2_n,
                                float* C, int64_t ldc, float beta, float* relu_out, int64_t ldr, float* ws,
                                int64_t ws_floats, cudaStream_t st) {
  using C_ = gts::Cfg<BN>;
  const bool dual = K2 > 0;
  gts::Params p{};
  p.M = M; p.N = N; p.K = K1 + K2;
  p.a_mn = lda1_k == 1 ? 0 : 1;
  p.b_mn = ldb1_k == 1 ? 0 : 1;
  if (dual && ((lda2_k == 1 ? 0 : 1) != p.a_mn)) return cudaErrorNotSupported;
  CUtensorMap ta, tb, tbl, ta2, tb2, tc, tr;
  bool ok = p.a_mn ? gemm_make_map(&ta, A1, M, K1, lda1_k, 32, true) : gemm_make_map(&ta, A1, K1, M, lda1_m, gts::BM, false);
  if (dual)
    ok = ok && (p.a_mn ? gemm_make_map(&ta2, A2, M, K2, lda2_k, 32, true)
                       : gemm_make_map(&ta2, A2, K2, M, lda2_m, gts::BM, false));
  else
    ta2 = ta;
  if (!ok) return cudaErrorNotSupported;
  p.mt = (M + gts::BM - 1) / gts::BM;
  p.nt = (N + BN - 1) / BN;
  p.nkb1 = (K1 + gts::BK - 1) / gts::BK;
  p.nkb = p.nkb1 + (K2 + gts::BK - 1) / gts::BK;
  const int sms = num_sms();
  int splits = 1;
  const int tiles = p.mt * p.nt;
  // split-K needs C for the reduction: a ReLU-only store (C == nullptr) keeps
  // one split
  if (!dual && C != nullptr && ws != nullptr && tiles < sms && p.nkb >= 8) {
    splits = sms / tiles;
    if (splits > p.nkb / 4) splits = p.nkb / 4;
    const int64_t by_ws = ws_floats / ((int64_t)M * N);
    if (splits > by_ws) splits = (int)by_ws;
    if (splits < 1) splits = 1;
  }
  p.kb_per_split = (p.nkb + splits - 1) / splits;
  p.splits = (p.nkb + p.kb_per_split - 1) / p.kb_per_split;
  p.C = C; p.ldc = ldc; p.beta = beta; p.relu_out = p.splits > 1 ? nullptr : relu_out; p.ldr = ldr;
  p.ws = p.splits > 1 ? ws : nullptr;
  // B pre-split once into the workspace (hi | lo, K-major, row stride Kp);
  // a dual GEMM's B2 rows start at K block nkb1
  const int kb2 = p.nkb1 * gts::BK;
  const int Kext = dual ? kb2 + K2 : K1;
  const int Kp = (Kext + 3) & ~3;
  static const bool no_bsplit = getenv("HB_GEMM_NO_BSPLIT") != nullptr;
  const bool b_tma = gemm_tma_ok(B1, ldb1_n, ldb1_k) && (!dual || gemm_tma_ok(B2, ldb2_n, ldb2_k));
  const bool want_split = p.splits == 1 && ws != nullptr && (int64_t)N * Kp <= (1 << 20) &&
                          2 * (int64_t)N * Kp <= ws_floats &&
                          (!b_tma || (!no_bsplit && (tiles >= 2 * sms || dual) && (p.nkb >= 4 || dual)));
  if (want_split) {
    float* hi = ws;
    float* lo = ws + (int64_t)N * Kp;
    cudaError_t e = gemm_bsplit_range(B1, ldb1_k, ldb1_n, K1, N, dual ? kb2 : Kp, Kp, 0, hi, lo, st);
    if (e == cudaSuccess && dual) e = gemm_bsplit_range(B2, ldb2_k, ldb2_n, K2, N, Kp - kb2, Kp, kb2, hi, lo, st);
    if (e != cudaSuccess) return e;
    if (!gemm_make_map(&tb, hi, Kext, N, Kp, BN, false) || !gemm_make_map(&tbl, lo, Kext, N, Kp, BN, false))
      return cudaErrorNotSupported;
    p.bsplit = 1;
    p.b_mn = 0;
    tb2 = tb;
  } else {
    if (dual && (ldb2_k == 1 ? 0 : 1) != p.b_mn) return cudaErrorNotSupported;
    ok = p.b_mn ? gemm_make_map(&tb, B1, N, K1, ldb1_k, 32, true) : gemm_make_map(&tb, B1, K1, N, ldb1_n, BN, false);
    if (dual)
      ok = ok && (p.b_mn ? gemm_make_map(&tb2, B2, N, K2, ldb2_k, 32, true)
                         : gemm_make_map(&tb2, B2, K2, N, ldb2_n, BN, false));
    else
      tb2 = tb;
    if (!ok) return cudaErrorNotSupported;
    tbl = tb;
  }
  // TMA-store epilogue: plain overwrite of a TMA-describable C (and ReLU copy)
  // C == nullptr: only the ReLU copy is stored (a hidden layer's z is not
  // needed after the forward: the backward masks with h = relu(z) > 0)
  static const bool no_tma_store = getenv("HB_GEMM_NO_TMA_STORE") != nullptr;
  static const bool no_tma_acc = getenv("HB_GEMM_NO_TMA_ACC") != nullptr;
  p.tma_store = !no_tma_store && (beta == 0.f || (C != nullptr && !no_tma_acc)) && p.splits == 1 &&
                (C == nullptr || gemm_tma_ok(C, ldc, 1)) &&
                (!p.relu_out || gemm_tma_ok(p.relu_out, ldr, 1)) &&
                (C == nullptr || gemm_make_map(&tc, C, N, M, ldc, 32, false)) &&
                (!p.relu_out || gemm_make_map(&tr, p.relu_out, N, M, ldr, 32, false));
  if (C == nullptr && (!p.tma_store || !p.relu_out)) return cudaErrorNotSupported;
  if (!p.tma_store) tc = tr = ta;
  else if (!p.relu_out) tr = tc;
  else if (C == nullptr) tc = tr;
  const int total = tiles * p.splits;
  const int grid = total < sms ? total : sms;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gts::gemm_ts_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C_::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  gts::gemm_ts_kernel<BN><<<grid, gts::kThreads, C_::SMEM, st>>>(ta, tb, tbl, ta2, tb2, tc, tr, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.splits > 1) e = gemm_splitk_reduce(ws, p.splits, M, N, C, ldc, beta, relu_out, ldr, st);
  return e;
}

cudaError_t launch_gemm_ts(int M, int N, int K, const float* A, int64_t lda_m, int64_t lda_k, const float* B,
                           int64_t ldb_k, int64_t ldb_n, float* C, int64_t ldc, float beta, float* relu_out, int64_t ldr,
                           float* ws, int64_t ws_floats, cudaStream_t st) {
  if (N <= 64)
    return launch_ts_bn<64>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, 0, nullptr, 0, 0, nullptr, 0, 0, C, ldc, beta,
                            relu_out, ldr, ws, ws_floats, st);
  return launch_ts_bn<128>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, 0, nullptr, 0, 0, nullptr, 0, 0, C, ldc, beta,
                           relu_out, ldr, ws, ws_floats, st);
}

// Dual GEMM on the A-in-TMEM kernel; cudaErrorNotSupported when an operand is
// not TMA-describable or the majors differ (the caller then runs two GEMMs).
cudaError_t launch_gemm_ts_dual(int M, int N, int K1, const float* A1, int64_t lda1_m, int64_t lda1_k,
                                const float* B1, int64_t ldb1_k, int64_t ldb1_n, int K2, const float* A2,
                                int64_t lda2_m, int64_t lda2_k, const float* B2, int64_t ldb2_k, int64_t ldb2_n,
                                float* C, int64_t ldc, float beta, float* relu_out, int64_t ldr, float* ws,
                                int64_t ws_floats, cudaStream_t st) {
  // B operands need not be TMA-describable: the dual path pre-splits them
  // into the workspace whenever it is large enough
  if (!gemm_tma_ok(A1, lda1_m, lda1_k) || !gemm_tma_ok(A2, lda2_m, lda2_k)) return cudaErrorNotSupported;
  if (N <= 64)
    return launch_ts_bn<64>(M, N, K1, A1, lda1_m, lda1_k, B1, ldb1_k, ldb1_n, K2, A2, lda2_m, lda2_k, B2, ldb2_k,
                            ldb2_n, C, ldc, beta, relu_out, ldr, ws, ws_floats, st);
  return launch_ts_bn<128>(M, N, K1, A1, lda1_m, lda1_k, B1, ldb1_k, ldb1_n, K2, A2, lda2_m, lda2_k, B2, ldb2_k,
                           ldb2_n, C, ldc, beta, relu_out, ldr, ws, ws_floats, st);
}


// Split-K weight-gradient GEMM on the A-in-TMEM kernel with decoupled A / B
// rings (gemm_dw_kernel).  cudaErrorNotSupported: caller uses the all-smem kernel.
template <int BN>
static cudaError_t launch_dw_bn(int M, int N, int K, const float* A, int64_t lda_m, int64_t lda_k, const float* B,
                                int64_t ldb_k, int64_t ldb_n, float* C, int64_t ldc, float beta, float* relu_out,
                                int64_t ldr, float* ws, int64_t ws_floats, cudaStream_t st) {
  using C_ = gts::DwCfg<BN>;
  gts::Params p{};
  p.M = M; p.N = N; p.K = K;
  p.a_mn = lda_k == 1 ? 0 : 1;
  p.b_mn = ldb_k == 1 ? 0 : 1;
  CUtensorMap ta, tb;
  bool ok = p.a_mn ? gemm_make_map(&ta, A, M, K, lda_k, 32, true) : gemm_make_map(&ta, A, K, M, lda_m, gts::BM, false);
  ok = ok && (p.b_mn ? gemm_make_map(&tb, B, N, K, ldb_k, 32, true) : gemm_make_map(&tb, B, K, N, ldb_n, BN, false));
  if (!ok) return cudaErrorNotSupported;
  p.mt = (M + gts::BM - 1) / gts::BM;
  p.nt = (N + BN - 1) / BN;
  p.nkb = (K + gts::BK - 1) / gts::BK;
  p.nkb1 = p.nkb;
  const int sms = num_sms();
  const int tiles = p.mt * p.nt;
  int splits = sms / tiles;
  if (splits > p.nkb / 4) splits = p.nkb / 4;
  const int64_t by_ws = ws_floats / ((int64_t)M * N);
  if (splits > by_ws) splits = (int)by_ws;
  if (splits < 1) splits = 1;
  p.kb_per_split = (p.nkb + splits - 1) / splits;
  p.splits = (p.nkb + p.kb_per_split - 1) / p.kb_per_split;
  p.C = C; p.ldc = ldc; p.beta = beta; p.relu_out = p.splits > 1 ? nullptr : relu_out; p.ldr = ldr;
  p.ws = p.splits > 1 ? ws : nullptr;
  const int total = tiles * p.splits;
  const int grid = total < sms ? total : sms;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gts::gemm_dw_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C_::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  gts::gemm_dw_kernel<BN><<<grid, gts::kThreads, C_::SMEM, st>>>(ta, tb, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.splits > 1) e = gemm_splitk_reduce(ws, p.splits, M, N, C, ldc, beta, relu_out, ldr, st);
  return e;
}

cudaError_t launch_gemm_dw(int M, int N, int K, const float* A, int64_t lda_m, int64_t lda_k, const float* B,
                           int64_t ldb_k, int64_t ldb_n, float* C, int64_t ldc, float beta, float* relu_out, int64_t ldr,
                           float* ws, int64_t ws_floats, cudaStream_t st) {
  if (N <= 64)
    return launch_dw_bn<64>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws, ws_floats, st);
  if (N <= 128)
    return launch_dw_bn<128>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws, ws_floats, st);
  return launch_dw_bn<256>(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws, ws_floats, st);
}

}  // namespace hb
