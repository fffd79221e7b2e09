// K3/K4 factored tiled path: SpMM with a 0/1 pattern and diagonal scalings,
//
//   Y[i, :] = r[i] * sum_{(i,j) in pattern} c[j] X[j, :]
//
// which is what the trainer's aggregation operators are (linalg.spmm,
// linalg.py:71-75, on the blocks of graph.py:120-141):
//   * SAGE mean        M  = D^-1 A           -> r = 1/deg,  c = 1
//   * its transpose    M^T = A^T D^-1        -> r = 1,      c = 1/deg
//   * GCN              Â  = D^-1/2 (A+I) D^-1/2 -> r = c = dinv.
// With the values factored out a tile record is the nonzero's column inside
// its 64-column window: ONE BYTE (the general kernel, spmm_tiled.cu, moves an
// 8-byte (col, val) record per nonzero through shared memory).  Each row's
// run of records is padded to whole 32-bit words (0xFF = padding) and read a
// word — 4 records — per broadcast load, unpacked with byte permutes, so the
// shared-memory datapath (the binding resource of a SIMT SpMM) carries the
// gathered X rows plus a quarter wavefront per nonzero: 8.25 wavefronts per
// nonzero at d = 256 instead of 9, with no per-record issue overhead beyond
// the general kernel's.
// Row blocks are 64 or 128 rows tall (16 consumer warps x 4 or 8 rows); taller
// blocks reuse each TMA-staged 64-row X window across more rows.  c is applied by a pre-pass into a
// caller-provided scratch copy of X (one HBM read + write of X), r to the
// accumulators before the store.
//
// Work items (row block, feature panel) are handed out in ascending order
// from a caller-provided counter pair {next item, CTAs finished} that must be
// zero on entry; the last CTA out re-arms it, so the same pair serves the
// next launch on the stream (and graph replays).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdlib>
#include "common.cuh"

namespace hb {

// narrow-row consumer layout (hb_spmm_set_narrow); 1 = the measured fastest
// per window width (255-column windows: balanced tail pairs)
int g_bin_narrow = getenv("HB_BIN_NARROW") ? atoi(getenv("HB_BIN_NARROW")) : 1;
// 128-row blocks, d > 128: 1 = 256-column panels (two records in flight), 0 = 128-column panels
int g_bin_wide128 = getenv("HB_BIN_WIDE128") ? atoi(getenv("HB_BIN_WIDE128")) : 1;

namespace sb {

// columns per window KW (64, or 128 for narrow rows): a record is col - c0 < KW
// record bytes per tile (ops.TiledCsr splits denser tiles): 2048, 4096 for
// 128-row x 255-column narrow tiles
constexpr int max_rec(int rb, int kw) { return rb == 128 && kw == 255 ? 4096 : 2048; }
// consumer warps per CTA (CW; a warp owns RB / CW rows of the block) + 1 producer
// u16 row offsets per tile: RB + 1 used, padded to a 16-byte multiple
constexpr int row_off_count(int rb) { return rb == 64 ? 72 : 136; }
constexpr int kQ = 4;

struct Args {
  int nrows, nblocks, npanels, d, pw;
  int* work;
  const int32_t* tile_ptr;
  const int32_t* tile_win;
  const int64_t* tile_off;        // byte offsets of each tile's records (multiples of 16)
  const uint16_t* tile_rowoff;    // [ntiles][row_off_count(RB)]
  const uint8_t* tile_rec;
  const int64_t* res_ptr;         // residual pattern (CSR without values)
  const int32_t* res_col;
  const float* row_scale;         // nullable
  const float* X;
  int64_t ldx;
  float* Y;
  int64_t ldy;
  const int32_t* block_order;     // nullable: item i works on row block block_order[i / npanels]
};

template <int RB, int NV, int G, int S, int KW = 64, bool TP = false>
struct Smem {
  // panel width in floats (TP: at most 48 columns, one panel)
  static constexpr int P = TP ? 48 : 4 * G * NV;
  static constexpr int X_BYTES = (KW * P * 4 + 127) / 128 * 128;   // TMA destinations: 128-byte aligned
  static constexpr int RO_BYTES = row_off_count(RB) * 2;
  static constexpr int MAXREC = max_rec(RB, KW);
  static constexpr int STAGE = X_BYTES + MAXREC + RO_BYTES + 112;   // 16-byte multiple
  static constexpr int TOTAL = S * STAGE + 128;
  static_assert(STAGE % 16 == 0, "stage alignment");
};

__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

template <int NV, int G>
__device__ __forceinline__ void add_row(float4 (&acc)[NV], const float4* __restrict__ x, int nlast) {
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    if (q < NV - 1 || nlast) {
      const float4 t = x[q * G];
      acc[q].x += t.x; acc[q].y += t.y; acc[q].z += t.z; acc[q].w += t.w;
    }
  }
}

// 1 CTA/SM: 17 warps are allocated registers as 20 (4-warp granularity), so
// 96 per thread is the most that launches; 2 CTAs/SM: 56
// RB rows per block (kRPW = RB / CW per warp), NV float4 per lane, G lanes
// per row group, S ring stages, MINB CTAs per SM, CW consumer warps
// TP ("tail pairs", 32 < d <= 48, G = 8, NV = 2): a lane group reads a
// nonzero's first 32 columns as one 128-byte quarter-warp access (all 32
// banks once: conflict-free wherever the row starts) and the 1-4 float4 tail
// of TWO nonzeros in a third access (lanes 0-3: the first's, lanes 4-7: the
// second's), so a pair costs 3 accesses instead of 4; acc[i][1] holds the
// tail sums, folded across the half-groups before the store.  With 4-lane
// groups (64-byte accesses, two rows per quarter-warp) the two halves of a
// quarter-warp collide in 7 of 8 bank alignments.
// barrier setup shared by the consumer layouts: S ring stages, kQ work-item slots
template <int S, int CW>
__device__ __forceinline__ void bin_init(uint64_t* full, uint64_t* empty, uint64_t* ifull, uint64_t* iempty) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    for (int q = 0; q < kQ; ++q) {
      mbar_init(&ifull[q], 1);
      mbar_init(&iempty[q], CW);
    }
    fence_mbar_init();
  }
  __syncthreads();
}

// producer warp: lane 0 claims work items (row block, panel) and posts them to
// the consumers; lane s feeds ring stage s (X window by TMA, the tile's
// records and row offsets by bulk copies)
template <class S_, int S, int KW, int kRowOff>
__device__ __forceinline__ void bin_producer(const CUtensorMap* tmX, const Args& a, uint8_t* smem, uint64_t* full,
                                             uint64_t* empty, uint64_t* ifull, uint64_t* iempty, int* item_q,
                                             int lane, int items, int P) {
  int it = 0;
  for (int qi = 0;; ++qi) {
    int item = 0;
    if (lane == 0) {
      item = atomicAdd(a.work, 1);
      const int q = qi % kQ;
      mbar_wait(&iempty[q], ((qi / kQ) & 1) ^ 1);
      item_q[q] = item;
      mbar_arrive_cta(&ifull[q]);
      if (item >= items && atomicAdd(a.work + 1, 1) == (int)gridDim.x - 1) {
        atomicExch(a.work, 0);
        atomicExch(a.work + 1, 0);
      }
    }
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= items) break;
    const int bi = item / a.npanels, pn = item % a.npanels;
    const int b = a.block_order ? __ldg(a.block_order + bi) : bi;
    const int t0 = a.tile_ptr[b], t1 = a.tile_ptr[b + 1];
    for (int t = t0; t < t1; ++t, ++it) {
      if (lane >= S || it % S != lane) continue;
      const int s = it % S;
      mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
      uint8_t* st = smem + s * S_::STAGE;
      const int64_t o0 = a.tile_off[t], o1 = a.tile_off[t + 1];
      const uint32_t rb = (uint32_t)(o1 - o0);
      mbar_expect_tx(&full[s], (uint32_t)(KW * a.pw * 4) + rb + S_::RO_BYTES);
      tma_2d(st, tmX, pn * P, a.tile_win[t] * KW, &full[s]);
      if (rb) tma_load_1d(st + S_::X_BYTES, a.tile_rec + o0, rb, &full[s]);
      tma_load_1d(st + S_::X_BYTES + S_::MAXREC, a.tile_rowoff + (int64_t)t * kRowOff, S_::RO_BYTES, &full[s]);
    }
  }
  __syncwarp();
}

template <int RB, int NV, int G, int S, int MINB, int CW, bool TP = false, int KW = 64>
__global__ void __maxnreg__(MINB == 1 ? (CW >= 24 ? 64 : 96) : 56)
spmm_bin_kernel(const __grid_constant__ CUtensorMap tmX, Args a) {
  using S_ = Smem<RB, NV, G, S, KW, TP>;
  constexpr int P = S_::P;
  constexpr int kConsumers = CW;
  constexpr int kRPW = RB / kConsumers;
  constexpr int kRowOff = row_off_count(RB);
  constexpr int NG = 32 / G;             // lane groups per warp (each owns whole rows)
  constexpr int RPG = kRPW / NG;         // rows per lane group
  static_assert(RPG >= 1 && kRPW % NG == 0, "row split");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  __shared__ __align__(8) uint64_t full[S], empty[S], ifull[kQ], iempty[kQ];
  __shared__ int item_q[kQ];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hg = lane / G, gl = lane % G;
  bin_init<S, kConsumers>(full, empty, ifull, iempty);
  const int items = a.nblocks * a.npanels;

  if (warp == kConsumers) {
    bin_producer<S_, S, KW, kRowOff>(&tmX, a, smem, full, empty, ifull, iempty, item_q, lane, items, P);
    return;
  }

  // ---------------- consumers: lane group hg owns rows hg, hg + NG, ... of
  // the warp's kRPW rows; lane gl holds NV float4 columns of the panel
  const int pw4 = a.pw / 4;
  // the last float4 of a lane may fall beyond the staged width (narrow panels)
  const int nlast = ((NV - 1) * G + gl) * 4 < a.pw;
  // TP: lane gl's tail float4 (8 + (gl & 3)) and whether the row has it
  const int tl = gl & 3;
  const bool tail_lane = (8 + tl) * 4 < a.pw;
  int it = 0;
  for (int qi = 0;; ++qi) {
    const int q = qi % kQ;
    mbar_wait(&ifull[q], (qi / kQ) & 1);
    const int item = item_q[q];
    __syncwarp();
    if (lane == 0) mbar_arrive_cta(&iempty[q]);
    if (item >= items) break;
    const int bi = item / a.npanels, pn = item % a.npanels;
    const int b = a.block_order ? __ldg(a.block_order + bi) : bi;
    const int r0 = b * RB + warp * kRPW;
    const int col0 = pn * P;
    float4 acc[RPG][NV];
#pragma unroll
    for (int i = 0; i < RPG; ++i)
#pragma unroll
      for (int v = 0; v < NV; ++v) acc[i][v] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int t = a.tile_ptr[b]; t < a.tile_ptr[b + 1]; ++t, ++it) {
      const int s = it % S;
      mbar_wait(&full[s], (it / S) & 1);
      const uint8_t* st = smem + s * S_::STAGE;
      const float4* xs = reinterpret_cast<const float4*>(st) + gl;
      const uint32_t* rec32 = reinterpret_cast<const uint32_t*>(st + S_::X_BYTES);
      const uint16_t* ro = reinterpret_cast<const uint16_t*>(st + S_::X_BYTES + S_::MAXREC) + warp * kRPW;
      // the warp's kRPW + 1 row offsets in two broadcast loads (not 2 per row)
      uint64_t ro_lo, ro_hi = 0;
      if constexpr (kRPW == 4) {
        ro_lo = *reinterpret_cast<const uint64_t*>(ro);
      } else {
        const uint4 v = *reinterpret_cast<const uint4*>(ro);
        ro_lo = ((uint64_t)v.y << 32) | v.x;
        ro_hi = ((uint64_t)v.w << 32) | v.z;
      }
      const int ro_end = ro[kRPW];
      auto row_off = [&](int q) -> int {
        if (q >= kRPW) return ro_end;
        const uint64_t v = q < 4 ? ro_lo : ro_hi;
        return (int)((v >> (16 * (q & 3))) & 0xffffu);
      };
#pragma unroll
      for (int i = 0; i < RPG; ++i) {
        const int rr = hg + i * NG;
        // the row's run of one-byte records, padded to whole words with 0xFF:
        // every word but the last holds 4 records
        const int w1 = row_off(rr + 1) >> 2;
        int w = row_off(rr) >> 2;
        if constexpr (G == 32) {
          // records in flight per warp: 4, or 2 when the accumulators of a
          // 128-row block (8 rows x NV float4) leave no registers for more
          constexpr int kU = RPG * NV > 8 || CW >= 24 ? 2 : 4;
          for (; w + 1 < w1; ++w) {
            const uint32_t q = rec32[w];                           // 4 records, one broadcast
#pragma unroll
            for (int u0 = 0; u0 < 4; u0 += kU) {
              float4 x[kU][NV];
#pragma unroll
              for (int u = 0; u < kU; ++u) {
                const int j = (int)__byte_perm(q, 0u, 0x4440u | (uint32_t)(u0 + u));
#pragma unroll
                for (int v = 0; v < NV; ++v)
                  if (v < NV - 1 || nlast) x[u][v] = xs[j * pw4 + v * G];
              }
#pragma unroll
              for (int u = 0; u < kU; ++u)
#pragma unroll
                for (int v = 0; v < NV; ++v)
                  if (v < NV - 1 || nlast) {
                    acc[i][v].x += x[u][v].x; acc[i][v].y += x[u][v].y;
                    acc[i][v].z += x[u][v].z; acc[i][v].w += x[u][v].w;
                  }
            }
          }
        } else if constexpr (TP) {
          static_assert(G == 8 && NV == 2, "tail pairs: 8-lane groups, main + tail float4");
          // pairs of nonzeros: two 128-byte main reads + one shared tail read;
          // the next record word is loaded before this word's X rows
          uint32_t qn = w + 1 < w1 ? rec32[w] : 0u;
          for (; w + 1 < w1; ++w) {
            const uint32_t q = qn;
            qn = rec32[w + 1];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int j0 = (int)__byte_perm(q, 0u, 0x4440u | (uint32_t)(2 * h));
              const int j1 = (int)__byte_perm(q, 0u, 0x4441u | (uint32_t)(2 * h));
              const float4 m0 = xs[j0 * pw4];
              const float4 m1 = xs[j1 * pw4];
              const int jt = gl < 4 ? j0 : j1;
              float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
              if (tail_lane) t = xs[jt * pw4 + 8 - gl + tl];
              acc[i][0].x += m0.x; acc[i][0].y += m0.y; acc[i][0].z += m0.z; acc[i][0].w += m0.w;
              acc[i][0].x += m1.x; acc[i][0].y += m1.y; acc[i][0].z += m1.z; acc[i][0].w += m1.w;
              acc[i][1].x += t.x; acc[i][1].y += t.y; acc[i][1].z += t.z; acc[i][1].w += t.w;
            }
          }
        } else {
          // narrow rows: each lane group walks its own row, two records at a time
          for (; w + 1 < w1; ++w) {
            const uint32_t q = rec32[w];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int j0 = (int)__byte_perm(q, 0u, 0x4440u | (uint32_t)(2 * h));
              const int j1 = (int)__byte_perm(q, 0u, 0x4441u | (uint32_t)(2 * h));
              float4 x0[NV], x1[NV];
#pragma unroll
              for (int v = 0; v < NV; ++v)
                if (v < NV - 1 || nlast) {
                  x0[v] = xs[j0 * pw4 + v * G];
                  x1[v] = xs[j1 * pw4 + v * G];
                }
#pragma unroll
              for (int v = 0; v < NV; ++v)
                if (v < NV - 1 || nlast) {
                  acc[i][v].x += x0[v].x; acc[i][v].y += x0[v].y; acc[i][v].z += x0[v].z; acc[i][v].w += x0[v].w;
                  acc[i][v].x += x1[v].x; acc[i][v].y += x1[v].y; acc[i][v].z += x1[v].z; acc[i][v].w += x1[v].w;
                }
            }
          }
        }
        if (w < w1) {                    // the run's last word: 0xFF bytes are padding
          const uint32_t q = rec32[w];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = (int)__byte_perm(q, 0u, 0x4440u | (uint32_t)u);
            if constexpr (TP) {
              if (j != 0xFF) {
                const float4 m = xs[j * pw4];
                acc[i][0].x += m.x; acc[i][0].y += m.y; acc[i][0].z += m.z; acc[i][0].w += m.w;
                if (gl < 4 && tail_lane) {
                  const float4 t = xs[j * pw4 + 8 - gl + tl];
                  acc[i][1].x += t.x; acc[i][1].y += t.y; acc[i][1].z += t.z; acc[i][1].w += t.w;
                }
              }
            } else {
              if (j != 0xFF) add_row<NV, G>(acc[i], xs + j * pw4, nlast);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&empty[s]);
    }
    if constexpr (TP) {
      // fold the second nonzero's tail sums (lanes 4-7) into lanes 0-3
#pragma unroll
      for (int i = 0; i < RPG; ++i) {
        float4& t = acc[i][1];
        const float x = __shfl_down_sync(0xffffffffu, t.x, 4, 8), y = __shfl_down_sync(0xffffffffu, t.y, 4, 8);
        const float z = __shfl_down_sync(0xffffffffu, t.z, 4, 8), w = __shfl_down_sync(0xffffffffu, t.w, 4, 8);
        if (gl < 4) { t.x += x; t.y += y; t.z += z; t.w += w; }
      }
    }
    // residual pattern entries gathered from global X, row scale, store
#pragma unroll
    for (int i = 0; i < RPG; ++i) {
      const int r = r0 + hg + i * NG;
      if (r >= a.nrows) continue;
      if constexpr (TP) {
        // lane gl: main float4 gl; lanes 0-3 also tail float4 8 + gl
        const int64_t e0 = a.res_ptr[r], e1 = a.res_ptr[r + 1];
        const bool has_t = gl < 4 && tail_lane;
        for (int64_t k = e0; k < e1; ++k) {
          const float4* xr = reinterpret_cast<const float4*>(a.X + (int64_t)__ldg(a.res_col + k) * a.ldx);
          if (gl * 4 < a.d) {
            const float4 t4 = __ldg(xr + gl);
            acc[i][0].x += t4.x; acc[i][0].y += t4.y; acc[i][0].z += t4.z; acc[i][0].w += t4.w;
          }
          if (has_t) {
            const float4 t4 = __ldg(xr + 8 + gl);
            acc[i][1].x += t4.x; acc[i][1].y += t4.y; acc[i][1].z += t4.z; acc[i][1].w += t4.w;
          }
        }
        const float sc = a.row_scale ? __ldg(a.row_scale + r) : 1.f;
        float* y = a.Y + (int64_t)r * a.ldy;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          if (v == 1 && !has_t) continue;
          const int col = v == 0 ? gl * 4 : (8 + gl) * 4;
          const int rem = a.d - col;
          const float4 o = make_float4(acc[i][v].x * sc, acc[i][v].y * sc, acc[i][v].z * sc, acc[i][v].w * sc);
          if (rem >= 4) {
            *reinterpret_cast<float4*>(y + col) = o;
          } else if (rem > 0) {
            y[col] = o.x;
            if (rem > 1) y[col + 1] = o.y;
            if (rem > 2) y[col + 2] = o.z;
          }
        }
        continue;
      }
      const float* Xp = a.X + col0;
      const int64_t e0 = a.res_ptr[r], e1 = a.res_ptr[r + 1];
      for (int64_t k = e0; k < e1; ++k) {
        const float4* xr = reinterpret_cast<const float4*>(Xp + (int64_t)__ldg(a.res_col + k) * a.ldx) + gl;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          if (col0 + (v * G + gl) * 4 < a.d) {
            const float4 t4 = __ldg(xr + v * G);
            acc[i][v].x += t4.x; acc[i][v].y += t4.y; acc[i][v].z += t4.z; acc[i][v].w += t4.w;
          }
        }
      }
      const float sc = a.row_scale ? __ldg(a.row_scale + r) : 1.f;
      float* y = a.Y + (int64_t)r * a.ldy + col0;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int col = (v * G + gl) * 4;
        const int rem = a.d - col0 - col;
        const float4 o = make_float4(acc[i][v].x * sc, acc[i][v].y * sc, acc[i][v].z * sc, acc[i][v].w * sc);
        if (rem >= 4) {
          *reinterpret_cast<float4*>(y + col) = o;
        } else if (rem > 0) {
          y[col] = o.x;
          if (rem > 1) y[col + 1] = o.y;
          if (rem > 2) y[col + 2] = o.z;
        }
      }
    }
  }
}

// Narrow rows (32 < d <= 48), 64-row blocks, tail pairs with GPR lane groups
// per row.  The tail-pair layout of spmm_bin_kernel gives each 8-lane group
// its own row, so a warp's four groups walk runs of different lengths and the
// warp waits for the longest; here GPR groups share one row, taking its
// record pairs round-robin (trip counts differ by at most one), and their
// partial sums are added with shuffles once the block is done.  A warp still
// owns 4 rows: SLOTS = 4 / GPR rows are in flight at a time, KS = GPR row
// sets in turn (acc holds KS rows x {main, tail}).  The summation order
// inside a row differs from CSR order (tolerance contract of hb_spmm_csr).
template <int S, int MINB, int GPR, int KW>
__global__ void __maxnreg__(MINB == 1 ? 96 : 56)
spmm_bin_tpb_kernel(const __grid_constant__ CUtensorMap tmX, Args a) {
  constexpr int RB = 64, CW = 16, G = 8, NV = 2;
  using S_ = Smem<RB, NV, G, S, KW, true>;
  constexpr int kRPW = RB / CW, NG = 32 / G, SLOTS = NG / GPR, KS = kRPW / SLOTS;
  constexpr int kRowOff = row_off_count(RB);
  static_assert(kRPW == 4 && NG == 4 && KS == GPR, "4 rows x 4 lane groups per warp");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  __shared__ __align__(8) uint64_t full[S], empty[S], ifull[kQ], iempty[kQ];
  __shared__ int item_q[kQ];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bin_init<S, CW>(full, empty, ifull, iempty);
  const int items = a.nblocks * a.npanels;
  if (warp == CW) {
    bin_producer<S_, S, KW, kRowOff>(&tmX, a, smem, full, empty, ifull, iempty, item_q, lane, items, S_::P);
    return;
  }
  const int hg = lane >> 3, gl = lane & 7;
  const int slot = hg / GPR, sub = hg % GPR;
  const int pw4 = a.pw / 4;
  const int tl = gl & 3;
  const bool tail_lane = (8 + tl) * 4 < a.pw;       // tail float4 8 + tl exists
  int it = 0;
  for (int qi = 0;; ++qi) {
    const int q = qi % kQ;
    mbar_wait(&ifull[q], (qi / kQ) & 1);
    const int item = item_q[q];
    __syncwarp();
    if (lane == 0) mbar_arrive_cta(&iempty[q]);
    if (item >= items) break;
    const int bi = item / a.npanels;
    const int b = a.block_order ? __ldg(a.block_order + bi) : bi;
    const int r0 = b * RB + warp * kRPW;
    float4 acc[KS][2];
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      acc[k][0] = make_float4(0.f, 0.f, 0.f, 0.f);
      acc[k][1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int t = a.tile_ptr[b]; t < a.tile_ptr[b + 1]; ++t, ++it) {
      const int s = it % S;
      mbar_wait(&full[s], (it / S) & 1);
      const uint8_t* st = smem + s * S_::STAGE;
      const float4* xs = reinterpret_cast<const float4*>(st);
      const uint32_t* rec32 = reinterpret_cast<const uint32_t*>(st + S_::X_BYTES);
      const uint16_t* ro = reinterpret_cast<const uint16_t*>(st + S_::X_BYTES + S_::MAXREC) + warp * kRPW;
      const uint64_t ro4 = *reinterpret_cast<const uint64_t*>(ro);     // the warp's 4 row offsets
      const int ro_end = ro[kRPW];
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        const int rr = k * SLOTS + slot;
        const int w0 = (int)((ro4 >> (16 * rr)) & 0xffffu) >> 2;
        const int w1 = (rr + 1 < kRPW ? (int)((ro4 >> (16 * (rr + 1))) & 0xffffu) : ro_end) >> 2;
        const int np = 2 * (w1 - w0);                              // record pairs (the last may be padding)
        for (int pp = sub; pp < np; pp += GPR) {
          const uint32_t qw = rec32[w0 + (pp >> 1)] >> (16 * (pp & 1));
          const int j0 = (int)(qw & 0xffu), j1 = (int)((qw >> 8) & 0xffu);
          if (j0 == 0xFF) break;                                   // padding ends the run
          const bool has1 = j1 != 0xFF;
          const float4 m0 = xs[j0 * pw4 + gl];
          float4 m1 = make_float4(0.f, 0.f, 0.f, 0.f);
          if (has1) m1 = xs[j1 * pw4 + gl];
          // one quarter-warp access for both tails: lanes 0-3 the first's, 4-7 the second's
          const int jt = gl < 4 ? j0 : j1;
          float4 tv = make_float4(0.f, 0.f, 0.f, 0.f);
          if (tail_lane && (gl < 4 || has1)) tv = xs[jt * pw4 + 8 + tl];
          acc[k][0].x += m0.x; acc[k][0].y += m0.y; acc[k][0].z += m0.z; acc[k][0].w += m0.w;
          if (has1) {
            acc[k][0].x += m1.x; acc[k][0].y += m1.y; acc[k][0].z += m1.z; acc[k][0].w += m1.w;
          }
          acc[k][1].x += tv.x; acc[k][1].y += tv.y; acc[k][1].z += tv.z; acc[k][1].w += tv.w;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&empty[s]);
    }
    // fold the second records' tails (lanes 4-7) into lanes 0-3, then add the
    // partial sums of the GPR groups that shared each row
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      float4& tv = acc[k][1];
      const float x = __shfl_down_sync(0xffffffffu, tv.x, 4, 8), y = __shfl_down_sync(0xffffffffu, tv.y, 4, 8);
      const float z = __shfl_down_sync(0xffffffffu, tv.z, 4, 8), w = __shfl_down_sync(0xffffffffu, tv.w, 4, 8);
      if (gl < 4) { tv.x += x; tv.y += y; tv.z += z; tv.w += w; }
#pragma unroll
      for (int o = 8; o < 8 * GPR; o <<= 1) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          float4& u = acc[k][v];
          u.x += __shfl_xor_sync(0xffffffffu, u.x, o);
          u.y += __shfl_xor_sync(0xffffffffu, u.y, o);
          u.z += __shfl_xor_sync(0xffffffffu, u.z, o);
          u.w += __shfl_xor_sync(0xffffffffu, u.w, o);
        }
      }
    }
    // group (slot, sub) finishes row set k = sub: residual gathers, row scale, store
    float4 am = make_float4(0.f, 0.f, 0.f, 0.f), at = am;
#pragma unroll
    for (int k = 0; k < KS; ++k)
      if (k == sub) { am = acc[k][0]; at = acc[k][1]; }
    const int r = r0 + sub * SLOTS + slot;
    if (r < a.nrows) {
      const int64_t e0 = a.res_ptr[r], e1 = a.res_ptr[r + 1];
      const bool has_t = gl < 4 && tail_lane;
      for (int64_t k = e0; k < e1; ++k) {
        const float4* xr = reinterpret_cast<const float4*>(a.X + (int64_t)__ldg(a.res_col + k) * a.ldx);
        if (gl * 4 < a.d) {
          const float4 t4 = __ldg(xr + gl);
          am.x += t4.x; am.y += t4.y; am.z += t4.z; am.w += t4.w;
        }
        if (has_t) {
          const float4 t4 = __ldg(xr + 8 + gl);
          at.x += t4.x; at.y += t4.y; at.z += t4.z; at.w += t4.w;
        }
      }
      const float sc = a.row_scale ? __ldg(a.row_scale + r) : 1.f;
      float* y = a.Y + (int64_t)r * a.ldy;
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        if (v == 1 && !has_t) continue;
        const float4 u = v == 0 ? am : at;
        const int col = v == 0 ? gl * 4 : (8 + gl) * 4;
        const int rem = a.d - col;
        const float4 o = make_float4(u.x * sc, u.y * sc, u.z * sc, u.w * sc);
        if (rem >= 4) {
          *reinterpret_cast<float4*>(y + col) = o;
        } else if (rem > 0) {
          y[col] = o.x;
          if (rem > 1) y[col + 1] = o.y;
          if (rem > 2) y[col + 2] = o.z;
        }
      }
    }
  }
}

// Xs[j, :d] = c[j] * X[j, :d]  (float4 rows: ld % 4 == 0, 16-byte aligned)
__global__ void scale_rows_kernel(const float* __restrict__ X, int64_t ldx, int rows, int d4,
                                  const float* __restrict__ c, float* __restrict__ Xs, int64_t ldxs) {
  const int64_t total = (int64_t)rows * d4;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d4, q = e - r * d4;
    const float s = __ldg(c + r);
    float4 v = __ldg(reinterpret_cast<const float4*>(X + r * ldx) + q);
    v.x *= s; v.y *= s; v.z *= s; v.w *= s;
    reinterpret_cast<float4*>(Xs + r * ldxs)[q] = v;
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

template <int RB, int NV, int G, int S, int MINB, int CW = 16, bool TP = false, int KW = 64>
static cudaError_t launch_nv(const Args& a0, int xrows, cudaStream_t stream) {
  using S_ = Smem<RB, NV, G, S, KW, TP>;
  static_assert(MINB * S_::TOTAL <= 227 * 1024, "smem");
  Args a = a0;
  a.npanels = (a.d + S_::P - 1) / S_::P;
  a.pw = a.npanels > 1 ? S_::P : (a.d + 3) / 4 * 4;
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)a.d, (cuuint64_t)xrows};
  cuuint64_t strides[1] = {(cuuint64_t)(a.ldx * 4)};
  cuuint32_t box[2] = {(cuuint32_t)a.pw, (cuuint32_t)KW};
  cuuint32_t es[2] = {1u, 1u};
  if (fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a.X), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(spmm_bin_kernel<RB, NV, G, S, MINB, CW, TP, KW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, S_::TOTAL);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int items = a.nblocks * a.npanels;
  const int grid = items < MINB * num_sms() ? items : MINB * num_sms();
  if (grid > 0) spmm_bin_kernel<RB, NV, G, S, MINB, CW, TP, KW><<<grid, 32 * (CW + 1), S_::TOTAL, stream>>>(map, a);
  return cudaGetLastError();
}

template <int S, int MINB, int GPR, int KW>
static cudaError_t launch_tpb(const Args& a0, int xrows, cudaStream_t stream) {
  using S_ = Smem<64, 2, 8, S, KW, true>;
  static_assert(MINB * S_::TOTAL <= 227 * 1024, "smem");
  Args a = a0;
  a.npanels = 1;
  a.pw = (a.d + 3) / 4 * 4;
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)a.d, (cuuint64_t)xrows};
  cuuint64_t strides[1] = {(cuuint64_t)(a.ldx * 4)};
  cuuint32_t box[2] = {(cuuint32_t)a.pw, (cuuint32_t)KW};
  cuuint32_t es[2] = {1u, 1u};
  if (fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a.X), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(spmm_bin_tpb_kernel<S, MINB, GPR, KW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, S_::TOTAL);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int items = a.nblocks;
  const int grid = items < MINB * num_sms() ? items : MINB * num_sms();
  if (grid > 0) spmm_bin_tpb_kernel<S, MINB, GPR, KW><<<grid, 32 * 17, S_::TOTAL, stream>>>(map, a);
  return cudaGetLastError();
}

}  // namespace sb

// Xs[j, :d] = c[j] * X[j, :d] (the column scaling of the factored operators)
cudaError_t launch_scale_rows(const float* X, int64_t ldx, int xrows, int d, const float* c, float* xs,
                              int64_t ldxs, cudaStream_t stream) {
  const int d4 = (d + 3) / 4;
  const int64_t total = (int64_t)xrows * d4;
  int grid = (int)((total + 255) / 256);
  if (grid > num_sms() * 16) grid = num_sms() * 16;
  if (grid > 0) sb::scale_rows_kernel<<<grid, 256, 0, stream>>>(X, ldx, xrows, d4, c, xs, ldxs);
  return cudaGetLastError();
}

cudaError_t launch_spmm_tiled_bin(int nrows, int xrows, int nblocks, const int32_t* tile_ptr,
                                  const int32_t* tile_win, const int64_t* tile_off, const uint16_t* tile_rowoff,
                                  const uint8_t* tile_rec, const int64_t* res_ptr, const int32_t* res_col,
                                  const float* row_scale, const float* col_scale, const float* X, int64_t ldx,
                                  int d, float* Y, int64_t ldy, float* xs, int64_t ldxs, int* work,
                                  int block_rows, int window_cols, const int32_t* block_order,
                                  cudaStream_t stream) {
  if (nrows <= 0 || d <= 0) return cudaSuccess;
  if ((ldx & 3) || (ldy & 3) || (((uintptr_t)X) & 15) || (((uintptr_t)Y) & 15)) return cudaErrorNotSupported;
  if (col_scale) {
    if (!xs || (ldxs & 3) || (((uintptr_t)xs) & 15) || ldxs < d) return cudaErrorInvalidValue;
    const cudaError_t e = launch_scale_rows(X, ldx, xrows, d, col_scale, xs, ldxs, stream);
    if (e != cudaSuccess) return e;
    X = xs;
    ldx = ldxs;
  }
  sb::Args a{};
  a.nrows = nrows; a.nblocks = nblocks; a.d = d; a.work = work;
  a.tile_ptr = tile_ptr; a.tile_win = tile_win; a.tile_off = tile_off; a.tile_rowoff = tile_rowoff;
  a.tile_rec = tile_rec; a.res_ptr = res_ptr; a.res_col = res_col; a.row_scale = row_scale;
  a.X = X; a.ldx = ldx; a.Y = Y; a.ldy = ldy; a.block_order = block_order;
  const int narrow = g_bin_narrow;
  if (window_cols == 255) {
    // 255-column windows (one-byte records 0..254, 0xFF = padding)
    if (d > 48) return cudaErrorInvalidValue;
    if (block_rows == 128) {
      // 128-row blocks: each staged window serves twice the rows; 16 consumer
      // warps x 8 rows (tail pairs, two rows per lane group), 2 CTAs per SM
      if (d <= 32) return cudaErrorInvalidValue;
      return sb::launch_nv<128, 2, 8, 2, 2, 16, true, 255>(a, xrows, stream);
    }
    if (block_rows != 64) return cudaErrorInvalidValue;
    // default (1, 4): tail pairs with two lane groups per row, 2 CTAs per SM
    // (0.95 / 1.00 ms at d = 41 on Reddit's mean operator / its transpose);
    // 3: tail pairs, a lane group per row (1.03 / 1.08 ms); 2: the same, 1
    // CTA per SM; 0 (or d <= 32): 4-lane groups
    if (d > 32 && (narrow == 1 || narrow == 4)) return sb::launch_tpb<2, 2, 2, 255>(a, xrows, stream);
    if (d > 32 && narrow == 2) return sb::launch_nv<64, 2, 8, 2, 1, 16, true, 255>(a, xrows, stream);
    if (d > 32 && narrow == 3) return sb::launch_nv<64, 2, 8, 2, 2, 16, true, 255>(a, xrows, stream);
    return sb::launch_nv<64, 3, 4, 2, 2, 8, false, 255>(a, xrows, stream);
  }
  if (window_cols == 128) {
    // 128-column windows (narrow rows): twice the nonzeros per (row, tile)
    // for the per-row record-run overhead
    if (block_rows != 64 || d > 48) return cudaErrorInvalidValue;
    if (d > 32 && narrow == 2) return sb::launch_nv<64, 2, 8, 2, 3, 8, true, 128>(a, xrows, stream);
    if (d > 32 && narrow == 3) return sb::launch_nv<64, 2, 8, 3, 2, 16, true, 128>(a, xrows, stream);
    if (narrow == 0) return sb::launch_nv<64, 3, 4, 4, 2, 8, false, 128>(a, xrows, stream);
    return sb::launch_nv<64, 3, 4, 2, 3, 8, false, 128>(a, xrows, stream);
  }
  if (window_cols != 64) return cudaErrorInvalidValue;
  if (block_rows == 64) {
    // d <= 48: 4-lane groups x 3 float4, 8 consumer warps x 8 rows, the warp's
    // 8 rows in parallel (one per group), 3 CTAs per SM
    if (d > 32 && d <= 48 && narrow == 2) return sb::launch_nv<64, 2, 8, 4, 2, 16, true>(a, xrows, stream);
    if (d > 32 && d <= 48 && narrow == 3) return sb::launch_nv<64, 2, 8, 4, 3, 8, true>(a, xrows, stream);
    if (d <= 48 && (narrow == 1 || narrow == 4)) return sb::launch_nv<64, 3, 4, 4, 3, 8>(a, xrows, stream);
    if (d <= 64) return sb::launch_nv<64, 2, 8, 4, 2>(a, xrows, stream);   // 4 rows of a warp in parallel
    if (d <= 128) return sb::launch_nv<64, 1, 32, 5, 1>(a, xrows, stream);
    return sb::launch_nv<64, 2, 32, 3, 1>(a, xrows, stream);              // 256-column panels
  }
  if (block_rows == 120) {
    // 30 consumer warps x 4 rows (64 registers, two records in flight): the
    // staged X window serves 120 rows, so its TMA writes into shared memory
    // cost 0.53x of a 64-row block's per nonzero
    if (d <= 128) return sb::launch_nv<120, 1, 32, 5, 1, 30>(a, xrows, stream);
    return sb::launch_nv<120, 2, 32, 3, 1, 30>(a, xrows, stream);
  }
  if (block_rows != 128) return cudaErrorInvalidValue;
  // 128-row blocks: 8 rows per warp; a TMA-staged X window serves twice the
  // rows (half the window writes into shared memory per nonzero).  256-column
  // panels with two records in flight per warp (register budget), 128-column
  // panels for d <= 128
  if (d <= 64) return sb::launch_nv<128, 2, 8, 4, 2>(a, xrows, stream);
  if (d <= 128 || g_bin_wide128 == 0) return sb::launch_nv<128, 1, 32, 5, 1>(a, xrows, stream);
  return sb::launch_nv<128, 2, 32, 3, 1>(a, xrows, stream);
}

}  // namespace hb
