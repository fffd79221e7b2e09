// K3/K4: CSR SpMM  Y = A * X  (reference linalg.spmm, linalg.py:71-75, used at
// trainer.py:291,293 for the aggregation and trainer.py:318,321 with the
// precomputed transposed block for the backward).
//
// One warp per output row.  The warp reads 32 (col, val) pairs with one
// coalesced load, then walks them with register shuffles; each nonzero
// gathers one X row as 128-bit loads (lane j owns columns 128q + 4j..+3).
// Accumulation is fp32 in index order (the reference sums in index order in
// f64).  The kernel is HBM/L2-gather bound: algorithmic bytes per launch are
// 8(n+1) + 8 nnz + 4 nnz d + 4 n d.
#include <cuda_runtime.h>
#include <cstdint>
#include "common.cuh"

namespace hb {

constexpr int kSpWarps = 8;

// NV float4 per lane, G lanes per nonzero group (32/G groups share a warp and
// walk interleaved nonzeros of the row), U nonzeros per group per step (loads
// in flight).  Narrow rows (d <= 64) put 2-4 nonzeros in one warp instruction;
// wide rows keep G = 32.  The groups' partial sums are combined with a
// butterfly at the end of the row.
template <int NV, int G, int U>
__global__ void __launch_bounds__(kSpWarps * 32)
spmm_rows_vec_kernel(int nrows, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                     const float* __restrict__ vals, const float* __restrict__ X, int64_t ldx, int d,
                     float* __restrict__ Y, int64_t ldy) {
  constexpr int NG = 32 / G;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  const int warp_global = blockIdx.x * kSpWarps + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * kSpWarps;
  for (int row = warp_global; row < nrows; row += nwarps) {
    const int64_t start = row_ptr[row], end = row_ptr[row + 1];
    float4 acc[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t base = start; base < end; base += 32) {
      const int64_t k = base + lane;
      const int my_c = k < end ? __ldg(col_idx + k) : 0;
      const float my_v = k < end ? __ldg(vals + k) : 0.f;
      const int n = (int)min((int64_t)32, end - base);
      for (int jj = 0; jj < n; jj += NG * U) {
        int c[U];
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = jj + u * NG + grp;          // j < 32 always (jj < n <= 32, steps of NG*U | 32)
          c[u] = __shfl_sync(0xffffffffu, my_c, j & 31);
          v[u] = __shfl_sync(0xffffffffu, my_v, j & 31);
          if (j >= n) v[u] = 0.f;                   // padding nonzero: row my_c of lane j (valid), weight 0
        }
        float4 x[U][NV];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float4* xr = reinterpret_cast<const float4*>(X + (int64_t)c[u] * ldx);
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            const int col = (q * G + gl) * 4;
            x[u][q] = col < d ? __ldg(xr + q * G + gl) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            acc[q].x = fmaf(v[u], x[u][q].x, acc[q].x); acc[q].y = fmaf(v[u], x[u][q].y, acc[q].y);
            acc[q].z = fmaf(v[u], x[u][q].z, acc[q].z); acc[q].w = fmaf(v[u], x[u][q].w, acc[q].w);
          }
      }
    }
#pragma unroll
    for (int off = G; off < 32; off <<= 1)
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        acc[q].x += __shfl_xor_sync(0xffffffffu, acc[q].x, off);
        acc[q].y += __shfl_xor_sync(0xffffffffu, acc[q].y, off);
        acc[q].z += __shfl_xor_sync(0xffffffffu, acc[q].z, off);
        acc[q].w += __shfl_xor_sync(0xffffffffu, acc[q].w, off);
      }
    if (grp == 0) {
      float* y = Y + (int64_t)row * ldy;
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const int col = (q * G + gl) * 4;
        if (col + 3 < d) {
          *reinterpret_cast<float4*>(y + col) = acc[q];
        } else if (col < d) {
          y[col] = acc[q].x;
          if (col + 1 < d) y[col + 1] = acc[q].y;
          if (col + 2 < d) y[col + 2] = acc[q].z;
        }
      }
    }
  }
}

// Column-sweep SpMM for long rows (K3/K4 on community-structured blocks).
// A CTA owns RB = 8*RW consecutive rows (RW per warp) and walks all of their
// nonzeros in lockstep column windows [w0, w0 + W): within a window each X row
// is pulled from L2 by the first row that needs it and served from L1 to the
// other rows of the block (the 8 warps advance window by window behind a CTA
// barrier; empty column ranges are skipped by a CTA-wide min of the rows' next
// columns).  W is sized so a window of X rows fits in L1 next to the other
// resident CTA.  Blocks whose rows are short (< kSweepMinAvg nonzeros on
// average) skip the windows and gather row by row.  Accumulation per row is
// fp32 in index order, like the row kernel.
constexpr int kSweepMinAvg = 16;

template <int NV, int RW, int U>
__device__ __forceinline__ void sweep_chunk(const float* __restrict__ X, int64_t ldx, int d, int lane, int c,
                                            float v, int n, float4 (&acc)[NV]) {
  for (int jj = 0; jj < n; jj += U) {
    int cc[U];
    float vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = jj + u;
      cc[u] = __shfl_sync(0xffffffffu, c, j < n ? j : 0);
      vv[u] = __shfl_sync(0xffffffffu, v, j < n ? j : 0);
      if (j >= n) vv[u] = 0.f;
    }
    float4 x[U][NV];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float4* xr = reinterpret_cast<const float4*>(X + (int64_t)cc[u] * ldx);
#pragma unroll
      for (int q = 0; q < NV; ++q)
        x[u][q] = (q * 32 + lane) * 4 < d ? __ldg(xr + q * 32 + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        acc[q].x = fmaf(vv[u], x[u][q].x, acc[q].x); acc[q].y = fmaf(vv[u], x[u][q].y, acc[q].y);
        acc[q].z = fmaf(vv[u], x[u][q].z, acc[q].z); acc[q].w = fmaf(vv[u], x[u][q].w, acc[q].w);
      }
  }
}

template <int NV, int RW, int U>
__global__ void __launch_bounds__(kSpWarps * 32, 2)
spmm_sweep_kernel(int nrows, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                  const float* __restrict__ vals, const float* __restrict__ X, int64_t ldx, int d,
                  float* __restrict__ Y, int64_t ldy, int W) {
  constexpr int RB = kSpWarps * RW;
  constexpr int NONE = 0x7fffffff;
  __shared__ int wmin[2][kSpWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nblocks = (nrows + RB - 1) / RB;
  int flip = 0;
  for (int blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
    const int r0 = blk * RB + warp * RW;
    const int rb_end = min(nrows, (blk + 1) * RB);
    const int64_t blk_nnz = row_ptr[rb_end] - row_ptr[blk * RB];
    int64_t pos[RW], end[RW];
#pragma unroll
    for (int i = 0; i < RW; ++i) {
      const int r = r0 + i;
      pos[i] = r < nrows ? row_ptr[r] : 0;
      end[i] = r < nrows ? row_ptr[r + 1] : 0;
    }
    float4 acc[RW][NV];
#pragma unroll
    for (int i = 0; i < RW; ++i)
#pragma unroll
      for (int q = 0; q < NV; ++q) acc[i][q] = make_float4(0.f, 0.f, 0.f, 0.f);

    if (blk_nnz < (int64_t)kSweepMinAvg * (rb_end - blk * RB)) {
      // short rows: plain row gather, no windows
#pragma unroll
      for (int i = 0; i < RW; ++i) {
        for (int64_t base = pos[i]; base < end[i]; base += 32) {
          const int64_t k = base + lane;
          const int c = k < end[i] ? __ldg(col_idx + k) : 0;
          const float v = k < end[i] ? __ldg(vals + k) : 0.f;
          sweep_chunk<NV, RW, U>(X, ldx, d, lane, c, v, (int)min((int64_t)32, end[i] - base), acc[i]);
        }
      }
    } else {
      int mymin = NONE;
#pragma unroll
      for (int i = 0; i < RW; ++i)
        if (pos[i] < end[i]) mymin = min(mymin, __ldg(col_idx + pos[i]));
      if (lane == 0) wmin[flip][warp] = mymin;
      __syncthreads();
      int w0 = NONE;
#pragma unroll
      for (int w = 0; w < kSpWarps; ++w) w0 = min(w0, wmin[flip][w]);
      flip ^= 1;
      while (w0 != NONE) {
        const int wend = w0 > NONE - W ? NONE : w0 + W;
        mymin = NONE;
#pragma unroll
        for (int i = 0; i < RW; ++i) {
          while (pos[i] < end[i]) {
            const int64_t k = pos[i] + lane;
            const int c = k < end[i] ? __ldg(col_idx + k) : NONE;
            const float v = k < end[i] ? __ldg(vals + k) : 0.f;
            const int n = __popc(__ballot_sync(0xffffffffu, c < wend));   // columns sorted: a prefix
            sweep_chunk<NV, RW, U>(X, ldx, d, lane, c, v, n, acc[i]);
            pos[i] += n;
            if (n < 32) {
              const int nc = __shfl_sync(0xffffffffu, c, n & 31);
              if (pos[i] < end[i]) mymin = min(mymin, nc);
              break;
            }
          }
        }
        if (lane == 0) wmin[flip][warp] = mymin;
        __syncthreads();
        w0 = NONE;
#pragma unroll
        for (int w = 0; w < kSpWarps; ++w) w0 = min(w0, wmin[flip][w]);
        flip ^= 1;
      }
    }
#pragma unroll
    for (int i = 0; i < RW; ++i) {
      const int r = r0 + i;
      if (r >= nrows) continue;
      float* y = Y + (int64_t)r * ldy;
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const int col = (q * 32 + lane) * 4;
        if (col + 3 < d) {
          *reinterpret_cast<float4*>(y + col) = acc[i][q];
        } else if (col < d) {
          y[col] = acc[i][q].x;
          if (col + 1 < d) y[col + 1] = acc[i][q].y;
          if (col + 2 < d) y[col + 2] = acc[i][q].z;
        }
      }
    }
  }
}

template <int NV, int RW, int U>
static void launch_sweep(int nrows, const int64_t* row_ptr, const int32_t* col_idx, const float* vals,
                         const float* X, int64_t ldx, int d, float* Y, int64_t ldy, int window, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {   // favour L1 over shared memory: the windows live in L1
    cudaFuncSetAttribute(spmm_sweep_kernel<NV, RW, U>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    attr = true;
  }
  constexpr int RB = kSpWarps * RW;
  const int nblocks = (nrows + RB - 1) / RB;
  const int cap = num_sms() * 2;
  const int grid = nblocks < cap ? nblocks : cap;
  int W = window;
  if (W <= 0) {
    W = (int)((64 * 1024) / (ldx * 4));   // ~64 KB of X rows per window (2 CTAs per SM)
    if (W < 16) W = 16;
  }
  spmm_sweep_kernel<NV, RW, U><<<grid, kSpWarps * 32, 0, st>>>(nrows, row_ptr, col_idx, vals, X, ldx, d, Y, ldy, W);
}

// Generic (unaligned leading dimensions): scalar columns, lane-strided.
__global__ void __launch_bounds__(kSpWarps * 32)
spmm_rows_scalar_kernel(int nrows, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                        const float* __restrict__ vals, const float* __restrict__ X, int64_t ldx, int d,
                        float* __restrict__ Y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int warp_global = blockIdx.x * kSpWarps + (threadIdx.x >> 5);
  for (int row = warp_global; row < nrows; row += gridDim.x * kSpWarps) {
    const int64_t start = row_ptr[row], end = row_ptr[row + 1];
    for (int cb = 0; cb < d; cb += 256) {
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int64_t k = start; k < end; ++k) {
        const int c = __ldg(col_idx + k);
        const float v = __ldg(vals + k);
        const float* xr = X + (int64_t)c * ldx;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int col = cb + e * 32 + lane;
          if (col < d) acc[e] = fmaf(v, __ldg(xr + col), acc[e]);
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int col = cb + e * 32 + lane;
        if (col < d) Y[(int64_t)row * ldy + col] = acc[e];
      }
    }
  }
}

// algo: 0 auto (column sweep when rows average >= 32 nonzeros and d > 64),
// 1 row gather, 2 column sweep (d > 64 only; else row gather).
cudaError_t launch_spmm(int nrows, const int64_t* row_ptr, const int32_t* col_idx, const float* vals,
                        const float* X, int64_t ldx, int d, float* Y, int64_t ldy, int64_t nnz, int algo,
                        int window, cudaStream_t st) {
  if (nrows <= 0 || d <= 0) return cudaSuccess;
  const int want = (nrows + kSpWarps - 1) / kSpWarps;
  const int cap = num_sms() * 8;
  const int grid = want < cap ? want : cap;
  const bool vec = (ldx % 4 == 0) && (ldy % 4 == 0) && ((((uintptr_t)X) & 15) == 0) &&
                   ((((uintptr_t)Y) & 15) == 0);
  const int d4 = (d + 3) / 4;
  const bool sweep = vec && d4 > 16 && d <= 1024 &&
                     (algo == 2 || (algo == 0 && nnz >= 0 && nnz >= (int64_t)32 * nrows));
  if (sweep) {
#define HB_W(NV, RW, U) launch_sweep<NV, RW, U>(nrows, row_ptr, col_idx, vals, X, ldx, d, Y, ldy, window, st)
    switch ((d4 + 31) / 32) {
      case 1: HB_W(1, 8, 4); break;
      case 2: HB_W(2, 8, 2); break;
      case 3: HB_W(3, 4, 2); break;
      case 4: HB_W(4, 4, 2); break;
      case 5: HB_W(5, 2, 2); break;
      case 6: HB_W(6, 2, 2); break;
      case 7: HB_W(7, 2, 1); break;
      default: HB_W(8, 2, 1); break;
    }
#undef HB_W
    return cudaGetLastError();
  }
  if (vec && d <= 1024) {
    const int d4 = (d + 3) / 4;
#define HB_S(NV, G, U) spmm_rows_vec_kernel<NV, G, U><<<grid, kSpWarps * 32, 0, st>>>(nrows, row_ptr, col_idx, vals, X, ldx, d, Y, ldy)
    if (d4 <= 8) HB_S(1, 8, 8);
    else if (d4 <= 16) {   // `window` doubles as an unroll override (tuning only)
      if (window == 4) HB_S(1, 16, 4);
      else if (window == 8) HB_S(1, 16, 8);
      else HB_S(1, 16, 16);
    }
    else switch ((d4 + 31) / 32) {
      case 1: HB_S(1, 32, 8); break;
      case 2:   // `window` doubles as an unroll override for the row kernel (tuning only)
        if (window == 1) HB_S(2, 32, 1);
        else if (window == 2) HB_S(2, 32, 2);
        else if (window == 8) HB_S(2, 32, 8);
        else HB_S(2, 32, 4);
        break;
      case 3: HB_S(3, 32, 2); break;
      case 4: HB_S(4, 32, 2); break;
      case 5: HB_S(5, 32, 2); break;
      case 6: HB_S(6, 32, 2); break;
      case 7: HB_S(7, 32, 2); break;
      default: HB_S(8, 32, 2); break;
    }
#undef HB_S
  } else {
    spmm_rows_scalar_kernel<<<grid, kSpWarps * 32, 0, st>>>(nrows, row_ptr, col_idx, vals, X, ldx, d, Y, ldy);
  }
  return cudaGetLastError();
}

}  // namespace hb
