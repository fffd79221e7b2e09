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

// algo: 0 auto, 1 row gather (the same kernel: the TMA-tiled path is a
// separate entry point, hb_spmm_tiled).  `window` > 0 overrides the number of
// nonzeros a lane group keeps in flight (tuning only).
cudaError_t launch_spmm(int nrows, const int64_t* row_ptr, const int32_t* col_idx, const float* vals,
                        const float* X, int64_t ldx, int d, float* Y, int64_t ldy, int64_t nnz, int algo,
                        int window, cudaStream_t st) {
  (void)nnz;
  (void)algo;
  if (nrows <= 0 || d <= 0) return cudaSuccess;
  const int want = (nrows + kSpWarps - 1) / kSpWarps;
  const int cap = num_sms() * 8;
  const int grid = want < cap ? want : cap;
  const bool vec = (ldx % 4 == 0) && (ldy % 4 == 0) && ((((uintptr_t)X) & 15) == 0) &&
                   ((((uintptr_t)Y) & 15) == 0);
  if (vec && d <= 1024) {
    const int d4 = (d + 3) / 4;
#define HB_S(NV, G, U) spmm_rows_vec_kernel<NV, G, U><<<grid, kSpWarps * 32, 0, st>>>(nrows, row_ptr, col_idx, vals, X, ldx, d, Y, ldy)
    if (d4 <= 8) HB_S(1, 8, 8);
    else if (d4 <= 16) {
      if (window == 4) HB_S(1, 16, 4);
      else if (window == 8) HB_S(1, 16, 8);
      else HB_S(1, 16, 16);
    }
    else switch ((d4 + 31) / 32) {
      case 1: HB_S(1, 32, 8); break;
      case 2:
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
