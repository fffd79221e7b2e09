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

template <int NV>
__global__ void __launch_bounds__(kSpWarps * 32)
spmm_rows_vec_kernel(int nrows, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                     const float* __restrict__ vals, const float* __restrict__ X, int64_t ldx, int d,
                     float* __restrict__ Y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
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
      int jj = 0;
      for (; jj + 2 <= n; jj += 2) {
        const int c0 = __shfl_sync(0xffffffffu, my_c, jj);
        const float v0 = __shfl_sync(0xffffffffu, my_v, jj);
        const int c1 = __shfl_sync(0xffffffffu, my_c, jj + 1);
        const float v1 = __shfl_sync(0xffffffffu, my_v, jj + 1);
        const float4* x0 = reinterpret_cast<const float4*>(X + (int64_t)c0 * ldx);
        const float4* x1 = reinterpret_cast<const float4*>(X + (int64_t)c1 * ldx);
        float4 a[NV], b[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          const int col = (q * 32 + lane) * 4;
          if (col < d) { a[q] = __ldg(x0 + q * 32 + lane); b[q] = __ldg(x1 + q * 32 + lane); }
        }
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          const int col = (q * 32 + lane) * 4;
          if (col < d) {
            acc[q].x = fmaf(v0, a[q].x, acc[q].x); acc[q].y = fmaf(v0, a[q].y, acc[q].y);
            acc[q].z = fmaf(v0, a[q].z, acc[q].z); acc[q].w = fmaf(v0, a[q].w, acc[q].w);
            acc[q].x = fmaf(v1, b[q].x, acc[q].x); acc[q].y = fmaf(v1, b[q].y, acc[q].y);
            acc[q].z = fmaf(v1, b[q].z, acc[q].z); acc[q].w = fmaf(v1, b[q].w, acc[q].w);
          }
        }
      }
      if (jj < n) {
        const int c0 = __shfl_sync(0xffffffffu, my_c, jj);
        const float v0 = __shfl_sync(0xffffffffu, my_v, jj);
        const float4* x0 = reinterpret_cast<const float4*>(X + (int64_t)c0 * ldx);
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          const int col = (q * 32 + lane) * 4;
          if (col < d) {
            const float4 a = __ldg(x0 + q * 32 + lane);
            acc[q].x = fmaf(v0, a.x, acc[q].x); acc[q].y = fmaf(v0, a.y, acc[q].y);
            acc[q].z = fmaf(v0, a.z, acc[q].z); acc[q].w = fmaf(v0, a.w, acc[q].w);
          }
        }
      }
    }
    float* y = Y + (int64_t)row * ldy;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int col = (q * 32 + lane) * 4;
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

cudaError_t launch_spmm(int nrows, const int64_t* row_ptr, const int32_t* col_idx, const float* vals,
                        const float* X, int64_t ldx, int d, float* Y, int64_t ldy, cudaStream_t st) {
  if (nrows <= 0 || d <= 0) return cudaSuccess;
  const int want = (nrows + kSpWarps - 1) / kSpWarps;
  const int cap = num_sms() * 8;
  const int grid = want < cap ? want : cap;
  const bool vec = (ldx % 4 == 0) && (ldy % 4 == 0) && ((((uintptr_t)X) & 15) == 0) &&
                   ((((uintptr_t)Y) & 15) == 0);
  if (vec && d <= 1024) {
    const int nv = (d + 127) / 128;
#define HB_S(N) spmm_rows_vec_kernel<N><<<grid, kSpWarps * 32, 0, st>>>(nrows, row_ptr, col_idx, vals, X, ldx, d, Y, ldy)
    switch (nv) {
      case 1: HB_S(1); break;
      case 2: HB_S(2); break;
      case 3: HB_S(3); break;
      case 4: HB_S(4); break;
      case 5: HB_S(5); break;
      case 6: HB_S(6); break;
      case 7: HB_S(7); break;
      default: HB_S(8); break;
    }
#undef HB_S
  } else {
    spmm_rows_scalar_kernel<<<grid, kSpWarps * 32, 0, st>>>(nrows, row_ptr, col_idx, vals, X, ldx, d, Y, ldy);
  }
  return cudaGetLastError();
}

}  // namespace hb
