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
#include <cstdlib>
#include <algorithm>
#include "common.cuh"

namespace hb {

constexpr int kSpWarps = 8;

// L2 residency: the row-gather kernel's hit rate depends on the local X rows
// of the community being aggregated staying in L2.  Everything read or written
// once — CSR entries, Y, and the halo rows (columns >= stream_col: copies of
// remote boundary nodes, each referenced by a handful of cut edges) — is
// marked evict-first so it does not push those rows out.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_f4_hint(const float4* a, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(a), "l"(pol));
  return r;
}
__device__ __forceinline__ int ld_i32_hint(const int32_t* a, uint64_t pol) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(a), "l"(pol));
  return r;
}
__device__ __forceinline__ float ld_f32_hint(const float* a, uint64_t pol) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(a), "l"(pol));
  return r;
}

// NV float4 per lane, G lanes per nonzero group (32/G groups share a warp and
// walk interleaved nonzeros of the row), U nonzeros per group per step (loads
// in flight).  Narrow rows (d <= 64) put 2-4 nonzeros in one warp instruction;
// wide rows keep G = 32.  The groups' partial sums are combined with a
// butterfly at the end of the row.
template <int NV, int G, int U>
__global__ void __launch_bounds__(kSpWarps * 32)
spmm_rows_vec_kernel(int nrows, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                     const float* __restrict__ vals, const float* __restrict__ X, int64_t ldx, int d,
                     float* __restrict__ Y, int64_t ldy, int stream_col, int hint, int* __restrict__ next_row,
                     int chunk) {
  constexpr int NG = 32 / G;
  const uint64_t pf = policy_evict_first();
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  const int warp_global = blockIdx.x * kSpWarps + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * kSpWarps;
  // Rows are handed out in ascending chunks from a global counter, so all
  // warps stay within a narrow band of rows: the X rows of the community being
  // aggregated stay L2-resident.  (A fixed grid-stride split lets warps drift
  // apart by several communities over the launch and multiplies HBM reads.)
  int r0 = 0, r1 = 0, row = warp_global;
  for (;;) {
    if (next_row) {
      if (row >= r1) {
        int got = 0;
        if (lane == 0) got = atomicAdd(next_row, chunk);
        r0 = __shfl_sync(0xffffffffu, got, 0);
        if (r0 >= nrows) {
          // the last warp out re-arms the counter for the next launch on this stream
          if (lane == 0 && atomicAdd(next_row + 1, 1) == nwarps - 1) {
            atomicExch(next_row, 0);
            atomicExch(next_row + 1, 0);
          }
          break;
        }
        r1 = min(nrows, r0 + chunk);
        row = r0;
      }
    } else if (row >= nrows) {
      break;
    }
    const int64_t start = row_ptr[row], end = row_ptr[row + 1];
    float4 acc[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t base = start; base < end; base += 32) {
      const int64_t k = base + lane;
      int my_c = 0;
      float my_v = 0.f;
      if (k < end) {
        if (hint) {
          my_c = ld_i32_hint(col_idx + k, pf);
          my_v = ld_f32_hint(vals + k, pf);
        } else {
          my_c = __ldg(col_idx + k);
          my_v = __ldg(vals + k);
        }
      }
      const int n = (int)min((int64_t)32, end - base);
      for (int jj = 0; jj < n; jj += NG * U) {
        int c[U];
        float v[U];
        bool live[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = jj + u * NG + grp;          // j < 32 always (jj < n <= 32, steps of NG*U | 32)
          c[u] = __shfl_sync(0xffffffffu, my_c, j & 31);
          v[u] = __shfl_sync(0xffffffffu, my_v, j & 31);
          live[u] = j < n;                          // padding slots issue no load
        }
        float4 x[U][NV];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float4* xr = reinterpret_cast<const float4*>(X + (int64_t)c[u] * ldx);
          const bool once = hint && c[u] >= stream_col;
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            const int col = (q * G + gl) * 4;
            x[u][q] = (col >= d || !live[u]) ? make_float4(0.f, 0.f, 0.f, 0.f)
                      : once ? ld_f4_hint(xr + q * G + gl, pf)
                             : __ldg(xr + q * G + gl);
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
          if (hint)
            __stcs(reinterpret_cast<float4*>(y + col), acc[q]);
          else
            *reinterpret_cast<float4*>(y + col) = acc[q];
        } else if (col < d) {
          y[col] = acc[q].x;
          if (col + 1 < d) y[col + 1] = acc[q].y;
          if (col + 2 < d) y[col + 2] = acc[q].z;
        }
      }
    }
    row = next_row ? row + 1 : row + nwarps;
  }
}

// Row-parallel variant: each group of G lanes owns one row (32/G rows of a
// warp in flight at once, no cross-group reduction).  The group reads its
// row's (col, val) pairs G at a time with one coalesced load and broadcasts
// them with width-G shuffles; U X rows in flight per group.  Rows come from
// the same ascending chunk counter as spmm_rows_vec_kernel.
template <int NV, int G, int U>
__global__ void __launch_bounds__(kSpWarps * 32)
spmm_rows_par_kernel(int nrows, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                     const float* __restrict__ vals, const float* __restrict__ X, int64_t ldx, int d,
                     float* __restrict__ Y, int64_t ldy, int* __restrict__ next_row, int chunk) {
  constexpr int NG = 32 / G;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (grp * G);
  const int nwarps = gridDim.x * kSpWarps;
  int r0 = 0, r1 = 0;
  for (;;) {
    int got = 0;
    if (lane == 0) got = atomicAdd(next_row, chunk);
    r0 = __shfl_sync(0xffffffffu, got, 0);
    if (r0 >= nrows) {
      if (lane == 0 && atomicAdd(next_row + 1, 1) == nwarps - 1) {
        atomicExch(next_row, 0);
        atomicExch(next_row + 1, 0);
      }
      break;
    }
    r1 = min(nrows, r0 + chunk);
    for (int row = r0 + grp; row < r1; row += NG) {
      const int64_t start = row_ptr[row], end = row_ptr[row + 1];
      float4 acc[NV];
#pragma unroll
      for (int q = 0; q < NV; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int64_t base = start; base < end; base += G) {
        const int64_t k = base + gl;
        const int my_c = k < end ? __ldg(col_idx + k) : 0;
        const float my_v = k < end ? __ldg(vals + k) : 0.f;
        const int n = (int)min((int64_t)G, end - base);
        for (int jj = 0; jj < n; jj += U) {
          int c[U];
          float v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            c[u] = __shfl_sync(gmask, my_c, (jj + u) % G, G);
            v[u] = __shfl_sync(gmask, my_v, (jj + u) % G, G);
          }
          float4 x[U][NV];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const float4* xr = reinterpret_cast<const float4*>(X + (int64_t)c[u] * ldx);
#pragma unroll
            for (int q = 0; q < NV; ++q) {
              const int col = (q * G + gl) * 4;
              x[u][q] = (col >= d || jj + u >= n) ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldg(xr + q * G + gl);
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
// `work`: caller-provided pair of ints {next work item, workers finished},
// zero on entry, left at zero by the last worker out (so one pair serves every
// launch on a stream, graph replays included).  NULL: static grid-stride rows.
cudaError_t launch_spmm(int nrows, const int64_t* row_ptr, const int32_t* col_idx, const float* vals,
                        const float* X, int64_t ldx, int d, float* Y, int64_t ldy, int64_t nnz, int algo,
                        int window, int stream_col, int* work, cudaStream_t st) {
  (void)nnz;
  (void)algo;
  if (nrows <= 0 || d <= 0) return cudaSuccess;
  const int want = (nrows + kSpWarps - 1) / kSpWarps;
  const int cap = num_sms() * 8;
  const int grid = want < cap ? want : cap;
  const bool vec = (ldx % 4 == 0) && (ldy % 4 == 0) && ((((uintptr_t)X) & 15) == 0) &&
                   ((((uintptr_t)Y) & 15) == 0);
  static const int hint = getenv("HB_SPMM_HINT") ? atoi(getenv("HB_SPMM_HINT")) : 0;
  static const int dyn_env = getenv("HB_SPMM_DYN") ? atoi(getenv("HB_SPMM_DYN")) : 1;
  const int dyn = dyn_env && work != nullptr;
  static const int chunk_env = getenv("HB_SPMM_CHUNK") ? atoi(getenv("HB_SPMM_CHUNK")) : 0;
  int* next_row = nullptr;
  int chunk = 1;
  if (dyn) {
    next_row = work;
    // ~192 nonzeros per grab
    const int64_t avg = nnz > 0 ? (nnz + nrows - 1) / nrows : 32;
    chunk = chunk_env > 0 ? chunk_env : (int)std::max<int64_t>(1, std::min<int64_t>(32, 192 / std::max<int64_t>(1, avg)));
  }
  static const int par = getenv("HB_SPMM_PAR") ? atoi(getenv("HB_SPMM_PAR")) : 1;
  if (vec && dyn && par && d <= 128) {
    // row-parallel lane groups (chunks rounded to whole groups of rows)
    const int ch = (chunk + 3) & ~3;
    // d <= 64: 8-lane groups x 2 float4, 4 rows in flight per group; 64 < d <=
    // 128: 8-lane groups x 4 float4, 2 in flight (17.5 TB/s gathered on the
    // ogbn 128-wide operator, the raw L2 gather ceiling; 16-lane groups x 2
    // float4: 16.5; profiles/r2_kbench_ogbn_rows.txt)
    if (d <= 64) spmm_rows_par_kernel<2, 8, 4><<<grid, kSpWarps * 32, 0, st>>>(nrows, row_ptr, col_idx, vals, X, ldx, d, Y, ldy, next_row, ch);
    else spmm_rows_par_kernel<4, 8, 2><<<grid, kSpWarps * 32, 0, st>>>(nrows, row_ptr, col_idx, vals, X, ldx, d, Y, ldy, next_row, ch);
    return cudaGetLastError();
  }
  if (vec && d <= 1024) {
    const int d4 = (d + 3) / 4;
#define HB_S(NV, G, U) spmm_rows_vec_kernel<NV, G, U><<<grid, kSpWarps * 32, 0, st>>>(nrows, row_ptr, col_idx, vals, X, ldx, d, Y, ldy, stream_col, hint, next_row, chunk)
    if (d4 <= 8) HB_S(1, 8, 8);
    else if (d4 <= 16) {
      // 4 nonzeros in flight per 16-lane group (8 per warp) and more resident
      // warps beat deeper per-group windows on both short and long rows
      const int w = window > 0 ? window : 4;
      if (w == 4) HB_S(1, 16, 4);
      else if (w == 8) HB_S(1, 16, 8);
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
      case 3:   // Yelp's 300-wide layer-1 operator: 4 nonzeros in flight 1.44 ms, 1 in flight 1.60
                // (profiles/r2_kbench_yelp_rows.txt)
        if (window == 1) HB_S(3, 32, 1);
        else if (window == 2) HB_S(3, 32, 2);
        else HB_S(3, 32, 4);
        break;
      case 4:
        if (window == 1) HB_S(4, 32, 1);
        else if (window == 2) HB_S(4, 32, 2);
        else HB_S(4, 32, 4);
        break;
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
