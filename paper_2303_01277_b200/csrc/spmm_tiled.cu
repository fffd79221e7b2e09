// K3/K4 tiled path: CSR SpMM with TMA staging of X tiles in shared memory.
//
//   Y[i, :] = sum_k A[i, k] X[k, :]      (linalg.spmm, linalg.py:71-75)
//
// The matrix is pre-split (once, on the device: ops.TiledCsr) into
//   * dense tiles: (row block of kTRB rows) x (column window of kTW columns)
//     holding >= a threshold of nonzeros, stored as row-sorted (col - c0, val)
//     records plus kTRB+1 row offsets per tile;
//   * a residual CSR with every other nonzero.
// A persistent CTA takes (row block, feature panel) work items in ascending
// order from a global counter (dynamic: the CTAs finish within one item of
// each other, and all of them work on neighbouring row blocks, whose X windows
// share L2), passed from the producer warp to the consumers through a small
// smem queue.  A producer
// warp streams the block's tiles through a 2-stage smem ring: one TMA 2-D
// box load of the X window (kTW rows x panel columns) plus two bulk copies of
// the tile's records and row offsets, all completing on one mbarrier.  Sixteen
// consumer warps own 4 rows each (register accumulators, lane = 4 columns of
// the panel per float4) and read X rows from smem, so a staged X row is
// reused by every row of the block that touches it instead of being gathered
// from L2 once per nonzero.  Residual nonzeros are gathered from global X
// (the row kernel's access pattern) before the block's rows are stored.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdlib>
#include "common.cuh"

namespace hb {
namespace st {

constexpr int kTRB = 64;         // rows per block (16 consumer warps x 4 rows)
constexpr int kTW = 64;          // columns per window
constexpr int kRowOff = 72;      // row offsets per tile (65 used, padded to 144 bytes)
constexpr int kRPW = 4;          // rows per consumer warp
constexpr int kMaxRec = 1024;    // records per tile (ops.TiledCsr splits denser tiles)
constexpr int kConsumers = kTRB / kRPW;
constexpr int kThreads = 32 * (kConsumers + 1);
constexpr int kQ = 4;            // work-item queue depth (producer -> consumers)

struct Args {
  int nrows, nblocks, npanels, d;
  int* next_item;                // {next item, CTAs finished}: caller's self-resetting counter pair
  int pw;                        // staged panel width (floats): min(P, d rounded up to 4)
  const int32_t* tile_ptr;       // [nblocks + 1]
  const int32_t* tile_win;       // [ntiles]
  const int64_t* tile_off;       // [ntiles + 1] record offsets (even: 16-byte aligned)
  const uint16_t* tile_rowoff;   // [ntiles][kRowOff]
  const int2* tile_nz;           // (col - c0, float bits of val)
  const int64_t* res_ptr;        // residual CSR
  const int32_t* res_col;
  const float* res_val;
  const float* X;
  int64_t ldx;
  float* Y;
  int64_t ldy;
};

// NV float4 per lane, G lanes per record group (32, or 16 for d <= 64 so two
// records go through one warp instruction), S pipeline stages.
template <int NV, int G, int S>
struct Smem {
  static constexpr int P = 4 * G * NV;                   // panel width (floats)
  static constexpr int X_BYTES = kTW * P * 4;
  static constexpr int NZ_BYTES = kMaxRec * 8;
  static constexpr int RO_BYTES = kRowOff * 2;
  static constexpr int STAGE = X_BYTES + NZ_BYTES + 256;
  static constexpr int TOTAL = S * STAGE + 128;
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
__device__ __forceinline__ void fma_row(float4 (&acc)[NV], float v, const float4* __restrict__ x) {
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const float4 t = x[q * G];
    acc[q].x = fmaf(v, t.x, acc[q].x); acc[q].y = fmaf(v, t.y, acc[q].y);
    acc[q].z = fmaf(v, t.z, acc[q].z); acc[q].w = fmaf(v, t.w, acc[q].w);
  }
}

template <int NV, int G, int S, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
spmm_tiled_kernel(const __grid_constant__ CUtensorMap tmX, Args a) {
  using S_ = Smem<NV, G, S>;
  constexpr int P = S_::P;
  constexpr int NG = 32 / G;
  extern __shared__ uint8_t smem_raw[];
  // aligned by pointer arithmetic on the __shared__ array (an integer round
  // trip would hide the address space and turn every access generic)
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  __shared__ __align__(8) uint64_t full[S], empty[S], ifull[kQ], iempty[kQ];
  __shared__ int item_q[kQ];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hg = lane / G, gl = lane % G;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    for (int q = 0; q < kQ; ++q) {
      mbar_init(&ifull[q], 1);
      mbar_init(&iempty[q], kConsumers);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int items = a.nblocks * a.npanels;

  if (warp == kConsumers) {
    // ---------------- producer ----------------
    // one producer lane per ring stage (lane s issues every tile that lands
    // in stage s, so each barrier is still waited on in phase order by a
    // single thread): the tiles' metadata loads (tile_off / tile_win,
    // dependent global reads) are then S deep in flight ahead of the ring
    int it = 0;
    for (int qi = 0;; ++qi) {
      // lane 0 claims the next item and publishes it to the consumers
      int item = 0;
      if (lane == 0) {
        item = atomicAdd(a.next_item, 1);
        const int q = qi % kQ;
        mbar_wait(&iempty[q], ((qi / kQ) & 1) ^ 1);
        item_q[q] = item;
        mbar_arrive_cta(&ifull[q]);
        if (item >= items && atomicAdd(a.next_item + 1, 1) == (int)gridDim.x - 1) {
          atomicExch(a.next_item, 0);      // last CTA out re-arms the counter pair
          atomicExch(a.next_item + 1, 0);
        }
      }
      item = __shfl_sync(0xffffffffu, item, 0);
      if (item >= items) break;
      const int b = item / a.npanels, pn = item % a.npanels;
      const int t0 = a.tile_ptr[b], t1 = a.tile_ptr[b + 1];
      // lane s issues every tile that lands in ring stage s (each barrier is
      // waited on in phase order by a single thread); the tiles' metadata
      // loads are then S deep in flight ahead of the ring
      for (int t = t0; t < t1; ++t, ++it) {
        if (lane >= S || it % S != lane) continue;
        const int s = it % S;
        mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
        uint8_t* st = smem + s * S_::STAGE;
        const int64_t o0 = a.tile_off[t], o1 = a.tile_off[t + 1];
        const uint32_t nzb = (uint32_t)((o1 - o0) * 8);
        mbar_expect_tx(&full[s], (uint32_t)(kTW * a.pw * 4) + nzb + S_::RO_BYTES);
        tma_2d(st, &tmX, pn * P, a.tile_win[t] * kTW, &full[s]);
        if (nzb) tma_load_1d(st + S_::X_BYTES, a.tile_nz + o0, nzb, &full[s]);
        tma_load_1d(st + S_::X_BYTES + S_::NZ_BYTES, a.tile_rowoff + (int64_t)t * kRowOff, S_::RO_BYTES,
                    &full[s]);
      }
    }
    __syncwarp();
    return;
  }

  // ---------------- consumers ----------------
  int it = 0;
  const int pw4 = a.pw / 4;
  for (int qi = 0;; ++qi) {
    const int q = qi % kQ;
    mbar_wait(&ifull[q], (qi / kQ) & 1);
    const int item = item_q[q];
    __syncwarp();
    if (lane == 0) mbar_arrive_cta(&iempty[q]);
    if (item >= items) break;
    const int b = item / a.npanels, pn = item % a.npanels;
    const int r0 = b * kTRB + warp * kRPW;
    const int col0 = pn * P;
    if constexpr (G < 32 && G * NG == 32 && kRPW % NG == 0 && (G == 8 || NV >= 4)) {
      // row-parallel consumers: lane group hg (G lanes x NV float4) owns rows
      // hg, hg + NG, ... of the warp's kRPW rows outright (no cross-group
      // reduction), so the warp walks NG rows at once
      constexpr int RPG = kRPW / NG;
      float4 acc1[RPG][NV];
#pragma unroll
      for (int i = 0; i < RPG; ++i)
#pragma unroll
        for (int qv = 0; qv < NV; ++qv) acc1[i][qv] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int t = a.tile_ptr[b]; t < a.tile_ptr[b + 1]; ++t, ++it) {
        const int s = it % S;
        mbar_wait(&full[s], (it / S) & 1);
        const uint8_t* st = smem + s * S_::STAGE;
        const float4* xs = reinterpret_cast<const float4*>(st) + gl;
        const int2* nz = reinterpret_cast<const int2*>(st + S_::X_BYTES);
        const uint16_t* ro = reinterpret_cast<const uint16_t*>(st + S_::X_BYTES + S_::NZ_BYTES) + warp * kRPW;
#pragma unroll
        for (int i = 0; i < RPG; ++i) {
          const int rr = hg + i * NG;
          const int k1 = ro[rr + 1];
          int k = ro[rr];
          for (; k + 1 < k1; k += 2) {
            const int2 e0 = nz[k], e1 = nz[k + 1];
            fma_row<NV, G>(acc1[i], __int_as_float(e0.y), xs + e0.x * pw4);
            fma_row<NV, G>(acc1[i], __int_as_float(e1.y), xs + e1.x * pw4);
          }
          if (k < k1) {
            const int2 e = nz[k];
            fma_row<NV, G>(acc1[i], __int_as_float(e.y), xs + e.x * pw4);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_cta(&empty[s]);
      }
#pragma unroll
      for (int i = 0; i < RPG; ++i) {
        const int r = r0 + hg + i * NG;
        if (r >= a.nrows) continue;
        const float* Xp = a.X + col0;
        const int64_t e0 = a.res_ptr[r], e1 = a.res_ptr[r + 1];
        for (int64_t k = e0; k < e1; ++k) {
          const int c = __ldg(a.res_col + k);
          const float v = __ldg(a.res_val + k);
          const float4* xr = reinterpret_cast<const float4*>(Xp + (int64_t)c * a.ldx) + gl;
#pragma unroll
          for (int qv = 0; qv < NV; ++qv) {
            if (col0 + (qv * G + gl) * 4 < a.d) {
              const float4 t4 = __ldg(xr + qv * G);
              acc1[i][qv].x = fmaf(v, t4.x, acc1[i][qv].x); acc1[i][qv].y = fmaf(v, t4.y, acc1[i][qv].y);
              acc1[i][qv].z = fmaf(v, t4.z, acc1[i][qv].z); acc1[i][qv].w = fmaf(v, t4.w, acc1[i][qv].w);
            }
          }
        }
        float* y = a.Y + (int64_t)r * a.ldy + col0;
#pragma unroll
        for (int qv = 0; qv < NV; ++qv) {
          const int col = (qv * G + gl) * 4;
          const int rem = a.d - col0 - col;
          if (rem >= 4) {
            *reinterpret_cast<float4*>(y + col) = acc1[i][qv];
          } else if (rem > 0) {
            y[col] = acc1[i][qv].x;
            if (rem > 1) y[col + 1] = acc1[i][qv].y;
            if (rem > 2) y[col + 2] = acc1[i][qv].z;
          }
        }
      }
      continue;
    }
    float4 acc[kRPW][NV];
#pragma unroll
    for (int i = 0; i < kRPW; ++i)
#pragma unroll
      for (int q = 0; q < NV; ++q) acc[i][q] = make_float4(0.f, 0.f, 0.f, 0.f);

    for (int t = a.tile_ptr[b]; t < a.tile_ptr[b + 1]; ++t, ++it) {
      const int s = it % S;
      mbar_wait(&full[s], (it / S) & 1);
      const uint8_t* st = smem + s * S_::STAGE;
      const float4* xs = reinterpret_cast<const float4*>(st) + gl;
      const int2* nz = reinterpret_cast<const int2*>(st + S_::X_BYTES);
      const uint16_t* ro = reinterpret_cast<const uint16_t*>(st + S_::X_BYTES + S_::NZ_BYTES) + warp * kRPW;
#pragma unroll
      for (int i = 0; i < kRPW; ++i) {
        const int k1 = ro[i + 1];
        int k = ro[i] + hg;                    // group hg takes records hg, hg + NG, ...
        for (; k + 3 * NG < k1; k += 4 * NG) {
          const int2 e0 = nz[k], e1 = nz[k + NG], e2 = nz[k + 2 * NG], e3 = nz[k + 3 * NG];
          fma_row<NV, G>(acc[i], __int_as_float(e0.y), xs + e0.x * pw4);
          fma_row<NV, G>(acc[i], __int_as_float(e1.y), xs + e1.x * pw4);
          fma_row<NV, G>(acc[i], __int_as_float(e2.y), xs + e2.x * pw4);
          fma_row<NV, G>(acc[i], __int_as_float(e3.y), xs + e3.x * pw4);
        }
        for (; k < k1; k += NG) {
          const int2 e = nz[k];
          fma_row<NV, G>(acc[i], __int_as_float(e.y), xs + e.x * pw4);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&empty[s]);
    }

    // residual nonzeros: gathered from global X (group hg takes every NG-th)
    const float* Xp = a.X + col0;
#pragma unroll
    for (int i = 0; i < kRPW; ++i) {
      const int r = r0 + i;
      if (r >= a.nrows) continue;
      const int64_t e0 = a.res_ptr[r], e1 = a.res_ptr[r + 1];
      for (int64_t base = e0; base < e1; base += 32) {
        const int64_t k = base + lane;
        const int my_c = k < e1 ? __ldg(a.res_col + k) : 0;
        const float my_v = k < e1 ? __ldg(a.res_val + k) : 0.f;
        const int n = (int)min((int64_t)32, e1 - base);
        for (int j0 = 0; j0 < n; j0 += NG) {
          const int j = j0 + hg;
          const int c = __shfl_sync(0xffffffffu, my_c, j & 31);
          const float vj = __shfl_sync(0xffffffffu, my_v, j & 31);   // every lane shuffles
          const float v = j < n ? vj : 0.f;
          const float4* xr = reinterpret_cast<const float4*>(Xp + (int64_t)c * a.ldx) + gl;
#pragma unroll
          for (int q = 0; q < NV; ++q) {
            if (col0 + (q * G + gl) * 4 < a.d) {
              const float4 t4 = __ldg(xr + q * G);
              acc[i][q].x = fmaf(v, t4.x, acc[i][q].x); acc[i][q].y = fmaf(v, t4.y, acc[i][q].y);
              acc[i][q].z = fmaf(v, t4.z, acc[i][q].z); acc[i][q].w = fmaf(v, t4.w, acc[i][q].w);
            }
          }
        }
      }
    }
    // combine the record groups, store the panel
#pragma unroll
    for (int i = 0; i < kRPW; ++i)
#pragma unroll
      for (int off = G; off < 32; off <<= 1)
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          acc[i][q].x += __shfl_xor_sync(0xffffffffu, acc[i][q].x, off);
          acc[i][q].y += __shfl_xor_sync(0xffffffffu, acc[i][q].y, off);
          acc[i][q].z += __shfl_xor_sync(0xffffffffu, acc[i][q].z, off);
          acc[i][q].w += __shfl_xor_sync(0xffffffffu, acc[i][q].w, off);
        }
    if (hg != 0) continue;
#pragma unroll
    for (int i = 0; i < kRPW; ++i) {
      const int r = r0 + i;
      if (r >= a.nrows) continue;
      float* y = a.Y + (int64_t)r * a.ldy + col0;
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const int col = (q * G + gl) * 4;
        const int rem = a.d - col0 - col;
        if (rem >= 4) {
          *reinterpret_cast<float4*>(y + col) = acc[i][q];
        } else if (rem > 0) {
          y[col] = acc[i][q].x;
          if (rem > 1) y[col + 1] = acc[i][q].y;
          if (rem > 2) y[col + 2] = acc[i][q].z;
        }
      }
    }
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

template <int NV, int G, int S, int MINB = 1>
static cudaError_t launch_nv(const Args& a0, int xrows, cudaStream_t stream) {
  using S_ = Smem<NV, G, S>;
  static_assert(S_::TOTAL <= 227 * 1024, "smem");
  Args a = a0;
  a.npanels = (a.d + S_::P - 1) / S_::P;
  a.pw = a.npanels > 1 ? S_::P : (a.d + 3) / 4 * 4;
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)a.d, (cuuint64_t)xrows};
  cuuint64_t strides[1] = {(cuuint64_t)(a.ldx * 4)};
  cuuint32_t box[2] = {(cuuint32_t)a.pw, (cuuint32_t)kTW};
  cuuint32_t es[2] = {1u, 1u};
  if (fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a.X), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(spmm_tiled_kernel<NV, G, S, MINB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, S_::TOTAL);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int items = a.nblocks * a.npanels;
  const int grid = items < MINB * num_sms() ? items : MINB * num_sms();
  if (grid > 0) spmm_tiled_kernel<NV, G, S, MINB><<<grid, kThreads, S_::TOTAL, stream>>>(map, a);
  return cudaGetLastError();
}

}  // namespace st

cudaError_t launch_spmm_tiled(int nrows, int xrows, int nblocks, const int32_t* tile_ptr, const int32_t* tile_win,
                              const int64_t* tile_off, const uint16_t* tile_rowoff, const int2* tile_nz,
                              const int64_t* res_ptr, const int32_t* res_col, const float* res_val, const float* X,
                              int64_t ldx, int d, float* Y, int64_t ldy, int* work, cudaStream_t stream) {
  if (nrows <= 0 || d <= 0) return cudaSuccess;
  if ((ldx & 3) || (ldy & 3) || (((uintptr_t)X) & 15) || (((uintptr_t)Y) & 15)) return cudaErrorNotSupported;
  st::Args a{};
  a.nrows = nrows; a.nblocks = nblocks; a.d = d;
  a.tile_ptr = tile_ptr; a.tile_win = tile_win; a.tile_off = tile_off; a.tile_rowoff = tile_rowoff;
  a.tile_nz = tile_nz; a.res_ptr = res_ptr; a.res_col = res_col; a.res_val = res_val;
  a.X = X; a.ldx = ldx; a.Y = Y; a.ldy = ldy;
  a.next_item = work;
  if (!a.next_item) return cudaErrorInvalidValue;
  // d <= 64: a lane group of 8 lanes per row (4 rows of a warp in parallel),
  // 2 CTAs per SM; wider panels: HB_TILED_ROWPAR=1 selects the same row-per-
  // group consumer (8 lanes x NV float4)
  static const int rowpar = getenv("HB_TILED_ROWPAR") ? atoi(getenv("HB_TILED_ROWPAR")) : 0;
  if (d <= 64) return st::launch_nv<2, 8, 4, 2>(a, xrows, stream);
  if (d <= 128) return rowpar ? st::launch_nv<4, 8, 5>(a, xrows, stream) : st::launch_nv<1, 32, 5>(a, xrows, stream);
  if (rowpar == 1) return st::launch_nv<8, 8, 3>(a, xrows, stream);
  if (rowpar == 2) return st::launch_nv<4, 16, 3>(a, xrows, stream);
  return st::launch_nv<2, 32, 3>(a, xrows, stream);                  // 72 KB stages, 256-column panels
}

}  // namespace hb
