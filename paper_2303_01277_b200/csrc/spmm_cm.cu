// K3/K4 factored tiled SpMM, column-major tiles ("cm"):
//
//   Y[i, :] = r[i] * sum_{(i,j) in pattern} c[j] X[j, :]
//
// the trainer's aggregation operators (linalg.spmm, linalg.py:71-75, on the
// partition blocks of graph.py:120-141; r / c as in spmm_bin.cu).
//
// Why a second tile format.  A SIMT SpMM that stages X windows in shared
// memory is bound by the shared-memory datapath (128 B/clk/SM): every
// nonzero moves its whole X row (1 KB at d = 256, 8 wavefronts) from shared
// memory to registers.  spmm_bin.cu walks each row's nonzeros, so a column
// shared by several rows of a warp is read once per row.  Here a warp owns 8
// rows of a 128-row block and walks the *columns* of the tile's 64-column
// window that any of its rows touches: each tile record is one (column,
// 8-bit row mask) pair, the X row is read once and added to every masked
// row's accumulators.  On the Reddit-shaped graph (in-community density
// ~8.7 %) a column entry serves ~1.35 rows, so the X reads per nonzero drop
// from 8 to ~6 wavefronts.  Each row still receives its tile contributions in
// ascending column order, then its residual ones: the summation order of
// spmm_bin.cu and hb_spmm_csr.
//
// Layout per tile (built by ops.TiledCsr(..., fmt="cm")): u16 entries
// (column | mask << 8), grouped by warp, each warp's run padded with zero
// entries to a multiple of 8 (one 16-byte broadcast load per 8 entries);
// kCmWoff u16 warp offsets (in entries).  A tile holds at most 16 x 64
// entries, so dense windows never split.
//
// Work items (row block, feature panel) come from the caller's counter pair
// {next item, CTAs finished}, zero on entry, re-armed by the last CTA.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdlib>
#include "common.cuh"

namespace hb {
namespace scm {

constexpr int kRB = 128;                         // rows per block
constexpr int kCW = 16;                          // consumer warps (8 rows each)
constexpr int kRPW = kRB / kCW;
constexpr int kKW = 64;                          // columns per window
constexpr int kWoff = 24;                        // u16 warp offsets per tile (kCW + 1 used)
constexpr int kMaxEnt = kCW * kKW + kCW * 7;     // (warp, column) pairs + per-warp padding
constexpr int kQ = 4;

struct Args {
  int nrows, nblocks, npanels, d, pw;
  int* work;
  const int32_t* tile_ptr;
  const int32_t* tile_win;
  const int64_t* tile_off;       // byte offsets of each tile's entries (multiples of 16)
  const uint16_t* tile_woff;     // [ntiles][kWoff]
  const uint16_t* tile_ent;
  const int64_t* res_ptr;        // residual pattern (CSR without values)
  const int32_t* res_col;
  const float* row_scale;        // nullable
  const float* X;
  int64_t ldx;
  float* Y;
  int64_t ldy;
};

template <int NV, int S>
struct Smem {
  static constexpr int P = 128 * NV;                        // panel width (floats)
  static constexpr int X_BYTES = kKW * P * 4;
  static constexpr int E_BYTES = (kMaxEnt * 2 + 15) / 16 * 16;
  static constexpr int W_BYTES = kWoff * 2;
  static constexpr int STAGE = (X_BYTES + E_BYTES + W_BYTES + 127) / 128 * 128;
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

template <int NV, bool FULL>
__device__ __forceinline__ void add4(float4 (&acc)[NV], const float4 (&x)[NV], int nlast) {
#pragma unroll
  for (int v = 0; v < NV; ++v)
    if (FULL || v < NV - 1 || nlast) {
      acc[v].x += x[v].x; acc[v].y += x[v].y; acc[v].z += x[v].z; acc[v].w += x[v].w;
    }
}

// acc[r] += x for every set bit r of the (warp-uniform) 8-bit row mask:
// a tree of warp-uniform branches (most entries carry one row), no
// predicated adds for absent rows
#define HB_CM_ADD(R) if (m & (1u << (R))) add4<NV, FULL>(acc[R], x, nlast)
template <int NV, bool FULL>
__device__ __forceinline__ void add_masked(float4 (&acc)[kRPW][NV], const float4 (&x)[NV], uint32_t m, int nlast) {
  if (m & 0x0Fu) {
    if (m & 0x03u) { HB_CM_ADD(0); HB_CM_ADD(1); }
    if (m & 0x0Cu) { HB_CM_ADD(2); HB_CM_ADD(3); }
  }
  if (m & 0xF0u) {
    if (m & 0x30u) { HB_CM_ADD(4); HB_CM_ADD(5); }
    if (m & 0xC0u) { HB_CM_ADD(6); HB_CM_ADD(7); }
  }
}
#undef HB_CM_ADD

// 17 warps are allocated registers as 20: 96 per thread is the most that
// launches one CTA per SM
template <int NV, int S, bool FULL>
__global__ void __maxnreg__(96)
spmm_cm_kernel(const __grid_constant__ CUtensorMap tmX, Args a) {
  using S_ = Smem<NV, S>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  __shared__ __align__(8) uint64_t full[S], empty[S], ifull[kQ], iempty[kQ];
  __shared__ int item_q[kQ];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCW);
    }
    for (int q = 0; q < kQ; ++q) {
      mbar_init(&ifull[q], 1);
      mbar_init(&iempty[q], kCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int items = a.nblocks * a.npanels;

  if (warp == kCW) {
    // ---------------- producer: lane 0 claims items, lane s feeds ring stage s
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
      const int b = item / a.npanels, pn = item % a.npanels;
      const int t0 = a.tile_ptr[b], t1 = a.tile_ptr[b + 1];
      for (int t = t0; t < t1; ++t, ++it) {
        if (lane >= S || it % S != lane) continue;
        const int s = it % S;
        mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
        uint8_t* st = smem + s * S_::STAGE;
        const int64_t o0 = a.tile_off[t], o1 = a.tile_off[t + 1];
        const uint32_t eb = (uint32_t)(o1 - o0);
        mbar_expect_tx(&full[s], (uint32_t)(kKW * a.pw * 4) + eb + S_::W_BYTES);
        tma_2d(st, &tmX, pn * S_::P, a.tile_win[t] * kKW, &full[s]);
        if (eb) tma_load_1d(st + S_::X_BYTES, reinterpret_cast<const uint8_t*>(a.tile_ent) + o0, eb, &full[s]);
        tma_load_1d(st + S_::X_BYTES + S_::E_BYTES, a.tile_woff + (int64_t)t * kWoff, S_::W_BYTES, &full[s]);
      }
    }
    __syncwarp();
    return;
  }

  // ---------------- consumers: warp owns rows warp*8 .. warp*8+7 of the block;
  // lane holds NV float4 columns (lane, lane + 32, ...) of the panel
  const int pw4 = a.pw / 4;
  const int nlast = FULL || ((NV - 1) * 32 + lane) * 4 < a.pw;
  int it = 0;
  for (int qi = 0;; ++qi) {
    const int q = qi % kQ;
    mbar_wait(&ifull[q], (qi / kQ) & 1);
    const int item = item_q[q];
    __syncwarp();
    if (lane == 0) mbar_arrive_cta(&iempty[q]);
    if (item >= items) break;
    const int b = item / a.npanels, pn = item % a.npanels;
    const int r0 = b * kRB + warp * kRPW;
    const int col0 = pn * S_::P;
    float4 acc[kRPW][NV];
#pragma unroll
    for (int i = 0; i < kRPW; ++i)
#pragma unroll
      for (int v = 0; v < NV; ++v) acc[i][v] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int t = a.tile_ptr[b]; t < a.tile_ptr[b + 1]; ++t, ++it) {
      const int s = it % S;
      mbar_wait(&full[s], (it / S) & 1);
      const uint8_t* st = smem + s * S_::STAGE;
      const float4* xs = reinterpret_cast<const float4*>(st) + lane;
      const uint16_t* wop = reinterpret_cast<const uint16_t*>(st + S_::X_BYTES + S_::E_BYTES) + warp;
      const int w0 = wop[0], w1 = wop[1];
      const uint4* ent = reinterpret_cast<const uint4*>(st + S_::X_BYTES) + (w0 >> 3);
      const int ng = (w1 - w0) >> 3;
      for (int g = 0; g < ng; ++g) {
        const uint4 qv = ent[g];                       // 8 entries, one broadcast load
        const uint32_t w4[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          // two entries in flight: both X rows are loaded before either is added;
          // the entry word is the same in every lane (a broadcast): lane 0's copy
          // makes that visible to the compiler (uniform branches)
          const uint32_t wu = __shfl_sync(0xffffffffu, w4[h], 0);
          const uint32_t ea = wu & 0xffffu, eb = wu >> 16;
          const uint32_t ma = ea >> 8, mb = eb >> 8;
          if (ma == 0) break;                          // zero entries pad the warp's run
          float4 xa[NV], xb[NV];
#pragma unroll
          for (int v = 0; v < NV; ++v)
            if (FULL || v < NV - 1 || nlast) xa[v] = xs[(int)(ea & 0xffu) * pw4 + v * 32];
          if (mb) {
#pragma unroll
            for (int v = 0; v < NV; ++v)
              if (FULL || v < NV - 1 || nlast) xb[v] = xs[(int)(eb & 0xffu) * pw4 + v * 32];
          }
          add_masked<NV, FULL>(acc, xa, ma, nlast);
          if (mb == 0) break;
          add_masked<NV, FULL>(acc, xb, mb, nlast);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&empty[s]);
    }
    // residual pattern entries gathered from global X, row scale, store
#pragma unroll
    for (int i = 0; i < kRPW; ++i) {
      const int r = r0 + i;
      if (r >= a.nrows) continue;
      const float* Xp = a.X + col0;
      const int64_t e0 = a.res_ptr[r], e1 = a.res_ptr[r + 1];
      for (int64_t k = e0; k < e1; ++k) {
        const float4* xr = reinterpret_cast<const float4*>(Xp + (int64_t)__ldg(a.res_col + k) * a.ldx) + lane;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          if (col0 + (v * 32 + lane) * 4 < a.d) {
            const float4 t4 = __ldg(xr + v * 32);
            acc[i][v].x += t4.x; acc[i][v].y += t4.y; acc[i][v].z += t4.z; acc[i][v].w += t4.w;
          }
        }
      }
      const float sc = a.row_scale ? __ldg(a.row_scale + r) : 1.f;
      float* y = a.Y + (int64_t)r * a.ldy + col0;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int col = (v * 32 + lane) * 4;
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

template <int NV, int S, bool FULL>
static cudaError_t launch_nv(const Args& a0, int xrows, cudaStream_t stream) {
  using S_ = Smem<NV, S>;
  static_assert(S_::TOTAL <= 227 * 1024, "smem");
  Args a = a0;
  a.npanels = (a.d + S_::P - 1) / S_::P;
  a.pw = a.npanels > 1 ? S_::P : (a.d + 3) / 4 * 4;
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)a.d, (cuuint64_t)xrows};
  cuuint64_t strides[1] = {(cuuint64_t)(a.ldx * 4)};
  cuuint32_t box[2] = {(cuuint32_t)a.pw, (cuuint32_t)kKW};
  cuuint32_t es[2] = {1u, 1u};
  if (fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a.X), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorNotSupported;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(spmm_cm_kernel<NV, S, FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         S_::TOTAL);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int items = a.nblocks * a.npanels;
  const int grid = items < num_sms() ? items : num_sms();
  if (grid > 0) spmm_cm_kernel<NV, S, FULL><<<grid, 32 * (kCW + 1), S_::TOTAL, stream>>>(map, a);
  return cudaGetLastError();
}

}  // namespace scm

cudaError_t launch_spmm_tiled_cm(int nrows, int xrows, int nblocks, const int32_t* tile_ptr,
                                 const int32_t* tile_win, const int64_t* tile_off, const uint16_t* tile_woff,
                                 const uint16_t* tile_ent, const int64_t* res_ptr, const int32_t* res_col,
                                 const float* row_scale, const float* col_scale, const float* X, int64_t ldx,
                                 int d, float* Y, int64_t ldy, float* xs, int64_t ldxs, int* work,
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
  scm::Args a{};
  a.nrows = nrows; a.nblocks = nblocks; a.d = d; a.work = work;
  a.tile_ptr = tile_ptr; a.tile_win = tile_win; a.tile_off = tile_off; a.tile_woff = tile_woff;
  a.tile_ent = tile_ent; a.res_ptr = res_ptr; a.res_col = res_col; a.row_scale = row_scale;
  a.X = X; a.ldx = ldx; a.Y = Y; a.ldy = ldy;
  // FULL: every panel is 128 * NV columns wide (no partial last float4 per lane)
  if (d <= 128) return d == 128 ? scm::launch_nv<1, 5, true>(a, xrows, stream)
                                : scm::launch_nv<1, 5, false>(a, xrows, stream);
  static const int nv_env = getenv("HB_CM_NV") ? atoi(getenv("HB_CM_NV")) : 2;
  if (nv_env == 1)                                    // 128-column panels
    return d % 128 == 0 ? scm::launch_nv<1, 5, true>(a, xrows, stream)
                        : scm::launch_nv<1, 5, false>(a, xrows, stream);
  return d % 256 == 0 ? scm::launch_nv<2, 3, true>(a, xrows, stream)      // 256-column panels
                      : scm::launch_nv<2, 3, false>(a, xrows, stream);
}

}  // namespace hb
