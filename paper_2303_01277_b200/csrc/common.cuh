// Shared helpers for the halo-path kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "halob200.h"

namespace hb {

constexpr int kWarp = 32;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Largest s with segs[s].row_begin <= row (segs sorted, segs[0].row_begin == 0).
__device__ __forceinline__ int find_segment(const hb_segment_t* segs, int nseg, int row) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].row_begin <= row) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Number of SMs of the current device (cached per process).
int num_sms();

}  // namespace hb
