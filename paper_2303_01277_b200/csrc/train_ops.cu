// Small fused elementwise/row kernels around the halo path (K8):
// masked softmax-CE + grad (linalg.py:87-112), ReLU / relu' product
// (linalg.py:78-84, trainer.py:295,312), Adam (linalg.py:115-140),
// argmax accuracy (trainer.py:129-144), keyed dropout (trainer.py:285-289) and
// the multi-label sigmoid BCE extension.
#include <cuda_runtime.h>
#include <cstdint>
#include "common.cuh"
#include "philox.cuh"

namespace hb {

// ---- masked softmax cross-entropy: warp per row ------------------------------
__global__ void xent_rows_kernel(const float* __restrict__ logits, int64_t ld, int n, int C,
                                 const int32_t* __restrict__ labels, const uint8_t* __restrict__ mask,
                                 double norm, float* __restrict__ grad, int64_t ldg,
                                 double* __restrict__ row_loss, int keep_unmasked) {
  const int lane = threadIdx.x & 31;
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n;
       row += gridDim.x * (blockDim.x >> 5)) {
    float* g = grad + (int64_t)row * ldg;
    if (!mask[row]) {
      if (keep_unmasked) continue;         // caller's buffers already hold the zeros
      for (int c = lane; c < C; c += 32) g[c] = 0.f;
      if (lane == 0) row_loss[row] = 0.0;
      continue;
    }
    const float* z = logits + (int64_t)row * ld;
    const int y = labels[row];
    if (C <= 128) {
      // one f64 exp per class: the (up to 4) logits of this lane stay in registers
      float zv[4];
      float m = -__int_as_float(0x7f800000);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = lane + 32 * k;
        zv[k] = c < C ? z[c] : 0.f;
        if (c < C) m = fmaxf(m, zv[k]);
      }
      m = warp_max(m);
      double ev[4], s = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        ev[k] = (lane + 32 * k < C) ? exp((double)zv[k] - (double)m) : 0.0;
        s += ev[k];
      }
      s = warp_sum_d(s);
      const double inv = 1.0 / s;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = lane + 32 * k;
        if (c < C) g[c] = (float)((ev[k] * inv - (c == y ? 1.0 : 0.0)) / norm);
      }
      if (lane == 0) row_loss[row] = -(((double)z[y] - (double)m) - log(s)) / norm;
      continue;
    }
    float m = -__int_as_float(0x7f800000);
    for (int c = lane; c < C; c += 32) m = fmaxf(m, z[c]);
    m = warp_max(m);
    double s = 0.0;
    for (int c = lane; c < C; c += 32) s += exp((double)z[c] - (double)m);
    s = warp_sum_d(s);
    const double inv = 1.0 / s;
    for (int c = lane; c < C; c += 32) {
      const double p = exp((double)z[c] - (double)m) * inv;
      g[c] = (float)((p - (c == y ? 1.0 : 0.0)) / norm);
    }
    if (lane == 0) row_loss[row] = -(((double)z[y] - (double)m) - log(s)) / norm;
  }
}

// Deterministic fixed-order sum of row_loss in two passes: block b reduces
// the contiguous slice [b*chunk, (b+1)*chunk) into part[b] (fixed tree), then
// one block sums the parts in order.  The block count depends on n only, so
// the result is run-to-run bit-identical.
constexpr int kSumBlocks = 256;
__global__ void __launch_bounds__(256) sum_f64_part_kernel(const double* __restrict__ x, int n, int chunk,
                                                           double* __restrict__ part) {
  __shared__ double sh[256];
  const int b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  double acc = 0.0;
  for (int i = b0 + threadIdx.x; i < b1; i += 256) acc += x[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(256) sum_f64_kernel(const double* __restrict__ x, int n,
                                                      double* __restrict__ out) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) acc += x[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// ---- ReLU and relu' product ----------------------------------------------------
// Row-tiled elementwise kernels: one warp walks a row with float4 accesses
// when the rows are 16-byte aligned (the trainer's buffers are), scalar
// otherwise; no per-element 64-bit division.
template <typename F>
__device__ __forceinline__ void rows_apply(int n, int d, bool vec, F f) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    if (vec) {
      const int d4 = d >> 2;
      for (int c4 = lane; c4 < d4; c4 += 32) f.vec4(r, 4 * c4);
      for (int c = 4 * d4 + lane; c < d; c += 32) f.one(r, c);
    } else {
      for (int c = lane; c < d; c += 32) f.one(r, c);
    }
  }
}

__device__ __forceinline__ float relu1(float v) { return (v > 0.f || v != v) ? v : 0.f; }  // np.maximum keeps NaN

struct ReluOp {
  const float* z; int64_t ldz; float* y; int64_t ldy;
  __device__ void one(int r, int c) const { y[(int64_t)r * ldy + c] = relu1(z[(int64_t)r * ldz + c]); }
  __device__ void vec4(int r, int c) const {
    const float4 v = *reinterpret_cast<const float4*>(z + (int64_t)r * ldz + c);
    *reinterpret_cast<float4*>(y + (int64_t)r * ldy + c) = make_float4(relu1(v.x), relu1(v.y), relu1(v.z), relu1(v.w));
  }
};

struct ReluGradOp {
  const float* j; int64_t ldj; const float* h; int64_t ldh; float* m; int64_t ldm;
  __device__ void one(int r, int c) const {
    m[(int64_t)r * ldm + c] = h[(int64_t)r * ldh + c] > 0.f ? j[(int64_t)r * ldj + c] : 0.f;
  }
  __device__ void vec4(int r, int c) const {
    const float4 a = *reinterpret_cast<const float4*>(j + (int64_t)r * ldj + c);
    const float4 b = *reinterpret_cast<const float4*>(h + (int64_t)r * ldh + c);
    *reinterpret_cast<float4*>(m + (int64_t)r * ldm + c) =
        make_float4(b.x > 0.f ? a.x : 0.f, b.y > 0.f ? a.y : 0.f, b.z > 0.f ? a.z : 0.f, b.w > 0.f ? a.w : 0.f);
  }
};

__global__ void relu_kernel(const float* __restrict__ z, int64_t ldz, int n, int d, float* __restrict__ y,
                            int64_t ldy, bool vec) {
  rows_apply(n, d, vec, ReluOp{z, ldz, y, ldy});
}

__global__ void relu_grad_mul_kernel(const float* __restrict__ j, int64_t ldj, const float* __restrict__ h,
                                     int64_t ldh, int n, int d, float* __restrict__ m, int64_t ldm, bool vec) {
  rows_apply(n, d, vec, ReluGradOp{j, ldj, h, ldh, m, ldm});
}

static bool al16(const void* p, int64_t ld) { return ((((uintptr_t)p) & 15) == 0) && (ld % 4 == 0); }

static int rows_grid(int n) {
  const int want = (n + 7) / 8;
  const int cap = num_sms() * 16;
  return want < cap ? (want > 0 ? want : 1) : cap;
}

// ---- Adam ------------------------------------------------------------------------
// guard (optional): the step is skipped when *loss is not finite or a flag
// word is non-zero — the reference's NaN check before Adam (trainer.py:361-366)
// evaluated on the device, so the host can read the epoch's loss later
__global__ void adam_kernel(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, int64_t n, float lr, float b1, float b2, float eps,
                            double bc1, double bc2, const double* __restrict__ loss,
                            const uint32_t* __restrict__ flags, const uint32_t* __restrict__ flags2,
                            const double* __restrict__ bc) {
  if (loss != nullptr && !isfinite(*loss)) return;
  if (bc != nullptr) {          // bias corrections from device memory (CUDA-graph replays)
    bc1 = bc[0];
    bc2 = bc[1];
  }
  if (flags != nullptr && *flags != 0u) return;
  if (flags2 != nullptr && *flags2 != 0u) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = g[i];
    const double mi = (double)b1 * m[i] + (1.0 - (double)b1) * gi;
    const double vi = (double)b2 * v[i] + (1.0 - (double)b2) * gi * gi;
    m[i] = (float)mi;
    v[i] = (float)vi;
    const double upd = (double)lr * (mi / bc1) / (sqrt(vi / bc2) + (double)eps);
    w[i] = (float)((double)w[i] - upd);
  }
}

// ---- argmax accuracy ---------------------------------------------------------
__global__ void argmax_acc_kernel(const float* __restrict__ logits, int64_t ld, int n, int C,
                                  const int32_t* __restrict__ labels, const uint8_t* __restrict__ mask,
                                  unsigned long long* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  unsigned long long local[6] = {0, 0, 0, 0, 0, 0};
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n;
       row += gridDim.x * (blockDim.x >> 5)) {
    const int mk = mask[row];
    if (mk < 1 || mk > 3) continue;
    const float* z = logits + (int64_t)row * ld;
    float best = -__int_as_float(0x7f800000);
    int arg = 0x7fffffff;
    for (int c = lane; c < C; c += 32) {
      const float v = z[c];
      if (v > best || (v == best && c < arg)) { best = v; arg = c; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (ob > best || (ob == best && oa < arg)) { best = ob; arg = oa; }
    }
    if (lane == 0) {
      local[2 * (mk - 1)] += 1;
      local[2 * (mk - 1) + 1] += (arg == labels[row]) ? 1 : 0;
    }
  }
  if (lane == 0)
    for (int k = 0; k < 6; ++k)
      if (local[k]) atomicAdd(counts + k, local[k]);
}

// ---- masked multi-label sigmoid BCE (extension: the reference has only the
// softmax CE; used for the Yelp-shaped multi-label config) ------
// row loss = sum_c [max(z,0) - z y + log1p(exp(-|z|))] / (norm C); grad =
// (sigmoid(z) - y) / (norm C); f64 math, one fp32 rounding of the gradient.
__global__ void bce_rows_kernel(const float* __restrict__ logits, int64_t ld, int n, int C,
                                const uint8_t* __restrict__ Y, int64_t ldy, const uint8_t* __restrict__ mask,
                                double norm, float* __restrict__ grad, int64_t ldg, double* __restrict__ row_loss,
                                int keep_unmasked) {
  const int lane = threadIdx.x & 31;
  const double scale = 1.0 / (norm * (double)C);
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n;
       row += gridDim.x * (blockDim.x >> 5)) {
    float* g = grad + (int64_t)row * ldg;
    if (!mask[row]) {
      if (keep_unmasked) continue;
      for (int c = lane; c < C; c += 32) g[c] = 0.f;
      if (lane == 0) row_loss[row] = 0.0;
      continue;
    }
    const float* z = logits + (int64_t)row * ld;
    const uint8_t* y = Y + (int64_t)row * ldy;
    double s = 0.0;
    for (int c = lane; c < C; c += 32) {
      const double zc = (double)z[c], yc = y[c] ? 1.0 : 0.0;
      s += fmax(zc, 0.0) - zc * yc + log1p(exp(-fabs(zc)));
      g[c] = (float)((1.0 / (1.0 + exp(-zc)) - yc) * scale);
    }
    s = warp_sum_d(s);
    if (lane == 0) row_loss[row] = s * scale;
  }
}

// Multi-label counts per mask value k = 1..3 (train / val / test):
// counts[3(k-1)] = true positives, +1 false positives, +2 false negatives of
// the prediction z > 0 (micro-F1 = 2TP / (2TP + FP + FN)).
__global__ void multilabel_counts_kernel(const float* __restrict__ logits, int64_t ld, int n, int C,
                                         const uint8_t* __restrict__ Y, int64_t ldy,
                                         const uint8_t* __restrict__ mask, unsigned long long* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  unsigned long long local[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n;
       row += gridDim.x * (blockDim.x >> 5)) {
    const int mk = mask[row];
    if (mk < 1 || mk > 3) continue;
    const float* z = logits + (int64_t)row * ld;
    const uint8_t* y = Y + (int64_t)row * ldy;
    unsigned tp = 0, fp = 0, fn = 0;
    for (int c = lane; c < C; c += 32) {
      const bool p = z[c] > 0.f, t = y[c] != 0;
      tp += p && t;
      fp += p && !t;
      fn += !p && t;
    }
    local[3 * (mk - 1)] += tp;
    local[3 * (mk - 1) + 1] += fp;
    local[3 * (mk - 1) + 2] += fn;
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    unsigned long long v = local[k];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && v) atomicAdd(counts + k, v);
  }
}

// ---- keyed dropout -----------------------------------------------------------------
__global__ void dropout_kernel(const float* __restrict__ x, int64_t ldx, int nrows, int64_t row0, int d,
                               uint64_t k0, uint64_t k1, double p, float scale, float* __restrict__ out,
                               int64_t ldo) {
  const uint64_t e_begin = (uint64_t)row0 * d, e_end = (uint64_t)(row0 + nrows) * d;
  const uint64_t b_first = e_begin >> 2, b_last = (e_end - 1) >> 2;
  for (uint64_t b = b_first + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b <= b_last;
       b += (uint64_t)gridDim.x * blockDim.x) {
    const U64x4 u = philox4x64_10(b + 1, k0, k1);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const uint64_t e = 4 * b + s;
      if (e < e_begin || e >= e_end) continue;
      const int64_t r = (int64_t)(e / d) - row0, c = (int64_t)(e % d);
      const bool keep = u53_to_double(pick(u, s)) >= p;
      out[r * ldo + c] = keep ? x[r * ldx + c] * scale : 0.f;
    }
  }
}

static int grid_for(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  return g < 1 ? 1 : (int)g;
}

cudaError_t launch_xent(const float* logits, int64_t ld, int n, int C, const int32_t* labels,
                        const uint8_t* mask, double norm, float* grad, int64_t ldg, double* row_loss,
                        double* loss_out, int keep_unmasked, double* partials, cudaStream_t st) {
  if (n > 0)
    xent_rows_kernel<<<grid_for(n, 8), 256, 0, st>>>(logits, ld, n, C, labels, mask, norm, grad, ldg, row_loss,
                                                     keep_unmasked);
  if (n <= 16 * 1024) {
    sum_f64_kernel<<<1, 256, 0, st>>>(row_loss, n, loss_out);
  } else {
    double* part = partials;            // caller's HB_XENT_PARTIALS doubles
    if (!part) return cudaErrorInvalidValue;
    const int chunk = (n + kSumBlocks - 1) / kSumBlocks;
    sum_f64_part_kernel<<<kSumBlocks, 256, 0, st>>>(row_loss, n, chunk, part);
    sum_f64_kernel<<<1, 256, 0, st>>>(part, kSumBlocks, loss_out);
  }
  return cudaGetLastError();
}

cudaError_t launch_relu(const float* z, int64_t ldz, int n, int d, float* y, int64_t ldy, cudaStream_t st) {
  if ((int64_t)n * d <= 0) return cudaSuccess;
  relu_kernel<<<rows_grid(n), 256, 0, st>>>(z, ldz, n, d, y, ldy, al16(z, ldz) && al16(y, ldy));
  return cudaGetLastError();
}

cudaError_t launch_relu_grad_mul(const float* j, int64_t ldj, const float* h, int64_t ldh, int n, int d,
                                 float* m, int64_t ldm, cudaStream_t st) {
  if ((int64_t)n * d <= 0) return cudaSuccess;
  relu_grad_mul_kernel<<<rows_grid(n), 256, 0, st>>>(j, ldj, h, ldh, n, d, m, ldm,
                                                     al16(j, ldj) && al16(h, ldh) && al16(m, ldm));
  return cudaGetLastError();
}

cudaError_t launch_adam(float* w, const float* g, float* m, float* v, int64_t n, float lr, float b1,
                        float b2, float eps, double bc1, double bc2, const double* loss, const uint32_t* flags,
                        const uint32_t* flags2, const double* bc, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  adam_kernel<<<grid_for(n, 256), 256, 0, st>>>(w, g, m, v, n, lr, b1, b2, eps, bc1, bc2, loss, flags, flags2, bc);
  return cudaGetLastError();
}

cudaError_t launch_argmax_accuracy(const float* logits, int64_t ld, int n, int C, const int32_t* labels,
                                   const uint8_t* mask, int64_t* counts, cudaStream_t st) {
  cudaMemsetAsync(counts, 0, 6 * sizeof(int64_t), st);
  if (n > 0)
    argmax_acc_kernel<<<grid_for(n, 8), 256, 0, st>>>(logits, ld, n, C, labels, mask,
                                                       reinterpret_cast<unsigned long long*>(counts));
  return cudaGetLastError();
}

cudaError_t launch_bce(const float* logits, int64_t ld, int n, int C, const uint8_t* Y, int64_t ldy,
                       const uint8_t* mask, double norm, float* grad, int64_t ldg, double* row_loss,
                       double* loss_out, int keep_unmasked, double* partials, cudaStream_t st) {
  if (n > 0)
    bce_rows_kernel<<<grid_for(n, 8), 256, 0, st>>>(logits, ld, n, C, Y, ldy, mask, norm, grad, ldg, row_loss,
                                                    keep_unmasked);
  if (n <= 16 * 1024) {
    sum_f64_kernel<<<1, 256, 0, st>>>(row_loss, n, loss_out);
  } else {
    if (!partials) return cudaErrorInvalidValue;
    const int chunk = (n + kSumBlocks - 1) / kSumBlocks;
    sum_f64_part_kernel<<<kSumBlocks, 256, 0, st>>>(row_loss, n, chunk, partials);
    sum_f64_kernel<<<1, 256, 0, st>>>(partials, kSumBlocks, loss_out);
  }
  return cudaGetLastError();
}

cudaError_t launch_multilabel_counts(const float* logits, int64_t ld, int n, int C, const uint8_t* Y, int64_t ldy,
                                     const uint8_t* mask, int64_t* counts, cudaStream_t st) {
  cudaMemsetAsync(counts, 0, 9 * sizeof(int64_t), st);
  if (n > 0)
    multilabel_counts_kernel<<<grid_for(n, 8), 256, 0, st>>>(logits, ld, n, C, Y, ldy, mask,
                                                             reinterpret_cast<unsigned long long*>(counts));
  return cudaGetLastError();
}

cudaError_t launch_dropout(const float* x, int64_t ldx, int nrows, int64_t row0, int d, uint64_t k0,
                           uint64_t k1, float p, float* out, int64_t ldo, cudaStream_t st) {
  if ((int64_t)nrows * d <= 0) return cudaSuccess;
  const float scale = (float)(1.0 / (1.0 - (double)p));
  dropout_kernel<<<grid_for(((int64_t)nrows * d) / 4 + 2, 256), 256, 0, st>>>(x, ldx, nrows, row0, d, k0, k1,
                                                                              (double)p, scale, out, ldo);
  return cudaGetLastError();
}

}  // namespace hb
