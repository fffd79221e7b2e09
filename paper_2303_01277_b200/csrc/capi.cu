// extern "C" entry points of libhalob200.so (declared in include/halob200.h).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include "common.cuh"

namespace hb {
cudaError_t launch_quantize_gather(const float*, int64_t, const int32_t*, int, const hb_segment_t*, int,
                                   int, int, uint32_t*, cudaStream_t);
cudaError_t launch_dequant_gather(const hb_segment_t*, int, int, const int32_t*, const int32_t*,
                                  const int32_t*, int, int, float*, int64_t, int, cudaStream_t);
cudaError_t launch_philox_uniforms(uint64_t, uint64_t, uint64_t, int64_t, double*, cudaStream_t);
cudaError_t launch_spmm(int, const int64_t*, const int32_t*, const float*, const float*, int64_t, int,
                        float*, int64_t, int64_t, int, int, int, int*, cudaStream_t);
cudaError_t launch_xent(const float*, int64_t, int, int, const int32_t*, const uint8_t*, double, float*,
                        int64_t, double*, double*, int, double*, cudaStream_t);
cudaError_t launch_relu(const float*, int64_t, int, int, float*, int64_t, cudaStream_t);
cudaError_t launch_relu_grad_mul(const float*, int64_t, const float*, int64_t, int, int, float*, int64_t,
                                 cudaStream_t);
cudaError_t launch_adam(float*, const float*, float*, float*, int64_t, float, float, float, float, double,
                        double, const double*, const uint32_t*, const uint32_t*, const double*, cudaStream_t);
cudaError_t launch_argmax_accuracy(const float*, int64_t, int, int, const int32_t*, const uint8_t*,
                                   int64_t*, cudaStream_t);
cudaError_t launch_dropout(const float*, int64_t, int, int64_t, int, uint64_t, uint64_t, float, float*,
                           int64_t, cudaStream_t);
cudaError_t launch_bce(const float*, int64_t, int, int, const uint8_t*, int64_t, const uint8_t*, double, float*,
                       int64_t, double*, double*, int, double*, cudaStream_t);
cudaError_t launch_multilabel_counts(const float*, int64_t, int, int, const uint8_t*, int64_t, const uint8_t*,
                                     int64_t*, cudaStream_t);

cudaError_t launch_gemm_tf32x3(int, int, int, const float*, int64_t, int64_t, const float*, int64_t, int64_t,
                               float*, int64_t, float, float*, int64_t, float*, int64_t, cudaStream_t);
cudaError_t launch_gemm2_tf32x3(int, int, int, const float*, int64_t, int64_t, const float*, int64_t, int64_t, int,
                                const float*, int64_t, int64_t, const float*, int64_t, int64_t, float*, int64_t, float,
                                float*, int64_t, float*, int64_t, cudaStream_t);
extern int g_gemm_path;
extern int g_bin_narrow;
extern int g_gemm_ts;
cudaError_t launch_spmm_tiled(int, int, int, const int32_t*, const int32_t*, const int64_t*, const uint16_t*,
                              const int2*, const int64_t*, const int32_t*, const float*, const float*, int64_t, int,
                              float*, int64_t, int*, cudaStream_t);
cudaError_t launch_spmm_tiled_bin(int, int, int, const int32_t*, const int32_t*, const int64_t*, const uint16_t*,
                                  const uint8_t*, const int64_t*, const int32_t*, const float*, const float*,
                                  const float*, int64_t, int, float*, int64_t, float*, int64_t, int*, int, int,
                                  const int32_t*, cudaStream_t);

cudaError_t launch_p2p_signal(unsigned long long* const*, int, cudaStream_t);
cudaError_t launch_p2p_wait(const unsigned long long*, unsigned long long, const unsigned long long*, uint32_t*,
                            uint32_t, unsigned long long, cudaStream_t);
cudaError_t alloc_base(const void*, void**);

int num_sms() {
  static int cached = 0;
  if (!cached) {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached = n > 0 ? n : 148;
  }
  return cached;
}
}  // namespace hb

static thread_local std::string g_last_error;

static int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

static int check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(HB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return HB_OK;
}

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static bool valid_bits(int b) { return (b >= 1 && b <= 8) || b == 16 || b == 32; }

extern "C" {

const char* hb_version(void) { return "halob200 0.1 sm_100a"; }

const char* hb_last_error(void) { return g_last_error.c_str(); }

int hb_philox_uniforms(uint64_t key0, uint64_t key1, uint64_t start, int64_t n, double* out, void* stream) {
  if (n < 0 || (n > 0 && !out)) return fail(HB_EINVAL, "hb_philox_uniforms: bad arguments");
  return check(hb::launch_philox_uniforms(key0, key1, start, n, out, S(stream)), "hb_philox_uniforms");
}

int hb_quantize_gather(const float* src, int64_t ld, const int32_t* row_idx, int32_t total_rows,
                       const hb_segment_t* segs, int32_t nseg, int32_t d, int32_t bits, uint32_t* flags,
                       void* stream) {
  if (!valid_bits(bits)) return fail(HB_EINVAL, "unsupported bit width " + std::to_string(bits));
  if (total_rows < 0 || d <= 0 || ld < d || (total_rows > 0 && (!src || !row_idx || !segs || nseg <= 0)) ||
      !flags)
    return fail(HB_EINVAL, "hb_quantize_gather: bad arguments");
  return check(hb::launch_quantize_gather(src, ld, row_idx, total_rows, segs, nseg, d, bits, flags, S(stream)),
               "hb_quantize_gather");
}

int hb_dequant_gather(const hb_segment_t* segs, int32_t nseg, int32_t num_dst, const int32_t* dst_rows,
                      const int32_t* src_ptr, const int32_t* src_rows, int32_t d, int32_t bits, float* dst,
                      int64_t ld, int32_t accumulate, void* stream) {
  if (!valid_bits(bits)) return fail(HB_EINVAL, "unsupported bit width " + std::to_string(bits));
  if (num_dst < 0 || d <= 0 || ld < d || (num_dst > 0 && (!segs || nseg <= 0 || !dst_rows || !src_ptr || !dst)))
    return fail(HB_EINVAL, "hb_dequant_gather: bad arguments");
  return check(hb::launch_dequant_gather(segs, nseg, num_dst, dst_rows, src_ptr, src_rows, d, bits, dst, ld,
                                         accumulate, S(stream)),
               "hb_dequant_gather");
}

int hb_spmm_csr(int32_t nrows, const int64_t* row_ptr, const int32_t* col_idx, const float* vals,
                const float* X, int64_t ldx, int32_t d, float* Y, int64_t ldy, void* stream) {
  if (nrows < 0 || d < 0 || ldx < d || ldy < d || (nrows > 0 && (!row_ptr || !Y)))
    return fail(HB_EINVAL, "hb_spmm_csr: bad arguments");
  return check(hb::launch_spmm(nrows, row_ptr, col_idx, vals, X, ldx, d, Y, ldy, -1, 1, 0, INT32_MAX, nullptr,
                               S(stream)),
               "hb_spmm_csr");
}

int hb_spmm_csr_ex(int32_t nrows, const int64_t* row_ptr, const int32_t* col_idx, const float* vals,
                   const float* X, int64_t ldx, int32_t d, float* Y, int64_t ldy, int64_t nnz, int32_t algo,
                   int32_t window, int32_t stream_col, int32_t* work, void* stream) {
  if (nrows < 0 || d < 0 || ldx < d || ldy < d || (nrows > 0 && (!row_ptr || !Y)) || algo < 0 || algo > 1)
    return fail(HB_EINVAL, "hb_spmm_csr_ex: bad arguments");
  return check(hb::launch_spmm(nrows, row_ptr, col_idx, vals, X, ldx, d, Y, ldy, nnz, algo, window, stream_col,
                               work, S(stream)),
               "hb_spmm_csr_ex");
}

int hb_spmm_tiled(int32_t nrows, int32_t xrows, int32_t nblocks, const int32_t* tile_ptr, const int32_t* tile_win,
                  const int64_t* tile_off, const uint16_t* tile_rowoff, const void* tile_nz, const int64_t* res_ptr,
                  const int32_t* res_col, const float* res_val, const float* X, int64_t ldx, int32_t d, float* Y,
                  int64_t ldy, int32_t* work, void* stream) {
  if (nrows < 0 || d < 0 || ldx < d || ldy < d || nblocks != (nrows + 63) / 64 ||
      (nrows > 0 && (!tile_ptr || !res_ptr || !X || !Y || !work)))
    return fail(HB_EINVAL, "hb_spmm_tiled: bad arguments");
  const cudaError_t e = hb::launch_spmm_tiled(nrows, xrows, nblocks, tile_ptr, tile_win, tile_off, tile_rowoff,
                                              reinterpret_cast<const int2*>(tile_nz), res_ptr, res_col, res_val, X,
                                              ldx, d, Y, ldy, work, S(stream));
  if (e == cudaErrorNotSupported)
    return fail(HB_EINVAL, "hb_spmm_tiled: X/Y need 16-byte aligned rows (ld % 4 == 0)");
  return check(e, "hb_spmm_tiled");
}

int hb_spmm_tiled_bin(int32_t nrows, int32_t xrows, int32_t nblocks, const int32_t* tile_ptr,
                      const int32_t* tile_win, const int64_t* tile_off, const uint16_t* tile_rowoff,
                      const uint8_t* tile_rec, const int64_t* res_ptr, const int32_t* res_col,
                      const float* row_scale, const float* col_scale, const float* X, int64_t ldx, int32_t d,
                      float* Y, int64_t ldy, float* xs, int64_t ldxs, int32_t* work, int32_t block_rows,
                      int32_t window_cols, const int32_t* block_order, void* stream) {
  if (nrows < 0 || d < 0 || ldx < d || ldy < d || (block_rows != 64 && block_rows != 120 && block_rows != 128) ||
      (window_cols != 64 && window_cols != 128 && window_cols != 255) ||
      (window_cols != 64 && d > 48) || (window_cols == 128 && block_rows != 64) ||
      (window_cols == 255 && block_rows == 128 && d <= 32) || (block_rows == 120 && window_cols != 64) ||
      nblocks != (nrows + block_rows - 1) / block_rows ||
      (nrows > 0 && (!tile_ptr || !res_ptr || !X || !Y || !work)) || (col_scale && (!xs || ldxs < d)))
    return fail(HB_EINVAL, "hb_spmm_tiled_bin: bad arguments");
  const cudaError_t e = hb::launch_spmm_tiled_bin(nrows, xrows, nblocks, tile_ptr, tile_win, tile_off, tile_rowoff,
                                                  tile_rec, res_ptr, res_col, row_scale, col_scale, X, ldx, d, Y,
                                                  ldy, xs, ldxs, work, block_rows, window_cols, block_order,
                                                  S(stream));
  if (e == cudaErrorNotSupported)
    return fail(HB_EINVAL, "hb_spmm_tiled_bin: X/Y need 16-byte aligned rows (ld % 4 == 0)");
  return check(e, "hb_spmm_tiled_bin");
}

int hb_gemm_f32(int32_t M, int32_t N, int32_t K, const float* A, int64_t lda_m, int64_t lda_k, const float* B,
                int64_t ldb_k, int64_t ldb_n, float* C, int64_t ldc, float beta, float* relu_out, int64_t ldr,
                float* ws, int64_t ws_floats, void* stream) {
  if (M < 0 || N < 0 || K < 0 || (M > 0 && N > 0 && (!A || !B || K == 0)) || (C && ldc < N) ||
      (!C && (!relu_out || beta != 0.f)))
    return fail(HB_EINVAL, "hb_gemm_f32: bad arguments");
  return check(hb::launch_gemm_tf32x3(M, N, K, A, lda_m, lda_k, B, ldb_k, ldb_n, C, ldc, beta, relu_out, ldr, ws,
                                      ws_floats, S(stream)),
               "hb_gemm_f32");
}

int hb_gemm2_f32(int32_t M, int32_t N, int32_t K1, const float* A1, int64_t lda1_m, int64_t lda1_k, const float* B1,
                 int64_t ldb1_k, int64_t ldb1_n, int32_t K2, const float* A2, int64_t lda2_m, int64_t lda2_k,
                 const float* B2, int64_t ldb2_k, int64_t ldb2_n, float* C, int64_t ldc, float beta,
                 float* relu_out, int64_t ldr, float* ws, int64_t ws_floats, void* stream) {
  if (M < 0 || N < 0 || K1 <= 0 || K2 <= 0 || (C && ldc < N) || (!C && (!relu_out || beta != 0.f)) ||
      (M > 0 && N > 0 && (!A1 || !B1 || !A2 || !B2)))
    return fail(HB_EINVAL, "hb_gemm2_f32: bad arguments");
  return check(hb::launch_gemm2_tf32x3(M, N, K1, A1, lda1_m, lda1_k, B1, ldb1_k, ldb1_n, K2, A2, lda2_m, lda2_k, B2,
                                       ldb2_k, ldb2_n, C, ldc, beta, relu_out, ldr, ws, ws_floats, S(stream)),
               "hb_gemm2_f32");
}

int hb_gemm_set_path(int32_t path) {
  if (path < 0 || path > 3 || path == 2)
    return fail(HB_EINVAL, "hb_gemm_set_path: path must be 0 (auto), 1 (SIMT-staged) or 3 (A in TMEM)");
  hb::g_gemm_path = path == 1 ? 1 : 0;
  hb::g_gemm_ts = path == 3 ? 1 : 0;
  return HB_OK;
}

int hb_spmm_set_narrow(int32_t variant) {
  if (variant < 0 || variant > 4)
    return fail(HB_EINVAL, "hb_spmm_set_narrow: variant must be 0..4");
  hb::g_bin_narrow = variant;
  return HB_OK;
}

int hb_softmax_xent(const float* logits, int64_t ld, int32_t n, int32_t C, const int32_t* labels,
                    const uint8_t* mask, double norm, float* grad, int64_t ldg, double* row_loss,
                    double* loss_out, int32_t keep_unmasked, double* partials, void* stream) {
  if (n < 0 || C <= 0 || norm <= 0 || !loss_out || (n > 0 && (!logits || !labels || !mask || !grad || !row_loss)) ||
      (n > 16 * 1024 && !partials))
    return fail(HB_EINVAL, "hb_softmax_xent: bad arguments");
  return check(hb::launch_xent(logits, ld, n, C, labels, mask, norm, grad, ldg, row_loss, loss_out, keep_unmasked,
                               partials, S(stream)),
               "hb_softmax_xent");
}

int hb_sigmoid_bce(const float* logits, int64_t ld, int32_t n, int32_t C, const uint8_t* labels, int64_t ldl,
                   const uint8_t* mask, double norm, float* grad, int64_t ldg, double* row_loss, double* loss_out,
                   int32_t keep_unmasked, double* partials, void* stream) {
  if (n < 0 || C <= 0 || norm <= 0 || !loss_out || ldl < C ||
      (n > 0 && (!logits || !labels || !mask || !grad || !row_loss)) || (n > 16 * 1024 && !partials))
    return fail(HB_EINVAL, "hb_sigmoid_bce: bad arguments");
  return check(hb::launch_bce(logits, ld, n, C, labels, ldl, mask, norm, grad, ldg, row_loss, loss_out,
                              keep_unmasked, partials, S(stream)),
               "hb_sigmoid_bce");
}

int hb_multilabel_counts(const float* logits, int64_t ld, int32_t n, int32_t C, const uint8_t* labels, int64_t ldl,
                         const uint8_t* mask, int64_t* counts, void* stream) {
  if (n < 0 || C <= 0 || ldl < C || !counts || (n > 0 && (!logits || !labels || !mask)))
    return fail(HB_EINVAL, "hb_multilabel_counts: bad arguments");
  return check(hb::launch_multilabel_counts(logits, ld, n, C, labels, ldl, mask, counts, S(stream)),
               "hb_multilabel_counts");
}

int hb_relu(const float* z, int64_t ldz, int32_t n, int32_t d, float* y, int64_t ldy, void* stream) {
  if (n < 0 || d < 0) return fail(HB_EINVAL, "hb_relu: bad arguments");
  return check(hb::launch_relu(z, ldz, n, d, y, ldy, S(stream)), "hb_relu");
}

int hb_relu_grad_mul(const float* j, int64_t ldj, const float* h, int64_t ldh, int32_t n, int32_t d, float* m,
                     int64_t ldm, void* stream) {
  if (n < 0 || d < 0) return fail(HB_EINVAL, "hb_relu_grad_mul: bad arguments");
  return check(hb::launch_relu_grad_mul(j, ldj, h, ldh, n, d, m, ldm, S(stream)), "hb_relu_grad_mul");
}

int hb_adam_step(float* w, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                 float eps, double bc1, double bc2, void* stream) {
  if (n < 0 || bc1 <= 0 || bc2 <= 0) return fail(HB_EINVAL, "hb_adam_step: bad arguments");
  return check(hb::launch_adam(w, g, m, v, n, lr, b1, b2, eps, bc1, bc2, nullptr, nullptr, nullptr, nullptr, S(stream)),
               "hb_adam_step");
}

int hb_adam_step_guarded(float* w, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                         float eps, double bc1, double bc2, const double* loss, const uint32_t* flags,
                         const uint32_t* flags2, void* stream) {
  if (n < 0 || bc1 <= 0 || bc2 <= 0 || !loss) return fail(HB_EINVAL, "hb_adam_step_guarded: bad arguments");
  return check(hb::launch_adam(w, g, m, v, n, lr, b1, b2, eps, bc1, bc2, loss, flags, flags2, nullptr, S(stream)),
               "hb_adam_step_guarded");
}

// Per-epoch words are small (K1 tables: 40 B per message): the copy is a
// one-CTA kernel reading the pinned buffer through its device mapping, not a
// copy-engine transfer — a copy engine busy with the next step's 562 MB feature
// upload would otherwise hold the compute stream up to the end of that upload.
__global__ void fetch_host_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, int64_t bytes) {
  const bool w4 = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 3) == 0;
  const int64_t nw = w4 ? bytes >> 2 : 0;
  for (int64_t i = threadIdx.x; i < nw; i += blockDim.x)
    reinterpret_cast<uint32_t*>(dst)[i] = reinterpret_cast<const volatile uint32_t*>(src)[i];
  for (int64_t i = nw * 4 + threadIdx.x; i < bytes; i += blockDim.x)
    dst[i] = reinterpret_cast<const volatile uint8_t*>(src)[i];
}

int hb_upload_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(HB_EINVAL, "hb_upload_async: bad arguments");
  if (bytes == 0) return HB_OK;
  void* dsrc = nullptr;
  if (bytes <= (1 << 20) && cudaHostGetDevicePointer(&dsrc, const_cast<void*>(src), 0) == cudaSuccess && dsrc) {
    fetch_host_kernel<<<1, 256, 0, S(stream)>>>(static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(dsrc),
                                                bytes);
    return check(cudaGetLastError(), "hb_upload_async");
  }
  cudaGetLastError();            // not a mapped pinned buffer (or large): a copy-engine transfer
  return check(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, S(stream)), "hb_upload_async");
}

int hb_adam_step_dev(float* w, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                     float eps, const double* bc, const double* loss, const uint32_t* flags, const uint32_t* flags2,
                     void* stream) {
  if (n < 0 || !bc || !loss) return fail(HB_EINVAL, "hb_adam_step_dev: bad arguments");
  return check(hb::launch_adam(w, g, m, v, n, lr, b1, b2, eps, 1.0, 1.0, loss, flags, flags2, bc, S(stream)),
               "hb_adam_step_dev");
}

int hb_argmax_accuracy(const float* logits, int64_t ld, int32_t n, int32_t C, const int32_t* labels,
                       const uint8_t* mask, int64_t* counts, void* stream) {
  if (n < 0 || C <= 0 || !counts) return fail(HB_EINVAL, "hb_argmax_accuracy: bad arguments");
  return check(hb::launch_argmax_accuracy(logits, ld, n, C, labels, mask, counts, S(stream)),
               "hb_argmax_accuracy");
}

int hb_dropout(const float* x, int64_t ldx, int32_t nrows, int64_t row0, int32_t d, uint64_t key0, uint64_t key1,
               float p, float* out, int64_t ldo, void* stream) {
  if (nrows < 0 || d < 0 || row0 < 0 || !(p >= 0.f && p < 1.f)) return fail(HB_EINVAL, "hb_dropout: bad arguments");
  return check(hb::launch_dropout(x, ldx, nrows, row0, d, key0, key1, p, out, ldo, S(stream)), "hb_dropout");
}

int hb_ipc_get_handle(const void* ptr, void* handle, int64_t* offset) {
  if (!ptr || !handle || !offset) return fail(HB_EINVAL, "hb_ipc_get_handle: bad arguments");
  void* base = nullptr;
  cudaError_t e = hb::alloc_base(ptr, &base);
  if (e != cudaSuccess) return check(e, "hb_ipc_get_handle (allocation base)");
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, base);
  if (e != cudaSuccess) return check(e, "hb_ipc_get_handle");
  memcpy(handle, &h, sizeof(h));
  *offset = static_cast<const char*>(ptr) - static_cast<const char*>(base);
  return HB_OK;
}

int hb_ipc_open_handle(const void* handle, void** base) {
  if (!handle || !base) return fail(HB_EINVAL, "hb_ipc_open_handle: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return check(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess), "hb_ipc_open_handle");
}

int hb_ipc_close(void* base) {
  if (!base) return fail(HB_EINVAL, "hb_ipc_close: bad arguments");
  return check(cudaIpcCloseMemHandle(base), "hb_ipc_close");
}

int hb_p2p_signal(uint64_t* const* counters, int32_t n, void* stream) {
  if (n < 0 || (n > 0 && !counters)) return fail(HB_EINVAL, "hb_p2p_signal: bad arguments");
  return check(hb::launch_p2p_signal(reinterpret_cast<unsigned long long* const*>(counters), n, S(stream)),
               "hb_p2p_signal");
}

int hb_p2p_wait(const uint64_t* counter, uint64_t target, const uint64_t* target_dev, uint32_t* flags,
                uint32_t flag_bit, uint64_t timeout_ns, void* stream) {
  if (!counter) return fail(HB_EINVAL, "hb_p2p_wait: bad arguments");
  return check(hb::launch_p2p_wait(reinterpret_cast<const unsigned long long*>(counter), target,
                                   reinterpret_cast<const unsigned long long*>(target_dev), flags, flag_bit,
                                   timeout_ns, S(stream)),
               "hb_p2p_wait");
}

}  // extern "C"
