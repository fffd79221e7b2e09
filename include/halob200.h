/*
 * halob200.h — C ABI of the B200-native Sylvie halo path (libhalob200.so).
 *
 * The reference (halobit, pure Python) has no FFI: the path sits behind
 * Python call boundaries.  Each entry point below replaces one reference
 * function (cited file:line under /root/reference/pkg/src/halobit); the Python
 * host layer (paper_2303_01277_b200/) binds them with ctypes and keeps the
 * reference's names, argument meaning and exceptions.  See INTEGRATION.md.
 *
 * Conventions
 *   - All pointers are device pointers unless named h_*; sizes are element
 *     counts; matrices are row-major with an explicit leading dimension (ld,
 *     in elements).
 *   - Every call is asynchronous on `stream` (a cudaStream_t passed as void*)
 *     and returns 0 on success or a negative HB_E* code; hb_last_error()
 *     returns a thread-local message for the last failure.
 *   - No call allocates device memory; the caller (PyTorch) owns every
 *     buffer, scratch included (`work` counter pairs, xent partials, the
 *     column-scaled X copy of hb_spmm_tiled_bin).
 */
#ifndef HALOB200_H_
#define HALOB200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HB_OK 0
#define HB_EINVAL (-1)     /* bad argument (maps to CodecError / ShapeError)   */
#define HB_ECUDA (-2)      /* CUDA launch/runtime failure                        */
#define HB_ENONFINITE (-3) /* reported via the device flag word, see hb_quantize_gather */

/* Flag bits written (atomicOr) into the caller's device flag word. */
#define HB_FLAG_NONFINITE 1u

/* Wire block = the reference's QuantizedBlock.to_bytes() layout
 * (codec.py:22-25, 71-76): 12-byte header <BBHII {1, bits, 0, rows, dim},
 * rows x {f32 row_min, f32 row_scale}, rows x ceil(dim*bits/8) payload bytes.
 * bits == 32 (passthrough): header + rows*dim fp32 (the accounting basis,
 * codec.py:110-114).                                                         */
#define HB_HEADER_BYTES 12

/* Doubles of caller scratch hb_softmax_xent needs for n > 16384 rows. */
#define HB_XENT_PARTIALS 256

/* One message = one (source partition -> destination partition) block of an
 * exchange (transport.py:184-192).  40 bytes, 8-byte aligned. */
typedef struct hb_segment {
  uint64_t key0, key1;   /* Philox key of the sender's stream (rngstream.py:19-23)   */
  uint64_t elem_offset;  /* stream index of element (row 0, col 0) of this block    */
  uint64_t out;          /* device address of the block's wire image (header start) */
  int32_t row_begin;     /* first row of this block in the flattened row list       */
  int32_t num_rows;      /* rows in the block (> 0)                                  */
} hb_segment_t;

const char* hb_version(void);
const char* hb_last_error(void);

/* Replaces RngStream.uniforms (rngstream.py:38-39): out[i] = uniform of stream
 * element start+i.  Used by parity tests to pin the device generator. */
int hb_philox_uniforms(uint64_t key0, uint64_t key1, uint64_t start, int64_t n,
                       double* out, void* stream);

/* K1 — replaces the send half of exchange() (transport.py:184-192) fused with
 * the gather of _fwd_outgoing/_bwd_outgoing (trainer.py:182,199) and
 * quantize_rows + pack_code_matrix (codec.py:124-196):
 *   for every segment s, row r of s:  x = src[row_idx[s.row_begin + r] * ld + 0..d)
 *   writes the wire block of s at s.out (header written by the block's row 0).
 * bits in {1..8, 16, 32}.  Non-finite input sets HB_FLAG_NONFINITE in *flags
 * (the reference raises CodecError, codec.py:167-168; the host checks the flag
 * at the exchange boundary).  `segs` is a device array of nseg descriptors
 * sorted by row_begin. */
int hb_quantize_gather(const float* src, int64_t ld, const int32_t* row_idx, int32_t total_rows,
                       const hb_segment_t* segs, int32_t nseg, int32_t d, int32_t bits,
                       uint32_t* flags, void* stream);

/* K2 — replaces the receive half of exchange() (transport.py:195-204:
 * dequantize_rows, codec.py:199-207) fused with _assemble_halo
 * (trainer.py:208-212, accumulate = 0) or _integrate (trainer.py:214-216,
 * accumulate = 1):
 *   for i in [0, num_dst):  row t = dst_rows[i]
 *     v = accumulate ? f64(dst[t]) : 0
 *     for k in [src_ptr[i], src_ptr[i+1]):  v += dequant(received row src_rows[k])
 *     dst[t] = f32(v)
 * Received row q lives in the segment s with s.row_begin <= q < s.row_begin +
 * s.num_rows (segs sorted by row_begin); sources are listed in ascending peer
 * order, so the f64 sum follows the reference's ascending-peer integration. */
int hb_dequant_gather(const hb_segment_t* segs, int32_t nseg, int32_t num_dst,
                      const int32_t* dst_rows, const int32_t* src_ptr, const int32_t* src_rows,
                      int32_t d, int32_t bits, float* dst, int64_t ld, int32_t accumulate,
                      void* stream);

/* K3/K4 — replaces linalg.spmm (linalg.py:71-75; called at trainer.py:291,293
 * and, with the transposed block, trainer.py:318,321):
 *   Y[i, 0:d) = sum_{k in [row_ptr[i], row_ptr[i+1])} vals[k] * X[col_idx[k], 0:d)
 * (fp32, accumulated in index order). */
int hb_spmm_csr(int32_t nrows, const int64_t* row_ptr, const int32_t* col_idx, const float* vals,
                const float* X, int64_t ldx, int32_t d, float* Y, int64_t ldy, void* stream);

/* K3/K4 row-gather kernel with its knobs exposed: algo 0 = auto, 1 = row
 * gather (rows handed out in ascending chunks; d <= 128: an 8- or 16-lane
 * group owns a row, wider rows a warp; several nonzeros in flight);
 * window > 0 = nonzeros kept in flight per warp for d > 128 (tuning; 0 =
 * default); nnz = stored entries (sizes the row chunks);
 * stream_col: X rows >= stream_col (the halo copies) are referenced a few
 * times each and are read L2-evict-first, like the CSR arrays and Y, so the
 * local rows being aggregated stay L2-resident (INT32_MAX: no hint).
 * work: a device pair of int32 {next row chunk, warps finished}, zero on
 * entry and left at zero (one pair per stream serves every launch, graph
 * replays included); NULL = static grid-stride row schedule.  Same result
 * contract as hb_spmm_csr. */
int hb_spmm_csr_ex(int32_t nrows, const int64_t* row_ptr, const int32_t* col_idx, const float* vals,
                   const float* X, int64_t ldx, int32_t d, float* Y, int64_t ldy, int64_t nnz, int32_t algo,
                   int32_t window, int32_t stream_col, int32_t* work, void* stream);

/* K3/K4 tiled path (same result contract as hb_spmm_csr, fp32 accumulation
 * in tile-then-residual order).  The matrix is pre-split (ops.TiledCsr, built
 * on the device from the CSR) into dense tiles of 64 rows x 64 columns —
 * tile_ptr[b]..tile_ptr[b+1] are the tiles of row block b (nblocks =
 * ceil(nrows / 64)), tile_win[t] the tile's column window (columns
 * 64*win .. +63), tile_nz[tile_off[t] .. tile_off[t+1]) its row-sorted
 * records {int32 col - 64*win, float val} (offsets even: 16-byte aligned),
 * tile_rowoff[t*72 .. +65) the records' row offsets — and a residual CSR
 * (res_ptr / res_col / res_val over all nrows) for every other nonzero.
 * X windows (64 rows x 128/256-column panels) are staged in shared memory by
 * TMA; xrows = rows of X.  X and Y rows must be 16-byte aligned.  work: the
 * (row block, panel) item counter pair, as hb_spmm_csr_ex (required). */
int hb_spmm_tiled(int32_t nrows, int32_t xrows, int32_t nblocks, const int32_t* tile_ptr, const int32_t* tile_win,
                  const int64_t* tile_off, const uint16_t* tile_rowoff, const void* tile_nz, const int64_t* res_ptr,
                  const int32_t* res_col, const float* res_val, const float* X, int64_t ldx, int32_t d, float* Y,
                  int64_t ldy, int32_t* work, void* stream);

/* K3/K4 factored tiled path for the trainer's aggregation operators, whose
 * values are diagonal scalings of a 0/1 pattern (graph.py:120-141: SAGE mean
 * D^-1 A, its transpose A^T D^-1, GCN D^-1/2 (A+I) D^-1/2):
 *   Y[i, 0:d) = r[i] * sum_{(i,j) in pattern} c[j] * X[j, 0:d)
 * row_scale r / col_scale c may each be NULL (= 1).  Tiles are block_rows
 * (64, 120 or 128) rows x window_cols columns: 64; for d <= 48 also 128
 * (64-row blocks) or 255 (64-row blocks, or 128-row blocks with 32 < d <= 48;
 * records up to 4096 bytes per tile then) (nblocks = ceil(nrows /
 * block_rows)); a record is one byte, the column inside the tile's window;
 * tile_rec[tile_off[t] .. tile_off[t+1]) (byte offsets, multiples of 16) are
 * tile t's row-sorted records and tile_rowoff[t*R .. +block_rows+1) their
 * row offsets (R = 72 for 64-row blocks, 136 for 120 and 128); res_ptr /
 * res_col the residual pattern.  With col_scale, c X is first written to xs
 * (xrows x ldxs floats, 16-byte aligned rows).  block_order (nullable): a
 * permutation of the row blocks, the order in which the dynamically
 * scheduled work items are handed out (heaviest first balances the SMs; the
 * results do not depend on it).  fp32 accumulation, tile-then-residual order
 * (same fp32 tolerance contract as hb_spmm_csr).  work as hb_spmm_tiled. */
int hb_spmm_tiled_bin(int32_t nrows, int32_t xrows, int32_t nblocks, const int32_t* tile_ptr,
                      const int32_t* tile_win, const int64_t* tile_off, const uint16_t* tile_rowoff,
                      const uint8_t* tile_rec, const int64_t* res_ptr, const int32_t* res_col,
                      const float* row_scale, const float* col_scale, const float* X, int64_t ldx, int32_t d,
                      float* Y, int64_t ldy, float* xs, int64_t ldxs, int32_t* work, int32_t block_rows,
                      int32_t window_cols, const int32_t* block_order, void* stream);

/* K5-K7 — the dense combine GEMMs (trainer.py:294, 313, 318-321) on tcgen05
 * tensor cores with the 3xTF32 split (fp32 accuracy):
 *   C[m, n] = sum_k A(m, k) B(k, n) (+ beta * C[m, n])
 *   A(m, k) = A[m*lda_m + k*lda_k],  B(k, n) = B[k*ldb_k + n*ldb_n]  (any strides)
 * relu_out (optional, not with split-K): relu_out[m*ldr + n] = max(C[m, n], 0).
 * ws (optional, ws_floats capacity): enables a deterministic split-K for
 * small M*N with long K (the weight gradient G = P^T m).  C may be NULL with
 * beta 0 and relu_out given: only relu(A B) is stored (A-in-TMEM kernel). */
int hb_gemm_f32(int32_t M, int32_t N, int32_t K, const float* A, int64_t lda_m, int64_t lda_k,
                const float* B, int64_t ldb_k, int64_t ldb_n, float* C, int64_t ldc, float beta,
                float* relu_out, int64_t ldr, float* ws, int64_t ws_floats, void* stream);

/* Dual dense combine C = A1 B1 + A2 B2 (+ beta C), optional ReLU copy: the
 * SAGE layer z = [h | A h] [W_top; W_bot] (trainer.py:294) and its input
 * gradient j = [S | m] [W_bot^T; W_top^T] (trainer.py:318-321) without
 * materialising the concatenation.  One pass of the A-in-TMEM kernel over
 * both K ranges (C written once, never read back) when all operands are
 * TMA-describable with matching major order; otherwise two hb_gemm_f32
 * passes.  Operand conventions as hb_gemm_f32; K1, K2 > 0.  C may be NULL
 * (beta 0, relu_out given): only the ReLU copy is written — a hidden layer's
 * pre-activation is not needed after the forward; returns HB_ECUDA
 * (cudaErrorNotSupported) if the single-pass kernel cannot take the operands. */
int hb_gemm2_f32(int32_t M, int32_t N, int32_t K1, const float* A1, int64_t lda1_m, int64_t lda1_k,
                 const float* B1, int64_t ldb1_k, int64_t ldb1_n, int32_t K2, const float* A2,
                 int64_t lda2_m, int64_t lda2_k, const float* B2, int64_t ldb2_k, int64_t ldb2_n,
                 float* C, int64_t ldc, float beta, float* relu_out, int64_t ldr, float* ws,
                 int64_t ws_floats, void* stream);

/* Selects the K5-K7 kernel: 0 = TMA-fed warp-specialised tcgen05 kernel
 * whenever both operands are TMA-describable (16-byte aligned, unit stride on
 * one axis, 16-byte row stride), else the SIMT-staged tcgen05 kernel;
 * 1 = SIMT-staged kernel only (2 is not a path: the CTA-pair kernel
 * measured no faster and was removed); 3 = the A-in-TMEM kernel for every shape (A split into tf32 hi/lo in
 * registers and stored with tcgen05.st, MMAs take A from TMEM).  Under 0 the
 * A-in-TMEM kernel already runs tall GEMMs (>= 148 output tiles). */
int hb_gemm_set_path(int32_t path);

/* Tuning / test hook: the consumer layout of hb_spmm_tiled_bin for narrow
 * rows (d <= 48, 64-row blocks).  64- and 128-column windows: 0 = 8-lane
 * groups x 2 float4 (2 CTAs/SM); 1 = 4-lane groups x 3 float4, 8 consumer
 * warps x 8 rows (3 CTAs/SM) — the default; 2 / 3 = "tail pairs" (32 < d <=
 * 48): 8-lane groups read a nonzero's first 32 columns as one 128-byte
 * access and the tails of two nonzeros in a third (16 / 8 consumer warps).
 * 255-column windows: 1 or 4 (default) = tail pairs with two lane groups
 * sharing each row (record pairs round-robin: balanced run lengths), 2
 * CTAs/SM; 3 = tail pairs, a lane group per row, 2 CTAs/SM; 2 = the same,
 * 1 CTA/SM; 0 = 4-lane groups.  64- and 128-column windows treat 4 as 1. */
int hb_spmm_set_narrow(int32_t variant);

/* K8 — softmax_cross_entropy (linalg.py:87-112) on the rows of one rank:
 * grad rows outside the mask are zero, masked rows get (softmax - onehot)/norm;
 * row_loss[i] = -log softmax[label] / norm (0 outside the mask) in f64.
 * *loss_out = fixed-order sum of row_loss (deterministic two-pass reduction).
 * keep_unmasked = 1: rows outside the mask are not written (the caller's
 * grad / row_loss rows there already hold zeros, e.g. from the previous
 * epoch).  partials: HB_XENT_PARTIALS doubles of device scratch, required
 * when n > 16384 (NULL otherwise allowed). */
int hb_softmax_xent(const float* logits, int64_t ld, int32_t n, int32_t C, const int32_t* labels,
                    const uint8_t* mask, double norm, float* grad, int64_t ldg, double* row_loss,
                    double* loss_out, int32_t keep_unmasked, double* partials, void* stream);

/* Multi-label extension (not in the reference, whose only loss is the
 * softmax CE; used for the Yelp-shaped "multilabel 100" config):
 * masked sigmoid binary cross-entropy over C labels, labels[i*ldl + c] in
 * {0, 1}: row_loss[i] = sum_c [max(z,0) - z y + log1p(exp(-|z|))] / (norm C),
 * grad = (sigmoid(z) - y) / (norm C) (0 outside the mask), f64 math;
 * *loss_out, keep_unmasked and partials as hb_softmax_xent. */
int hb_sigmoid_bce(const float* logits, int64_t ld, int32_t n, int32_t C, const uint8_t* labels, int64_t ldl,
                   const uint8_t* mask, double norm, float* grad, int64_t ldg, double* row_loss,
                   double* loss_out, int32_t keep_unmasked, double* partials, void* stream);

/* Multi-label evaluation counts (prediction z > 0) per mask value k = 1..3:
 * counts[3(k-1)] true positives, +1 false positives, +2 false negatives. */
int hb_multilabel_counts(const float* logits, int64_t ld, int32_t n, int32_t C, const uint8_t* labels,
                         int64_t ldl, const uint8_t* mask, int64_t* counts, void* stream);

/* ReLU epilogue (linalg.py:78-80): y = max(z, 0), in place allowed. */
int hb_relu(const float* z, int64_t ldz, int32_t n, int32_t d, float* y, int64_t ldy, void* stream);

/* relu_grad (linalg.py:83-84) fused with the product m = j * (h > 0)
 * (trainer.py:312), where h = relu(z) of the same layer. */
int hb_relu_grad_mul(const float* j, int64_t ldj, const float* h, int64_t ldh, int32_t n, int32_t d,
                     float* m, int64_t ldm, void* stream);

/* adam_step (linalg.py:115-140), bias corrections bc1 = 1-b1^t, bc2 = 1-b2^t. */
int hb_adam_step(float* w, const float* g, float* m, float* v, int64_t n, float lr, float b1,
                 float b2, float eps, double bc1, double bc2, void* stream);

/* hb_adam_step that skips the update on the device when *loss (device f64)
 * is not finite or a flag word (flags, flags2: device words, nullable) is
 * non-zero: the reference's check before Adam (trainer.py:361-366) without a
 * host synchronisation, so an epoch's loss can be read back after the next
 * epoch is issued (a failed epoch leaves the weights untouched, as the
 * reference's abort does). */
int hb_adam_step_guarded(float* w, const float* g, float* m, float* v, int64_t n, float lr, float b1,
                         float b2, float eps, double bc1, double bc2, const double* loss,
                         const uint32_t* flags, const uint32_t* flags2, void* stream);

/* Stream-ordered copy of `bytes` from PINNED host memory to the device: the
 * per-epoch words (K1 descriptor tables with the epoch's Philox keys, Adam's
 * bias corrections).  Up to 1 MiB from a mapped pinned buffer it is a one-CTA
 * kernel reading the buffer through its device mapping (no copy engine, so it
 * never queues behind a large feature upload on another stream); otherwise a
 * cudaMemcpyAsync.  Inside a CUDA-graph capture it becomes a node that reads
 * the host buffer when the graph replays. */
int hb_upload_async(void* dst, const void* src, int64_t bytes, void* stream);

/* hb_adam_step_guarded with the bias corrections read from device memory
 * (bc[0] = 1-b1^t, bc[1] = 1-b2^t, f64): the launch's arguments no longer
 * change from epoch to epoch, so a captured CUDA graph of the epoch replays it
 * (the host uploads bc with the epoch's other per-epoch words). */
int hb_adam_step_dev(float* w, const float* g, float* m, float* v, int64_t n, float lr, float b1,
                     float b2, float eps, const double* bc, const double* loss, const uint32_t* flags,
                     const uint32_t* flags2, void* stream);

/* ---- peer-memory halo exchange (N > 1, one process per GPU) ---------------
 * Replaces the NCCL send/recv of `exchange` (transport.py:172-205): every
 * rank's receive buffers are exported once as CUDA IPC handles and mapped by
 * the other ranks, K1 writes remote messages straight into the receiver's
 * buffer over NVLink, and 64-bit counters order arrival and reuse.
 *
 * hb_ipc_get_handle: the 64-byte cudaIpcMemHandle of the allocation holding
 * ptr, and ptr's byte offset in it.  hb_ipc_open_handle / hb_ipc_close: map /
 * unmap a peer's allocation (base address; add the offset). */
int hb_ipc_get_handle(const void* ptr, void* handle, int64_t* offset);
int hb_ipc_open_handle(const void* handle, void** base);
int hb_ipc_close(void* base);

/* Stream-ordered: after the work queued before it, atomically add 1 to each
 * of the n counters (device array of n pointers, peer-mapped addresses
 * allowed) with system-scope release semantics. */
int hb_p2p_signal(uint64_t* const* counters, int32_t n, void* stream);

/* Stream-ordered: block the stream until *counter >= target (system-scope
 * acquire); target_dev (nullable, device memory) overrides target, so a
 * captured CUDA graph can wait for a different count each replay.  After
 * timeout_ns the wait gives up and ORs flag_bit into *flags (nullable) — a
 * stalled or diverged peer surfaces as an error at the next host check
 * instead of a hung GPU. */
int hb_p2p_wait(const uint64_t* counter, uint64_t target, const uint64_t* target_dev, uint32_t* flags,
                uint32_t flag_bit, uint64_t timeout_ns, void* stream);

/* Argmax accuracy counts for evaluate() (trainer.py:129-144):
 * counts[2*k] = #rows with mask==k+1, counts[2*k+1] = #correct among them, k=0..2. */
int hb_argmax_accuracy(const float* logits, int64_t ld, int32_t n, int32_t C, const int32_t* labels,
                       const uint8_t* mask, int64_t* counts, void* stream);

/* Dropout on h~ (trainer.py:285-289, 322-323): keep = u >= p, drawn from the
 * keyed stream (seed, "dropout", part, epoch, layer) over h~ of shape
 * (nl+nh, d) in row-major order; out = keep ? x / (1-p) : 0.  Row r of this
 * call is row (row0 + r) of the partition's h~, so the forward (on h~) and
 * the backward (on j_full) regenerate the identical mask. */
int hb_dropout(const float* x, int64_t ldx, int32_t nrows, int64_t row0, int32_t d, uint64_t key0,
               uint64_t key1, float p, float* out, int64_t ldo, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HALOB200_H_ */
