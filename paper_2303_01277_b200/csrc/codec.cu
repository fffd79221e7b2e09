// K1 (gather + quantize + pack) and K2 (unpack + dequantize + gather/scatter)
// of the Sylvie Low-bit Module, bit-exact with halobit's codec.
//
// Reference semantics (halobit/codec.py:158-207, transport.py:184-204):
//   row_min   = f32(min(x)),  row_scale = f32((f64(max) - f64(min)) / B)
//   code      = clip(floor(h) + (u < h - floor(h)), 0, B),
//   h         = (f64(x) - f64(row_min)) / f64(row_scale)     (rows with scale > 0)
//   u         = uniform of stream element (elem_offset + r*d + c)
//   payload   = codes LSB-first, row padded to whole bytes (codec.py:124-134)
//   dequant   = f64(scale) * code + f64(min)
//
// Layout choices (B200-first):
//  * one warp per gathered row; the row (d <= 1149 fp32) stays in registers
//    between the min/max pass and the quantize pass, so HBM is read once;
//  * lanes are laid out in the *Philox frame*: lane j of chunk t owns Philox
//    block (e_row/4 + 32t + j), i.e. columns 128t + 4j - delta + {0..3} with
//    delta = e_row % 4 — every lane computes exactly one Philox4x64-10 block per
//    4 elements and no block is computed twice;
//  * h is evaluated in fp32 with a rigorous error bound; only elements whose
//    rounding decision could differ from the fp64 reference (near-integer h or
//    u within the bound of frac(h)) take the exact fp64 path;
//  * codes are OR-ed into a per-warp shared-memory row image (any bit width,
//    any row alignment), then written to the wire block with coalesced stores.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include "common.cuh"
#include "philox.cuh"

namespace hb {

constexpr int kQWarps = 8;                 // warps per CTA in K1/K2
constexpr int kMaxSmemSegs = 128;          // segment table cached in smem
constexpr int kK1SmallWords = 320;         // per-warp row image: pow2 b<=8 up to d=1149, b=16 up to d~600
constexpr int kK1LargeWords = 1160;        // b <= 16 up to d = 2300

__device__ __forceinline__ int find_segment_smem(const int32_t* begin, int nseg, int row) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (begin[mid] <= row) lo = mid; else hi = mid - 1;
  }
  return lo;
}

struct QuantRowCtx {
  float mn, s, inv_s, E, Eu;
  int B, bits;
  bool live, fast;
};

// Exact fp64 reference decision (codec.py:185-193); rarely executed.
__device__ __noinline__ int quant_exact(float x, float mn, float s, int B, uint64_t w) {
  const double D = __dsub_rn((double)x, (double)mn);
  const double h = __ddiv_rn(D, (double)s);
  const double f = floor(h);
  const double fr = __dsub_rn(h, f);
  const double u = u53_to_double(w);
  const int code = (int)f + (u < fr ? 1 : 0);
  return min(max(code, 0), B);
}

// fp32 decision + "ambiguous" flag.  With |h32 - h64| <= E (rigorous bound for
// the fp32 evaluation) and u in [ut, ut + 2^-23):
//   * floor(h) is certain unless frac(h32) is within E of an integer;
//   * (u < frac) is certain unless |frac32 - ut| < E + 2^-22.
// Ambiguous elements are recomputed with the exact fp64 path.
__device__ __forceinline__ int quant_fast(float x, const QuantRowCtx& q, uint64_t w, bool& amb) {
  const float xm = __fsub_rn(x, q.mn);
  const float h = __fmul_rn(xm, q.inv_s);
  const float fl = floorf(h);
  const float fr = __fsub_rn(h, fl);
  const float ut = __fsub_rn(__uint_as_float(((uint32_t)(w >> 32) >> 9) | 0x3f800000u), 1.0f);
  amb = (x != q.mn) & ((fr <= q.E) | (fr >= 1.0f - q.E) | (fabsf(__fsub_rn(fr, ut)) <= q.Eu) |
                        !(h < 8388608.0f));
  const int code = (int)fl + (ut < fr ? 1 : 0);
  return min(max(code, 0), q.B);
}

// b = 1: h in [0, 1 + eps]; a non-ambiguous element has floor(h) = 0, so the
// code is just (u < h).
// 1 bit: code = clip(floor(hbar) + (u < hbar - floor(hbar)), 0, 1) = (u < hbar)
// for hbar in [0, 1) and 1 for hbar >= 1.  With |h - hbar| <= E and
// ut <= u < ut + 2^-23, the fp32 decision (ut < h) can only differ from the
// exact one when |h - ut| <= Eu = E + 2^-22 — including at the row maximum
// (hbar ~ 1: ut <= 1 - 2^-23, so ut < h unless they are within Eu) and near
// the minimum — so that single test routes every undecidable element to the
// f64 path.
// 1 bit: code = (u < h), exact unless |h - ut| <= Eu.  x == row_min gives
// h == 0 exactly and code 0 on both paths, so it needs no exclusion here
// (it only reaches the exact path when ut <= Eu, probability ~1e-6).
__device__ __forceinline__ uint32_t quant_fast_b1(float x, const QuantRowCtx& q, uint64_t w, bool& amb) {
  const float h = __fmul_rn(__fsub_rn(x, q.mn), q.inv_s);
  const float ut = __fsub_rn(__uint_as_float(((uint32_t)(w >> 32) >> 9) | 0x3f800000u), 1.0f);
  amb = fabsf(__fsub_rn(h, ut)) <= q.Eu;
  return ut < h ? 1u : 0u;
}

// General b, no clamp needed: a non-ambiguous element has floor(h) <= B - 1.
__device__ __forceinline__ uint32_t quant_fast_nc(float x, const QuantRowCtx& q, uint64_t w, bool& amb) {
  const float h = __fmul_rn(__fsub_rn(x, q.mn), q.inv_s);
  const float fl = floorf(h);
  const float fr = __fsub_rn(h, fl);
  const float ut = __fsub_rn(__uint_as_float(((uint32_t)(w >> 32) >> 9) | 0x3f800000u), 1.0f);
  amb = (x != q.mn) & ((fr <= q.E) | (fr >= 1.0f - q.E) | (fabsf(__fsub_rn(fr, ut)) <= q.Eu) |
                        !(h < 8388608.0f));
  const float cf = __fadd_rn(fl, ut < fr ? 1.0f : 0.0f);
  return __float_as_uint(__fadd_rn(cf, 8388608.0f)) & 0x7fffffu;   // exact small integer
}

__device__ __forceinline__ float sel4(const float (&a)[4], int k) {
  return k == 0 ? a[0] : (k == 1 ? a[1] : (k == 2 ? a[2] : a[3]));
}

__device__ __forceinline__ void write_header(uint8_t* out, int bits, int rows, int d) {
  out[0] = 1;
  out[1] = (uint8_t)bits;
  out[2] = 0;
  out[3] = 0;
  for (int k = 0; k < 4; ++k) out[4 + k] = (uint8_t)((uint32_t)rows >> (8 * k));
  for (int k = 0; k < 4; ++k) out[8 + k] = (uint8_t)((uint32_t)d >> (8 * k));
}

// K1, register-lean layout (occupancy matters: Philox4x64-10 is a chain of
// dependent 64-bit multiplies, so the SM needs many warps in flight).
//   pass 1: stream the row once (128-bit loads) for min / max / finiteness;
//   pass 2: per 128-column chunk, each lane computes one Philox block (4
//           uniforms), re-reads its 4 columns (L1 hits) in the Philox frame,
//           quantizes and packs.
// MAXW: row-image words per warp in shared memory (bounds d).
//
// Packing: for bits in {1, 2, 4, 8} each lane's 4 codes form a 4b-bit field;
// a shuffle-OR over 8/b lanes assembles 32-bit words of the chunk image
// (chunk bit q = 4b*lane + b*i + j), stored to a per-warp smem array; the row
// image is then the chunk stream shifted right by delta*b bits (the Philox
// frame starts delta columns before the row).  Other widths OR codes into the
// smem row image with shared-memory atomics.
template <bool B1, int MAXW>
__global__ void __launch_bounds__(kQWarps * 32, 4)
quantize_gather_kernel(const float* __restrict__ src, int64_t ld, const int32_t* __restrict__ row_idx,
                       int total_rows, const hb_segment_t* __restrict__ segs_g, int nseg, int d,
                       int bits, uint32_t* __restrict__ flags) {
  __shared__ hb_segment_t segs_s[kMaxSmemSegs];
  __shared__ int32_t seg_begin[kMaxSmemSegs];
  __shared__ uint32_t rowbuf[kQWarps][MAXW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool smem_segs = nseg <= kMaxSmemSegs;
  if (smem_segs) {
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
      segs_s[i] = segs_g[i];
      seg_begin[i] = segs_g[i].row_begin;
    }
    __syncthreads();
  }
  const int B = (1 << bits) - 1;
  const int rb = (d * bits + 7) >> 3;
  const bool pow2 = bits <= 8 && (bits & (bits - 1)) == 0;
  const bool vec = ((ld & 3) == 0) && ((((uintptr_t)src) & 15) == 0);
  uint32_t* buf = rowbuf[warp];

  for (int row = blockIdx.x * kQWarps + warp; row < total_rows; row += gridDim.x * kQWarps) {
    const int si = smem_segs ? find_segment_smem(seg_begin, nseg, row) : find_segment(segs_g, nseg, row);
    const hb_segment_t sg = smem_segs ? segs_s[si] : segs_g[si];
    const int r = row - sg.row_begin;
    const float* __restrict__ x = src + (int64_t)row_idx[row] * ld;
    const uint64_t e_row = sg.elem_offset + (uint64_t)r * (uint64_t)d;
    const int delta = (int)(e_row & 3ull);
    const uint64_t blk0 = e_row >> 2;
    const int nchunks = (d + delta + 127) >> 7;
    uint8_t* out = reinterpret_cast<uint8_t*>(sg.out);

    // ---- pass 1: min / max / finiteness ---------------------------------------
    float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
    bool bad = false;
    if (vec) {
      const int d4 = d >> 2;
      for (int k = lane; k < d4; k += 32) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(x) + k);
        mn = fminf(fminf(mn, a.x), fminf(a.y, fminf(a.z, a.w)));
        mx = fmaxf(fmaxf(mx, a.x), fmaxf(a.y, fmaxf(a.z, a.w)));
        bad |= !(isfinite(a.x) & isfinite(a.y) & isfinite(a.z) & isfinite(a.w));
      }
      for (int c = 4 * d4 + lane; c < d; c += 32) {
        const float a = __ldg(x + c);
        mn = fminf(mn, a);
        mx = fmaxf(mx, a);
        bad |= !isfinite(a);
      }
    } else {
      for (int c = lane; c < d; c += 32) {
        const float a = __ldg(x + c);
        mn = fminf(mn, a);
        mx = fmaxf(mx, a);
        bad |= !isfinite(a);
      }
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    if (__any_sync(0xffffffffu, bad)) {
      if (lane == 0) atomicOr(flags, HB_FLAG_NONFINITE);
      continue;  // the host raises CodecError; the block contents are undefined
    }
    if (r == 0 && lane == 0) write_header(out, bits, sg.num_rows, d);

    if (bits == 32) {  // passthrough: fp32 rows after the header (no metadata)
      float* prow = reinterpret_cast<float*>(out + HB_HEADER_BYTES) + (int64_t)r * d;
      for (int c = lane; c < d; c += 32) prow[c] = __ldg(x + c);
      continue;
    }

    QuantRowCtx q;
    q.bits = bits;
    q.B = B;
    q.mn = mn;
    q.s = __double2float_rn(__ddiv_rn(__dsub_rn((double)mx, (double)mn), (double)B));
    q.live = q.s > 0.0f;
    q.inv_s = q.live ? __frcp_rn(q.s) : 0.f;
    q.fast = q.live && q.s >= 7.888609052210118e-31f /* 2^-100 */ &&
             fabsf(mn) <= 1.2676506002282294e30f && fabsf(mx) <= 1.2676506002282294e30f;
    q.E = (float)(B + 2) * 2.384185791015625e-07f;  // (B+2) * 2^-22
    q.Eu = q.E + 2.384185791015625e-07f;
    if (lane == 0) {
      *reinterpret_cast<float*>(out + HB_HEADER_BYTES + 8 * (int64_t)r) = q.mn;
      *reinterpret_cast<float*>(out + HB_HEADER_BYTES + 8 * (int64_t)r + 4) = q.s;
    }
    uint8_t* pay = out + HB_HEADER_BYTES + 8 * (int64_t)sg.num_rows + (int64_t)r * rb;

    // ---- pass 2: Philox + quantize + pack --------------------------------------
    const int nw_chunk = 4 * bits;                          // chunk image words (pow2 path)
    if (!pow2) {
      const int buf_words = ((64 + bits * (nchunks * 128)) >> 5) + 3;
      for (int k = lane; k < buf_words; k += 32) buf[k] = 0u;
      __syncwarp();
    }
    for (int t = 0; t < nchunks; ++t) {
      uint32_t field = 0, field_hi = 0;
      if (q.live) {
        const U64x4 u = philox4x64_10(blk0 + (uint64_t)(32 * t + lane) + 1ull, sg.key0, sg.key1);
        const int c0 = 128 * t + 4 * lane - delta;
        const bool full = q.fast && (128 * t - delta >= 0) && (128 * t - delta + 128 <= d);
        uint32_t code[4];
        bool amb[4];
        if (full) {
          const float xv[4] = {__ldg(x + c0), __ldg(x + c0 + 1), __ldg(x + c0 + 2), __ldg(x + c0 + 3)};
          const uint64_t ws[4] = {u.w0, u.w1, u.w2, u.w3};
#pragma unroll
          for (int i = 0; i < 4; ++i)
            code[i] = B1 ? quant_fast_b1(xv[i], q, ws[i], amb[i]) : quant_fast_nc(xv[i], q, ws[i], amb[i]);
        } else {
          const uint64_t ws[4] = {u.w0, u.w1, u.w2, u.w3};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int c = c0 + i;
            amb[i] = false;
            code[i] = 0;
            if (c >= 0 && c < d) {
              const float xv = __ldg(x + c);
              if (q.fast) code[i] = B1 ? quant_fast_b1(xv, q, ws[i], amb[i]) : quant_fast_nc(xv, q, ws[i], amb[i]);
              else amb[i] = true;
            }
          }
        }
        if (__any_sync(0xffffffffu, amb[0] | amb[1] | amb[2] | amb[3])) {
          const uint64_t ws[4] = {u.w0, u.w1, u.w2, u.w3};
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (amb[i]) code[i] = (uint32_t)quant_exact(__ldg(x + c0 + i), q.mn, q.s, q.B, ws[i]);
        }
        if (bits <= 8) {
#pragma unroll
          for (int i = 0; i < 4; ++i) field |= code[i] << (i * bits);
        } else {  // bits == 16
          field = code[0] | (code[1] << 16);
          field_hi = code[2] | (code[3] << 16);
        }
      }
      if (pow2) {
        // chunk image word k = OR of fields of lanes [k*L, (k+1)*L), L = 8/bits
        // L = 8 / bits lanes share a word: shifts, not a runtime division
        const int lgL = B1 ? 3 : 3 - (__ffs(bits) - 1);
        const int L = 1 << lgL;
        uint32_t w = field << ((4 * bits) * (lane & (L - 1)));
        if (L >= 2) w |= __shfl_xor_sync(0xffffffffu, w, 1);
        if (L >= 4) w |= __shfl_xor_sync(0xffffffffu, w, 2);
        if (L >= 8) w |= __shfl_xor_sync(0xffffffffu, w, 4);
        if ((lane & (L - 1)) == 0) buf[nw_chunk * t + (lane >> lgL)] = w;
      } else if (field | field_hi) {
        const int c0 = 128 * t + 4 * lane - delta;
        const int pos = 64 + bits * c0;                     // >= 16 for bits <= 16
        const int wd = pos >> 5, sh = pos & 31;
        const uint64_t f64v = (uint64_t)field | ((uint64_t)field_hi << 32);
        const uint64_t lo = f64v << sh;
        atomicOr(&buf[wd], (uint32_t)lo);
        if ((uint32_t)(lo >> 32)) atomicOr(&buf[wd + 1], (uint32_t)(lo >> 32));
        if (sh && (f64v >> (64 - sh))) atomicOr(&buf[wd + 2], (uint32_t)(f64v >> (64 - sh)));
      }
    }
    __syncwarp();
    // ---- emit the row image ------------------------------------------------------
    const int nrw = (rb + 3) >> 2;                            // row words
    const bool wordstore = ((((uintptr_t)pay) & 3) == 0) && ((rb & 3) == 0);
    if (pow2) {
      const int sh = delta * bits;                            // 0..24
      const int total_w = nw_chunk * nchunks;
      for (int m = lane; m < nrw; m += 32) {
        const uint32_t lo = buf[m];
        const uint32_t hi = (m + 1 < total_w) ? buf[m + 1] : 0u;
        const uint32_t rw = sh ? ((lo >> sh) | (hi << (32 - sh))) : lo;
        if (wordstore) {
          reinterpret_cast<uint32_t*>(pay)[m] = rw;
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (4 * m + k < rb) pay[4 * m + k] = (uint8_t)(rw >> (8 * k));
        }
      }
    } else {
      const uint8_t* img = reinterpret_cast<const uint8_t*>(buf) + 8;
      if (wordstore) {
        const uint32_t* iw = buf + 2;
        for (int k = lane; k < nrw; k += 32) reinterpret_cast<uint32_t*>(pay)[k] = iw[k];
      } else {
        for (int k = lane; k < rb; k += 32) pay[k] = img[k];
      }
    }
    __syncwarp();
  }
}

// K1 with TMA staging: each warp streams its rows through two shared-memory
// row buffers filled by 1-D bulk async copies (cp.async.bulk + mbarrier), one
// row ahead, so HBM latency hides behind the Philox work of the current row
// and the row is read from HBM exactly once (128-bit bulk transfers).
// Requires ld % 4 == 0 and a 16-byte aligned source.
template <bool B1, int MINB>
__global__ void __launch_bounds__(kQWarps * 32, MINB)
quantize_gather_tma_kernel(const float* __restrict__ src, int64_t ld, const int32_t* __restrict__ row_idx,
                           int total_rows, const hb_segment_t* __restrict__ segs_g, int nseg, int d,
                           int bits, uint32_t* __restrict__ flags, int ldr, int imgw) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ hb_segment_t segs_s[kMaxSmemSegs];
  __shared__ int32_t seg_begin[kMaxSmemSegs];
  __shared__ __align__(8) uint64_t bars[kQWarps][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool smem_segs = nseg <= kMaxSmemSegs;
  if (smem_segs) {
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
      segs_s[i] = segs_g[i];
      seg_begin[i] = segs_g[i].row_begin;
    }
  }
  float* rows_s = reinterpret_cast<float*>(dsm + (size_t)warp * (2 * ldr * 4 + imgw * 4));
  uint32_t* buf = reinterpret_cast<uint32_t*>(rows_s + 2 * ldr);
  if (lane == 0) {
    mbar_init(&bars[warp][0], 1);
    mbar_init(&bars[warp][1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int B = (1 << bits) - 1;
  const int rb = (d * bits + 7) >> 3;
  const bool pow2 = bits <= 8 && (bits & (bits - 1)) == 0;
  const uint32_t bytes = (uint32_t)(((d + 3) & ~3) * 4);
  const int stride = gridDim.x * kQWarps;
  uint32_t phase_bits = 0u;          // bit s = parity of barrier s (a register, not local memory)
  int cseg = 0;

  int row = blockIdx.x * kQWarps + warp;
  if (row < total_rows && lane == 0) {
    mbar_expect_tx(&bars[warp][0], bytes);
    tma_load_1d(rows_s, src + (int64_t)__ldg(row_idx + row) * ld, bytes, &bars[warp][0]);
  }
  for (int k = 0; row < total_rows; row += stride, ++k) {
    const int cur = k & 1;
    const int nxt = row + stride;
    if (nxt < total_rows && lane == 0) {
      fence_proxy_async_smem();
      mbar_expect_tx(&bars[warp][cur ^ 1], bytes);
      tma_load_1d(rows_s + (cur ^ 1) * ldr, src + (int64_t)__ldg(row_idx + nxt) * ld, bytes,
                  &bars[warp][cur ^ 1]);
    }
    // rows are visited in ascending order: try the previous segment first
    if (smem_segs) {
      if (!(row >= seg_begin[cseg] && (cseg + 1 >= nseg || row < seg_begin[cseg + 1])))
        cseg = find_segment_smem(seg_begin, nseg, row);
    } else {
      cseg = find_segment(segs_g, nseg, row);
    }
    const int si = cseg;
    const hb_segment_t sg = smem_segs ? segs_s[si] : segs_g[si];
    const int r = row - sg.row_begin;
    const uint64_t e_row = sg.elem_offset + (uint64_t)r * (uint64_t)d;
    const int delta = (int)(e_row & 3ull);
    const uint64_t blk0 = e_row >> 2;
    const int nchunks = (d + delta + 127) >> 7;
    uint8_t* out = reinterpret_cast<uint8_t*>(sg.out);
    const float* xs = rows_s + cur * ldr;
    mbar_wait(&bars[warp][cur], (phase_bits >> cur) & 1u);
    phase_bits ^= 1u << cur;

    // ---- pass 1 (smem): min / max / finiteness ----------------------------------
    float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
    bool bad = false;
    const int d4 = d >> 2;
    for (int c4 = lane; c4 < d4; c4 += 32) {
      const float4 a = reinterpret_cast<const float4*>(xs)[c4];
      mn = fminf(fminf(mn, a.x), fminf(a.y, fminf(a.z, a.w)));
      mx = fmaxf(fmaxf(mx, a.x), fmaxf(a.y, fmaxf(a.z, a.w)));
      bad |= !(isfinite(a.x) & isfinite(a.y) & isfinite(a.z) & isfinite(a.w));
    }
    for (int c = 4 * d4 + lane; c < d; c += 32) {
      const float a = xs[c];
      mn = fminf(mn, a);
      mx = fmaxf(mx, a);
      bad |= !isfinite(a);
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    if (__any_sync(0xffffffffu, bad)) {
      if (lane == 0) atomicOr(flags, HB_FLAG_NONFINITE);
      __syncwarp();
      continue;  // the host raises CodecError; the block contents are undefined
    }
    if (r == 0 && lane == 0) write_header(out, bits, sg.num_rows, d);
    QuantRowCtx q;
    q.bits = bits;
    q.B = B;
    q.mn = mn;
    q.s = __double2float_rn(__ddiv_rn(__dsub_rn((double)mx, (double)mn), (double)B));
    q.live = q.s > 0.0f;
    q.inv_s = q.live ? __frcp_rn(q.s) : 0.f;
    q.fast = q.live && q.s >= 7.888609052210118e-31f /* 2^-100 */ &&
             fabsf(mn) <= 1.2676506002282294e30f && fabsf(mx) <= 1.2676506002282294e30f;
    q.E = (float)(B + 2) * 2.384185791015625e-07f;  // (B+2) * 2^-22
    q.Eu = q.E + 2.384185791015625e-07f;
    if (lane == 0) {
      *reinterpret_cast<float*>(out + HB_HEADER_BYTES + 8 * (int64_t)r) = q.mn;
      *reinterpret_cast<float*>(out + HB_HEADER_BYTES + 8 * (int64_t)r + 4) = q.s;
    }
    uint8_t* pay = out + HB_HEADER_BYTES + 8 * (int64_t)sg.num_rows + (int64_t)r * rb;

    // ---- pass 2: Philox + quantize + pack --------------------------------------
    const int nw_chunk = 4 * bits;
    if (!pow2) {
      const int buf_words = ((64 + bits * (nchunks * 128)) >> 5) + 3;
      for (int w = lane; w < buf_words; w += 32) buf[w] = 0u;
      __syncwarp();
    }
    for (int t = 0; t < nchunks; ++t) {
      uint32_t field = 0, field_hi = 0;
      if (q.live) {
        const U64x4 u = philox4x64_10(blk0 + (uint64_t)(32 * t + lane) + 1ull, sg.key0, sg.key1);
        const uint64_t ws[4] = {u.w0, u.w1, u.w2, u.w3};
        const int c0 = 128 * t + 4 * lane - delta;
        const bool full = q.fast && (128 * t - delta >= 0) && (128 * t - delta + 128 <= d);
        uint32_t code[4];
        bool amb[4];
        if (full) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            code[i] = B1 ? quant_fast_b1(xs[c0 + i], q, ws[i], amb[i]) : quant_fast_nc(xs[c0 + i], q, ws[i], amb[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int c = c0 + i;
            amb[i] = false;
            code[i] = 0;
            if (c >= 0 && c < d) {
              if (q.fast) code[i] = B1 ? quant_fast_b1(xs[c], q, ws[i], amb[i]) : quant_fast_nc(xs[c], q, ws[i], amb[i]);
              else amb[i] = true;
            }
          }
        }
        if (__any_sync(0xffffffffu, amb[0] | amb[1] | amb[2] | amb[3])) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (amb[i]) code[i] = (uint32_t)quant_exact(xs[c0 + i], q.mn, q.s, q.B, ws[i]);
        }
        if (bits <= 8) {
#pragma unroll
          for (int i = 0; i < 4; ++i) field |= code[i] << (i * bits);
        } else {  // bits == 16
          field = code[0] | (code[1] << 16);
          field_hi = code[2] | (code[3] << 16);
        }
      }
      if (pow2) {
        // L = 8 / bits lanes share a word: shifts, not a runtime division
        const int lgL = B1 ? 3 : 3 - (__ffs(bits) - 1);
        const int L = 1 << lgL;
        uint32_t w = field << ((4 * bits) * (lane & (L - 1)));
        if (L >= 2) w |= __shfl_xor_sync(0xffffffffu, w, 1);
        if (L >= 4) w |= __shfl_xor_sync(0xffffffffu, w, 2);
        if (L >= 8) w |= __shfl_xor_sync(0xffffffffu, w, 4);
        if ((lane & (L - 1)) == 0) buf[nw_chunk * t + (lane >> lgL)] = w;
      } else if (field | field_hi) {
        const int c0 = 128 * t + 4 * lane - delta;
        const int pos = 64 + bits * c0;
        const int wd = pos >> 5, sh = pos & 31;
        const uint64_t f64v = (uint64_t)field | ((uint64_t)field_hi << 32);
        const uint64_t lo = f64v << sh;
        atomicOr(&buf[wd], (uint32_t)lo);
        if ((uint32_t)(lo >> 32)) atomicOr(&buf[wd + 1], (uint32_t)(lo >> 32));
        if (sh && (f64v >> (64 - sh))) atomicOr(&buf[wd + 2], (uint32_t)(f64v >> (64 - sh)));
      }
    }
    __syncwarp();
    const int nrw = (rb + 3) >> 2;
    const bool wordstore = ((((uintptr_t)pay) & 3) == 0) && ((rb & 3) == 0);
    if (pow2) {
      const int sh = delta * bits;
      const int total_w = nw_chunk * nchunks;
      for (int m = lane; m < nrw; m += 32) {
        const uint32_t lo = buf[m];
        const uint32_t hi = (m + 1 < total_w) ? buf[m + 1] : 0u;
        const uint32_t rw = sh ? ((lo >> sh) | (hi << (32 - sh))) : lo;
        if (wordstore) {
          reinterpret_cast<uint32_t*>(pay)[m] = rw;
        } else {
#pragma unroll
          for (int b4 = 0; b4 < 4; ++b4)
            if (4 * m + b4 < rb) pay[4 * m + b4] = (uint8_t)(rw >> (8 * b4));
        }
      }
    } else {
      const uint8_t* img = reinterpret_cast<const uint8_t*>(buf) + 8;
      if (wordstore) {
        const uint32_t* iw = buf + 2;
        for (int w = lane; w < nrw; w += 32) reinterpret_cast<uint32_t*>(pay)[w] = iw[w];
      } else {
        for (int w = lane; w < rb; w += 32) pay[w] = img[w];
      }
    }
    __syncwarp();
  }
}

// K1, 1-bit: two rows per warp, one per 16-lane half.  The per-row work that
// does not scale with d (segment lookup, TMA issue, min/max reductions, the
// f64 scale, metadata) is shared by the two rows of a warp instruction, and
// each lane runs two interleaved Philox4x64-10 blocks (64-column chunks in
// pairs) for twice the multiply-chain ILP.  Each half streams its rows through
// two TMA-filled smem row buffers, one row ahead, like the 32-lane kernel.
template <int MAXT, int MINB, int NBUF>
__global__ void __launch_bounds__(MAXT, MINB)
quantize_b1_hw_kernel(const float* __restrict__ src, int64_t ld, const int32_t* __restrict__ row_idx,
                      int total_rows, const hb_segment_t* __restrict__ segs_g, int nseg, int d,
                      uint32_t* __restrict__ flags, int ldr, int imgw) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ hb_segment_t segs_s[kMaxSmemSegs];
  __shared__ int32_t seg_begin[kMaxSmemSegs + 1];
  __shared__ __align__(8) uint64_t bars[kQWarps][2][2];   // [warp][half][buffer]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hw = lane >> 4, hl = lane & 15;
  for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
    segs_s[i] = segs_g[i];
    seg_begin[i] = segs_g[i].row_begin;
  }
  if (threadIdx.x == 0) seg_begin[nseg] = 0x7fffffff;
  const size_t per_half = (size_t)NBUF * ldr * 4 + (size_t)imgw * 4;
  float* rows_s = reinterpret_cast<float*>(dsm + (size_t)(2 * warp + hw) * per_half);
  uint32_t* buf = reinterpret_cast<uint32_t*>(rows_s + NBUF * ldr);
  if (hl == 0) {
    mbar_init(&bars[warp][hw][0], 1);
    mbar_init(&bars[warp][hw][1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const unsigned hmask = 0xffffu << (16 * hw);
  const int rb = (d + 7) >> 3;
  const uint32_t bytes = (uint32_t)(((d + 3) & ~3) * 4);
  const int nwarps = blockDim.x >> 5;                           // <= kQWarps
  // blocked rows per half-warp: consecutive rows stay in one message (the
  // cached segment hits) and their gather indices are neighbours
  const int nhalves = gridDim.x * nwarps * 2;
  const int chunk = (total_rows + nhalves - 1) / nhalves;
  const int hid = (blockIdx.x * nwarps + warp) * 2 + hw;
  const int row_end = min(total_rows, (hid + 1) * chunk);
  const int stride = 1;
  uint32_t phase_bits = 0u;
  int cseg = 0;
  int row = hid * chunk;
  if (row < row_end && hl == 0) {
    mbar_expect_tx(&bars[warp][hw][0], bytes);
    tma_load_1d(rows_s, src + (int64_t)__ldg(row_idx + row) * ld, bytes, &bars[warp][hw][0]);
  }
  for (int k = 0;; row += stride, ++k) {
    const bool active = row < row_end;
    if (!__any_sync(0xffffffffu, active)) break;
    const int cur = NBUF == 2 ? (k & 1) : 0;
    const int nxt = row + stride;
    if (NBUF == 2 && nxt < row_end && hl == 0) {
      fence_proxy_async_smem();
      mbar_expect_tx(&bars[warp][hw][cur ^ 1], bytes);
      tma_load_1d(rows_s + (cur ^ 1) * ldr, src + (int64_t)__ldg(row_idx + nxt) * ld, bytes,
                  &bars[warp][hw][cur ^ 1]);
    }
    if (NBUF == 1 && k > 0 && active && hl == 0) {
      // single buffer: this row's load is issued once the previous row's
      // passes are done with the buffer (other warps cover its latency)
      fence_proxy_async_smem();
      mbar_expect_tx(&bars[warp][hw][0], bytes);
      tma_load_1d(rows_s, src + (int64_t)__ldg(row_idx + row) * ld, bytes, &bars[warp][hw][0]);
    }
    if (active && !(row >= seg_begin[cseg] && row < seg_begin[cseg + 1]))
      cseg = find_segment_smem(seg_begin, nseg, row);
    const hb_segment_t& sg = segs_s[cseg];
    const int r = row - sg.row_begin;
    const uint64_t e_row = sg.elem_offset + (uint64_t)r * (uint64_t)d;
    const int delta = (int)(e_row & 3ull);
    const uint64_t blk0 = e_row >> 2;
    const int nch = (d + delta + 63) >> 6;                        // 64-column chunks of this half
    const int nch2 = max(nch, __shfl_xor_sync(0xffffffffu, nch, 16));
    uint8_t* out = reinterpret_cast<uint8_t*>(sg.out);
    const float* xs = rows_s + cur * ldr;
    if (active) {
      mbar_wait(&bars[warp][hw][cur], (phase_bits >> cur) & 1u);
      phase_bits ^= 1u << cur;
    }
    __syncwarp();

    // ---- pass 1 (smem): min / max / finiteness, reduced within the half --------
    float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
    bool bad = false;
    if (active) {
      const int d4 = d >> 2;
      for (int c4 = hl; c4 < d4; c4 += 16) {
        const float4 a = reinterpret_cast<const float4*>(xs)[c4];
        mn = fminf(fminf(mn, a.x), fminf(a.y, fminf(a.z, a.w)));
        mx = fmaxf(fmaxf(mx, a.x), fmaxf(a.y, fmaxf(a.z, a.w)));
        bad |= !(isfinite(a.x) & isfinite(a.y) & isfinite(a.z) & isfinite(a.w));
      }
      for (int c = 4 * d4 + hl; c < d; c += 16) {
        const float a = xs[c];
        mn = fminf(mn, a);
        mx = fmaxf(mx, a);
        bad |= !isfinite(a);
      }
    }
#pragma unroll
    for (int o = 8; o; o >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const bool badh = (__ballot_sync(0xffffffffu, bad) & hmask) != 0u;
    if (badh && active && hl == 0) atomicOr(flags, HB_FLAG_NONFINITE);
    const bool live_row = active && !badh;
    if (live_row && r == 0 && hl == 0) write_header(out, 1, sg.num_rows, d);
    QuantRowCtx q;
    q.bits = 1;
    q.B = 1;
    q.mn = mn;
    q.s = live_row ? __double2float_rn(__dsub_rn((double)mx, (double)mn)) : 0.f;
    q.live = q.s > 0.0f;
    q.inv_s = q.live ? __frcp_rn(q.s) : 0.f;
    q.fast = q.live && q.s >= 7.888609052210118e-31f && fabsf(mn) <= 1.2676506002282294e30f &&
             fabsf(mx) <= 1.2676506002282294e30f;
    q.E = 3.0f * 2.384185791015625e-07f;                          // (B+2) * 2^-22
    q.Eu = q.E + 2.384185791015625e-07f;
    if (live_row && hl == 0) {
      *reinterpret_cast<float*>(out + HB_HEADER_BYTES + 8 * (int64_t)r) = q.mn;
      *reinterpret_cast<float*>(out + HB_HEADER_BYTES + 8 * (int64_t)r + 4) = q.s;
    }

    // ---- pass 2: chunk pairs, two interleaved Philox blocks per lane ------------
    for (int t = 0; t < nch2; t += 2) {
      uint32_t f2[2] = {0u, 0u};
      if (q.live) {
        U64x4 ua, ub;
        philox4x64_10_x2(blk0 + (uint64_t)(16 * t + hl) + 1ull, blk0 + (uint64_t)(16 * (t + 1) + hl) + 1ull,
                         sg.key0, sg.key1, ua, ub);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const U64x4& u = j ? ub : ua;
          const uint64_t ws[4] = {u.w0, u.w1, u.w2, u.w3};
          const int tt = t + j;
          const int c0 = 64 * tt + 4 * hl - delta;
          const bool full = q.fast && (64 * tt - delta >= 0) && (64 * tt - delta + 64 <= d);
          uint32_t code[4];
          bool amb[4];
          if (full) {
#pragma unroll
            for (int i = 0; i < 4; ++i) code[i] = quant_fast_b1(xs[c0 + i], q, ws[i], amb[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int c = c0 + i;
              amb[i] = false;
              code[i] = 0;
              if (c >= 0 && c < d) {
                if (q.fast) code[i] = quant_fast_b1(xs[c], q, ws[i], amb[i]);
                else amb[i] = true;
              }
            }
          }
          if (amb[0] | amb[1] | amb[2] | amb[3]) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (amb[i]) code[i] = (uint32_t)quant_exact(xs[c0 + i], q.mn, q.s, 1, ws[i]);
          }
          f2[j] = code[0] | (code[1] << 1) | (code[2] << 2) | (code[3] << 3);
        }
      }
      // 64-bit chunk image = 16 lanes x 4 bits: word (hl >> 3) from lanes 8w .. 8w+7
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        uint32_t w = f2[j] << (4 * (hl & 7));
        w |= __shfl_xor_sync(0xffffffffu, w, 1);
        w |= __shfl_xor_sync(0xffffffffu, w, 2);
        w |= __shfl_xor_sync(0xffffffffu, w, 4);
        if ((hl & 7) == 0 && t + j < nch) buf[2 * (t + j) + (hl >> 3)] = w;
      }
    }
    __syncwarp();
    // ---- emit the row image (the Philox frame starts delta columns early) --------
    if (live_row) {
      uint8_t* pay = out + HB_HEADER_BYTES + 8 * (int64_t)sg.num_rows + (int64_t)r * rb;
      const int nrw = (rb + 3) >> 2;
      const int total_w = 2 * nch;
      const bool wordstore = ((((uintptr_t)pay) & 3) == 0) && ((rb & 3) == 0);
      for (int m = hl; m < nrw; m += 16) {
        const uint32_t lo = buf[m];
        const uint32_t hi = (m + 1 < total_w) ? buf[m + 1] : 0u;
        const uint32_t rw = delta ? ((lo >> delta) | (hi << (32 - delta))) : lo;
        if (wordstore) {
          reinterpret_cast<uint32_t*>(pay)[m] = rw;
        } else {
#pragma unroll
          for (int b4 = 0; b4 < 4; ++b4)
            if (4 * m + b4 < rb) pay[4 * m + b4] = (uint8_t)(rw >> (8 * b4));
        }
      }
    }
    __syncwarp();
  }
}

// Generic per-element path (rows wider than the smem row image).
__global__ void __launch_bounds__(kQWarps * 32)
quantize_gather_wide_kernel(const float* __restrict__ src, int64_t ld, const int32_t* __restrict__ row_idx,
                            int total_rows, const hb_segment_t* __restrict__ segs, int nseg, int d,
                            int bits, uint32_t* __restrict__ flags) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int B = (1 << bits) - 1;
  const int rb = (d * bits + 7) >> 3;
  for (int row = blockIdx.x * kQWarps + warp; row < total_rows; row += gridDim.x * kQWarps) {
    const hb_segment_t sg = segs[find_segment(segs, nseg, row)];
    const int r = row - sg.row_begin;
    const float* x = src + (int64_t)row_idx[row] * ld;
    const uint64_t e_row = sg.elem_offset + (uint64_t)r * (uint64_t)d;
    uint8_t* out = reinterpret_cast<uint8_t*>(sg.out);
    float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
    bool bad = false;
    for (int c = lane; c < d; c += 32) {
      const float a = __ldg(x + c);
      mn = fminf(mn, a);
      mx = fmaxf(mx, a);
      bad |= !isfinite(a);
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    if (__any_sync(0xffffffffu, bad)) {
      if (lane == 0) atomicOr(flags, HB_FLAG_NONFINITE);
      continue;
    }
    if (r == 0 && lane == 0) write_header(out, bits, sg.num_rows, d);
    if (bits == 32) {
      float* prow = reinterpret_cast<float*>(out + HB_HEADER_BYTES) + (int64_t)r * d;
      for (int c = lane; c < d; c += 32) prow[c] = __ldg(x + c);
      continue;
    }
    const float s = __double2float_rn(__ddiv_rn(__dsub_rn((double)mx, (double)mn), (double)B));
    if (lane == 0) {
      *reinterpret_cast<float*>(out + HB_HEADER_BYTES + 8 * (int64_t)r) = mn;
      *reinterpret_cast<float*>(out + HB_HEADER_BYTES + 8 * (int64_t)r + 4) = s;
    }
    uint8_t* pay = out + HB_HEADER_BYTES + 8 * (int64_t)sg.num_rows + (int64_t)r * rb;
    for (int byte = lane; byte < rb; byte += 32) {
      uint32_t acc = 0;
      const int c_first = (byte * 8) / bits, c_last = min(d - 1, (byte * 8 + 7) / bits);
      for (int c = c_first; c <= c_last; ++c) {
        int code = 0;
        if (s > 0.0f) {
          const uint64_t e = e_row + (uint64_t)c;
          const U64x4 u = philox4x64_10((e >> 2) + 1, sg.key0, sg.key1);
          code = quant_exact(__ldg(x + c), mn, s, B, pick(u, (int)(e & 3)));
        }
        const int pos = c * bits - byte * 8;  // may be negative for straddling codes
        acc |= pos >= 0 ? ((uint32_t)code << pos) : ((uint32_t)code >> (-pos));
      }
      pay[byte] = (uint8_t)(acc & 0xffu);
    }
  }
}

// ----------------------------------------------------------------------------
// K2: per destination row, sum (in f64, ascending peer order) the dequantized
// received rows listed for it, optionally on top of the current row.
__device__ __forceinline__ void codes4(const uint8_t* __restrict__ p, int rb, int c0, int bits,
                                       int d, int code[4]) {
  if (bits == 16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = c0 + i;
      code[i] = c < d ? (int)(p[2 * c] | ((uint32_t)p[2 * c + 1] << 8)) : 0;
    }
    return;
  }
  const int bit0 = c0 * bits;
  const int byte0 = bit0 >> 3;
  const int nb = ((bit0 & 7) + 4 * bits + 7) >> 3;  // <= 5
  uint64_t win = 0;
#pragma unroll
  for (int k = 0; k < 5; ++k)
    if (k < nb && byte0 + k < rb) win |= (uint64_t)p[byte0 + k] << (8 * k);
  win >>= (bit0 & 7);
  const uint32_t m = (1u << bits) - 1u;
#pragma unroll
  for (int i = 0; i < 4; ++i) code[i] = (int)((win >> (i * bits)) & m);
}

__global__ void __launch_bounds__(kQWarps * 32)
dequant_gather_kernel(const hb_segment_t* __restrict__ segs_g, int nseg, int num_dst,
                      const int32_t* __restrict__ dst_rows, const int32_t* __restrict__ src_ptr,
                      const int32_t* __restrict__ src_rows, int d, int bits, float* __restrict__ dst,
                      int64_t ld, int accumulate) {
  __shared__ hb_segment_t segs_s[kMaxSmemSegs];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool smem_segs = nseg <= kMaxSmemSegs;
  if (smem_segs) {
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) segs_s[i] = segs_g[i];
    __syncthreads();
  }
  const hb_segment_t* segs = smem_segs ? segs_s : segs_g;
  const int rb = bits == 32 ? 4 * d : (d * bits + 7) >> 3;
  const bool vec = ((ld & 3) == 0) && ((((uintptr_t)dst) & 15) == 0);

  for (int i = blockIdx.x * kQWarps + warp; i < num_dst; i += gridDim.x * kQWarps) {
    float* out = dst + (int64_t)dst_rows[i] * ld;
    const int k0 = src_ptr[i], k1 = src_ptr[i + 1];
    for (int cb = 0; cb < d; cb += 128) {
      const int c0 = cb + 4 * lane;
      if (c0 >= d) continue;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      const bool full = c0 + 3 < d;
      if (accumulate) {
        if (vec && full) {
          const float4 o = *reinterpret_cast<const float4*>(out + c0);
          acc[0] = o.x; acc[1] = o.y; acc[2] = o.z; acc[3] = o.w;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (c0 + e < d) acc[e] = out[c0 + e];
        }
      }
      for (int k = k0; k < k1; ++k) {
        const int q = src_rows[k];
        const hb_segment_t sg = segs[find_segment(segs, nseg, q)];
        const int r = q - sg.row_begin;
        const uint8_t* blk = reinterpret_cast<const uint8_t*>(sg.out);
        if (bits == 32) {
          const float* prow = reinterpret_cast<const float*>(blk + HB_HEADER_BYTES) + (int64_t)r * d;
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (c0 + e < d) acc[e] = __dadd_rn(acc[e], (double)prow[c0 + e]);
          continue;
        }
        const float mn = *reinterpret_cast<const float*>(blk + HB_HEADER_BYTES + 8 * (int64_t)r);
        const float sc = *reinterpret_cast<const float*>(blk + HB_HEADER_BYTES + 8 * (int64_t)r + 4);
        const uint8_t* pay = blk + HB_HEADER_BYTES + 8 * (int64_t)sg.num_rows + (int64_t)r * rb;
        int code[4];
        codes4(pay, rb, c0, bits, d, code);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          acc[e] = __dadd_rn(acc[e], __dadd_rn(__dmul_rn((double)sc, (double)code[e]), (double)mn));
      }
      if (vec && full) {
        *reinterpret_cast<float4*>(out + c0) =
            make_float4(__double2float_rn(acc[0]), __double2float_rn(acc[1]),
                        __double2float_rn(acc[2]), __double2float_rn(acc[3]));
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (c0 + e < d) out[c0 + e] = __double2float_rn(acc[e]);
      }
    }
  }
}

// K2, restructured for latency: the received row's metadata is read once per
// (destination, source) and the lane walks all of its 128-column chunks;
// the segment of a received row is found from a per-warp cached segment
// (received rows are visited in ascending order) before falling back to the
// binary search.  Forward 1-bit rows take an fp32 path that is bit-identical
// to the f64 formula (f32(f64(sc)*c + f64(mn)) == __fadd_rn(sc, mn) for c = 1:
// two fp32 operands, so the f64 sum is exact or rounds far below an fp32
// half-ulp); everything else accumulates in f64 exactly as before.
template <int NCH, bool FAST1>
__global__ void __launch_bounds__(kQWarps * 32)
dequant_rows_kernel(const hb_segment_t* __restrict__ segs_g, int nseg, int num_dst,
                    const int32_t* __restrict__ dst_rows, const int32_t* __restrict__ src_ptr,
                    const int32_t* __restrict__ src_rows, int d, int bits, float* __restrict__ dst,
                    int64_t ld, int accumulate) {
  __shared__ hb_segment_t segs_s[kMaxSmemSegs];
  __shared__ int32_t seg_begin[kMaxSmemSegs + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
    segs_s[i] = segs_g[i];
    seg_begin[i] = segs_g[i].row_begin;
  }
  if (threadIdx.x == 0) seg_begin[nseg] = 0x7fffffff;
  __syncthreads();
  const int rb = bits == 32 ? 4 * d : (d * bits + 7) >> 3;
  const bool vec = ((ld & 3) == 0) && ((((uintptr_t)dst) & 15) == 0);
  constexpr bool fast1 = FAST1;     // caller guarantees !accumulate && bits == 1
  constexpr int NA = FAST1 ? 1 : NCH;
  int cs = 0;
  for (int i = blockIdx.x * kQWarps + warp; i < num_dst; i += gridDim.x * kQWarps) {
    float* out = dst + (int64_t)dst_rows[i] * ld;
    const int k0 = src_ptr[i], k1 = src_ptr[i + 1];
    if (FAST1 && k1 - k0 != 1) {
      // several (or no) received rows for one destination: chunk-wise f64 sum
      for (int c0 = 4 * lane; c0 < d; c0 += 128) {
        double a4[4] = {0.0, 0.0, 0.0, 0.0};
        for (int k = k0; k < k1; ++k) {
          const int q = src_rows[k];
          const hb_segment_t& sg = segs_s[find_segment_smem(seg_begin, nseg, q)];
          const int r = q - sg.row_begin;
          const uint8_t* blk = reinterpret_cast<const uint8_t*>(sg.out);
          const float* mp = reinterpret_cast<const float*>(blk + HB_HEADER_BYTES + 8 * (int64_t)r);  // 4-byte aligned
          const float2 meta = make_float2(mp[0], mp[1]);
          const uint8_t* pay = blk + HB_HEADER_BYTES + 8 * (int64_t)sg.num_rows + (int64_t)r * rb;
          int code[4];
          codes4(pay, rb, c0, 1, d, code);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            a4[e] = __dadd_rn(a4[e], __dadd_rn(__dmul_rn((double)meta.y, (double)code[e]), (double)meta.x));
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (c0 + e < d) out[c0 + e] = __double2float_rn(a4[e]);
      }
      continue;
    }
    double acc[NA][4];
#pragma unroll
    for (int ch = 0; ch < NA; ++ch)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = ch * 128 + 4 * lane + e;
        acc[ch][e] = (!FAST1 && accumulate && c < d) ? (double)out[c] : 0.0;
      }
    for (int k = k0; k < k1; ++k) {
      const int q = src_rows[k];
      if (!(q >= seg_begin[cs] && q < seg_begin[cs + 1])) cs = find_segment_smem(seg_begin, nseg, q);
      const hb_segment_t& sg = segs_s[cs];
      const int r = q - sg.row_begin;
      const uint8_t* blk = reinterpret_cast<const uint8_t*>(sg.out);
      if (!FAST1 && bits == 32) {
        const float* prow = reinterpret_cast<const float*>(blk + HB_HEADER_BYTES) + (int64_t)r * d;
#pragma unroll
        for (int ch = 0; ch < NA; ++ch)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c = ch * 128 + 4 * lane + e;
            if (c < d) acc[ch][e] = __dadd_rn(acc[ch][e], (double)prow[c]);
          }
        continue;
      }
      const float* mp = reinterpret_cast<const float*>(blk + HB_HEADER_BYTES + 8 * (int64_t)r);  // 4-byte aligned
          const float2 meta = make_float2(mp[0], mp[1]);
      const uint8_t* pay = blk + HB_HEADER_BYTES + 8 * (int64_t)sg.num_rows + (int64_t)r * rb;
      if (fast1) {
        const float one = __fadd_rn(meta.y, meta.x);
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const int c0 = ch * 128 + 4 * lane;
          if (c0 >= d) continue;
          const uint32_t nib = (uint32_t)(pay[c0 >> 3] >> (c0 & 7));
          const float4 v = make_float4((nib & 1u) ? one : meta.x, (nib & 2u) ? one : meta.x,
                                       (nib & 4u) ? one : meta.x, (nib & 8u) ? one : meta.x);
          if (vec && c0 + 3 < d) {
            *reinterpret_cast<float4*>(out + c0) = v;
          } else {
            out[c0] = v.x;
            if (c0 + 1 < d) out[c0 + 1] = v.y;
            if (c0 + 2 < d) out[c0 + 2] = v.z;
            if (c0 + 3 < d) out[c0 + 3] = v.w;
          }
        }
        continue;
      }
#pragma unroll
      for (int ch = 0; ch < NA; ++ch) {
        const int c0 = ch * 128 + 4 * lane;
        if (c0 >= d) continue;
        int code[4];
        codes4(pay, rb, c0, bits, d, code);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          acc[ch][e] = __dadd_rn(acc[ch][e], __dadd_rn(__dmul_rn((double)meta.y, (double)code[e]), (double)meta.x));
      }
    }
    if (FAST1) continue;     // stored directly
#pragma unroll
    for (int ch = 0; ch < NA; ++ch) {
      const int c0 = ch * 128 + 4 * lane;
      if (c0 >= d) continue;
      if (vec && c0 + 3 < d) {
        *reinterpret_cast<float4*>(out + c0) =
            make_float4(__double2float_rn(acc[ch][0]), __double2float_rn(acc[ch][1]),
                        __double2float_rn(acc[ch][2]), __double2float_rn(acc[ch][3]));
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (c0 + e < d) out[c0 + e] = __double2float_rn(acc[ch][e]);
      }
    }
  }
}

// K2 forward, 1 bit, batched: a warp takes 32 consecutive destinations at a
// time, lane l resolves destination l (indices, segment, metadata, payload
// pointer) with independent loads, and the rows are then written one after
// another from register broadcasts — the dependent index/metadata chain is
// paid once per 32 rows instead of once per row.  Values are bit-identical to
// dequant_rows_kernel's fp32 fast path.
template <int NCH>
__global__ void __launch_bounds__(kQWarps * 32)
dequant_b1_batched_kernel(const hb_segment_t* __restrict__ segs_g, int nseg, int num_dst,
                          const int32_t* __restrict__ dst_rows, const int32_t* __restrict__ src_ptr,
                          const int32_t* __restrict__ src_rows, int d, float* __restrict__ dst, int64_t ld) {
  __shared__ hb_segment_t segs_s[kMaxSmemSegs];
  __shared__ int32_t seg_begin[kMaxSmemSegs + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
    segs_s[i] = segs_g[i];
    seg_begin[i] = segs_g[i].row_begin;
  }
  if (threadIdx.x == 0) seg_begin[nseg] = 0x7fffffff;
  __syncthreads();
  const int rb = (d + 7) >> 3;
  const bool vec = ((ld & 3) == 0) && ((((uintptr_t)dst) & 15) == 0);
  int cs = 0;
  for (int i0 = (blockIdx.x * kQWarps + warp) * 32; i0 < num_dst; i0 += gridDim.x * kQWarps * 32) {
    const int i = i0 + lane;
    const bool valid = i < num_dst;
    const int my_t = valid ? dst_rows[i] : 0;
    const int my_k0 = valid ? src_ptr[i] : 0;
    const int my_k1 = valid ? src_ptr[i + 1] : 0;
    const bool my_single = valid && my_k1 - my_k0 == 1;
    const int my_q = my_single ? src_rows[my_k0] : 0;
    if (my_single && !(my_q >= seg_begin[cs] && my_q < seg_begin[cs + 1]))
      cs = find_segment_smem(seg_begin, nseg, my_q);
    float my_mn = 0.f, my_one = 0.f;
    uint64_t my_pay = 0;
    if (my_single) {
      const hb_segment_t& sg = segs_s[cs];
      const int r = my_q - sg.row_begin;
      const uint8_t* blk = reinterpret_cast<const uint8_t*>(sg.out);
      const float* mp = reinterpret_cast<const float*>(blk + HB_HEADER_BYTES + 8 * (int64_t)r);
      my_mn = mp[0];
      my_one = __fadd_rn(mp[1], my_mn);
      my_pay = reinterpret_cast<uint64_t>(blk + HB_HEADER_BYTES + 8 * (int64_t)sg.num_rows + (int64_t)r * rb);
    }
    const unsigned singles = __ballot_sync(0xffffffffu, my_single);
    const int n = min(32, num_dst - i0);
    // rows of a warp's batch are written U at a time: the payload bytes of all
    // U rows are loaded before the first store, so the load latency is paid
    // once per U rows (U = 1 for wide rows: the byte registers would spill)
    constexpr int U = NCH <= 2 ? 4 : (NCH <= 5 ? 2 : 1);
    for (int j0 = 0; j0 < n; j0 += U) {
      uint32_t bits[U][NCH];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + u;
        const uint8_t* pay = reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, my_pay, j & 31));
        const bool ld_ok = j < n && ((singles >> (j & 31)) & 1u);
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const int c0 = ch * 128 + 4 * lane;
          bits[u][ch] = (ld_ok && c0 < d) ? (uint32_t)__ldg(pay + (c0 >> 3)) : 0u;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + u;
        if (j >= n) break;
        const int t = __shfl_sync(0xffffffffu, my_t, j);
        float* out = dst + (int64_t)t * ld;
        if (!((singles >> j) & 1u)) {
          // zero or several received rows for this destination: chunk-wise f64 sum
          const int k0 = __shfl_sync(0xffffffffu, my_k0, j), k1 = __shfl_sync(0xffffffffu, my_k1, j);
          for (int c0 = 4 * lane; c0 < d; c0 += 128) {
            double a4[4] = {0.0, 0.0, 0.0, 0.0};
            for (int k = k0; k < k1; ++k) {
              const int q = src_rows[k];
              const hb_segment_t& sg = segs_s[find_segment_smem(seg_begin, nseg, q)];
              const int r = q - sg.row_begin;
              const uint8_t* blk = reinterpret_cast<const uint8_t*>(sg.out);
              const float* mp = reinterpret_cast<const float*>(blk + HB_HEADER_BYTES + 8 * (int64_t)r);
              const uint8_t* pay = blk + HB_HEADER_BYTES + 8 * (int64_t)sg.num_rows + (int64_t)r * rb;
              int code[4];
              codes4(pay, rb, c0, 1, d, code);
#pragma unroll
              for (int e = 0; e < 4; ++e)
                a4[e] = __dadd_rn(a4[e], __dadd_rn(__dmul_rn((double)mp[1], (double)code[e]), (double)mp[0]));
            }
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (c0 + e < d) out[c0 + e] = __double2float_rn(a4[e]);
          }
          continue;
        }
        const float mn = __shfl_sync(0xffffffffu, my_mn, j);
        const float one = __shfl_sync(0xffffffffu, my_one, j);
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const int c0 = ch * 128 + 4 * lane;
          if (c0 >= d) continue;
          const uint32_t nib = bits[u][ch] >> (c0 & 7);
          const float4 v = make_float4((nib & 1u) ? one : mn, (nib & 2u) ? one : mn, (nib & 4u) ? one : mn,
                                       (nib & 8u) ? one : mn);
          if (vec && c0 + 3 < d) {
            *reinterpret_cast<float4*>(out + c0) = v;
          } else {
            out[c0] = v.x;
            if (c0 + 1 < d) out[c0 + 1] = v.y;
            if (c0 + 2 < d) out[c0 + 2] = v.z;
            if (c0 + 3 < d) out[c0 + 3] = v.w;
          }
        }
      }
    }
  }
}

// K2 general (any b <= 16, overwrite or ascending-peer accumulate), batched
// like dequant_b1_batched_kernel: 32 destinations per warp; their received
// rows are contiguous in src_rows, so a sliding window of 32 sources is
// resolved lane-parallel (segment, metadata, payload pointer) and broadcast.
// Per element: f64(sc) * code + f64(mn) (separate mul and add), summed in
// f64 on top of the current value when accumulating, one fp32 rounding —
// exactly dequant_rows_kernel's arithmetic.
template <int NCH>
__global__ void __launch_bounds__(kQWarps * 32)
dequant_batched_kernel(const hb_segment_t* __restrict__ segs_g, int nseg, int num_dst,
                       const int32_t* __restrict__ dst_rows, const int32_t* __restrict__ src_ptr,
                       const int32_t* __restrict__ src_rows, int d, int bits, float* __restrict__ dst,
                       int64_t ld, int accumulate) {
  __shared__ hb_segment_t segs_s[kMaxSmemSegs];
  __shared__ int32_t seg_begin[kMaxSmemSegs + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
    segs_s[i] = segs_g[i];
    seg_begin[i] = segs_g[i].row_begin;
  }
  if (threadIdx.x == 0) seg_begin[nseg] = 0x7fffffff;
  __syncthreads();
  const int rb = (d * bits + 7) >> 3;
  const bool vec = ((ld & 3) == 0) && ((((uintptr_t)dst) & 15) == 0);
  int cs = 0;
  float my_mn = 0.f, my_sc = 0.f;
  uint64_t my_pay = 0;
  auto prepare = [&](int w0, int s1) {
    const int k = w0 + lane;
    my_mn = 0.f;
    my_sc = 0.f;
    my_pay = 0;
    if (k < s1) {
      const int q = src_rows[k];
      if (!(q >= seg_begin[cs] && q < seg_begin[cs + 1])) cs = find_segment_smem(seg_begin, nseg, q);
      const hb_segment_t& sg = segs_s[cs];
      const int r = q - sg.row_begin;
      const uint8_t* blk = reinterpret_cast<const uint8_t*>(sg.out);
      const float* mp = reinterpret_cast<const float*>(blk + HB_HEADER_BYTES + 8 * (int64_t)r);
      my_mn = mp[0];
      my_sc = mp[1];
      my_pay = reinterpret_cast<uint64_t>(blk + HB_HEADER_BYTES + 8 * (int64_t)sg.num_rows + (int64_t)r * rb);
    }
  };
  for (int i0 = (blockIdx.x * kQWarps + warp) * 32; i0 < num_dst; i0 += gridDim.x * kQWarps * 32) {
    const int i = i0 + lane;
    const bool valid = i < num_dst;
    const int my_t = valid ? dst_rows[i] : 0;
    const int my_k0 = valid ? src_ptr[i] : 0;
    const int my_k1 = valid ? src_ptr[i + 1] : 0;
    const int n = min(32, num_dst - i0);
    const int s0 = __shfl_sync(0xffffffffu, my_k0, 0);
    const int s1 = __shfl_sync(0xffffffffu, my_k1, n - 1);
    int w0 = s0;
    prepare(w0, s1);
    for (int j = 0; j < n; ++j) {
      const int t = __shfl_sync(0xffffffffu, my_t, j);
      const int k0 = __shfl_sync(0xffffffffu, my_k0, j), k1 = __shfl_sync(0xffffffffu, my_k1, j);
      float* out = dst + (int64_t)t * ld;
      double acc[NCH][4];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int c = ch * 128 + 4 * lane + e;
          acc[ch][e] = (accumulate && c < d) ? (double)out[c] : 0.0;
        }
      for (int k = k0; k < k1; ++k) {
        if (k >= w0 + 32) {           // warp-uniform: slide the source window
          w0 = k;
          prepare(w0, s1);
        }
        const int sl = k - w0;
        const double mn = (double)__shfl_sync(0xffffffffu, my_mn, sl);
        const double sc = (double)__shfl_sync(0xffffffffu, my_sc, sl);
        const uint8_t* pay = reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, my_pay, sl));
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const int c0 = ch * 128 + 4 * lane;
          if (c0 >= d) continue;
          int code[4];
          codes4(pay, rb, c0, bits, d, code);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            acc[ch][e] = __dadd_rn(acc[ch][e], __dadd_rn(__dmul_rn(sc, (double)code[e]), mn));
        }
      }
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int c0 = ch * 128 + 4 * lane;
        if (c0 >= d) continue;
        if (vec && c0 + 3 < d) {
          *reinterpret_cast<float4*>(out + c0) =
              make_float4(__double2float_rn(acc[ch][0]), __double2float_rn(acc[ch][1]),
                          __double2float_rn(acc[ch][2]), __double2float_rn(acc[ch][3]));
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (c0 + e < d) out[c0 + e] = __double2float_rn(acc[ch][e]);
        }
      }
    }
  }
}

// K2 backward, 1 bit, ascending-peer accumulate (trainer.py:339-350 order):
// out[t] = fp32( f64(out[t]) + sum_k (f64(sc_k) * code + f64(mn_k)) ), the
// same operation sequence as dequant_batched_kernel — with code in {0, 1} the
// per-source term is one of two per-source constants v0 = 0 + mn, v1 = sc + mn
// (f64 mul by 0/1 is exact), so each element costs one f64 add per source.
// The destination rows' current values are read as float4 one row ahead of
// the row being accumulated (software-pipelined), so the read-modify-write
// latency of consecutive rows overlaps.
template <int NCH>
__global__ void __launch_bounds__(kQWarps * 32)
dequant_b1_acc_kernel(const hb_segment_t* __restrict__ segs_g, int nseg, int num_dst,
                      const int32_t* __restrict__ dst_rows, const int32_t* __restrict__ src_ptr,
                      const int32_t* __restrict__ src_rows, int d, float* __restrict__ dst, int64_t ld) {
  __shared__ hb_segment_t segs_s[kMaxSmemSegs];
  __shared__ int32_t seg_begin[kMaxSmemSegs + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
    segs_s[i] = segs_g[i];
    seg_begin[i] = segs_g[i].row_begin;
  }
  if (threadIdx.x == 0) seg_begin[nseg] = 0x7fffffff;
  __syncthreads();
  const int rb = (d + 7) >> 3;
  int cs = 0;
  float my_mn = 0.f, my_sc = 0.f;
  uint64_t my_pay = 0;
  auto prepare = [&](int w0, int s1) {
    const int k = w0 + lane;
    my_mn = 0.f;
    my_sc = 0.f;
    my_pay = 0;
    if (k < s1) {
      const int q = src_rows[k];
      if (!(q >= seg_begin[cs] && q < seg_begin[cs + 1])) cs = find_segment_smem(seg_begin, nseg, q);
      const hb_segment_t& sg = segs_s[cs];
      const int r = q - sg.row_begin;
      const uint8_t* blk = reinterpret_cast<const uint8_t*>(sg.out);
      const float* mp = reinterpret_cast<const float*>(blk + HB_HEADER_BYTES + 8 * (int64_t)r);
      my_mn = mp[0];
      my_sc = mp[1];
      my_pay = reinterpret_cast<uint64_t>(blk + HB_HEADER_BYTES + 8 * (int64_t)sg.num_rows + (int64_t)r * rb);
    }
  };
  auto load_row = [&](int t, float4 (&o)[NCH]) {
    const float* row = dst + (int64_t)t * ld;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      const int c0 = ch * 128 + 4 * lane;
      o[ch] = c0 + 3 < d ? *reinterpret_cast<const float4*>(row + c0)
                         : make_float4(c0 < d ? row[c0] : 0.f, c0 + 1 < d ? row[c0 + 1] : 0.f,
                                       c0 + 2 < d ? row[c0 + 2] : 0.f, 0.f);
    }
  };
  for (int i0 = (blockIdx.x * kQWarps + warp) * 32; i0 < num_dst; i0 += gridDim.x * kQWarps * 32) {
    const int i = i0 + lane;
    const bool valid = i < num_dst;
    const int my_t = valid ? dst_rows[i] : 0;
    const int my_k0 = valid ? src_ptr[i] : 0;
    const int my_k1 = valid ? src_ptr[i + 1] : 0;
    const int n = min(32, num_dst - i0);
    const int s0 = __shfl_sync(0xffffffffu, my_k0, 0);
    const int s1 = __shfl_sync(0xffffffffu, my_k1, n - 1);
    int w0 = s0;
    prepare(w0, s1);
    float4 cur[NCH];
    load_row(__shfl_sync(0xffffffffu, my_t, 0), cur);
    // the first source's payload bits of the next row are fetched while the
    // current row accumulates (most destinations have a single source)
    auto first_bits = [&](int jj, uint32_t (&nb)[NCH]) -> bool {
      const int ka = __shfl_sync(0xffffffffu, my_k0, jj), kb = __shfl_sync(0xffffffffu, my_k1, jj);
      if (!(ka < kb && ka >= w0 && ka < w0 + 32)) return false;      // warp-uniform
      const uint8_t* pay = reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, my_pay, ka - w0));
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int c0 = ch * 128 + 4 * lane;
        // the raw byte: shifting here would make the prefetch wait for its load
        nb[ch] = c0 < d ? (uint32_t)__ldg(pay + (c0 >> 3)) : 0u;
      }
      return true;
    };
    uint32_t nib_cur[NCH];
    bool have_cur = first_bits(0, nib_cur);
    // narrow rows (NCH <= 2) keep two rows in flight ahead of the one being
    // accumulated (nxt = j + 1 loaded one iteration early, nn = j + 2)
    constexpr bool kTwo = NCH <= 2;
    float4 nxt[NCH];
    uint32_t nib_nxt[NCH];
    bool have_nxt = false;
    if (kTwo && n > 1) {
      load_row(__shfl_sync(0xffffffffu, my_t, 1), nxt);
      have_nxt = first_bits(1, nib_nxt);
    }
    for (int j = 0; j < n; ++j) {
      const int t = __shfl_sync(0xffffffffu, my_t, j);
      const int k0 = __shfl_sync(0xffffffffu, my_k0, j), k1 = __shfl_sync(0xffffffffu, my_k1, j);
      const int ja = kTwo ? j + 2 : j + 1;                 // the row loaded this iteration
      const int ta = __shfl_sync(0xffffffffu, my_t, ja & 31);
      float4 nn[NCH];
      uint32_t nib_nn[NCH];
      bool have_nn = false;
      if (ja < n) {
        load_row(ta, nn);
        have_nn = first_bits(ja, nib_nn);
      }
      double acc[NCH][4];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        acc[ch][0] = (double)cur[ch].x; acc[ch][1] = (double)cur[ch].y;
        acc[ch][2] = (double)cur[ch].z; acc[ch][3] = (double)cur[ch].w;
      }
      for (int k = k0; k < k1; ++k) {
        if (k >= w0 + 32) {           // warp-uniform: slide the source window
          w0 = k;
          prepare(w0, s1);
        }
        const int sl = k - w0;
        const double mn = (double)__shfl_sync(0xffffffffu, my_mn, sl);
        const double sc = (double)__shfl_sync(0xffffffffu, my_sc, sl);
        const uint8_t* pay = reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, my_pay, sl));
        const double v0 = __dadd_rn(__dmul_rn(sc, 0.0), mn), v1 = __dadd_rn(__dmul_rn(sc, 1.0), mn);
        const bool pre = have_cur && k == k0;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const int c0 = ch * 128 + 4 * lane;
          if (c0 >= d) continue;
          const uint32_t nib = (pre ? nib_cur[ch] : (uint32_t)pay[c0 >> 3]) >> (c0 & 7);
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[ch][e] = __dadd_rn(acc[ch][e], ((nib >> e) & 1u) ? v1 : v0);
        }
      }
      float* out = dst + (int64_t)t * ld;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int c0 = ch * 128 + 4 * lane;
        if (c0 >= d) continue;
        const float4 v = make_float4(__double2float_rn(acc[ch][0]), __double2float_rn(acc[ch][1]),
                                     __double2float_rn(acc[ch][2]), __double2float_rn(acc[ch][3]));
        if (c0 + 3 < d) {
          *reinterpret_cast<float4*>(out + c0) = v;
        } else {
          out[c0] = v.x;
          if (c0 + 1 < d) out[c0 + 1] = v.y;
          if (c0 + 2 < d) out[c0 + 2] = v.z;
        }
      }
      if (kTwo) {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          cur[ch] = nxt[ch];
          nib_cur[ch] = nib_nxt[ch];
          nxt[ch] = nn[ch];
          nib_nxt[ch] = nib_nn[ch];
        }
        have_cur = have_nxt;
        have_nxt = have_nn;
      } else if (j + 1 < n) {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          cur[ch] = nn[ch];
          nib_cur[ch] = nib_nn[ch];
        }
        have_cur = have_nn;
      }
    }
  }
}

__global__ void philox_uniforms_kernel(uint64_t k0, uint64_t k1, uint64_t start, int64_t n,
                                       double* __restrict__ out) {
  const uint64_t first_blk = start >> 2;
  const uint64_t last_blk = (start + (uint64_t)n - 1) >> 2;
  for (uint64_t b = first_blk + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b <= last_blk;
       b += (uint64_t)gridDim.x * blockDim.x) {
    const U64x4 u = philox4x64_10(b + 1, k0, k1);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const uint64_t e = 4 * b + s;
      if (e >= start && e < start + (uint64_t)n) out[e - start] = u53_to_double(pick(u, s));
    }
  }
}

// ---- passthrough (bits = 32): K1 / K2 as pure gather / scatter copies ------
// codec.py:186-187 (quantize_rows returns the rows) and :202-203 (dequantize
// returns them): no metadata, no RNG.  A warp per row, lane-contiguous 4-byte
// accesses (a wire row starts 12 bytes past a 16-byte boundary, so wider
// accesses would be misaligned; lane-contiguous words still give 128-byte
// warp transactions), four words in flight per lane.  Segments are looked up
// from a per-warp cache (rows are visited in ascending order).
__device__ __forceinline__ int seg_lookup(const int32_t* seg_begin, int nseg, int row, int& cs) {
  if (!(row >= seg_begin[cs] && row < seg_begin[cs + 1])) cs = find_segment_smem(seg_begin, nseg, row);
  return cs;
}

// Row copy with the next row's words already in flight (K2 passthrough: 0.90-0.995
// of HBM at 1M-10M rows x 128-256, from 0.75-0.80): a warp holds row t
// (U words per lane, d <= 32 U) in registers while row t+1's loads issue, so
// each lane keeps up to 2U independent 4-byte loads outstanding.
template <int U>
__device__ __forceinline__ void pass_load(float (&v)[U], const float* p, int d, int lane) {
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = (p != nullptr && lane + 32 * u < d) ? __ldg(p + lane + 32 * u) : 0.f;
}

template <int U>
__device__ __forceinline__ bool pass_store(const float (&v)[U], float* p, int d, int lane) {
  bool bad = false;
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (lane + 32 * u < d) {
      bad |= !isfinite(v[u]);
      p[lane + 32 * u] = v[u];
    }
  return bad;
}

// rows t = 0..n-1 of a warp's batch: src / dst pointers broadcast from lane t
template <int U>
__device__ __forceinline__ bool pass_rows(const float* src_l, float* dst_l, int n, int d, int lane) {
  float cur[U], nxt[U];
  bool bad = false;
  pass_load<U>(cur, reinterpret_cast<const float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(src_l), 0)),
               d, lane);
  for (int t = 0; t < n; ++t) {
    const float* ns = reinterpret_cast<const float*>(
        __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(src_l), t + 1 < n ? t + 1 : t));
    float* dp = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(dst_l), t));
    pass_load<U>(nxt, t + 1 < n ? ns : nullptr, d, lane);
    bad |= pass_store<U>(cur, dp, d, lane);
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = nxt[u];
  }
  return bad;
}

__global__ void __launch_bounds__(kQWarps * 32)
quantize_pass_kernel(const float* __restrict__ src, int64_t ld, const int32_t* __restrict__ row_idx,
                     int total_rows, const hb_segment_t* __restrict__ segs_g, int nseg, int d,
                     uint32_t* __restrict__ flags) {
  __shared__ hb_segment_t segs_s[kMaxSmemSegs];
  __shared__ int32_t seg_begin[kMaxSmemSegs + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
    segs_s[i] = segs_g[i];
    seg_begin[i] = segs_g[i].row_begin;
  }
  if (threadIdx.x == 0) seg_begin[nseg] = 0x7fffffff;
  __syncthreads();
  int cs = 0;
  // 32 rows per warp at a time: lane l resolves row l's source and wire
  // pointers (and writes its block header), then the rows are copied one
  // after another from register broadcasts
  const int nwarps = gridDim.x * kQWarps;
  for (int r0 = (blockIdx.x * kQWarps + warp) * 32; r0 < total_rows; r0 += nwarps * 32) {
    const int row = r0 + lane;
    const float* x_l = nullptr;
    float* p_l = nullptr;
    if (row < total_rows) {
      const hb_segment_t& sg = segs_s[seg_lookup(seg_begin, nseg, row, cs)];
      const int r = row - sg.row_begin;
      uint8_t* out = reinterpret_cast<uint8_t*>(sg.out);
      x_l = src + (int64_t)row_idx[row] * ld;
      p_l = reinterpret_cast<float*>(out + HB_HEADER_BYTES) + (int64_t)r * d;
      if (r == 0) write_header(out, 32, sg.num_rows, d);
    }
    const int n = min(32, total_rows - r0);
    bool bad = false;
    // (the two-rows-in-flight copy of K2's passthrough measured slower here:
    // 0.72-0.79 of HBM vs 0.83-0.91 at 1M-10M rows x 128-256)
    for (int t = 0; t < n; ++t) {
      const float* x = reinterpret_cast<const float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(x_l), t));
      float* prow = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(p_l), t));
      for (int c = lane; c < d; c += 128) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = c + 32 * u < d ? __ldg(x + c + 32 * u) : 0.f;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c + 32 * u < d) {
            bad |= !isfinite(v[u]);
            prow[c + 32 * u] = v[u];
          }
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, HB_FLAG_NONFINITE);
  }
}

__global__ void __launch_bounds__(kQWarps * 32)
dequant_pass_kernel(const hb_segment_t* __restrict__ segs_g, int nseg, int num_dst,
                    const int32_t* __restrict__ dst_rows, const int32_t* __restrict__ src_ptr,
                    const int32_t* __restrict__ src_rows, int d, float* __restrict__ dst, int64_t ld,
                    int accumulate) {
  __shared__ hb_segment_t segs_s[kMaxSmemSegs];
  __shared__ int32_t seg_begin[kMaxSmemSegs + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
    segs_s[i] = segs_g[i];
    seg_begin[i] = segs_g[i].row_begin;
  }
  if (threadIdx.x == 0) seg_begin[nseg] = 0x7fffffff;
  __syncthreads();
  int cs = 0;
  // a warp takes 32 destinations at a time: lane l resolves destination l's
  // indices, segment and source row pointer with independent loads, then the
  // rows are copied one after another from register broadcasts (the index
  // chain is paid once per 32 rows, not once per row)
  const int nwarps = gridDim.x * kQWarps;
  for (int i0 = (blockIdx.x * kQWarps + warp) * 32; i0 < num_dst; i0 += nwarps * 32) {
    const int i = i0 + lane;
    int k0 = 0, k1 = 0;
    float* out_l = nullptr;
    const float* src_l = nullptr;
    if (i < num_dst) {
      out_l = dst + (int64_t)dst_rows[i] * ld;
      k0 = src_ptr[i];
      k1 = src_ptr[i + 1];
      if (k1 - k0 == 1) {
        const int q = src_rows[k0];
        const hb_segment_t& sg = segs_s[seg_lookup(seg_begin, nseg, q, cs)];
        src_l = reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(sg.out) + HB_HEADER_BYTES) +
                (int64_t)(q - sg.row_begin) * d;
      }
    }
    const int n = min(32, num_dst - i0);
    if (!accumulate && d <= 512 && __all_sync(0xffffffffu, i >= num_dst || k1 - k0 == 1)) {
      // forward halo rows: straight copies, the next row's loads in flight
      if (d <= 128) pass_rows<4>(src_l, out_l, n, d, lane);
      else if (d <= 256) pass_rows<8>(src_l, out_l, n, d, lane);
      else pass_rows<16>(src_l, out_l, n, d, lane);
      continue;
    }
    for (int t = 0; t < n; ++t) {
      float* out = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(out_l), t));
      const float* prow =
          reinterpret_cast<const float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(src_l), t));
      const int tk0 = __shfl_sync(0xffffffffu, k0, t), tk1 = __shfl_sync(0xffffffffu, k1, t);
      if (!accumulate && tk1 - tk0 == 1) {        // forward halo row: a straight copy
        for (int c = lane; c < d; c += 128) {
          float v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = c + 32 * u < d ? prow[c + 32 * u] : 0.f;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (c + 32 * u < d) out[c + 32 * u] = v[u];
        }
        continue;
      }
      // f64 sum (destination first when accumulating, then the sources in
      // ascending peer order), one fp32 rounding — as dequant_rows_kernel
      for (int c = lane; c < d; c += 128) {
        double acc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = (accumulate && c + 32 * u < d) ? (double)out[c + 32 * u] : 0.0;
        for (int k = tk0; k < tk1; ++k) {
          const int q = src_rows[k];
          const hb_segment_t& sg = segs_s[find_segment_smem(seg_begin, nseg, q)];
          const float* pr = reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(sg.out) +
                                                           HB_HEADER_BYTES) + (int64_t)(q - sg.row_begin) * d;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (c + 32 * u < d) acc[u] = __dadd_rn(acc[u], (double)pr[c + 32 * u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c + 32 * u < d) out[c + 32 * u] = __double2float_rn(acc[u]);
      }
    }
  }
}

// ----------------------------------------------------------------------------
cudaError_t launch_quantize_gather(const float* src, int64_t ld, const int32_t* row_idx,
                                   int total_rows, const hb_segment_t* segs, int nseg, int d,
                                   int bits, uint32_t* flags, cudaStream_t st) {
  if (total_rows <= 0) return cudaSuccess;
  const int nch = (d + 3 + 127) / 128;
  const bool pow2 = bits <= 8 && (bits & (bits - 1)) == 0;
  const int need = pow2 ? 4 * bits * nch + 1 : ((64 + (bits == 32 ? 0 : bits) * nch * 128) >> 5) + 3;
  const int want = (total_rows + kQWarps - 1) / kQWarps;
  const int grid = want < num_sms() * 16 ? want : num_sms() * 16;
  const dim3 blk(kQWarps * 32);
  static const bool legacy_pass = getenv("HB_PASS_LEGACY") != nullptr;
  if (bits == 32 && nseg <= kMaxSmemSegs && !legacy_pass) {
    const int want32 = (total_rows + 32 * kQWarps - 1) / (32 * kQWarps);
    const int g = want32 < num_sms() * 16 ? want32 : num_sms() * 16;
    quantize_pass_kernel<<<g, blk, 0, st>>>(src, ld, row_idx, total_rows, segs, nseg, d, flags);
    return cudaGetLastError();
  }
#define ARGS src, ld, row_idx, total_rows, segs, nseg, d, bits, flags
  static const bool no_tma = getenv("HB_K1_NO_TMA") != nullptr;
  static const bool no_hw = getenv("HB_K1_NO_HW") != nullptr;
  const bool aligned = (ld % 4 == 0) && ((((uintptr_t)src) & 15) == 0);
  if (!no_tma && !no_hw && aligned && bits == 1 && d <= 4096 && nseg <= kMaxSmemSegs) {
    const int ldr = (d + 3) & ~3;
    const int nch64 = (d + 3 + 63) >> 6;
    const int imgw = (2 * nch64 + 2 + 3) & ~3;
    // HB_K1_NBUF (tuning): row buffers per half-warp (2 = next row prefetched)
    static const int nbuf = getenv("HB_K1_NBUF") ? atoi(getenv("HB_K1_NBUF")) : 2;
    // wide rows: smaller CTAs so the per-warp row buffers do not cap the warps per SM
    const size_t per_warp = (size_t)2 * (nbuf * ldr * 4 + imgw * 4);
    const int wpc = per_warp > 6 * 1024 ? 4 : kQWarps;
    const size_t dyn = (size_t)wpc * per_warp;
    if (dyn <= 200 * 1024) {
      static const int minb = getenv("HB_K1_MINB") ? atoi(getenv("HB_K1_MINB")) : 3;
      // occupancy variants (128-thread CTAs for wide rows): <threads, CTAs/SM, buffers>
      auto kern = wpc == 4 ? (nbuf == 1 ? (minb >= 8 ? quantize_b1_hw_kernel<128, 8, 1>
                                                     : quantize_b1_hw_kernel<128, 6, 1>)
                                        : quantize_b1_hw_kernel<128, 5, 2>)
                           : (nbuf == 1 ? quantize_b1_hw_kernel<256, 4, 1> : quantize_b1_hw_kernel<256, 3, 2>);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
      const int want2 = (total_rows + 2 * wpc - 1) / (2 * wpc);
      const int cap = num_sms() * 16 * (kQWarps / wpc);
      const int grid2 = want2 < cap ? want2 : cap;
      kern<<<grid2, wpc * 32, dyn, st>>>(src, ld, row_idx, total_rows, segs, nseg, d, flags, ldr, imgw);
      return cudaGetLastError();
    }
  }
  if (!no_tma && aligned && bits != 32 && d <= 4096) {
    const int ldr = (d + 3) & ~3;
    const int imgw = ((pow2 ? 4 * bits * nch + 2 : ((64 + bits * nch * 128) >> 5) + 4) + 3) & ~3;  // 16B multiple
    const size_t dyn = (size_t)kQWarps * (2 * ldr * 4 + imgw * 4);
    if (dyn <= 200 * 1024) {
      static const int minb = getenv("HB_K1_MINB") ? atoi(getenv("HB_K1_MINB")) : 3;
      auto kern = bits == 1 ? (minb == 4 ? quantize_gather_tma_kernel<true, 4>
                               : minb == 2 ? quantize_gather_tma_kernel<true, 2> : quantize_gather_tma_kernel<true, 3>)
                            : (minb == 4 ? quantize_gather_tma_kernel<false, 4>
                               : minb == 2 ? quantize_gather_tma_kernel<false, 2> : quantize_gather_tma_kernel<false, 3>);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
      kern<<<grid, blk, dyn, st>>>(ARGS, ldr, imgw);
#undef ARGS
      return cudaGetLastError();
    }
  }
#define ARGS src, ld, row_idx, total_rows, segs, nseg, d, bits, flags
  if (bits == 32 || need <= kK1SmallWords) {
    if (bits == 1) quantize_gather_kernel<true, kK1SmallWords><<<grid, blk, 0, st>>>(ARGS);
    else quantize_gather_kernel<false, kK1SmallWords><<<grid, blk, 0, st>>>(ARGS);
  } else if (need <= kK1LargeWords) {
    if (bits == 1) quantize_gather_kernel<true, kK1LargeWords><<<grid, blk, 0, st>>>(ARGS);
    else quantize_gather_kernel<false, kK1LargeWords><<<grid, blk, 0, st>>>(ARGS);
  } else {
    quantize_gather_wide_kernel<<<grid, blk, 0, st>>>(ARGS);
  }
#undef ARGS
  return cudaGetLastError();
}

cudaError_t launch_dequant_gather(const hb_segment_t* segs, int nseg, int num_dst,
                                  const int32_t* dst_rows, const int32_t* src_ptr,
                                  const int32_t* src_rows, int d, int bits, float* dst, int64_t ld,
                                  int accumulate, cudaStream_t st) {
  if (num_dst <= 0) return cudaSuccess;
  const int want = (num_dst + kQWarps - 1) / kQWarps;
  const int grid = want < num_sms() * 8 ? want : num_sms() * 8;
  const int nch = (d + 127) / 128;
  static const bool legacy = getenv("HB_K2_LEGACY") != nullptr;
  static const bool no_acc = getenv("HB_K2_NO_B1ACC") != nullptr;
  const bool vec_dst = !no_acc && ((ld & 3) == 0) && ((((uintptr_t)dst) & 15) == 0);
  static const bool legacy_pass = getenv("HB_PASS_LEGACY") != nullptr;
  if (bits == 32 && nseg <= kMaxSmemSegs && !legacy_pass) {
    const int want32 = (num_dst + 32 * kQWarps - 1) / (32 * kQWarps);
    const int g = want32 < num_sms() * 16 ? want32 : num_sms() * 16;
    dequant_pass_kernel<<<g, kQWarps * 32, 0, st>>>(segs, nseg, num_dst, dst_rows, src_ptr, src_rows, d, dst, ld,
                                                   accumulate);
    return cudaGetLastError();
  }
  if (!legacy && nseg <= kMaxSmemSegs && nch <= 8) {
#define HB_K2(N, F) dequant_rows_kernel<N, F><<<grid, kQWarps * 32, 0, st>>>(segs, nseg, num_dst, dst_rows, \
                                                                       src_ptr, src_rows, d, bits, dst, ld, accumulate)
    // one received row per destination, 1 bit, overwrite: the fp32 fast path
    if (!accumulate && bits == 1) {
      const int want32 = (num_dst + 32 * kQWarps - 1) / (32 * kQWarps);
      // one wave: the resident CTAs per SM (register-limited) times the SMs
      auto one_wave = [&](const void* f) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, kQWarps * 32, 0) != cudaSuccess || per_sm < 1)
          per_sm = 4;
        // one resident wave for the 4-rows-ahead layout (d <= 256); the wide
        // rows measured faster with two (Reddit d = 602: 0.25 vs 0.27 ms)
        const int cap = num_sms() * (nch <= 2 ? per_sm : 8);
        return want32 < cap ? want32 : cap;
      };
#define HB_K2B(N) dequant_b1_batched_kernel<N><<<one_wave((const void*)dequant_b1_batched_kernel<N>), kQWarps * 32, 0, \
                                                 st>>>(segs, nseg, num_dst, dst_rows, src_ptr, src_rows, d, dst, ld)
      if (nch <= 1) HB_K2B(1);
      else if (nch <= 2) HB_K2B(2);
      else if (nch <= 4) HB_K2B(4);
      else if (nch <= 5) HB_K2B(5);
      else HB_K2B(8);
#undef HB_K2B
    } else if (accumulate && bits == 1 && vec_dst) {
      const int want32 = (num_dst + 32 * kQWarps - 1) / (32 * kQWarps);
      auto one_wave = [&](const void* f) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, kQWarps * 32, 0) != cudaSuccess || per_sm < 1)
          per_sm = 4;
        const int cap = num_sms() * per_sm;
        return want32 < cap ? want32 : cap;
      };
#define HB_K2A(N) dequant_b1_acc_kernel<N><<<one_wave((const void*)dequant_b1_acc_kernel<N>), kQWarps * 32, 0, \
                                             st>>>(segs, nseg, num_dst, dst_rows, src_ptr, src_rows, d, dst, ld)
      if (nch <= 1) HB_K2A(1);
      else if (nch <= 2) HB_K2A(2);
      else if (nch <= 4) HB_K2A(4);
      else if (nch <= 5) HB_K2A(5);
      else HB_K2A(8);
#undef HB_K2A
    } else if (bits != 32 && nch <= 4) {
      const int want32 = (num_dst + 32 * kQWarps - 1) / (32 * kQWarps);
      const int g32 = want32 < num_sms() * 8 ? want32 : num_sms() * 8;
#define HB_K2G(N) dequant_batched_kernel<N><<<g32, kQWarps * 32, 0, st>>>(segs, nseg, num_dst, dst_rows, src_ptr, \
                                                                       src_rows, d, bits, dst, ld, accumulate)
      if (nch <= 1) HB_K2G(1);
      else if (nch <= 2) HB_K2G(2);
      else HB_K2G(4);
#undef HB_K2G
    } else if (nch == 1) HB_K2(1, false);
    else if (nch == 2) HB_K2(2, false);
    else if (nch == 3) HB_K2(3, false);
    else if (nch == 4) HB_K2(4, false);
    else if (nch == 5) HB_K2(5, false);
    else HB_K2(8, false);
#undef HB_K2
    return cudaGetLastError();
  }
  dequant_gather_kernel<<<grid, kQWarps * 32, 0, st>>>(segs, nseg, num_dst, dst_rows, src_ptr,
                                                       src_rows, d, bits, dst, ld, accumulate);
  return cudaGetLastError();
}

cudaError_t launch_philox_uniforms(uint64_t k0, uint64_t k1, uint64_t start, int64_t n, double* out,
                                   cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = ((int64_t)((start + n + 3) >> 2) - (int64_t)(start >> 2));
  int grid = (int)((blocks + 255) / 256);
  if (grid > num_sms() * 16) grid = num_sms() * 16;
  philox_uniforms_kernel<<<grid, 256, 0, st>>>(k0, k1, start, n, out);
  return cudaGetLastError();
}

}  // namespace hb
