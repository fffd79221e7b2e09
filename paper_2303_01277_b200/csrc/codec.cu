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
#include "common.cuh"
#include "philox.cuh"

namespace hb {

constexpr int kQWarps = 8;                 // warps per CTA in K1/K2
constexpr int kMaxSmemSegs = 128;          // segment table cached in smem
constexpr int kMaxChunks = 9;              // d <= 9*128 - 3 keeps the row in registers
constexpr int kRowBufWords = 2 + (kMaxChunks * 128 * 16) / 32 + 4;  // b <= 16, 64-bit lead

struct QuantRowCtx {
  float mn, s, inv_s, E;
  int B, bits;
  bool live, fast;
};

// Exact fp64 reference decision (codec.py:185-193).
__device__ __forceinline__ int quant_exact(float x, const QuantRowCtx& q, uint64_t w) {
  const double D = __dsub_rn((double)x, (double)q.mn);
  const double h = __ddiv_rn(D, (double)q.s);
  const double f = floor(h);
  const double fr = __dsub_rn(h, f);
  const double u = u53_to_double(w);
  int code = (int)f + (u < fr ? 1 : 0);
  return min(max(code, 0), q.B);
}

// fp32 filter: returns the code, or -1 when the decision needs fp64.
__device__ __forceinline__ int quant_fast(float x, const QuantRowCtx& q, uint64_t w) {
  if (x == q.mn) return 0;                       // h == 0 exactly on both paths
  const float xm = __fsub_rn(x, q.mn);
  const float h = __fmul_rn(xm, q.inv_s);
  if (!(h < 8388608.0f)) return -1;
  const float fl = floorf(h);
  const float fr = __fsub_rn(h, fl);             // exact
  if (fr < q.E || fr > 1.0f - q.E) return -1;    // floor(h) itself is uncertain
  const float ut = __uint2float_rn((uint32_t)(w >> 40)) * 5.9604644775390625e-08f;  // top 24 bits
  int up;
  if (ut + 5.9604644775390625e-08f + q.E <= fr) up = 1;   // u < ut + 2^-24 <= frac
  else if (ut >= fr + q.E) up = 0;                         // u >= ut >= frac
  else return -1;
  const int code = (int)fl + up;
  return min(max(code, 0), q.B);
}

__device__ __forceinline__ int quant_one(float x, const QuantRowCtx& q, uint64_t w) {
  if (q.fast) {
    const int c = quant_fast(x, q, w);
    if (c >= 0) return c;
  }
  return quant_exact(x, q, w);
}

__device__ __forceinline__ void write_header(uint8_t* out, int bits, int rows, int d) {
  out[0] = 1;
  out[1] = (uint8_t)bits;
  out[2] = 0;
  out[3] = 0;
  for (int k = 0; k < 4; ++k) out[4 + k] = (uint8_t)((uint32_t)rows >> (8 * k));
  for (int k = 0; k < 4; ++k) out[8 + k] = (uint8_t)((uint32_t)d >> (8 * k));
}

__device__ __forceinline__ void store_f32_unaligned4(uint8_t* p, float v) {
  // p is 4-byte aligned by construction (12 + 8r offsets from a 16B-aligned block)
  *reinterpret_cast<float*>(p) = v;
}

// NCH > 0: the row is held in registers (NCH chunks of 128 columns, Philox frame).
// NCH == 0: generic path for very wide rows (re-reads x in the second pass).
template <int NCH>
__global__ void __launch_bounds__(kQWarps * 32)
quantize_gather_kernel(const float* __restrict__ src, int64_t ld, const int32_t* __restrict__ row_idx,
                       int total_rows, const hb_segment_t* __restrict__ segs_g, int nseg, int d,
                       int bits, uint32_t* __restrict__ flags) {
  __shared__ hb_segment_t segs_s[kMaxSmemSegs];
  __shared__ uint32_t rowbuf[kQWarps][NCH > 0 ? kRowBufWords : 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool smem_segs = nseg <= kMaxSmemSegs;
  if (smem_segs) {
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) segs_s[i] = segs_g[i];
    __syncthreads();
  }
  const hb_segment_t* segs = smem_segs ? segs_s : segs_g;
  const int B = (1 << bits) - 1;
  const int rb = (d * bits + 7) >> 3;
  const int nchunks_max = (d + 3 + 127) >> 7;
  uint32_t* buf = rowbuf[warp];
  const int buf_words = (NCH > 0) ? ((64 + bits * (nchunks_max * 128)) >> 5) + 3 : 0;

  for (int row = blockIdx.x * kQWarps + warp; row < total_rows; row += gridDim.x * kQWarps) {
    const hb_segment_t sg = segs[find_segment(segs, nseg, row)];
    const int r = row - sg.row_begin;
    const float* x = src + (int64_t)row_idx[row] * ld;
    const uint64_t e_row = sg.elem_offset + (uint64_t)r * (uint64_t)d;
    const int delta = (int)(e_row & 3ull);
    const uint64_t blk0 = e_row >> 2;
    const int nchunks = (d + delta + 127) >> 7;
    uint8_t* out = reinterpret_cast<uint8_t*>(sg.out);

    // ---- pass 1: load (Philox frame) + row min/max + finiteness -------------
    float v[NCH > 0 ? NCH : 1][4];
    float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
    bool bad = false;
    if (NCH > 0) {
#pragma unroll
      for (int t = 0; t < (NCH > 0 ? NCH : 1); ++t) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int c = 128 * t + 4 * lane + i - delta;
          float xv = 0.f;
          if (t < nchunks && c >= 0 && c < d) {
            xv = __ldg(x + c);
            mn = fminf(mn, xv);
            mx = fmaxf(mx, xv);
            bad |= !isfinite(xv);
          }
          v[t][i] = xv;
        }
      }
    } else {
      for (int c = lane; c < d; c += 32) {
        const float xv = __ldg(x + c);
        mn = fminf(mn, xv);
        mx = fmaxf(mx, xv);
        bad |= !isfinite(xv);
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
             fabsf(mn) <= 1.2676506002282294e30f && fabsf(mx) <= 1.2676506002282294e30f &&
             bits <= 16;
    q.E = (float)(B + 2) * 2.384185791015625e-07f;  // (B+2) * 2^-22
    if (lane == 0) {
      store_f32_unaligned4(out + HB_HEADER_BYTES + 8 * (int64_t)r, q.mn);
      store_f32_unaligned4(out + HB_HEADER_BYTES + 8 * (int64_t)r + 4, q.s);
    }
    uint8_t* pay = out + HB_HEADER_BYTES + 8 * (int64_t)sg.num_rows + (int64_t)r * rb;

    if (NCH == 0) {
      // generic wide-row path: direct byte-wise OR is impossible without atomics on
      // global memory, so each lane assembles whole payload bytes itself.
      for (int byte = lane; byte < rb; byte += 32) {
        uint32_t acc = 0;
        const int c_first = (byte * 8) / bits, c_last = min(d - 1, (byte * 8 + 7) / bits);
        for (int c = c_first; c <= c_last; ++c) {
          int code = 0;
          if (q.live) {
            const uint64_t e = e_row + (uint64_t)c;
            const U64x4 u = philox4x64_10((e >> 2) + 1, sg.key0, sg.key1);
            code = quant_one(__ldg(x + c), q, pick(u, (int)(e & 3)));
          }
          const int pos = c * bits - byte * 8;  // may be negative for straddling codes
          acc |= pos >= 0 ? ((uint32_t)code << pos) : ((uint32_t)code >> (-pos));
        }
        pay[byte] = (uint8_t)(acc & 0xffu);
      }
      continue;
    }

    // ---- pass 2: Philox + quantize + pack into the smem row image ------------
    for (int k = lane; k < buf_words; k += 32) buf[k] = 0u;
    __syncwarp();
    if (q.live) {
#pragma unroll
      for (int t = 0; t < (NCH > 0 ? NCH : 1); ++t) {
        if (t < nchunks) {
          const U64x4 u = philox4x64_10(blk0 + (uint64_t)(32 * t + lane) + 1ull, sg.key0, sg.key1);
          const int c0 = 128 * t + 4 * lane - delta;
          uint64_t field = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int c = c0 + i;
            if (c >= 0 && c < d) {
              const uint64_t w = i == 0 ? u.w0 : (i == 1 ? u.w1 : (i == 2 ? u.w2 : u.w3));
              field |= (uint64_t)quant_one(v[t][i], q, w) << (i * bits);
            }
          }
          if (field) {
            const int pos = 64 + bits * c0;           // >= 16 for bits <= 16
            const int wd = pos >> 5, sh = pos & 31;
            const uint64_t lo = field << sh;
            atomicOr(&buf[wd], (uint32_t)lo);
            if ((uint32_t)(lo >> 32)) atomicOr(&buf[wd + 1], (uint32_t)(lo >> 32));
            if (sh && (field >> (64 - sh))) atomicOr(&buf[wd + 2], (uint32_t)(field >> (64 - sh)));
          }
        }
      }
    }
    __syncwarp();
    const uint8_t* img = reinterpret_cast<const uint8_t*>(buf) + 8;
    if ((((uintptr_t)pay) & 3) == 0 && (rb & 3) == 0) {
      uint32_t* pw = reinterpret_cast<uint32_t*>(pay);
      const uint32_t* iw = buf + 2;
      for (int k = lane; k < (rb >> 2); k += 32) pw[k] = iw[k];
    } else {
      for (int k = lane; k < rb; k += 32) pay[k] = img[k];
    }
    __syncwarp();
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

// ----------------------------------------------------------------------------
cudaError_t launch_quantize_gather(const float* src, int64_t ld, const int32_t* row_idx,
                                   int total_rows, const hb_segment_t* segs, int nseg, int d,
                                   int bits, uint32_t* flags, cudaStream_t st) {
  if (total_rows <= 0) return cudaSuccess;
  const int nch = (d + 3 + 127) / 128;
  const int want = (total_rows + kQWarps - 1) / kQWarps;
  const int grid = want < num_sms() * 8 ? want : num_sms() * 8;
  const dim3 blk(kQWarps * 32);
#define HB_Q(N) quantize_gather_kernel<N><<<grid, blk, 0, st>>>(src, ld, row_idx, total_rows, segs, nseg, d, bits, flags)
  switch (nch) {
    case 1: HB_Q(1); break;
    case 2: HB_Q(2); break;
    case 3: HB_Q(3); break;
    case 4: HB_Q(4); break;
    case 5: HB_Q(5); break;
    case 6: HB_Q(6); break;
    case 7: HB_Q(7); break;
    case 8: HB_Q(8); break;
    case 9: HB_Q(9); break;
    default: HB_Q(0); break;
  }
#undef HB_Q
  return cudaGetLastError();
}

cudaError_t launch_dequant_gather(const hb_segment_t* segs, int nseg, int num_dst,
                                  const int32_t* dst_rows, const int32_t* src_ptr,
                                  const int32_t* src_rows, int d, int bits, float* dst, int64_t ld,
                                  int accumulate, cudaStream_t st) {
  if (num_dst <= 0) return cudaSuccess;
  const int want = (num_dst + kQWarps - 1) / kQWarps;
  const int grid = want < num_sms() * 8 ? want : num_sms() * 8;
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
