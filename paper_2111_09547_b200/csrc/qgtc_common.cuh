// Shared device helpers for the QGTC sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/qgtc_b200.h"

#define QG_WARP 32
#define QG_FULL 0xffffffffu

namespace qg {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Record the first offending linear index (status cells start at 0x7f7f...).
__device__ __forceinline__ void status_min(int64_t* status, int64_t idx) {
  if (status) atomicMin(reinterpret_cast<unsigned long long*>(status), (unsigned long long)idx);
}

// Eq.2 quantization in fp64 (quantize.py:102-104): clip(floor((x - amin) / scale)).
// Division/subtraction are IEEE round-to-nearest; nothing here can contract.
__device__ __forceinline__ uint32_t quantize_code(double x, double amin, double scale, uint32_t maxv) {
  double v = floor(__ddiv_rn(__dsub_rn(x, amin), scale));
  if (!(v > 0.0)) return 0u;              // also maps NaN to 0 (flagged separately)
  if (v >= (double)maxv) return maxv;
  return (uint32_t)v;
}

// Correctly rounded a / b from y = RN(1/b) (host-computed): q0 = a*y, one
// Newton correction makes q1 faithful, then Markstein's theorem makes
// q2 = RN(q1 + (a - b*q1)*y) the correctly rounded quotient, with the
// remainders exact through fma.  Outside a safe exponent range (zero,
// subnormal, huge, inf/nan) it falls back to the IEEE division, so the result
// is always bit-identical to __ddiv_rn(a, b) (checked by qg_test_div tests).
// IEEE fallback kept out of line so the (rare) slow path does not bloat every call site.
static __device__ __noinline__ double div_rn_ieee(double a, double b) { return __ddiv_rn(a, b); }
// tanh evaluated at fp32 precision (bitgemm.py:206-207); out of line (rarely used, large)
static __device__ __noinline__ double tanh_f32(double x) { return (double)(float)tanh(x); }

__device__ __forceinline__ double div_rn(double a, double b, double y) {
  // +-0 / finite b: IEEE gives a zero signed sign(a)^sign(b) == a * y exactly (ReLU
  // outputs on an alpha_min = 0 grid hit this for half the elements)
  if (a == 0.0 && fabs(y) < 0x1p+1000) return __dmul_rn(a, y);
  const double aa = fabs(a), bb = fabs(b);
  double q = __dmul_rn(a, y);
  const double qq = fabs(q);
  if (!(aa < 0x1p+900 && aa > 0x1p-900 && bb < 0x1p+900 && bb > 0x1p-900 && qq < 0x1p+900 && qq > 0x1p-900))
    return div_rn_ieee(a, b);
  double r = __fma_rn(-q, b, a);
  q = __fma_rn(r, y, q);
  r = __fma_rn(-q, b, a);
  return __fma_rn(r, y, q);
}

// Eq.2 requantization in the epilogue: code = clamp(floor(RN(a / scale)), 0, maxv),
// a = RN(x - amin), bit-identical to the reference (quantize.py:102-104).
// Only the floor of the correctly rounded quotient is needed, so the common case
// avoids the division: q0 = a * RN(1/scale) has |q0 - a/scale| <= 2^-52 * 256 < 2^-43
// for q0 < maxv + 1 <= 256, and RN(a/scale) is within 2^-45 of a/scale; if q0's
// fractional part is farther than 2^-40 from an integer, every candidate quotient has
// the same floor.  floor(q0) comes from a round-down add of 2^52 (no F2I, which
// runs at ~1/4 of the DFMA rate on B200).  Near-integer cases take IEEE __ddiv_rn.
__device__ __forceinline__ uint32_t quantize_code_fast(double x, double amin, double scale, double inv_scale,
                                                       uint32_t maxv) {
  const double a = __dsub_rn(x, amin);
  if (!(a > 0.0)) return 0u;                  // a <= 0 (or NaN): floor(a/scale) <= 0 -> 0
  const double q0 = __dmul_rn(a, inv_scale);
  if (q0 >= (double)maxv + 1.0) return maxv;  // quotient >= maxv + 1 - 2^-43 > maxv
  const double t = __dadd_rd(q0, 0x1p52);     // 2^52 + floor(q0)
  const double fl = __dsub_rn(t, 0x1p52);     // exact
  const double frac = __dsub_rn(q0, fl);      // exact (Sterbenz), in [0, 1)
  uint32_t k;
  if (frac > 0x1p-40 && frac < 1.0 - 0x1p-40) {
    k = (uint32_t)__double2loint(t);
  } else {
    const double v = __ddiv_rn(a, scale);
    k = v >= 1.0 ? (uint32_t)__double2int_rd(fmin(v, (double)maxv)) : 0u;
  }
  return k < maxv ? k : maxv;
}

// Epilogue requant with three fp64 ops.  q0 = RN(RN(x - amin) * RN(1/scale)) is
// within 2^-44 of the true quotient for quotients < 2^8; r = RN(q0 + 2^12) then has
// ulp 2^-40, so for r in [2^12, 2^13) its high word is 0x40B00000 + (floor << 8) +
// (top 8 fraction bits) and its low word the rest of the fraction (units of 2^-40).
// The fast decode is integer-only and valid when the caller's screen passes:
//   hi < 0x40C00000 unsigned  -> r in [+0, 2^13): finite, not negative, q0 < 4096
//   not (lo + 1 <= 2 && hi != 0x40B00000) -> the fraction is >= 2 units from an
//       integer, so floor(RN(a / scale)) == floor(q0) (margin 2^-39 - 2^-41 - 2^-44);
//       r == 2^12 exactly (q0 within 2^-41 of 0, e.g. ReLU zeros) is code 0 either way.
// Anything the screen flags goes to quantize_code_fast (exact, with the IEEE
// division fallback).  Bit-identity: tests/test_gpu_kernels.py.
struct R12 {
  uint32_t code;
  bool flag;   // screen failed: recompute exactly
};
__device__ __forceinline__ R12 quantize_code_r12(double x, double amin, double inv_scale, uint32_t maxv) {
  const double r = __dadd_rn(__dmul_rn(__dsub_rn(x, amin), inv_scale), 0x1p12);
  const uint32_t hi = (uint32_t)__double2hiint(r), lo = (uint32_t)__double2loint(r);
  const int kc = (int)(hi >> 8) - 0x40B000;            // floor for r in [2^12, 2^13)
  R12 o;
  o.code = (uint32_t)min(max(kc, 0), (int)maxv);
  o.flag = (hi >= 0x40C00000u) | ((lo + 1u <= 2u) & (hi != 0x40B00000u));
  return o;
}

// Same decode with the tight near-integer test: flag only when the 40-bit fraction
// (top 8 bits in hi, 32 in lo) is within one unit of an integer.  Inputs that are
// exactly representable at low precision (fp32 features: x * 2^k has a short
// fraction, so lo == 0 for almost every element) would trip the coarse lo-only test
// of quantize_code_r12 on nearly every element.
__device__ __forceinline__ R12 quantize_code_r12_tight(double x, double amin, double inv_scale, uint32_t maxv) {
  const double r = __dadd_rn(__dmul_rn(__dsub_rn(x, amin), inv_scale), 0x1p12);
  const uint32_t hi = (uint32_t)__double2hiint(r), lo = (uint32_t)__double2loint(r);
  const int kc = (int)(hi >> 8) - 0x40B000;
  const uint32_t f8 = hi & 0xFFu;
  R12 o;
  o.code = (uint32_t)min(max(kc, 0), (int)maxv);
  o.flag = (hi >= 0x40C00000u) | (((f8 == 0u) & (lo <= 1u)) & (hi != 0x40B00000u)) | ((f8 == 0xFFu) & (lo == ~0u));
  return o;
}

// Reference formulation (tests): floor of the IEEE quotient, clamped.
__device__ __forceinline__ uint32_t quantize_code_ref(double x, double amin, double scale, uint32_t maxv) {
  const double v = floor(__ddiv_rn(__dsub_rn(x, amin), scale));
  if (!(v > 0.0)) return 0u;
  if (v >= (double)maxv) return maxv;
  return (uint32_t)v;
}

// 8x8 bit-matrix transpose of a u64 (byte i = row i): afterwards byte j holds
// bit j of every input byte (Hacker's Delight 7-3).  Used to turn 8 codes into
// 8 plane bytes in a handful of ops.
__device__ __forceinline__ uint64_t transpose8x8(uint64_t x) {
  uint64_t t;
  t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;  x = x ^ t ^ (t << 7);
  t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull; x = x ^ t ^ (t << 14);
  t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull; x = x ^ t ^ (t << 28);
  return x;
}

// 4 packed bits -> 4 bytes of 0/1 (bit i -> byte i).
__device__ __forceinline__ uint32_t expand_nibble(uint32_t nib) {
  return (nib * 0x00204081u) & 0x01010101u;
}

// ------------------------------------------------------------------ epilogue
// Per-element fp64 epilogue: identical expression order to the reference
// (bitgemm.py:156-207), with explicit _rn intrinsics so no FMA contraction.
__device__ __forceinline__ double epi_real(const qg_epilogue& e, int64_t acc, int64_t r, int64_t c) {
  double real = __dmul_rn(e.k_acc, (double)acc);
  if (e.use_row) real = __dadd_rn(real, __dmul_rn(e.k_row, (double)e.row_sums[r]));
  if (e.use_col) real = __dadd_rn(real, __dmul_rn(e.k_col, (double)e.col_sums[c]));
  if (e.use_const) real = __dadd_rn(real, e.k_const);
  if (e.bias) real = __dadd_rn(real, e.bias[c]);
  if (e.bn_mean) {
    real = __dadd_rn(__dmul_rn(__ddiv_rn(__dsub_rn(real, e.bn_mean[c]), e.bn_denom[c]), e.bn_gamma[c]),
                     e.bn_beta[c]);
  }
  if (e.act == QG_ACT_RELU) {
    real = (real < 0.0) ? 0.0 : real;
  } else if (e.act == QG_ACT_TANH) {
    real = tanh_f32(real);
  }
  return real;
}

// Warp-collective epilogue over a 32-row x 32-column chunk.  Lane l owns row
// r0 + l; `get8(sub, v)` delivers acc(row, c0 + 8*sub + jj) for jj < 8 (TMEM
// slices in the GEMM, global loads in the stand-alone kernel).  All 32 lanes
// must call it; r0 and c0 are multiples of 32; rows/cols are logical dims.
template <typename Get8>
__device__ __forceinline__ void epi_chunk32(const qg_epilogue& e, int64_t r0, int64_t c0, Get8 get8,
                                            int64_t rows, int64_t cols) {
  const int lane = threadIdx.x & 31;
  const int64_t r = r0 + lane;
  const bool rvalid = r < rows;
  if (e.out_kind == QG_OUT_REAL) {
    for (int sub = 0; sub < 4; ++sub) {
      uint32_t v[8];
      get8(sub, v);
      if (rvalid) {
        double* dst = e.out_real + r * cols;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int64_t c = c0 + sub * 8 + jj;
          if (c < cols) dst[c] = epi_real(e, (int64_t)(int32_t)v[jj], r, c);
        }
      }
    }
    return;
  }
  // requantize -> codes (0 outside the logical matrix so padding stays zero) -> bit planes
  const uint32_t maxv = (1u << e.q_bits) - 1u;
  const bool colwise = e.q_orientation == QG_COLUMN_WISE;
  uint32_t w[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) w[p] = 0;
  int64_t rsum = 0;
  for (int sub = 0; sub < 4; ++sub) {
    uint32_t v[8];
    get8(sub, v);
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int j = sub * 8 + jj;
      const int64_t c = c0 + j;
      uint32_t q = 0;
      if (rvalid && c < cols) {
        const double real = epi_real(e, (int64_t)(int32_t)v[jj], r, c);
        if (!isfinite(real)) status_min(e.status, r * cols + c);
        q = quantize_code_fast(real, e.q_amin, e.q_scale, e.q_inv_scale, maxv);
        rsum += q;
        if (e.q_codes) e.q_codes[e.q_codes_colmajor ? c * e.q_codes_ld + r : r * e.q_codes_ld + c] = (uint8_t)q;
      }
      if (colwise) {
        // this lane's row: bit j of word (r, c0/32)
#pragma unroll
        for (int p = 0; p < 8; ++p) w[p] |= ((q >> p) & 1u) << j;
      } else {
        // column c0+j over the warp's 32 rows: lane j keeps the ballot
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          if (p < e.q_bits) {
            const uint32_t b = __ballot_sync(QG_FULL, (q >> p) & 1u);
            if (lane == j) w[p] = b;
          }
        }
      }
    }
  }
  if (e.q_row_sums && rvalid && rsum) atomicAdd(reinterpret_cast<unsigned long long*>(e.q_row_sums + r),
                                                (unsigned long long)rsum);
  if (e.q_skip_planes) return;
  if (colwise) {
    const int64_t wpr = e.q_pcols >> 5;
    const int64_t wpp = e.q_prows * wpr;
    if (r < e.q_prows && (c0 >> 5) < wpr) {
#pragma unroll
      for (int p = 0; p < 8; ++p)
        if (p < e.q_bits) e.q_planes[p * wpp + r * wpr + (c0 >> 5)] = w[p];
    }
  } else {
    const int64_t wpc = e.q_prows >> 5;   // words per column
    const int64_t wpp = e.q_pcols * wpc;
    const int64_t c = c0 + lane;
    if (c < e.q_pcols && (r0 >> 5) < wpc) {
#pragma unroll
      for (int p = 0; p < 8; ++p)
        if (p < e.q_bits) e.q_planes[p * wpp + c * wpc + (r0 >> 5)] = w[p];
    }
  }
}

__device__ __forceinline__ uint4 ldg128(const uint32_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d));
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  // K-major, SWIZZLE_NONE canonical layout: core matrix = 8 rows x 16 B;
  // LBO = 128 B (next core along K), SBO = 1024 B (next 8-row group).
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ uint32_t idesc_u8(int n) {
  return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);  // S32 acc, u8 x u8, K-major
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  }
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;   // src-size 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int kThreads = 256;

// smem address of (operand row r, K-core c) in the UMMA K-major interleaved layout
__device__ __forceinline__ uint32_t umma_off(int r, int c) { return (uint32_t)((r >> 3) * 1024 + c * 128 + (r & 7) * 16); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// A operand in TENSOR MEMORY (lane = row, column c = K bytes 4c..4c+3 little endian;
// measured: probes/ts_probe.cu)
__device__ __forceinline__ void umma_i8_ts(uint32_t tmem, uint32_t ta, uint64_t db, uint32_t idesc, uint32_t accum) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(tmem), "r"(ta), "l"(db), "r"(idesc), "r"(accum));
}
// 32 consecutive TMEM columns of this thread's lane (tcgen05.st.32x32b.x32)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&x)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]), "r"(x[7]), "r"(x[8]), "r"(x[9]),
      "r"(x[10]), "r"(x[11]), "r"(x[12]), "r"(x[13]), "r"(x[14]), "r"(x[15]), "r"(x[16]), "r"(x[17]), "r"(x[18]),
      "r"(x[19]), "r"(x[20]), "r"(x[21]), "r"(x[22]), "r"(x[23]), "r"(x[24]), "r"(x[25]), "r"(x[26]), "r"(x[27]),
      "r"(x[28]), "r"(x[29]), "r"(x[30]), "r"(x[31]));
}
__device__ __forceinline__ void umma_i8(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accum) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(accum));
}

// Tiled (UMMA K-major interleaved) operand layouts in HBM.  A 128-wide K slab of a
// left operand holds [rows/8][8 K-cores][8 rows][16 B]; a 128-row block of it is a
// contiguous 16 KB that lands in shared memory exactly as the MMA descriptor reads
// it (LBO 128 B, SBO 1024 B).  Right operands use the same per-slab layout over the
// N columns, so any 8-aligned column range of a slab is contiguous.
__device__ __forceinline__ int64_t left_tile_off(int64_t r, int64_t k, int64_t r128) {
  return (k >> 7) * (r128 << 7) + (r >> 3) * 1024 + ((k & 127) >> 4) * 128 + (r & 7) * 16 + (k & 15);
}
__device__ __forceinline__ int64_t right_tile_off(int64_t k, int64_t n, int64_t npad) {
  return (k >> 7) * (npad << 7) + (n >> 3) * 1024 + ((k & 127) >> 4) * 128 + (n & 7) * 16 + (k & 15);
}

}  // namespace qg
