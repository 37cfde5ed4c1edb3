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
    real = (double)(float)tanh(real);     // bitgemm.py:206-207 evaluates tanh at fp32 precision
  }
  return real;
}

// Warp-collective epilogue over a 32-row x 32-column chunk.  Lane l owns row
// r0 + l and holds v[j] = acc(row, c0 + j).  All 32 lanes must call it.
// rows/cols are the logical output dims; r0 is a multiple of 32.
template <typename AccT>
__device__ __forceinline__ void epi_chunk32(const qg_epilogue& e, int64_t r0, int64_t c0, const AccT* v,
                                            int64_t rows, int64_t cols) {
  const int lane = threadIdx.x & 31;
  const int64_t r = r0 + lane;
  const bool rvalid = r < rows;
  if (e.out_kind == QG_OUT_REAL) {
    if (rvalid) {
      double* dst = e.out_real + r * cols;
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        int64_t c = c0 + j;
        if (c < cols) dst[c] = epi_real(e, (int64_t)v[j], r, c);
      }
    }
    return;
  }
  // requantize -> codes (0 outside the logical matrix so padding stays zero)
  const uint32_t maxv = (1u << e.q_bits) - 1u;
  uint32_t code[32];
  int64_t rsum = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    int64_t c = c0 + j;
    uint32_t q = 0;
    if (rvalid && c < cols) {
      double real = epi_real(e, (int64_t)v[j], r, c);
      if (!isfinite(real)) status_min(e.status, r * cols + c);
      q = quantize_code(real, e.q_amin, e.q_scale, maxv);
      rsum += q;
    }
    code[j] = q;
  }
  if (e.q_row_sums && rvalid && rsum) atomicAdd(reinterpret_cast<unsigned long long*>(e.q_row_sums + r),
                                                (unsigned long long)rsum);
  if (e.q_orientation == QG_COLUMN_WISE) {
    // word (r, c0/32) per plane: this lane's row, 32 consecutive columns
    const int64_t wpr = e.q_pcols >> 5;
    const int64_t wpp = e.q_prows * wpr;
    if (r < e.q_prows && (c0 >> 5) < wpr) {
      for (int p = 0; p < e.q_bits; ++p) {
        uint32_t w = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) w |= ((code[j] >> p) & 1u) << j;
        e.q_planes[p * wpp + r * wpr + (c0 >> 5)] = w;
      }
    }
  } else {
    // word (c, r0/32) per plane: 32 consecutive rows (the warp's lanes) of one column
    const int64_t wpc = e.q_prows >> 5;   // words per column
    const int64_t wpp = e.q_pcols * wpc;
    for (int p = 0; p < e.q_bits; ++p) {
      uint32_t mine = 0;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        uint32_t b = __ballot_sync(QG_FULL, (code[j] >> p) & 1u);
        if (lane == j) mine = b;
      }
      int64_t c = c0 + lane;
      if (c < e.q_pcols && (r0 >> 5) < wpc) e.q_planes[p * wpp + c * wpc + (r0 >> 5)] = mine;
    }
  }
}

}  // namespace qg
