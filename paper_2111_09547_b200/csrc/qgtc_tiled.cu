// Tiled, warp-specialised bit-GEMM for sm_100a (the engine's fast path).
//
// Operands live in HBM in the UMMA K-major interleaved layout (qgtc_common.cuh
// left/right_tile_off): the 1-bit adjacency as 16 KB byte blocks (only the
// non-zero 128x128 blocks, expanded once per batch), activations and weights as
// u8 code caches written by the previous epilogue.  Per K tile a stage is
// therefore exactly two contiguous bulk copies (TMA engine, UBLKCP) completing on
// one mbarrier:
//   warp 0 lane 0  producer   wait empty[s] -> expect_tx -> 2x cp.async.bulk
//   warp 1 lane 0  MMA        wait full[s]  -> 4x tcgen05.mma kind::i8 -> commit empty[s]
//   all 8 warps    epilogue   wait done     -> tcgen05.ld -> fp64 dequant/bias/BN/act
//                                              -> requant -> tiled u8 codes + row sums
//                                              (or fp64 logits / int32)
// No per-tile __syncthreads.  One launch may cover many batches ("segments"):
// CTA -> (segment, 128-row block, N tile), so an epoch layer stage over all
// subgraph batches is a single grid.
//
// Variants: CHAIN (qg_chain) runs a second, dense GEMM behind the epilogue over the
// requantized codes left in the ring's shared memory (aggregation -> update in one
// launch); tc_pair_kernel runs cta_group::2 MMAs (M = 256) for large int32 GEMMs.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cuda.h>
#include "qgtc_common.cuh"

namespace qg {

struct TiledParams {
  alignas(64) CUtensorMap zero_map;   // pair mode: 16 KB zero block (rows of 128 B)
  alignas(64) CUtensorMap w2_map;     // chained pair mode: stage-2 weights, boxes of bn2/2 rows of 128 B
  const qg_tseg* segs;
  int32_t nsegs;
  int32_t a_blocks;         // 1: left operand = adjacency blocks (schedule), 0: dense left slabs
  int64_t b_npad;           // right operand padded N (slab pitch = b_npad * 128)
  int64_t n;                // logical output columns
  int32_t bn, log2bn, n_tiles, stages;
  int32_t mode;             // QG_GEMM_I32 / QG_GEMM_EPILOGUE
  int32_t out_layout;       // 0 fp64/int32 row-major, 1 left-tiled codes, 2 right-tiled codes
  int64_t out_npad;         // right-tiled output: padded N of the output (slab pitch)
  qg_epilogue epi;          // shared scalars + per-column vectors (per-row pointers come from segs)
  int64_t* phase_ns;        // optional per-tile %globaltimer stamps (tools/phase_tiled.py)
  int64_t total_ctas;       // work items (segment, row block, N tile) of this stage
  int32_t pair;             // 1: CTA pairs (cluster of 2) run cta_group::2 MMAs, M = 256
  int32_t pair_swizzle;     // pair kernels: row-block pairs per N-major group (1 = plain order)
  int32_t slot_bn;          // ring slot B capacity in columns: max(bn, bn2)
  int32_t screen;           // fp32 requant screen enabled (QG_NO_SCREEN=1 disables)
  int32_t a_bits;           // a_blocks: the adjacency ships as PACKED 2 KB blocks, expanded in smem (1)
                            // or into tensor memory (2)
  int32_t a_slots, a_col0;  // a_bits 2: TMEM A ring slots (32 columns each) and its first column
  int32_t persist;          // CTAs loop over work items (grid = resident CTAs); the producer
                            // prefetches the next item's first K tiles during the epilogue
  int32_t dbg;              // QG_EPI_DBG knock-out bits (experiments; screened epilogue only, built with
                            // -DQG_EPI_KNOCKOUTS): 1 no stores, 2 no math, 4 no TMEM loads
  // chained stage 2 (qg_tiled_args.chain): a dense GEMM over this stage's requantized
  // codes, which never leave shared memory; one CTA per row block (n_tiles 1).
  int32_t chain, bn2, k2, out_layout2;
  int64_t n2, out_npad2, w2_npad;
  const uint8_t* w2;
  qg_epilogue epi2;
};

// Segment of a work item: the last segment with cta_begin <= w (cta_begin ascending).
// Warp-cooperative: every lane tests its own segments with independent loads (one L2
// round trip per 32 segments instead of a dependent binary search).
template <typename Seg, typename Begin>
__device__ __forceinline__ int find_seg_by(const Seg* segs, int nsegs, int64_t w, Begin begin) {
  const int lane = threadIdx.x & 31;
  int cnt = 0;
  for (int base = 0; base < nsegs; base += 32) {
    const int i = base + lane;
    const bool le = i < nsegs && begin(segs[i]) <= w;
    cnt += __popc(__ballot_sync(0xffffffffu, le));
  }
  return cnt - 1;
}
__device__ __forceinline__ int find_seg(const qg_tseg* segs, int nsegs, int64_t w) {
  return find_seg_by(segs, nsegs, w, [](const qg_tseg& g) { return g.cta_begin; });
}

static __device__ __forceinline__ void tstamp(const TiledParams& P, int64_t tile, int k) {
  if (P.phase_ns) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.phase_ns[tile * 8 + k] = (int64_t)t;
    if (k == 0) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      P.phase_ns[tile * 8 + 6] = (int64_t)smid;
      P.phase_ns[tile * 8 + 7] = 0;             // chained launches overwrite it (stage-2 accumulator ready)
    }
  }
}

constexpr int kTThreads = 256;

// exact requant of one element with the non-finite report (rare path, kept out of line)
static __device__ __noinline__ uint32_t requant_exact(double x, double amin, double scale, double inv, uint32_t maxv,
                                                      int64_t* status, int64_t flat) {
  if (!isfinite(x) && status) status_min(status, flat);
  return quantize_code_fast(x, amin, scale, inv, maxv);
}

// ---------------------------------------------------------------- fp32 requant screen
// For epilogues without batch norm the requantized code of an element is
// clamp(floor(q), 0, maxv), q the reference's fp64 quotient RN(RN(x - amin) / scale) of
// the dequantized (+bias, ReLU) value x.  In exact arithmetic over the fp64 constants
// q ~ Y = alpha acc + beta_r + gamma_c (alpha = k_acc / scale > 0, beta_r = (rterm_r -
// amin) / scale, gamma_c = (C_c + K + B_c) / scale).  beta_r and gamma_c are large and
// cancel against alpha acc, so the screen shifts in INTEGERS first: acc' = acc - acc0_r -
// acc0_c (acc0 = rint(-beta / alpha)), converts acc' to fp32 (exact below 2^24, else
// relative 2^-24) and evaluates y = fma(acc', alpha, delta_r) + delta_c, |delta| <= alpha/2.
// Then |y - q| <= 2^-24 (4 |Y| + 3 alpha) + 2^-40 < margin = 2^-21 (maxv + 3 + 2 alpha +
// |q0|) wherever the code is decided (|Y| <= maxv + 2).  ReLU is max(q, q0) with q0 the
// quotient of x = 0 (monotone, exact); floor(clamp(z, 0.5, maxv + 0.5)) ==
// clamp(floor(z), 0, maxv).  An element whose clamped estimate lies within the margin
// of an integer takes the exact fp64 path (per element, divergent; ~2.5e-4 of the
// elements at 8 bits), so the codes are bit-identical to the reference's.
struct ScreenRow {
  bool on;          // screen usable for this tile (else every slice runs the fp64 path)
  int32_t a0r;      // acc0_r
  float dr;         // delta_r
  float alpha;
  float mrg;        // margin; -1: invalid row (never exact), +inf: always exact
  float hc;         // RN(0.5 - mrg): the flag test is |frac(y) - 1/2| > RN(hc - 2^-21 y)
  float lo, hi;     // clamp bounds: max(q0, 0.5) (ReLU) or 0.5; maxv + 0.5
  const int32_t* sA0;  // per column acc0_c (row-only stages: unused)
  const float* sD;     // per column delta_c
};

// doubles of per-column constants one stage stages in shared memory: the fp64 terms
// (C, B [, BN x5]) + the screen's acc0_c / delta_c; none for a row-only stage
__host__ __device__ __forceinline__ int col_doubles(int bn, bool row_only, bool has_bn) {
  if (row_only && !has_bn) return 0;
  return has_bn ? 7 * bn : 3 * bn;
}
// bytes of one ring slot of the single-CTA kernel (a_bits adds the 2 KB packed block,
// slots 1 KB aligned for the UMMA descriptors)
__host__ __device__ __forceinline__ uint32_t tiled_stage_bytes(int slot_bn, int a_bits) {
  if (a_bits == 2) return ((uint32_t)slot_bn * 128u + 2048u + 1023u) & ~1023u;   // no A bytes in smem
  const uint32_t b = 16384u + (uint32_t)slot_bn * 128u;
  return a_bits ? ((b + 2048u + 1023u) & ~1023u) : b;
}
__device__ __forceinline__ bool epi_row_only(const qg_epilogue& E) { return !E.use_col && !E.use_const && !E.bias; }

// per-column screen constants (staging warps; stages without batch norm); a column whose
// shift does not fit turns the stage's screen off (*off)
// alpha = k_acc / scale and ~1/alpha without fp64 divisions (software routines on the GPU):
// the screen only needs its integer shifts near -beta / alpha; the identities
// y = alpha acc' + delta hold exactly for the alpha used (relative 2^-52 off the quotient,
// far inside the margin)
__device__ __forceinline__ double screen_alpha(const qg_epilogue& E, double& inv_alpha) {
  const double alpha = E.k_acc * E.q_inv_scale;
  double r = (double)__frcp_rn((float)alpha);
  r = r * (2.0 - alpha * r);
  r = r * (2.0 - alpha * r);
  inv_alpha = r;
  return alpha;
}

__device__ __forceinline__ void screen_col(const qg_epilogue& E, int i, double C, double B, int32_t* sA0, float* sD,
                                           int* off) {
  double ia;
  const double alpha = screen_alpha(E, ia);
  const double K = E.use_const ? E.k_const : 0.0;
  const double gam = ((C + K) + B) * E.q_inv_scale;
  const double a0 = rint(-gam * ia);
  if (!(fabs(a0) <= 0x1p29)) {
    *off = 1;
    sA0[i] = 0;
    sD[i] = 0.0f;
    return;
  }
  sA0[i] = (int32_t)a0;
  sD[i] = (float)(gam + a0 * alpha);
}

// Per-column epilogue constants of one stage into shared memory (col_doubles layout):
// C = RN(k_col * col_sum), B = bias [, BN mean / denom / gamma / beta / inv_denom], and the
// screen's acc0_c / delta_c.  Columns n0 + i for i = t, t + nt, ... < bn.
__device__ __forceinline__ void stage_cols(const qg_epilogue& E, double* sC, int bn, int64_t n0, int64_t n, int t,
                                           int nt, int* off) {
  if (!col_doubles(bn, epi_row_only(E), E.bn_mean != nullptr)) return;
  for (int i = t; i < bn; i += nt) {
    const int64_t c = n0 + i;
    const bool ok = c < n;
    // absent terms are +0.0: x + 0.0 == x bit for bit here (x is never -0: the first
    // term k_acc*acc is >= +0 and RN sums that cancel give +0), so the dequant below
    // evaluates the reference's grouping without per-element branches
    const double cC = (ok && E.use_col) ? __dmul_rn(E.k_col, (double)E.col_sums[c]) : 0.0;
    const double cB = (ok && E.bias) ? E.bias[c] : 0.0;
    sC[0 * bn + i] = cC;
    sC[1 * bn + i] = cB;
    if (E.bn_mean) {
      sC[2 * bn + i] = ok ? E.bn_mean[c] : 0.0;
      sC[3 * bn + i] = ok ? E.bn_denom[c] : 1.0;
      sC[4 * bn + i] = ok ? E.bn_gamma[c] : 0.0;
      sC[5 * bn + i] = ok ? E.bn_beta[c] : 0.0;
      sC[6 * bn + i] = ok ? E.bn_inv_denom[c] : 1.0;
    } else {
      screen_col(E, i, cC, cB, reinterpret_cast<int32_t*>(sC + 2 * bn), reinterpret_cast<float*>(sC + 2 * bn) + bn,
                 off);
    }
  }
}

// Per-thread epilogue context: this lane owns one accumulator row (TMEM lane) and
// walks 8-column slices first, first+2, ...
struct EpiLane {
  uint32_t tmem_row;
  double* stage_real;         // fp64 outputs staged in shared memory (tile-local rows), or NULL
  bool has_acc, rvalid;
  int first, step, nslices, nvalid;   // this lane's slices: first, first + step, ...
  int64_t myrow, n0;
  __device__ __forceinline__ void load8(int cl8, uint32_t (&v)[8]) const {
    if (has_acc) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                     "=r"(v[7])
                   : "r"(tmem_row + (uint32_t)cl8));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    } else {
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) v[jj] = 0;
    }
  }
};

// Fused epilogue over this lane's slices, specialised on activation and BN so the
// 8 fp64 chains of a slice are straight-line code the scheduler can interleave.
// Dequant: ((((k_acc*acc) + rows) + cols) + const) + bias -- the reference's
// grouping (bitgemm.py:156-160); absent terms are +0.0 (exact, see sCol fill).
// Returns this lane's requantized code sum (packed output) for the row sums.
// ST: 0 = this stage to global memory; 1 = chained stage 1, codes into the shared
// memory operand of stage 2 (mid[k tile]); 2 = chained stage 2 (P.epi2, bn2, n2).
// The exact fp64 requant of ONE element (no batch norm): the screen's rare fallback.
struct ExactArgs {
  double k_acc, kconst, q_amin, q_scale, q_inv;
  uint32_t maxv;
};
template <int ACT, bool ROW_ONLY>
static __device__ __noinline__ uint32_t exact_code(const ExactArgs A, const double* sC, const double* sB, int cl,
                                                   uint32_t acc, double rterm, int64_t* status, int64_t flat) {
  double x = __dadd_rn(__dmul_rn(A.k_acc, (double)(int32_t)acc), rterm);
  if (!ROW_ONLY) x = __dadd_rn(__dadd_rn(__dadd_rn(x, sC[cl]), A.kconst), sB[cl]);
  if (ACT == QG_ACT_RELU) {
    const int hi = __double2hiint(x), m = ~(hi >> 31);
    x = __hiloint2double(hi & m, __double2loint(x) & m);
  }
  const R12 c = quantize_code_r12(x, A.q_amin, A.q_inv, A.maxv);
  return c.flag ? requant_exact(x, A.q_amin, A.q_scale, A.q_inv, A.maxv, status, flat) : c.code;
}

// The screened epilogue (ScreenRow) of this lane's slices, lean: per element one integer
// shift, one I2FP, 2 FFMA/FADD, a clamp, the floor and the margin test; bytes packed with
// PRMT, row sums with DP4A, one store per slice (8 byte stores for right-tiled outputs).
// Slices with a flagged element, ragged columns or rows past m are deferred to a second,
// warp-uniform pass (TMEM reloaded) that evaluates the exact fp64 path -- kept out of the
// main loop so its registers do not burden it.
// LAYOUT: 0 = chained stage 1 into the stage-2 operand in shared memory (mid0 / mid1),
// 1 = next LEFT operand (left-tiled codes), 2 = next RIGHT operand (right-tiled codes).
template <bool ROW_ONLY, int ST, int LAYOUT>
__device__ __forceinline__ void epi_store(const EpiLane& L, uint8_t* q_codes, int64_t r128, int64_t rbase, int lrow,
                                          uint8_t* mid0, uint8_t* mid1, int cl8, uint2 w, bool full) {
  const int64_t c = L.n0 + cl8;
  if (LAYOUT == 0) {
    uint8_t* dst = ((c >> 7) ? mid1 : mid0) + (lrow >> 3) * 1024 + ((c & 127) >> 4) * 128 + (lrow & 7) * 16 + (c & 15);
    *reinterpret_cast<uint2*>(dst) = w;
  } else if (L.rvalid) {
    if (LAYOUT == 1) {
      *reinterpret_cast<uint2*>(q_codes + (c >> 7) * (r128 << 7) + rbase + ((c & 127) >> 4) * 128 + (c & 15)) = w;
    } else {
      uint8_t* base = q_codes + rbase + (c >> 3) * 1024;
      if (full) {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          base[jj * 16] = (uint8_t)(w.x >> (8 * jj));
          base[(jj + 4) * 16] = (uint8_t)(w.y >> (8 * jj));
        }
      } else {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
          if (cl8 + jj < L.nvalid) base[jj * 16] = (uint8_t)((jj < 4 ? w.x : w.y) >> (8 * (jj & 3)));
      }
    }
  }
}

// Main-loop store of one full 8-column slice of a VALID row (rows past m and ragged slices
// go through the deferred pass): per-row bases precomputed by epi_fast, 32-bit column math.
// LAYOUT 0: shared-memory address (ms0 / ms1: the two 128-column K slots of stage 2's left
// operand at this row); 1: rowp = this row's left-tiled base, slab = bytes per 128 K
// columns; 2: rowp = this row's right-tiled base (K = row).
template <int LAYOUT>
__device__ __forceinline__ void epi_store_fast(uint8_t* rowp, uint32_t ms0, uint32_t ms1, int64_t slab, int c,
                                               uint2 w) {
  if (LAYOUT == 0) {
    const uint32_t a = ((c >> 7) ? ms1 : ms0) + (uint32_t)(((c & 127) >> 4) * 128 + (c & 15));
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(a), "r"(w.x), "r"(w.y) : "memory");
  } else if (LAYOUT == 1) {
    *reinterpret_cast<uint2*>(rowp + (int64_t)(c >> 7) * slab + (((c & 127) >> 4) * 128 + (c & 15))) = w;
  } else {
    uint8_t* base = rowp + (int64_t)(c >> 3) * 1024;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      base[jj * 16] = (uint8_t)(w.x >> (8 * jj));
      base[(jj + 4) * 16] = (uint8_t)(w.y >> (8 * jj));
    }
  }
}

// Screened estimate of one element: clamped fp32 y (floor bits in *f) and whether it is
// within the per-element margin 2^-21 (|y| + 2 alpha) of an integer (>= 2x the error bound
// 2^-24 (4 |Y| + 3 alpha) of ScreenRow).
template <bool ROW_ONLY>
__device__ __forceinline__ bool screen1(const ScreenRow& S, uint32_t acc, int32_t a0c, float dc, uint32_t& f) {
  const int32_t sh = ROW_ONLY ? (int32_t)acc - S.a0r : (int32_t)acc - S.a0r - a0c;
  float y = fmaf((float)sh, S.alpha, S.dr);
  if (!ROW_ONLY) y += dc;
  y = fminf(fmaxf(y, S.lo), S.hi);
  const float fl = __fadd_rd(y, 12582912.0f);              // 1.5 * 2^23 + floor(y)
  const float d = y - (fl - 12582912.0f);                  // y - floor(y), exact
  // distance to the nearest integer 1/2 - |d - 1/2| (d - 1/2 exact: d is a multiple of
  // ulp(y) >= 2^-24) against the margin; h = 1/2 - margin within 2^-25, the margin's slack
  // over the error bound is >= 2^-23
  const float h = fmaf(y, -0x1p-21f, S.hc);                // y >= 0.5 > 0 after the clamp
  f = __float_as_uint(fl);
  return fabsf(d - 0.5f) > h;
}

// Two elements of screen1 with the fp32 adds/FMAs in packed f32x2 form (FFMA2 / FADD2: one
// issue slot per pair; lane-wise the same IEEE operations and roundings as screen1, so the
// estimates, floors and flags are bit-identical to it -- the deferred pass re-derives them
// with screen1).
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t f2add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2add_rm(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2sub(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
template <bool ROW_ONLY>
__device__ __forceinline__ bool screen2(const ScreenRow& S, uint32_t acc0, uint32_t acc1, int32_t a0c0, int32_t a0c1,
                                        float dc0, float dc1, uint32_t& f0, uint32_t& f1) {
  const int32_t sh0 = ROW_ONLY ? (int32_t)acc0 - S.a0r : (int32_t)acc0 - S.a0r - a0c0;
  const int32_t sh1 = ROW_ONLY ? (int32_t)acc1 - S.a0r : (int32_t)acc1 - S.a0r - a0c1;
  uint64_t y = f2fma(f2pack((float)sh0, (float)sh1), f2pack(S.alpha, S.alpha), f2pack(S.dr, S.dr));
  if (!ROW_ONLY) y = f2add(y, f2pack(dc0, dc1));
  float y0, y1;
  f2unpack(y, y0, y1);
  y0 = fminf(fmaxf(y0, S.lo), S.hi);
  y1 = fminf(fmaxf(y1, S.lo), S.hi);
  y = f2pack(y0, y1);
  const uint64_t C = f2pack(12582912.0f, 12582912.0f);
  const uint64_t fl = f2add_rm(y, C);                       // 1.5 * 2^23 + floor(y)
  const uint64_t d = f2sub(y, f2sub(fl, C));                // y - floor(y), exact
  const uint64_t e = f2sub(d, f2pack(0.5f, 0.5f));
  const uint64_t h = f2fma(y, f2pack(-0x1p-21f, -0x1p-21f), f2pack(S.hc, S.hc));
  float e0, e1, h0, h1, l0, l1;
  f2unpack(e, e0, e1);
  f2unpack(h, h0, h1);
  f2unpack(fl, l0, l1);
  f0 = __float_as_uint(l0);
  f1 = __float_as_uint(l1);
  return (fabsf(e0) > h0) | (fabsf(e1) > h1);
}

template <bool ROW_ONLY, int ST, int LAYOUT>
__device__ __forceinline__ uint32_t epi_fast(const TiledParams& P, const qg_tseg& G, const EpiLane& L,
                                             const double* __restrict__ sCol, double rterm, uint8_t* mid0,
                                             uint8_t* mid1, const ScreenRow& S) {
  const int bn = ST == 2 ? P.bn2 : P.bn;
  uint8_t* const q_codes = G.q_codes;
  const int64_t myrow = L.myrow;
  const int lrow = (int)(myrow & 127);
  int64_t rbase = 0;
  if (LAYOUT == 1) rbase = (myrow >> 3) * 1024 + (myrow & 7) * 16;
  if (LAYOUT == 2) {
    const int64_t npad = ST == 2 ? P.out_npad2 : P.out_npad;
    rbase = (myrow >> 7) * (npad << 7) + ((myrow & 127) >> 4) * 128 + (myrow & 15);
  }
  const int64_t r128 = G.r128;
  const int nval = L.rvalid ? L.nvalid : 0;
  uint32_t rsum = 0, deferred = 0;
  // loop-invariant per-row bases (the slice loop only adds 32-bit column offsets)
  uint8_t* const rowp = q_codes + rbase;
  const int64_t slab = r128 << 7;
  const int n0i = (int)L.n0;
  uint32_t ms0 = 0, ms1 = 0;
  if (LAYOUT == 0) {
    const uint32_t ro = (uint32_t)((lrow >> 3) * 1024 + (lrow & 7) * 16);
    ms0 = smem_u32(mid0) + ro;
    ms1 = smem_u32(mid1) + ro;
  }
  const uint32_t sA0 = ROW_ONLY ? 0u : smem_u32(S.sA0), sD = ROW_ONLY ? 0u : smem_u32(S.sD);
  int k = 0;
  for (int sl = L.first; sl < L.nslices; sl += L.step, ++k) {
    const int cl8 = sl * 8;
    uint32_t v[8];
#ifdef QG_EPI_KNOCKOUTS
    if (P.dbg & 4) {
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) v[jj] = (uint32_t)(cl8 * 131 + jj * 17 + lrow);
    } else
#endif
      L.load8(cl8, v);
    int32_t a0[8];
    float dc[8];
    if (!ROW_ONLY) {
      uint32_t x[8], z[8];
      asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]) : "r"(sA0 + cl8 * 4));
      asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]) : "r"(sA0 + cl8 * 4 + 16));
      asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(z[0]), "=r"(z[1]), "=r"(z[2]), "=r"(z[3]) : "r"(sD + cl8 * 4));
      asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(z[4]), "=r"(z[5]), "=r"(z[6]), "=r"(z[7]) : "r"(sD + cl8 * 4 + 16));
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        a0[jj] = (int32_t)x[jj];
        dc[jj] = __uint_as_float(z[jj]);
      }
    }
    uint32_t t[8];
    bool bad = cl8 + 8 > nval;                               // ragged slice or row past m
#ifdef QG_EPI_KNOCKOUTS
    if (P.dbg & 2) {
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) t[jj] = v[jj];
    } else
#endif
    {
#pragma unroll
      for (int jj = 0; jj < 8; jj += 2)
        bad |= screen2<ROW_ONLY>(S, v[jj], v[jj + 1], ROW_ONLY ? 0 : a0[jj], ROW_ONLY ? 0 : a0[jj + 1],
                                 ROW_ONLY ? 0.f : dc[jj], ROW_ONLY ? 0.f : dc[jj + 1], t[jj], t[jj + 1]);
    }
    if (bad) {
      deferred |= 1u << k;
      continue;
    }
    uint2 w;
    w.x = __byte_perm(__byte_perm(t[0], t[1], 0x0040), __byte_perm(t[2], t[3], 0x0040), 0x5410);
    w.y = __byte_perm(__byte_perm(t[4], t[5], 0x0040), __byte_perm(t[6], t[7], 0x0040), 0x5410);
    rsum = __dp4a(w.x, 0x01010101u, rsum);
    rsum = __dp4a(w.y, 0x01010101u, rsum);
#ifdef QG_EPI_KNOCKOUTS
    if (P.dbg & 1) continue;
#endif
    epi_store_fast<LAYOUT>(rowp, ms0, ms1, slab, n0i + cl8, w);
  }
  // ---- deferred slices (warp-uniform walk: tcgen05.ld is collective): screened codes
  // again, the exact fp64 path only for the flagged elements, zeros past the valid region
  const uint32_t any = __reduce_or_sync(QG_FULL, deferred);
  if (any) {
    const qg_epilogue& E = ST == 2 ? P.epi2 : P.epi;
    const double k_acc = E.k_acc, kconst = E.use_const ? E.k_const : 0.0;
    const double q_amin = E.q_amin, q_scale = E.q_scale, q_inv = E.q_inv_scale;
    const uint32_t maxv = (1u << E.q_bits) - 1u;
    const bool relu = E.act == QG_ACT_RELU;
    const double* sC = sCol;
    const double* sB = sCol + bn;
    const int64_t pn = ST == 2 ? P.n2 : P.n;
    k = 0;
    for (int sl = L.first; sl < L.nslices; sl += L.step, ++k) {
      if (!((any >> k) & 1u)) continue;
      const int cl8 = sl * 8;
      uint32_t v[8];
      L.load8(cl8, v);
      if (!((deferred >> k) & 1u)) continue;
      uint32_t q[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const int c = cl8 + jj;
        uint32_t f = 0;
        const bool flag = screen1<ROW_ONLY>(S, v[jj], ROW_ONLY ? 0 : S.sA0[c], ROW_ONLY ? 0.f : S.sD[c], f);
        q[jj] = f & 0xFFu;
        if (c >= nval) {
          q[jj] = 0u;                                      // padding column / row past m: code 0
        } else if (flag) {
          double x = __dadd_rn(__dmul_rn(k_acc, (double)(int32_t)v[jj]), rterm);
          if (!ROW_ONLY) x = __dadd_rn(__dadd_rn(__dadd_rn(x, sC[c]), kconst), sB[c]);
          if (relu) {
            const int hh = __double2hiint(x), m = ~(hh >> 31);
            x = __hiloint2double(hh & m, __double2loint(x) & m);
          }
          const R12 r = quantize_code_r12(x, q_amin, q_inv, maxv);
          q[jj] = r.flag ? requant_exact(x, q_amin, q_scale, q_inv, maxv, G.status, myrow * pn + L.n0 + c) : r.code;
        }
      }
      const uint2 w = make_uint2(q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24),
                                 q[4] | (q[5] << 8) | (q[6] << 16) | (q[7] << 24));
      rsum = __dp4a(w.x, 0x01010101u, rsum);
      rsum = __dp4a(w.y, 0x01010101u, rsum);
      epi_store<ROW_ONLY, ST, LAYOUT>(L, q_codes, r128, rbase, lrow, mid0, mid1, cl8, w, cl8 + 8 <= nval);
    }
  }
  return rsum;
}

template <int ACT, bool HAS_BN, bool ROW_ONLY, int ST>
__device__ __forceinline__ uint32_t epi_slices(const TiledParams& P, const qg_tseg& G, const EpiLane& L,
                                               const double* __restrict__ sCol, double rterm, uint8_t* mid0,
                                               uint8_t* mid1) {
  const qg_epilogue& E = ST == 2 ? P.epi2 : P.epi;
  const int bn = ST == 2 ? P.bn2 : P.bn;
  const double* sC = sCol;
  const double* sB = sCol + bn;
  const double* sMean = sCol + 2 * bn;
  const double* sDen = sCol + 3 * bn;
  const double* sInv = sCol + 6 * bn;       // RN(1 / denom): div_rn's correctly rounded division
  const double* sGam = sCol + 4 * bn;
  const double* sBeta = sCol + 5 * bn;
  const double k_acc = E.k_acc;
  const double kconst = E.use_const ? E.k_const : 0.0;
  const bool packed = E.out_kind == QG_OUT_PLANES;
  const uint32_t maxv = packed ? (1u << E.q_bits) - 1u : 0u;
  const double q_amin = E.q_amin, q_scale = E.q_scale, q_inv = E.q_inv_scale;
  const int out_layout = ST == 2 ? P.out_layout2 : P.out_layout;
  // segment fields in registers (G lives in global memory; the code stores below
  // could alias it, so the compiler would otherwise reload every slice)
  uint8_t* const q_codes = G.q_codes;
  double* const out_real = G.out_real;
  int64_t* const status = G.status;
  const int64_t r128 = G.r128, out_npad = ST == 2 ? P.out_npad2 : P.out_npad, pn = ST == 2 ? P.n2 : P.n;
  const int lrow = (int)(L.myrow & 127);
  uint32_t rsum = 0;                                        // <= 256 cols x 255: fits u32
  for (int sl = L.first; sl < L.nslices; sl += L.step) {
    const int cl8 = sl * 8;
    uint32_t v[8];
    L.load8(cl8, v);
    const bool full = L.rvalid && cl8 + 8 <= L.nvalid;
    uint32_t q[8];
    {
    double real[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const int cl = cl8 + jj;
      double x = __dadd_rn(__dmul_rn(k_acc, (double)(int32_t)v[jj]), rterm);
      // ROW_ONLY (aggregation: exact 0/1 left operand, no bias): the reference adds
      // nothing else; otherwise the absent terms are +0.0
      if (!ROW_ONLY) x = __dadd_rn(__dadd_rn(__dadd_rn(x, sC[cl]), kconst), sB[cl]);
      if (HAS_BN) x = __dadd_rn(__dmul_rn(div_rn(__dsub_rn(x, sMean[cl]), sDen[cl], sInv[cl]), sGam[cl]), sBeta[cl]);
      if (ACT == QG_ACT_RELU) {
        if (packed) {
          // sign mask: -0 also maps to +0, which requantizes to the same code
          const int hi = __double2hiint(x), m = ~(hi >> 31);
          x = __hiloint2double(hi & m, __double2loint(x) & m);
        } else {
          x = (x < 0.0) ? 0.0 : x;
        }
      }
      if (ACT == QG_ACT_TANH) x = tanh_f32(x);
      real[jj] = x;
    }
    if (!packed) {
      if (L.rvalid) {
        double* dst = L.stage_real ? L.stage_real + (int64_t)lrow * pn : out_real + L.myrow * pn + L.n0;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
          if (cl8 + jj < L.nvalid) dst[cl8 + jj] = real[jj];
      }
      continue;
    }
    // requant: branch-free candidates; one (rare, divergent) exact pass for ragged
    // edges, non-finite values or quotients within 2^-40 of a code boundary
    bool slow = !full;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const R12 c = quantize_code_r12(real[jj], q_amin, q_inv, maxv);
      q[jj] = c.code;
      slow |= c.flag;
    }
    if (slow) {
      // non-finite x always lands here: r is then inf/NaN (hi >= 0x7ff00000) or negative
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
        q[jj] = (L.rvalid && cl8 + jj < L.nvalid)
                    ? requant_exact(real[jj], q_amin, q_scale, q_inv, maxv, status, L.myrow * pn + L.n0 + cl8 + jj)
                    : 0u;
    }
    }
    const uint32_t lo = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
    const uint32_t hi = q[4] | (q[5] << 8) | (q[6] << 16) | (q[7] << 24);
    rsum += ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
    if (ST == 1) {
      // stage 2's LEFT operand in shared memory (UMMA K-major core matrices, one 16 KB
      // slot per 128 K columns); rows past m hold zeros (their stage-2 rows are not stored).
      const int c = (int)L.n0 + cl8;
      uint8_t* dst = ((c >> 7) ? mid1 : mid0) + (lrow >> 3) * 1024 + ((c & 127) >> 4) * 128 + (lrow & 7) * 16 +
                     (c & 15);
      *reinterpret_cast<uint2*>(dst) = make_uint2(lo, hi);
      continue;
    }
    if (L.rvalid) {
      const int64_t cb = L.n0 + cl8;
      if (out_layout == 1) {
        // next LEFT operand: 8 consecutive K bytes of this row = one 8-byte store
        *reinterpret_cast<uint2*>(q_codes + left_tile_off(L.myrow, cb, r128)) = make_uint2(lo, hi);
      } else {
        // next RIGHT operand (K = this row): consecutive lanes write consecutive bytes
        uint8_t* base = q_codes + right_tile_off(L.myrow, cb, out_npad);
        if (full) {
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) base[jj * 16] = (uint8_t)q[jj];   // n += 1 -> +16 B
        } else {
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            if (cl8 + jj < L.nvalid) base[jj * 16] = (uint8_t)q[jj];
        }
      }
    }
  }
  return rsum;
}

// Per-CTA state of the tile pipeline (ring position, accumulator phase).
struct TileRing {
  uint8_t* stage0;            // S ring slots of (16 KB + bn_max * 128 B)
  double* sCol;               // per-column epilogue constants
  uint64_t* full;
  uint64_t* empty;
  uint64_t* aready;           // a_bits: the expanded A operand of a ring slot is ready
  uint64_t* aempty;           // a_bits 2: the MMAs reading a TMEM A slot completed
  uint64_t* done;
  unsigned long long* sRowSum;
  double* sRowTerm;
  int64_t* sRowIn;            // the stage's left-operand row sums (staged with the row terms)
  int* sOff;                  // [stage 1, stage 2]: a column's screen shift is out of range
  uint32_t tmem;
  int S;
  uint32_t it0;               // ring position (K tiles issued so far)
  uint32_t ndone;             // accumulator phases completed so far
  uint32_t ring_bytes;        // bytes of the ring (free for output staging after the last MMA)
  bool pdl_wait;              // griddepcontrol.wait still pending (PDL-launched single tile)
  int pref;                   // producer: K tiles of the CURRENT tile already issued (persistent prefetch)
};

// Epilogue of one 128-row x bn tile held in this CTA's TMEM: 8-column slices over all
// 8 warps, fused dequant/BN/act/requant (or fp64 / int32 output); the lane's code row
// sum is accumulated into R.sRowSum (flushed to global by the caller).  ST as in
// epi_slices (1: chained stage 1 into mid0/mid1; 2: chained stage 2).
template <int ST>
__device__ __forceinline__ void tile_epilogue(const TiledParams& P, const qg_tseg& G, TileRing& R, int64_t tile,
                                              int64_t rb, int64_t n0, int nk, uint32_t tmem, const double* sCol,
                                              bool fused, uint8_t* mid0 = nullptr, uint8_t* mid1 = nullptr) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int bn = ST == 2 ? P.bn2 : P.bn;
  const int64_t pn = ST == 2 ? P.n2 : P.n;
  const qg_epilogue& E = ST == 2 ? P.epi2 : P.epi;
  // ---------------- epilogue: 8-column TMEM slices over all 8 warps ----------------
  // warps 4q..4q+3 cover the 128 TMEM lanes; the blockDim/128 warp groups split the slices
  const int quad = warp & 3, half = warp >> 2, groups = (int)(blockDim.x >> 7);
  const int64_t r0 = rb * 128 + quad * 32;
  const int64_t myrow = r0 + lane;
  const bool rvalid = myrow < G.m;
  const int64_t rem_cols = pn - n0;
  const int ncols_cta = rem_cols <= 0 ? 0 : (rem_cols < bn ? (int)rem_cols : bn);
  const int nslices = (ncols_cta + 7) >> 3;
  const bool packed = fused && E.out_kind == QG_OUT_PLANES;
  EpiLane L;
  L.stage_real = nullptr;
  // fp64 outputs of a tile that spans all output columns form ONE contiguous block of
  // rows in out_real: stage them in the (now idle) ring and store them coalesced
  const bool stage_out = fused && E.out_kind == QG_OUT_REAL && n0 == 0 && pn <= bn &&
                         (uint64_t)128 * (uint64_t)pn * 8u <= R.ring_bytes;
  if (stage_out) L.stage_real = reinterpret_cast<double*>(R.stage0);
  L.tmem_row = tmem + ((uint32_t)(quad * 32) << 16);
  L.has_acc = nk > 0;
  L.first = half;
  L.step = groups;
  L.nslices = nslices;
  L.nvalid = (int)(pn - n0);
  L.rvalid = myrow < G.m;
  L.myrow = myrow;
  L.n0 = n0;
  uint32_t rsum = 0;
  if (ST == 0 && !fused) {
    const bool vec_ok = (P.n & 3) == 0 && (reinterpret_cast<uintptr_t>(G.out_i32) & 15) == 0;
    for (int sl = half; sl < nslices; sl += groups) {
      uint32_t v[8];
      L.load8(sl * 8, v);
      if (rvalid) {
        int32_t* dst = G.out_i32 + myrow * P.n + n0 + sl * 8;
        if (vec_ok && sl * 8 + 8 <= L.nvalid) {
          // 8 consecutive columns of this row: two 16-byte stores (n % 4 == 0 keeps them aligned)
          reinterpret_cast<int4*>(dst)[0] = make_int4((int)v[0], (int)v[1], (int)v[2], (int)v[3]);
          reinterpret_cast<int4*>(dst)[1] = make_int4((int)v[4], (int)v[5], (int)v[6], (int)v[7]);
        } else {
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            if (sl * 8 + jj < L.nvalid) dst[jj] = (int32_t)v[jj];
        }
      }
    }
  } else {
    // one uniform dispatch per tile: the slice loop below is straight-line per variant
    const double rterm = rvalid ? R.sRowTerm[quad * 32 + lane] : 0.0;
    const bool row_only = !E.use_col && !E.use_const && !E.bias;
    ScreenRow S;
    S.on = false;
    if (packed && P.screen && E.screen_rmax > 0.0 && E.act != QG_ACT_TANH && !E.bn_mean && !R.sOff[ST == 2]) {
      // per-row acc bound (unsigned codes): left row sum x max right code; the integer
      // shift acc - acc0_r - acc0_c must not overflow (acc < 2^30, |acc0| <= 2^29)
      int64_t rs = 0;
      bool known = true;
      if (ST == 2) rs = (int64_t)R.sRowSum[quad * 32 + lane];
      else if (G.row_sums) rs = R.sRowIn ? R.sRowIn[quad * 32 + lane] : (rvalid ? G.row_sums[myrow] : 0);
      else known = false;
      const double accmax = (double)rs * E.screen_rmax;
      double ia;
      const double alpha = screen_alpha(E, ia);
      const double beta = (rterm - E.q_amin) * E.q_inv_scale;
      double a0 = rint(-beta * ia);
      const bool a0_ok = fabs(a0) <= 0x1p29;
      if (!a0_ok) a0 = 0.0;
      // CTA-uniform (the staged code stores below rely on it); a warp whose rows could
      // overflow the integer shift (acc >= 2^30) or lack row sums sends every element to
      // the exact path instead (margin +inf)
      const bool warp_ok = __all_sync(QG_FULL, known && accmax < 0x1p30);
      S.on = alpha > 0.0 && alpha < 0x1p60;
      if (S.on) {
        const uint32_t maxv = (1u << E.q_bits) - 1u;
        float lo = 0.5f;
        double q0 = 0.0;
        if (E.act == QG_ACT_RELU) {
          // q0 ~ the reference quotient of x = 0 (quantize.py:102-104); its fp32 copy is
          // inside the margin (y >= lo >= q0f)
          q0 = -E.q_amin * E.q_inv_scale;
          lo = fmaxf(lo, (float)q0);
        }
        // per-element margin 2^-21 (|y| + 2 alpha) (screen1): this is its constant part; +inf
        // sends every element of the row to the exact path, -1 (rows past m) none
        const double margin = (2.0 * alpha + (double)maxv * 0x1p-20) * 0x1p-21 + 0x1p-40;
        S.mrg = !rvalid ? -1.0f
                        : (warp_ok && a0_ok && margin < 0.125 && fabs(q0) < 0x1p20) ? __double2float_ru(margin)
                                                                                    : __int_as_float(0x7f800000);
        S.hc = 0.5f - S.mrg;
        S.a0r = (int32_t)a0;
        S.dr = (float)(beta + a0 * alpha);
        S.alpha = (float)alpha;
        S.lo = lo;
        S.hi = (float)maxv + 0.5f;
        S.sA0 = reinterpret_cast<const int32_t*>(sCol + 2 * bn);
        S.sD = reinterpret_cast<const float*>(sCol + 2 * bn) + bn;
      }
    }
    const int out_layout = ST == 2 ? P.out_layout2 : P.out_layout;
    if (S.on && (ST == 1 || out_layout == 1 || out_layout == 2)) {
      if (ST == 1) {
        rsum = row_only ? epi_fast<true, ST, 0>(P, G, L, sCol, rterm, mid0, mid1, S)
                        : epi_fast<false, ST, 0>(P, G, L, sCol, rterm, mid0, mid1, S);
      } else if (out_layout == 1) {
        rsum = row_only ? epi_fast<true, ST, 1>(P, G, L, sCol, rterm, mid0, mid1, S)
                        : epi_fast<false, ST, 1>(P, G, L, sCol, rterm, mid0, mid1, S);
      } else {
        rsum = row_only ? epi_fast<true, ST, 2>(P, G, L, sCol, rterm, mid0, mid1, S)
                        : epi_fast<false, ST, 2>(P, G, L, sCol, rterm, mid0, mid1, S);
      }
    } else
    switch ((E.act * 2 + (E.bn_mean != nullptr ? 1 : 0)) * 2 + (row_only ? 1 : 0)) {
#define QG_EPI_CASE(i, A, B, Rw) \
  case i: rsum = epi_slices<A, B, Rw, ST>(P, G, L, sCol, rterm, mid0, mid1); break;
      QG_EPI_CASE(0, QG_ACT_NONE, false, false)
      QG_EPI_CASE(1, QG_ACT_NONE, false, true)
      QG_EPI_CASE(2, QG_ACT_NONE, true, false)
      QG_EPI_CASE(3, QG_ACT_NONE, true, true)
      QG_EPI_CASE(4, QG_ACT_RELU, false, false)
      QG_EPI_CASE(5, QG_ACT_RELU, false, true)
      QG_EPI_CASE(6, QG_ACT_RELU, true, false)
      QG_EPI_CASE(7, QG_ACT_RELU, true, true)
      QG_EPI_CASE(8, QG_ACT_TANH, false, false)
      QG_EPI_CASE(9, QG_ACT_TANH, false, true)
      QG_EPI_CASE(10, QG_ACT_TANH, true, false)
      default: rsum = epi_slices<QG_ACT_TANH, true, true, ST>(P, G, L, sCol, rterm, mid0, mid1); break;
#undef QG_EPI_CASE
    }
  }
  // chained stage 2 accumulates into the second half of sRowSum
  if (packed && (ST == 1 || G.q_row_sums) && rsum)
    atomicAdd(&R.sRowSum[(ST == 2 ? 128 : 0) + quad * 32 + lane], (unsigned long long)rsum);
  if (stage_out) {
    // the tile's rows [rb*128, min(m, rb*128 + 128)) x pn doubles, contiguous in out_real
    __syncthreads();
    const int64_t rows = G.m - rb * 128 < 128 ? G.m - rb * 128 : 128;
    // consecutive threads -> consecutive doubles (segment bases are only 8-byte aligned)
    const int64_t total = rows * pn;
    double* dst = G.out_real + rb * 128 * pn;
    for (int64_t i = tid; i < total; i += blockDim.x) dst[i] = L.stage_real[i];
  }
}

// One work item: (segment, 128-row block, N tile) -> fused GEMM tile.  Ends with a
// CTA barrier so the next tile may overwrite TMEM / shared staging.
template <int TMEM_COLS, bool CHAIN>
__device__ __forceinline__ void tiled_tile(const TiledParams& P, int64_t tile, TileRing& R) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int bn = P.bn, S = R.S;
  if (tid == 0) tstamp(P, tile, 0);

  // ---- segment lookup (uniform): last segment with cta_begin <= tile
  const qg_tseg& G = P.segs[find_seg(P.segs, P.nsegs, tile)];
  const int64_t local = tile - G.cta_begin;
  const int64_t rb = local / P.n_tiles;
  const int nt = (int)(local % P.n_tiles);
  const int64_t n0 = (int64_t)nt * bn;
  // persistent: the next work item of this CTA (warp-cooperative lookup, all threads)
  const int64_t next = tile + (int64_t)gridDim.x;
  const bool has_next = P.persist && next < P.total_ctas;
  const qg_tseg& Gn = P.segs[has_next ? find_seg(P.segs, P.nsegs, next) : 0];
  const int64_t localn = has_next ? next - Gn.cta_begin : 0;
  const int64_t rbn = localn / P.n_tiles;
  const int64_t n0n = (int64_t)(localn % P.n_tiles) * bn;

  // stage = [A: 16 KB UMMA bytes][B: bn x 128 B]                       (bytes)
  //         [A: 16 KB UMMA bytes][B: bn x 128 B][2 KB packed bit block] (a_bits 1: A expanded in smem)
  //         [B: bn x 128 B][2 KB packed bit block]                       (a_bits 2: A expanded into TMEM)
  const uint32_t b_bytes = (uint32_t)bn * 128u, slot_b = (uint32_t)P.slot_bn * 128u;
  uint8_t* stage0 = R.stage0;
  const bool ats = P.a_blocks && P.a_bits == 2;            // A operand from tensor memory
  const bool abits = P.a_blocks && P.a_bits == 1;
  const uint32_t a_bytes = ats ? 0u : 16384u;              // offset of B in a slot
  const uint32_t bits_off = a_bytes + slot_b;              // offset of the packed bits
  const uint32_t stage_bytes = tiled_stage_bytes(P.slot_bn, P.a_bits);
  double* sCol = R.sCol;
  uint64_t* full = R.full;
  uint64_t* empty = R.empty;
  const uint32_t tmem = R.tmem;
  const uint32_t it0 = R.it0;

  int nk, kbase = 0;
  if (P.a_blocks) { nk = G.blk_count[rb]; kbase = G.blk_base[rb]; }
  else nk = G.k_tiles;
  R.it0 += (uint32_t)nk;                                  // every thread tracks the ring position

  const bool fused = P.mode == QG_GEMM_EPILOGUE;
  const qg_epilogue& E = P.epi;
  // chained stage 2: per-column constants after stage 1's
  double* sCol2 = sCol + col_doubles(bn, epi_row_only(E), E.bn_mean != nullptr);
  if (tid < 128) R.sRowSum[tid] = 0ull;
  if (CHAIN && tid < 128) R.sRowSum[128 + tid] = 0ull;
  if (tid == 0) tstamp(P, tile, 1);

  if (warp == 0 && lane == 0) {
    // ---------------- producer: two bulk copies per K tile ----------------
    const uint8_t* bbase = G.b + (n0 >> 3) * 1024;
    int it_begin = 0;
    if (R.pdl_wait) {
      // PDL: the STATIC operand of the first ring-full of K tiles (adjacency blocks, or the
      // weights of a dense-left GEMM) is fetched while the predecessor grid drains; the
      // operand it produced only after griddepcontrol.wait
      const int pre = nk < S ? nk : S;
      uint8_t* dst0 = stage0;
      for (int it = 0; it < pre; ++it) {
        uint8_t* dst = dst0 + (size_t)((it0 + it) % S) * stage_bytes;
        uint64_t* fb = &full[(it0 + it) % S];
        if (abits || ats) {
          mbar_expect_tx(fb, 2048u + b_bytes);
          bulk_g2s(dst + bits_off, G.a + (int64_t)(kbase + it) * 2048, 2048u, fb);
        } else if (P.a_blocks) {
          mbar_expect_tx(fb, 16384u + b_bytes);
          bulk_g2s(dst, G.a + (int64_t)(kbase + it) * 16384, 16384u, fb);
        } else {
          mbar_expect_tx(fb, a_bytes + b_bytes);
          bulk_g2s(dst + a_bytes, bbase + (int64_t)it * (P.b_npad << 7), b_bytes, fb);
        }
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");
      for (int it = 0; it < pre; ++it) {
        uint8_t* dst = dst0 + (size_t)((it0 + it) % S) * stage_bytes;
        uint64_t* fb = &full[(it0 + it) % S];
        if (P.a_blocks)
          bulk_g2s(dst + a_bytes, bbase + (int64_t)G.blk_kt[kbase + it] * (P.b_npad << 7), b_bytes, fb);
        else
          bulk_g2s(dst, G.a + (int64_t)it * (G.r128 << 7) + rb * 16384, a_bytes, fb);
      }
      it_begin = pre;
    }
    // one K tile `it` of work item (Gx, rbx, n0x, kbasex) into ring position g
    auto issue = [&](const qg_tseg& Gx, int64_t rbx, int64_t n0x, int kbasex, int it, uint32_t g) {
      const int s = (int)(g % (uint32_t)S);
      if (g >= (uint32_t)S) mbar_wait(smem_u32(&empty[s]), ((g / S) - 1) & 1);
      int kt;
      const uint8_t* asrc;
      uint8_t* dst = stage0 + (size_t)s * stage_bytes;
      if (abits || ats) {
        // 2 KB packed block -> staging; the expander warps build the operand (smem or TMEM)
        kt = Gx.blk_kt[kbasex + it];
        mbar_expect_tx(&full[s], 2048u + b_bytes);
        bulk_g2s(dst + bits_off, Gx.a + (int64_t)(kbasex + it) * 2048, 2048u, &full[s]);
      } else {
        if (P.a_blocks) { kt = Gx.blk_kt[kbasex + it]; asrc = Gx.a + (int64_t)(kbasex + it) * 16384; }
        else { kt = it; asrc = Gx.a + (int64_t)kt * (Gx.r128 << 7) + rbx * 16384; }
        mbar_expect_tx(&full[s], a_bytes + b_bytes);
        bulk_g2s(dst, asrc, a_bytes, &full[s]);
      }
      bulk_g2s(dst + a_bytes, Gx.b + (n0x >> 3) * 1024 + (int64_t)kt * (P.b_npad << 7), b_bytes, &full[s]);
    };
    if (R.pref > it_begin) it_begin = R.pref;            // issued during the previous item's epilogue
    R.pref = 0;
    for (int it = it_begin; it < nk; ++it) issue(G, rb, n0, kbase, it, it0 + (uint32_t)it);
    if (!CHAIN && has_next) {
      // persistent: the next work item's first ring-full, behind this item's K tiles (the
      // slots free up as this item's MMAs retire; no dependence on the epilogue)
      int nnk, nkb = 0;
      if (P.a_blocks) { nnk = Gn.blk_count[rbn]; nkb = Gn.blk_base[rbn]; }
      else nnk = Gn.k_tiles;
      const int pre = nnk < S ? nnk : S;
      for (int j = 0; j < pre; ++j) issue(Gn, rbn, n0n, nkb, j, it0 + (uint32_t)nk + (uint32_t)j);
      R.pref = pre;
    }
    if (CHAIN) {
      // stage 2's (static) right operand, one K tile per ring position after stage 1's;
      // its left operand is written into the same slots by the stage-1 epilogue
      const uint32_t wb = (uint32_t)P.bn2 * 128u;
      for (int j = 0; j < P.k2; ++j) {
        const uint32_t g = it0 + (uint32_t)nk + (uint32_t)j;
        const int s = (int)(g % (uint32_t)S);
        if (g >= (uint32_t)S) mbar_wait(smem_u32(&empty[s]), ((g / S) - 1) & 1);
        mbar_expect_tx(&full[s], wb);
        bulk_g2s(stage0 + (size_t)s * stage_bytes + a_bytes, P.w2 + (int64_t)j * (P.w2_npad << 7), wb, &full[s]);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = idesc_u8(bn);
    for (int it = 0; it < nk; ++it) {
      const uint32_t g = it0 + (uint32_t)it;
      const int s = (int)(g % (uint32_t)S);
      mbar_wait(smem_u32((abits || ats) ? &R.aready[s] : &full[s]), (g / S) & 1);
      if (it == 0) tstamp(P, tile, 2);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = smem_u32(stage0 + (size_t)s * stage_bytes), b0 = a0 + a_bytes;
      if (ats) {
        // A from the TMEM ring slot g % a_slots (lane = row, 4 K bytes per column): 8 columns
        // per K = 32
        const uint32_t sa = g % (uint32_t)P.a_slots;
        const uint32_t at = tmem + (uint32_t)P.a_col0 + 32u * sa;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_i8_ts(tmem, at + 8u * (uint32_t)kk, umma_desc(b0 + kk * 256u), idesc, (it > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&R.aempty[sa]);
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_i8(tmem, umma_desc(a0 + kk * 256u), umma_desc(b0 + kk * 256u), idesc, (it > 0 || kk > 0) ? 1u : 0u);
      }
      umma_commit(&empty[s]);
    }
    if (nk > 0) umma_commit(R.done);
  } else if (warp >= 2 && fused) {
    // warps 2..7 stage the epilogue constants while the main loop runs: the row terms
    // RN(k_row * row_sum) (predecessor outputs) and the per-column constants
    const int t = tid - 64;
    if (R.pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (t < 128) {
      const int64_t row = rb * 128 + t;
      const int64_t rsin = (G.row_sums && row < G.m) ? G.row_sums[row] : 0;
      if (R.sRowIn) R.sRowIn[t] = rsin;
      R.sRowTerm[t] = (E.use_row && row < G.m) ? __dmul_rn(E.k_row, (double)rsin) : 0.0;
    }
    stage_cols(E, sCol, bn, n0, P.n, t, (int)blockDim.x - 64, &R.sOff[0]);
    if (CHAIN) stage_cols(P.epi2, sCol2, P.bn2, 0, P.n2, t, (int)blockDim.x - 64, &R.sOff[1]);
  }
  if (abits && warp >= 2) {
    // expander warps: packed 128x128 bit block -> UMMA K-major 0/1 bytes (16 KB) per ring
    // slot, one 16-byte store per (row, 16-bit K-core); unit u = (row/8, K-core, row%8) is
    // the core-matrix order, so consecutive lanes store consecutive 16 B
    const int et = tid - 64, nt = (int)blockDim.x - 64;
    for (int it = 0; it < nk; ++it) {
      const uint32_t g = it0 + (uint32_t)it;
      const int s = (int)(g % (uint32_t)S);
      mbar_wait(smem_u32(&full[s]), (g / S) & 1);
      uint8_t* slot = stage0 + (size_t)s * stage_bytes;
      const uint32_t* bits = reinterpret_cast<const uint32_t*>(slot + a_bytes + slot_b);
      for (int u = et; u < 1024; u += nt) {
        const int r = ((u >> 6) << 3) | (u & 7), c = (u >> 3) & 7;
        const uint32_t x = bits[r * 4 + (c >> 1)] >> ((c & 1) * 16);
        *reinterpret_cast<uint4*>(slot + u * 16) =
            make_uint4(expand_nibble(x & 0xFu), expand_nibble((x >> 4) & 0xFu), expand_nibble((x >> 8) & 0xFu),
                       expand_nibble((x >> 12) & 0xFu));
      }
      // generic-proxy smem writes -> visible to the tensor core (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&R.aready[s]);
    }
  }
  if (ats && warp >= 4 && warp < 8) {
    // A into TENSOR MEMORY: warp w (lanes 32 (w % 4) ..) expands its 32 rows -- thread =
    // row, 128 bits -> 128 bytes of 0/1 = 32 TMEM columns -- with one tcgen05.st per K
    // tile; no shared-memory traffic for A beyond the 2 KB of bits
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t SA = (uint32_t)P.a_slots;
    for (int it = 0; it < nk; ++it) {
      const uint32_t g = it0 + (uint32_t)it;
      const int s = (int)(g % (uint32_t)S);
      const uint32_t sa = g % SA;
      mbar_wait(smem_u32(&full[s]), (g / S) & 1);
      if (g >= SA) mbar_wait(smem_u32(&R.aempty[sa]), ((g / SA) - 1) & 1);   // slot read by the MMA
      const uint4 b4 = *reinterpret_cast<const uint4*>(stage0 + (size_t)s * stage_bytes + bits_off + r * 16);
      const uint32_t wv[4] = {b4.x, b4.y, b4.z, b4.w};
      uint32_t x[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) x[c] = expand_nibble((wv[c >> 3] >> (4 * (c & 7))) & 0xFu);
      tmem_st32(tmem + lane_base + (uint32_t)P.a_col0 + 32u * sa, x);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&R.aready[s]);
    }
  }
  __syncwarp();
  // every thread is past the predecessor grid before any global write (nk == 0 tiles
  // reach the epilogue without waiting on the pipeline)
  if (R.pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  R.pdl_wait = false;
  if (nk > 0) {
    mbar_wait(smem_u32(R.done), R.ndone & 1);
    R.ndone += 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  __syncthreads();   // sCol / row terms / zeroed row sums visible to all epilogue warps
  if (tid == 0) tstamp(P, tile, 3);

  if (CHAIN) {
    // ---- chained stage 2: stage 1's codes -> shared memory -> dense GEMM -> epilogue 2
    const uint32_t itc = R.it0;                          // ring position of stage-2 K tile 0
    R.it0 += (uint32_t)P.k2;
    uint8_t* mid0 = stage0 + (size_t)(itc % (uint32_t)S) * stage_bytes;
    uint8_t* mid1 = stage0 + (size_t)((itc + 1) % (uint32_t)S) * stage_bytes;
    tile_epilogue<1>(P, G, R, tile, rb, n0, nk, tmem, sCol, true, mid0, mid1);
    // generic-proxy code stores -> visible to the tensor core; TMEM reads retired
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const qg_epilogue& E2 = P.epi2;
    if (tid < 128) {
      // stage 2's row terms: RN(k_row * code row sum), the sums of the codes just written
      const int64_t row = rb * 128 + tid;
      const unsigned long long rs = R.sRowSum[tid];
      R.sRowTerm[tid] = (E2.use_row && row < G.m) ? __dmul_rn(E2.k_row, (double)rs) : 0.0;
    }
    if (warp == 1 && lane == 0) {
      const uint32_t idesc2 = idesc_u8(P.bn2);
      for (int j = 0; j < P.k2; ++j) {
        const uint32_t g = itc + (uint32_t)j;
        const int s = (int)(g % (uint32_t)S);
        mbar_wait(smem_u32(&full[s]), (g / S) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a0 = smem_u32(stage0 + (size_t)s * stage_bytes), b0 = a0 + a_bytes;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_i8(tmem, umma_desc(a0 + kk * 256u), umma_desc(b0 + kk * 256u), idesc2, (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit(&empty[s]);
      }
      umma_commit(R.done);
    }
    mbar_wait(smem_u32(R.done), R.ndone & 1);
    R.ndone += 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
    __syncthreads();                                     // stage-2 row terms visible
    if (tid == 0) tstamp(P, tile, 7);
    tile_epilogue<2>(P, G, R, tile, rb, 0, P.k2, tmem, sCol2, true);
    if (tid == 0) tstamp(P, tile, 4);
    if (E2.out_kind == QG_OUT_PLANES && G.q_row_sums) {
      __syncthreads();
      if (tid < 128 && rb * 128 + tid < G.m && R.sRowSum[128 + tid])
        atomicAdd(reinterpret_cast<unsigned long long*>(G.q_row_sums + rb * 128 + tid), R.sRowSum[128 + tid]);
    }
  } else {
    tile_epilogue<0>(P, G, R, tile, rb, n0, nk, tmem, sCol, fused);
    if (tid == 0) tstamp(P, tile, 4);
    if (P.mode == QG_GEMM_EPILOGUE && E.out_kind == QG_OUT_PLANES && G.q_row_sums) {
      __syncthreads();
      if (tid < 128 && rb * 128 + tid < G.m && R.sRowSum[tid])
        atomicAdd(reinterpret_cast<unsigned long long*>(G.q_row_sums + rb * 128 + tid), R.sRowSum[tid]);
    }
  }
  if (tid < 2) R.sOff[tid] = 0;                          // next work item re-derives its screen flags
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) tstamp(P, tile, 5);
}

// CTA setup: TMEM allocation, ring barriers.
template <int TMEM_COLS>
__device__ __forceinline__ void tiled_setup(TileRing& R, uint8_t* smem, uint64_t* full, uint64_t* empty,
                                            uint64_t* aready, uint64_t* aempty, bool a_tmem,
                                            uint64_t* done, uint32_t* tmem_base_s, unsigned long long* sRowSum,
                                            double* sRowTerm, int S, uint32_t stage_bytes_max) {
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_s)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    // aready: one arrival per expander warp (warps 2.. for smem expansion, 4..7 for TMEM)
    for (int i = 0; i < S; ++i) mbar_init(&aready[i], a_tmem ? 4u : (blockDim.x >> 5) - 2);
    for (int i = 0; i < 4; ++i) mbar_init(&aempty[i], 1);
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  R.stage0 = smem;
  R.aready = aready;
  R.aempty = aempty;
  R.sCol = reinterpret_cast<double*>(smem + (size_t)S * stage_bytes_max);
  R.full = full;
  R.empty = empty;
  R.done = done;
  R.sRowSum = sRowSum;
  R.sRowTerm = sRowTerm;
  R.S = S;
  R.ring_bytes = (uint32_t)S * stage_bytes_max;
  R.it0 = 0;
  R.ndone = 0;
  R.pdl_wait = false;
  R.pref = 0;
}

template <int TMEM_COLS, int MINB, int NT, bool CHAIN = false>
__global__ void __launch_bounds__(NT, MINB) tc_tiled_kernel(const __grid_constant__ TiledParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[8], empty[8], aready[8], aempty[4], done;
  __shared__ uint32_t tmem_base_s;
  __shared__ unsigned long long sRowSum[CHAIN ? 256 : 128];   // chained: [stage 1 | stage 2]
  __shared__ double sRowTerm[128];
  // staged input row sums; the 3-CTA/SM variant keeps its static footprint (reads global)
  __shared__ int64_t sRowIn[MINB >= 3 ? 1 : 128];
  __shared__ int sOff[2];
  TileRing R;
  if (threadIdx.x < 2) sOff[threadIdx.x] = 0;
  R.sOff = sOff;
  R.sRowIn = MINB >= 3 ? nullptr : sRowIn;
  // schedule arrays and the segment table are static for the lifetime of a launch
  // sequence; only predecessor OUTPUTS need griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;");
  tiled_setup<TMEM_COLS>(R, smem, full, empty, aready, aempty, P.a_blocks && P.a_bits == 2, &done, &tmem_base_s, sRowSum, sRowTerm, P.stages,
                         tiled_stage_bytes(P.slot_bn, P.a_bits));
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  R.tmem = tmem_base_s;
  // the predecessor grid's outputs (activations, row sums) are read only after
  // griddepcontrol.wait, issued per role inside the tile (static operands prefetch first)
  R.pdl_wait = true;
  for (int64_t tile = blockIdx.x; tile < P.total_ctas; tile += gridDim.x) {
    tiled_tile<TMEM_COLS, CHAIN>(P, tile, R);
    if (!P.persist) break;
  }
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(R.tmem), "n"(TMEM_COLS));
}


// ------------------------------------------------ 2-SM (CTA pair) variant
// A cluster of 2 CTAs computes a 256-row x bn tile with cta_group::2 MMAs (M = 256):
// each CTA stages its OWN 128-row A block and HALF of the B tile (bn/2 columns), so a
// K tile costs 16 KB + bn*64 B of shared memory / L2 traffic per CTA instead of
// 16 KB + bn*128 B.  The leader (rank 0) issues the MMAs once both CTAs' stages have
// landed (the peer relays its stage completion to the leader with a remote mbarrier
// arrive) and commits to the empty / done barriers of both CTAs (multicast).  Adjacency
// row blocks of a pair generally have different non-zero K lists: the pair walks their
// UNION, and a CTA whose row block has no block at that K tile stages a zero block.
__device__ __align__(1024) uint8_t g_zero_block[16384];

__device__ __forceinline__ uint32_t mapa_cluster(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void tma_2d_pair(void* dst, const void* tmap, int32_t x, int32_t y, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.cta_group::2 [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)), "l"(tmap), "r"(x), "r"(y), "r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// wait on a local mbarrier whose arrivals come from the peer CTA (acquire at cluster scope)
__device__ __forceinline__ void mbar_wait_cluster(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr), "r"(parity) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ void umma_i8_pair(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accum) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(accum));
}

// Union of two ascending K lists: the i-th K tile of the pair, and whether each row
// block has a block there (advancing the cursors).
struct UnionCursor {
  const int32_t* l0;
  const int32_t* l1;
  int n0, n1, i0, i1;
  __device__ __forceinline__ int next(bool& has0, bool& has1) {
    const int k0 = i0 < n0 ? l0[i0] : 0x7fffffff, k1 = i1 < n1 ? l1[i1] : 0x7fffffff;
    const int kt = k0 < k1 ? k0 : k1;
    has0 = k0 == kt;
    has1 = k1 == kt;
    i0 += has0;
    i1 += has1;
    return kt;
  }
};

// Work-item order of the pair kernels within a segment: groups of `gh` row-block pairs
// walked N-tile-major, so the tiles in flight at once share their A row blocks and B
// column tiles in L2 (gh = 1: row-pair-major, the plain order).  A bijection on
// [0, nrbp * n_tiles).
__device__ __forceinline__ void pair_swizzle(int64_t local, int64_t nrbp, int n_tiles, int gh, int64_t& rbp, int& nt) {
  if (gh <= 1) {
    rbp = local / n_tiles;
    nt = (int)(local % n_tiles);
    return;
  }
  const int64_t group = (int64_t)gh * n_tiles, g = local / group, r = local % group;
  const int64_t rows = nrbp - g * gh < gh ? nrbp - g * gh : gh;
  nt = (int)(r / rows);
  rbp = g * gh + r % rows;
}

// CHAIN: the pair also runs the chained dense stage 2 (qg_chain) over its 256 rows.  Each
// CTA's stage-1 epilogue writes its 128 rows of requantized codes into its own ring slots
// (the stage-2 LEFT operand, UMMA K-major), fences them to the async proxy and arrives on
// the leader's mid barrier; each CTA stages HALF of every weight tile (TMA, leader's full
// barrier); the leader then issues the stage-2 cta_group::2 MMAs (M = 256, N = bn2) into
// the same TMEM columns and both CTAs run epilogue 2 on their own rows.
template <int TMEM_COLS, bool CHAIN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTThreads)
    tc_pair_kernel(const __grid_constant__ TiledParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[8], empty[8], done, midbar;
  __shared__ uint32_t tmem_base_s;
  __shared__ unsigned long long sRowSum[CHAIN ? 256 : 128];
  __shared__ double sRowTerm[128];
  __shared__ int64_t sRowIn[128];
  __shared__ int sOff[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int bn = P.bn, S = P.stages, bh = bn >> 1;
  const int64_t pair = (int64_t)(blockIdx.x >> 1);
  if (tid == 0) tstamp(P, (int64_t)blockIdx.x, 0);

  // ---- work item of the pair: (segment, row-block pair, N tile); cta_begin counts PAIRS
  const qg_tseg& G = P.segs[find_seg(P.segs, P.nsegs, pair)];
  const int64_t local = pair - G.cta_begin;
  const int64_t nrb = G.r128 >> 7;
  int64_t rbp;
  int nt;
  pair_swizzle(local, (nrb + 1) >> 1, P.n_tiles, P.pair_swizzle, rbp, nt);
  const int64_t n0 = (int64_t)nt * bn;
  const int64_t rb = rbp * 2 + rank;                     // this CTA's row block (may be past the end)
  const bool rb_ok = rb < nrb;

  // K schedule of the pair (identical in both CTAs)
  UnionCursor U{};
  int nk = 0, kbase_me = 0;
  if (P.a_blocks) {
    const int64_t rb0 = rbp * 2, rb1 = rbp * 2 + 1;
    U.l0 = G.blk_kt + G.blk_base[rb0];
    U.n0 = G.blk_count[rb0];
    U.l1 = rb1 < nrb ? G.blk_kt + G.blk_base[rb1] : nullptr;
    U.n1 = rb1 < nrb ? G.blk_count[rb1] : 0;
    kbase_me = rb_ok ? G.blk_base[rb] : 0;
    UnionCursor c = U;
    bool h0, h1;
    while (c.i0 < c.n0 || c.i1 < c.n1) { c.next(h0, h1); ++nk; }
  } else {
    nk = G.k_tiles;
  }
  asm volatile("griddepcontrol.launch_dependents;");

  const uint32_t a_bytes = 16384u, bh_bytes = (uint32_t)bh * 128u;
  const uint32_t stage_bytes = a_bytes + (uint32_t)(P.slot_bn >> 1) * 128u;
  uint8_t* stage0 = smem;
  const bool fused = P.mode == QG_GEMM_EPILOGUE;
  const qg_epilogue& E = P.epi;
  double* sCol = reinterpret_cast<double*>(smem + (size_t)S * stage_bytes);
  double* sCol2 = sCol + (fused ? col_doubles(bn, epi_row_only(E), E.bn_mean != nullptr) : 0);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 32) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&done, 1);
    mbar_init(&midbar, 2);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 128) sRowSum[tid] = 0ull;
  if (CHAIN && tid < 128) sRowSum[128 + tid] = 0ull;
  if (tid < 2) sOff[tid] = 0;
  // PDL: the setup above and the STATIC operands below (adjacency / left blocks, column
  // constants) overlap the predecessor grid's tail; its OUTPUTS (the B operand, row sums)
  // are read only after griddepcontrol.wait (per role)
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();                                    // barriers of both CTAs initialised
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;
  TileRing R;
  R.stage0 = stage0; R.sCol = sCol; R.full = full; R.empty = empty; R.done = &done;
  R.sRowSum = sRowSum; R.sRowTerm = sRowTerm; R.S = S; R.it0 = 0; R.ndone = 0; R.pdl_wait = false; R.tmem = tmem;
  R.ring_bytes = (uint32_t)S * stage_bytes;
  R.sOff = sOff;
  R.sRowIn = sRowIn;
  const int k2 = CHAIN ? P.k2 : 0;
  if (tid == 0) tstamp(P, (int64_t)blockIdx.x, 1);

  if (warp == 0 && lane == 0) {
    // ---------------- producer (both CTAs): own A block + own half of B ----------------
    // TMA copies (cta_group::2) complete on the LEADER's full[s]; the leader arms it with
    // the bytes of both CTAs (a peer's bytes may land first: the tx count runs ahead)
    const uint32_t leader_full = mapa_cluster(smem_u32(&full[0]), 0);
    const int64_t b_row0 = ((n0 + (int64_t)rank * bh) >> 3) * 8;      // 128-byte rows
    UnionCursor c = U;
    int i_me = 0;
    // the first ring-full: A (static) before the predecessor finishes, B after
    const int pre = nk < S ? nk : S;
    int kts[8];
    for (int it = 0; it < nk; ++it) {
      const int s = it % S;
      if (it >= S) mbar_wait(smem_u32(&empty[s]), ((it / S) - 1) & 1);
      const void* amap;
      int64_t arow;
      int kt;
      if (P.a_blocks) {
        bool h0, h1;
        kt = c.next(h0, h1);
        const bool mine = rank == 0 ? h0 : h1;
        const bool real = rb_ok && mine;
        amap = real ? (const void*)G.tmap_a : (const void*)&P.zero_map;
        arow = real ? (int64_t)(kbase_me + i_me) * 128 : 0;
        i_me += mine;
      } else {
        kt = it;
        amap = rb_ok ? (const void*)G.tmap_a : (const void*)&P.zero_map;
        arow = rb_ok ? (((int64_t)kt * (G.r128 << 7) + rb * 16384) >> 7) : 0;
      }
      uint8_t* dst = stage0 + (size_t)s * stage_bytes;
      if (rank == 0) mbar_expect_tx(&full[s], 2u * (a_bytes + bh_bytes));
      const uint32_t bar = leader_full + (uint32_t)s * 8u;
      tma_2d_pair(dst, amap, 0, (int32_t)arow, bar);
      if (it < pre) {
        kts[it] = kt;
        if (it == pre - 1) {
          asm volatile("griddepcontrol.wait;" ::: "memory");
          for (int j = 0; j < pre; ++j)
            tma_2d_pair(stage0 + (size_t)j * stage_bytes + a_bytes, G.tmap_b, 0,
                        (int32_t)(((int64_t)kts[j] * (P.b_npad << 7) >> 7) + b_row0),
                        leader_full + (uint32_t)j * 8u);
        }
        continue;
      }
      tma_2d_pair(dst + a_bytes, G.tmap_b, 0, (int32_t)(((int64_t)kt * (P.b_npad << 7) >> 7) + b_row0), bar);
    }
    if (CHAIN) {
      // stage 2's weights: this CTA's half of every K tile, into the slots after stage 1's
      const int bh2 = P.bn2 >> 1;
      const uint32_t wh_bytes = (uint32_t)bh2 * 128u;
      for (int j = 0; j < k2; ++j) {
        const int g = nk + j, s = g % S;
        if (g >= S) mbar_wait(smem_u32(&empty[s]), ((g / S) - 1) & 1);
        if (rank == 0) mbar_expect_tx(&full[s], 2u * wh_bytes);
        tma_2d_pair(stage0 + (size_t)s * stage_bytes + a_bytes, &P.w2_map, 0,
                    (int32_t)((int64_t)j * P.w2_npad + (int64_t)rank * bh2), leader_full + (uint32_t)s * 8u);
      }
    }
  } else if (warp == 1 && lane == 0) {
    if (rank == 0) {
      // ---------------- MMA issuer (leader): both CTAs' stages, M = 256 ----------------
      const uint32_t idesc = (2u << 4) | ((uint32_t)(bn >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
      for (int it = 0; it < nk; ++it) {
        const int s = it % S;
        mbar_wait(smem_u32(&full[s]), (it / S) & 1);
        if (it == 0) { tstamp(P, (int64_t)blockIdx.x, 2); tstamp(P, (int64_t)blockIdx.x + 1, 2); }
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a0 = smem_u32(stage0 + (size_t)s * stage_bytes), b0 = a0 + a_bytes;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_i8_pair(tmem, umma_desc(a0 + kk * 256u), umma_desc(b0 + kk * 256u), idesc,
                       (it > 0 || kk > 0) ? 1u : 0u);
        umma_commit_pair(&empty[s]);
      }
      if (nk > 0) umma_commit_pair(&done);
    }
  } else if (warp >= 2 && fused) {
    const int t = tid - 64;
    stage_cols(E, sCol, bn, n0, P.n, t, (int)blockDim.x - 64, &sOff[0]);
    if (CHAIN) stage_cols(P.epi2, sCol2, P.bn2, 0, P.n2, t, (int)blockDim.x - 64, &sOff[1]);
    asm volatile("griddepcontrol.wait;" ::: "memory");   // row sums: predecessor outputs
    if (t < 128) {
      const int64_t row = rb * 128 + t;
      const int64_t rsin = (G.row_sums && rb_ok && row < G.m) ? G.row_sums[row] : 0;
      sRowIn[t] = rsin;
      sRowTerm[t] = (E.use_row && rb_ok && row < G.m) ? __dmul_rn(E.k_row, (double)rsin) : 0.0;
    }
  }
  __syncwarp();
  // every thread is past the predecessor grid before any global write
  asm volatile("griddepcontrol.wait;" ::: "memory");
  uint32_t ndone = 0;
  if (nk > 0) {
    mbar_wait(smem_u32(&done), 0);
    ndone = 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  __syncthreads();
  if (tid == 0) tstamp(P, (int64_t)blockIdx.x, 3);
  if (CHAIN) {
    uint8_t* mid0 = stage0 + (size_t)(nk % S) * stage_bytes;
    uint8_t* mid1 = stage0 + (size_t)((nk + 1) % S) * stage_bytes;
    if (nk == 0 && tid == 0) tstamp(P, (int64_t)blockIdx.x, 2);
    if (rb_ok) tile_epilogue<1>(P, G, R, (int64_t)blockIdx.x, rb, 0, nk, tmem, sCol, true, mid0, mid1);
    // codes (generic proxy) -> visible to the leader's tensor core; TMEM reads retired
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid == 0) mbar_arrive_remote(mapa_cluster(smem_u32(&midbar), 0));
    if (rank == 0 && warp == 1 && lane == 0) {
      // ---- stage-2 MMAs (leader): both CTAs' epilogue 1 drained the accumulator and
      // wrote their codes (mid barrier); the weight halves land on full[]
      mbar_wait_cluster(smem_u32(&midbar), 0);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t idesc2 = (2u << 4) | ((uint32_t)(P.bn2 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
      for (int j = 0; j < k2; ++j) {
        const int g = nk + j, s = g % S;
        mbar_wait(smem_u32(&full[s]), (g / S) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a0 = smem_u32(stage0 + (size_t)s * stage_bytes), b0 = a0 + a_bytes;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_i8_pair(tmem, umma_desc(a0 + kk * 256u), umma_desc(b0 + kk * 256u), idesc2,
                       (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit_pair(&empty[s]);
      }
      umma_commit_pair(&done);
    }
    __syncwarp();
    const qg_epilogue& E2 = P.epi2;
    if (tid < 128) {
      const int64_t row = rb * 128 + tid;
      R.sRowTerm[tid] = (E2.use_row && rb_ok && row < G.m) ? __dmul_rn(E2.k_row, (double)sRowSum[tid]) : 0.0;
    }
    mbar_wait(smem_u32(&done), ndone & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    __syncthreads();                                     // stage-2 row terms visible
    if (tid == 0) tstamp(P, (int64_t)blockIdx.x, 7);
    if (rb_ok) {
      tile_epilogue<2>(P, G, R, (int64_t)blockIdx.x, rb, 0, k2, tmem, sCol2, true);
      if (tid == 0) tstamp(P, (int64_t)blockIdx.x, 4);
      if (E2.out_kind == QG_OUT_PLANES && G.q_row_sums) {
        __syncthreads();
        if (tid < 128 && rb * 128 + tid < G.m && sRowSum[128 + tid])
          atomicAdd(reinterpret_cast<unsigned long long*>(G.q_row_sums + rb * 128 + tid), sRowSum[128 + tid]);
      }
    }
  } else if (rb_ok) {
    if (nk == 0 && tid == 0) tstamp(P, (int64_t)blockIdx.x, 2);
    tile_epilogue<0>(P, G, R, (int64_t)blockIdx.x, rb, n0, nk, tmem, sCol, fused);
    if (tid == 0) tstamp(P, (int64_t)blockIdx.x, 4);
    if (fused && E.out_kind == QG_OUT_PLANES && G.q_row_sums) {
      __syncthreads();
      if (tid < 128 && rb * 128 + tid < G.m && sRowSum[tid])
        atomicAdd(reinterpret_cast<unsigned long long*>(G.q_row_sums + rb * 128 + tid), sRowSum[tid]);
    }
  }
  if (!rb_ok && tid == 0) tstamp(P, (int64_t)blockIdx.x, 4);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();                                    // both CTAs done with TMEM and the ring
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
  if (tid == 0) tstamp(P, (int64_t)blockIdx.x, 5);
}

// ------------------------------------------------ adjacency block preparation
// Gather the non-zero 128x128 blocks of a column-wise packed 1-bit matrix into a
// compact array of packed blocks (128 rows x 4 words = 2 KB each), following the
// schedule (blk_base / blk_kt).  One warp per block.
__global__ void block_gather_kernel(const uint32_t* __restrict__ a, int64_t prows, int64_t pcols,
                                    const int32_t* __restrict__ blk_rb, const int32_t* __restrict__ blk_kt,
                                    int64_t nblocks, uint32_t* __restrict__ packed) {
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= nblocks) return;
  const int64_t rb = blk_rb[b], kt = blk_kt[b], wpr = pcols >> 5;
  for (int r = lane; r < 128; r += 32) {
    const int64_t row = rb * 128 + r;
    uint4 q = make_uint4(0, 0, 0, 0);
    if (row < prows) q = __ldg(reinterpret_cast<const uint4*>(a + row * wpr + kt * 4));
    reinterpret_cast<uint4*>(packed)[b * 128 + r] = q;
  }
}

// Expand packed blocks to UMMA-layout byte blocks (16 KB each) and accumulate the
// row degrees (popcount) -- graph.py:292-295.  Block = 256 threads per packed block:
// thread -> (row r = t & 127, K-core pair), 4 K-cores of 16 bytes each.
__global__ void __launch_bounds__(256) block_expand_kernel(const uint32_t* __restrict__ packed, int64_t nblocks,
                                                           const int32_t* __restrict__ blk_rb,
                                                           uint8_t* __restrict__ bytes, int64_t* __restrict__ degrees,
                                                           int64_t rows) {
  const int64_t b = blockIdx.x;
  if (b >= nblocks) return;
  const int t = threadIdx.x, r = t & 127, h = t >> 7;
  const uint4 w4 = __ldg(reinterpret_cast<const uint4*>(packed) + b * 128 + r);
  const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
  if (bytes) {                                // NULL: degrees only (blocks expanded in the GEMM)
    uint8_t* blk = bytes + b * 16384;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = h + 2 * i;                 // K-core: bits 16c..16c+15 = word c>>1, half c&1
      const uint32_t x = w[c >> 1] >> ((c & 1) * 16);
      const uint4 o = make_uint4(expand_nibble(x & 0xFu), expand_nibble((x >> 4) & 0xFu),
                                 expand_nibble((x >> 8) & 0xFu), expand_nibble((x >> 12) & 0xFu));
      *reinterpret_cast<uint4*>(blk + umma_off(r, c)) = o;
    }
  }
  if (degrees && h == 0) {
    const int64_t row = (int64_t)blk_rb[b] * 128 + r;
    const int d = __popc(w4.x) + __popc(w4.y) + __popc(w4.z) + __popc(w4.w);
    if (row < rows && d) atomicAdd(reinterpret_cast<unsigned long long*>(degrees + row), (unsigned long long)d);
  }
}

// Grouped variant over many batches (one launch per epoch on the e2e path): block ->
// segment by binary search on block_begin, then the same expansion + degrees.
__global__ void __launch_bounds__(256) block_expand_grouped_kernel(const qg_block_seg* __restrict__ segs, int nsegs,
                                                                   int64_t total_blocks) {
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t gb = blockIdx.x;
  if (gb >= total_blocks) return;
  const qg_block_seg& S = segs[find_seg_by(segs, nsegs, gb, [](const qg_block_seg& g) { return g.block_begin; })];
  const int64_t b = gb - S.block_begin;
  const int t = threadIdx.x, r = t & 127, h = t >> 7;
  const uint4 w4 = __ldg(reinterpret_cast<const uint4*>(S.packed) + b * 128 + r);
  const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
  if (S.bytes) {
    uint8_t* blk = S.bytes + b * 16384;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = h + 2 * i;
      const uint32_t x = w[c >> 1] >> ((c & 1) * 16);
      *reinterpret_cast<uint4*>(blk + umma_off(r, c)) =
          make_uint4(expand_nibble(x & 0xFu), expand_nibble((x >> 4) & 0xFu), expand_nibble((x >> 8) & 0xFu),
                     expand_nibble((x >> 12) & 0xFu));
    }
  }
  if (S.degrees && h == 0) {
    const int64_t row = (int64_t)S.blk_rb[b] * 128 + r;
    const int d = __popc(w4.x) + __popc(w4.y) + __popc(w4.z) + __popc(w4.w);
    if (row < S.rows && d) atomicAdd(reinterpret_cast<unsigned long long*>(S.degrees + row), (unsigned long long)d);
  }
}

// Plain code matrix (row-major [rows][ld]) -> left- or right-tiled layout.
__global__ void codes_to_tiles_kernel(const uint8_t* __restrict__ codes, int64_t rows, int64_t cols, int64_t ld,
                                      int right, int64_t pitch, uint8_t* __restrict__ tiles) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * cols) return;
  const int64_t r = i / cols, c = i % cols;
  // left: rows = M, cols = K (pitch = r128); right: rows = K, cols = N (pitch = npad)
  const int64_t off = right ? right_tile_off(r, c, pitch) : left_tile_off(r, c, pitch);
  tiles[off] = codes[r * ld + c];
}

// Tiled codes -> plain row-major codes (materialising plane views of code caches).
__global__ void tiles_to_codes_kernel(const uint8_t* __restrict__ tiles, int64_t rows, int64_t cols, int right,
                                      int64_t pitch, uint8_t* __restrict__ codes, int64_t ld) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * cols) return;
  const int64_t r = i / cols, c = i % cols;
  const int64_t off = right ? right_tile_off(r, c, pitch) : left_tile_off(r, c, pitch);
  codes[r * ld + c] = tiles[off];
}

// Grouped entry conversion: row-wise feature planes of all batches -> tiled u8 codes.  Unit =
// 256 rows (8 plane words per column) x 128 columns; thread t (128 per CTA) owns column c0 + t and
// reads, per plane, its 8 consecutive row words with two 16-byte loads (one 32-B sector),
// then expands them into 256 code bytes (bit i of plane p -> bit p of byte i).
// Right-tiled (K = rows): every 32 rows of column c are two 16-byte K-cores -> direct
// vector stores.  Left-tiled (K = columns): transpose through shared memory, then every
// thread stores 16-byte K-cores of rows; row code sums reduce over the unit's 128 columns
// before one atomic per row.
template <int kEntryWords>                              // row words (x 32 rows) per unit: 8 or 1
__global__ void __launch_bounds__(128, 5) entry_tiles_kernel(const qg_entry_seg* __restrict__ segs, int nsegs,
                                                          int nplanes, int right) {
  // the first GEMM (PDL-launched) may start its prologue + static-operand prefetch now;
  // it reads this kernel's output only after griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;");
  __shared__ __align__(16) uint8_t tile[32 * kEntryWords][128 + 16];
  const qg_entry_seg& G =
      segs[find_seg_by(segs, nsegs, (int64_t)blockIdx.x, [](const qg_entry_seg& g) { return g.unit_begin; })];
  // PDL-launched: everything above read only the (static) segment table; the planes and
  // the zeroed row sums come from the stream predecessor
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t u = (int64_t)blockIdx.x - G.unit_begin;
  const int64_t wpl = G.pr >> 5;                          // words per column of one plane
  const int64_t ncg = right ? (G.pitch + 127) >> 7 : (G.pc + 127) >> 7;
  const int64_t vb = (u / ncg) * kEntryWords, cg = u % ncg;   // first row word, 128-column group
  const int t = threadIdx.x;
  const int64_t wpp = wpl * G.pc;
  const int64_t c = cg * 128 + (t & 127);
  const int nw = (int)(wpl - vb < kEntryWords ? wpl - vb : kEntryWords);   // valid row words
  uint32_t w[8][kEntryWords];                              // [plane][row word]
#pragma unroll
  for (int p = 0; p < 8; ++p)
#pragma unroll
    for (int j = 0; j < kEntryWords; ++j) w[p][j] = 0u;
  if (t < 128 && c < G.pc) {
    const uint32_t* col = G.words + c * wpl + vb;          // 16-byte aligned: wpl % 4 == 0, vb % 8 == 0
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      if (p < nplanes) {
        const uint32_t* src = col + p * wpp;
        if (kEntryWords == 8 && nw == 8) {
          const uint4 a = __ldg(reinterpret_cast<const uint4*>(src));
          const uint4 b = __ldg(reinterpret_cast<const uint4*>(src) + 1);
          w[p][0] = a.x; w[p][1] = a.y; w[p][2] = a.z; w[p][3] = a.w;
          w[p][4 % kEntryWords] = b.x; w[p][5 % kEntryWords] = b.y; w[p][6 % kEntryWords] = b.z;
          w[p][7 % kEntryWords] = b.w;
        } else {
#pragma unroll
          for (int j = 0; j < kEntryWords; ++j) w[p][j] = j < nw ? __ldg(src + j) : 0u;
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kEntryWords; ++j) {
    // 32 code bytes (rows 32(vb + j) ..): for each 8-row group g gather byte g of the 8
    // plane words (byte p = plane p, PRMT) and transpose the 8x8 bit matrix -- byte i of the
    // result holds bit p of row 8g + i for every plane p, i.e. the code of row 8g + i
    uint32_t o[8];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint32_t sel = (uint32_t)g | ((uint32_t)(g + 4) << 4);      // [a.byte g, b.byte g]
      const uint32_t p01 = __byte_perm(w[0][j], w[1][j], sel), p23 = __byte_perm(w[2][j], w[3][j], sel);
      const uint32_t p45 = __byte_perm(w[4][j], w[5][j], sel), p67 = __byte_perm(w[6][j], w[7][j], sel);
      const uint64_t x = ((uint64_t)__byte_perm(p45, p67, 0x5410) << 32) | __byte_perm(p01, p23, 0x5410);
      const uint64_t tt = transpose8x8(x);
      o[2 * g] = (uint32_t)tt;
      o[2 * g + 1] = (uint32_t)(tt >> 32);
    }
    if (right) {
      if (t < 128 && c < G.pitch && j < nw) {
        const int64_t k0 = (vb + j) * 32;
        *reinterpret_cast<uint4*>(G.tiles + right_tile_off(k0, c, G.pitch)) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4*>(G.tiles + right_tile_off(k0 + 16, c, G.pitch)) =
            make_uint4(o[4], o[5], o[6], o[7]);
      }
    } else if (t < 128) {
#pragma unroll
      for (int i = 0; i < 32; ++i) tile[32 * j + i][t] = (uint8_t)(o[i >> 2] >> (8 * (i & 3)));
    }
  }
  if (right) return;
  __syncthreads();
  // 256 rows x 8 K-cores = 2048 16-byte stores, 16 per thread; the 8 cores of a row are 8
  // consecutive lanes (row sums reduce over them)
  for (int idx = t; idx < 32 * kEntryWords * 8; idx += 128) {
    const int r = idx >> 3, core = idx & 7;
    const int64_t row = vb * 32 + r, k = cg * 128 + core * 16;
    const uint4 q = *reinterpret_cast<const uint4*>(&tile[r][core * 16]);
    if (row < G.pitch) *reinterpret_cast<uint4*>(G.tiles + left_tile_off(row, k, G.pitch)) = q;
    if (G.row_sums) {
      const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
      uint32_t sum = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) sum = __dp4a(w4[i], 0x01010101u, sum);
#pragma unroll
      for (int off = 4; off > 0; off >>= 1) sum += __shfl_xor_sync(QG_FULL, sum, off);
      if (core == 0 && row < G.rows && sum)
        atomicAdd(reinterpret_cast<unsigned long long*>(G.row_sums + row), (unsigned long long)sum);
    }
  }
}

}  // namespace qg

using namespace qg;

extern "C" int qg_entry_tiles(const qg_entry_seg* segs, int32_t nsegs, int32_t nplanes, int32_t right,
                              int32_t words_per_unit, int64_t total_units, void* stream) {
  if (!segs || nsegs < 1 || nplanes < 1 || nplanes > 8 || total_units < 0 ||
      (words_per_unit != 1 && words_per_unit != 8))
    return QG_ERR_ARG;
  if (total_units == 0) return QG_OK;
  // programmatic dependent launch: the launch overlaps the predecessor's tail (the slab
  // reset of a captured epoch); the kernel waits before reading any predecessor output
  static const bool pdl = getenv("QG_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)total_units);
  cfg.blockDim = dim3(128);          // one thread per column of the unit; 5 CTAs per SM
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (words_per_unit == 8) cudaLaunchKernelEx(&cfg, entry_tiles_kernel<8>, segs, (int)nsegs, (int)nplanes, (int)right);
  else cudaLaunchKernelEx(&cfg, entry_tiles_kernel<1>, segs, (int)nsegs, (int)nplanes, (int)right);
  return cudaGetLastError() == cudaSuccess ? QG_OK : QG_ERR_CUDA;
}

static inline int tstatus() { return cudaGetLastError() == cudaSuccess ? QG_OK : QG_ERR_CUDA; }

template <int COLS, int MINB, int NT, bool CHAIN>
static void tiled_attr(size_t bytes) {
  static size_t done = 0;
  if (bytes > done) {
    cudaFuncSetAttribute(tc_tiled_kernel<COLS, MINB, NT, CHAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    cudaFuncSetAttribute(tc_tiled_kernel<COLS, MINB, NT, CHAIN>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    done = bytes;
  }
}

// Programmatic dependent launch: the grid may start while its stream predecessor is
// still running; the kernel's griddepcontrol.wait (after its prologue) orders every
// read of predecessor outputs, so launch latency + TMEM/barrier setup overlap the
// previous layer's tail.  Captured into CUDA graphs as programmatic edges.
template <int COLS, int MINB, int NT = kTThreads, bool CHAIN = false>
static void launch_tiled(const TiledParams& P, unsigned grid, size_t smem, cudaStream_t st) {
  tiled_attr<COLS, MINB, NT, CHAIN>(smem);
  if (P.persist) {
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const unsigned resident = (unsigned)(sms * MINB);
    if (grid > resident) grid = resident;
  }
  static const bool pdl = getenv("QG_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, tc_tiled_kernel<COLS, MINB, NT, CHAIN>, P);
}

// qg_tiled_args -> kernel parameters; returns the per-column constant bytes the
// epilogue stages in shared memory (0 on an argument error, see *rc).
static size_t tiled_params(const qg_tiled_args* a, TiledParams& P, int& rc) {
  rc = QG_OK;
  if (!a || !a->segs || a->nsegs < 1 || a->total_ctas < 1) { rc = QG_ERR_ARG; return 0; }
  if (a->bn < 16 || a->bn > 256 || (a->bn & (a->bn - 1))) { rc = QG_ERR_ARG; return 0; }
  if (a->mode != QG_GEMM_I32 && a->mode != QG_GEMM_EPILOGUE) { rc = QG_ERR_ARG; return 0; }
  if (a->mode == QG_GEMM_EPILOGUE && !a->epi) { rc = QG_ERR_ARG; return 0; }
  // batch norm needs all five vectors (bn_inv_denom = RN(1 / bn_denom) drives the division)
  if (a->epi && a->epi->bn_mean && !(a->epi->bn_denom && a->epi->bn_gamma && a->epi->bn_beta && a->epi->bn_inv_denom))
    { rc = QG_ERR_ARG; return 0; }
  if (a->b_npad % 8 || a->b_npad < (int64_t)a->n_tiles * a->bn) { rc = QG_ERR_SHAPE; return 0; }
  // reserved fields (round-1 opt-in variants, removed) must be zero
  if ((a->a_bits && (!a->a_blocks || a->pair)) || a->a_bits < 0 || a->a_bits > 2 ||
      (a->a_bits == 2 && (a->chain || a->bn > 128)) || a->reserved1 || a->reserved2 || a->reserved3 ||
      (a->epi && a->epi->reserved_d1 != 0.0))
    { rc = QG_ERR_UNSUPPORTED; return 0; }
  P = TiledParams{};
  P.segs = a->segs; P.nsegs = a->nsegs; P.a_blocks = a->a_blocks; P.b_npad = a->b_npad; P.n = a->n;
  P.bn = a->bn; P.n_tiles = a->n_tiles; P.mode = a->mode; P.out_layout = a->out_layout; P.out_npad = a->out_npad;
  P.log2bn = 5;
  while ((1 << P.log2bn) < P.bn) ++P.log2bn;
  if (a->epi) P.epi = *a->epi;
  P.phase_ns = a->phase_ns;
  P.total_ctas = a->total_ctas;
  P.pair = a->pair;
  P.a_bits = a->a_blocks ? a->a_bits : 0;
  P.slot_bn = P.bn;
  // per-column constants: fp64 terms + the fp32 screen's acc0_c / delta_c (col_doubles)
  const qg_epilogue* e1 = a->epi;
  size_t cols = e1 ? (size_t)col_doubles(P.bn, !e1->use_col && !e1->use_const && !e1->bias, e1->bn_mean != nullptr) * 8
                   : 0;
  static const bool screen = getenv("QG_NO_SCREEN") == nullptr;
  P.screen = screen ? 1 : 0;
  static const int dbg = getenv("QG_EPI_DBG") ? atoi(getenv("QG_EPI_DBG")) : 0;
  P.dbg = dbg;
  static const bool persist = getenv("QG_PERSIST") != nullptr && atoi(getenv("QG_PERSIST")) != 0;
  P.persist = persist ? 1 : 0;
  if (a->chain) {
    const qg_chain* c = a->chain;
    // stage 1: one N tile covering all its columns, packed codes
    if (a->mode != QG_GEMM_EPILOGUE || a->n_tiles != 1 || a->n > a->bn || c->reserved ||
        a->epi->out_kind != QG_OUT_PLANES)
      { rc = QG_ERR_UNSUPPORTED; return 0; }
    if (!c->w || !c->epi || c->w_npad < 32 || c->w_npad > 256 || (c->w_npad & (c->w_npad - 1)) || c->n < 1 ||
        c->n > c->w_npad || (c->out_layout != 0 && c->out_layout != 2) ||
        (c->out_layout == 0) != (c->epi->out_kind == QG_OUT_REAL) ||
        (c->epi->bn_mean && !(c->epi->bn_denom && c->epi->bn_gamma && c->epi->bn_beta && c->epi->bn_inv_denom)))
      { rc = QG_ERR_ARG; return 0; }
    P.chain = 1;
    P.bn2 = (int32_t)c->w_npad;
    P.k2 = (int32_t)((a->n + 127) / 128);
    P.n2 = c->n;
    P.out_layout2 = c->out_layout;
    P.out_npad2 = c->out_npad;
    P.w2 = c->w;
    P.w2_npad = c->w_npad;
    P.epi2 = *c->epi;
    P.slot_bn = std::max(P.bn, P.bn2);
    if (c->epi->reserved_d1 != 0.0) { rc = QG_ERR_UNSUPPORTED; return 0; }
    const qg_epilogue* e2 = c->epi;
    cols += (size_t)col_doubles(P.bn2, !e2->use_col && !e2->use_const && !e2->bias, e2->bn_mean != nullptr) * 8;
  }
  return cols;
}

// the kernel is epilogue-heavy: size the ring so TWO CTAs fit per SM (one CTA's fp64
// epilogue overlaps the other's bulk-copy/MMA main loop); TMEM 2 x 256 cols fits
static size_t smem_budget() {
  size_t budget = 113 * 1024 - 4096;
  static const char* env_budget = getenv("QG_TILED_SMEM_KB");   // tuning experiments only
  if (env_budget) budget = (size_t)atoi(env_budget) * 1024;
  return budget;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

extern "C" int qg_encode_linear_map(const void* base, int64_t bytes, int32_t box_rows, void* out) {
  if (!base || !out || bytes <= 0 || (bytes & 127) || box_rows < 1 || box_rows > 256 ||
      (reinterpret_cast<uintptr_t>(base) & 15))
    return QG_ERR_ARG;
  EncodeTiledFn fn = encode_fn();
  if (!fn) return QG_ERR_UNSUPPORTED;
  const cuuint64_t dims[2] = {128, (cuuint64_t)(bytes >> 7)};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base),
                        dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? QG_OK : QG_ERR_ARG;
}

template <int COLS, bool CHAIN>
static void launch_pair(const TiledParams& P, unsigned grid, size_t smem, cudaStream_t st) {
  static size_t attr_done = 0;
  if (smem > attr_done) {
    cudaFuncSetAttribute(tc_pair_kernel<COLS, CHAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(tc_pair_kernel<COLS, CHAIN>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    attr_done = smem;
  }
  static const bool pdl = getenv("QG_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, tc_pair_kernel<COLS, CHAIN>, P);
}

extern "C" int qg_tiled_gemm(const qg_tiled_args* a, void* stream) {
  TiledParams P;
  int rc;
  const size_t cols = tiled_params(a, P, rc);
  if (rc != QG_OK) return rc;
  if (P.pair) {
    // total_ctas = 2 x pairs; a stage holds the own A block + half of the B tile
    if ((a->total_ctas & 1) || P.bn < 64 || (P.chain && P.bn2 < 32)) return QG_ERR_UNSUPPORTED;
    void* zero = nullptr;
    cudaGetSymbolAddress(&zero, g_zero_block);
    if (qg_encode_linear_map(zero, 16384, 128, &P.zero_map) != QG_OK) return QG_ERR_UNSUPPORTED;
    if (P.chain &&
        qg_encode_linear_map(P.w2, (int64_t)P.k2 * P.w2_npad * 128, P.bn2 >> 1, &P.w2_map) != QG_OK)
      return QG_ERR_UNSUPPORTED;
    // 8 row-block pairs per N-major group: the ~148 pairs in flight then share A row
    // blocks and B column tiles in L2 (C5 16k: 73% -> 79% of the int8 peak)
    static const int swz = getenv("QG_PAIR_SWIZZLE") ? atoi(getenv("QG_PAIR_SWIZZLE")) : 8;
    P.pair_swizzle = swz < 1 ? 1 : swz;
    const size_t stage = 16384 + (size_t)P.slot_bn * 64;
    cudaStream_t st = (cudaStream_t)stream;
    P.stages = (int32_t)std::max<size_t>(P.chain ? 3 : 2, std::min<size_t>(8, (smem_budget() - cols) / stage));
    const size_t smem = (size_t)P.stages * stage + cols;
    const unsigned grid = (unsigned)a->total_ctas;
    const int tcols = std::max(32, (int)P.slot_bn);
    if (P.chain) {
      switch (tcols) {
        case 64: launch_pair<64, true>(P, grid, smem, st); break;
        case 128: launch_pair<128, true>(P, grid, smem, st); break;
        default: launch_pair<256, true>(P, grid, smem, st); break;
      }
    } else {
      switch (tcols) {
        case 64: launch_pair<64, false>(P, grid, smem, st); break;
        case 128: launch_pair<128, false>(P, grid, smem, st); break;
        default: launch_pair<256, false>(P, grid, smem, st); break;
      }
    }
    return tstatus();
  }
  const size_t stage = tiled_stage_bytes(P.slot_bn, P.a_bits);
  // Occupancy: 2 CTAs/SM by default (one CTA's fp64 epilogue overlaps the other's main
  // loop).  Stages with N tiles <= 128 and >= 3 CTAs per SM of work run 3 CTAs/SM
  // (80-register variant, 72 KB ring, 3 x <= 128 TMEM columns): more warps hide the
  // epilogue's latency (C3: 0.29 -> 0.25 ms/epoch).
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  static const bool env_budget = getenv("QG_TILED_SMEM_KB") != nullptr;
  // TMEM columns: the widest accumulator (stage 1 or the chained stage 2)
  const int tcols = std::max(32, (int)P.slot_bn);     // TMEM allocations are >= 32 columns
  const bool three = !env_budget && !P.chain && tcols <= 128 && a->total_ctas >= 3 * (int64_t)sms &&
                     (P.a_bits != 2 || P.bn <= 64);
  static const bool wide = getenv("QG_WIDE") != nullptr && atoi(getenv("QG_WIDE")) != 0;
  const size_t budget = three ? 72 * 1024 : smem_budget();
  P.stages = (int32_t)std::max<size_t>(2, std::min<size_t>(8, (budget - cols) / stage));
  const size_t smem = (size_t)P.stages * stage + cols;
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned grid = (unsigned)a->total_ctas;
  if (P.a_bits == 2) {
    // A in tensor memory: the accumulator at columns [0, bn), the A ring of 32-column slots
    // after it -- 3 CTAs/SM: 128 columns (bn <= 64, 2 slots); else 256 columns (4 slots)
    if (three) {
      P.a_col0 = 64; P.a_slots = 2;
      launch_tiled<128, 3>(P, grid, smem, st);
    } else {
      P.a_col0 = 128; P.a_slots = 4;
      launch_tiled<256, 2>(P, grid, smem, st);
    }
    return tstatus();
  }
  if (P.chain) {
    // chained aggregate -> update: one tile per CTA.  A chained stage has half the CTAs of
    // the split-N stages it replaces and two epilogues per tile: with fewer tiles than
    // SMs, 16 warps (1 CTA/SM) split the epilogue slices 4 ways
    static const bool force16 = getenv("QG_CHAIN_16W") != nullptr && atoi(getenv("QG_CHAIN_16W")) != 0;
    const bool wide16 = a->total_ctas <= (int64_t)sms || force16;
    static const bool chain_wide = getenv("QG_CHAIN_WIDE") != nullptr && atoi(getenv("QG_CHAIN_WIDE")) != 0;
    if (!wide16 && chain_wide && tcols == 256) {
      // 12 warps: 3 warp groups split the two epilogues' slices (opt-in, measured)
      launch_tiled<256, 2, 384, true>(P, grid, smem, st);
    } else if (wide16) {
      switch (tcols) {
        case 32: launch_tiled<32, 1, 512, true>(P, grid, smem, st); break;
        case 64: launch_tiled<64, 1, 512, true>(P, grid, smem, st); break;
        case 128: launch_tiled<128, 1, 512, true>(P, grid, smem, st); break;
        default: launch_tiled<256, 1, 512, true>(P, grid, smem, st); break;
      }
    } else {
      switch (tcols) {
        case 32: launch_tiled<32, 2, kTThreads, true>(P, grid, smem, st); break;
        case 64: launch_tiled<64, 2, kTThreads, true>(P, grid, smem, st); break;
        case 128: launch_tiled<128, 2, kTThreads, true>(P, grid, smem, st); break;
        default: launch_tiled<256, 2, kTThreads, true>(P, grid, smem, st); break;
      }
    }
  } else if (three) {
    switch (tcols) {
      case 32: launch_tiled<32, 3>(P, grid, smem, st); break;
      case 64: launch_tiled<64, 3>(P, grid, smem, st); break;
      default: launch_tiled<128, 3>(P, grid, smem, st); break;
    }
  } else {
    switch (tcols) {
      case 32: launch_tiled<32, 2>(P, grid, smem, st); break;
      case 64: launch_tiled<64, 2>(P, grid, smem, st); break;
      case 128: launch_tiled<128, 2>(P, grid, smem, st); break;
      default:
        // QG_WIDE=1: 12 warps (80 registers) for the epilogue-bound dense-left (update) GEMMs.
        // It paid off for the fp64 epilogue (C4 -3.5%); with the lean screened epilogue the
        // 8-warp, 128-register variant is faster (C4 first update 1.06 -> 0.96 ms, r04h)
        if (wide && !P.a_blocks && !P.chain && P.mode == QG_GEMM_EPILOGUE) launch_tiled<256, 2, 384>(P, grid, smem, st);
        else launch_tiled<256, 2>(P, grid, smem, st);
        break;
    }
  }
  return tstatus();
}

extern "C" int qg_block_prepare(const uint32_t* a_words, int64_t rows, int64_t padded_rows, int64_t padded_cols,
                                const int32_t* blk_rb, const int32_t* blk_kt, int64_t nblocks, uint32_t* packed,
                                uint8_t* bytes, int64_t* degrees, void* stream) {
  if (nblocks < 0 || (nblocks && (!blk_rb || !packed))) return QG_ERR_ARG;
  if (nblocks == 0) return QG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (a_words)   // gather from the dense packed matrix; otherwise `packed` is already filled
    block_gather_kernel<<<(unsigned)((nblocks * 32 + 255) / 256), 256, 0, st>>>(a_words, padded_rows, padded_cols,
                                                                                blk_rb, blk_kt, nblocks, packed);
  block_expand_kernel<<<(unsigned)nblocks, 256, 0, st>>>(packed, nblocks, blk_rb, bytes, degrees, rows);
  return tstatus();
}

extern "C" int qg_block_prepare_grouped(const qg_block_seg* segs, int32_t nsegs, int64_t total_blocks,
                                        void* stream) {
  if (!segs || nsegs < 1 || total_blocks < 0) return QG_ERR_ARG;
  if (total_blocks == 0) return QG_OK;
  block_expand_grouped_kernel<<<(unsigned)total_blocks, 256, 0, (cudaStream_t)stream>>>(segs, nsegs, total_blocks);
  return tstatus();
}

extern "C" int qg_codes_to_tiles(const uint8_t* codes, int64_t rows, int64_t cols, int64_t ld, int right,
                                 int64_t pitch, uint8_t* tiles, void* stream) {
  if (!codes || !tiles || rows < 0 || cols < 0 || ld < cols) return QG_ERR_ARG;
  const int64_t n = rows * cols;
  if (n == 0) return QG_OK;
  codes_to_tiles_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(codes, rows, cols, ld, right,
                                                                                      pitch, tiles);
  return tstatus();
}

extern "C" int qg_tiles_to_codes(const uint8_t* tiles, int64_t rows, int64_t cols, int right, int64_t pitch,
                                 uint8_t* codes, int64_t ld, void* stream) {
  if (!codes || !tiles || rows < 0 || cols < 0 || ld < cols) return QG_ERR_ARG;
  const int64_t n = rows * cols;
  if (n == 0) return QG_OK;
  tiles_to_codes_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(tiles, rows, cols, right, pitch,
                                                                                      codes, ld);
  return tstatus();
}
