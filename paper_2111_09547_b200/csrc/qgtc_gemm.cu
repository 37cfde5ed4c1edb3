// Any-bitwidth bit-GEMM for sm_100a.
//
// TCGEN05 path (default): per CTA one 128-row block of L times one N tile of
// R.  For every non-zero 128-bit K tile of the row block (zero-tile jumping
// schedule from qg_tile_scan) the 4 warps load the packed plane words of L
// (rows) and R (columns), recompose the planes into u8 codes in registers
// (code byte = sum_p 2^p bit_p -- the shift-add of the plane partial sums
// moved in front of the MMA, exact by linearity) and store them in the UMMA
// K-major canonical layout; one thread issues 4x tcgen05.mma.kind::i8
// (M=128, N=BN, K=32) into a TMEM s32 accumulator.  Two smem stages: the
// expansion of tile i+1 overlaps the MMAs of tile i (mbarrier via
// tcgen05.commit).  Epilogue: tcgen05.ld 32x32b -> registers -> shared fp64
// epilogue device function -> requantized planes (+ row sums) or fp64 / int32.
//
// PER_PLANE variant (bmm_1bit_by_nbit API, cross-bit reuse ablation): R plane
// p is expanded to 0/1 bytes, giving A . X_p exactly (<= K, no overflow).
//
// POPC path: CUDA-core AND+popcount over packed words with exact int64
// accumulation and int32 overflow detection (the reference's semantics for
// shapes where the s32 tensor accumulator could wrap).
#include <algorithm>
#include "qgtc_common.cuh"

namespace qg {

struct GemmParams {
  const uint32_t* lhs;
  const uint32_t* rhs;
  int64_t m, m_padded, n, n_padded;
  int64_t lwpr, lwpp, rwpr, rwpp;  // words per row/col and per plane
  int32_t lbits, rbits;
  int32_t k_tiles;                 // k_padded / 128
  int32_t bn;                      // N tile (multiple of 32, <= 256)
  int32_t n_tiles;
  int32_t mode;
  int64_t vstride;                 // PER_PLANE: virtual column stride of one R plane
  int64_t n_ext;                   // computed (virtual) column extent, <= n_tiles*bn
  int32_t raw_stages;              // cp.async ring depth for the packed plane words (2..4)
  int32_t log2bn;                  // bn is a power of two (32..256)
  const uint8_t* lhs_codes; int64_t lhs_ld;   // optional u8 code operands (K-major, UMMA-ready)
  const uint8_t* rhs_codes; int64_t rhs_ld;
  int32_t pf_dist;                 // cp.async prefetch distance (raw_stages - 2, >= 1)
  const int32_t* blk_list;
  const int32_t* blk_count;
  int32_t* out_i32;
  int32_t* overflow;
  int64_t* phase_ns;
  qg_epilogue epi;
};

constexpr int kStampStride = 6 + 4 * 16;   // 6 phase stamps + 4 per main-loop iteration (first 16)
__device__ __forceinline__ void phase_stamp(const GemmParams& P, int k) {
  if (P.phase_ns && threadIdx.x == 0) {
    uint64_t t;
    if (k == 0 || k == 5) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));   // ns, comparable across SMs
    else t = (uint64_t)clock64();                                             // SM cycles, fine-grained
    P.phase_ns[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * kStampStride + k] = (int64_t)t;
  }
}

// Expand one unit = (operand row, K-core c): 16 code bytes from `nb` plane
// words (raw[p*stride + row*4 + (c>>1)]).  Codes: sum_p bit_p << p; ZERO_ONE:
// a single plane's 0/1 bytes.
template <bool ZERO_ONE>
__device__ __forceinline__ void expand_unit(const uint32_t* raw, int pstride, int row, int c, int nb, uint32_t dst) {
  const int sh0 = (c & 1) * 16;
  const uint32_t* src = raw + row * 4 + (c >> 1);
  uint32_t o0 = 0, o1 = 0, o2 = 0, o3 = 0;
#pragma unroll 1
  for (int p = 0; p < nb; ++p) {
    const uint32_t w = src[p * pstride] >> sh0;
    const int sh = ZERO_ONE ? 0 : p;
    o0 |= expand_nibble(w & 0xFu) << sh;
    o1 |= expand_nibble((w >> 4) & 0xFu) << sh;
    o2 |= expand_nibble((w >> 8) & 0xFu) << sh;
    o3 |= expand_nibble((w >> 12) & 0xFu) << sh;
  }
  sts128(dst, o0, o1, o2, o3);
}


template <bool PER_PLANE, int TMEM_COLS>
__global__ void __launch_bounds__(kThreads) tc_bitgemm_kernel(const __grid_constant__ GemmParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar_x[2];     // expanded-stage reuse (MMA of it-2 done)
  __shared__ __align__(8) uint64_t mbar_r[4];     // raw-stage reuse (MMA of it-NR done)
  __shared__ uint32_t tmem_base_s;
  phase_stamp(P, 0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int bn = P.bn;
  const int64_t rb = blockIdx.x;
  const int nt = (int)blockIdx.y;
  const int lb = P.lbits;
  const int rbits = PER_PLANE ? 1 : P.rbits;
  const bool a_codes = P.lhs_codes != nullptr, b_codes = P.rhs_codes != nullptr;
  const bool expand = !a_codes || !b_codes;
  const int NR = P.raw_stages, PD = P.pf_dist;
  // dynamic smem: [sA 2x16K if A expanded][sB 2x bn*128 if B expanded][rawA NR][rawB NR][sCol 7*bn*8]
  const uint32_t base = smem_u32(smem);
  uint32_t off = 0;
  const uint32_t sA0 = base + off;  if (!a_codes) off += 2 * 16384u;
  const uint32_t bstage = (uint32_t)bn * 128u;
  const uint32_t sB0 = base + off;  if (!b_codes) off += 2 * bstage;
  const uint32_t rawA_bytes = a_codes ? 16384u : (uint32_t)lb * 2048u;
  const uint32_t rawB_bytes = b_codes ? bstage : (uint32_t)rbits * bn * 16u;
  uint8_t* rawA = smem + off;  off += NR * rawA_bytes;
  uint8_t* rawB = smem + off;  off += NR * rawB_bytes;
  // [7][bn] per-column epilogue constants, beyond the 32 KB epilogue scratch at the base
  double* sCol = reinterpret_cast<double*>(smem + (off > 32768u ? off : 32768u));

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar_x[i])));
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar_r[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }

  const int nk = P.blk_count ? P.blk_count[rb] : P.k_tiles;
  const int32_t* klist = P.blk_list ? P.blk_list + rb * (int64_t)P.k_tiles : nullptr;

  // cp.async of K tile `kt` into raw stage `rs`
  auto issue = [&](int kt, int rs) {
    uint8_t* ra = rawA + rs * rawA_bytes;
    uint8_t* rbp = rawB + rs * rawB_bytes;
    if (a_codes) {
      // 128 rows x 8 16-byte K-cores, straight into the UMMA layout (8 lanes = one 128 B row)
      for (int u = tid; u < 1024; u += kThreads) {
        const int c = u & 7, r = u >> 3;
        const int64_t row = rb * 128 + r;
        const bool ok = row < P.m;
        cp_async16(smem_u32(ra) + umma_off(r, c), P.lhs_codes + (ok ? row : 0) * P.lhs_ld + kt * 128 + c * 16, ok);
      }
    } else {
      for (int u = tid; u < lb * 128; u += kThreads) {
        const int p = u >> 7, r = u & 127;
        const int64_t row = rb * 128 + r;
        const bool ok = row < P.m_padded;
        cp_async16(smem_u32(ra) + (p * 128 + r) * 16, P.lhs + p * P.lwpp + (ok ? row : 0) * P.lwpr + kt * 4, ok);
      }
    }
    if (b_codes) {
      for (int u = tid; u < bn * 8; u += kThreads) {
        const int c = u & 7, j = u >> 3;
        const int64_t col = (int64_t)nt * bn + j;
        const bool ok = col < P.n;
        cp_async16(smem_u32(rbp) + umma_off(j, c), P.rhs_codes + (ok ? col : 0) * P.rhs_ld + kt * 128 + c * 16, ok);
      }
    } else {
      for (int u = tid; u < rbits * bn; u += kThreads) {
        const int p = u >> P.log2bn, j = u & (bn - 1);
        const int64_t vc = (int64_t)nt * bn + j;
        int64_t col = vc, pl = p;
        if (PER_PLANE) { pl = vc / P.vstride; col = vc % P.vstride; }
        const bool ok = pl < P.rbits && col < P.n_padded && vc < P.n_ext;
        cp_async16(smem_u32(rbp) + (p * bn + j) * 16, P.rhs + (ok ? pl * P.rwpp + col * P.rwpr : 0) + kt * 4, ok);
      }
    }
  };

  // prologue: prefetch the first PD K tiles (empty groups keep the group count uniform)
  for (int s0 = 0; s0 < PD; ++s0) {
    if (s0 < nk) issue(klist ? klist[s0] : s0, s0 % NR);
    cp_async_commit();
  }
  if (P.mode == QG_GEMM_EPILOGUE) {
    // per-column epilogue constants of this CTA's columns (same fp64 products as the
    // reference's broadcast terms, computed once instead of per element)
    const qg_epilogue& E0 = P.epi;
    for (int i = tid; i < bn; i += kThreads) {
      const int64_t c = (int64_t)nt * bn + i;
      const bool ok = c < P.n;
      sCol[0 * bn + i] = (ok && E0.use_col) ? __dmul_rn(E0.k_col, (double)E0.col_sums[c]) : 0.0;
      sCol[1 * bn + i] = (ok && E0.bias) ? E0.bias[c] : 0.0;
      if (E0.bn_mean) {
        sCol[2 * bn + i] = ok ? E0.bn_mean[c] : 0.0;
        sCol[3 * bn + i] = ok ? E0.bn_denom[c] : 1.0;
        sCol[4 * bn + i] = ok ? E0.bn_inv_denom[c] : 1.0;
        sCol[5 * bn + i] = ok ? E0.bn_gamma[c] : 0.0;
        sCol[6 * bn + i] = ok ? E0.bn_beta[c] : 0.0;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;
  const uint32_t idesc = idesc_u8(bn);
  phase_stamp(P, 1);

  for (int it = 0; it < nk; ++it) {
    const int st = it & 1, rs = it % NR;
    const int pf = it + PD;
    if (pf < nk) {
      if (pf >= NR) mbar_wait(smem_u32(&mbar_r[pf % NR]), ((pf - NR) / NR) & 1);   // stage free again
      issue(klist ? klist[pf] : pf, pf % NR);
    }
    cp_async_commit();
    if (PD >= 2) cp_async_wait<2>(); else cp_async_wait<1>();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // cp.async data -> tensor-core reads
    __syncthreads();                                   // raw stage rs visible to every thread
    if (it < 16) phase_stamp(P, 6 + 4 * it);
    if (expand && it >= 2) mbar_wait(smem_u32(&mbar_x[st]), ((it - 2) >> 1) & 1);
    if (it < 16) phase_stamp(P, 7 + 4 * it);
    if (expand) {
      const uint32_t* ra = reinterpret_cast<const uint32_t*>(rawA + rs * rawA_bytes);
      const uint32_t* rbw = reinterpret_cast<const uint32_t*>(rawB + rs * rawB_bytes);
      if (!a_codes) {
        // A: thread -> row r = tid&127, K-cores h, h+2, h+4, h+6 (h = tid>>7): one 128-bit
        // shared load per plane feeds four independent expansion chains.
        const int r = tid & 127, h = tid >> 7;
        uint32_t o[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0;
#pragma unroll 1
        for (int p = 0; p < lb; ++p) {
          const uint4 w4 = *reinterpret_cast<const uint4*>(ra + (p * 128 + r) * 4);
          const uint32_t wv[4] = {w4.x >> (16 * h), w4.y >> (16 * h), w4.z >> (16 * h), w4.w >> (16 * h)};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            o[i][0] |= expand_nibble(wv[i] & 0xFu) << p;
            o[i][1] |= expand_nibble((wv[i] >> 4) & 0xFu) << p;
            o[i][2] |= expand_nibble((wv[i] >> 8) & 0xFu) << p;
            o[i][3] |= expand_nibble((wv[i] >> 12) & 0xFu) << p;
          }
        }
        const uint32_t abase = sA0 + st * 16384u;
#pragma unroll
        for (int i = 0; i < 4; ++i) sts128(abase + umma_off(r, h + 2 * i), o[i][0], o[i][1], o[i][2], o[i][3]);
      }
      if (!b_codes) {
        // B: thread -> column j = tid & (bn-1), K-cores c0, c0+cs, ... (bn/32 of them)
        const int j = tid & (bn - 1), c0 = tid >> P.log2bn, cs = kThreads >> P.log2bn;
        const uint32_t bbase = sB0 + st * bstage;
#pragma unroll 1
        for (int c = c0; c < 8; c += cs) {
          const int wi = c >> 1, sh = (c & 1) * 16;
          uint32_t o0 = 0, o1 = 0, o2 = 0, o3 = 0;
#pragma unroll 1
          for (int p = 0; p < rbits; ++p) {
            const uint32_t w = rbw[(p * bn + j) * 4 + wi] >> sh;
            const int shp = PER_PLANE ? 0 : p;
            o0 |= expand_nibble(w & 0xFu) << shp;
            o1 |= expand_nibble((w >> 4) & 0xFu) << shp;
            o2 |= expand_nibble((w >> 8) & 0xFu) << shp;
            o3 |= expand_nibble((w >> 12) & 0xFu) << shp;
          }
          sts128(bbase + umma_off(j, c), o0, o1, o2, o3);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
    }
    if (it < 16) phase_stamp(P, 8 + 4 * it);
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t abase = a_codes ? smem_u32(rawA + rs * rawA_bytes) : sA0 + st * 16384u;
      const uint32_t bbase = b_codes ? smem_u32(rawB + rs * rawB_bytes) : sB0 + st * bstage;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t da = umma_desc(abase + kk * 256u);
        const uint64_t db = umma_desc(bbase + kk * 256u);
        const uint32_t accum = (it > 0 || kk > 0) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(accum));
      }
      if (expand)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&mbar_x[st])) : "memory");
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&mbar_r[rs])) : "memory");
    }
    if (it < 16) phase_stamp(P, 9 + 4 * it);
  }
  cp_async_wait<0>();
  if (nk > 0) {
    mbar_wait(smem_u32(&mbar_r[(nk - 1) % NR]), ((nk - 1) / NR) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  phase_stamp(P, 2);

  // ---- epilogue: 8-column TMEM slices spread over all 8 warps ----
  // warp w owns TMEM lanes 32*(w%4).. (rows) and slices s = w/4, w/4 + 2, ...
  const int quad = warp & 3, half = warp >> 2;
  const int64_t r0 = rb * 128 + quad * 32;
  const int64_t myrow = r0 + lane;
  const int64_t col_lo = (int64_t)nt * bn;
  const int64_t rem_cols = P.n_ext - col_lo;
  const int ncols_cta = rem_cols <= 0 ? 0 : (rem_cols < bn ? (int)rem_cols : bn);
  const int nslices = (ncols_cta + 7) >> 3;
  const qg_epilogue& E = P.epi;
  const bool fused = P.mode == QG_GEMM_EPILOGUE;
  const bool packed = fused && E.out_kind == QG_OUT_PLANES;
  const bool colwise = packed && E.q_orientation == QG_COLUMN_WISE;
  // colwise words of the CTA tile are OR-accumulated in smem (reusing the sA stages)
  uint32_t* sWords = reinterpret_cast<uint32_t*>(smem);     // [128 rows][bn/32 words][8 planes]
  __shared__ unsigned long long sRowSum[128];
  const int wpc_cta = (bn + 31) >> 5;
  if (packed) {
    for (int i = tid; i < 128 * wpc_cta * 8; i += kThreads) sWords[i] = 0;
    if (tid < 128) sRowSum[tid] = 0ull;
  }
  __syncthreads();
  const bool rvalid = myrow < P.m;
  const uint32_t maxv = packed ? (1u << E.q_bits) - 1u : 0u;
  // row term k_row * row_sums[r] is identical for every column (hoisted)
  const double rterm = (fused && E.use_row && rvalid) ? __dmul_rn(E.k_row, (double)E.row_sums[myrow]) : 0.0;
  unsigned long long rsum = 0;
  const int wpc_rows = packed ? (int)(E.q_prows >> 5) : 0;
  for (int sl = half; sl < nslices; sl += 2) {
    const int64_t cb = col_lo + sl * 8;
    uint64_t codes8 = 0;                 // byte jj = requantized code of column cb+jj (colwise packing)
#pragma unroll 1
    for (int g = 0; g < 2; ++g) {        // two groups of 4 columns: small code, 4 independent chains
      uint32_t v[4];
      if (nk > 0) {
        const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(sl * 8 + g * 4);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      } else {
        v[0] = v[1] = v[2] = v[3] = 0;
      }
      const int64_t c4 = cb + g * 4;
      if (!fused) {
        if (rvalid) {
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int64_t vc = c4 + jj;
            if (PER_PLANE) {
              const int64_t pl = vc / P.vstride, col = vc % P.vstride;
              if (pl < P.rbits && col < P.n) P.out_i32[(pl * P.m + myrow) * P.n + col] = (int32_t)v[jj];
            } else if (vc < P.n) {
              P.out_i32[myrow * P.n + vc] = (int32_t)v[jj];
            }
          }
        }
        continue;
      }
      double real[4];
      const int cl4 = sl * 8 + g * 4;             // CTA-local column of element 0
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int cl = cl4 + jj;
        double x = __dmul_rn(E.k_acc, (double)(int32_t)v[jj]);
        if (E.use_row) x = __dadd_rn(x, rterm);
        if (E.use_col) x = __dadd_rn(x, sCol[cl]);
        if (E.use_const) x = __dadd_rn(x, E.k_const);
        if (E.bias) x = __dadd_rn(x, sCol[bn + cl]);
        if (E.bn_mean)
          x = __dadd_rn(__dmul_rn(__ddiv_rn(__dsub_rn(x, sCol[2 * bn + cl]), sCol[3 * bn + cl]), sCol[5 * bn + cl]),
                        sCol[6 * bn + cl]);
        if (E.act == QG_ACT_RELU) x = (x < 0.0) ? 0.0 : x;
        else if (E.act == QG_ACT_TANH) x = tanh_f32(x);
        real[jj] = x;
      }
      if (!packed) {
        if (rvalid) {
          double* dst = E.out_real + myrow * P.n;
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            if (c4 + jj < P.n) dst[c4 + jj] = real[jj];
        }
        continue;
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int64_t c = c4 + jj;
        uint32_t q = 0;
        if (rvalid && c < P.n) {
          if (!isfinite(real[jj])) status_min(E.status, myrow * P.n + c);
          q = quantize_code_fast(real[jj], E.q_amin, E.q_scale, E.q_inv_scale, maxv);
          rsum += q;
        }
        codes8 |= (uint64_t)q << (8 * (g * 4 + jj));
      }
    }
    if (packed && E.q_codes && rvalid) {
      // u8 code cache in the next GEMM's K-major operand layout
      if (E.q_codes_colmajor) {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
          if (cb + jj < P.n) E.q_codes[(cb + jj) * E.q_codes_ld + myrow] = (uint8_t)(codes8 >> (8 * jj));
      } else {
        *reinterpret_cast<uint64_t*>(E.q_codes + myrow * E.q_codes_ld + cb) = codes8;
      }
    }
    if (packed && !colwise && !E.q_skip_planes) {
      // row-wise words: column cb+jj over the warp's 32 rows; lane jj keeps the ballot
      // of column jj, then 8 lanes store one word per plane
      const uint64_t planes8 = transpose8x8(codes8);   // byte p, bit jj = bit p of code jj
      const int64_t c = cb + lane;
      const bool in = lane < 8 && c < E.q_pcols && (r0 >> 5) < wpc_rows;
      uint32_t* dst = E.q_planes + (in ? c * wpc_rows + (r0 >> 5) : 0);
      const int64_t pstride = E.q_pcols * wpc_rows;
#pragma unroll 1
      for (int p = 0; p < E.q_bits; ++p) {
        const uint32_t byte = (uint32_t)(planes8 >> (8 * p)) & 0xFFu;
        uint32_t mine = 0;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const uint32_t b = __ballot_sync(QG_FULL, (byte >> jj) & 1u);
          mine = (lane == jj) ? b : mine;
        }
        if (in) dst[p * pstride] = mine;
      }
    }
    if (colwise && !E.q_skip_planes) {
      // byte p of the transpose = plane p's 8 bits of this slice
      const uint64_t planes8 = transpose8x8(codes8);
      const int lr = quad * 32 + lane;
      const int wi = (sl * 8) >> 5, sh = (sl * 8) & 31;
#pragma unroll 1
      for (int p = 0; p < E.q_bits; ++p) {
        const uint32_t b = (uint32_t)(planes8 >> (8 * p)) & 0xFFu;
        if (b) atomicOr(&sWords[(lr * wpc_cta + wi) * 8 + p], b << sh);
      }
    }
  }
  phase_stamp(P, 3);
  if (packed) {
    if (rsum) atomicAdd(&sRowSum[quad * 32 + lane], rsum);
    __syncthreads();
    if (colwise && !E.q_skip_planes) {
      const int64_t wpr = E.q_pcols >> 5, wpp = E.q_prows * wpr;
      const int64_t w0 = col_lo >> 5;
      for (int i = tid; i < 128 * wpc_cta * 8; i += kThreads) {
        const int p = i & 7, wi = (i >> 3) % wpc_cta, lr = (i >> 3) / wpc_cta;
        const int64_t row = rb * 128 + lr;
        if (p < E.q_bits && row < E.q_prows && w0 + wi < wpr) E.q_planes[p * wpp + row * wpr + w0 + wi] = sWords[i];
      }
    }
    if (E.q_row_sums && tid < 128 && rb * 128 + tid < P.m && sRowSum[tid])
      atomicAdd(reinterpret_cast<unsigned long long*>(E.q_row_sums + rb * 128 + tid), sRowSum[tid]);
  }
  phase_stamp(P, 4);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
  phase_stamp(P, 5);
}

// ----------------------------------------------------------- POPC (exact)
// One thread per output element; lanes of a warp share the L row (broadcast)
// and walk their own R column.  Exact: per plane pair the 128-bit popcount
// sum is shifted by p+q into an int64 accumulator.
template <bool PER_PLANE>
__global__ void __launch_bounds__(256) popc_bitgemm_kernel(const __grid_constant__ GemmParams P,
                                                           int32_t* __restrict__ out, int plane) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= P.m * P.n) return;
  const int64_t r = idx / P.n, c = idx % P.n;
  const int64_t rblk = r >> 7;
  const int nk = P.blk_count ? P.blk_count[rblk] : P.k_tiles;
  const int32_t* klist = P.blk_list ? P.blk_list + rblk * (int64_t)P.k_tiles : nullptr;
  long long total = 0;
  for (int it = 0; it < nk; ++it) {
    const int kt = klist ? klist[it] : it;
    for (int p = 0; p < P.lbits; ++p) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(P.lhs + p * P.lwpp + r * P.lwpr + kt * 4));
      if (PER_PLANE) {
        const uint4 b = __ldg(reinterpret_cast<const uint4*>(P.rhs + plane * P.rwpp + c * P.rwpr + kt * 4));
        total += __popc(a.x & b.x) + __popc(a.y & b.y) + __popc(a.z & b.z) + __popc(a.w & b.w);
      } else {
        for (int q = 0; q < P.rbits; ++q) {
          const uint4 b = __ldg(reinterpret_cast<const uint4*>(P.rhs + q * P.rwpp + c * P.rwpr + kt * 4));
          const long long s = __popc(a.x & b.x) + __popc(a.y & b.y) + __popc(a.z & b.z) + __popc(a.w & b.w);
          total += s << (p + q);
        }
      }
    }
  }
  if (total > 2147483647LL || total < -2147483648LL) {
    if (P.overflow) atomicExch(P.overflow, 1);
  }
  out[(PER_PLANE ? (int64_t)plane * P.m * P.n : 0) + idx] = (int32_t)total;
}

// ------------------------------------------------------- standalone epilogue
__global__ void __launch_bounds__(256) epilogue_kernel(const int32_t* __restrict__ acc, int64_t rows, int64_t cols,
                                                       const __grid_constant__ qg_epilogue E) {
  const int lane = threadIdx.x & 31;
  const int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t cchunks = (cols + 31) >> 5;
  // cover the padded output so every 32-row group gets its row-wise words
  const int64_t rgroups = (rows + 31) >> 5;
  if (item >= rgroups * cchunks) return;
  const int64_t r0 = (item / cchunks) * 32, c0 = (item % cchunks) * 32;
  const int64_t r = r0 + lane;
  auto get8 = [&](int sub, uint32_t (&v)[8]) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t c = c0 + sub * 8 + j;
      v[j] = (r < rows && c < cols) ? (uint32_t)acc[r * cols + c] : 0u;
    }
  };
  epi_chunk32(E, r0, c0, get8, rows, cols);
}

}  // namespace qg

using namespace qg;

static inline int launch_status_g() { return cudaGetLastError() == cudaSuccess ? QG_OK : QG_ERR_CUDA; }

static int epilogue_launch(const int32_t* acc, int64_t rows, int64_t cols, const qg_epilogue& e, cudaStream_t st) {
  const int64_t warps = ((rows + 31) / 32) * ((cols + 31) / 32);
  if (warps == 0) return QG_OK;
  epilogue_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(acc, rows, cols, e);
  return launch_status_g();
}

static int check_epilogue(const qg_epilogue* e) {
  if (!e) return QG_ERR_ARG;
  if (e->use_row && !e->row_sums) return QG_ERR_ARG;
  if (e->use_col && !e->col_sums) return QG_ERR_ARG;
  if (e->out_kind == QG_OUT_REAL) return e->out_real ? QG_OK : QG_ERR_ARG;
  if (e->out_kind != QG_OUT_PLANES) return QG_ERR_ARG;
  if (!e->q_planes && !(e->q_skip_planes && e->q_codes)) return QG_ERR_ARG;
  if (e->q_codes && e->q_codes_ld % 16) return QG_ERR_SHAPE;
  if (e->q_bits < 1 || e->q_bits > 8) return QG_ERR_BITS;
  if (e->q_prows % 8 || e->q_pcols % 8) return QG_ERR_SHAPE;
  if (e->q_orientation == QG_ROW_WISE && e->q_prows % 128) return QG_ERR_SHAPE;
  if (e->q_orientation == QG_COLUMN_WISE && e->q_pcols % 128) return QG_ERR_SHAPE;
  return QG_OK;
}

extern "C" int qg_epilogue_apply(const int32_t* acc, int64_t rows, int64_t cols, const qg_epilogue* epi,
                                 void* stream) {
  if (rows < 0 || cols < 0 || (rows * cols > 0 && !acc)) return QG_ERR_ARG;
  int rc = check_epilogue(epi);
  if (rc != QG_OK) return rc;
  if (epi->out_kind == QG_OUT_PLANES && (epi->q_prows < rows || epi->q_pcols < cols)) return QG_ERR_SHAPE;
  return epilogue_launch(acc, rows, cols, *epi, (cudaStream_t)stream);
}

template <bool PER_PLANE, int COLS>
static void set_smem_attr(size_t bytes) {
  static size_t done = 0;
  if (bytes > done) {
    cudaFuncSetAttribute(tc_bitgemm_kernel<PER_PLANE, COLS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)bytes);
    done = bytes;
  }
}

template <bool PER_PLANE>
static int launch_tc(GemmParams P, dim3 grid, cudaStream_t st) {
  const int rbits = PER_PLANE ? 1 : P.rbits;
  const bool ac = P.lhs_codes != nullptr, bc = P.rhs_codes != nullptr;
  const size_t expanded = (ac ? 0 : 2 * 16384) + (bc ? 0 : 2 * (size_t)P.bn * 128);
  const size_t colc = 7 * (size_t)P.bn * 8;
  const size_t stage = (ac ? 16384 : (size_t)P.lbits * 2048) + (bc ? (size_t)P.bn * 128 : (size_t)rbits * P.bn * 16);
  const size_t budget = 227 * 1024 - 4096;           // keep room for static smem
  P.raw_stages = (int32_t)std::max<size_t>(2, std::min<size_t>(4, (budget - expanded - colc) / stage));
  P.pf_dist = std::max(1, P.raw_stages - 2);
  // layout: [expanded stages][raw ring] then sCol, never below the 32 KB epilogue scratch
  const size_t smem = std::max<size_t>(expanded + (size_t)P.raw_stages * stage, 32768) + colc;
  const int cols = P.bn <= 32 ? 32 : P.bn <= 64 ? 64 : P.bn <= 128 ? 128 : 256;
  switch (cols) {
    case 32: set_smem_attr<PER_PLANE, 32>(smem); tc_bitgemm_kernel<PER_PLANE, 32><<<grid, kThreads, smem, st>>>(P); break;
    case 64: set_smem_attr<PER_PLANE, 64>(smem); tc_bitgemm_kernel<PER_PLANE, 64><<<grid, kThreads, smem, st>>>(P); break;
    case 128: set_smem_attr<PER_PLANE, 128>(smem); tc_bitgemm_kernel<PER_PLANE, 128><<<grid, kThreads, smem, st>>>(P); break;
    default: set_smem_attr<PER_PLANE, 256>(smem); tc_bitgemm_kernel<PER_PLANE, 256><<<grid, kThreads, smem, st>>>(P); break;
  }
  return launch_status_g();
}

extern "C" int qg_bitgemm(const qg_gemm_args* a, void* stream) {
  if (!a || !a->lhs || !a->rhs) return QG_ERR_ARG;
  if (a->lbits < 1 || a->lbits > 8 || a->rbits < 1 || a->rbits > 8) return QG_ERR_BITS;
  if (a->m < 0 || a->n < 0 || a->k < 0 || a->m_padded < a->m || a->n_padded < a->n) return QG_ERR_SHAPE;
  if (a->k_padded % 128 || a->m_padded % 8 || a->n_padded % 8) return QG_ERR_SHAPE;
  if (a->mode == QG_GEMM_PER_PLANE && a->lbits != 1) return QG_ERR_ARG;
  if (a->mode == QG_GEMM_EPILOGUE) {
    int rc = check_epilogue(a->epi);
    if (rc != QG_OK) return rc;
  } else if (!a->out_i32) {
    return QG_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (a->m == 0 || a->n == 0) return QG_OK;
  GemmParams P{};
  P.lhs = a->lhs; P.rhs = a->rhs;
  P.m = a->m; P.m_padded = a->m_padded; P.n = a->n; P.n_padded = a->n_padded;
  P.lwpr = a->k_padded / 32; P.lwpp = a->m_padded * P.lwpr;
  P.rwpr = a->k_padded / 32; P.rwpp = a->n_padded * P.rwpr;
  P.lbits = a->lbits; P.rbits = a->rbits;
  P.k_tiles = (int32_t)(a->k_padded / 128);
  P.mode = a->mode;
  P.blk_list = a->blk_list; P.blk_count = a->blk_count;
  P.out_i32 = a->out_i32; P.overflow = a->overflow; P.phase_ns = a->phase_ns;
  P.lhs_codes = a->lhs_codes; P.lhs_ld = a->lhs_ld; P.rhs_codes = a->rhs_codes; P.rhs_ld = a->rhs_ld;
  if ((P.lhs_codes && (P.lhs_ld < a->k_padded || P.lhs_ld % 16)) || (P.rhs_codes && (P.rhs_ld < a->k_padded || P.rhs_ld % 16)))
    return QG_ERR_SHAPE;
  if (a->epi) P.epi = *a->epi;

  // the s32 tensor accumulator is exact iff the largest possible sum fits
  const double maxsum = (a->mode == QG_GEMM_PER_PLANE)
                            ? (double)a->k
                            : (double)((1 << a->lbits) - 1) * (double)((1 << a->rbits) - 1) * (double)a->k;
  int algo = a->algo;
  if (algo == QG_ALGO_AUTO) algo = maxsum < 2147483647.0 ? QG_ALGO_TCGEN05 : QG_ALGO_POPC;
  if (algo == QG_ALGO_TCGEN05 && maxsum >= 2147483647.0) return QG_ERR_UNSUPPORTED;
  if (algo == QG_ALGO_POPC && (P.lhs_codes || P.rhs_codes)) return QG_ERR_UNSUPPORTED;   // POPC reads planes

  if (algo == QG_ALGO_TCGEN05) {
    const int64_t row_blocks = (a->m_padded + 127) / 128;
    // column extent actually computed: logical columns (padding columns of R are zero)
    int64_t vtotal;
    if (a->mode == QG_GEMM_PER_PLANE) {
      const int64_t n32 = (a->n + 31) / 32 * 32;
      if (a->cross_bit || n32 > 256) {
        P.vstride = std::max<int64_t>(32, n32);                    // one plane per tile group
        P.vstride = (P.vstride + 255) / 256 * 256 > 256 ? (P.vstride + 255) / 256 * 256 : P.vstride;
      } else {
        P.vstride = a->n;                                          // planes stacked along N
      }
      vtotal = P.vstride * a->rbits;
    } else {
      P.vstride = a->n_padded;
      vtotal = a->n;
    }
    P.n_ext = vtotal;
    const int64_t ext32 = std::max<int64_t>(32, (vtotal + 31) / 32 * 32);
    // largest power-of-two N tile (32..256) that still gives >= one full wave of CTAs
    int bn = 32;
    while (bn < 256 && bn < ext32) bn *= 2;
    while (bn > 32 && row_blocks * ((ext32 + bn - 1) / bn) < 148) bn /= 2;
    if (a->mode == QG_GEMM_PER_PLANE && a->cross_bit)
      while (bn > 32 && bn > P.vstride) bn /= 2;
    P.bn = bn;
    P.log2bn = 5;
    while ((1 << P.log2bn) < bn) ++P.log2bn;
    P.n_tiles = (int32_t)((ext32 + bn - 1) / bn);
    dim3 grid((unsigned)row_blocks, (unsigned)P.n_tiles);
    if (a->mode == QG_GEMM_PER_PLANE) return launch_tc<true>(P, grid, st);
    return launch_tc<false>(P, grid, st);
  }
  // POPC path
  const int64_t total = a->m * a->n;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  if (a->mode == QG_GEMM_PER_PLANE) {
    for (int p = 0; p < a->rbits; ++p) popc_bitgemm_kernel<true><<<blocks, 256, 0, st>>>(P, a->out_i32, p);
    return launch_status_g();
  }
  int32_t* dst = a->mode == QG_GEMM_I32 ? a->out_i32 : a->scratch_i32;
  if (!dst) return QG_ERR_ARG;
  popc_bitgemm_kernel<false><<<blocks, 256, 0, st>>>(P, dst, 0);
  int rc = launch_status_g();
  if (rc != QG_OK || a->mode == QG_GEMM_I32) return rc;
  return epilogue_launch(dst, a->m, a->n, *a->epi, st);
}

namespace qg {
__global__ void test_div_kernel(const double* a, const double* b, const double* y, int64_t n, double* out,
                                double* ref) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = div_rn(a[i], b[i], y[i]);
  ref[i] = __ddiv_rn(a[i], b[i]);
}
}  // namespace qg

extern "C" int qg_test_div(const double* a, const double* b, const double* inv_b, int64_t n, double* out,
                           double* ref, void* stream) {
  if (n < 0 || (n && (!a || !b || !inv_b || !out || !ref))) return QG_ERR_ARG;
  if (n == 0) return QG_OK;
  qg::test_div_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(a, b, inv_b, n, out, ref);
  return launch_status_g();
}

namespace qg {
// Direct case: the packed axis of the planes is the contiguous axis of the code
// layout (row-wise planes -> col-major codes, column-wise planes -> row-major
// codes).  Thread per word position: 32 codes = 32 contiguous bytes, built with
// the nibble-expansion trick (bit i of plane p -> bit p of byte i).
__global__ void planes_to_codes_direct_kernel(const uint32_t* __restrict__ words, int nplanes, int64_t lines,
                                              int64_t line_len, int64_t wpl, int64_t wpp,
                                              uint8_t* __restrict__ codes, int64_t ld) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nw = (line_len + 31) >> 5;
  if (idx >= lines * nw) return;
  const int64_t line = idx / nw, w = idx % nw;
  uint32_t o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int p = 0; p < nplanes; ++p) {
    const uint32_t x = __ldg(words + p * wpp + line * wpl + w);
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] |= expand_nibble((x >> (4 * q)) & 0xFu) << p;
  }
  uint8_t* dst = codes + line * ld + w * 32;
  const int64_t rem = line_len - w * 32;
  if (rem >= 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
    reinterpret_cast<uint4*>(dst)[0] = make_uint4(o[0], o[1], o[2], o[3]);
    reinterpret_cast<uint4*>(dst)[1] = make_uint4(o[4], o[5], o[6], o[7]);
  } else {
    for (int i = 0; i < 32 && i < rem; ++i) dst[i] = (uint8_t)(o[i >> 2] >> (8 * (i & 3)));
  }
}

// Transpose case: row-wise planes -> row-major codes (or column-wise -> col-major).
// Block = 32 output lines x 256 positions: thread t owns position t, expands its
// word of 32 lines into a shared tile, then the tile is written line-major with
// coalesced stores.  Optional per-line sums (row sums of the codes).
__global__ void __launch_bounds__(256) planes_to_codes_transpose_kernel(
    const uint32_t* __restrict__ words, int nplanes, int64_t lines, int64_t positions, int64_t wpl, int64_t wpp,
    uint8_t* __restrict__ codes, int64_t ld, int64_t* __restrict__ line_sums) {
  __shared__ uint8_t tile[32][256 + 16];
  const int t = threadIdx.x;
  const int64_t v = blockIdx.y;                 // 32-line group
  const int64_t pos = (int64_t)blockIdx.x * 256 + t;
  uint32_t o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (pos < positions) {
    for (int p = 0; p < nplanes; ++p) {
      const uint32_t x = __ldg(words + p * wpp + pos * wpl + v);
#pragma unroll
      for (int q = 0; q < 8; ++q) o[q] |= expand_nibble((x >> (4 * q)) & 0xFu) << p;
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) tile[i][t] = (uint8_t)(o[i >> 2] >> (8 * (i & 3)));
  __syncthreads();
  // each warp writes 4 lines of 256 bytes
  const int warp = t >> 5, lane = t & 31;
  for (int i = warp; i < 32; i += 8) {
    const int64_t line = v * 32 + i;
    if (line >= lines) break;
    uint32_t sum = 0;
    for (int j = lane; j < 256; j += 32) {
      const int64_t q = (int64_t)blockIdx.x * 256 + j;
      if (q < positions) {
        codes[line * ld + q] = tile[i][j];
        sum += tile[i][j];
      }
    }
    if (line_sums) {
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) sum += __shfl_xor_sync(QG_FULL, sum, o2);
      if (lane == 0 && sum) atomicAdd(reinterpret_cast<unsigned long long*>(line_sums + line), (unsigned long long)sum);
    }
  }
}
}  // namespace qg

extern "C" int qg_planes_to_codes(const uint32_t* words, int64_t nplanes, int64_t rows, int64_t cols,
                                  int64_t padded_rows, int64_t padded_cols, int orientation, uint8_t* codes,
                                  int64_t ld, int colmajor, int64_t* row_sums, void* stream) {
  if (!words || !codes || nplanes < 1 || nplanes > 8 || rows < 0 || cols < 0) return QG_ERR_ARG;
  if (ld < (colmajor ? rows : cols)) return QG_ERR_SHAPE;
  if (rows * cols == 0) return QG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t wpp = padded_rows * padded_cols / 32;
  const bool rowwise = orientation == QG_ROW_WISE;
  if (rowwise == (bool)colmajor) {
    // packed axis == contiguous code axis
    const int64_t lines = colmajor ? cols : rows, len = colmajor ? rows : cols;
    const int64_t wpl = rowwise ? padded_rows / 32 : padded_cols / 32;
    const int64_t n = lines * ((len + 31) / 32);
    qg::planes_to_codes_direct_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        words, (int)nplanes, lines, len, wpl, wpp, codes, ld);
    if (row_sums) return QG_ERR_UNSUPPORTED;   // row sums only on the transpose (left-operand) path
  } else {
    // row-wise planes -> row-major codes: lines = rows, positions = columns
    const int64_t lines = colmajor ? cols : rows, positions = colmajor ? rows : cols;
    const int64_t wpl = rowwise ? padded_rows / 32 : padded_cols / 32;
    dim3 grid((unsigned)((positions + 255) / 256), (unsigned)((lines + 31) / 32));
    qg::planes_to_codes_transpose_kernel<<<grid, 256, 0, st>>>(words, (int)nplanes, lines, positions, wpl, wpp,
                                                               codes, ld, colmajor ? nullptr : row_sums);
  }
  return launch_status_g();
}

namespace qg {
__global__ void test_requant_kernel(const double* x, int64_t n, double amin, double scale, double inv, int bits,
                                    uint32_t* out, uint32_t* ref) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t maxv = (1u << bits) - 1u;
  const uint32_t fast = quantize_code_fast(x[i], amin, scale, inv, maxv);
  // the tiled epilogue's form: branch-free candidate, exact pass when flagged
  const R12 c = quantize_code_r12(x[i], amin, inv, maxv);
  const uint32_t nb = (c.flag || !isfinite(x[i])) ? fast : c.code;
  out[i] = nb == fast ? fast : 0xFFFFFFFFu;
  ref[i] = quantize_code_ref(x[i], amin, scale, maxv);
}
}  // namespace qg

extern "C" int qg_test_requant(const double* x, int64_t n, double amin, double scale, double inv_scale, int bits,
                               uint32_t* out, uint32_t* ref, void* stream) {
  if (n < 0 || (n && (!x || !out || !ref)) || bits < 1 || bits > 8) return QG_ERR_ARG;
  if (n == 0) return QG_OK;
  qg::test_requant_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, n, amin, scale,
                                                                                       inv_scale, bits, out, ref);
  return launch_status_g();
}

extern "C" int qg_version(void) { return 30; }  // == number of exported entry points

// ---------------------------------------------------------------------------
// Reference-shaped entry points over qg_bitgemm / cudaMemcpyAsync,
// and the OpCounters closed forms (host-only).
extern "C" int qg_bmm_1xs(const qg_gemm_args* a, void* stream) {
  if (!a) return QG_ERR_ARG;
  if (a->lbits != 1) return QG_ERR_BITS;
  return qg_bitgemm(a, stream);
}

extern "C" int qg_gemm_sxt(const qg_gemm_args* a, void* stream) {
  if (!a) return QG_ERR_ARG;
  if (a->mode != QG_GEMM_I32 && a->mode != QG_GEMM_EPILOGUE) return QG_ERR_ARG;
  return qg_bitgemm(a, stream);
}

extern "C" int qg_batch_h2d(const void* pinned_src, int64_t nbytes, void* device_dst, void* stream) {
  if (nbytes < 0 || (nbytes && (!pinned_src || !device_dst))) return QG_ERR_ARG;
  if (nbytes == 0) return QG_OK;
  const cudaError_t e = cudaMemcpyAsync(device_dst, pinned_src, (size_t)nbytes, cudaMemcpyHostToDevice,
                                        (cudaStream_t)stream);
  return e == cudaSuccess ? QG_OK : QG_ERR_CUDA;
}

extern "C" int qg_bmm_counters(int64_t rt, int64_t ct, int64_t zero_tiles, int32_t s, int64_t n_chunks, int32_t jump,
                               int32_t cross_tile, qg_counters* out) {
  if (!out || rt < 0 || ct < 0 || n_chunks < 0 || s < 1 || s > 8 || zero_tiles < 0 || zero_tiles > rt * ct)
    return QG_ERR_ARG;
  const int64_t total = rt * ct;
  const int64_t nz = jump ? total - zero_tiles : total;
  out->tile_mma_count = (int64_t)s * nz * n_chunks;
  out->tile_fetch_count = cross_tile ? nz : (int64_t)s * nz;
  out->tiles_skipped = jump ? zero_tiles : 0;
  out->word_and_popcount_count = 256 * out->tile_mma_count;
  out->tiles_total = total;
  return QG_OK;
}

extern "C" int qg_gemm_counters(int64_t rt, int64_t ct, const int64_t* plane_zero_tiles, int32_t s, int32_t t,
                                int64_t n_chunks, int32_t jump, int32_t cross_tile, qg_counters* out) {
  if (!out || !plane_zero_tiles || rt < 0 || ct < 0 || n_chunks < 0 || s < 1 || s > 8 || t < 1 || t > 8)
    return QG_ERR_ARG;
  const int64_t per_plane = rt * ct;
  int64_t nz = 0, zeros = 0;
  for (int i = 0; i < s; ++i) {
    if (plane_zero_tiles[i] < 0 || plane_zero_tiles[i] > per_plane) return QG_ERR_ARG;
    nz += jump ? per_plane - plane_zero_tiles[i] : per_plane;
    zeros += plane_zero_tiles[i];
  }
  out->tile_mma_count = (int64_t)t * nz * n_chunks;
  out->tile_fetch_count = cross_tile ? nz : (int64_t)t * nz;
  out->tiles_skipped = jump ? zeros : 0;
  out->word_and_popcount_count = 256 * out->tile_mma_count;
  out->tiles_total = (int64_t)s * per_plane;
  return QG_OK;
}
