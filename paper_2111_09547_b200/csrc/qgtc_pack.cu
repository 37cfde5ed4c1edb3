// bit_qnt and layout kernels: fused quantize + bit-decompose + pack, plane
// packing, unpack/to_val, warp bit-transpose repack, zero-tile scan.
// All HBM-bound; every warp access is a coalesced 128 B row segment.
#include <algorithm>
#include "qgtc_common.cuh"

namespace qg {

// ------------------------------------------------------------ quantize+pack
template <typename SrcT>
__device__ __forceinline__ uint32_t load_code(const SrcT* src, int kind, int64_t r, int64_t c, int64_t ld,
                                              int64_t cols, double amin, double scale, uint32_t maxv,
                                              int64_t* status, int64_t status_base) {
  if constexpr (sizeof(SrcT) == 1) {
    uint32_t v = src[r * ld + c];
    if (v > maxv) { status_min(status, status_base + r * cols + c); v &= maxv; }
    return v;
  } else {
    double x = (double)src[r * ld + c];
    if (!isfinite(x)) status_min(status, status_base + r * cols + c);
    return quantize_code(x, amin, scale, maxv);
  }
}

// Column-wise: one warp per (row, chunk of 32 words).  Lane l reads column
// 32*w + l for each word w of the chunk; ballots form the words; lane j keeps
// word j of the chunk so the final stores are coalesced.
template <typename SrcT, int BITS>
__global__ void __launch_bounds__(256) quantize_pack_col_kernel(
    const SrcT* __restrict__ src, int64_t rows, int64_t cols, int64_t ld, double amin, double scale,
    int64_t prows, int64_t pcols, uint32_t* __restrict__ planes, uint8_t* __restrict__ codes,
    int64_t* __restrict__ row_sums, int64_t* status, int64_t status_base) {
  const int lane = threadIdx.x & 31;
  const int64_t wpr = pcols >> 5;
  const int64_t chunks = (wpr + 31) >> 5;
  const int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (item >= prows * chunks) return;
  const int64_t r = item / chunks;
  const int64_t w0 = (item % chunks) * 32;
  const int nw = (int)(wpr - w0 < 32 ? wpr - w0 : 32);
  const uint32_t maxv = (1u << BITS) - 1u;
  uint32_t mine[BITS];
#pragma unroll
  for (int p = 0; p < BITS; ++p) mine[p] = 0;
  int64_t rsum = 0;
  const bool rvalid = r < rows;
  for (int it = 0; it < nw; ++it) {
    const int64_t c = (w0 + it) * 32 + lane;
    uint32_t code = 0;
    if (rvalid && c < cols) {
      code = load_code<SrcT>(src, 0, r, c, ld, cols, amin, scale, maxv, status, status_base);
      rsum += code;
      if (codes) codes[r * cols + c] = (uint8_t)code;
    }
#pragma unroll
    for (int p = 0; p < BITS; ++p) {
      uint32_t b = __ballot_sync(QG_FULL, (code >> p) & 1u);
      if (lane == it) mine[p] = b;
    }
  }
  if (lane < nw) {
    const int64_t wpp = prows * wpr;
#pragma unroll
    for (int p = 0; p < BITS; ++p) planes[p * wpp + r * wpr + w0 + lane] = mine[p];
  }
  if (row_sums && rvalid) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rsum += __shfl_xor_sync(QG_FULL, rsum, o);
    if (lane == 0 && rsum) atomicAdd(reinterpret_cast<unsigned long long*>(row_sums + r), (unsigned long long)rsum);
  }
}

// Row-wise bit_qnt (the feature path, bitpack.py:181-191 + quantize.py:93-105).
// CTA = 8 warps over a tile of 8 row groups (256 rows) x 32 columns.  Warp w owns row
// group v0 + w, lane = column: every row step is one fully coalesced 128-byte warp load
// (fp32), 8 rows are loaded ahead (independent loads in flight).  Requant: the exact
// division-free form (quantize_code_r12_tight; IEEE fallback only within 2^-40 of a
// code boundary).  The 8 codes of a column's 8-row step go into the bytes of a u64 and
// one 8x8 bit transpose (transpose8x8) turns them into the 8 plane bytes of that step,
// so the plane words (bit i = row 32v + i) are built in registers with no cross-lane
// traffic.  Row sums: one redux.sync per row.  Plane words are staged in shared memory
// so each (plane, column) is stored as 8 consecutive words (32 B) along the row-group
// index instead of 4-byte stores one column pitch apart.
// exact requant of one flagged element (+ the DataError position), kept out of line
template <typename SrcT>
static __device__ __noinline__ uint32_t requant_slow(SrcT x, double amin, double scale, double inv, uint32_t maxv,
                                                     int64_t* status, int64_t flat) {
  if constexpr (sizeof(SrcT) == 1) {
    status_min(status, flat);
    return (uint32_t)x & maxv;
  } else {
    const double xd = (double)x;
    if (!isfinite(xd)) status_min(status, flat);
    return quantize_code_fast(xd, amin, scale, inv, maxv);
  }
}

constexpr int kRowTileCols = 32, kRowTileGroups = 8;

template <typename SrcT, int BITS>
__global__ void __launch_bounds__(256, 3) quantize_pack_row_vec_kernel(
    const SrcT* __restrict__ src, int64_t rows, int64_t cols, int64_t ld, double amin, double scale, double inv,
    int64_t prows, int64_t pcols, uint32_t* __restrict__ planes, uint8_t* __restrict__ codes,
    int64_t* __restrict__ row_sums, int64_t* status, int64_t status_base, int64_t ncolt) {
  __shared__ uint32_t sw[BITS][kRowTileCols][kRowTileGroups + 1];
  const bool single_tile = ncolt == 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wpc = prows >> 5;                          // words per column (row groups)
  // 1-D grid, column tiles fastest: the CTAs covering one row band run together, so the
  // sectors shared by neighbouring (unaligned) column tiles come from L2, not HBM twice
  const int64_t rt = (int64_t)blockIdx.x / ncolt, ct = (int64_t)blockIdx.x % ncolt;
  const int64_t v0 = rt * kRowTileGroups, v = v0 + warp;
  const int64_t c = ct * kRowTileCols + lane;
  const bool cok = c < cols;
  const uint32_t maxv = (1u << BITS) - 1u;
  uint32_t word[BITS];
#pragma unroll
  for (int p = 0; p < BITS; ++p) word[p] = 0u;
  uint32_t my_pair = 0;                                    // lane i: rows 32v + (i & ~1) + {0, 1}
  uint32_t tlo[4] = {0u, 0u, 0u, 0u}, thi[4] = {0u, 0u, 0u, 0u};   // transposed 8-row steps
  // fp32 sources: an fp32 screen y = fma(x, RN32(1/scale), RN32(-amin/scale)) with
  // |y - q| <= 2^-24 (2|y| + 2|c|) against the reference quotient q = RN(RN(x - amin) /
  // scale) (x is exact in fp64); elements within 2^-21 (|y| + |c|) of a code boundary,
  // and non-finite ones, take the exact fp64 path (requant_slow)
  const float inv32 = (float)inv, c32 = (float)(-amin * inv);
  const float mc = fabsf(c32) * 0x1p-21f + 0x1p-40f, hic = (float)maxv + 0.5f, hc = 0.5f - mc;
  if (v < wpc) {
    const int64_t rbase = v * 32;
    const SrcT* colp = src + rbase * ld + c;
    // the loads of kPre 8-row steps are issued before any of them is processed (4 KB per
    // warp in flight for fp32 sources instead of 1 KB: the kernel is HBM-latency bound)
    constexpr int kPre = sizeof(SrcT) >= 8 ? 2 : 4;
#pragma unroll
    for (int s0 = 0; s0 < 4; s0 += kPre) {
    SrcT xs[kPre][8];
#pragma unroll
    for (int s = 0; s < kPre; ++s) {
      const int64_t left = rows - (rbase + (s0 + s) * 8);
      const int nk = left <= 0 ? 0 : (left < 8 ? (int)left : 8);
      const SrcT* p0 = colp + (int64_t)(s0 + s) * 8 * ld;
#pragma unroll
      for (int k = 0; k < 8; ++k) xs[s][k] = (cok && k < nk) ? p0[(int64_t)k * ld] : SrcT(0);
    }
#pragma unroll
    for (int s = 0; s < kPre; ++s) {
      const int i0 = (s0 + s) * 8;
      const int64_t left = rows - (rbase + i0);
      const int nk = left <= 0 ? 0 : (left < 8 ? (int)left : 8);   // valid rows of this step
      const SrcT* x = xs[s];
      uint32_t q[8];
      uint32_t lo, hi;
      if constexpr (sizeof(SrcT) == 4) {
        // per element: FFMA y, 2 FMNMX, FADD.RM floor, 2 FADD frac, FADD frac - 1/2 (exact:
        // frac is a multiple of ulp(yc) >= 2^-24), FFMA h = RN(1/2 - mc) - 2^-21 yc (within
        // 2^-25 of 1/2 - margin; the margin's slack over the error bound is >= 3 * 2^-24),
        // one FSETP |frac - 1/2| > h; non-finite inputs through an FFMA chain (x * 0 is NaN
        // iff x is not finite)
        uint32_t f[8];
        bool bad = false;
        float nf = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float y = fmaf((float)x[k], inv32, c32);
          const float yc = fminf(fmaxf(y, 0.5f), hic);
          const float fl = __fadd_rd(yc, 12582912.0f);     // 1.5 * 2^23 + floor(yc)
          const float d = yc - (fl - 12582912.0f);
          const float h = fmaf(yc, -0x1p-21f, hc);
          f[k] = __float_as_uint(fl);
          bad |= fabsf(d - 0.5f) > h;
          nf = fmaf((float)x[k], 0.f, nf);
        }
        bad |= !(nf == 0.f);
        if (bad && cok) {
          // rare: recheck per element; near-boundary / out-of-range / non-finite ones take
          // the exact path (out of line)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float y = fmaf((float)x[k], inv32, c32);
            const float yc = fminf(fmaxf(y, 0.5f), hic);
            const float d = yc - (__uint_as_float(f[k]) - 12582912.0f);
            const bool fk = (fabsf(d - 0.5f) > fmaf(yc, -0x1p-21f, hc)) |
                            !(fabsf((float)x[k]) <= 3.4028234663852886e38f);
            if (fk && k < nk)
              f[k] = (f[k] & ~0xFFFFu) |
                     requant_slow<SrcT>(x[k], amin, scale, inv, maxv, status, status_base + (rbase + i0 + k) * cols + c);
          }
        }
        if (!(cok && nk == 8)) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (!(cok && k < nk)) f[k] &= ~0xFFFFu;
        }
        // the low 16 bits of f are the code (byte 1 is zero): pairs for the row sums, then
        // the 4-code words
        uint32_t pr[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) pr[k] = __byte_perm(f[2 * k], f[2 * k + 1], 0x5410);
        lo = __byte_perm(pr[0], pr[1], 0x6420);
        hi = __byte_perm(pr[2], pr[3], 0x6420);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t sum = __reduce_add_sync(QG_FULL, pr[k]);
          if ((lane >> 1) == (i0 >> 1) + k) my_pair = sum;
        }
        if (codes) {
#pragma unroll
          for (int k = 0; k < 8; ++k) q[k] = f[k] & 0xFFu;
        }
      } else {
      uint32_t fm = 0u;                                   // elements needing the exact path
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if constexpr (sizeof(SrcT) == 1) {
          q[k] = (uint32_t)x[k];
          fm |= (uint32_t)(q[k] > maxv) << k;
        } else {
          const R12 rq = quantize_code_r12_tight((double)x[k], amin, inv, maxv);
          q[k] = rq.code;
          fm |= (uint32_t)rq.flag << k;
        }
      }
      if (fm && cok) {
        // rare: out-of-range / near-boundary / non-finite elements (out of line)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (((fm >> k) & 1u) && k < nk)
            q[k] = requant_slow<SrcT>(x[k], amin, scale, inv, maxv, status,
                                      status_base + (rbase + i0 + k) * cols + c);
      }
      lo = 0u;
      hi = 0u;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (!(cok && k < nk)) q[k] = 0u;
        if (k < 4) lo |= q[k] << (8 * k);
        else hi |= q[k] << (8 * (k - 4));
      }
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        // rows i0 + k and i0 + k + 1 in the two 16-bit halves (sum <= 32 * 255 < 2^16)
        const uint32_t sum = __reduce_add_sync(QG_FULL, q[k] | (q[k + 1] << 16));
        if ((lane >> 1) == ((i0 + k) >> 1)) my_pair = sum;
      }
      }
      if (codes && cok) {
        uint8_t* cp = codes + (rbase + i0) * cols + c;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < nk) cp[(int64_t)k * cols] = (uint8_t)q[k];
      }
      // byte p of t = plane p of the 8 rows (bit k = row i0 + k)
      const uint64_t t = transpose8x8(((uint64_t)hi << 32) | lo);
      tlo[s0 + s] = (uint32_t)t;
      thi[s0 + s] = (uint32_t)(t >> 32);
    }
    }
    // word p = [byte p of step 0 .. step 3]: 3 PRMT per plane
#pragma unroll
    for (int p = 0; p < BITS; ++p) {
      const uint32_t* tv = p < 4 ? tlo : thi;
      const uint32_t sel = (uint32_t)(p & 3) | ((uint32_t)(4 + (p & 3)) << 4);
      word[p] = __byte_perm(__byte_perm(tv[0], tv[1], sel), __byte_perm(tv[2], tv[3], sel), 0x5410);
    }
    const uint32_t my_sum = (lane & 1) ? my_pair >> 16 : my_pair & 0xFFFFu;
    if (row_sums) {
      const int64_t r = v * 32 + lane;
      if (r < rows && my_sum) {
        if (single_tile) row_sums[r] += (int64_t)my_sum;   // the only writer of row r
        else atomicAdd(reinterpret_cast<unsigned long long*>(row_sums + r), (unsigned long long)my_sum);
      }
    }
  }
#pragma unroll
  for (int p = 0; p < BITS; ++p) sw[p][lane][warp] = word[p];
  __syncthreads();
  // plane p, column c0 + cc, row group v0 + w: word p * wpp + (c0 + cc) * wpc + v0 + w
  const int64_t wpp = pcols * wpc, c0 = ct * kRowTileCols;
  for (int idx = threadIdx.x; idx < BITS * kRowTileCols * kRowTileGroups; idx += blockDim.x) {
    const int w = idx & 7, cc = (idx >> 3) & 31, p = idx >> 8;
    const int64_t col = c0 + cc, vg = v0 + w;
    if (col < pcols && vg < wpc) planes[p * wpp + col * wpc + vg] = sw[p][cc][w];
  }
}

template <typename SrcT>
__global__ void col_sums_kernel(const SrcT* __restrict__ src, int64_t rows, int64_t cols, int64_t ld,
                                double amin, double scale, uint32_t maxv, int64_t* __restrict__ col_sums) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  int64_t s = 0;
  for (int64_t r = 0; r < rows; ++r) {
    if constexpr (sizeof(SrcT) == 1) {
      s += (src[r * ld + c] < maxv ? (uint32_t)src[r * ld + c] : maxv);
    } else {
      s += quantize_code((double)src[r * ld + c], amin, scale, maxv);
    }
  }
  col_sums[c] += s;
}

template <typename SrcT, int BITS>
int launch_quantize_pack(const SrcT* src, int64_t rows, int64_t cols, int64_t ld, double amin, double scale,
                         int orientation, int64_t prows, int64_t pcols, uint32_t* planes, uint8_t* codes,
                         int64_t* row_sums, int64_t* col_sums, int64_t* status, int64_t status_base,
                         cudaStream_t st) {
  int64_t warps;
  if (orientation == QG_COLUMN_WISE) {
    warps = prows * (((pcols >> 5) + 31) >> 5);
  } else {
    warps = (prows >> 5) * ((pcols + 31) >> 5);
  }
  if (warps > 0) {
    const int64_t blocks = (warps * 32 + 255) / 256;
    if (orientation == QG_COLUMN_WISE)
      quantize_pack_col_kernel<SrcT, BITS><<<(unsigned)blocks, 256, 0, st>>>(
          src, rows, cols, ld, amin, scale, prows, pcols, planes, codes, row_sums, status, status_base);
    else {
      const int64_t nrowt = ((prows >> 5) + kRowTileGroups - 1) / kRowTileGroups;
      const int64_t ncolt = (pcols + kRowTileCols - 1) / kRowTileCols;
      quantize_pack_row_vec_kernel<SrcT, BITS><<<(unsigned)(nrowt * ncolt), 256, 0, st>>>(
          src, rows, cols, ld, amin, scale, 1.0 / scale, prows, pcols, planes, codes, row_sums, status, status_base,
          ncolt);
    }
  }
  if (col_sums && cols > 0 && rows > 0)
    col_sums_kernel<SrcT><<<(unsigned)((cols + 127) / 128), 128, 0, st>>>(src, rows, cols, ld, amin, scale,
                                                                          (1u << BITS) - 1u, col_sums);
  return QG_OK;
}

template <typename SrcT>
int dispatch_quantize_pack(const SrcT* src, int64_t rows, int64_t cols, int64_t ld, double amin,
                           double scale, int bits, int orientation, int64_t prows, int64_t pcols,
                           uint32_t* planes, uint8_t* codes, int64_t* row_sums, int64_t* col_sums,
                           int64_t* status, int64_t status_base, cudaStream_t st) {
  switch (bits) {
#define QG_CASE(B) \
  case B:          \
    return launch_quantize_pack<SrcT, B>(src, rows, cols, ld, amin, scale, orientation, prows, pcols, planes, \
                                         codes, row_sums, col_sums, status, status_base, st);
    QG_CASE(1) QG_CASE(2) QG_CASE(3) QG_CASE(4) QG_CASE(5) QG_CASE(6) QG_CASE(7) QG_CASE(8)
#undef QG_CASE
    default:
      return QG_ERR_BITS;
  }
}

// ---------------------------------------------------------------- unpack
__global__ void unpack_kernel(const uint32_t* __restrict__ words, int64_t nplanes, int64_t rows, int64_t cols,
                              int64_t prows, int64_t pcols, int orientation, uint8_t* __restrict__ out_planes,
                              int32_t* __restrict__ out_codes) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  const int64_t r = idx / cols, c = idx % cols;
  const int64_t wpp = prows * pcols / 32;
  int64_t off;
  int bit;
  if (orientation == QG_COLUMN_WISE) {
    off = r * (pcols >> 5) + (c >> 5);
    bit = (int)(c & 31);
  } else {
    off = c * (prows >> 5) + (r >> 5);
    bit = (int)(r & 31);
  }
  int32_t code = 0;
  for (int64_t p = 0; p < nplanes; ++p) {
    uint32_t b = (__ldg(words + p * wpp + off) >> bit) & 1u;
    if (out_planes) out_planes[p * rows * cols + idx] = (uint8_t)b;
    code |= (int32_t)(b << p);
  }
  if (out_codes) out_codes[idx] = code;
}

// ---------------------------------------------------------------- repack
// Warp-level 32x32 bit transpose through ballots: lane i loads the source word
// of line i; ballot j collects bit j of every lane = destination word j.
__global__ void __launch_bounds__(256) repack_kernel(const uint32_t* __restrict__ src, int64_t nplanes,
                                                     int64_t spr, int64_t spc, int src_orientation,
                                                     uint32_t* __restrict__ dst, int64_t dpr, int64_t dpc) {
  const int lane = threadIdx.x & 31;
  // block grid over (row groups of 32) x (column groups of 32) of the padded union
  const int64_t rmax = max(spr, dpr), cmax = max(spc, dpc);
  const int64_t rg = (rmax + 31) >> 5, cg = (cmax + 31) >> 5;
  const int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (item >= rg * cg * nplanes) return;
  const int64_t p = item / (rg * cg);
  const int64_t rem = item % (rg * cg);
  const int64_t v = rem / cg;   // 32-row group
  const int64_t w = rem % cg;   // 32-col group
  const int64_t swpp = spr * spc / 32, dwpp = dpr * dpc / 32;
  uint32_t x = 0;
  if (src_orientation == QG_COLUMN_WISE) {
    // lane i: row 32v+i, word w (cols 32w..)
    const int64_t r = v * 32 + lane;
    if (r < spr && w < (spc >> 5)) x = src[p * swpp + r * (spc >> 5) + w];
  } else {
    // lane i: column 32w+i, word v (rows 32v..)
    const int64_t c = w * 32 + lane;
    if (c < spc && v < (spr >> 5)) x = src[p * swpp + c * (spr >> 5) + v];
  }
  uint32_t mine = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    uint32_t b = __ballot_sync(QG_FULL, (x >> j) & 1u);
    if (lane == j) mine = b;
  }
  if (src_orientation == QG_COLUMN_WISE) {
    // destination row-wise: lane j holds column 32w+j, rows 32v..32v+31
    const int64_t c = w * 32 + lane;
    if (c < dpc && v < (dpr >> 5)) dst[p * dwpp + c * (dpr >> 5) + v] = mine;
  } else {
    // destination column-wise: lane j holds row 32v+j, cols 32w..32w+31
    const int64_t r = v * 32 + lane;
    if (r < dpr && w < (dpc >> 5)) dst[p * dwpp + r * (dpc >> 5) + w] = mine;
  }
}

// -------------------------------------------------------------- tile scan
// One warp per 8-row tile group; lane handles K tiles lane, lane+32, ...
// Each row contributes a 16 B (uint4) load per K tile: 32 lanes read 512
// consecutive bytes of one row -> fully coalesced.
__global__ void __launch_bounds__(256) tile_scan_kernel(const uint32_t* __restrict__ a, int64_t rows,
                                                        int64_t prows, int64_t pcols,
                                                        uint8_t* __restrict__ flags, int64_t* __restrict__ degrees,
                                                        int64_t* __restrict__ zero_count) {
  const int lane = threadIdx.x & 31;
  const int64_t rt = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (rt >= (prows >> 3)) return;
  const int64_t ct = pcols >> 7, wpr = pcols >> 5;
  uint32_t deg[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) deg[i] = 0;
  int64_t zeros = 0;
  for (int64_t t = lane; t < ct; t += 32) {
    uint32_t any = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(a + (rt * 8 + i) * wpr + t * 4));
      any |= q.x | q.y | q.z | q.w;
      deg[i] += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
    }
    if (flags) flags[rt * ct + t] = any == 0;
    zeros += any == 0;
  }
  if (degrees) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t d = deg[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(QG_FULL, d, o);
      if (lane == 0 && rt * 8 + i < rows) degrees[rt * 8 + i] = d;
    }
  }
  if (zero_count) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) zeros += __shfl_xor_sync(QG_FULL, zeros, o);
    if (lane == 0 && zeros) atomicAdd(reinterpret_cast<unsigned long long*>(zero_count), (unsigned long long)zeros);
  }
}

// Zero-tile-jumping schedule: per 128-row block, the ordered list of K tiles
// with at least one set bit, derived from the 8x128 flags (16 flags per
// 128x128 block).  One warp per row block; lanes read consecutive flags.
__global__ void block_list_kernel(const uint8_t* __restrict__ flags, int64_t prows, int64_t pcols,
                                  int32_t* __restrict__ blk_list, int32_t* __restrict__ blk_count) {
  const int lane = threadIdx.x & 31;
  const int64_t rb = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nrb = (prows + 127) >> 7;
  if (rb >= nrb) return;
  const int64_t ct = pcols >> 7, rt = prows >> 3;
  const int64_t t_lo = rb * 16, t_hi = (rt < t_lo + 16 ? rt : t_lo + 16);
  int32_t count = 0;
  for (int64_t k0 = 0; k0 < ct; k0 += 32) {
    const int64_t k = k0 + lane;
    bool nz = false;
    if (k < ct) {
#pragma unroll 4
      for (int64_t t = t_lo; t < t_hi; ++t) nz |= flags[t * ct + k] == 0;
    }
    const uint32_t m = __ballot_sync(QG_FULL, nz);
    if (nz) blk_list[rb * ct + count + __popc(m & ((1u << lane) - 1u))] = (int32_t)k;
    count += __popc(m);
  }
  if (lane == 0) blk_count[rb] = count;
}

__global__ void plane_zero_tiles_kernel(const uint32_t* __restrict__ a, int64_t nplanes, int64_t prows,
                                        int64_t pcols, int64_t* __restrict__ zero_counts) {
  const int64_t rt_n = prows >> 3, ct = pcols >> 7, wpr = pcols >> 5;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nplanes * rt_n * ct) return;
  const int64_t p = idx / (rt_n * ct);
  const int64_t rem = idx % (rt_n * ct);
  const int64_t rt = rem / ct, t = rem % ct;
  const uint32_t* base = a + p * prows * wpr;
  uint32_t any = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(base + (rt * 8 + i) * wpr + t * 4));
    any |= q.x | q.y | q.z | q.w;
  }
  if (!any) atomicAdd(reinterpret_cast<unsigned long long*>(zero_counts + p), 1ull);
}

__global__ void status_reset_kernel(int64_t* s, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) s[i] = 0x7f7f7f7f7f7f7f7fLL;
}

__global__ void popcount_kernel(const uint32_t* __restrict__ in, int64_t n, int32_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __popc(in[i]);
}

__global__ void reduce_planes_kernel(const int64_t* __restrict__ accs, int64_t nplanes, int64_t n,
                                     int32_t* __restrict__ out, int32_t* overflow) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // exact int64 shift-sum (wraps only beyond 2^63, far outside any valid input)
  long long total = 0;
  for (int64_t p = 0; p < nplanes; ++p) total += (long long)((unsigned long long)accs[p * n + i] << p);
  if (total > 2147483647LL || total < -2147483648LL) {
    if (overflow) atomicExch(overflow, 1);
  }
  out[i] = (int32_t)total;
}

}  // namespace qg

// ======================================================================= ABI
using namespace qg;

static inline int launch_status() {
  return cudaGetLastError() == cudaSuccess ? QG_OK : QG_ERR_CUDA;
}
static inline bool bad_pad(int pad) { return pad != 8 && pad != 128; }
static inline int64_t pad_up(int64_t n, int64_t m) { return (n + m - 1) / m * m; }

// Per-epoch slab reset in ONE kernel: zero the accumulator slab, clear the status slab.
__global__ void slab_reset_kernel(int64_t* zero, int64_t nz, int64_t* status, int64_t ns) {
  // a PDL-launched successor (the epoch's entry conversion) may start launching now; it
  // waits for this grid's completion before touching any memory
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nz + ns; i += stride) {
    if (i < nz) zero[i] = 0;
    else status[i - nz] = 0x7f7f7f7f7f7f7f7fLL;
  }
}

extern "C" int qg_slab_reset(int64_t* zero, int64_t nzero, int64_t* status, int64_t nstatus, void* stream) {
  if (nzero < 0 || nstatus < 0 || (nzero && !zero) || (nstatus && !status)) return QG_ERR_ARG;
  const int64_t n = nzero + nstatus;
  if (n == 0) return QG_OK;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 1184);
  slab_reset_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(zero, nzero, status, nstatus);
  return launch_status();
}

extern "C" int qg_status_reset(int64_t* status, int64_t n, void* stream) {
  if (!status || n < 0) return QG_ERR_ARG;
  if (n == 0) return QG_OK;
  status_reset_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(status, n);
  return launch_status();
}

extern "C" int qg_quantize_pack(const void* src, int src_kind, int64_t rows, int64_t cols, int64_t ld,
                                double alpha_min, double scale, int bits, int orientation, int pad_to,
                                uint32_t* planes, uint8_t* codes, int64_t* row_sums, int64_t* col_sums,
                                int64_t* status, void* stream) {
  if (rows < 0 || cols < 0 || ld < cols || (rows * cols > 0 && !src) || !planes) return QG_ERR_ARG;
  if (bits < 1 || bits > 8) return QG_ERR_BITS;
  if (orientation != QG_COLUMN_WISE && orientation != QG_ROW_WISE) return QG_ERR_ARG;
  if (bad_pad(pad_to)) return QG_ERR_ARG;
  const int64_t prows = orientation == QG_COLUMN_WISE ? pad_up(rows, pad_to) : pad_up(rows, 128);
  const int64_t pcols = orientation == QG_COLUMN_WISE ? pad_up(cols, 128) : pad_up(cols, pad_to);
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  switch (src_kind) {
    case QG_SRC_F32:
      rc = dispatch_quantize_pack<float>((const float*)src, rows, cols, ld, alpha_min, scale, bits, orientation,
                                         prows, pcols, planes, codes, row_sums, col_sums, status, 0, st);
      break;
    case QG_SRC_F64:
      rc = dispatch_quantize_pack<double>((const double*)src, rows, cols, ld, alpha_min, scale, bits, orientation,
                                          prows, pcols, planes, codes, row_sums, col_sums, status, 0, st);
      break;
    case QG_SRC_U8:
      rc = dispatch_quantize_pack<uint8_t>((const uint8_t*)src, rows, cols, ld, alpha_min, scale, bits,
                                           orientation, prows, pcols, planes, codes, row_sums, col_sums, status, 0,
                                           st);
      break;
    default:
      return QG_ERR_ARG;
  }
  return rc != QG_OK ? rc : launch_status();
}

extern "C" int qg_pack_planes(const uint8_t* planes01, int64_t nplanes, int64_t rows, int64_t cols,
                              int orientation, int pad_to, uint32_t* words, int64_t* status, void* stream) {
  if (nplanes < 0 || rows < 0 || cols < 0 || !words || (nplanes * rows * cols > 0 && !planes01)) return QG_ERR_ARG;
  if (orientation != QG_COLUMN_WISE && orientation != QG_ROW_WISE) return QG_ERR_ARG;
  if (bad_pad(pad_to)) return QG_ERR_ARG;
  const int64_t prows = orientation == QG_COLUMN_WISE ? pad_up(rows, pad_to) : pad_up(rows, 128);
  const int64_t pcols = orientation == QG_COLUMN_WISE ? pad_up(cols, 128) : pad_up(cols, pad_to);
  const int64_t wpp = prows * pcols / 32;
  for (int64_t p = 0; p < nplanes; ++p) {
    int rc = launch_quantize_pack<uint8_t, 1>(planes01 + p * rows * cols, rows, cols, cols, 0.0, 1.0, orientation,
                                              prows, pcols, words + p * wpp, nullptr, nullptr, nullptr, status,
                                              p * rows * cols, (cudaStream_t)stream);
    if (rc != QG_OK) return rc;
  }
  return launch_status();
}

extern "C" int qg_unpack(const uint32_t* words, int64_t nplanes, int64_t rows, int64_t cols, int64_t padded_rows,
                         int64_t padded_cols, int orientation, uint8_t* out_planes, int32_t* out_codes,
                         void* stream) {
  if (nplanes < 1 || rows < 0 || cols < 0 || !words) return QG_ERR_ARG;
  if (padded_rows < rows || padded_cols < cols) return QG_ERR_SHAPE;
  const int64_t n = rows * cols;
  if (n == 0) return QG_OK;
  unpack_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      words, nplanes, rows, cols, padded_rows, padded_cols, orientation, out_planes, out_codes);
  return launch_status();
}

extern "C" int qg_repack(const uint32_t* src, int64_t nplanes, int64_t src_pr, int64_t src_pc, int src_orientation,
                         uint32_t* dst, int64_t dst_pr, int64_t dst_pc, void* stream) {
  if (!src || !dst || nplanes < 1) return QG_ERR_ARG;
  if (src_pr % 8 || src_pc % 8 || dst_pr % 8 || dst_pc % 8) return QG_ERR_SHAPE;
  const int64_t rg = (std::max(src_pr, dst_pr) + 31) / 32, cg = (std::max(src_pc, dst_pc) + 31) / 32;
  const int64_t warps = rg * cg * nplanes;
  if (warps == 0) return QG_OK;
  repack_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      src, nplanes, src_pr, src_pc, src_orientation, dst, dst_pr, dst_pc);
  return launch_status();
}

extern "C" int qg_tile_scan(const uint32_t* a_words, int64_t rows, int64_t padded_rows, int64_t padded_cols,
                            uint8_t* zero_flags, int64_t* degrees, int64_t* zero_count, int32_t* blk_list,
                            int32_t* blk_count, void* stream) {
  if (!a_words || padded_rows % 8 || padded_cols % 128 || rows > padded_rows) return QG_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rt = padded_rows / 8;
  if (rt > 0 && (zero_flags || degrees || zero_count))
    tile_scan_kernel<<<(unsigned)((rt * 32 + 255) / 256), 256, 0, st>>>(a_words, rows, padded_rows, padded_cols,
                                                                         zero_flags, degrees, zero_count);
  if (blk_list && blk_count) {
    if (!zero_flags) return QG_ERR_ARG;   // the schedule is derived from the 8x128 flags
    const int64_t nrb = (padded_rows + 127) / 128;
    if (nrb > 0)
      block_list_kernel<<<(unsigned)((nrb * 32 + 127) / 128), 128, 0, st>>>(zero_flags, padded_rows, padded_cols,
                                                                             blk_list, blk_count);
  }
  return launch_status();
}

extern "C" int qg_plane_zero_tiles(const uint32_t* words, int64_t nplanes, int64_t padded_rows,
                                   int64_t padded_cols, int64_t* zero_counts, void* stream) {
  if (!words || !zero_counts || padded_rows % 8 || padded_cols % 128) return QG_ERR_ARG;
  const int64_t n = nplanes * (padded_rows / 8) * (padded_cols / 128);
  if (n == 0) return QG_OK;
  plane_zero_tiles_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      words, nplanes, padded_rows, padded_cols, zero_counts);
  return launch_status();
}

extern "C" int qg_popcount32(const uint32_t* in, int64_t n, int32_t* out, void* stream) {
  if (n < 0 || (n && (!in || !out))) return QG_ERR_ARG;
  if (n == 0) return QG_OK;
  popcount_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(in, n, out);
  return launch_status();
}

extern "C" int qg_reduce_planes(const int64_t* accs, int64_t nplanes, int64_t n, int32_t* out, int32_t* overflow,
                                void* stream) {
  if (nplanes < 1 || nplanes > 62 || n < 0 || (n && (!accs || !out))) return QG_ERR_ARG;
  if (n == 0) return QG_OK;
  reduce_planes_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(accs, nplanes, n, out,
                                                                                      overflow);
  return launch_status();
}

namespace qg {
// One thread per edge: set bit (src, dst) in column-wise words (zero-initialised).
__global__ void edges_to_bits_kernel(const int64_t* __restrict__ src, const int64_t* __restrict__ dst, int64_t n_edges,
                                     int64_t rows, uint32_t* __restrict__ words, int64_t wpr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_edges) return;
  const int64_t r = src[i], c = dst[i];
  if (r < 0 || r >= rows || c < 0) return;
  atomicOr(words + r * wpr + (c >> 5), 1u << (c & 31));
}
}  // namespace qg

extern "C" int qg_edges_to_bits(const int64_t* src, const int64_t* dst, int64_t n_edges, int64_t rows,
                                uint32_t* words, int64_t padded_rows, int64_t padded_cols, void* stream) {
  if (!words || n_edges < 0 || (n_edges && (!src || !dst)) || padded_cols % 128 || rows > padded_rows)
    return QG_ERR_ARG;
  if (n_edges == 0) return QG_OK;
  qg::edges_to_bits_kernel<<<(unsigned)((n_edges + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      src, dst, n_edges, rows, words, padded_cols / 32);
  return cudaGetLastError() == cudaSuccess ? QG_OK : QG_ERR_CUDA;
}
