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
  const int32_t* blk_list;
  const int32_t* blk_count;
  int32_t* out_i32;
  int32_t* overflow;
  qg_epilogue epi;
};

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

// Expand one 128-bit K slice of `nb` stacked planes (w[p] = 4 words) to 128
// code bytes and store them as the 8 K-cores of one UMMA row.
template <bool ZERO_ONE>
__device__ __forceinline__ void expand_store_row(const uint4* w, int nb, uint32_t row_base) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    uint32_t o[4];
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int sh = 4 * ((c & 1) * 4 + jj);
      uint32_t acc = 0;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        if (p < nb) {
          const uint32_t word = (c >> 1) == 0 ? w[p].x : (c >> 1) == 1 ? w[p].y : (c >> 1) == 2 ? w[p].z : w[p].w;
          const uint32_t e = expand_nibble((word >> sh) & 0xFu);
          acc |= ZERO_ONE ? e : (e << p);
        }
      }
      o[jj] = acc;
    }
    sts128(row_base + c * 128, o[0], o[1], o[2], o[3]);
  }
}

template <bool PER_PLANE, int TMEM_COLS>
__global__ void __launch_bounds__(128) tc_bitgemm_kernel(const __grid_constant__ GemmParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int bn = P.bn;
  const int64_t rb = blockIdx.x;
  const int nt = (int)blockIdx.y;
  uint8_t* sA = smem;                       // 2 x 16 KB
  uint8_t* sB = smem + 2 * 16384;           // 2 x bn*128 B
  const uint32_t sA0 = smem_u32(sA), sB0 = smem_u32(sB);
  const uint32_t bstage = (uint32_t)bn * 128u;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;

  const int nk = P.blk_count ? P.blk_count[rb] : P.k_tiles;
  const int32_t* klist = P.blk_list ? P.blk_list + rb * (int64_t)P.k_tiles : nullptr;
  const int64_t row = rb * 128 + tid;
  const int lb = P.lbits;
  const int rb_bits = PER_PLANE ? 1 : P.rbits;
  const uint32_t idesc = idesc_u8(bn);
  // per-thread R columns: tid, tid+128 (bn <= 256).  PER_PLANE: virtual column
  // v -> (plane v / vstride, column v % vstride) so one CTA can cover several planes.
  const uint32_t* rcol[2] = {nullptr, nullptr};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int t = tid + 128 * h;
    if (t >= bn) continue;
    const int64_t vc = (int64_t)nt * bn + t;
    int64_t col = vc, pl = 0;
    if (PER_PLANE) { pl = vc / P.vstride; col = vc % P.vstride; }
    if (pl < P.rbits && col < P.n_padded) rcol[h] = P.rhs + pl * P.rwpp + col * P.rwpr;
  }
  const bool has_c0 = tid < bn, has_c1 = tid + 128 < bn;

  for (int it = 0; it < nk; ++it) {
    const int st = it & 1;
    const int kt = klist ? klist[it] : it;
    uint4 wa[8], wb0[8], wb1[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      wa[p] = make_uint4(0, 0, 0, 0);
      wb0[p] = make_uint4(0, 0, 0, 0);
      wb1[p] = make_uint4(0, 0, 0, 0);
      if (p < lb && row < P.m_padded) wa[p] = ldg128(P.lhs + p * P.lwpp + row * P.lwpr + kt * 4);
      if (p < rb_bits) {
        if (rcol[0]) wb0[p] = ldg128(rcol[0] + p * P.rwpp + kt * 4);
        if (rcol[1]) wb1[p] = ldg128(rcol[1] + p * P.rwpp + kt * 4);
      }
    }
    if (it >= 2) mbar_wait(smem_u32(&mbar[st]), ((it - 2) >> 1) & 1);
    // A row tid -> group tid/8, row-in-core tid%8
    const uint32_t a_row = sA0 + st * 16384u + (uint32_t)((tid >> 3) * 1024 + (tid & 7) * 16);
    expand_store_row<false>(wa, lb, a_row);
    if (has_c0) {
      const uint32_t b_row = sB0 + st * bstage + (uint32_t)((tid >> 3) * 1024 + (tid & 7) * 16);
      if (PER_PLANE) expand_store_row<true>(wb0, 1, b_row); else expand_store_row<false>(wb0, rb_bits, b_row);
    }
    if (has_c1) {
      const int t1 = tid + 128;
      const uint32_t b_row = sB0 + st * bstage + (uint32_t)((t1 >> 3) * 1024 + (t1 & 7) * 16);
      if (PER_PLANE) expand_store_row<true>(wb1, 1, b_row); else expand_store_row<false>(wb1, rb_bits, b_row);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t da = umma_desc(sA0 + st * 16384u + kk * 256u);
        const uint64_t db = umma_desc(sB0 + st * bstage + kk * 256u);
        const uint32_t accum = (it > 0 || kk > 0) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(accum));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&mbar[st])) : "memory");
    }
  }
  if (nk > 0) {
    mbar_wait(smem_u32(&mbar[(nk - 1) & 1]), ((nk - 1) >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
  }

  // ---------------- epilogue: TMEM -> registers (lane = row) ----------------
  const int64_t r0 = rb * 128 + warp * 32;
  const int64_t myrow = r0 + lane;
  for (int c0 = 0; c0 < bn; c0 += 32) {
    uint32_t v[32];
    if (nk > 0) {
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
            "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
            "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = 0;
    }
    const int64_t cbase = (int64_t)nt * bn + c0;
    if (P.mode == QG_GEMM_EPILOGUE) {
      const int32_t* sv = reinterpret_cast<const int32_t*>(v);
      epi_chunk32<int32_t>(P.epi, r0, cbase, sv, P.m, P.n);
    } else if (myrow < P.m) {
      if (PER_PLANE) {
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
          const int64_t vc = cbase + j;
          const int64_t pl = vc / P.vstride, col = vc % P.vstride;
          if (pl < P.rbits && col < P.n) P.out_i32[(pl * P.m + myrow) * P.n + col] = (int32_t)v[j];
        }
      } else {
        int32_t* dst = P.out_i32 + myrow * P.n;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (cbase + j < P.n) dst[cbase + j] = (int32_t)v[j];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
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
  int32_t v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = (r < rows && c0 + j < cols) ? acc[r * cols + c0 + j] : 0;
  epi_chunk32<int32_t>(E, r0, c0, v, rows, cols);
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
  if (e->out_kind != QG_OUT_PLANES || !e->q_planes) return QG_ERR_ARG;
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
static int launch_tc(const GemmParams& P, dim3 grid, cudaStream_t st) {
  const size_t smem = 2 * 16384 + 2 * (size_t)P.bn * 128;
  const int cols = P.bn <= 32 ? 32 : P.bn <= 64 ? 64 : P.bn <= 128 ? 128 : 256;
  switch (cols) {
    case 32: set_smem_attr<PER_PLANE, 32>(smem); tc_bitgemm_kernel<PER_PLANE, 32><<<grid, 128, smem, st>>>(P); break;
    case 64: set_smem_attr<PER_PLANE, 64>(smem); tc_bitgemm_kernel<PER_PLANE, 64><<<grid, 128, smem, st>>>(P); break;
    case 128: set_smem_attr<PER_PLANE, 128>(smem); tc_bitgemm_kernel<PER_PLANE, 128><<<grid, 128, smem, st>>>(P); break;
    default: set_smem_attr<PER_PLANE, 256>(smem); tc_bitgemm_kernel<PER_PLANE, 256><<<grid, 128, smem, st>>>(P); break;
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
  P.out_i32 = a->out_i32; P.overflow = a->overflow;
  if (a->epi) P.epi = *a->epi;

  // the s32 tensor accumulator is exact iff the largest possible sum fits
  const double maxsum = (a->mode == QG_GEMM_PER_PLANE)
                            ? (double)a->k
                            : (double)((1 << a->lbits) - 1) * (double)((1 << a->rbits) - 1) * (double)a->k;
  int algo = a->algo;
  if (algo == QG_ALGO_AUTO) algo = maxsum < 2147483647.0 ? QG_ALGO_TCGEN05 : QG_ALGO_POPC;
  if (algo == QG_ALGO_TCGEN05 && maxsum >= 2147483647.0) return QG_ERR_UNSUPPORTED;

  if (algo == QG_ALGO_TCGEN05) {
    const int64_t row_blocks = (a->m_padded + 127) / 128;
    if (a->mode == QG_GEMM_PER_PLANE) {
      const int64_t n32 = (a->n_padded + 31) / 32 * 32;
      int64_t vtotal;
      if (a->cross_bit || n32 > 256) {
        // one plane per tile: stride rounded to a whole number of tiles
        P.bn = (int32_t)std::min<int64_t>(256, n32);
        P.vstride = (a->n_padded + P.bn - 1) / P.bn * P.bn;
        vtotal = P.vstride * a->rbits;
      } else {
        // planes stacked along N: each L tile is expanded once for several planes
        P.vstride = a->n_padded;
        vtotal = P.vstride * a->rbits;
        P.bn = (int32_t)std::min<int64_t>(256, (vtotal + 31) / 32 * 32);
      }
      P.n_tiles = (int32_t)((vtotal + P.bn - 1) / P.bn);
      dim3 grid((unsigned)row_blocks, (unsigned)P.n_tiles);
      return launch_tc<true>(P, grid, st);
    }
    const int64_t nround = (a->n_padded + 31) / 32 * 32;
    P.bn = (int32_t)std::min<int64_t>(256, nround);
    P.n_tiles = (int32_t)((a->n_padded + P.bn - 1) / P.bn);
    dim3 grid((unsigned)row_blocks, (unsigned)P.n_tiles);
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

extern "C" int qg_version(void) { return 13; }
