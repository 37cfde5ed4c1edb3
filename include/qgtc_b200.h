/*
 * qgtc_b200.h -- C-ABI of the B200-native QGTC hot path (sm_100a).
 *
 * The reference (`bitgnn`, /root/reference/pkg/src/bitgnn) is a pure
 * Python/numpy package with no FFI; its drop-in boundary is the Python API.
 * Each entry point below replaces the compute of one reference function
 * (cited as file:line); the Python mirror package `paper_2111_09547_b200`
 * binds them with ctypes and keeps the reference names, argument meaning and
 * exceptions.
 *
 * Conventions
 *  - All pointers are DEVICE pointers (caller-owned; no hidden allocation).
 *    `stream` is a cudaStream_t passed as void*; every call is stream-ordered
 *    and asynchronous.
 *  - Packed planes use the reference layouts verbatim (bitpack.py:3-14):
 *      column-wise: words[plane][padded_rows][padded_cols/32]
 *      row-wise:    words[plane][padded_cols][padded_rows/32]
 *    bit j of a word is element 32*w + j; every padding bit is zero.
 *  - Return value: QG_OK or a QG_ERR_* code for host-side argument errors
 *    (raised eagerly, before any launch, like the reference's ShapeError /
 *    ValueError).  Data-dependent conditions detected on the device
 *    (non-finite input, non-binary plane, int32 overflow) are reported
 *    through caller-provided device status words, read by the caller after
 *    the stream synchronises.
 *  - `status` words are int64 "first bad linear index" cells updated with
 *    atomicMin; initialise them with qg_status_reset (0x7f.. pattern).
 */
#ifndef QGTC_B200_H
#define QGTC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QG_OK 0
#define QG_ERR_ARG 1          /* null pointer / negative size / bad enum   */
#define QG_ERR_SHAPE 2        /* operand dims or orientations incompatible */
#define QG_ERR_BITS 3         /* bit width outside [1, 8]                   */
#define QG_ERR_CUDA 4         /* launch failure (cudaGetLastError)          */
#define QG_ERR_UNSUPPORTED 5  /* shape the selected algorithm cannot run    */

#define QG_COLUMN_WISE 0
#define QG_ROW_WISE 1

#define QG_SRC_F32 0
#define QG_SRC_F64 1
#define QG_SRC_U8 2           /* codes already quantized; validated < 2**bits */

#define QG_ACT_NONE 0
#define QG_ACT_RELU 1
#define QG_ACT_TANH 2

#define QG_OUT_REAL 0         /* fp64 matrix [rows][cols]                   */
#define QG_OUT_PLANES 1       /* requantized packed planes (+ row sums)     */

#define QG_GEMM_PER_PLANE 0   /* out_i32[p][rows][cols] = L(1-bit) . R_p     */
#define QG_GEMM_I32 1         /* out_i32[rows][cols] = sum (L_i . R_j) << (i+j) */
#define QG_GEMM_EPILOGUE 2    /* reduced accumulator -> fused epilogue      */

#define QG_ALGO_AUTO 0
#define QG_ALGO_TCGEN05 1     /* tcgen05.mma kind::i8, planes recomposed on chip */
#define QG_ALGO_POPC 2        /* CUDA-core AND+POPC over packed words (exact int64) */

/* Library identity / sanity: returns the number of exported compute entry points. */
int qg_version(void);

/* Reset `n` int64 status cells to "no error" (0x7f7f.. > any index). */
int qg_status_reset(int64_t* status, int64_t n, void* stream);

/* Per-forward reset of a runtime's slabs in one kernel: `zero` (nzero int64 words,
 * the atomic accumulators) := 0, `status` (nstatus cells) := the clear pattern. */
int qg_slab_reset(int64_t* zero, int64_t nzero, int64_t* status, int64_t nstatus, void* stream);

/*
 * Fused Eq.2 quantization + bit decomposition + packing (bit_qnt).
 * Replaces quantize_matrix (quantize.py:93-105) + bit_decompose
 * (quantize.py:108-112) + pack_planes (bitpack.py:213-228), and the row/column
 * code sums the engine derives from them (engine.py:150, 203, 280).
 *   src:        row-major rows x cols (leading dim ld) of f32/f64 reals, or u8 codes
 *   code = clip(floor((x - alpha_min) / scale), 0, 2**bits - 1), fp64, no FMA
 *   planes:     bits x words_per_plane output, fully written (padding = 0)
 *   codes:      optional u8 [rows][cols] copy of the codes (QuantMatrix.values)
 *   row_sums:   optional int64 [rows], ACCUMULATED (caller zeroes)
 *   col_sums:   optional int64 [cols], ACCUMULATED (caller zeroes)
 *   status:     first non-finite (f32/f64) or out-of-range (u8) index r*cols+c
 */
int qg_quantize_pack(const void* src, int src_kind, int64_t rows, int64_t cols, int64_t ld,
                     double alpha_min, double scale, int bits, int orientation, int pad_to,
                     uint32_t* planes, uint8_t* codes, int64_t* row_sums, int64_t* col_sums,
                     int64_t* status, void* stream);

/*
 * Pack `nplanes` logical 0/1 planes (u8 [nplanes][rows][cols]).  Replaces
 * pack_colwise / pack_rowwise / pack_planes (bitpack.py:169-228); status
 * receives the first non-binary index p*rows*cols + r*cols + c
 * (_as_binary, bitpack.py:153-160).
 */
int qg_pack_planes(const uint8_t* planes01, int64_t nplanes, int64_t rows, int64_t cols,
                   int orientation, int pad_to, uint32_t* words, int64_t* status, void* stream);

/*
 * Unpack to logical planes and/or codes.  Replaces unpack / to_planes
 * (bitpack.py:194-233) and to_val (quantize.py:115-129).
 *   out_planes: optional u8 [nplanes][rows][cols]
 *   out_codes:  optional int32 [rows][cols] = sum_p plane_p << p
 */
int qg_unpack(const uint32_t* words, int64_t nplanes, int64_t rows, int64_t cols,
              int64_t padded_rows, int64_t padded_cols, int orientation,
              uint8_t* out_planes, int32_t* out_codes, void* stream);

/*
 * Re-orient a stack through 32x32 warp bit transposes (no logical planes in
 * HBM).  Replaces repack (bitpack.py:236-238) and the engine's _oriented
 * (engine.py:173-176).  dst dims are the destination padded dims.
 */
int qg_repack(const uint32_t* src, int64_t nplanes, int64_t src_pr, int64_t src_pc,
              int src_orientation, uint32_t* dst, int64_t dst_pr, int64_t dst_pc, void* stream);

/*
 * Zero-tile scan of a column-wise 1-bit operand over 8x128 tiles plus
 * popcount row degrees.  Replaces scan_zero_tiles (bitgemm.py:214-233) and
 * SubgraphBatch.degrees (graph.py:292-295).
 *   zero_flags: optional u8 [pr/8][pc/128] (1 = all-zero tile)
 *   degrees:    optional int64 [rows]
 *   zero_count: optional int64 [1], ACCUMULATED (caller zeroes)
 *   blk_list / blk_count: optional (requires zero_flags) per-128-row-block lists of non-zero
 *     128-bit K tiles (the zero-tile-jumping schedule of the GEMM kernels):
 *     blk_list[rb * (pc/128) + i], i < blk_count[rb].
 */
int qg_tile_scan(const uint32_t* a_words, int64_t rows, int64_t padded_rows, int64_t padded_cols,
                 uint8_t* zero_flags, int64_t* degrees, int64_t* zero_count,
                 int32_t* blk_list, int32_t* blk_count, void* stream);

/* Per-plane zero 8x128 tile counts of a column-wise stack (GEMM counters,
 * bitgemm.py:426-427); zero_counts int64 [nplanes], ACCUMULATED. */
int qg_plane_zero_tiles(const uint32_t* words, int64_t nplanes, int64_t padded_rows,
                        int64_t padded_cols, int64_t* zero_counts, void* stream);

/* Fused epilogue parameters (EpilogueSpec, bitgemm.py:125-153; the
 * coefficients are the reference's fp64 term grouping, bitgemm.py:156-179,
 * precomputed on the host so the device evaluates the identical expression). */
typedef struct {
  int32_t act;                 /* QG_ACT_*                                        */
  int32_t use_row, use_col, use_const;
  double k_acc;                /* sa * sb                                         */
  double k_row;                /* sa * amb      (times lhs_row_sums[r])           */
  double k_col;                /* sb * ama      (times rhs_col_sums[c])           */
  double k_const;              /* (inner_dim * ama) * amb                         */
  const int64_t* row_sums;     /* [rows]                                          */
  const int64_t* col_sums;     /* [cols]                                          */
  const double* bias;          /* [cols] or NULL                                  */
  const double* bn_mean;       /* [cols] or NULL (all four or none)               */
  const double* bn_denom;      /* sqrt(var + eps), host-computed                  */
  const double* bn_gamma;
  const double* bn_beta;
  const double* bn_inv_denom;  /* RN(1 / bn_denom), host-computed (fast exact division) */
  double q_inv_scale;          /* RN(1 / q_scale), host-computed                       */
  int32_t out_kind;            /* QG_OUT_REAL / QG_OUT_PLANES                     */
  int32_t q_bits;              /* requant grid (quantize.py:93-105)               */
  double q_amin, q_scale;
  int32_t q_orientation;       /* QG_COLUMN_WISE / QG_ROW_WISE                    */
  int32_t pad_;
  int64_t q_prows, q_pcols;    /* padded dims of the output stack                 */
  double* out_real;            /* [rows][cols] for QG_OUT_REAL                    */
  uint32_t* q_planes;          /* q_bits x words; caller zero-fills               */
  int64_t* q_row_sums;         /* optional [rows], ACCUMULATED (caller zeroes)    */
  int64_t* status;             /* optional: first non-finite requant input index  */
  uint8_t* q_codes;            /* optional u8 code cache of the requantized output, the
                                  K-major operand layout of the next bit-GEMM:
                                  row-major [rows][ld] (next lhs) or col-major
                                  [cols][ld] (next rhs); padding must be zero      */
  int64_t q_codes_ld;
  int32_t q_codes_colmajor;
  int32_t q_skip_planes;       /* 1: write only the code cache (planes built lazily) */
  double screen_rmax;          /* tiled fast path: max code of the RIGHT operand (2^bits - 1)
                                  enables the fp32 requant screen (0 = exact fp64 path for
                                  every element); per-row acc bound = row_sums[r] * this   */
  double reserved_d1;          /* reserved, 0                                          */
} qg_epilogue;

/*
 * Stand-alone epilogue over an int32 accumulator [rows][cols].  Replaces
 * apply_epilogue (bitgemm.py:182-211).  The fused GEMM path evaluates the
 * same device function, so fused == unfused bit for bit.
 */
int qg_epilogue_apply(const int32_t* acc, int64_t rows, int64_t cols, const qg_epilogue* epi,
                      void* stream);

/* Any-bitwidth bit-GEMM arguments.  L is column-wise (M x K, lbits planes),
 * R is row-wise (K x N, rbits planes) with the same padded K. */
typedef struct {
  const uint32_t* lhs; int32_t lbits; int32_t pad0;
  int64_t m, m_padded;         /* logical / padded rows of L                      */
  int64_t k, k_padded;         /* logical / padded shared dim (k_padded % 128 == 0) */
  const uint32_t* rhs; int32_t rbits; int32_t pad1;
  int64_t n, n_padded;         /* logical / padded cols of R                      */
  const int32_t* blk_list;     /* optional zero-tile-jumping schedule (qg_tile_scan) */
  const int32_t* blk_count;
  int32_t mode;                /* QG_GEMM_*                                       */
  int32_t algo;                /* QG_ALGO_*                                       */
  int32_t* out_i32;            /* PER_PLANE: [rbits][m][n]; I32: [m][n]          */
  const qg_epilogue* epi;      /* EPILOGUE mode                                   */
  int32_t* overflow;           /* optional device flag, set to 1 on int32 overflow */
  int32_t* scratch_i32;        /* [m][n] scratch for the POPC epilogue path       */
  const uint8_t* lhs_codes;    /* optional: L as u8 codes [>= m][lhs_ld] (K contiguous,
                                  zero beyond k); used instead of the planes (TCGEN05) */
  int64_t lhs_ld;
  const uint8_t* rhs_codes;    /* optional: R as u8 codes [>= n][rhs_ld] (K contiguous) */
  int64_t rhs_ld;
  int64_t* phase_ns;           /* optional profiling hook: per CTA 6 %globaltimer stamps
                                  (entry, setup done, MMAs done, epilogue computed, stored, exit) */
  int32_t cross_bit;           /* PER_PLANE: 1 = one plane per CTA (cross-bit reuse),
                                  0 = planes stacked along N so each L tile is
                                  expanded once for all planes (cross-tile reuse) */
  int32_t pad2;
} qg_gemm_args;

/*
 * Bit-GEMM.  Replaces bmm_1bit_by_nbit (bitgemm.py:306-371; mode PER_PLANE),
 * gemm_sbit_by_tbit (bitgemm.py:374-475; modes I32 / EPILOGUE) and
 * reduce_bitplanes + apply_epilogue inside the engine (engine.py:235-317).
 * The TCGEN05 algorithm recomposes plane stacks into u8 codes in shared
 * memory (sum_p 2^p plane_p, exact) and runs tcgen05.mma kind::i8; it is
 * selected only when (2^lbits-1)(2^rbits-1)k < 2^31 so the s32 tensor
 * accumulator cannot wrap.  POPC is exact in int64 and flags overflow like
 * _narrow_int32 (bitgemm.py:282-288).
 */
int qg_bitgemm(const qg_gemm_args* args, void* stream);

/* ---- tiled fast path (engine) ------------------------------------------------
 * Operands in HBM in the UMMA K-major interleaved "tiled" layout: a left operand
 * (M x K) is stored as K slabs of 128, each [pad128(M)/8][8 K-cores][8 rows][16 B]
 * (a 128-row block of a slab is a contiguous 16 KB); a right operand (K x N) as K
 * slabs of [npad/8][8][8][16 B].  The 1-bit adjacency is stored as the array of
 * its non-zero 128x128 blocks expanded to 0/1 bytes (16 KB each), addressed by a
 * per-128-row-block schedule.  One segment = one subgraph batch; a launch covers
 * any number of segments (CTA -> segment, row block, N tile).                   */
typedef struct {
  const uint8_t* a;            /* left tiles: dense slabs, or adjacency blocks       */
  const uint8_t* b;            /* right tiles (slab pitch b_npad * 128)              */
  const int32_t* blk_count;    /* adjacency: non-zero K tiles per 128-row block      */
  const int32_t* blk_base;     /* adjacency: first block index of each row block     */
  const int32_t* blk_kt;       /* adjacency: K tile of each block                    */
  const int64_t* row_sums;     /* epilogue lhs row sums (degrees / code row sums)    */
  uint8_t* q_codes;            /* epilogue: tiled u8 code output                     */
  int64_t* q_row_sums;         /* epilogue: int64 row sums of the codes, ACCUMULATED */
  double* out_real;            /* fp64 logits [m][n]                                 */
  int32_t* out_i32;            /* int32 accumulator [m][n] (QG_GEMM_I32)             */
  int64_t* status;             /* first non-finite requant input index               */
  int64_t m;                   /* logical rows                                       */
  int64_t r128;                /* rows padded to 128 (left slab pitch / left output) */
  int64_t cta_begin;           /* first CTA of this segment                          */
  int32_t k_tiles;             /* dense left: K tiles                                */
  int32_t pad_;
  int64_t reserved0;           /* reserved, 0                                         */
  /* pair mode (qg_tiled_args.pair): 2-D TMA descriptors (CUtensorMap, 128 B, 64-B
   * aligned; qg_encode_linear_map) of the A source and the B source viewed as rows of
   * 128 bytes -- the pair's copies signal the leader CTA's mbarrier (cta_group::2) */
  uint8_t tmap_a[128];
  uint8_t tmap_b[128];
} qg_tseg;

/* Encode a 2-D TMA descriptor over a linear device buffer of `bytes` (multiple of 128)
 * viewed as rows of 128 bytes, box = box_rows rows (a contiguous box_rows*128-byte
 * copy).  Host-only; out = 128 bytes. */
int qg_encode_linear_map(const void* base, int64_t bytes, int32_t box_rows, void* out);

typedef struct {
  const qg_tseg* segs;         /* DEVICE array of segments (sorted by cta_begin)     */
  int32_t nsegs;
  int32_t a_blocks;            /* 1: left = adjacency blocks, 0: dense left slabs    */
  int64_t total_ctas;
  int64_t b_npad;              /* right operand padded N (multiple of bn)            */
  int64_t n;                   /* logical output columns                             */
  int32_t bn, n_tiles;         /* N tile (power of two 16..256) and tiles per row block */
  int32_t mode;                /* QG_GEMM_I32 or QG_GEMM_EPILOGUE                    */
  int32_t out_layout;          /* 0 row-major fp64/int32, 1 left-tiled codes, 2 right-tiled codes */
  int64_t out_npad;            /* right-tiled output: padded N                       */
  const qg_epilogue* epi;      /* shared epilogue scalars / per-column vectors       */
  int64_t* phase_ns;           /* optional [total_ctas][8] %globaltimer stamps (tools/) */
  int32_t a_bits;              /* a_blocks only: 1 = segs[].a holds PACKED blocks (2 KB:
                                  128 rows x 4 words, the column-wise bits of the block),
                                  expanded to the UMMA byte layout in shared memory;
                                  0 = pre-expanded 16 KB byte blocks                    */
  int32_t pair;                /* 1: CTA pairs (cluster of 2) with cta_group::2 MMAs, M = 256;
                                  segs[].cta_begin then counts PAIRS, total_ctas = 2 x pairs,
                                  bn >= 64 (each CTA stages bn/2 columns of B)             */
  const struct qg_chain* chain; /* optional: fuse a dense stage-2 GEMM behind this stage   */
  void* reserved1;             /* reserved, NULL (round-1 dataflow epoch, removed)       */
  void* reserved2;
  int32_t reserved3;
  int32_t pad3_;
} qg_tiled_args;

/* Chained stage 2 of a tiled GEMM (qg_tiled_args.chain): an aggregation and the update
 * that consumes its rows (engine.py:282-334: aggregate -> update inside a GCN layer, or
 * a GIN layer's aggregation -> the next layer's update) in one launch.  Stage 1
 * (n_tiles == 1; EPILOGUE mode, packed output) requantizes its tile into u8
 * codes that stay in shared memory as the LEFT operand of stage 2, whose right operand
 * is `w` (right-tiled, K = stage-1 n); stage 2's epilogue uses the code row sums of
 * that tile.  segs[].q_codes / q_row_sums / out_real / status are then stage 2's
 * outputs; stage 1's codes are never written to HBM. */
typedef struct qg_chain {
  const uint8_t* w;            /* right-tiled stage-2 operand (slab pitch w_npad * 128)  */
  int64_t w_npad;              /* padded N of w: power of two 32..256                    */
  int64_t n;                   /* stage-2 logical output columns (<= w_npad)             */
  int32_t out_layout;          /* 0 fp64 row-major, 2 right-tiled codes                  */
  int32_t reserved;            /* reserved, 0 (round-1 DSMEM split chain, removed)        */
  int64_t out_npad;            /* right-tiled output: padded N                           */
  const qg_epilogue* epi;      /* stage-2 epilogue                                       */
} qg_chain;

/* Warp-specialised tiled bit-GEMM (cp.async.bulk producer, single-thread
 * tcgen05.mma kind::i8 issuer, 8-warp fused epilogue).  Same arithmetic as
 * qg_bitgemm's EPILOGUE / I32 modes; replaces the per-batch loop of
 * engine.py:320-332 for a whole epoch layer stage. */
int qg_tiled_gemm(const qg_tiled_args* args, void* stream);

/* Gather the non-zero 128x128 blocks (blk_rb/blk_kt) of a column-wise 1-bit matrix
 * into `packed` (2 KB each; skipped when a_words == NULL and `packed` is already
 * filled, e.g. shipped by the QGT3 tile-sparse wire format), expand them to 16 KB
 * UMMA byte blocks (skipped when bytes == NULL: qg_tiled_gemm a_bits mode expands in
 * shared memory) and accumulate row degrees (graph.py:292-295; degrees zeroed). */
int qg_block_prepare(const uint32_t* a_words, int64_t rows, int64_t padded_rows, int64_t padded_cols,
                     const int32_t* blk_rb, const int32_t* blk_kt, int64_t nblocks, uint32_t* packed,
                     uint8_t* bytes, int64_t* degrees, void* stream);

/* qg_block_prepare over many batches in ONE launch (shipped blocks, no gather): the
 * per-epoch block expansion + degrees of the multi-batch end-to-end path. */
typedef struct {
  const uint32_t* packed;      /* [nblocks][128][4] packed blocks                     */
  const int32_t* blk_rb;       /* row block of each block                            */
  uint8_t* bytes;              /* 16 KB UMMA byte blocks out, or NULL (degrees only)  */
  int64_t* degrees;            /* [rows] ACCUMULATED (caller zeroes), or NULL         */
  int64_t rows;
  int64_t block_begin;         /* first global block index of this batch             */
} qg_block_seg;

int qg_block_prepare_grouped(const qg_block_seg* segs, int32_t nsegs, int64_t total_blocks, void* stream);

/* Plain row-major u8 codes [rows][ld] <-> left (right = 0, pitch = pad128(rows)) or
 * right (right = 1, pitch = npad) tiled layout. */
int qg_codes_to_tiles(const uint8_t* codes, int64_t rows, int64_t cols, int64_t ld, int right, int64_t pitch,
                      uint8_t* tiles, void* stream);
int qg_tiles_to_codes(const uint8_t* tiles, int64_t rows, int64_t cols, int right, int64_t pitch, uint8_t* codes,
                      int64_t ld, void* stream);

/* Grouped entry conversion (engine.py:164-176 _entry_state/_oriented + the code
 * recomposition sum_p 2^p plane_p, quantize.py:115-129): the ROW-WISE packed
 * feature planes of every batch -> u8 codes directly in the tiled operand layout
 * of the first GEMM, one launch for all batches.  right = 0: left-tiled M x K
 * (GIN update, X as rows x features; optional int64 row code sums, ZEROED by the
 * caller); right = 1: right-tiled K x N (GCN aggregation, pitch = padded N).
 * A work unit is 32 * words_per_unit rows (words_per_unit = 8 or 1: 32-byte plane loads
 * for large inputs, more units for small ones) x 128 columns; unit_begin = first unit of
 * the segment. */
typedef struct {
  const uint32_t* words;       /* (bits, pad128(rows)/32 * pc) row-wise plane words   */
  uint8_t* tiles;              /* tiled u8 output                                    */
  int64_t* row_sums;           /* left only: int64 row sums of the codes (or NULL)   */
  int64_t rows, cols;          /* logical                                            */
  int64_t pr, pc;              /* padded plane dims (pr = pad128(rows))              */
  int64_t pitch;               /* left: pad128(rows); right: padded N (>= cols)      */
  int64_t unit_begin;          /* first work unit of this segment                    */
} qg_entry_seg;

int qg_entry_tiles(const qg_entry_seg* segs, int32_t nsegs, int32_t nplanes, int32_t right,
                   int32_t words_per_unit, int64_t total_units, void* stream);

/* Shifted reduction sum_p acc[p] << p (int64 in) narrowed to int32 with an
 * overflow flag.  Replaces reduce_bitplanes (bitgemm.py:291-298). */
int qg_reduce_planes(const int64_t* accs, int64_t nplanes, int64_t n, int32_t* out,
                     int32_t* overflow, void* stream);

/* Packed planes -> u8 codes (sum_p bit_p << p) in a K-major operand layout:
 * row-major [rows][ld] or col-major [cols][ld].  Padding entries are not written.
 * row_sums (optional, row-major output of row-wise planes only): int64 [rows],
 * ACCUMULATED -- the left operand's row code sums (engine.py:280). */
int qg_planes_to_codes(const uint32_t* words, int64_t nplanes, int64_t rows, int64_t cols,
                       int64_t padded_rows, int64_t padded_cols, int orientation, uint8_t* codes,
                       int64_t ld, int colmajor, int64_t* row_sums, void* stream);

/* Set adjacency bits from an edge list into zero-initialised column-wise
 * words (row = src, col = dst).  Replaces the dense total x total build +
 * pack_colwise of build_batch (graph.py:334-342) without a dense matrix. */
int qg_edges_to_bits(const int64_t* src, const int64_t* dst, int64_t n_edges, int64_t rows,
                     uint32_t* words, int64_t padded_rows, int64_t padded_cols, void* stream);

/* Test hook: out[i] = a[i] / b[i] through the epilogue's division routine
 * (Markstein reciprocal sequence + IEEE fallback) and ref[i] through IEEE
 * __ddiv_rn, so tests can prove the fast path is correctly rounded. */
int qg_test_div(const double* a, const double* b, const double* inv_b, int64_t n, double* out, double* ref,
                void* stream);

/* Test hook: out[i] = the epilogue's requantization code of x[i] (filtered
 * reciprocal path) and ref[i] = clamp(floor(__ddiv_rn(x - amin, scale))), so
 * tests can prove the fast path bit-identical to quantize.py:102-104. */
int qg_test_requant(const double* x, int64_t n, double alpha_min, double scale, double inv_scale, int bits,
                    uint32_t* out, uint32_t* ref, void* stream);

/* popcount32 (bitgemm.py:58-60) on the device. */
int qg_popcount32(const uint32_t* in, int64_t n, int32_t* out, void* stream);

/* ---- reference-shaped entry points (SURVEY.md 8(b) export table) ---------------
 * qg_bmm_1xs: bmm_1bit_by_nbit (bitgemm.py:306-371) -- qg_bitgemm with lbits == 1
 *   (QG_ERR_BITS otherwise); mode PER_PLANE (the reference's per-plane list), I32
 *   (reduce_bitplanes fused) or EPILOGUE.
 * qg_gemm_sxt: gemm_sbit_by_tbit (bitgemm.py:374-475) -- qg_bitgemm, mode I32 or
 *   EPILOGUE (QG_ERR_ARG for PER_PLANE).
 * qg_batch_h2d: the single H2D of a packed compound buffer (pack_batch /
 *   unpack_batch, graph.py:374-431; QGT2/QGT3 images) from PINNED host memory,
 *   stream-ordered (capturable in a CUDA graph). */
int qg_bmm_1xs(const qg_gemm_args* args, void* stream);
int qg_gemm_sxt(const qg_gemm_args* args, void* stream);
int qg_batch_h2d(const void* pinned_src, int64_t nbytes, void* device_dst, void* stream);

/* OpCounters closed forms (bitgemm.py:72-100, 335-370, 409-461), host-only:
 *   bmm:  rt x ct 8x128 tiles of A, `zero_tiles` of them all-zero, s planes of X,
 *         n_chunks = padded N / 8;
 *   gemm: per plane i < s of X its zero tiles plane_zero_tiles[i], t planes of W.
 * jump = 0 counts every tile; cross_tile = 0 is the cross-bit reuse mode. */
typedef struct {
  int64_t tile_mma_count;
  int64_t tile_fetch_count;
  int64_t tiles_skipped;
  int64_t word_and_popcount_count;
  int64_t tiles_total;
} qg_counters;

int qg_bmm_counters(int64_t rt, int64_t ct, int64_t zero_tiles, int32_t s, int64_t n_chunks, int32_t jump,
                    int32_t cross_tile, qg_counters* out);
int qg_gemm_counters(int64_t rt, int64_t ct, const int64_t* plane_zero_tiles, int32_t s, int32_t t,
                     int64_t n_chunks, int32_t jump, int32_t cross_tile, qg_counters* out);

/*
 * Host partitioner (no device work).  Replaces partition() (graph.py:190-229, the
 * balanced BFS-grown greedy METIS stand-in): identical decisions for the same seed
 * (Python random.Random(seed).randrange reproduced).  Input: CSR of the undirected,
 * sorted, self-loop-free neighbour lists (Graph.neighbors, graph.py:73-81).
 * part_of: int64 [n], written.  QG_ERR_ARG unless 1 <= num_parts <= n.
 */
int qg_partition_bfs(int64_t n, const int64_t* indptr, const int64_t* nbrs, int64_t num_parts, int64_t seed,
                     int64_t* part_of);

#ifdef __cplusplus
}
#endif
#endif /* QGTC_B200_H */
