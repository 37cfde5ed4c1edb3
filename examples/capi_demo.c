/* Plain-C consumer of the C-ABI (include/qgtc_b200.h): what a non-Python host
 * binds.  Host-only part (always): library version + the OpCounters closed forms
 * of bmm_1bit_by_nbit / gemm_sbit_by_tbit.  With a GPU (argv[1] == "gpu"): bit_qnt
 * of a small fp32 matrix into row-wise bit planes through qg_quantize_pack, checked
 * against the scalar definition of quantize.py:93-105.
 *
 *   gcc -O2 -I include examples/capi_demo.c -L paper_2111_09547_b200/_lib -lqgtc_b200 \
 *       -L/usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,$PWD/paper_2111_09547_b200/_lib -o capi_demo
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "qgtc_b200.h"

/* the CUDA runtime calls the demo needs, declared here so the demo builds with gcc alone */
extern int cudaMalloc(void** p, size_t n);
extern int cudaFree(void* p);
extern int cudaMemcpy(void* dst, const void* src, size_t n, int kind);
extern int cudaDeviceSynchronize(void);

int main(int argc, char** argv) {
  printf("libqgtc_b200 exports %d entry points\n", qg_version());
  qg_counters c;
  /* 4 x 2 tiles of 8x128 bits, 3 of them all-zero, 4-bit X, 16 chunks of 8 columns */
  if (qg_bmm_counters(4, 2, 3, 4, 16, 1, 1, &c) != QG_OK) return 1;
  printf("bmm counters: mma=%lld fetch=%lld skipped=%lld words=%lld total=%lld\n", (long long)c.tile_mma_count,
         (long long)c.tile_fetch_count, (long long)c.tiles_skipped, (long long)c.word_and_popcount_count,
         (long long)c.tiles_total);
  if (c.tile_mma_count != 4 * 5 * 16 || c.tiles_skipped != 3 || c.word_and_popcount_count != 256 * 320) return 2;
  const int64_t zeros[2] = {1, 0};
  if (qg_gemm_counters(2, 2, zeros, 2, 3, 4, 1, 0, &c) != QG_OK) return 3;   /* cross-bit reuse */
  if (c.tile_mma_count != 3 * 7 * 4 || c.tile_fetch_count != 3 * 7 || c.tiles_total != 8) return 4;
  if (qg_bmm_counters(2, 2, 9, 1, 1, 1, 1, &c) != QG_ERR_ARG) return 5;   /* host-side validation */
  if (argc < 2 || strcmp(argv[1], "gpu") != 0) {
    printf("host-only checks OK\n");
    return 0;
  }
  /* bit_qnt on the device: 3 x 40 fp32, grid [0, 1) with 4 bits, row-wise planes, pad 8 */
  enum { R = 3, C = 40, BITS = 4 };
  float x[R * C];
  for (int i = 0; i < R * C; ++i) x[i] = (float)((i * 37) % 101) / 101.0f;
  const int64_t pr = 128, pc = 40;                     /* row-wise: rows -> pad 128, cols -> pad 8 */
  const int64_t words = pr * pc / 32;
  void *dx, *dplanes, *dstatus;
  int64_t status = 0x7f7f7f7f7f7f7f7fLL;
  if (cudaMalloc(&dx, sizeof x) || cudaMalloc(&dplanes, BITS * words * 4) || cudaMalloc(&dstatus, 8)) return 6;
  cudaMemcpy(dx, x, sizeof x, 1);
  cudaMemcpy(dstatus, &status, 8, 1);
  const double amin = 0.0, scale = 1.0 / (1 << BITS);
  if (qg_quantize_pack(dx, QG_SRC_F32, R, C, C, amin, scale, BITS, QG_ROW_WISE, 8, (uint32_t*)dplanes, NULL, NULL,
                       NULL, (int64_t*)dstatus, NULL) != QG_OK)
    return 7;
  cudaDeviceSynchronize();
  uint32_t* planes = (uint32_t*)malloc(BITS * words * 4);
  cudaMemcpy(planes, dplanes, BITS * words * 4, 2);
  int bad = 0;
  for (int r = 0; r < R; ++r)
    for (int col = 0; col < C; ++col) {
      const double q = floor(((double)x[r * C + col] - amin) / scale);
      const unsigned want = q < 0 ? 0u : (q > 15 ? 15u : (unsigned)q);
      unsigned got = 0;
      for (int p = 0; p < BITS; ++p) {    /* row-wise word (col, r / 32), bit r % 32 */
        const uint32_t w = planes[p * words + col * (pr / 32) + r / 32];
        got |= ((w >> (r % 32)) & 1u) << p;
      }
      bad += got != want;
    }
  printf("device bit_qnt: %s (%d mismatches)\n", bad ? "FAIL" : "OK", bad);
  free(planes);
  cudaFree(dx);
  cudaFree(dplanes);
  cudaFree(dstatus);
  return bad ? 8 : 0;
}
