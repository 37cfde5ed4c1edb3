// Probe: cycles of the fused fp64 epilogue element chain (dequant -> bias -> requant) in isolation.
#include <cstdio>
#include <cstdint>
#include "../paper_2111_09547_b200/csrc/qgtc_common.cuh"
using namespace qg;
__global__ void k(const int* acc, const double* colv, int n_elem, long long* out, uint32_t* sink, int mode) {
  const int tid = threadIdx.x;
  const double k_acc = 0.0123, rterm = 1.5, k_const = -0.25, amin = -3.0, scale = 0.37, inv = 1.0 / 0.37;
  uint32_t s = 0;
  long long t0 = clock64();
  for (int e = 0; e < n_elem; e += 4) {
    double x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int a = acc[(tid * 131 + e + j) & 1023];
      double v = __dmul_rn(k_acc, (double)a);
      v = __dadd_rn(v, rterm);
      v = __dadd_rn(v, colv[(e + j) & 63]);
      v = __dadd_rn(v, k_const);
      x[j] = v;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t q;
      if (mode == 0) q = quantize_code_fast(x[j], amin, scale, inv, 15u);
      else if (mode == 1) q = quantize_code(x[j], amin, scale, 15u);
      else q = (uint32_t)x[j];
      s += q;
    }
  }
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + tid] = s;
  if (tid == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
  int* acc; double* colv; long long* d; uint32_t* sink;
  cudaMalloc(&acc, 4096); cudaMalloc(&colv, 512); cudaMalloc(&d, 8 * 148); cudaMalloc(&sink, 4 * 148 * 256);
  cudaMemset(acc, 1, 4096); cudaMemset(colv, 0, 512);
  for (int mode : {0, 1, 2}) {
    k<<<148, 256>>>(acc, colv, 16, d, sink, mode);
    k<<<148, 256>>>(acc, colv, 16, d, sink, mode);
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("mode=%d (0 markstein, 1 ieee div, 2 no div): %lld cycles for 16 elements/thread, 256 threads/SM\n", mode, h);
  }
}
