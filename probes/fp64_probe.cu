// Probe: per-SM throughput of DFMA, DADD, I2F.F64, F2I.F64, FFMA on this GPU.
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void k(double* outd, float* outf, long long* cyc, int iters) {
  double a[8]; float f[8]; int ii[8];
  for (int j = 0; j < 8; ++j) { a[j] = 1.0 + threadIdx.x * 1e-3 + j; f[j] = 1.0f + j; ii[j] = threadIdx.x + j; }
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) a[j] = fma(a[j], 1.0000001, 1e-9);
      if (MODE == 1) a[j] = a[j] + 1e-9;
      if (MODE == 2) { a[j] += (double)ii[j]; ii[j] += 1; }
      if (MODE == 3) { ii[j] += (int)a[j]; a[j] += 0.5; }
      if (MODE == 4) f[j] = fmaf(f[j], 1.0000001f, 1e-9f);
    }
  }
  long long t1 = clock64();
  double s = 0; float sf = 0;
  for (int j = 0; j < 8; ++j) { s += a[j] + ii[j]; sf += f[j]; }
  outd[blockIdx.x * blockDim.x + threadIdx.x] = s; outf[blockIdx.x * blockDim.x + threadIdx.x] = sf;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* d; float* f; long long* c;
  cudaMalloc(&d, 8 * 148 * 1024); cudaMalloc(&f, 4 * 148 * 1024); cudaMalloc(&c, 8 * 148);
  const int iters = 4096, threads = 1024;
  const char* names[] = {"DFMA", "DADD", "I2F.F64+DADD", "F2I.F64+DADD", "FFMA"};
  for (int m = 0; m < 5; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) k<0><<<148, threads>>>(d, f, c, iters);
      if (m == 1) k<1><<<148, threads>>>(d, f, c, iters);
      if (m == 2) k<2><<<148, threads>>>(d, f, c, iters);
      if (m == 3) k<3><<<148, threads>>>(d, f, c, iters);
      if (m == 4) k<4><<<148, threads>>>(d, f, c, iters);
    }
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double ops = (double)iters * 8 * threads;
    printf("%-14s %.2f ops/clk/SM\n", names[m], ops / h);
  }
}
