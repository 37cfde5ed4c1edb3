// Pipe-choice microbenchmarks for the bit-GEMM (north star item 2), sm_100a.
// Standalone; not part of the product.  Each kernel runs a register-resident inner
// loop long enough that launch overhead is negligible and reports the sustained
// rate in 1-bit MACs per second (one AND+POPC over a 32-bit word = 32 bit-MACs; one
// mma.sync m16n8k256 b1 = 16*8*256 bit-MACs):
//   popc   : CUDA-core AND + POPC + IADD over 32-bit words (the reference's kernel,
//            bitgemm.py:48-60 / 236-253, on the SIMT pipes)
//   mma_b1 : warp-level mma.sync.m16n8k256.row.col.s32.b1.b1.s32.and.popc
// The tcgen05 kind::i8 rate is probes/tc_i8_probe.cu (profiles/int8_peak.json): one
// u8 x u8 MAC there retires all s x t bit-plane pairs of an s-bit x t-bit product.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pipe_probe pipe_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s\n", cudaGetErrorString(e)); return 1; } } while (0)

// 8x8 register tile of word pairs per thread: 64 AND+POPC+ADD per k step
__global__ void popc_kernel(const uint32_t* seed, int iters, uint32_t* out) {
  uint32_t a[8], b[8], acc[8][8];
  const uint32_t s = seed[threadIdx.x & 31] ^ (blockIdx.x * 0x9E3779B9u);
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = s * (i + 1) + 0x1234567u * i; b[i] = s ^ (0xABCDEF01u * (i + 3)); }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] += __popc(a[i] & b[j]);
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = __funnelshift_l(a[i], a[i], 1); b[i] += 0x9E3779B9u; }
  }
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) r ^= acc[i][j];
  if (r == 0x12345678u) out[blockIdx.x] = r;
}

// 4 independent m16n8k256 b1 MMAs per step (4 accumulator sets)
__global__ void mma_b1_kernel(const uint32_t* seed, int iters, uint32_t* out) {
  uint32_t a[4], b[2];
  int32_t c[4][4];
  const uint32_t s = seed[threadIdx.x & 31] ^ blockIdx.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = s * (2 * i + 1);
  b[0] = s ^ 0x55555555u;
  b[1] = s ^ 0x33333333u;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[q][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile(
          "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+r"(c[q][0]), "+r"(c[q][1]), "+r"(c[q][2]), "+r"(c[q][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  int32_t r = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int i = 0; i < 4; ++i) r ^= c[q][i];
  if (r == 0x12345678) out[blockIdx.x] = (uint32_t)r;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  uint32_t* seed;
  uint32_t* out;
  CK(cudaMalloc(&seed, 32 * 4));
  CK(cudaMalloc(&out, 1 << 20));
  uint32_t hs[32];
  for (int i = 0; i < 32; ++i) hs[i] = 0x9E3779B9u * (i + 7);
  CK(cudaMemcpy(seed, hs, sizeof(hs), cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  // popc: 64 AND+POPC per thread per iteration, 32 bit-MACs each
  {
    const int iters = 20000;
    popc_kernel<<<blocks, threads>>>(seed, 100, out);
    cudaEventRecord(e0);
    popc_kernel<<<blocks, threads>>>(seed, iters, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bitmacs = (double)blocks * threads * iters * 64.0 * 32.0;
    printf(", \"popc_ms\": %.3f, \"popc_bit_tmacs\": %.2f", ms, bitmacs / (ms * 1e-3) / 1e12);
  }
  // mma.sync b1: per warp per iteration 4 x 16*8*256 bit-MACs
  {
    const int iters = 20000;
    mma_b1_kernel<<<blocks, threads>>>(seed, 100, out);
    cudaEventRecord(e0);
    mma_b1_kernel<<<blocks, threads>>>(seed, iters, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bitmacs = (double)blocks * (threads / 32) * iters * 4.0 * 16 * 8 * 256;
    printf(", \"mma_b1_ms\": %.3f, \"mma_b1_bit_tmacs\": %.2f", ms, bitmacs / (ms * 1e-3) / 1e12);
  }
  printf("}\n");
  return 0;
}
