// Probe: cycles of the A-operand plane expansion (smem raw words -> UMMA layout) in isolation.
#include <cstdio>
#include <cstdint>
#include "../paper_2111_09547_b200/csrc/qgtc_common.cuh"
using namespace qg;
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d));
}
__device__ __forceinline__ uint32_t umma_off(int r, int c) { return (uint32_t)((r >> 3) * 1024 + c * 128 + (r & 7) * 16); }
__global__ void k(int lb, int iters, long long* out, int fence) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint32_t* raw = reinterpret_cast<uint32_t*>(smem + 32768);
  const int tid = threadIdx.x;
  for (int i = tid; i < lb * 512; i += blockDim.x) raw[i] = i * 2654435761u;
  __syncthreads();
  const uint32_t sA0 = smem_u32(smem);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int r = tid & 127, h = tid >> 7;
    uint32_t o[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0;
#pragma unroll 1
    for (int p = 0; p < lb; ++p) {
      const uint4 w4 = *reinterpret_cast<const uint4*>(raw + (p * 128 + r) * 4);
      const uint32_t wv[4] = {w4.x >> (16 * h), w4.y >> (16 * h), w4.z >> (16 * h), w4.w >> (16 * h)};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        o[i][0] |= expand_nibble(wv[i] & 0xFu) << p;
        o[i][1] |= expand_nibble((wv[i] >> 4) & 0xFu) << p;
        o[i][2] |= expand_nibble((wv[i] >> 8) & 0xFu) << p;
        o[i][3] |= expand_nibble((wv[i] >> 12) & 0xFu) << p;
      }
    }
    const uint32_t abase = sA0 + (it & 1) * 16384u;
#pragma unroll
    for (int i = 0; i < 4; ++i) sts128(abase + umma_off(r, h + 2 * i), o[i][0], o[i][1], o[i][2], o[i][3]);
    if (fence) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = (t1 - t0) / iters;
}
int main() {
  long long* d; cudaMalloc(&d, 8 * 148);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  for (int lb : {1, 4, 8})
    for (int fence : {0, 1}) {
      k<<<148, 256, 100000>>>(lb, 1000, d, fence);
      long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("lb=%d fence=%d: %lld cycles / iteration (256 threads)\n", lb, fence, h);
    }
}
