// Which resource limits co-residency of the tiled GEMM kernels to 1 CTA/SM in the
// occupancy API / cooperative launches?  Variants: plain, +tcgen05.alloc, +griddepcontrol.
#include <cstdio>
#include <cstdint>
__global__ void k_plain(int* p) { extern __shared__ uint8_t s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
__global__ void k_tmem(int* p) {
  extern __shared__ uint8_t s[];
  __shared__ uint32_t base;
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((uint32_t)__cvta_generic_to_shared(&base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (p) p[threadIdx.x] = s[threadIdx.x] + base;
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(base));
}
__global__ void k_gdc(int* p) {
  extern __shared__ uint8_t s[];
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p) p[threadIdx.x] = s[threadIdx.x];
}
template <typename K>
void q(const char* name, K k, int smem) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int n = -1;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 256, smem);
  printf("%-8s smem=%6d occ=%d %s\n", name, smem, n, e == cudaSuccess ? "" : cudaGetErrorString(e));
}
int main() {
  for (int smem : {1024, 60 * 1024, 100 * 1024}) {
    q("plain", k_plain, smem);
    q("tmem", k_tmem, smem);
    q("gdc", k_gdc, smem);
  }
  return 0;
}
