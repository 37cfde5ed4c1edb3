// Probe: 2-SM (cta_group::2) tcgen05.mma kind::i8, M=256 (128 rows per CTA), N=256
// (each CTA holds half of B), K=128, operands staged in shared memory by plain stores.
// Checks the pair's result against a CPU product and times repeated MMAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tc2_probe tc2_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t umma_off(int r, int c) { return (uint32_t)((r >> 3) * 1024 + c * 128 + (r & 7) * 16); }
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// A: [256][128] u8 row-major (rows = M), B: [256][128] u8 (row n = column n of the K x N operand)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) tc2_kernel(const uint8_t* A, const uint8_t* B,
                                                                             int32_t* D, int reps) {
  __shared__ __align__(1024) uint8_t sA[16384];
  __shared__ __align__(1024) uint8_t sB[16384];
  __shared__ __align__(8) uint64_t bar_done;
  __shared__ uint32_t tmem_base;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // this CTA's 128 rows of A and 128 columns (n) of B, in the UMMA K-major layout
  for (int u = tid; u < 128 * 8; u += 128) {
    const int r = u >> 3, c = u & 7;
    const uint4 a = *reinterpret_cast<const uint4*>(A + (size_t)(rank * 128 + r) * 128 + c * 16);
    const uint4 b = *reinterpret_cast<const uint4*>(B + (size_t)(rank * 128 + r) * 128 + c * 16);
    *reinterpret_cast<uint4*>(sA + umma_off(r, c)) = a;
    *reinterpret_cast<uint4*>(sB + umma_off(r, c)) = b;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_done)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  long long t0 = 0, t1 = 0;
  if (rank == 0 && tid == 0) {
    // S32 accumulate, u8 x u8, K-major; M = 256 (pair), N = 256
    const uint32_t idesc = (2u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t da = umma_desc(smem_u32(sA) + kk * 256), db = umma_desc(smem_u32(sB) + kk * 256);
        const uint32_t acc = (kk > 0) ? 1u : 0u;   // every rep recomputes the same product
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(&bar_done)), "h"((uint16_t)3) : "memory");
  }
  mbar_wait(smem_u32(&bar_done), 0);
  if (rank == 0 && tid == 0) {
    t1 = clock64();
    D[256 * 256] = (int32_t)(t1 - t0);
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: warp w reads TMEM lanes 32w..32w+31 = rows rank*128 + 32w + lane
  const int row = rank * 128 + warp * 32 + lane;
  for (int c0 = 0; c0 < 256; c0 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) D[(size_t)row * 256 + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 1;
  std::vector<uint8_t> A(256 * 128), B(256 * 128);
  srand(1);
  for (auto& x : A) x = rand() & 255;
  for (auto& x : B) x = rand() & 255;
  uint8_t *dA, *dB;
  int32_t* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, (256 * 256 + 1) * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, (256 * 256 + 1) * 4);
  tc2_kernel<<<2, 128>>>(dA, dB, dD, reps);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("launch error: %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<int32_t> D(256 * 256 + 1);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < 256; ++n) {
      long s = 0;
      for (int k = 0; k < 128; ++k) s += (long)A[m * 128 + k] * B[n * 128 + k];
      if (s != D[m * 256 + n]) {
        if (bad < 5) printf("mismatch m=%d n=%d got %d want %ld\n", m, n, D[m * 256 + n], s);
        ++bad;
      }
    }
  const double cyc = D[256 * 256];
  printf("cta_group::2 kind::i8 M=256 N=256 K=128: %s (%ld mismatches); reps=%d cycles=%.0f -> %.1f MAC/clk per SM\n",
         bad ? "FAIL" : "OK", bad, reps, cyc, cyc > 0 ? 256.0 * 256 * 128 * reps / cyc / 2 : 0.0);
  return bad ? 1 : 0;
}
