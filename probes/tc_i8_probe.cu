// Probe: validate tcgen05.mma kind::i8 descriptor encodings (K-major, no swizzle)
// and tcgen05.ld 32x32b readback on sm_100a. Standalone; not part of the product.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  return d;                 // layout type 0 = SWIZZLE_NONE, base offset 0
}
__device__ __forceinline__ uint32_t make_idesc_i8(int M, int N, int a_signed, int b_signed) {
  uint32_t d = 0;
  d |= 2u << 4;                       // c_format S32
  d |= (uint32_t)a_signed << 7;       // a_format (0 = u8)
  d |= (uint32_t)b_signed << 10;      // b_format
  d |= (uint32_t)(N >> 3) << 17;
  d |= (uint32_t)(M >> 4) << 24;
  return d;
}

// A: M=128 rows x K bytes (row-major, K contiguous); B: N rows x K bytes (K contiguous).
// smem canonical K-major interleave: [group8][kcore][8 rows][16 B]
template <int N, int K>
__global__ void probe(const uint8_t* A, const uint8_t* B, int32_t* D, long long* cycles, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                       // 128*K
  uint8_t* sB = smem + 128 * K;             // N*K
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int KC = K / 16;  // k-cores
  for (int i = tid; i < 128 * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    sA[((r >> 3) * KC + (k >> 4)) * 128 + (r & 7) * 16 + (k & 15)] = A[i];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    sB[((r >> 3) * KC + (k >> 4)) * 128 + (r & 7) * 16 + (k & 15)] = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tbase = tmem_base;
  uint32_t idesc = make_idesc_i8(128, N, 0, 0);
  long long t0 = clock64();
  if (tid == 0) {
    for (int rep = 0; rep < reps; ++rep) {
      for (int kk = 0; kk < K / 32; ++kk) {
        uint64_t da = make_desc(smem_u32(sA) + kk * 256, 128, KC * 128);
        uint64_t db = make_desc(smem_u32(sB) + kk * 256, 128, KC * 128);
        uint32_t acc = (rep > 0 || kk > 0) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tbase), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  // wait phase 0
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  long long t1 = clock64();
  if (tid == 0) cycles[blockIdx.x] = t1 - t0;
  // read back: warp w lanes 32w.. ; 16 columns at a time
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    uint32_t taddr = tbase + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    int row = warp * 32 + lane;
    for (int j = 0; j < 16; ++j) D[(size_t)blockIdx.x * 128 * N + row * N + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(256));
}

template <int N, int K>
int run(int reps, int blocks) {
  std::vector<uint8_t> hA(128 * K), hB(N * K);
  srand(1);
  for (auto& x : hA) x = rand() & 0xFF;
  for (auto& x : hB) x = rand() & 0xFF;
  uint8_t *dA, *dB; int32_t* dD; long long* dc;
  cudaMalloc(&dA, hA.size()); cudaMalloc(&dB, hB.size());
  cudaMalloc(&dD, sizeof(int32_t) * 128 * N * blocks); cudaMalloc(&dc, sizeof(long long) * blocks);
  cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice);
  size_t smem = 128 * K + N * K + 1024;
  cudaFuncSetAttribute(probe<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  probe<N, K><<<blocks, 128, smem>>>(dA, dB, dD, dc, reps);
  cudaEventRecord(e0);
  probe<N, K><<<blocks, 128, smem>>>(dA, dB, dD, dc, reps);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("N=%d K=%d CUDA error %s\n", N, K, cudaGetErrorString(err)); return 1; }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<int32_t> hD(128 * N);
  cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
  long long cyc; cudaMemcpy(&cyc, dc, sizeof(cyc), cudaMemcpyDeviceToHost);
  long long bad = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < N; ++j) {
      long long ref = 0;
      for (int k = 0; k < K; ++k) ref += (long long)hA[i * K + k] * hB[j * K + k];
      ref *= reps;
      ref = (int32_t)(uint32_t)(ref & 0xFFFFFFFFLL);
      if (ref != hD[i * N + j]) { if (bad < 5) printf("  mismatch (%d,%d) got %d want %lld\n", i, j, hD[i * N + j], ref); ++bad; }
    }
  double macs = 128.0 * N * K * reps * blocks;
  printf("N=%d K=%d reps=%d blocks=%d: %s  cycles/blk=%lld  MAC/cyc/SM=%.1f  TOPS(int8 ops)=%.1f\n", N, K, reps, blocks,
         bad ? "FAIL" : "OK", cyc, 128.0 * N * K * reps / cyc, 2 * macs / (ms * 1e-3) / 1e12);
  cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
  return bad ? 1 : 0;
}

int main() {
  int rc = 0;
  rc |= run<64, 128>(1, 1);
  rc |= run<256, 128>(1, 1);
  rc |= run<16, 64>(1, 1);
  rc |= run<64, 128>(2000, 148);
  rc |= run<128, 128>(2000, 148);
  rc |= run<256, 128>(2000, 148);
  rc |= run<256, 128>(2000, 296);
  return rc;
}
