// Probe: tcgen05.mma kind::i8 with A in TENSOR MEMORY ("TS" form) on sm_100a.
// A (128 x 128 u8) is written into TMEM by the threads with tcgen05.st.32x32b.x32
// (thread = row = TMEM lane, 32 columns of 4 bytes = K bytes 4c..4c+3, little endian);
// B (N x 128 u8) sits in shared memory in the UMMA K-major core layout.  The product is
// read back and checked against the host.  Standalone; not part of the product.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o ts_probe ts_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ uint32_t make_idesc_i8(int M, int N) {
  return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N>
__global__ void probe(const uint8_t* A, const uint8_t* B, int32_t* D, int mode) {
  constexpr int K = 128, KC = K / 16;
  __shared__ __align__(1024) uint8_t sB[N * K];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    sB[((r >> 3) * KC + (k >> 4)) * 128 + (r & 7) * 16 + (k & 15)] = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(256));
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
  const uint32_t tbase = tmem_base, acc_t = tbase, a_t = tbase + 128;
  // A row tid -> TMEM lane tid, 32 columns
  {
    uint32_t w[32];
    for (int c = 0; c < 32; ++c) {
      const uint8_t* p = A + tid * K + 4 * c;
      w[c] = mode == 0 ? (p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24))
                       : (p[3] | (p[2] << 8) | (p[1] << 16) | ((uint32_t)p[0] << 24));
    }
    const uint32_t taddr = a_t + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]),
        "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]),
        "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]),
        "r"(w[27]), "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t idesc = make_idesc_i8(128, N);
    for (int kk = 0; kk < K / 32; ++kk) {
      const uint64_t db = make_desc(smem_u32(sB) + kk * 256, 128, KC * 128);
      const uint32_t acc = kk > 0 ? 1u : 0u;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(acc_t),
                   "r"(a_t + (uint32_t)(kk * 8)), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = acc_t + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) D[tid * N + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(256));
}

int main() {
  constexpr int N = 64, K = 128;
  std::vector<uint8_t> hA(128 * K), hB(N * K);
  srand(7);
  for (auto& x : hA) x = rand() & 0xFF;
  for (auto& x : hB) x = rand() & 0xFF;
  uint8_t *dA, *dB;
  int32_t* dD;
  cudaMalloc(&dA, hA.size());
  cudaMalloc(&dB, hB.size());
  cudaMalloc(&dD, 4 * 128 * N);
  cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 2; ++mode) {
    probe<N><<<1, 128>>>(dA, dB, dD, mode);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(err)); return 1; }
    std::vector<int32_t> hD(128 * N);
    cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
    long long bad = 0;
    for (int i = 0; i < 128; ++i)
      for (int j = 0; j < N; ++j) {
        long long ref = 0;
        for (int k = 0; k < K; ++k) ref += (long long)hA[i * K + k] * hB[j * K + k];
        if (ref != hD[i * N + j]) {
          if (bad < 3) printf("  mode %d mismatch (%d,%d) got %d want %lld\n", mode, i, j, hD[i * N + j], ref);
          ++bad;
        }
      }
    printf("{\"ts_mode\": %d, \"layout\": \"%s\", \"mismatches\": %lld}\n", mode,
           mode == 0 ? "lane=row, column c = K bytes 4c..4c+3 little-endian" : "big-endian bytes", bad);
  }
  return 0;
}
