// Probe of the 5th-generation tensor core INT8 path on sm_100a:
// D[128 x 64] (s32, TMEM) = A[128 x K] (s8, smem, K-major) * B[64 x K]^T (s8, smem, K-major),
// K = 64 as two tcgen05.mma.kind::i8 instructions (K = 32 each), operands in the
// no-swizzle canonical K-major layout (8-row x 16-byte core matrices), result read
// back with tcgen05.ld.32x32b. Checked against a host product; then timed as a
// back-to-back stream of MMAs (int8 ops/s of one SM and of the whole GPU).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_i8_probe tools/umma_i8_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e = (x);                                                                  \
    if (e != cudaSuccess) {                                                               \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);     \
      exit(1);                                                                            \
    }                                                                                     \
  } while (0)

#ifndef PROBE_N
#define PROBE_N 64
#endif
constexpr int M = 128, N = PROBE_N, K = 64;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// byte offset of element (row r, k) in the canonical no-swizzle K-major layout
// of an R x 64 int8 operand: core matrix (r / 8, k / 16) of 8 x 16 bytes,
// k-chunks of a row group adjacent (LBO = 128 B), row groups 512 B apart (SBO)
__host__ __device__ __forceinline__ int kmaj_off(int r, int k) {
  return ((r >> 3) * 4 + (k >> 4)) * 128 + (r & 7) * 16 + (k & 15);
}

__device__ __forceinline__ uint64_t smem_desc(const void* base, int lbo, int sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(base) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
  return d;
}

__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4)      // D format S32
         | (1u << 7)    // A signed 8-bit
         | (1u << 10)   // B signed 8-bit
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, int acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

__global__ void k_probe(const int8_t* __restrict__ A, const int8_t* __restrict__ B, int* __restrict__ D, int reps,
                        long long* __restrict__ cycles) {
  __shared__ __align__(1024) int8_t sA[M * K];
  __shared__ __align__(1024) int8_t sB[N * K];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) unsigned long long mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < M * K; e += blockDim.x) sA[kmaj_off(e / K, e % K)] = A[e];
  for (int e = tid; e < N * K; e += blockDim.x) sB[kmaj_off(e / K, e % K)] = B[e];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(N < 32 ? 32 : N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> tensor core reads
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t dt = tmem_base;
  const uint32_t id = idesc_i8(M, N);
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int kk = 0; kk < K / 32; ++kk) {
        // K = 32 per instruction: the two 16-byte k-chunks kk*2, kk*2+1
        const uint64_t ad = smem_desc(sA + kk * 2 * 128, 128, 512);
        const uint64_t bd = smem_desc(sB + kk * 2 * 128, 128, 512);
        mma_i8(dt, ad, bd, id, (r > 0 || kk > 0) ? 1 : 0);
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&mbar))
                 : "memory");
  }
  // wait for the MMAs (phase 0)
  {
    unsigned done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&mbar))
          : "memory");
    }
  }
  if (tid == 0) {
    t1 = clock64();
    cycles[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: warp w (0..3) reads TMEM lanes 32w..32w+31 (rows), 64 columns
  if (warp < 4) {
    const int row = 32 * warp + lane;
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t v[8];
      const uint32_t addr = dt + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 8; ++j) D[row * N + c0 + j] = (int)v[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(dt), "n"(N < 32 ? 32 : N));
}

int main() {
  std::vector<int8_t> A(M * K), B(N * K);
  srand(7);
  for (auto& a : A) a = (int8_t)((rand() % 255) - 127);
  for (auto& b : B) b = (int8_t)((rand() % 255) - 127);
  int8_t *dA, *dB;
  int* dD;
  long long* dc;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dD, sizeof(int) * M * N));
  CK(cudaMalloc(&dc, sizeof(long long)));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  k_probe<<<1, 128>>>(dA, dB, dD, 1, dc);
  CK(cudaDeviceSynchronize());
  std::vector<int> D(M * N);
  CK(cudaMemcpy(D.data(), dD, sizeof(int) * M * N, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int ref = 0;
      for (int k = 0; k < K; ++k) ref += (int)A[i * K + k] * (int)B[j * K + k];
      if (ref != D[i * N + j]) {
        if (bad < 5) printf("mismatch (%d,%d): %d vs %d\n", i, j, D[i * N + j], ref);
        ++bad;
      }
    }
  printf("int8 tcgen05 128x%dx64: %s (%ld mismatches)\n", N, bad ? "FAIL" : "exact", bad);
  // throughput: reps x (2 MMAs of 128x64x32)
  const int reps = 4096;
  k_probe<<<1, 128>>>(dA, dB, dD, reps, dc);
  CK(cudaDeviceSynchronize());
  long long cyc;
  CK(cudaMemcpy(&cyc, dc, sizeof(cyc), cudaMemcpyDeviceToHost));
  const double macs = (double)reps * M * N * K;
  printf("one SM: %lld cycles for %d x 128x%dx64 -> %.0f int8 MAC/clk/SM (%.2f cycles per 128x%dx32 MMA)\n", cyc,
         reps, N, macs / cyc, (double)cyc / (2.0 * reps), N);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_probe<<<148, 128>>>(dA, dB, dD, reps, dc);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("148 SMs: %.3f ms -> %.1f int8 TOPS (2 ops per MAC)\n", ms, 2.0 * macs * 148 / (ms * 1e-3) / 1e12);
  return bad ? 1 : 0;
}
