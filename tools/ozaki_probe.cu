// Probe of the emulated-FP64 tile product on the INT8 tensor cores
// (Ozaki-style splitting; the building block of an int8 tcgen05 path for the
// dense Cholesky's trailing updates):
//   C (64 x 64) = X (64 x K) * Y (64 x K)^T, FP64 in, FP64 out, K = 64 * nk.
// Every row r of X and Y carries a power-of-two scale 2^e_r >= max |row|; the
// scaled entries are split into 8 balanced base-2^7 digits (int8, |d| <= 64):
//   x = d1 / 2^6 + d2 / 2^13 + ... + d8 / 2^55  (+ |rest| <= 2^-56).
// Digit pairs (p, q) with p + q <= 9 (+ the even-p pairs of p + q = 10) are
// multiplied exactly on tcgen05.mma.kind::i8 into int32 TMEM accumulators,
// one per shift group: A = two stacked digit planes of X (M = 128), B = one
// digit plane of Y (N = 64), so lanes 0-63 of column block b hold the odd-p
// pairs of shift b and lanes 64-127 the even-p pairs of shift b + 1. The
// epilogue converts the 8 blocks to FP64 with exact power-of-two scales.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ozaki_probe tools/ozaki_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

#ifndef OZ_N
#define OZ_N 128
#endif
constexpr int TS = 64;
constexpr int NDIG = 8;
constexpr int PLANE = TS * TS;  // bytes per digit plane of a tile

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__host__ __device__ __forceinline__ int kmaj_off(int r, int k) {
  return ((r >> 3) * 4 + (k >> 4)) * 128 + (r & 7) * 16 + (k & 15);
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, int lbo, int sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, int acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

// digits of one tile (64 rows x 64 k) into 8 planes, canonical K-major layout
__global__ void k_slice(const double* __restrict__ X, int ldx, int nk, const int* __restrict__ e,
                        int8_t* __restrict__ out /* nk tiles x 8 planes x 4 KB */) {
  const int kt = blockIdx.x;
  for (int q = threadIdx.x; q < TS * TS; q += blockDim.x) {
    const int r = q / TS, c = q % TS;
    double x = ldexp(X[(size_t)r * ldx + kt * TS + c], -e[r]);
    int8_t* o = out + (size_t)kt * NDIG * PLANE + kmaj_off(r, c);
    double d = rint(x * 64.0);
    o[0] = (int8_t)d;
    x = x * 64.0 - d;
#pragma unroll
    for (int p = 1; p < NDIG; ++p) {
      x *= 128.0;
      d = rint(x);
      o[p * PLANE] = (int8_t)d;
      x -= d;
    }
  }
}

// one CTA: C = X Y^T over nk k-tiles; 256 threads (8 warps)
__global__ void __launch_bounds__(256, 1) k_ozaki_tile(const int8_t* __restrict__ xs, const int8_t* __restrict__ ys,
                                                     int nk, const int* __restrict__ ex, const int* __restrict__ ey,
                                                     double* __restrict__ C, long long* __restrict__ cyc) {
  extern __shared__ __align__(1024) int8_t sm[];
  int8_t* sA = sm;                       // 8 planes x 4 KB
  int8_t* sB = sm + NDIG * PLANE;        // 8 planes x 4 KB
  double* P = reinterpret_cast<double*>(sm + 2 * NDIG * PLANE);  // 64 x 64 staging
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) unsigned long long mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t dt = tmem_base;
  const uint32_t idesc = idesc_i8(128, OZ_N);
  long long t0 = clock64();
  unsigned phase = 0;
  for (int kt = 0; kt < nk; ++kt) {
    // stage the k-tile's digit planes (uint4 copies), then hand them to the tensor core
    const uint4* gx = reinterpret_cast<const uint4*>(xs + (size_t)kt * NDIG * PLANE);
    const uint4* gy = reinterpret_cast<const uint4*>(ys + (size_t)kt * NDIG * PLANE);
    uint4* ax = reinterpret_cast<uint4*>(sA);
    uint4* ay = reinterpret_cast<uint4*>(sB);
    for (int q = tid; q < NDIG * PLANE / 16; q += blockDim.x) {
      ax[q] = gx[q];
      ay[q] = gy[q];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid == 0) {
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
#if OZ_N == 64
#pragma unroll
      for (int h = 0; h < 4; ++h)
#pragma unroll
        for (int q = 1; q <= NDIG; ++q) {
          const int b = 2 * h + 1 + q;  // column block (shift group of the odd-p lanes)
          if (b > 9) continue;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const uint64_t ad = smem_desc(a0 + 2 * h * PLANE + kk * 256, 128, 512);
            const uint64_t bd = smem_desc(b0 + (q - 1) * PLANE + kk * 256, 128, 512);
            // every block b is first reached by (h = 0, q = b - 1): that MMA
            // (k-tile 0, kk = 0) overwrites the accumulator, the rest accumulate
            mma_i8(dt + (uint32_t)((b - 2) * 64), ad, bd, idesc, (kt == 0 && kk == 0 && h == 0) ? 0 : 1);
          }
        }
#else
      // N = 128: B = digit planes (q, q + 1), q odd; block b = 2h + 1 + q (even)
      // is 128 columns: quadrant (lanes 0-63 | 64-127) x (cols 0-63 | 64-127)
      // holds shift b | b + 1 / b + 1 | b + 2
#pragma unroll
      for (int h = 0; h < 4; ++h)
#pragma unroll
        for (int q = 1; q <= NDIG; q += 2) {
          const int b = 2 * h + 1 + q;
          if (b > 9) continue;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const uint64_t ad = smem_desc(a0 + 2 * h * PLANE + kk * 256, 128, 512);
            const uint64_t bd = smem_desc(b0 + (q - 1) * PLANE + kk * 256, 128, 512);
            mma_i8(dt + (uint32_t)((b - 2) / 2 * 128), ad, bd, idesc, (kt == 0 && kk == 0 && h == 0) ? 0 : 1);
          }
        }
#endif
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&mbar))
                   : "memory");
    }
    // wait for this k-tile's MMAs before the next staging overwrites sA / sB
    unsigned done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&mbar)), "r"(phase)
          : "memory");
    }
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  // ---- epilogue: warp (quarter qd = warp % 4, column half ch = warp / 4)
  const int qd = warp & 3, ch = warp >> 2;
  const int lrow = 32 * qd + lane;  // TMEM lane
  const int r = lrow & 63;
  double v[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) v[c] = 0.0;
  // Horner over the shift groups, largest weight first: block b carries
  // 2^-(7 t - 2) with t = b (lanes 0-63) or t = b + 1 (lanes 64-127)
#pragma unroll 1
  for (int blk = 0; blk < 8; ++blk) {
    uint32_t u[32];
#if OZ_N == 64
    const int b = blk + 2;
    const uint32_t addr = dt + ((uint32_t)(32 * qd) << 16) + (uint32_t)((b - 2) * 64 + 32 * ch);
#else
    // blk = 2 x (block) + column half: block b = 2 + 2 (blk / 2), cols (blk & 1) * 64 + 32 ch
    const int b = 2 + 2 * (blk >> 1) + (blk & 1);  // the lanes 0-63 shift of this column half
    const uint32_t addr = dt + ((uint32_t)(32 * qd) << 16) + (uint32_t)((blk >> 1) * 128 + (blk & 1) * 64 + 32 * ch);
#endif
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
          "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15]),
          "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]),
          "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int t = b + (qd >= 2 ? 1 : 0);
    const double w = ldexp(1.0, -(7 * t - 2));
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = fma((double)(int)u[c], w, v[c]);
  }
  if (qd < 2) {
#pragma unroll
    for (int c = 0; c < 32; ++c) P[r * TS + 32 * ch + c] = v[c];
  }
  __syncthreads();
  if (qd >= 2) {
#pragma unroll
    for (int c = 0; c < 32; ++c) P[r * TS + 32 * ch + c] += v[c];
  }
  __syncthreads();
  if (tid == 0) cyc[0] = clock64() - t0;
  for (int q = tid; q < TS * TS; q += blockDim.x) {
    const int rr = q / TS, cc = q % TS;
    C[q] = ldexp(P[q], ex[rr] + ey[cc]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(dt), "n"(512));
}

int main(int argc, char** argv) {
  const int nk = argc > 1 ? atoi(argv[1]) : 4;
  const int K = TS * nk;
  std::vector<double> X(TS * K), Y(TS * K);
  srand(11);
  auto rnd = [] { return (rand() / (double)RAND_MAX) * 2.0 - 1.0; };
  std::vector<int> ex(TS), ey(TS);
  for (int r = 0; r < TS; ++r) {
    const double sx = std::pow(10.0, 3.0 * rnd()), sy = std::pow(10.0, 3.0 * rnd());  // rows over 6 decades
    double mx = 0, my = 0;
    for (int k = 0; k < K; ++k) {
      X[r * K + k] = sx * rnd() * (k % 7 == 3 ? 1e-6 : 1.0);
      Y[r * K + k] = sy * rnd();
      mx = std::max(mx, std::fabs(X[r * K + k]));
      my = std::max(my, std::fabs(Y[r * K + k]));
    }
    ex[r] = (int)std::floor(std::log2(mx)) + 1;  // |x| / 2^e < 1
    ey[r] = (int)std::floor(std::log2(my)) + 1;
  }
  double *dX, *dY, *dC;
  int *dex, *dey;
  int8_t *xs, *ys;
  long long* dc;
  CK(cudaMalloc(&dX, 8 * X.size()));
  CK(cudaMalloc(&dY, 8 * Y.size()));
  CK(cudaMalloc(&dC, 8 * TS * TS));
  CK(cudaMalloc(&dex, 4 * TS));
  CK(cudaMalloc(&dey, 4 * TS));
  CK(cudaMalloc(&xs, (size_t)nk * NDIG * PLANE));
  CK(cudaMalloc(&ys, (size_t)nk * NDIG * PLANE));
  CK(cudaMalloc(&dc, 8));
  CK(cudaMemcpy(dX, X.data(), 8 * X.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dY, Y.data(), 8 * Y.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dex, ex.data(), 4 * TS, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dey, ey.data(), 4 * TS, cudaMemcpyHostToDevice));
  k_slice<<<nk, 256>>>(dX, K, nk, dex, xs);
  k_slice<<<nk, 256>>>(dY, K, nk, dey, ys);
  const size_t smem = 2 * NDIG * PLANE + 8 * TS * TS;
  CK(cudaFuncSetAttribute(k_ozaki_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_ozaki_tile<<<1, 256, smem>>>(xs, ys, nk, dex, dey, dC, dc);
  CK(cudaDeviceSynchronize());
  std::vector<double> C(TS * TS);
  CK(cudaMemcpy(C.data(), dC, 8 * TS * TS, cudaMemcpyDeviceToHost));
  long long cyc;
  CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
  // reference in long double, error relative to |x_r| |y_c| (the Ozaki bound) and to |C|
  double worst_norm = 0, worst_rel = 0, worst_fp64 = 0;
  for (int i = 0; i < TS; ++i)
    for (int j = 0; j < TS; ++j) {
      long double s = 0, a = 0;
      double f = 0;
      for (int k = 0; k < K; ++k) {
        s += (long double)X[i * K + k] * (long double)Y[j * K + k];
        a += std::fabs((long double)X[i * K + k] * (long double)Y[j * K + k]);
        f = std::fma(X[i * K + k], Y[j * K + k], f);
      }
      const double err = (double)std::fabs((long double)C[i * TS + j] - s);
      worst_norm = std::max(worst_norm, err / (double)a);
      worst_fp64 = std::max(worst_fp64, (double)std::fabs((long double)f - s) / (double)a);
      if (std::fabs((double)s) > 1e-3 * (double)a) worst_rel = std::max(worst_rel, err / std::fabs((double)s));
    }
  printf("K = %d: ozaki-int8 error / sum|x y| = %.3e (fp64 fma chain: %.3e), relative (well-conditioned entries) "
         "%.3e; %lld cycles (%.1f per k-tile)\n",
         K, worst_norm, worst_fp64, worst_rel, cyc, (double)cyc / nk);
  return worst_norm < 1e-14 ? 0 : 1;
}
