// Latency of the pieces of the 16-pivot warp kernel on sm_100a (diagnostics):
// dependent chains of DFMA, DMUL, MUFU.RCP64H / RSQ64H (+ refinement), a
// double shuffle (two 32-bit SHFL), and an STS -> __syncwarp -> LDS broadcast.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_fp64 tools/lat_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcp_approx(double x) {
  double y;
  asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double rsq_approx(double x) {
  double y;
  asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double shfl_f64(double v, int src) {
  const int lo = __shfl_sync(0xffffffffu, __double2loint(v), src);
  const int hi = __shfl_sync(0xffffffffu, __double2hiint(v), src);
  return __hiloint2double(hi, lo);
}

__global__ void k_lat(double seed, long long* out, double* sink) {
  __shared__ double buf[64];
  const int lane = threadIdx.x;
  const int N = 256;
  double x = seed + lane * 1e-3;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = fma(x, 0.999999, 1e-9);
  t1 = clock64();
  if (lane == 0) out[0] = (t1 - t0) / N;
  // DMUL chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = x * 1.0000001;
  t1 = clock64();
  if (lane == 0) out[1] = (t1 - t0) / N;
  // MUFU rcp chain (approx only)
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = rcp_approx(x + 1.0);
  t1 = clock64();
  if (lane == 0) out[2] = (t1 - t0) / N;
  // rcp + cubic correction chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) {
    const double a = x + 1.0;
    double y = rcp_approx(a);
    const double e = fma(-a, y, 1.0);
    const double t = fma(e, e, e);
    x = fma(y, t, y);
  }
  t1 = clock64();
  if (lane == 0) out[3] = (t1 - t0) / N;
  // rsqrt approx chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = rsq_approx(x + 1.0);
  t1 = clock64();
  if (lane == 0) out[4] = (t1 - t0) / N;
  // double shuffle chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = shfl_f64(x, (lane + 1) & 31) + 1e-9;
  t1 = clock64();
  if (lane == 0) out[5] = (t1 - t0) / N;
  // STS -> syncwarp -> LDS broadcast chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) {
    if (lane == (i & 15)) buf[i & 31] = x;
    __syncwarp();
    x = buf[i & 31] + 1e-9;
    __syncwarp();
  }
  t1 = clock64();
  if (lane == 0) out[6] = (t1 - t0) / N;
  // 2 x 32-bit shuffles issued back to back, single 32-bit chain
  int ix = __double2loint(x);
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) ix = __shfl_sync(0xffffffffu, ix, (lane + 1) & 31) + 1;
  t1 = clock64();
  if (lane == 0) out[7] = (t1 - t0) / N;
  sink[lane] = x + ix;
}

int main() {
  long long* d;
  double* s;
  cudaMalloc(&d, 8 * 8);
  cudaMalloc(&s, 32 * 8);
  k_lat<<<1, 32>>>(1.5, d, s);
  cudaDeviceSynchronize();
  long long h[8];
  cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  const char* n[8] = {"DFMA", "DMUL", "MUFU rcp64h", "rcp + 3 DFMA", "MUFU rsq64h", "shfl f64 (2x32)+DADD",
                      "STS/syncwarp/LDS+DADD", "shfl 32 + IADD"};
  for (int i = 0; i < 8; ++i) printf("%-24s %lld cycles (loop-carried)\n", n[i], h[i]);
  return 0;
}
