// Dependent-chain latencies on sm_100a (diagnostics): DFMA, DMUL, rsqrt/rcp
// approx f64, double shuffle, f32 rsqrt. One warp, clock64 around 1024 deps.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double seed) {
  double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0, t1;
  const int R = 1024;
#define TIME(idx, BODY)                                   \
  t0 = clock64();                                         \
  for (int i = 0; i < R; ++i) { BODY; }                   \
  t1 = clock64();                                         \
  if (threadIdx.x == 0) cyc[idx] = (t1 - t0) / R;
  TIME(0, x = fma(x, y, 1e-30))
  TIME(1, x = x * y)
  TIME(2, asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(x)); x = x * 0.25 + 1.0)
  TIME(3, asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x)); x = x * 0.25 + 1.0)
  TIME(4, x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31))
  TIME(5, { float f = (float)x; asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(f)); x = (double)f; })
  TIME(6, x = sqrt(x) + 1.0)
  TIME(7, x = 1.0 / x + 1.0)
  out[threadIdx.x] = x;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64 * 8);
  k<<<1, 32>>>(o, c, 1.5); cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
  const char* n[8] = {"dfma", "dmul", "rsqrt.approx.f64 + dfma", "rcp.approx.f64 + dfma", "shfl f64",
                      "cvt+rsqrt.f32+cvt", "sqrt.rn.f64 + dadd", "div.rn.f64 + dadd"};
  for (int i = 0; i < 8; ++i) printf("%-26s %lld cyc/iter\n", n[i], h[i]);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
