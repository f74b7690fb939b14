#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
int main() {
  const size_t B = 3 * 128061 * 8;
  void *d, *ha, *hr;
  cudaMalloc(&d, B);
  cudaHostAlloc(&ha, B, cudaHostAllocDefault);
  hr = aligned_alloc(4096, (B + 4095) / 4096 * 4096);
  cudaHostRegister(hr, (B + 4095) / 4096 * 4096, cudaHostRegisterDefault);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[2] = {"hostalloc", "registered"};
  void* hs[2] = {ha, hr};
  for (int rep = 0; rep < 2; ++rep)
  for (int k = 0; k < 2; ++k) {
    for (int dir = 0; dir < 2; ++dir) {
      float best = 1e9;
      for (int i = 0; i < 20; ++i) {
        cudaEventRecord(e0, s);
        if (dir == 0) cudaMemcpyAsync(d, hs[k], B, cudaMemcpyHostToDevice, s);
        else cudaMemcpyAsync(hs[k], d, B, cudaMemcpyDeviceToHost, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("%s %s: %.1f us = %.1f GB/s\n", names[k], dir ? "D2H" : "H2D", best * 1e3, B / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
