// Microbenchmark of the diagonal-tile factorization pieces (diagnostics).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2008_01541_b200/csrc potrf_bench.cu ...
#ifndef NOPROF
#define SPB_POTRF_PROF 1
#ifndef SPB_POTRF_PROF_T
#define SPB_POTRF_PROF_T 32
#endif
#endif
#include "../paper_2008_01541_b200/csrc/dense.cu"

namespace spb {
void set_error(const std::string&) {}
}
using namespace spb;

__global__ void __launch_bounds__(288, 1) k_potrf_bench(const double* A, double* L, double* LiT, int* info,
                                                       long long* cycles, int reps, const double* U) {
  extern __shared__ __align__(128) double smd[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 8) return;  // consumers only (named barrier 1 counts 256)
  const int wr = warp >> 2, wc = warp & 3;
  Acc acc;
  acc_foreach(wr, wc, lane, [&](int mb, int nb, int r, int c) {
    acc.c[mb][nb][0] = A[r * 64 + c];
    acc.c[mb][nb][1] = A[r * 64 + c + 1];
  });
  // the sub-diagonal tile sits in the shared scratch tile in the kernel
  double* Us = nullptr;
  if (U) {
    Us = smd + SM_SCR;
    for (int q = tid; q < TILE; q += 256) Us[q] = U[q];
  }
  cons_sync();
  long long t0 = clock64();
  const DensePeers nop{};
  for (int r = 0; r < reps; ++r)
    potrf_blocked_tile<false>(acc, smd, smd + 128 * LSP, L, LiT, 0, info, nullptr, wr, wc, lane, nop, Us);
  long long t1 = clock64();
  // diag16 alone
  for (int r = 0; r < reps; ++r) {
    if (warp == 0) potrf_diag16(smd, smd + 128 * LSP, 0, 0, info, lane);
    cons_sync();
  }
  long long t2 = clock64();
  for (int r = 0; r < reps; ++r) cons_sync();
  long long t3 = clock64();
  if (tid == 0) {
    cycles[0] = (t1 - t0) / reps;
    cycles[1] = (t2 - t1) / reps;
    cycles[2] = (t3 - t2) / reps;
  }
}

int main() {
  double hA[4096];
  for (int r = 0; r < 64; ++r)
    for (int c = 0; c < 64; ++c) hA[r * 64 + c] = (r == c ? 100.0 : 0.0) + 1.0 / (1.0 + r + c);
  double *A, *L, *LiT;
  int* info;
  long long* cyc;
  cudaMalloc(&A, 4096 * 8);
  cudaMalloc(&L, 4096 * 8);
  cudaMalloc(&LiT, 4096 * 8);
  cudaMalloc(&info, 4);
  cudaMalloc(&cyc, 3 * 8);
  cudaMemset(info, 0, 4);
  cudaMemcpy(A, hA, 4096 * 8, cudaMemcpyHostToDevice);
  size_t smem = cholesky_smem_bytes();
  cudaFuncSetAttribute(k_potrf_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // U (swizzled 64 x 64, the diagonal task's sub-diagonal tile): its rank-64
  // update A - U U^T runs in block 0 (POTRF_UPD=1) or is skipped
  double hU[4096];
  const bool with_u = getenv("POTRF_UPD") && getenv("POTRF_UPD")[0] == '1';
  for (int r = 0; r < 64; ++r)
    for (int c = 0; c < 64; ++c) hU[swz(r, c)] = 0.05 * ((r * 7 + c * 13) % 11 - 5) / 5.0;
  double* U;
  cudaMalloc(&U, 4096 * 8);
  cudaMemcpy(U, hU, 4096 * 8, cudaMemcpyHostToDevice);
  k_potrf_bench<<<1, 288, smem>>>(A, L, LiT, info, cyc, 20, with_u ? U : nullptr);
  cudaDeviceSynchronize();
  long long h[3];
  cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
  int hi;
  cudaMemcpy(&hi, info, 4, cudaMemcpyDeviceToHost);
  printf("err=%s info=%d potrf_blocked %lld cyc (%.2f us @1.9GHz), diag16 %lld cyc, cons_sync %lld cyc\n",
         cudaGetErrorString(cudaGetLastError()), hi, h[0], h[0] / 1900.0, h[1], h[2]);
#ifndef NOPROF
  long long prof[32];
  cudaMemcpyFromSymbol(prof, g_potrf_prof, sizeof(prof));
  // phases are cumulative clocks over 20 reps (+ the diag16-only loop does not mark)
  const char* names[15] = {"start", "init", "upd+d16_0", "pan_0", "upd+d16_1", "pan_1", "upd+d16_2", "pan_2",
                           "upd+d16_3", "pan_3", "", "", "", "", "store"};
  long long prev = prof[1];
  printf("  %-10s %8.0f cyc\n", "init", (prof[1] - prof[0]) / 20.0);
  for (int k = 2; k < 10; ++k) {
    printf("  %-10s %8.0f cyc\n", names[k], (prof[k] - prev) / 20.0);
    prev = prof[k];
  }
  printf("  %-10s %8.0f cyc\n", "store", (prof[14] - prev) / 20.0);
  // block 1, the profiled thread of warps 1-7 (from the block's start = mark 3 of block 0)
  printf("  block 1 thread %d: +%.0f to its branch, init_rows %.0f, store_cols %.0f, trailing update %.0f (warp 0 done at +%.0f; barrier at +%.0f)\n",
         SPB_POTRF_PROF_T, (prof[16] - prof[3]) / 20.0, (prof[17] - prof[16]) / 20.0, (prof[18] - prof[17]) / 20.0,
         (prof[19] - prof[18]) / 20.0, (prof[24] - prof[3]) / 20.0, (prof[4] - prof[3]) / 20.0);
#endif
  double hL[4096];
  cudaMemcpy(hL, L, 4096 * 8, cudaMemcpyDeviceToHost);
  // check L L^T == A - U U^T
  double err = 0;
  for (int r = 0; r < 64; ++r)
    for (int c = 0; c <= r; ++c) {
      double s = 0;
      for (int k = 0; k <= c; ++k) s += hL[swz(r, k)] * hL[swz(c, k)];
      double a = hA[r * 64 + c];
      if (with_u)
        for (int k = 0; k < 64; ++k) a -= hU[swz(r, k)] * hU[swz(c, k)];
      err = fmax(err, fabs(s - a));
    }
  // and L^-T: L^T (L^-T) = I
  double hLi[4096], erri = 0;
  cudaMemcpy(hLi, LiT, 4096 * 8, cudaMemcpyDeviceToHost);
  for (int r = 0; r < 64; ++r)
    for (int c = 0; c < 64; ++c) {
      double s = 0;
      for (int k = 0; k < 64; ++k) s += hL[swz(k, r)] * hLi[swz(k, c)];
      erri = fmax(erri, fabs(s - (r == c ? 1.0 : 0.0)));
    }
  printf("max |L^T L^-T - I| = %.3e\n", erri);
  printf("max |LL^T - A| = %.3e\n", err);
  return 0;
}
