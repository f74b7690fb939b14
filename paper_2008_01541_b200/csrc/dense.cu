// Dense FP64 Schur-complement kernels (the inner-loop system of Algorithm 1,
// PAPER.md:402-441; reference linalg.py:432-461 + solver.py:430-440).
//
//   k_cholesky_tiles   H = sigma0 + C22 assembled on the fly and factored
//                      LL^T in ONE persistent launch: left-looking 64x64 tile
//                      tasks claimed in dependency order, per-tile readiness
//                      flags (acquire/release), trailing products on the FP64
//                      tensor pipe (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4;
//                      tcgen05 has no f64 kind). The RHS g rides along as an
//                      extra tile ROW of the matrix, so the forward
//                      substitution y = L^-1 g is produced by the same tasks.
//   k_dense_backward   u = L^-T y, one CTA per tile column, flag chained.
//   k_sym_gemv_*       sigma0 u (symmetric, lower tiles read once) for the
//                      f~2 maintenance and the residual (solver.py:436-440).
//
// Layout: tile (i,j), i >= j, at index i(i+1)/2 + j, 64x64 row-major. The
// order m is padded to 64 N with an identity tail.
#include "common.cuh"
#include "kernels.cuh"

namespace spb {

constexpr int TS = 64;     // tile size
constexpr int LDS = 68;    // padded smem row (8-byte bank slots (4g+t) mod 16 distinct)
constexpr int TILE_SMEM = TS * LDS;

__host__ __device__ __forceinline__ int tidx(int i, int j) { return i * (i + 1) / 2 + j; }
int dense_tile_count(int N) { return N * (N + 1) / 2; }
size_t cholesky_smem_bytes() { return sizeof(double) * (4 * TILE_SMEM + 2 * TS) + 16; }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// global tile (row-major 64x64) -> smem tile (row stride LDS), 256 threads
__device__ __forceinline__ void load_tile_async(double* s, const double* g) {
  for (int q = threadIdx.x; q < TS * TS / 2; q += blockDim.x) {
    int r = q >> 5, c2 = (q & 31) * 2;
    cp_async16(s + r * LDS + c2, g + r * TS + c2);
  }
}

__device__ __forceinline__ void wait_flag(const int* f) {
  if (threadIdx.x == 0) {
    while (ld_acquire(f) == 0) __nanosleep(64);
  }
  __syncthreads();
}

// Warp tile: 32 rows x 16 cols; 8 warps cover 64x64 as 2 (rows) x 4 (cols).
struct Acc {
  double c[4][2][2];
};

__device__ __forceinline__ void acc_zero(Acc& a) {
#pragma unroll
  for (int mb = 0; mb < 4; ++mb)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) a.c[mb][nb][0] = a.c[mb][nb][1] = 0.0;
}

// acc += sign * A * B^T over K = 64, A and B row-major 64x64 smem tiles.
template <bool NEG>
__device__ __forceinline__ void tile_gemm_abt(Acc& acc, const double* sA, const double* sB, int wr, int wc,
                                              int lane) {
  const int g = lane >> 2, t = lane & 3;
  const double* pa = sA + (wr * 32 + g) * LDS + t;
  const double* pb = sB + (wc * 16 + g) * LDS + t;
#pragma unroll 4
  for (int kk = 0; kk < TS; kk += 4) {
    double a[4], b[2];
#pragma unroll
    for (int mb = 0; mb < 4; ++mb) a[mb] = NEG ? -pa[mb * 8 * LDS + kk] : pa[mb * 8 * LDS + kk];
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) b[nb] = pb[nb * 8 * LDS + kk];
#pragma unroll
    for (int mb = 0; mb < 4; ++mb)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) dmma(acc.c[mb][nb][0], acc.c[mb][nb][1], a[mb], b[nb]);
  }
}

// fragment <-> smem tile (row stride LDS)
__device__ __forceinline__ void acc_to_smem(const Acc& acc, double* s, int wr, int wc, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mb = 0; mb < 4; ++mb)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      int r = wr * 32 + mb * 8 + g, c = wc * 16 + nb * 8 + 2 * t;
      s[r * LDS + c] = acc.c[mb][nb][0];
      s[r * LDS + c + 1] = acc.c[mb][nb][1];
    }
}
__device__ __forceinline__ void smem_to_acc(Acc& acc, const double* s, int wr, int wc, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mb = 0; mb < 4; ++mb)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      int r = wr * 32 + mb * 8 + g, c = wc * 16 + nb * 8 + 2 * t;
      acc.c[mb][nb][0] = s[r * LDS + c];
      acc.c[mb][nb][1] = s[r * LDS + c + 1];
    }
}
__device__ __forceinline__ void acc_to_global(const Acc& acc, double* gt, int wr, int wc, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mb = 0; mb < 4; ++mb)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      int r = wr * 32 + mb * 8 + g, c = wc * 16 + nb * 8 + 2 * t;
      *reinterpret_cast<double2*>(gt + r * TS + c) = make_double2(acc.c[mb][nb][0], acc.c[mb][nb][1]);
    }
}

// In-smem Cholesky of a 64x64 SPD tile (lower), then its triangular inverse.
// Writes L (strict upper zeroed) and inv(L) to global. Returns via *info the
// 1-based global column of the first non-positive pivot (dpotrf semantics).
__device__ void potrf_inv_tile(double* S, double* col, double* gL, double* gLinv, int j, int* info) {
  const int tid = threadIdx.x;
  for (int k = 0; k < TS; ++k) {
    double d = S[k * LDS + k];
    if (!(d > 0.0)) {
      if (tid == 0) atomicCAS(info, 0, j * TS + k + 1);
    }
    double dk = sqrt(d);
    if (tid > k && tid < TS) {
      double l = S[tid * LDS + k] / dk;
      col[tid] = l;
      S[tid * LDS + k] = l;
    }
    __syncthreads();
    if (tid == 0) S[k * LDS + k] = dk;
    // trailing update of rows/cols > k (lower part)
    const int rem = TS - 1 - k;
    for (int q = tid; q < rem * rem; q += blockDim.x) {
      int r = k + 1 + q / rem, c = k + 1 + q % rem;
      if (c <= r) S[r * LDS + c] -= col[r] * col[c];
    }
    __syncthreads();
  }
  // write L (zero strict upper)
  for (int q = tid; q < TS * TS; q += blockDim.x) {
    int r = q >> 6, c = q & 63;
    gL[q] = (c <= r) ? S[r * LDS + c] : 0.0;
  }
  // inverse: column c of X = L^-1 by forward substitution (one thread per column)
  double* X = S + TS * LDS;  // second tile buffer (caller guarantees space)
  if (tid < TS) {
    const int c = tid;
    for (int r = 0; r < TS; ++r) {
      double v;
      if (r < c) {
        v = 0.0;
      } else {
        double s = (r == c) ? 1.0 : 0.0;
        for (int k = c; k < r; ++k) s -= S[r * LDS + k] * X[k * LDS + c];
        v = s / S[r * LDS + r];
      }
      X[r * LDS + c] = v;
    }
  }
  __syncthreads();
  for (int q = tid; q < TS * TS; q += blockDim.x) {
    int r = q >> 6, c = q & 63;
    gLinv[q] = X[r * LDS + c];
  }
}

// Add C22 contributions of the active proxies to one tile held in smem
// (contributions summed in the reference's COO order, then added: h = sigma0 + c22).
__device__ __forceinline__ void add_c22(const DenseDev& d, int tile, double* S) {
  int e0 = d.c22_tile_ptr[tile], e1 = d.c22_tile_ptr[tile + 1];
  for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    double s = 0.0;
    bool any = false;
    for (int q = d.c22_ent_ptr[e]; q < d.c22_ent_ptr[e + 1]; ++q) {
      int code = d.c22_contrib[q];
      int j = code >> 4, a = (code >> 2) & 3, b = code & 3;
      if (!d.active[j]) continue;
      double v = d.proxy_c[j] * (d.proxy_w[4 * j + a] * d.proxy_w[4 * j + b]);
      s = any ? s + v : v;
      any = true;
    }
    if (any) {
      int rc = d.c22_ent_rc[e];
      S[(rc >> 6) * LDS + (rc & 63)] += s;
    }
  }
}

__global__ void __launch_bounds__(256, 1) k_cholesky_tiles(DenseDev d, const int2* __restrict__ tasks, int ntasks) {
  extern __shared__ __align__(16) double smem[];
  double* sA[2] = {smem, smem + TILE_SMEM};
  double* sB[2] = {smem + 2 * TILE_SMEM, smem + 3 * TILE_SMEM};
  double* col = smem + 4 * TILE_SMEM;
  __shared__ int s_task;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wr = warp >> 2, wc = warp & 3;
  const int N = d.N;
  const int ntiles = N * (N + 1) / 2;

  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(d.counter, 1);
    __syncthreads();
    const int task = s_task;
    __syncthreads();
    if (task >= ntasks) break;
    const int2 ij = tasks[task];
    const int i = ij.x, j = ij.y;
    const bool rhs = (i == N);
    const double* src = rhs ? d.Y + (int64_t)j * TS * TS : d.sigma0 + (int64_t)tidx(i, j) * TS * TS;

    // ---- acc <- H tile (sigma0 + C22) or g^T tile
    Acc acc;
    load_tile_async(sA[0], src);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    if (!rhs && d.c22_tile_ptr) {
      add_c22(d, tidx(i, j), sA[0]);
      __syncthreads();
    }
    smem_to_acc(acc, sA[0], wr, wc, lane);
    __syncthreads();

    // ---- left-looking accumulation over k < j, double-buffered
    if (j > 0) {
      auto fa = [&](int k) -> const int* { return d.flags + (rhs ? ntiles + k : tidx(i, k)); };
      auto ta = [&](int k) -> const double* {
        return rhs ? d.Y + (int64_t)k * TS * TS : d.L + (int64_t)tidx(i, k) * TS * TS;
      };
      wait_flag(fa(0));
      wait_flag(d.flags + tidx(j, 0));
      load_tile_async(sA[0], ta(0));
      load_tile_async(sB[0], d.L + (int64_t)tidx(j, 0) * TS * TS);
      cp_async_commit();
      for (int k = 0; k < j; ++k) {
        const int cur = k & 1;
        if (k + 1 < j) {
          wait_flag(fa(k + 1));
          wait_flag(d.flags + tidx(j, k + 1));
          load_tile_async(sA[cur ^ 1], ta(k + 1));
          load_tile_async(sB[cur ^ 1], d.L + (int64_t)tidx(j, k + 1) * TS * TS);
          cp_async_commit();
          cp_async_wait_1();
        } else {
          cp_async_wait_all();
        }
        __syncthreads();
        tile_gemm_abt<true>(acc, sA[cur], sB[cur], wr, wc, lane);
        __syncthreads();
      }
    }

    // ---- finalize
    int* myflag = d.flags + (rhs ? ntiles + j : tidx(i, j));
    if (i == j) {
      acc_to_smem(acc, sA[0], wr, wc, lane);
      __syncthreads();
      // sA[0] holds S, sA[1] is scratch for the inverse
      potrf_inv_tile(sA[0], col, d.L + (int64_t)tidx(j, j) * TS * TS, d.Linv + (int64_t)j * TS * TS, j, d.info);
    } else {
      wait_flag(d.flags + tidx(j, j));
      load_tile_async(sB[0], d.Linv + (int64_t)j * TS * TS);
      cp_async_commit();
      acc_to_smem(acc, sA[0], wr, wc, lane);
      cp_async_wait_all();
      __syncthreads();
      Acc out;
      acc_zero(out);
      tile_gemm_abt<false>(out, sA[0], sB[0], wr, wc, lane);  // acc * inv(Ljj)^T
      double* dst = rhs ? d.Y + (int64_t)j * TS * TS : d.L + (int64_t)tidx(i, j) * TS * TS;
      acc_to_global(out, dst, wr, wc, lane);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release(myflag, 1);
  }
}

// u = L^-T y: x_j^T = (y_j^T - sum_{i>j} x_i^T L_ij) inv(L_jj). CTA b handles
// block j = N-1-b; blocks only wait on lower CTA indices.
__global__ void __launch_bounds__(256) k_dense_backward(DenseDev d, int* __restrict__ xflags,
                                                        double* __restrict__ xrows /* N*3*64 */,
                                                        double* __restrict__ u, int m) {
  __shared__ double xi[3 * TS];
  __shared__ double acc_s[3 * TS];
  const int N = d.N;
  const int j = N - 1 - blockIdx.x;
  const int tid = threadIdx.x;
  const int r = tid >> 6, c = tid & 63;  // r < 3 valid (192 threads)
  double acc = 0.0;
  for (int i = N - 1; i > j; --i) {
    wait_flag(xflags + i);
    if (tid < 3 * TS) xi[tid] = xrows[(int64_t)i * 3 * TS + tid];
    __syncthreads();
    if (r < 3) {
      const double* L = d.L + (int64_t)tidx(i, j) * TS * TS;
      double s = 0.0;
#pragma unroll 8
      for (int k = 0; k < TS; ++k) s += xi[r * TS + k] * L[k * TS + c];
      acc += s;
    }
    __syncthreads();
  }
  if (r < 3) acc_s[r * TS + c] = d.Y[(int64_t)j * TS * TS + r * TS + c] - acc;
  __syncthreads();
  if (r < 3) {
    const double* Li = d.Linv + (int64_t)j * TS * TS;
    double s = 0.0;
#pragma unroll 8
    for (int k = 0; k < TS; ++k) s += acc_s[r * TS + k] * Li[k * TS + c];
    xrows[(int64_t)j * 3 * TS + r * TS + c] = s;
    int row = j * TS + c;
    if (row < m) u[3 * row + r] = s;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) st_release(xflags + j, 1);
}

// sigma0 u: per lower tile, the row and (off-diagonal) column contributions.
__global__ void __launch_bounds__(256) k_sym_gemv_tiles(DenseDev d, const double* __restrict__ u,
                                                        double* __restrict__ partial) {
  const int t = blockIdx.x;
  // decode tile (i, j)
  int i = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while (tidx(i + 1, 0) <= t) ++i;
  while (tidx(i, 0) > t) --i;
  const int j = t - tidx(i, 0);
  __shared__ double ui[3 * TS], uj[3 * TS];
  __shared__ double colred[4][3 * TS];
  const int tid = threadIdx.x;
  const int m = d.m;
  if (tid < TS) {
    int ri = i * TS + tid, rj = j * TS + tid;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      ui[q * TS + tid] = ri < m ? u[3 * ri + q] : 0.0;
      uj[q * TS + tid] = rj < m ? u[3 * rj + q] : 0.0;
    }
  }
  __syncthreads();
  const double* T = d.sigma0 + (int64_t)t * TS * TS;
  // row contribution: warp w handles rows w*8..w*8+7, lanes over columns
  const int lane = tid & 31, w = tid >> 5;
  double* out_row = partial + (int64_t)t * 2 * 3 * TS;
  double* out_col = out_row + 3 * TS;
  for (int rr = 0; rr < 8; ++rr) {
    int row = w * 8 + rr;
    double a0 = T[row * TS + lane], a1 = T[row * TS + lane + 32];
    double s0 = a0 * uj[lane] + a1 * uj[lane + 32];
    double s1 = a0 * uj[TS + lane] + a1 * uj[TS + lane + 32];
    double s2 = a0 * uj[2 * TS + lane] + a1 * uj[2 * TS + lane + 32];
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      out_row[row] = s0;
      out_row[TS + row] = s1;
      out_row[2 * TS + row] = s2;
    }
  }
  if (i != j) {
    // column contribution: T^T ui -> thread (cgrp, col): partial over 16 rows
    const int cc = tid & 63, grp = tid >> 6;
    double s0 = 0, s1 = 0, s2 = 0;
    for (int rr = grp * 16; rr < grp * 16 + 16; ++rr) {
      double a = T[rr * TS + cc];
      s0 += a * ui[rr];
      s1 += a * ui[TS + rr];
      s2 += a * ui[2 * TS + rr];
    }
    colred[grp][cc] = s0;
    colred[grp][TS + cc] = s1;
    colred[grp][2 * TS + cc] = s2;
    __syncthreads();
    if (tid < 3 * TS) out_col[tid] = ((colred[0][tid] + colred[1][tid]) + colred[2][tid]) + colred[3][tid];
  }
}

__global__ void k_sym_gemv_reduce(DenseDev d, const double* __restrict__ partial, double* __restrict__ out) {
  // block b: out rows b*64..; sum row parts (b, j<=b) then column parts (i>b, b)
  const int b = blockIdx.x, tid = threadIdx.x;
  if (tid >= 3 * TS) return;
  const int q = tid / TS, r = tid % TS;
  double s = 0.0;
  for (int j = 0; j <= b; ++j) s += partial[(int64_t)tidx(b, j) * 6 * TS + q * TS + r];
  for (int i = b + 1; i < d.N; ++i) s += partial[(int64_t)tidx(i, b) * 6 * TS + 3 * TS + q * TS + r];
  int row = b * TS + r;
  if (row < d.m) out[3 * row + q] = s;
}

// ------------------------------------------------------------- launchers
void launch_cholesky_tiles(cudaStream_t st, const DenseDev& d, const int2* tasks, int ntasks, int grid) {
  static bool attr = false;
  size_t smem = cholesky_smem_bytes();
  if (!attr) {
    cudaFuncSetAttribute(k_cholesky_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_cholesky_tiles<<<grid, 256, smem, st>>>(d, tasks, ntasks);
}

void launch_dense_backward(cudaStream_t st, const DenseDev& d, int* xflags, double* xrows, double* u) {
  k_dense_backward<<<d.N, 256, 0, st>>>(d, xflags, xrows, u, d.m);
}

void launch_sym_tile_gemv(cudaStream_t st, const DenseDev& d, const double* u, double* partial) {
  k_sym_gemv_tiles<<<dense_tile_count(d.N), 256, 0, st>>>(d, u, partial);
}

void launch_sym_tile_gemv_reduce(cudaStream_t st, const DenseDev& d, const double* partial, double* out) {
  k_sym_gemv_reduce<<<d.N, 192, 0, st>>>(d, partial, out);
}

}  // namespace spb
