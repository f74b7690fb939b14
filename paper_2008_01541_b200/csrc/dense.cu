// Dense FP64 Schur-complement kernels (the inner-loop system of Algorithm 1,
// PAPER.md:402-441; reference linalg.py:432-461 + solver.py:430-440).
//
//   k_cholesky_tiles   H = sigma0 + C22 assembled on the fly and factored
//                      LL^T in ONE persistent launch over 64x64 tiles:
//                      left-looking tile tasks claimed from a global counter
//                      in dependency order (diagonal tasks claimed LEAD columns
//                      ahead), per-tile readiness flags (release / relaxed poll
//                      + acquire fence). Per CTA a producer warp streams the
//                      (L_ik, L_jk) tile pairs with 1D bulk async copies (TMA)
//                      into a 3-stage mbarrier ring while 8 consumer warps run
//                      the trailing products on the FP64 tensor pipe
//                      (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4; tcgen05 has no
//                      f64 kind). The RHS g rides along as an extra tile ROW,
//                      so y = L^-1 g comes out of the same tasks. Diagonal
//                      tiles are factored register-resident as the augmented
//                      panel [A; I], giving L_jj and L_jj^-T in one sweep.
//   k_dense_backward   u = L^-T y, one CTA per tile column, flag chained.
//   k_sym_gemv_*       sigma0 u (lower tiles read once) for the f~2 upkeep
//                      and the residual (solver.py:436-440).
//
// Layout: tile (i,j), i >= j, at index i(i+1)/2 + j; 64x64 swizzled row-major
// (common.cuh swz). The order m is padded to 64 N with an identity tail.
#include "common.cuh"
#include "kernels.cuh"

namespace spb {

constexpr int TS = 64;
constexpr int TILE = TS * TS;            // doubles per tile (global, row-major)
constexpr int TILE_BYTES = TILE * 8;     // 32 KB
constexpr int PTILE = TILE;              // doubles per smem stage tile (swizzled, unpadded)
constexpr int NSTAGE = 3;
constexpr int NCONS = 256;               // consumer threads (8 warps)
constexpr int NTHREADS = NCONS + 32;     // + 1 producer warp
constexpr int LDP = 66;
// RHS row tiles move only their first 8 rows (g^T in rows 0..2, zeros in 3..7;
// swz keeps every row inside its own 64 doubles). Rows 8..63 of a Y tile are
// scratch that no reader uses (each output row depends on its own input row).
constexpr int RHS_BYTES = 8 * TS * 8;                  // plain row stride of the potrf scratch

__host__ __device__ __forceinline__ int tidx(int i, int j) { return i * (i + 1) / 2 + j; }
int dense_tile_count(int N) { return N * (N + 1) / 2; }

// dynamic smem: [stage s][slot a/b] swizzled tiles, a finalize scratch tile,
// then the stage mbarriers, the task-ring mbarriers and the 2 task slots
constexpr int SM_STAGES = NSTAGE * 2 * PTILE;
constexpr int SM_SCR = SM_STAGES;
constexpr int SM_BAR = SM_SCR + PTILE;  // in doubles (8-byte aligned)
size_t cholesky_smem_bytes() { return sizeof(double) * (SM_BAR + 2 * NSTAGE + 4 + 1 + 2); }  // + INT8 path: accumulator barrier, TMEM slot

struct CholSmem {
  double* stage0;
  double* scratch;            // one tile: regular-tile finalize
  unsigned long long* full;   // [NSTAGE]
  unsigned long long* empty;  // [NSTAGE]
  unsigned long long* tfull;  // [2] task ring: the producer published a task id
  unsigned long long* tempty; // [2] task ring: every consumer warp read it
  int* task;                  // [2]
  __device__ __forceinline__ double* slot(int s, int k) const { return stage0 + (s * 2 + k) * PTILE; }
};

// ------------------------------------------------------------- primitives
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, int bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, int parity) {
  asm volatile(
      "{\n .reg .pred P1;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n }\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, int bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NCONS) : "memory"); }

// Spin (one thread) until a readiness flag is set, then order later reads
// (generic and async proxy) after the producer's release.
// MULTI: the flag may be released by a peer GPU (system scope).
template <bool MULTI = false>
__device__ __forceinline__ void poll_flag(const int* f, int v) {
  if (MULTI) {
    if (ld_relaxed_sys(f) < v) {
      SpinGuard g;  // a peer that never releases traps after kSpinLimitNs
      while (ld_relaxed_sys(f) < v) {
        __nanosleep(64);
        g.tick();
      }
    }
    fence_acq_rel_sys();
  } else {
    if (ld_relaxed(f) < v) {
      SpinGuard g;
      while (ld_relaxed(f) < v) {
        __nanosleep(32);
        g.tick();
      }
    }
    fence_acq_rel_gpu();
  }
  fence_proxy_async_global();
}

// Tile-cyclic mode: after a CTA's threads stored a finished tile into the
// local and the peer replicas, order those stores before the flag releases.
template <bool MULTI>
__device__ __forceinline__ void fence_tile_stores() {
  if (MULTI) __threadfence_system();
  else __threadfence();
}
// thread 0: release flag `idx` with value v in every peer replica
__device__ __forceinline__ void release_peers(const DensePeers& pr, int idx, int v) {
  for (int p = 0; p < pr.n; ++p) st_release_sys(pr.flags[p] + idx, v);
}

// Warp tile 32 rows x 16 cols; 8 warps cover 64x64 as 2 x 4.
struct Acc {
  double c[4][2][2];
};
__device__ __forceinline__ void acc_zero(Acc& a) {
#pragma unroll
  for (int mb = 0; mb < 4; ++mb)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) a.c[mb][nb][0] = a.c[mb][nb][1] = 0.0;
}

// acc (+/-)= A * B^T over K = 64, A and B swizzled smem tiles (rows of B are
// the n index). Lane (g, t) reads logical column 16a + 4b + t of rows with
// (row & 3) = g & 3, i.e. physical column 16a + 4(b ^ (g & 3)) + t: four
// per-lane base offsets (one per b) plus immediates.
template <bool NEG>
__device__ __forceinline__ void mma_abt(Acc& acc, const double* sA, const double* sB, int wr, int wc, int lane) {
  const int g = lane >> 2, t = lane & 3, gq = g & 3;
  const double* pa = sA + (wr * 32 + g) * TS + t;
  const double* pb = sB + (wc * 16 + g) * TS + t;
  int ob[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) ob[b] = 4 * (b ^ gq);
#pragma unroll
  for (int a16 = 0; a16 < TS; a16 += 16) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      double av[4], bv[2];
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) {
        const double v = pa[ob[b] + mb * 8 * TS + a16];
        av[mb] = NEG ? -v : v;
      }
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) bv[nb] = pb[ob[b] + nb * 8 * TS + a16];
#pragma unroll
      for (int mb = 0; mb < 4; ++mb)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) dmma(acc.c[mb][nb][0], acc.c[mb][nb][1], av[mb], bv[nb]);
    }
  }
}

// The RHS row's k-step: only rows 0..7 of A (g^T packed in rows 0..2, rows
// 3..7 zero) carry data, so only the warps of rows 0..31 (wr = 0) work, on
// their first m8 block: 1/8 of the DMMAs of a full tile, with the same
// fragment order as mma_abt for those rows (bit-identical results).
template <bool NEG>
__device__ __forceinline__ void mma_abt_m8(Acc& acc, const double* sA, const double* sB, int wc, int lane) {
  const int g = lane >> 2, t = lane & 3, gq = g & 3;
  const double* pa = sA + g * TS + t;
  const double* pb = sB + (wc * 16 + g) * TS + t;
  int ob[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) ob[b] = 4 * (b ^ gq);
#pragma unroll
  for (int a16 = 0; a16 < TS; a16 += 16) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const double v = pa[ob[b] + a16];
      const double av = NEG ? -v : v;
      double bv[2];
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) bv[nb] = pb[ob[b] + nb * 8 * TS + a16];
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) dmma(acc.c[0][nb][0], acc.c[0][nb][1], av, bv[nb]);
    }
  }
}

// acc += A * B, A swizzled (M x K), B swizzled row-major (K x N): b = B[k0+t][n0+g]
// at row k0+t, physical column (n0+g) ^ (t << 2) (a per-lane constant per nb).
__device__ __forceinline__ void mma_ab(Acc& acc, const double* sA, const double* sB, int wr, int wc, int lane) {
  const int g = lane >> 2, t = lane & 3, gq = g & 3;
  const double* pa = sA + (wr * 32 + g) * TS + t;
  int ob[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) ob[b] = 4 * (b ^ gq);
  const double* pb0 = sB + t * TS + ((wc * 16 + 0 + g) ^ (t << 2));
  const double* pb1 = sB + t * TS + ((wc * 16 + 8 + g) ^ (t << 2));
#pragma unroll
  for (int a16 = 0; a16 < TS; a16 += 16) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int k0 = a16 + 4 * b;
      double av[4], bv[2];
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) av[mb] = pa[ob[b] + mb * 8 * TS + a16];
      bv[0] = pb0[k0 * TS];
      bv[1] = pb1[k0 * TS];
#pragma unroll
      for (int mb = 0; mb < 4; ++mb)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) dmma(acc.c[mb][nb][0], acc.c[mb][nb][1], av[mb], bv[nb]);
    }
  }
}

// out = A * U with U = inv(L_jj)^T upper triangular (U[k][n] = 0 for k > n,
// stored as exact zeros). Column block cb (16 columns) needs only k < 16(cb+1),
// so the warp tiling pairs blocks {0,3} and {1,2}: warp w takes rows
// 16(w >> 1) .. +15 of both blocks of its pair and issues 80 DMMAs where the
// dense 32 x 16 tiling issues 128. The skipped products are zero and come last
// in k order, so the sums are those of the dense product.
struct TriAcc {
  double c[2][2][2][2];  // [pair block][mb][nb][2]
};
__device__ __forceinline__ int tri_block(int warp, int blk) { return (warp & 1) ? 1 + blk : 3 * blk; }
__device__ __forceinline__ void mma_ab_upper(TriAcc& acc, const double* sA, const double* sU, int warp, int lane) {
  const int g = lane >> 2, t = lane & 3, gq = g & 3;
  const int cb0 = tri_block(warp, 0), cb1 = tri_block(warp, 1);
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) acc.c[q][mb][nb][0] = acc.c[q][mb][nb][1] = 0.0;
  const double* pa = sA + ((warp >> 1) * 16 + g) * TS + t;
  int ob[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) ob[b] = 4 * (b ^ gq);
  const double* pb[2][2];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) pb[q][nb] = sU + t * TS + (((q ? cb1 : cb0) * 16 + nb * 8 + g) ^ (t << 2));
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int k0 = kb * 16 + 4 * b;
      double av[2];
#pragma unroll
      for (int mb = 0; mb < 2; ++mb) av[mb] = pa[ob[b] + mb * 8 * TS + kb * 16];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (kb > (q ? cb1 : cb0)) continue;  // warp-uniform
        double bv[2];
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) bv[nb] = pb[q][nb][k0 * TS];
#pragma unroll
        for (int mb = 0; mb < 2; ++mb)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb) dmma(acc.c[q][mb][nb][0], acc.c[q][mb][nb][1], av[mb], bv[nb]);
      }
    }
  }
}
__device__ __forceinline__ void tri_to_swz(const TriAcc& acc, double* s, int warp, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        const int r = (warp >> 1) * 16 + mb * 8 + g, c = tri_block(warp, q) * 16 + nb * 8 + 2 * t;
        *reinterpret_cast<double2*>(s + swz(r, c)) = make_double2(acc.c[q][mb][nb][0], acc.c[q][mb][nb][1]);
      }
}

// fragment (row r0+g, cols c0+2t, c0+2t+1) <-> swizzled tiles (smem or global)
template <typename F>
__device__ __forceinline__ void acc_foreach(int wr, int wc, int lane, F f) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mb = 0; mb < 4; ++mb)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) f(mb, nb, wr * 32 + mb * 8 + g, wc * 16 + nb * 8 + 2 * t);
}
__device__ __forceinline__ void smem_to_acc(Acc& acc, const double* s, int wr, int wc, int lane) {
  acc_foreach(wr, wc, lane, [&](int mb, int nb, int r, int c) {
    double2 v = *reinterpret_cast<const double2*>(s + swz(r, c));
    acc.c[mb][nb][0] = v.x;
    acc.c[mb][nb][1] = v.y;
  });
}
__device__ __forceinline__ void acc_to_swz(const Acc& acc, double* s, int wr, int wc, int lane) {
  acc_foreach(wr, wc, lane, [&](int mb, int nb, int r, int c) {
    *reinterpret_cast<double2*>(s + swz(r, c)) = make_double2(acc.c[mb][nb][0], acc.c[mb][nb][1]);
  });
}
__device__ __forceinline__ void acc_to_plain(const Acc& acc, double* s, int wr, int wc, int lane) {
  acc_foreach(wr, wc, lane, [&](int mb, int nb, int r, int c) {
    s[r * LDP + c] = acc.c[mb][nb][0];
    s[r * LDP + c + 1] = acc.c[mb][nb][1];
  });
}

// Add the active proxies' C22 entries of one tile (swizzled smem). Each entry
// sums its contributions in the reference's COO order, then h = sigma0 + c22.
__device__ __forceinline__ void add_c22(const DenseDev& d, int tile, double* S) {
  int e0 = d.c22_tile_ptr[tile], e1 = d.c22_tile_ptr[tile + 1];
  for (int e = e0 + (int)threadIdx.x; e < e1; e += NCONS) {
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
      S[swz(rc >> 6, rc & 63)] += s;
    }
  }
}

// digit planes of a swizzled FP64 tile (INT8 tensor-core path, defined below)
__device__ __forceinline__ void tile_digits(const double* __restrict__ src, const int* __restrict__ erow, int rb,
                                            signed char* __restrict__ dst, int t0, int nt, int r0 = 0, int r1 = 64);

// ------------------------------------------------ diagonal tile factorization
// Blocked factorization of the augmented 128 x 64 panel [A; I] held in shared
// memory (row stride LSP, conflict-free DMMA fragments): for each 16-column
// block, warp 0 factors the 16 x 16 diagonal block with shuffles (its lanes
// 16..31 carry the identity rows, producing D^-T alongside), then all warps
// solve the panel (rows below, incl. the identity rows) against D^-T and apply
// the rank-16 trailing update on the FP64 tensor pipe. Rows 0..63 end as
// L_jj (lower), rows 64..127 as L_jj^-T (upper). 3 consumer barriers per
// block instead of one per column.
constexpr int LSP = 68;        // row stride of the augmented panel (bank slots (4g + t) mod 16)
constexpr int LDT = 20;
constexpr int UPD_WARPS = NCONS / 32 - 1;  // consumer warps beside warp 0        // row stride of the 16 x 16 D^-T block

// 1/sqrt(x) for the (positive, normal) pivots without the library's
// special-case call path, whose ABI spills the live panel registers on every
// column: hardware approximation + two Newton steps (~1 ulp).
__device__ __forceinline__ double pivot_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // one third-order correction, y (1 + e/2 + 3 e^2 / 8) with e = 1 - x y^2:
  // relative error O(e^3) from the ~2^-22 approximation (4 dependent ops
  // instead of the 6 of two Newton steps)
  const double e = fma(-(x * y), y, 1.0);
  const double p = fma(e, 0.375, 0.5);
  return fma(y * e, p, y);
}

// 1/x for the pivot chain: hardware approximation + one cubic correction,
// y (1 + e + e^2) with e = 1 - x y (3 dependent FMAs)
__device__ __forceinline__ double pivot_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  const double t = fma(e, e, e);
  return fma(y, t, y);
}

// double shuffle as two explicit 32-bit shuffles (the generic overload makes
// the register allocator shuffle the halves around with XOR swaps)
__device__ __forceinline__ double shfl_f64(double v, int src) {
  const int lo = __shfl_sync(0xffffffffu, __double2loint(v), src);
  const int hi = __shfl_sync(0xffffffffu, __double2hiint(v), src);
  return __hiloint2double(hi, lo);
}

__device__ __forceinline__ void potrf_diag16(double* S, double* DT, int o, int j, int* info, int lane) {
  // lanes 0..15: row r = lane of D; lanes 16..31: identity row i = lane - 16
  double v[16];
  const bool drow = lane < 16;
#pragma unroll
  for (int c = 0; c < 16; ++c) v[c] = drow ? S[(o + lane) * LSP + o + c] : ((c == lane - 16) ? 1.0 : 0.0);
  int badk = -1;  // first non-positive pivot of the block
  double dnext = shfl_f64(v[0], 0);
#pragma unroll 16
  for (int k = 0; k < 16; ++k) {
    const double dkk = dnext;
    badk = (badk < 0 && !(dkk > 0.0)) ? k : badk;
    const double ip = pivot_rsqrt(dkk);
    const bool active = lane > k;  // rows below the pivot (all identity lanes)
    const double u = v[k];
    const double l = u * ip;
    // one select per column instead of one per updated entry: rows at or
    // above the pivot multiply by zero (their entries stay as they are)
    const double lm = active ? l : 0.0;
    v[k] = (lane == k) ? dkk * ip : (active ? l : v[k]);
    if (k < 15) {
      // critical chain first: lane k+1's next pivot needs only its own
      // entries, a_{k+1,k+1} - a_{k+1,k}^2 / d_k: the chain runs through one
      // reciprocal (the column scaling's rsqrt is off it), then one shuffle
      dnext = shfl_f64(fma(-(u * u), pivot_rcp(dkk), v[k + 1]), k + 1);
    }
    // broadcast the column through shared memory: one store per lane and one
    // broadcast load per entry instead of two 32-bit shuffles per entry
    double* lb = DT + 16 * LDT + 16 * (k & 1);
    if (lane < 16) lb[lane] = l;
    __syncwarp();
#pragma unroll 16
    for (int c = 0; c < 16; ++c) {
      if (c > k) v[c] = fma(-lm, lb[c], v[c]);
    }
  }
  if (badk >= 0 && lane == 0) atomicCAS(info, 0, j * TS + o + badk + 1);
  if (drow) {
#pragma unroll
    for (int c = 0; c < 16; ++c) S[(o + lane) * LSP + o + c] = (c <= lane) ? v[c] : 0.0;
  } else {
#pragma unroll
    for (int c = 0; c < 16; ++c) DT[(lane - 16) * LDT + c] = v[c];
  }
}

#ifdef SPB_POTRF_PROF  // tools/potrf_bench.cu: per-phase clocks of thread 0
__device__ long long g_potrf_prof[32];
#define POTRF_MARK(n) \
  if (threadIdx.x == 0) g_potrf_prof[n] += clock64();
#define POTRF_MARKW(n) \
  if (threadIdx.x == SPB_POTRF_PROF_T) g_potrf_prof[16 + (n)] += clock64();
#define POTRF_MARK0(n) \
  if (threadIdx.x == 0) g_potrf_prof[n] += clock64();
#else
#define POTRF_MARK(n)
#define POTRF_MARKW(n) \
  do {                 \
  } while (0);
#define POTRF_MARK0(n) \
  do {                 \
  } while (0);
#endif

// rank-16 update of the 8x8 block (rb, cb) of the augmented panel by the
// factored column block o: S[rb][cb] -= P[rb][o:o+16] P[cb][o:o+16]^T,
// two blocks per call so their DMMA chains overlap
__device__ __forceinline__ void upd_block2(double* S, int o, int rbA, int cbA, bool okA, int rbB, int cbB, bool okB,
                                           int g, int t) {
  const int rb[2] = {okA ? rbA : 0, okB ? rbB : 0}, cb[2] = {okA ? cbA : 0, okB ? cbB : 0};
  const bool ok[2] = {okA, okB};
  double c0[2], c1[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const double* pc = S + (rb[u] * 8 + g) * LSP + cb[u] * 8 + 2 * t;
    c0[u] = ok[u] ? pc[0] : 0.0;
    c1[u] = ok[u] ? pc[1] : 0.0;
  }
#pragma unroll
  for (int k0 = 0; k0 < 16; k0 += 4)
#pragma unroll
    for (int u = 0; u < 2; ++u)
      dmma(c0[u], c1[u], -S[(rb[u] * 8 + g) * LSP + o + t + k0], S[(cb[u] * 8 + g) * LSP + o + t + k0]);
#pragma unroll
  for (int u = 0; u < 2; ++u)
    if (ok[u]) {
      double* pc = S + (rb[u] * 8 + g) * LSP + cb[u] * 8 + 2 * t;
      pc[0] = c0[u];
      pc[1] = c1[u];
    }
}

// S[rb][cb] -= U[rb rows] U[cb rows]^T over K = 64 with U a swizzled 64x64
// tile (the sub-diagonal L(j, j-1) of the diagonal task), two 8x8 blocks per
// call; the k order and the DMMA accumulation are those of mma_abt<true>, so
// the result is bitwise the register-tile update it replaces
__device__ __forceinline__ void upd_block2_tile(double* S, const double* U, int rbA, int cbA, bool okA, int rbB,
                                                int cbB, bool okB, int g, int t) {
  const int rb[2] = {okA ? rbA : 0, okB ? rbB : 0}, cb[2] = {okA ? cbA : 0, okB ? cbB : 0};
  const bool ok[2] = {okA, okB};
  double c0[2], c1[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const double* pc = S + (rb[u] * 8 + g) * LSP + cb[u] * 8 + 2 * t;
    c0[u] = ok[u] ? pc[0] : 0.0;
    c1[u] = ok[u] ? pc[1] : 0.0;
  }
#pragma unroll
  for (int k0 = 0; k0 < TS; k0 += 4)
#pragma unroll
    for (int u = 0; u < 2; ++u)
      dmma(c0[u], c1[u], -U[swz(rb[u] * 8 + g, k0 + t)], U[swz(cb[u] * 8 + g, k0 + t)]);
#pragma unroll
  for (int u = 0; u < 2; ++u)
    if (ok[u]) {
      double* pc = S + (rb[u] * 8 + g) * LSP + cb[u] * 8 + 2 * t;
      pc[0] = c0[u];
      pc[1] = c1[u];
    }
}

// Look-ahead blocked factorization: after the panel solve of column block kb,
// warp 0 updates the next 16x16 diagonal block and factors it right away while
// warps 1-7 apply the rest of the rank-16 trailing update, so the sequential
// 16-pivot kernels overlap the update work (2 consumer barriers per block).
template <bool MULTI>
// upd (optional): a swizzled tile U whose rank-64 update A -= U U^T is still
// due (the diagonal task's sub-diagonal tile): warp 0 applies it to the first
// 16x16 block and starts factoring while warps 1-7 apply the rest.
// rel_flag (optional): the flag of that tile, released (value 2, and in the
// peers' replicas at rel_idx) by warp 7 while warp 0 factors the first block.
__device__ void potrf_blocked_tile(const Acc& acc, double* S, double* DT, double* gL, double* gLinvT, int j,
                                   int* info, int* flag, int wr, int wc, int lane, const DensePeers& pr,
                                   const double* upd, int* rel_flag = nullptr, int rel_idx = 0,
                                   signed char* dig_out = nullptr, const int* erow = nullptr) {
  const int tid = threadIdx.x, warp = tid >> 5;
  POTRF_MARK(0)
  const int g = lane >> 2, t = lane & 3;
  // identity rows 64 + [r0, r0 + 16) of the inverse half (row 64 + i is first
  // read by the panel solve of block i / 16: each block's rows are set while
  // warp 0 factors the block before)
  auto init_rows = [&](int r0, int t0, int nt) {
    for (int q = t0; q < 16 * 64; q += nt) {
      const int r = r0 + (q >> 6), c = q & 63;
      S[(64 + r) * LSP + c] = (r == c) ? 1.0 : 0.0;
    }
  };
  // columns [c0, c0 + 16) are final once their block's panel is solved:
  // L_jj (lower) and L_jj^-T (upper; rows below the diagonal are zero and
  // may not be initialized yet) go out while later blocks are factored
  auto store_cols = [&](int c0, int t0, int nt, bool linv, bool l) {
    for (int q = t0; q < 64 * 16; q += nt) {
      const int r = q >> 4, c = c0 + (q & 15);
      if (linv) {
        const double v = (r <= c) ? S[(64 + r) * LSP + c] : 0.0;
        gLinvT[swz(r, c)] = v;
        if (MULTI)
          for (int p = 0; p < pr.n; ++p) pr.LinvT[p][(size_t)j * TILE + swz(r, c)] = v;
      }
      if (l) {
        const double v = (c <= r) ? S[r * LSP + c] : 0.0;
        gL[swz(r, c)] = v;
        if (MULTI)
          for (int p = 0; p < pr.n; ++p) pr.L[p][(size_t)tidx(j, j) * TILE + swz(r, c)] = v;
      }
    }
  };
  cons_sync();  // every warp has finished reading the stage area
  acc_foreach(wr, wc, lane, [&](int mb, int nb, int r, int c) {
    S[r * LSP + c] = acc.c[mb][nb][0];
    S[r * LSP + c + 1] = acc.c[mb][nb][1];
  });
  init_rows(0, tid, NCONS);
  cons_sync();
  POTRF_MARK(1)
#pragma unroll 1
  for (int kb = 0; kb < 4; ++kb) {
    const int o = 16 * kb;
    // (a) the trailing update by column block kb-1 (rows [o, 128) x cols
    // [o, 64)): warp 0 updates the 16x16 diagonal block of kb and factors it
    // right away (one call site: the unrolled 16-pivot kernel is large);
    // warps 1..7 update every other block meanwhile
    if (kb == 0 && upd && warp < 4) {
      // the first 16x16 block of A -= U U^T is on the chain: warps 0-3 (one
      // per SM sub-partition) each take a quarter of K for its three 8x8
      // blocks, warp 0 adds the quarters in fixed order
      double* part = DT + 16 * LDT + 64;  // 4 x 3 x 64 doubles past the pivot buffers
      double c[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      const int brb[3] = {0, 1, 1}, bcb[3] = {0, 0, 1};
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        const int k0 = 16 * warp + 4 * s4;
#pragma unroll
        for (int b = 0; b < 3; ++b)
          dmma(c[b][0], c[b][1], -upd[swz(brb[b] * 8 + g, k0 + t)], upd[swz(bcb[b] * 8 + g, k0 + t)]);
      }
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        part[(warp * 3 + b) * 64 + g * 8 + 2 * t] = c[b][0];
        part[(warp * 3 + b) * 64 + g * 8 + 2 * t + 1] = c[b][1];
      }
      asm volatile("bar.sync 3, 128;" ::: "memory");
      if (warp == 0) {
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int q = g * 8 + 2 * t + e;
            double* ps = S + (brb[b] * 8 + g) * LSP + bcb[b] * 8 + 2 * t + e;
            *ps += (part[(0 * 3 + b) * 64 + q] + part[(1 * 3 + b) * 64 + q]) +
                   (part[(2 * 3 + b) * 64 + q] + part[(3 * 3 + b) * 64 + q]);
          }
        __syncwarp();
      }
    }
    if (warp == 0) {
      if (kb > 0) {
        const int d0 = o >> 3;
        upd_block2(S, o - 16, d0, d0, true, d0 + 1, d0, true, g, t);
        upd_block2(S, o - 16, d0 + 1, d0 + 1, true, 0, 0, false, g, t);
        __syncwarp();
      }
      potrf_diag16(S, DT, o, j, info, lane);
    } else {
      if (kb < 2 && rel_flag && dig_out) {
        // INT8 path: the sub-diagonal tile's digit planes, written by warps
        // 1-7 while warp 0 pivots blocks 0 and 1 (half the rows each), precede
        // its release (the partial (j+1, j) that reads them has ~5 us of slack)
        tile_digits(upd, erow, j, dig_out, tid - 32, NCONS - 32, 32 * kb, 32 * kb + 32);
        fence_proxy_async_global();
        if (kb == 1) asm volatile("bar.sync 4, %0;" ::"n"(NCONS - 32) : "memory");
      }
      if (kb == (dig_out ? 1 : 0) && rel_flag && warp == NCONS / 32 - 1 && lane == 0) {
        // every thread's stores of the tile precede the barriers above
        fence_tile_stores<MULTI>();
        st_release(rel_flag, 2);
        if (MULTI) release_peers(pr, rel_idx, 2);
      }
      if (kb == 0 && upd) {
        // the rest of A -= U U^T: lower 8x8 blocks of rows 16..63 (33 blocks)
        constexpr int NB = 33;
        for (int b2 = warp - 1; b2 < NB; b2 += 2 * UPD_WARPS) {
          int rbu[2], cbu[2];
          bool oku[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            int bidx = b2 + u * UPD_WARPS, rb = 2;
            oku[u] = bidx < NB;
            while (oku[u] && bidx > rb) {
              bidx -= rb + 1;
              ++rb;
            }
            rbu[u] = rb;
            cbu[u] = oku[u] ? bidx : 0;
          }
          upd_block2_tile(S, upd, rbu[0], cbu[0], oku[0], rbu[1], cbu[1], oku[1], g, t);
        }
      }
      if (kb == 1) POTRF_MARKW(0)
      if (kb < 3) init_rows(o + 16, tid - 32, NCONS - 32);
      if (kb == 1) POTRF_MARKW(1)
      if (kb > 0) store_cols(o - 16, tid - 32, NCONS - 32, true, true);
      if (kb == 1) POTRF_MARKW(2)
    }
    if (warp > 0 && kb > 0) {
      // only the 8x8 blocks the update changes, listed compactly: the lower
      // blocks of A below warp 0's two block rows, then the rows of the
      // inverse half that are nonzero in the panel (row 64 + i of [A; I]
      // stays e_i in every column < i, so rows i >= o are still zero in
      // panel columns [o - 16, o))
      const int rb0 = o >> 3, cb0 = rb0, ncb = 8 - cb0;
      int ntop = 0;
      for (int rb = rb0 + 2; rb < 8; ++rb) ntop += rb - cb0 + 1;
      const int nblk = ntop + (o >> 3) * ncb;
      for (int b2 = warp - 1; b2 < nblk; b2 += 2 * UPD_WARPS) {
        int rbu[2], cbu[2];
        bool oku[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          int bidx = b2 + u * UPD_WARPS;
          oku[u] = bidx < nblk;
          if (bidx < ntop) {
            int rb = rb0 + 2;
            while (bidx >= rb - cb0 + 1) {
              bidx -= rb - cb0 + 1;
              ++rb;
            }
            rbu[u] = rb;
            cbu[u] = cb0 + bidx;
          } else {
            bidx -= ntop;
            rbu[u] = 8 + bidx / ncb;
            cbu[u] = cb0 + bidx % ncb;
          }
        }
        upd_block2(S, o - 16, rbu[0], cbu[0], oku[0], rbu[1], cbu[1], oku[1], g, t);
      }
    }
    if (kb == 1) POTRF_MARKW(3)
    if (kb == 1) POTRF_MARK0(24)  // warp 0 done (block 1)
    cons_sync();
    POTRF_MARK(2 + 2 * kb)
    // (b) panel: rows [o+16, 128) x cols [o, o+16): P = S_panel * D^-T (in place)
    // (rows 64 + i of the inverse half with i >= o + 16 are still zero here)
    const int pb0 = (o + 16) >> 3, pb1 = min(16, 8 + ((o + 16) >> 3));
    for (int rb = pb0 + warp; rb < pb1; rb += NCONS / 32) {
      double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
      const double* pa = S + (rb * 8 + g) * LSP + o + t;
#pragma unroll
      for (int k0 = 0; k0 < 16; k0 += 4) {
        const double a = pa[k0];
        dmma(c0[0], c0[1], a, DT[(k0 + t) * LDT + 0 + g]);
        dmma(c1[0], c1[1], a, DT[(k0 + t) * LDT + 8 + g]);
      }
      __syncwarp();
      double* pw = S + (rb * 8 + g) * LSP + o + 2 * t;
      pw[0] = c0[0];
      pw[1] = c0[1];
      pw[8] = c1[0];
      pw[9] = c1[1];
    }
    cons_sync();
    POTRF_MARK(3 + 2 * kb)
  }
  // the last columns of L_jj^-T (the next tasks read only it: the kernel
  // never reads the diagonal L tiles), publish, then the last columns of L_jj
  store_cols(48, tid, NCONS, true, false);
  if (flag) {
    fence_proxy_async_global();
    fence_tile_stores<MULTI>();
    cons_sync();
    if (tid == 0) {
      st_release(flag, 1);
      if (MULTI) release_peers(pr, tidx(j, j), 1);
    }
  }
  store_cols(48, tid, NCONS, false, true);
  POTRF_MARK(14)
}

// ---------------------------------------------------------------- kernel
// The producer warp runs one task ahead: it claims task t+1 and streams its
// tiles while the consumers finalize task t (task ids pass through a 2-slot
// mbarrier ring), so claim latency, the first tile's TMA latency and the
// finalize overlap. Diagonal tasks factor in the stage area, so across them
// the producer waits for the consumers (named barrier 2).
template <bool MULTI>
__device__ __forceinline__ void cholesky_body(const DenseDev& d, const int2* __restrict__ tasks, int ntasks) {
  extern __shared__ __align__(128) double smd[];
  CholSmem sm;
  sm.stage0 = smd;
  sm.scratch = smd + SM_SCR;
  sm.full = reinterpret_cast<unsigned long long*>(smd + SM_BAR);
  sm.empty = sm.full + NSTAGE;
  sm.tfull = sm.empty + NSTAGE;
  sm.tempty = sm.tfull + 2;
  sm.task = reinterpret_cast<int*>(sm.tempty + 2);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool producer = warp == 8;
  const int wr = warp >> 2, wc = warp & 3;
  const int N = d.N;
  const int ntiles = N * (N + 1) / 2;
  // a PDL successor (the frame's dense backward) may be scheduled onto the
  // SMs this grid frees in its tail; it waits on the tile flags itself
  if (tid == 0) pdl_trigger();
  if (tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], NCONS / 32);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&sm.tfull[k], 1);
      mbar_init(&sm.tempty[k], NCONS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int it = 0;  // stage-use counter, advanced identically by producer and consumers
  if (producer) {
    auto fill = [&](const double* a, const double* b, int slot_a, int abytes = TILE_BYTES) {
      const int s = it % NSTAGE;
      if (lane == 0) {
        mbar_wait(&sm.empty[s], ((it / NSTAGE) & 1) ^ 1);
        mbar_expect_tx(&sm.full[s], abytes + (b ? TILE_BYTES : 0));
        bulk_g2s(sm.slot(s, slot_a), a, abytes, &sm.full[s]);
        if (b) bulk_g2s(sm.slot(s, 1), b, TILE_BYTES, &sm.full[s]);
      }
      __syncwarp();
      ++it;
    };
    auto wait_ready = [&](const int* f, int v) {
      if (lane == 0) poll_flag<MULTI>(f, v);
      __syncwarp();
    };
    // flag values: 1 = final; the sub-diagonal tile (k+1, k) is first
    // published as a partial sum (1) and finalized by diagonal task k+1 (2)
    auto tile_ready = [&](int r, int c) { wait_ready(d.flags + tidx(r, c), r == c + 1 ? 2 : 1); };
    for (int use = 0;; ++use) {
      const int k2 = use & 1;
      int task = 0;
      if (lane == 0) {
        task = atomicAdd(d.counter, 1);
        mbar_wait(&sm.tempty[k2], ((use >> 1) & 1) ^ 1);
        sm.task[k2] = task;
        mbar_arrive(&sm.tfull[k2]);  // release: the id is visible to the waiters
      }
      task = __shfl_sync(0xffffffffu, task, 0);
      if (task >= ntasks) break;
      const int2 ij = tasks[task];
      const int i = ij.x, j = ij.y;
      const bool rhs = (i == N);
      const double* src = rhs ? d.Y + (size_t)j * TILE : d.sigma0 + (size_t)tidx(i, j) * TILE;
      if (rhs && lane == 0) {
        // launched programmatically behind build_g: g is complete only after
        // the predecessor grid (no-op in an ordinary launch)
        pdl_wait();
        fence_proxy_async_global();
      }
      fill(src, nullptr, 0, rhs ? RHS_BYTES : TILE_BYTES);
      if (i == j) {
        // diagonal task: A = B = L_jk (one copy), then the partial sum of the
        // sub-diagonal tile (j, j-1) with inv(L_{j-1,j-1})^T for its finalize
        for (int k = 0; k < j - 1; ++k) {
          tile_ready(j, k);
          fill(d.L + (size_t)tidx(j, k) * TILE, nullptr, 0);
        }
        if (j > 0) {
          // the partial is usually ready long before diag j-1: only the
          // 32 KB inv(L_{j-1,j-1})^T transfer waits on the chain
          wait_ready(d.flags + tidx(j, j - 1), 1);
          fill(d.L + (size_t)tidx(j, j - 1) * TILE, nullptr, 0);
          wait_ready(d.flags + tidx(j - 1, j - 1), 1);
          fill(d.LinvT + (size_t)(j - 1) * TILE, nullptr, 1);
        }
        // the factorization uses the whole stage area: no prefetch across it
        asm volatile("bar.sync 2, %0;" ::"n"(NTHREADS) : "memory");
      } else {
        for (int k = 0; k < j; ++k) {
          if (rhs) wait_ready(d.flags + ntiles + k, 1);
          else tile_ready(i, k);
          tile_ready(j, k);
          if (rhs) fill(d.Y + (size_t)k * TILE, d.L + (size_t)tidx(j, k) * TILE, 0, RHS_BYTES);
          else fill(d.L + (size_t)tidx(i, k) * TILE, d.L + (size_t)tidx(j, k) * TILE, 0);
        }
        if (i != j + 1 || rhs) {
          wait_ready(d.flags + tidx(j, j), 1);
          fill(d.LinvT + (size_t)j * TILE, nullptr, 1);
        }
      }
    }
    return;
  }
  // ---------------------------------------------------------- consumers
  unsigned long long t_claim = 0, t_kdone = 0, t_fin = 0;
  for (int use = 0;; ++use) {
    const int k2 = use & 1;
    mbar_wait(&sm.tfull[k2], (use >> 1) & 1);
    const int task = sm.task[k2];
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.tempty[k2]);
    if (task >= ntasks) break;
    const int2 ij = tasks[task];
    const int i = ij.x, j = ij.y;
    const bool rhs = (i == N);
    if (d.trace && tid == 0) t_claim = globaltimer();
    int* myflag = d.flags + (rhs ? ntiles + j : tidx(i, j));
    // ---- acc <- H tile (sigma0 + C22) or the g^T tile
    Acc acc;
    int s = it % NSTAGE;
    mbar_wait(&sm.full[s], (it / NSTAGE) & 1);
    // only tiles holding C22 entries (near the diagonal) need the add + barrier
    if (!rhs && d.c22_tile_ptr && d.c22_tile_ptr[tidx(i, j)] < d.c22_tile_ptr[tidx(i, j) + 1]) {
      add_c22(d, tidx(i, j), sm.slot(s, 0));
      cons_sync();
    }
    smem_to_acc(acc, sm.slot(s, 0), wr, wc, lane);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s]);
    ++it;
    const int nk = (i == j) ? j - 1 : j;  // the diagonal task's last k comes from the partial
    for (int k = 0; k < nk; ++k) {
      // ---- left-looking accumulation
      s = it % NSTAGE;
      mbar_wait(&sm.full[s], (it / NSTAGE) & 1);
      if (!rhs) mma_abt<true>(acc, sm.slot(s, 0), sm.slot(s, i == j ? 0 : 1), wr, wc, lane);
      else if (wr == 0) mma_abt_m8<true>(acc, sm.slot(s, 0), sm.slot(s, 1), wc, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
      ++it;
    }
    if (i == j && j > 0) {
      // ---- finalize the sub-diagonal tile on the critical chain:
      // L(j, j-1) = partial * inv(L_{j-1,j-1})^T, publish it (flag 2), and
      // apply its rank-64 update here; diag(j-1) -> diag(j) crosses one flag
      const int sa = it % NSTAGE;  // slot 0: the partial sum
      mbar_wait(&sm.full[sa], (it / NSTAGE) & 1);
      ++it;
      const int sb = it % NSTAGE;  // slot 1: inv(L_{j-1,j-1})^T
      mbar_wait(&sm.full[sb], (it / NSTAGE) & 1);
      ++it;
      TriAcc out;
      mma_ab_upper(out, sm.slot(sa, 0), sm.slot(sb, 1), warp, lane);
      cons_sync();  // every warp has finished reading both stages
      double* scratch = sm.scratch;
      tri_to_swz(out, scratch, warp, lane);
      tri_to_swz(out, d.L + (size_t)tidx(j, j - 1) * TILE, warp, lane);
      if (MULTI)
        for (int p = 0; p < d.peers.n; ++p) tri_to_swz(out, d.peers.L[p] + (size_t)tidx(j, j - 1) * TILE, warp, lane);
      // its rank-64 update A -= L(j, j-1) L(j, j-1)^T is applied inside the
      // factorization (from the scratch copy), off the chain but its first
      // block; the tile's release (flag 2) is issued inside the factorization
      // too, by a warp off the pivot chain, after the factorization's first
      // CTA barrier has ordered every thread's stores before it
      fence_proxy_async_global();
      if (lane == 0) {
        mbar_arrive(&sm.empty[sa]);
        mbar_arrive(&sm.empty[sb]);
      }
    }
    // ---- finalize
    if (d.trace && tid == 0) t_kdone = globaltimer();
    if (i == j) {
      // the producer is parked: the whole stage area holds the augmented panel + D^-T
      potrf_blocked_tile<MULTI>(acc, sm.stage0, sm.stage0 + 128 * LSP, d.L + (size_t)tidx(j, j) * TILE,
                                d.LinvT + (size_t)j * TILE, j, d.info, myflag, wr, wc, lane, d.peers,
                                j > 0 ? sm.scratch : nullptr, j > 0 ? d.flags + tidx(j, j - 1) : nullptr,
                                j > 0 ? tidx(j, j - 1) : 0);
    } else if (i == j + 1 && !rhs) {
      // sub-diagonal tile: publish the partial sum; diagonal task j+1 finalizes it
      acc_to_swz(acc, d.L + (size_t)tidx(i, j) * TILE, wr, wc, lane);
    } else {
      // the producer may already be filling stages for the next task: the
      // finalize works in the dedicated scratch tile
      acc_to_swz(acc, sm.scratch, wr, wc, lane);
      cons_sync();
      s = it % NSTAGE;
      mbar_wait(&sm.full[s], (it / NSTAGE) & 1);
      TriAcc out;
      mma_ab_upper(out, sm.scratch, sm.slot(s, 1), warp, lane);  // acc * inv(L_jj)^T = acc * LinvT
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
      ++it;
      double* dst = rhs ? d.Y + (size_t)j * TILE : d.L + (size_t)tidx(i, j) * TILE;
      tri_to_swz(out, dst, warp, lane);
      if (MULTI)  // tile-cyclic: no RHS row
        for (int p = 0; p < d.peers.n; ++p) tri_to_swz(out, d.peers.L[p] + (size_t)tidx(i, j) * TILE, warp, lane);
    }
    if (d.trace && tid == 0) t_fin = globaltimer();
    fence_proxy_async_smem();    // generic smem writes before later bulk copies into the stages
    fence_proxy_async_global();  // generic global tile stores before other CTAs' bulk reads
    fence_tile_stores<MULTI>();
    cons_sync();  // every consumer's stores are fenced; the scratch tile is free again
    if (tid == 0) {
      st_release(myflag, 1);
      // peers get final tiles only: the diagonal released its own, a partial
      // (j+1, j) is finalized (flag 2) by the diagonal task j+1 on this rank
      if (MULTI && i > j + 1) release_peers(d.peers, tidx(i, j), 1);
      if (d.trace) {
        unsigned long long* tr = d.trace + 4 * (size_t)task;
        tr[0] = t_claim;
        tr[1] = t_kdone;
        tr[2] = globaltimer();
        tr[3] = t_fin;
      }
    }
    if (i == j) asm volatile("bar.sync 2, %0;" ::"n"(NTHREADS) : "memory");  // release the producer
  }
}

__global__ void __launch_bounds__(NTHREADS, 1) k_cholesky_tiles(DenseDev d, const int2* __restrict__ tasks,
                                                                int ntasks) {
  cholesky_body<false>(d, tasks, ntasks);
}

// Tile-cyclic factorization: CTA b serves rank b % P (P = 1 on a real
// multi-GPU rank, P = world size when one GPU emulates all ranks' replicas).
__global__ void __launch_bounds__(NTHREADS, 1) k_cholesky_ranks(const DenseRankJob* __restrict__ jobs, int P) {
  const DenseRankJob& job = jobs[blockIdx.x % P];
  cholesky_body<true>(job.d, job.tasks, job.ntasks);
}

// =====================================================================
// Emulated-FP64 trailing updates on the INT8 tensor cores (tcgen05)
// ---------------------------------------------------------------------
// The left-looking accumulation S = sum_k L_ik L_jk^T is the FP64 work of the
// factorization (m^3 / 3 flops). DMMA (mma.sync m8n8k4.f64) tops out at ~37
// TF on B200; tcgen05 has no FP64 kind. Here every finalized L tile is also
// stored as 8 base-2^7 digit planes (Ozaki-style splitting, int8): row r of
// L is scaled by a power of two 2^erow[r] > max |L_r.| (bounded a priori by
// sqrt(H_rr) >= |L_rc|, since L L^T = H), and
//   L_rc / 2^e_r = d1 / 2^6 + d2 / 2^13 + ... + d8 / 2^55  (|d_p| <= 64).
// The digit products d_p(L_ik) d_q(L_jk)^T are exact in int32 on
// tcgen05.mma.kind::i8 (|sum| < 2^28 per product over any K of this
// problem), accumulated in TMEM per shift group p + q, and converted to FP64
// with exact power-of-two scales: an error ~1e-17 of sum |L_rk L_ck|,
// below that of an FP64 FMA chain (tools/ozaki_probe.cu). Pairs with
// p + q <= 9 (plus the even-p pairs of 10) are kept.
//
// MMA shape M = 128 (two stacked digit planes of L_ik: 2h+1, 2h+2), N = 128
// (planes q, q+1 of L_jk, q odd), K = 32; per 64-deep k-step 20 MMAs
// (1,280 tensor cycles against 4,096 for the 64^3 DMMA step). TMEM block
// bi = (2h + 1 + q - 2) / 2 (128 columns, all 512 columns used): its
// quadrant (lanes 0-63 | 64-127) x (cols 0-63 | 64-127) accumulates shift
// b | b+1 / b+1 | b+2 with b = 2 + 2 bi.
constexpr int NDIG = 8;
constexpr int DPLANE = TS * TS;        // bytes per digit plane of a tile
constexpr int DTILE = NDIG * DPLANE;   // 32 KB: the digits of one L tile

__host__ __device__ __forceinline__ int kmaj_off(int r, int k) {
  return ((r >> 3) * 4 + (k >> 4)) * 128 + (r & 7) * 16 + (k & 15);
}
// 2^k as a double, exact for -1022 <= k <= 1023 (bit construction)
__device__ __forceinline__ double pow2i(int k) { return __longlong_as_double((long long)(k + 1023) << 52); }
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  // no-swizzle K-major: 8-row x 16-byte core matrices, k-chunks 128 B apart
  // (LBO), 8-row groups 512 B apart (SBO), sm_100 descriptor version 1
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46);
}
// instruction descriptor: D s32, A/B signed 8-bit, K-major, N = 128, M = 128
constexpr uint32_t OZ_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
__device__ __forceinline__ void umma_i8(uint32_t dtmem, uint64_t ad, uint64_t bd, int acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dtmem),
      "l"(ad), "l"(bd), "r"(OZ_IDESC), "r"(acc));
}
__device__ __forceinline__ void umma_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t addr, uint32_t (&u)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
        "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15]),
        "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]),
        "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// digits of a swizzled FP64 tile (rows of block `rb`) into the tile's 8
// planes in global memory; 4 consecutive columns (one 32-bit word per plane)
// per work item, threads t0, t0 + nt, ... Each digit is 3 FP64 operations: the
// magic-number round (t = fma(x, 2^7, 1.5 * 2^52) holds rint(128 x) in its low
// bits; no float -> int conversion), the exact remainder fma(x, 2^7, -d).
__device__ __forceinline__ void tile_digits(const double* __restrict__ src, const int* __restrict__ erow, int rb,
                                            signed char* __restrict__ dst, int t0, int nt, int r0, int r1) {
  constexpr double MAGIC = 6755399441055744.0;  // 1.5 * 2^52
  for (int w = r0 * 16 + t0; w < r1 * 16; w += nt) {
    const int r = w >> 4, c0 = (w & 15) * 4;
    const double sc = pow2i(-erow[rb * TS + r]);  // exact scaling
    // the 4 logical columns c0 .. c0+3 are 4 adjacent physical ones (swz XORs a multiple of 4)
    const double2 v01 = *reinterpret_cast<const double2*>(src + swz(r, c0));
    const double2 v23 = *reinterpret_cast<const double2*>(src + swz(r, c0) + 2);
    const double xs[4] = {v01.x * sc, v01.y * sc, v23.x * sc, v23.y * sc};
    uint32_t word[NDIG];
#pragma unroll
    for (int p = 0; p < NDIG; ++p) word[p] = 0u;
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      double x = xs[cc];
#pragma unroll
      for (int p = 0; p < NDIG; ++p) {
        const double m = p == 0 ? 64.0 : 128.0;
        const double t = fma(x, m, MAGIC);
        const double dd = t - MAGIC;
        x = fma(x, m, -dd);
        word[p] |= ((uint32_t)__double2loint(t) & 0xFFu) << (8 * cc);
      }
    }
    const int off = kmaj_off(r, c0);
#pragma unroll
    for (int p = 0; p < NDIG; ++p) *reinterpret_cast<uint32_t*>(dst + p * DPLANE + off) = word[p];
  }
}

// One 64-deep k-step of S += L_a L_b^T from their digit planes in smem
// (sa, sb: 32 KB each; sa == sb for the diagonal tasks). first: the task's
// first k-step (the first MMA into each TMEM block overwrites).
__device__ int g_oz_diag_nomma = 0;  // DIAGNOSTIC ONLY (SPB_OZ_DIAG_NOMMA, traced launches): skip the MMAs
__device__ __forceinline__ void oz_kstep(uint32_t tmem, const signed char* sa, const signed char* sb, bool first) {
  if (g_oz_diag_nomma) return;
  const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
#pragma unroll
  for (int h = 0; h < 4; ++h)
#pragma unroll
    for (int q = 1; q <= NDIG; q += 2) {
      const int b = 2 * h + 1 + q;
      if (b > 9) continue;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk)
        umma_i8(tmem + (uint32_t)((b - 2) / 2 * 128), umma_desc(a0 + 2 * h * DPLANE + kk * 256),
                umma_desc(b0 + (q - 1) * DPLANE + kk * 256), (first && h == 0 && kk == 0) ? 0 : 1);
    }
}

// TMEM accumulators -> acc -= 2^(e_r + e_c) S over the tile (all 8 consumer
// warps; warp w reads TMEM lane quarter w % 4, column half w / 4); P: the
// swizzled scratch tile. Leaves TMEM free (fenced, behind a consumer barrier).
__device__ __forceinline__ void oz_epilogue(uint32_t tmem, Acc& acc, double* P, const int* __restrict__ erow,
                                            int ib, int jb, int warp, int lane, int wr, int wc) {
  const int qd = warp & 3, ch = warp >> 2;
  const int r = (32 * qd + lane) & 63;
  double v[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) v[c] = 0.0;
#pragma unroll 1
  for (int blk = 0; blk < 8; ++blk) {
    uint32_t u[32];
    tmem_ld32(tmem + ((uint32_t)(32 * qd) << 16) + (uint32_t)((blk >> 1) * 128 + (blk & 1) * 64 + 32 * ch), u);
    const int t = 2 + 2 * (blk >> 1) + (blk & 1) + (qd >= 2 ? 1 : 0);
    const double w = __longlong_as_double((long long)(1023 - (7 * t - 2)) << 52);  // 2^-(7t-2), exact
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = fma((double)(int)u[c], w, v[c]);
  }
  tc_fence_before();
  if (qd < 2) {
#pragma unroll
    for (int c = 0; c < 32; ++c) P[swz(r, 32 * ch + c)] = v[c];
  }
  cons_sync();
  if (qd >= 2) {
#pragma unroll
    for (int c = 0; c < 32; ++c) P[swz(r, 32 * ch + c)] += v[c];
  }
  cons_sync();
  acc_foreach(wr, wc, lane, [&](int mb, int nb, int rr, int cc) {
    const int er = erow[ib * TS + rr];
    const double2 pv = *reinterpret_cast<const double2*>(P + swz(rr, cc));
    acc.c[mb][nb][0] -= pv.x * pow2i(er + erow[jb * TS + cc]);
    acc.c[mb][nb][1] -= pv.y * pow2i(er + erow[jb * TS + cc + 1]);
  });
  cons_sync();  // P (the scratch tile) is free again
}

// The left-looking tile Cholesky of cholesky_body with the k-loop on the INT8
// tensor cores (single GPU; the tile-cyclic MULTI path stays on DMMA). Task
// list, flags, diagonal chain, RHS row and finalizes are those of
// cholesky_body; what changes:
//   * the producer streams the 32 KB digit tiles of L_ik / L_jk instead of
//     the FP64 tiles for the k-loop (RHS row and finalize inputs stay FP64);
//   * consumer warp 0, lane 0 issues the 20 MMAs per k-step and releases
//     the stage with tcgen05.commit (8 arrivals: the empty barriers keep
//     their 8-warp count); the last k-step commits to the accumulator barrier;
//   * every finalized L tile (regular tiles and the sub-diagonal tile the
//     diagonal task finalizes) also gets its digit planes before its flag.
__global__ void __launch_bounds__(NTHREADS, 1) k_cholesky_oz(DenseDev d, const int2* __restrict__ tasks, int ntasks) {
  extern __shared__ __align__(1024) double smd[];
  CholSmem sm;
  sm.stage0 = smd;
  sm.scratch = smd + SM_SCR;
  sm.full = reinterpret_cast<unsigned long long*>(smd + SM_BAR);
  sm.empty = sm.full + NSTAGE;
  sm.tfull = sm.empty + NSTAGE;
  sm.tempty = sm.tfull + 2;
  sm.task = reinterpret_cast<int*>(sm.tempty + 2);
  unsigned long long* accf = reinterpret_cast<unsigned long long*>(sm.task + 2);  // 8-byte aligned (task: 2 ints)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool producer = warp == 8;
  const int wr = warp >> 2, wc = warp & 3;
  const int N = d.N;
  const int ntiles = N * (N + 1) / 2;
  if (tid == 0) pdl_trigger();
  if (tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], NCONS / 32);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&sm.tfull[k], 1);
      mbar_init(&sm.tempty[k], NCONS / 32);
    }
    mbar_init(accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  int it = 0;
  if (producer) {
    auto fill = [&](const void* a, const void* b, int slot_a, int abytes = TILE_BYTES) {
      const int s = it % NSTAGE;
      if (lane == 0) {
        mbar_wait(&sm.empty[s], ((it / NSTAGE) & 1) ^ 1);
        mbar_expect_tx(&sm.full[s], abytes + (b ? TILE_BYTES : 0));
        bulk_g2s(sm.slot(s, slot_a), a, abytes, &sm.full[s]);
        if (b) bulk_g2s(sm.slot(s, 1), b, TILE_BYTES, &sm.full[s]);
      }
      __syncwarp();
      ++it;
    };
    auto wait_ready = [&](const int* f, int v) {
      if (lane == 0) poll_flag<false>(f, v);
      __syncwarp();
    };
    // flags in this kernel: a regular tile (r >= c + 2) is final in FP64 at 1
    // and has its digit planes at 2; a sub-diagonal tile (c + 1, c) is a
    // partial sum at 1 and final (FP64) at 2 -- no task ever reads its digits
    // (the k-step k = j - 1 of every task runs in FP64, see below)
    auto fp64_ready = [&](int r, int c) { wait_ready(d.flags + tidx(r, c), r == c + 1 ? 2 : 1); };
    auto digits_ready = [&](int r, int c) { wait_ready(d.flags + tidx(r, c), 2); };
    // Batched readiness: the warp loads the flags of 16 k-steps at once (lanes
    // 0-15: tile (ra, k), lanes 16-31: tile (rb, k)); one fence then covers
    // every flag observed ready, and only the k-steps whose flags were not
    // yet set are polled one by one. (A per-k-step poll is two dependent L2
    // round trips + fences: longer than the INT8 k-step itself.)
    // digits: both tiles' digit planes (flag 2; regular tiles only); else
    // FP64 readiness (ra = N: the RHS row, flags ntiles + k)
    auto ready_mask = [&](int ra, int rb, int k0, int kmax, bool digits) -> unsigned {
      const int kk = k0 + (lane & 15);
      bool ok = true;
      if (kk < kmax) {
        const int r = lane < 16 ? ra : rb;
        const int* f = (r == N) ? d.flags + ntiles + kk : d.flags + tidx(r, kk);
        const int v = digits ? 2 : ((r != N && r == kk + 1) ? 2 : 1);
        ok = ld_relaxed(f) >= v;
      }
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      if (lane == 0) {
        fence_acq_rel_gpu();
        fence_proxy_async_global();
      }
      __syncwarp();
      return (m & 0xFFFFu) & (m >> 16);  // bit l: both tiles of k-step k0 + l ready
    };
    for (int use = 0;; ++use) {
      const int k2 = use & 1;
      int task = 0;
      if (lane == 0) {
        task = atomicAdd(d.counter, 1);
        mbar_wait(&sm.tempty[k2], ((use >> 1) & 1) ^ 1);
        sm.task[k2] = task;
        mbar_arrive(&sm.tfull[k2]);
      }
      task = __shfl_sync(0xffffffffu, task, 0);
      if (task >= ntasks) break;
      const int2 ij = tasks[task];
      const int i = ij.x, j = ij.y;
      const bool rhs = (i == N);
      const double* src = rhs ? d.Y + (size_t)j * TILE : d.sigma0 + (size_t)tidx(i, j) * TILE;
      if (rhs && lane == 0) {
        pdl_wait();
        fence_proxy_async_global();
      }
      fill(src, nullptr, 0, rhs ? RHS_BYTES : TILE_BYTES);
      if (i == j) {
        unsigned rm = 0;
        for (int k = 0; k < j - 1; ++k) {
          if ((k & 15) == 0) rm = ready_mask(j, j, k, j - 1, true);
          if (!((rm >> (k & 15)) & 1u)) digits_ready(j, k);
          fill(d.Lq + (size_t)tidx(j, k) * DTILE, nullptr, 0);
        }
        if (j > 0) {
          wait_ready(d.flags + tidx(j, j - 1), 1);
          fill(d.L + (size_t)tidx(j, j - 1) * TILE, nullptr, 0);
          wait_ready(d.flags + tidx(j - 1, j - 1), 1);
          fill(d.LinvT + (size_t)(j - 1) * TILE, nullptr, 1);
        }
        asm volatile("bar.sync 2, %0;" ::"n"(NTHREADS) : "memory");
      } else {
        unsigned rm = 0;
        // every matrix task takes its last k-step (k = j - 1: the fresh
        // sub-diagonal L(j, j - 1) and L(i, j - 1), at the diagonal chain) in
        // FP64 from the FP64 tiles: no task waits for digit planes of a tile
        // finalized in the last column (RHS row: FP64 throughout)
        const int kq = rhs ? j : j - 1;
        for (int k = 0; k < kq; ++k) {
          if ((k & 15) == 0) rm = ready_mask(i, j, k, kq, !rhs);
          if (!((rm >> (k & 15)) & 1u)) {
            if (rhs) {
              wait_ready(d.flags + ntiles + k, 1);
              fp64_ready(j, k);
            } else {
              digits_ready(i, k);
              digits_ready(j, k);
            }
          }
          if (rhs) fill(d.Y + (size_t)k * TILE, d.L + (size_t)tidx(j, k) * TILE, 0, RHS_BYTES);
          else fill(d.Lq + (size_t)tidx(i, k) * DTILE, d.Lq + (size_t)tidx(j, k) * DTILE, 0);
        }
        if (!rhs && j > 0) {
          fp64_ready(i, j - 1);
          fp64_ready(j, j - 1);
          fill(d.L + (size_t)tidx(i, j - 1) * TILE, d.L + (size_t)tidx(j, j - 1) * TILE, 0);
        }
        if (i != j + 1 || rhs) {
          wait_ready(d.flags + tidx(j, j), 1);
          fill(d.LinvT + (size_t)j * TILE, nullptr, 1);
        }
      }
    }
    return;
  }
  // ---------------------------------------------------------- consumers
  int acc_phase = 0;
  unsigned long long t_claim = 0, t_kdone = 0, t_fin = 0;
  for (int use = 0;; ++use) {
    const int k2 = use & 1;
    mbar_wait(&sm.tfull[k2], (use >> 1) & 1);
    const int task = sm.task[k2];
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.tempty[k2]);
    if (task >= ntasks) break;
    const int2 ij = tasks[task];
    const int i = ij.x, j = ij.y;
    const bool rhs = (i == N);
    int* myflag = d.flags + (rhs ? ntiles + j : tidx(i, j));
    if (d.trace && tid == 0) t_claim = globaltimer();
    Acc acc;
    int s = it % NSTAGE;
    mbar_wait(&sm.full[s], (it / NSTAGE) & 1);
    if (!rhs && d.c22_tile_ptr && d.c22_tile_ptr[tidx(i, j)] < d.c22_tile_ptr[tidx(i, j) + 1]) {
      add_c22(d, tidx(i, j), sm.slot(s, 0));
      cons_sync();
    }
    smem_to_acc(acc, sm.slot(s, 0), wr, wc, lane);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s]);
    ++it;
    const int nk = rhs ? j : j - 1;  // digit-plane k-steps (RHS: FP64 k-steps)
    if (rhs) {
      for (int k = 0; k < nk; ++k) {
        s = it % NSTAGE;
        mbar_wait(&sm.full[s], (it / NSTAGE) & 1);
        if (wr == 0) mma_abt_m8<true>(acc, sm.slot(s, 0), sm.slot(s, 1), wc, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);
        ++it;
      }
    }
    if (!rhs && nk > 0) {
      // ---- the k-loop on the tensor cores: one thread issues, commits free the stages
      if (warp == 0) {
        // the whole warp waits (no divergent spin beside the issuing lane);
        // lane 0 issues
        for (int k = 0; k < nk; ++k) {
          s = (it + k) % NSTAGE;
          mbar_wait(&sm.full[s], ((it + k) / NSTAGE) & 1);
          tc_fence_after();
          if (lane == 0) {
            const signed char* sa = reinterpret_cast<const signed char*>(sm.slot(s, 0));
            const signed char* sb = (i == j) ? sa : reinterpret_cast<const signed char*>(sm.slot(s, 1));
            oz_kstep(tmem, sa, sb, k == 0);
#pragma unroll
            for (int w = 0; w < NCONS / 32; ++w) umma_commit(&sm.empty[s]);  // 8 arrivals when the MMAs are done
            if (k == nk - 1) umma_commit(accf);
          }
          __syncwarp();
        }
      }
      it += nk;
      mbar_wait(accf, acc_phase);
      acc_phase ^= 1;
      tc_fence_after();
      oz_epilogue(tmem, acc, sm.scratch, d.erow, i, j, warp, lane, wr, wc);
    }
    if (!rhs && i != j && j > 0) {
      // ---- the last k-step (k = j - 1) in FP64 on DMMA
      s = it % NSTAGE;
      mbar_wait(&sm.full[s], (it / NSTAGE) & 1);
      mma_abt<true>(acc, sm.slot(s, 0), sm.slot(s, 1), wr, wc, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
      ++it;
    }
    if (i == j && j > 0) {
      // ---- finalize the sub-diagonal tile on the chain (as cholesky_body),
      // plus its digit planes before it is released (inside the factorization)
      const int sa = it % NSTAGE;
      mbar_wait(&sm.full[sa], (it / NSTAGE) & 1);
      ++it;
      const int sb = it % NSTAGE;
      mbar_wait(&sm.full[sb], (it / NSTAGE) & 1);
      ++it;
      TriAcc out;
      mma_ab_upper(out, sm.slot(sa, 0), sm.slot(sb, 1), warp, lane);
      cons_sync();
      double* scratch = sm.scratch;
      tri_to_swz(out, scratch, warp, lane);
      tri_to_swz(out, d.L + (size_t)tidx(j, j - 1) * TILE, warp, lane);
      // its digit planes are written inside the factorization, off the pivot chain
      fence_proxy_async_global();
      if (lane == 0) {
        mbar_arrive(&sm.empty[sa]);
        mbar_arrive(&sm.empty[sb]);
      }
    }
    if (d.trace && tid == 0) t_kdone = globaltimer();
    if (i == j) {
      potrf_blocked_tile<false>(acc, sm.stage0, sm.stage0 + 128 * LSP, d.L + (size_t)tidx(j, j) * TILE,
                                d.LinvT + (size_t)j * TILE, j, d.info, myflag, wr, wc, lane, d.peers,
                                j > 0 ? sm.scratch : nullptr, j > 0 ? d.flags + tidx(j, j - 1) : nullptr,
                                j > 0 ? tidx(j, j - 1) : 0);
      if (d.trace && tid == 0) t_fin = globaltimer();  // the factorization (and the diagonal's release) is done
    } else if (i == j + 1 && !rhs) {
      acc_to_swz(acc, d.L + (size_t)tidx(i, j) * TILE, wr, wc, lane);
    } else {
      acc_to_swz(acc, sm.scratch, wr, wc, lane);
      cons_sync();
      s = it % NSTAGE;
      mbar_wait(&sm.full[s], (it / NSTAGE) & 1);
      TriAcc out;
      mma_ab_upper(out, sm.scratch, sm.slot(s, 1), warp, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
      ++it;
      double* dst = rhs ? d.Y + (size_t)j * TILE : d.L + (size_t)tidx(i, j) * TILE;
      tri_to_swz(out, dst, warp, lane);
      if (!rhs) {
        // the FP64 tile is final (flag 1: the FP64 last k-steps of column i
        // and the dense backward read it), then its digit planes (flag 2)
        fence_proxy_async_global();
        fence_tile_stores<false>();
        cons_sync();  // also: every warp is done reading the scratch tile
        if (tid == 0) st_release(myflag, 1);
        tri_to_swz(out, sm.scratch, warp, lane);
        cons_sync();
        tile_digits(sm.scratch, d.erow, i, d.Lq + (size_t)tidx(i, j) * DTILE, tid, NCONS);
      }
    }
    if (d.trace && tid == 0 && i != j) t_fin = globaltimer();
    fence_proxy_async_smem();
    fence_proxy_async_global();
    fence_tile_stores<false>();
    cons_sync();
    if (tid == 0) {
      // regular tiles: 2 = digit planes written too; partials, diagonals, RHS: 1
      st_release(myflag, (!rhs && i >= j + 2) ? 2 : 1);
      if (d.trace) {
        unsigned long long* tr = d.trace + 4 * (size_t)task;
        tr[0] = t_claim;
        tr[1] = t_kdone;
        tr[2] = globaltimer();
        tr[3] = t_fin;
      }
    }
    if (i == j) asm volatile("bar.sync 2, %0;" ::"n"(NTHREADS) : "memory");
  }
  // consumers: release TMEM (every MMA of this CTA has been waited on)
  tc_fence_before();
  cons_sync();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// u = L^-T y, block rows from the bottom: x_j = (y_j - sum_{i>j} x_i L_ij) W_j
// with W_j = inv(L_jj)^T (x_j, y_j: 3 x 64 row blocks; x_i L_ij: 3x64 * 64x64).
// CTA b owns block j = N-1-b and only waits on lower CTA indices.
// The chain step j+1 -> j is cut to one small GEMV: at launch every CTA
// precomputes M_j = L_{j+1,j} W_j in shared memory and prefetches L_{j+2,j};
// the contributions of x_i, i >= j+2, and c_j = (y_j - sum_{i>=j+2} x_i L_ij) W_j
// are formed while x_{j+1} is still being solved, so after it arrives only
// x_j = c_j - x_{j+1} M_j (3 x 64 x 64, split 4 ways + fixed-order reduce) remains.
// No flags: xrows is preset to an all-ones NaN that arithmetic never produces
// (results are canonicalised), producers store each value with a relaxed
// store and one consumer warp polls the 192 values themselves, so a chain
// step costs one store -> load visibility instead of store, fence, release
// flag, poll, acquire and reload.
constexpr int BW_LDS = 65;  // padded row stride of the shared tiles (conflict-free column access)
constexpr int BW_SMEM_DOUBLES = 4 * TS * BW_LDS + 6 * TS + 12 * TS + 3 * TS + 3 * TS + 1;
constexpr unsigned long long BW_EMPTY = ~0ull;  // sentinel (negative NaN, all payload bits set)

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// warp 0 waits until block i of xrows is complete and stages it in xi
// (3 x 64); with `also` >= 0 it also stages block `also` into xi + 192 if that
// one is complete by then. Returns (to every thread) how many were staged.
__device__ __forceinline__ int bw_fetch(const double* xrows, int i, double* xi, int also, int* nflag) {
  if (threadIdx.x < 32) {
    const double* src = xrows + (size_t)i * 3 * TS;
    const double* src2 = xrows + (size_t)(also >= 0 ? also : i) * 3 * TS;
    unsigned long long v[6], w[6];
    bool ready, ready2;
    SpinGuard g;
    do {
      g.tick();
      ready = ready2 = true;
#pragma unroll
      for (int e = 0; e < 6; ++e) {
        v[e] = ld_relaxed_u64(src + threadIdx.x + 32 * e);
        w[e] = ld_relaxed_u64(src2 + threadIdx.x + 32 * e);
        ready &= (v[e] != BW_EMPTY);
        ready2 &= (w[e] != BW_EMPTY);
      }
    } while (!__all_sync(0xffffffffu, ready));
    const bool two = also >= 0 && __all_sync(0xffffffffu, ready2);
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      xi[threadIdx.x + 32 * e] = __longlong_as_double((long long)v[e]);
      if (two) xi[3 * TS + threadIdx.x + 32 * e] = __longlong_as_double((long long)w[e]);
    }
    if (threadIdx.x == 0) *nflag = two ? 2 : 1;
  }
  __syncthreads();
  return *nflag;
}

// part[grp][r][c] = sum_{k in group} x[r][k] T[k][c]   (T plain, stride BW_LDS)
__device__ __forceinline__ void bw_gemv_part(const double* x, const double* T, double* part, int c, int grp) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
  for (int k = grp * 16; k < grp * 16 + 16; ++k) {
    const double l = T[k * BW_LDS + c];
    a0 += x[k] * l;
    a1 += x[TS + k] * l;
    a2 += x[2 * TS + k] * l;
  }
  part[(grp * 3 + 0) * TS + c] = a0;
  part[(grp * 3 + 1) * TS + c] = a1;
  part[(grp * 3 + 2) * TS + c] = a2;
}
__device__ __forceinline__ double bw_reduce(const double* part, int tid) {
  const int r = tid >> 6, c = tid & 63;
  return ((part[(0 * 3 + r) * TS + c] + part[(1 * 3 + r) * TS + c]) + part[(2 * 3 + r) * TS + c]) +
         part[(3 * 3 + r) * TS + c];
}

__global__ void __launch_bounds__(256) k_dense_backward(DenseDev d, double* __restrict__ xrows /* N*3*64 */,
                                                        double* __restrict__ u, int m,
                                                        unsigned long long* __restrict__ trace /* 5 per CTA or null */,
                                                        int await_flags) {
  unsigned long long tt[5] = {0, 0, 0, 0, 0};
  if (trace && threadIdx.x == 0) tt[0] = globaltimer();
  extern __shared__ double bw_sm[];
  double* sW = bw_sm;                   // W[k][c] = inv(L_jj)[c][k]
  double* sM = sW + TS * BW_LDS;        // M = L_{j+1,j} W
  double* sL1 = sM + TS * BW_LDS;       // L_{j+1,j} (plain rows)
  double* sL2 = sL1 + TS * BW_LDS;      // L_{j+2,j}
  double* xi = sL2 + TS * BW_LDS;       // 2 x 3 x 64
  double* part = xi + 6 * TS;           // 4 x 3 x 64 partial sums
  double* cj = part + 12 * TS;          // 3 x 64
  double* yj = cj + 3 * TS;             // 3 x 64: y_j, prefetched
  int* nflag = reinterpret_cast<int*>(yj + 3 * TS);
  double* sM2 = sL1;                    // M2 = L_{j+2,j} W (overwrites L_{j+1,j} once M is formed)
  const int N = d.N;
  const int j = N - 1 - blockIdx.x;
  const int tid = threadIdx.x;
  const int c = tid & 63, grp = tid >> 6;  // 4 groups x 64 columns
  if (tid == 0) pdl_trigger();  // the u2 consumer behind may launch (it waits for this grid)
  if (await_flags) {
    // launched programmatically behind the factorization: column j of L,
    // inv(L_jj)^T and y_j are read only once their flags are released
    if (tid < 32) {
      const int ntiles = N * (N + 1) / 2;
      for (int i = j + tid; i <= N; i += 32) {
        const int* f = i == N ? d.flags + ntiles + j : d.flags + tidx(i, j);
        const int v = (i == j + 1 && i < N) ? 2 : 1;  // the sub-diagonal tile is final at 2
        // bounded in time (SpinGuard): this CTA may wait for the whole
        // factorization, so the bound is a clock limit, not a spin count
        SpinGuard g;
        while (ld_relaxed(f) < v) {
          __nanosleep(256);
          g.tick();
        }
      }
      fence_acq_rel_gpu();
    }
    __syncthreads();
  }
  // ---- prologue (off the chain): W, L_{j+1,j}, L_{j+2,j} -> smem; M = L_{j+1,j} W
  for (int q = tid; q < TILE; q += 256) {
    const int k = q >> 6, cc = q & 63;
    sW[cc * BW_LDS + k] = d.LinvT[(size_t)j * TILE + swz(k, cc)];  // LinvT row k = column k of inv(L_jj)
    if (j + 1 < N) sL1[k * BW_LDS + cc] = d.L[(size_t)tidx(j + 1, j) * TILE + swz(k, cc)];
    if (j + 2 < N) sL2[k * BW_LDS + cc] = d.L[(size_t)tidx(j + 2, j) * TILE + swz(k, cc)];
  }
  if (tid < 3 * TS) yj[tid] = d.Y[(size_t)j * TILE + swz(tid >> 6, c)];
  __syncthreads();
  // M[k][c] = sum_p A[k][p] W[p][c] for A = L_{j+1,j} and (then) L_{j+2,j}:
  // thread (grp, c) forms rows k = grp + 4 q
  auto times_w = [&](const double* A, double* out) {
#pragma unroll 1
    for (int q = 0; q < 16; ++q) {
      const int k = grp + 4 * q;
      double s = 0.0;
#pragma unroll 16
      for (int p = 0; p < TS; ++p) s = fma(A[k * BW_LDS + p], sW[p * BW_LDS + c], s);
      out[k * BW_LDS + c] = s;
    }
  };
  if (j + 1 < N) times_w(sL1, sM);
  if (j + 2 < N) {
    __syncthreads();  // L_{j+1,j} consumed: its buffer takes M2
    times_w(sL2, sM2);
  }
  // ---- contributions of x_i, i >= j+3, from the global tiles: the next two
  // tiles are loaded into registers ahead of their x, and when this CTA is
  // behind the solved frontier it consumes two ready blocks per round
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  auto load_tile = [&](int i, double (&t)[16]) {
    const double* L = d.L + (size_t)tidx(i, j) * TILE;
#pragma unroll
    for (int q = 0; q < 16; ++q) t[q] = L[swz(grp * 16 + q, c)];
  };
  auto consume = [&](const double* x, const double (&t)[16]) {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int k = grp * 16 + q;
      acc0 += x[k] * t[q];
      acc1 += x[TS + k] * t[q];
      acc2 += x[2 * TS + k] * t[q];
    }
  };
  {
    double ta[16], tb[16];
    int i = N - 1;
    if (i >= j + 3) load_tile(i, ta);
    if (i - 1 >= j + 3) load_tile(i - 1, tb);
    while (i >= j + 3) {
      const int got = bw_fetch(xrows, i, xi, i - 1 >= j + 3 ? i - 1 : -1, nflag);
      consume(xi, ta);
      if (got == 2) {
        consume(xi + 3 * TS, tb);
        if (i - 2 >= j + 3) load_tile(i - 2, ta);
        if (i - 3 >= j + 3) load_tile(i - 3, tb);
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) ta[q] = tb[q];
        if (i - 2 >= j + 3) load_tile(i - 2, tb);
      }
      i -= got;
      __syncthreads();
    }
  }
  if (trace && threadIdx.x == 0) tt[1] = globaltimer();
  // ---- c'_j = (y_j - sum_{i>=j+3} x_i L_ij) W as soon as those sums are in;
  // then x_{j+2} costs one GEMV with M2 = L_{j+2,j} W when it arrives
  part[(grp * 3 + 0) * TS + c] = acc0;
  part[(grp * 3 + 1) * TS + c] = acc1;
  part[(grp * 3 + 2) * TS + c] = acc2;
  __syncthreads();
  if (tid < 3 * TS) xi[tid] = yj[tid] - bw_reduce(part, tid);
  __syncthreads();
  bw_gemv_part(xi, sW, part, c, grp);
  __syncthreads();
  if (tid < 3 * TS) cj[tid] = bw_reduce(part, tid);
  if (j + 2 < N) {
    __syncthreads();  // xi and part free
    bw_fetch(xrows, j + 2, xi, -1, nflag);
    bw_gemv_part(xi, sM2, part, c, grp);
    __syncthreads();
    if (tid < 3 * TS) cj[tid] -= bw_reduce(part, tid);
  }
  if (trace && threadIdx.x == 0) tt[2] = globaltimer();
  // ---- the chain step: x_j = c_j - x_{j+1} M
  double x = 0.0;
  if (j + 1 < N) {
    __syncthreads();  // cj complete; xi free
    bw_fetch(xrows, j + 1, xi, -1, nflag);
    if (trace && threadIdx.x == 0) tt[3] = globaltimer();
    bw_gemv_part(xi, sM, part, c, grp);
    __syncthreads();
    if (tid < 3 * TS) x = cj[tid] - bw_reduce(part, tid);
  } else if (tid < 3 * TS) {
    x = cj[tid];
  }
  if (tid < 3 * TS) {
    if (isnan(x)) x = CUDART_NAN;  // canonical: never the sentinel
    st_relaxed_f64(xrows + (size_t)j * 3 * TS + tid, x);
    if (trace && threadIdx.x == 0) {
      tt[4] = globaltimer();
      for (int k = 0; k < 5; ++k) trace[5 * (size_t)blockIdx.x + k] = tt[k];
    }
    const int row = j * TS + c;
    if (row < m) u[3 * row + (tid >> 6)] = x;
  }
}

// sigma0 u: per lower tile, the row and (off-diagonal) column contributions.
// Thread (row group g, column c) loads its 16 tile entries once (coalesced
// across c), forms the column part in registers and the row part with one
// 16-way warp transpose-sum per RHS; fixed-order shared reductions finish both.
__device__ __forceinline__ double gemv_transpose_sum16(double (&v)[16], int lane) {
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], 16);
#pragma unroll
  for (int off = 8; off >= 1; off >>= 1) {
    const bool upper = lane & off;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const double send = upper ? v[i] : v[i + off];
      const double keep = upper ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];  // lane l: the total of entry l % 16
}

__global__ void __launch_bounds__(256) k_sym_gemv_tiles(DenseDev d, const double* __restrict__ u,
                                                        double* __restrict__ partial) {
  const int t = blockIdx.x;
  int i = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while (tidx(i + 1, 0) <= t) ++i;
  while (tidx(i, 0) > t) --i;
  const int j = t - tidx(i, 0);
  __shared__ double ui[3 * TS], uj[3 * TS];
  __shared__ double colred[4][3 * TS];
  __shared__ double rowred[2][3 * TS];
  const int tid = threadIdx.x, lane = tid & 31;
  const int c = tid & 63, g = tid >> 6;
  const int m = d.m;
  if (tid < TS) {
    const int ri = i * TS + tid, rj = j * TS + tid;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      ui[q * TS + tid] = ri < m ? u[3 * ri + q] : 0.0;
      uj[q * TS + tid] = rj < m ? u[3 * rj + q] : 0.0;
    }
  }
  const double* T = d.sigma0 + (size_t)t * TILE;
  double a[16];
#pragma unroll
  for (int rr = 0; rr < 16; ++rr) a[rr] = T[swz(16 * g + rr, c)];
  __syncthreads();
  double* out_row = partial + (size_t)t * 6 * TS;
  double* out_col = out_row + 3 * TS;
  // row part: sum over c of a[r][c] uj[c]; warps hold 32 columns x 16 rows
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const double w = uj[q * TS + c];
    double v[16];
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) v[rr] = a[rr] * w;
    const double sum = gemv_transpose_sum16(v, lane);
    if (lane < 16) rowred[c >> 5][q * TS + 16 * g + lane] = sum;
  }
  if (i != j) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      double s = 0.0;
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) s += a[rr] * ui[q * TS + 16 * g + rr];
      colred[g][q * TS + c] = s;
    }
  }
  __syncthreads();
  if (tid < 3 * TS) {
    out_row[tid] = rowred[0][tid] + rowred[1][tid];
    if (i != j) out_col[tid] = ((colred[0][tid] + colred[1][tid]) + colred[2][tid]) + colred[3][tid];
  }
}

// ---------------------------------------------- streaming symmetric mat-vec
// partial = per-tile products of sigma0 u (3 RHS) over the lower tiles
// (solver.py:436-440: the f~2 upkeep and the residual share this one pass).
// Persistent: every CTA streams tiles t = blockIdx.x + k * gridDim.x through a
// 3-stage ring of 32 KB bulk copies (cp.async.bulk + mbarrier), so HBM sees a
// continuous stream instead of one short-lived CTA per tile; the u blocks of
// the next tile are prefetched into registers while the current one computes.
//   row part    (block row i): T u_j on the FP64 tensor pipe (DMMA m8n8k4,
//               RHS in the n dimension): warp w owns rows 8w..8w+7, 16 k-steps;
//               the fragments read the swizzled tile conflict-free;
//   column part (block j, i != j): T^T u_i with FMAs, thread = column,
//               16 rows per thread, 4 row groups summed in fixed order.
// k_sym_gemv_reduce4 then sums every block's partials in fixed tile order.
#ifndef SG_STAGES_CFG
#define SG_STAGES_CFG 2
#define SG_CTAS_CFG 3
#endif
constexpr int SG_STAGES = SG_STAGES_CFG;
constexpr int SG_THREADS = 256;
constexpr int SG_CTAS_PER_SM = SG_CTAS_CFG;
constexpr size_t SG_SMEM = (size_t)SG_STAGES * TILE_BYTES + 8 * (6 * TS + 4 * 3 * TS + 3 * TS) + 64;

__device__ __forceinline__ void sgemv_tile_ij(int t, int& i, int& j) {
  i = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while (tidx(i + 1, 0) <= t) ++i;
  while (tidx(i, 0) > t) --i;
  j = t - tidx(i, 0);
}

__global__ void __launch_bounds__(SG_THREADS, SG_CTAS_PER_SM) k_sym_gemv_stream(
    DenseDev d, const double* __restrict__ u, double* __restrict__ partial) {
  extern __shared__ __align__(128) double sgm[];
  double* stage = sgm;                      // SG_STAGES x 64 x 64 (swizzled, as in global)
  double* ubuf = sgm + SG_STAGES * TILE;    // [u_i (3 x 64) | u_j (3 x 64)], RHS-major
  double* colred = ubuf + 6 * TS;           // 4 row groups x 3 x 64
  double* rowout = colred + 4 * 3 * TS;     // 3 x 64
  unsigned long long* full = reinterpret_cast<unsigned long long*>(rowout + 3 * TS);  // SG_STAGES
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int ntiles = d.N * (d.N + 1) / 2;
  const int m = d.m;
  if (tid == 0) {
    for (int k = 0; k < SG_STAGES; ++k) mbar_init(&full[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int nmine = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) ++nmine;
  if (tid == 0) {  // sigma0 is constant: the ring fills while the predecessor finishes
    for (int k = 0; k < SG_STAGES && k < nmine; ++k) {
      const int t = blockIdx.x + k * gridDim.x;
      mbar_expect_tx(&full[k], TILE_BYTES);
      bulk_g2s(stage + k * TILE, d.sigma0 + (size_t)t * TILE, TILE_BYTES, &full[k]);
    }
  }
  pdl_wait();  // u comes from the predecessor (dense backward solve)
  double pu[6];
  {
    int i, j;
    sgemv_tile_ij(blockIdx.x, i, j);
    if (tid < TS && nmine > 0) {
      const int ri = i * TS + tid, rj = j * TS + tid;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        pu[q] = ri < m ? u[3 * ri + q] : 0.0;
        pu[3 + q] = rj < m ? u[3 * rj + q] : 0.0;
      }
    }
  }
  for (int k = 0; k < nmine; ++k) {
    const int t = blockIdx.x + k * gridDim.x;
    const int sidx = k % SG_STAGES;
    double* ui = ubuf;  // rewritten only after the previous tile's last barrier
    double* uj = ui + 3 * TS;
    int i, j;
    sgemv_tile_ij(t, i, j);
    if (tid < TS) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        ui[q * TS + tid] = pu[q];
        uj[q * TS + tid] = pu[3 + q];
      }
      // prefetch the next tile's u blocks (latency hidden behind this tile)
      if (k + 1 < nmine) {
        int i2, j2;
        sgemv_tile_ij(t + gridDim.x, i2, j2);
        const int ri = i2 * TS + tid, rj = j2 * TS + tid;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          pu[q] = ri < m ? u[3 * ri + q] : 0.0;
          pu[3 + q] = rj < m ? u[3 * rj + q] : 0.0;
        }
      }
    }
    __syncthreads();  // u blocks staged; the previous tile's rowout/colred were read
    mbar_wait(&full[sidx], (k / SG_STAGES) & 1);
    const double* T = stage + sidx * TILE;
    // ---- row part on DMMA: rows 8w + g8, RHS in n (columns 0..2 of 8);
    // two accumulator chains (even / odd k-steps) summed at the end
    {
      // four independent accumulator chains (k-steps mod 4), summed in fixed order
      double cc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      const int r = 8 * warp + g8;
#pragma unroll
      for (int ks = 0; ks < 16; ks += 4) {
        double a[4], bb[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          a[h] = T[swz(r, 4 * (ks + h) + t4)];
          bb[h] = g8 < 3 ? uj[g8 * TS + 4 * (ks + h) + t4] : 0.0;
        }
#pragma unroll
        for (int h = 0; h < 4; ++h) dmma(cc[h][0], cc[h][1], a[h], bb[h]);
      }
      const double c0 = (cc[0][0] + cc[1][0]) + (cc[2][0] + cc[3][0]);
      const double c1 = (cc[0][1] + cc[1][1]) + (cc[2][1] + cc[3][1]);
      // lane (g8, t4) holds C[g8][2 t4], C[g8][2 t4 + 1]: RHS 0,1 (t4 = 0), RHS 2 (t4 = 1)
      if (t4 == 0) {
        rowout[0 * TS + r] = c0;
        rowout[1 * TS + r] = c1;
      } else if (t4 == 1) {
        rowout[2 * TS + r] = c0;
      }
    }
    // ---- column part: thread = column c, rows 16 g .. 16 g + 15
    if (i != j) {
      const int c = tid & 63, g = tid >> 6;
      double sv[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};  // even / odd rows
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) {
        const int r = 16 * g + rr;
        const double a = T[swz(r, c)];
#pragma unroll
        for (int q = 0; q < 3; ++q) sv[rr & 1][q] = fma(a, ui[q * TS + r], sv[rr & 1][q]);
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) colred[(g * 3 + q) * TS + c] = sv[0][q] + sv[1][q];
    }
    __syncthreads();  // stage sidx is free; rowout/colred complete
    if (tid == 0 && k + SG_STAGES < nmine) {
      const int tn = blockIdx.x + (k + SG_STAGES) * gridDim.x;
      fence_proxy_async_smem();
      mbar_expect_tx(&full[sidx], TILE_BYTES);
      bulk_g2s(stage + sidx * TILE, d.sigma0 + (size_t)tn * TILE, TILE_BYTES, &full[sidx]);
    }
    double* out_row = partial + (size_t)t * 6 * TS;
    double* out_col = out_row + 3 * TS;
    if (tid < 3 * TS) {
      out_row[tid] = rowout[tid];
      if (i != j) {
        const int q = tid / TS, c = tid % TS;
        out_col[tid] = ((colred[(0 * 3 + q) * TS + c] + colred[(1 * 3 + q) * TS + c]) +
                        colred[(2 * 3 + q) * TS + c]) + colred[(3 * 3 + q) * TS + c];
      }
    }
  }
  if (tid == 0) pdl_trigger();
}

// out[b] = the sum over the tiles of block row/column b in fixed tile order:
// 4 thread groups each sum a fixed quarter of the tiles, then group 0 adds
// the four quarter sums in fixed order (4x the loads in flight of a single
// sequential sum; bitwise deterministic).
__global__ void __launch_bounds__(768) k_sym_gemv_reduce4(DenseDev d, const double* __restrict__ partial,
                                                          double* __restrict__ out) {
  __shared__ double qs[4][3 * TS];
  pdl_wait();
  const int b = blockIdx.x, tid = threadIdx.x;
  const int grp = tid / (3 * TS), e = tid % (3 * TS);
  const int q = e / TS, r = e % TS;
  const int N = d.N;  // block b touches N tiles: (b, 0..b) then (b+1..N-1, b)
  const int k0 = (grp * N) / 4, k1 = ((grp + 1) * N) / 4;
  double s = 0.0;
  int k = k0;
  for (; k + 8 <= k1; k += 8) {
    double v[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const int kk = k + h;
      v[h] = kk <= b ? partial[(size_t)tidx(b, kk) * 6 * TS + q * TS + r]
                     : partial[(size_t)tidx(kk, b) * 6 * TS + 3 * TS + q * TS + r];
    }
#pragma unroll
    for (int h = 0; h < 8; ++h) s += v[h];
  }
  for (; k < k1; ++k)
    s += k <= b ? partial[(size_t)tidx(b, k) * 6 * TS + q * TS + r]
                : partial[(size_t)tidx(k, b) * 6 * TS + 3 * TS + q * TS + r];
  qs[grp][e] = s;
  __syncthreads();
  if (grp == 0) {
    const double tot = ((qs[0][e] + qs[1][e]) + qs[2][e]) + qs[3][e];
    const int row = b * TS + r;
    if (row < d.m) out[3 * row + q] = tot;
  }
  if (tid == 0) pdl_trigger();
}

// out[b] = sum over the tiles of block row/column b, in fixed order (loads
// unrolled so they are in flight together; the adds stay sequential)
__global__ void k_sym_gemv_reduce(DenseDev d, const double* __restrict__ partial, double* __restrict__ out) {
  const int b = blockIdx.x, tid = threadIdx.x;
  if (tid >= 3 * TS) return;
  const int q = tid / TS, r = tid % TS;
  double s = 0.0;
  int j = 0;
  for (; j + 8 <= b + 1; j += 8) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = partial[(size_t)tidx(b, j + k) * 6 * TS + q * TS + r];
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
  }
  for (; j <= b; ++j) s += partial[(size_t)tidx(b, j) * 6 * TS + q * TS + r];
  int i = b + 1;
  for (; i + 8 <= d.N; i += 8) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = partial[(size_t)tidx(i + k, b) * 6 * TS + 3 * TS + q * TS + r];
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
  }
  for (; i < d.N; ++i) s += partial[(size_t)tidx(i, b) * 6 * TS + 3 * TS + q * TS + r];
  int row = b * TS + r;
  if (row < d.m) out[3 * row + q] = s;
}

// ------------------------------------------------------------- launchers
void launch_cholesky_tiles(cudaStream_t st, const DenseDev& d, const int2* tasks, int ntasks, int grid, bool pdl) {
  static bool attr = false;
  size_t smem = cholesky_smem_bytes();
  if (!attr) {
    cudaFuncSetAttribute(k_cholesky_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  if (pdl) {
    launch_pdl(k_cholesky_tiles, dim3(grid), dim3(NTHREADS), smem, st, d, tasks, ntasks);
    return;
  }
  k_cholesky_tiles<<<grid, NTHREADS, smem, st>>>(d, tasks, ntasks);
}

void launch_cholesky(cudaStream_t st, const DenseDev& d, const int2* tasks, int ntasks, int grid, bool pdl,
                     bool int8) {
  if (!int8) {
    launch_cholesky_tiles(st, d, tasks, ntasks, grid, pdl);
    return;
  }
  static bool attr = false;
  size_t smem = cholesky_smem_bytes();
  if (!attr) {
    cudaFuncSetAttribute(k_cholesky_oz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  if (pdl) {
    launch_pdl(k_cholesky_oz, dim3(grid), dim3(NTHREADS), smem, st, d, tasks, ntasks);
    return;
  }
  k_cholesky_oz<<<grid, NTHREADS, smem, st>>>(d, tasks, ntasks);
}

void chol_int8_diag_nomma(int on) { cudaMemcpyToSymbol(g_oz_diag_nomma, &on, sizeof(int)); }

bool chol_int8_enabled() {
  static const bool on = !(getenv("SPB_CHOL_INT8") && getenv("SPB_CHOL_INT8")[0] == '0');
  return on;
}

void launch_cholesky_ranks(cudaStream_t st, const DenseRankJob* jobs, int P, int grid) {
  static bool attr = false;
  size_t smem = cholesky_smem_bytes();
  if (!attr) {
    cudaFuncSetAttribute(k_cholesky_ranks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_cholesky_ranks<<<grid, NTHREADS, smem, st>>>(jobs, P);
}

void dense_backward_preset(cudaStream_t st, const DenseDev& d, double* xrows) {
  cudaMemsetAsync(xrows, 0xff, sizeof(double) * 3 * TS * (size_t)d.N, st);  // BW_EMPTY everywhere
}

void launch_dense_backward(cudaStream_t st, const DenseDev& d, double* xrows, double* u,
                           unsigned long long* trace, bool preset) {
  static bool attr = false;
  const size_t smem = sizeof(double) * BW_SMEM_DOUBLES;
  if (!attr) {
    cudaFuncSetAttribute(k_dense_backward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  if (!preset) {
    dense_backward_preset(st, d, xrows);
    k_dense_backward<<<d.N, 256, smem, st>>>(d, xrows, u, d.m, trace, 0);
  } else {
    // rows preset off the path: start behind the factorization (PDL) and
    // wait on its tile flags, so the prologues run in its tail
    launch_pdl(k_dense_backward, dim3(d.N), dim3(256), smem, st, d, xrows, u, d.m, trace, 1);
  }
}

void launch_sym_tile_gemv(cudaStream_t st, const DenseDev& d, const double* u, double* partial) {
  k_sym_gemv_tiles<<<dense_tile_count(d.N), 256, 0, st>>>(d, u, partial);
}

void launch_sym_tile_gemv_reduce(cudaStream_t st, const DenseDev& d, const double* partial, double* out) {
  k_sym_gemv_reduce<<<d.N, 192, 0, st>>>(d, partial, out);
}

// out = sigma0 u: the streaming tile pass, then the fixed-order block sums
// (both programmatic launches when pdl).
void launch_sym_gemv(cudaStream_t st, const DenseDev& d, const double* u, double* partial, double* out, bool pdl,
                     int max_ctas) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sym_gemv_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SG_SMEM);
    attr = true;
  }
  static int per_sm = 0;
  if (!per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sym_gemv_stream, SG_THREADS, SG_SMEM);
    per_sm = std::max(1, std::min(per_sm, SG_CTAS_PER_SM));
  }
  int grid = std::min(dense_tile_count(d.N), NUM_SMS_B200 * per_sm);
  if (max_ctas > 0) grid = std::min(grid, max_ctas);  // results do not depend on the grid
  if (pdl) {
    launch_pdl(k_sym_gemv_stream, dim3(grid), dim3(SG_THREADS), SG_SMEM, st, d, u, partial);
    launch_pdl(k_sym_gemv_reduce4, dim3(d.N), dim3(4 * 3 * TS), 0, st, d, (const double*)partial, out);
    return;
  }
  k_sym_gemv_stream<<<grid, SG_THREADS, SG_SMEM, st>>>(d, u, partial);
  k_sym_gemv_reduce4<<<d.N, 4 * 3 * TS, 0, st>>>(d, partial, out);
}

// Task order: column-major (below-diagonal tiles, RHS row), with diagonal
// task d and the partial sum of its sub-diagonal tile (d, d-1) claimed
// `lead` columns ahead (optionally growing as lead + d / ldiv). A sweep on
// cfg3 (tools/chol_sweep.sh) found a fixed lead of 1-2 best (2.93 ms); a lead
// growing with d claims CTAs that then stall in the throughput-bound middle.
// At most 2 (lead + N / ldiv + 1) claimed tasks wait on unclaimed ones, far
// below the 148-CTA grid, so the order cannot deadlock.
std::vector<int2> cholesky_task_order(int N, bool with_rhs, int lead) {
  int ldiv = 1 << 30, pmode = 0;
  if (const char* e = getenv("SPB_CHOL_LEAD")) lead = atoi(e);  // diagnostics overrides
  if (const char* e = getenv("SPB_CHOL_LDIV")) ldiv = std::max(1, atoi(e));
  if (const char* e = getenv("SPB_CHOL_PMODE")) pmode = atoi(e);  // 1: partial heads its column
  std::vector<int2> tk;
  int next_diag = 0;
  for (int j = 0; j < N; ++j) {
    while (next_diag < N && next_diag - (lead + next_diag / ldiv) <= j) {
      if (next_diag > 0 && pmode == 0) tk.push_back(make_int2(next_diag, next_diag - 1));  // partial (d, d-1)
      tk.push_back(make_int2(next_diag, next_diag));
      ++next_diag;
    }
    if (pmode == 1 && j + 1 < N) tk.push_back(make_int2(j + 1, j));
    for (int i = j + 2; i < N; ++i) tk.push_back(make_int2(i, j));
    if (with_rhs) tk.push_back(make_int2(N, j));
  }
  return tk;
}

// Tile-cyclic ownership: column j belongs to rank j mod P, except the
// sub-diagonal partial (j+1, j), which belongs to the rank of diagonal j+1
// (the diagonal task finalizes it, so the partial never leaves that rank).
int dense_tile_owner(int i, int j, int nranks) { return (i == j + 1 ? i : j) % nranks; }

// A rank's tasks in the global claim order: every cross-rank dependency
// points to an earlier task of the global order, so with all ranks' CTAs
// resident the globally first unfinished task always progresses.
std::vector<int2> cholesky_rank_tasks(int N, int rank, int nranks, int lead) {
  std::vector<int2> all = cholesky_task_order(N, false, lead), mine;
  for (const int2& t : all)
    if (dense_tile_owner(t.x, t.y, nranks) == rank) mine.push_back(t);
  return mine;
}

}  // namespace spb
