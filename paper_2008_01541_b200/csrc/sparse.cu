// Sparse three-step-solve kernels on the prefactored interior
// (reference linalg.py:385-414 forward_sub / backward_sub with the
// numba column solves _lsolve/_ltsolve, linalg.py:203-223).
//
// The factor is supernodal with PARTITIONED-INVERSE panels (precompute.cpp):
// for supernode s with nc columns and nr rows, M_s = [inv(L_ss); L_b inv(L_ss)]
// (nr x nc, column-major). Then
//   forward : v_s = b_s + sum_children U_c (extend-add),
//             y_s = inv(L_ss) v_top,   U_s = v_below - W v_top
//   backward: x_s = inv(L_ss)^T y_s - W^T x_below
// i.e. ONE dense GEMV (3 RHS) per supernode; supernodes of the same
// elimination-tree height run concurrently (one launch per level). The x2
// rows of the panels are the coupling C, so the forward sweep also yields
// f~2 = f2 - C y1 and the backward sweep consumes C^T u2 (linalg.py:395, :408).
// Update vectors are pulled by their consumer in fixed child order: no float
// atomics, bitwise run-to-run determinism (test_solver.py:275-283).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace spb {

struct SnDev {
  int64_t valoff;
  int rowoff, nc, nr, first, uoff, pad;
};

struct LevelTasks {
  int cta_off, ncta, warp_off, nwarp;
  int max_nc;  // forward CTA tasks: columns staged in smem
};

struct DeviceFactor {
  int n1 = 0, n2 = 0, ns = 0, nlevels = 0;
  int64_t nrows_total = 0, urows = 0, nval = 0;
  SnDev* sn = nullptr;
  int* rows = nullptr;
  double* M = nullptr;
  int* asm_ptr = nullptr;
  int* asm_src = nullptr;
  int* x2_ptr = nullptr;
  int* x2_src = nullptr;
  int2* fw_cta = nullptr;   // (s, row0)
  int2* fw_warp = nullptr;  // (s, row0)
  int2* bw_cta = nullptr;   // (s, col0)
  int* bw_warp = nullptr;   // s
  std::vector<LevelTasks> fw, bw;
  ~DeviceFactor() {
    for (void* p : {(void*)sn, (void*)rows, (void*)M, (void*)asm_ptr, (void*)asm_src, (void*)x2_ptr,
                    (void*)x2_src, (void*)fw_cta, (void*)fw_warp, (void*)bw_cta, (void*)bw_warp})
      if (p) cudaFree(p);
  }
};

size_t device_factor_ubuf(const DeviceFactor& df) { return (size_t)df.urows; }
int device_factor_levels(const DeviceFactor& df) { return df.nlevels; }

constexpr int FW_ROWS = 32;     // rows per forward task
constexpr int BW_COLS = 16;     // columns per backward CTA task
constexpr int WARP_NC = 32;     // supernodes with nc <= this use warp tasks
constexpr int CH_FW = 4096;     // forward column chunk staged in smem
constexpr int CH_BW = 4096;     // backward row chunk staged in smem

// -------------------------------------------------------------- forward
__device__ __forceinline__ double asm_sum(const int* __restrict__ ap, const int* __restrict__ as,
                                          const double* __restrict__ U, int64_t p, int q, double init) {
  double v = init;
  for (int k = ap[p]; k < ap[p + 1]; ++k) v += U[3 * (int64_t)as[k] + q];
  return v;
}

__global__ void __launch_bounds__(256) k_forward_level(const SnDev* __restrict__ sn, const double* __restrict__ M,
                                                       const int* __restrict__ ap, const int* __restrict__ as,
                                                       const int2* __restrict__ cta_tasks, int ncta,
                                                       const int2* __restrict__ warp_tasks, int nwarp,
                                                       const double* __restrict__ b, double* __restrict__ y,
                                                       double* __restrict__ U) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if ((int)blockIdx.x < ncta) {
    // ---------------- CTA task: 32 rows, columns split over 8 warps
    const int2 tk = cta_tasks[blockIdx.x];
    const SnDev S = sn[tk.x];
    const int r = tk.y + lane;
    const bool valid = r < S.nr;
    const int cmax = (tk.y < S.nc) ? min(S.nc, tk.y + FW_ROWS) : S.nc;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    const double* Mp = M + S.valoff + r;
    for (int c0 = 0; c0 < cmax; c0 += CH_FW) {
      const int c1 = min(cmax, c0 + CH_FW);
      __syncthreads();
      for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
        int64_t p = (int64_t)S.rowoff + c;
        int gi = S.first + c;
#pragma unroll
        for (int q = 0; q < 3; ++q) sm[3 * (c - c0) + q] = asm_sum(ap, as, U, p, q, b[3 * (int64_t)gi + q]);
      }
      __syncthreads();
      if (valid) {
        int c = c0 + warp;
#pragma unroll 4
        for (; c < c1; c += 8) {
          double mv = Mp[(int64_t)c * S.nr];
          const double* v = sm + 3 * (c - c0);
          a0 += mv * v[0];
          a1 += mv * v[1];
          a2 += mv * v[2];
        }
      }
    }
    __syncthreads();
    double* red = sm;  // [8][32][3]
    red[(warp * 32 + lane) * 3 + 0] = a0;
    red[(warp * 32 + lane) * 3 + 1] = a1;
    red[(warp * 32 + lane) * 3 + 2] = a2;
    __syncthreads();
    if (threadIdx.x < 96) {
      const int rl = threadIdx.x / 3, q = threadIdx.x % 3;
      const int rr = tk.y + rl;
      if (rr < S.nr) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += red[(w * 32 + rl) * 3 + q];
        if (rr < S.nc) {
          y[3 * (int64_t)(S.first + rr) + q] = s;
        } else {
          double vb = asm_sum(ap, as, U, (int64_t)S.rowoff + rr, q, 0.0);
          U[3 * (int64_t)(S.uoff + rr - S.nc) + q] = vb - s;
        }
      }
    }
  } else {
    // ---------------- warp task: whole small panel row block in one warp
    const int t = ((int)blockIdx.x - ncta) * 8 + warp;
    if (t >= nwarp) return;
    const int2 tk = warp_tasks[t];
    const SnDev S = sn[tk.x];
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    if (lane < S.nc) {
      int64_t p = (int64_t)S.rowoff + lane;
      int gi = S.first + lane;
      v0 = asm_sum(ap, as, U, p, 0, b[3 * (int64_t)gi + 0]);
      v1 = asm_sum(ap, as, U, p, 1, b[3 * (int64_t)gi + 1]);
      v2 = asm_sum(ap, as, U, p, 2, b[3 * (int64_t)gi + 2]);
    }
    const int r = tk.y + lane;
    const bool valid = r < S.nr;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    const double* Mp = M + S.valoff + (valid ? r : 0);
    for (int c = 0; c < S.nc; ++c) {
      double mv = valid ? Mp[(int64_t)c * S.nr] : 0.0;
      a0 += mv * __shfl_sync(0xffffffffu, v0, c);
      a1 += mv * __shfl_sync(0xffffffffu, v1, c);
      a2 += mv * __shfl_sync(0xffffffffu, v2, c);
    }
    if (valid) {
      if (r < S.nc) {
        y[3 * (int64_t)(S.first + r) + 0] = a0;
        y[3 * (int64_t)(S.first + r) + 1] = a1;
        y[3 * (int64_t)(S.first + r) + 2] = a2;
      } else {
        int64_t p = (int64_t)S.rowoff + r;
        int64_t o = 3 * (int64_t)(S.uoff + r - S.nc);
        U[o + 0] = asm_sum(ap, as, U, p, 0, 0.0) - a0;
        U[o + 1] = asm_sum(ap, as, U, p, 1, 0.0) - a1;
        U[o + 2] = asm_sum(ap, as, U, p, 2, 0.0) - a2;
      }
    }
  }
}

// f~2[k] = f2[k] + sum of root update entries on x2 row k (= f2 - C y1).
__global__ void k_forward_x2(int n1, int n2, const int* __restrict__ xp, const int* __restrict__ xs,
                             const double* __restrict__ U, const double* __restrict__ b, double* __restrict__ f2) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= 3 * n2) return;
  int row = k / 3, q = k % 3;
  double v = b[3 * (int64_t)(n1 + row) + q];
  for (int t = xp[row]; t < xp[row + 1]; ++t) v += U[3 * (int64_t)xs[t] + q];
  f2[k] = v;
}

// ------------------------------------------------------------- backward
// XF: (n,3) with rows [0,n1) = x1 solution (being produced), [n1,n) = x2 input.
__global__ void __launch_bounds__(256) k_backward_level(const SnDev* __restrict__ sn, const double* __restrict__ M,
                                                        const int* __restrict__ rows,
                                                        const int2* __restrict__ cta_tasks, int ncta,
                                                        const int* __restrict__ warp_tasks, int nwarp,
                                                        const double* __restrict__ y, double* __restrict__ XF) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if ((int)blockIdx.x < ncta) {
    const int2 tk = cta_tasks[blockIdx.x];
    const SnDev S = sn[tk.x];
    const int* rw = rows + S.rowoff;
    double acc[2][3] = {{0, 0, 0}, {0, 0, 0}};
    const int cA = tk.y + warp * 2;
    // rows < c never contribute to column c (inv(L_ss) is lower triangular)
    const int rstart = tk.y;
    for (int r0 = rstart; r0 < S.nr; r0 += CH_BW) {
      const int r1 = min(S.nr, r0 + CH_BW);
      __syncthreads();
      for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        if (r < S.nc) {
#pragma unroll
          for (int q = 0; q < 3; ++q) sm[3 * (r - r0) + q] = y[3 * (int64_t)(S.first + r) + q];
        } else {
          const int64_t g = rw[r];
#pragma unroll
          for (int q = 0; q < 3; ++q) sm[3 * (r - r0) + q] = -XF[3 * g + q];
        }
      }
      __syncthreads();
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const int c = cA + cc;
        if (c >= S.nc) continue;
        const double* Mc = M + S.valoff + (int64_t)c * S.nr;
        for (int r = max(r0, c) + lane; r < r1; r += 32) {
          double mv = Mc[r];
          const double* z = sm + 3 * (r - r0);
          acc[cc][0] += mv * z[0];
          acc[cc][1] += mv * z[1];
          acc[cc][2] += mv * z[2];
        }
      }
    }
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      const int c = cA + cc;
      double s0 = warp_sum(acc[cc][0]), s1 = warp_sum(acc[cc][1]), s2 = warp_sum(acc[cc][2]);
      if (lane == 0 && c < S.nc) {
        XF[3 * (int64_t)(S.first + c) + 0] = s0;
        XF[3 * (int64_t)(S.first + c) + 1] = s1;
        XF[3 * (int64_t)(S.first + c) + 2] = s2;
      }
    }
  } else {
    const int t = ((int)blockIdx.x - ncta) * 8 + warp;
    if (t >= nwarp) return;
    const SnDev S = sn[warp_tasks[t]];
    const int* rw = rows + S.rowoff;
    const int c = lane;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    const double* Mc = M + S.valoff + (int64_t)(c < S.nc ? c : 0) * S.nr;
    for (int r = 0; r < S.nr; ++r) {
      double z0, z1, z2;
      if (r < S.nc) {
        z0 = y[3 * (int64_t)(S.first + r) + 0];
        z1 = y[3 * (int64_t)(S.first + r) + 1];
        z2 = y[3 * (int64_t)(S.first + r) + 2];
      } else {
        const int64_t g = rw[r];
        z0 = -XF[3 * g + 0];
        z1 = -XF[3 * g + 1];
        z2 = -XF[3 * g + 2];
      }
      if (c < S.nc && r >= c) {
        double mv = Mc[r];
        a0 += mv * z0;
        a1 += mv * z1;
        a2 += mv * z2;
      }
    }
    if (c < S.nc) {
      XF[3 * (int64_t)(S.first + c) + 0] = a0;
      XF[3 * (int64_t)(S.first + c) + 1] = a1;
      XF[3 * (int64_t)(S.first + c) + 2] = a2;
    }
  }
}

// ---------------------------------------------------------------- host
template <typename T>
static int upload(T** dst, const std::vector<T>& v) {
  size_t bytes = sizeof(T) * std::max<size_t>(v.size(), 1);
  SPB_CUDA(cudaMalloc(dst, bytes));
  if (!v.empty()) SPB_CUDA(cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return SPB_OK;
}

int build_device_factor(Factor& f) {
  if (f.dev) return SPB_OK;
  auto* d = new DeviceFactor();
  const int64_t ns = f.nsuper;
  d->n1 = (int)f.n1;
  d->n2 = (int)f.n2;
  d->ns = (int)ns;
  d->nlevels = (int)f.nlevels;
  d->nrows_total = f.sn_rowptr.empty() ? 0 : f.sn_rowptr[ns];
  d->nval = f.sn_valptr.empty() ? 0 : f.sn_valptr[ns];
  if (d->nrows_total >= (int64_t)1 << 31) { delete d; set_error("factor too large (row index > 2^31)"); return SPB_ERR_SETUP; }
  std::vector<SnDev> sn(ns);
  int64_t uoff = 0;
  for (int64_t s = 0; s < ns; ++s) {
    SnDev& S = sn[s];
    S.valoff = f.sn_valptr[s];
    S.rowoff = (int)f.sn_rowptr[s];
    S.nc = (int)(f.sn_first[s + 1] - f.sn_first[s]);
    S.nr = (int)(f.sn_rowptr[s + 1] - f.sn_rowptr[s]);
    S.first = (int)f.sn_first[s];
    S.uoff = (int)uoff;
    S.pad = 0;
    uoff += S.nr - S.nc;
  }
  d->urows = uoff;
  std::vector<int> rows(d->nrows_total);
  for (int64_t k = 0; k < d->nrows_total; ++k) rows[k] = (int)f.sn_rows[k];
  // forward extend-add maps (children in ascending order)
  std::vector<std::vector<int64_t>> children(ns);
  for (int64_t s = 0; s < ns; ++s)
    if (f.sn_parent[s] >= 0) children[f.sn_parent[s]].push_back(s);
  std::vector<int> cnt(d->nrows_total + 1, 0);
  std::vector<int> xcnt(f.n2 + 1, 0);
  std::vector<int> pos(f.n, -1);
  auto for_each_map = [&](auto&& emit) {
    for (int64_t s = 0; s < ns; ++s) {
      const SnDev& S = sn[s];
      for (int k = 0; k < S.nr; ++k) pos[rows[S.rowoff + k]] = k;
      for (int64_t c : children[s]) {
        const SnDev& C = sn[c];
        for (int q = 0; q < C.nr - C.nc; ++q) {
          int p = pos[rows[C.rowoff + C.nc + q]];
          emit(false, (int64_t)S.rowoff + p, C.uoff + q);
        }
      }
      for (int k = 0; k < S.nr; ++k) pos[rows[S.rowoff + k]] = -1;
    }
    for (int64_t s = 0; s < ns; ++s) {
      if (f.sn_parent[s] >= 0) continue;
      const SnDev& C = sn[s];
      for (int q = 0; q < C.nr - C.nc; ++q) emit(true, rows[C.rowoff + C.nc + q] - f.n1, C.uoff + q);
    }
  };
  for_each_map([&](bool x2, int64_t p, int) {
    if (x2) xcnt[p + 1]++; else cnt[p + 1]++;
  });
  for (int64_t k = 0; k < d->nrows_total; ++k) cnt[k + 1] += cnt[k];
  for (int64_t k = 0; k < f.n2; ++k) xcnt[k + 1] += xcnt[k];
  std::vector<int> asrc(cnt[d->nrows_total]), xsrc(xcnt[f.n2]);
  {
    std::vector<int> fill(cnt.begin(), cnt.end() - 1), xfill(xcnt.begin(), xcnt.end() - 1);
    for_each_map([&](bool x2, int64_t p, int src) {
      if (x2) xsrc[xfill[p]++] = src; else asrc[fill[p]++] = src;
    });
  }
  // level task lists
  std::vector<std::vector<int64_t>> bylevel(f.nlevels);
  for (int64_t s = 0; s < ns; ++s) bylevel[f.sn_level[s]].push_back(s);
  std::vector<int2> fwc, fww, bwc;
  std::vector<int> bww;
  d->fw.resize(f.nlevels);
  d->bw.resize(f.nlevels);
  for (int64_t l = 0; l < f.nlevels; ++l) {
    LevelTasks& F = d->fw[l];
    LevelTasks& B = d->bw[l];
    F.cta_off = (int)fwc.size();
    F.warp_off = (int)fww.size();
    B.cta_off = (int)bwc.size();
    B.warp_off = (int)bww.size();
    F.max_nc = 0;
    for (int64_t s : bylevel[l]) {
      const SnDev& S = sn[s];
      bool small = S.nc <= WARP_NC;
      for (int r0 = 0; r0 < S.nr; r0 += FW_ROWS) {
        if (small) fww.push_back(make_int2((int)s, r0));
        else fwc.push_back(make_int2((int)s, r0));
      }
      if (!small) F.max_nc = std::max(F.max_nc, S.nc);
      if (small) bww.push_back((int)s);
      else
        for (int c0 = 0; c0 < S.nc; c0 += BW_COLS) bwc.push_back(make_int2((int)s, c0));
    }
    F.ncta = (int)fwc.size() - F.cta_off;
    F.nwarp = (int)fww.size() - F.warp_off;
    B.ncta = (int)bwc.size() - B.cta_off;
    B.nwarp = (int)bww.size() - B.warp_off;
  }
  int rc;
  if ((rc = upload(&d->sn, sn)) || (rc = upload(&d->rows, rows)) || (rc = upload(&d->M, f.Mval)) ||
      (rc = upload(&d->asm_ptr, cnt)) || (rc = upload(&d->asm_src, asrc)) || (rc = upload(&d->x2_ptr, xcnt)) ||
      (rc = upload(&d->x2_src, xsrc)) || (rc = upload(&d->fw_cta, fwc)) || (rc = upload(&d->fw_warp, fww)) ||
      (rc = upload(&d->bw_cta, bwc)) || (rc = upload(&d->bw_warp, bww))) {
    delete d;
    return rc;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_forward_level, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * CH_FW * 8 + 64);
    cudaFuncSetAttribute(k_backward_level, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * CH_BW * 8 + 64);
    attr = true;
  }
  f.dev = d;
  return SPB_OK;
}

void sparse_forward(cudaStream_t st, const DeviceFactor& d, const double* b, double* y, double* U, double* f2,
                    int* launches) {
  for (int l = 0; l < d.nlevels; ++l) {
    const LevelTasks& T = d.fw[l];
    int grid = T.ncta + (T.nwarp + 7) / 8;
    if (grid == 0) continue;
    size_t smem = T.ncta ? std::max<size_t>(sizeof(double) * 3 * std::min(T.max_nc, CH_FW), 8 * 32 * 3 * 8) : 0;
    k_forward_level<<<grid, 256, smem, st>>>(d.sn, d.M, d.asm_ptr, d.asm_src, d.fw_cta + T.cta_off, T.ncta,
                                             d.fw_warp + T.warp_off, T.nwarp, b, y, U);
    if (launches) ++*launches;
  }
  if (d.n2 > 0) {
    k_forward_x2<<<ceil_div(3 * (int64_t)d.n2, 256), 256, 0, st>>>(d.n1, d.n2, d.x2_ptr, d.x2_src, U, b, f2);
    if (launches) ++*launches;
  }
}

void sparse_backward(cudaStream_t st, const DeviceFactor& d, const double* y, double* XF, int* launches) {
  for (int l = d.nlevels - 1; l >= 0; --l) {
    const LevelTasks& T = d.bw[l];
    int grid = T.ncta + (T.nwarp + 7) / 8;
    if (grid == 0) continue;
    size_t smem = T.ncta ? sizeof(double) * 3 * CH_BW : 0;
    k_backward_level<<<grid, 256, smem, st>>>(d.sn, d.M, d.rows, d.bw_cta + T.cta_off, T.ncta,
                                              d.bw_warp + T.warp_off, T.nwarp, y, XF);
    if (launches) ++*launches;
  }
}

}  // namespace spb

spb::Factor::~Factor() { delete dev; }
