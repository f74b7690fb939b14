// Inner-loop bookkeeping and end-of-frame metrics (reference
// solver.py:435-440 and _finish_metrics solver.py:373-384):
//   x2 += u2;  f~2 -= sigma0 u2 - K22_beta u2;  u2_accum += u2;
//   residual = |H u2 - g| / max(|g|, tiny) with H u2 = sigma0 u2 + C22 u2;
//   x1 += u1 after the backward sweep; energy / penetration / active count.
// All reductions are fixed-order (block partials, single-block finish).
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"

namespace spb {

// v_j = c_j * (w_j . u2[local nodes of j]) for active proxies (C22 u2 = W^T diag(c) W u2)
__global__ void k_proxy_wu(ProxyDev px, const uint8_t* __restrict__ active, const double* __restrict__ u2,
                           double* __restrict__ v) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= px.P) return;
  double s0 = 0, s1 = 0, s2 = 0;
  if (active[j]) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      double wb = px.w[4 * j + b];
      int l = px.local[4 * j + b];
      s0 += wb * u2[3 * l + 0];
      s1 += wb * u2[3 * l + 1];
      s2 += wb * u2[3 * l + 2];
    }
    double c = px.c[j];
    s0 *= c; s1 *= c; s2 *= c;
  }
  v[3 * j + 0] = s0;
  v[3 * j + 1] = s1;
  v[3 * j + 2] = s2;
}

__global__ void __launch_bounds__(256) k_inner_update(int m, const double* __restrict__ u2,
                                                      const double* __restrict__ s0u, const int* __restrict__ kptr,
                                                      const int* __restrict__ kidx, const double* __restrict__ kval,
                                                      const double* __restrict__ g, const double* __restrict__ pw,
                                                      const double* __restrict__ vprox, const int* __restrict__ cptr,
                                                      const int* __restrict__ csrc, double* __restrict__ f_tilde2,
                                                      double* __restrict__ u2acc, double* __restrict__ x,
                                                      const int* __restrict__ x2_ids,
                                                      double* __restrict__ rpartial /* 2 per block */) {
  __shared__ double sr[8], sg[8];
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  double rr = 0.0, gg = 0.0;
  if (k < m) {
    double ku[3] = {0, 0, 0};
    for (int q = kptr[k]; q < kptr[k + 1]; ++q) {
      double a = kval[q];
      int c = kidx[q];
      ku[0] += a * u2[3 * c + 0];
      ku[1] += a * u2[3 * c + 1];
      ku[2] += a * u2[3 * c + 2];
    }
    double cu[3] = {0, 0, 0};
    for (int q = cptr[k]; q < cptr[k + 1]; ++q) {
      int s = csrc[q];
      int j = s >> 2, a = s & 3;
      double wa = pw[4 * j + a];
      cu[0] += wa * vprox[3 * j + 0];
      cu[1] += wa * vprox[3 * j + 1];
      cu[2] += wa * vprox[3 * j + 2];
    }
    const int64_t node = x2_ids[k];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      double u = u2[3 * k + q];
      double s = s0u[3 * k + q];
      double r = (s + cu[q]) - g[3 * k + q];
      rr += r * r;
      gg += g[3 * k + q] * g[3 * k + q];
      x[3 * node + q] += u;
      f_tilde2[3 * k + q] -= s - ku[q];
      if (u2acc) u2acc[3 * k + q] += u;  // null: k_u2acc_to_xf already did it
    }
  }
  rr = warp_sum(rr);
  gg = warp_sum(gg);
  if ((threadIdx.x & 31) == 0) {
    sr[threadIdx.x >> 5] = rr;
    sg[threadIdx.x >> 5] = gg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < 8; ++w) { a += sr[w]; b += sg[w]; }
    rpartial[2 * blockIdx.x + 0] = a;
    rpartial[2 * blockIdx.x + 1] = b;
  }
}

// x[node(k)] += X[k] for the x1 rows in factor order (linalg.py:411 scatter back
// through fill_perm, solver.py:445).
__global__ void k_scatter_add(int cnt, const int* __restrict__ node, const double* __restrict__ X,
                              double* __restrict__ x) {
  pdl_wait();  // X of the backward sweep's last launch
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= 3 * cnt) return;
  int row = k / 3, q = k % 3;
  x[3 * (int64_t)node[row] + q] += X[k];
}

// b-vector gather for the one-shot ops: out[k] = src[idx[k]] (3 columns)
__global__ void k_gather3(int cnt, const int* __restrict__ idx, const double* __restrict__ src,
                          double* __restrict__ out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= 3 * cnt) return;
  out[k] = src[3 * (int64_t)idx[k / 3] + k % 3];
}

__global__ void __launch_bounds__(256) k_attachment_energy(int na, const int* __restrict__ nodes,
                                                           const double* __restrict__ ak,
                                                           const double* __restrict__ tgt,
                                                           const double* __restrict__ x,
                                                           double* __restrict__ partial) {
  __shared__ double red[8];
  int a = blockIdx.x * blockDim.x + threadIdx.x;
  double e = 0.0;
  if (a < na) {
    int64_t i = nodes[a];
    double d0 = x[3 * i + 0] - tgt[3 * a + 0], d1 = x[3 * i + 1] - tgt[3 * a + 1], d2 = x[3 * i + 2] - tgt[3 * a + 2];
    e = 0.5 * ak[a] * ((d0 * d0 + d1 * d1) + d2 * d2);
  }
  e = warp_sum(e);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    partial[blockIdx.x] = s;
  }
}

// out[0] energy, [1] max penetration, [2] residual, [3] active count
__global__ void k_finish_metrics(const double* __restrict__ e_part, int ne_b, const double* __restrict__ a_part,
                                 int na_b, const double* __restrict__ p_part, int np_b,
                                 const double* __restrict__ r_part, int nr_b, const uint8_t* __restrict__ active,
                                 int P, int have_residual, double* __restrict__ out) {
  __shared__ double s_e[256], s_a[256], s_p[256], s_d[256], s_r[256], s_g[256], s_c[256];
  const int t = threadIdx.x;
  double e = 0, a = 0, p = 0, dmax = 0, rr = 0, gg = 0, cnt = 0;
  for (int i = t; i < ne_b; i += 256) e += e_part[i];
  for (int i = t; i < na_b; i += 256) a += a_part[i];
  for (int i = t; i < np_b; i += 256) {
    p += p_part[2 * i];
    dmax = fmax(dmax, p_part[2 * i + 1]);
  }
  for (int i = t; i < nr_b; i += 256) {
    rr += r_part[2 * i];
    gg += r_part[2 * i + 1];
  }
  for (int i = t; i < P; i += 256) cnt += active[i] ? 1.0 : 0.0;
  s_e[t] = e; s_a[t] = a; s_p[t] = p; s_d[t] = dmax; s_r[t] = rr; s_g[t] = gg; s_c[t] = cnt;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (t < o) {
      s_e[t] += s_e[t + o]; s_a[t] += s_a[t + o]; s_p[t] += s_p[t + o];
      s_d[t] = fmax(s_d[t], s_d[t + o]);
      s_r[t] += s_r[t + o]; s_g[t] += s_g[t + o]; s_c[t] += s_c[t + o];
    }
    __syncthreads();
  }
  if (t == 0) {
    out[0] = (s_e[0] + s_a[0]) + 0.5 * s_p[0];
    out[1] = s_d[0];
    if (have_residual) out[2] = sqrt(s_r[0]) / fmax(sqrt(s_g[0]), DBL_MIN);
    out[3] = s_c[0];
  }
}

// ------------------------------------------------------------- launchers
void launch_proxy_wu(cudaStream_t st, const ProxyDev& px, const uint8_t* active, const double* u2, double* v) {
  if (px.P <= 0) return;
  k_proxy_wu<<<ceil_div(px.P, 128), 128, 0, st>>>(px, active, u2, v);
}

int update_blocks(int m) { return m > 0 ? ceil_div(m, 256) : 0; }

void launch_inner_update(cudaStream_t st, int m, const double* u2, const double* s0u, const int* kptr,
                         const int* kidx, const double* kval, const double* g, const double* pw, const double* v,
                         const int* cptr, const int* csrc, double* f_tilde2, double* u2acc, double* x,
                         const int* x2_ids, double* rpartial) {
  if (m <= 0) return;
  k_inner_update<<<update_blocks(m), 256, 0, st>>>(m, u2, s0u, kptr, kidx, kval, g, pw, v, cptr, csrc, f_tilde2,
                                                   u2acc, x, x2_ids, rpartial);
}

// The last inner pass's u2_accum upkeep, split off k_inner_update so the
// backward sweep can start while the sigma0 mat-vec and the f~2 upkeep run on
// a second stream: u2acc += u2 (the same single add), XF's x2 rows = u2acc.
__global__ void k_u2acc_to_xf(int m3, const double* __restrict__ u2, double* __restrict__ u2acc,
                              double* __restrict__ xf2) {
  if (threadIdx.x == 0) pdl_trigger();  // the backward sweep's first launch may follow
  pdl_wait();                           // u2 of the dense backward
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m3) return;
  const double v = u2acc[k] + u2[k];
  u2acc[k] = v;
  xf2[k] = v;
}

void launch_u2acc_to_xf(cudaStream_t st, int m, const double* u2, double* u2acc, double* xf2) {
  if (m <= 0) return;
  launch_pdl(k_u2acc_to_xf, dim3(ceil_div(3 * (int64_t)m, 256)), dim3(256), 0, st, 3 * m, u2, u2acc, xf2);
}

void launch_scatter_add(cudaStream_t st, int cnt, const int* node, const double* X, double* x) {
  if (cnt <= 0) return;
  launch_pdl(k_scatter_add, dim3(ceil_div(3 * (int64_t)cnt, 256)), dim3(256), 0, st, cnt, node, X, x);
}

void launch_gather3(cudaStream_t st, int cnt, const int* idx, const double* src, double* out) {
  if (cnt <= 0) return;
  k_gather3<<<ceil_div(3 * (int64_t)cnt, 256), 256, 0, st>>>(cnt, idx, src, out);
}

int attachment_blocks(int na) { return na > 0 ? ceil_div(na, 256) : 0; }

void launch_attachment_energy(cudaStream_t st, int na, const int* nodes, const double* k, const double* tgt,
                              const double* x, double* partial) {
  if (na <= 0) return;
  k_attachment_energy<<<attachment_blocks(na), 256, 0, st>>>(na, nodes, k, tgt, x, partial);
}

void launch_finish_metrics(cudaStream_t st, const double* e_part, int ne_b, const double* a_part, int na_b,
                           const double* p_part, int np_b, const double* r_part, int nr_b, const uint8_t* active,
                           int P, int have_residual, double* out) {
  k_finish_metrics<<<1, 256, 0, st>>>(e_part, ne_b, a_part, na_b, p_part, np_b, r_part, nr_b, active, P,
                                      have_residual, out);
}

}  // namespace spb
