// Element kernels: deformation gradient, sign-carrying 3x3 SVD, best-fit
// rotation / bi-phasic projection, Piola stress and per-element node forces,
// deterministic node gathers, and the elastic energy.
//
// Compiled with -fmad=false: every product/sum below is evaluated in the
// reference's order and rounding (numba kernels are non-fused LLVM;
// numpy's stacked 3x3 matmul is the fused chain fma(a2,b2,fma(a1,b1,a0*b0)),
// written explicitly). Rotations are therefore bit-identical to the
// reference on identical x (tests/test_gpu_parity.py::test_svd_bitwise).
//
// Reference: material.py:69-245 (SVD, R, Q), mesh.py:239-244 (F),
// material.py:328-378 (forces, energy), solver.py:327-346 (beta forces).
#include "common.cuh"
#include "kernels.cuh"

namespace spb {

// F = Ds * Dm^-1 with numpy's fused chain per entry (mesh.py:243-244).
__device__ __forceinline__ void deformation_gradient(const double* __restrict__ x, int4 t,
                                                     const double* __restrict__ dmi, int64_t ne, int64_t e,
                                                     double F[9]) {
  double x0[3], ds[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i) x0[i] = x[3 * (int64_t)t.x + i];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    ds[i][0] = x[3 * (int64_t)t.y + i] - x0[i];
    ds[i][1] = x[3 * (int64_t)t.z + i] - x0[i];
    ds[i][2] = x[3 * (int64_t)t.w + i] - x0[i];
  }
  double D[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) D[c] = dmi[c * ne + e];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) F[3 * i + j] = fma(ds[i][2], D[6 + j], fma(ds[i][1], D[3 + j], ds[i][0] * D[j]));
}

// Cyclic Jacobi on A = F^T F (material.py:69-113), non-fused arithmetic.
__device__ __forceinline__ void jacobi_eigh3(double A[3][3], double V[3][3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) V[i][j] = (i == j) ? 1.0 : 0.0;
  double scale = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double a = fabs(A[i][j]);
      scale = (a > scale) ? a : scale;
    }
  if (scale == 0.0) return;
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = fabs(A[0][1]) + fabs(A[0][2]) + fabs(A[1][2]);
    if (off <= 1e-30 * scale) break;
#pragma unroll
    for (int pq = 0; pq < 3; ++pq) {
      const int p = (pq < 2) ? 0 : 1;
      const int q = (pq == 0) ? 1 : 2;
      double apq = A[p][q];
      if (apq == 0.0) continue;
      double tau = (A[q][q] - A[p][p]) / (2.0 * apq);
      double t = (tau >= 0.0) ? 1.0 / (tau + sqrt(1.0 + tau * tau)) : -1.0 / (-tau + sqrt(1.0 + tau * tau));
      double c = 1.0 / sqrt(1.0 + t * t);
      double s = t * c;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double akp = A[k][p], akq = A[k][q];
        A[k][p] = c * akp - s * akq;
        A[k][q] = s * akp + c * akq;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double apk = A[p][k], aqk = A[q][k];
        A[p][k] = c * apk - s * aqk;
        A[q][k] = s * apk + c * aqk;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double vkp = V[k][p], vkq = V[k][q];
        V[k][p] = c * vkp - s * vkq;
        V[k][q] = s * vkp + c * vkq;
      }
    }
  }
}

// Sign-carrying SVD of one F (row-major), material.py:116-221.
__device__ void signed_svd(const double f[9], double u[9], double S[3], double v[9]) {
  double A[3][3], Ve[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) acc += f[3 * k + i] * f[3 * k + j];
      A[i][j] = acc;
    }
  jacobi_eigh3(A, Ve);
  double d0 = A[0][0], d1 = A[1][1], d2 = A[2][2], tmp;
  int i0 = 0, i1 = 1, i2 = 2, ti;
  if (d1 > d0) { tmp = d0; d0 = d1; d1 = tmp; ti = i0; i0 = i1; i1 = ti; }
  if (d2 > d0) { tmp = d0; d0 = d2; d2 = tmp; ti = i0; i0 = i2; i2 = ti; }
  if (d2 > d1) { tmp = d1; d1 = d2; d2 = tmp; ti = i1; i1 = i2; i2 = ti; }
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    v[3 * r + 0] = Ve[r][i0];
    v[3 * r + 1] = Ve[r][i1];
    v[3 * r + 2] = Ve[r][i2];
  }
  double detv = v[0] * (v[4] * v[8] - v[5] * v[7]) - v[1] * (v[3] * v[8] - v[5] * v[6]) +
                v[2] * (v[3] * v[7] - v[4] * v[6]);
  if (detv < 0.0) {
    v[2] = -v[2];
    v[5] = -v[5];
    v[8] = -v[8];
  }
  double w0x = f[0] * v[0] + f[1] * v[3] + f[2] * v[6];
  double w0y = f[3] * v[0] + f[4] * v[3] + f[5] * v[6];
  double w0z = f[6] * v[0] + f[7] * v[3] + f[8] * v[6];
  double s0 = sqrt(w0x * w0x + w0y * w0y + w0z * w0z);
  if (s0 <= 1e-300) {
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      u[c] = (c % 4 == 0) ? 1.0 : 0.0;
      v[c] = (c % 4 == 0) ? 1.0 : 0.0;
    }
    S[0] = S[1] = S[2] = 0.0;
    return;
  }
  u[0] = w0x / s0;
  u[3] = w0y / s0;
  u[6] = w0z / s0;
  double w1x = f[0] * v[1] + f[1] * v[4] + f[2] * v[7];
  double w1y = f[3] * v[1] + f[4] * v[4] + f[5] * v[7];
  double w1z = f[6] * v[1] + f[7] * v[4] + f[8] * v[7];
  double dot01 = u[0] * w1x + u[3] * w1y + u[6] * w1z;
  w1x -= dot01 * u[0];
  w1y -= dot01 * u[3];
  w1z -= dot01 * u[6];
  double n1 = sqrt(w1x * w1x + w1y * w1y + w1z * w1z);
  double s1;
  if (n1 > 1e-12 * s0) {
    u[1] = w1x / n1;
    u[4] = w1y / n1;
    u[7] = w1z / n1;
    s1 = n1;
  } else {
    double ax = fabs(u[0]), ay = fabs(u[3]), az = fabs(u[6]);
    double tx, ty, tz;
    if (ax <= ay && ax <= az) { tx = 1.0; ty = 0.0; tz = 0.0; }
    else if (ay <= az) { tx = 0.0; ty = 1.0; tz = 0.0; }
    else { tx = 0.0; ty = 0.0; tz = 1.0; }
    double dt = u[0] * tx + u[3] * ty + u[6] * tz;
    tx -= dt * u[0];
    ty -= dt * u[3];
    tz -= dt * u[6];
    double nt = sqrt(tx * tx + ty * ty + tz * tz);
    u[1] = tx / nt;
    u[4] = ty / nt;
    u[7] = tz / nt;
    s1 = 0.0;
  }
  u[2] = u[3] * u[7] - u[6] * u[4];
  u[5] = u[6] * u[1] - u[0] * u[7];
  u[8] = u[0] * u[4] - u[3] * u[1];
  S[0] = s0;
  S[1] = s1;
  double w2x = f[0] * v[2] + f[1] * v[5] + f[2] * v[8];
  double w2y = f[3] * v[2] + f[4] * v[5] + f[5] * v[8];
  double w2z = f[6] * v[2] + f[7] * v[5] + f[8] * v[8];
  S[2] = u[2] * w2x + u[5] * w2y + u[8] * w2z;
}

__device__ __forceinline__ void uvt(const double u[9], const double v[9], double R[9]) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) acc += u[3 * r + k] * v[3 * c + k];
      R[3 * r + c] = acc;
    }
}

__device__ __forceinline__ void udvt(const double u[9], const double S[3], const double v[9], double smin,
                                     double smax, double Q[9]) {
  double s[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) s[k] = fmin(fmax(S[k], smin), smax);  // np.clip (material.py:287)
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 3; ++k) acc += u[3 * r + k] * s[k] * v[3 * c + k];
      Q[3 * r + c] = acc;
    }
}

// Piola stress and the 4 node forces of one element (material.py:347-356).
__device__ __forceinline__ void element_forces(const double F[9], const double R[9], const double* Q,
                                               const double D[9], double vol, const ElemParams& p,
                                               double out[12]) {
  double P[9];
  const double two_mu = 2.0 * p.mu;
#pragma unroll
  for (int c = 0; c < 9; ++c) P[c] = two_mu * (F[c] - R[c]);
  if (Q) {
    const double two_mup = 2.0 * p.mu_prime;
#pragma unroll
    for (int c = 0; c < 9; ++c) P[c] = P[c] + two_mup * (F[c] - Q[c]);
  }
  const double nv = -vol;
  double G[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      G[i][j] = nv * fma(P[3 * i + 2], D[3 * j + 2], fma(P[3 * i + 1], D[3 * j + 1], P[3 * i + 0] * D[3 * j + 0]));
#pragma unroll
  for (int i = 0; i < 3; ++i) out[i] = -((G[i][0] + G[i][1]) + G[i][2]);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int i = 0; i < 3; ++i) out[3 * (a + 1) + i] = G[i][a];
}

// One thread per element of the subset: R (and Q) <- polar(F), and the
// per-element node forces G (SoA: G[(slot*3+d)*nsub + i]).
// 6 CTAs per SM (80 registers, a small L1-resident spill): the Jacobi SVD is
// FP64-latency bound, and 24 instead of 16 resident warps per SM take the
// alpha step from ~195 to ~186 us at cfg3 (alternated A/B, tools/lib_ab.sh)
__global__ void __launch_bounds__(128, 6) k_local_forces(int nsub, const int* __restrict__ sub,
                                                      const int4* __restrict__ tets, const double* __restrict__ x,
                                                      const double* __restrict__ dmi,
                                                      const double* __restrict__ vol, int64_t ne,
                                                      double* __restrict__ R, double* __restrict__ Q,
                                                      ElemParams p, double* __restrict__ G, int project) {
  if (threadIdx.x == 0) pdl_trigger();  // the node gather behind may launch (it waits for G)
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsub) return;
  int64_t e = sub ? sub[i] : i;
  int4 t = tets[e];
  double F[9], Rl[9], Ql[9], D[9];
  deformation_gradient(x, t, dmi, ne, e, F);
  if (project) {
    double u[9], v[9], S[3];
    signed_svd(F, u, S, v);
    uvt(u, v, Rl);
#pragma unroll
    for (int c = 0; c < 9; ++c) R[c * ne + e] = Rl[c];
    if (p.biphasic) {
      udvt(u, S, v, p.smin, p.smax, Ql);
#pragma unroll
      for (int c = 0; c < 9; ++c) Q[c * ne + e] = Ql[c];
    }
  } else {
#pragma unroll
    for (int c = 0; c < 9; ++c) Rl[c] = R[c * ne + e];
    if (p.biphasic)
#pragma unroll
      for (int c = 0; c < 9; ++c) Ql[c] = Q[c * ne + e];
  }
  if (G) {
#pragma unroll
    for (int c = 0; c < 9; ++c) D[c] = dmi[c * ne + e];
    double out[12];
    element_forces(F, Rl, p.biphasic ? Ql : nullptr, D, vol[e], p, out);
#pragma unroll
    for (int c = 0; c < 12; ++c) G[(int64_t)c * nsub + i] = out[c];
  }
}

// Deterministic node gather: out[k] = sum of the listed element-slot forces in
// list order (the reference's np.add.at order: slot-major, element order),
// then attachment springs k (t - x) in attachment-list order (solver.py:187-190).
__global__ void __launch_bounds__(256) k_gather_forces(int nout, const int* __restrict__ ptr,
                                                       const int* __restrict__ src, const double* __restrict__ G,
                                                       int nsub, const int* __restrict__ out_node,
                                                       const int* __restrict__ aptr, const int* __restrict__ aidx,
                                                       const double* __restrict__ ak,
                                                       const double* __restrict__ atgt,
                                                       const double* __restrict__ x, double* __restrict__ out) {
  if (threadIdx.x == 0) pdl_trigger();  // the forward sweep behind waits for b itself
  pdl_wait();                           // G of the element kernel before
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nout) return;
  double f0 = 0.0, f1 = 0.0, f2 = 0.0;
  for (int q = ptr[k]; q < ptr[k + 1]; ++q) {
    int s = src[q];
    int i = s >> 2, slot = s & 3;
    f0 += G[(int64_t)(slot * 3 + 0) * nsub + i];
    f1 += G[(int64_t)(slot * 3 + 1) * nsub + i];
    f2 += G[(int64_t)(slot * 3 + 2) * nsub + i];
  }
  if (aptr) {
    int64_t node = out_node[k];
    for (int a = aptr[k]; a < aptr[k + 1]; ++a) {
      int j = aidx[a];
      double kk = ak[j];
      f0 += kk * (atgt[3 * j + 0] - x[3 * node + 0]);
      f1 += kk * (atgt[3 * j + 1] - x[3 * node + 1]);
      f2 += kk * (atgt[3 * j + 2] - x[3 * node + 2]);
    }
  }
  out[3 * k + 0] = f0;
  out[3 * k + 1] = f1;
  out[3 * k + 2] = f2;
}

// Elastic energy density per element reduced per block (material.py:360-378);
// partial sums are combined in fixed order by k_finish_metrics.
__global__ void __launch_bounds__(256) k_elastic_energy(int64_t ne, const int4* __restrict__ tets,
                                                        const double* __restrict__ x,
                                                        const double* __restrict__ dmi,
                                                        const double* __restrict__ vol,
                                                        const double* __restrict__ R,
                                                        const double* __restrict__ Q, ElemParams p,
                                                        double* __restrict__ partial) {
  __shared__ double red[8];
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double val = 0.0;
  if (e < ne) {
    double F[9];
    deformation_gradient(x, tets[e], dmi, ne, e, F);
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      double d = F[c] - R[c * ne + e];
      s += d * d;
    }
    double dens = p.mu * s;
    if (p.biphasic) {
      double sq = 0.0;
#pragma unroll
      for (int c = 0; c < 9; ++c) {
        double d = F[c] - Q[c * ne + e];
        sq += d * d;
      }
      dens = dens + p.mu_prime * sq;
    }
    val = vol[e] * dens;
  }
  val = warp_sum(val);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = val;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    partial[blockIdx.x] = s;
  }
}

// F of a subset (op helper).
__global__ void k_deformation_gradients(int nsub, const int* __restrict__ sub, const int4* __restrict__ tets,
                                        const double* __restrict__ x, const double* __restrict__ dmi, int64_t ne,
                                        double* __restrict__ F) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsub) return;
  int64_t e = sub ? sub[i] : i;
  double f[9];
  deformation_gradient(x, tets[e], dmi, ne, e, f);
#pragma unroll
  for (int c = 0; c < 9; ++c) F[9 * (int64_t)i + c] = f[c];
}

// SVD / polar / clamp of a stack of row-major F (op helper).
__global__ void k_svd_op(int64_t k, const double* __restrict__ F, double* U, double* S, double* V, double* R,
                         double* Q, double smin, double smax) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  double f[9], u[9], v[9], s[3], r[9];
#pragma unroll
  for (int c = 0; c < 9; ++c) f[c] = F[9 * i + c];
  signed_svd(f, u, s, v);
  if (U)
    for (int c = 0; c < 9; ++c) U[9 * i + c] = u[c];
  if (V)
    for (int c = 0; c < 9; ++c) V[9 * i + c] = v[c];
  if (S)
    for (int c = 0; c < 3; ++c) S[3 * i + c] = s[c];
  if (R) {
    uvt(u, v, r);
    for (int c = 0; c < 9; ++c) R[9 * i + c] = r[c];
  }
  if (Q) {
    udvt(u, s, v, smin, smax, r);
    for (int c = 0; c < 9; ++c) Q[9 * i + c] = r[c];
  }
}

// ------------------------------------------------------------- launchers
void launch_local_forces(cudaStream_t st, int nsub, const int* sub, const int4* tets, const double* x,
                         const double* dmi, const double* vol, int64_t ne, double* R, double* Q,
                         const ElemParams& p, double* G, int project) {
  if (nsub <= 0) return;
  k_local_forces<<<ceil_div(nsub, 128), 128, 0, st>>>(nsub, sub, tets, x, dmi, vol, ne, R, Q, p, G, project);
}

void launch_gather_forces(cudaStream_t st, int nout, const int* ptr, const int* src, const double* G, int nsub,
                          const int* out_node, const int* aptr, const int* aidx, const double* ak,
                          const double* atgt, const double* x, double* out) {
  if (nout <= 0) return;
  launch_pdl(k_gather_forces, dim3(ceil_div(nout, 256)), dim3(256), 0, st, nout, ptr, src, G, nsub, out_node, aptr,
             aidx, ak, atgt, x, out);
}

int energy_blocks(int64_t ne) { return ceil_div(ne, 256); }

void launch_elastic_energy(cudaStream_t st, int64_t ne, const int4* tets, const double* x, const double* dmi,
                           const double* vol, const double* R, const double* Q, const ElemParams& p,
                           double* partial) {
  if (ne <= 0) return;
  k_elastic_energy<<<energy_blocks(ne), 256, 0, st>>>(ne, tets, x, dmi, vol, R, Q, p, partial);
}

void launch_deformation_gradients(cudaStream_t st, int nsub, const int* sub, const int4* tets, const double* x,
                                  const double* dmi, int64_t ne, double* F) {
  if (nsub <= 0) return;
  k_deformation_gradients<<<ceil_div(nsub, 128), 128, 0, st>>>(nsub, sub, tets, x, dmi, ne, F);
}

void launch_svd_op(cudaStream_t st, int64_t k, const double* F, double* U, double* S, double* V, double* R,
                   double* Q, double smin, double smax) {
  if (k <= 0) return;
  k_svd_op<<<ceil_div(k, 128), 128, 0, st>>>(k, F, U, S, V, R, Q, smin, smax);
}

}  // namespace spb
