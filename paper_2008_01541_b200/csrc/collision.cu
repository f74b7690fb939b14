// Collision kernels: proxy positions, signed distances of the posed implicit
// colliders, deepest-collider detection with frozen targets, the reduced
// inner right-hand side g = f~2 + f_beta + f_col, and the end-of-frame proxy
// metrics (collision energy, penetration depth).
//
// Compiled with -fmad=false. Proxy positions follow numpy's einsum order
// (sequential, non-fused: collision.py:309). Signed distances go through
// BLAS dgemv/dgemm in the reference (collision.py:51, :70, :111), whose
// per-row order is not reproducible; flags are therefore certified by the
// sign-band protocol of SURVEY.md §7 H3 (tests/test_gpu_parity.py).
//
// Reference: collision.py:43-203 (shapes, transforms), :316-342 (detect),
// :345-374 (penetration, energy), solver.py:349-364 (collision forces),
// solver.py:432-433 (g).
#include "common.cuh"
#include "kernels.cuh"

namespace spb {

__device__ __forceinline__ void proxy_point(const int4* __restrict__ tets, const double* __restrict__ x,
                                            const int* __restrict__ elem, const double* __restrict__ w, int j,
                                            double p[3]) {
  int4 t = tets[elem[j]];
  double w0 = w[4 * j + 0], w1 = w[4 * j + 1], w2 = w[4 * j + 2], w3 = w[4 * j + 3];
#pragma unroll
  for (int d = 0; d < 3; ++d)
    p[d] = ((w0 * x[3 * (int64_t)t.x + d] + w1 * x[3 * (int64_t)t.y + d]) + w2 * x[3 * (int64_t)t.z + d]) +
           w3 * x[3 * (int64_t)t.w + d];
}

__device__ __forceinline__ double norm3(double a, double b, double c) { return sqrt((a * a + b * b) + c * c); }

__device__ double grid_sample(const ShapeDev& s, double qx, double qy, double qz) {
  // collision.py:145-167; +inf outside the inclusive bounds
  const double sp = s.p[3];
  double gx = (qx - s.p[0]) / sp, gy = (qy - s.p[1]) / sp, gz = (qz - s.p[2]) / sp;
  const int nx = s.dims[0], ny = s.dims[1], nz = s.dims[2];
  if (!(gx >= 0 && gx <= nx - 1 && gy >= 0 && gy <= ny - 1 && gz >= 0 && gz <= nz - 1)) return CUDART_INF;
  int ix = min((int)gx, nx - 2), iy = min((int)gy, ny - 2), iz = min((int)gz, nz - 2);
  double fx = gx - ix, fy = gy - iy, fz = gz - iz;
  const double* v = s.values;
  auto at = [&](int i, int j, int k) { return v[i + (int64_t)nx * (j + (int64_t)ny * k)]; };
  double c00 = at(ix, iy, iz) * (1 - fx) + at(ix + 1, iy, iz) * fx;
  double c10 = at(ix, iy + 1, iz) * (1 - fx) + at(ix + 1, iy + 1, iz) * fx;
  double c01 = at(ix, iy, iz + 1) * (1 - fx) + at(ix + 1, iy, iz + 1) * fx;
  double c11 = at(ix, iy + 1, iz + 1) * (1 - fx) + at(ix + 1, iy + 1, iz + 1) * fx;
  return (c00 * (1 - fy) + c10 * fy) * (1 - fz) + (c01 * (1 - fy) + c11 * fy) * fz;
}

__device__ __forceinline__ void capsule_closest(const ShapeDev& s, const double q[3], double c[3]) {
  double ax = s.p[3] - s.p[0], ay = s.p[4] - s.p[1], az = s.p[5] - s.p[2];
  double denom = (ax * ax + ay * ay) + az * az;
  if (denom == 0.0) {
    c[0] = s.p[0]; c[1] = s.p[1]; c[2] = s.p[2];
    return;
  }
  double t = (((q[0] - s.p[0]) * ax + (q[1] - s.p[1]) * ay) + (q[2] - s.p[2]) * az) / denom;
  t = fmin(fmax(t, 0.0), 1.0);
  c[0] = s.p[0] + t * ax;
  c[1] = s.p[1] + t * ay;
  c[2] = s.p[2] + t * az;
}

__device__ double sd_local(const ShapeDev& s, const double q[3]) {
  switch (s.kind) {
    case SPB_SHAPE_HALF_SPACE:
      return ((q[0] - s.p[0]) * s.p[3] + (q[1] - s.p[1]) * s.p[4]) + (q[2] - s.p[2]) * s.p[5];
    case SPB_SHAPE_SPHERE:
      return norm3(q[0] - s.p[0], q[1] - s.p[1], q[2] - s.p[2]) - s.p[3];
    case SPB_SHAPE_CAPSULE: {
      double c[3];
      capsule_closest(s, q, c);
      return norm3(q[0] - c[0], q[1] - c[1], q[2] - c[2]) - s.p[6];
    }
    default:
      return grid_sample(s, q[0], q[1], q[2]);
  }
}

__device__ void grad_local(const ShapeDev& s, const double q[3], double g[3]) {
  switch (s.kind) {
    case SPB_SHAPE_HALF_SPACE:
      g[0] = s.p[3]; g[1] = s.p[4]; g[2] = s.p[5];
      return;
    case SPB_SHAPE_SPHERE:
    case SPB_SHAPE_CAPSULE: {
      double c[3];
      if (s.kind == SPB_SHAPE_SPHERE) { c[0] = s.p[0]; c[1] = s.p[1]; c[2] = s.p[2]; }
      else capsule_closest(s, q, c);
      double d0 = q[0] - c[0], d1 = q[1] - c[1], d2 = q[2] - c[2];
      double r = norm3(d0, d1, d2);
      if (r > 0) { g[0] = d0 / r; g[1] = d1 / r; g[2] = d2 / r; }
      else { g[0] = 1.0; g[1] = 0.0; g[2] = 0.0; }  // collision.py:92, :121
      return;
    }
    default: {
      const double h = 0.5 * s.p[3];
      for (int a = 0; a < 3; ++a) {
        double qp[3] = {q[0], q[1], q[2]}, qm[3] = {q[0], q[1], q[2]};
        qp[a] = q[a] + h;
        qm[a] = q[a] - h;
        g[a] = (grid_sample(s, qp[0], qp[1], qp[2]) - grid_sample(s, qm[0], qm[1], qm[2])) / (2 * h);
      }
      if (!(isfinite(g[0]) && isfinite(g[1]) && isfinite(g[2]))) g[0] = g[1] = g[2] = 0.0;  // collision.py:179
    }
  }
}

__device__ __forceinline__ void to_local(const PosedDev& c, const double p[3], double q[3]) {
  double d0 = p[0] - c.t[0], d1 = p[1] - c.t[1], d2 = p[2] - c.t[2];
#pragma unroll
  for (int j = 0; j < 3; ++j) q[j] = (d0 * c.R[0 + j] + d1 * c.R[3 + j]) + d2 * c.R[6 + j];
}

// Deepest collider per proxy (strict <, first listed wins ties), active iff
// phi < 0, target = p - phi * R grad (collision.py:316-342, :196-203).
__global__ void __launch_bounds__(128) k_detect(ProxyDev px, const int4* __restrict__ tets,
                                                const double* __restrict__ x, const ShapeDev* __restrict__ shapes,
                                                const ColliderSet* __restrict__ cols, uint8_t* __restrict__ active,
                                                double* __restrict__ target, double* __restrict__ depth) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= px.P) return;
  double p[3];
  proxy_point(tets, x, px.elem, px.w, j, p);
  const int nc = cols->n;
  double best = CUDART_INF;
  int bi = -1;
  for (int ci = 0; ci < nc; ++ci) {
    const PosedDev& c = cols->posed[ci];
    double q[3];
    to_local(c, p, q);
    double phi = sd_local(shapes[c.shape], q);
    if (phi < best) { best = phi; bi = ci; }
  }
  bool act = best < 0.0;
  double t0 = 0.0, t1 = 0.0, t2 = 0.0;
  if (act) {
    const PosedDev& c = cols->posed[bi];
    const ShapeDev& s = shapes[c.shape];
    double q[3], g[3];
    to_local(c, p, q);
    double phi = sd_local(s, q);
    grad_local(s, q, g);
    if (!isfinite(phi)) phi = 0.0;
    double w0 = (g[0] * c.R[0] + g[1] * c.R[1]) + g[2] * c.R[2];
    double w1 = (g[0] * c.R[3] + g[1] * c.R[4]) + g[2] * c.R[5];
    double w2 = (g[0] * c.R[6] + g[1] * c.R[7]) + g[2] * c.R[8];
    t0 = p[0] - phi * w0;
    t1 = p[1] - phi * w1;
    t2 = p[2] - phi * w2;
  }
  if (active) active[j] = act ? 1 : 0;
  if (target) {
    target[3 * j + 0] = t0;
    target[3 * j + 1] = t1;
    target[3 * j + 2] = t2;
  }
  if (depth) depth[j] = isfinite(best) ? fmax(0.0, -best) : 0.0;
}

// g[k] = (f~2[k] + f_beta[k]) + f_col[k] for every trailing-local row k
// (solver.py:432-433). f_beta gathers the beta elements' slot forces in the
// reference's np.add.at order; f_col gathers w_a * (-c (p - t)) of active
// proxies in (slot, proxy) order (solver.py:356-364).
__global__ void __launch_bounds__(256) k_build_g(int m, const double* __restrict__ f_tilde2,
                                                 const int* __restrict__ bptr, const int* __restrict__ bsrc,
                                                 const double* __restrict__ Gb, int nbeta, ProxyDev px,
                                                 const int4* __restrict__ tets, const double* __restrict__ x,
                                                 const uint8_t* __restrict__ active,
                                                 const double* __restrict__ target, const int* __restrict__ cptr,
                                                 const int* __restrict__ csrc, double* __restrict__ g,
                                                 double* __restrict__ ytile /* RHS tile row or null */) {
  if (threadIdx.x == 0) pdl_trigger();  // the factorization behind may start; its RHS row waits for g
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  double b0 = 0.0, b1 = 0.0, b2 = 0.0;
  for (int q = bptr[k]; q < bptr[k + 1]; ++q) {
    int s = bsrc[q];
    int i = s >> 2, slot = s & 3;
    b0 += Gb[(int64_t)(slot * 3 + 0) * nbeta + i];
    b1 += Gb[(int64_t)(slot * 3 + 1) * nbeta + i];
    b2 += Gb[(int64_t)(slot * 3 + 2) * nbeta + i];
  }
  double c0 = 0.0, c1 = 0.0, c2 = 0.0;
  for (int q = cptr[k]; q < cptr[k + 1]; ++q) {
    int s = csrc[q];
    int j = s >> 2, a = s & 3;
    if (!active[j]) continue;
    double p[3];
    proxy_point(tets, x, px.elem, px.w, j, p);
    double nc = -px.c[j];
    double wa = px.w[4 * j + a];
    c0 += wa * (nc * (p[0] - target[3 * j + 0]));
    c1 += wa * (nc * (p[1] - target[3 * j + 1]));
    c2 += wa * (nc * (p[2] - target[3 * j + 2]));
  }
  double g0 = (f_tilde2[3 * k + 0] + b0) + c0;
  double g1 = (f_tilde2[3 * k + 1] + b1) + c1;
  double g2 = (f_tilde2[3 * k + 2] + b2) + c2;
  g[3 * k + 0] = g0;
  g[3 * k + 1] = g1;
  g[3 * k + 2] = g2;
  if (ytile) {
    // tile j = k/64 of the RHS row holds g^T (rows 0..2, swizzled layout)
    int tj = k >> 6, c = k & 63;
    double* t = ytile + (int64_t)tj * 4096;
    t[swz(0, c)] = g0;
    t[swz(1, c)] = g1;
    t[swz(2, c)] = g2;
  }
}

// End-of-frame proxy terms: collision energy (collision.py:362-374) and the
// penetration depth against every posed collider (collision.py:345-359).
__global__ void __launch_bounds__(128) k_proxy_final(ProxyDev px, const int4* __restrict__ tets,
                                                     const double* __restrict__ x,
                                                     const ShapeDev* __restrict__ shapes,
                                                     const ColliderSet* __restrict__ cols,
                                                     const uint8_t* __restrict__ active,
                                                     const double* __restrict__ target,
                                                     double* __restrict__ partial /* 2 per block */) {
  __shared__ double se[4], sd[4];
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  double e = 0.0, dep = 0.0;
  if (j < px.P) {
    double p[3];
    proxy_point(tets, x, px.elem, px.w, j, p);
    if (active[j]) {
      double d0 = p[0] - target[3 * j + 0], d1 = p[1] - target[3 * j + 1], d2 = p[2] - target[3 * j + 2];
      e = px.c[j] * ((d0 * d0 + d1 * d1) + d2 * d2);
    }
    double best = CUDART_INF;
    for (int ci = 0; ci < cols->n; ++ci) {
      double q[3];
      to_local(cols->posed[ci], p, q);
      best = fmin(best, sd_local(shapes[cols->posed[ci].shape], q));
    }
    dep = isfinite(best) ? fmax(0.0, -best) : 0.0;
  }
  e = warp_sum(e);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dep = fmax(dep, __shfl_xor_sync(0xffffffffu, dep, o));
  if ((threadIdx.x & 31) == 0) {
    se[threadIdx.x >> 5] = e;
    sd[threadIdx.x >> 5] = dep;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0, d = 0.0;
    for (int w = 0; w < 4; ++w) {
      s += se[w];
      d = fmax(d, sd[w]);
    }
    partial[2 * blockIdx.x + 0] = s;
    partial[2 * blockIdx.x + 1] = d;
  }
}

// ------------------------------------------------------------- launchers
void launch_detect(cudaStream_t st, const ProxyDev& px, const int4* tets, const double* x, const ShapeDev* shapes,
                   const ColliderSet* cols, uint8_t* active, double* target, double* depth) {
  if (px.P <= 0) return;
  k_detect<<<ceil_div(px.P, 128), 128, 0, st>>>(px, tets, x, shapes, cols, active, target, depth);
}

void launch_build_g(cudaStream_t st, int m, const double* f_tilde2, const int* bptr, const int* bsrc,
                    const double* Gb, int nbeta, const ProxyDev& px, const int4* tets, const double* x,
                    const uint8_t* active, const double* target, const int* cptr, const int* csrc, double* g,
                    double* ytile) {
  if (m <= 0) return;
  k_build_g<<<ceil_div(m, 256), 256, 0, st>>>(m, f_tilde2, bptr, bsrc, Gb, nbeta, px, tets, x, active, target,
                                              cptr, csrc, g, ytile);
}

int proxy_blocks(int P) { return P > 0 ? ceil_div(P, 128) : 0; }

void launch_proxy_final(cudaStream_t st, const ProxyDev& px, const int4* tets, const double* x,
                        const ShapeDev* shapes, const ColliderSet* cols, const uint8_t* active,
                        const double* target, double* partial) {
  if (px.P <= 0) return;
  k_proxy_final<<<proxy_blocks(px.P), 128, 0, st>>>(px, tets, x, shapes, cols, active, target, partial);
}

}  // namespace spb
