// One-shot device ops behind the public helper functions of the drop-in API
// (mesh.deformation_gradients, material.signed_svd/polar_rotations/
// biphasic_projections/elastic_forces/elastic_energy, collision.detect/
// penetration_depths, linalg.forward_sub/backward_sub/dense_factor/
// dense_solve). Each call uploads its inputs, runs the same kernels the frame
// solver uses, and downloads the result. No host fallback exists.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

static int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

namespace spb {
void set_error(const std::string& msg);

namespace {
template <typename T>
struct Tmp {
  T* p = nullptr;
  explicit Tmp(size_t n) {
    if (cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1)) != cudaSuccess) p = nullptr;
  }
  ~Tmp() {
    if (p) cudaFree(p);
  }
  bool ok() const { return p != nullptr; }
};

#define TMP(T, name, count)                                   \
  Tmp<T> name(count);                                         \
  if (!name.ok()) {                                           \
    set_error("cudaMalloc failed in op");                     \
    return SPB_ERR_CUDA;                                      \
  }
#define H2D(dst, src, bytes) SPB_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice))
#define D2H(dst, src, bytes) SPB_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost))

int upload_mesh(int64_t ne, const int64_t* tets, const double* dmi, Tmp<int4>& t4, Tmp<double>& dsoa) {
  std::vector<int4> t(ne);
  for (int64_t e = 0; e < ne; ++e)
    t[e] = make_int4((int)tets[4 * e], (int)tets[4 * e + 1], (int)tets[4 * e + 2], (int)tets[4 * e + 3]);
  H2D(t4.p, t.data(), sizeof(int4) * ne);
  std::vector<double> soa(9 * ne);
  for (int64_t e = 0; e < ne; ++e)
    for (int c = 0; c < 9; ++c) soa[c * ne + e] = dmi[9 * e + c];
  H2D(dsoa.p, soa.data(), sizeof(double) * 9 * ne);
  return SPB_OK;
}

// tile helpers for the dense ops
constexpr int TS = 64;
int pack_tiles(int64_t m, int N, const double* h, std::vector<double>& tiles) {
  tiles.assign((size_t)N * (N + 1) / 2 * 4096, 0.0);
  for (int i = 0; i < N; ++i)
    for (int j = 0; j <= i; ++j) {
      double* T = tiles.data() + (size_t)(i * (i + 1) / 2 + j) * 4096;
      for (int r = 0; r < 64; ++r)
        for (int c = 0; c < 64; ++c) {
          int64_t gr = i * 64 + r, gc = j * 64 + c;
          T[swz(r, c)] = (gr < m && gc < m) ? h[gr * m + gc] : (gr == gc ? 1.0 : 0.0);
        }
    }
  return SPB_OK;
}
}  // namespace
}  // namespace spb

using namespace spb;

extern "C" {

int32_t spb_op_deformation_gradients(int64_t ne, const int64_t* tets, const double* dm_inverse, int64_t n,
                                     const double* x, int64_t k, const int64_t* elements, double* F) {
  SPB_GUARD_BEGIN
  if (k <= 0) return SPB_OK;
  TMP(int4, t4, ne);
  TMP(double, dsoa, 9 * ne);
  {
    int rc = upload_mesh(ne, tets, dm_inverse, t4, dsoa);
    if (rc) return rc;
  }
  TMP(double, dx, 3 * n);
  H2D(dx.p, x, sizeof(double) * 3 * n);
  TMP(int, dsub, k);
  if (elements) {
    std::vector<int> s(elements, elements + k);
    H2D(dsub.p, s.data(), sizeof(int) * k);
  }
  TMP(double, dF, 9 * k);
  launch_deformation_gradients(0, (int)k, elements ? dsub.p : nullptr, t4.p, dx.p, dsoa.p, ne, dF.p);
  SPB_CUDA(cudaGetLastError());
  D2H(F, dF.p, sizeof(double) * 9 * k);
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_op_svd(int64_t k, const double* F, double* U, double* S, double* V, double* R, double* Q,
                   double sigma_min, double sigma_max) {
  SPB_GUARD_BEGIN
  if (k <= 0) return SPB_OK;
  TMP(double, dF, 9 * k);
  H2D(dF.p, F, sizeof(double) * 9 * k);
  Tmp<double> dU(U ? 9 * k : 0), dS(S ? 3 * k : 0), dV(V ? 9 * k : 0), dR(R ? 9 * k : 0), dQ(Q ? 9 * k : 0);
  launch_svd_op(0, k, dF.p, U ? dU.p : nullptr, S ? dS.p : nullptr, V ? dV.p : nullptr, R ? dR.p : nullptr,
                Q ? dQ.p : nullptr, sigma_min, sigma_max);
  SPB_CUDA(cudaGetLastError());
  if (U) D2H(U, dU.p, sizeof(double) * 9 * k);
  if (S) D2H(S, dS.p, sizeof(double) * 3 * k);
  if (V) D2H(V, dV.p, sizeof(double) * 9 * k);
  if (R) D2H(R, dR.p, sizeof(double) * 9 * k);
  if (Q) D2H(Q, dQ.p, sizeof(double) * 9 * k);
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_op_elastic(int64_t ne, const int64_t* tets, const double* dm_inverse, const double* volume, int64_t n,
                       const double* x, const double* R, const double* Q, double mu, double mu_prime, int64_t k,
                       const int64_t* elements, double* forces, double* energy) {
  SPB_GUARD_BEGIN
  TMP(int4, t4, ne);
  TMP(double, dsoa, 9 * ne);
  {
    int rc = upload_mesh(ne, tets, dm_inverse, t4, dsoa);
    if (rc) return rc;
  }
  TMP(double, dvol, ne);
  H2D(dvol.p, volume, sizeof(double) * ne);
  TMP(double, dx, 3 * n);
  H2D(dx.p, x, sizeof(double) * 3 * n);
  std::vector<double> soa(9 * ne);
  TMP(double, dR, 9 * ne);
  for (int64_t e = 0; e < ne; ++e)
    for (int c = 0; c < 9; ++c) soa[c * ne + e] = R[9 * e + c];
  H2D(dR.p, soa.data(), sizeof(double) * 9 * ne);
  bool bip = Q != nullptr && mu_prime > 0.0;
  TMP(double, dQ, bip ? 9 * ne : 1);
  if (bip) {
    for (int64_t e = 0; e < ne; ++e)
      for (int c = 0; c < 9; ++c) soa[c * ne + e] = Q[9 * e + c];
    H2D(dQ.p, soa.data(), sizeof(double) * 9 * ne);
  }
  ElemParams ep{mu, mu_prime, 0.0, 0.0, bip ? 1 : 0};
  const int64_t nsub = elements ? k : ne;
  if (forces) {
    TMP(int, dsub, nsub);
    if (elements) {
      std::vector<int> s(elements, elements + k);
      H2D(dsub.p, s.data(), sizeof(int) * k);
    }
    TMP(double, G, 12 * nsub);
    launch_local_forces(0, (int)nsub, elements ? dsub.p : nullptr, t4.p, dx.p, dsoa.p, dvol.p, ne, dR.p, dQ.p, ep,
                        G.p, 0);
    // slot-major, element-order node gather (material.py:354-356)
    std::vector<int> ptr(n + 1, 0), src;
    std::vector<std::pair<int, int>> pairs;
    for (int a = 0; a < 4; ++a)
      for (int64_t i = 0; i < nsub; ++i) {
        int64_t e = elements ? elements[i] : i;
        pairs.emplace_back((int)tets[4 * e + a], (int)(i * 4 + a));
      }
    for (auto& kv : pairs) ptr[kv.first + 1]++;
    for (int64_t v = 0; v < n; ++v) ptr[v + 1] += ptr[v];
    src.resize(pairs.size());
    std::vector<int> fill(ptr.begin(), ptr.end() - 1);
    for (auto& kv : pairs) src[fill[kv.first]++] = kv.second;
    TMP(int, dptr, n + 1);
    TMP(int, dsrc, src.size());
    H2D(dptr.p, ptr.data(), sizeof(int) * (n + 1));
    if (!src.empty()) H2D(dsrc.p, src.data(), sizeof(int) * src.size());
    TMP(double, dout, 3 * n);
    launch_gather_forces(0, (int)n, dptr.p, dsrc.p, G.p, (int)nsub, nullptr, nullptr, nullptr, nullptr, nullptr,
                         dx.p, dout.p);
    SPB_CUDA(cudaGetLastError());
    D2H(forces, dout.p, sizeof(double) * 3 * n);
  }
  if (energy) {
    if (elements) {
      // energy over a subset: gather the subset into a compact mesh
      std::vector<int64_t> te(4 * k);
      std::vector<double> dm(9 * k), vo(k), rr(9 * k), qq(bip ? 9 * k : 0);
      for (int64_t i = 0; i < k; ++i) {
        int64_t e = elements[i];
        for (int a = 0; a < 4; ++a) te[4 * i + a] = tets[4 * e + a];
        for (int c = 0; c < 9; ++c) {
          dm[9 * i + c] = dm_inverse[9 * e + c];
          rr[9 * i + c] = R[9 * e + c];
          if (bip) qq[9 * i + c] = Q[9 * e + c];
        }
        vo[i] = volume[e];
      }
      return spb_op_elastic(k, te.data(), dm.data(), vo.data(), n, x, rr.data(), bip ? qq.data() : nullptr, mu,
                            mu_prime, 0, nullptr, nullptr, energy);
    }
    int nb = energy_blocks(ne);
    TMP(double, part, nb);
    launch_elastic_energy(0, ne, t4.p, dx.p, dsoa.p, dvol.p, dR.p, dQ.p, ep, part.p);
    TMP(double, out, 4);
    launch_finish_metrics(0, part.p, nb, nullptr, 0, nullptr, 0, nullptr, 0, nullptr, 0, 0, out.p);
    SPB_CUDA(cudaGetLastError());
    D2H(energy, out.p, sizeof(double));
  }
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_op_detect(int64_t n, const double* x, const int64_t* tets, int64_t P, const int64_t* proxy_elements,
                      const double* proxy_weights, int32_t num_shapes, const spb_shape_desc* shapes,
                      const spb_posed_collider* colliders, uint8_t* active, double* target, double* depth) {
  SPB_GUARD_BEGIN
  if (P <= 0) return SPB_OK;
  if (num_shapes > MAX_COLLIDERS) { set_error("too many colliders"); return SPB_ERR_ARG; }
  // compact mesh of the proxy elements
  std::vector<int4> t4(P);
  std::vector<int> pe(P);
  for (int64_t j = 0; j < P; ++j) {
    int64_t e = proxy_elements[j];
    t4[j] = make_int4((int)tets[4 * e], (int)tets[4 * e + 1], (int)tets[4 * e + 2], (int)tets[4 * e + 3]);
    pe[j] = (int)j;
  }
  TMP(int4, dt, P);
  H2D(dt.p, t4.data(), sizeof(int4) * P);
  TMP(int, dpe, P);
  H2D(dpe.p, pe.data(), sizeof(int) * P);
  TMP(double, dw, 4 * P);
  H2D(dw.p, proxy_weights, sizeof(double) * 4 * P);
  TMP(double, dx, 3 * n);
  H2D(dx.p, x, sizeof(double) * 3 * n);
  std::vector<ShapeDev> sh(num_shapes);
  std::vector<Tmp<double>*> vals;
  for (int s = 0; s < num_shapes; ++s) {
    sh[s].kind = shapes[s].kind;
    for (int k = 0; k < 7; ++k) sh[s].p[k] = shapes[s].params[k];
    sh[s].values = nullptr;
    if (shapes[s].kind == SPB_SHAPE_LEVELSET) {
      size_t cnt = (size_t)shapes[s].dims[0] * shapes[s].dims[1] * shapes[s].dims[2];
      for (int k = 0; k < 3; ++k) sh[s].dims[k] = (int)shapes[s].dims[k];
      auto* v = new Tmp<double>(cnt);
      vals.push_back(v);
      H2D(v->p, shapes[s].values, sizeof(double) * cnt);
      sh[s].values = v->p;
    }
  }
  TMP(ShapeDev, dsh, std::max(num_shapes, 1));
  if (num_shapes) H2D(dsh.p, sh.data(), sizeof(ShapeDev) * num_shapes);
  ColliderSet cs{};
  cs.n = num_shapes;
  for (int s = 0; s < num_shapes; ++s) {
    cs.posed[s].shape = s;
    for (int k = 0; k < 9; ++k) cs.posed[s].R[k] = colliders[s].rotation[k];
    for (int k = 0; k < 3; ++k) cs.posed[s].t[k] = colliders[s].translation[k];
  }
  TMP(ColliderSet, dcs, 1);
  H2D(dcs.p, &cs, sizeof(ColliderSet));
  TMP(uint8_t, dact, P);
  TMP(double, dtg, 3 * P);
  TMP(double, ddep, P);
  ProxyDev px{(int)P, dpe.p, dw.p, nullptr, nullptr};
  launch_detect(0, px, dt.p, dx.p, dsh.p, dcs.p, dact.p, dtg.p, ddep.p);
  SPB_CUDA(cudaGetLastError());
  if (active) D2H(active, dact.p, P);
  if (target) D2H(target, dtg.p, sizeof(double) * 3 * P);
  if (depth) D2H(depth, ddep.p, sizeof(double) * P);
  for (auto* v : vals) delete v;
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_op_dense_factor(int64_t m, const double* h, double* chol, int64_t* info) {
  SPB_GUARD_BEGIN
  *info = 0;
  if (m <= 0) return SPB_OK;
  const int N = (int)((m + 63) / 64);
  const int nt = dense_tile_count(N);
  std::vector<double> tiles;
  pack_tiles(m, N, h, tiles);
  TMP(double, dS, (size_t)nt * 4096);
  H2D(dS.p, tiles.data(), sizeof(double) * tiles.size());
  TMP(double, dL, (size_t)nt * 4096);
  TMP(double, dLi, (size_t)N * 4096);
  TMP(double, dY, (size_t)N * 4096);
  TMP(int, dflags, nt + N);
  TMP(int, dcnt, 1);
  TMP(int, dinfo, 1);
  SPB_CUDA(cudaMemset(dflags.p, 0, sizeof(int) * (nt + N)));
  SPB_CUDA(cudaMemset(dcnt.p, 0, sizeof(int)));
  SPB_CUDA(cudaMemset(dinfo.p, 0, sizeof(int)));
  SPB_CUDA(cudaMemset(dY.p, 0, sizeof(double) * N * 4096));
  std::vector<int2> tk = cholesky_task_order(N, false, CHOL_LEAD);
  TMP(int2, dtk, tk.size());
  H2D(dtk.p, tk.data(), sizeof(int2) * tk.size());
  DenseDev d{(int)m, N, dS.p, dL.p, dLi.p, dY.p, dflags.p, dcnt.p, dinfo.p, nullptr, nullptr, nullptr, nullptr,
             nullptr, nullptr, nullptr};
  launch_cholesky_tiles(0, d, dtk.p, (int)tk.size(), std::min<int>(NUM_SMS_B200, (int)tk.size()));
  SPB_CUDA(cudaGetLastError());
  SPB_CUDA(cudaDeviceSynchronize());
  int hinfo = 0;
  D2H(&hinfo, dinfo.p, sizeof(int));
  D2H(tiles.data(), dL.p, sizeof(double) * tiles.size());
  for (int64_t r = 0; r < m; ++r)
    for (int64_t c = 0; c < m; ++c) {
      int i = (int)(r / 64), j = (int)(c / 64);
      chol[r * m + c] =
          (c <= r) ? tiles[(size_t)(i * (i + 1) / 2 + j) * 4096 + swz((int)(r % 64), (int)(c % 64))] : 0.0;
    }
  if (hinfo > 0) {
    *info = hinfo;
    set_error("dense factorization failed: non-positive pivot");
    return SPB_ERR_INDEFINITE;
  }
  return SPB_OK;
  SPB_GUARD_END
}

// Solve with a given lower factor: its tiles and the transposed inverses of its
// diagonal tiles (host, O(N 64^3)) feed the device sweeps: the forward sweep is
// the tile kernel's RHS-row tasks with every L tile marked ready, the backward
// sweep is k_dense_backward.
int32_t spb_op_dense_solve(int64_t m, const double* chol, int64_t nrhs, const double* g, double* out) {
  SPB_GUARD_BEGIN
  if (m <= 0 || nrhs <= 0) return SPB_OK;
  const int N = (int)((m + 63) / 64);
  const int nt = dense_tile_count(N);
  std::vector<double> lower((size_t)m * m);
  for (int64_t r = 0; r < m; ++r)
    for (int64_t c = 0; c < m; ++c) lower[r * m + c] = (c <= r) ? chol[r * m + c] : 0.0;
  std::vector<double> tiles;
  pack_tiles(m, N, lower.data(), tiles);
  std::vector<double> linvT((size_t)N * 4096, 0.0);
  std::vector<double> T(4096), X(4096);
  for (int i = 0; i < N; ++i) {
    const double* Ts = tiles.data() + (size_t)(i * (i + 1) / 2 + i) * 4096;
    for (int r = 0; r < 64; ++r)
      for (int c = 0; c < 64; ++c) T[r * 64 + c] = Ts[swz(r, c)];
    std::fill(X.begin(), X.end(), 0.0);
    for (int c = 0; c < 64; ++c)
      for (int r = c; r < 64; ++r) {
        double s = (r == c) ? 1.0 : 0.0;
        for (int k = c; k < r; ++k) s -= T[r * 64 + k] * X[k * 64 + c];
        X[r * 64 + c] = s / T[r * 64 + r];
      }
    double* D = linvT.data() + (size_t)i * 4096;
    for (int r = 0; r < 64; ++r)
      for (int c = 0; c < 64; ++c) D[swz(c, r)] = X[r * 64 + c];  // transpose
  }
  TMP(double, dL, (size_t)nt * 4096);
  H2D(dL.p, tiles.data(), sizeof(double) * tiles.size());
  TMP(double, dLi, (size_t)N * 4096);
  H2D(dLi.p, linvT.data(), sizeof(double) * linvT.size());
  TMP(double, dY, (size_t)N * 4096);
  TMP(int, dflags, nt + N);
  TMP(int, dcnt, 1);
  TMP(int, dinfo, 1);
  TMP(double, xrows, (size_t)N * 3 * 64);
  TMP(double, du, 3 * m);
  std::vector<int2> tk;
  for (int j = 0; j < N; ++j) tk.push_back(make_int2(N, j));
  TMP(int2, dtk, tk.size());
  H2D(dtk.p, tk.data(), sizeof(int2) * tk.size());
  std::vector<int> ready(nt + N, 0);
  for (int t = 0; t < nt; ++t) ready[t] = 2;  // final (sub-diagonal tiles need 2)
  DenseDev d{(int)m, N, nullptr, dL.p, dLi.p, dY.p, dflags.p, dcnt.p, dinfo.p, nullptr, nullptr, nullptr, nullptr,
             nullptr, nullptr, nullptr};
  std::vector<double> ytile((size_t)N * 4096);
  std::vector<double> u(3 * m);
  for (int64_t c0 = 0; c0 < nrhs; c0 += 3) {
    std::fill(ytile.begin(), ytile.end(), 0.0);
    for (int64_t r = 0; r < m; ++r)
      for (int q = 0; q < 3 && c0 + q < nrhs; ++q)
        ytile[(size_t)(r / 64) * 4096 + swz(q, (int)(r % 64))] = g[r * nrhs + c0 + q];
    H2D(dY.p, ytile.data(), sizeof(double) * ytile.size());
    H2D(dflags.p, ready.data(), sizeof(int) * ready.size());
    SPB_CUDA(cudaMemset(dcnt.p, 0, sizeof(int)));
    launch_cholesky_tiles(0, d, dtk.p, (int)tk.size(), std::min<int>(NUM_SMS_B200, N));
    launch_dense_backward(0, d, xrows.p, du.p);
    SPB_CUDA(cudaGetLastError());
    D2H(u.data(), du.p, sizeof(double) * 3 * m);
    for (int64_t r = 0; r < m; ++r)
      for (int q = 0; q < 3 && c0 + q < nrhs; ++q) out[r * nrhs + c0 + q] = u[3 * r + q];
  }
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_op_forward_sub(const spb_factor* fp, int64_t nrhs, const double* b1, const double* b2, double* y1,
                           double* y2) {
  SPB_GUARD_BEGIN
  Factor* f = const_cast<Factor*>(reinterpret_cast<const Factor*>(fp));
  const int64_t n1 = f->n1, n2 = f->n2, n = f->n;
  if (n1 > 0) {
    int rc = build_device_factor(*f);
    if (rc) return rc;
  }
  TMP(double, db, 3 * n);
  TMP(double, dy, 3 * std::max<int64_t>(n1, 1));
  TMP(double, dU, 3 * (n1 > 0 ? std::max<size_t>(device_factor_ubuf(*f->dev_on(cur_device())), 1) : 1));
  TMP(double, df2, 3 * std::max<int64_t>(n2, 1));
  std::vector<double> bh(3 * n), yh(3 * n1), f2h(3 * n2);
  for (int64_t c0 = 0; c0 < nrhs; c0 += 3) {
    std::fill(bh.begin(), bh.end(), 0.0);
    for (int64_t k = 0; k < n1; ++k)
      for (int q = 0; q < 3 && c0 + q < nrhs; ++q) bh[3 * k + q] = b1[f->fill_perm[k] * nrhs + c0 + q];
    for (int64_t k = 0; k < n2; ++k)
      for (int q = 0; q < 3 && c0 + q < nrhs; ++q) bh[3 * (n1 + k) + q] = b2[k * nrhs + c0 + q];
    H2D(db.p, bh.data(), sizeof(double) * 3 * n);
    if (n1 > 0) {
      sparse_forward(0, *f->dev_on(cur_device()), db.p, dy.p, dU.p, df2.p, nullptr);
      SPB_CUDA(cudaGetLastError());
      D2H(yh.data(), dy.p, sizeof(double) * 3 * n1);
      if (n2 > 0) D2H(f2h.data(), df2.p, sizeof(double) * 3 * n2);
    } else {
      for (int64_t k = 0; k < 3 * n2; ++k) f2h[k] = bh[k];
    }
    for (int64_t k = 0; k < n1; ++k)
      for (int q = 0; q < 3 && c0 + q < nrhs; ++q) y1[k * nrhs + c0 + q] = yh[3 * k + q];
    for (int64_t k = 0; k < n2; ++k)
      for (int q = 0; q < 3 && c0 + q < nrhs; ++q) y2[k * nrhs + c0 + q] = f2h[3 * k + q];
  }
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_op_backward_sub(const spb_factor* fp, int64_t nrhs, const double* y1, const double* x2, double* x1) {
  SPB_GUARD_BEGIN
  Factor* f = const_cast<Factor*>(reinterpret_cast<const Factor*>(fp));
  const int64_t n1 = f->n1, n2 = f->n2, n = f->n;
  if (n1 == 0) return SPB_OK;
  {
    int rc = build_device_factor(*f);
    if (rc) return rc;
  }
  TMP(double, dXF, 3 * n);
  TMP(double, dy, 3 * n1);
  std::vector<double> xf(3 * n), yh(3 * n1);
  for (int64_t c0 = 0; c0 < nrhs; c0 += 3) {
    std::fill(xf.begin(), xf.end(), 0.0);
    std::fill(yh.begin(), yh.end(), 0.0);
    for (int64_t k = 0; k < n1; ++k)
      for (int q = 0; q < 3 && c0 + q < nrhs; ++q) yh[3 * k + q] = y1[k * nrhs + c0 + q];
    for (int64_t k = 0; k < n2; ++k)
      for (int q = 0; q < 3 && c0 + q < nrhs; ++q) xf[3 * (n1 + k) + q] = x2[k * nrhs + c0 + q];
    H2D(dy.p, yh.data(), sizeof(double) * 3 * n1);
    H2D(dXF.p, xf.data(), sizeof(double) * 3 * n);
    sparse_backward(0, *f->dev_on(cur_device()), dy.p, dXF.p, nullptr);
    SPB_CUDA(cudaGetLastError());
    D2H(xf.data(), dXF.p, sizeof(double) * 3 * n1);
    for (int64_t k = 0; k < n1; ++k)
      for (int q = 0; q < 3 && c0 + q < nrhs; ++q) x1[f->fill_perm[k] * nrhs + c0 + q] = xf[3 * k + q];
  }
  return SPB_OK;
  SPB_GUARD_END
}

}  // extern "C"
