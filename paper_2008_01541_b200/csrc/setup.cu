// Proxy setup on the device: collision.scatter_proxies
// (reference collision.py:255-300).
//
// For every surface triangle whose three vertices lie in the region, the
// owning tetrahedron is the FIRST tet (in element order) with that face (the
// reference's owner map is a setdefault over all tets' faces,
// collision.py:_surface_owner_map); the proxy weights put the sub-triangle
// barycentric points on the owner's slots of the face vertices in the
// owner's winding, 0 on the opposite vertex. Output order: surface-triangle
// order, then sample-point order (the reference's append order).
//
// Device form: every tet face is packed to one sorted-vertex int64 key
// (node ids < 2^21, as mesh.boundary_face_index packs them) and stably
// radix-sorted with its (element * 4 + face) index, so the first match of a
// key is the first owner; each selected surface triangle finds it by binary
// search, and an exclusive scan of the per-triangle counts places its proxies.
// Everything is integer work plus copies of the given barycentric points:
// the result is bit-identical to the reference's.
#include <algorithm>

#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.cuh"

namespace spb {
void set_error(const std::string& msg);

namespace {
__constant__ int kTetFaces[4][3] = {{0, 2, 1}, {0, 1, 3}, {0, 3, 2}, {1, 2, 3}};  // mesh.TET_FACES

__device__ __forceinline__ unsigned long long face_key(long long a, long long b, long long c) {
  // sort the triple (3 compare-swaps), pack 21 bits each
  if (a > b) { const long long t = a; a = b; b = t; }
  if (b > c) { const long long t = b; b = c; c = t; }
  if (a > b) { const long long t = a; a = b; b = t; }
  return ((unsigned long long)a << 42) | ((unsigned long long)b << 21) | (unsigned long long)c;
}

__global__ void k_face_keys(const long long* __restrict__ tets, long long ne, unsigned long long* __restrict__ keys,
                            long long* __restrict__ vals) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= 4 * ne) return;
  const long long e = i >> 2;
  const int f = (int)(i & 3);
  const long long* t = tets + 4 * e;
  keys[i] = face_key(t[kTetFaces[f][0]], t[kTetFaces[f][1]], t[kTetFaces[f][2]]);
  vals[i] = i;
}

__global__ void k_scatter_count(const long long* __restrict__ tris, long long ns, const unsigned char* __restrict__ mask,
                                int per, int* __restrict__ cnt) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= ns) return;
  const long long* v = tris + 3 * t;
  cnt[t] = (mask[v[0]] && mask[v[1]] && mask[v[2]]) ? per : 0;
}

__global__ void k_scatter_emit(const long long* __restrict__ tris, long long ns, const int* __restrict__ cnt,
                               const int* __restrict__ off, int per, const double* __restrict__ bary,
                               const unsigned long long* __restrict__ keys, const long long* __restrict__ vals,
                               long long nf, const long long* __restrict__ tets, long long* __restrict__ out_elem,
                               double* __restrict__ out_w, int* __restrict__ err) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= ns || cnt[t] == 0) return;
  const long long* v = tris + 3 * t;
  const unsigned long long key = face_key(v[0], v[1], v[2]);
  long long lo = 0, hi = nf;  // first sorted face with this key
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (keys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  if (lo >= nf || keys[lo] != key) {
    atomicExch(err, 1);  // not a face of any tet (the reference raises KeyError)
    return;
  }
  const long long fv = vals[lo];
  const long long e = fv >> 2;
  const int f = (int)(fv & 3);
  const long long* tet = tets + 4 * e;
  int slot[3];
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const long long w = tet[kTetFaces[f][l]];  // the owner's winding
    int s = 3;
    for (int k = 3; k >= 0; --k)
      if (tet[k] == w) s = k;  // first slot holding the vertex (tet.index)
    slot[l] = s;
  }
  for (int b = 0; b < per; ++b) {
    const long long o = (long long)off[t] + b;
    double w4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int l = 0; l < 3; ++l) w4[slot[l]] = bary[3 * b + l];  // later slots win, as the reference's loop
    out_elem[o] = e;
#pragma unroll
    for (int k = 0; k < 4; ++k) out_w[4 * o + k] = w4[k];
  }
}

template <typename T>
struct Buf {
  T* p = nullptr;
  explicit Buf(size_t n) {
    if (cudaMalloc(&p, sizeof(T) * (n ? n : 1)) != cudaSuccess) p = nullptr;
  }
  ~Buf() {
    if (p) cudaFree(p);
  }
};
}  // namespace
}  // namespace spb

using namespace spb;

extern "C" {

// collision.scatter_proxies on the device. out_elem / out_weights hold
// ns * per_element entries; *count receives the number written. Returns
// SPB_ERR_ARG when a node id does not fit the 21-bit face key or a selected
// surface triangle is no tet's face (the host path then applies).
int32_t spb_scatter_proxies(const int64_t* tets, int64_t ne, int64_t n, const int64_t* surface_tris, int64_t ns,
                            const uint8_t* node_mask, int32_t per_element, const double* bary, int64_t* out_elem,
                            double* out_weights, int64_t* count) {
  SPB_GUARD_BEGIN
  if (!count || ne < 0 || ns < 0 || n < 0 || per_element < 1) {
    set_error("spb_scatter_proxies: bad arguments");
    return SPB_ERR_ARG;
  }
  *count = 0;
  if (n >= (int64_t(1) << 21)) { set_error("node ids exceed the 21-bit face key"); return SPB_ERR_ARG; }
  if (ns == 0 || ne == 0) return SPB_OK;
  const long long nf = 4 * ne;
  Buf<long long> d_tets(4 * ne), d_tris(3 * ns), d_vals(nf), d_vals2(nf), d_elem(ns * per_element);
  Buf<unsigned long long> d_keys(nf), d_keys2(nf);
  Buf<unsigned char> d_mask(n);
  Buf<int> d_cnt(ns), d_off(ns), d_err(1);
  Buf<double> d_bary(3 * per_element), d_w(4 * ns * per_element);
  if (!d_tets.p || !d_tris.p || !d_vals.p || !d_vals2.p || !d_elem.p || !d_keys.p || !d_keys2.p || !d_mask.p ||
      !d_cnt.p || !d_off.p || !d_err.p || !d_bary.p || !d_w.p) {
    set_error("cudaMalloc failed (scatter_proxies)");
    return SPB_ERR_CUDA;
  }
  SPB_CUDA(cudaMemcpy(d_tets.p, tets, sizeof(long long) * 4 * ne, cudaMemcpyHostToDevice));
  SPB_CUDA(cudaMemcpy(d_tris.p, surface_tris, sizeof(long long) * 3 * ns, cudaMemcpyHostToDevice));
  SPB_CUDA(cudaMemcpy(d_mask.p, node_mask, n, cudaMemcpyHostToDevice));
  SPB_CUDA(cudaMemcpy(d_bary.p, bary, sizeof(double) * 3 * per_element, cudaMemcpyHostToDevice));
  SPB_CUDA(cudaMemset(d_err.p, 0, sizeof(int)));
  const int B = 256;
  k_face_keys<<<(unsigned)((nf + B - 1) / B), B>>>(d_tets.p, ne, d_keys.p, d_vals.p);
  SPB_CUDA(cudaGetLastError());
  // stable radix sort on the 63-bit keys: equal keys keep element order
  size_t tmp_bytes = 0, tmp2 = 0;
  SPB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_keys.p, d_keys2.p, d_vals.p, d_vals2.p, (int)nf, 0,
                                           63));
  SPB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, d_cnt.p, d_off.p, (int)ns));
  Buf<unsigned char> d_tmp(std::max(tmp_bytes, tmp2));
  if (!d_tmp.p) { set_error("cudaMalloc failed (scatter_proxies)"); return SPB_ERR_CUDA; }
  SPB_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp.p, tmp_bytes, d_keys.p, d_keys2.p, d_vals.p, d_vals2.p, (int)nf, 0,
                                           63));
  k_scatter_count<<<(unsigned)((ns + B - 1) / B), B>>>(d_tris.p, ns, d_mask.p, per_element, d_cnt.p);
  SPB_CUDA(cudaGetLastError());
  size_t t2 = std::max(tmp_bytes, tmp2);
  SPB_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp.p, t2, d_cnt.p, d_off.p, (int)ns));
  k_scatter_emit<<<(unsigned)((ns + B - 1) / B), B>>>(d_tris.p, ns, d_cnt.p, d_off.p, per_element, d_bary.p, d_keys2.p,
                                                      d_vals2.p, nf, d_tets.p, d_elem.p, d_w.p, d_err.p);
  SPB_CUDA(cudaGetLastError());
  int err = 0, last_off = 0, last_cnt = 0;
  SPB_CUDA(cudaMemcpy(&err, d_err.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (err) { set_error("a selected surface triangle is no tet's face"); return SPB_ERR_ARG; }
  SPB_CUDA(cudaMemcpy(&last_off, d_off.p + (ns - 1), sizeof(int), cudaMemcpyDeviceToHost));
  SPB_CUDA(cudaMemcpy(&last_cnt, d_cnt.p + (ns - 1), sizeof(int), cudaMemcpyDeviceToHost));
  const int64_t total = (int64_t)last_off + last_cnt;
  if (total > 0) {
    SPB_CUDA(cudaMemcpy(out_elem, d_elem.p, sizeof(long long) * total, cudaMemcpyDeviceToHost));
    SPB_CUDA(cudaMemcpy(out_weights, d_w.p, sizeof(double) * 4 * total, cudaMemcpyDeviceToHost));
  }
  *count = total;
  return SPB_OK;
  SPB_GUARD_END
}

}  // extern "C"
