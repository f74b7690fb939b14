// Standalone dense Schur-complement Cholesky (BASELINE config 4: the scaling
// sweep over dense SPD orders, and the tile-cyclic multi-GPU factorization).
//
// The same persistent tile kernel as the frame solver (dense.cu,
// k_cholesky_tiles) factors an m x m SPD matrix held as lower 64x64 swizzled
// tiles. The matrix comes from the host (spb_dense_set_matrix) or from the
// synthetic generator below (an exponential kernel on
// a sqrt(m) x sqrt(m) surface grid, tuned like the measured sigma0).
//
// Tile-cyclic mode (nranks > 1, one process per GPU): every rank holds a full
// replica of L. Rank r runs the tasks of the tile columns it owns
// (dense_tile_owner), and each finished tile is stored into every peer's
// replica over NVLink through CUDA-IPC mappings, with its readiness flag
// released at system scope. Dependencies are the same per-tile flags as on
// one GPU, so the factorization needs no collective call and the transfer of
// a tile overlaps the math of the next. Emulated mode runs all ranks' replicas
// as ONE launch on one GPU (CTA b serves rank b % P) to test that data path
// where only one GPU exists.
//
// Replaces: linalg.dense_factor (reference linalg.py:432-440, scipy.linalg.
// cholesky / LAPACK dpotrf) for the standalone factorization; info follows
// dpotrf (first failing column, 1-based).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace spb {
void set_error(const std::string& msg);

namespace {
constexpr int TS = 64;
constexpr int TILE = TS * TS;

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// One rank's factor image in one allocation (one IPC handle covers it):
// [L tiles][LinvT tiles][flags (ntiles + N)][counter][info]
struct ReplicaLayout {
  size_t off_L, off_LinvT, off_flags, off_counter, off_info, bytes;
  explicit ReplicaLayout(int N) {
    const size_t nt = (size_t)N * (N + 1) / 2;
    off_L = 0;
    off_LinvT = align256(off_L + nt * TILE * sizeof(double));
    off_flags = align256(off_LinvT + (size_t)N * TILE * sizeof(double));
    off_counter = align256(off_flags + (nt + N) * sizeof(int));
    off_info = off_counter + 256;
    bytes = off_info + 256;
  }
};

struct Replica {
  char* base = nullptr;
  bool owned = false;  // false: an IPC mapping of a peer's allocation
  double* L(const ReplicaLayout& lo) const { return reinterpret_cast<double*>(base + lo.off_L); }
  double* LinvT(const ReplicaLayout& lo) const { return reinterpret_cast<double*>(base + lo.off_LinvT); }
  int* flags(const ReplicaLayout& lo) const { return reinterpret_cast<int*>(base + lo.off_flags); }
  int* counter(const ReplicaLayout& lo) const { return reinterpret_cast<int*>(base + lo.off_counter); }
  int* info(const ReplicaLayout& lo) const { return reinterpret_cast<int*>(base + lo.off_info); }
};

__device__ __forceinline__ void tile_of(int t, int& i, int& j) {
  i = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  j = t - i * (i + 1) / 2;
}

// K_rc = a exp(-|p_r - p_c| / ell) + b delta_rc, p_r = (r mod g, r div g);
// padding rows/columns beyond m are the identity. One CTA per lower tile.
__global__ void __launch_bounds__(256) k_synth_tiles(double* __restrict__ S, int m, int g, double a, double b,
                                                     double inv_ell) {
  int i, j;
  tile_of(blockIdx.x, i, j);
  double* T = S + (size_t)blockIdx.x * TILE;
  for (int q = threadIdx.x; q < TILE; q += 256) {
    const int r = q >> 6, c = q & 63;
    const int gr = i * TS + r, gc = j * TS + c;
    double v;
    if (gr < m && gc < m) {
      const double dx = (double)(gr % g - gc % g), dy = (double)(gr / g - gc / g);
      v = a * exp(-sqrt(dx * dx + dy * dy) * inv_ell) + (gr == gc ? b : 0.0);
    } else {
      v = (gr == gc) ? 1.0 : 0.0;
    }
    T[swz(r, c)] = v;
  }
}

// Row-major m x m (device) -> lower swizzled tiles; the lower triangle of h
// is read and mirrored into the full diagonal tiles; padding = identity.
__global__ void __launch_bounds__(256) k_pack_tiles(const double* __restrict__ h, int64_t m, double* __restrict__ S) {
  int i, j;
  tile_of(blockIdx.x, i, j);
  double* T = S + (size_t)blockIdx.x * TILE;
  for (int q = threadIdx.x; q < TILE; q += 256) {
    const int r = q >> 6, c = q & 63;
    const int64_t gr = (int64_t)i * TS + r, gc = (int64_t)j * TS + c;
    double v;
    if (gr < m && gc < m) v = gc <= gr ? h[gr * m + gc] : h[gc * m + gr];
    else v = (gr == gc) ? 1.0 : 0.0;
    T[swz(r, c)] = v;
  }
}

// Lower swizzled tiles -> row-major m x m (device, preset to zero): the lower
// triangle, plus its mirror when `mirror` (a symmetric matrix).
__global__ void __launch_bounds__(256) k_unpack_tiles(const double* __restrict__ S, int64_t m, int mirror,
                                                      double* __restrict__ h) {
  int i, j;
  tile_of(blockIdx.x, i, j);
  const double* T = S + (size_t)blockIdx.x * TILE;
  for (int q = threadIdx.x; q < TILE; q += 256) {
    const int r = q >> 6, c = q & 63;
    const int64_t gr = (int64_t)i * TS + r, gc = (int64_t)j * TS + c;
    if (gr >= m || gc > gr) continue;
    const double v = T[swz(r, c)];
    h[gr * m + gc] = v;
    if (mirror && gc < gr) h[gc * m + gr] = v;
  }
}

// y_b = sum over the tiles of block row b (fixed order, no atomics):
//   mode 0: A x with A symmetric stored as lower tiles (diagonal tiles full)
//   mode 1: L x,   mode 2: L^T x   (L lower, diagonal tiles lower)
// Row part (tiles (b, j), j <= b): thread (r, q) dots 16 columns of row r.
// Column part (tiles (i, b)): thread (c, grp) dots column c of every 4th tile.
__global__ void __launch_bounds__(256) k_tile_matvec(const double* __restrict__ T, int N, int mode,
                                                     const double* __restrict__ x, double* __restrict__ y) {
  const int b = blockIdx.x, tid = threadIdx.x;
  __shared__ double colp[4][TS];
  double rowacc = 0.0;
  if (mode != 2) {
    const int r = tid >> 2, q = tid & 3;
    for (int j = 0; j <= b; ++j) {
      const double* Tt = T + (size_t)(b * (b + 1) / 2 + j) * TILE;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int c = q * 16 + k;
        rowacc += Tt[swz(r, c)] * x[j * TS + c];
      }
    }
    rowacc += __shfl_xor_sync(0xffffffffu, rowacc, 1);
    rowacc += __shfl_xor_sync(0xffffffffu, rowacc, 2);
  }
  {
    const int c = tid & 63, grp = tid >> 6;
    double acc = 0.0;
    if (mode != 1) {
      for (int i = (mode == 0 ? b + 1 : b) + grp; i < N; i += 4) {
        const double* Tt = T + (size_t)(i * (i + 1) / 2 + b) * TILE;
        for (int r = 0; r < TS; ++r) acc += Tt[swz(r, c)] * x[i * TS + r];
      }
    }
    colp[grp][c] = acc;
  }
  __syncthreads();
  if ((tid & 3) == 0) {
    const int r = tid >> 2;
    y[b * TS + r] = rowacc + ((colp[0][r] + colp[1][r]) + (colp[2][r] + colp[3][r]));
  }
}
// Per-row exponent bounds of the INT8 trailing updates (k_cholesky_oz):
// 2^erow[r] > sqrt(H_rr) >= |L_rc| (L L^T = H), from the diagonal tiles.
__global__ void k_erow_from_diag(const double* __restrict__ tiles, int N, int* __restrict__ erow) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N * TS) return;
  const int b = r / TS, rr = r % TS;
  const double h = tiles[(size_t)(b * (b + 1) / 2 + b) * TILE + swz(rr, rr)];
  int ex = 0;
  frexp(sqrt(fmax(h, 1e-300)), &ex);
  erow[r] = ex;
}
}  // namespace
}  // namespace spb

struct spb_dense {
  int device = 0, rank = 0, nranks = 1, emulate = 0;
  int64_t m = 0;
  int N = 0, grid = 0;
  spb::ReplicaLayout lo{1};
  double* sigma0 = nullptr;
  std::vector<spb::Replica> reps;     // own replica (real) or all P replicas (emulated)
  std::vector<spb::Replica> peers;    // IPC mappings of the other ranks' replicas (real multi-rank)
  std::vector<int2*> tasks;           // per replica
  std::vector<int> ntasks;
  spb::DenseRankJob* jobs = nullptr;  // device copy (MULTI kernel)
  bool jobs_ready = false;
  // single GPU: trailing updates on the INT8 tensor cores (SPB_CHOL_INT8, default on)
  bool int8 = false;
  int* erow = nullptr;
  signed char* Lq = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ~spb_dense() {
    cudaSetDevice(device);
    for (auto& p : peers)
      if (p.base) cudaIpcCloseMemHandle(p.base);
    for (auto& r : reps)
      if (r.base && r.owned) cudaFree(r.base);
    for (auto* t : tasks) cudaFree(t);
    if (jobs) cudaFree(jobs);
    if (sigma0) cudaFree(sigma0);
    if (erow) cudaFree(erow);
    if (Lq) cudaFree(Lq);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (st) cudaStreamDestroy(st);
  }
  bool multi() const { return emulate || nranks > 1; }
  size_t ntiles() const { return (size_t)N * (N + 1) / 2; }
};

namespace spb {
namespace {
int upload_jobs(spb_dense* d) {
  const int R = (int)d->reps.size();
  std::vector<DenseRankJob> jobs(R);
  for (int r = 0; r < R; ++r) {
    DenseRankJob& jb = jobs[r];
    memset(&jb, 0, sizeof(jb));
    const Replica& me = d->reps[r];
    jb.d.m = (int)d->m;
    jb.d.N = d->N;
    jb.d.sigma0 = d->sigma0;
    jb.d.L = me.L(d->lo);
    jb.d.LinvT = me.LinvT(d->lo);
    jb.d.flags = me.flags(d->lo);
    jb.d.counter = me.counter(d->lo);
    jb.d.info = me.info(d->lo);
    // peers: the other emulated replicas, or the IPC-mapped ones
    std::vector<const Replica*> others;
    if (d->emulate) {
      for (int p = 0; p < R; ++p)
        if (p != r) others.push_back(&d->reps[p]);
    } else {
      for (auto& p : d->peers) others.push_back(&p);
    }
    jb.d.peers.n = (int)others.size();
    for (size_t p = 0; p < others.size(); ++p) {
      jb.d.peers.L[p] = others[p]->L(d->lo);
      jb.d.peers.LinvT[p] = others[p]->LinvT(d->lo);
      jb.d.peers.flags[p] = others[p]->flags(d->lo);
    }
    jb.tasks = d->tasks[r];
    jb.ntasks = d->ntasks[r];
  }
  if (!d->jobs) SPB_CUDA(cudaMalloc(&d->jobs, sizeof(DenseRankJob) * R));
  SPB_CUDA(cudaMemcpy(d->jobs, jobs.data(), sizeof(DenseRankJob) * R, cudaMemcpyHostToDevice));
  d->jobs_ready = true;
  return SPB_OK;
}

int check(const spb_dense* d) {
  if (!d) {
    set_error("null dense context");
    return SPB_ERR_ARG;
  }
  SPB_CUDA(cudaSetDevice(d->device));
  return SPB_OK;
}
#define DCHECK(d)                      \
  do {                                 \
    int _s = spb::check(d);            \
    if (_s != SPB_OK) return _s;       \
  } while (0)
}  // namespace
}  // namespace spb

extern "C" {

int32_t spb_dense_rank_tasks(int64_t m, int32_t rank, int32_t nranks, int32_t* ij, int64_t* count) {
  SPB_GUARD_BEGIN
  if (m <= 0 || nranks < 1 || nranks > spb::MAX_DENSE_PEERS + 1 || rank < 0 || rank >= nranks || !count) {
    spb::set_error("spb_dense_rank_tasks: bad arguments");
    return SPB_ERR_ARG;
  }
  const int N = (int)((m + 63) / 64);
  std::vector<int2> tk = nranks == 1 ? spb::cholesky_task_order(N, false, spb::CHOL_LEAD)
                                     : spb::cholesky_rank_tasks(N, rank, nranks, spb::CHOL_LEAD);
  if (ij) {
    if (*count < (int64_t)tk.size()) {
      spb::set_error("spb_dense_rank_tasks: output too small");
      return SPB_ERR_ARG;
    }
    for (size_t t = 0; t < tk.size(); ++t) {
      ij[2 * t] = tk[t].x;
      ij[2 * t + 1] = tk[t].y;
    }
  }
  *count = (int64_t)tk.size();
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_dense_create(int64_t m, int32_t device, int32_t rank, int32_t nranks, int32_t emulate,
                         spb_dense** out) {
  SPB_GUARD_BEGIN
  if (!out || m <= 0 || m > (int64_t)64 * 2000 || nranks < 1 || nranks > spb::MAX_DENSE_PEERS + 1 ||
      (emulate != 0 && emulate != 1) || (!emulate && (rank < 0 || rank >= nranks))) {
    spb::set_error("spb_dense_create: bad arguments");
    return SPB_ERR_ARG;
  }
  *out = nullptr;
  int ndev = 0;
  SPB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) {
    spb::set_error("spb_dense_create: no such CUDA device");
    return SPB_ERR_CUDA;
  }
  SPB_CUDA(cudaSetDevice(device));
  auto d = new spb_dense();
  std::unique_ptr<spb_dense> guard(d);
  d->device = device;
  d->rank = emulate ? 0 : rank;
  d->nranks = nranks;
  d->emulate = emulate;
  d->m = m;
  d->N = (int)((m + 63) / 64);
  d->lo = spb::ReplicaLayout(d->N);
  SPB_CUDA(cudaStreamCreateWithFlags(&d->st, cudaStreamNonBlocking));
  SPB_CUDA(cudaEventCreate(&d->e0));
  SPB_CUDA(cudaEventCreate(&d->e1));
  SPB_CUDA(cudaMalloc(&d->sigma0, d->ntiles() * spb::TILE * sizeof(double)));
  const int R = emulate ? nranks : 1;
  d->reps.resize(R);
  int total = 0;
  for (int r = 0; r < R; ++r) {
    SPB_CUDA(cudaMalloc(&d->reps[r].base, d->lo.bytes));
    d->reps[r].owned = true;
    SPB_CUDA(cudaMemset(d->reps[r].base, 0, d->lo.bytes));
    const int rid = emulate ? r : rank;
    std::vector<int2> tk = nranks == 1 ? spb::cholesky_task_order(d->N, false, spb::CHOL_LEAD)
                                       : spb::cholesky_rank_tasks(d->N, rid, nranks, spb::CHOL_LEAD);
    int2* dt = nullptr;
    SPB_CUDA(cudaMalloc(&dt, sizeof(int2) * std::max<size_t>(1, tk.size())));
    if (!tk.empty()) SPB_CUDA(cudaMemcpy(dt, tk.data(), sizeof(int2) * tk.size(), cudaMemcpyHostToDevice));
    d->tasks.push_back(dt);
    d->ntasks.push_back((int)tk.size());
    total += (int)tk.size();
  }
  // persistent grid: every SM (emulated ranks share them), never more CTAs than tasks
  d->grid = std::max(1, std::min(spb::NUM_SMS_B200, emulate ? std::max(total, R) : d->ntasks[0]));
  if (emulate) d->grid = std::max(d->grid, R);
  if (emulate || nranks == 1) {
    int s = spb::upload_jobs(d);
    if (s != SPB_OK) return s;
  }
  // one GPU: the INT8 tensor-core path needs the per-row bounds and 32 KB of
  // digit planes per tile (int32 accumulation stays exact up to m ~ 98K:
  // 4 digit pairs x 64^2 x m < 2^31)
  d->int8 = !d->multi() && spb::chol_int8_enabled() && m <= 98304;
  if (d->int8) {
    SPB_CUDA(cudaMalloc(&d->erow, sizeof(int) * (size_t)d->N * spb::TS));
    SPB_CUDA(cudaMalloc(&d->Lq, d->ntiles() * (size_t)32768));
  }
  *out = guard.release();
  return SPB_OK;
  SPB_GUARD_END
}

void spb_dense_destroy(spb_dense* d) { delete d; }

int32_t spb_dense_set_matrix(spb_dense* d, const double* h) {
  SPB_GUARD_BEGIN
  DCHECK(d);
  if (!h) {
    spb::set_error("spb_dense_set_matrix: null matrix");
    return SPB_ERR_ARG;
  }
  const size_t bytes = sizeof(double) * (size_t)d->m * (size_t)d->m;
  double* tmp = nullptr;
  SPB_CUDA(cudaMallocAsync(&tmp, bytes, d->st));
  cudaError_t e = cudaMemcpyAsync(tmp, h, bytes, cudaMemcpyHostToDevice, d->st);
  if (e == cudaSuccess) spb::k_pack_tiles<<<(unsigned)d->ntiles(), 256, 0, d->st>>>(tmp, d->m, d->sigma0);
  cudaFreeAsync(tmp, d->st);
  SPB_CUDA(e);
  SPB_CUDA(cudaGetLastError());
  SPB_CUDA(cudaStreamSynchronize(d->st));
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_dense_synthetic(spb_dense* d, double a, double b, double ell) {
  SPB_GUARD_BEGIN
  DCHECK(d);
  if (!(ell > 0.0)) {
    spb::set_error("spb_dense_synthetic: ell must be positive");
    return SPB_ERR_ARG;
  }
  const int g = (int)std::ceil(std::sqrt((double)d->m));
  spb::k_synth_tiles<<<(unsigned)d->ntiles(), 256, 0, d->st>>>(d->sigma0, (int)d->m, g, a, b, 1.0 / ell);
  SPB_CUDA(cudaGetLastError());
  SPB_CUDA(cudaStreamSynchronize(d->st));
  return SPB_OK;
  SPB_GUARD_END
}

static int32_t unpack(spb_dense* d, const double* tiles_dev, double* h, bool lower_only) {
  const size_t bytes = sizeof(double) * (size_t)d->m * (size_t)d->m;
  double* tmp = nullptr;
  SPB_CUDA(cudaMallocAsync(&tmp, bytes, d->st));
  cudaError_t e = cudaMemsetAsync(tmp, 0, bytes, d->st);
  if (e == cudaSuccess) {
    spb::k_unpack_tiles<<<(unsigned)d->ntiles(), 256, 0, d->st>>>(tiles_dev, d->m, lower_only ? 0 : 1, tmp);
    e = cudaMemcpyAsync(h, tmp, bytes, cudaMemcpyDeviceToHost, d->st);
  }
  cudaFreeAsync(tmp, d->st);
  SPB_CUDA(e);
  SPB_CUDA(cudaGetLastError());
  SPB_CUDA(cudaStreamSynchronize(d->st));
  return SPB_OK;
}

int32_t spb_dense_get_matrix(spb_dense* d, double* h) {
  SPB_GUARD_BEGIN
  DCHECK(d);
  SPB_CUDA(cudaStreamSynchronize(d->st));
  return unpack(d, d->sigma0, h, false);
  SPB_GUARD_END
}

int32_t spb_dense_get_factor(spb_dense* d, int32_t replica, double* chol) {
  SPB_GUARD_BEGIN
  DCHECK(d);
  if (replica < 0 || replica >= (int)d->reps.size() || !chol) {
    spb::set_error("spb_dense_get_factor: bad replica");
    return SPB_ERR_ARG;
  }
  SPB_CUDA(cudaStreamSynchronize(d->st));
  return unpack(d, d->reps[replica].L(d->lo), chol, true);
  SPB_GUARD_END
}

int32_t spb_dense_ipc_handle(spb_dense* d, uint8_t* out) {
  SPB_GUARD_BEGIN
  DCHECK(d);
  if (!out || d->emulate) {
    spb::set_error("spb_dense_ipc_handle: needs a real (non-emulated) context");
    return SPB_ERR_ARG;
  }
  cudaIpcMemHandle_t h;
  SPB_CUDA(cudaIpcGetMemHandle(&h, d->reps[0].base));
  memcpy(out, &h, sizeof(h));
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_dense_open_peers(spb_dense* d, const uint8_t* handles) {
  SPB_GUARD_BEGIN
  DCHECK(d);
  if (!handles || d->emulate || d->nranks < 2 || !d->peers.empty()) {
    spb::set_error("spb_dense_open_peers: needs a real multi-rank context, once");
    return SPB_ERR_ARG;
  }
  for (int p = 0; p < d->nranks; ++p) {
    if (p == d->rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + (size_t)p * SPB_DENSE_IPC_BYTES, sizeof(h));
    void* ptr = nullptr;
    SPB_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    spb::Replica r;
    r.base = static_cast<char*>(ptr);
    r.owned = false;
    d->peers.push_back(r);
  }
  return spb::upload_jobs(d);
  SPB_GUARD_END
}

// Diagnostics of the IPC plumbing without any kernel that waits on a peer:
// write `value` into the own replica's first L tile and its flag words, or
// read the first L value and flag word of peer slot `peer` (rank order,
// own rank skipped) through the mapped allocation.
int32_t spb_dense_debug_replica(spb_dense* d, int32_t peer, double value, double* out_value, int32_t* out_flag) {
  SPB_GUARD_BEGIN
  DCHECK(d);
  if (peer < 0) {
    std::vector<double> t(spb::TILE, value);
    SPB_CUDA(cudaMemcpy(d->reps[0].L(d->lo), t.data(), sizeof(double) * spb::TILE, cudaMemcpyHostToDevice));
    std::vector<int> f(16, (int)value);
    SPB_CUDA(cudaMemcpy(d->reps[0].flags(d->lo), f.data(), sizeof(int) * 16, cudaMemcpyHostToDevice));
    return SPB_OK;
  }
  if (peer >= (int)d->peers.size() || !out_value || !out_flag) {
    spb::set_error("spb_dense_debug_replica: no such peer");
    return SPB_ERR_ARG;
  }
  SPB_CUDA(cudaMemcpy(out_value, d->peers[peer].L(d->lo), sizeof(double), cudaMemcpyDeviceToHost));
  SPB_CUDA(cudaMemcpy(out_flag, d->peers[peer].flags(d->lo), sizeof(int), cudaMemcpyDeviceToHost));
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_dense_reset(spb_dense* d) {
  SPB_GUARD_BEGIN
  DCHECK(d);
  for (auto& r : d->reps) {
    SPB_CUDA(cudaMemsetAsync(r.flags(d->lo), 0, sizeof(int) * (d->ntiles() + d->N), d->st));
    SPB_CUDA(cudaMemsetAsync(r.base + d->lo.off_counter, 0, 512, d->st));  // counter + info
  }
  SPB_CUDA(cudaStreamSynchronize(d->st));
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_dense_set_cholesky_kind(spb_dense* d, int32_t kind) {
  SPB_GUARD_BEGIN
  DCHECK(d);
  if (kind == 1 && (d->multi() || d->m > 98304)) {
    spb::set_error("spb_dense_set_cholesky_kind: the INT8 path is single-GPU, m <= 98304");
    return SPB_ERR_ARG;
  }
  d->int8 = kind == 1;
  if (d->int8 && !d->erow) {
    SPB_CUDA(cudaMalloc(&d->erow, sizeof(int) * (size_t)d->N * spb::TS));
    SPB_CUDA(cudaMalloc(&d->Lq, d->ntiles() * (size_t)32768));
  }
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_dense_cholesky_kind(spb_dense* d, int32_t* kind) {
  if (!d || !kind) {
    spb::set_error("spb_dense_cholesky_kind: bad arguments");
    return SPB_ERR_ARG;
  }
  *kind = d->int8 ? 1 : 0;
  return SPB_OK;
}

int32_t spb_dense_launch(spb_dense* d) {
  SPB_GUARD_BEGIN
  DCHECK(d);
  if (!d->jobs_ready) {
    spb::set_error("spb_dense_launch: peers not opened (spb_dense_open_peers)");
    return SPB_ERR_ARG;
  }
  SPB_CUDA(cudaEventRecord(d->e0, d->st));
  if (!d->multi()) {
    const spb::Replica& r = d->reps[0];
    spb::DenseDev dd{};
    dd.m = (int)d->m;
    dd.N = d->N;
    dd.sigma0 = d->sigma0;
    dd.L = r.L(d->lo);
    dd.LinvT = r.LinvT(d->lo);
    dd.flags = r.flags(d->lo);
    dd.counter = r.counter(d->lo);
    dd.info = r.info(d->lo);
    if (d->int8) {
      spb::k_erow_from_diag<<<(d->N * spb::TS + 255) / 256, 256, 0, d->st>>>(d->sigma0, d->N, d->erow);
      dd.erow = d->erow;
      dd.Lq = d->Lq;
    }
    spb::launch_cholesky(d->st, dd, d->tasks[0], d->ntasks[0], d->grid, false, d->int8);
  } else {
    spb::launch_cholesky_ranks(d->st, d->jobs, (int)d->reps.size(), d->grid);
  }
  SPB_CUDA(cudaGetLastError());
  SPB_CUDA(cudaEventRecord(d->e1, d->st));
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_dense_finish(spb_dense* d, double* ms, int64_t* info) {
  SPB_GUARD_BEGIN
  DCHECK(d);
  SPB_CUDA(cudaEventSynchronize(d->e1));
  SPB_CUDA(cudaGetLastError());
  float t = 0.f;
  SPB_CUDA(cudaEventElapsedTime(&t, d->e0, d->e1));
  if (ms) *ms = t;
  int64_t first = 0;
  for (auto& r : d->reps) {
    int hi = 0;
    SPB_CUDA(cudaMemcpy(&hi, r.info(d->lo), sizeof(int), cudaMemcpyDeviceToHost));
    if (hi > 0 && (first == 0 || hi < first)) first = hi;
  }
  if (info) *info = first;
  if (first > 0) {
    spb::set_error("dense factorization failed: non-positive pivot");
    return SPB_ERR_INDEFINITE;
  }
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_dense_factor(spb_dense* d, int32_t reps, double* ms, int64_t* info) {
  SPB_GUARD_BEGIN
  DCHECK(d);
  if (reps < 1 || (d->nranks > 1 && !d->emulate)) {
    spb::set_error("spb_dense_factor: single-process contexts only (multi-rank: reset/launch/finish)");
    return SPB_ERR_ARG;
  }
  double total = 0.0;
  for (int k = 0; k < reps; ++k) {
    int s = spb_dense_reset(d);
    if (s != SPB_OK) return s;
    s = spb_dense_launch(d);
    if (s != SPB_OK) return s;
    double t = 0.0;
    s = spb_dense_finish(d, &t, info);
    if (s != SPB_OK) return s;
    total += t;
  }
  if (ms) *ms = total / reps;
  return SPB_OK;
  SPB_GUARD_END
}

int32_t spb_dense_residual(spb_dense* d, int32_t replica, const double* v, double* out2) {
  SPB_GUARD_BEGIN
  DCHECK(d);
  if (replica < 0 || replica >= (int)d->reps.size() || !v || !out2) {
    spb::set_error("spb_dense_residual: bad arguments");
    return SPB_ERR_ARG;
  }
  const size_t n = (size_t)d->N * 64;
  std::vector<double> hv(n, 0.0), a(n), b(n);
  std::copy(v, v + d->m, hv.begin());
  struct Buf {  // x | A v | L^T v | L L^T v
    double* p = nullptr;
    ~Buf() {
      if (p) cudaFree(p);
    }
  } buf;
  SPB_CUDA(cudaMalloc(&buf.p, 4 * n * sizeof(double)));
  double *x = buf.p, *y = x + n, *w = y + n, *z = w + n;
  SPB_CUDA(cudaMemcpy(x, hv.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  const double* L = d->reps[replica].L(d->lo);
  spb::k_tile_matvec<<<d->N, 256, 0, d->st>>>(d->sigma0, d->N, 0, x, y);  // A v
  spb::k_tile_matvec<<<d->N, 256, 0, d->st>>>(L, d->N, 2, x, w);          // L^T v
  spb::k_tile_matvec<<<d->N, 256, 0, d->st>>>(L, d->N, 1, w, z);          // L L^T v
  SPB_CUDA(cudaGetLastError());
  SPB_CUDA(cudaStreamSynchronize(d->st));
  SPB_CUDA(cudaMemcpy(a.data(), y, n * sizeof(double), cudaMemcpyDeviceToHost));
  SPB_CUDA(cudaMemcpy(b.data(), z, n * sizeof(double), cudaMemcpyDeviceToHost));
  double rr = 0.0, aa = 0.0;
  for (int64_t k = 0; k < d->m; ++k) {
    rr += (a[k] - b[k]) * (a[k] - b[k]);
    aa += a[k] * a[k];
  }
  out2[0] = std::sqrt(rr);
  out2[1] = std::sqrt(aa);
  return SPB_OK;
  SPB_GUARD_END
}

}  // extern "C"
