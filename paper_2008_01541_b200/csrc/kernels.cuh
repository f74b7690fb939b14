// Host-side launchers of the device kernels (one translation unit per family).
#pragma once

#include <vector>

#include "common.cuh"

namespace spb {

// ---------------------------------------------------------------- element.cu
void launch_local_forces(cudaStream_t st, int nsub, const int* sub, const int4* tets, const double* x,
                         const double* dmi, const double* vol, int64_t ne, double* R, double* Q,
                         const ElemParams& p, double* G, int project);
void launch_gather_forces(cudaStream_t st, int nout, const int* ptr, const int* src, const double* G, int nsub,
                          const int* out_node, const int* aptr, const int* aidx, const double* ak,
                          const double* atgt, const double* x, double* out);
int energy_blocks(int64_t ne);
void launch_elastic_energy(cudaStream_t st, int64_t ne, const int4* tets, const double* x, const double* dmi,
                           const double* vol, const double* R, const double* Q, const ElemParams& p,
                           double* partial);
void launch_deformation_gradients(cudaStream_t st, int nsub, const int* sub, const int4* tets, const double* x,
                                  const double* dmi, int64_t ne, double* F);
void launch_svd_op(cudaStream_t st, int64_t k, const double* F, double* U, double* S, double* V, double* R,
                   double* Q, double smin, double smax);

// -------------------------------------------------------------- collision.cu
struct ProxyDev {
  int P;
  const int* elem;    // (P)
  const double* w;    // (P,4)
  const double* c;    // (P)
  const int* local;   // (P,4) trailing-local node ids (perm - n1)
};
void launch_detect(cudaStream_t st, const ProxyDev& px, const int4* tets, const double* x, const ShapeDev* shapes,
                   const ColliderSet* cols, uint8_t* active, double* target, double* depth);
void launch_build_g(cudaStream_t st, int m, const double* f_tilde2, const int* bptr, const int* bsrc,
                    const double* Gb, int nbeta, const ProxyDev& px, const int4* tets, const double* x,
                    const uint8_t* active, const double* target, const int* cptr, const int* csrc, double* g,
                    double* ytile);
int proxy_blocks(int P);
void launch_proxy_final(cudaStream_t st, const ProxyDev& px, const int4* tets, const double* x,
                        const ShapeDev* shapes, const ColliderSet* cols, const uint8_t* active,
                        const double* target, double* partial);

// ------------------------------------------------------------------ dense.cu
// Tile-cyclic multi-GPU factorization (BASELINE config 4): every rank keeps a
// full replica of L; the CTA that finishes a tile also stores it into each
// peer's replica over NVLink (P2P stores through CUDA-IPC mappings) and
// releases the peer's readiness flag at system scope. n = 0 on one GPU.
constexpr int MAX_DENSE_PEERS = 7;
struct DensePeers {
  int n;
  double* L[MAX_DENSE_PEERS];
  double* LinvT[MAX_DENSE_PEERS];
  int* flags[MAX_DENSE_PEERS];
};
struct DenseDev {
  int m, N;                  // order and tile count (T = 64)
  const double* sigma0;      // lower tiles, tile-major (diagonal tiles full)
  double* L;                 // factor tiles
  double* LinvT;             // transposed inverse diagonal tiles (N)
  double* Y;                 // RHS tile row (N tiles): rows 0..2 = g^T, then y^T
  int* flags;                // N(N+1)/2 + N readiness flags
  int* counter;              // task counter
  int* info;                 // first failing column + 1 (0 = ok)
  // C22 by tile: entries (tile-local r*64+c) and their contributions
  // (proxy j, slot a, slot b) in the reference's COO order
  const int* c22_tile_ptr;   // (ntiles+1)
  const int* c22_ent_rc;     // (E)
  const int* c22_ent_ptr;    // (E+1)
  const int* c22_contrib;    // (C) j*16 + a*4 + b
  const double* proxy_w;
  const double* proxy_c;
  const uint8_t* active;
  unsigned long long* trace;  // optional: per task {claim, k-loop done, finalize done, sm}
  DensePeers peers;           // replicas this rank also writes (tile-cyclic mode)
  // emulated-FP64 trailing updates on the INT8 tensor cores (k_cholesky_oz):
  // per row a power-of-two bound 2^erow[r] > max |L_r.|, and per L tile its 8
  // base-2^7 digit planes (int8, canonical K-major tcgen05 layout, 32 KB)
  const int* erow;
  signed char* Lq;
};
// one rank's share of a tile-cyclic factorization: its replica, peers and task list
struct DenseRankJob {
  DenseDev d;
  const int2* tasks;
  int ntasks;
};
int dense_tile_count(int N);
size_t cholesky_smem_bytes();
// pdl: launched programmatically behind build_g (only the RHS row waits for it)
void launch_cholesky_tiles(cudaStream_t st, const DenseDev& d, const int2* tasks, int ntasks, int grid, bool pdl = false);
// the frame's factorization: k_cholesky_oz (INT8 tensor-core k-loop) when
// int8, else k_cholesky_tiles (FP64 DMMA)
void launch_cholesky(cudaStream_t st, const DenseDev& d, const int2* tasks, int ntasks, int grid, bool pdl, bool int8);
// SPB_CHOL_INT8 (default 1): contexts factor with the INT8 tensor-core path
bool chol_int8_enabled();
void chol_int8_diag_nomma(int on);  // diagnostics (trace only): skip the INT8 MMAs
std::vector<int2> cholesky_task_order(int N, bool with_rhs, int lead);
// P ranks (real: one job per process, P = 1 per launch; emulated: one launch
// over all ranks' replicas, CTA b serving rank b % P)
void launch_cholesky_ranks(cudaStream_t st, const DenseRankJob* jobs, int P, int grid);
int dense_tile_owner(int i, int j, int nranks);
std::vector<int2> cholesky_rank_tasks(int N, int rank, int nranks, int lead);
constexpr int CHOL_LEAD = 2;
void launch_dense_backward(cudaStream_t st, const DenseDev& d, double* xrows, double* u,
                           unsigned long long* trace = nullptr, bool preset = false);
void dense_backward_preset(cudaStream_t st, const DenseDev& d, double* xrows);  // xrows <- sentinel
void launch_sym_tile_gemv(cudaStream_t st, const DenseDev& d, const double* u, double* partial);
void launch_sym_tile_gemv_reduce(cudaStream_t st, const DenseDev& d, const double* partial, double* out);
// max_ctas > 0 caps the persistent grid (beside the backward sweep); the
// result is bitwise independent of the grid (per-tile partials, fixed-order sums)
void launch_sym_gemv(cudaStream_t st, const DenseDev& d, const double* u, double* partial, double* out, bool pdl,
                     int max_ctas = 0);

// -------------------------------------------------------------------- pcg.cu
struct PcgDev {
  int n;                                     // rows (context factor order)
  const int* rowptr;
  const int* col;
  const double* val;                         // A + C22, full CSR
  const double* dinv;                        // Jacobi: 1 / diag
  const double* b;                           // (n,3)
  double *x, *r, *z, *p, *q;                 // (n,3)
  double* partial;                           // pcg_partial_doubles()
  unsigned* bar;                             // grid barrier counter
  double tol;
  int max_iters;
  int* iters;                                // [3] per column, [3] = iteration of a p'Ap <= 0 (0: none)
  double* resid;                             // [3] |A x - b| / |b|
};
int pcg_grid();
size_t pcg_partial_doubles();
int launch_pcg_values(cudaStream_t st, int nnz, const double* aval, double* val, int nent, const int* pos,
                      const int* eptr, const int* contrib, const double* w, const double* cst,
                      const uint8_t* active, int n, const int* diag_pos, double* dinv);
int launch_pcg(cudaStream_t st, const PcgDev& d);

// ----------------------------------------------------------------- sparse.cu
struct DeviceFactor;
int build_device_factor(Factor& f);
struct SweepWork {
  double* VZ = nullptr;     // gathered rows (forward v / backward z)
  double* P = nullptr;      // backward tile partials
  int* chunk_cnt = nullptr; // backward chunk arrivals
  int* flow_cnt = nullptr;  // dataflow counters
};
int sweep_work_alloc(const DeviceFactor& d, SweepWork& w);
void sweep_work_free(SweepWork& w);
// w == nullptr: the factor's own workspace (one-shot ops; not for concurrent use)
void sparse_forward(cudaStream_t st, const DeviceFactor& d, const double* b, double* y, double* U, double* f2,
                    int* launches, const SweepWork* w = nullptr);
void sparse_backward(cudaStream_t st, const DeviceFactor& d, const double* y, double* XF, int* launches,
                     const SweepWork* w = nullptr);
size_t device_factor_ubuf(const DeviceFactor& df);
int device_factor_levels(const DeviceFactor& df);

// ----------------------------------------------------------------- update.cu
void launch_proxy_wu(cudaStream_t st, const ProxyDev& px, const uint8_t* active, const double* u2, double* v);
int update_blocks(int m);
void launch_inner_update(cudaStream_t st, int m, const double* u2, const double* s0u, const int* kptr,
                         const int* kidx, const double* kval, const double* g, const double* pw, const double* v,
                         const int* cptr, const int* csrc, double* f_tilde2, double* u2acc, double* x,
                         const int* x2_ids, double* rpartial);
void launch_scatter_add(cudaStream_t st, int cnt, const int* node, const double* X, double* x);
void launch_u2acc_to_xf(cudaStream_t st, int m, const double* u2, double* u2acc, double* xf2);
void launch_gather3(cudaStream_t st, int cnt, const int* idx, const double* src, double* out);
int attachment_blocks(int na);
void launch_attachment_energy(cudaStream_t st, int na, const int* nodes, const double* k, const double* tgt,
                              const double* x, double* partial);
void launch_finish_metrics(cudaStream_t st, const double* e_part, int ne_b, const double* a_part, int na_b,
                           const double* p_part, int np_b, const double* r_part, int nr_b, const uint8_t* active,
                           int P, int have_residual, double* out);

}  // namespace spb
