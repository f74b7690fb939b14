/*
 * schurpd_b200 — C ABI of the B200-native per-frame Schur-complement PD solve.
 *
 * Drop-in boundary for the reference package `schurpd` (arXiv 2008.01541
 * reference, /root/reference/pkg/src/schurpd). The reference has no FFI of its
 * own; its seam is the Python solver registry and dataclasses
 * (solver.py:606-614 `SOLVE_FUNCTIONS` / `solve_frame`). Every entry point
 * below replaces one reference function at that seam and is bound by the
 * Python shim `paper_2008_01541_b200/_native.py` (ctypes):
 *
 *   spb_factor_*        <- linalg.partial_cholesky          (linalg.py:329-382)
 *                          + fill_ordering                  (linalg.py:280-292)
 *   spb_ctx_create      <- build_system's device residency  (solver.py:246-296)
 *   spb_ctx_step        <- solve_frame_schur                (solver.py:387-455)
 *                          incl. _finish_metrics            (solver.py:373-384)
 *   spb_ctx_set_pose    <- harness.Simulation.pose output   (harness.py:575-590)
 *   spb_ctx_frame_pcg   <- solve_frame_pcg                  (solver.py:542-603)
 *   spb_ctx_set_state / spb_ctx_get_state
 *                       <- SolverState fields               (solver.py:116-145)
 *   spb_op_*            <- the public per-op helpers of the hot path:
 *                          mesh.deformation_gradients       (mesh.py:239-244)
 *                          material.polar_rotations/signed_svd/biphasic_projections
 *                                                           (material.py:248-294)
 *                          material.elastic_forces/elastic_energy (material.py:328-378)
 *                          collision.detect/penetration_depths (collision.py:316-359)
 *                          linalg.forward_sub/backward_sub  (linalg.py:385-414)
 *                          linalg.dense_factor/dense_solve  (linalg.py:432-461)
 *   spb_dense_*         <- linalg.dense_factor as a standalone, possibly
 *                          tile-cyclic multi-GPU factorization (linalg.py:432-440;
 *                          BASELINE config 4)
 *
 * Conventions: plain pointers and sizes, no torch types. All arrays are
 * host memory, C-contiguous, float64 / int64 unless stated. Every call returns
 * an SPB_* status; spb_last_error() returns the thread's last message.
 * Status -> reference exception (errors.py:4-61), mapped by the shim:
 *   SPB_ERR_ARG        -> InvalidArgumentError
 *   SPB_ERR_INDEFINITE -> IndefiniteMatrixError(column = *info)
 *   SPB_ERR_PARTITION  -> PartitionError
 *   SPB_ERR_SETUP      -> SolverSetupError
 *   SPB_ERR_CUDA       -> DeviceError (no CPU fallback exists)
 * Threading: one context = one device + one stream + one host thread
 * ("one frame is solved by a single logical thread of control").
 */
#ifndef SCHURPD_B200_H
#define SCHURPD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPB_OK 0
#define SPB_ERR_ARG 1
#define SPB_ERR_INDEFINITE 2
#define SPB_ERR_PARTITION 3
#define SPB_ERR_SETUP 4
#define SPB_ERR_CUDA 5
#define SPB_ERR_ALLOC 6

#define SPB_SHAPE_HALF_SPACE 0
#define SPB_SHAPE_SPHERE 1
#define SPB_SHAPE_CAPSULE 2
#define SPB_SHAPE_LEVELSET 3

#define SPB_CADENCE_INNER 0
#define SPB_CADENCE_FRAME 1
#define SPB_CADENCE_NEVER 2

typedef struct spb_factor spb_factor;
typedef struct spb_ctx spb_ctx;

/* Library identity and last error (thread local). */
int32_t spb_version(void);
const char *spb_last_error(void);
int32_t spb_device_count(int32_t *count);
/* The calling thread's current CUDA device (contexts default to it, or to
 * LOCAL_RANK under torchrun: one process per GPU). */
int32_t spb_get_device(int32_t *device);
/* Page-lock a caller-owned host range so spb_ctx_set_state / get_state move
 * it by DMA without staging (e.g. a SolverState.x reused every frame); the
 * caller unregisters it before freeing the memory. */
int32_t spb_host_register(void *ptr, int64_t bytes);
int32_t spb_host_unregister(void *ptr);

/* ----------------------------------------------------------- precompute */

/* Register the host BLAS/LAPACK (Fortran ABI, 32-bit ints) used by the
 * multifrontal precompute: dgemm, dsyrk, dtrsm, dpotrf, dtrtri. */
int32_t spb_set_host_blas(void *dgemm, void *dsyrk, void *dtrsm, void *dpotrf, void *dtrtri);

/* Partial factorization of the symmetric scalar block A (n x n, given as its
 * upper triangle in CSC: Ap[n+1], Ai, Ax) already permuted x1-first; the
 * leading n1 unknowns are eliminated and the dense Schur complement sigma0 of
 * the trailing n-n1 is retained (linalg.py:329-382).
 *   coords   (n1,3) rest coordinates of the x1 nodes for geometric nested
 *            dissection, or NULL (graph nested dissection)
 *   ordering 0 = identity, 1 = nested dissection (+ etree postorder)
 *   relax    1 = relaxed supernode amalgamation
 * On SPB_ERR_INDEFINITE, *bad_column is the failing x1 column in the
 * caller's (pre-fill) numbering (linalg.py:351-356). */
int32_t spb_factor_create(int64_t n, int64_t n1, const int64_t *Ap, const int64_t *Ai, const double *Ax,
                          const double *coords, int32_t ordering, int32_t relax, spb_factor **out,
                          int64_t *bad_column);
void spb_factor_destroy(spb_factor *f);
/* info[8] = {n1, n2, n_supernodes, nnz(L1), nnz(C), tree levels, panel values, panel rows} */
int32_t spb_factor_info(const spb_factor *f, int64_t *info);
int32_t spb_factor_fill_perm(const spb_factor *f, int64_t *out /* n1 */);
/* L1 in CSC (diagonal first per column), sized by info[3] */
int32_t spb_factor_export_l1(const spb_factor *f, int64_t *indptr, int64_t *indices, double *data);
/* coupling C = A21 L1^-T as CSR (n2 x n1), sized by info[4] */
int32_t spb_factor_export_coupling(const spb_factor *f, int64_t *indptr, int64_t *indices, double *data);
int32_t spb_factor_sigma0(const spb_factor *f, double *out /* n2*n2 row-major */);
int32_t spb_factor_supernodes(const spb_factor *f, int64_t *first, int64_t *rowptr, int64_t *rows,
                              int64_t *parent, int64_t *level);

/* Nested-dissection fill ordering of a symmetric pattern (upper CSC), with
 * optional rest coordinates; out[new] = old (linalg.fill_ordering). */
int32_t spb_fill_ordering(int64_t n, const int64_t *Ap, const int64_t *Ai, const double *coords, int64_t *out);
/* Symbolic Cholesky nnz (incl. diagonal) of a symmetric pattern (upper CSC). */
int32_t spb_symbolic_nnz(int64_t n, const int64_t *Ap, const int64_t *Ai, int64_t *nnz);

/* ---------------------------------------------------------- scene context */

typedef struct {
  int64_t num_nodes, num_elements;
  const int64_t *tets;       /* (ne,4) */
  const double *dm_inverse;  /* (ne,3,3) */
  const double *volume;      /* (ne,) */
  double mu, mu_prime, sigma_min, sigma_max;
  /* partition (partition.py:20-44) */
  int64_t n1, n2;
  const int64_t *perm;       /* (n,) perm[old] = new */
  int64_t num_alpha, num_beta;
  const int64_t *e_alpha, *e_beta;
  /* attachments, list order (solver.py:60-71) */
  int64_t num_attachments;
  const int64_t *att_nodes;  /* (na,) */
  const double *att_stiffness;
  /* collision proxies (collision.py:23-40) */
  int64_t num_proxies;
  const int64_t *proxy_elements; /* (P,) */
  const double *proxy_weights;   /* (P,4) */
  const double *proxy_stiffness; /* (P,) */
  /* prone-element stiffness K22_beta (solver.py:274-285), CSR m x m */
  const int64_t *k22_indptr, *k22_indices;
  const double *k22_data;
} spb_scene_desc;

/* Collider shape geometry (collision.py:57-180). params by kind:
 *   half_space: point[3], normal[3]      sphere: center[3], radius
 *   capsule: p0[3], p1[3], radius        levelset: origin[3], spacing (+dims, values) */
typedef struct {
  int32_t kind;
  double params[7];
  int64_t dims[3];
  const double *values; /* levelset samples, x fastest (collision.py:142-143) */
} spb_shape_desc;

/* One posed collider: registered shape id + rigid transform (collision.py:43-54). */
typedef struct {
  int32_t shape;
  double rotation[9]; /* row-major */
  double translation[3];
} spb_posed_collider;

typedef struct {
  int32_t outer_iters, inner_iters, cadence;
  int32_t use_graph;          /* capture/replay the frame as a CUDA graph */
  int32_t first_detection_done_unused;
  double early_exit_residual; /* < 0: disabled (solver.py:448-452) */
} spb_step_config;

/* FrameMetrics (solver.py:96-113); device-timed phases in ms. */
typedef struct {
  double t_local_ms, t_forward_ms, t_detect_ms, t_dense_ms, t_backward_ms, t_total_ms;
  double energy;
  int64_t active_proxies;
  double max_penetration, residual;
  int64_t info;               /* failing column on SPB_ERR_INDEFINITE */
  int64_t kernel_launches;    /* kernels this step launched */
  int64_t outer_passes;       /* outer passes run (< outer_iters after an early exit, solver.py:448-452) */
} spb_frame_metrics;

int32_t spb_ctx_create(const spb_scene_desc *scene, const spb_factor *factor, int32_t device, spb_ctx **out);
void spb_ctx_destroy(spb_ctx *ctx);
int32_t spb_ctx_add_shape(spb_ctx *ctx, const spb_shape_desc *shape, int32_t *shape_id);
/* Per-frame pose: attachment targets (na,3) in list order, posed colliders. */
int32_t spb_ctx_set_pose(spb_ctx *ctx, const double *att_targets, int32_t num_colliders,
                         const spb_posed_collider *colliders);
/* Upload a SolverState (R/Q may be NULL: identity / untouched). */
int32_t spb_ctx_set_state(spb_ctx *ctx, const double *x, const double *R, const double *Q, const uint8_t *active,
                          const double *target, const double *f_tilde2, const double *u2_accum);
/* One frame of solve_frame_schur on the context's state. */
int32_t spb_ctx_step(spb_ctx *ctx, const spb_step_config *cfg, spb_frame_metrics *metrics);
/* One whole frame in one call (what Simulation.step does per frame,
 * harness.py:592-596 -> solver.py:387-455): upload the pose (attachment
 * targets, posed colliders) and the state (x, active, target), run the frame
 * (CUDA graph), download x / active / target in place and f_tilde2 / u2_accum,
 * fill the metrics; one stream synchronisation. R/Q stay on the device
 * (spb_ctx_get_state pulls them). */
int32_t spb_ctx_frame(spb_ctx *ctx, const double *att_targets, int32_t num_colliders,
                      const spb_posed_collider *colliders, double *x, uint8_t *active, double *target,
                      const spb_step_config *cfg, double *f_tilde2, double *u2_accum, spb_frame_metrics *metrics);
/* spb_ctx_frame with the incoming active set / targets read from *_in and the
 * outgoing ones written to active / target (a caller that keeps the previous
 * frame's arrays, as SolverState does, passes them as *_in and fresh arrays
 * as outputs; no copy on the host). */
int32_t spb_ctx_frame_io(spb_ctx *ctx, const double *att_targets, int32_t num_colliders,
                         const spb_posed_collider *colliders, double *x, const uint8_t *active_in,
                         const double *target_in, uint8_t *active, double *target, const spb_step_config *cfg,
                         double *f_tilde2, double *u2_accum, spb_frame_metrics *metrics);
/* PCG baseline (reference solve_frame_pcg, solver.py:542-603; the paper's
 * §5.4 comparison solver), on the device. spb_ctx_set_operator hands over the
 * global matrix A (reference GlobalSystem.A: upper CSC in partition order,
 * n x n scalar); spb_ctx_frame_pcg then runs one frame like spb_ctx_frame:
 * per inner pass A_col = A + C22 (active set), b = all-element elastic +
 * attachment + collision forces, three Jacobi-PCG solves (one per coordinate,
 * |r|/|b| <= tol or max_iters) in one cooperative launch, x += dx.
 * pcg_iterations = worst per-pass count; metrics->residual = max_c
 * |A_col dx_c - b_c| / |b_c| of the last pass. p'Ap <= 0 returns
 * SPB_ERR_INDEFINITE with metrics->info = -1 (IndefiniteOperatorError). */
int32_t spb_ctx_set_operator(spb_ctx *ctx, int64_t n, const int64_t *indptr, const int64_t *indices,
                             const double *data);
int32_t spb_ctx_frame_pcg(spb_ctx *ctx, const double *att_targets, int32_t num_colliders,
                          const spb_posed_collider *colliders, double *x, uint8_t *active, double *target,
                          const spb_step_config *cfg, double tol, int64_t max_iters, spb_frame_metrics *metrics,
                          int64_t *pcg_iterations);
/* A batch of frames (BASELINE config 5 through the public API): the
 * arguments of spb_ctx_frame per context; every frame is in flight before
 * the host waits on any. metrics: n entries. Returns the first error. */
typedef struct {
  const double *att_targets;
  int32_t num_colliders;
  const spb_posed_collider *colliders;
  double *x;
  uint8_t *active;
  double *target;
  double *f_tilde2;
  double *u2_accum;
} spb_frame_io;
int32_t spb_frame_batch(spb_ctx **ctxs, int32_t n, const spb_frame_io *io, const spb_step_config *cfg,
                        spb_frame_metrics *metrics);
/* Download state; any pointer may be NULL to skip that field. */
int32_t spb_ctx_get_state(spb_ctx *ctx, double *x, double *R, double *Q, uint8_t *active, double *target,
                          double *f_tilde2, double *u2_accum);
/* Device-resident timing: run `frames` steps back to back with inputs
 * resident in HBM; reports the mean device ms per frame (CUDA events). */
int32_t spb_ctx_bench(spb_ctx *ctx, const spb_step_config *cfg, int32_t frames, double *ms_per_frame,
                      double *phase_ms /* [6]: local, forward, inner-detect, dense, backward, metrics */);
/* Diagnostics: per-task timestamps of one tile-Cholesky launch (see context.cu). */
int32_t spb_ctx_trace_cholesky(spb_ctx *ctx, uint64_t *out, int32_t *tasks_out, int32_t *ntasks);
/* Which factorization the context runs: 1 = trailing updates on the INT8
 * tensor cores (emulated FP64, k_cholesky_oz), 0 = FP64 DMMA (k_cholesky_tiles;
 * SPB_CHOL_INT8=0 at context creation). */
int32_t spb_ctx_cholesky_kind(spb_ctx *ctx, int32_t *kind);
/* Cholesky-only timing on the context's current H (tile kernel), ms per launch. */
int32_t spb_ctx_bench_cholesky(spb_ctx *ctx, int32_t reps, double *ms);
/* Diagnostics: per-block timestamps of one dense backward solve (5 per block). */
int32_t spb_ctx_trace_dense_backward(spb_ctx *ctx, uint64_t *out, int32_t *nblocks);
/* Graph-replay mean time of one piece of the frame on the current buffers:
 * 0 tile Cholesky, 1 dense backward solve, 2 sigma0 mat-vec, 3 sparse forward
 * sweep, 4 sparse backward sweep (bench.py rooflines). */
int32_t spb_ctx_bench_kernel(spb_ctx *ctx, int32_t which, int32_t reps, double *ms);
/* Batch throughput (BASELINE config 5): n contexts (e.g. scenes sharing one
 * factor) stepped concurrently, one stream each; mean device ms per round of
 * one frame of every context. */
int32_t spb_bench_batch(spb_ctx **ctxs, int32_t n, const spb_step_config *cfg, int32_t rounds,
                        double *ms_per_round);
/* Hint: n contexts step concurrently on this device (batch of scenes). The
 * tile Cholesky then takes about 1/n of the SMs, so the scenes' chain-bound
 * factorizations overlap; n = 1 restores the single-scene grid. spb_bench_batch
 * applies its own n. Results are bitwise independent of the hint. */
int32_t spb_ctx_set_concurrency(spb_ctx *ctx, int32_t n);

/* ------------------------------------------------------- one-shot ops */
int32_t spb_op_deformation_gradients(int64_t ne, const int64_t *tets, const double *dm_inverse, int64_t n,
                                     const double *x, int64_t k, const int64_t *elements, double *F);
/* signed SVD / polar / clamp of k 3x3 matrices; U,S,V,R,Q may be NULL */
int32_t spb_op_svd(int64_t k, const double *F, double *U, double *S, double *V, double *R, double *Q,
                   double sigma_min, double sigma_max);
int32_t spb_op_elastic(int64_t ne, const int64_t *tets, const double *dm_inverse, const double *volume,
                       int64_t n, const double *x, const double *R, const double *Q, double mu, double mu_prime,
                       int64_t k, const int64_t *elements, double *forces /* (n,3) or NULL */,
                       double *energy /* or NULL */);
int32_t spb_op_detect(int64_t n, const double *x, const int64_t *tets, int64_t P, const int64_t *proxy_elements,
                      const double *proxy_weights, int32_t num_shapes, const spb_shape_desc *shapes,
                      const spb_posed_collider *colliders, uint8_t *active, double *target, double *depth);
/* collision.scatter_proxies (reference collision.py:255-300) on the device,
 * the proxies of every surface triangle (ns x 3) whose three
 * vertices have node_mask set, per_element each at the given barycentric
 * points (per_element x 3), owned by the first tet (element order) with that
 * face; out_elem[ns * per_element], out_weights[ns * per_element * 4];
 * *count = proxies written (surface-triangle order, then point order).
 * SPB_ERR_ARG: node ids >= 2^21 or a selected triangle that is no tet's face. */
int32_t spb_scatter_proxies(const int64_t *tets, int64_t ne, int64_t n, const int64_t *surface_tris, int64_t ns,
                            const uint8_t *node_mask, int32_t per_element, const double *bary, int64_t *out_elem,
                            double *out_weights, int64_t *count);
/* dense SPD factor (lower, in place on a row-major m x m copy) and solve with nrhs columns */
int32_t spb_op_dense_factor(int64_t m, const double *h, double *chol, int64_t *info);
int32_t spb_op_dense_solve(int64_t m, const double *chol, int64_t nrhs, const double *g, double *x);
/* three-step solve pieces on a factor (linalg.py:385-414), nrhs columns (<= 3 per sweep) */
int32_t spb_op_forward_sub(const spb_factor *f, int64_t nrhs, const double *b1, const double *b2, double *y1,
                           double *y2);
int32_t spb_op_backward_sub(const spb_factor *f, int64_t nrhs, const double *y1, const double *x2, double *x1);

/* ------------------------------------- standalone dense Cholesky (config 4)
 * Replaces linalg.dense_factor (linalg.py:432-440: scipy.linalg.cholesky,
 * LAPACK dpotrf, lower) for one m x m SPD matrix held on the device as 64x64
 * tiles, factored by the frame solver's persistent tile kernel.
 * nranks == 1: one GPU. nranks > 1, emulate == 0: tile-cyclic over nranks
 * processes (one per GPU, `rank` = this process): each rank keeps a full L
 * replica and pushes every tile it finishes into the peers' replicas over
 * NVLink (CUDA IPC); exchange handles with spb_dense_ipc_handle /
 * spb_dense_open_peers, then per factorization on every rank:
 *   spb_dense_reset -> barrier -> spb_dense_launch -> spb_dense_finish -> barrier
 * emulate == 1: all nranks replicas on this one GPU, factored by ONE launch
 * (tests of the multi-rank data path on a single GPU). info: dpotrf's first
 * failing column (1-based), SPB_ERR_INDEFINITE when > 0. */
typedef struct spb_dense spb_dense;
#define SPB_DENSE_IPC_BYTES 64
int32_t spb_dense_create(int64_t m, int32_t device, int32_t rank, int32_t nranks, int32_t emulate,
                         spb_dense **out);
void spb_dense_destroy(spb_dense *d);
/* the lower triangle of a row-major m x m matrix is read (then mirrored) */
int32_t spb_dense_set_matrix(spb_dense *d, const double *h);
/* K_rc = a exp(-|p_r - p_c| / ell) + b delta_rc on a ceil(sqrt(m))^2 grid, generated on the device */
int32_t spb_dense_synthetic(spb_dense *d, double a, double b, double ell);
int32_t spb_dense_get_matrix(spb_dense *d, double *h /* m x m row-major, symmetric */);
int32_t spb_dense_get_factor(spb_dense *d, int32_t replica, double *chol /* m x m row-major, lower */);
int32_t spb_dense_ipc_handle(spb_dense *d, uint8_t *out /* SPB_DENSE_IPC_BYTES */);
int32_t spb_dense_open_peers(spb_dense *d, const uint8_t *handles /* nranks * SPB_DENSE_IPC_BYTES, rank order */);
/* diagnostics: peer < 0 fills the own replica's first L tile (and 16 flag
 * words) with `value`; peer >= 0 reads the first L value and flag word of the
 * peer's IPC-mapped replica (peer slots in rank order, own rank skipped) */
int32_t spb_dense_debug_replica(spb_dense *d, int32_t peer, double value, double *out_value, int32_t *out_flag);
/* 1: one GPU, trailing updates on the INT8 tensor cores (emulated FP64,
 * k_cholesky_oz); 0: FP64 DMMA (tile-cyclic / emulated ranks, SPB_CHOL_INT8=0) */
int32_t spb_dense_cholesky_kind(spb_dense *d, int32_t *kind);
int32_t spb_dense_set_cholesky_kind(spb_dense *d, int32_t kind);
int32_t spb_dense_reset(spb_dense *d);
int32_t spb_dense_launch(spb_dense *d);
int32_t spb_dense_finish(spb_dense *d, double *ms, int64_t *info);
/* single-process convenience: reps x (reset, launch, finish); mean ms per factorization */
int32_t spb_dense_factor(spb_dense *d, int32_t reps, double *ms, int64_t *info);
/* out2 = { ||A v - L (L^T v)||_2, ||A v||_2 } on the device (full-size check) */
int32_t spb_dense_residual(spb_dense *d, int32_t replica, const double *v, double *out2);
/* host only: the (i, j) tile tasks rank `rank` of nranks runs, in claim order;
 * ij == NULL returns the count; else *count is the capacity (pairs) */
int32_t spb_dense_rank_tasks(int64_t m, int32_t rank, int32_t nranks, int32_t *ij, int64_t *count);

#ifdef __cplusplus
}
#endif
#endif /* SCHURPD_B200_H */
