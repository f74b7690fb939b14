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
// elimination-tree height are independent. Each level runs as
//   (1) a gather kernel that assembles every struct row of the level once into
//       a contiguous buffer (forward: v = b + children's update entries;
//       backward: z = [y_s ; -x_below]), then
//   (2) GEMV kernels that stream the panels with coalesced loads and many
//       independent loads in flight (CTA tasks for wide supernodes, warp tasks
//       for nc <= 16).
// The x2 rows of the panels are the coupling C, so the forward sweep also yields
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
  int pos_off, npos;  // struct positions of the level (gather kernels)
  int max_nc;         // forward CTA tasks: columns staged in smem
  int rows;           // forward CTA task height (8..128)
  int bw_rows;        // backward tile height (128..4096)
};

struct DeviceFactor {
  int n1 = 0, n2 = 0, ns = 0, nlevels = 0;
  int64_t nrows_total = 0, urows = 0, nval = 0;
  SnDev* sn = nullptr;
  int* rows = nullptr;      // struct rows (factor positions)
  int* pos_owner = nullptr; // per struct position: factor index of an own column (top rows) or -1
  int* lvl_pos = nullptr;   // struct positions grouped by level
  double* M = nullptr;
  double* VZ = nullptr;     // per struct position x 3: assembled v (forward) / z (backward)
  int* asm_ptr = nullptr;
  int* asm_src = nullptr;
  int* x2_ptr = nullptr;
  int* x2_src = nullptr;
  int2* fw_cta = nullptr;   // (s, row0)
  int2* fw_warp = nullptr;  // (s, row0)
  int4* bw_tiles = nullptr;   // (s, c0, r0, partial slot)
  int4* bw_chunks = nullptr;  // (s, c0, first slot, ntiles)
  int* bw_tile_chunk = nullptr;  // chunk (global index) of every tile
  int* bw_chunk_cnt = nullptr;   // arrivals per chunk, zeroed per sweep
  double* P = nullptr;        // backward tile partials
  int* bw_warp = nullptr;     // s
  // bottom subtrees (levels < fuse): one CTA per group walks its supernodes
  // level by level (gather, GEMV) with block barriers instead of launches
  int fuse = 0, ngroups = 0;
  int* sub_pos = nullptr;     // struct positions, [group][level] ranges
  int* sub_pos_off = nullptr; // ngroups * fuse + 1
  int2* sub_fw = nullptr;     // forward warp tasks (s, r0)
  int* sub_fw_off = nullptr;
  int2* sub_bw = nullptr;     // backward warp tasks (s, c0), 8 columns each
  int* sub_bw_off = nullptr;
  // dataflow sweeps over the levels >= fuse (one persistent launch each)
  int flow = 0, nft = 0, nbt = 0, nbch = 0;
  int* parent = nullptr;       // supernode parent or -1
  int4* ftasks = nullptr;      // (kind 0 gather / 1 rows, s, r0, -)
  int* f_need = nullptr;       // row tasks of the children a supernode's gather waits for
  int4* btasks = nullptr;      // gather: (-(s+1), 0, 0, 0); tile: (s, c0, r0, slot)
  int* btask_chunk = nullptr;  // chunk of a tile task
  int4* bchunks = nullptr;     // (s, c0, first slot, ntiles)
  int* b_need = nullptr;       // column chunks of the parent a supernode's gather waits for
  int* flow_cnt = nullptr;     // counters, zeroed per sweep: [claim | per supernode x 2 | per chunk]
  int fw_grid = 0, bw_grid = 0;
  size_t fw_smem = 0;
  size_t p_slots = 0, nchunks = 0;  // sizes of the per-sweep workspace
  std::vector<LevelTasks> lv;
  std::vector<int> bwt_off, bwr_off, bww_off;  // backward tile / chunk / warp offsets per level
  ~DeviceFactor() {
    for (void* p : {(void*)sn, (void*)rows, (void*)pos_owner, (void*)lvl_pos, (void*)M, (void*)VZ,
                    (void*)asm_ptr, (void*)asm_src, (void*)x2_ptr, (void*)x2_src, (void*)fw_cta, (void*)fw_warp,
                    (void*)bw_tiles, (void*)bw_chunks, (void*)P, (void*)bw_warp, (void*)sub_pos,
                    (void*)sub_pos_off, (void*)sub_fw, (void*)sub_fw_off, (void*)sub_bw, (void*)sub_bw_off,
                    (void*)bw_tile_chunk, (void*)bw_chunk_cnt, (void*)parent, (void*)ftasks, (void*)f_need, (void*)btasks, (void*)btask_chunk,
                    (void*)bchunks, (void*)b_need, (void*)flow_cnt})
      if (p) cudaFree(p);
  }
};

size_t device_factor_ubuf(const DeviceFactor& df) { return (size_t)df.urows; }
int device_factor_levels(const DeviceFactor& df) { return df.nlevels; }

constexpr int FW_ROWS = 32;     // rows per forward CTA task (16 column groups x 32 rows)
constexpr int FW_THREADS = 512;
constexpr int FW_WARPS = FW_THREADS / 32;
constexpr int BT_ROWS = 512;       // backward tile rows
constexpr int BT_COLS = 32;        // backward tile columns (8 warps x 4)
constexpr int BW_WARP_MAXNR = 128; // small supernodes with longer columns take the tile path
constexpr int FW_WROWS = 32;    // rows per forward warp task
constexpr int WARP_NC = 16;     // supernodes with nc <= this use warp tasks
constexpr int CH_FW = 4096;     // forward column chunk staged in smem

// ------------------------------------------------------------- gathers
// forward: V[p] = b[own column] (top rows) + sum of the children's update
// entries landing on struct position p, in fixed child order.
__global__ void k_fw_gather(const int* __restrict__ lvl_pos, int npos, const int* __restrict__ owner,
                            const int* __restrict__ ap, const int* __restrict__ as, const double* __restrict__ U,
                            const double* __restrict__ b, double* __restrict__ V) {
  pdl_trigger();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= npos) return;
  const int p = lvl_pos[t];
  const int o = owner[p];
  const int k0 = ap[p], k1 = ap[p + 1];
  pdl_wait();  // U from the previous level
  double v0 = 0.0, v1 = 0.0, v2 = 0.0;
  if (o >= 0) {
    v0 = b[3 * (int64_t)o + 0];
    v1 = b[3 * (int64_t)o + 1];
    v2 = b[3 * (int64_t)o + 2];
  }
  for (int k = k0; k < k1; ++k) {
    const double* u = U + 3 * (int64_t)as[k];
    v0 += u[0];
    v1 += u[1];
    v2 += u[2];
  }
  V[3 * (int64_t)p + 0] = v0;
  V[3 * (int64_t)p + 1] = v1;
  V[3 * (int64_t)p + 2] = v2;
}

// backward: Z[p] = y[own column] for top rows, -x[row] below (x2 rows hold u2_accum)
__global__ void k_bw_gather(const int* __restrict__ lvl_pos, int npos, const int* __restrict__ owner,
                            const int* __restrict__ rows, const double* __restrict__ y,
                            const double* __restrict__ XF, double* __restrict__ Z) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= npos) return;
  const int p = lvl_pos[t];
  const int o = owner[p];
  double z0, z1, z2;
  if (o >= 0) {
    z0 = y[3 * (int64_t)o + 0];
    z1 = y[3 * (int64_t)o + 1];
    z2 = y[3 * (int64_t)o + 2];
  } else {
    const double* x = XF + 3 * (int64_t)rows[p];
    z0 = -x[0];
    z1 = -x[1];
    z2 = -x[2];
  }
  Z[3 * (int64_t)p + 0] = z0;
  Z[3 * (int64_t)p + 1] = z1;
  Z[3 * (int64_t)p + 2] = z2;
}

// -------------------------------------------------------------- forward
// CTA task (s, r0): rows r0..r0+31 of M_s; warp w walks columns w, w+8, ...
// (8 independent loads in flight per lane); partials summed in fixed order.
// Warp task (s, r0): one lane per row, the <= 16 inputs broadcast by shuffles.
__global__ void __launch_bounds__(FW_THREADS) k_forward_level(const SnDev* __restrict__ sn, const double* __restrict__ M,
                                                       const double* __restrict__ V,
                                                       const int2* __restrict__ cta_tasks, int ncta,
                                                       const int2* __restrict__ warp_tasks, int nwarp, int rows,
                                                       double* __restrict__ y, double* __restrict__ U) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if ((int)blockIdx.x < ncta) {
    // task (s, r0): rows r0..r0+R-1 of M_s; lane = row + R * column group, the
    // 16 * (32/R) column groups stride the columns (many loads in flight),
    // partials summed in fixed group order
    const int2 tk = cta_tasks[blockIdx.x];
    const SnDev S = sn[tk.x];
    const int R = rows, ngrp = 32 / rows;
    const int rl = lane % R, cg = lane / R;
    const int r = tk.y + rl;
    const bool valid = r < S.nr;
    const int cmax = (tk.y < S.nc) ? min(S.nc, tk.y + R) : S.nc;
    const double* Vs = V + 3 * (int64_t)S.rowoff;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    const double* Mp = M + S.valoff + (valid ? r : 0);
    const int stride = FW_WARPS * ngrp;
    for (int c0 = 0; c0 < cmax; c0 += CH_FW) {
      const int c1 = min(cmax, c0 + CH_FW);
      __syncthreads();
      for (int q = threadIdx.x; q < 3 * (c1 - c0); q += blockDim.x) sm[q] = Vs[3 * c0 + q];
      __syncthreads();
      if (valid) {
        int c = c0 + warp * ngrp + cg;
#pragma unroll 16
        for (; c < c1; c += stride) {
          const double mv = Mp[(int64_t)c * S.nr];
          const double* v = sm + 3 * (c - c0);
          a0 += mv * v[0];
          a1 += mv * v[1];
          a2 += mv * v[2];
        }
      }
    }
    __syncthreads();
    double* red = sm;  // [FW_WARPS * ngrp][R][3]
    const int grp = warp * ngrp + cg;
    red[(grp * R + rl) * 3 + 0] = a0;
    red[(grp * R + rl) * 3 + 1] = a1;
    red[(grp * R + rl) * 3 + 2] = a2;
    __syncthreads();
    if ((int)threadIdx.x < 3 * R) {
      const int rr0 = threadIdx.x / 3, q = threadIdx.x % 3;
      const int rr = tk.y + rr0;
      if (rr < S.nr) {
        double s = 0.0;
        for (int w = 0; w < stride; ++w) s += red[(w * R + rr0) * 3 + q];
        if (rr < S.nc) y[3 * (int64_t)(S.first + rr) + q] = s;
        else U[3 * (int64_t)(S.uoff + rr - S.nc) + q] = Vs[3 * rr + q] - s;
      }
    }
  } else {
    const int t = ((int)blockIdx.x - ncta) * FW_WARPS + warp;
    if (t >= nwarp) return;
    const int2 tk = warp_tasks[t];
    const SnDev S = sn[tk.x];
    const double* Vs = V + 3 * (int64_t)S.rowoff;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    if (lane < S.nc) {
      v0 = Vs[3 * lane + 0];
      v1 = Vs[3 * lane + 1];
      v2 = Vs[3 * lane + 2];
    }
    const int r = tk.y + lane;
    const bool valid = r < S.nr;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    const double* Mp = M + S.valoff + (valid ? r : 0);
#pragma unroll
    for (int c = 0; c < WARP_NC; ++c) {
      if (c < S.nc) {
        const double mv = valid ? Mp[(int64_t)c * S.nr] : 0.0;
        a0 += mv * __shfl_sync(0xffffffffu, v0, c);
        a1 += mv * __shfl_sync(0xffffffffu, v1, c);
        a2 += mv * __shfl_sync(0xffffffffu, v2, c);
      }
    }
    if (valid) {
      if (r < S.nc) {
        y[3 * (int64_t)(S.first + r) + 0] = a0;
        y[3 * (int64_t)(S.first + r) + 1] = a1;
        y[3 * (int64_t)(S.first + r) + 2] = a2;
      } else {
        const int64_t o = 3 * (int64_t)(S.uoff + r - S.nc);
        U[o + 0] = Vs[3 * r + 0] - a0;
        U[o + 1] = Vs[3 * r + 1] - a1;
        U[o + 2] = Vs[3 * r + 2] - a2;
      }
    }
  }
}

// f~2[k] = f2[k] + sum of root update entries on x2 row k (= f2 - C y1).
__global__ void k_forward_x2(int n1, int n2, const int* __restrict__ xp, const int* __restrict__ xs,
                             const double* __restrict__ U, const double* __restrict__ b, double* __restrict__ f2) {
  pdl_trigger();
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= 3 * n2) return;
  int row = k / 3, q = k % 3;
  pdl_wait();
  double v = b[3 * (int64_t)(n1 + row) + q];
  for (int t = xp[row]; t < xp[row + 1]; ++t) v += U[3 * (int64_t)xs[t] + q];
  f2[k] = v;
}

// ------------------------------------------------------------- backward
// Sum v[0..16) over the 32 lanes so that lane l ends with the total of entry
// l % 16 (all-to-all butterfly: 31 shuffles instead of 16 x 5).
__device__ __forceinline__ double warp_transpose_sum16(double (&v)[16], int lane) {
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
  return v[0];
}

// Backward 2D tiles: tile (s, c0, r0) covers rows [r0, r0+BT_ROWS) x columns
// [c0, c0+32) of M_s. The z chunk is staged in smem once per tile; warp w owns
// 4 columns, lanes walk rows (coalesced), 16 panel loads in flight per lane.
// Per-tile partial sums go to P[slot]; k_bw_reduce adds the row-chunk partials
// of every column in fixed order (deterministic, no atomics).
__global__ void __launch_bounds__(256) k_bw_tile(const SnDev* __restrict__ sn, const double* __restrict__ M,
                                                 const double* __restrict__ Z, const int4* __restrict__ tiles,
                                                 double* __restrict__ P) {
  __shared__ double zs[3 * BT_ROWS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int4 tk = tiles[blockIdx.x];  // (s, c0, r0, slot)
  const SnDev S = sn[tk.x];
  const int c0 = tk.y, r0 = tk.z;
  const int nrt = min(BT_ROWS, S.nr - r0);
  const double* Zs = Z + 3 * ((int64_t)S.rowoff + r0);
  for (int q = threadIdx.x; q < 3 * nrt; q += 256) zs[q] = Zs[q];
  __syncthreads();
  double acc[4][3];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = 0.0;
  const int cb = c0 + 4 * warp;
  const double* Mt = M + S.valoff + (int64_t)cb * S.nr + r0;
  const int nci = max(0, min(4, S.nc - cb));
  if (nci > 0) {
#pragma unroll 4
    for (int k = lane; k < nrt; k += 32) {
      const double z0 = zs[3 * k], z1 = zs[3 * k + 1], z2 = zs[3 * k + 2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i < nci) {
          const double m = Mt[(int64_t)i * S.nr + k];
          acc[i][0] += m * z0;
          acc[i][1] += m * z1;
          acc[i][2] += m * z2;
        }
      }
    }
  }
  double* out = P + (int64_t)tk.w * (BT_COLS * 3);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double v = warp_sum(acc[i][q]);
      if (lane == 0) out[(4 * warp + i) * 3 + q] = v;
    }
}

// x[first + c0 + cc] = sum over the chunk's row tiles (ascending r0) of P.
__global__ void k_bw_reduce(const SnDev* __restrict__ sn, const int4* __restrict__ chunks, int nchunks,
                            const double* __restrict__ P, double* __restrict__ XF) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nchunks * BT_COLS * 3) return;
  const int ch = t / (BT_COLS * 3), e = t % (BT_COLS * 3);
  const int cc = e / 3, q = e % 3;
  const int4 c = chunks[ch];  // (s, c0, first slot, ntiles)
  const SnDev S = sn[c.x];
  if (c.y + cc >= S.nc) return;
  double s = 0.0;
  for (int k = 0; k < c.w; ++k) s += P[((int64_t)(c.z + k) * BT_COLS + cc) * 3 + q];
  XF[3 * (int64_t)(S.first + c.y + cc) + q] = s;
}

// Warp task (s), nc <= 16: lanes over rows, one RHS at a time (low register
// footprint for occupancy), then the butterfly.
__global__ void __launch_bounds__(256) k_backward_warp(const SnDev* __restrict__ sn, const double* __restrict__ M,
                                                       const double* __restrict__ Z,
                                                       const int* __restrict__ warp_tasks, int nwarp,
                                                       double* __restrict__ XF) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = blockIdx.x * 8 + warp;
  if (t >= nwarp) return;
  const SnDev S = sn[warp_tasks[t]];
  const double* Zs = Z + 3 * (int64_t)S.rowoff;
  const double* Mc = M + S.valoff;
  double out[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    double acc[16];
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) acc[cc] = 0.0;
    for (int r = lane; r < S.nr; r += 32) {
      const double z = Zs[3 * r + q];
#pragma unroll
      for (int cc = 0; cc < 16; ++cc)
        if (cc < S.nc) acc[cc] += Mc[(int64_t)cc * S.nr + r] * z;
    }
    out[q] = warp_transpose_sum16(acc, lane);
  }
  if (lane < S.nc) {
    XF[3 * (int64_t)(S.first + lane) + 0] = out[0];
    XF[3 * (int64_t)(S.first + lane) + 1] = out[1];
    XF[3 * (int64_t)(S.first + lane) + 2] = out[2];
  }
}

// --------------------------------------------- fused level kernels (>= fuse)
// One launch per level and sweep: the gathers are folded into the GEMV tasks
// (each task assembles the inputs it reads) and the backward column-chunk
// reduction is done by the chunk's last tile (atomic arrival count; the sum
// itself runs in fixed row-tile order), so a level costs one launch instead of
// 2 (forward) or 3-4 (backward).
__device__ __forceinline__ double bw_gather_q(int p, int q, const int* __restrict__ owner,
                                              const int* __restrict__ rows, const double* __restrict__ y,
                                              const double* __restrict__ XF) {
  const int o = owner[p];
  return o >= 0 ? y[3 * (int64_t)o + q] : -XF[3 * (int64_t)rows[p] + q];
}

// CTA task (s, r0): rows r0 .. r0 + R - 1, R in {8, ..., 128}: lanes cover
// RL = min(R, 32) rows x 32/RL column subgroups, warps cover G = R/32 row
// groups x 16/G column groups; every thread strides its column group.
template <int FW_BATCH, int FW_MINB>
__global__ void __launch_bounds__(FW_THREADS, FW_MINB) k_fw_level(
    const SnDev* __restrict__ sn, const double* __restrict__ M, const int2* __restrict__ cta_tasks, int ncta,
    const int2* __restrict__ warp_tasks, int nwarp, int R, const double* __restrict__ V, double* __restrict__ y,
    double* __restrict__ U) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_trigger();
  if ((int)blockIdx.x < ncta) {
    const int2 tk = cta_tasks[blockIdx.x];
    const SnDev S = sn[tk.x];
    const double* Vs = V + 3 * (int64_t)S.rowoff;
    pdl_wait();  // V comes from this level's gather
    const int r0 = tk.y;
    const int RL = min(R, 32), G = max(1, R >> 5);
    const int rg = warp % G, row_in = 32 * rg + lane % RL;
    const int cgi = (warp / G) * (32 / RL) + lane / RL, ncg = (FW_WARPS / G) * (32 / RL);
    const int r = r0 + row_in;
    const bool valid = r < S.nr && row_in < R;
    const int cmax = (r0 < S.nc) ? min(S.nc, r0 + R) : S.nc;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    const double* Mp = M + S.valoff + (valid ? r : 0);
    for (int c0 = 0; c0 < cmax; c0 += CH_FW) {
      const int c1 = min(cmax, c0 + CH_FW);
      __syncthreads();
      for (int e = threadIdx.x; e < 3 * (c1 - c0); e += FW_THREADS) sm[e] = Vs[3 * c0 + e];
      __syncthreads();
      if (valid) {
        // predicated batches of FW_BATCH loads: every batch (the last,
        // partial one included) keeps FW_BATCH panel loads in flight; the
        // accumulation order (c ascending) is unchanged
        for (int cb = c0 + cgi; cb < c1; cb += FW_BATCH * ncg) {
          double mv[FW_BATCH];
#pragma unroll
          for (int u = 0; u < FW_BATCH; ++u) {
            const int c = cb + u * ncg;
            mv[u] = c < c1 ? Mp[(int64_t)c * S.nr] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < FW_BATCH; ++u) {
            const int c = cb + u * ncg;
            if (c < c1) {
              const double* v = sm + 3 * (c - c0);
              a0 += mv[u] * v[0];
              a1 += mv[u] * v[1];
              a2 += mv[u] * v[2];
            }
          }
        }
      }
    }
    __syncthreads();
    double* red = sm;  // [column group][row in task][3]
    if (row_in < R) {
      const int e0 = (cgi * R + row_in) * 3;
      red[e0 + 0] = a0;
      red[e0 + 1] = a1;
      red[e0 + 2] = a2;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 3 * R; e += FW_THREADS) {
      const int rl = e / 3, q = e % 3;
      const int rr = r0 + rl;
      if (rr >= S.nr) continue;
      double sum = 0.0;
      for (int g2 = 0; g2 < ncg; ++g2) sum += red[(g2 * R + rl) * 3 + q];
      if (rr < S.nc) y[3 * (int64_t)(S.first + rr) + q] = sum;
      else U[3 * (int64_t)(S.uoff + rr - S.nc) + q] = Vs[3 * rr + q] - sum;
    }
  } else {
    const int t = ((int)blockIdx.x - ncta) * FW_WARPS + warp;
    if (t >= nwarp) return;
    const int2 tk = warp_tasks[t];
    const SnDev S = sn[tk.x];
    const double* Vs = V + 3 * (int64_t)S.rowoff;
    pdl_wait();
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    if (lane < S.nc) {
      v0 = Vs[3 * lane + 0];
      v1 = Vs[3 * lane + 1];
      v2 = Vs[3 * lane + 2];
    }
    const int r = tk.y + lane;
    const bool valid = r < S.nr;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    const double* Mp = M + S.valoff + (valid ? r : 0);
#pragma unroll
    for (int c = 0; c < WARP_NC; ++c) {
      if (c < S.nc) {
        const double mv = valid ? Mp[(int64_t)c * S.nr] : 0.0;
        a0 += mv * __shfl_sync(0xffffffffu, v0, c);
        a1 += mv * __shfl_sync(0xffffffffu, v1, c);
        a2 += mv * __shfl_sync(0xffffffffu, v2, c);
      }
    }
    if (valid) {
      if (r < S.nc) {
        y[3 * (int64_t)(S.first + r) + 0] = a0;
        y[3 * (int64_t)(S.first + r) + 1] = a1;
        y[3 * (int64_t)(S.first + r) + 2] = a2;
      } else {
        const int64_t o = 3 * (int64_t)(S.uoff + r - S.nc);
        U[o + 0] = Vs[3 * r + 0] - a0;
        U[o + 1] = Vs[3 * r + 1] - a1;
        U[o + 2] = Vs[3 * r + 2] - a2;
      }
    }
  }
}

// k_fw_level variants: panel loads in flight per thread x resident CTAs per SM
// (SPB_FW_VARIANT for diagnostics; the level task heights follow the slots)
using FwLevelFn = void (*)(const SnDev*, const double*, const int2*, int, const int2*, int, int, const double*,
                           double*, double*);
static int fw_variant() {
  // swept on cfg3 (tools/slots_sweep.sh): 4 loads x 3 CTAs/SM, 4 x 148 slots
  // 277 us; 8 x 2: 282 us; 12 x 2: 290 us; unbatched remainder loop: 288 us
  static const int v = getenv("SPB_FW_VARIANT") ? atoi(getenv("SPB_FW_VARIANT")) : 0;
  return v;
}
static FwLevelFn fw_level_kernel() {
  switch (fw_variant()) {
    case 0: return k_fw_level<4, 3>;
    case 2: return k_fw_level<12, 2>;
    default: return k_fw_level<8, 2>;
  }
}

// Tile (s, c0, r0): rows [r0, r0 + RT) x columns [c0, c0 + 32) of M_s (RT per
// level, sized so the level's tiles fit the resident CTA slots); z gathered
// straight into shared memory.
__global__ void __launch_bounds__(256) k_bw_level(
    const SnDev* __restrict__ sn, const double* __restrict__ M, const int4* __restrict__ tiles, int RT,
    const int* __restrict__ tile_chunk, const int4* __restrict__ chunks, int* __restrict__ chunk_cnt,
    const int* __restrict__ owner, const int* __restrict__ rows, const double* __restrict__ y,
    double* __restrict__ P, double* __restrict__ XF) {
  extern __shared__ double zs[];  // 3 x RT
  __shared__ int last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_trigger();
  const int4 tk = tiles[blockIdx.x];  // (s, c0, r0, slot)
  const SnDev S = sn[tk.x];
  const int c0 = tk.y, r0 = tk.z;
  const int nrt = min(RT, S.nr - r0);
  pdl_wait();  // x of the ancestors (previous level) and the chunk counters
  for (int e = threadIdx.x; e < 3 * nrt; e += 256) zs[e] = bw_gather_q(S.rowoff + r0 + e / 3, e % 3, owner, rows, y, XF);
  __syncthreads();
  double acc[4][3];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = 0.0;
  const int cb = c0 + 4 * warp;
  const double* Mt = M + S.valoff + (int64_t)cb * S.nr + r0;
  const int nci = max(0, min(4, S.nc - cb));
  if (nci > 0) {
#pragma unroll 4
    for (int k = lane; k < nrt; k += 32) {
      const double z0 = zs[3 * k], z1 = zs[3 * k + 1], z2 = zs[3 * k + 2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i < nci) {
          const double m = Mt[(int64_t)i * S.nr + k];
          acc[i][0] += m * z0;
          acc[i][1] += m * z1;
          acc[i][2] += m * z2;
        }
      }
    }
  }
  double* out = P + (int64_t)tk.w * (BT_COLS * 3);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const double v = warp_sum(acc[i][q]);
      if (lane == 0) out[(4 * warp + i) * 3 + q] = v;
    }
  // the chunk's last tile sums the partials in row-tile order
  __threadfence();
  __syncthreads();
  const int ch = tile_chunk[blockIdx.x];
  const int4 C = chunks[ch];  // (s, c0, first slot, ntiles)
  if (threadIdx.x == 0) last = (atomicAdd(chunk_cnt + ch, 1) == C.w - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < BT_COLS * 3) {
    const int cc = threadIdx.x / 3, q = threadIdx.x % 3;
    if (C.y + cc < S.nc) {
      double sum = 0.0;
      for (int k = 0; k < C.w; ++k) sum += __ldcg(P + ((int64_t)(C.z + k) * BT_COLS + cc) * 3 + q);
      XF[3 * (int64_t)(S.first + C.y + cc) + q] = sum;
    }
  }
}

// warp task (s), nc <= 16 and nr <= BW_WARP_MAXNR: lanes over rows, one RHS at
// a time, butterfly (separate kernel: rare above the fused subtrees)
__global__ void __launch_bounds__(256) k_bw_level_warp(const SnDev* __restrict__ sn, const double* __restrict__ M,
                                                       const int* __restrict__ warp_tasks, int nwarp,
                                                       const int* __restrict__ owner, const int* __restrict__ rows,
                                                       const double* __restrict__ y, double* __restrict__ XF) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_trigger();
  const int t = blockIdx.x * 8 + warp;
  if (t >= nwarp) return;
  const SnDev S = sn[warp_tasks[t]];
  const double* Mc = M + S.valoff;
  pdl_wait();
  double out[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    double acc[16];
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) acc[cc] = 0.0;
    for (int r = lane; r < S.nr; r += 32) {
      const double z = bw_gather_q(S.rowoff + r, q, owner, rows, y, XF);
#pragma unroll
      for (int cc = 0; cc < 16; ++cc)
        if (cc < S.nc) acc[cc] += Mc[(int64_t)cc * S.nr + r] * z;
    }
    out[q] = warp_transpose_sum16(acc, lane);
  }
  if (lane < S.nc) {
    XF[3 * (int64_t)(S.first + lane) + 0] = out[0];
    XF[3 * (int64_t)(S.first + lane) + 1] = out[1];
    XF[3 * (int64_t)(S.first + lane) + 2] = out[2];
  }
}

// ------------------------------------------------- bottom-subtree kernels
// The lower elimination-tree levels hold thousands of small supernodes
// (cfg3: levels 0-6 = 5.5K supernodes, 105 MB of panels) whose per-level
// launches are latency-bound. Whole subtrees are grouped (balanced by panel
// bytes) and one CTA per group runs all those levels, with block barriers
// between the dependent steps; the children's updates and the ancestors' x are
// produced by the same CTA (or by the level kernels before/after the launch).
constexpr int SUB_THREADS = 512;
constexpr int SUB_WARPS = SUB_THREADS / 32;
constexpr int SUB_BWC = 8;  // backward warp task width (columns)

// One warp: rows r0..r0+31 of M_s times the assembled v (any nc), in column order.
__device__ __forceinline__ void fw_warp_rows(const SnDev& S, int r0, int lane, const double* __restrict__ M,
                                             const double* V, double* y, double* U) {
  const int r = r0 + lane;
  const bool valid = r < S.nr;
  const int cmax = (r0 < S.nc) ? min(S.nc, r0 + 32) : S.nc;  // inv(L_ss) is lower triangular
  const double* Vs = V + 3 * (int64_t)S.rowoff;
  const double* Mp = M + S.valoff + (valid ? r : 0);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  // 16 independent panel loads in flight per lane (latency-bound otherwise);
  // the chunk's 48 v entries come in with two coalesced loads and are
  // broadcast by shuffles (entry e = 3u + q sits in lane e % 32 of load e / 32)
  for (int c = 0; c < cmax; c += 16) {
    double mv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) mv[u] = (c + u < cmax) ? Mp[(int64_t)(c + u) * S.nr] : 0.0;
    const int nv = 3 * min(16, cmax - c);
    const double vlo = lane < nv ? Vs[3 * c + lane] : 0.0;
    const double vhi = lane + 32 < nv ? Vs[3 * c + 32 + lane] : 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const double v0 = (3 * u + 0 < 32) ? __shfl_sync(0xffffffffu, vlo, (3 * u + 0) & 31)
                                         : __shfl_sync(0xffffffffu, vhi, (3 * u + 0) & 31);
      const double v1 = (3 * u + 1 < 32) ? __shfl_sync(0xffffffffu, vlo, (3 * u + 1) & 31)
                                         : __shfl_sync(0xffffffffu, vhi, (3 * u + 1) & 31);
      const double v2 = (3 * u + 2 < 32) ? __shfl_sync(0xffffffffu, vlo, (3 * u + 2) & 31)
                                         : __shfl_sync(0xffffffffu, vhi, (3 * u + 2) & 31);
      if (c + u < cmax) {
        a0 += mv[u] * v0;
        a1 += mv[u] * v1;
        a2 += mv[u] * v2;
      }
    }
  }
  if (!valid) return;
  if (r < S.nc) {
    y[3 * (int64_t)(S.first + r) + 0] = a0;
    y[3 * (int64_t)(S.first + r) + 1] = a1;
    y[3 * (int64_t)(S.first + r) + 2] = a2;
  } else {
    const int64_t o = 3 * (int64_t)(S.uoff + r - S.nc);
    U[o + 0] = Vs[3 * r + 0] - a0;
    U[o + 1] = Vs[3 * r + 1] - a1;
    U[o + 2] = Vs[3 * r + 2] - a2;
  }
}

// lane l ends with the warp total of entry l % 8
__device__ __forceinline__ double warp_transpose_sum8(double (&v)[8], int lane) {
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], 16);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], 8);
#pragma unroll
  for (int off = 4; off >= 1; off >>= 1) {
    const bool upper = lane & off;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const double send = upper ? v[i] : v[i + off];
      const double keep = upper ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

__global__ void __launch_bounds__(SUB_THREADS) k_subtree_forward(
    const SnDev* __restrict__ sn, const double* __restrict__ M, const int* __restrict__ pos,
    const int* __restrict__ pos_off, const int2* __restrict__ tasks, const int* __restrict__ task_off, int fuse,
    const int* __restrict__ owner, const int* __restrict__ ap, const int* __restrict__ as,
    const double* __restrict__ b, double* V, double* y, double* U) {
  const int g = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_trigger();
  pdl_wait();
  for (int l = 0; l < fuse; ++l) {
    const int q0 = pos_off[g * fuse + l], q1 = pos_off[g * fuse + l + 1];
    for (int t = q0 + (int)threadIdx.x; t < q1; t += SUB_THREADS) {
      const int p = pos[t];
      const int o = owner[p];
      double v0 = 0.0, v1 = 0.0, v2 = 0.0;
      if (o >= 0) {
        v0 = b[3 * (int64_t)o + 0];
        v1 = b[3 * (int64_t)o + 1];
        v2 = b[3 * (int64_t)o + 2];
      }
      for (int k = ap[p]; k < ap[p + 1]; ++k) {
        const double* u = U + 3 * (int64_t)as[k];
        v0 += u[0];
        v1 += u[1];
        v2 += u[2];
      }
      V[3 * (int64_t)p + 0] = v0;
      V[3 * (int64_t)p + 1] = v1;
      V[3 * (int64_t)p + 2] = v2;
    }
    __syncthreads();
    const int t0 = task_off[g * fuse + l], t1 = task_off[g * fuse + l + 1];
    for (int t = t0 + warp; t < t1; t += SUB_WARPS) {
      const int2 tk = tasks[t];
      fw_warp_rows(sn[tk.x], tk.y, lane, M, V, y, U);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(SUB_THREADS) k_subtree_backward(
    const SnDev* __restrict__ sn, const double* __restrict__ M, const int* __restrict__ pos,
    const int* __restrict__ pos_off, const int2* __restrict__ tasks, const int* __restrict__ task_off, int fuse,
    const int* __restrict__ owner, const int* __restrict__ rows, const double* __restrict__ y, double* Z,
    double* XF) {
  const int g = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_trigger();
  pdl_wait();
  for (int l = fuse - 1; l >= 0; --l) {
    const int q0 = pos_off[g * fuse + l], q1 = pos_off[g * fuse + l + 1];
    for (int t = q0 + (int)threadIdx.x; t < q1; t += SUB_THREADS) {
      const int p = pos[t];
      const int o = owner[p];
      double z0, z1, z2;
      if (o >= 0) {
        z0 = y[3 * (int64_t)o + 0];
        z1 = y[3 * (int64_t)o + 1];
        z2 = y[3 * (int64_t)o + 2];
      } else {
        const double* x = XF + 3 * (int64_t)rows[p];
        z0 = -x[0];
        z1 = -x[1];
        z2 = -x[2];
      }
      Z[3 * (int64_t)p + 0] = z0;
      Z[3 * (int64_t)p + 1] = z1;
      Z[3 * (int64_t)p + 2] = z2;
    }
    __syncthreads();
    const int t0 = task_off[g * fuse + l], t1 = task_off[g * fuse + l + 1];
    for (int t = t0 + warp; t < t1; t += SUB_WARPS) {
      const int2 tk = tasks[t];  // (s, c0)
      const SnDev S = sn[tk.x];
      const int c0 = tk.y, ncc = min(SUB_BWC, S.nc - c0);
      const double* Zs = Z + 3 * (int64_t)S.rowoff;
      const double* Mc = M + S.valoff + (int64_t)c0 * S.nr;
      double acc[3][SUB_BWC];
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int cc = 0; cc < SUB_BWC; ++cc) acc[q][cc] = 0.0;
      // rows above c0 are zero in the inv(L_ss) block; two row steps per
      // iteration keep 16 panel loads in flight per lane
      for (int r = c0 + lane; r < S.nr; r += 64) {
        double z[2][3], mv[2][SUB_BWC];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int rr = r + 32 * h;
          const bool ok = rr < S.nr;
#pragma unroll
          for (int q = 0; q < 3; ++q) z[h][q] = ok ? Zs[3 * rr + q] : 0.0;
#pragma unroll
          for (int cc = 0; cc < SUB_BWC; ++cc) mv[h][cc] = (ok && cc < ncc) ? Mc[(int64_t)cc * S.nr + rr] : 0.0;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int cc = 0; cc < SUB_BWC; ++cc) {
            acc[0][cc] += mv[h][cc] * z[h][0];
            acc[1][cc] += mv[h][cc] * z[h][1];
            acc[2][cc] += mv[h][cc] * z[h][2];
          }
      }
      const double o0 = warp_transpose_sum8(acc[0], lane);
      const double o1 = warp_transpose_sum8(acc[1], lane);
      const double o2 = warp_transpose_sum8(acc[2], lane);
      if (lane < ncc) {
        XF[3 * (int64_t)(S.first + c0 + lane) + 0] = o0;
        XF[3 * (int64_t)(S.first + c0 + lane) + 1] = o1;
        XF[3 * (int64_t)(S.first + c0 + lane) + 2] = o2;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------- dataflow sweeps
// The upper levels (>= fuse) as ONE persistent launch per sweep: tasks are
// claimed from a global counter in topological order (forward: leaves up;
// backward: root down), and each waits only for the tasks it reads, through
// per-supernode counters (release/acquire), instead of a kernel boundary per
// level. Every claimed task waits only on earlier-claimed tasks, so a
// persistent grid always makes progress. Summation orders are fixed (no float
// atomics): bitwise-deterministic.
constexpr int FL_FW_THREADS = 512;
constexpr int FL_BW_THREADS = 256;
constexpr int FL_ROWS = 32;

__device__ __forceinline__ void flow_wait(const int* c, int need) {
  if (threadIdx.x == 0 && need > 0) {
    SpinGuard g;
    while (ld_relaxed(c) < need) g.tick();
    fence_acq_rel_gpu();
  }
  __syncthreads();
}

__device__ __forceinline__ int flow_claim(int* counter, int* slot) {
  __syncthreads();  // the previous task is finished with the slot
  if (threadIdx.x == 0) *slot = atomicAdd(counter, 1);
  __syncthreads();
  return *slot;
}

__global__ void __launch_bounds__(FL_FW_THREADS) k_forward_flow(
    const SnDev* __restrict__ sn, const double* __restrict__ M, const int4* __restrict__ tasks, int ntasks,
    const int* __restrict__ need, const int* __restrict__ parent, int* cnt /* [claim | done(ns) | gathered(ns)] */,
    int ns, const int* __restrict__ owner, const int* __restrict__ ap, const int* __restrict__ as,
    const double* __restrict__ b, double* V, double* y, double* U) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int slot;
  int* done = cnt + 1;
  int* gathered = cnt + 1 + ns;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    const int t = flow_claim(cnt, &slot);
    if (t >= ntasks) break;
    const int4 tk = tasks[t];
    const SnDev S = sn[tk.y];
    if (tk.x == 0) {
      // gather: V = b (own columns) + children's update entries, fixed order
      flow_wait(done + tk.y, need[tk.y]);
      for (int k = threadIdx.x; k < S.nr; k += FL_FW_THREADS) {
        const int p = S.rowoff + k;
        const int o = owner[p];
        double v0 = 0.0, v1 = 0.0, v2 = 0.0;
        if (o >= 0) {
          v0 = b[3 * (int64_t)o + 0];
          v1 = b[3 * (int64_t)o + 1];
          v2 = b[3 * (int64_t)o + 2];
        }
        for (int q = ap[p]; q < ap[p + 1]; ++q) {
          // written by other CTAs of this launch: bypass L1 (lines may be stale)
          const double* u = U + 3 * (int64_t)as[q];
          v0 += __ldcg(u + 0);
          v1 += __ldcg(u + 1);
          v2 += __ldcg(u + 2);
        }
        V[3 * (int64_t)p + 0] = v0;
        V[3 * (int64_t)p + 1] = v1;
        V[3 * (int64_t)p + 2] = v2;
      }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) st_release(gathered + tk.y, 1);
      continue;
    }
    // rows r0..r0+31 of M_s (16 warps stride the columns), like k_forward_level
    flow_wait(gathered + tk.y, 1);
    const int r0 = tk.z;
    const int r = r0 + lane;
    const bool valid = r < S.nr;
    const int cmax = (r0 < S.nc) ? min(S.nc, r0 + FL_ROWS) : S.nc;
    const double* Vs = V + 3 * (int64_t)S.rowoff;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    const double* Mp = M + S.valoff + (valid ? r : 0);
    for (int c0 = 0; c0 < cmax; c0 += CH_FW) {
      const int c1 = min(cmax, c0 + CH_FW);
      __syncthreads();
      for (int q = threadIdx.x; q < 3 * (c1 - c0); q += FL_FW_THREADS) sm[q] = __ldcg(Vs + 3 * c0 + q);
      __syncthreads();
      if (valid) {
        int c = c0 + warp;
#pragma unroll 16
        for (; c < c1; c += FL_FW_THREADS / 32) {
          const double mv = Mp[(int64_t)c * S.nr];
          const double* v = sm + 3 * (c - c0);
          a0 += mv * v[0];
          a1 += mv * v[1];
          a2 += mv * v[2];
        }
      }
    }
    __syncthreads();
    double* red = sm;  // [16 warps][32][3]
    red[(warp * 32 + lane) * 3 + 0] = a0;
    red[(warp * 32 + lane) * 3 + 1] = a1;
    red[(warp * 32 + lane) * 3 + 2] = a2;
    __syncthreads();
    if (threadIdx.x < 96) {
      const int rl = threadIdx.x / 3, q = threadIdx.x % 3;
      const int rr = r0 + rl;
      if (rr < S.nr) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < FL_FW_THREADS / 32; ++w) s += red[(w * 32 + rl) * 3 + q];
        if (rr < S.nc) y[3 * (int64_t)(S.first + rr) + q] = s;
        else U[3 * (int64_t)(S.uoff + rr - S.nc) + q] = __ldcg(Vs + 3 * rr + q) - s;
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0 && parent[tk.y] >= 0) atomicAdd(done + parent[tk.y], 1);
  }
}

__global__ void __launch_bounds__(FL_BW_THREADS) k_backward_flow(
    const SnDev* __restrict__ sn, const double* __restrict__ M, const int4* __restrict__ tasks,
    const int* __restrict__ task_chunk, int ntasks, const int4* __restrict__ chunks, const int* __restrict__ need,
    const int* __restrict__ parent, int* cnt /* [claim | done(ns) | gathered(ns) | chunk(nch)] */, int ns,
    const int* __restrict__ owner, const int* __restrict__ rows, const double* __restrict__ y, double* Z, double* P,
    double* XF) {
  __shared__ double zs[3 * BT_ROWS];
  __shared__ int slot, last;
  int* done = cnt + 1;
  int* gathered = cnt + 1 + ns;
  int* chunk_cnt = cnt + 1 + 2 * ns;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    const int t = flow_claim(cnt, &slot);
    if (t >= ntasks) break;
    const int4 tk = tasks[t];
    if (tk.x < 0) {
      // gather z_s = [y own ; -x below]; the below rows are the ancestors' x
      const int s = -tk.x - 1;
      const SnDev S = sn[s];
      if (parent[s] >= 0) flow_wait(done + parent[s], need[s]);
      for (int k = threadIdx.x; k < S.nr; k += FL_BW_THREADS) {
        const int p = S.rowoff + k;
        const int o = owner[p];
        double z0, z1, z2;
        if (o >= 0) {
          z0 = y[3 * (int64_t)o + 0];
          z1 = y[3 * (int64_t)o + 1];
          z2 = y[3 * (int64_t)o + 2];
        } else {
          const double* x = XF + 3 * (int64_t)rows[p];
          z0 = -__ldcg(x + 0);
          z1 = -__ldcg(x + 1);
          z2 = -__ldcg(x + 2);
        }
        Z[3 * (int64_t)p + 0] = z0;
        Z[3 * (int64_t)p + 1] = z1;
        Z[3 * (int64_t)p + 2] = z2;
      }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) st_release(gathered + s, 1);
      continue;
    }
    // tile (s, c0, r0): partial x over rows [r0, r0+512) x columns [c0, c0+32)
    const SnDev S = sn[tk.x];
    flow_wait(gathered + tk.x, 1);
    const int c0 = tk.y, r0 = tk.z;
    const int nrt = min(BT_ROWS, S.nr - r0);
    const double* Zs = Z + 3 * ((int64_t)S.rowoff + r0);
    for (int q = threadIdx.x; q < 3 * nrt; q += FL_BW_THREADS) zs[q] = __ldcg(Zs + q);
    __syncthreads();
    double acc[4][3];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = 0.0;
    const int cb = c0 + 4 * warp;
    const double* Mt = M + S.valoff + (int64_t)cb * S.nr + r0;
    const int nci = max(0, min(4, S.nc - cb));
    if (nci > 0) {
#pragma unroll 4
      for (int k = lane; k < nrt; k += 32) {
        const double z0 = zs[3 * k], z1 = zs[3 * k + 1], z2 = zs[3 * k + 2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i < nci) {
            const double m = Mt[(int64_t)i * S.nr + k];
            acc[i][0] += m * z0;
            acc[i][1] += m * z1;
            acc[i][2] += m * z2;
          }
        }
      }
    }
    double* out = P + (int64_t)tk.w * (BT_COLS * 3);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const double v = warp_sum(acc[i][q]);
        if (lane == 0) out[(4 * warp + i) * 3 + q] = v;
      }
    // the last tile of the column chunk sums the partials in row-tile order
    __threadfence();
    __syncthreads();
    const int ch = task_chunk[t];
    const int4 C = chunks[ch];
    if (threadIdx.x == 0) last = (atomicAdd(chunk_cnt + ch, 1) == C.w - 1);
    __syncthreads();
    if (!last) continue;
    __threadfence();
    if (threadIdx.x < BT_COLS * 3) {
      const int cc = threadIdx.x / 3, q = threadIdx.x % 3;
      if (C.y + cc < S.nc) {
        double s = 0.0;
        for (int k = 0; k < C.w; ++k) s += __ldcg(P + ((int64_t)(C.z + k) * BT_COLS + cc) * 3 + q);
        XF[3 * (int64_t)(S.first + C.y + cc) + q] = s;
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(done + tk.x, 1);
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
  int cur = 0;
  SPB_CUDA(cudaGetDevice(&cur));
  if (cur < 0 || cur >= Factor::kMaxDevices) { set_error("device id out of range"); return SPB_ERR_ARG; }
  if (f.devs[cur]) return SPB_OK;
  auto* d = new DeviceFactor();
  const int64_t ns = f.nsuper;
  d->n1 = (int)f.n1;
  d->n2 = (int)f.n2;
  d->ns = (int)ns;
  d->nlevels = (int)f.nlevels;
  d->nrows_total = f.sn_rowptr.empty() ? 0 : f.sn_rowptr[ns];
  d->nval = f.sn_valptr.empty() ? 0 : f.sn_valptr[ns];
  if (d->nrows_total >= (int64_t)1 << 31) {
    delete d;
    set_error("factor too large (row index > 2^31)");
    return SPB_ERR_SETUP;
  }
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
  std::vector<int> rows(d->nrows_total), owner(d->nrows_total, -1);
  for (int64_t k = 0; k < d->nrows_total; ++k) rows[k] = (int)f.sn_rows[k];
  for (int64_t s = 0; s < ns; ++s)
    for (int k = 0; k < sn[s].nc; ++k) owner[sn[s].rowoff + k] = sn[s].first + k;
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
    if (x2) xcnt[p + 1]++;
    else cnt[p + 1]++;
  });
  for (int64_t k = 0; k < d->nrows_total; ++k) cnt[k + 1] += cnt[k];
  for (int64_t k = 0; k < f.n2; ++k) xcnt[k + 1] += xcnt[k];
  std::vector<int> asrc(cnt[d->nrows_total]), xsrc(xcnt[f.n2]);
  {
    std::vector<int> fill(cnt.begin(), cnt.end() - 1), xfill(xcnt.begin(), xcnt.end() - 1);
    for_each_map([&](bool x2, int64_t p, int src) {
      if (x2) xsrc[xfill[p]++] = src;
      else asrc[fill[p]++] = src;
    });
  }
  // per level: forward tasks, backward tasks, struct positions
  std::vector<std::vector<int64_t>> bylevel(f.nlevels);
  for (int64_t s = 0; s < ns; ++s) bylevel[f.sn_level[s]].push_back(s);
  std::vector<int2> fwc, fww;
  std::vector<int4> bwt, bwr;
  std::vector<int> btc;
  std::vector<int> bww, lpos;
  lpos.reserve(d->nrows_total);
  d->lv.resize(f.nlevels);
  d->bwt_off.assign(f.nlevels + 1, 0);
  d->bwr_off.assign(f.nlevels + 1, 0);
  d->bww_off.assign(f.nlevels + 1, 0);
  for (int64_t l = 0; l < f.nlevels; ++l) {
    LevelTasks& T = d->lv[l];
    T.cta_off = (int)fwc.size();
    T.warp_off = (int)fww.size();
    T.pos_off = (int)lpos.size();
    T.max_nc = 0;
    d->bwt_off[l] = (int)bwt.size();
    d->bwr_off[l] = (int)bwr.size();
    d->bww_off[l] = (int)bww.size();
    {
      // forward CTA task height: the largest of 32/16/8 rows giving >= 4 waves
      int64_t n32 = 0;
      for (int64_t s : bylevel[l])
        if (sn[s].nc > WARP_NC) n32 += (sn[s].nr + 31) / 32;
      // task height R: the smallest of 8..128 whose task count still fits
      // the resident CTA slots (~4 x 148): a task streams at a roughly fixed
      // rate, so the level is fastest when all of it runs concurrently in as
      // many tasks as possible (wide top levels: short tasks; levels of many
      // small supernodes: tall tasks, one wave)
      static const int slots = (getenv("SPB_FW_SLOTS") ? atoi(getenv("SPB_FW_SLOTS")) : 4) * NUM_SMS_B200;
      (void)n32;
      T.rows = 128;
      for (int R = 8; R <= 128; R *= 2) {
        int64_t nt = 0;
        for (int64_t s : bylevel[l])
          if (sn[s].nc > WARP_NC) nt += (sn[s].nr + R - 1) / R;
        if (nt <= slots) {
          T.rows = R;
          break;
        }
      }
      for (int64_t s : bylevel[l]) {
        const SnDev& S = sn[s];
        if (S.nc <= WARP_NC) continue;
        for (int r0 = 0; r0 < S.nr; r0 += T.rows) fwc.push_back(make_int2((int)s, r0));
        T.max_nc = std::max(T.max_nc, S.nc);
      }
    }
    {
      // backward tile height: the smallest of 128..4096 whose tile count fits
      // the resident slots (~4 x 148 CTAs of 256 threads; swept on cfg3)
      static const int bslots = (getenv("SPB_BW_SLOTS") ? atoi(getenv("SPB_BW_SLOTS")) : 4) * NUM_SMS_B200;
      T.bw_rows = 4096;
      for (int RT = 128; RT <= 4096; RT *= 2) {
        int64_t nt = 0;
        for (int64_t s : bylevel[l]) {
          const SnDev& S = sn[s];
          if (S.nc <= WARP_NC && S.nr <= BW_WARP_MAXNR) continue;
          for (int c0 = 0; c0 < S.nc; c0 += BT_COLS)
            for (int r0 = 0; r0 < S.nr; r0 += RT)
              if (r0 + RT > c0) ++nt;
        }
        if (nt <= bslots) {
          T.bw_rows = RT;
          break;
        }
      }
    }
    for (int64_t s : bylevel[l]) {
      const SnDev& S = sn[s];
      const bool small = S.nc <= WARP_NC;
      if (small) {
        for (int r0 = 0; r0 < S.nr; r0 += FW_WROWS) fww.push_back(make_int2((int)s, r0));
      }
      if (small && S.nr <= BW_WARP_MAXNR) {
        bww.push_back((int)s);
      } else {
        const int RT = l < d->fuse ? BT_ROWS : T.bw_rows;
        for (int c0 = 0; c0 < S.nc; c0 += BT_COLS) {
          const int slot0 = (int)bwt.size();
          for (int r0 = 0; r0 < S.nr; r0 += RT) {
            if (r0 + RT <= c0) continue;  // entirely above the diagonal of inv(L_ss): zero
            bwt.push_back(make_int4((int)s, c0, r0, (int)bwt.size()));
          }
          for (int k = slot0; k < (int)bwt.size(); ++k) btc.push_back((int)bwr.size());
          bwr.push_back(make_int4((int)s, c0, slot0, (int)bwt.size() - slot0));
        }
      }
      for (int k = 0; k < S.nr; ++k) lpos.push_back(S.rowoff + k);
    }
    T.ncta = (int)fwc.size() - T.cta_off;
    T.nwarp = (int)fww.size() - T.warp_off;
    T.npos = (int)lpos.size() - T.pos_off;
  }
  d->bwt_off[f.nlevels] = (int)bwt.size();
  d->bwr_off[f.nlevels] = (int)bwr.size();
  d->bww_off[f.nlevels] = (int)bww.size();
  // ---- bottom subtrees: choose the fuse height f by a small cost model
  // (slowest group's panel bytes at ~25 GB/s effective per SM + ~20 us per remaining
  // level launch pair + ~8 us per fused level), group whole subtrees (LPT on
  // bytes, 148 groups)
  {
    std::vector<std::vector<int64_t>> kids(ns);
    for (int64_t s = 0; s < ns; ++s)
      if (f.sn_parent[s] >= 0) kids[f.sn_parent[s]].push_back(s);
    auto plan = [&](int fz, std::vector<int64_t>& roots, std::vector<std::vector<int64_t>>& members,
                    std::vector<int>& group_of_root, int& G) -> double {
      roots.clear();
      for (int64_t s = 0; s < ns; ++s)
        if (f.sn_level[s] < fz && (f.sn_parent[s] < 0 || f.sn_level[f.sn_parent[s]] >= fz)) roots.push_back(s);
      members.assign(roots.size(), {});
      std::vector<double> work(roots.size(), 0.0);
      for (size_t k = 0; k < roots.size(); ++k) {
        std::vector<int64_t> stack{roots[k]};
        while (!stack.empty()) {
          int64_t s = stack.back();
          stack.pop_back();
          members[k].push_back(s);
          work[k] += (double)sn[s].nc * sn[s].nr;
          for (int64_t c : kids[s]) stack.push_back(c);
        }
      }
      G = (int)std::min<size_t>(NUM_SMS_B200, roots.size());
      group_of_root.assign(roots.size(), 0);
      if (G == 0) return 1e30;
      std::vector<size_t> ord(roots.size());
      for (size_t k = 0; k < ord.size(); ++k) ord[k] = k;
      std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return work[a] > work[b]; });
      std::vector<double> load(G, 0.0);
      for (size_t k : ord) {
        int gmin = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        load[gmin] += work[k];
        group_of_root[k] = gmin;
      }
      const double maxb = 8.0 * *std::max_element(load.begin(), load.end());
      // + ~8 us per fused level: each is a block-barrier-separated pass with
      // its own dependent latency (cfg2: picks 6 levels, 167 us for both
      // sweeps, against 190 us at 7 without this term; cfg3 keeps 6)
      return maxb / 25e9 + 20e-6 * (double)(f.nlevels - fz) + 8e-6 * (double)fz;
    };
    int best = 0;
    double best_t = 20e-6 * (double)f.nlevels;
    std::vector<int64_t> roots;
    std::vector<std::vector<int64_t>> members;
    std::vector<int> gor;
    int G = 0;
    const char* env = getenv("SPB_SWEEP_FUSE");
    if (env) {
      best = std::max(0, std::min((int)f.nlevels, atoi(env)));
    } else {
      for (int fz = 1; fz <= (int)f.nlevels; ++fz) {
        const double t = plan(fz, roots, members, gor, G);
        if (t < best_t) best_t = t, best = fz;
      }
    }
    d->fuse = best;
    if (best > 0) plan(best, roots, members, gor, G);
    d->ngroups = best > 0 ? G : 0;
    std::vector<int> spos, spos_off, sfw_off, sbw_off;
    std::vector<int2> sfw, sbw;
    if (best > 0) {
      std::vector<std::vector<std::vector<int64_t>>> byg(G, std::vector<std::vector<int64_t>>(best));
      for (size_t k = 0; k < roots.size(); ++k)
        for (int64_t s : members[k]) byg[gor[k]][f.sn_level[s]].push_back(s);
      for (int g = 0; g < G; ++g)
        for (int l = 0; l < best; ++l) {
          auto& v = byg[g][l];
          std::sort(v.begin(), v.end());
          spos_off.push_back((int)spos.size());
          sfw_off.push_back((int)sfw.size());
          sbw_off.push_back((int)sbw.size());
          for (int64_t s : v) {
            const SnDev& S = sn[s];
            for (int k = 0; k < S.nr; ++k) spos.push_back(S.rowoff + k);
            for (int r0 = 0; r0 < S.nr; r0 += 32) sfw.push_back(make_int2((int)s, r0));
            for (int c0 = 0; c0 < S.nc; c0 += SUB_BWC) sbw.push_back(make_int2((int)s, c0));
          }
        }
      spos_off.push_back((int)spos.size());
      sfw_off.push_back((int)sfw.size());
      sbw_off.push_back((int)sbw.size());
    }
    int rc2;
    if ((rc2 = upload(&d->sub_pos, spos)) || (rc2 = upload(&d->sub_pos_off, spos_off)) ||
        (rc2 = upload(&d->sub_fw, sfw)) || (rc2 = upload(&d->sub_fw_off, sfw_off)) ||
        (rc2 = upload(&d->sub_bw, sbw)) || (rc2 = upload(&d->sub_bw_off, sbw_off))) {
      delete d;
      return rc2;
    }
  }
  // ---- dataflow task lists for the levels >= fuse
  size_t flow_slots = 0;
  {
    const char* fe = getenv("SPB_SWEEP_FLOW");
    // experimental (SPB_SWEEP_FLOW=1): on cfg3 the per-level launches are
    // faster, since a persistent CTA serialises its tasks' latency chains
    d->flow = fe ? atoi(fe) : 0;
    std::vector<int> par(ns), fneed(ns, 0), bneed(ns, 0), bchunk_of;
    std::vector<int4> ft, bt, bch;
    std::vector<int> nch_of(ns, 0);
    for (int64_t s = 0; s < ns; ++s) par[s] = (int)f.sn_parent[s];
    for (int64_t l = d->fuse; l < f.nlevels; ++l)
      for (int64_t s : bylevel[l]) {
        ft.push_back(make_int4(0, (int)s, 0, 0));
        for (int r0 = 0; r0 < sn[s].nr; r0 += FL_ROWS) ft.push_back(make_int4(1, (int)s, r0, 0));
        if (par[s] >= 0) fneed[par[s]] += (sn[s].nr + FL_ROWS - 1) / FL_ROWS;
      }
    int slot = 0;
    for (int64_t l = f.nlevels - 1; l >= d->fuse; --l)
      for (int64_t s : bylevel[l]) {
        bt.push_back(make_int4(-(int)(s + 1), 0, 0, 0));
        bchunk_of.push_back(-1);
        const SnDev& S = sn[s];
        for (int c0 = 0; c0 < S.nc; c0 += BT_COLS) {
          const int slot0 = slot, ch = (int)bch.size();
          for (int r0 = 0; r0 < S.nr; r0 += BT_ROWS) {
            if (r0 + BT_ROWS <= c0) continue;  // entirely above the diagonal of inv(L_ss): zero
            bt.push_back(make_int4((int)s, c0, r0, slot++));
            bchunk_of.push_back(ch);
          }
          bch.push_back(make_int4((int)s, c0, slot0, slot - slot0));
          nch_of[s]++;
        }
      }
    for (int64_t s = 0; s < ns; ++s)
      if (f.sn_level[s] >= d->fuse && par[s] >= 0) bneed[s] = nch_of[par[s]];
    int maxnc = 0;
    for (int64_t s = 0; s < ns; ++s)
      if (f.sn_level[s] >= d->fuse) maxnc = std::max(maxnc, sn[s].nc);
    d->fw_smem = sizeof(double) * std::max(3 * std::min(maxnc, CH_FW), 3 * FL_FW_THREADS);
    d->nft = (int)ft.size();
    d->nbt = (int)bt.size();
    d->nbch = (int)bch.size();
    flow_slots = (size_t)slot;
    std::vector<int> zero(1 + 2 * ns + bch.size(), 0);
    int rc3;
    if ((rc3 = upload(&d->parent, par)) || (rc3 = upload(&d->ftasks, ft)) || (rc3 = upload(&d->f_need, fneed)) ||
        (rc3 = upload(&d->btasks, bt)) || (rc3 = upload(&d->btask_chunk, bchunk_of)) ||
        (rc3 = upload(&d->bchunks, bch)) || (rc3 = upload(&d->b_need, bneed)) ||
        (rc3 = upload(&d->flow_cnt, zero))) {
      delete d;
      return rc3;
    }
  }
  int rc;
  if ((rc = upload(&d->sn, sn)) || (rc = upload(&d->rows, rows)) || (rc = upload(&d->pos_owner, owner)) ||
      (rc = upload(&d->lvl_pos, lpos)) || (rc = upload(&d->M, f.Mval)) || (rc = upload(&d->asm_ptr, cnt)) ||
      (rc = upload(&d->asm_src, asrc)) || (rc = upload(&d->x2_ptr, xcnt)) || (rc = upload(&d->x2_src, xsrc)) ||
      (rc = upload(&d->fw_cta, fwc)) || (rc = upload(&d->fw_warp, fww)) || (rc = upload(&d->bw_tiles, bwt)) ||
      (rc = upload(&d->bw_chunks, bwr)) || (rc = upload(&d->bw_tile_chunk, btc)) ||
      (rc = upload(&d->bw_chunk_cnt, std::vector<int>(std::max<size_t>(bwr.size(), 1), 0))) ||
      (rc = upload(&d->bw_warp, bww))) {
    delete d;
    return rc;
  }
  d->p_slots = std::max<size_t>(std::max(bwt.size(), flow_slots), 1);
  d->nchunks = std::max<size_t>(bwr.size(), 1);
  if (cudaMalloc(&d->VZ, sizeof(double) * 3 * std::max<int64_t>(d->nrows_total, 1)) != cudaSuccess ||
      cudaMalloc(&d->P, sizeof(double) * 3 * BT_COLS * std::max<size_t>(std::max(bwt.size(), flow_slots), 1)) !=
          cudaSuccess) {
    delete d;
    set_error("cudaMalloc failed (sweep buffer)");
    return SPB_ERR_CUDA;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_forward_level, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * CH_FW * 8 + 64);
    cudaFuncSetAttribute(k_forward_flow, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * CH_FW * 8 + 64);
    for (FwLevelFn fn : {k_fw_level<4, 3>, k_fw_level<8, 2>, k_fw_level<12, 2>})
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * CH_FW * 8 + 64);
    cudaFuncSetAttribute(k_bw_level, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 4096 * 8);
    attr = true;
  }
  // persistent grids: exactly the resident CTAs
  {
    int nf = 0, nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nf, k_forward_flow, FL_FW_THREADS, d->fw_smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_backward_flow, FL_BW_THREADS, 0);
    d->fw_grid = std::max(1, nf) * NUM_SMS_B200;
    d->bw_grid = std::max(1, nb) * NUM_SMS_B200;
  }
  f.devs[cur] = d;
  return SPB_OK;
}

// Per-context sweep workspace (contexts sharing one factor step concurrently).
int sweep_work_alloc(const DeviceFactor& d, SweepWork& w) {
  w = SweepWork{};
  if (cudaMalloc(&w.VZ, sizeof(double) * 3 * std::max<int64_t>(d.nrows_total, 1)) != cudaSuccess ||
      cudaMalloc(&w.P, sizeof(double) * 3 * BT_COLS * d.p_slots) != cudaSuccess ||
      cudaMalloc(&w.chunk_cnt, sizeof(int) * d.nchunks) != cudaSuccess ||
      cudaMalloc(&w.flow_cnt, sizeof(int) * (1 + 2 * (size_t)d.ns + d.nbch)) != cudaSuccess) {
    sweep_work_free(w);
    set_error("cudaMalloc failed (sweep workspace)");
    return SPB_ERR_CUDA;
  }
  return SPB_OK;
}
void sweep_work_free(SweepWork& w) {
  for (void* p : {(void*)w.VZ, (void*)w.P, (void*)w.chunk_cnt, (void*)w.flow_cnt})
    if (p) cudaFree(p);
  w = SweepWork{};
}

// DIAGNOSTIC ONLY (tools/sweep_levels.sh): skip the launches of the upper
// levels in the SPB_SWEEP_SKIP bitmask (level kernels and gathers) or of the
// gathers in SPB_SWEEP_SKIPG; the results are then wrong, the timing tells
// each level's marginal cost in the PDL-chained sweep
static long sweep_skip(bool gather) {
  static const long m = getenv("SPB_SWEEP_SKIP") ? strtol(getenv("SPB_SWEEP_SKIP"), nullptr, 0) : 0;
  static const long g = getenv("SPB_SWEEP_SKIPG") ? strtol(getenv("SPB_SWEEP_SKIPG"), nullptr, 0) : 0;
  return gather ? (m | g) : m;
}

void sparse_forward(cudaStream_t st, const DeviceFactor& d, const double* b, double* y, double* U, double* f2,
                    int* launches, const SweepWork* w) {
  double* VZ = w ? w->VZ : d.VZ;
  int* flow_cnt = w ? w->flow_cnt : d.flow_cnt;
  if (d.fuse > 0) {
    launch_pdl(k_subtree_forward, dim3(d.ngroups), dim3(SUB_THREADS), 0, st, (const SnDev*)d.sn, (const double*)d.M,
               (const int*)d.sub_pos, (const int*)d.sub_pos_off, (const int2*)d.sub_fw, (const int*)d.sub_fw_off,
               d.fuse, (const int*)d.pos_owner, (const int*)d.asm_ptr, (const int*)d.asm_src, b, VZ, y, U);
    if (launches) ++*launches;
  }
  if (d.flow && d.nft > 0) {
    cudaMemsetAsync(flow_cnt, 0, sizeof(int) * (1 + 2 * (size_t)d.ns + d.nbch), st);
    k_forward_flow<<<d.fw_grid, FL_FW_THREADS, d.fw_smem, st>>>(d.sn, d.M, d.ftasks, d.nft, d.f_need, d.parent,
                                                                  flow_cnt, d.ns, d.pos_owner, d.asm_ptr, d.asm_src,
                                                                  b, VZ, y, U);
    if (launches) ++*launches;
  }
  for (int l = d.fuse; l < d.nlevels && !d.flow; ++l) {
    const LevelTasks& T = d.lv[l];
    if (T.npos == 0 || ((sweep_skip(false) >> l) & 1)) continue;
    if (!((sweep_skip(true) >> l) & 1))
    launch_pdl(k_fw_gather, dim3(ceil_div(T.npos, 256)), dim3(256), 0, st, (const int*)(d.lvl_pos + T.pos_off),
               T.npos, (const int*)d.pos_owner, (const int*)d.asm_ptr, (const int*)d.asm_src, (const double*)U, b,
               VZ);
    const int grid = T.ncta + (T.nwarp + FW_WARPS - 1) / FW_WARPS;
    const size_t smem = sizeof(double) * std::max(3 * std::min(T.max_nc, CH_FW), 3 * FW_THREADS);
    launch_pdl(fw_level_kernel(), dim3(grid), dim3(FW_THREADS), smem, st, (const SnDev*)d.sn, (const double*)d.M,
               (const int2*)(d.fw_cta + T.cta_off), T.ncta, (const int2*)(d.fw_warp + T.warp_off), T.nwarp,
               T.rows, (const double*)VZ, y, U);
    if (launches) *launches += 2;
  }
  if (d.n2 > 0) {
    launch_pdl(k_forward_x2, dim3(ceil_div(3 * (int64_t)d.n2, 256)), dim3(256), 0, st, d.n1, d.n2,
               (const int*)d.x2_ptr, (const int*)d.x2_src, (const double*)U, b, f2);
    if (launches) ++*launches;
  }
}

void sparse_backward(cudaStream_t st, const DeviceFactor& d, const double* y, double* XF, int* launches,
                     const SweepWork* w) {
  double* VZ = w ? w->VZ : d.VZ;
  double* Pw = w ? w->P : d.P;
  int* chunk_cnt = w ? w->chunk_cnt : d.bw_chunk_cnt;
  int* flow_cnt = w ? w->flow_cnt : d.flow_cnt;
  if (d.flow && d.nbt > 0) {
    cudaMemsetAsync(flow_cnt, 0, sizeof(int) * (1 + 2 * (size_t)d.ns + d.nbch), st);
    k_backward_flow<<<d.bw_grid, FL_BW_THREADS, 0, st>>>(d.sn, d.M, d.btasks, d.btask_chunk, d.nbt, d.bchunks,
                                                                d.b_need, d.parent, flow_cnt, d.ns, d.pos_owner,
                                                                d.rows, y, VZ, Pw, XF);
    if (launches) ++*launches;
  }
  if (!d.flow && d.nlevels > d.fuse)
    cudaMemsetAsync(chunk_cnt, 0, sizeof(int) * std::max(d.bwr_off[d.nlevels], 1), st);
  for (int l = d.nlevels - 1; l >= d.fuse && !d.flow; --l) {
    const LevelTasks& T = d.lv[l];
    if (T.npos == 0) continue;
    const int nt = d.bwt_off[l + 1] - d.bwt_off[l];
    const int nw = d.bww_off[l + 1] - d.bww_off[l];
    if (nt + nw == 0 || ((sweep_skip(false) >> l) & 1)) continue;
    if (nt)
      launch_pdl(k_bw_level, dim3(nt), dim3(256), sizeof(double) * 3 * T.bw_rows, st, (const SnDev*)d.sn,
                 (const double*)d.M, (const int4*)(d.bw_tiles + d.bwt_off[l]), T.bw_rows,
                 (const int*)(d.bw_tile_chunk + d.bwt_off[l]), (const int4*)d.bw_chunks, chunk_cnt,
                 (const int*)d.pos_owner, (const int*)d.rows, y, Pw, XF);
    if (nw)
      launch_pdl(k_bw_level_warp, dim3((nw + 7) / 8), dim3(256), 0, st, (const SnDev*)d.sn, (const double*)d.M,
                 (const int*)(d.bw_warp + d.bww_off[l]), nw, (const int*)d.pos_owner, (const int*)d.rows, y, XF);
    if (launches) *launches += (nt > 0) + (nw > 0);
  }
  if (d.fuse > 0) {
    launch_pdl(k_subtree_backward, dim3(d.ngroups), dim3(SUB_THREADS), 0, st, (const SnDev*)d.sn,
               (const double*)d.M, (const int*)d.sub_pos, (const int*)d.sub_pos_off, (const int2*)d.sub_bw,
               (const int*)d.sub_bw_off, d.fuse, (const int*)d.pos_owner, (const int*)d.rows, y, VZ, XF);
    if (launches) ++*launches;
  }
}

}  // namespace spb

spb::Factor::~Factor() {
  int cur = -1;
  cudaGetDevice(&cur);
  for (int k = 0; k < kMaxDevices; ++k)
    if (devs[k]) {
      cudaSetDevice(k);
      delete devs[k];
    }
  if (cur >= 0) cudaSetDevice(cur);
}
