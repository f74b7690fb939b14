// Shared device-side definitions (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>
#include <math_constants.h>

#include "spb_internal.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "schurpd_b200 is built for sm_100a only"
#endif

namespace spb {

constexpr int NUM_SMS_B200 = 148;

#define SPB_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess) {                                                            \
      spb::set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " +    \
                     __FILE__ + ":" + std::to_string(__LINE__) + " (" #call ")");       \
      return SPB_ERR_CUDA;                                                              \
    }                                                                                   \
  } while (0)

// ------------------------------------------------------------ bounded spins
// Every inter-CTA / inter-GPU wait (tile flags, solved-row sentinels, grid
// barriers, dataflow counters) is bounded in TIME: a wait longer than
// kSpinLimitNs (a dead peer GPU, a lost flag) traps, which fails the launch
// with an error instead of leaving the device hung. The clock is read only
// every 64th spin, so a flag that is already set costs nothing extra.
constexpr unsigned long long kSpinLimitNs = 60ull * 1000ull * 1000ull * 1000ull;  // 60 s

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct SpinGuard {
  unsigned long long t0 = 0;
  unsigned it = 0;
  __device__ __forceinline__ void tick() {
    if ((++it & 63u) == 0u) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > kSpinLimitNs) __trap();
    }
  }
};

// ------------------------------------------------------------ collider data
struct ShapeDev {
  int kind;
  double p[7];
  int dims[3];
  const double* values;  // device, indexed [ix + nx*(iy + ny*iz)]
};

struct PosedDev {
  int shape;
  double R[9];
  double t[3];
};

constexpr int MAX_COLLIDERS = 32;

struct ColliderSet {
  int n;
  PosedDev posed[MAX_COLLIDERS];
};

// ------------------------------------------------------------ element data
struct ElemParams {
  double mu, mu_prime, smin, smax;
  int biphasic;
};

// ------------------------------------------------------------ small utils
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// Dense 64x64 FP64 tiles are stored "swizzled row-major": element (r, c) at
// r*64 + (c ^ ((r & 3) << 2)). The XOR moves 4-column groups so that DMMA
// fragment loads (8 rows x 4 consecutive k) hit 16 distinct 8-byte bank slots
// per half-warp, while whole tiles stay contiguous for one 32 KB bulk (TMA)
// copy. The XOR only touches column bits 2-3, which are lane constants in the
// fragment loads, so those keep register + immediate addressing.
__host__ __device__ __forceinline__ int swz(int r, int c) { return r * 64 + (c ^ ((r & 3) << 2)); }

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// system scope: flags written by peer GPUs over NVLink
__device__ __forceinline__ int ld_relaxed_sys(const int* p) {
  int v;
  asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// Programmatic dependent launch: a kernel launched with launch_pdl() may start
// while its predecessor drains; it must call pdl_wait() before touching data
// the predecessor writes (no-op without a programmatic predecessor).
// pdl_trigger() lets the successor start launching as this CTA proceeds.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Set while a concurrent-scene frame is enqueued: there, kernels placed early
// by PDL hold SMs the other scenes' work needs (cfg5: 4,467 scene-frames/s
// without PDL against 4,321 with it), so every launch_pdl is an ordinary launch.
inline thread_local bool tl_pdl_off = false;

template <typename... K, typename... A>
inline cudaError_t launch_pdl(void (*kernel)(K...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  static const bool off = getenv("SPB_PDL") && getenv("SPB_PDL")[0] == '0';  // A/B diagnostics
  cfg.attrs = at;
  cfg.numAttrs = (off || tl_pdl_off) ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}

}  // namespace spb
