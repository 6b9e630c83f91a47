// Shared helpers for the xdg_b200 kernels (sm_100a).
//
// Error model: every exported entry point returns an int status (XDG_OK = 0)
// and records a message retrievable through xdg_last_error().  The Python
// layer maps statuses onto the reference's exception classes
// (cutdg/errors.py: DimensionMismatchError, SingularSystemError, ...).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <stdio.h>

#include "../../include/xdg_b200.h"
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3 (no library to link)

namespace xdg {

// NVTX range for the lifetime of a scope: the solver phases show up as named
// ranges in nsys / ncu --nvtx timelines (no cost when no tool is attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

void set_error(const char* fmt, ...);

#define XDG_TRY_CUDA(expr)                                                 \
  do {                                                                     \
    cudaError_t _e = (expr);                                               \
    if (_e != cudaSuccess) {                                               \
      ::xdg::set_error("%s:%d: %s -> %s", __FILE__, __LINE__, #expr,       \
                       cudaGetErrorString(_e));                            \
      return XDG_ERR_CUDA;                                                 \
    }                                                                      \
  } while (0)

#define XDG_TRY(expr)                 \
  do {                                \
    int _st = (expr);                 \
    if (_st != XDG_OK) return _st;    \
  } while (0)

#define XDG_CHECK_LAUNCH() XDG_TRY_CUDA(cudaGetLastError())

#define XDG_REQUIRE(cond, code, ...)                                       \
  do {                                                                     \
    if (!(cond)) {                                                         \
      ::xdg::set_error(__VA_ARGS__);                                       \
      return (code);                                                       \
    }                                                                      \
  } while (0)

// Device-resident column-count variants of the RM kernels (xdg_vec.cu):
// launched for max_cols columns, the kernels use min(max_cols, *ncols_dev).
int gemv_t_dev(int64_t L, int max_cols, const int* ncols_dev, const double* W, int64_t ldw,
               const double* w, double* coeff, void* ws, cudaStream_t s);
int gemv_update2_dev(int64_t L, int max_cols, const int* ncols_dev, const double* W,
                     const double* Z, int64_t ld, const double* cw, const double* cz,
                     double* w, double* z, cudaStream_t s);
int add_small_dev(int max_n, const int* n_dev, const double* a, const double* b, double* out,
                  cudaStream_t s);

// Scalar arithmetic with the same rounding on the host and on the device
// (separately rounded mul / add / div; no contraction), so a decision made
// by a 1-thread kernel equals the host driver's bit for bit.
__host__ __device__ __forceinline__ double rmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  volatile double r = a * b;
  return r;
#endif
}
__host__ __device__ __forceinline__ double radd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  volatile double r = a + b;
  return r;
#endif
}
__host__ __device__ __forceinline__ double rdiv(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  volatile double r = a / b;
  return r;
#endif
}
__host__ __device__ __forceinline__ double rsqrt_(double a) {
#ifdef __CUDA_ARCH__
  return __dsqrt_rn(a);
#else
  return sqrt(a);  // IEEE correctly rounded on both sides
#endif
}
// hypot(a, b) = m sqrt(1 + (s / m)^2), m = max(|a|, |b|): no overflow, the
// same bits on host and device (np.hypot, solvers.py:813, to ~1 ulp).
__host__ __device__ __forceinline__ double xhypot(double a, double b) {
  const double x = fabs(a), y = fabs(b);
  const double m = x > y ? x : y, t = x > y ? y : x;
  if (m == 0.0) return 0.0;
  const double q = rdiv(t, m);
  return rmul(m, rsqrt_(radd(1.0, rmul(q, q))));
}

// Number of SMs on the current device (cached per process; one device per
// process is the deployment model).
int sm_count();

// Grid for a grid-stride kernel: enough CTAs to cover `work` threads but at
// most `per_sm` resident CTAs on every SM (persistent-style sizing in
// multiples of the SM count).
inline int grid_for(int64_t work, int threads, int per_sm) {
  int64_t need = (work + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count() * per_sm;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

// Grid for a grid-stride kernel sized to exactly one resident wave:
// SMs x (CTAs of this kernel that fit on one SM), capped by the work.  A
// grid larger than the resident capacity leaves a partial second wave whose
// CTAs carry a full share of the grid-stride work (tail effect).
template <typename Kernel>
int resident_grid(Kernel kernel, int threads, size_t smem, int64_t work) {
  static thread_local const void* keys[64];
  static thread_local int vals[64];
  static thread_local int n = 0;
  const void* key = reinterpret_cast<const void*>(kernel);
  int per_sm = 0;
  for (int i = 0; i < n; ++i)
    if (keys[i] == key) per_sm = vals[i];
  if (per_sm == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads,
                                                      smem) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    if (n < 64) {
      keys[n] = key;
      vals[n] = per_sm;
      ++n;
    }
  }
  int64_t need = (work + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count() * per_sm;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

// ---------------------------------------------------------------------------
// Deterministic reductions.  A CTA reduces its threads' values through a
// fixed shuffle tree, writes one partial per CTA, and the last CTA to finish
// (ticket counter) sums the partials in CTA order.  No floating-point
// atomics, so results are bit-reproducible run to run.

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum `v` over the CTA; result valid in thread 0.  blockDim.x % 32 == 0.
__device__ __forceinline__ double block_sum(double v, double* smem32) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) smem32[warp] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  double r = 0.0;
  if (warp == 0) {
    r = lane < nw ? smem32[lane] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;
}

// Workspace layout for the reductions: [counter(8 B)][partials...].
// Every CTA calls this with its thread-0 value; the last CTA writes
// out[0] = sum of partials in CTA order and re-arms the counter.
__device__ __forceinline__ void grid_finalize(double cta_value, double* ws,
                                              double* out) {
  __shared__ bool am_last;
  unsigned int* counter = reinterpret_cast<unsigned int*>(ws);
  double* partials = ws + 1;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = cta_value;
    __threadfence();
    unsigned int t = atomicAdd(counter, 1u);
    am_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (am_last) {
    __threadfence();
    // fixed-order sum of the partials by warp 0, lanes striding, then a
    // shuffle tree: deterministic for a fixed grid size.
    double s = 0.0;
    if (threadIdx.x < 32) {
      for (int i = threadIdx.x; i < (int)gridDim.x; i += 32)
        s += ((volatile double*)partials)[i];
      s = warp_sum(s);
      if (threadIdx.x == 0) {
        out[0] = s;
        *counter = 0u;
      }
    }
  }
}

}  // namespace xdg
