// Batched dense LU solves (forward + backward substitution with partial
// pivoting), one CTA per system, variable sizes.
//
// Used for the low-order systems of the degree-separated preconditioner
// (cutdg solvers.py:208-221 factor, 249-251 solve; the reference uses SuperLU,
// blockmatrix.py:203-227) -- one system per Schwarz block, or one global
// system for GMRES -- and for the coarsest multigrid level / the "direct"
// solver (solvers.py:661-666, 698-710).
//
// Factors come from a dense LU with partial pivoting (A = P L U, L unit
// lower, packed row-major, torch.linalg.lu_factor at setup).  The pivot is
// pre-composed with the gather from the global vector: rhs_i = b[src_i].
//
// Algorithm (per CTA): panels of T = 32 rows.  For each panel, the warps
// first apply the already-solved part as a GEMV (lanes stride along the
// row: coalesced reads of the row-major factor), then warp 0 solves the
// 32x32 triangle with shuffles.  Forward then backward.  Bound: HBM (the
// factor is streamed once per solve: 8 n^2 bytes).
#include "xdg_common.cuh"

namespace xdg {
namespace {

constexpr int kT = 512;   // threads per CTA
constexpr int kPanel = 32;

__global__ void __launch_bounds__(kT)
lu_solve_batched_kernel(const int64_t* __restrict__ lu_off,
                        const int* __restrict__ dims,
                        const int64_t* __restrict__ vec_off,
                        const double* __restrict__ LU,
                        const int* __restrict__ src, const double* __restrict__ b,
                        double* __restrict__ xout) {
  const int s = blockIdx.x;
  const int n = dims[s];
  if (n == 0) return;
  const double* A = LU + lu_off[s];
  const int* sidx = src + vec_off[s];
  double* x = xout + vec_off[s];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int nwarps = kT / 32;

  for (int i = threadIdx.x; i < n; i += kT) x[i] = b[sidx[i]];
  __syncthreads();

  // ---- forward: L y = P^T b (unit diagonal) ----
  for (int p0 = 0; p0 < n; p0 += kPanel) {
    const int pe = min(p0 + kPanel, n);
    if (p0 > 0) {
      for (int i = p0 + warp; i < pe; i += nwarps) {
        const double* row = A + (int64_t)i * n;
        double acc = 0.0;
        for (int j = lane; j < p0; j += 32) acc = fma(row[j], x[j], acc);
        acc = warp_sum(acc);
        if (lane == 0) x[i] -= acc;
      }
      __syncthreads();
    }
    if (warp == 0) {
      const int i = p0 + lane;
      double t = i < pe ? x[i] : 0.0;
      for (int j = p0; j < pe; ++j) {
        const double yj = __shfl_sync(0xffffffffu, t, j - p0);
        if (i > j && i < pe) t = fma(-A[(int64_t)i * n + j], yj, t);
      }
      if (i < pe) x[i] = t;
    }
    __syncthreads();
  }

  // ---- backward: U x = y ----
  for (int pe = n; pe > 0; pe -= kPanel) {
    const int p0 = max(pe - kPanel, 0);
    if (pe < n) {
      for (int i = p0 + warp; i < pe; i += nwarps) {
        const double* row = A + (int64_t)i * n;
        double acc = 0.0;
        for (int j = pe + lane; j < n; j += 32) acc = fma(row[j], x[j], acc);
        acc = warp_sum(acc);
        if (lane == 0) x[i] -= acc;
      }
      __syncthreads();
    }
    if (warp == 0) {
      const int i = p0 + lane;
      double t = i < pe ? x[i] : 0.0;
      for (int j = pe - 1; j >= p0; --j) {
        if (i == j) t = t / A[(int64_t)j * n + j];
        const double xj = __shfl_sync(0xffffffffu, t, j - p0);
        if (i < j) t = fma(-A[(int64_t)i * n + j], xj, t);
      }
      if (i < pe) x[i] = t;
    }
    __syncthreads();
  }
}

// ipiv (LAPACK, 1-based sequential row swaps) -> permutation, one thread
// per system (setup only).
__global__ void ipiv_to_perm_kernel(int nsys, const int* __restrict__ dims,
                                    const int64_t* __restrict__ vec_off,
                                    const int* __restrict__ ipiv,
                                    int* __restrict__ perm) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nsys) return;
  const int n = dims[s];
  int* p = perm + vec_off[s];
  const int* ip = ipiv + vec_off[s];
  for (int i = 0; i < n; ++i) p[i] = i;
  for (int i = 0; i < n; ++i) {
    const int j = ip[i] - 1;
    const int t = p[i];
    p[i] = p[j];
    p[j] = t;
  }
}

}  // namespace
}  // namespace xdg

extern "C" int xdg_lu_solve_batched(int nsys, const int64_t* lu_off,
                                    const int* dims, const int64_t* vec_off,
                                    const double* LU, const int* src,
                                    const double* b, double* x,
                                    xdg_stream_t stream) {
  using namespace xdg;
  XDG_REQUIRE(nsys >= 0, XDG_ERR_ARG, "negative system count");
  if (nsys == 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  lu_solve_batched_kernel<<<nsys, kT, 0, s>>>(lu_off, dims, vec_off, LU, src,
                                              b, x);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_ipiv_to_perm(int nsys, const int* dims,
                                const int64_t* vec_off, const int* ipiv,
                                int* perm, xdg_stream_t stream) {
  using namespace xdg;
  if (nsys <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  ipiv_to_perm_kernel<<<(nsys + 127) / 128, 128, 0, s>>>(nsys, dims, vec_off,
                                                          ipiv, perm);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

// ===========================================================================
// Multi-CTA panel triangular solves for ONE large system (the global
// low-order system of GMRES-PMG, solvers.py:800 with all cells, and large
// coarsest levels).  One CTA per 64-row panel; panels are claimed through an
// atomic ticket in launch order, so every panel a CTA waits for has already
// started (no deadlock without a cooperative launch).  A monotone counter
// publishes how many panels are solved; a waiting CTA folds each newly
// solved panel into LANE-PARTIAL accumulators (lane l always sums columns
// l, l+64, ... in panel order) and reduces across lanes only once, so the
// result does not depend on timing: bit-reproducible.  The diagonal 64x64
// blocks are applied through their precomputed inverses (setup), turning the
// sequential triangle into a small GEMV.  Bound: HBM (each factor is read
// once, 8 n^2 / 2 bytes per direction) plus the panel chain latency.
namespace xdg {
namespace {

constexpr int kP = 64;        // panel rows
constexpr int kPT = 256;      // threads per CTA (8 warps x 8 rows)

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// FORWARD: y = Linv-panels applied to (P^T b - L_offdiag y).  counters[0] =
// ticket, counters[1] = solved panels.  BACKWARD uses U and counts from the
// bottom.
template <bool FORWARD>
__global__ void __launch_bounds__(kPT)
panel_trsv_kernel(int n, const double* __restrict__ LU,
                  const double* __restrict__ Dinv, const int* __restrict__ src,
                  const double* __restrict__ b, double* y, int* counters) {
  __shared__ int s_panel, s_ready;
  __shared__ double t[kP];
  const int np = (n + kP - 1) / kP;
  if (threadIdx.x == 0) s_panel = atomicAdd(counters, 1);
  __syncthreads();
  const int seq = s_panel;                       // position in the chain
  const int p = FORWARD ? seq : np - 1 - seq;    // panel index
  const int r0 = p * kP;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // warp w owns panel rows w*8 .. w*8+7; lane covers columns lane, lane+32
  double part[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) part[q] = 0.0;
  int folded = 0;
  while (folded < seq) {
    if (threadIdx.x == 0) {
      int r;
      while ((r = ld_acquire(counters + 1)) == folded) __nanosleep(64);
      s_ready = r;
    }
    __syncthreads();
    const int ready = s_ready;
    __syncthreads();
    for (int k = folded; k < ready; ++k) {
      const int qp = FORWARD ? k : np - 1 - k;   // solved panel to fold
      const int c0 = qp * kP;
      const double y0 = (c0 + lane < n) ? ((volatile double*)y)[c0 + lane] : 0.0;
      const double y1 = (c0 + lane + 32 < n) ? ((volatile double*)y)[c0 + lane + 32] : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int row = r0 + warp * 8 + q;
        if (row < n) {
          const double* A = LU + (int64_t)row * n + c0;
          if (c0 + lane < n) part[q] = fma(A[lane], y0, part[q]);
          if (c0 + lane + 32 < n) part[q] = fma(A[lane + 32], y1, part[q]);
        }
      }
    }
    folded = ready;
  }
  // t = rhs - (sum over folded panels)
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const double s = warp_sum(part[q]);
    const int lr = warp * 8 + q, row = r0 + lr;
    if (lane == 0)
      t[lr] = row < n ? ((FORWARD ? b[src[row]] : ((volatile double*)y)[row]) - s) : 0.0;
  }
  __syncthreads();
  // y_panel = Dinv_p t  (64 x 64 row-major, identity-padded past n)
  const double* D = Dinv + (int64_t)p * kP * kP;
  double out[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int lr = warp * 8 + q;
    double s = fma(D[lr * kP + lane], t[lane], 0.0);
    s = fma(D[lr * kP + lane + 32], t[lane + 32], s);
    out[q] = warp_sum(s);
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int row = r0 + warp * 8 + q;
      if (row < n) y[row] = out[q];
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) st_release(counters + 1, seq + 1);
}

}  // namespace
}  // namespace xdg

extern "C" int xdg_lu_solve_panels(int n, const double* LU, const double* Linv,
                                   const double* Uinv, const int* src,
                                   const double* b, double* x, int* counters,
                                   xdg_stream_t stream) {
  using namespace xdg;
  XDG_REQUIRE(n >= 0, XDG_ERR_ARG, "negative size");
  if (n == 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int np = (n + kP - 1) / kP;
  XDG_TRY_CUDA(cudaMemsetAsync(counters, 0, 4 * sizeof(int), s));
  // forward writes y into x; the backward pass reads its right-hand side
  // from x (in place: each panel reads its own rows before overwriting)
  panel_trsv_kernel<true><<<np, kPT, 0, s>>>(n, LU, Linv, src, b, x, counters);
  XDG_CHECK_LAUNCH();
  panel_trsv_kernel<false><<<np, kPT, 0, s>>>(n, LU, Uinv, src, b, x, counters + 2);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}
