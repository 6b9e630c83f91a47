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
