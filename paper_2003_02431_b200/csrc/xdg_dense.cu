// Dense LU solves of the low-order PMG systems (cutdg solvers.py:208-221
// factor, 249-251 solve; SuperLU in the reference, blockmatrix.py:203-227)
// and of the coarsest multigrid level / "direct" solver (solvers.py:661-666,
// 698-710).
//
// Factors: partial-pivoting LU at setup (torch.linalg.lu_factor_ex ->
// cuSOLVER getrf), then the explicit inverses of its triangular factors
// (setup).  Every solve is x = U^-1 (L^-1 (P^T b)): two triangular GEMVs
// over the same 8 n^2 bytes forward/backward substitution would stream,
// but with no sequential dependence chain -- every row is an independent,
// coalesced dot product.  Bound: HBM.  The pivot is pre-composed with the
// gather from the global vector: rhs_i = b[src_i].
#include "xdg_common.cuh"

namespace xdg {
namespace {

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
// Solves through explicit triangular inverses of the partial-pivoting LU:
// INV (row-major n x n per system) holds L^-1 strictly below the diagonal
// (unit diagonal implicit) and U^-1 on and above it.  x = U^-1 (L^-1 P^T b)
// is two triangular GEMVs -- the same 8 n^2 bytes as forward/backward
// substitution, but no sequential chain: every row is an independent
// coalesced dot product (deterministic lane-strided partials + shuffle tree).
namespace xdg {
namespace {

constexpr int kIT = 512;  // threads per CTA (16 warps)

template <bool LOWER>
__device__ __forceinline__ double tri_row_dot(const double* __restrict__ row,
                                              const double* v, int i, int n,
                                              int lane) {
  // LOWER: sum_{j<i} row[j] v[j];  UPPER: sum_{j>=i} row[j] v[j].
  // 8 independent loads per lane in flight (memory-level parallelism for a
  // single SM streaming a whole factor), 4 accumulators, fixed order.
  const int j0 = LOWER ? 0 : i, j1 = LOWER ? i : n;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int j = j0 + lane;
  for (; j + 224 < j1; j += 256) {
    double r[8], q[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      r[u] = __ldg(row + j + 32 * u);
      q[u] = v[j + 32 * u];
    }
    a0 = fma(r[0], q[0], a0);
    a1 = fma(r[1], q[1], a1);
    a2 = fma(r[2], q[2], a2);
    a3 = fma(r[3], q[3], a3);
    a0 = fma(r[4], q[4], a0);
    a1 = fma(r[5], q[5], a1);
    a2 = fma(r[6], q[6], a2);
    a3 = fma(r[7], q[7], a3);
  }
  for (; j < j1; j += 32) a0 = fma(__ldg(row + j), v[j], a0);
  return warp_sum((a0 + a1) + (a2 + a3));
}

// one CTA per system, vectors staged in shared memory (2 n doubles)
__global__ void __launch_bounds__(kIT)
inv_apply_batched_kernel(const int64_t* __restrict__ off,
                         const int* __restrict__ dims,
                         const int64_t* __restrict__ vec_off,
                         const double* __restrict__ INV,
                         const int* __restrict__ src,
                         const double* __restrict__ b, double* __restrict__ xout) {
  extern __shared__ double sm[];
  const int s = blockIdx.x;
  const int n = dims[s];
  if (n == 0) return;
  const double* A = INV + off[s];
  const int* sidx = src + vec_off[s];
  double* x = xout + vec_off[s];
  double* t = sm;       // P^T b
  double* y = sm + n;   // L^-1 t
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int nw = kIT / 32;
  for (int i = threadIdx.x; i < n; i += kIT) t[i] = b[sidx[i]];
  __syncthreads();
  for (int i = warp; i < n; i += nw) {
    const double d = tri_row_dot<true>(A + (int64_t)i * n, t, i, n, lane);
    if (lane == 0) y[i] = __dadd_rn(t[i], d);
  }
  __syncthreads();
  for (int i = warp; i < n; i += nw) {
    const double d = tri_row_dot<false>(A + (int64_t)i * n, y, i, n, lane);
    if (lane == 0) x[i] = d;
  }
}

// one large system: warp per row over the whole GPU, rows interleaved so
// long and short triangle rows mix on every SM
__global__ void __launch_bounds__(256)
gather_kernel(int n, const int* __restrict__ src, const double* __restrict__ b,
              double* __restrict__ t) {
  for (int i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256)
    t[i] = b[src[i]];
}

template <bool LOWER>
__global__ void __launch_bounds__(256)
inv_apply_rows_kernel(int n, const double* __restrict__ A,
                      const double* __restrict__ v, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * 8;
  for (int w = blockIdx.x * 8 + (threadIdx.x >> 5); w < n; w += nw) {
    // pair long and short rows: w -> rows alternate from both ends
    const int i = (w & 1) ? n - 1 - (w >> 1) : (w >> 1);
    const double d = tri_row_dot<LOWER>(A + (int64_t)i * n, v, i, n, lane);
    if (lane == 0) out[i] = LOWER ? __dadd_rn(v[i], d) : d;
  }
}

}  // namespace
}  // namespace xdg

extern "C" int xdg_lu_inv_apply_batched(int nsys, const int64_t* off,
                                        const int* dims, const int64_t* vec_off,
                                        const double* INV, const int* src,
                                        const double* b, double* x,
                                        int max_n, xdg_stream_t stream) {
  using namespace xdg;
  if (nsys <= 0) return XDG_OK;
  const size_t smem = (size_t)2 * max_n * sizeof(double);
  XDG_REQUIRE(smem <= 200 * 1024, XDG_ERR_ARG,
              "batched inverse apply: system of %d unknowns exceeds shared memory", max_n);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  static thread_local bool attr = false;
  if (!attr) {
    XDG_TRY_CUDA(cudaFuncSetAttribute(inv_apply_batched_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024));
    attr = true;
  }
  inv_apply_batched_kernel<<<nsys, kIT, smem, s>>>(off, dims, vec_off, INV, src, b, x);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_lu_inv_apply_large(int n, const double* INV, const int* src,
                                      const double* b, double* x,
                                      double* scratch, xdg_stream_t stream) {
  using namespace xdg;
  if (n <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  double* t = scratch;
  double* y = scratch + n;
  gather_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(n, src, b, t);
  XDG_CHECK_LAUNCH();
  const int g = resident_grid(inv_apply_rows_kernel<true>, 256, 0, (int64_t)n * 32);
  inv_apply_rows_kernel<true><<<g, 256, 0, s>>>(n, INV, t, y);
  XDG_CHECK_LAUNCH();
  inv_apply_rows_kernel<false><<<g, 256, 0, s>>>(n, INV, y, x);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}
