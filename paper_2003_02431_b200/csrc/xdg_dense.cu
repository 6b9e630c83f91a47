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


template <bool LOWER>
__device__ __forceinline__ double tri_row_dot(const double* __restrict__ row,
                                              const double* v, int i, int n,
                                              int lane) {
  // LOWER: sum_{j<i} row[j] v[j];  UPPER: sum_{j>=i} row[j] v[j].
  // Chunks of 256 columns: every lane issues its 8 loads of a chunk
  // together (predicated past the end), so short rows and row tails keep
  // the same memory-level parallelism as long rows.  4 accumulators, fixed
  // order: deterministic.
  const int j0 = LOWER ? 0 : i, j1 = LOWER ? i : n;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int jb = j0;
  for (; jb + 256 <= j1; jb += 256) {  // full chunks: no predicates
    double r[8], q[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      r[u] = __ldg(row + jb + lane + 32 * u);
      q[u] = v[jb + lane + 32 * u];
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
  if (jb < j1) {  // one predicated chunk for the tail
    double r[8], q[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = jb + lane + 32 * u;
      const bool in = j < j1;
      r[u] = in ? __ldg(row + j) : 0.0;
      q[u] = in ? v[j] : 0.0;
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
  return warp_sum((a0 + a1) + (a2 + a3));
}

// All systems at once, warp per row over the whole GPU.  Global row g of
// the batch belongs to system row_sys[g] (rows of a system are contiguous,
// starting at vec_off[s]); rows are visited in an interleaved order so long
// and short triangle rows mix on every SM.
__global__ void __launch_bounds__(256)
gather_kernel(int64_t total, const int* __restrict__ src,
              const double* __restrict__ b, double* __restrict__ t) {
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * 256)
    t[i] = b[src[i]];
}

template <bool LOWER>
__global__ void __launch_bounds__(256)
inv_rows_kernel(int64_t total, const int* __restrict__ row_sys,
                const int64_t* __restrict__ off, const int* __restrict__ dims,
                const int64_t* __restrict__ vec_off, const double* __restrict__ INV,
                const double* __restrict__ v, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t w = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); w < total; w += nw) {
    const int64_t g = (w & 1) ? total - 1 - (w >> 1) : (w >> 1);
    const int s = row_sys[g];
    const int64_t base = vec_off[s];
    const int n = dims[s];
    const int i = (int)(g - base);
    const double* vs = v + base;
    const double d = tri_row_dot<LOWER>(INV + off[s] + (int64_t)i * n, vs, i, n, lane);
    if (lane == 0) out[g] = LOWER ? __dadd_rn(vs[i], d) : d;
  }
}

}  // namespace
}  // namespace xdg

extern "C" int xdg_lu_inv_apply(int nsys, int64_t total, const int* row_sys,
                                const int64_t* off, const int* dims,
                                const int64_t* vec_off, const double* INV,
                                const int* src, const double* b, double* x,
                                double* scratch, xdg_stream_t stream) {
  using namespace xdg;
  XDG_REQUIRE(nsys >= 0 && total >= 0, XDG_ERR_ARG, "bad batch");
  if (nsys == 0 || total == 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  double* t = scratch;
  double* y = scratch + total;
  gather_kernel<<<grid_for(total, 256, 4), 256, 0, s>>>(total, src, b, t);
  XDG_CHECK_LAUNCH();
  const int g = resident_grid(inv_rows_kernel<true>, 256, 0, total * 32);
  inv_rows_kernel<true><<<g, 256, 0, s>>>(total, row_sys, off, dims, vec_off, INV, t, y);
  XDG_CHECK_LAUNCH();
  inv_rows_kernel<false><<<g, 256, 0, s>>>(total, row_sys, off, dims, vec_off, INV, y, x);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}
