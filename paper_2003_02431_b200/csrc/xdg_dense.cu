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

// ===========================================================================
// Same solves, CTA per (system, block of rows): the system's right-hand side
// (n doubles) is staged in shared memory once per task, so every lane's
// registers hold only matrix loads -- 16 in flight per lane instead of
// 8 matrix + 8 vector.  Used when every system fits the staging buffer.
namespace xdg {
namespace {

template <bool LOWER>
__device__ __forceinline__ double tri_row_dot_smem(const double* __restrict__ row,
                                                   const double* sv, int i, int n,
                                                   int lane) {
  const int j0 = LOWER ? 0 : i, j1 = LOWER ? i : n;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int jb = j0;
  for (; jb + 512 <= j1; jb += 512) {
    double r[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) r[u] = __ldg(row + jb + lane + 32 * u);
#pragma unroll
    for (int u = 0; u < 16; u += 4) {
      a0 = fma(r[u], sv[jb + lane + 32 * u], a0);
      a1 = fma(r[u + 1], sv[jb + lane + 32 * (u + 1)], a1);
      a2 = fma(r[u + 2], sv[jb + lane + 32 * (u + 2)], a2);
      a3 = fma(r[u + 3], sv[jb + lane + 32 * (u + 3)], a3);
    }
  }
  if (jb < j1) {  // clamped tail chunk: loads stay unpredicated
    double r[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) r[u] = __ldg(row + min(jb + lane + 32 * u, j1 - 1));
#pragma unroll
    for (int u = 0; u < 16; u += 4) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = jb + lane + 32 * (u + k);
        const double q = j < j1 ? sv[j] : 0.0;
        if (k == 0) a0 = fma(r[u], q, a0);
        if (k == 1) a1 = fma(r[u + 1], q, a1);
        if (k == 2) a2 = fma(r[u + 2], q, a2);
        if (k == 3) a3 = fma(r[u + 3], q, a3);
      }
    }
  }
  return warp_sum((a0 + a1) + (a2 + a3));
}

template <bool LOWER>
__global__ void __launch_bounds__(256, 4)
inv_rows_smem_kernel(int64_t ntasks, const int* __restrict__ task_sys,
                     const int* __restrict__ task_row0, int rows_per_task,
                     const int64_t* __restrict__ off, const int* __restrict__ dims,
                     const int64_t* __restrict__ vec_off, const double* __restrict__ INV,
                     const double* __restrict__ v, double* __restrict__ out) {
  extern __shared__ double sv[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t t = blockIdx.x; t < ntasks; t += gridDim.x) {
    const int s = task_sys[t];
    const int i0 = task_row0[t];
    const int n = dims[s];
    const int64_t base = vec_off[s];
    __syncthreads();  // the previous task is done with sv
    for (int j = threadIdx.x; j < n; j += 256) sv[j] = v[base + j];
    __syncthreads();
    const int i1 = min(i0 + rows_per_task, n);
    const double* A = INV + off[s];
    for (int i = i0 + warp; i < i1; i += 8) {
      const double d = tri_row_dot_smem<LOWER>(A + (int64_t)i * n, sv, i, n, lane);
      if (lane == 0) out[base + i] = LOWER ? __dadd_rn(sv[i], d) : d;
    }
  }
}

}  // namespace
}  // namespace xdg

extern "C" int xdg_lu_inv_apply_tasks(int64_t ntasks, const int* task_sys,
                                      const int* task_row0, int rows_per_task,
                                      int max_dim, int64_t total, const int64_t* off,
                                      const int* dims, const int64_t* vec_off,
                                      const double* INV, const int* src, const double* b,
                                      double* x, double* scratch, xdg_stream_t stream) {
  using namespace xdg;
  XDG_REQUIRE(ntasks >= 0 && total >= 0 && rows_per_task > 0 && max_dim >= 0,
              XDG_ERR_ARG, "bad batch");
  if (ntasks == 0 || total == 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t smem = sizeof(double) * (size_t)max_dim;
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    XDG_TRY_CUDA(cudaFuncSetAttribute(inv_rows_smem_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    XDG_TRY_CUDA(cudaFuncSetAttribute(inv_rows_smem_kernel<false>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  double* t = scratch;
  double* y = scratch + total;
  gather_kernel<<<grid_for(total, 256, 4), 256, 0, s>>>(total, src, b, t);
  XDG_CHECK_LAUNCH();
  const int g = resident_grid(inv_rows_smem_kernel<true>, 256, smem, ntasks * 256);
  inv_rows_smem_kernel<true><<<g, 256, smem, s>>>(ntasks, task_sys, task_row0, rows_per_task,
                                                  off, dims, vec_off, INV, t, y);
  XDG_CHECK_LAUNCH();
  inv_rows_smem_kernel<false><<<g, 256, smem, s>>>(ntasks, task_sys, task_row0,
                                                   rows_per_task, off, dims, vec_off, INV, y,
                                                   x);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}
