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
#include <stdlib.h>

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

// Ring variant: the factor rows stream through a per-warp ring of
// shared-memory stages filled by cp.async (LDGSTS: no registers held by
// loads in flight), kRingStages - 1 chunks of kRingChunk doubles ahead of
// the FMAs.  A warp's rows of a task form one chunk stream, so the memory
// pipeline does not drain between rows (the register version issues a row's
// loads, reduces, then starts the next row).
constexpr int kRingChunk = 512;  // doubles per stage (4 KB)
constexpr int kRingStages = 4;

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem_src) : "memory");
}

template <bool LOWER>
__global__ void __launch_bounds__(256, 1)
inv_rows_ring_kernel(int64_t ntasks, const int* __restrict__ task_sys,
                     const int* __restrict__ task_row0, int rows_per_task, int sv_len,
                     const int64_t* __restrict__ off, const int* __restrict__ dims,
                     const int64_t* __restrict__ vec_off, const double* __restrict__ INV,
                     const double* __restrict__ v, double* __restrict__ out) {
  extern __shared__ double sm[];
  double* sv = sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* ring = sm + sv_len + warp * (kRingStages * kRingChunk);
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
    // prefetch cursor (pi, pj) and consume cursor (ci, cj) over this warp's
    // rows i0 + warp, + 8, ...; row i spans columns [lo(i), hi(i))
    auto lo = [&](int i) { return LOWER ? 0 : i; };
    auto hi = [&](int i) { return LOWER ? i : n; };
    int pi = i0 + warp, pj = pi < i1 ? lo(pi) : 0;
    int ci = pi, cj = pj;
    int pstage = 0, cstage = 0;
    auto issue = [&]() {  // one chunk of the prefetch stream (or an empty group)
      while (pi < i1 && pj >= hi(pi)) {  // next row (rows may be empty: L^-1 row 0)
        pi += 8;
        pj = pi < i1 ? lo(pi) : 0;
      }
      if (pi < i1) {
        const int len = min(kRingChunk, hi(pi) - pj);
        const double* src = A + (int64_t)pi * n + pj;
        double* dst = ring + pstage * kRingChunk;
        for (int e = lane; e < len; e += 32) cp_async8(dst + e, src + e);
        pj += len;
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      pstage = (pstage + 1) % kRingStages;
    };
#pragma unroll
    for (int q = 0; q < kRingStages - 1; ++q) issue();
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    while (ci < i1) {
      if (cj >= hi(ci)) {  // row done (or empty)
        const double d = warp_sum((a0 + a1) + (a2 + a3));
        if (lane == 0) out[base + ci] = LOWER ? __dadd_rn(sv[ci], d) : d;
        a0 = a1 = a2 = a3 = 0.0;
        ci += 8;
        cj = ci < i1 ? lo(ci) : 0;
        continue;
      }
      issue();
      asm volatile("cp.async.wait_group %0;" ::"n"(kRingStages - 1) : "memory");
      __syncwarp();
      const int len = min(kRingChunk, hi(ci) - cj);
      const double* buf = ring + cstage * kRingChunk;
#pragma unroll 4
      for (int e = lane; e < len; e += 128) {
        a0 = fma(buf[e], sv[cj + e], a0);
        if (e + 32 < len) a1 = fma(buf[e + 32], sv[cj + e + 32], a1);
        if (e + 64 < len) a2 = fma(buf[e + 64], sv[cj + e + 64], a2);
        if (e + 96 < len) a3 = fma(buf[e + 96], sv[cj + e + 96], a3);
      }
      __syncwarp();  // the stage is refilled by the next issue()
      cj += len;
      cstage = (cstage + 1) % kRingStages;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
}

bool inv_ring_enabled() {
  static const bool on = [] {
    const char* e = getenv("XDG_INV_RING");
    return e != nullptr && atoi(e) != 0;
  }();
  return on;
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
  const int sv_len = (max_dim + 1) & ~1;
  const size_t rsmem = sizeof(double) * ((size_t)sv_len + 8 * kRingStages * kRingChunk);
  if (inv_ring_enabled() && rsmem <= 200 * 1024) {
    static size_t rattr = 0;
    if (rsmem > rattr) {
      XDG_TRY_CUDA(cudaFuncSetAttribute(inv_rows_ring_kernel<true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)rsmem));
      XDG_TRY_CUDA(cudaFuncSetAttribute(inv_rows_ring_kernel<false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)rsmem));
      rattr = rsmem;
    }
    const int g = resident_grid(inv_rows_ring_kernel<true>, 256, rsmem, ntasks * 256);
    inv_rows_ring_kernel<true><<<g, 256, rsmem, s>>>(ntasks, task_sys, task_row0,
                                                      rows_per_task, sv_len, off, dims,
                                                      vec_off, INV, t, y);
    XDG_CHECK_LAUNCH();
    inv_rows_ring_kernel<false><<<g, 256, rsmem, s>>>(ntasks, task_sys, task_row0,
                                                       rows_per_task, sv_len, off, dims,
                                                       vec_off, INV, y, x);
    XDG_CHECK_LAUNCH();
    return XDG_OK;
  }
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
