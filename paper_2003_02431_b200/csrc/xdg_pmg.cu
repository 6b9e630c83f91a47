// Degree-separated block preconditioner (p-multigrid, cutdg solvers.py:183-305)
// and the additive overlapping Schwarz combination (solvers.py:460-478).
//
// One "plan" covers a set of systems (Schwarz blocks, or the single global
// cell set of GMRES-PMG).  Work item = one cell (block row) of one system.
//
//  xdg_pmg_build_low   (setup)  dense low-order matrices A_s, one per system:
//                               A_s[(lr*m+p), (lc*m+q)] = M[c_lr, c_lc](p, q)
//                               over the blocks whose row AND column are in
//                               the system (extract_block_submatrix,
//                               blockmatrix.py:153-167; solvers.py:208-215)
//  xdg_pmg_gather_high (setup)  per-cell high-order diagonal blocks
//                               H_c = M[c, c](m:, m:)      (solvers.py:232)
//  xdg_pmg_high        (apply)  fused: local residual on the high rows
//                               r = b - M_II x_lo (only the low columns of
//                               each block are touched, the high part of x is
//                               zero: solvers.py:257) + per-cell pivoted LU
//                               solve of H_c (solvers.py:258-262), one warp
//                               per cell, factors column-major so a lane
//                               per row reads coalesced columns
//  xdg_pmg_combine     (apply)  z = (sum of overlapping contributions in
//                               Schwarz-block order) ./ damping, no atomics
//                               (solvers.py:473-478)
#include <algorithm>

#include "xdg_common.cuh"

namespace xdg {
namespace {

constexpr int kT = 256;

__global__ void __launch_bounds__(kT)
build_low_kernel(int nwork, int N, int m, const int* __restrict__ wi_ptr,
                 const int* __restrict__ wi_blk, const int* __restrict__ wi_lcol,
                 const int* __restrict__ wi_lrow, const int* __restrict__ wi_sys,
                 const int64_t* __restrict__ lu_off, const int* __restrict__ dims,
                 const double* __restrict__ val_t, double* __restrict__ A) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * kT) >> 5;
  for (int w = (blockIdx.x * kT + threadIdx.x) >> 5; w < nwork; w += warps) {
    const int s = wi_sys[w];
    const int n = dims[s];
    double* As = A + lu_off[s];
    const int lr = wi_lrow[w];
    for (int e = wi_ptr[w]; e < wi_ptr[w + 1]; ++e) {
      const int64_t k = wi_blk[e];
      const int lc = wi_lcol[e];
      const double* v = val_t + k * N * N;
      for (int pq = lane; pq < m * m; pq += 32) {
        const int p = pq / m, q = pq - p * m;
        As[(int64_t)(lr * m + p) * n + lc * m + q] = v[q * N + p];
      }
    }
  }
}

__global__ void __launch_bounds__(kT)
gather_high_kernel(int ncells, int N, int m, const int* __restrict__ cells,
                   const int* __restrict__ diag_blk,
                   const double* __restrict__ val_t, double* __restrict__ H) {
  const int nh = N - m;
  const int64_t total = (int64_t)ncells * nh * nh;
  for (int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * kT) {
    const int ci = (int)(t / (nh * nh));
    const int r = (int)(t - (int64_t)ci * nh * nh);
    const int i = r / nh, j = r - i * nh;  // row-major H(i, j)
    const int64_t k = diag_blk[ci];
    H[t] = val_t[k * N * N + (int64_t)(m + j) * N + (m + i)];
  }
  (void)cells;
}

// rows of the high block owned by a lane: i = lane (slot 0), lane+32 (slot 1)
template <int SLOTS>
__global__ void __launch_bounds__(kT)
pmg_high_kernel(int nwork, int N, int m, const int* __restrict__ wi_ptr,
                const int* __restrict__ wi_blk, const int* __restrict__ wi_lcol,
                const int* __restrict__ wi_cell, const int* __restrict__ wi_lrow,
                const int64_t* __restrict__ wi_xlo, const int* __restrict__ wi_hidx,
                const int64_t* __restrict__ wi_out,
                const double* __restrict__ val_t, const double* __restrict__ HLU,
                const int* __restrict__ hperm, const double* __restrict__ b,
                const double* __restrict__ xlo_buf, double* __restrict__ out_buf) {
  const int nh = N - m;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * kT) >> 5;
  for (int w = (blockIdx.x * kT + threadIdx.x) >> 5; w < nwork; w += warps) {
    const int c = wi_cell[w];
    const double* xlo = xlo_buf + wi_xlo[w];
    double acc[SLOTS];
#pragma unroll
    for (int sl = 0; sl < SLOTS; ++sl) acc[sl] = 0.0;
    // ---- local residual r = b - M_II x (high rows, low columns) ----
    for (int e = wi_ptr[w]; e < wi_ptr[w + 1]; ++e) {
      const int64_t k = wi_blk[e];
      const double* v = val_t + k * N * N + m;  // column q: v[q*N + i]
      const double* xq = xlo + (int64_t)wi_lcol[e] * m;
      for (int q = 0; q < m; ++q) {
        const double xv = __ldg(xq + q);
#pragma unroll
        for (int sl = 0; sl < SLOTS; ++sl) {
          const int i = lane + 32 * sl;
          if (i < nh) acc[sl] = __dadd_rn(acc[sl], __dmul_rn(__ldg(v + q * N + i), xv));
        }
      }
    }
    double r[SLOTS];
#pragma unroll
    for (int sl = 0; sl < SLOTS; ++sl) {
      const int i = lane + 32 * sl;
      r[sl] = i < nh ? __dadd_rn(b[(int64_t)c * N + m + i], -acc[sl]) : 0.0;
    }
    // ---- pivoted LU solve of H_c (column-major LU, perm composed) ----
    const int hi = wi_hidx[w];
    const double* F = HLU + (int64_t)hi * nh * nh;
    const int* P = hperm + (int64_t)hi * nh;
    double t[SLOTS];
#pragma unroll
    for (int sl = 0; sl < SLOTS; ++sl) {
      const int i = lane + 32 * sl;
      const int pi = i < nh ? P[i] : 0;
      double got = 0.0;
#pragma unroll
      for (int s2 = 0; s2 < SLOTS; ++s2) {
        const double v2 = __shfl_sync(0xffffffffu, r[s2], pi & 31);
        if ((pi >> 5) == s2) got = v2;
      }
      t[sl] = got;
    }
    for (int j = 0; j < nh; ++j) {  // unit lower, column-oriented
      const double send = SLOTS == 1 ? t[0] : ((j >> 5) == 0 ? t[0] : t[SLOTS - 1]);
      const double yj = __shfl_sync(0xffffffffu, send, j & 31);
#pragma unroll
      for (int sl = 0; sl < SLOTS; ++sl) {
        const int i = lane + 32 * sl;
        if (i > j && i < nh) t[sl] = __dadd_rn(t[sl], -__dmul_rn(yj, F[(int64_t)j * nh + i]));
      }
    }
    for (int j = nh - 1; j >= 0; --j) {  // upper, column-oriented
#pragma unroll
      for (int sl = 0; sl < SLOTS; ++sl)
        if (lane + 32 * sl == j) t[sl] = __ddiv_rn(t[sl], F[(int64_t)j * nh + j]);
      const double send = SLOTS == 1 ? t[0] : ((j >> 5) == 0 ? t[0] : t[SLOTS - 1]);
      const double xj = __shfl_sync(0xffffffffu, send, j & 31);
#pragma unroll
      for (int sl = 0; sl < SLOTS; ++sl) {
        const int i = lane + 32 * sl;
        if (i < j) t[sl] = __dadd_rn(t[sl], -__dmul_rn(xj, F[(int64_t)j * nh + i]));
      }
    }
    // ---- write the cell's full local solution (low copy + high) ----
    double* o = out_buf + wi_out[w];
    const double* self = xlo + (int64_t)wi_lrow[w] * m;
    for (int q = lane; q < m; q += 32) o[q] = self[q];
#pragma unroll
    for (int sl = 0; sl < SLOTS; ++sl) {
      const int i = lane + 32 * sl;
      if (i < nh) o[m + i] = t[sl];
    }
  }
}

// nh <= 16: floor(32/nh) cells per warp, lane group g owns cell w_base + g,
// lane i of the group owns high row i.  Same arithmetic order per row as
// pmg_high_kernel (blocks in order, low columns in order, separate mul/add;
// column-oriented LU substitutions).
// N_T / M_T > 0: block size and low modes known at compile time (the
// BASELINE shapes): the residual's column loop and the substitution loops
// unroll, and the lane's row of the LU factor is loaded up front -- the
// serial shuffle chain then waits for no memory (it waited for one dependent
// global load per step: 2 nh round trips per cell).  Same operations in the
// same order as the generic instantiation (bit-identical).
template <int N_T, int M_T>
__global__ void __launch_bounds__(kT)
pmg_high_packed_kernel(int nwork, int N_rt, int m_rt, const int* __restrict__ wi_ptr,
                       const int* __restrict__ wi_blk, const int* __restrict__ wi_lcol,
                       const int* __restrict__ wi_cell, const int* __restrict__ wi_lrow,
                       const int64_t* __restrict__ wi_xlo,
                       const int* __restrict__ wi_hidx,
                       const int64_t* __restrict__ wi_out,
                       const double* __restrict__ val_t,
                       const double* __restrict__ HLU, const int* __restrict__ hperm,
                       const double* __restrict__ b, const double* __restrict__ xlo_buf,
                       double* __restrict__ out_buf) {
  constexpr bool FIX = N_T > 0;
  const int N = FIX ? N_T : N_rt;
  const int m = FIX ? M_T : m_rt;
  const int nh = N - m;
  constexpr int NH_T = FIX ? N_T - M_T : 1;
  const int cpw = 32 / nh;
  const int lane = threadIdx.x & 31;
  const int grp = lane / nh;
  const int i = lane - grp * nh;
  const int base = grp * nh;
  const bool lane_ok = grp < cpw;
  const int warps = (gridDim.x * kT) >> 5;
  for (int wb = ((blockIdx.x * kT + threadIdx.x) >> 5) * cpw; wb < nwork;
       wb += warps * cpw) {
    const int w = wb + grp;
    const bool active = lane_ok && w < nwork;
    int e0 = 0, e1 = 0;
    const double* xlo = xlo_buf;
    int c = 0, hi = 0;
    if (active) {
      e0 = wi_ptr[w];
      e1 = wi_ptr[w + 1];
      xlo = xlo_buf + wi_xlo[w];
      c = wi_cell[w];
      hi = wi_hidx[w];
    }
    const double* F = HLU + (int64_t)hi * nh * nh;
    double frow[NH_T];  // F[j * nh + i], j = 0 .. nh-1: this lane's row of the LU
    double bi = 0.0;
    int pi = i;
    if (FIX && active) {
#pragma unroll
      for (int j = 0; j < NH_T; ++j) frow[j] = __ldg(F + j * NH_T + i);
      bi = b[(int64_t)c * N + m + i];
      pi = hperm[(int64_t)hi * nh + i];
    }
    const int cnt = __reduce_max_sync(0xffffffffu, e1 - e0);
    double acc = 0.0;
    for (int t = 0; t < cnt; ++t) {
      const int e = e0 + t;
      if (active && e < e1) {
        const int64_t k = wi_blk[e];
        const double* v = val_t + k * N * N + m + i;
        const double* xq = xlo + (int64_t)wi_lcol[e] * m;
        if (FIX) {
          double vv[M_T > 0 ? M_T : 1], xx[M_T > 0 ? M_T : 1];
#pragma unroll
          for (int q = 0; q < M_T; ++q) {
            vv[q] = __ldg(v + q * N_T);
            xx[q] = __ldg(xq + q);
          }
#pragma unroll
          for (int q = 0; q < M_T; ++q) acc = __dadd_rn(acc, __dmul_rn(vv[q], xx[q]));
        } else {
          for (int q = 0; q < m; ++q)
            acc = __dadd_rn(acc, __dmul_rn(__ldg(v + q * N), __ldg(xq + q)));
        }
      }
    }
    double r = 0.0;
    if (active) {
      if (!FIX) {
        bi = b[(int64_t)c * N + m + i];
        pi = hperm[(int64_t)hi * nh + i];
      }
      r = __dadd_rn(bi, -acc);
    }
    double t = __shfl_sync(0xffffffffu, r, base + pi);
    if (FIX) {
#pragma unroll
      for (int j = 0; j < NH_T; ++j) {  // unit lower, column-oriented
        const double yj = __shfl_sync(0xffffffffu, t, base + j);
        if (active && i > j) t = __dadd_rn(t, -__dmul_rn(yj, frow[j]));
      }
#pragma unroll
      for (int j = NH_T - 1; j >= 0; --j) {  // upper, column-oriented
        if (active && i == j) t = __ddiv_rn(t, frow[j]);
        const double xj = __shfl_sync(0xffffffffu, t, base + j);
        if (active && i < j) t = __dadd_rn(t, -__dmul_rn(xj, frow[j]));
      }
    } else {
      for (int j = 0; j < nh; ++j) {  // unit lower, column-oriented
        const double yj = __shfl_sync(0xffffffffu, t, base + j);
        if (active && i > j) t = __dadd_rn(t, -__dmul_rn(yj, F[(int64_t)j * nh + i]));
      }
      for (int j = nh - 1; j >= 0; --j) {  // upper, column-oriented
        if (active && i == j) t = __ddiv_rn(t, F[(int64_t)j * nh + j]);
        const double xj = __shfl_sync(0xffffffffu, t, base + j);
        if (active && i < j) t = __dadd_rn(t, -__dmul_rn(xj, F[(int64_t)j * nh + i]));
      }
    }
    if (active) {
      double* o = out_buf + wi_out[w];
      const double* self = xlo + (int64_t)wi_lrow[w] * m;
      for (int q = i; q < m; q += nh) o[q] = self[q];
      o[m + i] = t;
    }
  }
}

__global__ void __launch_bounds__(kT)
combine_kernel(int nbr, int N, const int* __restrict__ cptr,
               const int64_t* __restrict__ cpos, const double* __restrict__ out,
               const double* __restrict__ damping, double* __restrict__ z) {
  const int64_t total = (int64_t)nbr * N;
  for (int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * kT) {
    const int bi = (int)(t / N);
    const int i = (int)(t - (int64_t)bi * N);
    double s = 0.0;
    for (int e = cptr[bi]; e < cptr[bi + 1]; ++e) s = __dadd_rn(s, out[cpos[e] + i]);
    z[t] = damping ? __ddiv_rn(s, damping[t]) : s;
  }
}

// Systems q of a size bucket on grid x, element ranges on grid y:
// packed[q] (P x P) <-> the system's n x n row-major matrix at
// flat + off[sys[q]].  Pack writes the identity in the padding (rows /
// columns n..P-1).  32-bit index math (P * P < 2^31).
__global__ void __launch_bounds__(kT)
pack_square_kernel(int64_t nsys, const int64_t* __restrict__ sys,
                   const int* __restrict__ dims, const int64_t* __restrict__ off, int P,
                   double* __restrict__ packed, double* __restrict__ flat, int unpack) {
  for (int64_t q = blockIdx.x; q < nsys; q += gridDim.x) {
    const int64_t sq = sys[q];
    const int n = dims[sq];
    double* src = flat + off[sq];
    double* dst = packed + q * (int64_t)P * P;
    const int64_t cnt = unpack ? (int64_t)n * n : (int64_t)P * P;
    const int w = unpack ? n : P;
    // 64-bit loop counter (the stride may step past INT_MAX near the end);
    // i, j stay 32-bit (k < P * P < 2^31 inside the loop)
    for (int64_t k = (int64_t)blockIdx.y * kT + threadIdx.x; k < cnt;
         k += (int64_t)kT * gridDim.y) {
      const int kk = (int)k;
      const int i = kk / w, j = kk - i * w;
      if (unpack)
        src[kk] = dst[i * P + j];
      else
        dst[kk] = (i < n && j < n) ? src[i * n + j] : (i == j ? 1.0 : 0.0);
    }
  }
}

}  // namespace
}  // namespace xdg

using namespace xdg;

extern "C" int xdg_pmg_build_low(int nwork, int N, int m, const int* wi_ptr,
                                 const int* wi_blk, const int* wi_lcol,
                                 const int* wi_lrow, const int* wi_sys,
                                 const int64_t* lu_off, const int* dims,
                                 const double* val_t, double* A,
                                 xdg_stream_t stream) {
  XDG_REQUIRE(N >= 1 && m >= 1 && m <= N, XDG_ERR_ARG, "bad N=%d m=%d", N, m);
  if (nwork <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  build_low_kernel<<<grid_for((int64_t)nwork * 32, kT, 8), kT, 0, s>>>(
      nwork, N, m, wi_ptr, wi_blk, wi_lcol, wi_lrow, wi_sys, lu_off, dims,
      val_t, A);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_pmg_gather_high(int ncells, int N, int m, const int* cells,
                                   const int* diag_blk, const double* val_t,
                                   double* H, xdg_stream_t stream) {
  XDG_REQUIRE(m < N, XDG_ERR_ARG, "no high-order modes (m=%d, N=%d)", m, N);
  if (ncells <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t total = (int64_t)ncells * (N - m) * (N - m);
  gather_high_kernel<<<grid_for(total, kT, 8), kT, 0, s>>>(ncells, N, m, cells,
                                                           diag_blk, val_t, H);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_pmg_high(int nwork, int N, int m, const int* wi_ptr,
                            const int* wi_blk, const int* wi_lcol,
                            const int* wi_cell, const int* wi_lrow,
                            const int64_t* wi_xlo, const int* wi_hidx,
                            const int64_t* wi_out, const double* val_t,
                            const double* HLU, const int* hperm,
                            const double* b, const double* xlo, double* out,
                            xdg_stream_t stream) {
  const int nh = N - m;
  XDG_REQUIRE(nh >= 1 && nh <= 64, XDG_ERR_UNSUPPORTED,
              "high-order block size %d outside [1, 64]", nh);
  if (nwork <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (nh <= 16) {
    const int cpw = 32 / nh;
    const int64_t warps = ((int64_t)nwork + cpw - 1) / cpw;
#define XDG_PACKED(NN, MM)                                                              \
  if (N == NN && m == MM) {                                                             \
    const int g = resident_grid(pmg_high_packed_kernel<NN, MM>, kT, 0, warps * 32);     \
    pmg_high_packed_kernel<NN, MM><<<g, kT, 0, s>>>(nwork, N, m, wi_ptr, wi_blk,        \
                                                    wi_lcol, wi_cell, wi_lrow, wi_xlo,  \
                                                    wi_hidx, wi_out, val_t, HLU, hperm, \
                                                    b, xlo, out);                       \
    XDG_CHECK_LAUNCH();                                                                 \
    return XDG_OK;                                                                      \
  }
    // (N, m) of the BASELINE configs: 3D p=3 k_lo=2 / 1, p=2 k_lo=1, p=1 k_lo=0... and 2D p=2
    XDG_PACKED(20, 10) XDG_PACKED(20, 4) XDG_PACKED(10, 4) XDG_PACKED(10, 1)
    XDG_PACKED(6, 3) XDG_PACKED(6, 1) XDG_PACKED(4, 1) XDG_PACKED(35, 20)
#undef XDG_PACKED
    const int g = resident_grid(pmg_high_packed_kernel<0, 0>, kT, 0, warps * 32);
    pmg_high_packed_kernel<0, 0><<<g, kT, 0, s>>>(nwork, N, m, wi_ptr, wi_blk, wi_lcol,
                                                  wi_cell, wi_lrow, wi_xlo, wi_hidx,
                                                  wi_out, val_t, HLU, hperm, b, xlo, out);
    XDG_CHECK_LAUNCH();
    return XDG_OK;
  }
  const int grid = grid_for((int64_t)nwork * 32, kT, 8);
  if (nh <= 32)
    pmg_high_kernel<1><<<grid, kT, 0, s>>>(nwork, N, m, wi_ptr, wi_blk, wi_lcol,
                                           wi_cell, wi_lrow, wi_xlo, wi_hidx,
                                           wi_out, val_t, HLU, hperm, b, xlo, out);
  else
    pmg_high_kernel<2><<<grid, kT, 0, s>>>(nwork, N, m, wi_ptr, wi_blk, wi_lcol,
                                           wi_cell, wi_lrow, wi_xlo, wi_hidx,
                                           wi_out, val_t, HLU, hperm, b, xlo, out);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_pmg_combine(int nbr, int N, const int* cptr,
                               const int64_t* cpos, const double* out,
                               const double* damping, double* z,
                               xdg_stream_t stream) {
  if (nbr <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  combine_kernel<<<grid_for((int64_t)nbr * N, kT, 8), kT, 0, s>>>(
      nbr, N, cptr, cpos, out, damping, z);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_pack_square(int64_t nsys, const int64_t* sys, const int* dims,
                               const int64_t* off, int P, double* packed, double* flat,
                               int unpack, xdg_stream_t stream) {
  XDG_REQUIRE(P >= 1, XDG_ERR_ARG, "bad pad size P=%d", P);
  if (nsys <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  XDG_REQUIRE((int64_t)P * P < (1LL << 31), XDG_ERR_ARG, "pad size P=%d too large", P);
  // about 8 elements per thread, at most 65535 parts per system
  const int64_t parts = std::min<int64_t>(65535, ((int64_t)P * P + 8 * kT - 1) / (8 * kT));
  const int64_t gx = std::min<int64_t>(nsys, std::max<int64_t>(1, 8 * sm_count() / parts));
  pack_square_kernel<<<dim3((unsigned)gx, (unsigned)parts), kT, 0, s>>>(nsys, sys, dims, off,
                                                                      P, packed, flat, unpack);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}
