// Block-sparse (uniform N x N blocks) FP64 matrix-vector product for sm_100a.
//
// Replaces cutdg BlockSparseMatrix.matvec (blockmatrix.py:119-125), which
// routes through a cached scipy CSR (blockmatrix.py:91-114) and scipy's
// single-threaded csr_matvec.
//
// Bound: HBM.  Algorithmic bytes per launch = 8 N^2 nnzb (blocks)
// + 4 nnzb (col) + 4 (nbr+1) (row_ptr) + 8 L (x) + 8 L (y) [+ 8 L for b].
//
// Mapping.  One thread owns one scalar row (block row bi, row i of the
// block).  Blocks are stored column-major (BSR-T), so for a fixed block k
// and column j the N threads of a block row read N consecutive doubles: a
// fully coalesced 8N-byte segment per (k, j).  Summation order per scalar
// row: blocks in column order, then columns j in order, with separately
// rounded mul and add -- exactly csr_matvec's order over tocsr(), which
// makes the product bit-identical to the reference.
//
//  * N <= 32: rows are packed warp-aligned (floor(32/N) block rows per
//    warp); lane i loads x[c*N+i] once and the block row's lanes exchange
//    the N values through shuffles instead of N redundant loads.
//  * N  > 32: flat thread-per-scalar-row mapping, x through L1 broadcast.
//
// Grid-stride persistent sizing: grid = min(work, 148 SMs x CTAs/SM).
#include "xdg_common.cuh"

namespace xdg {
namespace {

constexpr int kThreads = 256;

// Minimum resident CTAs per SM requested from ptxas for the warp-aligned
// kernel (0: no hint).  A hint lets ptxas keep a whole block column of
// loads in flight (measured with tools/tune_spmv.py; see profiles/).
#ifndef XDG_SPMV_MINB_SMALL
#define XDG_SPMV_MINB_SMALL 3  // N <= 12
#endif
#ifndef XDG_SPMV_MINB_LARGE
#define XDG_SPMV_MINB_LARGE 3  // N > 12
#endif
template <int N>
struct MinBlocks {
  static constexpr int v = N <= 12 ? XDG_SPMV_MINB_SMALL : XDG_SPMV_MINB_LARGE;
};
#define XDG_LB(N) __launch_bounds__(kThreads, MinBlocks<N>::v > 0 ? MinBlocks<N>::v : 1)
#define XDG_LB_HINTED(N) (MinBlocks<N>::v > 0)

enum EpiMode { EPI_PLAIN = 0, EPI_AXPBY = 1, EPI_RESID = 2 };

template <int MODE>
__device__ __forceinline__ double epilogue(double acc, int64_t gi,
                                           const double* __restrict__ b,
                                           const double* y, double alpha,
                                           double beta) {
  if (MODE == EPI_RESID) return __dadd_rn(b[gi], -acc);
  if (MODE == EPI_AXPBY) {
    double v = __dmul_rn(alpha, acc);
    if (beta != 0.0) v = __dadd_rn(v, __dmul_rn(beta, y[gi]));
    return v;
  }
  return acc;
}

// ---- N <= 32: warp-aligned block rows, x exchanged through shuffles -------
template <int N, int MODE, bool NORM>
__global__ void XDG_LB(N)
spmv_warp_rows(int row_begin, int row_end, const int* __restrict__ row_ptr,
               const int* __restrict__ col, const double* __restrict__ val,
               const double* __restrict__ x, double* y, double alpha,
               double beta, const double* __restrict__ b, double* norm_out,
               double* ws) {
  constexpr int RPW = 32 / N;  // block rows per warp
  const int lane = threadIdx.x & 31;
  const int r = lane / N;      // block row within the warp
  const int i = lane - r * N;  // row within the block
  const bool lane_ok = r < RPW;
  const int warps_total = (gridDim.x * kThreads) >> 5;
  const int nrows = row_end - row_begin;
  const int nwork = (nrows + RPW - 1) / RPW;
  double sq = 0.0;
  for (int w = (blockIdx.x * kThreads + threadIdx.x) >> 5; w < nwork;
       w += warps_total) {
    const int bi = row_begin + w * RPW + r;
    const bool active = lane_ok && (bi < row_end);
    int k0 = 0, k1 = 0;
    if (active) {
      k0 = __ldg(row_ptr + bi);
      k1 = __ldg(row_ptr + bi + 1);
    }
    // uniform trip count across the warp so the shuffles see every lane
    const int cnt = __reduce_max_sync(0xffffffffu, k1 - k0);
    double acc = 0.0;
    for (int t = 0; t < cnt; ++t) {
      const int k = k0 + t;
      const bool has = active && (k < k1);
      double xv = 0.0;
      const double* v = val;
      if (has) {
        const int c = __ldg(col + k);
        xv = __ldg(x + (int64_t)c * N + i);
        v = val + (int64_t)k * (N * N) + i;
      }
      double vv[N];
#pragma unroll
      for (int j = 0; j < N; ++j) vv[j] = has ? __ldg(v + j * N) : 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const double xj = __shfl_sync(0xffffffffu, xv, r * N + j);
        if (has) acc = __dadd_rn(acc, __dmul_rn(vv[j], xj));
      }
    }
    if (active) {
      const int64_t gi = (int64_t)bi * N + i;
      const double out = epilogue<MODE>(acc, gi, b, y, alpha, beta);
      y[gi] = out;
      if (NORM) sq += out * out;
    }
  }
  if (NORM) {
    __shared__ double red[kThreads / 32];
    const double s = block_sum(sq, red);
    grid_finalize(s, ws, norm_out);
  }
}

// ---- generic / large N: flat thread-per-scalar-row ------------------------
template <int N_T, int MODE, bool NORM>
__global__ void __launch_bounds__(kThreads)
spmv_flat(int row_begin, int row_end, int N_rt, const int* __restrict__ row_ptr,
          const int* __restrict__ col, const double* __restrict__ val,
          const double* __restrict__ x, double* y, double alpha, double beta,
          const double* __restrict__ b, double* norm_out, double* ws) {
  const int N = N_T > 0 ? N_T : N_rt;
  const int64_t nscalar = (int64_t)(row_end - row_begin) * N;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  double sq = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x; t < nscalar;
       t += stride) {
    const int bi = row_begin + (int)(t / N);
    const int i = (int)(t - (int64_t)(bi - row_begin) * N);
    const int k0 = __ldg(row_ptr + bi), k1 = __ldg(row_ptr + bi + 1);
    double acc = 0.0;
    for (int k = k0; k < k1; ++k) {
      const int c = __ldg(col + k);
      const double* v = val + (int64_t)k * N * N + i;
      const double* xc = x + (int64_t)c * N;
      if (N_T > 0) {
#pragma unroll 8
        for (int j = 0; j < N_T; ++j)
          acc = __dadd_rn(acc, __dmul_rn(__ldg(v + j * N_T), __ldg(xc + j)));
      } else {
        for (int j = 0; j < N; ++j)
          acc = __dadd_rn(acc, __dmul_rn(__ldg(v + j * N), __ldg(xc + j)));
      }
    }
    const int64_t gi = (int64_t)bi * N + i;
    const double out = epilogue<MODE>(acc, gi, b, y, alpha, beta);
    y[gi] = out;
    if (NORM) sq += out * out;
  }
  if (NORM) {
    __shared__ double red[kThreads / 32];
    const double s = block_sum(sq, red);
    grid_finalize(s, ws, norm_out);
  }
}

template <int N, int MODE, bool NORM>
cudaError_t launch_warp(int rb, int re, const int* rp, const int* col,
                        const double* val, const double* x, double* y,
                        double a, double bt, const double* b, double* nrm,
                        double* ws, cudaStream_t s) {
  constexpr int RPW = 32 / N;
  const int64_t warps = ((int64_t)(re - rb) + RPW - 1) / RPW;
  const int grid = resident_grid(spmv_warp_rows<N, MODE, NORM>, kThreads, 0,
                                 warps * 32);
  spmv_warp_rows<N, MODE, NORM>
      <<<grid, kThreads, 0, s>>>(rb, re, rp, col, val, x, y, a, bt, b, nrm, ws);
  return cudaGetLastError();
}

template <int NT, int MODE, bool NORM>
cudaError_t launch_flat(int rb, int re, int N, const int* rp, const int* col,
                        const double* val, const double* x, double* y,
                        double a, double bt, const double* b, double* nrm,
                        double* ws, cudaStream_t s) {
  const int grid = resident_grid(spmv_flat<NT, MODE, NORM>, kThreads, 0,
                                 (int64_t)(re - rb) * N);
  spmv_flat<NT, MODE, NORM><<<grid, kThreads, 0, s>>>(rb, re, N, rp, col, val,
                                                      x, y, a, bt, b, nrm, ws);
  return cudaGetLastError();
}

template <int MODE, bool NORM>
cudaError_t dispatch_n(int rb, int re, int N, const int* rp, const int* col,
                       const double* val, const double* x, double* y, double a,
                       double bt, const double* b, double* nrm, double* ws,
                       cudaStream_t s) {
#define XDG_W(NN) \
  case NN:        \
    return launch_warp<NN, MODE, NORM>(rb, re, rp, col, val, x, y, a, bt, b, nrm, ws, s);
#define XDG_F(NN) \
  case NN:        \
    return launch_flat<NN, MODE, NORM>(rb, re, N, rp, col, val, x, y, a, bt, b, nrm, ws, s);
#ifndef XDG_SPMV_FLAT20
#define XDG_SPMV_FLAT20 0
#endif
  switch (N) {
    XDG_W(1) XDG_W(2) XDG_W(3) XDG_W(4) XDG_W(6) XDG_W(10) XDG_W(15)
#if XDG_SPMV_FLAT20
    XDG_F(20)
#else
    XDG_W(20)
#endif
    XDG_W(21) XDG_W(28)
    XDG_F(35) XDG_F(56)
    default:
      if (N <= 32) break;
      return launch_flat<0, MODE, NORM>(rb, re, N, rp, col, val, x, y, a, bt,
                                        b, nrm, ws, s);
  }
#undef XDG_W
#undef XDG_F
  // remaining small N without a dedicated instantiation
  return launch_flat<0, MODE, NORM>(rb, re, N, rp, col, val, x, y, a, bt, b,
                                    nrm, ws, s);
}

}  // namespace
}  // namespace xdg

extern "C" int xdg_bsr_spmv(int row_begin, int row_end, int N,
                            const int* row_ptr, const int* col,
                            const double* val_t, const double* x, double* y,
                            double alpha, double beta, const double* b,
                            double* norm2_out, void* ws, xdg_stream_t stream) {
  using namespace xdg;
  XDG_REQUIRE(N >= 1, XDG_ERR_ARG, "block size N=%d must be >= 1", N);
  XDG_REQUIRE(row_begin >= 0 && row_end >= row_begin, XDG_ERR_ARG,
              "bad row range [%d,%d)", row_begin, row_end);
  XDG_REQUIRE(norm2_out == nullptr || ws != nullptr, XDG_ERR_ARG,
              "norm requested without workspace");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (row_end == row_begin) {
    if (norm2_out) XDG_TRY_CUDA(cudaMemsetAsync(norm2_out, 0, sizeof(double), s));
    return XDG_OK;
  }
  double* w = static_cast<double*>(ws);
  cudaError_t e;
  const bool nrm = norm2_out != nullptr;
  if (b != nullptr) {
    e = nrm ? dispatch_n<EPI_RESID, true>(row_begin, row_end, N, row_ptr, col, val_t, x, y, 1.0, 0.0, b, norm2_out, w, s)
            : dispatch_n<EPI_RESID, false>(row_begin, row_end, N, row_ptr, col, val_t, x, y, 1.0, 0.0, b, norm2_out, w, s);
  } else if (alpha == 1.0 && beta == 0.0) {
    e = nrm ? dispatch_n<EPI_PLAIN, true>(row_begin, row_end, N, row_ptr, col, val_t, x, y, 1.0, 0.0, b, norm2_out, w, s)
            : dispatch_n<EPI_PLAIN, false>(row_begin, row_end, N, row_ptr, col, val_t, x, y, 1.0, 0.0, b, norm2_out, w, s);
  } else {
    e = nrm ? dispatch_n<EPI_AXPBY, true>(row_begin, row_end, N, row_ptr, col, val_t, x, y, alpha, beta, b, norm2_out, w, s)
            : dispatch_n<EPI_AXPBY, false>(row_begin, row_end, N, row_ptr, col, val_t, x, y, alpha, beta, b, norm2_out, w, s);
  }
  XDG_TRY_CUDA(e);
  return XDG_OK;
}
