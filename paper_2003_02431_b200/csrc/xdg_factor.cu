// Batched partial-pivoting LU with triangular inverses (sm_100a).
//
// Replaces the reference's factorizations on the solver path:
//   * `_PmgFactors.__init__` (cutdg solvers.py:191-243): SuperLU `splu` of
//     the low-order system (blockmatrix.py:203-216) and the per-cell
//     `scipy.linalg.lu_factor(diag[N_lo:, N_lo:])` (solvers.py:225-243);
//   * `direct_factor` (blockmatrix.py:203-216) of the coarsest level;
//   * the fronts of the multifrontal factorization (multifrontal.py) that
//     replaces SuperLU for the large systems: a front of n = P + B unknowns
//     eliminates only its first P columns (pivots among its first P rows);
//     afterwards the trailing B x B block holds the Schur complement
//     F_BB - L_BP U_PB, rows P.. of the first P columns hold L_BP = F_BP U^-1
//     and rows ..P of the last B columns U_PB = L^-1 P F_PB.
//
// One call factors a batch of row-major matrices of any sizes (matrix b at
// A + off[b], leading dimension ld[b], n[b] x n[b], p[b] <= n[b] columns
// eliminated), right-looking, blocked by NB columns:
//   panel   one thread-block CLUSTER per matrix holds the (n - k0) x NB panel
//           in distributed shared memory (rows split over the C CTAs of the
//           cluster); per column: CTA-local arg-max, cluster barrier, the
//           global pivot from the C candidates (DSMEM reads), row exchange
//           between the owning CTAs, scale + rank-1 update of the local rows
//           -- two cluster barriers per column, no global-memory round trips.
//           Full rows are swapped (LAPACK getrf semantics: the swaps reach
//           the L columns left of the panel and the trailing columns).
//   trsm    U12 = L11^-1 A12 (thread per column, L11 in shared memory).
//   update  A22 -= L21 U12, 64 x 64 tiles, K = NB, 4 x 4 FP64 per thread
//           (FP64 is vector-pipe work on B200; tcgen05 has no f64 kind).
// With `invert`, the top-left p x p LU is then overwritten by its
// triangular inverses in the layout the solve kernels read
// (xdg_lu_inv_apply: L^-1 strictly below the diagonal, unit diagonal
// implicit; U^-1 on and above it), blocked the same way:
//   diag    every NB x NB diagonal block of L and U inverted in shared memory;
//   sweep   block column j of U^-1: T = triu(X11) U12, X12 = -T X_jj;
//           block row i of L^-1:    T = L21 tril1(X11), X21 = -X_ii T.
// The permutation is returned directly (perm[i] = original row now at
// position i, the form xdg_lu_inv_apply / pmg_high consume), and info[b] =
// first column whose pivot is zero or not finite (+1), 0 if none.
#include <cooperative_groups.h>

#include <algorithm>

#include "xdg_common.cuh"

namespace cg = cooperative_groups;

namespace xdg {
namespace {

constexpr int kPT = 256;       // panel CTA threads
constexpr int kTile = 64;      // update tile edge
constexpr int kKc = 16;        // K chunk of the update tile
constexpr int kMaxCluster = 16;

struct Mat {
  double* a;
  int n, p, ld;
};

__device__ __forceinline__ Mat mat_of(double* A, const int64_t* off, const int* n,
                                      const int* p, const int* ld, int b) {
  Mat m;
  m.a = A + off[b];
  m.n = n[b];
  m.p = p[b];
  m.ld = ld[b];
  return m;
}

// ---------------------------------------------------------------------------
// panel: cluster of C CTAs per matrix; CTA r of the cluster owns panel rows
// [k0 + r*rpc, k0 + (r+1)*rpc) in its shared memory (stride nb+1 doubles:
// conflict-free column walks).
__global__ void __launch_bounds__(kPT)
lu_panel_kernel(int64_t nmat, double* __restrict__ A, const int64_t* __restrict__ off,
                const int* __restrict__ dn, const int* __restrict__ dp,
                const int* __restrict__ dld, int* __restrict__ perm,
                const int64_t* __restrict__ perm_off, int* __restrict__ info, int k0,
                int NB, int rpc) {
  extern __shared__ double smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int crank = (int)cluster.block_rank();
  const int64_t b = blockIdx.x / C;
  if (b >= nmat) return;  // whole clusters only (grid = nmat * C)
  const Mat M = mat_of(A, off, dn, dp, dld, (int)b);
  const int S = NB + 1;
  double* pan = smem;                       // rpc x S
  double* prow = pan + (size_t)rpc * S;     // pivot row (NB)
  double* xrow = prow + NB;                 // row received in an exchange (NB)
  double* cval = xrow + NB;                 // [0] candidate |value|
  int* cidx = reinterpret_cast<int*>(cval + 1);  // [0] candidate row, [1] pivot
  __shared__ double wv[kPT / 32];
  __shared__ int wi[kPT / 32];
  const int tid = threadIdx.x;
  const bool active = k0 < M.p;
  const int kb = active ? min(NB, M.p - k0) : 0;
  const int r0 = k0 + crank * rpc;                 // first global row of this CTA
  const int nloc = active ? max(0, min(rpc, M.n - r0)) : 0;
  int* pm = perm + perm_off[b];
  // load the panel rows (columns k0 .. k0+kb-1)
  for (int e = tid; e < nloc * kb; e += kPT) {
    const int r = e / kb, c = e - r * kb;
    pan[r * S + c] = M.a[(int64_t)(r0 + r) * M.ld + k0 + c];
  }
  if (active && k0 == 0 && crank == 0)
    for (int i = tid; i < M.p; i += kPT) pm[i] = i;
  __syncthreads();
  int bad = 0;
  for (int jj = 0; jj < kb; ++jj) {
    const int j = k0 + jj;
    // 1. local arg-max of |a(i, j)| over rows i in [j, p) held here
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int r = tid; r < nloc; r += kPT) {
      const int gi = r0 + r;
      if (gi < j || gi >= M.p) continue;
      const double v = fabs(pan[r * S + jj]);
      if (v > best || (v == best && gi < bi)) {  // NaN never wins
        best = v;
        bi = gi;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if ((tid & 31) == 0) {
      wv[tid >> 5] = best;
      wi[tid >> 5] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < kPT / 32; ++w)
        if (wv[w] > best || (wv[w] == best && wi[w] < bi)) {
          best = wv[w];
          bi = wi[w];
        }
      cval[0] = best;
      cidx[0] = bi;
    }
    cluster.sync();  // (A) candidates visible cluster-wide
    // 2. global pivot from the C candidates (warp 0), broadcast in smem
    if (tid < 32) {
      double v = -1.0;
      int vi = 0x7fffffff;
      if (tid < C) {
        v = *cluster.map_shared_rank(cval, tid);
        vi = *cluster.map_shared_rank(cidx, tid);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, vi, o);
        if (ov > v || (ov == v && oi < vi)) {
          v = ov;
          vi = oi;
        }
      }
      if (tid == 0) cidx[1] = (v >= 0.0 && vi < M.p) ? vi : j;
    }
    __syncthreads();
    const int piv = cidx[1];
    const int own_j = (j - k0) / rpc, own_p = (piv - k0) / rpc;
    // 3. every CTA fetches the pivot row (old row piv) of the panel; the
    //    owner of row piv also fetches row j (the exchange partner)
    for (int c = tid; c < kb; c += kPT) {
      const double* src = cluster.map_shared_rank(pan, own_p) + (piv - k0 - own_p * rpc) * S;
      prow[c] = src[c];
      if (crank == own_p && piv != j) {
        const double* sj = cluster.map_shared_rank(pan, own_j) + (j - k0 - own_j * rpc) * S;
        xrow[c] = sj[c];
      }
    }
    cluster.sync();  // (B) all remote reads done before any row is rewritten
    if (piv != j) {
      if (crank == own_j)
        for (int c = tid; c < kb; c += kPT) pan[(j - r0) * S + c] = prow[c];
      if (crank == own_p)
        for (int c = tid; c < kb; c += kPT) pan[(piv - r0) * S + c] = xrow[c];
      // full-row swap outside the panel columns (ordered: a column is owned
      // by one thread for every swap of this launch)
      for (int c = crank * kPT + tid; c < M.n; c += C * kPT) {
        if (c >= k0 && c < k0 + kb) continue;
        double* ra = M.a + (int64_t)j * M.ld + c;
        double* rb = M.a + (int64_t)piv * M.ld + c;
        const double t = *ra;
        *ra = *rb;
        *rb = t;
      }
      if (crank == 0 && tid == 0) {
        const int t = pm[j];
        pm[j] = pm[piv];
        pm[piv] = t;
      }
    }
    __syncthreads();
    // 4. scale the column below the pivot, rank-1 update of the panel
    const double pv = prow[jj];
    if (pv == 0.0 || !isfinite(pv)) {
      bad = bad ? bad : j + 1;
      continue;  // LAPACK: no scaling on a zero pivot (column is zero)
    }
    const double rinv = 1.0 / pv;
    const int w = kb - jj - 1;
    const int rlo = max(0, j + 1 - r0);
    for (int r = rlo + tid; r < nloc; r += kPT) pan[r * S + jj] *= rinv;
    __syncthreads();
    if (w > 0) {
      const int cnt = (nloc - rlo) * w;
      for (int e = tid; e < cnt; e += kPT) {
        const int r = rlo + e / w, c = jj + 1 + e % w;
        pan[r * S + c] = __fma_rn(-pan[r * S + jj], prow[c], pan[r * S + c]);
      }
    }
    __syncthreads();
  }
  // write the panel back
  for (int e = tid; e < nloc * kb; e += kPT) {
    const int r = e / kb, c = e - r * kb;
    M.a[(int64_t)(r0 + r) * M.ld + k0 + c] = pan[r * S + c];
  }
  if (bad && crank == 0 && tid == 0 && info[b] == 0) info[b] = bad;
  cluster.sync();  // no CTA leaves while its shared memory may still be read
}

// U12 = L11^-1 A12: rows k0..k0+kb-1, columns k0+kb..n-1; grid (column
// chunks of kPT, matrices).
__global__ void __launch_bounds__(kPT)
lu_trsm_kernel(double* __restrict__ A, const int64_t* __restrict__ off,
               const int* __restrict__ dn, const int* __restrict__ dp,
               const int* __restrict__ dld, int k0, int NB) {
  extern __shared__ double L[];  // kb x kb
  const Mat M = mat_of(A, off, dn, dp, dld, blockIdx.y);
  if (k0 >= M.p) return;
  const int kb = min(NB, M.p - k0);
  const int c0 = k0 + kb + blockIdx.x * kPT;
  if (c0 >= M.n) return;
  for (int e = threadIdx.x; e < kb * kb; e += kPT)
    L[e] = M.a[(int64_t)(k0 + e / kb) * M.ld + k0 + e % kb];
  __syncthreads();
  const int c = c0 + threadIdx.x;
  if (c >= M.n) return;
  double x[64];
  double* col = M.a + (int64_t)k0 * M.ld + c;
#pragma unroll 4
  for (int i = 0; i < kb; ++i) {
    double s = col[(int64_t)i * M.ld];
    for (int t = 0; t < i; ++t) s = __fma_rn(-L[i * kb + t], x[t], s);
    x[i] = s;
    col[(int64_t)i * M.ld] = s;
  }
}

// 64 x 64 tile of C (+)= alpha * A B accumulated over K in chunks, 4 x 4
// per thread.  Loader callbacks give A(i, k) / B(k, j) (zero outside).
struct TileAcc {
  double c[4][4];
};

template <class FA, class FB>
__device__ __forceinline__ void tile_mma(TileAcc& acc, int K, FA fa, FB fb,
                                         double (*As)[kTile + 1], double (*Bs)[kTile + 1]) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc.c[i][j] = 0.0;
  for (int kc = 0; kc < K; kc += kKc) {
    // As[k][i] = A(i, kc + k), Bs[k][j] = B(kc + k, j)
    for (int e = threadIdx.x; e < kKc * kTile; e += 256) {
      const int i = e / kKc, k = e - i * kKc;  // k fastest: row-contiguous A reads
      As[k][i] = fa(i, kc + k);
      const int kk = e / kTile, j = e - kk * kTile;
      Bs[kk][j] = fb(kc + kk, j);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kKc; ++k) {
      double a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc.c[i][j] = __fma_rn(a[i], bb[j], acc.c[i][j]);
    }
    __syncthreads();
  }
}

// A22 -= L21 U12 over rows/columns k0+kb..n-1; grid (tiles, matrices).
__global__ void __launch_bounds__(256)
lu_update_kernel(double* __restrict__ A, const int64_t* __restrict__ off,
                 const int* __restrict__ dn, const int* __restrict__ dp,
                 const int* __restrict__ dld, int k0, int NB) {
  __shared__ double As[kKc][kTile + 1];
  __shared__ double Bs[kKc][kTile + 1];
  const Mat M = mat_of(A, off, dn, dp, dld, blockIdx.y);
  if (k0 >= M.p) return;
  const int kb = min(NB, M.p - k0);
  const int s = k0 + kb;
  const int m = M.n - s;
  if (m <= 0) return;
  const int nt = (m + kTile - 1) / kTile;
  if ((int)blockIdx.x >= nt * nt) return;
  const int ti = blockIdx.x / nt, tj = blockIdx.x - ti * nt;
  const int i0 = s + ti * kTile, j0 = s + tj * kTile;
  const double* a = M.a;
  const int ld = M.ld, n = M.n;
  TileAcc acc;
  tile_mma(
      acc, kb,
      [&](int i, int k) {
        return (i0 + i < n && k < kb) ? a[(int64_t)(i0 + i) * ld + k0 + k] : 0.0;
      },
      [&](int k, int j) {
        return (j0 + j < n && k < kb) ? a[(int64_t)(k0 + k) * ld + j0 + j] : 0.0;
      },
      As, Bs);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gi = i0 + ty * 4 + i;
    if (gi >= n) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gj = j0 + tx * 4 + j;
      if (gj < n) M.a[(int64_t)gi * ld + gj] -= acc.c[i][j];
    }
  }
}

// ---------------------------------------------------------------------------
// triangular inverses of the p x p LU (in place)

// Invert every NB x NB diagonal block: U_dd (upper, with diagonal) and the
// unit-lower L_dd; grid (diag blocks, matrices), 256 threads.
__global__ void __launch_bounds__(256)
trtri_diag_kernel(double* __restrict__ A, const int64_t* __restrict__ off,
                  const int* __restrict__ dn, const int* __restrict__ dp,
                  const int* __restrict__ dld, int NB) {
  extern __shared__ double sm[];
  const Mat M = mat_of(A, off, dn, dp, dld, blockIdx.y);
  const int d0 = blockIdx.x * NB;
  if (d0 >= M.p) return;
  const int kb = min(NB, M.p - d0);
  double* T = sm;             // the block, kb x kb
  double* X = sm + kb * kb;   // its inverse parts
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x)
    T[e] = M.a[(int64_t)(d0 + e / kb) * M.ld + d0 + e % kb];
  __syncthreads();
  // U^-1 column by column: x_jj = 1/u_jj, x_ij = -(sum_{k=i}^{j-1} x_ik u_kj) x_jj
  // L^-1 row by row:       x_ij = -(l_ij + sum_{k=j+1}^{i-1} l_ik x_kj), i > j
  for (int t = 0; t < kb; ++t) {
    // U column t (threads i < t), diag by thread t
    for (int i = threadIdx.x; i <= t; i += blockDim.x) {
      const double xjj = 1.0 / T[t * kb + t];
      if (i == t) {
        X[t * kb + t] = xjj;
      } else {
        double s = 0.0;
        for (int k = i; k < t; ++k) s = __fma_rn(X[i * kb + k], T[k * kb + t], s);
        X[i * kb + t] = -s * xjj;
      }
    }
    // L row t (threads j < t)
    for (int jx = threadIdx.x; jx < t; jx += blockDim.x) {
      double s = T[t * kb + jx];
      for (int k = jx + 1; k < t; ++k) s = __fma_rn(T[t * kb + k], X[k * kb + jx], s);
      X[t * kb + jx] = -s;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x)
    M.a[(int64_t)(d0 + e / kb) * M.ld + d0 + e % kb] = X[e];
}

// Block column j0 of U^-1 (z = 0) or block row j0 of L^-1 (z = 1), first
// half: T = triu(X[0:j0,0:j0]) U[0:j0, j0:j0+kb]   (z = 0, T: j0 x kb)
//       T = L[j0:j0+kb, 0:j0] tril1(X[0:j0,0:j0])   (z = 1, T: kb x j0)
// into the workspace (matrix b, sweep z at W + (2b + z) * wstride, row-major,
// kb-wide / j0-wide).
// grid (64-row (z=0) / 64-column (z=1) tiles, matrices, 2).
__global__ void __launch_bounds__(256)
trtri_sweep_t_kernel(double* __restrict__ A, const int64_t* __restrict__ off,
                     const int* __restrict__ dn, const int* __restrict__ dp,
                     const int* __restrict__ dld, double* __restrict__ W,
                     int64_t wstride, int j0, int NB) {
  __shared__ double As[kKc][kTile + 1];
  __shared__ double Bs[kKc][kTile + 1];
  const Mat M = mat_of(A, off, dn, dp, dld, blockIdx.y);
  if (j0 >= M.p) return;
  const int kb = min(NB, M.p - j0);
  const double* a = M.a;
  const int ld = M.ld;
  double* T = W + (2 * (int64_t)blockIdx.y + blockIdx.z) * wstride;
  const int t0 = blockIdx.x * kTile;
  if (t0 >= j0) return;
  TileAcc acc;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  if (blockIdx.z == 0) {
    // rows t0.., K runs over k in [t0, j0) with k >= i (upper triangle)
    const int K = j0 - t0;
    tile_mma(
        acc, K,
        [&](int i, int k) {
          const int gi = t0 + i, gk = t0 + k;
          return (gi < j0 && gk < j0 && gk >= gi) ? a[(int64_t)gi * ld + gk] : 0.0;
        },
        [&](int k, int jx) {
          const int gk = t0 + k;
          return (gk < j0 && jx < kb) ? a[(int64_t)gk * ld + j0 + jx] : 0.0;
        },
        As, Bs);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int gi = t0 + ty * 4 + i;
      if (gi >= j0) continue;
#pragma unroll
      for (int jx = 0; jx < 4; ++jx) {
        const int c = tx * 4 + jx;
        if (c < kb) T[(int64_t)gi * kb + c] = acc.c[i][jx];
      }
    }
  } else {
    // columns t0.., K over k in [t0, j0) with k >= column (unit lower X)
    const int K = j0 - t0;
    tile_mma(
        acc, K,
        [&](int i, int k) {
          const int gk = t0 + k;
          return (i < kb && gk < j0) ? a[(int64_t)(j0 + i) * ld + gk] : 0.0;
        },
        [&](int k, int jx) {
          const int gk = t0 + k, gc = t0 + jx;
          if (gk >= j0 || gc >= j0 || gk < gc) return 0.0;
          return gk == gc ? 1.0 : a[(int64_t)gk * ld + gc];
        },
        As, Bs);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = ty * 4 + i;
      if (r >= kb) continue;
#pragma unroll
      for (int jx = 0; jx < 4; ++jx) {
        const int gc = t0 + tx * 4 + jx;
        if (gc < j0) T[(int64_t)r * j0 + gc] = acc.c[i][jx];
      }
    }
  }
}

// Second half: X[0:j0, j0:j0+kb] = -T X_jj   (z = 0)
//              X[j0:j0+kb, 0:j0] = -X_jj T   (z = 1)
// grid (64-row / 64-column tiles, matrices, 2).
__global__ void __launch_bounds__(256)
trtri_sweep_x_kernel(double* __restrict__ A, const int64_t* __restrict__ off,
                     const int* __restrict__ dn, const int* __restrict__ dp,
                     const int* __restrict__ dld, const double* __restrict__ W,
                     int64_t wstride, int j0, int NB) {
  __shared__ double As[kKc][kTile + 1];
  __shared__ double Bs[kKc][kTile + 1];
  const Mat M = mat_of(A, off, dn, dp, dld, blockIdx.y);
  if (j0 >= M.p) return;
  const int kb = min(NB, M.p - j0);
  const int t0 = blockIdx.x * kTile;
  if (t0 >= j0) return;
  const double* a = M.a;
  const int ld = M.ld;
  const double* T = W + (2 * (int64_t)blockIdx.y + blockIdx.z) * wstride;
  TileAcc acc;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  if (blockIdx.z == 0) {
    tile_mma(
        acc, kb,
        [&](int i, int k) {
          const int gi = t0 + i;
          return (gi < j0 && k < kb) ? T[(int64_t)gi * kb + k] : 0.0;
        },
        [&](int k, int jx) {  // X_jj upper (with diagonal)
          return (k < kb && jx < kb && k <= jx) ? a[(int64_t)(j0 + k) * ld + j0 + jx] : 0.0;
        },
        As, Bs);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int gi = t0 + ty * 4 + i;
      if (gi >= j0) continue;
#pragma unroll
      for (int jx = 0; jx < 4; ++jx) {
        const int c = tx * 4 + jx;
        if (c < kb) M.a[(int64_t)gi * ld + j0 + c] = -acc.c[i][jx];
      }
    }
  } else {
    tile_mma(
        acc, kb,
        [&](int i, int k) {  // X_jj unit lower
          if (i >= kb || k >= kb || k > i) return 0.0;
          return k == i ? 1.0 : a[(int64_t)(j0 + i) * ld + j0 + k];
        },
        [&](int k, int jx) {
          const int gc = t0 + jx;
          return (k < kb && gc < j0) ? T[(int64_t)k * j0 + gc] : 0.0;
        },
        As, Bs);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = ty * 4 + i;
      if (r >= kb) continue;
#pragma unroll
      for (int jx = 0; jx < 4; ++jx) {
        const int gc = t0 + tx * 4 + jx;
        if (gc < j0) M.a[(int64_t)(j0 + r) * ld + gc] = -acc.c[i][jx];
      }
    }
  }
}

int panel_nb(int max_n) {
  // NB x (max_n / 16 rows) must fit one CTA's shared memory
  if (max_n <= 6144) return 64;
  if (max_n <= 12288) return 32;
  if (max_n <= 24576) return 16;
  return 8;
}

constexpr size_t kSmemCap = 200 * 1024;

}  // namespace
}  // namespace xdg

using namespace xdg;

extern "C" int64_t xdg_batched_factor_ws_bytes(int64_t nmat, int max_p) {
  // per matrix: the U sweep's j0 x NB and the L sweep's NB x j0 temporaries
  // (j0 < max_p; NB as chosen for max_n >= max_p, at most panel_nb(max_p))
  const int NB = panel_nb(max_p);
  return 2 * nmat * (int64_t)std::max(max_p, 1) * NB * 8;
}

extern "C" int xdg_batched_factor(int64_t nmat, const int64_t* off, const int* n,
                                  const int* p, const int* ld, int max_n, int max_p,
                                  double* A, int* perm, const int64_t* perm_off, int* info,
                                  int invert, double* ws, xdg_stream_t stream) {
  if (nmat <= 0 || max_p <= 0) return XDG_OK;
  XDG_REQUIRE(max_p <= max_n && nmat < 65536, XDG_ERR_ARG,
              "bad batch: nmat=%lld max_n=%d max_p=%d (nmat < 65536 per call)",
              (long long)nmat, max_n, max_p);
  XDG_REQUIRE(!invert || ws != nullptr, XDG_ERR_ARG, "invert needs the workspace");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int NB = panel_nb(max_n);
  static bool attr_done = false;
  if (!attr_done) {
    XDG_TRY_CUDA(cudaFuncSetAttribute(lu_panel_kernel,
                                      cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    XDG_TRY_CUDA(cudaFuncSetAttribute(lu_panel_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kSmemCap + 4096));
    XDG_TRY_CUDA(cudaFuncSetAttribute(trtri_diag_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      2 * 64 * 64 * 8));
    attr_done = true;
  }
  XDG_TRY_CUDA(cudaMemsetAsync(info, 0, sizeof(int) * nmat, s));
  for (int k0 = 0; k0 < max_p; k0 += NB) {
    const int rows = max_n - k0;
    // smallest cluster whose row share fits the shared-memory budget
    int C = 1;
    auto need = [&](int c) {
      const int rpc = (rows + c - 1) / c;
      return (size_t)rpc * (NB + 1) * 8 + 2 * NB * 8 + 64;
    };
    while (C < kMaxCluster && need(C) > kSmemCap) C *= 2;
    XDG_REQUIRE(need(C) <= kSmemCap, XDG_ERR_ARG, "matrix too large (n=%d)", max_n);
    const int rpc = (rows + C - 1) / C;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nmat * C));
    cfg.blockDim = dim3(kPT);
    cfg.dynamicSmemBytes = need(C);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    XDG_TRY_CUDA(cudaLaunchKernelEx(&cfg, lu_panel_kernel, nmat, A, off, n, p, ld, perm,
                                    perm_off, info, k0, NB, rpc));
    const int right = max_n - k0 - 1;  // upper bound of columns right of the panel
    if (right > 0) {
      dim3 g1((unsigned)((right + kPT - 1) / kPT), (unsigned)nmat);
      lu_trsm_kernel<<<g1, kPT, NB * NB * 8, s>>>(A, off, n, p, ld, k0, NB);
      XDG_CHECK_LAUNCH();
      const int nt = (right + kTile - 1) / kTile;
      dim3 g2((unsigned)(nt * nt), (unsigned)nmat);
      lu_update_kernel<<<g2, 256, 0, s>>>(A, off, n, p, ld, k0, NB);
      XDG_CHECK_LAUNCH();
    }
  }
  if (!invert) return XDG_OK;
  const int nd = (max_p + NB - 1) / NB;
  trtri_diag_kernel<<<dim3((unsigned)nd, (unsigned)nmat), 256, 2 * NB * NB * 8, s>>>(
      A, off, n, p, ld, NB);
  XDG_CHECK_LAUNCH();
  const int64_t wstride = (int64_t)max_p * NB;
  for (int j0 = NB; j0 < max_p; j0 += NB) {
    dim3 g((unsigned)((j0 + kTile - 1) / kTile), (unsigned)nmat, 2);
    trtri_sweep_t_kernel<<<g, 256, 0, s>>>(A, off, n, p, ld, ws, wstride, j0, NB);
    XDG_CHECK_LAUNCH();
    trtri_sweep_x_kernel<<<g, 256, 0, s>>>(A, off, n, p, ld, ws, wstride, j0, NB);
    XDG_CHECK_LAUNCH();
  }
  return XDG_OK;
}
