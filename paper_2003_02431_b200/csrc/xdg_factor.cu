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
// implicit; U^-1 on and above it): blocked TRSMs with the identity, block
// row by block row (GEMM with the rows already inverted, then substitution
// with the diagonal block), see trtri_gemm_kernel / trtri_solve_kernel.
// The permutation is returned directly (perm[i] = original row now at
// position i, the form xdg_lu_inv_apply / pmg_high consume), and info[b] =
// first column whose pivot is zero or not finite (+1), 0 if none.
#include <cooperative_groups.h>

#include <stdlib.h>

#include <algorithm>

#include "xdg_common.cuh"
#include "xdg_dmma.cuh"

namespace cg = cooperative_groups;

namespace xdg {
namespace {

constexpr int kPT = 256;       // panel CTA threads
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
                int NB, int rpc, int S) {
  extern __shared__ double smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int crank = (int)cluster.block_rank();
  const int64_t b = blockIdx.x / C;
  if (b >= nmat) return;  // whole clusters only (grid = nmat * C)
  const Mat M = mat_of(A, off, dn, dp, dld, (int)b);
  // S = widest panel of this launch + 1 (min(NB, max_p - k0) + 1: fronts of
  // 10-60 pivots leave room for several CTAs per SM)
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

// U12 = L11^-1 A12: rows k0..k0+kb-1, columns right of the panel inside
// [c_lo, c_hi); grid (column chunks of kPT, matrices).
__global__ void __launch_bounds__(kPT)
lu_trsm_kernel(double* __restrict__ A, const int64_t* __restrict__ off,
               const int* __restrict__ dn, const int* __restrict__ dp,
               const int* __restrict__ dld, int k0, int NB, int c_lo, int c_hi) {
  extern __shared__ double L[];  // kb x kb
  Mat M = mat_of(A, off, dn, dp, dld, blockIdx.y);
  if (k0 >= M.p) return;
  const int kb = min(NB, M.p - k0);
  // columns [max(k0 + kb, c_lo), min(c_hi, n))
  const int c0 = max(k0 + kb, c_lo) + blockIdx.x * kPT;
  M.n = min(M.n, c_hi);
  if (c0 >= M.n) return;
  for (int e = threadIdx.x; e < kb * kb; e += kPT)
    L[e] = M.a[(int64_t)(k0 + e / kb) * M.ld + k0 + e % kb];
  __syncthreads();
  const int c = c0 + threadIdx.x;
  if (c >= M.n) return;
  double x[64];
  double* col = M.a + (int64_t)k0 * M.ld + c;
  // the column's kb entries first (independent loads, all in flight), then
  // the substitution, then the stores
#pragma unroll 16
  for (int i = 0; i < kb; ++i) x[i] = col[(int64_t)i * M.ld];
  for (int i = 1; i < kb; ++i) {
    double s = x[i];
    for (int t = 0; t < i; ++t) s = __fma_rn(-L[i * kb + t], x[t], s);
    x[i] = s;
  }
#pragma unroll 16
  for (int i = 1; i < kb; ++i) col[(int64_t)i * M.ld] = x[i];
}

// A[r0:r1, c0:c1] -= A[r0:r1, q0:q1] A[q0:q1, c0:c1] inside every matrix of
// the batch (ranges clipped to the matrix: rows / columns to n, the K range
// to its eliminated columns p); grid (tiles, matrices).  The trailing update
// of the blocked LU (A22 -= L21 U12) and its deferred parts.
template <int BT>
__global__ void __launch_bounds__(256, BT >= 128 ? 1 : 2)
lu_update_kernel(double* __restrict__ A, const int64_t* __restrict__ off,
                 const int* __restrict__ dn, const int* __restrict__ dp,
                 const int* __restrict__ dld, int r0, int r1, int c0, int c1, int q0, int q1,
                 int ntc, int after_panel) {
  __shared__ DmmaSmem<BT, BT> sm;
  const Mat M = mat_of(A, off, dn, dp, dld, blockIdx.y);
  const int qe = min(q1, M.p), ce = min(c1, M.n);
  if (qe <= q0) return;
  // flags: 1 / 2 -- the row / column range starts right after this
  // matrix's own eliminated columns [q0, qe) (qe < q1 when its p falls
  // inside them); 4 -- the row range ends at this matrix's p
  if (after_panel & 1) r0 = qe;
  if (after_panel & 2) c0 = qe;
  const int re = min((after_panel & 4) ? min(r1, M.p) : r1, M.n);
  const int ti = blockIdx.x / ntc, tj = blockIdx.x - ti * ntc;
  const int i0 = r0 + ti * BT, j0 = c0 + tj * BT;
  if (i0 >= re || j0 >= ce) return;
  double* a = M.a;
  const int ld = M.ld;
  tile_dmma<BT, BT>(
      qe - q0,
      [&](int i, int k) {
        return (i0 + i < re && q0 + k < qe) ? a[(int64_t)(i0 + i) * ld + q0 + k] : 0.0;
      },
      [&](int k, int j) {
        return (j0 + j < ce && q0 + k < qe) ? a[(int64_t)(q0 + k) * ld + j0 + j] : 0.0;
      },
      [&](int i, int j, double v) {
        if (i0 + i < re && j0 + j < ce) a[(int64_t)(i0 + i) * ld + j0 + j] -= v;
      },
      sm);
}

// ---------------------------------------------------------------------------
// Triangular inverses of the p x p LU, in place, as blocked TRSMs with the
// identity (U X = I bottom-up, L X = I top-down: the right-residual method
// LAPACK's dtrtrs / scipy solve_triangular(U, I) use; multiplying by
// explicit inverses of the diagonal blocks instead loses up to two digits
// on the 1:1000 jump-coefficient systems, measured).  Step s handles block
// row i = nblk-1-s of U^-1 (z = 0) and block row i = s of L^-1 (z = 1):
//   gemm   R = E_i - U[i, i+1:] X[i+1:, :]   (z = 0, columns [i0, p))
//          R = E_i - L[i, :i] X[:i, :]       (z = 1, columns [0, i0 + kb))
//          into the workspace, with a copy of the diagonal block
//   solve  U_ii X_i = R by back substitution / L_ii X_i = R by forward
//          substitution, thread per column, written into the upper / strictly
//          lower part of block row i only.
// The U sweep reads and writes only on/above the diagonal, the L sweep only
// below it: both run in the same launches.  Workspace per (matrix, sweep):
// NB x p for R, then NB x NB for the diagonal block.

__device__ __forceinline__ double* trtri_ws(double* W, int64_t wstride, int b, int z) {
  return W + (2 * (int64_t)b + z) * wstride;
}

constexpr int kTN = 128;  // column tile of the trtri product

// grid (128-column tiles, matrices, 2); block rows of NB <= 64
__global__ void __launch_bounds__(256)
trtri_gemm_kernel(double* __restrict__ A, const int64_t* __restrict__ off,
                  const int* __restrict__ dn, const int* __restrict__ dp,
                  const int* __restrict__ dld, double* __restrict__ W, int64_t wstride,
                  int step, int NB) {
  __shared__ DmmaSmem<64, kTN> sm;
  const Mat M = mat_of(A, off, dn, dp, dld, blockIdx.y);
  const int nblk = (M.p + NB - 1) / NB;
  if (step >= nblk) return;
  const int z = blockIdx.z;
  const int i = z == 0 ? nblk - 1 - step : step;
  const int i0 = i * NB, kb = min(NB, M.p - i0);
  const int cbeg = z == 0 ? i0 : 0;
  const int cend = z == 0 ? M.p : i0 + kb;
  const int j0 = cbeg + blockIdx.x * kTN;
  if (j0 >= cend) return;
  const double* a = M.a;
  const int ld = M.ld, P = M.p;
  double* R = trtri_ws(W, wstride, blockIdx.y, z);
  double* Dg = R + (int64_t)NB * P;
  if (blockIdx.x == 0)  // original diagonal block for the solve step
    for (int e = threadIdx.x; e < kb * kb; e += 256)
      Dg[e] = a[(int64_t)(i0 + e / kb) * ld + i0 + e % kb];
  auto store = [&](int r, int c, double v) {
    const int gj = j0 + c;
    if (r < kb && gj < cend) R[(int64_t)r * P + gj] = (gj == i0 + r ? 1.0 : 0.0) - v;
  };
  if (z == 0) {
    // K over k in [i0 + kb, min(P, j0 + tile)): X[k][j] upper (k <= j)
    const int kbeg = i0 + kb, kend = min(P, j0 + kTN);
    tile_dmma<64, kTN>(
        max(0, kend - kbeg),
        [&](int r, int k) {
          const int gk = kbeg + k;
          return (r < kb && gk < kend) ? a[(int64_t)(i0 + r) * ld + gk] : 0.0;
        },
        [&](int k, int c) {
          const int gk = kbeg + k, gj = j0 + c;
          return (gk < kend && gj < cend && gk <= gj) ? a[(int64_t)gk * ld + gj] : 0.0;
        },
        store, sm);
  } else {
    // K over k in [j0, i0): X[k][j] unit lower (k > j stored, k == j -> 1)
    const int kbeg = j0, kend = i0;
    tile_dmma<64, kTN>(
        max(0, kend - kbeg),
        [&](int r, int k) {
          const int gk = kbeg + k;
          return (r < kb && gk < kend) ? a[(int64_t)(i0 + r) * ld + gk] : 0.0;
        },
        [&](int k, int c) {
          const int gk = kbeg + k, gj = j0 + c;
          if (gk >= kend || gj >= cend || gk < gj) return 0.0;
          return gk == gj ? 1.0 : a[(int64_t)gk * ld + gj];
        },
        store, sm);
  }
}

// grid (256-column chunks, matrices, 2)
__global__ void __launch_bounds__(256)
trtri_solve_kernel(double* __restrict__ A, const int64_t* __restrict__ off,
                   const int* __restrict__ dn, const int* __restrict__ dp,
                   const int* __restrict__ dld, const double* __restrict__ W,
                   int64_t wstride, int step, int NB) {
  __shared__ double D[64 * 65];
  const Mat M = mat_of(A, off, dn, dp, dld, blockIdx.y);
  const int nblk = (M.p + NB - 1) / NB;
  if (step >= nblk) return;
  const int z = blockIdx.z;
  const int i = z == 0 ? nblk - 1 - step : step;
  const int i0 = i * NB, kb = min(NB, M.p - i0);
  const int cbeg = z == 0 ? i0 : 0;
  const int cend = z == 0 ? M.p : i0 + kb;
  const int P = M.p;
  const double* R = trtri_ws(const_cast<double*>(W), wstride, blockIdx.y, z);
  const double* Dg = R + (int64_t)NB * P;
  if (cbeg + (int)blockIdx.x * 256 >= cend) return;
  for (int e = threadIdx.x; e < kb * kb; e += 256) D[(e / kb) * 65 + e % kb] = Dg[e];
  __syncthreads();
  const int j = cbeg + blockIdx.x * 256 + threadIdx.x;
  if (j >= cend) return;
  double x[64];
  if (z == 0) {  // back substitution, rows kb-1 .. 0
    const int rmax = j < i0 + kb ? j - i0 : kb - 1;  // X_ii upper: rows <= j - i0
#pragma unroll 16
    for (int r = 0; r < kb; ++r) x[r] = (r <= rmax) ? R[(int64_t)r * P + j] : 0.0;
    for (int r = rmax; r >= 0; --r) {
      double v = x[r];
      for (int c = r + 1; c <= rmax; ++c) v = __fma_rn(-D[r * 65 + c], x[c], v);
      x[r] = v / D[r * 65 + r];
    }
    for (int r = 0; r <= rmax; ++r) M.a[(int64_t)(i0 + r) * M.ld + j] = x[r];
  } else {  // forward substitution with the unit-lower L_ii
    // X_ii unit lower: column j - i0 of it starts at its unit diagonal
    // (R = 1 there), which takes part in the substitution but is not stored
    const int rlo = j >= i0 ? j - i0 : 0;
#pragma unroll 16
    for (int r = 0; r < kb; ++r) x[r] = (r >= rlo) ? R[(int64_t)r * P + j] : 0.0;
    for (int r = rlo + 1; r < kb; ++r) {
      double v = x[r];
      for (int c = rlo; c < r; ++c) v = __fma_rn(-D[r * 65 + c], x[c], v);
      x[r] = v;
    }
    for (int r = j >= i0 ? rlo + 1 : 0; r < kb; ++r) M.a[(int64_t)(i0 + r) * M.ld + j] = x[r];
  }
}

int panel_nb(int max_n) {
  // XDG_FACTOR_NB (8/16/32/64) overrides the panel width (experiments)
  static const int forced = [] {
    const char* e = getenv("XDG_FACTOR_NB");
    const int v = e ? atoi(e) : 0;
    return (v == 8 || v == 16 || v == 32 || v == 64) ? v : 0;
  }();
  // NB x (max_n / 16 rows) must fit one CTA's shared memory
  if (forced && (size_t)(max_n + 15) / 16 * (forced + 1) * 8 <= 200 * 1024) return forced;
  if (max_n <= 6144) return 64;
  if (max_n <= 12288) return 32;
  if (max_n <= 24576) return 16;
  return 8;
}

constexpr size_t kSmemCap = 200 * 1024;
constexpr int kTrtriNB = 64;  // block rows of the triangular inverses

// width of a super-panel: its inner panels (NB columns, bounded by the
// cluster's shared memory) update only the super-panel's own rows and
// columns; the rest of the trailing matrix gets one update with K = KB
int super_nb(int max_n, int NB) {
  static const int forced = [] {
    const char* e = getenv("XDG_FACTOR_KB");
    return e ? atoi(e) : 0;
  }();
  int kb = max_n > 1024 ? 256 : (max_n > 256 ? 128 : NB);
  if (forced >= NB && forced % NB == 0) kb = forced;
  return std::max(kb, NB);
}

}  // namespace
}  // namespace xdg

using namespace xdg;

extern "C" int64_t xdg_batched_factor_ws_bytes(int64_t nmat, int max_p) {
  // per matrix and sweep: NB x max_p (R) + NB x NB (diagonal block); NB as
  // chosen for max_n >= max_p is at most panel_nb(max_p)
  (void)panel_nb;
  const int NB = kTrtriNB;
  return 2 * nmat * ((int64_t)NB * std::max(max_p, 1) + (int64_t)NB * NB) * 8;
}

extern "C" int xdg_batched_factor(int64_t nmat, const int64_t* off, const int* n,
                                  const int* p, const int* ld, int max_n, int max_p,
                                  double* A, int* perm, const int64_t* perm_off, int* info,
                                  int invert, double* ws, xdg_stream_t stream) {
  if (nmat <= 0 || max_p <= 0) return XDG_OK;
  NvtxRange nv("xdg_batched_factor");
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
    attr_done = true;
  }
  XDG_TRY_CUDA(cudaMemsetAsync(info, 0, sizeof(int) * nmat, s));
  const int KB = super_nb(max_n, NB);
  auto update = [&](int r0, int r1, int c0, int c1, int q0, int q1, int flags) -> int {
    r1 = std::min(r1, max_n);
    c1 = std::min(c1, max_n);
    // tile counts for the widest per-matrix range (a range that starts
    // after a matrix's own panel starts at q0 + 1 at the earliest)
    const int nr = r1 - ((flags & 1) ? q0 + 1 : r0);
    const int nc = c1 - ((flags & 2) ? q0 + 1 : c0);
    if (nr <= 0 || nc <= 0 || q1 <= q0) return XDG_OK;
    if (std::max(nr, nc) > 256) {
      const int ntr = (nr + 127) / 128, ntc = (nc + 127) / 128;
      lu_update_kernel<128><<<dim3((unsigned)(ntr * ntc), (unsigned)nmat), 256, 0, s>>>(
          A, off, n, p, ld, r0, r1, c0, c1, q0, q1, ntc, flags);
    } else {
      const int ntr = (nr + 63) / 64, ntc = (nc + 63) / 64;
      lu_update_kernel<64><<<dim3((unsigned)(ntr * ntc), (unsigned)nmat), 256, 0, s>>>(
          A, off, n, p, ld, r0, r1, c0, c1, q0, q1, ntc, flags);
    }
    XDG_CHECK_LAUNCH();
    return XDG_OK;
  };
  auto trsm = [&](int k0, int c_lo, int c_hi) -> int {
    const int lo = std::max(k0 + 1, c_lo), hi = std::min(c_hi, max_n);
    if (hi <= lo) return XDG_OK;
    dim3 g1((unsigned)((hi - lo + kPT - 1) / kPT), (unsigned)nmat);
    lu_trsm_kernel<<<g1, kPT, NB * NB * 8, s>>>(A, off, n, p, ld, k0, NB, c_lo, c_hi);
    XDG_CHECK_LAUNCH();
    return XDG_OK;
  };
  // Two-level right-looking LU.  Inside a super-panel [K0, K1) the inner
  // panels (NB columns) update only the super-panel's columns; the columns
  // right of it see the row interchanges only (full-row swaps) until the
  // super-panel is done, then U12 = L11^-1 A12 block row by block row and one
  // trailing update with K = KB (LAPACK's getrf order: laswp, trsm, gemm).
  for (int K0 = 0; K0 < max_p; K0 += KB) {
    const int K1 = std::min(K0 + KB, max_n), Kp = std::min(K0 + KB, max_p);
    for (int k0 = K0; k0 < Kp; k0 += NB) {
      const int rows = max_n - k0;
      // smallest cluster whose row share fits the shared-memory budget
      int C = 1;
      const int S = (std::min(NB, max_p - k0) + 1) | 1;  // odd: conflict-free column walks
      auto need = [&](int c) {
        const int rpc = (rows + c - 1) / c;
        return (size_t)rpc * S * 8 + 2 * NB * 8 + 64;
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
                                      perm_off, info, k0, NB, rpc, S));
      // inside the super-panel: U12 and the update of its remaining columns
      XDG_TRY(trsm(k0, 0, K1));
      XDG_TRY(update(0, max_n, 0, K1, k0, k0 + NB, 1 | 2));
    }
    if (K1 < max_n) {
      // right of the super-panel: block rows of U12 in order, each after the
      // products with the block rows above it, then the deferred update
      for (int k0 = K0; k0 < Kp; k0 += NB) {
        if (k0 > K0) XDG_TRY(update(k0, k0 + NB, K1, max_n, K0, k0, 4));
        XDG_TRY(trsm(k0, K1, max_n));
      }
      XDG_TRY(update(0, max_n, K1, max_n, K0, K0 + KB, 1));
    }
  }
  if (!invert) return XDG_OK;
  // workspace per (matrix, sweep): NB x max_p for R + NB x NB diagonal block
  const int TB = kTrtriNB;
  const int64_t wstride = (int64_t)TB * max_p + (int64_t)TB * TB;
  const int nblk = (max_p + TB - 1) / TB;
  for (int st = 0; st < nblk; ++st) {
    dim3 g1((unsigned)((max_p + kTN - 1) / kTN), (unsigned)nmat, 2);
    trtri_gemm_kernel<<<g1, 256, 0, s>>>(A, off, n, p, ld, ws, wstride, st, TB);
    XDG_CHECK_LAUNCH();
    dim3 g2((unsigned)((max_p + 255) / 256), (unsigned)nmat, 2);
    trtri_solve_kernel<<<g2, 256, 0, s>>>(A, off, n, p, ld, ws, wstride, st, TB);
    XDG_CHECK_LAUNCH();
  }
  return XDG_OK;
}
