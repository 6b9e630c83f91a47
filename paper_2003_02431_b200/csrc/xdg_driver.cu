// Native solver driver: the control loops of the reference's residual
// minimisation (solvers.py:559-625), orthonormalization multigrid
// (solvers.py:669-749) and preconditioned GMRES (solvers.py:756-846), run
// in C++ over device-resident data.  Scalar decisions (dependent candidate,
// accept / reject, Givens rotations, convergence) stay on the host exactly
// as in the reference; every vector operation is a kernel of this library.
// Host syncs: one per rm_step (four scalars read back together), one per
// GMRES inner iteration (the Hessenberg column), one per multigrid
// iteration of the entry level is implied by the rm_step syncs.
//
// Fused kernels introduced here:
//   mgs_kernel        cooperative: all j+1 MGS steps of one GMRES iteration,
//                     one grid-wide sync per step (double-buffered partials),
//                     the axpy of step i fused with the dot of step i+1
//   rm_normalize      w /= ||w||, z /= ||w|| with ||w|| = sqrt(device dot)
//   rm_commit         y += alpha z ; x = x0 + y ; r = r0 - My_new
//   rm_restart        x0 += y ; r0 -= My ; y = My = 0 ; x = x0 ; r = r0
//   rm_current        x = x0 + y ; r = r0 - My
#include <cooperative_groups.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "xdg_common.cuh"

namespace cg = cooperative_groups;

namespace xdg {
namespace {

constexpr int kT = 256;
constexpr int kPerSm = 4;

__global__ void __launch_bounds__(kT)
rm_normalize_kernel(int64_t n, const double* __restrict__ nw2, double* w,
                    double* z) {
  const double d = sqrt(*nw2);
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride) {
    w[i] = __ddiv_rn(w[i], d);
    z[i] = __ddiv_rn(z[i], d);
  }
}

__global__ void __launch_bounds__(kT)
rm_commit_kernel(int64_t n, const double* __restrict__ alpha,
                 const double* __restrict__ z, double* __restrict__ y,
                 const double* __restrict__ x0, const double* __restrict__ r0,
                 const double* __restrict__ My_new, double* __restrict__ x,
                 double* __restrict__ r) {
  const double a = *alpha;
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride) {
    const double yi = __dadd_rn(y[i], __dmul_rn(a, z[i]));
    y[i] = yi;
    x[i] = __dadd_rn(x0[i], yi);
    r[i] = __dadd_rn(r0[i], -My_new[i]);
  }
}

__global__ void __launch_bounds__(kT)
rm_restart_kernel(int64_t n, double* __restrict__ x0, double* __restrict__ r0,
                  double* __restrict__ y, double* __restrict__ My,
                  double* __restrict__ x, double* __restrict__ r) {
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride) {
    const double xn = __dadd_rn(x0[i], y[i]);
    const double rn = __dadd_rn(r0[i], -My[i]);
    x0[i] = xn;
    r0[i] = rn;
    y[i] = 0.0;
    My[i] = 0.0;
    x[i] = xn;
    r[i] = rn;
  }
}

__global__ void __launch_bounds__(kT)
rm_current_kernel(int64_t n, const double* __restrict__ x0,
                  const double* __restrict__ y, const double* __restrict__ r0,
                  const double* __restrict__ My, double* __restrict__ x,
                  double* __restrict__ r) {
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride) {
    x[i] = __dadd_rn(x0[i], y[i]);
    r[i] = __dadd_rn(r0[i], -My[i]);
  }
}

// ---- fused modified Gram-Schmidt (cooperative) ----------------------------
__global__ void __launch_bounds__(kT)
mgs_kernel(int64_t n, int j, double* __restrict__ V, int64_t ldv,
           double* __restrict__ w, double* __restrict__ h,
           double* __restrict__ parts, const int* __restrict__ j_dev) {
  cg::grid_group grid = cg::this_grid();
  if (j_dev) j = *j_dev;  // graph-captured GMRES: the step index lives on the device
  __shared__ double red[kT / 32];
  const int G = gridDim.x;
  const int64_t stride = (int64_t)G * kT;
  const int64_t i0 = (int64_t)blockIdx.x * kT + threadIdx.x;
  // step 0 dot: V_0 . w
  double s = 0.0;
  for (int64_t e = i0; e < n; e += stride) s = fma(V[e], w[e], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) parts[blockIdx.x] = s;
  grid.sync();
  for (int i = 0; i <= j; ++i) {
    const double* P = parts + (int64_t)(i & 1) * G;
    double hi = 0.0;
    for (int g = 0; g < G; ++g) hi += P[g];  // same order in every CTA
    if (blockIdx.x == 0 && threadIdx.x == 0) h[i] = hi;
    const double* Vi = V + (int64_t)i * ldv;
    const double* Vn = V + (int64_t)(i + 1) * ldv;
    double t = 0.0;
    for (int64_t e = i0; e < n; e += stride) {
      const double we = __dadd_rn(w[e], -__dmul_rn(hi, Vi[e]));
      w[e] = we;
      t = (i < j) ? fma(Vn[e], we, t) : fma(we, we, t);
    }
    t = block_sum(t, red);
    if (threadIdx.x == 0) parts[(int64_t)((i + 1) & 1) * G + blockIdx.x] = t;
    grid.sync();
  }
  const double* P = parts + (int64_t)((j + 1) & 1) * G;
  double nrm2 = 0.0;
  for (int g = 0; g < G; ++g) nrm2 += P[g];
  const double hn = sqrt(nrm2);
  if (blockIdx.x == 0 && threadIdx.x == 0) h[j + 1] = hn;
  double* Vj1 = V + (int64_t)(j + 1) * ldv;
  for (int64_t e = i0; e < n; e += stride)
    Vj1[e] = hn > 0.0 ? __ddiv_rn(w[e], hn) : 0.0;
}

// Same steps, same arithmetic and order, with each thread's w and current
// basis column elements (at most K per thread) held in registers across the
// grid syncs: a step streams only V_{i+1} (the axpy's V_i is the previous
// step's V_{i+1}, w never leaves the SM) -- 1 instead of 3-4 vector passes
// per step, bit-identical to mgs_kernel on the same grid.
constexpr int kMgsK = 16;

__global__ void __launch_bounds__(kT, 2)
mgs_reg_kernel(int64_t n, int j, double* __restrict__ V, int64_t ldv,
               double* __restrict__ w, double* __restrict__ h,
               double* __restrict__ parts, const int* __restrict__ j_dev) {
  cg::grid_group grid = cg::this_grid();
  if (j_dev) j = *j_dev;
  __shared__ double red[kT / 32];
  const int G = gridDim.x;
  const int64_t stride = (int64_t)G * kT;
  const int64_t i0 = (int64_t)blockIdx.x * kT + threadIdx.x;
  double wr[kMgsK], vr[kMgsK];
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kMgsK; ++k) {
    const int64_t e = i0 + k * stride;
    wr[k] = vr[k] = 0.0;
    if (e < n) {
      wr[k] = w[e];
      vr[k] = V[e];
      s = fma(vr[k], wr[k], s);
    }
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) parts[blockIdx.x] = s;
  grid.sync();
  for (int i = 0; i <= j; ++i) {
    const double* P = parts + (int64_t)(i & 1) * G;
    double hi = 0.0;
    for (int g = 0; g < G; ++g) hi += P[g];  // same order in every CTA
    if (blockIdx.x == 0 && threadIdx.x == 0) h[i] = hi;
    const double* Vn = V + (int64_t)(i + 1) * ldv;
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < kMgsK; ++k) {
      const int64_t e = i0 + k * stride;
      if (e < n) {
        const double we = __dadd_rn(wr[k], -__dmul_rn(hi, vr[k]));
        wr[k] = we;
        if (i < j) {
          vr[k] = Vn[e];
          t = fma(vr[k], we, t);
        } else {
          t = fma(we, we, t);
        }
      }
    }
    t = block_sum(t, red);
    if (threadIdx.x == 0) parts[(int64_t)((i + 1) & 1) * G + blockIdx.x] = t;
    grid.sync();
  }
  const double* P = parts + (int64_t)((j + 1) & 1) * G;
  double nrm2 = 0.0;
  for (int g = 0; g < G; ++g) nrm2 += P[g];
  const double hn = sqrt(nrm2);
  if (blockIdx.x == 0 && threadIdx.x == 0) h[j + 1] = hn;
  double* Vj1 = V + (int64_t)(j + 1) * ldv;
#pragma unroll
  for (int k = 0; k < kMgsK; ++k) {
    const int64_t e = i0 + k * stride;
    if (e < n) {
      w[e] = wr[k];
      Vj1[e] = hn > 0.0 ? __ddiv_rn(wr[k], hn) : 0.0;
    }
  }
}

// ---------------------------------------------------------------------------
// host helpers

// Algorithmic bytes of every kernel the driver launches (minimal traffic of
// each op: SURVEY 8(d) formulas), accumulated per solve so a solve can
// report achieved bandwidth = bytes / time against the HBM roofline.
thread_local double g_bytes = 0.0;
inline void count(double b) { g_bytes += b; }
inline double spmv_bytes(const xdg_bsr* M, bool fused_b) {
  const double N = M->N;
  return 8.0 * N * N * M->nnzb + 4.0 * M->nnzb + 4.0 * (M->nbr + 1) +
         8.0 * N * (M->nbc + M->nbr) + (fused_b ? 8.0 * N * M->nbr : 0.0);
}

cudaError_t sync_read(double* host, const double* dev, int count, cudaStream_t s) {
  cudaError_t e = cudaMemcpyAsync(host, dev, sizeof(double) * count,
                                  cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

int spmv(const xdg_bsr* M, const double* x, double* y, const double* b,
         double* nrm, void* ws, cudaStream_t s) {
  count(spmv_bytes(M, b != nullptr));
  return xdg_bsr_spmv(0, M->nbr, M->N, M->row_ptr, M->col, M->val_t, x, y, 1.0,
                      0.0, b, nrm, ws, reinterpret_cast<xdg_stream_t>(s));
}

}  // namespace
}  // namespace xdg

using namespace xdg;

// ---------------------------------------------------------------------------
// The plan struct is operator-agnostic; the operator's blocks come in M.
static int pmg_apply_op(const xdg_pmg* P, const xdg_bsr* M, const double* b,
                        double* z, cudaStream_t s) {
  xdg_stream_t st = reinterpret_cast<xdg_stream_t>(s);
  count(P->apply_bytes);
  double* xlo = (P->direct && !P->has_high) ? z : P->xlo;
  if (P->mf)
    XDG_TRY(xdg_mf_solve(P->mf, b, xlo, st));
  else if (P->task_sys)
    XDG_TRY(xdg_lu_inv_apply_tasks(P->ntasks, P->task_sys, P->task_row0, P->rows_per_task,
                                   P->max_dim, P->total, P->lu_off, P->dims, P->vec_off,
                                   P->LU, P->src, b, xlo, P->scratch, st));
  else
    XDG_TRY(xdg_lu_inv_apply(P->nsys, P->total, P->row_sys, P->lu_off, P->dims,
                             P->vec_off, P->LU, P->src, b, xlo, P->scratch, st));
  if (P->has_high) {
    double* out = P->direct ? z : P->out;
    XDG_TRY(xdg_pmg_high(P->nwork, P->N, P->m, P->wi_ptr, P->wi_blk, P->wi_lcol,
                         P->wi_cell, P->wi_lrow, P->wi_xlo, P->wi_hidx,
                         P->wi_out, M->val_t, P->HLU, P->hperm, b, xlo, out, st));
  }
  if (!P->direct)
    XDG_TRY(xdg_pmg_combine(M->nbr, P->N, P->cptr, P->cpos, P->out, P->damping,
                            z, st));
  return XDG_OK;
}

extern "C" int xdg_pmg_apply_op(const xdg_pmg* P, const xdg_bsr* M,
                                const double* b, double* z,
                                xdg_stream_t stream) {
  NvtxRange nv("xdg_pmg_apply");
  return pmg_apply_op(P, M, b, z, reinterpret_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------------------
extern "C" int xdg_rm_current(xdg_rm* rm, xdg_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  count(48.0 * rm->n);
  rm_current_kernel<<<grid_for(rm->n, kT, kPerSm), kT, 0, s>>>(
      rm->n, rm->x0, rm->y, rm->r0, rm->My, rm->x, rm->r);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_rm_init(xdg_rm* rm, const double* x0, const double* r0,
                           xdg_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t bytes = sizeof(double) * rm->n;
  if (x0 != rm->x0) XDG_TRY_CUDA(cudaMemcpyAsync(rm->x0, x0, bytes, cudaMemcpyDeviceToDevice, s));
  if (r0 != rm->r0) XDG_TRY_CUDA(cudaMemcpyAsync(rm->r0, r0, bytes, cudaMemcpyDeviceToDevice, s));
  XDG_TRY_CUDA(cudaMemsetAsync(rm->y, 0, bytes, s));
  XDG_TRY_CUDA(cudaMemsetAsync(rm->My, 0, bytes, s));
  XDG_TRY(xdg_dot(rm->n, rm->r0, rm->r0, rm->sc + 7, rm->ws, stream));
  double v;
  XDG_TRY_CUDA(sync_read(&v, rm->sc + 7, 1, s));
  rm->best_norm = sqrt(v);
  rm->ncols = 0;
  rm->last_dependent = 0;
  rm->dependent_count = rm->rejected_count = rm->restart_count = 0;
  return XDG_OK;
}

static int rm_restart(xdg_rm* rm, cudaStream_t s) {
  // best_norm is unchanged: it already is || r0 - My || of the very vector
  // that becomes the new r0 (same kernel, same data -> same bits), which is
  // what solvers.py:554 recomputes.
  count(80.0 * rm->n);
  rm_restart_kernel<<<grid_for(rm->n, kT, kPerSm), kT, 0, s>>>(
      rm->n, rm->x0, rm->r0, rm->y, rm->My, rm->x, rm->r);
  XDG_CHECK_LAUNCH();
  rm->ncols = 0;
  rm->restart_count += 1;
  return XDG_OK;
}

extern "C" int xdg_rm_step(xdg_rm* rm, const xdg_bsr* M, const double* zc,
                           xdg_stream_t stream) {
  NvtxRange nv("xdg_rm_step");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t n = rm->n;
  if (rm->ncols >= rm->max_columns) XDG_TRY(rm_restart(rm, s));
  const int col = rm->ncols;
  double* z = rm->Z + (int64_t)col * n;  // candidate lives in its would-be column
  double* w = rm->W + (int64_t)col * n;
  if (zc != z) {
    count(16.0 * n);
    XDG_TRY_CUDA(cudaMemcpyAsync(z, zc, sizeof(double) * n,
                                 cudaMemcpyDeviceToDevice, s));
  }
  double* sc = rm->sc;
  XDG_TRY(spmv(M, z, w, nullptr, sc + 0, rm->ws, s));          // w = M z
  if (col > 0) {
    // two classical Gram-Schmidt passes (solvers.py:589-592).  The two z
    // updates are merged into z -= Z (c1 + c2): one pass over Z instead of
    // two (a roundoff-level reassociation of (z - Z c1) - Z c2); w is
    // updated exactly as in the reference.
    double* c1 = rm->coeff;
    double* c2 = rm->coeff + rm->max_columns;
    double* cs = rm->coeff + 2 * (int64_t)rm->max_columns;
    // W read 3x (two W^T w, one w-only update), W+Z once, vectors
    count(8.0 * col * n * 5 + 8.0 * n * 10);
    XDG_TRY(xdg_gemv_t(n, col, rm->W, n, w, c1, rm->gemv_ws, stream));
    XDG_TRY(xdg_gemv_update2(n, col, rm->W, nullptr, n, c1, nullptr, w, nullptr,
                             stream));
    XDG_TRY(xdg_gemv_t(n, col, rm->W, n, w, c2, rm->gemv_ws, stream));
    XDG_TRY(xdg_add_small(col, c1, c2, cs, stream));
    XDG_TRY(xdg_gemv_update2(n, col, rm->W, rm->Z, n, c2, cs, w, z, stream));
  }
  count(16.0 * n + 32.0 * n + 16.0 * n + 32.0 * n);  // dot, normalize, dot, update
  XDG_TRY(xdg_dot(n, w, w, sc + 1, rm->ws, stream));          // ||w||^2
  // speculative tail (discarded when the candidate is dependent)
  rm_normalize_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, sc + 1, w, z);
  XDG_CHECK_LAUNCH();
  XDG_TRY(xdg_dot(n, w, rm->r0, sc + 2, rm->ws, stream));     // alpha = w . r0
  XDG_TRY(spmv(M, z, rm->Mz, nullptr, nullptr, nullptr, s));  // exact image
  XDG_TRY(xdg_rm_update(n, rm->r0, rm->My, rm->Mz, sc + 2, rm->My_new, sc + 3,
                        rm->ws, stream));
  double h[4];
  XDG_TRY_CUDA(sync_read(h, sc, 4, s));
  const double scale = sqrt(h[0]), norm_w = sqrt(h[1]);
  if (scale == 0.0 || norm_w <= 1e-13 * scale) {               // solvers.py:594-599
    rm->last_dependent = 1;
    rm->dependent_count += 1;
    return xdg_rm_current(rm, stream);
  }
  const double alpha = h[2], rho = sqrt(h[3]);
  rm->last_dependent = 0;
  if (rho > rm->best_norm) {                                   // solvers.py:609-615
    rm->rejected_count += 1;
    return rm_restart(rm, s);
  }
  rm->alpha_host[col] = alpha;
  count(64.0 * n);
  rm_commit_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(
      n, sc + 2, z, rm->y, rm->x0, rm->r0, rm->My_new, rm->x, rm->r);
  XDG_CHECK_LAUNCH();
  double* t = rm->My;
  rm->My = rm->My_new;
  rm->My_new = t;
  rm->best_norm = rho;
  rm->ncols = col + 1;
  return XDG_OK;
}

// ---------------------------------------------------------------------------
// ortho_mg_solve

namespace {

struct OmgRun {
  xdg_omg_level* L;
  int nlevels, entry;
  double tol;
  int max_it, coarse_it;
  cudaStream_t s;
};

// Solves level `lam` (0-based) for rhs b_dev into x_dev.  Returns status;
// iterations / history only recorded for the entry level.
int omg_level(OmgRun& R, int lam, const double* b, double* x, int has_x0,
              int* iters, double* hist, int* hist_len, double* final_res) {
  xdg_omg_level& lv = R.L[lam];
  xdg_stream_t st = reinterpret_cast<xdg_stream_t>(R.s);
  xdg_rm& rm = lv.rm;
  const int64_t n = (int64_t)lv.M.nbr * lv.M.N;
  if (lam == R.nlevels - 1 || !lv.has_restriction) {           // solvers.py:698-710
    const xdg_direct& D = lv.direct;
    if (D.mf) {
      count(D.mf->apply_bytes);
      XDG_TRY(xdg_mf_solve(D.mf, b, x, st));
    } else {
      count(8.0 * D.n * (double)D.n + 32.0 * D.n);
      if (D.task_sys)
        XDG_TRY(xdg_lu_inv_apply_tasks(D.ntasks, D.task_sys, D.task_row0, D.rows_per_task,
                                       D.max_dim, D.n, D.zero_off, D.dims, D.zero_off, D.LU,
                                       D.perm, b, x, D.scratch, st));
      else
        XDG_TRY(xdg_lu_inv_apply(1, D.n, D.row_sys, D.zero_off, D.dims, D.zero_off,
                                 D.LU, D.perm, b, x, D.scratch, st));
    }
    if (lam == R.entry) {
      XDG_TRY(spmv(&lv.M, x, rm.r, b, rm.sc + 6, rm.ws, R.s));
      double v;
      XDG_TRY_CUDA(sync_read(&v, rm.sc + 6, 1, R.s));
      *final_res = sqrt(v);
      hist[0] = *final_res;
      *hist_len = 1;
      *iters = 0;
    }
    return XDG_OK;
  }
  if (!has_x0) XDG_TRY_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, R.s));
  // r = b - M x ; RmState(x, r)
  XDG_TRY(spmv(&lv.M, x, rm.r, b, nullptr, nullptr, R.s));
  XDG_TRY(xdg_rm_init(&rm, x, rm.r, st));
  double* H = (lam == R.entry) ? hist : nullptr;
  int hl = 0;
  double last = rm.best_norm;
  if (H) H[hl] = last;
  ++hl;
  const int budget = (lam == R.entry) ? R.max_it : R.coarse_it;
  int it = 0;
  xdg_omg_level& nx = R.L[lam + 1];
  while (last > R.tol && it < budget) {
    ++it;
    XDG_TRY(pmg_apply_op(&lv.schwarz, &lv.M, rm.r, lv.z, R.s));
    XDG_TRY(xdg_rm_step(&rm, &lv.M, lv.z, st));
    XDG_TRY(spmv(&lv.Rt, rm.r, nx.b, nullptr, nullptr, nullptr, R.s));  // r_c = R^T r
    XDG_TRY(omg_level(R, lam + 1, nx.b, nx.rm.x, 0, nullptr, nullptr, nullptr, nullptr));
    // the coarse solution sits in nx.rm.x (for the coarsest: written there)
    XDG_TRY(spmv(&lv.R, nx.rm.x, lv.xf, nullptr, nullptr, nullptr, R.s));
    XDG_TRY(xdg_rm_step(&rm, &lv.M, lv.xf, st));
    XDG_TRY(pmg_apply_op(&lv.schwarz, &lv.M, rm.r, lv.z, R.s));
    XDG_TRY(xdg_rm_step(&rm, &lv.M, lv.z, st));
    // ||r|| of the returned residual == best_norm (every rm_step exit leaves
    // r = r0 - My whose norm is best_norm)
    last = rm.best_norm;
    if (H) H[hl] = last;
    ++hl;
  }
  if (it > 0 && x != rm.x)
    XDG_TRY_CUDA(cudaMemcpyAsync(x, rm.x, sizeof(double) * n,
                                 cudaMemcpyDeviceToDevice, R.s));
  if (lam == R.entry) {
    *iters = it;
    *hist_len = hl;
    *final_res = last;
  }
  return XDG_OK;
}


}  // namespace

namespace xdg {
namespace omg_graph {

// ===========================================================================
// Graph-captured ortho_mg_solve: the whole Alg. 4 recursion as ONE CUDA graph
// with device-side control flow -- no host round trip per rm_step or
// iteration (the host-decision driver above reads 4 scalars back after every
// rm_step and one per level visit: ~11 blocking D2H reads per level-1
// iteration at cfg1).
//   * RmState scalars (column count, best norm, counters) live on the
//     device (RmDev); rm_step's three outcomes (solvers.py:594-615:
//     dependent -> current(), reject -> restart(), accept -> commit) are the
//     bodies of a SWITCH node whose value a 1-thread decision kernel sets;
//     the restart at a full space (solvers.py:574-575) is an IF node.
//   * Each level's iteration loop (solvers.py:719-738: `while ||r|| > tol
//     and it < budget`) is a WHILE node; the loop-end kernel appends the
//     history entry and re-evaluates the condition.  Coarse levels nest
//     their WHILE node inside the finer level's body.
//   * The candidate w of a step is built in a per-level scratch vector and
//     copied into its column on accept (the host driver builds it in the
//     column itself); My takes My_new's values on accept (the host driver
//     swaps the pointers).  Same kernels, same grids, same arithmetic: the
//     results are bit-identical to the host-decision driver
//     (tests/test_omg_graph_gpu.py).
//   * Algorithmic bytes: the decision kernels add each rm_step's bytes for
//     the path actually taken, the loop-end kernels each body's fixed bytes.

struct RmDev {
  double best_norm, last, bytes, pad0;
  int ncols, last_dependent, dependent_count, rejected_count, restart_count;
  int col, path, it, budget, ticket;
};

// ---- rm_step control without conditional nodes (XDG_OMG_FLAT) -------------
// The IF (restart when full) and SWITCH (accept / dependent / rejected) nodes
// of an rm_step become two ordinary kernels: every CTA takes the decision
// from the same device state (thread 0, broadcast through shared memory),
// does its slice of the chosen path, and the LAST CTA to finish (ticket
// counter) writes the state updates -- no CTA reads the state after it
// changed.  Same arithmetic as the conditional bodies (bit-identical); a
// kernel whose path has no vector work exits at once.
__device__ __forceinline__ bool last_cta(int* ticket) {
  __shared__ int is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int t = atomicAdd(ticket, 1);
    is_last = t == (int)gridDim.x - 1;
    if (is_last) *ticket = 0;
  }
  __syncthreads();
  return is_last != 0;
}

__global__ void __launch_bounds__(kT)
rm_flat_begin_kernel(int64_t n, RmDev* st, int max_columns, double restart_bytes,
                     double* gbytes, double* __restrict__ x0, double* __restrict__ r0,
                     double* __restrict__ y, double* __restrict__ My, double* __restrict__ x,
                     double* __restrict__ r) {
  __shared__ int full_s;
  if (threadIdx.x == 0) full_s = *(volatile int*)&st->ncols >= max_columns;
  __syncthreads();
  if (!full_s) return;  // uniform over the grid: nobody takes a ticket
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride) {
    const double xn = __dadd_rn(x0[i], y[i]);
    const double rn = __dadd_rn(r0[i], -My[i]);
    x0[i] = xn;
    r0[i] = rn;
    y[i] = 0.0;
    My[i] = 0.0;
    x[i] = xn;
    r[i] = rn;
  }
  if (last_cta(&st->ticket) && threadIdx.x == 0) {
    st->ncols = 0;
    st->restart_count += 1;
    *gbytes += restart_bytes;
  }
}

__global__ void __launch_bounds__(kT)
rm_flat_finish_kernel(int64_t n, RmDev* st, const double* sc, double* gbytes, double spmv2,
                      double cgs_per_col, double cgs_fixed, const double* __restrict__ z,
                      const double* __restrict__ w, double* __restrict__ y,
                      double* __restrict__ x0, double* __restrict__ r0,
                      const double* __restrict__ My_new, double* __restrict__ My,
                      double* __restrict__ x, double* __restrict__ r, double* __restrict__ Z,
                      double* __restrict__ W) {
  __shared__ int path_s, col_s;
  __shared__ double rho_s;
  if (threadIdx.x == 0) {  // rm_dev_decide_kernel's decision, state untouched
    const double scale = sqrt(sc[0]), norm_w = sqrt(sc[1]);
    int path;
    double rho = 0.0;
    if (scale == 0.0 || norm_w <= 1e-13 * scale) {
      path = 1;
    } else {
      rho = sqrt(sc[3]);
      path = rho > *(volatile double*)&st->best_norm ? 2 : 0;
    }
    path_s = path;
    col_s = *(volatile int*)&st->ncols;
    rho_s = rho;
  }
  __syncthreads();
  const int path = path_s;
  const int64_t col = col_s;
  const int64_t stride = (int64_t)gridDim.x * kT;
  const int64_t i0 = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (path == 0) {  // accept (rm_dev_commit_kernel)
    const double a = sc[2];
    double* Zc = Z + col * n;
    double* Wc = W + col * n;
    for (int64_t i = i0; i < n; i += stride) {
      const double zi = z[i];
      const double yi = __dadd_rn(y[i], __dmul_rn(a, zi));
      const double mn = My_new[i];
      y[i] = yi;
      x[i] = __dadd_rn(x0[i], yi);
      r[i] = __dadd_rn(r0[i], -mn);
      My[i] = mn;
      Zc[i] = zi;
      Wc[i] = w[i];
    }
  } else if (path == 1) {  // dependent (rm_current_kernel)
    for (int64_t i = i0; i < n; i += stride) {
      x[i] = __dadd_rn(x0[i], y[i]);
      r[i] = __dadd_rn(r0[i], -My[i]);
    }
  } else {  // rejected: restart (rm_dev_restart_kernel)
    for (int64_t i = i0; i < n; i += stride) {
      const double xn = __dadd_rn(x0[i], y[i]);
      const double rn = __dadd_rn(r0[i], -My[i]);
      x0[i] = xn;
      r0[i] = rn;
      y[i] = 0.0;
      My[i] = 0.0;
      x[i] = xn;
      r[i] = rn;
    }
  }
  if (last_cta(&st->ticket) && threadIdx.x == 0) {
    const double nn = (double)n;
    double bytes = spmv2 + 96.0 * nn + (col > 0 ? cgs_per_col * col + cgs_fixed : 0.0);
    if (path == 1) {
      st->last_dependent = 1;
      st->dependent_count += 1;
      bytes += 48.0 * nn;
    } else if (path == 2) {
      st->last_dependent = 0;
      st->rejected_count += 1;
      st->ncols = 0;
      st->restart_count += 1;
      bytes += 80.0 * nn;
    } else {
      st->last_dependent = 0;
      st->col = (int)col;
      st->ncols = (int)col + 1;
      st->best_norm = rho_s;
      bytes += 64.0 * nn;
    }
    st->path = path;
    *gbytes += bytes;
  }
}

bool omg_flat_enabled() {
  static const bool on = [] {
    const char* e = getenv("XDG_OMG_FLAT");
    return e != nullptr && atoi(e) != 0;
  }();
  return on;
}

__global__ void rm_dev_pre_kernel(RmDev* st, int max_columns, cudaGraphConditionalHandle h,
                                  double restart_bytes, double* gbytes) {
  const int full = st->ncols >= max_columns;
  if (full) *gbytes += restart_bytes;
  cudaGraphSetConditional(h, full);
}

__global__ void __launch_bounds__(kT)
rm_dev_restart_kernel(int64_t n, RmDev* st, double* __restrict__ x0, double* __restrict__ r0,
                      double* __restrict__ y, double* __restrict__ My, double* __restrict__ x,
                      double* __restrict__ r) {
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride) {
    const double xn = __dadd_rn(x0[i], y[i]);
    const double rn = __dadd_rn(r0[i], -My[i]);
    x0[i] = xn;
    r0[i] = rn;
    y[i] = 0.0;
    My[i] = 0.0;
    x[i] = xn;
    r[i] = rn;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->ncols = 0;
    st->restart_count += 1;
  }
}

// rm_step decision (solvers.py:594-615) on the device
__global__ void rm_dev_decide_kernel(RmDev* st, const double* sc, cudaGraphConditionalHandle h,
                                     double* gbytes, double n, double spmv2, double cgs_per_col,
                                     double cgs_fixed) {
  const int col = st->ncols;
  double bytes = spmv2 + 96.0 * n + (col > 0 ? cgs_per_col * col + cgs_fixed : 0.0);
  const double scale = sqrt(sc[0]), norm_w = sqrt(sc[1]);
  int path;
  if (scale == 0.0 || norm_w <= 1e-13 * scale) {
    st->last_dependent = 1;
    st->dependent_count += 1;
    path = 1;
    bytes += 48.0 * n;
  } else {
    const double rho = sqrt(sc[3]);
    st->last_dependent = 0;
    if (rho > st->best_norm) {
      st->rejected_count += 1;  // the restart body zeroes ncols, counts the restart
      path = 2;
      bytes += 80.0 * n;
    } else {
      st->col = col;
      st->ncols = col + 1;
      st->best_norm = rho;
      path = 0;
      bytes += 64.0 * n;
    }
  }
  st->path = path;
  *gbytes += bytes;
  cudaGraphSetConditional(h, (unsigned)path);
}

// accept: y += alpha z; x = x0 + y; r = r0 - My_new; My = My_new; the
// candidate (z, w) becomes column `col` of (Z, W)
__global__ void __launch_bounds__(kT)
rm_dev_commit_kernel(int64_t n, const RmDev* st, const double* __restrict__ alpha,
                     const double* __restrict__ z, const double* __restrict__ w,
                     double* __restrict__ y, const double* __restrict__ x0,
                     const double* __restrict__ r0, const double* __restrict__ My_new,
                     double* __restrict__ My, double* __restrict__ x, double* __restrict__ r,
                     double* __restrict__ Z, double* __restrict__ W) {
  const double a = *alpha;
  const int64_t col = st->col;
  double* Zc = Z + col * n;
  double* Wc = W + col * n;
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride) {
    const double zi = z[i];
    const double yi = __dadd_rn(y[i], __dmul_rn(a, zi));
    const double mn = My_new[i];
    y[i] = yi;
    x[i] = __dadd_rn(x0[i], yi);
    r[i] = __dadd_rn(r0[i], -mn);
    My[i] = mn;
    Zc[i] = zi;
    Wc[i] = w[i];
  }
}

__global__ void __launch_bounds__(kT)
copy_kernel(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride) b[i] = a[i];
}

__global__ void __launch_bounds__(kT)
zero2_kernel(int64_t n, double* __restrict__ a, double* __restrict__ b) {
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride) {
    a[i] = 0.0;
    if (b) b[i] = 0.0;
  }
}

// RmState(x, r) scalars + the level loop's first condition
__global__ void rm_dev_init_kernel(RmDev* st, const double* nr2, int budget, double tol,
                                   double* hist, cudaGraphConditionalHandle h) {
  const double bn = sqrt(*nr2);
  st->best_norm = bn;
  st->last = bn;
  st->ncols = st->last_dependent = st->dependent_count = 0;
  st->rejected_count = st->restart_count = 0;
  st->it = 0;
  st->budget = budget;
  if (hist) hist[0] = bn;
  cudaGraphSetConditional(h, (bn > tol && budget > 0) ? 1u : 0u);
}

__global__ void level_loop_end_kernel(RmDev* st, double tol, double* hist,
                                      cudaGraphConditionalHandle h, double* gbytes,
                                      double body_bytes) {
  const int it = st->it + 1;
  st->it = it;
  const double last = st->best_norm;
  st->last = last;
  if (hist) hist[it] = last;
  *gbytes += body_bytes;
  cudaGraphSetConditional(h, (last > tol && it < st->budget) ? 1u : 0u);
}

// x = rm.x when the loop ran at least once
__global__ void __launch_bounds__(kT)
copy_if_ran_kernel(int64_t n, const RmDev* st, const double* __restrict__ a,
                   double* __restrict__ b) {
  if (st->it <= 0) return;
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride) b[i] = a[i];
}

struct GraphOmg {
  xdg_omg_level* L;
  int nlevels, entry;
  double tol;
  int max_it, coarse_it;
  std::vector<cudaStream_t> streams;  // one capture stream per nesting depth
  RmDev* dev = nullptr;               // per level
  double* wc = nullptr;               // per level candidate-w scratch (offsets)
  std::vector<int64_t> wc_off;
  double* hist = nullptr;
  double* gbytes = nullptr;
  cudaGraph_t top = nullptr;
};

cudaStream_t cap_stream(GraphOmg& G, int depth) {
  while ((int)G.streams.size() <= depth) {
    cudaStream_t t;
    if (cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    G.streams.push_back(t);
  }
  return G.streams[depth];
}

// A conditional handle on the graph stream s is capturing into.
int make_handle(cudaStream_t s, cudaGraphConditionalHandle* h) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  XDG_TRY_CUDA(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, nullptr, nullptr));
  XDG_REQUIRE(cs == cudaStreamCaptureStatusActive, XDG_ERR_CUDA, "stream not capturing");
  XDG_TRY_CUDA(cudaGraphConditionalHandleCreate(h, g, 0, 0));
  return XDG_OK;
}

// Add a conditional node (handle h) at the capture frontier of stream s;
// returns its body graphs.
int add_cond_node(cudaStream_t s, cudaGraphConditionalHandle h,
                  cudaGraphConditionalNodeType type, int size, cudaGraph_t* bodies) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  XDG_TRY_CUDA(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &nd));
  XDG_REQUIRE(cs == cudaStreamCaptureStatusActive, XDG_ERR_CUDA, "stream not capturing");
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = type;
  p.conditional.size = size;
  cudaGraphNode_t node;
  XDG_TRY_CUDA(cudaGraphAddNode(&node, g, deps, nd, &p));
  for (int i = 0; i < size; ++i) bodies[i] = p.conditional.phGraph_out[i];
  XDG_TRY_CUDA(cudaStreamUpdateCaptureDependencies(s, &node, 1,
                                                   cudaStreamSetCaptureDependencies));
  return XDG_OK;
}

int begin_body(GraphOmg& G, int depth, cudaGraph_t body, cudaStream_t* out) {
  cudaStream_t t = cap_stream(G, depth);
  XDG_REQUIRE(t != nullptr, XDG_ERR_CUDA, "no capture stream");
  XDG_TRY_CUDA(cudaStreamBeginCaptureToGraph(t, body, nullptr, nullptr, 0,
                                             cudaStreamCaptureModeRelaxed));
  *out = t;
  return XDG_OK;
}

int end_body(cudaStream_t t) {
  cudaGraph_t g;
  XDG_TRY_CUDA(cudaStreamEndCapture(t, &g));
  return XDG_OK;
}

// One rm_step (solvers.py:559-625) of level lam on the candidate z (updated
// in place), captured on stream s at nesting depth `depth`.
int cap_rm_step(GraphOmg& G, int lam, double* z, cudaStream_t s, int depth) {
  xdg_omg_level& lv = G.L[lam];
  xdg_rm& rm = lv.rm;
  RmDev* st = G.dev + lam;
  const int64_t n = rm.n;
  const double saved = g_bytes;  // rm_step bytes are counted on the device
  double* w = G.wc + G.wc_off[lam];
  double* sc = rm.sc;
  const int mc = rm.max_columns;
  const xdg_stream_t xs = reinterpret_cast<xdg_stream_t>(s);
  const int* ncols = &st->ncols;
  // restart when the space is full (solvers.py:574-575)
  const bool flat = omg_flat_enabled();
  if (flat) {
    rm_flat_begin_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(
        n, st, mc, 80.0 * n, G.gbytes, rm.x0, rm.r0, rm.y, rm.My, rm.x, rm.r);
    XDG_CHECK_LAUNCH();
  } else {
    cudaGraphConditionalHandle h;
    XDG_TRY(make_handle(s, &h));
    rm_dev_pre_kernel<<<1, 1, 0, s>>>(st, mc, h, 80.0 * n, G.gbytes);
    XDG_CHECK_LAUNCH();
    cudaGraph_t body;
    XDG_TRY(add_cond_node(s, h, cudaGraphCondTypeIf, 1, &body));
    cudaStream_t t;
    XDG_TRY(begin_body(G, depth + 1, body, &t));
    rm_dev_restart_kernel<<<grid_for(n, kT, kPerSm), kT, 0, t>>>(n, st, rm.x0, rm.r0, rm.y,
                                                                  rm.My, rm.x, rm.r);
    XDG_CHECK_LAUNCH();
    XDG_TRY(end_body(t));
  }
  XDG_TRY(spmv(&lv.M, z, w, nullptr, sc + 0, rm.ws, s));           // w = M z
  // two classical Gram-Schmidt passes (solvers.py:589-592), columns on the
  // device (no-ops while the space is empty)
  double* c1 = rm.coeff;
  double* c2 = rm.coeff + mc;
  double* cs = rm.coeff + 2 * (int64_t)mc;
  XDG_TRY(gemv_t_dev(n, mc, ncols, rm.W, n, w, c1, rm.gemv_ws, s));
  XDG_TRY(gemv_update2_dev(n, mc, ncols, rm.W, nullptr, n, c1, nullptr, w, nullptr, s));
  XDG_TRY(gemv_t_dev(n, mc, ncols, rm.W, n, w, c2, rm.gemv_ws, s));
  XDG_TRY(add_small_dev(mc, ncols, c1, c2, cs, s));
  XDG_TRY(gemv_update2_dev(n, mc, ncols, rm.W, rm.Z, n, c2, cs, w, z, s));
  XDG_TRY(xdg_dot(n, w, w, sc + 1, rm.ws, xs));                     // ||w||^2
  rm_normalize_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, sc + 1, w, z);
  XDG_CHECK_LAUNCH();
  XDG_TRY(xdg_dot(n, w, rm.r0, sc + 2, rm.ws, xs));                 // alpha
  XDG_TRY(spmv(&lv.M, z, rm.Mz, nullptr, nullptr, nullptr, s));    // exact image
  XDG_TRY(xdg_rm_update(n, rm.r0, rm.My, rm.Mz, sc + 2, rm.My_new, sc + 3, rm.ws, xs));
  g_bytes = saved;
  if (flat) {
    const double sb = spmv_bytes(&lv.M, false);
    rm_flat_finish_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(
        n, st, sc, G.gbytes, 2.0 * sb, 8.0 * n * 5, 8.0 * n * 10, z, w, rm.y, rm.x0, rm.r0,
        rm.My_new, rm.My, rm.x, rm.r, rm.Z, rm.W);
    XDG_CHECK_LAUNCH();
  } else {
    cudaGraphConditionalHandle h;
    XDG_TRY(make_handle(s, &h));
    const double sb = spmv_bytes(&lv.M, false);
    rm_dev_decide_kernel<<<1, 1, 0, s>>>(st, sc, h, G.gbytes, (double)n, 2.0 * sb,
                                         8.0 * n * 5, 8.0 * n * 10);
    XDG_CHECK_LAUNCH();
    cudaGraph_t bodies[3];
    XDG_TRY(add_cond_node(s, h, cudaGraphCondTypeSwitch, 3, bodies));
    cudaStream_t t;
    XDG_TRY(begin_body(G, depth + 1, bodies[0], &t));             // accept
    rm_dev_commit_kernel<<<grid_for(n, kT, kPerSm), kT, 0, t>>>(
        n, st, sc + 2, z, w, rm.y, rm.x0, rm.r0, rm.My_new, rm.My, rm.x, rm.r, rm.Z, rm.W);
    XDG_CHECK_LAUNCH();
    XDG_TRY(end_body(t));
    XDG_TRY(begin_body(G, depth + 1, bodies[1], &t));             // dependent
    rm_current_kernel<<<grid_for(n, kT, kPerSm), kT, 0, t>>>(n, rm.x0, rm.y, rm.r0, rm.My,
                                                              rm.x, rm.r);
    XDG_CHECK_LAUNCH();
    XDG_TRY(end_body(t));
    XDG_TRY(begin_body(G, depth + 1, bodies[2], &t));             // rejected
    rm_dev_restart_kernel<<<grid_for(n, kT, kPerSm), kT, 0, t>>>(n, st, rm.x0, rm.r0, rm.y,
                                                                  rm.My, rm.x, rm.r);
    XDG_CHECK_LAUNCH();
    XDG_TRY(end_body(t));
  }
  return XDG_OK;
}

int cap_direct(xdg_omg_level& lv, const double* b, double* x, cudaStream_t s) {
  const xdg_direct& D = lv.direct;
  const xdg_stream_t st = reinterpret_cast<xdg_stream_t>(s);
  if (D.mf) {
    count(D.mf->apply_bytes);
    return xdg_mf_solve(D.mf, b, x, st);
  }
  count(8.0 * D.n * (double)D.n + 32.0 * D.n);
  if (D.task_sys)
    return xdg_lu_inv_apply_tasks(D.ntasks, D.task_sys, D.task_row0, D.rows_per_task,
                                  D.max_dim, D.n, D.zero_off, D.dims, D.zero_off, D.LU,
                                  D.perm, b, x, D.scratch, st);
  return xdg_lu_inv_apply(1, D.n, D.row_sys, D.zero_off, D.dims, D.zero_off, D.LU, D.perm, b,
                          x, D.scratch, st);
}

// Level lam (not the coarsest) solving for b into x (solvers.py:696-738),
// captured on s at depth `depth`.
int cap_level(GraphOmg& G, int lam, const double* b, double* x, int has_x0, cudaStream_t s,
              int depth) {
  xdg_omg_level& lv = G.L[lam];
  xdg_rm& rm = lv.rm;
  RmDev* st = G.dev + lam;
  const int64_t n = (int64_t)lv.M.nbr * lv.M.N;
  const bool entry = lam == G.entry;
  double* hist = entry ? G.hist : nullptr;
  if (!has_x0) {
    zero2_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, x, nullptr);
    XDG_CHECK_LAUNCH();
  }
  XDG_TRY(spmv(&lv.M, x, rm.r, b, nullptr, nullptr, s));          // r = b - M x
  // RmState(x, r)
  count(48.0 * n);
  copy_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, x, rm.x0);
  XDG_CHECK_LAUNCH();
  copy_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, rm.r, rm.r0);
  XDG_CHECK_LAUNCH();
  zero2_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, rm.y, rm.My);
  XDG_CHECK_LAUNCH();
  XDG_TRY(xdg_dot(n, rm.r0, rm.r0, rm.sc + 7, rm.ws, reinterpret_cast<xdg_stream_t>(s)));
  cudaGraphConditionalHandle h;
  XDG_TRY(make_handle(s, &h));
  rm_dev_init_kernel<<<1, 1, 0, s>>>(st, rm.sc + 7, entry ? G.max_it : G.coarse_it, G.tol,
                                     hist, h);
  XDG_CHECK_LAUNCH();
  cudaGraph_t body;
  XDG_TRY(add_cond_node(s, h, cudaGraphCondTypeWhile, 1, &body));
  cudaStream_t t;
  XDG_TRY(begin_body(G, depth + 1, body, &t));
  const double b0 = g_bytes;
  xdg_omg_level& nx = G.L[lam + 1];
  const bool coarsest_next = lam + 1 == G.nlevels - 1 || !nx.has_restriction;
  XDG_TRY(pmg_apply_op(&lv.schwarz, &lv.M, rm.r, lv.z, t));
  XDG_TRY(cap_rm_step(G, lam, lv.z, t, depth + 1));
  XDG_TRY(spmv(&lv.Rt, rm.r, nx.b, nullptr, nullptr, nullptr, t));  // r_c = R^T r
  if (coarsest_next)
    XDG_TRY(cap_direct(nx, nx.b, nx.rm.x, t));
  else
    XDG_TRY(cap_level(G, lam + 1, nx.b, nx.rm.x, 0, t, depth + 1));
  XDG_TRY(spmv(&lv.R, nx.rm.x, lv.xf, nullptr, nullptr, nullptr, t));
  XDG_TRY(cap_rm_step(G, lam, lv.xf, t, depth + 1));
  XDG_TRY(pmg_apply_op(&lv.schwarz, &lv.M, rm.r, lv.z, t));
  XDG_TRY(cap_rm_step(G, lam, lv.z, t, depth + 1));
  const double body_bytes = g_bytes - b0;
  g_bytes = b0;
  level_loop_end_kernel<<<1, 1, 0, t>>>(st, G.tol, hist, h, G.gbytes, body_bytes);
  XDG_CHECK_LAUNCH();
  XDG_TRY(end_body(t));
  if (x != rm.x) {
    copy_if_ran_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, st, rm.x, x);
    XDG_CHECK_LAUNCH();
  }
  return XDG_OK;
}

bool omg_graph_enabled() {
  static const bool on = [] {
    const char* e = getenv("XDG_OMG_GRAPH");
    return e == nullptr || atoi(e) != 0;
  }();
  return on;
}

// Whole solve as one graph launch.  Returns XDG_OK with the outputs filled.
int omg_solve_graph(xdg_omg_level* levels, int nlevels, int entry, double tolerance,
                    int max_iterations, int coarse_cycle_iterations, const double* b,
                    double* x, int has_x0, int* iterations, double* history, int* hist_len,
                    double* final_residual, cudaStream_t s) {
  GraphOmg G;
  G.L = levels;
  G.nlevels = nlevels;
  G.entry = entry;
  G.tol = tolerance;
  G.max_it = max_iterations;
  G.coarse_it = coarse_cycle_iterations;
  // device state: RmDev per level, candidate-w scratch per level, history,
  // byte counter
  int64_t tot = 0;
  G.wc_off.assign(nlevels, 0);
  for (int l = 0; l < nlevels; ++l) {
    G.wc_off[l] = tot;
    tot += (int64_t)levels[l].M.nbr * levels[l].M.N;
  }
  const size_t bytes_state = sizeof(RmDev) * nlevels;
  const size_t bytes_all = bytes_state + sizeof(double) * (tot + max_iterations + 2 + 1);
  char* buf = nullptr;
  XDG_TRY_CUDA(cudaMallocAsync(&buf, bytes_all, s));
  XDG_TRY_CUDA(cudaMemsetAsync(buf, 0, bytes_all, s));
  G.dev = reinterpret_cast<RmDev*>(buf);
  G.wc = reinterpret_cast<double*>(buf + bytes_state);
  G.hist = G.wc + tot;
  G.gbytes = G.hist + max_iterations + 2;
  cudaStream_t s0 = cap_stream(G, 0);
  int st = XDG_OK;
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  if (s0 == nullptr) {
    st = XDG_ERR_CUDA;
  } else {
    // the capture stream waits for the caller's stream (allocation, memset)
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(ev, s);
    cudaStreamWaitEvent(s0, ev, 0);
    cudaEventDestroy(ev);
    XDG_TRY_CUDA(cudaStreamBeginCapture(s0, cudaStreamCaptureModeRelaxed));
    st = cap_level(G, entry, b, x, has_x0, s0, 0);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(s0, &g);
    if (st == XDG_OK && e != cudaSuccess) {
      set_error("graph capture: %s", cudaGetErrorString(e));
      st = XDG_ERR_CUDA;
    }
    graph = g;
    if (st == XDG_OK) {
      e = cudaGraphInstantiate(&exec, graph, 0);
      if (e != cudaSuccess) {
        set_error("graph instantiate: %s", cudaGetErrorString(e));
        st = XDG_ERR_CUDA;
      }
    }
    if (st == XDG_OK) {
      e = cudaGraphLaunch(exec, s);
      if (e != cudaSuccess) {
        set_error("graph launch: %s", cudaGetErrorString(e));
        st = XDG_ERR_CUDA;
      }
    }
  }
  RmDev top;
  double dbytes = 0.0;
  if (st == XDG_OK) {
    cudaError_t e = cudaMemcpyAsync(&top, G.dev + entry, sizeof(RmDev), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&dbytes, G.gbytes, sizeof(double),
                                              cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) {
      *iterations = top.it;
      *hist_len = top.it + 1;
      e = cudaMemcpy(history, G.hist, sizeof(double) * (top.it + 1), cudaMemcpyDeviceToHost);
    }
    if (e != cudaSuccess) {
      set_error("graph readback: %s", cudaGetErrorString(e));
      st = XDG_ERR_CUDA;
    }
    *final_residual = top.last;
    // level state back into the host structs (counters the Python side reads)
    xdg_rm& rm = levels[entry].rm;
    rm.ncols = top.ncols;
    rm.best_norm = top.best_norm;
    rm.last_dependent = top.last_dependent;
    rm.dependent_count = top.dependent_count;
    rm.rejected_count = top.rejected_count;
    rm.restart_count = top.restart_count;
    g_bytes += dbytes;
  }
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  cudaFreeAsync(buf, s);
  for (cudaStream_t t : G.streams) cudaStreamDestroy(t);
  return st;
}

}  // namespace omg_graph
}  // namespace xdg

using xdg::omg_graph::omg_graph_enabled;
using xdg::omg_graph::omg_solve_graph;


extern "C" int xdg_omg_solve(xdg_omg_level* levels, int nlevels, int entry,
                             double tolerance, int max_iterations,
                             int coarse_cycle_iterations, const double* b,
                             double* x, int has_x0, int* iterations,
                             double* history, int* hist_len,
                             double* final_residual, double* bytes_out,
                             xdg_stream_t stream) {
  NvtxRange nv("xdg_omg_solve");
  g_bytes = 0.0;
  XDG_REQUIRE(nlevels >= 1 && entry >= 0 && entry < nlevels, XDG_ERR_ARG,
              "bad level range");
  OmgRun R{levels, nlevels, entry, tolerance, max_iterations,
           coarse_cycle_iterations, reinterpret_cast<cudaStream_t>(stream)};
  const bool coarsest = entry == nlevels - 1 || !levels[entry].has_restriction;
  // one CUDA graph with device-side control flow (XDG_OMG_GRAPH=0: the
  // host-decision driver, same arithmetic)
  int st = (omg_graph_enabled() && !coarsest)
               ? omg_solve_graph(levels, nlevels, entry, tolerance, max_iterations,
                                 coarse_cycle_iterations, b, x, has_x0, iterations, history,
                                 hist_len, final_residual, R.s)
               : omg_level(R, entry, b, x, has_x0, iterations, history, hist_len,
                           final_residual);
  if (st != XDG_OK) return st;
  XDG_TRY_CUDA(cudaStreamSynchronize(R.s));
  if (bytes_out) *bytes_out = g_bytes;
  return XDG_OK;
}

// ---------------------------------------------------------------------------
// GMRES

// One Givens step of restarted GMRES (solvers.py:808-823) on column j of
// the row-major (m+1) x m Hessenberg H: copy the MGS column hc, apply the
// previous rotations, form rotation j, update g; *est = |g[j+1]|.  Returns
// 1 on a zero rotation denominator (SingularSystemError, solvers.py:813-817).
// Host and device evaluate it with the same rounding (rmul/radd/rdiv).
__host__ __device__ inline int givens_step(double* H, int m, double* cs, double* sn,
                                           double* g, const double* hc, int j, double* est) {
#define HC(i, k) H[(size_t)(i) * m + (k)]
  for (int i = 0; i <= j + 1; ++i) HC(i, j) = hc[i];
  for (int i = 0; i < j; ++i) {
    const double hij = radd(rmul(cs[i], HC(i, j)), rmul(sn[i], HC(i + 1, j)));
    HC(i + 1, j) = radd(rmul(-sn[i], HC(i, j)), rmul(cs[i], HC(i + 1, j)));
    HC(i, j) = hij;
  }
  const double denom = xhypot(HC(j, j), HC(j + 1, j));
  if (denom == 0.0) return 1;
  cs[j] = rdiv(HC(j, j), denom);
  sn[j] = rdiv(HC(j + 1, j), denom);
  HC(j, j) = radd(rmul(cs[j], HC(j, j)), rmul(sn[j], HC(j + 1, j)));
  g[j + 1] = rmul(-sn[j], g[j]);
  g[j] = rmul(cs[j], g[j]);
  HC(j + 1, j) = 0.0;
  *est = fabs(g[j + 1]);
  return 0;
}

// y = -H[:j,:j]^-1 g[:j] (upper triangular back substitution, solvers.py:831;
// negated for x -= Z y with the w -= W c kernel)
__host__ __device__ inline void gmres_backsolve(const double* H, int m, const double* g, int j,
                                                double* y) {
  for (int i = j - 1; i >= 0; --i) {
    double t = g[i];
    for (int k = i + 1; k < j; ++k) t = radd(t, -rmul(HC(i, k), y[k]));
    y[i] = rdiv(t, HC(i, i));
  }
  for (int i = 0; i < j; ++i) y[i] = -y[i];
#undef HC
}

// MGS of GMRES step j (j_dev != NULL: read on the device, graph capture).
static int mgs_launch(int64_t n, int j, const int* j_dev, double* V, int64_t ldv, double* w,
                      double* h, void* ws, cudaStream_t s) {
  static thread_local int per_sm = 0;
  if (per_sm == 0) {
    XDG_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mgs_kernel,
                                                               kT, 0));
    if (per_sm < 1) per_sm = 1;
  }
  int64_t need = (n + kT - 1) / kT;
  int64_t cap = (int64_t)sm_count() * (per_sm < 2 ? per_sm : 2);
  int grid = (int)(need < cap ? (need < 1 ? 1 : need) : cap);
  // partials: 2 x grid doubles after the reduction counter slot
  double* parts = static_cast<double*>(ws) + 1;
  void* args[] = {&n, &j, &V, &ldv, &w, &h, &parts, const_cast<int**>(&j_dev)};
  // register-resident variant on the same grid when it fits (XDG_MGS_REG=0
  // forces the streaming kernel)
  static thread_local int reg_per_sm = -1;
  static const bool reg_ok = [] {
    const char* e = getenv("XDG_MGS_REG");
    return e == nullptr || atoi(e) != 0;
  }();
  if (reg_per_sm < 0 &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&reg_per_sm, mgs_reg_kernel, kT, 0) !=
          cudaSuccess)
    reg_per_sm = 0;
  const bool use_reg = reg_ok && n >= 32768 &&  // small n: grid-sync bound either way
                       (int64_t)grid <= (int64_t)sm_count() * reg_per_sm &&
                       n <= (int64_t)kMgsK * grid * kT;
  XDG_TRY_CUDA(cudaLaunchCooperativeKernel(
      use_reg ? (const void*)mgs_reg_kernel : (const void*)mgs_kernel, dim3(grid), dim3(kT),
      args, 0, s));
  return XDG_OK;
}

extern "C" int xdg_mgs(int64_t n, int j, double* V, int64_t ldv, double* w,
                       double* h, void* ws, xdg_stream_t stream) {
  return mgs_launch(n, j, nullptr, V, ldv, w, h, ws, reinterpret_cast<cudaStream_t>(stream));
}

namespace xdg {
namespace omg_graph {
bool gmres_graph_enabled();
int gmres_solve_graph(const xdg_bsr* M, const xdg_pmg* pmg, int m, double tol, int max_it,
                      const double* b, double* x, int has_x0, double* V, double* Zb, double* w,
                      double* r, double* sc, double* ycoef, void* ws, int* iterations,
                      double* history, int* hist_len, double* final_residual, cudaStream_t s);
}  // namespace omg_graph
}  // namespace xdg

extern "C" int xdg_gmres_solve(const xdg_bsr* M, const xdg_pmg* pmg,
                               int restart, double tolerance,
                               int max_iterations, const double* b, double* x,
                               int has_x0, double* V, double* Zb, double* w,
                               double* r, double* sc, double* ycoef, void* ws,
                               void* gemv_ws, int* iterations, double* history,
                               int* hist_len, double* final_residual,
                               double* bytes_out, xdg_stream_t stream) {
  NvtxRange nv("xdg_gmres_solve");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  g_bytes = 0.0;
  if (xdg::omg_graph::gmres_graph_enabled()) {  // one CUDA graph (XDG_GMRES_GRAPH=0: host loop)
    const int rc = xdg::omg_graph::gmres_solve_graph(
        M, pmg, restart, tolerance, max_iterations, b, x, has_x0, V, Zb, w, r, sc, ycoef, ws,
        iterations, history, hist_len, final_residual, s);
    if (bytes_out) *bytes_out = g_bytes;
    return rc;
  }
  const int m = restart;
  const int64_t n = (int64_t)M->nbr * M->N;
  (void)gemv_ws;
  if (!has_x0) XDG_TRY_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
  XDG_TRY(spmv(M, x, r, b, sc, ws, s));
  double v;
  XDG_TRY_CUDA(sync_read(&v, sc, 1, s));
  double beta = sqrt(v);
  int hl = 0, total = 0;
  history[hl++] = beta;
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), hc(m + 2),
      y(m);
  while (beta > tolerance && total < max_iterations) {
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(cs.begin(), cs.end(), 0.0);
    std::fill(sn.begin(), sn.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    count(16.0 * n);
    XDG_TRY(xdg_scale(n, beta, nullptr, 1, r, V, stream));      // V_0 = r / beta
    int j = 0;
    while (j < m && total < max_iterations) {
      ++total;
      double* Vj = V + (int64_t)j * n;
      double* Zj = Zb + (int64_t)j * n;
      XDG_TRY(pmg_apply_op(pmg, M, Vj, Zj, s));
      XDG_TRY(spmv(M, Zj, w, nullptr, nullptr, nullptr, s));
      // MGS of iteration j moves 8 n (2 (j + 1) + 3) bytes
      count(8.0 * n * (2.0 * (j + 1) + 3.0));
      XDG_TRY(xdg_mgs(n, j, V, n, w, sc, ws, stream));
      XDG_TRY_CUDA(sync_read(hc.data(), sc, j + 2, s));
      double est;
      if (givens_step(H.data(), m, cs.data(), sn.data(), g.data(), hc.data(), j, &est)) {
        set_error("preconditioned operator produced a zero column");
        return XDG_ERR_SINGULAR;
      }
      history[hl++] = est;
      ++j;
      if (est <= tolerance) break;
    }
    gmres_backsolve(H.data(), m, g.data(), j, y.data());       // y := -H^-1 g
    XDG_TRY_CUDA(cudaMemcpyAsync(ycoef, y.data(), sizeof(double) * j,
                                 cudaMemcpyHostToDevice, s));
    count(8.0 * j * n + 16.0 * n);
    XDG_TRY(xdg_gemv_update2(n, j, Zb, nullptr, n, ycoef, nullptr, x, nullptr,
                             stream));
    XDG_TRY(spmv(M, x, r, b, sc, ws, s));
    XDG_TRY_CUDA(sync_read(&v, sc, 1, s));
    beta = sqrt(v);
    history[hl - 1] = beta;
  }
  *iterations = total;
  *hist_len = hl;
  *final_residual = beta;
  if (bytes_out) *bytes_out = g_bytes;
  return XDG_OK;
}

// ===========================================================================
// Graph-captured gmres_pmg_solve (solvers.py:756-846): the restart cycles
// and the Arnoldi steps are nested WHILE nodes of one CUDA graph; the MGS
// step index, the Hessenberg column, the Givens rotations, the back
// substitution and the convergence tests live on the device (1-thread
// kernels evaluating givens_step / gmres_backsolve, the same functions and
// rounding as the host driver above: bit-identical results).  V_j and Z_j
// are addressed through device-indexed copies into fixed buffers.
namespace xdg {
namespace omg_graph {

struct GmDev {
  double beta, est;
  int j, total, hl, err;
};

__global__ void gm_init_kernel(GmDev* st, const double* nr2, double tol, int max_it,
                               double* hist, cudaGraphConditionalHandle h) {
  const double beta = sqrt(*nr2);
  st->beta = beta;
  st->est = beta;
  st->j = st->total = st->err = 0;
  st->hl = 1;
  hist[0] = beta;
  cudaGraphSetConditional(h, (beta > tol && max_it > 0) ? 1u : 0u);
}

__global__ void gm_cycle_init_kernel(GmDev* st, double* H, double* cs, double* sn, double* g,
                                     int m, cudaGraphConditionalHandle h) {
  for (int i = 0; i < (m + 1) * m; ++i) H[i] = 0.0;
  for (int i = 0; i < m; ++i) cs[i] = sn[i] = 0.0;
  for (int i = 0; i <= m; ++i) g[i] = 0.0;
  g[0] = st->beta;
  st->j = 0;
  cudaGraphSetConditional(h, m > 0 ? 1u : 0u);
}

__global__ void __launch_bounds__(kT)
gm_col_copy_kernel(int64_t n, const GmDev* st, const double* __restrict__ src, int64_t lds,
                   double* __restrict__ dst, int64_t ldd) {
  const int64_t j = st->j;
  const double* a = src + j * lds;
  double* b = dst + j * ldd;
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride) b[i] = a[i];
}

__global__ void gm_givens_kernel(GmDev* st, const double* hc, double* H, double* cs, double* sn,
                                 double* g, int m, double tol, int max_it, double* hist,
                                 cudaGraphConditionalHandle h, double* gbytes, double n,
                                 double fixed_bytes) {
  const int j = st->j;
  double est = 0.0;
  *gbytes += fixed_bytes + 8.0 * n * (2.0 * (j + 1) + 3.0);
  if (givens_step(H, m, cs, sn, g, hc, j, &est)) {
    st->err = 1;
    cudaGraphSetConditional(h, 0u);
    return;
  }
  st->est = est;
  hist[st->hl++] = est;
  st->total += 1;
  st->j = j + 1;
  cudaGraphSetConditional(h, (j + 1 < m && st->total < max_it && est > tol) ? 1u : 0u);
}

__global__ void gm_backsolve_kernel(const GmDev* st, const double* H, const double* g, int m,
                                    double* ycoef, double* gbytes, double n) {
  if (st->err) return;
  gmres_backsolve(H, m, g, st->j, ycoef);
  *gbytes += 8.0 * st->j * n + 16.0 * n;
}

__global__ void gm_cycle_end_kernel(GmDev* st, const double* nr2, double tol, int max_it,
                                    double* hist, cudaGraphConditionalHandle h) {
  if (st->err) {
    cudaGraphSetConditional(h, 0u);
    return;
  }
  const double beta = sqrt(*nr2);
  st->beta = beta;
  hist[st->hl - 1] = beta;
  cudaGraphSetConditional(h, (beta > tol && st->total < max_it) ? 1u : 0u);
}

bool gmres_graph_enabled() {
  static const bool on = [] {
    const char* e = getenv("XDG_GMRES_GRAPH");
    return e == nullptr || atoi(e) != 0;
  }();
  return on;
}

int gmres_solve_graph(const xdg_bsr* M, const xdg_pmg* pmg, int m, double tol, int max_it,
                      const double* b, double* x, int has_x0, double* V, double* Zb, double* w,
                      double* r, double* sc, double* ycoef, void* ws, int* iterations,
                      double* history, int* hist_len, double* final_residual, cudaStream_t s) {
  const int64_t n = (int64_t)M->nbr * M->N;
  GraphOmg G;  // capture streams
  const size_t nH = (size_t)(m + 1) * m, ndbl = nH + 3 * (size_t)m + 1 + (max_it + 2) + 1 +
                                                2 * (size_t)n;
  char* buf = nullptr;
  XDG_TRY_CUDA(cudaMallocAsync(&buf, sizeof(GmDev) + sizeof(double) * ndbl, s));
  XDG_TRY_CUDA(cudaMemsetAsync(buf, 0, sizeof(GmDev) + sizeof(double) * ndbl, s));
  GmDev* st = reinterpret_cast<GmDev*>(buf);
  double* H = reinterpret_cast<double*>(buf + sizeof(GmDev));
  double* cs = H + nH;
  double* sn = cs + m;
  double* g = sn + m;           // m + 1
  double* hist = g + m + 1;     // max_it + 2
  double* gbytes = hist + max_it + 2;
  double* vbuf = gbytes + 1;
  double* zbuf = vbuf + n;
  cudaStream_t s0 = cap_stream(G, 0);
  int rc = XDG_OK;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  const xdg_stream_t x0s = reinterpret_cast<xdg_stream_t>(s0);
  auto capture = [&]() -> int {
    if (!has_x0) {
      zero2_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s0>>>(n, x, nullptr);
      XDG_CHECK_LAUNCH();
    }
    XDG_TRY(spmv(M, x, r, b, sc, ws, s0));                          // r = b - M x
    cudaGraphConditionalHandle ho;
    XDG_TRY(make_handle(s0, &ho));
    gm_init_kernel<<<1, 1, 0, s0>>>(st, sc, tol, max_it, hist, ho);
    XDG_CHECK_LAUNCH();
    cudaGraph_t outer;
    XDG_TRY(add_cond_node(s0, ho, cudaGraphCondTypeWhile, 1, &outer));
    cudaStream_t s1;
    XDG_TRY(begin_body(G, 1, outer, &s1));
    const xdg_stream_t x1 = reinterpret_cast<xdg_stream_t>(s1);
    {
      cudaGraphConditionalHandle hi;
      XDG_TRY(make_handle(s1, &hi));
      gm_cycle_init_kernel<<<1, 1, 0, s1>>>(st, H, cs, sn, g, m, hi);
      XDG_CHECK_LAUNCH();
      count(16.0 * n);
      // V_0 = r / beta (device beta; same rounding as xdg_scale with a host beta)
      XDG_TRY(xdg_scale(n, 1.0, &st->beta, 1, r, V, x1));
      cudaGraph_t inner;
      XDG_TRY(add_cond_node(s1, hi, cudaGraphCondTypeWhile, 1, &inner));
      cudaStream_t s2;
      XDG_TRY(begin_body(G, 2, inner, &s2));
      const double b0 = g_bytes;
      gm_col_copy_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s2>>>(n, st, V, n, vbuf, 0);
      XDG_CHECK_LAUNCH();
      XDG_TRY(pmg_apply_op(pmg, M, vbuf, zbuf, s2));
      XDG_TRY(spmv(M, zbuf, w, nullptr, nullptr, nullptr, s2));
      gm_col_copy_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s2>>>(n, st, zbuf, 0, Zb, n);
      XDG_CHECK_LAUNCH();
      XDG_TRY(mgs_launch(n, 0, &st->j, V, n, w, sc, ws, s2));
      const double fixed = g_bytes - b0;
      g_bytes = b0;
      gm_givens_kernel<<<1, 1, 0, s2>>>(st, sc, H, cs, sn, g, m, tol, max_it, hist, hi, gbytes,
                                        (double)n, fixed);
      XDG_CHECK_LAUNCH();
      XDG_TRY(end_body(s2));
      gm_backsolve_kernel<<<1, 1, 0, s1>>>(st, H, g, m, ycoef, gbytes, (double)n);
      XDG_CHECK_LAUNCH();
      XDG_TRY(gemv_update2_dev(n, m, &st->j, Zb, nullptr, n, ycoef, nullptr, x, nullptr, s1));
      const double b1 = g_bytes;
      XDG_TRY(spmv(M, x, r, b, sc, ws, s1));
      (void)b1;
      gm_cycle_end_kernel<<<1, 1, 0, s1>>>(st, sc, tol, max_it, hist, ho);
      XDG_CHECK_LAUNCH();
    }
    XDG_TRY(end_body(s1));
    (void)x0s;
    return XDG_OK;
  };
  if (s0 == nullptr) {
    rc = XDG_ERR_CUDA;
  } else {
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(ev, s);
    cudaStreamWaitEvent(s0, ev, 0);
    cudaEventDestroy(ev);
    XDG_TRY_CUDA(cudaStreamBeginCapture(s0, cudaStreamCaptureModeRelaxed));
    // the restart cycles' spmv bytes (once per cycle) are counted on the host
    // at capture; scale the per-cycle part by the cycle count afterwards
    const double cap0 = g_bytes;
    rc = capture();
    const double per_capture = g_bytes - cap0;
    g_bytes = cap0;
    cudaError_t e = cudaStreamEndCapture(s0, &graph);
    if (rc == XDG_OK && e != cudaSuccess) {
      set_error("gmres graph capture: %s", cudaGetErrorString(e));
      rc = XDG_ERR_CUDA;
    }
    if (rc == XDG_OK && (e = cudaGraphInstantiate(&exec, graph, 0)) != cudaSuccess) {
      set_error("gmres graph instantiate: %s", cudaGetErrorString(e));
      rc = XDG_ERR_CUDA;
    }
    if (rc == XDG_OK && (e = cudaGraphLaunch(exec, s)) != cudaSuccess) {
      set_error("gmres graph launch: %s", cudaGetErrorString(e));
      rc = XDG_ERR_CUDA;
    }
    if (rc == XDG_OK) {
      GmDev top;
      double dbytes = 0.0;
      e = cudaMemcpyAsync(&top, st, sizeof(GmDev), cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(&dbytes, gbytes, sizeof(double), cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e == cudaSuccess)
        e = cudaMemcpy(history, hist, sizeof(double) * top.hl, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) {
        set_error("gmres graph readback: %s", cudaGetErrorString(e));
        rc = XDG_ERR_CUDA;
      } else if (top.err) {
        set_error("preconditioned operator produced a zero column");
        rc = XDG_ERR_SINGULAR;
      } else {
        *iterations = top.total;
        *hist_len = top.hl;
        *final_residual = top.beta;
        // host-counted capture bytes: the initial residual once, the cycle
        // setup (V_0 scaling + residual) once per restart cycle
        const int cycles = (top.total + m - 1) / (m > 0 ? m : 1);
        g_bytes += per_capture * (cycles > 0 ? cycles : 1) + dbytes;
      }
    }
  }
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  cudaFreeAsync(buf, s);
  for (cudaStream_t t : G.streams) cudaStreamDestroy(t);
  return rc;
}

}  // namespace omg_graph
}  // namespace xdg

// Exported pieces of rm_step for the multi-GPU driver (dist_solvers.py),
// which interleaves them with all-reduces.
extern "C" int xdg_rm_normalize(int64_t n, const double* nw2_dev, double* w,
                                double* z, xdg_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n <= 0) return XDG_OK;
  rm_normalize_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, nw2_dev, w, z);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_rm_commit(int64_t n, const double* alpha_dev, const double* z,
                             double* y, const double* x0, const double* r0,
                             const double* My_new, double* x, double* r,
                             xdg_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n <= 0) return XDG_OK;
  rm_commit_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, alpha_dev, z, y, x0, r0,
                                                          My_new, x, r);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_rm_restart_vec(int64_t n, double* x0, double* r0, double* y,
                                  double* My, double* x, double* r,
                                  xdg_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n <= 0) return XDG_OK;
  rm_restart_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, x0, r0, y, My, x, r);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_rm_restart(xdg_rm* rm, xdg_stream_t stream) {
  return rm_restart(rm, reinterpret_cast<cudaStream_t>(stream));
}
