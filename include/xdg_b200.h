/*
 * xdg_b200 — C-ABI of the B200 (sm_100a) XDG solver hot path.
 *
 * Drop-in boundary for the reference package `cutdg` (arXiv 2003.02431
 * restatement, /root/reference/pkg/src/cutdg).  Every entry point takes plain
 * device pointers and sizes, returns an int status (XDG_OK == 0) and runs on
 * the caller's CUDA stream.  No torch types cross this boundary; the Python
 * host layer (paper_2003_02431_b200/) binds it with ctypes.
 *
 * Data layout ("BSR-T"): a uniform-block sparse matrix with nbr block rows
 * and N x N dense blocks is (row_ptr int32[nbr+1], col int32[nnzb],
 * val f64[nnzb][N][N]) with blocks sorted by (block row, block col) -- the
 * order BlockSparseMatrix.tocsr() uses (blockmatrix.py:98) -- and every
 * block stored COLUMN-major: val[k*N*N + j*N + i] = block_k(i, j).
 * xdg_blocks_transpose() converts the reference's row-major blocks.
 * Vectors are f64, block-major (block b owns [b*N, (b+1)*N)).
 *
 * Reductions (dot, norms) are deterministic: per-CTA partials are summed in
 * CTA order by the last CTA; they need a workspace of
 * xdg_reduce_workspace_bytes() bytes, zero-initialised once by the caller.
 */
#ifndef XDG_B200_H_
#define XDG_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* xdg_stream_t; /* == cudaStream_t */

enum {
  XDG_OK = 0,
  XDG_ERR_ARG = 1,      /* -> DimensionMismatchError / InvalidConfigError */
  XDG_ERR_CUDA = 2,     /* CUDA runtime failure                           */
  XDG_ERR_SINGULAR = 3, /* -> SingularSystemError                         */
  XDG_ERR_UNSUPPORTED = 4
};

/* ---- library info ------------------------------------------------------ */
int xdg_version(void);
/* sizeof of the plain-pointer structs, in the order xdg_bsr, xdg_pmg,
 * xdg_direct, xdg_rm, xdg_omg_level, xdg_mf, xdg_mf_node (binding checks);
 * returns the number of entries. */
int xdg_struct_sizes(int64_t* out, int n);
const char* xdg_last_error(void);
/* Bytes of reduction workspace the reduction entry points need. */
int64_t xdg_reduce_workspace_bytes(void);

/* ---- block layout ------------------------------------------------------ */
/* Row-major -> column-major block storage (and back: the op is an
 * involution on square blocks).  in and out must not alias.
 * Replaces the cached CSR build, cutdg blockmatrix.py:91-114. */
int xdg_blocks_transpose(int64_t nnzb, int N, const double* in, double* out,
                         xdg_stream_t stream);

/* out[i*N + q] = x[idx[i]*N + q]: packs the owned x blocks a neighbouring
 * rank needs (multi-GPU halo send buffer). */
int xdg_gather_blocks(int64_t nidx, int N, const int* idx, const double* x,
                      double* out, xdg_stream_t stream);

/* y[idx[i]*N + q] += src[i*N + q] (idx without duplicates): adds the
 * partial Schwarz sums other ranks computed for this rank's cells. */
/* y[idx[i]*N + q] = src[i*N + q] (idx without duplicates): unpacks
 * values received from other ranks (multi-GPU multifrontal exchange). */
int xdg_scatter_blocks(int64_t nidx, int N, const int* idx, const double* src, double* y,
                       xdg_stream_t stream);
int xdg_scatter_add_blocks(int64_t nidx, int N, const int* idx,
                           const double* src, double* y, xdg_stream_t stream);
/* out[k*m + q] = x[k*N + q], q < m: the low-order modes of nblk blocks (the
 * owned part of the distributed low-order right-hand side, solvers.py:250). */
int xdg_gather_modes(int64_t nblk, int N, int m, const double* x, double* out,
                     xdg_stream_t stream);

/* ---- block-sparse matrix-vector product -------------------------------- */
/* Block rows [row_begin, row_end) of
 *     b == NULL :  y = alpha * (M x) + beta * y   (beta == 0: y not read)
 *     b != NULL :  y = b - M x                    (alpha, beta ignored)
 * Each scalar row is summed over its blocks in column order, then over the
 * block's columns in order, with separately rounded multiply and add: the
 * summation order of scipy's csr_matvec on BlockSparseMatrix.tocsr(), so
 * alpha=1, beta=0 reproduces cutdg BlockSparseMatrix.matvec
 * (blockmatrix.py:119-125) bit for bit.
 * If norm2_out != NULL, *norm2_out (device) = sum over the computed rows of
 * y_i^2 (deterministic), using ws (xdg_reduce_workspace_bytes()).
 * x is indexed by block column (it may be longer than M's rows: owned
 * blocks followed by halo blocks on a multi-GPU rank). */
int xdg_bsr_spmv(int row_begin, int row_end, int N, const int* row_ptr,
                 const int* col, const double* val_t, const double* x,
                 double* y, double alpha, double beta, const double* b,
                 double* norm2_out, void* ws, xdg_stream_t stream);

/* ---- vector kernels (deterministic reductions) ------------------------- */
/* *out = sum_i x_i * y_i  (device scalar).   numpy `x @ y`,
 * used at solvers.py:587,594,604,607,700,782,803,805,834. */
int xdg_dot(int64_t n, const double* x, const double* y, double* out,
            void* ws, xdg_stream_t stream);
/* y += s * x with s = a            if a_dev == NULL
 *                 s = a * (*a_dev) otherwise (device scalar)   */
int xdg_axpy(int64_t n, double a, const double* a_dev, const double* x,
             double* y, xdg_stream_t stream);
/* One modified Gram-Schmidt step in one pass (distributed GMRES,
 * solvers.py:802-805): y += c * x with c = a * (*a_dev) (a_dev != NULL) or
 * c = a, then *out = sum_i v_i y_i over the updated y (v == NULL: sum y_i^2);
 * deterministic reduction (ws as for xdg_dot). */
int xdg_axpy_dot(int64_t n, double a, const double* a_dev, const double* x,
                 double* y, const double* v, double* out, void* ws,
                 xdg_stream_t stream);
/* y = s * x with s = a                   if a_dev == NULL and !invert
 *                s = a * (*a_dev)        if a_dev != NULL and !invert
 * y = a * (x / (*a_dev))                 if a_dev != NULL and invert
 * y = x / a                              if a_dev == NULL and invert
 * (division per element, x_i / d, like numpy `w /= norm_w`, solvers.py:601) */
int xdg_scale(int64_t n, double a, const double* a_dev, int invert,
              const double* x, double* y, xdg_stream_t stream);
/* out = x + y (elementwise): RmState.current() x0 + y (solvers.py:546). */
int xdg_add(int64_t n, const double* x, const double* y, double* out,
            xdg_stream_t stream);
/* rm_step's exact-image update (solvers.py:605-607), fused:
 *   My_new = My + (*alpha_dev) * Mz ;  *rho2 = ||r0 - My_new||^2 (device). */
int xdg_rm_update(int64_t n, const double* r0, const double* My,
                  const double* Mz, const double* alpha_dev, double* My_new,
                  double* rho2, void* ws, xdg_stream_t stream);
/* r = b - y (elementwise). */
int xdg_sub(int64_t n, const double* b, const double* y, double* r,
            xdg_stream_t stream);
/* y = x ./ d (elementwise), the overlap damping of schwarz_apply
 * (solvers.py:478). */
int xdg_div(int64_t n, const double* x, const double* d, double* y,
            xdg_stream_t stream);

/* ---- tall-skinny kernels for residual minimisation / GMRES ------------- */
/* coeff[c] = sum_i W[c*ldw + i] * w[i], c < ncols: `W.T @ w`
 * (solvers.py:590).  Deterministic; ws >= xdg_gemv_t_workspace_bytes. */
int64_t xdg_gemv_t_workspace_bytes(int ncols);
int xdg_gemv_t(int64_t L, int ncols, const double* W, int64_t ldw,
               const double* w, double* coeff, void* ws, xdg_stream_t stream);
/* w -= W coeff ; z -= Z coeff_z (coeff_z NULL: coeff; Z may be NULL): the
 * update pair of a classical Gram-Schmidt pass, solvers.py:591-592. */
int xdg_gemv_update2(int64_t L, int ncols, const double* W, const double* Z,
                     int64_t ld, const double* coeff, const double* coeff_z,
                     double* w, double* z, xdg_stream_t stream);
/* out = a + b for short device vectors (coefficient sums). */
int xdg_add_small(int n, const double* a, const double* b, double* out,
                  xdg_stream_t stream);


/* ---- dense LU solves (batched, variable size) --------------------------- */
/* Factors: a partial-pivoting LU (A = P L U, L unit lower) stored as its
 * TRIANGULAR INVERSES, INV (row-major n x n per system): L^-1 strictly below
 * the diagonal (unit diagonal implicit), U^-1 on and above it.  A solve
 * x = U^-1 L^-1 P^T b is two triangular GEMVs (8 n^2 bytes, the same as
 * forward/backward substitution, without the sequential chain).
 * Replaces SuperLU solve (blockmatrix.py:224) for the low-order PMG systems
 * (solvers.py:249-251) and the coarsest-level direct solve (solvers.py:699).
 *
 * For s < nsys: n = dims[s], INV + off[s], and x + vec_off[s] receives
 * A_s^-1 (b[src[vec_off[s]+i]])_i -- pivot permutation pre-composed with the
 * gather.  Systems are packed back to back (vec_off[s+1] = vec_off[s] +
 * dims[s]), total = sum of dims, row_sys[g] = system of packed row g.  All
 * systems at once, warp per row over the whole GPU (3 launches: gather,
 * L^-1 rows, U^-1 rows); scratch: 2 total doubles. */
int xdg_lu_inv_apply(int nsys, int64_t total, const int* row_sys,
                     const int64_t* off, const int* dims,
                     const int64_t* vec_off, const double* INV, const int* src,
                     const double* b, double* x, double* scratch,
                     xdg_stream_t stream);
/* The same solves with CTA tasks (system task_sys[t], rows task_row0[t] ..
 * + rows_per_task): each system's right-hand side is staged in shared memory
 * (max_dim doubles), so the row dots keep only matrix loads in flight. */
int xdg_lu_inv_apply_tasks(int64_t ntasks, const int* task_sys,
                           const int* task_row0, int rows_per_task, int max_dim,
                           int64_t total, const int64_t* off, const int* dims,
                           const int64_t* vec_off, const double* INV,
                           const int* src, const double* b, double* x,
                           double* scratch, xdg_stream_t stream);
/* ---- batched dense factorization (setup, xdg_factor.cu) --------------- */
/* Partial-pivoting LU of a batch of row-major matrices of any sizes, in
 * place: matrix b at A + off[b] (elements), leading dimension ld[b],
 * n[b] x n[b], its first p[b] <= n[b] columns eliminated with pivots chosen
 * among its first p[b] rows (p = n: a full LU; p < n: a multifrontal front,
 * leaving L_BP = F_BP U^-1, U_PB = L^-1 P F_PB and the Schur complement
 * F_BB - L_BP U_PB in place).  max_n / max_p bound n[b] / p[b] (grid
 * sizing).  perm[perm_off[b] + i] (i < p[b]) = original row at position i
 * ((P b)[i] = b[perm[i]]); info[b] = 1 + first column with a zero or
 * non-finite pivot, 0 if none (the caller raises SingularSystemError).
 * invert != 0: the top-left p x p LU is replaced by the triangular
 * inverses xdg_lu_inv_apply reads (L^-1 strictly below the diagonal, U^-1
 * on and above), using ws (xdg_batched_factor_ws_bytes(nmat, max_p)).
 * nmat < 65536 per call.
 * Replaces scipy lu_factor (cutdg solvers.py:233), SuperLU splu
 * (blockmatrix.py:213) and the dense factor of direct_factor
 * (blockmatrix.py:203-216) -- SURVEY 8(b)'s xdg_batched_factor. */
int xdg_batched_factor(int64_t nmat, const int64_t* off, const int* n,
                       const int* p, const int* ld, int max_n, int max_p,
                       double* A, int* perm, const int64_t* perm_off, int* info,
                       int invert, double* ws, xdg_stream_t stream);
int64_t xdg_batched_factor_ws_bytes(int64_t nmat, int max_p);
/* LAPACK ipiv (1-based sequential swaps) -> permutation perm with
 * (P^T b)[i] = b[perm[i]], per system (setup). */
int xdg_ipiv_to_perm(int nsys, const int* dims, const int64_t* vec_off,
                     const int* ipiv, int* perm, xdg_stream_t stream);

/* ---- degree-separated preconditioner / Schwarz -------------------------- */
/* Work item w = one cell (block row) of one system; its blocks restricted
 * to the system's cell set are wi_blk[wi_ptr[w] .. wi_ptr[w+1]) with local
 * column index wi_lcol (sorted by column).  m = number of low modes.
 * Setup: dense low-order matrices A_s (zero-initialised by the caller)
 * (solvers.py:208-215). */
int xdg_pmg_build_low(int nwork, int N, int m, const int* wi_ptr,
                      const int* wi_blk, const int* wi_lcol, const int* wi_lrow,
                      const int* wi_sys, const int64_t* lu_off, const int* dims,
                      const double* val_t, double* A, xdg_stream_t stream);
/* Setup: size-bucket staging of the batched dense factorization.
 * unpack = 0: packed[q] (P x P) = the n x n row-major system sys[q]
 * (n = dims[sys[q]], at flat + off[sys[q]]), identity in the padding;
 * unpack = 1: the n x n top-left of packed[q] back to flat.  Replaces the
 * per-system copies around the reference's per-block lu_factor
 * (solvers.py:208-221). */
int xdg_pack_square(int64_t nsys, const int64_t* sys, const int* dims,
                    const int64_t* off, int P, double* packed, double* flat,
                    int unpack, xdg_stream_t stream);
/* Setup: H[c] = M[cells[c], cells[c]](m:, m:), row-major, diag_blk[c] the
 * block index of the diagonal block (solvers.py:232). */
int xdg_pmg_gather_high(int ncells, int N, int m, const int* cells,
                        const int* diag_blk, const double* val_t, double* H,
                        xdg_stream_t stream);
/* Apply, fused: for every work item, r = b_hi - M_II(hi, lo) x_lo over the
 * system's blocks (solvers.py:257), x_hi = H^-1 r with the cell's pivoted
 * column-major LU (HLU + wi_hidx*nh*nh, hperm) (solvers.py:258-262), and
 * out[wi_out + 0..N) = [x_lo(cell), x_hi].  N - m <= 64. */
int xdg_pmg_high(int nwork, int N, int m, const int* wi_ptr, const int* wi_blk,
                 const int* wi_lcol, const int* wi_cell, const int* wi_lrow,
                 const int64_t* wi_xlo, const int* wi_hidx,
                 const int64_t* wi_out, const double* val_t, const double* HLU,
                 const int* hperm, const double* b, const double* xlo,
                 double* out, xdg_stream_t stream);
/* z[bi*N+i] = (sum_e out[cpos[e] + i], e in [cptr[bi], cptr[bi+1]) in
 * order) / damping[bi*N+i]  (damping may be NULL): the additive Schwarz
 * sum and overlap damping of schwarz_apply (solvers.py:473-478). */
int xdg_pmg_combine(int nbr, int N, const int* cptr, const int64_t* cpos,
                    const double* out, const double* damping, double* z,
                    xdg_stream_t stream);

/* ---- Galerkin coarse operator (transfer.py:344-351) -------------------- */
/* Mc = R^T M R where R has one block per fine row.  Output block o of Mc
 * accumulates, in order, the terms t in [tptr[o], tptr[o+1]):
 *   R[t_ri[t]]^T  M[t_e[t]]  R[t_rk[t]]   (all blocks column-major, N <= 64).
 * One CTA per output block; deterministic. */
int xdg_galerkin(int nout, int N, const int* tptr, const int* t_e,
                 const int* t_ri, const int* t_rk, const double* Mv,
                 const double* Rv, double* Cv, xdg_stream_t stream);

/* ---- SIP-DG raw operator formation (assembly.py:255-367) -------------- */
/* out[o] = sum_{t in [tptr[o],tptr[o+1])} coef[t] * tables[tid[t]]
 *        + sum_{d in [dptr[o],dptr[o+1])} dense[didx[d]]
 * All blocks N x N column-major; one warp per output block; deterministic.
 * Replaces the per-block add_block accumulation of assemble_sip
 * (assembly.py:271-367, blockmatrix.py:65-76). */
int xdg_assemble_blocks(int nout, int N, const int* tptr, const int* tid,
                        const double* coef, const double* tables, const int* dptr,
                        const int* didx, const double* dense, double* out,
                        xdg_stream_t stream);

/* ---- multifrontal sparse LU (nested-dissection forest) ---------------- */
/* Replaces SuperLU splu/solve (cutdg blockmatrix.py:203-227) for the
 * low-order PMG systems (solvers.py:208-221, 249-251), the coarsest level /
 * "direct" solver (solvers.py:661-666, 698-710).  Built by multifrontal.py.
 * Factor storage F (device): per front row-major INV (p x p, leading dim
 * ldp: L^-1 strictly lower, U^-1 upper), L_BP (b x p, ld ldp), U_PB
 * (p x b, ld ldb). */
typedef struct xdg_mf_node {
  int32_t p, b, ldp, ldb;      /* pivot / boundary unknowns, leading dims */
  int32_t gp, gb, ldr, pad1;   /* lanes per row for p- / b-long rows (2^k);
                                  ldr > 0: lbp holds the column-major forward
                                  copy FT[k][r] of [L^-1; M_BP], ld = ldr   */
  int64_t inv, lbp, upb;       /* offsets into F */
  int64_t w, y, c;             /* offsets into W (p+b), Y (p), C (b) */
  int64_t bx, px;              /* offsets into bidx (b), pdst (p) */
} xdg_mf_node;

typedef struct xdg_mf {
  int32_t nlevels, nnodes;
  int64_t total;               /* unknowns */
  const int64_t* lev_ent;      /* HOST [nlevels+1] gather-entry ranges      */
  const int64_t* lev_task;     /* HOST [4][nlevels+1] warp-task ranges of the
                                  phases lower, bound, upb, upper            */
  const int64_t* ent_w;        /* gather entry -> W index                   */
  const int64_t* ent_src;      /* -> index into b, or -1                    */
  const int64_t* ent_cptr;     /* CSR of child contributions (into C)       */
  const int64_t* ent_cidx;
  const int32_t* tasks;        /* int4 (node, first row, rows, -1) warp tasks */
  const xdg_mf_node* nodes;
  const int64_t* bidx;         /* Y index of each boundary unknown          */
  const int64_t* pdst;         /* x index of each pivot unknown             */
  const double* ent_scale;     /* equilibration: W = ent_scale * b[src] ... */
  const double* pscale;        /*   ... x[pdst] = pscale * (U^-1 T)         */
  const double* F;
  double* W;
  double* Y;
  double* C;
  double apply_bytes;          /* algorithmic bytes of one solve            */
  /* Fused low levels: heights [0, fuse_levels) run as nfbatch launches per
   * sweep, one CTA per group of fronts, each group a sequence of stages
   * (fronts of one height, children in earlier stages of the group).      */
  int32_t fuse_levels, nfbatch;
  int64_t nfstages;
  const int64_t* fb_grp;       /* HOST [nfbatch+1] group ranges per launch   */
  const int64_t* g_stage;      /* [ngroups+1] stage ranges per group         */
  const int64_t* st_ent;       /* [nfstages+1] ranges into fent              */
  const int64_t* st_task;      /* [4][nfstages+1] ranges into ftask per phase */
  const int64_t* fent;         /* gather entry ids, stage by stage           */
  const int32_t* ftask;        /* int4 warp tasks, stage by stage            */
  /* Merged phases: the factors hold M_BP = L_BP L^-1 (at lbp) and N_PB =
   * U^-1 U_PB (at upb), see xdg_mf_merge; one row launch per height and
   * sweep: lev_task then has 6 ranges per level -- [0] forward warp tasks
   * (rows 0..p+b-1 of every front), [1] forward group tasks (long rows),
   * [2] / [3] the same for the backward rows 0..p-1, [4] forward
   * thread-per-row tasks of the fronts with a column-major copy (ldr > 0),
   * [5] reserved; X[p] = equilibrated solution (bidx indexes X).
   * Excludes the fused low levels.                                        */
  double* X;
  int32_t merged, pad_;
} xdg_mf;

/* Setup: extend-add of one round of children's Schur complements into
 * their parents' fronts (pair = 7 int64 per (parent, child): parent base,
 * parent stride, child base, child stride, child pivot pad, n, U offset).
 * Replaces the per-child assembly of the factorization SuperLU does inside
 * splu (cutdg blockmatrix.py:203-227). */
int xdg_mf_extend_add(int64_t npairs, const int64_t* pair, const int64_t* U,
                      const double* child, double* parent, int64_t max_n,
                      xdg_stream_t stream);
/* Setup of the merged phases: for nb fronts (each an n x n row-major
 * buffer, n = P + B, as xdg_batched_factor(invert) left it) write
 * out_m[q] = L_BP L^-1 (B x P) and out_n[q] = U^-1 U_PB (P x B), dense
 * row-major, front after front.  Same role as the triangular solves inside
 * SuperLU's supernodal solve (cutdg blockmatrix.py:218-227), moved to the
 * factorization. */
int xdg_mf_merge(int64_t nb, int P, int B, const double* fronts, double* out_m,
                 double* out_n, xdg_stream_t stream);
/* Rows per warp task of a front whose rows take a whole warp. */
int xdg_mf_rows_per_warp(void);
/* Host-side symbolic analysis (csrc/xdg_ordering.cu).  Nested dissection
 * of the graph (ptr, col) with nv vertices into a post-ordered forest:
 * node_ptr[nnodes+1], node_verts[nv], parent[nnodes] (capacities nv+1, nv,
 * nv); returns nnodes. */
int64_t xdg_nd_order(int64_t nv, const int64_t* ptr, const int64_t* col,
                     int64_t leaf, int64_t* node_ptr, int64_t* node_verts,
                     int64_t* parent);
/* Boundary sets of the fronts (ancestor vertices adjacent to the subtree,
 * sorted by (owner, vertex)); returns their total size, copied out by
 * xdg_nd_boundaries_copy(b_ptr[nnodes+1], b_verts[total]). */
int64_t xdg_nd_boundaries(int64_t nv, const int64_t* ptr, const int64_t* col,
                          int64_t nnodes, const int64_t* node_ptr,
                          const int64_t* node_verts, const int64_t* parent);
int xdg_nd_boundaries_copy(int64_t* b_ptr, int64_t* b_verts);
/* Overlapping Schwarz partition (cutdg schwarz_partition, solvers.py:
 * 384-457): greedy BFS cores of >= target DOFs over the graph (adj_ptr,
 * adj sorted), grown by one neighbour layer.  Returns the number of cores;
 * xdg_schwarz_sizes gives {#core nodes, #extended nodes}; xdg_schwarz_copy
 * writes core_ptr[ncore+1], core_nodes, ext_ptr[ncore+1], ext_nodes. */
int64_t xdg_schwarz_partition(int64_t n, const int64_t* adj_ptr,
                              const int64_t* adj, const int64_t* dofs,
                              int64_t target);
int xdg_schwarz_sizes(int64_t* out);
int xdg_schwarz_copy(int64_t* core_ptr, int64_t* core_nodes, int64_t* ext_ptr,
                     int64_t* ext_nodes);
/* x[pdst] = A^-1 b[src] for every system of the forest at once:
 * 3 launches per forward level, 2 per backward level. */
int xdg_mf_solve(const xdg_mf* mf, const double* b, double* x,
                 xdg_stream_t stream);
/* One sweep of xdg_mf_solve: phase 1 = forward (gather, L^-1, bound
 * contributions), 2 = backward (U_PB, U^-1, output), 3 = both.  The
 * multi-GPU factor (dist_multifrontal) runs the owned subtrees' forward
 * sweep, exchanges the subtree roots' contributions, runs the replicated
 * top fronts, then the owned backward sweep. */
int xdg_mf_solve_phase(const xdg_mf* mf, const double* b, double* x, int phase,
                       xdg_stream_t stream);

/* ======================================================================
 * Native solver driver (the reference's control loops, solvers.py:559-846,
 * run in C++ over device data: one host sync per rm_step / GMRES inner
 * iteration, no Python in the iteration loop).  Plain-pointer structs; the
 * host layer fills them from its device buffers.  All device pointers.
 * ====================================================================== */
typedef struct xdg_bsr {
  int32_t nbr, nbc, N, pad0;
  int64_t nnzb;
  const int* row_ptr;
  const int* col;
  const double* val_t;
} xdg_bsr;

typedef struct xdg_pmg {       /* PmgPlan of paper_2003_02431_b200/pmg.py */
  int32_t nsys, nwork, N, m, has_high, direct;
  int64_t total;               /* sum of the low-order system sizes */
  const int* row_sys;
  double* scratch;             /* 2 total doubles */
  const int64_t* lu_off;
  const int* dims;
  const int64_t* vec_off;
  const double* LU;            /* triangular-inverse factors (INV) */
  const int* src;
  double* xlo;
  const int* wi_ptr;
  const int* wi_blk;
  const int* wi_lcol;
  const int* wi_cell;
  const int* wi_lrow;
  const int64_t* wi_xlo;
  const int* wi_hidx;
  const int64_t* wi_out;
  const double* HLU;
  const int* hperm;
  double* out;
  const int* cptr;
  const int64_t* cpos;
  const double* damping;
  double apply_bytes;          /* algorithmic bytes of one apply (accounting) */
  const xdg_mf* mf;            /* sparse low-order factors (NULL: dense LU) */
  const int* task_sys;         /* dense solves by CTA tasks (NULL: per row) */
  const int* task_row0;
  int64_t ntasks;
  int32_t rows_per_task, max_dim;
} xdg_pmg;

typedef struct xdg_direct {    /* dense LU of one system (coarsest level) */
  int32_t n, pad0;
  const double* LU;            /* triangular-inverse factors (INV) */
  const int* perm;
  const int64_t* zero_off;     /* device {0} */
  const int* dims;             /* device {n} */
  const int* row_sys;          /* device zeros[n] */
  double* scratch;             /* 2 n doubles */
  const xdg_mf* mf;            /* sparse factors (NULL: dense LU)           */
  const int* task_sys;         /* dense solve by CTA tasks (NULL: per row)  */
  const int* task_row0;
  int64_t ntasks;
  int32_t rows_per_task, max_dim;
} xdg_direct;

typedef struct xdg_rm {        /* RmState (solvers.py:485-556) */
  int64_t n;
  int32_t max_columns, ncols;
  int32_t last_dependent, dependent_count, rejected_count, restart_count;
  double best_norm;
  double* W;                   /* [max_columns][n] */
  double* Z;                   /* [max_columns][n] */
  double* x0;
  double* r0;
  double* y;
  double* My;
  double* My_new;              /* swapped with My on accept */
  double* Mz;
  double* coeff;               /* [3 * max_columns]: c1, c2, c1 + c2 */
  double* sc;                  /* >= 8 device scalars */
  double* alpha_host;          /* HOST [max_columns] */
  double* x;                   /* current() outputs */
  double* r;
  void* ws;                    /* reduction workspace */
  void* gemv_ws;               /* xdg_gemv_t_workspace_bytes(max_columns) */
} xdg_rm;

typedef struct xdg_omg_level { /* one level of ortho_mg_solve */
  xdg_bsr M;
  xdg_bsr R;                   /* prolongation (fine rows x coarse cols) */
  xdg_bsr Rt;                  /* restriction */
  int32_t has_restriction, pad0;
  xdg_pmg schwarz;
  xdg_direct direct;           /* used when coarsest */
  xdg_rm rm;
  double* b;                   /* this level's right-hand side buffer */
  double* z;                   /* smoother output */
  double* xf;                  /* R x_c */
} xdg_omg_level;

/* One rm_step (solvers.py:559-625) on state `rm` with operator M and
 * candidate z (device, length rm->n).  Updates rm (host counters too) and
 * leaves the current point / true residual in rm->x, rm->r. */
int xdg_rm_step(xdg_rm* rm, const xdg_bsr* M, const double* z,
                xdg_stream_t stream);
/* RmState(x0, r0): copies x0, r0, zeroes y / My, best_norm = ||r0||. */
int xdg_rm_init(xdg_rm* rm, const double* x0, const double* r0,
                xdg_stream_t stream);
/* rm_step pieces for the multi-GPU driver (it all-reduces in between):
 * w /= sqrt(*nw2), z /= sqrt(*nw2)  (solvers.py:601-602);
 * y += alpha z, x = x0 + y, r = r0 - My_new  (accept, solvers.py:617-624);
 * x0 += y, r0 -= My, y = My = 0, x = x0, r = r0  (restart, 548-556). */
int xdg_rm_normalize(int64_t n, const double* nw2_dev, double* w, double* z,
                     xdg_stream_t stream);
int xdg_rm_commit(int64_t n, const double* alpha_dev, const double* z,
                  double* y, const double* x0, const double* r0,
                  const double* My_new, double* x, double* r,
                  xdg_stream_t stream);
int xdg_rm_restart_vec(int64_t n, double* x0, double* r0, double* y, double* My,
                       double* x, double* r, xdg_stream_t stream);
/* RmState.restart() (solvers.py:548-556); also leaves x = x0, r = r0. */
int xdg_rm_restart(xdg_rm* rm, xdg_stream_t stream);
/* x = x0 + y, r = r0 - My  (RmState.current()). */
int xdg_rm_current(xdg_rm* rm, xdg_stream_t stream);
/* z = PMG / Schwarz application of a plan over operator M
 * (pmg.PmgPlan.apply; solvers.py:245-265, 460-478). */
int xdg_pmg_apply_op(const xdg_pmg* plan, const xdg_bsr* M, const double* b,
                     double* z, xdg_stream_t stream);
/* ortho_mg_solve (solvers.py:669-749) entered at level index `entry`
 * (0-based) of `levels` (nlevels total).  x (device, entry level size) holds
 * the initial guess if has_x0, else is zeroed.  history: HOST array of
 * capacity max_iterations+1; *iterations, *hist_len, *final_residual set;
 * *bytes_out (if not NULL) = algorithmic bytes of all kernels launched. */
int xdg_omg_solve(xdg_omg_level* levels, int nlevels, int entry,
                  double tolerance, int max_iterations,
                  int coarse_cycle_iterations, const double* b, double* x,
                  int has_x0, int* iterations, double* history, int* hist_len,
                  double* final_residual, double* bytes_out,
                  xdg_stream_t stream);
/* Restarted GMRES with PMG on the right (solvers.py:756-846).  V: device
 * [restart+1][n], Zb: [restart][n], w: [n], r: [n], sc: device
 * [restart+8], ycoef: device [restart].  history: HOST, capacity
 * max_iterations+1.  Returns XDG_ERR_SINGULAR on a zero Givens column. */
int xdg_gmres_solve(const xdg_bsr* M, const xdg_pmg* pmg, int restart,
                    double tolerance, int max_iterations, const double* b,
                    double* x, int has_x0, double* V, double* Zb, double* w,
                    double* r, double* sc, double* ycoef, void* ws,
                    void* gemv_ws, int* iterations, double* history,
                    int* hist_len, double* final_residual, double* bytes_out,
                    xdg_stream_t stream);
/* Fused modified Gram-Schmidt of GMRES step j (solvers.py:802-807):
 * for i <= j: h_i = V_i . w ; w -= h_i V_i ; then h_{j+1} = ||w|| and
 * V_{j+1} = w / h_{j+1} (zero if h_{j+1} == 0).  h (device) receives
 * h_0..h_{j+1}.  One cooperative launch (grid-wide syncs between steps). */
int xdg_mgs(int64_t n, int j, double* V, int64_t ldv, double* w, double* h,
            void* ws, xdg_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* XDG_B200_H_ */
