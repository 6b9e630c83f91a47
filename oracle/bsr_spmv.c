/* oracle/bsr_spmv.c -- TEST INFRASTRUCTURE (CPU checker / CPU baseline).
 *
 * Restates cutdg BlockSparseMatrix.matvec (blockmatrix.py:119-125): the
 * reference converts its dict of blocks into CSR in sorted (bi, bj) order
 * (blockmatrix.py:91-114) and calls scipy's csr_matvec, which sums every
 * scalar row left to right (ascending column), starting from 0.0, with a
 * separately rounded multiply and add.  On the row-major BSR arrays that is:
 *     y[bi*N+i] = (((0 + A_k0(i,0) x_c0[0]) + A_k0(i,1) x_c0[1]) + ...)
 * over blocks k of row bi in column order.  Compiled with
 * -ffp-contract=off so no FMA contraction changes the rounding.
 *
 * nthreads > 1 splits the block rows into contiguous ranges over POSIX
 * threads (rows are independent: the result is identical for any count).
 */
#include <pthread.h>
#include <stdint.h>
#include <unistd.h>

typedef struct {
  int64_t r0, r1;
  int N;
  const int64_t *row_ptr, *col;
  const double *val, *x;
  double* y;
} job_t;

static void rows(int64_t r0, int64_t r1, int N, const int64_t* row_ptr,
                 const int64_t* col, const double* val, const double* x,
                 double* y) {
  for (int64_t bi = r0; bi < r1; ++bi) {
    for (int i = 0; i < N; ++i) {
      double sum = 0.0;
      for (int64_t k = row_ptr[bi]; k < row_ptr[bi + 1]; ++k) {
        const double* a = val + k * (int64_t)N * N + (int64_t)i * N;
        const double* xc = x + col[k] * (int64_t)N;
        for (int j = 0; j < N; ++j) {
          double p = a[j] * xc[j];
          sum = sum + p;
        }
      }
      y[bi * N + i] = sum;
    }
  }
}

static void* run(void* p) {
  job_t* j = (job_t*)p;
  rows(j->r0, j->r1, j->N, j->row_ptr, j->col, j->val, j->x, j->y);
  return 0;
}

void oracle_bsr_spmv(int64_t nbr, int N, const int64_t* row_ptr,
                     const int64_t* col, const double* val, const double* x,
                     double* y, int nthreads) {
  if (nthreads <= 1 || nbr < 1024) {
    rows(0, nbr, N, row_ptr, col, val, x, y);
    return;
  }
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  job_t jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = (job_t){nbr * t / nthreads, nbr * (t + 1) / nthreads, N,
                      row_ptr, col, val, x, y};
    pthread_create(&th[t], 0, run, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], 0);
}

int oracle_max_threads(void) { return (int)sysconf(_SC_NPROCESSORS_ONLN); }
