// Galerkin coarse operator Mc = R^T M R (cutdg transfer.py:344-351 via two
// dict-of-blocks SpGEMMs, blockmatrix.py:133-151) -- the paper's Table-2
// "sparse matrix-matrix product".
//
// R has exactly one N x N block per fine block row (nested aggregates,
// transfer.py:307-334), so every block M_ik contributes exactly one term
// R_i^T M_ik R_k to the coarse block (parent(i), parent(k)).  The host builds
// the output pattern and, per output block, its term list sorted by (i, k);
// this kernel runs one CTA per output block and accumulates the terms in that
// order (deterministic, no atomics).  Same association as the reference's
// bs_matmat(R^T, bs_matmat(M, R)): per fine row i the products M_ik R_k are
// summed first (P_i), then acc += R_i^T P_i -- with the large carrier
// coefficients of small cut pieces, forming R_i^T M_ik R_k term by term
// cancels far worse.  Compute <= 4 N^3 flops per term; bytes: 2 N^2 doubles
// read per term + N^2 per fine row + N^2 written per output block.
// All blocks column-major (BSR-T).
#include "xdg_common.cuh"

namespace xdg {
namespace {

constexpr int kGT = 256;
constexpr int kGMaxOwn = 16;  // outputs per thread: N^2 <= 16 * 256 (N <= 64)

__global__ void __launch_bounds__(kGT)
galerkin_kernel(int nout, int N, const int* __restrict__ tptr,
                const int* __restrict__ t_e, const int* __restrict__ t_ri,
                const int* __restrict__ t_rk, const double* __restrict__ Mv,
                const double* __restrict__ Rv, double* __restrict__ Cv) {
  extern __shared__ double sm[];
  const int NN = N * N;
  double* A = sm;            // M_ik      column-major: A[c*N + a] = M(a, c)
  double* B = sm + NN;       // R_k       column-major: B[b*N + c] = R_k(c, b)
  double* Ct = sm + 2 * NN;  // R_i^T     Ct[c*N + a] = R_i(c, a)
  double* P = sm + 3 * NN;   // M_ik R_k  column-major
  const int o = blockIdx.x;
  double acc[kGMaxOwn], pac[kGMaxOwn];
#pragma unroll
  for (int q = 0; q < kGMaxOwn; ++q) acc[q] = pac[q] = 0.0;
  const int tb = tptr[o], te = tptr[o + 1];
  for (int t = tb; t < te; ++t) {
    const double* Me = Mv + (int64_t)t_e[t] * NN;
    const double* Rk = Rv + (int64_t)t_rk[t] * NN;
    __syncthreads();
    for (int x = threadIdx.x; x < NN; x += kGT) {
      A[x] = Me[x];
      B[x] = Rk[x];
    }
    __syncthreads();
    // P_i += M_ik R_k   (reference order: (M R) first, blockmatrix.py:132-150)
#pragma unroll
    for (int q = 0; q < kGMaxOwn; ++q) {
      const int x = threadIdx.x + q * kGT;
      if (x < NN) {
        const int b = x / N, a = x - b * N;
        double s = 0.0;
        for (int c = 0; c < N; ++c) s = fma(A[c * N + a], B[b * N + c], s);
        pac[q] += s;
      }
    }
    const int ri = t_ri[t];
    if (t + 1 < te && t_ri[t + 1] == ri) continue;
    // last term of fine row i: acc += R_i^T P_i
    const double* Ri = Rv + (int64_t)ri * NN;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kGMaxOwn; ++q) {
      const int x = threadIdx.x + q * kGT;
      if (x < NN) {
        P[x] = pac[q];
        pac[q] = 0.0;
      }
    }
    for (int x = threadIdx.x; x < NN; x += kGT) {
      const int a = x / N, c = x - a * N;  // Ri column-major: x = a*N + c
      Ct[c * N + a] = Ri[x];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kGMaxOwn; ++q) {
      const int x = threadIdx.x + q * kGT;
      if (x < NN) {
        const int b = x / N, a = x - b * N;
        double s = 0.0;
        for (int c = 0; c < N; ++c) s = fma(Ct[c * N + a], P[b * N + c], s);
        acc[q] += s;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kGMaxOwn; ++q) {
    const int x = threadIdx.x + q * kGT;
    if (x < NN) Cv[(int64_t)o * NN + x] = acc[q];
  }
}

}  // namespace
}  // namespace xdg

extern "C" int xdg_galerkin(int nout, int N, const int* tptr, const int* t_e,
                            const int* t_ri, const int* t_rk, const double* Mv,
                            const double* Rv, double* Cv, xdg_stream_t stream) {
  using namespace xdg;
  XDG_REQUIRE(N >= 1 && N * N <= kGMaxOwn * kGT, XDG_ERR_UNSUPPORTED,
              "galerkin: block size %d outside [1, 64]", N);
  if (nout <= 0) return XDG_OK;
  const size_t smem = sizeof(double) * 4 * (size_t)N * N;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (smem > 48 * 1024)
    XDG_TRY_CUDA(cudaFuncSetAttribute(galerkin_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  galerkin_kernel<<<nout, kGT, smem, s>>>(nout, N, tptr, t_e, t_ri, t_rk, Mv, Rv, Cv);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}
