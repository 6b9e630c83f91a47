// SIP-DG raw operator formation (cutdg assembly.py:255-367).
//
// Every output block o of the raw BSR operator is
//     sum_{t in [tptr[o], tptr[o+1])} coef[t] * tables[tid[t]]
//   + sum_{d in [dptr[o], dptr[o+1])} dense[didx[d]]
// where the tables are the few reference blocks of regular contributions
// (uncut volume mu_s K, full-face consistency C and penalty P per axis/side)
// and the dense blocks are the exact per-item blocks of cut volumes, cut face
// portions and interface patches, built on the host.  All blocks are
// column-major (BSR-T), so element x of the output is a plain weighted sum of
// element x of its inputs: one warp per output block, lanes over the N^2
// elements, coalesced writes.  Tables (a few dozen N x N blocks) stay in L1/L2;
// the pass is bounded by the output write, 8 N^2 bytes per block.  Products
// and sums are separately rounded in term order, so the result is bit-identical
// to the host evaluation of the same term list (SipTerms.evaluate_host).
#include "xdg_common.cuh"

namespace xdg {
namespace {

constexpr int kAT = 256;

__global__ void __launch_bounds__(kAT)
assemble_kernel(int nout, int NN, const int* __restrict__ tptr,
                const int* __restrict__ tid, const double* __restrict__ coef,
                const double* __restrict__ tables, const int* __restrict__ dptr,
                const int* __restrict__ didx, const double* __restrict__ dense,
                double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (kAT / 32);
  for (int o = blockIdx.x * (kAT / 32) + (threadIdx.x >> 5); o < nout; o += warps) {
    const int t0 = tptr[o], t1 = tptr[o + 1];
    const int d0 = dptr[o], d1 = dptr[o + 1];
    double* dst = out + (int64_t)o * NN;
    for (int x = lane; x < NN; x += 32) {
      double acc = 0.0;
      for (int t = t0; t < t1; ++t)
        acc = __dadd_rn(acc, __dmul_rn(__ldg(coef + t),
                                       __ldg(tables + (int64_t)__ldg(tid + t) * NN + x)));
      for (int d = d0; d < d1; ++d)
        acc = __dadd_rn(acc, __ldg(dense + (int64_t)__ldg(didx + d) * NN + x));
      dst[x] = acc;
    }
  }
}

}  // namespace
}  // namespace xdg

extern "C" int xdg_assemble_blocks(int nout, int N, const int* tptr, const int* tid,
                                   const double* coef, const double* tables,
                                   const int* dptr, const int* didx, const double* dense,
                                   double* out, xdg_stream_t stream) {
  using namespace xdg;
  XDG_REQUIRE(N >= 1, XDG_ERR_ARG, "assemble_blocks: block size %d", N);
  if (nout <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int grid = resident_grid(assemble_kernel, kAT, 0, (nout + 7) / 8);
  assemble_kernel<<<grid, kAT, 0, s>>>(nout, N * N, tptr, tid, coef, tables, dptr, didx,
                                       dense, out);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}
