// Block storage conversion: row-major blocks (cutdg's dict-of-blocks /
// tocsr order, blockmatrix.py:91-114) <-> column-major blocks (BSR-T, the
// layout every xdg_b200 kernel streams).  One CTA per tile of blocks, staged
// through shared memory so both the read and the write are coalesced.
#include "xdg_common.cuh"

namespace xdg {
namespace {

constexpr int kT = 256;

__global__ void __launch_bounds__(kT)
blocks_transpose_kernel(int64_t nnzb, int N, const double* __restrict__ in,
                        double* __restrict__ out) {
  extern __shared__ double tile[];
  const int nn = N * N;
  const int per_tile = (4096 / nn) > 0 ? (4096 / nn) : 1;  // blocks per tile
  for (int64_t k0 = (int64_t)blockIdx.x * per_tile; k0 < nnzb;
       k0 += (int64_t)gridDim.x * per_tile) {
    const int nb = (int)((nnzb - k0) < per_tile ? (nnzb - k0) : per_tile);
    const int64_t base = k0 * nn;
    for (int e = threadIdx.x; e < nb * nn; e += kT) tile[e] = in[base + e];
    __syncthreads();
    for (int e = threadIdx.x; e < nb * nn; e += kT) {
      const int kb = e / nn, r = e - kb * nn;
      const int a = r / N, c = r - a * N;  // out element (a, c) of block kb
      out[base + e] = tile[kb * nn + c * N + a];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kT)
gather_blocks_kernel(int64_t nidx, int N, const int* __restrict__ idx,
                     const double* __restrict__ x, double* __restrict__ out) {
  const int64_t total = nidx * N;
  for (int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * kT) {
    const int64_t k = t / N;
    out[t] = x[(int64_t)idx[k] * N + (t - k * N)];
  }
}

__global__ void __launch_bounds__(kT)
gather_modes_kernel(int64_t nblk, int N, int m, const double* __restrict__ x,
                    double* __restrict__ out) {
  const int64_t total = nblk * m;
  for (int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * kT) {
    const int64_t k = t / m;
    out[t] = x[k * N + (t - k * m)];
  }
}

__global__ void __launch_bounds__(kT)
scatter_add_blocks_kernel(int64_t nidx, int N, const int* __restrict__ idx,
                          const double* __restrict__ src, double* __restrict__ y) {
  const int64_t total = nidx * N;
  for (int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * kT) {
    const int64_t k = t / N;
    double* d = y + (int64_t)idx[k] * N + (t - k * N);
    *d = __dadd_rn(*d, src[t]);
  }
}

__global__ void __launch_bounds__(kT)
scatter_blocks_kernel(int64_t nidx, int N, const int* __restrict__ idx,
                      const double* __restrict__ src, double* __restrict__ y) {
  const int64_t total = nidx * N;
  for (int64_t t = (int64_t)blockIdx.x * kT + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * kT) {
    const int64_t k = t / N;
    y[(int64_t)idx[k] * N + (t - k * N)] = src[t];
  }
}

}  // namespace
}  // namespace xdg

extern "C" int xdg_scatter_blocks(int64_t nidx, int N, const int* idx, const double* src,
                                  double* y, xdg_stream_t stream) {
  using namespace xdg;
  if (nidx <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  scatter_blocks_kernel<<<grid_for(nidx * N, kT, 8), kT, 0, s>>>(nidx, N, idx, src, y);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_scatter_add_blocks(int64_t nidx, int N, const int* idx,
                                      const double* src, double* y,
                                      xdg_stream_t stream) {
  using namespace xdg;
  if (nidx <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  scatter_add_blocks_kernel<<<grid_for(nidx * N, kT, 8), kT, 0, s>>>(nidx, N, idx,
                                                                     src, y);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_gather_modes(int64_t nblk, int N, int m, const double* x,
                                double* out, xdg_stream_t stream) {
  using namespace xdg;
  if (nblk <= 0) return XDG_OK;
  XDG_REQUIRE(m >= 1 && m <= N, XDG_ERR_ARG, "bad mode count %d of %d", m, N);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  gather_modes_kernel<<<grid_for(nblk * m, kT, 8), kT, 0, s>>>(nblk, N, m, x, out);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_gather_blocks(int64_t nidx, int N, const int* idx,
                                 const double* x, double* out,
                                 xdg_stream_t stream) {
  using namespace xdg;
  if (nidx <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  gather_blocks_kernel<<<grid_for(nidx * N, kT, 8), kT, 0, s>>>(nidx, N, idx,
                                                                x, out);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_blocks_transpose(int64_t nnzb, int N, const double* in,
                                    double* out, xdg_stream_t stream) {
  using namespace xdg;
  XDG_REQUIRE(N >= 1 && nnzb >= 0, XDG_ERR_ARG, "bad block shape");
  if (nnzb == 0) return XDG_OK;
  XDG_REQUIRE(in != out, XDG_ERR_ARG, "in-place transpose not supported");
  const int nn = N * N;
  const int per_tile = (4096 / nn) > 0 ? (4096 / nn) : 1;
  const size_t smem = sizeof(double) * (size_t)per_tile * nn;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (smem > 48 * 1024)
    XDG_TRY_CUDA(cudaFuncSetAttribute(blocks_transpose_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  const int64_t tiles = (nnzb + per_tile - 1) / per_tile;
  int grid = (int)(tiles < (int64_t)sm_count() * 8 ? tiles : (int64_t)sm_count() * 8);
  blocks_transpose_kernel<<<grid, kT, smem, s>>>(nnzb, N, in, out);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}
