// Vector and tall-skinny kernels of the Krylov / residual-minimisation loops
// (cutdg solvers.py:559-625 rm_step, 756-846 gmres_pmg_solve).
//
// All are HBM-bound streaming kernels; reductions are deterministic
// (fixed shuffle tree per CTA + CTA-ordered final sum, xdg_common.cuh).
#include <stdarg.h>
#include <string.h>

#include "xdg_common.cuh"

namespace xdg {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int sm_count() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) ==
            cudaSuccess && n > 0)
      cached = n;
    else
      cached = 148;
  }
  return cached;
}

namespace {

constexpr int kT = 256;
constexpr int kPerSm = 4;

__global__ void __launch_bounds__(kT)
dot_kernel(int64_t n, const double* __restrict__ x,
           const double* __restrict__ y, double* out, double* ws) {
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride)
    s = fma(__ldg(x + i), __ldg(y + i), s);
  __shared__ double red[kT / 32];
  grid_finalize(block_sum(s, red), ws, out);
}

__global__ void __launch_bounds__(kT)
axpy_kernel(int64_t n, double a, const double* __restrict__ a_dev,
            const double* __restrict__ x, double* __restrict__ y) {
  const double s = a_dev ? __dmul_rn(a, *a_dev) : a;
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride)
    y[i] = __dadd_rn(y[i], __dmul_rn(s, x[i]));
}

__global__ void __launch_bounds__(kT)
scale_kernel(int64_t n, double a, const double* __restrict__ a_dev, int invert,
             const double* __restrict__ x, double* __restrict__ y) {
  const int64_t stride = (int64_t)gridDim.x * kT;
  if (a_dev != nullptr && invert) {
    // numpy `w /= norm_w` divides every element (no reciprocal multiply)
    const double d = *a_dev;
    for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride)
      y[i] = __dmul_rn(a, __ddiv_rn(x[i], d));
    return;
  }
  if (invert) {  // host divisor: y = x / a
    for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride)
      y[i] = __ddiv_rn(x[i], a);
    return;
  }
  const double s = a_dev ? __dmul_rn(a, *a_dev) : a;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride)
    y[i] = __dmul_rn(s, x[i]);
}

// rm_step's exact-image update (solvers.py:605-607):
//   My_new = My + alpha * Mz ;  *rho2 = || r0 - My_new ||^2
__global__ void __launch_bounds__(kT)
rm_update_kernel(int64_t n, const double* __restrict__ r0,
                 const double* __restrict__ My, const double* __restrict__ Mz,
                 const double* __restrict__ alpha_dev, double* __restrict__ My_new,
                 double* rho2, double* ws) {
  const double a = *alpha_dev;
  double s = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride) {
    const double v = __dadd_rn(My[i], __dmul_rn(a, Mz[i]));
    My_new[i] = v;
    const double d = __dadd_rn(r0[i], -v);
    s = fma(d, d, s);
  }
  __shared__ double red[kT / 32];
  grid_finalize(block_sum(s, red), ws, rho2);
}

// out = x + y (elementwise) -- RmState.current(): x0 + y (solvers.py:546)
__global__ void __launch_bounds__(kT)
add_kernel(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
           double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride)
    out[i] = __dadd_rn(x[i], y[i]);
}

__global__ void __launch_bounds__(kT)
sub_kernel(int64_t n, const double* __restrict__ b,
           const double* __restrict__ y, double* __restrict__ r) {
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride)
    r[i] = __dadd_rn(b[i], -y[i]);
}

__global__ void __launch_bounds__(kT)
div_kernel(int64_t n, const double* __restrict__ x,
           const double* __restrict__ d, double* __restrict__ y) {
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride)
    y[i] = __ddiv_rn(x[i], d[i]);
}

// ---- W^T w over up to kCols columns per pass ------------------------------
// Each CTA streams a contiguous slice of the L rows; per column it forms a
// partial dot with a fixed shuffle tree and writes partial[c][cta].  A
// second, tiny kernel sums the partials per column in CTA order.
constexpr int kCols = 8;

__global__ void __launch_bounds__(kT)
gemv_t_partial(int64_t L, int ncols, const double* __restrict__ W, int64_t ldw,
               const double* __restrict__ w, double* __restrict__ partial) {
  const int64_t per = (L + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * per;
  const int64_t hi = lo + per < L ? lo + per : L;
  __shared__ double red[kCols][kT / 32];
  for (int c0 = 0; c0 < ncols; c0 += kCols) {
    double acc[kCols];
#pragma unroll
    for (int q = 0; q < kCols; ++q) acc[q] = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += kT) {
      const double wi = __ldg(w + i);
#pragma unroll
      for (int q = 0; q < kCols; ++q)
        if (c0 + q < ncols)
          acc[q] = fma(__ldg(W + (int64_t)(c0 + q) * ldw + i), wi, acc[q]);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < kCols; ++q) {
      const double v = warp_sum(acc[q]);
      if (lane == 0) red[q][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < kCols && c0 + (int)threadIdx.x < ncols) {
      double s = 0.0;
      for (int q = 0; q < kT / 32; ++q) s += red[threadIdx.x][q];
      partial[(int64_t)(c0 + threadIdx.x) * gridDim.x + blockIdx.x] = s;
    }
    __syncthreads();
  }
}

__global__ void gemv_t_final(int ncols, int nparts,
                             const double* __restrict__ partial,
                             double* __restrict__ coeff) {
  // one warp per column, fixed order
  const int c = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= ncols) return;
  double s = 0.0;
  for (int p = lane; p < nparts; p += 32) s += partial[(int64_t)c * nparts + p];
  s = warp_sum(s);
  if (lane == 0) coeff[c] = s;
}

// w -= W coeff ; z -= Z coeff.  Per element the column sum is formed in
// column order, then subtracted (numpy: tmp = W @ coeff; w -= tmp).
__global__ void __launch_bounds__(kT)
gemv_update2_kernel(int64_t L, int ncols, const double* __restrict__ W,
                    const double* __restrict__ Z, int64_t ld,
                    const double* __restrict__ coeff, double* __restrict__ w,
                    double* __restrict__ z) {
  extern __shared__ double sc[];
  for (int c = threadIdx.x; c < ncols; c += kT) sc[c] = coeff[c];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < L; i += stride) {
    double tw = 0.0, tz = 0.0;
    for (int c = 0; c < ncols; ++c) {
      tw = fma(__ldg(W + (int64_t)c * ld + i), sc[c], tw);
      if (Z) tz = fma(__ldg(Z + (int64_t)c * ld + i), sc[c], tz);
    }
    w[i] = __dadd_rn(w[i], -tw);
    if (Z) z[i] = __dadd_rn(z[i], -tz);
  }
}

int gemv_t_parts() { return sm_count() * 2; }

}  // namespace
}  // namespace xdg

using namespace xdg;

extern "C" int xdg_version(void) { return 1; }
extern "C" const char* xdg_last_error(void) { return g_err; }

extern "C" int64_t xdg_reduce_workspace_bytes(void) {
  // counter + one partial per CTA of the largest reduction grid
  return 8 * (1 + (int64_t)sm_count() * 16);
}

extern "C" int xdg_dot(int64_t n, const double* x, const double* y,
                       double* out, void* ws, xdg_stream_t stream) {
  XDG_REQUIRE(n >= 0, XDG_ERR_ARG, "negative length");
  XDG_REQUIRE(ws != nullptr, XDG_ERR_ARG, "dot needs a workspace");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  dot_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, x, y, out,
                                                     static_cast<double*>(ws));
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_axpy(int64_t n, double a, const double* a_dev,
                        const double* x, double* y, xdg_stream_t stream) {
  if (n <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  axpy_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, a, a_dev, x, y);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_scale(int64_t n, double a, const double* a_dev, int invert,
                         const double* x, double* y, xdg_stream_t stream) {
  if (n <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  scale_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, a, a_dev, invert, x,
                                                       y);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_rm_update(int64_t n, const double* r0, const double* My,
                             const double* Mz, const double* alpha_dev,
                             double* My_new, double* rho2, void* ws,
                             xdg_stream_t stream) {
  XDG_REQUIRE(ws != nullptr, XDG_ERR_ARG, "rm_update needs a workspace");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  rm_update_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(
      n, r0, My, Mz, alpha_dev, My_new, rho2, static_cast<double*>(ws));
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_add(int64_t n, const double* x, const double* y,
                       double* out, xdg_stream_t stream) {
  if (n <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  add_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, x, y, out);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_sub(int64_t n, const double* b, const double* y, double* r,
                       xdg_stream_t stream) {
  if (n <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  sub_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, b, y, r);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_div(int64_t n, const double* x, const double* d, double* y,
                       xdg_stream_t stream) {
  if (n <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  div_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, x, d, y);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int64_t xdg_gemv_t_workspace_bytes(int ncols) {
  return 8 * (int64_t)(ncols > 0 ? ncols : 1) * gemv_t_parts();
}

extern "C" int xdg_gemv_t(int64_t L, int ncols, const double* W, int64_t ldw,
                          const double* w, double* coeff, void* ws,
                          xdg_stream_t stream) {
  XDG_REQUIRE(L >= 0 && ncols >= 0 && ldw >= L, XDG_ERR_ARG,
              "gemv_t: bad shape L=%lld ncols=%d ldw=%lld", (long long)L, ncols,
              (long long)ldw);
  if (ncols == 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int parts = gemv_t_parts();
  if (L < (int64_t)parts * kT) parts = (int)((L + kT - 1) / kT);
  if (parts < 1) parts = 1;
  double* partial = static_cast<double*>(ws);
  gemv_t_partial<<<parts, kT, 0, s>>>(L, ncols, W, ldw, w, partial);
  XDG_CHECK_LAUNCH();
  gemv_t_final<<<(ncols + 7) / 8, 256, 0, s>>>(ncols, parts, partial, coeff);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_gemv_update2(int64_t L, int ncols, const double* W,
                                const double* Z, int64_t ld,
                                const double* coeff, double* w, double* z,
                                xdg_stream_t stream) {
  XDG_REQUIRE(L >= 0 && ncols >= 0 && ld >= L, XDG_ERR_ARG,
              "gemv_update2: bad shape");
  if (ncols == 0 || L == 0) return XDG_OK;
  XDG_REQUIRE(ncols <= 6000, XDG_ERR_ARG, "gemv_update2: ncols %d too large",
              ncols);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  gemv_update2_kernel<<<grid_for(L, kT, kPerSm), kT, ncols * sizeof(double),
                        s>>>(L, ncols, W, Z, ld, coeff, w, z);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}
