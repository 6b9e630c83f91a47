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

// One MGS step of the distributed GMRES (solvers.py:802-805) in one pass:
// y += c x with c = a * (*a_dev), then *out = sum_i v_i y_i (v == NULL:
// sum y_i^2) -- the axpy of step i fused with the dot of step i + 1, with
// the rounding of the single-GPU cooperative mgs_kernel.
__global__ void __launch_bounds__(kT)
axpy_dot_kernel(int64_t n, double a, const double* __restrict__ a_dev,
                const double* __restrict__ x, double* y, const double* v, double* out,
                double* ws) {
  const double c = a_dev ? __dmul_rn(a, *a_dev) : a;
  double t = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += stride) {
    const double yi = __dadd_rn(y[i], __dmul_rn(c, x[i]));
    y[i] = yi;
    t = v ? fma(v[i], yi, t) : fma(yi, yi, t);
  }
  __shared__ double red[kT / 32];
  grid_finalize(block_sum(t, red), ws, out);
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

// ---- W^T w -------------------------------------------------------------------
// Each CTA owns a tile of kTile rows: w's tile is staged in shared memory,
// warp j handles columns j, j+8, ...; for a column every lane issues
// kTile/32 independent coalesced loads, reduces them in a fixed order and
// the warp tree writes partial[c][tile].  gemv_t_final sums the tile
// partials per column in tile order (deterministic).
constexpr int kTile = 1024;
constexpr int kMaxTiles = 4096;

__global__ void __launch_bounds__(kT)
gemv_t_partial(int64_t L, int ncols, const double* __restrict__ W, int64_t ldw,
               const double* __restrict__ w, double* __restrict__ partial,
               const int* __restrict__ ncols_dev) {
  __shared__ double ws[kTile];
  if (ncols_dev) ncols = min(ncols, *ncols_dev);  // device-resident column count
  if (ncols <= 0) return;
  const int ntiles = gridDim.x;
  const int64_t rows_per = ((L + ntiles - 1) / ntiles + 31) / 32 * 32;
  const int64_t lo = (int64_t)blockIdx.x * rows_per;
  const int64_t hi = lo + rows_per < L ? lo + rows_per : L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t t0 = lo; t0 < hi; t0 += kTile) {
    const int len = (int)((hi - t0) < kTile ? (hi - t0) : kTile);
    __syncthreads();
    for (int i = threadIdx.x; i < kTile; i += kT) ws[i] = i < len ? w[t0 + i] : 0.0;
    __syncthreads();
    for (int c = warp; c < ncols; c += kT / 32) {
      const double* Wc = W + (int64_t)c * ldw + t0;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      if (len == kTile) {
#pragma unroll 8
        for (int k = 0; k < kTile / 32; k += 4) {
          const int i = lane + 32 * k;
          a0 = fma(__ldg(Wc + i), ws[i], a0);
          a1 = fma(__ldg(Wc + i + 32), ws[i + 32], a1);
          a2 = fma(__ldg(Wc + i + 64), ws[i + 64], a2);
          a3 = fma(__ldg(Wc + i + 96), ws[i + 96], a3);
        }
      } else {
        for (int i = lane; i < len; i += 32) a0 = fma(__ldg(Wc + i), ws[i], a0);
      }
      const double v = warp_sum((a0 + a1) + (a2 + a3));
      if (lane == 0) {
        double* pc = partial + (int64_t)c * ntiles + blockIdx.x;
        *pc = (t0 == lo) ? v : *pc + v;
      }
    }
  }
}

__global__ void gemv_t_final(int ncols, int nparts,
                             const double* __restrict__ partial,
                             double* __restrict__ coeff, const int* __restrict__ ncols_dev) {
  // one warp per column, fixed order
  if (ncols_dev) ncols = min(ncols, *ncols_dev);
  const int c = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= ncols) return;
  double s = 0.0;
  for (int p = lane; p < nparts; p += 32) s += partial[(int64_t)c * nparts + p];
  s = warp_sum(s);
  if (lane == 0) coeff[c] = s;
}

// w -= W cw ; z -= Z cz.  Per element the column sum is formed in column
// order (4 columns' loads issued together), then subtracted
// (numpy: tmp = W @ coeff; w -= tmp).
__global__ void __launch_bounds__(kT)
gemv_update2_kernel(int64_t L, int ncols, const double* __restrict__ W,
                    const double* __restrict__ Z, int64_t ld,
                    const double* __restrict__ cw, const double* __restrict__ cz,
                    double* __restrict__ w, double* __restrict__ z,
                    const int* __restrict__ ncols_dev) {
  extern __shared__ double sc[];
  if (ncols_dev) ncols = min(ncols, *ncols_dev);
  if (ncols <= 0) return;  // uniform: no column, no update
  double* scw = sc;
  double* scz = sc + ncols;
  for (int c = threadIdx.x; c < ncols; c += kT) {
    scw[c] = cw[c];
    scz[c] = cz[c];
  }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < L; i += stride) {
    double tw = 0.0, tz = 0.0;
    int c = 0;
    for (; c + 4 <= ncols; c += 4) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = __ldg(W + (int64_t)(c + u) * ld + i);
        b[u] = Z ? __ldg(Z + (int64_t)(c + u) * ld + i) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        tw = fma(a[u], scw[c + u], tw);
        if (Z) tz = fma(b[u], scz[c + u], tz);
      }
    }
    for (; c < ncols; ++c) {
      tw = fma(__ldg(W + (int64_t)c * ld + i), scw[c], tw);
      if (Z) tz = fma(__ldg(Z + (int64_t)c * ld + i), scz[c], tz);
    }
    w[i] = __dadd_rn(w[i], -tw);
    if (Z) z[i] = __dadd_rn(z[i], -tz);
  }
}

__global__ void add_small_kernel(int n, const double* a, const double* b, double* out,
                                 const int* n_dev) {
  if (n_dev) n = min(n, *n_dev);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = a[i] + b[i];
}

int gemv_t_parts(int64_t L) {
  int64_t t = (L + kTile - 1) / kTile;
  if (t > kMaxTiles) t = kMaxTiles;
  return t < 1 ? 1 : (int)t;
}

}  // namespace
}  // namespace xdg

using namespace xdg;

extern "C" int xdg_version(void) { return 1; }

extern "C" int xdg_struct_sizes(int64_t* out, int n) {
  const int64_t sz[] = {(int64_t)sizeof(xdg_bsr),     (int64_t)sizeof(xdg_pmg),
                        (int64_t)sizeof(xdg_direct),  (int64_t)sizeof(xdg_rm),
                        (int64_t)sizeof(xdg_omg_level), (int64_t)sizeof(xdg_mf),
                        (int64_t)sizeof(xdg_mf_node)};
  const int k = (int)(sizeof(sz) / sizeof(sz[0]));
  for (int i = 0; i < n && i < k; ++i) out[i] = sz[i];
  return k;
}
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

extern "C" int xdg_axpy_dot(int64_t n, double a, const double* a_dev, const double* x,
                            double* y, const double* v, double* out, void* ws,
                            xdg_stream_t stream) {
  XDG_REQUIRE(n >= 0 && ws != nullptr, XDG_ERR_ARG, "axpy_dot: bad length or workspace");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  axpy_dot_kernel<<<grid_for(n, kT, kPerSm), kT, 0, s>>>(n, a, a_dev, x, y, v, out,
                                                          static_cast<double*>(ws));
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
  return 8 * (int64_t)(ncols > 0 ? ncols : 1) * kMaxTiles;
}

extern "C" int xdg_gemv_t(int64_t L, int ncols, const double* W, int64_t ldw,
                          const double* w, double* coeff, void* ws,
                          xdg_stream_t stream) {
  XDG_REQUIRE(L >= 0 && ncols >= 0 && ldw >= L, XDG_ERR_ARG,
              "gemv_t: bad shape L=%lld ncols=%d ldw=%lld", (long long)L, ncols,
              (long long)ldw);
  if (ncols == 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int parts = gemv_t_parts(L);
  double* partial = static_cast<double*>(ws);
  gemv_t_partial<<<parts, kT, 0, s>>>(L, ncols, W, ldw, w, partial, nullptr);
  XDG_CHECK_LAUNCH();
  gemv_t_final<<<(ncols + 7) / 8, 256, 0, s>>>(ncols, parts, partial, coeff, nullptr);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_gemv_update2(int64_t L, int ncols, const double* W,
                                const double* Z, int64_t ld,
                                const double* coeff, const double* coeff_z,
                                double* w, double* z, xdg_stream_t stream) {
  XDG_REQUIRE(L >= 0 && ncols >= 0 && ld >= L, XDG_ERR_ARG,
              "gemv_update2: bad shape");
  if (ncols == 0 || L == 0) return XDG_OK;
  XDG_REQUIRE(ncols <= 6000, XDG_ERR_ARG, "gemv_update2: ncols %d too large",
              ncols);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t smem = 2 * ncols * sizeof(double);
  if (smem > 48 * 1024)
    XDG_TRY_CUDA(cudaFuncSetAttribute(gemv_update2_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  gemv_update2_kernel<<<grid_for(L, kT, kPerSm), kT, smem, s>>>(
      L, ncols, W, Z, ld, coeff, coeff_z ? coeff_z : coeff, w, z, nullptr);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

extern "C" int xdg_add_small(int n, const double* a, const double* b,
                             double* out, xdg_stream_t stream) {
  if (n <= 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  add_small_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, a, b, out, nullptr);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

// ---------------------------------------------------------------------------
// Device-resident column counts (the graph-captured ortho_mg_solve: the RM
// space's column count lives on the device; launches are sized for
// max_cols and the kernels read the actual count).  Same grids and the same
// arithmetic as the host-count entry points above: bit-identical results.
namespace xdg {

int gemv_t_dev(int64_t L, int max_cols, const int* ncols_dev, const double* W, int64_t ldw,
               const double* w, double* coeff, void* ws, cudaStream_t s) {
  if (max_cols <= 0 || L <= 0) return XDG_OK;
  const int parts = gemv_t_parts(L);
  double* partial = static_cast<double*>(ws);
  gemv_t_partial<<<parts, kT, 0, s>>>(L, max_cols, W, ldw, w, partial, ncols_dev);
  XDG_CHECK_LAUNCH();
  gemv_t_final<<<(max_cols + 7) / 8, 256, 0, s>>>(max_cols, parts, partial, coeff, ncols_dev);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

int gemv_update2_dev(int64_t L, int max_cols, const int* ncols_dev, const double* W,
                     const double* Z, int64_t ld, const double* cw, const double* cz,
                     double* w, double* z, cudaStream_t s) {
  if (max_cols <= 0 || L <= 0) return XDG_OK;
  XDG_REQUIRE(max_cols <= 6000, XDG_ERR_ARG, "gemv_update2: ncols %d too large", max_cols);
  const size_t smem = 2 * max_cols * sizeof(double);
  if (smem > 48 * 1024)
    XDG_TRY_CUDA(cudaFuncSetAttribute(gemv_update2_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gemv_update2_kernel<<<grid_for(L, kT, kPerSm), kT, smem, s>>>(L, max_cols, W, Z, ld, cw,
                                                                cz ? cz : cw, w, z, ncols_dev);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

int add_small_dev(int max_n, const int* n_dev, const double* a, const double* b, double* out,
                  cudaStream_t s) {
  if (max_n <= 0) return XDG_OK;
  add_small_kernel<<<(max_n + 255) / 256, 256, 0, s>>>(max_n, a, b, out, n_dev);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

}  // namespace xdg
