// Multifrontal sparse LU solves (nested-dissection elimination forest) for
// the low-order PMG systems, the Schwarz blocks' low-order systems and large
// direct / coarsest-level solves -- the systems the reference factors with
// SuperLU (cutdg blockmatrix.py:203-227 splu/solve; solvers.py:208-221,
// 249-251, 661-666, 698-710).
//
// Setup (multifrontal.py): nested dissection of each system's block graph
// into a forest of fronts; front t eliminates its pivot unknowns P_t
// (partial pivoting inside P_t) against its boundary B_t (ancestor
// separators).  Stored per front: INV_t (L^-1 strictly below the diagonal,
// U^-1 on/above it, p x p), L_BP = F_BP U^-1 (b x p), U_PB = L^-1 P F_PB
// (p x b), all row-major with padded leading dimensions.
//
// Solve, level by level (height h = 0 .. H-1 forward, H-1 .. 0 backward),
// every front of a level in one launch, warp per row:
//   F1 gather   W_t[i] = b[src] + sum of the children's contributions
//               (fixed order: deterministic), P part in pivot order
//   F2 lower    Y_t   = L^-1 W_t[P]                 (triangular GEMV)
//   F3 bound    C_t   = W_t[B] - L_BP Y_t           (contribution to parent)
//   B1 upb      T_t   = Y_t - U_PB x[B_t]           (x of ancestors)
//   B2 upper    x[P_t] = U^-1 T_t
// with the symmetric equilibration S folded in (b scaled in F1, x in B2).
// Bound: HBM -- each apply streams every stored factor once
// (8 (p^2 + 2 p b) bytes per front); no sequential substitution chains.
#include <algorithm>

#include "xdg_common.cuh"
#include "xdg_dmma.cuh"

namespace xdg {
namespace {

constexpr int kT = 256;

// Programmatic dependent launch for the level chain (gather_h -> rows_h ->
// gather_{h+1} ...): every launch of a sweep depends on the previous one only
// through the small vectors W / Y / C / X; tasks, nodes and the factor F are
// read-only.  Unless XDG_MF_PDL=0, a kernel lets its successor's CTAs become
// resident at once (launch_dependents) and the successor fetches its first
// descriptors (and touches its first factor rows) before it waits for the
// predecessor's stores (griddepcontrol.wait): the launch ramp and the
// descriptor -> node chain overlap the predecessor's tail.
bool mf_pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("XDG_MF_PDL");
    return e == nullptr || atoi(e) != 0;  // default on: cfg2 low-order solve 2.52 -> 2.42 ms
  }();
  return on;
}
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
template <typename... KArgs, typename... Args>
cudaError_t launch_chain(void (*kernel)(KArgs...), int grid, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kT);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = mf_pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, KArgs(args)...);
}

// Sub-warp row dots.  A warp task covers 32/G consecutive rows of one
// front, G lanes per row (G = power of two chosen per front from the row
// length, so short rows still keep the whole warp's loads in flight and long
// rows get the whole warp).  Lanes of a group stride G through the row, 8
// loads in flight per lane, fixed accumulation order; the group sum is a
// shuffle-xor tree inside the aligned group (deterministic).
#ifndef MF_U
#define MF_U 8  // loads in flight per lane per chunk
#endif
#ifndef MF_MINB
// resident CTAs per SM the row kernels are compiled for.  Measured with the
// PDL chain (cfg2 low-order solve, profiles/r2_mf_variants*.txt; MINB x rows
// per warp task x loads in flight): 3 x 2 x 8 2.42 ms, 2 x 3 x 8 2.23 ms,
// 2 x 4 x 8 2.34, 2 x 4 x 12 2.32, 2 x 3 x 6/10/12 2.31-2.32, 3 x 3 x 8 2.47,
// 4 x 2 x 8 3.38 (spills): three rows share each vector load and 128
// registers keep 24 factor loads per lane in flight.
#define MF_MINB 2
#endif

template <typename V>
__device__ __forceinline__ double group_dot(const double* __restrict__ row, V v,
                                            int j0, int j1, int gl, int G,
                                            bool active) {
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  if (active) {
    const int step = MF_U * G;
    for (int jb = j0; jb < j1; jb += step) {
      // clamped (always valid) unpredicated loads, so all of them are
      // issued before the first FMA; out-of-row lanes are zeroed afterwards
      double r[MF_U], q[MF_U];
#pragma unroll
      for (int u = 0; u < MF_U; ++u) {
        const int j = min(jb + gl + G * u, j1 - 1);
        r[u] = __ldg(row + j);
        q[u] = v(j);
      }
#pragma unroll
      for (int u = 0; u < MF_U; ++u)
        if (jb + gl + G * u >= j1) r[u] = 0.0;
#pragma unroll
      for (int u = 0; u < MF_U; ++u) a[u & 3] = fma(r[u], q[u], a[u & 3]);
    }
  }
  double s = (a[0] + a[1]) + (a[2] + a[3]);
  for (int o = 16; o > 0; o >>= 1)
    if (o < G) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// Two rows per lane group (row sets a and b of a two-set task) of the bound
// or upb phase, whose rows all span the same columns [0, n): one vector load
// per element serves both rows, and both rows' factor loads are issued
// together (2 x MF_U per lane in flight).  Each row keeps group_dot's
// chunking and accumulation order: bit-identical to two group_dot calls.
template <typename V>
__device__ __forceinline__ void group_dot2(const double* __restrict__ ra,
                                           const double* __restrict__ rb, V v, int j1,
                                           int gl, int G, bool acta, bool actb, double& da,
                                           double& db) {
  double x[4] = {0.0, 0.0, 0.0, 0.0}, y[4] = {0.0, 0.0, 0.0, 0.0};
  if (acta && j1 > 0) {
    const int step = MF_U * G;
    const double* rbb = actb ? rb : ra;
    for (int jb = 0; jb < j1; jb += step) {
      double p[MF_U], s[MF_U], q[MF_U];
#pragma unroll
      for (int u = 0; u < MF_U; ++u) {
        const int j = min(jb + gl + G * u, j1 - 1);
        p[u] = __ldg(ra + j);
        s[u] = __ldg(rbb + j);
        q[u] = v(j);
      }
#pragma unroll
      for (int u = 0; u < MF_U; ++u)
        if (jb + gl + G * u >= j1) q[u] = 0.0;
#pragma unroll
      for (int u = 0; u < MF_U; ++u) {
        x[u & 3] = fma(p[u], q[u], x[u & 3]);
        y[u & 3] = fma(s[u], q[u], y[u & 3]);
      }
    }
  }
  double sa = (x[0] + x[1]) + (x[2] + x[3]);
  double sb = (y[0] + y[1]) + (y[2] + y[3]);
  for (int o = 16; o > 0; o >>= 1)
    if (o < G) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
  da = sa;
  db = actb ? sb : 0.0;
}

// MR rows of one front against the same vector (whole warp, lanes stride
// 32): the vector is loaded once for all of them, so MU vector + MR*MU
// factor loads are in flight per lane.  Row q covers [r0[q], r1[q]) inside
// [lo, hi); loads are clamped to hi - 1 (inside the padded rows) and masked.
// Used for fronts whose rows get a whole warp (G = 32).
#ifndef MF_MR
#define MF_MR 3
#endif
#ifndef MF_MU
#define MF_MU 8
#endif
constexpr int kMR = MF_MR;
constexpr int kMU = MF_MU;

template <typename V>
__device__ __forceinline__ void multi_dot(const double* const* rows, V v, int lo, int hi,
                                          const int* r0, const int* r1, int lane, double* d) {
  double acc[kMR][2];
#pragma unroll
  for (int q = 0; q < kMR; ++q) acc[q][0] = acc[q][1] = 0.0;
  for (int jb = lo; jb < hi; jb += 32 * kMU) {
    double m[kMR][kMU], x[kMU];
    typename V::index_t ix[kMU];
#pragma unroll
    for (int u = 0; u < kMU; ++u) ix[u] = v.idx(min(jb + lane + 32 * u, hi - 1));
#pragma unroll
    for (int u = 0; u < kMU; ++u) {
      const int j = min(jb + lane + 32 * u, hi - 1);
#pragma unroll
      for (int q = 0; q < kMR; ++q) m[q][u] = __ldg(rows[q] + j);
    }
#pragma unroll
    for (int u = 0; u < kMU; ++u) x[u] = v.at(ix[u]);
#pragma unroll
    for (int u = 0; u < kMU; ++u) {
      const int j = jb + lane + 32 * u;
#pragma unroll
      for (int q = 0; q < kMR; ++q) {
        const double xq = (j >= r0[q] && j < r1[q]) ? x[u] : 0.0;
        acc[q][u & 1] = fma(m[q][u], xq, acc[q][u & 1]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kMR; ++q) d[q] = warp_sum(acc[q][0] + acc[q][1]);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Vector accessors.  idx(j) / at(i) split an element access in two so the
// loops can issue every index load of a chunk, then the factor loads, then
// the (dependent) vector loads: a gathered element costs one extra round
// trip per chunk, not one per element.
struct Direct {
  const double* p;
  typedef int index_t;
  __device__ __forceinline__ double operator()(int j) const { return p[j]; }
  __device__ __forceinline__ int idx(int j) const { return j; }
  __device__ __forceinline__ double at(int i) const { return p[i]; }
};

struct Gathered {
  const double* x;
  const int64_t* ix;
  typedef int64_t index_t;
  __device__ __forceinline__ double operator()(int j) const { return x[ix[j]]; }
  __device__ __forceinline__ int64_t idx(int j) const { return __ldg(ix + j); }
  __device__ __forceinline__ double at(int64_t i) const { return x[i]; }
};

// Task g of n in interleaved order (long and short rows mix on every SM).
__device__ __forceinline__ int64_t interleave(int64_t w, int64_t n) {
  return (w & 1) ? n - 1 - (w >> 1) : (w >> 1);
}

__global__ void __launch_bounds__(kT)
mf_gather_kernel(int64_t e0, int64_t e1, const int64_t* __restrict__ ent_w,
                 const int64_t* __restrict__ ent_src,
                 const int64_t* __restrict__ ent_cptr,
                 const int64_t* __restrict__ ent_cidx,
                 const double* __restrict__ ent_scale,
                 const double* __restrict__ b, const double* __restrict__ C,
                 double* __restrict__ W) {
  pdl_trigger();
  // the entry lists are static: the first entry's descriptors are loaded
  // before the wait for the previous launch's C (and for b)
  int64_t e = e0 + (int64_t)blockIdx.x * kT + threadIdx.x;
  int64_t s = -1, k0 = 0, k1 = 0, wi = 0;
  double sc = 0.0;
  if (e < e1) {
    s = ent_src[e];
    sc = ent_scale[e];
    k0 = ent_cptr[e];
    k1 = ent_cptr[e + 1];
    wi = ent_w[e];
  }
  pdl_wait();
  while (e < e1) {
    double v = s >= 0 ? __dmul_rn(sc, b[s]) : 0.0;
    for (int64_t k = k0; k < k1; ++k) v = __dadd_rn(v, C[ent_cidx[k]]);
    W[wi] = v;
    e += (int64_t)gridDim.x * kT;
    if (e < e1) {
      s = ent_src[e];
      sc = ent_scale[e];
      k0 = ent_cptr[e];
      k1 = ent_cptr[e + 1];
      wi = ent_w[e];
    }
  }
}

enum Phase { kLower = 0, kBound = 1, kUpb = 2, kUpper = 3 };

// The four row phases (p = pivot unknowns, b = boundary unknowns of a front):
//   kLower  Y[i]  = W[i] + L^-1[i, :i] . W[:i]              rows: P, G = gp
//   kBound  C[j]  = W[p+j] - L_BP[j, :] . Y                  rows: B, G = gp
//   kUpb    W[i]  = Y[i] - U_PB[i, :] . Y[bidx]              rows: P, G = gb
//   kUpper  Y[i] = U^-1[i, i:] . W[i:], x[pdst[i]] = s_i Y[i] rows: P, G = gp
// (in the backward sweep Y holds the equilibrated solution of the fronts
// already solved: the ancestors' values the U_PB rows read through bidx)
struct Ctx {
  const xdg_mf_node* nodes;
  const double* F;
  const int64_t* bidx;
  const int64_t* pdst;
  const double* pscale;
  double* W;
  double* Y;
  double* C;
  double* x;
  double* X;
};

template <int PH>
__device__ __forceinline__ void row_span(const xdg_mf_node& nd, int r, int& j0, int& j1) {
  j0 = (PH == kUpper) ? r : 0;
  j1 = (PH == kLower) ? r : (PH == kUpb ? nd.b : nd.p);
}

template <int PH>
__device__ __forceinline__ double row_part(const Ctx& c, const xdg_mf_node& nd, int r,
                                           int js, int je, int gl, int G, bool act) {
  if (PH == kLower)
    return group_dot(c.F + nd.inv + (int64_t)r * nd.ldp, Direct{c.W + nd.w}, js, je, gl, G,
                     act);
  if (PH == kBound)
    return group_dot(c.F + nd.lbp + (int64_t)r * nd.ldp, Direct{c.Y + nd.y}, js, je, gl, G,
                     act);
  if (PH == kUpb)
    return group_dot(c.F + nd.upb + (int64_t)r * nd.ldb, Gathered{c.Y, c.bidx + nd.bx}, js,
                     je, gl, G, act);
  return group_dot(c.F + nd.inv + (int64_t)r * nd.ldp, Direct{c.W + nd.w}, js, je, gl, G,
                   act);
}

template <int PH>
__device__ __forceinline__ void row_part2(const Ctx& c, const xdg_mf_node& nd, int ra,
                                          int rb, int gl, int G, bool acta, bool actb,
                                          double& da, double& db) {
  const int64_t mat = (PH == kBound) ? nd.lbp : nd.upb;
  const int ld = (PH == kUpb) ? nd.ldb : nd.ldp;
  const double* pa = c.F + mat + (int64_t)ra * ld;
  const double* pb = c.F + mat + (int64_t)rb * ld;
  if (PH == kUpb)
    group_dot2(pa, pb, Gathered{c.Y, c.bidx + nd.bx}, nd.b, gl, G, acta, actb, da, db);
  else
    group_dot2(pa, pb, Direct{c.Y + nd.y}, nd.p, gl, G, acta, actb, da, db);
}

template <int PH>
__device__ __forceinline__ void row_done(const Ctx& c, const xdg_mf_node& nd, int r,
                                         double d) {
  if (PH == kLower) c.Y[nd.y + r] = __dadd_rn(c.W[nd.w + r], d);
  if (PH == kBound) c.C[nd.c + r] = __dsub_rn(c.W[nd.w + nd.p + r], d);
  if (PH == kUpb) c.W[nd.w + r] = __dsub_rn(c.Y[nd.y + r], d);
  if (PH == kUpper) {
    c.Y[nd.y + r] = d;
    c.x[c.pdst[nd.px + r]] = __dmul_rn(c.pscale[nd.px + r], d);
  }
}

// Warp tasks (node, row, nrows, -1): fronts whose rows take a whole warp
// (G = 32) get kMR rows per task (multi_dot, shared vector loads); shorter
// rows get 32/G rows per task, G lanes each (nrows field 0).
template <int PH>
__device__ __forceinline__ void run_task(const Ctx& c, const int4 tk, const int lane) {
    const xdg_mf_node nd = c.nodes[tk.x];
    if (tk.z == kMR) {  // kMR rows r, r + 1, ... of a G = 32 front
      const int r = tk.y;
      const int nrows = (PH == kBound) ? nd.b : nd.p;
      const double* rows[kMR];
      int r0[kMR], r1[kMR];
      int lo = 1 << 30, hi = 0;
      const int64_t mat = (PH == kBound) ? nd.lbp : (PH == kUpb ? nd.upb : nd.inv);
      const int ld = (PH == kUpb) ? nd.ldb : nd.ldp;
#pragma unroll
      for (int q = 0; q < kMR; ++q) {
        const int rq = min(r + q, nrows - 1);
        rows[q] = c.F + mat + (int64_t)rq * ld;
        row_span<PH>(nd, rq, r0[q], r1[q]);
        if (r + q >= nrows) r1[q] = r0[q];  // past the front: empty row
        if (r1[q] > r0[q]) {
          lo = min(lo, r0[q]);
          hi = max(hi, r1[q]);
        }
      }
      double d[kMR];
#pragma unroll
      for (int q = 0; q < kMR; ++q) d[q] = 0.0;
      if (hi > lo) {
        if (PH == kUpb)
          multi_dot(rows, Gathered{c.Y, c.bidx + nd.bx}, lo, hi, r0, r1, lane, d);
        else
          multi_dot(rows, Direct{(PH == kBound) ? c.Y + nd.y : c.W + nd.w}, lo, hi, r0, r1,
                    lane, d);
      }
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < kMR; ++q)
          if (r + q < nrows) row_done<PH>(c, nd, r + q, d[q]);
      }
    } else if ((PH == kBound || PH == kUpb) && tk.z == -2) {
      // two row sets of 32/G rows: rows a and b = a + 32/G share the vector
      const int G = (PH == kUpb) ? nd.gb : nd.gp;
      const int gl = lane & (G - 1);
      const int ra = tk.y + lane / G, rb = ra + 32 / G;
      const int nrows = (PH == kBound) ? nd.b : nd.p;
      const bool acta = ra < nrows, actb = rb < nrows;
      double da, db;
      row_part2<PH>(c, nd, acta ? ra : 0, actb ? rb : 0, gl, G, acta, actb, da, db);
      if (acta && gl == 0) row_done<PH>(c, nd, ra, da);
      if (actb && gl == 0) row_done<PH>(c, nd, rb, db);
    } else {
      const int G = (PH == kUpb) ? nd.gb : nd.gp;
      const int gl = lane & (G - 1);
      const int r = tk.y + lane / G;
      const int nrows = (PH == kBound) ? nd.b : nd.p;
      const bool act = r < nrows;
      int j0 = 0, j1 = 0;
      if (act) row_span<PH>(nd, r, j0, j1);
      const double d = row_part<PH>(c, nd, r, j0, j1, gl, G, act && j1 > j0);
      if (act && gl == 0) row_done<PH>(c, nd, r, d);
    }
}

template <int PH>
__global__ void __launch_bounds__(kT, MF_MINB)
mf_rows_kernel(int64_t t0, int64_t ntasks, const int4* __restrict__ tasks, Ctx c) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (kT / 32);
  for (int64_t w = (int64_t)blockIdx.x * (kT / 32) + (threadIdx.x >> 5); w < ntasks;
       w += nw)
    run_task<PH>(c, tasks[t0 + interleave(w, ntasks)], lane);
}

// ---------------------------------------------------------------------------
// Merged phases (xdg_mf.merged): the factors are stored as
//   M_BP = L_BP L^-1   (b x p)   and   N_PB = U^-1 U_PB   (p x b)
// (products formed once at setup, xdg_mf_merge; same bytes as L_BP / U_PB),
// so that neither sweep has a phase that waits for the triangular solve of
// its own front:
//   forward   Y[i]  = W[i] + L^-1[i, :i] . W[:i]        rows 0 .. p-1
//             C[j]  = W[p+j] - M_BP[j, :] . W[:p]       rows p .. p+b-1
//   backward  X[i]  = U^-1[i, i:] . Y[i:] - N_PB[i, :] . X[bidx]
// One row launch per height and sweep (was two), every row of a front reads
// the same vector, and the short triangular rows share their launch with
// the long rectangular ones.  X is the equilibrated solution (Y keeps the
// forward result: rows of the same launch still read it).

// Rows a and b (lane group of G lanes, ranges [sa, ea) and [sb, eb) of the
// same vector): the vector element is loaded once for both rows, all loads
// of a chunk are issued before the first FMA.  Loads are clamped to hi - 1
// (inside the padded rows) and masked.
template <typename V>
__device__ __forceinline__ void group_dot2r(const double* __restrict__ ra,
                                            const double* __restrict__ rb, V v, int sa, int ea,
                                            int sb, int eb, int gl, int G, double& da,
                                            double& db) {
  double x[4] = {0.0, 0.0, 0.0, 0.0}, y[4] = {0.0, 0.0, 0.0, 0.0};
  const int lo = min(ea > sa ? sa : (1 << 30), eb > sb ? sb : (1 << 30));
  const int hi = max(ea > sa ? ea : 0, eb > sb ? eb : 0);
  if (hi > lo) {
    const int step = MF_U * G;
    for (int jb = lo; jb < hi; jb += step) {
      double p[MF_U], s[MF_U], q[MF_U];
      typename V::index_t ix[MF_U];
#pragma unroll
      for (int u = 0; u < MF_U; ++u) ix[u] = v.idx(min(jb + gl + G * u, hi - 1));
#pragma unroll
      for (int u = 0; u < MF_U; ++u) {
        const int j = min(jb + gl + G * u, hi - 1);
        p[u] = __ldg(ra + j);
        s[u] = __ldg(rb + j);
      }
#pragma unroll
      for (int u = 0; u < MF_U; ++u) q[u] = v.at(ix[u]);
#pragma unroll
      for (int u = 0; u < MF_U; ++u) {
        const int j = jb + gl + G * u;
        const double qa = (j >= sa && j < ea) ? q[u] : 0.0;
        const double qb = (j >= sb && j < eb) ? q[u] : 0.0;
        x[u & 3] = fma(p[u], qa, x[u & 3]);
        y[u & 3] = fma(s[u], qb, y[u & 3]);
      }
    }
  }
  double sa_ = (x[0] + x[1]) + (x[2] + x[3]);
  double sb_ = (y[0] + y[1]) + (y[2] + y[3]);
  for (int o = 16; o > 0; o >>= 1)
    if (o < G) {
      sa_ += __shfl_xor_sync(0xffffffffu, sa_, o);
      sb_ += __shfl_xor_sync(0xffffffffu, sb_, o);
    }
  da = sa_;
  db = sb_;
}

// forward row r of a front: pointer and length (the vector is W[w .. w+p))
__device__ __forceinline__ const double* fwd_row(const Ctx& c, const xdg_mf_node& nd, int r,
                                                 int& len) {
  if (r < nd.p) {
    len = r;
    return c.F + nd.inv + (int64_t)r * nd.ldp;
  }
  len = nd.p;
  return c.F + nd.lbp + (int64_t)(r - nd.p) * nd.ldp;
}

__device__ __forceinline__ void fwd_done(const Ctx& c, const xdg_mf_node& nd, int r, double d) {
  if (r < nd.p)
    c.Y[nd.y + r] = __dadd_rn(c.W[nd.w + r], d);
  else
    c.C[nd.c + (r - nd.p)] = __dsub_rn(c.W[nd.w + r], d);
}

__device__ __forceinline__ void fwd_store(const Ctx& c, const xdg_mf_node& nd, int r, double w,
                                          double d) {
  if (r < nd.p)
    c.Y[nd.y + r] = __dadd_rn(w, d);
  else
    c.C[nd.c + (r - nd.p)] = __dsub_rn(w, d);
}

__device__ __forceinline__ void bwd_done(const Ctx& c, const xdg_mf_node& nd, int r, double du,
                                         double dn) {
  const double d = __dsub_rn(du, dn);
  c.X[nd.y + r] = d;
  c.x[c.pdst[nd.px + r]] = __dmul_rn(c.pscale[nd.px + r], d);
}

// kMR consecutive rows r .. of one front over the chunks (j_off, j_step):
// d = the U^-1 / L^-1 / M_BP part, e = the N_PB part (backward only).
// this warp's share [lo + (hi-lo) w/n, lo + (hi-lo) (w+1)/n) of a range,
// cut at multiples of 32 elements (shares equal in bytes: the warps of a
// CTA task finish together)
__device__ __forceinline__ void warp_share(int& lo, int& hi, int w, int n) {
  if (n == 1 || hi <= lo) return;
  const int len = hi - lo;
  const int a = lo + (int)(((int64_t)len * w / n) & ~31LL);
  const int b = (w == n - 1) ? hi : lo + (int)(((int64_t)len * (w + 1) / n) & ~31LL);
  lo = a;
  hi = b;
}

template <bool FWD>
__device__ __forceinline__ void merged_rows(const Ctx& c, const xdg_mf_node& nd, int r,
                                            int nrows, int lane, int w, int nw, double* d,
                                            double* e) {
  const double* rows[kMR];
  int r0[kMR], r1[kMR];
  int lo = 1 << 30, hi = 0;
#pragma unroll
  for (int q = 0; q < kMR; ++q) {
    const int rq = min(r + q, nrows - 1);
    if (FWD) {
      r0[q] = 0;
      rows[q] = fwd_row(c, nd, rq, r1[q]);
    } else {
      rows[q] = c.F + nd.inv + (int64_t)rq * nd.ldp;
      r0[q] = rq;
      r1[q] = nd.p;
    }
    if (r + q >= nrows) r1[q] = r0[q];
    if (r1[q] > r0[q]) {
      lo = min(lo, r0[q]);
      hi = max(hi, r1[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < kMR; ++q) d[q] = e[q] = 0.0;
  warp_share(lo, hi, w, nw);
#pragma unroll
  for (int q = 0; q < kMR; ++q) {  // the rows' ranges inside this warp's share
    r0[q] = max(r0[q], lo);
    r1[q] = min(r1[q], hi);
  }
  if (hi > lo) multi_dot(rows, Direct{FWD ? c.W + nd.w : c.Y + nd.y}, lo, hi, r0, r1, lane, d);
  if (!FWD && nd.b > 0) {
#pragma unroll
    for (int q = 0; q < kMR; ++q) {
      const int rq = min(r + q, nrows - 1);
      rows[q] = c.F + nd.upb + (int64_t)rq * nd.ldb;
      r0[q] = 0;
      r1[q] = (r + q < nrows) ? nd.b : 0;
    }
    int nlo = 0, nhi = nd.b;
    warp_share(nlo, nhi, w, nw);
#pragma unroll
    for (int q = 0; q < kMR; ++q) {
      r0[q] = nlo;
      r1[q] = (r + q < nrows) ? nhi : nlo;
    }
    if (nhi > nlo) multi_dot(rows, Gathered{c.X, c.bidx + nd.bx}, nlo, nhi, r0, r1, lane, e);
  }
}

template <bool FWD>
__device__ __forceinline__ void run_merged(const Ctx& c, const int4 tk, const xdg_mf_node& nd,
                                           const int lane) {
  const int nrows = FWD ? nd.p + nd.b : nd.p;
  if (tk.z == kMR) {  // whole-warp rows: kMR rows share the vector loads
    const int r = tk.y;
    double d[kMR], e[kMR];
    merged_rows<FWD>(c, nd, r, nrows, lane, 0, 1, d, e);
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < kMR; ++q)
        if (r + q < nrows) {
          if (FWD)
            fwd_done(c, nd, r + q, d[q]);
          else
            bwd_done(c, nd, r + q, d[q], e[q]);
        }
    }
  } else {  // two sets of 32/G rows, G lanes per row
    const int G = FWD ? nd.gp : nd.gb;
    const int gl = lane & (G - 1);
    const int ra = tk.y + lane / G, rb = ra + 32 / G;
    const bool acta = ra < nrows, actb = rb < nrows;
    const int qa = acta ? ra : 0, qb = actb ? rb : 0;
    double da, db, ea = 0.0, eb = 0.0;
    if (FWD) {
      int la, lb;
      const double* pa = fwd_row(c, nd, qa, la);
      const double* pb = fwd_row(c, nd, qb, lb);
      // the rows' own W entries are loaded with the dot's loads, not after it
      const double wa = c.W[nd.w + qa], wb = c.W[nd.w + qb];
      group_dot2r(pa, pb, Direct{c.W + nd.w}, 0, acta ? la : 0, 0, actb ? lb : 0, gl, G, da, db);
      if (acta && gl == 0) fwd_store(c, nd, ra, wa, da);
      if (actb && gl == 0) fwd_store(c, nd, rb, wb, db);
    } else {
      const double* inv = c.F + nd.inv;
      group_dot2r(inv + (int64_t)qa * nd.ldp, inv + (int64_t)qb * nd.ldp, Direct{c.Y + nd.y},
                  qa, acta ? nd.p : qa, qb, actb ? nd.p : qb, gl, G, da, db);
      if (nd.b > 0) {
        const double* un = c.F + nd.upb;
        group_dot2r(un + (int64_t)qa * nd.ldb, un + (int64_t)qb * nd.ldb,
                    Gathered{c.X, c.bidx + nd.bx}, 0, acta ? nd.b : 0, 0, actb ? nd.b : 0, gl,
                    G, ea, eb);
      }
      if (acta && gl == 0) bwd_done(c, nd, ra, da, ea);
      if (actb && gl == 0) bwd_done(c, nd, rb, db, eb);
    }
  }
}

// Group task: kMR long rows shared by a group of kGW warps of the CTA, each
// warp an equal contiguous share of the columns; the warps' partial sums are
// added in warp order by the group's first lanes (deterministic).  Long rows
// as warp tasks leave a launch with fewer tasks than resident warps and a
// tail as long as its longest row (root front: 2 x 76 KB per task).
#ifndef MF_GW
#define MF_GW 4
#endif
constexpr int kGW = MF_GW;          // warps per group
constexpr int kNG = kT / 32 / kGW;  // groups per CTA

template <bool FWD>
__device__ __forceinline__ void run_merged_group(const Ctx& c, const int4 tk, int grp,
                                                 double (*part)[2 * kMR]) {
  const int lane = threadIdx.x & 31, gw = (threadIdx.x >> 5) % kGW;
  const xdg_mf_node nd = c.nodes[tk.x];
  const int nrows = FWD ? nd.p + nd.b : nd.p;
  const int r = tk.y;
  double d[kMR], e[kMR];
  merged_rows<FWD>(c, nd, r, nrows, lane, gw, kGW, d, e);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < kMR; ++q) {
      part[gw][q] = d[q];
      part[gw][kMR + q] = e[q];
    }
  }
  asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * kGW) : "memory");
  if (gw == 0 && lane < kMR && r + lane < nrows) {
    double ds = 0.0, es = 0.0;
#pragma unroll
    for (int w = 0; w < kGW; ++w) {
      ds += part[w][lane];
      es += part[w][kMR + lane];
    }
    if (FWD)
      fwd_done(c, nd, r + lane, ds);
    else
      bwd_done(c, nd, r + lane, ds, es);
  }
}

template <bool FWD>
__global__ void __launch_bounds__(kT, MF_MINB)
mf_merged_kernel(int64_t t0, int64_t ntasks, int64_t c0, int64_t nctasks,
                 const int4* __restrict__ tasks, Ctx c) {
  __shared__ double part[2][kNG][kGW][2 * kMR];
  pdl_trigger();
  // Warp tasks, software-pipelined through shared memory: while task k runs,
  // the node of task k + 1 and the descriptor of task k + 2 are in flight
  // (cp.async), so a task's chain of dependent loads is its factor rows only
  // -- not descriptor -> node -> rows.  The low levels (thousands of fronts
  // of 10-300 pivots, a few KB per task) are bound by exactly that chain.
  __shared__ __align__(16) int4 tks[kT / 32][2];
  __shared__ __align__(16) xdg_mf_node nds[kT / 32][2];
  static_assert(sizeof(xdg_mf_node) == 96, "node copies are 6 x 16 bytes");
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int64_t nw = (int64_t)gridDim.x * (kT / 32);
  const int64_t w0 = (int64_t)blockIdx.x * (kT / 32) + wp;
  auto fetch_task = [&](int64_t w, int slot) {  // lane 6: 16-byte descriptor
    if (lane == 6) cp_async16(&tks[wp][slot], tasks + t0 + interleave(w, ntasks));
  };
  auto fetch_node = [&](int node, int slot) {  // lanes 0-5: 96-byte node
    if (lane < 6)
      cp_async16(reinterpret_cast<char*>(&nds[wp][slot]) + 16 * lane,
                 reinterpret_cast<const char*>(c.nodes + node) + 16 * lane);
  };
  // static data only up to the wait: the first descriptor and node of this
  // warp's tasks (and of its group's first CTA task) are on their way while
  // the previous launch of the chain drains
  if (w0 < ntasks) {
    fetch_task(w0, 0);
    cp_async_wait_all();
    __syncwarp();
    fetch_node(tks[wp][0].x, 0);
    if (w0 + nw < ntasks) fetch_task(w0 + nw, 1);
  }
  pdl_wait();
  {
    const int grp = (threadIdx.x >> 5) / kGW;
    int par = 0;  // alternating buffers: one group barrier per task
    for (int64_t ct = (int64_t)blockIdx.x * kNG + grp; ct < nctasks;
         ct += (int64_t)gridDim.x * kNG, par ^= 1)
      run_merged_group<FWD>(c, tasks[c0 + interleave(ct, nctasks)], grp, part[par][grp]);
  }
  if (w0 >= ntasks) return;
  int k = 0;
  for (int64_t w = w0; w < ntasks; w += nw, k ^= 1) {
    cp_async_wait_all();
    __syncwarp();  // nds[k] and tks[k ^ 1] have landed
    const int4 tk = tks[wp][k];
    const bool more = w + nw < ntasks;
    const int next_node = more ? tks[wp][k ^ 1].x : 0;
    __syncwarp();  // every lane has read tks[k] before it is refilled
    if (more) fetch_node(next_node, k ^ 1);
    if (w + 2 * nw < ntasks) fetch_task(w + 2 * nw, k);
    run_merged<FWD>(c, tk, nds[wp][k], lane);
  }
}

template <bool FWD>
int launch_merged(const xdg_mf* mf, int h, double* x, cudaStream_t s) {
  // warp tasks: lev_task[0] / [2]; CTA tasks (long rows): lev_task[1] / [3]
  const int64_t* lev = mf->lev_task + (int64_t)(FWD ? 0 : 2) * (mf->nlevels + 1);
  const int64_t* levc = lev + (mf->nlevels + 1);
  const int64_t t0 = lev[h], nt = lev[h + 1] - t0;
  const int64_t c0 = levc[h], nc = levc[h + 1] - c0;
  if (nt <= 0 && nc <= 0) return XDG_OK;
  Ctx c{mf->nodes, mf->F, mf->bidx, mf->pdst, mf->pscale, mf->W, mf->Y, mf->C, x, mf->X};
  const int g = resident_grid(mf_merged_kernel<FWD>, kT, 0, (nt + nc * kGW) * 32);
  XDG_TRY_CUDA(launch_chain(mf_merged_kernel<FWD>, g, s, t0, nt, c0, nc,
                        reinterpret_cast<const int4*>(mf->tasks), c));
  return XDG_OK;
}

// Forward rows of the fronts with a column-major copy FT[k][r] of
// [L^-1 (strictly lower); M_BP] (nd.ldr > 0): one THREAD per row, a warp
// task = 32 consecutive rows.  Loads are coalesced across the rows, the
// vector entry W[k] is the same for every lane (one broadcast load), no
// reductions, no per-entry masks: ~0.15 instructions per matrix entry
// instead of ~2 for the lane groups on fronts of 10-300 pivots, and few
// enough registers for twice the resident warps.
#ifndef MF_CU
#define MF_CU 8  // columns (independent loads) in flight per thread
#endif
__global__ void __launch_bounds__(kT, 6)
mf_fwd_cols_kernel(int64_t t0, int64_t ntasks, const int4* __restrict__ tasks, Ctx c) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (kT / 32);
  for (int64_t w = (int64_t)blockIdx.x * (kT / 32) + (threadIdx.x >> 5); w < ntasks; w += nw) {
    const int4 tk = tasks[t0 + interleave(w, ntasks)];
    const xdg_mf_node nd = c.nodes[tk.x];
    const int p = nd.p, R = nd.p + nd.b;
    const int r = tk.y + lane;
    const bool act = r < R;
    // storage row: boundary rows sit after the padded pivot rows
    const int rs = act ? (r < p ? r : r + (nd.ldp - p)) : 0;
    // a block of pivot rows only needs the columns left of its last row
    const int kend = (tk.y + 32 <= p) ? tk.y + 31 : p;
    const double* ft = c.F + nd.lbp + rs;
    const double* wv = c.W + nd.w;
    const double wr = act ? wv[r] : 0.0;
    double acc[2] = {0.0, 0.0};
    for (int k0 = 0; k0 < kend; k0 += MF_CU) {
      double a[MF_CU], x[MF_CU];
#pragma unroll
      for (int u = 0; u < MF_CU; ++u) {
        const int k = min(k0 + u, kend - 1);
        a[u] = __ldg(ft + (int64_t)k * nd.ldr);
        x[u] = wv[k];
      }
#pragma unroll
      for (int u = 0; u < MF_CU; ++u)
        acc[u & 1] = fma(a[u], (k0 + u < kend) ? x[u] : 0.0, acc[u & 1]);
    }
    const double d = acc[0] + acc[1];
    if (act) {
      if (r < p)
        c.Y[nd.y + r] = __dadd_rn(wr, d);
      else
        c.C[nd.c + (r - p)] = __dsub_rn(wr, d);
    }
  }
}

int launch_fwd_cols(const xdg_mf* mf, int h, double* x, cudaStream_t s) {
  const int64_t* lev = mf->lev_task + (int64_t)4 * (mf->nlevels + 1);
  const int64_t t0 = lev[h], nt = lev[h + 1] - t0;
  if (nt <= 0) return XDG_OK;
  Ctx c{mf->nodes, mf->F, mf->bidx, mf->pdst, mf->pscale, mf->W, mf->Y, mf->C, x, mf->X};
  const int g = resident_grid(mf_fwd_cols_kernel, kT, 0, nt * 32);
  mf_fwd_cols_kernel<<<g, kT, 0, s>>>(t0, nt, reinterpret_cast<const int4*>(mf->tasks), c);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

// Gather entry e: W[ent_w] = scale * b[src] + children's contributions (in
// fixed order).  Plain loads: in the fused kernel C was written by the same
// launch (children of an earlier stage).
__device__ __forceinline__ void gather_entry(int64_t e, const xdg_mf& m, const double* b) {
  const int64_t s = m.ent_src[e];
  double v = s >= 0 ? __dmul_rn(m.ent_scale[e], b[s]) : 0.0;
  for (int64_t k = m.ent_cptr[e]; k < m.ent_cptr[e + 1]; ++k) v = __dadd_rn(v, m.C[m.ent_cidx[k]]);
  m.W[m.ent_w[e]] = v;
}

// Warps of the CTA stride over the warp tasks [t0, t1) of one stage.
template <int PH>
__device__ __forceinline__ void stage_tasks(const Ctx& c, const int4* tasks, int64_t t0,
                                            int64_t t1) {
  const int lane = threadIdx.x & 31;
  for (int64_t w = t0 + (threadIdx.x >> 5); w < t1; w += kT / 32) run_task<PH>(c, tasks[w], lane);
}

// Fused low levels: one CTA per group of fronts, the group's stages (sets
// of fronts of one height whose children are in earlier stages of the same
// group) in order, __syncthreads between phases.  Forward: gather, lower,
// bound per stage; backward (reverse stage order): upb, upper.  Every row
// runs the same run_task code as the per-level launches: bit-identical.
template <bool FWD>
__global__ void __launch_bounds__(kT, MF_MINB)
mf_fused_kernel(int64_t g0, int64_t g1, const xdg_mf m, const double* b, Ctx c) {
  const int64_t ns1 = m.nfstages + 1;
  const int4* ft = reinterpret_cast<const int4*>(m.ftask);
  for (int64_t g = g0 + blockIdx.x; g < g1; g += gridDim.x) {
    const int64_t s0 = m.g_stage[g], s1 = m.g_stage[g + 1];
    if (FWD) {
      for (int64_t s = s0; s < s1; ++s) {
        for (int64_t i = m.st_ent[s] + threadIdx.x; i < m.st_ent[s + 1]; i += kT)
          gather_entry(m.fent[i], m, b);
        __syncthreads();
        stage_tasks<kLower>(c, ft, m.st_task[s], m.st_task[s + 1]);
        __syncthreads();
        stage_tasks<kBound>(c, ft, m.st_task[ns1 + s], m.st_task[ns1 + s + 1]);
        __syncthreads();
      }
    } else {
      for (int64_t s = s1 - 1; s >= s0; --s) {
        stage_tasks<kUpb>(c, ft, m.st_task[2 * ns1 + s], m.st_task[2 * ns1 + s + 1]);
        __syncthreads();
        stage_tasks<kUpper>(c, ft, m.st_task[3 * ns1 + s], m.st_task[3 * ns1 + s + 1]);
        __syncthreads();
      }
    }
  }
}

template <bool FWD>
int launch_fused(const xdg_mf* mf, int k, const double* b, double* x, cudaStream_t s) {
  const int64_t g0 = mf->fb_grp[k], ng = mf->fb_grp[k + 1] - g0;
  if (ng <= 0) return XDG_OK;
  Ctx c{mf->nodes, mf->F, mf->bidx, mf->pdst, mf->pscale, mf->W, mf->Y, mf->C, x, mf->X};
  const int g = resident_grid(mf_fused_kernel<FWD>, kT, 0, ng * kT);
  mf_fused_kernel<FWD><<<g, kT, 0, s>>>(g0, g0 + ng, *mf, b, c);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

template <int PH>
int launch_rows(const xdg_mf* mf, int h, double* x, cudaStream_t s) {
  const int64_t* lev = mf->lev_task + (int64_t)PH * (mf->nlevels + 1);
  const int64_t t0 = lev[h], nt = lev[h + 1] - t0;
  if (nt <= 0) return XDG_OK;
  Ctx c{mf->nodes, mf->F, mf->bidx, mf->pdst, mf->pscale, mf->W, mf->Y, mf->C, x, mf->X};
  const int g = resident_grid(mf_rows_kernel<PH>, kT, 0, nt * 32);
  mf_rows_kernel<PH><<<g, kT, 0, s>>>(t0, nt, reinterpret_cast<const int4*>(mf->tasks), c);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

}  // namespace
}  // namespace xdg

extern "C" int xdg_mf_rows_per_warp(void) { return xdg::kMR; }

extern "C" int xdg_mf_solve_phase(const xdg_mf* mf, const double* b, double* x, int phase,
                                  xdg_stream_t stream) {
  using namespace xdg;
  XDG_REQUIRE(mf != nullptr && mf->nlevels >= 0 && phase >= 1 && phase <= 3, XDG_ERR_ARG,
              "bad multifrontal plan / phase");
  XDG_REQUIRE(!mf->merged || (mf->nfbatch == 0 && mf->X != nullptr), XDG_ERR_ARG,
              "merged multifrontal phases exclude the fused low levels and need X");
  NvtxRange nv("xdg_mf_solve");
  if (mf->total == 0 || mf->nlevels == 0) return XDG_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int H = mf->nlevels;
  const int HF = mf->fuse_levels;  // levels [0, HF) run as fused batches
  if (phase & 1) {  // forward: gather, lower, bound per height
    for (int k = 0; k < mf->nfbatch; ++k) XDG_TRY(launch_fused<true>(mf, k, b, x, s));
    for (int h = HF; h < H; ++h) {
      const int64_t e0 = mf->lev_ent[h], e1 = mf->lev_ent[h + 1];
      if (e1 > e0) {
        XDG_TRY_CUDA(launch_chain(mf_gather_kernel, grid_for(e1 - e0, kT, 8), s, e0, e1,
                              mf->ent_w, mf->ent_src, mf->ent_cptr, mf->ent_cidx,
                              mf->ent_scale, b, mf->C, mf->W));
      }
      if (mf->merged) {
        XDG_TRY(launch_fwd_cols(mf, h, x, s));
        XDG_TRY(launch_merged<true>(mf, h, x, s));
        continue;
      }
      XDG_TRY(launch_rows<kLower>(mf, h, x, s));
      XDG_TRY(launch_rows<kBound>(mf, h, x, s));
    }
  }
  if (phase & 2) {  // backward: upb, upper per height
    for (int h = H - 1; h >= HF; --h) {
      if (mf->merged) {
        XDG_TRY(launch_merged<false>(mf, h, x, s));
        continue;
      }
      XDG_TRY(launch_rows<kUpb>(mf, h, x, s));
      XDG_TRY(launch_rows<kUpper>(mf, h, x, s));
    }
    for (int k = mf->nfbatch - 1; k >= 0; --k) XDG_TRY(launch_fused<false>(mf, k, b, x, s));
  }
  return XDG_OK;
}

extern "C" int xdg_mf_solve(const xdg_mf* mf, const double* b, double* x,
                            xdg_stream_t stream) {
  return xdg_mf_solve_phase(mf, b, x, 3, stream);
}

// Setup: extend-add of the children's Schur complements into their parents'
// fronts, one CTA per (parent, child) pair of one round (the r-th child of
// every parent: targets are distinct, no atomics; rounds run in child order,
// so each entry receives its children's terms in the same order as the
// reference-ordered host loop -- bit-identical).  pair[7q ..] = (parent
// base, parent stride, child base, child stride, child pivot pad, boundary
// unknowns n, offset of the pair's n front rows in U).
namespace xdg {
namespace {
__global__ void __launch_bounds__(kT)
mf_extend_add_kernel(int64_t npairs, const int64_t* __restrict__ pair,
                     const int64_t* __restrict__ U, const double* __restrict__ child,
                     double* __restrict__ parent) {
  for (int64_t q = blockIdx.x; q < npairs; q += gridDim.x) {
    const int64_t* pq = pair + 7 * q;
    const int64_t tb = pq[0], ts = pq[1], cb = pq[2], cs = pq[3], cp = pq[4];
    const int n = (int)pq[5];
    const int64_t* u = U + pq[6];
    const int64_t nn = (int64_t)n * n;
    for (int64_t k = (int64_t)blockIdx.y * kT + threadIdx.x; k < nn;
         k += (int64_t)kT * gridDim.y) {  // 64-bit counter: no overflow past n^2
      const int kk = (int)k;
      const int i = kk / n, j = kk - i * n;
      double* d = parent + tb + u[i] * ts + u[j];
      *d = __dadd_rn(*d, child[cb + (cp + i) * cs + cp + j]);
    }
  }
}
}  // namespace
}  // namespace xdg

extern "C" int xdg_mf_extend_add(int64_t npairs, const int64_t* pair, const int64_t* U,
                                 const double* child, double* parent, int64_t max_n,
                                 xdg_stream_t stream) {
  using namespace xdg;
  if (npairs <= 0) return XDG_OK;
  XDG_REQUIRE(max_n * max_n < (1LL << 31), XDG_ERR_ARG, "boundary too large (%lld)",
              (long long)max_n);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // pairs on grid x, element ranges of a pair on grid y (~8 per thread)
  const int64_t parts = std::min<int64_t>(65535, std::max<int64_t>(
                                                     1, (max_n * max_n + 8 * kT - 1) / (8 * kT)));
  const int64_t gx = std::min<int64_t>(npairs, std::max<int64_t>(1, 8 * sm_count() / parts));
  mf_extend_add_kernel<<<dim3((unsigned)gx, (unsigned)parts), kT, 0, s>>>(npairs, pair, U,
                                                                        child, parent);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}

// Setup of the merged phases: for every front of a bucket (nb fronts, each
// an n x n row-major buffer, n = P + B, holding the partial factorization
// xdg_batched_factor left: triangular inverses in the leading P x P corner,
// L_BP below, U_PB to the right)
//   M = L_BP L^-1  (B x P, L^-1 unit lower: strictly-lower part stored)
//   N = U^-1 U_PB  (P x B, U^-1 upper incl. diagonal)
// written to the factor storage.  Tiled FP64 product, 64 x 64 tile per CTA,
// 4 x 4 per thread, the triangular operand masked while it is staged and
// the K range cut to its nonzero part.
namespace xdg {
namespace {
template <bool LOWER, int BT>  // true: M = L_BP L^-1;  false: N = U^-1 U_PB
__global__ void __launch_bounds__(256, BT >= 128 ? 1 : 2)
mf_merge_kernel(int P, int B, const double* __restrict__ Fb, double* __restrict__ out) {
  __shared__ DmmaSmem<BT, BT> sm;
  const int n = P + B;
  const double* F = Fb + (int64_t)blockIdx.z * n * n;
  const int rows = LOWER ? B : P, cols = LOWER ? P : B;
  double* O = out + (int64_t)blockIdx.z * rows * cols;
  const int i0 = blockIdx.y * BT, j0 = blockIdx.x * BT;
  // nonzero K range: L^-1[k, j] = 0 for k < j;  U^-1[i, k] = 0 for k < i
  const int kbeg = ((LOWER ? j0 : i0) / kDK) * kDK;
  tile_dmma<BT, BT>(
      P - kbeg,
      [&](int ii, int kk) {
        const int i = i0 + ii, k = kbeg + kk;
        if (i >= rows || k >= P) return 0.0;
        if (LOWER) return F[(int64_t)(P + i) * n + k];
        return (k >= i) ? F[(int64_t)i * n + k] : 0.0;
      },
      [&](int kk, int jj) {
        const int k = kbeg + kk, j = j0 + jj;
        if (j >= cols || k >= P) return 0.0;
        if (LOWER) return (k > j) ? F[(int64_t)k * n + j] : (k == j ? 1.0 : 0.0);
        return F[(int64_t)k * n + P + j];
      },
      [&](int ii, int jj, double v) {
        const int i = i0 + ii, j = j0 + jj;
        if (i < rows && j < cols) O[(int64_t)i * cols + j] = v;
      },
      sm);
}

template <int BT>
int launch_merge(int64_t nb, int P, int B, const double* fronts, double* out_m, double* out_n,
                 cudaStream_t s) {
  const unsigned tp = (unsigned)((P + BT - 1) / BT), tb = (unsigned)((B + BT - 1) / BT);
  mf_merge_kernel<true, BT><<<dim3(tp, tb, (unsigned)nb), 256, 0, s>>>(P, B, fronts, out_m);
  XDG_CHECK_LAUNCH();
  mf_merge_kernel<false, BT><<<dim3(tb, tp, (unsigned)nb), 256, 0, s>>>(P, B, fronts, out_n);
  XDG_CHECK_LAUNCH();
  return XDG_OK;
}
}  // namespace
}  // namespace xdg

extern "C" int xdg_mf_merge(int64_t nb, int P, int B, const double* fronts, double* out_m,
                            double* out_n, xdg_stream_t stream) {
  using namespace xdg;
  if (nb <= 0 || P <= 0 || B <= 0) return XDG_OK;
  XDG_REQUIRE(nb <= 65535, XDG_ERR_ARG, "xdg_mf_merge: at most 65535 fronts per call");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (std::max(P, B) > 256) return launch_merge<128>(nb, P, B, fronts, out_m, out_n, s);
  return launch_merge<64>(nb, P, B, fronts, out_m, out_n, s);
}
