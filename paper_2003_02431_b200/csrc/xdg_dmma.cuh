// FP64 tensor-core tile product shared by the factorization kernels
// (xdg_factor.cu: trailing updates, triangular inverses) and the
// multifrontal setup products (xdg_multifrontal.cu: xdg_mf_merge).
#pragma once

#include "xdg_common.cuh"

namespace xdg {

// FP64 tensor-core tile product (mma.sync m8n8k4 f64 -- DMMA; the
// factorization's block products are the compute-bound part of the path:
// north_star allows FP64 tensor cores there).  BM x BN tile of A B
// accumulated over K in chunks of 8, 256 threads = 2 x 4 warps, operands
// staged through double-buffered shared memory (next chunk prefetched into
// registers during the products).  Loader callbacks give A(i, k) / B(k, j)
// (zero outside); st(i, j, v) receives every tile entry.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

constexpr int kDK = 8;  // K chunk of the DMMA tiles

template <int BM, int BN>
struct DmmaSmem {
  double a[2][kDK][BM + 4];  // leading dimension = 4 mod 16: conflict-free fragments
  double b[2][kDK][BN + 4];
};

template <int BM, int BN, class FA, class FB, class ST>
__device__ __forceinline__ void tile_dmma(int K, FA fa, FB fb, ST st, DmmaSmem<BM, BN>& sm) {
  constexpr int WM = BM / 2, WN = BN / 4, MT = WM / 8, NT = WN / 8;
  constexpr int LA = BM * kDK / 256, LB = BN * kDK / 256;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp >> 2) * WM, wn0 = (warp & 3) * WN;
  const int lr = lane >> 2, lk = lane & 3;
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double ra[LA], rb[LB];
  auto fetch = [&](int kc) {
#pragma unroll
    for (int q = 0; q < LA; ++q) {
      const int e = tid + 256 * q;  // k fastest: row-contiguous A reads
      ra[q] = fa(e / kDK, kc + e % kDK);
    }
#pragma unroll
    for (int q = 0; q < LB; ++q) {
      const int e = tid + 256 * q;  // j fastest
      rb[q] = fb(kc + e / BN, e % BN);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int q = 0; q < LA; ++q) {
      const int e = tid + 256 * q;
      sm.a[buf][e % kDK][e / kDK] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < LB; ++q) {
      const int e = tid + 256 * q;
      sm.b[buf][e / BN][e % BN] = rb[q];
    }
  };
  if (K > 0) {
    fetch(0);
    stash(0);
  }
  __syncthreads();
  int buf = 0;
  for (int kc = 0; kc < K; kc += kDK, buf ^= 1) {
    const bool more = kc + kDK < K;
    if (more) fetch(kc + kDK);
#pragma unroll
    for (int ks = 0; ks < kDK; ks += 4) {
      double a[MT], b[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) a[i] = sm.a[buf][ks + lk][wm0 + 8 * i + lr];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = sm.b[buf][ks + lk][wn0 + 8 * j + lr];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int r = wm0 + 8 * i + lr, c = wn0 + 8 * j + 2 * lk;
      st(r, c, acc[i][j][0]);
      st(r, c + 1, acc[i][j][1]);
    }
}


}  // namespace xdg
