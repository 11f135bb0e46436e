// small_expm.cuh — exp(A) for n <= 16 inside one CTA of n*n threads (thread e
// owns element e of every n x n matrix; all matrices in shared memory):
// Taylor-16 in Paterson-Stockmeyer form (A^2, A^3, A^4, then three Horner
// products in A^4), then `sq` squarings — the construction of the DMMA path
// (k_model.cu expm_dev), without a launch per product. Used by the GRAPE build
// (k_sweep.cu) and by expm_dev for small n.
#pragma once
#include <cuda_runtime.h>

namespace lbg {

constexpr int kSmallN = 16, kSmallNN = kSmallN * kSmallN;

struct SmallCoef {
  double c[17];  // 1/k!, k = 0..16
};

__device__ __forceinline__ double2 small_mm(const double2* __restrict__ X, const double2* __restrict__ Y, int n,
                                            int r, int c) {
  double re = 0.0, im = 0.0;
  for (int k = 0; k < n; ++k) {
    const double2 a = X[r * n + k], b = Y[k * n + c];
    re = fma(a.x, b.x, re);
    re = fma(-a.y, b.y, re);
    im = fma(a.x, b.y, im);
    im = fma(a.y, b.x, im);
  }
  return make_double2(re, im);
}

// A holds the scaled argument on entry; the result is left in T. All threads
// of the CTA call this (contains __syncthreads).
__device__ __forceinline__ void small_taylor(double2* A, double2* A2, double2* A3, double2* A4, double2* T, int n,
                                             const double* cf, int sq) {
  const int e = threadIdx.x;
  const bool own = e < n * n;
  const int r = own ? e / n : 0, c = own ? e - r * n : 0;
  auto combo = [&](double2 x, double c0, double c1, double c2, double c3) {
    double2 v = x;
    if (r == c) v.x += c0;
    v.x += c1 * A[e].x;
    v.y += c1 * A[e].y;
    v.x += c2 * A2[e].x;
    v.y += c2 * A2[e].y;
    v.x += c3 * A3[e].x;
    v.y += c3 * A3[e].y;
    return v;
  };
  if (own) A2[e] = small_mm(A, A, n, r, c);
  __syncthreads();
  if (own) {
    A3[e] = small_mm(A2, A, n, r, c);
    A4[e] = small_mm(A2, A2, n, r, c);
  }
  __syncthreads();
  if (own) {  // T = c12 I + c13 A + c14 A2 + c15 A3 + c16 A4
    double2 v = combo(make_double2(0.0, 0.0), cf[12], cf[13], cf[14], cf[15]);
    v.x += cf[16] * A4[e].x;
    v.y += cf[16] * A4[e].y;
    T[e] = v;
  }
  __syncthreads();
  for (int j = 2; j >= 0; --j) {  // T = A4 T + B_j
    double2 v = make_double2(0.0, 0.0);
    if (own) v = combo(small_mm(A4, T, n, r, c), cf[4 * j], cf[4 * j + 1], cf[4 * j + 2], cf[4 * j + 3]);
    __syncthreads();
    if (own) T[e] = v;
    __syncthreads();
  }
  for (int q = 0; q < sq; ++q) {
    double2 v = make_double2(0.0, 0.0);
    if (own) v = small_mm(T, T, n, r, c);
    __syncthreads();
    if (own) T[e] = v;
    __syncthreads();
  }
}

}  // namespace lbg
