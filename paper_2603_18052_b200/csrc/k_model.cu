// k_model.cu — model-side kernels: Kronecker assembly of the vectorised
// Lindbladian (K5, single model), the GPU propagator P = exp(L dt) (K4,
// single matrix), the batched invariant check (K6) and the single-step shim.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "internal.hpp"
#include "small_expm.cuh"

namespace lbg {

namespace {

// Complex arithmetic with explicit round-to-nearest intrinsics: no FMA
// contraction, so the assembly reproduces the reference's std::complex
// arithmetic bit for bit (tests/test_gpu_parity.py checks L exactly).
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double2 conjd(double2 a) { return make_double2(a.x, -a.y); }

// (L_m^dag L_m)[i][j] accumulated like lb::matmul (complex_matrix.cpp:41-54):
// ascending q from zero, re += ar*br - ai*bi, im += ar*bi + ai*br, a = conj(L[q][i]).
__device__ __forceinline__ double2 ldl_entry(const double2* __restrict__ l, int d, int i, int j) {
  double re = 0.0, im = 0.0;
  for (int q = 0; q < d; ++q) {
    const double2 a = conjd(l[q * d + i]);
    const double2 b = l[q * d + j];
    re = __dadd_rn(re, __dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)));
    im = __dadd_rn(im, __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
  }
  return make_double2(re, im);
}

// K5: element (R = i*d + k, C = j*d + l) of
//   L = -i (H (x) I - I (x) H^T) + sum_m [ L_m (x) conj L_m - 1/2 L_m^dag L_m (x) I
//                                        - 1/2 I (x) (L_m^dag L_m)^T ]
// in the reference's evaluation order (lindblad.cpp:46-57): kron entries are
// a[i][j] * b[k][l] complex products, accumulated with add_scaled.
__device__ __forceinline__ double2 lindblad_entry(const double2* __restrict__ h, const double2* __restrict__ ops,
                                                  int n_ops, int d, long long e) {
  const int n = d * d;
  const int R = int(e / n), Cc = int(e - (long long)R * n);
  const int i = R / d, k = R - i * d, j = Cc / d, l = Cc - j * d;
  const double2 one = make_double2(1.0, 0.0), zero = make_double2(0.0, 0.0);
  const double2 dkl = (k == l) ? one : zero, dij = (i == j) ? one : zero;
  // -i * (kron(H, I) - kron(I, H^T))
  const double2 t1 = cmul(h[i * d + j], dkl);
  const double2 t2 = cmul(dij, h[l * d + k]);
  double2 acc = cmul(make_double2(0.0, -1.0), csub(t1, t2));
  for (int m = 0; m < n_ops; ++m) {
    const double2* lm = ops + (long long)m * d * d;
    acc = cadd(acc, cmul(one, cmul(lm[i * d + j], conjd(lm[k * d + l]))));
    const double2 a = (k == l) ? ldl_entry(lm, d, i, j) : zero;
    acc = cadd(acc, cmul(make_double2(-0.5, 0.0), cmul(a, dkl)));
    const double2 b = (i == j) ? ldl_entry(lm, d, l, k) : zero;
    acc = cadd(acc, cmul(make_double2(-0.5, 0.0), cmul(dij, b)));
  }
  return acc;
}
__global__ void build_lindbladian_kernel(const double2* __restrict__ h,
                                         const double2* __restrict__ ops, int n_ops, int d,
                                         double2* __restrict__ out) {
  const long long nn = (long long)(d * d) * (d * d);
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < nn) out[e] = lindblad_entry(h, ops, n_ops, d, e);
}
// batch of models: model b = (h + b d^2, ops + b n_ops d^2) -> out + b d^4
__global__ void build_lindbladian_batched_kernel(const double2* __restrict__ h, const double2* __restrict__ ops,
                                                 int n_ops, int d, long long total, double2* __restrict__ out) {
  const long long nn = (long long)(d * d) * (d * d);
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long b = q / nn, e = q - b * nn;
    out[q] = lindblad_entry(h + b * d * d, ops + b * n_ops * d * d, n_ops, d, e);
  }
}

// out = x + c0*I + c1*a1 + c2*a2 + c3*a3 + c4*a4   (any pointer may be null)
__global__ void combo_kernel(double2* __restrict__ out, const double2* __restrict__ x,
                             const double2* __restrict__ a1, const double2* __restrict__ a2,
                             const double2* __restrict__ a3, const double2* __restrict__ a4,
                             double c0, double c1, double c2, double c3, double c4, int n) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * n) return;
  const int r = int(e / n), c = int(e - (long long)r * n);
  double2 v = x ? x[e] : make_double2(0.0, 0.0);
  if (r == c) v.x += c0;
  if (a1) { v.x += c1 * a1[e].x; v.y += c1 * a1[e].y; }
  if (a2) { v.x += c2 * a2[e].x; v.y += c2 * a2[e].y; }
  if (a3) { v.x += c3 * a3[e].x; v.y += c3 * a3[e].y; }
  if (a4) { v.x += c4 * a4[e].x; v.y += c4 * a4[e].y; }
  out[e] = v;
}

__global__ void scale_kernel(double2* __restrict__ out, const double2* __restrict__ a, double s,
                             long long count) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < count) out[e] = make_double2(a[e].x * s, a[e].y * s);
}

// column sums of |a| -> colsum[n]: block = 32 columns x 8 row groups (coalesced
// rows, 8-way parallel sums; one thread per column took 0.29 ms at n = 729)
__global__ void colsum_kernel(const double2* __restrict__ a, int n, double* __restrict__ colsum) {
  __shared__ double part[8][33];
  const int tx = threadIdx.x, ty = threadIdx.y, c = blockIdx.x * 32 + tx;
  double s = 0.0;
  if (c < n)
    for (int r = ty; r < n; r += 8) s += hypot(a[(long long)r * n + c].x, a[(long long)r * n + c].y);
  part[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && c < n) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += part[k][tx];
    colsum[c] = t;
  }
}

// order-preserving map of a double to uint64 for atomic min/max
__device__ __forceinline__ unsigned long long okey(double v) {
  const unsigned long long b = __double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ounkey(unsigned long long k) {
  if (k == 0ull || k == ~0ull) return __longlong_as_double(0x7ff8000000000000ll);  // a NaN that won
  return __longlong_as_double((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k);
}
// NaN semantics of lb::check_state (validate.cpp:10-30): a NaN trace error or a
// NaN minimum diagonal (rho(0,0) NaN: std::min keeps its first operand) fails
// the state, so in the batch max / min a NaN must WIN (fmax / fmin would drop
// it); the Hermiticity max drops NaN like std::max does. NaN takes the keys 0
// and ~0, which no other double maps to.
__device__ __forceinline__ unsigned long long okey_max(double v) { return isnan(v) ? ~0ull : okey(v); }
__device__ __forceinline__ unsigned long long okey_min(double v) { return isnan(v) ? 0ull : okey(v); }
__device__ __forceinline__ double nanmax(double a, double b) { return isnan(a) ? a : (isnan(b) ? b : fmax(a, b)); }
__device__ __forceinline__ double nanmin(double a, double b) { return isnan(a) ? a : (isnan(b) ? b : fmin(a, b)); }
// std::min(m, x) = (x < m) ? x : m: a NaN x is dropped, a NaN m is kept
__device__ __forceinline__ double std_min(double m, double x) { return x < m ? x : m; }

// K6: validate.cpp:10-30 per trajectory, reduced over the batch.
__global__ void check_state_kernel(const double2* __restrict__ x, int d, long long batch,
                                   unsigned long long* __restrict__ keys) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double tr_err = 0.0, herm = 0.0, mind = 1e300;
  if (b < batch) {
    const double2* r = x + b * d * d;
    double tre = 0.0, tim = 0.0;
    mind = r[0].x;
    for (int i = 0; i < d; ++i) {
      tre += r[i * d + i].x;
      tim += r[i * d + i].y;
      mind = std_min(mind, r[i * d + i].x);
      for (int j = 0; j < d; ++j) {
        const double2 a = r[i * d + j], c = r[j * d + i];
        herm = fmax(herm, hypot(a.x - c.x, a.y + c.y));
      }
    }
    tr_err = hypot(tre - 1.0, tim);
  }
  for (int o = 16; o > 0; o >>= 1) {
    tr_err = nanmax(tr_err, __shfl_xor_sync(0xffffffffu, tr_err, o));
    herm = fmax(herm, __shfl_xor_sync(0xffffffffu, herm, o));
    mind = nanmin(mind, __shfl_xor_sync(0xffffffffu, mind, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&keys[0], okey_max(tr_err));
    atomicMax(&keys[1], okey(herm));
    atomicMin(&keys[2], okey_min(mind));
  }
}

// the same per state with one WARP per state (d >= 6): lanes split the d^2
// Hermiticity pairs; the trace is summed by lane 0 in the reference's order, so
// the results are bit-identical to the thread-per-state kernel
__global__ void check_state_warp_kernel(const double2* __restrict__ x, int d, long long batch,
                                        unsigned long long* __restrict__ keys) {
  const long long b = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  double tr_err = 0.0, herm = 0.0, mind = 1e300;
  if (b < batch) {
    const double2* r = x + b * d * d;
    for (int e = lane; e < d * d; e += 32) {
      const int i = e / d, j = e - i * d;
      const double2 a = r[e], c = r[j * d + i];
      herm = fmax(herm, hypot(a.x - c.x, a.y + c.y));
    }
    if (lane == 0) {
      double tre = 0.0, tim = 0.0;
      mind = r[0].x;
      for (int i = 0; i < d; ++i) {
        tre += r[i * d + i].x;
        tim += r[i * d + i].y;
        mind = std_min(mind, r[i * d + i].x);
      }
      tr_err = hypot(tre - 1.0, tim);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    tr_err = nanmax(tr_err, __shfl_xor_sync(0xffffffffu, tr_err, o));
    herm = fmax(herm, __shfl_xor_sync(0xffffffffu, herm, o));
    mind = nanmin(mind, __shfl_xor_sync(0xffffffffu, mind, o));
  }
  if (lane == 0) {
    atomicMax(&keys[0], okey_max(tr_err));
    atomicMax(&keys[1], okey(herm));
    atomicMin(&keys[2], okey_min(mind));
  }
}

__global__ void check_state_finish(const unsigned long long* __restrict__ keys, double* out3) {
  if (threadIdx.x < 3) out3[threadIdx.x] = ounkey(keys[threadIdx.x]);
}
__global__ void check_state_init(unsigned long long* keys) {
  if (threadIdx.x < 2) keys[threadIdx.x] = okey(0.0);
  if (threadIdx.x == 2) keys[2] = okey(1e300);
}

// one matvec out[i] = sum_j P[i][j] v[j] (the raw-pointer shim), ascending j
// exp(scale * a) for n <= 16 in one CTA (small_expm.cuh)
__global__ void __launch_bounds__(kSmallNN) small_expm_kernel(const double2* __restrict__ a, int n, double scale,
                                                              int sq, SmallCoef co, double2* __restrict__ out) {
  __shared__ double2 A[kSmallNN], A2[kSmallNN], A3[kSmallNN], A4[kSmallNN], T[kSmallNN];
  const int e = threadIdx.x;
  if (e < n * n) A[e] = make_double2(a[e].x * scale, a[e].y * scale);
  __syncthreads();
  small_taylor(A, A2, A3, A4, T, n, co.c, sq);
  if (e < n * n) out[e] = T[e];
}

// Batched exp(a_b dt) for n <= 16: one CTA per matrix, each with its own
// scaling: the 1-norm in colsum_kernel's summation order and expm_dev's
// squaring rule, then small_taylor — each out_b equals lbg_expm_dev(a_b).
// bad |= 1 for non-finite input, 2 for more than 64 squarings.
__global__ void __launch_bounds__(kSmallNN) small_expm_batched_kernel(const double2* __restrict__ a, int n, double dt,
                                                                      SmallCoef co, double2* __restrict__ out,
                                                                      unsigned* __restrict__ bad) {
  __shared__ double2 A[kSmallNN], A2[kSmallNN], A3[kSmallNN], A4[kSmallNN], T[kSmallNN];
  __shared__ double part[8][kSmallN + 1];
  __shared__ int s_sq;
  __shared__ double s_scale;
  const long long nn = (long long)n * n, b = blockIdx.x;
  const double2* ab = a + b * nn;
  const int e = threadIdx.x;
  {
    const int c = e & 15, ty = e >> 4;  // 16 columns x 16 row groups; groups 0..7 used
    if (ty < 8 && c < n) {
      double sum = 0.0;
      for (int r = ty; r < n; r += 8) sum += hypot(ab[r * n + c].x, ab[r * n + c].y);
      part[ty][c] = sum;
    }
  }
  __syncthreads();
  if (e == 0) {
    double nrm = 0.0;
    for (int c = 0; c < n; ++c) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += part[k][c];
      nrm = (isnan(t) || t > nrm) ? t : nrm;
    }
    nrm *= fabs(dt);
    int sq = 0;
    if (!isfinite(nrm)) {
      atomicOr(bad, 1u);
      sq = -1;
    } else if (nrm > 0.79) {
      sq = int(ceil(log2(nrm / 0.79)));
      if (sq > 64) {
        atomicOr(bad, 2u);
        sq = -1;
      }
    }
    s_sq = sq;
    s_scale = sq >= 0 ? dt * ldexp(1.0, -sq) : 0.0;
  }
  __syncthreads();
  const int sq = s_sq;
  if (sq < 0) return;
  if (e < nn) A[e] = make_double2(ab[e].x * s_scale, ab[e].y * s_scale);
  __syncthreads();
  small_taylor(A, A2, A3, A4, T, n, co.c, sq);
  if (e < nn) out[b * nn + e] = T[e];
}

// max over a batch of n x n matrices of the 1-norm (bits of a non-negative
// double, so unsigned max = double max; NaN sorts above every finite value)
__global__ void norm_batched_kernel(const double2* __restrict__ a, int n, long long batch,
                                    unsigned long long* __restrict__ nmax) {
  __shared__ double part[8][33];
  const long long nbx = (n + 31) / 32;
  const long long b = blockIdx.x / nbx;
  const int tx = threadIdx.x, ty = threadIdx.y, c = int(blockIdx.x - b * nbx) * 32 + tx;
  const double2* m = a + b * n * (long long)n;
  double sum = 0.0;
  if (c < n)
    for (int r = ty; r < n; r += 8) sum += hypot(m[(long long)r * n + c].x, m[(long long)r * n + c].y);
  part[ty][tx] = sum;
  __syncthreads();
  if (ty == 0) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += part[k][tx];
    for (int o = 16; o > 0; o >>= 1) {  // NaN-propagating max (fmax would drop a NaN column)
      const double u = __shfl_xor_sync(0xffffffffu, t, o);
      t = (isnan(t) || isnan(u)) ? __longlong_as_double(-1ll) : fmax(t, u);
    }
    if (tx == 0) atomicMax(nmax, (unsigned long long)__double_as_longlong(t));
  }
}

// out = x + c0 I + c1 a1 + c2 a2 + c3 a3 + c4 a4 over a batch (flat index)
__global__ void combo_flat_kernel(double2* __restrict__ out, const double2* __restrict__ x,
                                  const double2* __restrict__ a1, const double2* __restrict__ a2,
                                  const double2* __restrict__ a3, const double2* __restrict__ a4, double c0,
                                  double c1, double c2, double c3, double c4, int n, long long total) {
  const long long nn = (long long)n * n;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long e = q % nn;
    double2 v = x ? x[q] : make_double2(0.0, 0.0);
    if (e / n == e % n) v.x += c0;
    if (a1) { v.x += c1 * a1[q].x; v.y += c1 * a1[q].y; }
    if (a2) { v.x += c2 * a2[q].x; v.y += c2 * a2[q].y; }
    if (a3) { v.x += c3 * a3[q].x; v.y += c3 * a3[q].y; }
    if (a4) { v.x += c4 * a4[q].x; v.y += c4 * a4[q].y; }
    out[q] = v;
  }
}

unsigned grid_for(long long total) { return unsigned(std::min<long long>((total + 255) / 256, 148LL * 64)); }

// SoA planes <-> AoS (interleaved) for the AoS-only latency kernels
__global__ void planes_to_aos_kernel(const double* __restrict__ re, const double* __restrict__ im, long long count,
                                     double2* __restrict__ out) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < count) out[e] = make_double2(re[e], im[e]);
}
__global__ void aos_to_planes_kernel(const double2* __restrict__ in, long long count, double* __restrict__ re,
                                     double* __restrict__ im) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e < count) {
    const double2 z = in[e];
    re[e] = z.x;
    im[e] = z.y;
  }
}

__global__ void step_once_kernel(const double2* __restrict__ p, const double2* __restrict__ v,
                                 double2* __restrict__ out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double re = 0.0, im = 0.0;
  for (int j = 0; j < n; ++j) {
    const double2 a = p[(long long)i * n + j], b = v[j];
    re = fma(a.x, b.x, re);
    re = fma(-a.y, b.y, re);
    im = fma(a.x, b.y, im);
    im = fma(a.y, b.x, im);
  }
  out[i] = make_double2(re, im);
}

unsigned blocks_for(long long n, int t) { return unsigned((n + t - 1) / t); }

}  // namespace

void launch_build_lindbladian(size_t d, const double* h, size_t n_ops, const double* ops,
                              double* out, cudaStream_t s) {
  const long long nn = (long long)(d * d) * (long long)(d * d);
  build_lindbladian_kernel<<<blocks_for(nn, 256), 256, 0, s>>>(
      reinterpret_cast<const double2*>(h), reinterpret_cast<const double2*>(ops), int(n_ops),
      int(d), reinterpret_cast<double2*>(out));
  LBG_CHECK_LAUNCH("build_lindbladian_kernel");
}

void launch_build_lindbladian_batched(size_t d, const double* h, size_t n_ops, const double* ops, int64_t batch,
                                      double* out, cudaStream_t s) {
  if (batch <= 0) return;
  const long long total = (long long)batch * (long long)(d * d) * (long long)(d * d);
  build_lindbladian_batched_kernel<<<grid_for(total), 256, 0, s>>>(
      reinterpret_cast<const double2*>(h), reinterpret_cast<const double2*>(ops), int(n_ops), int(d), total,
      reinterpret_cast<double2*>(out));
  LBG_CHECK_LAUNCH("build_lindbladian_batched_kernel");
}

// Taylor coefficients 1/k!, k = 0..16
static double inv_fact(int k) {
  double f = 1.0;
  for (int i = 2; i <= k; ++i) f *= i;
  return 1.0 / f;
}

// P = exp(a dt): scaling and squaring around a degree-16 Taylor polynomial in
// Paterson-Stockmeyer form (s = 4): A2 = A A, A3 = A2 A, A4 = A2 A2,
//   P = B0 + A4 (B1 + A4 (B2 + A4 (B3 + c16 A4))),  B_j = sum_{i<4} c_{4j+i} A^i.
// 6 complex GEMMs on DMMA, no linear solve. Truncation error
// sum_{k>16} x^k/k! <= 2^-54 for x = ||A||_1 <= kTheta16 = 0.79 (A = a dt 2^-s).
// expm workspace: six n x n complex matrices, then the stream-K engine's control
// block for the large-n products (n >= kExpmStreamN)
static size_t expm_aux_offset(size_t n) { return (6 * n * n * 16 + 255) & ~size_t(255); }
size_t expm_workspace(size_t n) {
  return expm_aux_offset(n) + (n >= kExpmStreamN ? zgemm_stream_workspace(int(n)) : 0);
}

// Replaces lb::expm (expm.cpp:109-134: Pade-13, 6 matmuls + LU solve).
void expm_dev(const double* a, size_t n, double dt, double* out, double* work, cudaStream_t s) {
  constexpr double kTheta16 = 0.79;
  const long long nn = (long long)n * (long long)n;
  double2* w = reinterpret_cast<double2*>(work);
  double2 *A1 = w, *A2 = w + nn, *A3 = w + 2 * nn, *A4 = w + 3 * nn, *T = w + 4 * nn, *M = w + 5 * nn;
  double2* P = reinterpret_cast<double2*>(out);
  // ||a dt||_1 -> number of squarings (one host sync, like the reference's
  // synchronous expm; the result steers the launch sequence)
  double* colsum = reinterpret_cast<double*>(M);  // scratch
  colsum_kernel<<<blocks_for((long long)n, 32), dim3(32, 8), 0, s>>>(reinterpret_cast<const double2*>(a), int(n),
                                                                      colsum);
  LBG_CHECK_LAUNCH("colsum_kernel");
  std::vector<double> cs(n);
  check_cuda(cudaMemcpyAsync(cs.data(), colsum, sizeof(double) * n, cudaMemcpyDeviceToHost, s), "D2H norm");
  sync_stream_spin(s, "sync norm");
  double nrm = 0.0;
  for (double v : cs) nrm = (std::isnan(v) || v > nrm) ? v : nrm;  // a NaN column must not be dropped
  nrm *= std::fabs(dt);
  if (!std::isfinite(nrm)) throw invalid_argument("expm: non-finite entries in input");
  int sq = 0;
  if (nrm > kTheta16) {
    sq = int(std::ceil(std::log2(nrm / kTheta16)));
    if (sq > 64) throw runtime_error("expm: norm of a*dt requires more than 64 squarings");
  }
  const double scale = dt * std::ldexp(1.0, -sq);
  if (n <= size_t(kSmallN)) {  // one launch instead of eleven
    SmallCoef co;
    for (int k = 0; k <= 16; ++k) co.c[k] = inv_fact(k);
    small_expm_kernel<<<1, kSmallNN, 0, s>>>(reinterpret_cast<const double2*>(a), int(n), scale, sq, co, P);
    LBG_CHECK_LAUNCH("small_expm_kernel");
    return;
  }
  scale_kernel<<<blocks_for(nn, 256), 256, 0, s>>>(A1, reinterpret_cast<const double2*>(a), scale, nn);
  LBG_CHECK_LAUNCH("scale_kernel");
  const int ni = int(n);
  // one product per launch: stream-K on the persistent engine for large n (no
  // partial last wave), one tile per CTA below
  void* aux = reinterpret_cast<char*>(work) + expm_aux_offset(n);
  auto mm = [&](const double2* x, const double2* y, double2* z) {
    if (n >= kExpmStreamN)
      launch_zgemm_stream(reinterpret_cast<const double*>(x), reinterpret_cast<const double*>(y),
                          reinterpret_cast<double*>(z), ni, aux, s);
    else
      launch_zgemm(reinterpret_cast<const double*>(x), reinterpret_cast<const double*>(y), reinterpret_cast<double*>(z),
                   ni, 1, 0, 0, 0, s);
  };
  mm(A1, A1, A2);
  mm(A2, A1, A3);
  mm(A2, A2, A4);
  double c[17];
  for (int k = 0; k <= 16; ++k) c[k] = inv_fact(k);
  const unsigned g = blocks_for(nn, 256);
  // T = B3 + c16 A4
  combo_kernel<<<g, 256, 0, s>>>(T, nullptr, A1, A2, A3, A4, c[12], c[13], c[14], c[15], c[16], ni);
  LBG_CHECK_LAUNCH("combo_kernel");
  for (int j = 2; j >= 0; --j) {
    mm(A4, T, M);
    double2* dst = (j == 0 && sq == 0) ? P : T;
    combo_kernel<<<g, 256, 0, s>>>(dst, M, A1, A2, A3, nullptr, c[4 * j], c[4 * j + 1], c[4 * j + 2], c[4 * j + 3], 0.0, ni);
    LBG_CHECK_LAUNCH("combo_kernel");
  }
  // squarings: T holds the current value when sq > 0
  double2* cur = T;
  for (int i = 0; i < sq; ++i) {
    double2* dst = (i == sq - 1) ? P : (cur == T ? M : T);
    mm(cur, cur, dst);
    cur = dst;
  }
}

// Batched P_b = exp(a_b dt). n <= 16: one CTA per matrix (own scaling, equal
// to expm_dev per matrix). Larger n: the construction of expm_dev on batched
// tile GEMMs (launch_zgemm, the batch in chunks of 65,535 along grid z) with the
// batch's largest squaring count (one host sync for the norm, like expm_dev).
size_t expm_batched_workspace(size_t n, int64_t batch) {
  if (n <= size_t(kSmallN) || batch <= 0) return 256;
  return 6 * ((size_t(batch) * n * n * 16 + 255) & ~size_t(255)) + 256;
}
void expm_batched_dev(const double* a, size_t n, int64_t batch, double dt, double* out, void* work, cudaStream_t s) {
  if (batch <= 0) return;
  constexpr double kTheta16 = 0.79;
  const long long nn = (long long)n * (long long)n, total = (long long)batch * nn;
  char* w = static_cast<char*>(work);
  double c[17];
  for (int k = 0; k <= 16; ++k) c[k] = inv_fact(k);
  if (n <= size_t(kSmallN)) {
    unsigned* bad = reinterpret_cast<unsigned*>(w);
    check_cuda(cudaMemsetAsync(bad, 0, 4, s), "memset");
    SmallCoef co;
    for (int k = 0; k <= 16; ++k) co.c[k] = c[k];
    small_expm_batched_kernel<<<unsigned(batch), kSmallNN, 0, s>>>(reinterpret_cast<const double2*>(a), int(n), dt,
                                                                    co, reinterpret_cast<double2*>(out), bad);
    LBG_CHECK_LAUNCH("small_expm_batched_kernel");
    unsigned hbad = 0;
    check_cuda(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s), "D2H");
    sync_stream_spin(s, "sync");
    if (hbad & 1u) throw invalid_argument("expm: non-finite entries in input");
    if (hbad & 2u) throw runtime_error("expm: norm of a*dt requires more than 64 squarings");
    return;
  }
  const size_t mb = (size_t(total) * 16 + 255) & ~size_t(255);
  double2* M[6];
  for (int q = 0; q < 6; ++q) M[q] = reinterpret_cast<double2*>(w + q * mb);
  unsigned long long* nmax = reinterpret_cast<unsigned long long*>(w + 6 * mb);
  check_cuda(cudaMemsetAsync(nmax, 0, 8, s), "memset");
  norm_batched_kernel<<<unsigned(batch * ((static_cast<long long>(n) + 31) / 32)), dim3(32, 8), 0, s>>>(
      reinterpret_cast<const double2*>(a), int(n), batch, nmax);
  LBG_CHECK_LAUNCH("norm_batched_kernel");
  unsigned long long bits = 0;
  check_cuda(cudaMemcpyAsync(&bits, nmax, 8, cudaMemcpyDeviceToHost, s), "D2H norm");
  sync_stream_spin(s, "sync norm");
  double nrm;
  std::memcpy(&nrm, &bits, 8);
  nrm *= std::fabs(dt);
  if (!std::isfinite(nrm)) throw invalid_argument("expm: non-finite entries in input");
  int sq = 0;
  if (nrm > kTheta16) {
    sq = int(std::ceil(std::log2(nrm / kTheta16)));
    if (sq > 64) throw runtime_error("expm: norm of a*dt requires more than 64 squarings");
  }
  const double scale = dt * std::ldexp(1.0, -sq);
  double2 *A1 = M[0], *A2 = M[1], *A3 = M[2], *A4 = M[3], *T = M[4], *MM = M[5];
  double2* P = reinterpret_cast<double2*>(out);
  const unsigned g = grid_for(total);
  combo_flat_kernel<<<g, 256, 0, s>>>(A1, nullptr, reinterpret_cast<const double2*>(a), nullptr, nullptr, nullptr,
                                      0.0, scale, 0.0, 0.0, 0.0, int(n), total);
  LBG_CHECK_LAUNCH("combo_flat_kernel");
  auto mm = [&](const double2* x, const double2* y, double2* z) {
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
      const int cb = int(std::min<int64_t>(65535, batch - b0));
      launch_zgemm(reinterpret_cast<const double*>(x + b0 * nn), reinterpret_cast<const double*>(y + b0 * nn),
                   reinterpret_cast<double*>(z + b0 * nn), int(n), cb, nn, nn, nn, s);
    }
  };
  mm(A1, A1, A2);
  mm(A2, A1, A3);
  mm(A2, A2, A4);
  combo_flat_kernel<<<g, 256, 0, s>>>(T, nullptr, A1, A2, A3, A4, c[12], c[13], c[14], c[15], c[16], int(n), total);
  LBG_CHECK_LAUNCH("combo_flat_kernel");
  for (int j = 2; j >= 0; --j) {
    mm(A4, T, MM);
    double2* dst = (j == 0 && sq == 0) ? P : T;
    combo_flat_kernel<<<g, 256, 0, s>>>(dst, MM, A1, A2, A3, nullptr, c[4 * j], c[4 * j + 1], c[4 * j + 2],
                                        c[4 * j + 3], 0.0, int(n), total);
    LBG_CHECK_LAUNCH("combo_flat_kernel");
  }
  double2* cur = T;
  for (int i = 0; i < sq; ++i) {
    double2* dst = (i == sq - 1) ? P : (cur == T ? MM : T);
    mm(cur, cur, dst);
    cur = dst;
  }
}

void launch_check_state(const double* x, size_t d, int64_t batch, double* out3, cudaStream_t s) {
  // keys live in the 3 doubles after out3's slot? use a small static device buffer per call
  unsigned long long* keys = nullptr;
  check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&keys), 3 * sizeof(unsigned long long), s), "malloc keys");
  check_state_init<<<1, 32, 0, s>>>(keys);
  LBG_CHECK_LAUNCH("check_state_init");
  if (batch > 0) {
    if (d >= 6) {
      check_state_warp_kernel<<<blocks_for(batch * 32, 256), 256, 0, s>>>(reinterpret_cast<const double2*>(x),
                                                                         int(d), batch, keys);
      LBG_CHECK_LAUNCH("check_state_warp_kernel");
    } else {
      check_state_kernel<<<blocks_for(batch, 256), 256, 0, s>>>(reinterpret_cast<const double2*>(x), int(d), batch,
                                                                 keys);
      LBG_CHECK_LAUNCH("check_state_kernel");
    }
  }
  check_state_finish<<<1, 32, 0, s>>>(keys, out3);
  LBG_CHECK_LAUNCH("check_state_finish");
  check_cuda(cudaFreeAsync(keys, s), "free keys");
}

void launch_step_once(const double* p, const double* v, double* out, size_t n, cudaStream_t s) {
  step_once_kernel<<<blocks_for((long long)n, 128), 128, 0, s>>>(
      reinterpret_cast<const double2*>(p), reinterpret_cast<const double2*>(v),
      reinterpret_cast<double2*>(out), int(n));
  LBG_CHECK_LAUNCH("step_once_kernel");
}

void launch_planes_to_aos(const double* re, const double* im, long long count, double* out, cudaStream_t s) {
  if (count <= 0) return;
  planes_to_aos_kernel<<<unsigned((count + 255) / 256), 256, 0, s>>>(re, im, count, reinterpret_cast<double2*>(out));
  LBG_CHECK_LAUNCH("planes_to_aos_kernel");
}
void launch_aos_to_planes(const double* in, long long count, double* re, double* im, cudaStream_t s) {
  if (count <= 0) return;
  aos_to_planes_kernel<<<unsigned((count + 255) / 256), 256, 0, s>>>(reinterpret_cast<const double2*>(in), count,
                                                                     re, im);
  LBG_CHECK_LAUNCH("aos_to_planes_kernel");
}

}  // namespace lbg
