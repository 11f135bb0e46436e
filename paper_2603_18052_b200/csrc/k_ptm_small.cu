// k_ptm_small.cu — per-trajectory propagators for small systems (d <= 3,
// n = d^2 <= 9) in the real transfer-matrix representation (k_ptm.cu header):
// the "tiny d" regime of a parameter sweep, where one CTA per trajectory would
// leave most of the SM idle.
//
//   build: one WARP per trajectory — L_R assembled entrywise (dissipator part
//     precomputed once), per-trajectory 1-norm and squaring count, Taylor-16 in
//     Paterson-Stockmeyer form on n x n real matrices in the warp's slice of
//     shared memory (each lane owns n^2/32 entries), squarings; P_R -> HBM
//     (n^2 doubles per trajectory, 648 B at d = 3).
//   step: one THREAD per trajectory — P_R (n^2 doubles) and the state (n) in
//     registers for all steps, n independent FMA chains per step; populations
//     out; the ensemble sum reduced per warp with shuffles, one atomic per value.
//
// Replaces, per trajectory, make_model + build_lindbladian + expm + the step
// loop of lb::grape_chain (proj/src/propagate.cpp:130-160), as k_ptm.cu does
// for d = 9.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "internal.hpp"

namespace lbg {
namespace {

constexpr int kBuildWarps = 4;
constexpr double kTheta = 0.79;  // Taylor-16 truncation <= 2^-54 relative for ||A||_1 <= 0.79

template <int D>
__device__ __forceinline__ double2 kron_coh(const double2* __restrict__ h, int q, int p) {
  // -i (H (x) I - I (x) H^T) entry (q, p), q = (i,k), p = (j,l)
  const int i = q / D, k = q - i * D, j = p / D, l = p - j * D;
  double2 v = make_double2(0.0, 0.0);
  if (k == l) {
    const double2 a = h[i * D + j];
    v.x += a.y;
    v.y -= a.x;
  }
  if (i == j) {
    const double2 a = h[l * D + k];
    v.x -= a.y;
    v.y += a.x;
  }
  return v;
}

template <int D, class F>
__device__ __forceinline__ double real_entry_d(F&& lq, int q, int s) {
  const int si = s / D, sj = s - si * D;
  double2 c;
  if (si == sj) {
    c = lq(s);
  } else {
    const double2 a = lq(s), bt = lq(sj * D + si);
    c = si < sj ? make_double2(a.x + bt.x, a.y + bt.y) : make_double2(a.y - bt.y, bt.x - a.x);
  }
  const int qi = q / D, qj = q - qi * D;
  return qi <= qj ? c.x : -c.y;
}

template <int D>
__global__ void small_dissipator_kernel(const double2* __restrict__ dis, double* __restrict__ dr) {
  constexpr int N = D * D;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N * N) return;
  const int q = e / N, s = e - q * N;
  dr[e] = real_entry_d<D>([&](int p) { return dis[q * N + p]; }, q, s);
}

// warp-level n x n real product, lane-strided over the n^2 entries
template <int N>
__device__ __forceinline__ void warp_mm(const double* __restrict__ X, const double* __restrict__ Y,
                                        double* __restrict__ Z, int lane) {
  for (int e = lane; e < N * N; e += 32) {
    const int r = e / N, c = e - r * N;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) acc = fma(X[r * N + k], Y[k * N + c], acc);
    Z[e] = acc;
  }
  __syncwarp();
}

template <int D>
__global__ void __launch_bounds__(32 * kBuildWarps) small_build_kernel(
    const double* __restrict__ dr, const double2* __restrict__ h0, const double2* __restrict__ hd,
    const double2* __restrict__ hs, const double* __restrict__ delta, const double* __restrict__ scale, double dt,
    int64_t count, const double* __restrict__ cf, double* __restrict__ pr_out) {
  constexpr int N = D * D, NN = N * N;
  __shared__ double mats[kBuildWarps][6][NN];
  __shared__ double2 hbuf[kBuildWarps][D * D];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b = int64_t(blockIdx.x) * kBuildWarps + w;
  if (b >= count) return;  // whole warp
  double *A = mats[w][0], *A2 = mats[w][1], *A3 = mats[w][2], *A4 = mats[w][3], *T = mats[w][4], *U = mats[w][5];
  double2* hb = hbuf[w];
  const double db = delta[b], sb = scale[b];
  for (int e = lane; e < D * D; e += 32)
    hb[e] = make_double2(h0[e].x + db * hd[e].x + sb * hs[e].x, h0[e].y + db * hd[e].y + sb * hs[e].y);
  __syncwarp();
  for (int e = lane; e < NN; e += 32) {
    const int q = e / N, s = e - q * N;
    A[e] = (dr[e] + real_entry_d<D>([&](int p) { return kron_coh<D>(hb, q, p); }, q, s)) * dt;
  }
  __syncwarp();
  // ||A||_1 (max column sum) -> squarings, per trajectory
  double cs = 0.0;
  if (lane < N)
    for (int r = 0; r < N; ++r) cs += fabs(A[r * N + lane]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cs = fmax(cs, __shfl_xor_sync(0xffffffffu, cs, o));
  int sq = cs > kTheta ? int(ceil(log2(cs / kTheta))) : 0;
  sq = sq < 0 ? 0 : sq;
  const double sc = ldexp(1.0, -sq);
  for (int e = lane; e < NN; e += 32) A[e] *= sc;
  __syncwarp();
  warp_mm<N>(A, A, A2, lane);
  warp_mm<N>(A2, A, A3, lane);
  warp_mm<N>(A2, A2, A4, lane);
  auto combo = [&](int e, double x, double c0, double c1, double c2, double c3) {
    const int r = e / N, c = e - r * N;
    return x + (r == c ? c0 : 0.0) + c1 * A[e] + c2 * A2[e] + c3 * A3[e];
  };
  for (int e = lane; e < NN; e += 32) T[e] = combo(e, cf[16] * A4[e], cf[12], cf[13], cf[14], cf[15]);
  __syncwarp();
  for (int j = 2; j >= 0; --j) {  // T = A4 T + B_j
    warp_mm<N>(A4, T, U, lane);
    for (int e = lane; e < NN; e += 32) T[e] = combo(e, U[e], cf[4 * j], cf[4 * j + 1], cf[4 * j + 2], cf[4 * j + 3]);
    __syncwarp();
  }
  for (int q = 0; q < sq; ++q) {
    warp_mm<N>(T, T, U, lane);
    for (int e = lane; e < NN; e += 32) T[e] = U[e];
    __syncwarp();
  }
  for (int e = lane; e < NN; e += 32) pr_out[b * NN + e] = T[e];
}

// one thread per trajectory; P_R and the state in registers
template <int D>
__global__ void __launch_bounds__(128) small_step_kernel(const double* __restrict__ pr, const double* __restrict__ x0,
                                                         int64_t count, int64_t steps, double* __restrict__ pops,
                                                         double* __restrict__ ens_x) {
  constexpr int N = D * D;
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool live = b < count;
  double p[N * N], x[N];
#pragma unroll
  for (int e = 0; e < N * N; ++e) p[e] = live ? pr[b * N * N + e] : 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) x[i] = x0[i];
#pragma unroll 1
  for (int64_t s = 0; s < steps; ++s) {
    double y[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) a = fma(p[i * N + j], x[j], a);
      y[i] = a;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = y[i];
  }
  if (live)
#pragma unroll
    for (int i = 0; i < D; ++i) pops[b * D + i] = x[i * D + i];
  // ensemble: warp sum, then one atomic per value from lane 0
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double v = live ? x[i] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&ens_x[i], v);
  }
}

__global__ void small_rho_to_x_kernel(const double2* __restrict__ rho, int d, double* __restrict__ x) {
  const int p = threadIdx.x, n = d * d;
  if (p >= n) return;
  const int i = p / d, j = p - i * d;
  x[p] = i <= j ? rho[p].x : -rho[p].y;
}
__global__ void small_x_to_rho_kernel(const double* __restrict__ x, int d, double2* __restrict__ rho) {
  const int p = threadIdx.x, n = d * d;
  if (p >= n) return;
  const int i = p / d, j = p - i * d;
  if (i == j)
    rho[p] = make_double2(x[p], 0.0);
  else if (i < j)
    rho[p] = make_double2(x[p], x[j * d + i]);
  else
    rho[p] = make_double2(x[j * d + i], -x[p]);
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

template <int D>
void run_small(const double* h0, const double* hd, const double* hs, size_t n_ops, const double* ops,
               const double* delta, const double* scale, double dt, const double* rho0, int64_t batch,
               int64_t steps, double* pops, double* ens_sum, void* work, cudaStream_t s) {
  constexpr int N = D * D;
  char* w = static_cast<char*>(work);
  double* pr = reinterpret_cast<double*>(w);                                            // batch x N x N
  double2* dis = reinterpret_cast<double2*>(w + align_up(size_t(batch) * N * N * 8));     // N x N complex
  double2* zero_h = reinterpret_cast<double2*>(reinterpret_cast<char*>(dis) + align_up(size_t(N) * N * 16));
  double* dr = reinterpret_cast<double*>(zero_h + 16);  // after D x D (<= 16) complex zeros
  double* x0 = dr + N * N;            // N
  double* ens_x = x0 + 16;            // N
  double* cf = ens_x + 16;            // 17
  double hcf[17];
  hcf[0] = 1.0;
  for (int k = 1; k <= 16; ++k) hcf[k] = hcf[k - 1] / k;
  check_cuda(cudaMemcpyAsync(cf, hcf, sizeof hcf, cudaMemcpyHostToDevice, s), "H2D coefficients");
  check_cuda(cudaMemsetAsync(zero_h, 0, size_t(D) * D * 16, s), "memset");
  check_cuda(cudaMemsetAsync(ens_x, 0, N * 8, s), "memset");
  launch_build_lindbladian(D, reinterpret_cast<const double*>(zero_h), n_ops, ops, reinterpret_cast<double*>(dis), s);
  small_dissipator_kernel<D><<<(N * N + 255) / 256, 256, 0, s>>>(dis, dr);
  LBG_CHECK_LAUNCH("small_dissipator_kernel");
  small_rho_to_x_kernel<<<1, 32, 0, s>>>(reinterpret_cast<const double2*>(rho0), D, x0);
  LBG_CHECK_LAUNCH("small_rho_to_x_kernel");
  small_build_kernel<D><<<unsigned((batch + kBuildWarps - 1) / kBuildWarps), 32 * kBuildWarps, 0, s>>>(
      dr, reinterpret_cast<const double2*>(h0), reinterpret_cast<const double2*>(hd),
      reinterpret_cast<const double2*>(hs), delta, scale, dt, batch, cf, pr);
  LBG_CHECK_LAUNCH("small_build_kernel");
  small_step_kernel<D><<<unsigned((batch + 127) / 128), 128, 0, s>>>(pr, x0, batch, steps, pops, ens_x);
  LBG_CHECK_LAUNCH("small_step_kernel");
  small_x_to_rho_kernel<<<1, 32, 0, s>>>(ens_x, D, reinterpret_cast<double2*>(ens_sum));
  LBG_CHECK_LAUNCH("small_x_to_rho_kernel");
}

}  // namespace

bool ptm_small_supported(size_t d) { return d >= 2 && d <= 3; }  // P_R of d = 4 (256 doubles) would not fit in registers

size_t ptm_small_workspace(size_t d, int64_t batch) {
  const size_t n = d * d;
  return align_up(size_t(std::max<int64_t>(batch, 1)) * n * n * 8) + align_up(n * n * 16) +
         align_up((n * n + 16 + 16 + 24) * 8 + 16 * 16) + 256;
}

void launch_ptm_sweep_small(size_t d, const double* h0, const double* hd, const double* hs, size_t n_ops,
                            const double* ops, const double* delta, const double* scale, double dt,
                            const double* rho0, int64_t batch, int64_t steps, double* pops, double* ens_sum,
                            void* work, cudaStream_t s) {
  if (batch <= 0) {
    check_cuda(cudaMemsetAsync(ens_sum, 0, d * d * 16, s), "memset");
    return;
  }
  switch (d) {
    case 2: return run_small<2>(h0, hd, hs, n_ops, ops, delta, scale, dt, rho0, batch, steps, pops, ens_sum, work, s);
    case 3: return run_small<3>(h0, hd, hs, n_ops, ops, delta, scale, dt, rho0, batch, steps, pops, ens_sum, work, s);
    default: throw invalid_argument("small ptm sweep supports d in [2, 3]");
  }
}

}  // namespace lbg
