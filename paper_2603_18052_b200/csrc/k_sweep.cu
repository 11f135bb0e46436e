// k_sweep.cu — config 4 ("robustness atlas"): per-trajectory propagators.
// For every trajectory b:   H_b = h0 + delta_b hd + scale_b hs,
//   K5  L_b dt  assembled on the GPU by the Kronecker formula (dissipator part
//       D = sum_k [L_k (x) conj L_k - ...] is trajectory independent, built once),
//   K4  P_b = exp(L_b dt) by batched Taylor-16 / Paterson-Stockmeyer on DMMA
//       (the batched complex GEMM of k_tiled.cu),
//   K3  rho_b <- P_b^steps rho0 with P_b resident in shared memory; epilogue
//       writes the populations and adds rho_b into the ensemble sum.
// Trajectories are processed in chunks so the per-trajectory matrices
// (7 x 105 KB at d = 9) fit a bounded workspace; P_b never leaves the GPU.
//
// Replaces, per trajectory, make_model + build_lindbladian + expm + the step
// loop of lb::grape_chain (proj/src/propagate.cpp:130-160).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "internal.hpp"
#include "small_expm.cuh"

namespace lbg {

namespace {

constexpr int64_t kChunk = 4096;
constexpr int kThetaSq = 0;  // see host side

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// A_b = scale_dt * (D + coherent(H_b)),  coherent(H)[(i,k),(j,l)] = -i (H_ij d_kl - d_ij H_lk)
__global__ void sweep_assemble_kernel(const double2* __restrict__ dis, const double2* __restrict__ h0,
                                      const double2* __restrict__ hd, const double2* __restrict__ hs,
                                      const double* __restrict__ delta, const double* __restrict__ scale,
                                      int d, double sdt, double2* __restrict__ A, long long stride) {
  const int n = d * d;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (e >= n * n) return;
  const int R = e / n, C = e - R * n;
  const int i = R / d, k = R - i * d, j = C / d, l = C - j * d;
  const double db = delta[b], sb = scale[b];
  double2 acc = dis[e];
  // -i * x = (x.im, -x.re)
  if (k == l) {
    const double2 hij = make_double2(h0[i * d + j].x + db * hd[i * d + j].x + sb * hs[i * d + j].x,
                                     h0[i * d + j].y + db * hd[i * d + j].y + sb * hs[i * d + j].y);
    acc.x += hij.y;
    acc.y -= hij.x;
  }
  if (i == j) {
    const double2 hlk = make_double2(h0[l * d + k].x + db * hd[l * d + k].x + sb * hs[l * d + k].x,
                                     h0[l * d + k].y + db * hd[l * d + k].y + sb * hs[l * d + k].y);
    acc.x -= hlk.y;
    acc.y += hlk.x;
  }
  A[b * stride + e] = make_double2(acc.x * sdt, acc.y * sdt);
}

// batched out = x + c0 I + c1 a1 + c2 a2 + c3 a3 + c4 a4
__global__ void combo_batched_kernel(double2* __restrict__ out, const double2* __restrict__ x,
                                     const double2* __restrict__ a1, const double2* __restrict__ a2,
                                     const double2* __restrict__ a3, const double2* __restrict__ a4,
                                     double c0, double c1, double c2, double c3, double c4, int n,
                                     long long stride) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * n) return;
  const long long o = blockIdx.y * stride + e;
  const int r = e / n, c = e - r * n;
  double2 v = x ? x[o] : make_double2(0.0, 0.0);
  if (r == c) v.x += c0;
  if (a1) { v.x += c1 * a1[o].x; v.y += c1 * a1[o].y; }
  if (a2) { v.x += c2 * a2[o].x; v.y += c2 * a2[o].y; }
  if (a3) { v.x += c3 * a3[o].x; v.y += c3 * a3[o].y; }
  if (a4) { v.x += c4 * a4[o].x; v.y += c4 * a4[o].y; }
  out[o] = v;
}

// max over the batch of the 1-norms (max column sum of |A|): block = 32 columns
// x 8 row groups of one matrix (coalesced rows, 8-way parallel column sums)
__global__ void sweep_norm_kernel(const double2* __restrict__ A, int n, long long stride,
                                  unsigned long long* __restrict__ nmax) {
  __shared__ double part[8][33];
  const int tx = threadIdx.x, ty = threadIdx.y, c = blockIdx.x * 32 + tx;
  const double2* m = A + (long long)blockIdx.y * stride;
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

// K3: one CTA per trajectory, P_b resident in shared memory (row stride n = 81
// complex is odd, so the 32 rows a warp reads per j hit distinct 16-B groups).
__global__ void __launch_bounds__(96) sweep_step_kernel(const double2* __restrict__ P, long long stride,
                                                       const double2* __restrict__ rho0, int d,
                                                       int64_t steps, double* __restrict__ pops,
                                                       double* __restrict__ ens_sum) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = d * d;
  double2* ps = reinterpret_cast<double2*>(smem);
  double2* va = ps + n * n;
  double2* vb = va + n;
  const int b = blockIdx.x;
  const double2* pb = P + b * stride;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) ps[e] = pb[e];
  for (int e = threadIdx.x; e < n; e += blockDim.x) va[e] = rho0[e];
  __syncthreads();
  const int i = threadIdx.x;
  for (int64_t s = 0; s < steps; ++s) {
    if (i < n) {
      double re = 0.0, im = 0.0, re2 = 0.0, im2 = 0.0;
      const double2* row = ps + i * n;
      int j = 0;
      for (; j + 1 < n; j += 2) {
        const double2 a = row[j], v = va[j];
        const double2 a2 = row[j + 1], v2 = va[j + 1];
        re = fma(a.x, v.x, re);
        re = fma(-a.y, v.y, re);
        im = fma(a.x, v.y, im);
        im = fma(a.y, v.x, im);
        re2 = fma(a2.x, v2.x, re2);
        re2 = fma(-a2.y, v2.y, re2);
        im2 = fma(a2.x, v2.y, im2);
        im2 = fma(a2.y, v2.x, im2);
      }
      if (j < n) {
        const double2 a = row[j], v = va[j];
        re = fma(a.x, v.x, re);
        re = fma(-a.y, v.y, re);
        im = fma(a.x, v.y, im);
        im = fma(a.y, v.x, im);
      }
      vb[i] = make_double2(re + re2, im + im2);
    }
    __syncthreads();
    double2* t = va;
    va = vb;
    vb = t;
  }
  if (i < d) pops[(long long)b * d + i] = va[i * d + i].x;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    atomicAdd(&ens_sum[2 * e], va[e].x);
    atomicAdd(&ens_sum[2 * e + 1], va[e].y);
  }
}

// GRAPE segment propagators for n = d^2 <= 16 in ONE launch: one CTA per
// segment, thread e owns element e of every n x n matrix, everything in shared
// memory. Same construction as the batched path (sweep_assemble_kernel +
// Taylor-16 / Paterson-Stockmeyer), with the squaring count chosen per segment
// on the device (no host round trip for the norm).
__global__ void __launch_bounds__(kSmallN * kSmallN) grape_small_build_kernel(
    const double2* __restrict__ dis, const double2* __restrict__ h0, const double2* __restrict__ hc,
    const double* __restrict__ amps, int d, double dt, double theta, const double* __restrict__ cf,
    double2* __restrict__ props) {
  constexpr int NN = kSmallN * kSmallN;
  __shared__ double2 A[NN], A2[NN], A3[NN], A4[NN], T[NN];
  __shared__ double colsum[kSmallN];
  __shared__ int s_sq;
  const int n = d * d, e = threadIdx.x, seg = blockIdx.x;
  const bool own = e < n * n;
  const int r = own ? e / n : 0, c = own ? e - r * n : 0;
  const double aj = amps[seg];
  if (own) {  // dt * (D + coherent(h0 + a_j hc))
    const int i = r / d, k = r - i * d, j = c / d, l = c - j * d;
    double2 acc = dis[e];
    if (k == l) {
      const double2 hij = make_double2(h0[i * d + j].x + aj * hc[i * d + j].x, h0[i * d + j].y + aj * hc[i * d + j].y);
      acc.x += hij.y;
      acc.y -= hij.x;
    }
    if (i == j) {
      const double2 hlk = make_double2(h0[l * d + k].x + aj * hc[l * d + k].x, h0[l * d + k].y + aj * hc[l * d + k].y);
      acc.x -= hlk.y;
      acc.y += hlk.x;
    }
    A[e] = make_double2(acc.x * dt, acc.y * dt);
  }
  __syncthreads();
  if (e < n) {
    double cs = 0.0;
    for (int q = 0; q < n; ++q) cs += hypot(A[q * n + e].x, A[q * n + e].y);
    colsum[e] = cs;
  }
  __syncthreads();
  if (e == 0) {
    double nrm = 0.0;
    for (int q = 0; q < n; ++q) nrm = fmax(nrm, colsum[q]);
    int sq = nrm > theta ? int(ceil(log2(nrm / theta))) : 0;
    s_sq = sq < 0 ? 0 : sq;
  }
  __syncthreads();
  const int sq = s_sq;
  const double sc = ldexp(1.0, -sq);
  if (own) A[e] = make_double2(A[e].x * sc, A[e].y * sc);
  __syncthreads();
  small_taylor(A, A2, A3, A4, T, n, cf, sq);
  if (own) props[(long long)seg * n * n + e] = T[e];
}

double inv_fact(int k) {
  double f = 1.0;
  for (int i = 2; i <= k; ++i) f *= i;
  return 1.0 / f;
}

}  // namespace

size_t sweep_workspace(size_t d, int64_t batch) {
  const size_t n = d * d;
  const size_t chunk = size_t(std::min<int64_t>(std::max<int64_t>(batch, 1), kChunk));
  return 7 * align_up(chunk * n * n * 16) + align_up(n * n * 16) + 256;
}

// Batched complex propagators P_b = exp(dt (D + C(h0 + delta_b hd + scale_b hs)))
// for b in [0, batch), chunk by chunk: K5 assembly, one norm pass (common
// squaring count), Taylor-16 / Paterson-Stockmeyer on the batched DMMA GEMM.
// on_chunk(P, c0, cb) runs after chunk [c0, c0+cb)'s propagators are ready.
namespace {
template <class F>
void propagators_complex(size_t d, const double* h0, const double* hd, const double* hs, size_t n_ops,
                         const double* ops, const double* delta, const double* scale, double dt,
                         int64_t batch, void* work, cudaStream_t s, F&& on_chunk) {
  const int n = int(d * d);
  const long long nn = (long long)n * n;
  const size_t chunk = size_t(std::min<int64_t>(std::max<int64_t>(batch, 1), kChunk));
  char* w = static_cast<char*>(work);
  const size_t mb = align_up(chunk * nn * 16);
  double2* M[7];
  for (int q = 0; q < 7; ++q) M[q] = reinterpret_cast<double2*>(w + q * mb);
  double2* dis = reinterpret_cast<double2*>(w + 7 * mb);
  unsigned long long* nmax = reinterpret_cast<unsigned long long*>(w + 7 * mb + align_up(nn * 16));

  // trajectory-independent dissipator D = build_lindbladian(H = 0, ops)
  check_cuda(cudaMemsetAsync(M[0], 0, d * d * 16, s), "memset");
  launch_build_lindbladian(d, reinterpret_cast<const double*>(M[0]), n_ops, ops,
                           reinterpret_cast<double*>(dis), s);
  if (batch == 0) return;

  // one pass over all trajectories' norms fixes a common squaring count
  check_cuda(cudaMemsetAsync(nmax, 0, 8, s), "memset");
  for (int64_t c0 = 0; c0 < batch; c0 += int64_t(chunk)) {
    const int cb = int(std::min<int64_t>(int64_t(chunk), batch - c0));
    sweep_assemble_kernel<<<dim3((nn + 255) / 256, cb), 256, 0, s>>>(
        dis, reinterpret_cast<const double2*>(h0), reinterpret_cast<const double2*>(hd),
        reinterpret_cast<const double2*>(hs), delta + c0, scale + c0, int(d), dt, M[0], nn);
    LBG_CHECK_LAUNCH("sweep_assemble_kernel");
    sweep_norm_kernel<<<dim3(unsigned((n + 31) / 32), unsigned(cb)), dim3(32, 8), 0, s>>>(M[0], n, nn, nmax);
    LBG_CHECK_LAUNCH("sweep_norm_kernel");
  }
  unsigned long long bits = 0;
  check_cuda(cudaMemcpyAsync(&bits, nmax, 8, cudaMemcpyDeviceToHost, s), "D2H");
  sync_stream_spin(s, "sync");
  double nrm;
  std::memcpy(&nrm, &bits, 8);
  if (!std::isfinite(nrm)) throw invalid_argument("sweep: non-finite generator");
  constexpr double kTheta16 = 0.79;
  int sq = 0;
  if (nrm > kTheta16) sq = int(std::ceil(std::log2(nrm / kTheta16)));
  if (sq > 64) throw runtime_error("sweep: norm requires more than 64 squarings");
  const double sdt = dt * std::ldexp(1.0, -sq);
  (void)kThetaSq;

  double c[17];
  for (int k = 0; k <= 16; ++k) c[k] = inv_fact(k);
  double2 *A1 = M[0], *A2 = M[1], *A3 = M[2], *A4 = M[3], *T = M[4], *MM = M[5], *P = M[6];
  for (int64_t c0 = 0; c0 < batch; c0 += int64_t(chunk)) {
    const int cb = int(std::min<int64_t>(int64_t(chunk), batch - c0));
    const dim3 eg((nn + 255) / 256, cb);
    sweep_assemble_kernel<<<eg, 256, 0, s>>>(
        dis, reinterpret_cast<const double2*>(h0), reinterpret_cast<const double2*>(hd),
        reinterpret_cast<const double2*>(hs), delta + c0, scale + c0, int(d), sdt, A1, nn);
    LBG_CHECK_LAUNCH("sweep_assemble_kernel");
    auto mm = [&](const double2* a, const double2* b, double2* out) {
      launch_zgemm(reinterpret_cast<const double*>(a), reinterpret_cast<const double*>(b),
                   reinterpret_cast<double*>(out), n, cb, nn, nn, nn, s);
    };
    mm(A1, A1, A2);
    mm(A2, A1, A3);
    mm(A2, A2, A4);
    combo_batched_kernel<<<eg, 256, 0, s>>>(T, nullptr, A1, A2, A3, A4, c[12], c[13], c[14], c[15], c[16], n, nn);
    LBG_CHECK_LAUNCH("combo_batched_kernel");
    for (int j = 2; j >= 0; --j) {
      mm(A4, T, MM);
      double2* dst = (j == 0 && sq == 0) ? P : T;
      combo_batched_kernel<<<eg, 256, 0, s>>>(dst, MM, A1, A2, A3, nullptr, c[4 * j], c[4 * j + 1],
                                              c[4 * j + 2], c[4 * j + 3], 0.0, n, nn);
      LBG_CHECK_LAUNCH("combo_batched_kernel");
    }
    double2* cur = T;
    for (int i = 0; i < sq; ++i) {
      double2* dst = (i == sq - 1) ? P : (cur == T ? MM : T);
      mm(cur, cur, dst);
      cur = dst;
    }
    on_chunk(P, c0, cb);
  }
}

}  // namespace

void launch_sweep(size_t d, const double* h0, const double* hd, const double* hs, size_t n_ops,
                  const double* ops, const double* delta, const double* scale, double dt,
                  const double* rho0, int64_t batch, int64_t steps, double* pops, double* ens_sum,
                  void* work, cudaStream_t s) {
  if (!work) throw invalid_argument("sweep: workspace required");
  if (d * d > 96) throw invalid_argument("sweep: supports d*d <= 96");
  const int n = int(d * d);
  const long long nn = (long long)n * n;
  check_cuda(cudaMemsetAsync(ens_sum, 0, size_t(n) * 16, s), "memset ens");
  const size_t smem = size_t(nn + 2 * n) * 16;
  ensure_max_dyn_smem((const void*)sweep_step_kernel, int(smem));
  propagators_complex(d, h0, hd, hs, n_ops, ops, delta, scale, dt, batch, work, s,
                      [&](const double2* P, int64_t c0, int cb) {
                        sweep_step_kernel<<<cb, 96, smem, s>>>(P, nn, reinterpret_cast<const double2*>(rho0),
                                                               int(d), steps, pops + c0 * int64_t(d), ens_sum);
                        LBG_CHECK_LAUNCH("sweep_step_kernel");
                      });
}

size_t grape_workspace(size_t d, int64_t segments) {
  const size_t n = d * d;
  return sweep_workspace(d, segments) + align_up(size_t(segments) * n * n * 16) + align_up(n * 16) +
         std::max(tiled_workspace(n, 1), rowsplit_workspace(n, 1));
}

// GRAPE piecewise-constant chain (propagate.cpp:111-168): every segment's
// propagator P_j = exp(dt L(h0 + a_j hc)) is independent of the state, so all
// of them are built in ONE batched pass (timed as build), then the state walks
// the chain segment by segment on the step kernels (timed as chain).
void launch_grape(size_t d, const double* h0, const double* hc, const double* zero_h, size_t n_ops,
                  const double* ops, const double* amps, const double* zeros, int64_t segments,
                  int64_t steps_per_segment, double dt, double* x, void* work, cudaStream_t s,
                  cudaEvent_t ev_build_end) {
  const size_t n = d * d;
  const long long nn = (long long)n * n;
  char* w = static_cast<char*>(work);
  double2* props = reinterpret_cast<double2*>(w + sweep_workspace(d, segments));
  void* ework = w + sweep_workspace(d, segments) + align_up(size_t(segments) * nn * 16) + align_up(n * 16);
  if (n <= size_t(kSmallN)) {
    // small systems (d <= 4): two launches in total — every propagator in one
    // build kernel, then the whole chain in one kernel
    double2* dis = reinterpret_cast<double2*>(w);
    double* cf = reinterpret_cast<double*>(w + align_up(nn * 16));
    double hcf[17];
    for (int k = 0; k <= 16; ++k) hcf[k] = inv_fact(k);
    check_cuda(cudaMemcpyAsync(cf, hcf, sizeof hcf, cudaMemcpyHostToDevice, s), "H2D coefficients");
    launch_build_lindbladian(d, zero_h, n_ops, ops, reinterpret_cast<double*>(dis), s);
    grape_small_build_kernel<<<unsigned(segments), kSmallN * kSmallN, 0, s>>>(
        dis, reinterpret_cast<const double2*>(h0), reinterpret_cast<const double2*>(hc), amps, int(d), dt, 0.79,
        cf, props);
    LBG_CHECK_LAUNCH("grape_small_build_kernel");
    if (ev_build_end) check_cuda(cudaEventRecord(ev_build_end, s), "event");
    launch_chain_segments(reinterpret_cast<const double*>(props), n, segments, steps_per_segment, x, s);
    return;
  }
  propagators_complex(d, h0, hc, zero_h, n_ops, ops, amps, zeros, dt, segments, w, s,
                      [&](const double2* P, int64_t c0, int cb) {
                        check_cuda(cudaMemcpyAsync(props + c0 * nn, P, size_t(cb) * nn * 16,
                                                   cudaMemcpyDeviceToDevice, s),
                                   "D2D P");
                      });
  if (ev_build_end) check_cuda(cudaEventRecord(ev_build_end, s), "event");
  if (cta_chain_supported(n) && !chain_supported(n)) {  // d <= 9: the whole chain in one launch
    launch_cta_chain_segments(reinterpret_cast<const double*>(props), n, segments, steps_per_segment, x, s);
    return;
  }
  for (int64_t j = 0; j < segments; ++j) {
    const double* pj = reinterpret_cast<const double*>(props + j * nn);
    if (chain_supported(n))
      launch_chain(pj, n, nullptr, nullptr, x, 1, steps_per_segment, Layout::aos, s);
    else if (cta_chain_supported(n))
      launch_cta_chain(pj, n, x, 1, steps_per_segment, s);
    else if (rowsplit_supported(n, 1))
      launch_rowsplit(pj, n, x, 1, steps_per_segment, ework, s);
    else
      launch_tiled_evolve(pj, n, nullptr, nullptr, x, 1, steps_per_segment, Layout::aos, ework, s);
  }
}

}  // namespace lbg
