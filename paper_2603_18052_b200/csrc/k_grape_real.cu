// k_grape_real.cu — the GRAPE chain (propagate.cpp:111-168) for large d in the
// real transfer-matrix representation (k_ptm.cu header): a Hermitian rho0 and
// Hermiticity-preserving segment propagators make every step a REAL n x n
// matvec on rho's real coordinates, and every segment's propagator a real
// exponential — 4x fewer flops in the build, which dominates at d = 27.
//
//   build: L_R,j = D_R + coherent_R(h0 + a_j hc) assembled entrywise for all
//     segments at once (D_R from the complex Kronecker-assembled dissipator,
//     once); P_R,j = exp(dt L_R,j) by Taylor-16 / Paterson-Stockmeyer on the
//     real batched tile GEMM (k_tiled.cu launch_dgemm), one common squaring
//     count from one norm pass (like the complex batched path);
//   chain: one cooperative launch walks every segment — each CTA holds its
//     rows of the current P_R,j in shared memory (reloaded per segment), a
//     grid barrier per step (K2c's scheme, k_single.cu, on real data).
// Real matrices use an even leading dimension (TMA rows are 16-byte aligned).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "internal.hpp"

namespace lbg {
namespace {

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }
inline int even_ld(int n) { return n + (n & 1); }

__device__ __forceinline__ double real_coord(double2 z, int i, int j) { return i <= j ? z.x : -z.y; }

// real-form entry (q, s) of a complex operator given entrywise (k_ptm.cu)
template <class F>
__device__ __forceinline__ double real_entry_rt(F&& lq, int d, int q, int s) {
  const int si = s / d, sj = s - si * d;
  double2 c;
  if (si == sj) {
    c = lq(s);
  } else {
    const double2 a = lq(s), bt = lq(sj * d + si);
    c = si < sj ? make_double2(a.x + bt.x, a.y + bt.y) : make_double2(a.y - bt.y, bt.x - a.x);
  }
  const int qi = q / d, qj = q - qi * d;
  return real_coord(c, qi, qj);
}

// D (n x n complex, dense) -> D_R (n x ld real)
__global__ void dissipator_real_kernel(const double2* __restrict__ dis, int d, int ld, double* __restrict__ dr) {
  const int n = d * d;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * n) return;
  const int q = int(e / n), s = int(e - (long long)q * n);
  dr[(long long)q * ld + s] = real_entry_rt([&](int p) { return dis[(long long)q * n + p]; }, d, q, s);
}

// A_R,j = dt (D_R + coherent_R(h0 + a_j hc)), coherent(H)[(i,k),(j,l)] = -i (H_ij d_kl - d_ij H_lk)
__global__ void assemble_real_kernel(const double* __restrict__ dr, const double2* __restrict__ h0,
                                     const double2* __restrict__ hc, const double* __restrict__ amps, int d,
                                     int ld, double dt, double* __restrict__ A) {
  const int n = d * d;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int seg = blockIdx.y;
  if (e >= (long long)n * n) return;
  const int q = int(e / n), s = int(e - (long long)q * n);
  const double a = amps[seg];
  auto coh = [&](int p) {
    const int i = q / d, k = q - i * d, j = p / d, l = p - j * d;
    double2 v = make_double2(0.0, 0.0);
    if (k == l) {
      const double2 h = make_double2(h0[i * d + j].x + a * hc[i * d + j].x, h0[i * d + j].y + a * hc[i * d + j].y);
      v.x += h.y;
      v.y -= h.x;
    }
    if (i == j) {
      const double2 h = make_double2(h0[l * d + k].x + a * hc[l * d + k].x, h0[l * d + k].y + a * hc[l * d + k].y);
      v.x -= h.y;
      v.y += h.x;
    }
    return v;
  };
  const long long o = (long long)seg * n * ld + (long long)q * ld + s;
  A[o] = dt * (dr[(long long)q * ld + s] + real_entry_rt(coh, d, q, s));
}

// per-matrix 1-norm (max column sum), max over the batch into *nmax (bits).
// Block (32 columns x 8 row groups), grid (column blocks, matrices): coalesced
// rows, 8-way parallel column sums (a thread per whole column took 0.89 ms for
// 20 matrices at n = 729 — a fifth of the build).
__global__ void colsum_real_kernel(const double* __restrict__ A, int n, int ld, unsigned long long* __restrict__ nmax) {
  __shared__ double part[8][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int c = blockIdx.x * 32 + tx;
  const double* m = A + (long long)blockIdx.y * n * ld;
  double sum = 0.0;
  if (c < n)
    for (int r = ty; r < n; r += 8) sum += fabs(m[(long long)r * ld + c]);
  part[ty][tx] = sum;
  __syncthreads();
  if (ty == 0) {
    double tot = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) tot += part[k][tx];
    for (int o = 16; o > 0; o >>= 1) tot = fmax(tot, __shfl_xor_sync(0xffffffffu, tot, o));
    if (tx == 0) atomicMax(nmax, (unsigned long long)__double_as_longlong(tot));
  }
}

// A *= 2^-sq with sq decided on the device (squarings_kernel)
__global__ void scale_real_kernel(double* __restrict__ A, int n, int ld, const int* __restrict__ sq) {
  const int q = *sq;
  if (q == 0) return;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * n) return;
  const int r = int(e / n), c = int(e - (long long)r * n);
  A[(long long)blockIdx.y * n * ld + (long long)r * ld + c] *= ldexp(1.0, -q);
}

// the common squaring count from the batch's max 1-norm (Taylor-16: theta = 0.79)
__global__ void squarings_kernel(const unsigned long long* __restrict__ nmax, int sq_max, int* __restrict__ sq) {
  const double nrm = __longlong_as_double((long long)*nmax);
  int q = nrm > 0.79 ? int(ceil(log2(nrm / 0.79))) : 0;
  *sq = q < sq_max ? q : sq_max;  // the host bound covers it; the clamp only guards rounding
}

// out = x + c0 I + c1 a1 + c2 a2 + c3 a3 + c4 a4   (any of x, a4 may be null)
__global__ void combo_real_kernel(double* __restrict__ out, const double* __restrict__ x, const double* __restrict__ a1,
                                  const double* __restrict__ a2, const double* __restrict__ a3,
                                  const double* __restrict__ a4, double c0, double c1, double c2, double c3,
                                  double c4, int n, int ld) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * n) return;
  const int r = int(e / n), c = int(e - (long long)r * n);
  const long long o = (long long)blockIdx.y * n * ld + (long long)r * ld + c;
  double v = x ? x[o] : 0.0;
  if (r == c) v += c0;
  v += c1 * a1[o] + c2 * a2[o] + c3 * a3[o];
  if (a4) v += c4 * a4[o];
  out[o] = v;
}

// rho (d x d complex) <-> real coordinates (n)
__global__ void rho_to_x_real_kernel(const double2* __restrict__ rho, int d, double* __restrict__ x) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x, n = d * d;
  if (p >= n) return;
  const int i = p / d, j = p - i * d;
  x[p] = real_coord(rho[p], i, j);
}
__global__ void x_to_rho_real_kernel(const double* __restrict__ x, int d, double2* __restrict__ rho) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x, n = d * d;
  if (p >= n) return;
  const int i = p / d, j = p - i * d;
  rho[p] = i == j ? make_double2(x[p], 0.0)
                  : (i < j ? make_double2(x[p], x[j * d + i]) : make_double2(x[j * d + i], -x[p]));
}

// ---- the chain: real rows of P_R,j spread over every SM, one grid barrier per step
constexpr int RT = 256;

__global__ void __launch_bounds__(RT) rowsplit_real_kernel(const double* __restrict__ props, int n, int ld,
                                                           double* x0, double* x1, int64_t segments, int64_t sps,
                                                           unsigned int* bar) {
  extern __shared__ __align__(16) double smr[];
  const int r0 = int((long long)n * blockIdx.x / gridDim.x);
  const int r1 = int((long long)n * (blockIdx.x + 1) / gridDim.x);
  const int rows = r1 - r0;
  double* ps = smr;                    // rows x n
  double* vs = ps + size_t(rows) * n;  // n
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* cur = x0;
  double* nxt = x1;
  unsigned int epoch = 0;
#pragma unroll 1
  for (int64_t seg = 0; seg < segments; ++seg) {
    const double* p = props + seg * (long long)n * ld;
    for (int e = tid; e < rows * n; e += RT) {
      const int r = e / n, c = e - r * n;
      ps[e] = p[(long long)(r0 + r) * ld + c];
    }
#pragma unroll 1
    for (int64_t s = 0; s < sps; ++s) {
      for (int e = tid; e < n; e += RT) vs[e] = __ldcg(cur + e);  // other CTAs wrote it
      __syncthreads();
      for (int r = warp; r < rows; r += RT / 32) {
        const double* prow = ps + size_t(r) * n;
        double a0 = 0.0, a1 = 0.0;
        int j = lane;
        for (; j + 32 < n; j += 64) {
          a0 = fma(prow[j], vs[j], a0);
          a1 = fma(prow[j + 32], vs[j + 32], a1);
        }
        if (j < n) a0 = fma(prow[j], vs[j], a0);
        double v = a0 + a1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) nxt[r0 + r] = v;
      }
      grid_barrier_sync(bar, ++epoch * gridDim.x);
      double* t = cur;
      cur = nxt;
      nxt = t;
    }
  }
}

}  // namespace

bool grape_real_supported(size_t d) { return d * d > 96; }

size_t grape_real_workspace(size_t d, int64_t segments) {
  const size_t n = d * d, ld = size_t(even_ld(int(n)));
  const size_t mat = align_up(size_t(segments) * n * ld * 8);
  // D (complex), D_R, A, A2, A3, A4, T, M, P_R, x0 / x1 / barrier / norm
  return align_up(n * n * 16) + align_up(n * ld * 8) + 8 * mat + align_up(2 * n * 8) + 512;
}

void launch_grape_real(size_t d, const double* h0, const double* hc, const double* zero_h, size_t n_ops,
                       const double* ops, const double* amps, int64_t segments, int64_t sps, double dt, double* x_rho,
                       int squaring_bound, void* work, cudaStream_t s, cudaEvent_t ev_build_end) {
  const int n = int(d * d), ld = even_ld(n), dd = int(d);
  const size_t mat = align_up(size_t(segments) * n * ld * 8);
  char* w = static_cast<char*>(work);
  double2* dis = reinterpret_cast<double2*>(w);
  double* dr = reinterpret_cast<double*>(w + align_up(size_t(n) * n * 16));
  char* mats = w + align_up(size_t(n) * n * 16) + align_up(size_t(n) * ld * 8);
  double* A = reinterpret_cast<double*>(mats);
  double* A2 = reinterpret_cast<double*>(mats + mat);
  double* A3 = reinterpret_cast<double*>(mats + 2 * mat);
  double* A4 = reinterpret_cast<double*>(mats + 3 * mat);
  double* T = reinterpret_cast<double*>(mats + 4 * mat);
  double* M = reinterpret_cast<double*>(mats + 5 * mat);
  double* P = reinterpret_cast<double*>(mats + 6 * mat);
  double* x0 = reinterpret_cast<double*>(mats + 8 * mat);
  double* x1 = x0 + n;
  unsigned int* bar = reinterpret_cast<unsigned int*>(x1 + n);
  unsigned long long* nmax = reinterpret_cast<unsigned long long*>(bar + 4);
  int* sqd = reinterpret_cast<int*>(nmax + 1);
  // matrices start zeroed (the leading-dimension padding is never written)
  check_cuda(cudaMemsetAsync(mats, 0, 7 * mat, s), "memset");
  launch_build_lindbladian(d, zero_h, n_ops, ops, reinterpret_cast<double*>(dis), s);
  const long long nn = (long long)n * n;
  dissipator_real_kernel<<<unsigned((nn + 255) / 256), 256, 0, s>>>(dis, dd, ld, dr);
  LBG_CHECK_LAUNCH("dissipator_real_kernel");
  const dim3 eg(unsigned((nn + 255) / 256), unsigned(segments));
  assemble_real_kernel<<<eg, 256, 0, s>>>(dr, reinterpret_cast<const double2*>(h0),
                                          reinterpret_cast<const double2*>(hc), amps, dd, ld, dt, A);
  LBG_CHECK_LAUNCH("assemble_real_kernel");
  // one norm pass fixes a common squaring count (Taylor-16: theta = 0.79) on the
  // device; the host launches sq_max conditional products from an a-priori
  // bound, each a plain copy when beyond the device count — no host round trip
  check_cuda(cudaMemsetAsync(nmax, 0, 8, s), "memset");
  colsum_real_kernel<<<dim3(unsigned((n + 31) / 32), unsigned(segments)), dim3(32, 8), 0, s>>>(A, n, ld, nmax);
  LBG_CHECK_LAUNCH("colsum_real_kernel");
  const int sq_max = squaring_bound;
  squarings_kernel<<<1, 1, 0, s>>>(nmax, sq_max, sqd);
  LBG_CHECK_LAUNCH("squarings_kernel");
  if (sq_max > 0) {
    scale_real_kernel<<<eg, 256, 0, s>>>(A, n, ld, sqd);
    LBG_CHECK_LAUNCH("scale_real_kernel");
  }
  double c[17];
  c[0] = 1.0;
  for (int k = 1; k <= 16; ++k) c[k] = c[k - 1] / k;
  const long long st = (long long)n * ld;
  const int bs = int(segments);
  auto mm = [&](const double* a, const double* b, double* out) { launch_dgemm(a, b, out, n, ld, bs, st, st, st, s); };
  mm(A, A, A2);
  mm(A2, A, A3);
  mm(A2, A2, A4);
  combo_real_kernel<<<eg, 256, 0, s>>>(T, nullptr, A, A2, A3, A4, c[12], c[13], c[14], c[15], c[16], n, ld);
  LBG_CHECK_LAUNCH("combo_real_kernel");
  for (int j = 2; j >= 0; --j) {  // T = A4 T + B_j
    mm(A4, T, M);
    double* dst = (j == 0 && sq_max == 0) ? P : T;
    combo_real_kernel<<<eg, 256, 0, s>>>(dst, M, A, A2, A3, nullptr, c[4 * j], c[4 * j + 1], c[4 * j + 2],
                                         c[4 * j + 3], 0.0, n, ld);
    LBG_CHECK_LAUNCH("combo_real_kernel");
  }
  double* cur = T;
  for (int i = 0; i < sq_max; ++i) {  // T -> M -> T ... ending in P; copies past the device count
    double* dst = (i == sq_max - 1) ? P : (cur == T ? M : T);
    launch_dgemm(cur, cur, dst, n, ld, bs, st, st, st, s, sqd, i);
    cur = dst;
  }
  if (ev_build_end) check_cuda(cudaEventRecord(ev_build_end, s), "event");
  // ---- the chain ----
  rho_to_x_real_kernel<<<(n + 255) / 256, 256, 0, s>>>(reinterpret_cast<const double2*>(x_rho), dd, x0);
  LBG_CHECK_LAUNCH("rho_to_x_real_kernel");
  check_cuda(cudaMemsetAsync(bar, 0, 4, s), "memset");
  // measured (50 x 32 steps at d = 27): 148 CTAs 1.90 ms, 96 1.96, 74 2.46, 37 3.20 — the
  // per-CTA row work, not the barrier's participant count, sets the step time
  const int grid = std::min(sm_count(), n);
  const int rows_max = (n + grid - 1) / grid;
  const size_t smem = (size_t(rows_max) * n + n) * 8;
  ensure_max_dyn_smem((const void*)rowsplit_real_kernel, int(smem));
  const double* pp = P;
  int ni = n, li = ld;
  int64_t sg = segments, sp = sps;
  void* args[] = {(void*)&pp, (void*)&ni, (void*)&li, (void*)&x0, (void*)&x1, (void*)&sg, (void*)&sp, (void*)&bar};
  if (segments > 0 && sps > 0) {
    check_cuda(cudaLaunchCooperativeKernel((const void*)rowsplit_real_kernel, dim3(grid), dim3(RT), args, smem, s),
               "rowsplit_real_kernel (cooperative)");
    note_launch();
  }
  const double* fin = ((segments * sps) & 1) ? x1 : x0;
  x_to_rho_real_kernel<<<(n + 255) / 256, 256, 0, s>>>(fin, dd, reinterpret_cast<double2*>(x_rho));
  LBG_CHECK_LAUNCH("x_to_rho_real_kernel");
}

}  // namespace lbg
