// k_ptm.cu — config 4 in the real (transfer-matrix) representation.
//
// A Lindbladian maps Hermitian matrices to Hermitian matrices, so on the real
// coordinates of a density matrix
//     x[i*d+j] = Re rho_ij (i <= j),   x[i*d+j] = Im rho_ji = -Im rho_ij (i > j)
// (the same index space as row-major vec(rho)) it acts as a REAL d^2 x d^2
// matrix L_R = T L T^-1, and P_R = exp(L_R dt) = T P T^-1 is the same
// propagator as the reference's complex P = exp(L dt) in another basis. With
// n = d^2:
//   L_R[q][s] = f_q( c_qs ),  c_qs = L[q][s]                    (s diagonal)
//                                  = L[q][s] + L[q][s^T]         (s upper)
//                                  = i (L[q][s^T] - L[q][s])     (s lower)
//   f_q = Re for q upper/diagonal, -Im for q lower;  s^T = transposed index.
// Every L entry comes from the Kronecker formula of lindblad.cpp:37-59 (K5),
// so the assembly is elementwise. A real n x n matmul is 4x fewer FMAs than
// the complex one, and a step is n^2 real FMAs instead of 4 n^2.
//
// K4 (ptm_expm_kernel): one CTA per trajectory; A_R = dt L_R formed in shared
//   memory from three precomputed affine terms (ptm_terms_kernel); Taylor in
//   Paterson-Stockmeyer form with s = 3 (A2, A3, then Horner products in A3,
//   no solve): degree 12 in 5 real DMMA matmuls for ||A||_1 <= 0.36
//   (truncation <= 2.5e-16; config 4 sits at 0.327-0.342), degree 14 in 6 for
//   ||A||_1 <= 0.53 (<= 2^-54), scaling and squaring above;
//   three 88x92 padded matrices in shared memory, A and A^2 also kept at each
//   thread's own accumulator positions so the Horner epilogues never re-read
//   them. Writes P_R (n x n) to global memory.
// K3 (ptm_step_kernel): three trajectories per CTA; P_R register resident
//   (a 4 x 21 block per thread), x in shared memory; per step 84 FMAs in 12
//   chains, a 4-lane shuffle reduce-scatter, one barrier. The SM register file
//   (P_R = 13k registers per trajectory) caps residency at 3 trajectories per
//   SM. Epilogue: populations + ensemble sum.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "internal.hpp"

namespace lbg {
namespace {

constexpr int D = 9, N = 81;          // config 4 size
constexpr int MT = 11, KT = 21;       // 8-row m/n tiles (88), 4-wide k steps (84)
constexpr int RS = 92;                // smem row stride: 92 = 12 (mod 16) -> conflict free
constexpr int MAT = 88 * RS;          // doubles per padded matrix
constexpr int WARPS = 11, THREADS = 32 * WARPS;
constexpr double kTheta14 = 0.53;
// degree 12 (5 products) below 0.36: truncation <= 0.36^13 / 13! (1 + 0.36/14) = 2.5e-16
constexpr double kTheta12 = 0.36;
static_assert(THREADS == 4 * 88, "combine pass: 4 threads per padded column");

// coherent Kronecker entries  C[q][p] = -i (H[i][j] d_kl - d_ij H[l][k]),  q = (i,k), p = (j,l)
__device__ __forceinline__ double2 kron_c(const double2* __restrict__ h, int q, int p) {
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

// Real-representation entry L_R[q][s] of a complex generator given entry-wise.
template <class F>
__device__ __forceinline__ double real_entry(F&& lq, int q, int s) {
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

// The generator is affine in the sweep parameters, L(b) = L(h0) + delta_b L(hd)
// + s_b L(hs) with the dissipator in L(h0), and so is its real form. The three
// terms dt C0 = dt (D_R + coherent_R(h0)), dt Cd = dt coherent_R(hd),
// dt Cs = dt coherent_R(hs) are built ONCE (D from the complex
// Kronecker-assembled dissipator, k_model.cu build_lindbladian_kernel with
// H = 0), in the padded 88 x RS shared-memory layout of the expm kernel (zero
// padding), so each trajectory stages them with three bulk copies and forms
// A = dt L_R(b) with two FMAs per entry.
__global__ void ptm_terms_kernel(const double2* __restrict__ dis, const double2* __restrict__ h0,
                                 const double2* __restrict__ hd, const double2* __restrict__ hs, double dt,
                                 double* __restrict__ terms) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= MAT) return;
  const int q = e / RS, s = e - q * RS;
  const bool in = q < N && s < N;
  terms[e] = in ? dt * (real_entry([&](int p) { return dis[q * N + p]; }, q, s) +
                        real_entry([&](int p) { return kron_c(h0, q, p); }, q, s))
                : 0.0;
  terms[MAT + e] = in ? dt * real_entry([&](int p) { return kron_c(hd, q, p); }, q, s) : 0.0;
  terms[2 * MAT + e] = in ? dt * real_entry([&](int p) { return kron_c(hs, q, p); }, q, s) : 0.0;
}

// acc[m][0..1] = (X * Y)[m*8 + g][w*8 + 2t .. +1], X, Y padded 88 x RS
__device__ __forceinline__ void mm(const double* __restrict__ X, const double* __restrict__ Y,
                                   double (&acc)[MT][2], int w, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0.0;
  const double* xa = X + g * RS + t;
  const double* yb = Y + t * RS + w * 8 + g;
  double a_cur[MT], b_cur = yb[0];
#pragma unroll
  for (int m = 0; m < MT; ++m) a_cur[m] = xa[m * 8 * RS];
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    double a_nxt[MT], b_nxt = 0.0;
    if (k + 1 < KT) {
      b_nxt = yb[(k + 1) * 4 * RS];
#pragma unroll
      for (int m = 0; m < MT; ++m) a_nxt[m] = xa[m * 8 * RS + (k + 1) * 4];
    }
#pragma unroll
    for (int m = 0; m < MT; ++m) dmma(acc[m], a_cur[m], b_cur);
    if (k + 1 < KT) {
      b_cur = b_nxt;
#pragma unroll
      for (int m = 0; m < MT; ++m) a_cur[m] = a_nxt[m];
    }
  }
}

__device__ __forceinline__ void store(double* __restrict__ Z, const double (&v)[MT][2], int w, int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int m = 0; m < MT; ++m)
    *reinterpret_cast<double2*>(Z + (m * 8 + g) * RS + w * 8 + 2 * t) = make_double2(v[m][0], v[m][1]);
}

// acc = acc + c0 I + c1 a1 + c2 a2 at own positions (in place); zero in the padding
__device__ __forceinline__ void horner_epilogue(double (&acc)[MT][2],
                                                const double (&a1)[MT][2], const double (&a2)[MT][2],
                                                double c0, double c1, double c2, int w, int lane,
                                                bool with_acc) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int r = m * 8 + g, col = w * 8 + 2 * t + c;
      double x = (with_acc ? acc[m][c] : 0.0) + c1 * a1[m][c] + c2 * a2[m][c];
      if (r == col) x += c0;
      acc[m][c] = (r < N && col < N) ? x : 0.0;
    }
}

__global__ void __launch_bounds__(THREADS, 1)
    ptm_expm_kernel(const double* __restrict__ terms, const double* __restrict__ delta,
                    const double* __restrict__ scale, double* __restrict__ p_out) {
  extern __shared__ __align__(16) double sm[];
  double* S0 = sm;
  double* S1 = sm + MAT;
  double* S2 = sm + 2 * MAT;
  __shared__ double colpart[4][88];
  __shared__ int s_sq, s_deg12;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int b = blockIdx.x;
  // dt C0 / dt Cd / dt Cs -> S0 / S1 / S2: three bulk async copies on one mbarrier
  const unsigned sb32 = static_cast<unsigned>(__cvta_generic_to_shared(&bar));
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sb32));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb32), "r"(unsigned(3 * MAT * 8))
                 : "memory");
#pragma unroll
    for (int i = 0; i < 3; ++i)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              static_cast<unsigned>(__cvta_generic_to_shared(sm + i * MAT))),
          "l"(terms + i * MAT), "r"(unsigned(MAT * 8)), "r"(sb32)
          : "memory");
  }
  const double db = delta[b], sb = scale[b];
  __syncthreads();  // barrier initialised
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra WAIT_%=;\n}\n" ::"r"(
          sb32)
      : "memory");
  // A = dt C0 + delta dt Cd + s dt Cs in place in S0, fused with the column
  // sums of ||A||_1: thread = (column c, quarter of the rows); 4 x 88 = THREADS
  {
    const int c = tid % 88, q0 = (tid / 88) * 22;
    double cs = 0.0;
    if (c < N) {
#pragma unroll 2
      for (int r = q0; r < q0 + 22 && r < N; ++r) {
        const int o = r * RS + c;
        const double v = fma(sb, S2[o], fma(db, S1[o], S0[o]));
        S0[o] = v;
        cs += fabs(v);
      }
    }
    colpart[tid / 88][c] = cs;
  }
  __syncthreads();
  if (w == 0) {  // ||A||_1 -> squarings (per trajectory)
    double nrm = 0.0;
    for (int c = lane; c < N; c += 32)
      nrm = fmax(nrm, (colpart[0][c] + colpart[1][c]) + (colpart[2][c] + colpart[3][c]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nrm = fmax(nrm, __shfl_xor_sync(0xffffffffu, nrm, o));
    if (lane == 0) {
      s_sq = nrm > kTheta14 ? int(ceil(log2(nrm / kTheta14))) : 0;
      s_deg12 = nrm <= kTheta12;
    }
  }
  __syncthreads();
  const int sq = s_sq;
  const bool deg12 = s_deg12;
  if (sq > 0) {
    const double sc = ldexp(1.0, -sq);
    for (int e = tid; e < N * N; e += THREADS) {
      const int q = e / N, s = e - q * N;
      S0[q * RS + s] *= sc;
    }
    __syncthreads();
  }

  const int g = lane >> 2, t = lane & 3;
  double a1[MT][2], a2[MT][2], acc[MT][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int c = 0; c < 2; ++c) a1[m][c] = S0[(m * 8 + g) * RS + w * 8 + 2 * t + c];
  // Taylor coefficients 1/k!, k = 0..14
  double cf[15];
  cf[0] = 1.0;
#pragma unroll
  for (int k = 1; k < 15; ++k) cf[k] = cf[k - 1] / k;

  mm(S0, S0, acc, w, lane);  // A2
#pragma unroll
  for (int m = 0; m < MT; ++m) a2[m][0] = acc[m][0], a2[m][1] = acc[m][1];
  store(S1, acc, w, lane);
  __syncthreads();
  mm(S1, S0, acc, w, lane);  // A3
  __syncthreads();            // everyone done reading S0/S1
  store(S2, acc, w, lane);
  int j0;
  if (deg12) {  // T = B3 + c12 A3 (B4 = c12 I: no product)
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m][0] *= cf[12], acc[m][1] *= cf[12];
    horner_epilogue(acc, a1, a2, cf[9], cf[10], cf[11], w, lane, true);
    j0 = 2;
  } else {  // T = B4
    horner_epilogue(acc, a1, a2, cf[12], cf[13], cf[14], w, lane, false);
    j0 = 3;
  }
  store(S0, acc, w, lane);
  __syncthreads();
  double* tcur = S0;
  double* tnxt = S1;
#pragma unroll 1
  for (int j = j0; j >= 0; --j) {  // T = B_j + A3 T
    mm(S2, tcur, acc, w, lane);
    double c0 = cf[0], c1 = cf[1], c2 = cf[2];  // cf[3j .. 3j+2] without a local-memory index
#pragma unroll
    for (int jj = 1; jj < 4; ++jj)
      if (j == jj) c0 = cf[3 * jj], c1 = cf[3 * jj + 1], c2 = cf[3 * jj + 2];
    horner_epilogue(acc, a1, a2, c0, c1, c2, w, lane, true);
    if (j > 0 || sq > 0) {
      store(tnxt, acc, w, lane);
      __syncthreads();
      double* tt = tcur;
      tcur = tnxt;
      tnxt = tt;
    }
  }
  for (int i = 0; i < sq; ++i) {  // squarings
    mm(tcur, tcur, acc, w, lane);
    if (i + 1 < sq) {
      store(tnxt, acc, w, lane);
      __syncthreads();
      double* tt = tcur;
      tcur = tnxt;
      tnxt = tt;
    }
  }
  // ---- P_R -> global (n x n, unpadded) ----
  double* out = p_out + size_t(b) * N * N;
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    const int r = m * 8 + g, c0 = w * 8 + 2 * t;
    if (r < N) {
      if (c0 < N) out[r * N + c0] = acc[m][0];
      if (c0 + 1 < N) out[r * N + c0 + 1] = acc[m][1];
    }
  }
}

// K4, balanced: the DMMA tiles cover rows / columns / k 0..79 only (10 x 10
// output tiles, 20 k-steps: 2,000 DMMAs per product instead of 11 x 11 x 21 =
// 2,541, whose last m-tile, n-tile and k-step carry one real row / column / k
// each), 20 warps = five per sub-partition own 5 tiles each (half an n-tile
// column), so every sub-partition issues exactly 500 DMMAs per product (the
// 11-warp kernel: 693 on three of them). The 81st row / column go to DFMA:
// the k = 80 term is a rank-1 update on each lane's own tile entries, and the
// 161 fringe entries (column 80, rows 0..79, and row 80) are dot products
// split over 4 lanes (k = kq mod 4) and shuffle-reduced. Four 81 x 84
// matrices (A, A^2, A^3, T: 213 KB) in shared memory; the Horner epilogues
// read A and A^2 there, T is updated in place between two barriers.
constexpr int RS2 = 84;                      // = 4 (mod 16): conflict-free DMMA fragments
constexpr int MAT2 = N * RS2;                // doubles per matrix (81 rows)
constexpr int E_WARPS = 20, E_THREADS = 32 * E_WARPS;
constexpr int EMT = 5, EKT = 20;             // m-tiles per warp, DMMA k-steps (k < 80)
constexpr int E_PARTS = 7, E_PROWS = 12;     // combine pass: 7 row parts x 81 columns
constexpr int FRINGE = 2 * 80 + 1;           // column 80 (rows < 80) + row 80
static_assert(E_PARTS * 81 <= E_THREADS && E_PARTS * E_PROWS >= N, "combine pass");
static_assert(4 * MAT2 * 8 + E_PARTS * RS2 * 8 + 64 <= 232448, "shared memory");

struct TaylorCoef {
  double v[15];
};
constexpr TaylorCoef make_taylor() {
  TaylorCoef c{};
  c.v[0] = 1.0;
  for (int k = 1; k < 15; ++k) c.v[k] = c.v[k - 1] / k;
  return c;
}
__constant__ TaylorCoef c_taylor = make_taylor();

__global__ void ptm_terms2_kernel(const double2* __restrict__ dis, const double2* __restrict__ h0,
                                  const double2* __restrict__ hd, const double2* __restrict__ hs, double dt,
                                  double* __restrict__ terms) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= MAT2) return;
  const int q = e / RS2, s = e - q * RS2;
  const bool in = s < N;
  terms[e] = in ? dt * (real_entry([&](int p) { return dis[q * N + p]; }, q, s) +
                        real_entry([&](int p) { return kron_c(h0, q, p); }, q, s))
                : 0.0;
  terms[MAT2 + e] = in ? dt * real_entry([&](int p) { return kron_c(hd, q, p); }, q, s) : 0.0;
  terms[2 * MAT2 + e] = in ? dt * real_entry([&](int p) { return kron_c(hs, q, p); }, q, s) : 0.0;
}

struct Fringe {  // this lane's fringe dot products (the second only in warp 0)
  int r[2], c[2];
  bool own[2];   // lane kq == 0 of a valid dot: holds and stores the entry
};
__device__ __forceinline__ void fringe_rc(int d, int& r, int& c) {
  if (d < 80) r = d, c = 80;
  else r = 80, c = d - 80;
}

// (X Y) at this lane's tile entries (acc) and fringe entries (f)
__device__ __forceinline__ void mm2(const double* __restrict__ X, const double* __restrict__ Y,
                                    double (&acc)[EMT][2], double (&f)[2], const Fringe& fr, int w, int lane) {
  const int g = lane >> 2, t = lane & 3, nt = w >> 1, mh = w & 1;
#pragma unroll
  for (int m = 0; m < EMT; ++m) acc[m][0] = acc[m][1] = 0.0;
  const double* xa = X + (mh * EMT * 8 + g) * RS2 + t;
  const double* yb = Y + t * RS2 + nt * 8 + g;
#pragma unroll 4
  for (int k = 0; k < EKT; ++k) {
    const double b = yb[k * 4 * RS2];
    double a[EMT];
#pragma unroll
    for (int m = 0; m < EMT; ++m) a[m] = xa[m * 8 * RS2 + k * 4];
#pragma unroll
    for (int m = 0; m < EMT; ++m) dmma(acc[m], a[m], b);
  }
  {  // k = 80: rank-1 update of the own entries
    const double2 y = *reinterpret_cast<const double2*>(Y + 80 * RS2 + nt * 8 + 2 * t);
#pragma unroll
    for (int m = 0; m < EMT; ++m) {
      const double x = X[((mh * EMT + m) * 8 + g) * RS2 + 80];
      acc[m][0] = fma(x, y.x, acc[m][0]);
      acc[m][1] = fma(x, y.y, acc[m][1]);
    }
  }
  const int kq = lane & 3;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    if (i == 1 && w != 0) break;  // warp-uniform: only warp 0 has a second fringe dot
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    const double* xr = X + fr.r[i] * RS2;
    const double* yc = Y + fr.c[i];
#pragma unroll
    for (int j = 0; j < 21; ++j) {  // k = kq + 4 j <= 80: 21 terms for kq = 0, 20 otherwise
      const int k = kq + 4 * j;
      if (j == 20 && kq != 0) break;
      const double v = xr[k], y = yc[k * RS2];
      if (j % 3 == 0)
        s0 = fma(v, y, s0);
      else if (j % 3 == 1)
        s1 = fma(v, y, s1);
      else
        s2 = fma(v, y, s2);
    }
    double sum = (s0 + s1) + s2;
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    f[i] = sum;
  }
}

// acc = (with_acc ? acc : 0) + c0 I + c1 A + c2 A^2 at the own entries (A, A^2 from shared memory)
__device__ __forceinline__ void epi2(double (&acc)[EMT][2], double (&f)[2], const Fringe& fr,
                                     const double* __restrict__ SA, const double* __restrict__ SA2, double c0,
                                     double c1, double c2, bool with_acc, int w, int lane) {
  const int g = lane >> 2, t = lane & 3, nt = w >> 1, mh = w & 1;
#pragma unroll
  for (int m = 0; m < EMT; ++m) {
    const int r = (mh * EMT + m) * 8 + g, col = nt * 8 + 2 * t;
    const double2 a1 = *reinterpret_cast<const double2*>(SA + r * RS2 + col);
    const double2 a2 = *reinterpret_cast<const double2*>(SA2 + r * RS2 + col);
    double x0 = (with_acc ? acc[m][0] : 0.0) + c1 * a1.x + c2 * a2.x;
    double x1 = (with_acc ? acc[m][1] : 0.0) + c1 * a1.y + c2 * a2.y;
    if (r == col) x0 += c0;
    if (r == col + 1) x1 += c0;
    acc[m][0] = x0;
    acc[m][1] = x1;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    if (i == 1 && w != 0) break;
    const int o = fr.r[i] * RS2 + fr.c[i];
    double x = (with_acc ? f[i] : 0.0) + c1 * SA[o] + c2 * SA2[o];
    if (fr.r[i] == fr.c[i]) x += c0;
    f[i] = x;
  }
}

__device__ __forceinline__ void store2(double* __restrict__ Z, const double (&acc)[EMT][2], const double (&f)[2],
                                       const Fringe& fr, int w, int lane) {
  const int g = lane >> 2, t = lane & 3, nt = w >> 1, mh = w & 1;
#pragma unroll
  for (int m = 0; m < EMT; ++m)
    *reinterpret_cast<double2*>(Z + ((mh * EMT + m) * 8 + g) * RS2 + nt * 8 + 2 * t) =
        make_double2(acc[m][0], acc[m][1]);
#pragma unroll
  for (int i = 0; i < 2; ++i)
    if (fr.own[i]) Z[fr.r[i] * RS2 + fr.c[i]] = f[i];
}

__global__ void __launch_bounds__(E_THREADS, 1)
    ptm_expm2_kernel(const double* __restrict__ terms, const double* __restrict__ delta,
                     const double* __restrict__ scale, double* __restrict__ p_out) {
  extern __shared__ __align__(16) double sm[];
  double* SA = sm;
  double* SA2 = sm + MAT2;
  double* SA3 = sm + 2 * MAT2;
  double* ST = sm + 3 * MAT2;
  __shared__ double colpart[E_PARTS][RS2];
  __shared__ int s_sq, s_deg12;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int b = blockIdx.x;
  // dt C0 / dt Cd / dt Cs -> SA / SA2 / SA3: three bulk async copies on one mbarrier
  const unsigned sb32 = static_cast<unsigned>(__cvta_generic_to_shared(&bar));
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sb32));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sb32), "r"(unsigned(3 * MAT2 * 8))
                 : "memory");
#pragma unroll
    for (int i = 0; i < 3; ++i)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
              static_cast<unsigned>(__cvta_generic_to_shared(sm + i * MAT2))),
          "l"(terms + i * MAT2), "r"(unsigned(MAT2 * 8)), "r"(sb32)
          : "memory");
  }
  const double db = delta[b], sb = scale[b];
  // this lane's fringe dots: virtual lane v = tid (+ E_THREADS in warp 0), dot v / 4, k phase v % 4
  Fringe fr;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int v = tid + i * E_THREADS, d = v >> 2;
    const bool valid = d < FRINGE;
    fringe_rc(valid ? d : 0, fr.r[i], fr.c[i]);
    fr.own[i] = valid && (v & 3) == 0 && (i == 0 || w == 0);
  }
  __syncthreads();  // barrier initialised
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra WAIT_%=;\n}\n" ::"r"(
          sb32)
      : "memory");
  // A = dt C0 + delta dt Cd + s dt Cs in place in SA, fused with the column sums of ||A||_1
  if (tid < E_PARTS * 81) {
    const int c = tid % 81, q0 = (tid / 81) * E_PROWS;
    double cs = 0.0;
#pragma unroll 2
    for (int r = q0; r < q0 + E_PROWS && r < N; ++r) {
      const int o = r * RS2 + c;
      const double v = fma(sb, SA3[o], fma(db, SA2[o], SA[o]));
      SA[o] = v;
      cs += fabs(v);
    }
    colpart[tid / 81][c] = cs;
  }
  __syncthreads();
  if (w == 0) {  // ||A||_1 -> squarings (per trajectory)
    double nrm = 0.0;
    for (int c = lane; c < N; c += 32) {
      double cs = 0.0;
#pragma unroll
      for (int p = 0; p < E_PARTS; ++p) cs += colpart[p][c];
      nrm = fmax(nrm, cs);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nrm = fmax(nrm, __shfl_xor_sync(0xffffffffu, nrm, o));
    if (lane == 0) {
      s_sq = nrm > kTheta14 ? int(ceil(log2(nrm / kTheta14))) : 0;
      s_deg12 = nrm <= kTheta12;
    }
  }
  __syncthreads();
  const int sq = s_sq;
  const bool deg12 = s_deg12;
  if (sq > 0) {
    const double sc = ldexp(1.0, -sq);
    for (int e = tid; e < N * N; e += E_THREADS) {
      const int q = e / N, s = e - q * N;
      SA[q * RS2 + s] *= sc;
    }
    __syncthreads();
  }
  const double* cf = c_taylor.v;
  double acc[EMT][2], f[2] = {0.0, 0.0};
  mm2(SA, SA, acc, f, fr, w, lane);  // A^2
  store2(SA2, acc, f, fr, w, lane);
  __syncthreads();
  mm2(SA2, SA, acc, f, fr, w, lane);  // A^3
  store2(SA3, acc, f, fr, w, lane);
  int j0;
  if (deg12) {  // T = B3 + c12 A3 (B4 = c12 I: no product)
#pragma unroll
    for (int m = 0; m < EMT; ++m) acc[m][0] *= cf[12], acc[m][1] *= cf[12];
    f[0] *= cf[12];
    f[1] *= cf[12];
    epi2(acc, f, fr, SA, SA2, cf[9], cf[10], cf[11], true, w, lane);
    j0 = 2;
  } else {  // T = B4
    epi2(acc, f, fr, SA, SA2, cf[12], cf[13], cf[14], false, w, lane);
    j0 = 3;
  }
  store2(ST, acc, f, fr, w, lane);
  __syncthreads();
#pragma unroll 1
  for (int j = j0; j >= 0; --j) {  // T = B_j + A3 T
    mm2(SA3, ST, acc, f, fr, w, lane);
    epi2(acc, f, fr, SA, SA2, cf[3 * j], cf[3 * j + 1], cf[3 * j + 2], true, w, lane);
    if (j > 0 || sq > 0) {
      __syncthreads();  // every warp is done reading T
      store2(ST, acc, f, fr, w, lane);
      __syncthreads();
    }
  }
  for (int i = 0; i < sq; ++i) {  // squarings
    mm2(ST, ST, acc, f, fr, w, lane);
    if (i + 1 < sq) {
      __syncthreads();
      store2(ST, acc, f, fr, w, lane);
      __syncthreads();
    }
  }
  // ---- P_R -> global (n x n, unpadded) ----
  double* out = p_out + size_t(b) * N * N;
  const int g = lane >> 2, t = lane & 3, nt = w >> 1, mh = w & 1;
#pragma unroll
  for (int m = 0; m < EMT; ++m) {  // rows of 81 doubles: odd rows are not 16-byte aligned
    double* o = out + ((mh * EMT + m) * 8 + g) * N + nt * 8 + 2 * t;
    o[0] = acc[m][0];
    o[1] = acc[m][1];
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
    if (fr.own[i]) out[fr.r[i] * N + fr.c[i]] = f[i];
}

// K3: x <- P_R x for `steps` steps, P_R register resident.
// P_R is padded to 84 x 84 and cut into 4-row x 21-column blocks: one block
// (84 doubles) per thread, the 4 column blocks of a row group in 4 adjacent
// lanes. A step is 84 FMAs on 11 loads of the thread's 21 x values (earlier
// design — one 81-double row per thread — issued 41 broadcast loads per step
// and was shared-memory-wavefront bound: ncu 0.82 wavefronts/cycle, FP64 pipe
// 40%, profiles/r01_ncu_ptm_step_rowthread.json), then a 2-round butterfly
// reduce-scatter over the 4 lanes leaves each lane one finished row, one store
// and one barrier.
// DFMA latency is 23 cycles on B200 (profiles/r01_latency_probe.json): the 4
// row sums run as 12 independent chains of depth 7.
// Three trajectories per CTA: 63 groups of 4 lanes = 252 of 256 threads, two
// 224-register warps per sub-partition — all its 16K registers can carry.
// x lives in shared memory padded per column block (stride 22: 16-byte aligned
// pairs, the 4 blocks on disjoint banks).
constexpr int STEP_TRAJ = 3;
constexpr int STEP_THREADS = 256;
constexpr int SR = 4, SC = 21, SGROUPS = 21, XB = 22, XS = 4 * XB;
__device__ __forceinline__ int xpos(int c) { return (c / SC) * XB + c % SC; }
// One step of the 4 x 21 register-block matvec: the thread's 4 partial row
// sums over its column block x[0..20] (NA accumulators per row), then a
// butterfly reduce-scatter over the 4 column-block lanes (lane cb keeps the
// total of row cb of its group).
template <int NA>
__device__ __forceinline__ double block_row_step(const double (&p)[SR][SC], const double* __restrict__ x, bool hi2,
                                                 bool hi1) {
  double acc[SR][NA];
#pragma unroll
  for (int i = 0; i < SR; ++i)
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[i][a] = 0.0;
#pragma unroll
  for (int k = 0; k + 1 < SC; k += 2) {
    if (k % 10 == 0) asm volatile("" ::: "memory");  // bound how far loads are hoisted
    const double2 v = *reinterpret_cast<const double2*>(x + k);
#pragma unroll
    for (int i = 0; i < SR; ++i) {
      acc[i][k % NA] = fma(p[i][k], v.x, acc[i][k % NA]);
      acc[i][(k + 1) % NA] = fma(p[i][k + 1], v.y, acc[i][(k + 1) % NA]);
    }
  }
  {
    const double v = x[SC - 1];
#pragma unroll
    for (int i = 0; i < SR; ++i) acc[i][(SC - 1) % NA] = fma(p[i][SC - 1], v, acc[i][(SC - 1) % NA]);
  }
  double r4[SR];
#pragma unroll
  for (int i = 0; i < SR; ++i) {
#pragma unroll
    for (int w = 1; w < NA; w *= 2)
#pragma unroll
      for (int a = 0; a + w < NA; a += 2 * w) acc[i][a] += acc[i][a + w];
    r4[i] = acc[i][0];
  }
  double k0 = hi2 ? r4[2] : r4[0], k1 = hi2 ? r4[3] : r4[1];
  const double s0 = hi2 ? r4[0] : r4[2], s1 = hi2 ? r4[1] : r4[3];
  k0 += __shfl_xor_sync(0xffffffffu, s0, 2);
  k1 += __shfl_xor_sync(0xffffffffu, s1, 2);
  double kk = hi1 ? k1 : k0;
  kk += __shfl_xor_sync(0xffffffffu, hi1 ? k0 : k1, 1);
  return kk;
}

// GRAPE chain for d = 9 (propagate.cpp:144-156) in the real form: ONE CTA walks
// every segment, P_R,j register-resident in the same 4 x 21 blocks (21 groups
// of 4 lanes, 3 warps), reloaded from global memory (L2) at each segment
// switch. Latency-bound: 4 accumulators per row halve the FMA dependency depth
// of K3. (Measured: staging the next segment's blocks in shared memory by
// cp.async during the current segment made the chain slower, 0.47 vs 0.42 ms
// for 50 x 32 steps: the switch is not the cost, the step latency is.)
constexpr int CH_THREADS = 96;
__global__ void __launch_bounds__(CH_THREADS) ptm_chain_kernel(const double* __restrict__ props, int64_t segments,
                                                               int64_t sps, double2* __restrict__ rho) {
  __shared__ __align__(16) double xs[2][XS];
  const int tid = threadIdx.x, grp = tid >> 2, cb = tid & 3;
  const bool active = grp < SGROUPS;
  const int rg = active ? grp : SGROUPS - 1;
  for (int q = tid; q < XS; q += CH_THREADS) {
    const int c = (q / XB) * SC + q % XB;
    double v = 0.0;
    if (q % XB < SC && c < N) {
      const int i = c / D, j = c - i * D;
      v = i <= j ? rho[c].x : -rho[c].y;
    }
    xs[0][q] = v;
    xs[1][q] = 0.0;
  }
  const int row = rg * SR + cb;
  const bool writer = active && row < N;
  const int slot = xpos(row);
  const bool hi2 = cb & 2, hi1 = cb & 1;
  int cur = 0;
  double p[SR][SC];
#pragma unroll 1
  for (int64_t sg = 0; sg < segments; ++sg) {
    const double* pb = props + size_t(sg) * N * N;
#pragma unroll
    for (int i = 0; i < SR; ++i)
#pragma unroll
      for (int k = 0; k < SC; ++k) {
        const int r = rg * SR + i, c = cb * SC + k;
        p[i][k] = (r < N && c < N) ? pb[r * N + c] : 0.0;
      }
    __syncthreads();
#pragma unroll 1
    for (int64_t s = 0; s < sps; ++s) {
      const double kk = block_row_step<4>(p, xs[cur] + cb * XB, hi2, hi1);
      if (writer) xs[cur ^ 1][slot] = kk;
      __syncthreads();
      cur ^= 1;
    }
  }
  __syncthreads();
  if (tid < N) {
    const int i = tid / D, j = tid - i * D;
    const double a = xs[cur][xpos(tid)], bt = xs[cur][xpos(j * D + i)];
    rho[tid] = i == j ? make_double2(a, 0.0) : (i < j ? make_double2(a, bt) : make_double2(bt, -a));
  }
}

__global__ void __maxnreg__(224)
    ptm_step_kernel(const double* __restrict__ p_r, const double* __restrict__ x0, int64_t count, int64_t steps,
                    double* __restrict__ pops, double* __restrict__ ens_x) {
  __shared__ __align__(16) double xs[2][STEP_TRAJ][XS];
  const int tid = threadIdx.x;
  const int grp = tid >> 2, cb = tid & 3;
  const bool active = grp < STEP_TRAJ * SGROUPS;  // the 4 spare lanes shadow the last group
  const int tt = active ? grp / SGROUPS : STEP_TRAJ - 1;
  const int rg = active ? grp - tt * SGROUPS : SGROUPS - 1;
  const int64_t b = int64_t(blockIdx.x) * STEP_TRAJ + tt;
  const bool live = b < count;
  const double* pb = p_r + size_t(live ? b : 0) * N * N;
  double p[SR][SC];
#pragma unroll
  for (int i = 0; i < SR; ++i)
#pragma unroll
    for (int k = 0; k < SC; ++k) {
      const int r = rg * SR + i, c = cb * SC + k;
      p[i][k] = (r < N && c < N) ? pb[r * N + c] : 0.0;
    }
  for (int e = tid; e < STEP_TRAJ * XS; e += STEP_THREADS) {
    const int t = e / XS, q = e - t * XS, c = (q / XB) * SC + q % XB;
    xs[0][t][q] = (q % XB < SC && c < N) ? x0[c] : 0.0;
    xs[1][t][q] = 0.0;
  }
  __syncthreads();
  const int row = rg * SR + cb;  // the row this lane finishes
  const bool writer = active && row < N;
  const int slot = xpos(row);
  const bool hi2 = cb & 2, hi1 = cb & 1;
  int cur = 0;
#pragma unroll 1
  for (int64_t s = 0; s < steps; ++s) {
    const double kk = block_row_step<2>(p, xs[cur][tt] + cb * XB, hi2, hi1);
    if (writer) xs[cur ^ 1][tt][slot] = kk;
    __syncthreads();
    cur ^= 1;
  }
  if (writer && live) {
    const double v = xs[cur][tt][slot];
    if (row % (D + 1) == 0) pops[size_t(b) * D + row / (D + 1)] = v;
    atomicAdd(&ens_x[row], v);
  }
}

// complex rho (d x d) <-> real coordinates
__global__ void rho_to_x_kernel(const double2* __restrict__ rho, double* __restrict__ x) {
  const int p = threadIdx.x;
  if (p >= N) return;
  const int i = p / D, j = p - i * D;
  x[p] = i <= j ? rho[p].x : -rho[p].y;
}
__global__ void x_to_rho_kernel(const double* __restrict__ x, double2* __restrict__ rho) {
  const int p = threadIdx.x;
  if (p >= N) return;
  const int i = p / D, j = p - i * D;
  if (i == j)
    rho[p] = make_double2(x[p], 0.0);
  else if (i < j)
    rho[p] = make_double2(x[p], x[j * D + i]);
  else
    rho[p] = make_double2(x[j * D + i], -x[p]);
}

bool expm_v2() {  // A/B switch: LBG_PTM_EXPM=1 selects the 11-warp kernel
  static const bool v2 = [] {
    const char* e = std::getenv("LBG_PTM_EXPM");
    return !(e && std::atoi(e) == 1);
  }();
  return v2;
}
void launch_terms(const double2* dis, const double* h0, const double* hd, const double* hs, double dt,
                  double* terms, cudaStream_t s) {
  const auto* H0 = reinterpret_cast<const double2*>(h0);
  const auto* HD = reinterpret_cast<const double2*>(hd);
  const auto* HS = reinterpret_cast<const double2*>(hs);
  if (expm_v2()) {
    ptm_terms2_kernel<<<(MAT2 + 255) / 256, 256, 0, s>>>(dis, H0, HD, HS, dt, terms);
    LBG_CHECK_LAUNCH("ptm_terms2_kernel");
  } else {
    ptm_terms_kernel<<<(MAT + 255) / 256, 256, 0, s>>>(dis, H0, HD, HS, dt, terms);
    LBG_CHECK_LAUNCH("ptm_terms_kernel");
  }
}
void launch_expm(const double* terms, const double* delta, const double* scale, double* pr, int count,
                 cudaStream_t s) {
  if (expm_v2()) {
    const size_t smem = size_t(4) * MAT2 * 8;
    ensure_max_dyn_smem((const void*)ptm_expm2_kernel, int(smem));
    ptm_expm2_kernel<<<count, E_THREADS, smem, s>>>(terms, delta, scale, pr);
    LBG_CHECK_LAUNCH("ptm_expm2_kernel");
  } else {
    const size_t smem = size_t(3) * MAT * 8;
    ensure_max_dyn_smem((const void*)ptm_expm_kernel, int(smem));
    ptm_expm_kernel<<<count, THREADS, smem, s>>>(terms, delta, scale, pr);
    LBG_CHECK_LAUNCH("ptm_expm_kernel");
  }
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }
constexpr int64_t kChunk = 16384;

}  // namespace

size_t ptm_sweep_workspace(int64_t batch) {
  const size_t chunk = size_t(std::min<int64_t>(std::max<int64_t>(batch, 1), kChunk));
  return align_up(chunk * N * N * 8) + align_up(size_t(N) * N * 16) + align_up(2 * N * 8) +
         align_up(size_t(3) * MAT * 8) + 256;
}

bool ptm_sweep_supported(size_t d) { return d == size_t(D); }

void launch_ptm_sweep(size_t d, const double* h0, const double* hd, const double* hs, size_t n_ops,
                      const double* ops, const double* delta, const double* scale, double dt,
                      const double* rho0, int64_t batch, int64_t steps, double* pops, double* ens_sum,
                      void* work, cudaStream_t s) {
  if (d != size_t(D)) throw invalid_argument("ptm sweep: d must be 9");
  const size_t chunk = size_t(std::min<int64_t>(std::max<int64_t>(batch, 1), kChunk));
  char* w = static_cast<char*>(work);
  double* pr = reinterpret_cast<double*>(w);
  double2* dis = reinterpret_cast<double2*>(w + align_up(chunk * N * N * 8));
  double* xv = reinterpret_cast<double*>(w + align_up(chunk * N * N * 8) + align_up(size_t(N) * N * 16));
  double* x0 = xv;
  double* ens_x = xv + N;
  double* terms = reinterpret_cast<double*>(w + align_up(chunk * N * N * 8) + align_up(size_t(N) * N * 16) +
                                         align_up(2 * N * 8));
  // dissipator D = build_lindbladian(H = 0, ops) (K5, shared by all trajectories)
  check_cuda(cudaMemsetAsync(ens_x, 0, N * 8, s), "memset");
  check_cuda(cudaMemsetAsync(pr, 0, d * d * 16, s), "memset");
  launch_build_lindbladian(d, pr, n_ops, ops, reinterpret_cast<double*>(dis), s);
  launch_terms(dis, h0, hd, hs, dt, terms, s);
  rho_to_x_kernel<<<1, 96, 0, s>>>(reinterpret_cast<const double2*>(rho0), x0);
  LBG_CHECK_LAUNCH("rho_to_x_kernel");
  for (int64_t c0 = 0; c0 < batch; c0 += int64_t(chunk)) {
    const int cb = int(std::min<int64_t>(int64_t(chunk), batch - c0));
    launch_expm(terms, delta + c0, scale + c0, pr, cb, s);
    ptm_step_kernel<<<unsigned((cb + STEP_TRAJ - 1) / STEP_TRAJ), STEP_THREADS, 0, s>>>(
        pr, x0, cb, steps, pops + c0 * int64_t(D), ens_x);
    LBG_CHECK_LAUNCH("ptm_step_kernel");
  }
  x_to_rho_kernel<<<1, 96, 0, s>>>(ens_x, reinterpret_cast<double2*>(ens_sum));
  LBG_CHECK_LAUNCH("x_to_rho_kernel");
}

bool ptm_grape_supported(size_t d) { return d == size_t(D); }

size_t ptm_grape_workspace(int64_t segments) {
  return align_up(size_t(segments) * N * N * 8) + align_up(size_t(N) * N * 16) + align_up(size_t(3) * MAT * 8) +
         align_up(size_t(segments) * 8) + 256;
}

// GRAPE for d = 9 with an exactly Hermitian rho0: segment generators H_j = h0 +
// a_j hc are the affine family of config 4 with (delta, s) = (a_j, 0), so the
// build is ptm_terms_kernel + ONE ptm_expm_kernel launch over all segments;
// then ONE ptm_chain_kernel launch walks the chain. rho (d x d complex, device)
// is updated in place.
void launch_ptm_grape(const double* h0, const double* hc, const double* zero_h, size_t n_ops, const double* ops,
                      const double* amps, int64_t segments, int64_t sps, double dt, double* rho, void* work,
                      cudaStream_t s, cudaEvent_t ev_build_end) {
  char* w = static_cast<char*>(work);
  double* pr = reinterpret_cast<double*>(w);
  double2* dis = reinterpret_cast<double2*>(w + align_up(size_t(segments) * N * N * 8));
  double* terms = reinterpret_cast<double*>(reinterpret_cast<char*>(dis) + align_up(size_t(N) * N * 16));
  double* zeros = reinterpret_cast<double*>(reinterpret_cast<char*>(terms) + align_up(size_t(3) * MAT * 8));
  check_cuda(cudaMemsetAsync(zeros, 0, size_t(segments) * 8, s), "memset");
  launch_build_lindbladian(size_t(D), zero_h, n_ops, ops, reinterpret_cast<double*>(dis), s);
  launch_terms(dis, h0, hc, zero_h, dt, terms, s);
  launch_expm(terms, amps, zeros, pr, int(segments), s);
  if (ev_build_end) check_cuda(cudaEventRecord(ev_build_end, s), "event");
  ptm_chain_kernel<<<1, CH_THREADS, 0, s>>>(pr, segments, sps, reinterpret_cast<double2*>(rho));
  LBG_CHECK_LAUNCH("ptm_chain_kernel");
}

}  // namespace lbg
