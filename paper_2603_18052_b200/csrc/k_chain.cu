// k_chain.cu — K2: latency kernel for few trajectories (config 0: d = 3, one
// trajectory, 10^4 dependent steps).
//
// Regime: a single dependent chain of tiny matvecs has no throughput
// roofline; the bound is the per-step latency (shared-memory round trip + the
// FMA dependency depth). One warp owns one trajectory: lane r (r < 2n) owns
// real-form output row r and keeps that row of the real-form P in registers
// (2n doubles); each step every lane reads the current real vector from
// shared memory as broadcast 128-bit loads, forms its dot product in four
// interleaved FMA chains, writes its output element and __syncwarp()s.
// Several warps per CTA run independent trajectories.
//
// Replaces evolve's step loop (proj/src/propagate.cpp:88-92) around
// step_soa_kernel (proj/src/kernels_variants.cpp:26-41).
#include "common.cuh"
#include "internal.hpp"

namespace lbg {

namespace {

constexpr int kWarps = 4;

// `steps` steps of one warp's chain: lane `slot` writes its real-form output
// row; v0 / v1 ping-pong in shared memory. Returns the buffer holding the state.
template <int N>
__device__ __forceinline__ double* chain_steps(const double (&coef)[2 * N], double* v0, double* v1, int slot,
                                               int64_t steps) {
#pragma unroll 1
  for (int64_t s = 0; s < steps; ++s) {
    // issue every broadcast load of the state first: one shared-memory latency per step
    double2 vv[N];
#pragma unroll
    for (int j = 0; j < N; ++j) vv[j] = *reinterpret_cast<const double2*>(v0 + 2 * j);
    constexpr int NA = N >= 6 ? 6 : N;
    double acc[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      acc[j % NA] = fma(coef[2 * j], vv[j].x, acc[j % NA]);
      acc[j % NA] = fma(coef[2 * j + 1], vv[j].y, acc[j % NA]);
    }
#pragma unroll
    for (int w = 1; w < NA; w *= 2)
#pragma unroll
      for (int a = 0; a + w < NA; a += 2 * w) acc[a] += acc[a + w];
    v1[slot] = acc[0];
    __syncwarp();
    double* tmp = v0;
    v0 = v1;
    v1 = tmp;
  }
  return v0;
}

template <int N, Layout L>
__global__ void __launch_bounds__(32 * kWarps) chain_kernel(const double2* __restrict__ p,
                                                           double* __restrict__ x_re,
                                                           double* __restrict__ x_im,
                                                           double* __restrict__ x_aos,
                                                           int64_t batch, int64_t steps) {
  constexpr int R = 2 * N;  // real-form length
  __shared__ __align__(16) double vbuf[kWarps][2][R + 2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t t = blockIdx.x * (int64_t)kWarps + w;
  if (t >= batch) return;  // whole warp exits together
  const bool active = lane < R;
  const int i = lane >> 1, a = lane & 1;
  // real-form row r = 2i+a of P: coef[2j+b] = A'[2i+a][2j+b]
  double coef[R];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const double2 z = active ? p[i * N + j] : make_double2(0.0, 0.0);
    coef[2 * j] = a ? z.y : z.x;       // (a, b=0): re row -> Re, im row -> Im
    coef[2 * j + 1] = a ? z.x : -z.y;  // (a, b=1): re row -> -Im, im row -> Re
  }
  double* v0 = vbuf[w][0];
  double* v1 = vbuf[w][1];
  if (active) {
    if (L == Layout::soa)
      v0[lane] = a ? x_im[t * N + i] : x_re[t * N + i];
    else
      v0[lane] = x_aos[t * R + lane];
  }
  __syncwarp();
  // lanes >= R compute too (zero coefficients) and write a dummy slot, so the
  // step loop has no divergent branch
  const int slot = active ? lane : R;
  v0 = chain_steps<N>(coef, v0, v1, slot, steps);
  if (active) {
    if (L == Layout::soa) {
      if (a)
        x_im[t * N + i] = v0[lane];
      else
        x_re[t * N + i] = v0[lane];
    } else {
      x_aos[t * R + lane] = v0[lane];
    }
  }
}

template <int N>
void launch_n(const double* p, double* x_re, double* x_im, double* x_aos, int64_t batch,
              int64_t steps, Layout layout, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>((batch + kWarps - 1) / kWarps);
  const double2* p2 = reinterpret_cast<const double2*>(p);
  if (layout == Layout::soa)
    chain_kernel<N, Layout::soa><<<blocks, 32 * kWarps, 0, s>>>(p2, x_re, x_im, nullptr, batch, steps);
  else
    chain_kernel<N, Layout::aos><<<blocks, 32 * kWarps, 0, s>>>(p2, nullptr, nullptr, x_aos, batch, steps);
  LBG_CHECK_LAUNCH("chain_kernel");
}

// GRAPE chain (propagate.cpp:144-156) in ONE launch: segment j applies
// props[j] for sps steps. The next segment's real-form row is loaded into
// registers while the current segment runs, so a segment switch costs no
// global-memory latency and no kernel launch.
template <int N>
__global__ void __launch_bounds__(32 * kWarps) chain_segments_kernel(const double2* __restrict__ props,
                                                                     int64_t segments, int64_t sps,
                                                                     double* __restrict__ x_aos) {
  constexpr int R = 2 * N;
  // per-warp buffers as in chain_kernel (a lane-dependent address keeps the
  // state loads in the vector pipe, where ptxas issues them all up front)
  __shared__ __align__(16) double vbuf[kWarps][2][R + 2];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const bool active = lane < R;
  const int i = lane >> 1, a = lane & 1;
  double coef[R], next[R];
  auto load_row = [&](int64_t j, double (&c)[R]) {
    const double2* p = props + j * N * N;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const double2 z = active ? __ldg(p + i * N + k) : make_double2(0.0, 0.0);
      c[2 * k] = a ? z.y : z.x;
      c[2 * k + 1] = a ? z.x : -z.y;
    }
  };
  load_row(0, coef);
  double* v0 = vbuf[wi][0];
  if (active) v0[lane] = x_aos[lane];
  __syncwarp();
  const int slot = active ? lane : R;
#pragma unroll 1
  for (int64_t seg = 0; seg < segments; ++seg) {
    if (seg + 1 < segments) load_row(seg + 1, next);
    v0 = chain_steps<N>(coef, v0, v0 == vbuf[wi][0] ? vbuf[wi][1] : vbuf[wi][0], slot, sps);
#pragma unroll
    for (int k = 0; k < R; ++k) coef[k] = next[k];
  }
  if (active) x_aos[lane] = v0[lane];
}

}  // namespace

void launch_chain_segments(const double* props, std::size_t n, int64_t segments, int64_t sps, double* x_aos,
                           cudaStream_t s) {
  if (segments <= 0 || sps <= 0) return;
  const double2* p2 = reinterpret_cast<const double2*>(props);
  switch (n) {
#define LBG_CASE(N)                                                                    \
  case N:                                                                              \
    chain_segments_kernel<N><<<1, 32, 0, s>>>(p2, segments, sps, x_aos); \
    break;
    LBG_CASE(1) LBG_CASE(2) LBG_CASE(3) LBG_CASE(4) LBG_CASE(5) LBG_CASE(6) LBG_CASE(7)
    LBG_CASE(8) LBG_CASE(9) LBG_CASE(10) LBG_CASE(11) LBG_CASE(12) LBG_CASE(13) LBG_CASE(14)
    LBG_CASE(15) LBG_CASE(16)
#undef LBG_CASE
    default: throw invalid_argument("segmented chain kernel supports n <= 16");
  }
  LBG_CHECK_LAUNCH("chain_segments_kernel");
}

bool chain_supported(std::size_t n) { return n >= 1 && n <= 16; }

void launch_chain(const double* p_dev, std::size_t n, double* x_re, double* x_im, double* x_aos,
                  int64_t batch, int64_t steps, Layout layout, cudaStream_t s) {
  if (batch <= 0) return;
  switch (n) {
#define LBG_CASE(N) \
  case N: return launch_n<N>(p_dev, x_re, x_im, x_aos, batch, steps, layout, s);
    LBG_CASE(1) LBG_CASE(2) LBG_CASE(3) LBG_CASE(4) LBG_CASE(5) LBG_CASE(6) LBG_CASE(7)
    LBG_CASE(8) LBG_CASE(9) LBG_CASE(10) LBG_CASE(11) LBG_CASE(12) LBG_CASE(13) LBG_CASE(14)
    LBG_CASE(15) LBG_CASE(16)
#undef LBG_CASE
    default: throw invalid_argument("chain kernel supports n <= 16");
  }
}

}  // namespace lbg
