// k_single.cu — latency kernels for one (or a few) trajectories at larger n,
// the shape of GRAPE chains (propagate.cpp:111-168) and of lb::evolve on a
// single state (propagate.cpp:75-109). The batched kernels waste most of their
// tiles on one trajectory (K1b: 31/32 of each DMMA tile), so:
//
// K2b `cta_chain_kernel` (n <= 96): one CTA per trajectory; 4 threads per output
//   row, each holding its quarter row of P (<= 24 complex) in registers for all
//   steps, so a step reads only vec(rho) from shared memory (broadcast loads);
//   8 FMA chains (DFMA latency 23 cycles), 2-level shuffle reduction, one
//   barrier per step.
//
// K2c `rowsplit_kernel` (any n, batch <= 4): P's rows are spread over every SM's
//   shared memory (n = 729: 5 rows = 58 KB per CTA; 8.5 MB total on chip), so a
//   step reads only the state (n complex, L2) — per step each CTA pulls vec(rho)
//   into shared memory, each warp produces its rows by a lane-split dot product
//   and a warp shuffle reduction, then all CTAs meet at a grid barrier
//   (cooperative launch: all CTAs co-resident).
#include <algorithm>

#include "common.cuh"
#include "internal.hpp"

namespace lbg {
namespace {

constexpr int kMaxCtaN = 96;

// ---------------------------------------------------------------- K2b ------
// NT > 0: n known at compile time (n = 81: exact quarter rows, no predicates,
// constant addresses); NT == 0: runtime n. `segments` > 1 is the GRAPE chain
// in one launch: segment g applies props[g] for sps steps, and the next
// segment's P streams into shared memory (cp.async) while the current one runs.
template <int NT>
__global__ void __launch_bounds__(4 * kMaxCtaN) cta_chain_kernel(const double2* __restrict__ props, int n_rt,
                                                                double2* __restrict__ x, int64_t segments,
                                                                int64_t sps) {
  extern __shared__ __align__(16) double2 sm2[];
  const int n = NT > 0 ? NT : n_rt;
  const int S = n + ((4 - n % 8) + 8) % 8;  // row stride = 4 (mod 8) complex
  double2* ps = sm2;
  constexpr int VPAD = (kMaxCtaN + 3) / 4;  // quarter rows may read up to QMAX past n
  double2* va = ps + size_t(n) * S;
  double2* vb = va + n + VPAD;
  const int tid = threadIdx.x;
  const int i = tid >> 2, q = tid & 3;
  const int Q = NT > 0 ? (NT + 3) / 4 : (n + 3) / 4;
  double2* xb = x + size_t(blockIdx.x) * n;
  auto stage = [&](const double2* p) {  // P (n x n) -> padded shared memory, asynchronously
    for (int e = tid; e < n * S; e += blockDim.x) {
      const int r = e / S, c = e - r * S;
      cp_async16(ps + e, p + size_t(r) * n + (c < n ? c : 0), c < n);
    }
    cp_async_commit();
  };
  stage(props);
  for (int e = tid; e < 2 * (n + VPAD); e += blockDim.x) va[e] = e < n ? xb[e] : make_double2(0.0, 0.0);
  const bool active = i < n;
  const int j0 = q * Q;
  constexpr int QMAX = NT > 0 ? (NT + 3) / 4 : (kMaxCtaN + 3) / 4;
  constexpr int NC = NT > 0 ? 8 : 4;  // independent FMA chains per re / im (DFMA latency 23 cycles)
  double2 pr[QMAX];  // this thread's quarter row of P, register resident for a whole segment
#pragma unroll 1
  for (int64_t seg = 0; seg < segments; ++seg) {
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll
    for (int jj = 0; jj < QMAX; ++jj) {
      const int j = j0 + jj;
      pr[jj] = (active && jj < Q && j < n) ? ps[size_t(i) * S + j] : make_double2(0.0, 0.0);
    }
    __syncthreads();  // everyone holds its row before the buffer is refilled
    if (seg + 1 < segments) stage(props + (seg + 1) * size_t(n) * n);
#pragma unroll 1
    for (int64_t s = 0; s < sps; ++s) {
      const double2* vq = va + j0;
      double ar[NC], ai[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) ar[c] = ai[c] = 0.0;
#pragma unroll
      for (int jj = 0; jj < QMAX; ++jj) {  // 2 NC independent FMA chains
        if (NT > 0 || jj < Q) {
          const double2 a = pr[jj], v = vq[jj];
          const int c = jj % NC;
          ar[c] = fma(a.x, v.x, ar[c]);
          ar[c] = fma(-a.y, v.y, ar[c]);
          ai[c] = fma(a.x, v.y, ai[c]);
          ai[c] = fma(a.y, v.x, ai[c]);
        }
      }
#pragma unroll
      for (int w = 1; w < NC; w *= 2)
#pragma unroll
        for (int c = 0; c + w < NC; c += 2 * w) {
          ar[c] += ar[c + w];
          ai[c] += ai[c + w];
        }
      double re = ar[0], im = ai[0];
      re += __shfl_xor_sync(0xffffffffu, re, 1);
      im += __shfl_xor_sync(0xffffffffu, im, 1);
      re += __shfl_xor_sync(0xffffffffu, re, 2);
      im += __shfl_xor_sync(0xffffffffu, im, 2);
      if (active && q == 0) vb[i] = make_double2(re, im);
      __syncthreads();
      double2* t = va;
      va = vb;
      vb = t;
    }
  }
  for (int e = tid; e < n; e += blockDim.x) xb[e] = va[e];
}

// ---------------------------------------------------------------- K2c ------
constexpr int RS_THREADS = 256;


// x0/x1: batch x n complex ping-pong state in global memory (L2 resident)
__global__ void __launch_bounds__(RS_THREADS) rowsplit_kernel(const double2* __restrict__ p, int n,
                                                             double2* x0, double2* x1, int batch,
                                                             int64_t steps, unsigned int* bar) {
  extern __shared__ __align__(16) double2 sm2[];
  const int r0 = int((long long)n * blockIdx.x / gridDim.x);
  const int r1 = int((long long)n * (blockIdx.x + 1) / gridDim.x);
  const int rows = r1 - r0;
  double2* ps = sm2;                         // rows x n
  double2* vs = ps + size_t(rows) * n;       // batch x n
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < rows * n; e += RS_THREADS) ps[e] = p[size_t(r0) * n + e];
  double2* cur = x0;
  double2* nxt = x1;
#pragma unroll 1
  for (int64_t s = 0; s < steps; ++s) {
    for (int e = tid; e < batch * n; e += RS_THREADS) vs[e] = __ldcg(cur + e);  // L2: other CTAs wrote it
    __syncthreads();
    for (int task = warp; task < rows * batch; task += RS_THREADS / 32) {
      const int r = task % rows, b = task / rows;
      const double2* prow = ps + size_t(r) * n;
      const double2* v = vs + size_t(b) * n;
      double ar0 = 0.0, ai0 = 0.0, ar1 = 0.0, ai1 = 0.0;
      int j = lane;
      for (; j + 32 < n; j += 64) {
        const double2 a = prow[j], x = v[j], a2 = prow[j + 32], x2 = v[j + 32];
        ar0 = fma(a.x, x.x, ar0);
        ar0 = fma(-a.y, x.y, ar0);
        ai0 = fma(a.x, x.y, ai0);
        ai0 = fma(a.y, x.x, ai0);
        ar1 = fma(a2.x, x2.x, ar1);
        ar1 = fma(-a2.y, x2.y, ar1);
        ai1 = fma(a2.x, x2.y, ai1);
        ai1 = fma(a2.y, x2.x, ai1);
      }
      if (j < n) {
        const double2 a = prow[j], x = v[j];
        ar0 = fma(a.x, x.x, ar0);
        ar0 = fma(-a.y, x.y, ar0);
        ai0 = fma(a.x, x.y, ai0);
        ai0 = fma(a.y, x.x, ai0);
      }
      double re = ar0 + ar1, im = ai0 + ai1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, o);
        im += __shfl_xor_sync(0xffffffffu, im, o);
      }
      if (lane == 0) nxt[size_t(b) * n + r0 + r] = make_double2(re, im);
    }
    grid_barrier_sync(bar, unsigned(s + 1) * gridDim.x);
    double2* t = cur;
    cur = nxt;
    nxt = t;
  }
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

bool cta_chain_supported(size_t n) { return n >= 1 && n <= size_t(kMaxCtaN); }

static void cta_launch(const double* props, size_t n, double* x_aos, int64_t batch, int64_t segments, int64_t sps,
                       cudaStream_t s) {
  if (!cta_chain_supported(n)) throw invalid_argument("cta chain kernel supports n <= 96");
  const int ni = int(n);
  const int S = ni + ((4 - ni % 8) + 8) % 8;
  const size_t smem = (size_t(ni) * S + 2 * (ni + (kMaxCtaN + 3) / 4)) * sizeof(double2);
  const int threads = ((4 * ni + 31) / 32) * 32;
  const double2* p2 = reinterpret_cast<const double2*>(props);
  double2* x2 = reinterpret_cast<double2*>(x_aos);
  if (ni == 81) {
    ensure_max_dyn_smem((const void*)cta_chain_kernel<81>, int(smem));
    cta_chain_kernel<81><<<unsigned(batch), threads, smem, s>>>(p2, ni, x2, segments, sps);
  } else {
    ensure_max_dyn_smem((const void*)cta_chain_kernel<0>, int(smem));
    cta_chain_kernel<0><<<unsigned(batch), threads, smem, s>>>(p2, ni, x2, segments, sps);
  }
  LBG_CHECK_LAUNCH("cta_chain_kernel");
}

void launch_cta_chain(const double* p, size_t n, double* x_aos, int64_t batch, int64_t steps, cudaStream_t s) {
  if (batch <= 0 || steps <= 0) return;
  cta_launch(p, n, x_aos, batch, 1, steps, s);
}

// GRAPE chain of one trajectory over all segments in one launch
void launch_cta_chain_segments(const double* props, size_t n, int64_t segments, int64_t sps, double* x_aos,
                               cudaStream_t s) {
  if (segments <= 0 || sps <= 0) return;
  cta_launch(props, n, x_aos, 1, segments, sps, s);
}

// one CTA per SM (at most one per row); each holds ceil(n/grid) rows of P
int rowsplit_grid(size_t n) { return std::min<int>(sm_count(), int(n)); }

bool rowsplit_supported(size_t n, int64_t batch) {
  const int g = std::min<int>(sm_count(), int(n));
  const size_t rows = (n + g - 1) / g;
  return batch >= 1 && batch <= 4 && (rows * n + size_t(batch) * n) * 16 <= 220 * 1024;
}

size_t rowsplit_workspace(size_t n, int64_t batch) {
  return 2 * align_up(size_t(batch) * n * 16) + 256;
}

void launch_rowsplit(const double* p, size_t n, double* x_aos, int64_t batch, int64_t steps, void* work,
                     cudaStream_t s) {
  if (batch <= 0 || steps <= 0) return;
  if (!rowsplit_supported(n, batch)) throw invalid_argument("rowsplit kernel: shape not supported");
  if (!work) throw invalid_argument("rowsplit: workspace required");
  char* w = static_cast<char*>(work);
  double2* x0 = reinterpret_cast<double2*>(w);
  double2* x1 = reinterpret_cast<double2*>(w + align_up(size_t(batch) * n * 16));
  unsigned int* bar = reinterpret_cast<unsigned int*>(w + 2 * align_up(size_t(batch) * n * 16));
  check_cuda(cudaMemcpyAsync(x0, x_aos, size_t(batch) * n * 16, cudaMemcpyDeviceToDevice, s), "D2D");
  check_cuda(cudaMemsetAsync(bar, 0, sizeof(unsigned int), s), "memset");
  const int grid = rowsplit_grid(n);
  const int rows_max = int((n + grid - 1) / grid);
  const size_t smem = (size_t(rows_max) * n + size_t(batch) * n) * sizeof(double2);
  ensure_max_dyn_smem((const void*)rowsplit_kernel, int(smem));
  const double2* p2 = reinterpret_cast<const double2*>(p);
  int ni = int(n), bi = int(batch);
  int64_t st = steps;
  void* args[] = {(void*)&p2, (void*)&ni, (void*)&x0, (void*)&x1, (void*)&bi, (void*)&st, (void*)&bar};
  check_cuda(cudaLaunchCooperativeKernel((const void*)rowsplit_kernel, dim3(grid), dim3(RS_THREADS), args, smem, s),
             "rowsplit_kernel (cooperative)");
  note_launch();
  check_cuda(cudaMemcpyAsync(x_aos, (steps & 1) ? x1 : x0, size_t(batch) * n * 16, cudaMemcpyDeviceToDevice, s),
             "D2D");
}

}  // namespace lbg
