// k_density.cu — shared-P propagation of DENSITY MATRICES in their real
// coordinates (the transfer-matrix view of k_ptm.cu, for configs 0-3).
//
// lb::evolve only accepts physical states (propagate.cpp:77-80). A Lindblad
// propagator maps Hermitian matrices to Hermitian matrices, so on the real
// coordinates x[i*d+j] = Re rho_ij (i <= j), -Im rho_ij (i > j) it is the REAL
// n x n matrix P_R = T P T^-1 (n = d^2), built here entrywise from the complex P:
//   P_R[q][s] = f_q(c),  c = P[q][s] (s diagonal) | P[q][s] + P[q][s^T] (s upper)
//                            | i (P[q][s^T] - P[q][s]) (s lower),
//   f_q = Re for q upper / diagonal, -Im for q lower.
// A state splits exactly as rho = H + i H' with H = (rho + rho^dag)/2 and
// H' = (rho - rho^dag)/(2i) both Hermitian, and P(rho) = P(H) + i P(H'): the
// Hermitian part is one real vector, any anti-Hermitian part (zero for a
// physical state stored Hermitian, e.g. the configs' Ginibre GG^dag/tr) a second
// one. A step is n^2 real FMAs instead of 4 n^2 (8 d^4 -> 2 d^4 flops).
//
// Kernels: K1a-R `dfma9r_kernel` (n = 9: P_R in the constant bank, 81 DFMA per
// trajectory-step, one trajectory per thread), for n > 84 the real-arithmetic
// variant of the K1c tile engine (k_tiled.cu), and K1b-R `smem_real_kernel`
// (n <= 84: P_R resident in shared memory, real m8n8k4 DMMA, 32 vectors/CTA,
// 8 warps balanced over the 4 SMSPs).
#include <algorithm>
#include <map>
#include <mutex>

#include "../../include/lbg.h"
#include "common.cuh"
#include "internal.hpp"

namespace lbg {
namespace {

// Auto mode: the anti-Hermitian vectors follow the Hermitian ones (indices
// [half, count)); `flag` (device) says whether any of them is non-zero, so the
// stepping kernels skip them without a host round trip.
__device__ __forceinline__ int64_t live_count(int64_t count, int64_t half, const int* flag) {
  return (flag && *flag == 0) ? half : count;
}

// ---- conversions ------------------------------------------------------------
__device__ __forceinline__ double real_coord(double2 z, int i, int j) { return i <= j ? z.x : -z.y; }

// P (n x n complex, n = d^2) -> P_R (n x n real)
__global__ void p_to_real_kernel(const double2* __restrict__ p, int d, double* __restrict__ pr) {
  const int n = d * d;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * n) return;
  const int q = int(e / n), s = int(e - (long long)q * n);
  const int si = s / d, sj = s - si * d;
  double2 c;
  if (si == sj) {
    c = p[e];
  } else {
    const double2 a = p[e], bt = p[(long long)q * n + sj * d + si];
    c = si < sj ? make_double2(a.x + bt.x, a.y + bt.y) : make_double2(a.y - bt.y, bt.x - a.x);
  }
  const int qi = q / d, qj = q - qi * d;
  pr[e] = real_coord(c, qi, qj);
}

// rho (batch x n complex) -> x (batch x n real: Hermitian part) and, if xa is
// non-null, xa (batch x n real: the Hermitian matrix H' of the anti-Hermitian part)
__global__ void rho_to_real_kernel(const double2* __restrict__ rho, int d, long long count,
                                   double* __restrict__ x, double* __restrict__ xa, int* __restrict__ flag) {
  const int n = d * d;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= count * n) return;
  const long long b = e / n;
  const int p = int(e - b * n), i = p / d, j = p - i * d;
  const double2 z = rho[e], zt = rho[b * n + j * d + i];
  // H_ij = (rho_ij + conj rho_ji)/2 ;  H'_ij = (rho_ij - conj rho_ji)/(2i)
  const double2 h = make_double2(0.5 * (z.x + zt.x), 0.5 * (z.y - zt.y));
  x[e] = real_coord(h, i, j);
  if (xa) {
    const double2 dlt = make_double2(0.5 * (z.x - zt.x), 0.5 * (z.y + zt.y));  // (rho - rho^dag)/2
    const double2 hp = make_double2(dlt.y, -dlt.x);                            // divided by i
    const double c = real_coord(hp, i, j);
    xa[e] = c;
    if (flag) {  // one atomic per warp that saw a non-zero anti-Hermitian entry
      const unsigned m = __ballot_sync(__activemask(), c != 0.0);
      if (m && (threadIdx.x & 31) == __ffs(m) - 1) atomicOr(flag, 1);
    }
  }
}

// real coordinates -> rho = H(x) + i H(xa)
__global__ void real_to_rho_kernel(const double* __restrict__ x, const double* __restrict__ xa, int d,
                                   long long count, double2* __restrict__ rho, const int* __restrict__ flag) {
  const int n = d * d;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= count * n) return;
  const long long b = e / n;
  const int p = int(e - b * n), i = p / d, j = p - i * d;
  auto herm = [&](const double* v) {
    const double* vb = v + b * n;
    if (i == j) return make_double2(vb[p], 0.0);
    if (i < j) return make_double2(vb[p], vb[j * d + i]);
    return make_double2(vb[j * d + i], -vb[p]);
  };
  double2 r = herm(x);
  if (xa && !(flag && *flag == 0)) {
    const double2 a = herm(xa);
    r.x -= a.y;
    r.y += a.x;
  }
  rho[e] = r;
}

// ---- K1a-R: n = 9 --------------------------------------------------------------
constexpr int kSlots = 8;
__constant__ double c_pr9[kSlots][81];

template <int SLOT, int TPT>
__global__ void __launch_bounds__(128) dfma9r_kernel(double* __restrict__ x, int64_t count, int64_t half,
                                                     const int* __restrict__ flag, int64_t steps) {
  count = live_count(count, half, flag);
  if (int64_t(blockIdx.x) * 128 * TPT >= count) return;
  // TPT trajectories per thread (coalesced: t, t + 128, ...): each P operand
  // load feeds TPT FMAs, and TPT x 9 independent FMA chains hide DFMA latency
  const int64_t base = int64_t(blockIdx.x) * 128 * TPT + threadIdx.x;
  double v[TPT][9];
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const int64_t t = base + 128 * u;
#pragma unroll
    for (int j = 0; j < 9; ++j) v[u][j] = t < count ? x[t * 9 + j] : 0.0;
  }
  for (int64_t s = 0; s < steps; ++s) {
    // a loop-variant (always zero, uniform) offset keeps P's loads inside the
    // loop: every DFMA then takes its P operand from a uniform register
    // (LDCU -> DFMA R, R, UR, R) instead of ptxas hoisting 81 values into
    // the register file and shuttling them back through R2UR moves
    const double* __restrict__ p = c_pr9[SLOT] + (s >> 62);
    double nv[TPT][9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      // one accumulator per (trajectory, row): TPT x 9 independent 9-deep
      // chains, and no DADD tail (every FP64 instruction is a useful FMA)
      double a[TPT];
#pragma unroll
      for (int u = 0; u < TPT; ++u) a[u] = 0.0;
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        const double pij = p[i * 9 + j];
#pragma unroll
        for (int u = 0; u < TPT; ++u) a[u] = fma(pij, v[u][j], a[u]);
      }
#pragma unroll
      for (int u = 0; u < TPT; ++u) nv[u][i] = a[u];
    }
#pragma unroll
    for (int u = 0; u < TPT; ++u)
#pragma unroll
      for (int i = 0; i < 9; ++i) v[u][i] = nv[u][i];
  }
#pragma unroll
  for (int u = 0; u < TPT; ++u) {
    const int64_t t = base + 128 * u;
    if (t < count)
#pragma unroll
      for (int j = 0; j < 9; ++j) x[t * 9 + j] = v[u][j];
  }
}

struct SlotPool {
  std::mutex mu;
  cudaEvent_t ev[kSlots] = {};
  bool init = false;
  int next = 0;
};
SlotPool& pool() {  // per device: events and the constant bank belong to one device
  static std::mutex mu;
  static std::map<int, SlotPool*>* pools = new std::map<int, SlotPool*>;  // leaked: outlives CUDA teardown
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(mu);
  SlotPool*& p = (*pools)[dev];
  if (!p) p = new SlotPool;
  return *p;
}

// ---- K1b-R: n <= 84, real DMMA, P_R in shared memory ---------------------------
// 8 warps = 4 n-tiles x 2 row halves. The SMSP of warp w is w % 4, so each SMSP
// runs both halves of one n-tile: every SMSP issues exactly mt x kt DMMAs per
// step, no SMSP waits on a heavier one. Generic n (N == 0 instances): mt =
// ceil(n / 8) m-tiles split 6 + 5 at 11. n = 81 (the FRINGE specialisation):
// 10 DMMA m-tiles (real rows 0..79) split 5 + 5 over 20 k-steps (k < 80); the
// k = 80 rank-1 term and row 80 run on DFMA.
constexpr int kVec = 32, kWarpsR = 8;
struct RGeom {  // P_R: mt*8 rows x sp cols; V: kVec x sv
  int n, mt, kt, sp, sv;
  size_t p_bytes, v_bytes, total;
  __host__ __device__ RGeom(int n_) : n(n_) {
    mt = (n + 7) / 8;
    kt = (n + 3) / 4;
    sp = 4 * kt;
    sp += ((4 - sp % 16) + 16) % 16;  // = 4 (mod 16): conflict-free A fragments
    sv = 4 * kt;
    sv += ((4 - sv % 16) + 16) % 16;  // = 4 (mod 16): conflict-free B fragments
    p_bytes = size_t(mt) * 8 * sp * 8;
    v_bytes = size_t(kVec) * sv * 8;
    total = p_bytes + 2 * v_bytes;
  }
};

// N > 0: n known at compile time (n = 81 for config 2: no predicates, k loop
// fully unrolled); N == 0: runtime n. MG = m-tiles of the larger half.
// FRINGE (n = 81 only): the DMMA tiles cover rows and k 0..79 (10 m-tiles x 20
// k-steps, 5 + 5 per row half, instead of 11 x 21 over the 88 x 84 padding);
// the k = 80 term is a rank-1 DFMA update of each lane's own entries, and row 80
// is 32 dot products (8 lanes each, k = kq mod 8) split between the two warps
// of an n-tile -- the scheme of the c4 expm kernel (k_ptm.cu).
template <int N, int MG, bool FRINGE = false>
__global__ void __launch_bounds__(32 * kWarpsR, 1) smem_real_kernel(const double* __restrict__ pr, int n_rt,
                                                                    double* __restrict__ x, int64_t count,
                                                                    int64_t half, const int* __restrict__ flag,
                                                                    int64_t steps) {
  count = live_count(count, half, flag);
  if (int64_t(blockIdx.x) * kVec >= count) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = N > 0 ? N : n_rt;
  const RGeom g(n);
  double* ps = reinterpret_cast<double*>(smem);
  double* va = reinterpret_cast<double*>(smem + g.p_bytes);
  double* vb = reinterpret_cast<double*>(smem + g.p_bytes + g.v_bytes);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t b0 = int64_t(blockIdx.x) * kVec;
  for (int e = tid; e < g.mt * 8 * g.sp; e += blockDim.x) {
    const int i = e / g.sp, j = e - i * g.sp;
    ps[e] = (i < n && j < n) ? pr[size_t(i) * n + j] : 0.0;
  }
  for (int e = tid; e < kVec * g.sv; e += blockDim.x) {
    const int t = e / g.sv, r = e - t * g.sv;
    const int64_t b = b0 + t;
    va[e] = (b < count && r < n) ? x[b * n + r] : 0.0;
    vb[e] = 0.0;
  }
  __syncthreads();
  static_assert(!FRINGE || (N == 81 && MG == 5), "fringe layout: n = 81, 5 + 5 m-tiles");
  const int nt = warp & 3, rhalf = warp >> 2;
  const int mt_d = FRINGE ? 10 : g.mt, kt_d = FRINGE ? 20 : g.kt;
  const int m_split = (mt_d + 1) / 2;
  const int m_begin = rhalf ? m_split : 0;
  const int mcount = rhalf ? mt_d - m_split : m_split;
  const int gq = lane >> 2, tq = lane & 3;
  const double* pa = ps + size_t(m_begin * 8 + gq) * g.sp + tq;  // A frag: P_R[m*8+g][k*4+t]
  const int mstride = 8 * g.sp;
#pragma unroll 1
  for (int64_t s = 0; s < steps; ++s) {
    double acc[MG][2];
#pragma unroll
    for (int mi = 0; mi < MG; ++mi) acc[mi][0] = acc[mi][1] = 0.0;
    const double* vrow = va + (nt * 8 + gq) * g.sv + tq;  // B frag: V[n = nt*8+g][k*4+t]
    // register double buffer: fragments of k-step ks+1 load while ks computes
    double a_cur[MG], b_cur = vrow[0];
#pragma unroll
    for (int mi = 0; mi < MG; ++mi) a_cur[mi] = mi < mcount ? pa[mi * mstride] : 0.0;
#pragma unroll(N > 0 ? 21 : 1)
    for (int ks = 0; ks < kt_d; ++ks) {
      double a_nxt[MG], b_nxt = 0.0;
      const bool more = ks + 1 < kt_d;
      if (more) {
        b_nxt = vrow[(ks + 1) * 4];
#pragma unroll
        for (int mi = 0; mi < MG; ++mi) a_nxt[mi] = mi < mcount ? pa[mi * mstride + 4 * (ks + 1)] : 0.0;
      }
#pragma unroll
      for (int mi = 0; mi < MG; ++mi)
        if (mi < mcount) dmma(acc[mi], a_cur[mi], b_cur);
      if (more) {
        b_cur = b_nxt;
#pragma unroll
        for (int mi = 0; mi < MG; ++mi) a_cur[mi] = a_nxt[mi];
      }
    }
    if (FRINGE) {
      // k = 80: rank-1 update of the own entries
      const int t0 = nt * 8 + 2 * tq;
      const double v0 = va[t0 * g.sv + 80], v1 = va[(t0 + 1) * g.sv + 80];
#pragma unroll
      for (int mi = 0; mi < MG; ++mi) {
        const double pk = ps[size_t((m_begin + mi) * 8 + gq) * g.sp + 80];
        acc[mi][0] = fma(pk, v0, acc[mi][0]);
        acc[mi][1] = fma(pk, v1, acc[mi][1]);
      }
      // row 80 for vectors nt*8 + 4*rhalf + (lane >> 3): k = kq (mod 8)
      const int vec = nt * 8 + 4 * rhalf + (lane >> 3), kq = lane & 7;
      const double* p80 = ps + size_t(80) * g.sp;
      const double* vv = va + vec * g.sv;
      double f0 = 0.0, f1 = 0.0;
#pragma unroll
      for (int j = 0; j < 11; ++j) {
        const int k = kq + 8 * j;
        if (j == 10 && kq != 0) break;
        if (j & 1)
          f1 = fma(p80[k], vv[k], f1);
        else
          f0 = fma(p80[k], vv[k], f0);
      }
      double f = f0 + f1;
      f += __shfl_xor_sync(0xffffffffu, f, 1);
      f += __shfl_xor_sync(0xffffffffu, f, 2);
      f += __shfl_xor_sync(0xffffffffu, f, 4);
      if (kq == 0) vb[vec * g.sv + 80] = f;
    }
#pragma unroll
    for (int mi = 0; mi < MG; ++mi) {
      if (mi < mcount) {
        const int row = (m_begin + mi) * 8 + gq;  // C frag: row g, cols 2t, 2t+1
        const int t0 = nt * 8 + 2 * tq;
        if (row < n) {
          vb[t0 * g.sv + row] = acc[mi][0];
          vb[(t0 + 1) * g.sv + row] = acc[mi][1];
        }
      }
    }
    __syncthreads();
    double* tmp = va;
    va = vb;
    vb = tmp;
  }
  for (int e = tid; e < kVec * n; e += blockDim.x) {
    const int t = e / n, r = e - t * n;
    const int64_t b = b0 + t;
    if (b < count) x[b * n + r] = va[t * g.sv + r];
  }
}

template <int N, int MG, bool FRINGE = false>
void launch_smem_real(const double* pr, int n, double* x, int64_t count, int64_t half, const int* flag,
                      int64_t steps, cudaStream_t s) {
  const RGeom g(n);
  // one CTA per SM: the 8 warps are balanced over the 4 sub-partitions for ONE
  // CTA, and when the block scheduler stacks two live CTAs on an SM (observed
  // under ncu: 64 SMs x 2 instead of 128 x 1, 4.35 vs 2.2 ms at config 2) they
  // share its tensor pipes while other SMs idle. Asking for more than half the
  // SM's shared memory pins the residency to one.
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "device");
  int smem_sm = 0;
  check_cuda(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev), "attr");
  const size_t bytes = std::max(g.total, size_t(smem_sm / 2 + 1024));
  ensure_max_dyn_smem((const void*)smem_real_kernel<N, MG, FRINGE>, int(bytes));
  smem_real_kernel<N, MG, FRINGE><<<unsigned((count + kVec - 1) / kVec), 32 * kWarpsR, bytes, s>>>(
      pr, n, x, count, half, flag, steps);
  LBG_CHECK_LAUNCH("smem_real_kernel");
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

constexpr size_t kDirectMaxN = 84;  // K1a-R / K1b-R up to here, the real K1c tile engine beyond

bool density_supported(size_t n) { return n >= 1; }
bool density_uses_tile_engine(size_t n) { return n > kDirectMaxN; }

size_t density_workspace(size_t n, int64_t batch) {
  const size_t base = align_up(n * n * 8) + align_up(2 * size_t(batch) * n * 8) + 256;
  if (n <= kDirectMaxN) return base;
  // + the real tile engine's workspace for up to 2 batch vectors
  return base + align_up(tiled_real_workspace(n, 2 * batch));
}

// x: count real vectors of length n (in place)
static void step_real(const double* pr, size_t n, double* x, int64_t count, int64_t half, const int* flag,
                      int64_t steps, cudaStream_t s) {
  if (count <= 0 || steps <= 0) return;
  if (n == 9) {
    SlotPool& sp = pool();
    std::lock_guard<std::mutex> lk(sp.mu);
    if (!sp.init) {
      for (auto& e : sp.ev) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      sp.init = true;
    }
    const int slot = sp.next;
    sp.next = (sp.next + 1) % kSlots;
    check_cuda(cudaStreamWaitEvent(s, sp.ev[slot], 0), "stream wait");
    check_cuda(cudaMemcpyToSymbolAsync(c_pr9, pr, 81 * 8, size_t(81) * 8 * slot, cudaMemcpyDeviceToDevice, s),
               "P_R -> constant bank");
    constexpr int kTpt = 4;  // measured: 1 -> 112, 2 -> 185, 3 -> 190, 4 -> 195 G traj-steps/s (c1)
    const unsigned blocks = unsigned((count + 128 * kTpt - 1) / (128 * kTpt));
    switch (slot) {
#define LBG_SLOT(S) \
  case S: dfma9r_kernel<S, kTpt><<<blocks, 128, 0, s>>>(x, count, half, flag, steps); break;
      LBG_SLOT(0) LBG_SLOT(1) LBG_SLOT(2) LBG_SLOT(3) LBG_SLOT(4) LBG_SLOT(5) LBG_SLOT(6) LBG_SLOT(7)
#undef LBG_SLOT
    }
    LBG_CHECK_LAUNCH("dfma9r_kernel");
    check_cuda(cudaEventRecord(sp.ev[slot], s), "event record");
    return;
  }
  const int ni = int(n);
  // n = 81 (config 2): the fringe layout, 2.10 vs 2.24 ms per c2 pass over the 88 x 84 padded tiles
  if (ni == 81) return launch_smem_real<81, 5, true>(pr, ni, x, count, half, flag, steps, s);
  switch (((ni + 7) / 8 + 1) / 2) {
#define LBG_MG(M) \
  case M: return launch_smem_real<0, M>(pr, ni, x, count, half, flag, steps, s);
    LBG_MG(1) LBG_MG(2) LBG_MG(3) LBG_MG(4) LBG_MG(5) LBG_MG(6)
#undef LBG_MG
    default: throw invalid_argument("density: n too large for the shared-memory real kernel");
  }
}

void launch_density(const double* p, size_t d, double* rho, int64_t batch, int64_t steps, int mode, void* work,
                    cudaStream_t s) {
  const size_t n = d * d;
  if (!density_supported(n)) throw invalid_argument("density mode: empty state");
  if (mode < kDensityHermitian || mode > kDensityAuto) throw invalid_argument("density: unknown mode");
  if (batch <= 0) return;
  const bool tiled_auto = n > kDirectMaxN && mode == kDensityAuto;  // decided after one flag read (below)
  char* w = static_cast<char*>(work);
  double* pr = reinterpret_cast<double*>(w);
  double* x = reinterpret_cast<double*>(w + align_up(n * n * 8));
  double* xa = x + size_t(batch) * n;  // contiguous with x: one stepping launch covers both
  int* flag = reinterpret_cast<int*>(w + align_up(n * n * 8) + align_up(2 * size_t(batch) * n * 8));
  const bool general = mode != kDensityHermitian;
  int* live = mode == kDensityAuto ? flag : nullptr;
  if (live) check_cuda(cudaMemsetAsync(live, 0, sizeof(int), s), "memset flag");
  const long long nn = (long long)n * n, ne = (long long)batch * n;
  p_to_real_kernel<<<unsigned((nn + 255) / 256), 256, 0, s>>>(reinterpret_cast<const double2*>(p), int(d), pr);
  LBG_CHECK_LAUNCH("p_to_real_kernel");
  rho_to_real_kernel<<<unsigned((ne + 255) / 256), 256, 0, s>>>(reinterpret_cast<const double2*>(rho), int(d),
                                                                batch, x, general ? xa : nullptr, live);
  LBG_CHECK_LAUNCH("rho_to_real_kernel");
  // the two real vector sets are contiguous: one launch covers both (auto mode:
  // the anti-Hermitian half is skipped on the device when it is all zero)
  if (n <= kDirectMaxN) {
    step_real(pr, n, x, general ? 2 * batch : batch, batch, live, steps, s);
  } else {
    bool gen = general;
    if (tiled_auto) {  // read the flag (one 4-byte sync): the tile engine takes its vector count from the host
      int h = 0;
      check_cuda(cudaMemcpyAsync(&h, live, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H flag");
      sync_stream_spin(s, "sync flag");
      gen = h != 0;
    }
    void* inner = w + align_up(n * n * 8) + align_up(2 * size_t(batch) * n * 8) + 256;
    const int64_t nvec = gen ? 2 * batch : batch;
    launch_tiled_evolve_real(pr, n, x, nvec, steps, inner, s);  // K1c on real arithmetic
  }
  real_to_rho_kernel<<<unsigned((ne + 255) / 256), 256, 0, s>>>(x, general ? xa : nullptr, int(d), batch,
                                                                reinterpret_cast<double2*>(rho), live);
  LBG_CHECK_LAUNCH("real_to_rho_kernel");
}

}  // namespace lbg
