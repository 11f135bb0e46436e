// k_smem.cu — K1b: shared-P batched propagation with P resident in shared
// memory, FP64 tensor cores (DMMA) — config 2 (d = 9, n = 81, 4,096 trajectories).
//
// Each CTA owns 32 trajectories (four 8-wide MMA n-tiles) for ALL steps:
//   - P (n x n complex, 110 KB padded) is staged once into shared memory;
//   - the 32 state vectors live in shared memory in real form, ping-ponged;
//   - per step the CTA computes V_next' (2n x 32) = P' (2n x 2n) * V' (2n x 32)
//     as m8n8k4 DMMAs (real form of the complex product, common.cuh), 12 warps =
//     3 row groups x 4 n-tiles (3 warps per SMSP, balanced), then __syncthreads().
// HBM traffic is one read + one write of the state and one read of P per CTA;
// the bound is the DMMA pipe (tile use at n=81: 162/168 rows x 162/164 k = 95.3%).
// Shared-memory layouts are padded so every fragment load is conflict-free:
//   P row stride SP = 2 (mod 8) complex, V row stride SV = 4 (mod 16) doubles.
//
// Replaces step_soa_kernel (proj/src/kernels_variants.cpp:26-41) inside
// evolve (proj/src/propagate.cpp:85-92), batched over trajectories.
#include <cstdint>

#include "common.cuh"
#include "internal.hpp"

namespace lbg {

namespace {

constexpr int kTraj = 32;   // trajectories per CTA (4 n-tiles)
constexpr int kWarps = 12;  // 3 row groups x 4 n-tiles
constexpr int kMaxN = 84;

struct SmemGeom {
  int n, mt, kt, sp, sv;
  size_t p_bytes, v_bytes, total;
  __host__ __device__ SmemGeom(int n_) : n(n_) {
    mt = (n + 3) / 4;      // m8 tiles over 2n real rows
    kt = (n + 1) / 2;      // k4 steps over 2n real cols
    sp = 2 * kt;           // complex cols incl. K padding
    sp += (2 - (sp % 8) + 8) % 8;  // sp = 2 (mod 8)
    sv = 4 * kt;           // doubles per trajectory row incl. K padding
    sv += (4 - (sv % 16) + 16) % 16;  // sv = 4 (mod 16)
    p_bytes = size_t(mt) * 4 * sp * 16;
    v_bytes = size_t(kTraj) * sv * 8;
    total = p_bytes + 2 * v_bytes;
  }
};

// N > 0: n known at compile time (config 2 uses N = 81: no tile predicates,
// fully unrolled k loop); N == 0: runtime n.
template <int N, int MG, Layout L>
__global__ void __launch_bounds__(32 * kWarps, 1)
    smem_kernel(const double2* __restrict__ p, int n_rt, double* __restrict__ x_re,
                double* __restrict__ x_im, double* __restrict__ x_aos, int64_t batch,
                int64_t steps) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = N > 0 ? N : n_rt;
  const SmemGeom g(n);
  double2* ps = reinterpret_cast<double2*>(smem);
  double* va = reinterpret_cast<double*>(smem + g.p_bytes);
  double* vb = reinterpret_cast<double*>(smem + g.p_bytes + g.v_bytes);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t b0 = int64_t(blockIdx.x) * kTraj;

  // ---- stage P (zero padded) and the CTA's 32 state vectors (real form) ----
  const int prow = g.mt * 4;
  for (int e = tid; e < prow * g.sp; e += blockDim.x) {
    const int i = e / g.sp, j = e - i * g.sp;
    ps[e] = (i < n && j < n) ? p[size_t(i) * n + j] : make_double2(0.0, 0.0);
  }
  for (int e = tid; e < kTraj * g.sv; e += blockDim.x) {
    const int t = e / g.sv, r = e - t * g.sv;
    const int64_t b = b0 + t;
    double v = 0.0;
    if (b < batch && r < 2 * n) {
      if (L == Layout::soa)
        v = (r & 1) ? x_im[b * n + (r >> 1)] : x_re[b * n + (r >> 1)];
      else
        v = x_aos[b * 2 * n + r];
    }
    va[e] = v;
    vb[e] = 0.0;
  }
  __syncthreads();

  const AFragLane af(lane);
  const int mg = warp >> 2;  // row group 0..2
  const int nt = warp & 3;   // n-tile 0..3
  const int m_begin = mg * MG;
  const int bn = nt * 8 + (lane >> 2);  // B fragment column (trajectory in CTA)
  const int bk = lane & 3;              // B fragment k within the step
  // per-lane A fragment base (doubles) and per-m-tile stride
  const double* pa = reinterpret_cast<const double*>(ps) + size_t(m_begin * 4 + af.di) * 2 * g.sp +
                     2 * af.dj + af.comp;
  const int mstride = 4 * 2 * g.sp;
  int mcount = g.mt - m_begin;
  mcount = mcount < 0 ? 0 : (mcount > MG ? MG : mcount);

  for (int64_t s = 0; s < steps; ++s) {
    double acc[MG][2];
#pragma unroll
    for (int mi = 0; mi < MG; ++mi) acc[mi][0] = acc[mi][1] = 0.0;
    const double* vrow = va + bn * g.sv + bk;
    // register double buffer: fragments of step ks+1 load while ks computes
    double a_cur[MG], b_cur;
    b_cur = vrow[0];
#pragma unroll
    for (int mi = 0; mi < MG; ++mi) a_cur[mi] = (N > 0 || mi < mcount) ? af.sign(pa[mi * mstride]) : 0.0;
#pragma unroll(N > 0 ? 41 : 1)
    for (int ks = 0; ks < g.kt; ++ks) {
      double a_nxt[MG], b_nxt = 0.0;
      const bool more = ks + 1 < g.kt;
      if (more) {
        b_nxt = vrow[(ks + 1) * 4];
#pragma unroll
        for (int mi = 0; mi < MG; ++mi)
          a_nxt[mi] = (N > 0 || mi < mcount) ? af.sign(pa[mi * mstride + 4 * (ks + 1)]) : 0.0;
      }
#pragma unroll
      for (int mi = 0; mi < MG; ++mi)
        if (N > 0 || mi < mcount) dmma(acc[mi], a_cur[mi], b_cur);
      if (more) {
        b_cur = b_nxt;
#pragma unroll
        for (int mi = 0; mi < MG; ++mi) a_cur[mi] = a_nxt[mi];
      }
    }
    // epilogue: complex-pair the fragments and write V_next (real form)
#pragma unroll
    for (int mi = 0; mi < MG; ++mi) {
      if (N > 0 || mi < mcount) {
        int coff;
        const double2 z = pair_complex(acc[mi], lane, coff);
        const int i = (m_begin + mi) * 4 + (lane >> 3);
        const int t = nt * 8 + coff;
        if (i < n) *reinterpret_cast<double2*>(vb + t * g.sv + 2 * i) = z;
      }
    }
    __syncthreads();
    double* tmp = va;
    va = vb;
    vb = tmp;
  }

  // ---- write the final states back ----
  for (int e = tid; e < kTraj * 2 * n; e += blockDim.x) {
    const int t = e / (2 * n), r = e - t * 2 * n;
    const int64_t b = b0 + t;
    if (b >= batch) continue;
    const double v = va[t * g.sv + r];
    if (L == Layout::soa) {
      if (r & 1)
        x_im[b * n + (r >> 1)] = v;
      else
        x_re[b * n + (r >> 1)] = v;
    } else {
      x_aos[b * 2 * n + r] = v;
    }
  }
}

// K1b at the per-rank shares of config 2 (2,048 / 1,024 trajectories): NT = 2
// or 1 n-tiles per CTA instead of 4, so 256 / 128 n-tiles still fill 128 SMs.
// The 12 warps are 12 / NT row groups x NT n-tiles. The DMMA m-tiles cover
// complex rows 0..79 only (20 tiles of 8 real rows; a 21st tile would carry the
// single complex row 80 in 8 real rows): they are dealt to the row groups so
// that warps 8..11 (one per sub-partition) carry fewer (NT = 2: 4,4,4,4,2,2;
// NT = 1: eight groups of 2 and four of 1) and warp w runs on sub-partition
// w % 4: every sub-partition issues 10 (NT = 2) / 5 (NT = 1) DMMAs per k-step
// (NT = 4: 21). Complex row 80 is a DFMA dot product on warps 8..11 (T / 4
// trajectories each, 32 / (T / 4) k-slices per trajectory, shuffle-reduced)
// after their DMMAs, while the heavier warps still fill the pipe. The m-tile
// count is a template parameter (no predicated mma.sync; two code paths per
// kernel).
template <int MC, bool FR, int SL>
__device__ __forceinline__ double* nt_steps(const double* __restrict__ pa, int mstride, double* va, double* vb,
                                            int bn, int bk, int sv, int i0, int t0, int lane, int64_t steps,
                                            const double2* __restrict__ prow80, int tfr) {
  constexpr int KT = 41;
  for (int64_t s = 0; s < steps; ++s) {
    double acc[MC][2];
#pragma unroll
    for (int mi = 0; mi < MC; ++mi) acc[mi][0] = acc[mi][1] = 0.0;
    const double* vrow = va + bn * sv + bk;
    const AFragLane af(lane);
    double a_cur[MC], b_cur = vrow[0];
#pragma unroll
    for (int mi = 0; mi < MC; ++mi) a_cur[mi] = af.sign(pa[mi * mstride]);
#pragma unroll
    for (int ks = 0; ks < KT; ++ks) {
      double a_nxt[MC], b_nxt = 0.0;
      if (ks + 1 < KT) {
        b_nxt = vrow[(ks + 1) * 4];
#pragma unroll
        for (int mi = 0; mi < MC; ++mi) a_nxt[mi] = af.sign(pa[mi * mstride + 4 * (ks + 1)]);
      }
#pragma unroll
      for (int mi = 0; mi < MC; ++mi) dmma(acc[mi], a_cur[mi], b_cur);
      if (ks + 1 < KT) {
        b_cur = b_nxt;
#pragma unroll
        for (int mi = 0; mi < MC; ++mi) a_cur[mi] = a_nxt[mi];
      }
    }
#pragma unroll
    for (int mi = 0; mi < MC; ++mi) {
      int coff;
      const double2 z = pair_complex(acc[mi], lane, coff);
      const int i = i0 + mi * 4 + (lane >> 3);
      *reinterpret_cast<double2*>(vb + (t0 + coff) * sv + 2 * i) = z;
    }
    if constexpr (FR) {  // complex row 80 of trajectory tfr: k = ksl + SL j
      const int ksl = lane & (SL - 1);
      const double* x = va + tfr * sv;
      double r1 = 0.0, r2 = 0.0, i1 = 0.0, i2 = 0.0;
#pragma unroll
      for (int j = 0; j < (81 + SL - 1) / SL; ++j) {
        const int k = ksl + SL * j;
        if (k < 81) {
          const double2 pv = prow80[k];
          const double xr = x[2 * k], xi = x[2 * k + 1];
          r1 = fma(pv.x, xr, r1);
          r2 = fma(-pv.y, xi, r2);
          i1 = fma(pv.y, xr, i1);
          i2 = fma(pv.x, xi, i2);
        }
      }
      double re = r1 + r2, im = i1 + i2;
#pragma unroll
      for (int o = SL / 2; o >= 1; o >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, o);
        im += __shfl_xor_sync(0xffffffffu, im, o);
      }
      if (ksl == 0) *reinterpret_cast<double2*>(vb + tfr * sv + 160) = make_double2(re, im);
    }
    __syncthreads();
    double* tmp = va;
    va = vb;
    vb = tmp;
  }
  return va;
}

template <int NT, Layout L>
__global__ void __launch_bounds__(32 * kWarps, 1)
    smem81_nt_kernel(const double2* __restrict__ p, double* __restrict__ x_re, double* __restrict__ x_im,
                     double* __restrict__ x_aos, int64_t batch, int64_t steps) {
  extern __shared__ __align__(16) unsigned char smem[];
  // RGH heavy row groups of H m-tiles, then the 4 / NT light groups (warps 8..11) of LM
  constexpr int n = 81, T = 8 * NT, RG = kWarps / NT, RGH = RG - 4 / NT, H = NT == 2 ? 4 : 2, LM = H / 2;
  constexpr int TPW = T / 4, SL = 32 / TPW;  // row-80 trajectories per light warp, k-slices each
  static_assert(RGH * H + (RG - RGH) * LM == 20, "20 m-tiles (complex rows 0..79)");
  const SmemGeom g(n);
  double2* ps = reinterpret_cast<double2*>(smem);
  double* va = reinterpret_cast<double*>(smem + g.p_bytes);
  double* vb = reinterpret_cast<double*>(smem + g.p_bytes + g.v_bytes);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t b0 = int64_t(blockIdx.x) * T;
  for (int e = tid; e < g.mt * 4 * g.sp; e += blockDim.x) {
    const int i = e / g.sp, j = e - i * g.sp;
    ps[e] = (i < n && j < n) ? p[size_t(i) * n + j] : make_double2(0.0, 0.0);
  }
  for (int e = tid; e < T * g.sv; e += blockDim.x) {
    const int t = e / g.sv, r = e - t * g.sv;
    const int64_t b = b0 + t;
    double v = 0.0;
    if (b < batch && r < 2 * n) {
      if (L == Layout::soa)
        v = (r & 1) ? x_im[b * n + (r >> 1)] : x_re[b * n + (r >> 1)];
      else
        v = x_aos[b * 2 * n + r];
    }
    va[e] = v;
    vb[e] = 0.0;
  }
  __syncthreads();
  const AFragLane af(lane);
  const int rg = warp / NT, nt = warp % NT;
  const int m_begin = rg < RGH ? rg * H : RGH * H + (rg - RGH) * LM;
  const double* pa =
      reinterpret_cast<const double*>(ps) + size_t(m_begin * 4 + af.di) * 2 * g.sp + 2 * af.dj + af.comp;
  const int mstride = 4 * 2 * g.sp, bn = nt * 8 + (lane >> 2), bk = lane & 3;
  const double2* prow80 = ps + 80 * g.sp;
  const int tfr = (warp - 8) * TPW + lane / SL;  // light warps 8..11
  double* fin;
  if (rg < RGH)
    fin = nt_steps<H, false, SL>(pa, mstride, va, vb, bn, bk, g.sv, m_begin * 4, nt * 8, lane, steps, prow80, 0);
  else
    fin = nt_steps<LM, true, SL>(pa, mstride, va, vb, bn, bk, g.sv, m_begin * 4, nt * 8, lane, steps, prow80, tfr);
  for (int e = tid; e < T * 2 * n; e += blockDim.x) {
    const int t = e / (2 * n), r = e - t * 2 * n;
    const int64_t b = b0 + t;
    if (b >= batch) continue;
    const double v = fin[t * g.sv + r];
    if (L == Layout::soa) {
      if (r & 1)
        x_im[b * n + (r >> 1)] = v;
      else
        x_re[b * n + (r >> 1)] = v;
    } else {
      x_aos[b * 2 * n + r] = v;
    }
  }
}

template <int NT>
void launch_nt(const double* p, double* x_re, double* x_im, double* x_aos, int64_t batch, int64_t steps,
               Layout layout, cudaStream_t s) {
  const SmemGeom g(81);
  const unsigned blocks = static_cast<unsigned>((batch + 8 * NT - 1) / (8 * NT));
  const double2* p2 = reinterpret_cast<const double2*>(p);
  auto k = layout == Layout::soa ? smem81_nt_kernel<NT, Layout::soa> : smem81_nt_kernel<NT, Layout::aos>;
  ensure_max_dyn_smem((const void*)k, int(g.total));
  k<<<blocks, 32 * kWarps, g.total, s>>>(p2, x_re, x_im, x_aos, batch, steps);
  LBG_CHECK_LAUNCH("smem81_nt_kernel");
}

// n = 81: n-tiles per CTA (4, 2 or 1) with the shortest critical path, in DMMA
// issue slots per sub-partition and step: waves x busiest sub-partition's
// DMMAs per k-step x 41 k-steps (NT = 4 first: ties keep the measured kernel)
// (per-slot weights in percent: the measured pass time per DMMA slot of the
// NT = 2 / 1 kernels is ~9% / ~13% above NT = 4's — two code paths, the row-80 tail)
constexpr int kBusiest[3][3] = {{4, 21, 100}, {2, 10, 109}, {1, 5, 113}};
int smem81_nt(int64_t batch) {
  int64_t best = INT64_MAX;
  int nt_best = 4;
  const int64_t ntiles = (batch + 7) / 8;
  for (const auto& c : kBusiest) {
    const int64_t ctas = (ntiles + c[0] - 1) / c[0];
    const int64_t cost = ((ctas + sm_count() - 1) / sm_count()) * c[1] * 41 * c[2];
    if (cost < best) best = cost, nt_best = c[0];
  }
  return nt_best;
}

template <int N, int MG>
void launch_mg(const double* p, int n, double* x_re, double* x_im, double* x_aos, int64_t batch,
               int64_t steps, Layout layout, cudaStream_t s) {
  const SmemGeom g(n);
  const unsigned blocks = static_cast<unsigned>((batch + kTraj - 1) / kTraj);
  const double2* p2 = reinterpret_cast<const double2*>(p);
  if (layout == Layout::soa) {
    auto k = smem_kernel<N, MG, Layout::soa>;
    ensure_max_dyn_smem((const void*)k, int(g.total));
    k<<<blocks, 32 * kWarps, g.total, s>>>(p2, n, x_re, x_im, nullptr, batch, steps);
  } else {
    auto k = smem_kernel<N, MG, Layout::aos>;
    ensure_max_dyn_smem((const void*)k, int(g.total));
    k<<<blocks, 32 * kWarps, g.total, s>>>(p2, n, nullptr, nullptr, x_aos, batch, steps);
  }
  LBG_CHECK_LAUNCH("smem_kernel");
}

}  // namespace

bool smem_supported(std::size_t n) { return n >= 1 && n <= kMaxN; }

int64_t smem81_cost(int64_t batch) {
  const int nt = smem81_nt(batch);
  int busiest = 21, weight = 100;
  for (const auto& c : kBusiest)
    if (c[0] == nt) busiest = c[1], weight = c[2];
  const int64_t ctas = ((batch + 7) / 8 + nt - 1) / nt;
  return ((ctas + sm_count() - 1) / sm_count()) * busiest * 41 * weight / 100;
}

void launch_smem(const double* p_dev, std::size_t n, double* x_re, double* x_im, double* x_aos,
                 int64_t batch, int64_t steps, Layout layout, cudaStream_t s) {
  if (batch <= 0) return;
  if (!smem_supported(n)) throw invalid_argument("smem kernel supports n <= 84");
  if (n == 81) {
    const int nt = smem81_nt(batch);
    if (nt == 2) return launch_nt<2>(p_dev, x_re, x_im, x_aos, batch, steps, layout, s);
    if (nt == 1) return launch_nt<1>(p_dev, x_re, x_im, x_aos, batch, steps, layout, s);
    return launch_mg<81, 7>(p_dev, 81, x_re, x_im, x_aos, batch, steps, layout, s);
  }
  const int mt = (int(n) + 3) / 4;
  const int mg = (mt + 2) / 3;
  switch (mg) {
#define LBG_CASE(M) \
  case M: return launch_mg<0, M>(p_dev, int(n), x_re, x_im, x_aos, batch, steps, layout, s);
    LBG_CASE(1) LBG_CASE(2) LBG_CASE(3) LBG_CASE(4) LBG_CASE(5) LBG_CASE(6) LBG_CASE(7)
#undef LBG_CASE
    default: throw invalid_argument("smem kernel: n too large");
  }
}

}  // namespace lbg
