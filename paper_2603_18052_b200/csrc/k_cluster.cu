// k_cluster.cu — K1b-C: the shared-P stepper for n = 81 (config 2) on
// 2-CTA thread-block clusters, to remove the SM quantisation of K1b.
//
// K1b gives each CTA 32 trajectories (four 8-wide MMA n-tiles); 4,096
// trajectories are 512 n-tiles, so 128 of 148 SMs work and the step time is
// that of 4 n-tiles (86.5% of the machine at best). Here a cluster of two CTAs
// (two SMs) owns k <= 7 n-tiles: each CTA computes floor(k/2) n-tiles alone
// and, when k is odd, HALF of the rows of one shared n-tile; the two halves
// are exchanged through distributed shared memory (st.shared::cluster into
// the peer's next-state buffer) and one cluster barrier per step replaces the
// CTA barrier. 4,096 trajectories -> 74 clusters x 7 n-tiles on all 148 SMs,
// 3.5 n-tiles of work per SM instead of 4.
//
// Inside a CTA, 8 warps (two per SM sub-partition) each own a list of m-tiles
// (8 real rows of P) for ALL of the CTA's n-tiles, so an A fragment feeds up to
// four DMMAs; the lists are balanced on the host (longest-processing-time
// greedy over "heavy" m-tiles, which also carry the shared n-tile, and "light"
// ones), so every sub-partition issues the same number of DMMAs within one.
// Layouts are K1b's (k_smem.cu): P real-form A fragments from complex rows
// (stride 2 mod 8 complex), V[traj][2n] real form (stride 4 mod 16 doubles).
#include <algorithm>
#include <cstdint>
#include <vector>

#include "common.cuh"
#include "internal.hpp"

namespace lbg {
namespace {

constexpr int CN = 81;                 // n (config 2)
constexpr int CMT = (CN + 3) / 4;      // 21 m-tiles (4 complex rows = 8 real rows)
constexpr int CKT = (CN + 1) / 2;      // 41 k-steps (2 complex = 4 real columns)
constexpr int CWARPS = 8;              // two warps per sub-partition (w and w + 4)
constexpr int MAXM = 7;                // m-tiles per warp (LPT keeps it <= 6 at k = 7)
constexpr int SLOTS = 4;               // n-tile slots per CTA: own 0..h-1, shared = 3
constexpr int SP = [] {                // complex row stride of P: = 2 (mod 8)
  int sp = 2 * CKT;
  return sp + (2 - (sp % 8) + 8) % 8;
}();
constexpr int SV = [] {                // double row stride of V: = 4 (mod 16)
  int sv = 4 * CKT;
  return sv + (4 - (sv % 16) + 16) % 16;
}();
constexpr size_t P_BYTES = size_t(CMT) * 4 * SP * 16;
constexpr size_t V_BYTES = size_t(SLOTS) * 8 * SV * 8;
constexpr size_t SMEM_BYTES = P_BYTES + 2 * V_BYTES;

struct ClusterPlan {
  int k, h, shared;                 // n-tiles per cluster, own per CTA, 1 if an n-tile is split
  int lo[2], hi[2];                 // m-tile half [lo, hi) each rank computes of the shared n-tile
  signed char mlist[2][CWARPS][MAXM];  // heavy m-tiles first
  signed char mcount[2][CWARPS];
  signed char nheavy[2][CWARPS];
};

// One warp's step loop. NH "heavy" m-tiles (3 own n-tiles + the shared one)
// and NL "light" m-tiles (own n-tiles only) are compile-time counts, so the
// DMMA sequence has no predicates (a runtime count makes ptxas wrap every
// mma.sync in WARPSYNC / BSSY convergence code, measured 4x slower).
template <int NH, int NL>
__device__ __forceinline__ double* warp_steps(const double* __restrict__ pbase, const signed char* mlist,
                                              double* va, double* vb, unsigned va_peer0, unsigned vb_peer0,
                                              uint64_t* xbar, unsigned peer_bar0, unsigned in_bytes, int lane,
                                              int64_t steps) {
  constexpr int NM = NH + NL, NQ = SLOTS;  // slot 3 = the shared n-tile (heavy m-tiles only)
  int mrow[NM > 0 ? NM : 1];
#pragma unroll
  for (int mi = 0; mi < NM; ++mi) mrow[mi] = mlist[mi];  // heavy first, then light
  const AFragLane af(lane);
  const int bn = lane >> 2, bk = lane & 3;
  bool flip = false;
#pragma unroll 1
  for (int64_t s = 0; s < steps; ++s) {
    // step parity selects the mbarrier: the peer cannot run two steps ahead
    const int par = int(s & 1);
    if (threadIdx.x == 0) mbar_expect_tx(&xbar[par], in_bytes);
    double acc[NM > 0 ? NM : 1][NQ][2];
#pragma unroll
    for (int mi = 0; mi < NM; ++mi)
#pragma unroll
      for (int q = 0; q < NQ; ++q) acc[mi][q][0] = acc[mi][q][1] = 0.0;
    const double* vrow = va + bn * SV + bk;
    double a_cur[NM > 0 ? NM : 1], b_cur[NQ];
#pragma unroll
    for (int mi = 0; mi < NM; ++mi) a_cur[mi] = af.sign(pbase[size_t(mrow[mi]) * 4 * 2 * SP]);
#pragma unroll
    for (int q = 0; q < NQ; ++q) b_cur[q] = vrow[q * 8 * SV];
#pragma unroll  // fully: a rolled loop makes ptxas shuffle the accumulators around every DMMA
    for (int ks = 0; ks < CKT; ++ks) {
      double a_nxt[NM > 0 ? NM : 1], b_nxt[NQ];
      const int kn = ks + 1 < CKT ? ks + 1 : ks;  // last iteration reloads (harmless)
#pragma unroll
      for (int q = 0; q < NQ; ++q) b_nxt[q] = vrow[q * 8 * SV + kn * 4];
#pragma unroll
      for (int mi = 0; mi < NM; ++mi) a_nxt[mi] = af.sign(pbase[size_t(mrow[mi]) * 4 * 2 * SP + 4 * kn]);
#pragma unroll
      for (int mi = 0; mi < NM; ++mi) {
#pragma unroll
        for (int q = 0; q < NQ - 1; ++q) dmma(acc[mi][q], a_cur[mi], b_cur[q]);
        if (mi < NH) dmma(acc[mi][NQ - 1], a_cur[mi], b_cur[NQ - 1]);
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) b_cur[q] = b_nxt[q];
#pragma unroll
      for (int mi = 0; mi < NM; ++mi) a_cur[mi] = a_nxt[mi];
    }
    const unsigned vb_peer = flip ? va_peer0 : vb_peer0;
    const unsigned peer_bar = peer_bar0 + unsigned(par) * 8u;
#pragma unroll
    for (int mi = 0; mi < NM; ++mi) {
      const int i = mrow[mi] * 4 + (lane >> 3);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        if (q == NQ - 1 && mi >= NH) continue;
        int coff;
        const double2 z = pair_complex(acc[mi][q], lane, coff);
        const int t = q * 8 + coff;
        if (i < CN) {
          *reinterpret_cast<double2*>(vb + t * SV + 2 * i) = z;
          if (q == NQ - 1) st_async_f64x2(vb_peer + unsigned(t * SV + 2 * i) * 8u, z, peer_bar);
        }
      }
    }
    __syncthreads();                                    // own results written locally
    mbar_wait_parity_cluster(&xbar[par], unsigned((s >> 1) & 1));  // the peer's half has landed
    double* tmp = va;
    va = vb;
    vb = tmp;
    flip = !flip;
  }
  return va;
}

// k = 7 n-tiles per cluster: CTA r owns n-tiles 3r..3r+2 of the cluster and
// computes m-tiles [lo_r, hi_r) of the shared 7th. Per-warp (heavy, light)
// m-tile counts come from the host plan; each combination is one template.
template <Layout L>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32 * CWARPS, 1)
    smem_cluster_kernel(const double2* __restrict__ p, double* __restrict__ x_re, double* __restrict__ x_im,
                        double* __restrict__ x_aos, int64_t batch, int64_t steps, const ClusterPlan plan) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2* ps = reinterpret_cast<double2*>(smem);
  double* va = reinterpret_cast<double*>(smem + P_BYTES);
  double* vb = reinterpret_cast<double*>(smem + P_BYTES + V_BYTES);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned rank = cluster_ctarank(), peer = rank ^ 1u;
  const int64_t cl = blockIdx.x >> 1;
  constexpr int K = 7, H = 3;
  // n-tile of slot s: own s < 3, shared s == 3
  auto slot_tile = [&](int s) -> int64_t { return s < H ? cl * K + int64_t(rank) * H + s : cl * K + 2 * H; };

  // ---- stage P (zero padded) and the slots' state vectors (real form) ----
  for (int e = tid; e < CMT * 4 * SP; e += blockDim.x) {
    const int i = e / SP, j = e - i * SP;
    ps[e] = (i < CN && j < CN) ? p[size_t(i) * CN + j] : make_double2(0.0, 0.0);
  }
  for (int e = tid; e < SLOTS * 8 * SV; e += blockDim.x) {
    const int t = e / SV, r = e - t * SV;
    const int64_t b = slot_tile(t >> 3) * 8 + (t & 7);
    double v = 0.0;
    if (b < batch && r < 2 * CN) {
      if (L == Layout::soa)
        v = (r & 1) ? x_im[b * CN + (r >> 1)] : x_re[b * CN + (r >> 1)];
      else
        v = x_aos[b * 2 * CN + r];
    }
    va[e] = v;
    vb[e] = 0.0;
  }
  __shared__ __align__(8) uint64_t xbar[2];
  if (tid == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(
          static_cast<unsigned>(__cvta_generic_to_shared(&xbar[b]))));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  cluster_sync_all();  // the peer's buffers and mbarriers exist before any remote store

  const AFragLane af(lane);
  const double* pbase = reinterpret_cast<const double*>(ps) + size_t(af.di) * 2 * SP + 2 * af.dj + af.comp;
  const unsigned vb_peer0 = mapa_shared(vb, peer), va_peer0 = mapa_shared(va, peer);
  const unsigned peer_bar0 = mapa_shared(&xbar[0], peer);
  // bytes the peer sends per step: its half's valid complex rows x 8 trajectories x 16 B
  const int prow0 = plan.lo[peer] * 4, prow1 = min(plan.hi[peer] * 4, CN);
  const unsigned in_bytes = unsigned(prow1 - prow0) * 8u * 16u;
  const signed char* ml = plan.mlist[rank][warp];
  const int nh = plan.nheavy[rank][warp], nl = plan.mcount[rank][warp] - nh;
  double* fin = va;
  switch (nh * 8 + nl) {  // kCombos: the only shapes make_plan() may choose
#define LBG_WARP(NH, NL) \
  case NH * 8 + NL:                                                                                            \
    fin = warp_steps<NH, NL>(pbase, ml, va, vb, va_peer0, vb_peer0, xbar, peer_bar0, in_bytes, lane, steps); \
    break;
    LBG_WARP(2, 0) LBG_WARP(2, 1) LBG_WARP(1, 1) LBG_WARP(0, 3) LBG_WARP(1, 2) LBG_WARP(0, 2)
#undef LBG_WARP
    default: __trap();
  }

  cluster_sync_all();  // no CTA exits while its peer may still address its shared memory
  // ---- write back: own slots; the shared slot by rank 0 ----
  for (int e = tid; e < SLOTS * 8 * 2 * CN; e += blockDim.x) {
    const int t = e / (2 * CN), r = e - t * 2 * CN;
    const int q = t >> 3;
    if (q == SLOTS - 1 && rank != 0) continue;
    const int64_t b = slot_tile(q) * 8 + (t & 7);
    if (b >= batch) continue;
    const double v = fin[t * SV + r];
    if (L == Layout::soa) {
      if (r & 1)
        x_im[b * CN + (r >> 1)] = v;
      else
        x_re[b * CN + (r >> 1)] = v;
    } else {
      x_aos[b * 2 * CN + r] = v;
    }
  }
}

// Per-warp (heavy, light) m-tile counts minimising the busiest sub-partition
// (heavy = 4 DMMAs per k-step, light = 3), found by exhaustive search over
// the 4-way compositions once on the host; then the m-tile ids are dealt out.
constexpr int kCombos[][2] = {{2, 0}, {2, 1}, {1, 1}, {0, 3}, {1, 2}, {0, 2}};
ClusterPlan make_plan() {
  ClusterPlan pl{};
  pl.k = 7;
  pl.h = 3;
  pl.shared = 1;
  pl.lo[0] = 0;
  pl.hi[0] = (CMT + 1) / 2;
  pl.lo[1] = (CMT + 1) / 2;
  pl.hi[1] = CMT;
  for (int r = 0; r < 2; ++r) {
    const int H = pl.hi[r] - pl.lo[r], Lc = CMT - H;
    constexpr int SM4 = 4;  // sub-partitions
    int best = 1 << 30, bh[SM4] = {}, bl[SM4] = {};
    int nh[SM4], nl[SM4];
    for (nh[0] = 0; nh[0] <= H; ++nh[0])
      for (nh[1] = 0; nh[0] + nh[1] <= H; ++nh[1])
        for (nh[2] = 0; nh[0] + nh[1] + nh[2] <= H; ++nh[2]) {
          nh[3] = H - nh[0] - nh[1] - nh[2];
          for (nl[0] = 0; nl[0] <= Lc; ++nl[0])
            for (nl[1] = 0; nl[0] + nl[1] <= Lc; ++nl[1])
              for (nl[2] = 0; nl[0] + nl[1] + nl[2] <= Lc; ++nl[2]) {
                nl[3] = Lc - nl[0] - nl[1] - nl[2];
                int worst = 0, ok = 1;
                for (int w = 0; w < SM4; ++w) {
                  // the two warps of the sub-partition split its list
                  const int a[2][2] = {{(nh[w] + 1) / 2, nl[w] / 2}, {nh[w] / 2, nl[w] - nl[w] / 2}};
                  for (auto& c2 : a) {
                    bool known = false;
                    for (auto& c : kCombos) known = known || (c[0] == c2[0] && c[1] == c2[1]);
                    if (!known || c2[0] + c2[1] > MAXM) ok = 0;
                  }
                  worst = std::max(worst, 4 * nh[w] + 3 * nl[w]);
                }
                if (ok && worst < best) {
                  best = worst;
                  std::copy(nh, nh + SM4, bh);
                  std::copy(nl, nl + SM4, bl);
                }
              }
        }
    if (best == (1 << 30)) throw invalid_argument("cluster plan: no balanced split");
    int mh = pl.lo[r], ml = 0;
    auto next_light = [&]() {
      while (ml >= pl.lo[r] && ml < pl.hi[r]) ++ml;
      return ml++;
    };
    for (int q = 0; q < SM4; ++q) {
      const int split[2][2] = {{(bh[q] + 1) / 2, bl[q] / 2}, {bh[q] / 2, bl[q] - bl[q] / 2}};
      for (int half = 0; half < 2; ++half) {
        const int w = q + 4 * half;  // warps q and q + 4 share sub-partition q
        for (int i = 0; i < split[half][0]; ++i) pl.mlist[r][w][pl.mcount[r][w]++] = static_cast<signed char>(mh++);
        pl.nheavy[r][w] = static_cast<signed char>(split[half][0]);
        for (int i = 0; i < split[half][1]; ++i)
          pl.mlist[r][w][pl.mcount[r][w]++] = static_cast<signed char>(next_light());
      }
    }
  }
  return pl;
}

const ClusterPlan& plan7() {
  static const ClusterPlan pl = make_plan();
  return pl;
}

}  // namespace

bool cluster_supported(std::size_t n) { return n == size_t(CN); }

// Critical paths in DMMA issue slots per sub-partition and step: K1b-C =
// waves x the busiest sub-partition's DMMAs per k-step x 41 k-steps; K1b =
// waves x 21 (3 warps x 7 m-tiles) x 41.
int64_t cluster_cost(std::size_t n, int64_t batch) {
  if (n != size_t(CN) || batch <= 0) return INT64_MAX;
  const int sms = sm_count();
  const int64_t nt = (batch + 7) / 8;
  const ClusterPlan& pl = plan7();
  int busiest = 0;
  for (int r = 0; r < 2; ++r)
    for (int q = 0; q < 4; ++q) {
      int load = 0;
      for (int w : {q, q + 4}) load += 4 * pl.nheavy[r][w] + 3 * (pl.mcount[r][w] - pl.nheavy[r][w]);
      busiest = std::max(busiest, load);
    }
  const int64_t clusters = (nt + 6) / 7, per_wave = std::max(1, sms / 2);
  return ((clusters + per_wave - 1) / per_wave) * busiest * CKT;
}
// Is the cluster kernel's critical path shorter than K1b's?
bool cluster_preferred(std::size_t n, int64_t batch) {
  return n == size_t(CN) && batch > 0 && cluster_cost(n, batch) < smem81_cost(batch);
}

void launch_smem_cluster(const double* p_dev, double* x_re, double* x_im, double* x_aos, int64_t batch,
                         int64_t steps, Layout layout, cudaStream_t s) {
  if (batch <= 0) return;
  const int64_t nt = (batch + 7) / 8;
  const int64_t clusters = (nt + 6) / 7;
  const ClusterPlan& pl = plan7();
  const double2* p2 = reinterpret_cast<const double2*>(p_dev);
  const dim3 grid(unsigned(2 * clusters));
  if (layout == Layout::soa) {
    ensure_max_dyn_smem((const void*)smem_cluster_kernel<Layout::soa>, int(SMEM_BYTES));
    smem_cluster_kernel<Layout::soa><<<grid, 32 * CWARPS, SMEM_BYTES, s>>>(p2, x_re, x_im, nullptr, batch, steps, pl);
  } else {
    ensure_max_dyn_smem((const void*)smem_cluster_kernel<Layout::aos>, int(SMEM_BYTES));
    smem_cluster_kernel<Layout::aos><<<grid, 32 * CWARPS, SMEM_BYTES, s>>>(p2, nullptr, nullptr, x_aos, batch, steps,
                                                                           pl);
  }
  LBG_CHECK_LAUNCH("smem_cluster_kernel");
}

}  // namespace lbg
