// k_ksplit.cu — K1b-K: the shared-P stepper for n = 81 (config 2) at SMALL
// batches: the per-GPU share of config 2 when 4,096 trajectories are sharded
// over 2 / 4 / 8 GPUs (2,048 / 1,024 / 512 trajectories).
//
// K1b / K1b-C give a CTA (or a 2-CTA cluster) whole n-tiles of 8 trajectories
// and ALL 81 rows of P. 512 trajectories are 64 n-tiles: at 4 (K1b) or 3.5
// (K1b-C) n-tiles per SM only 16-19 of 148 SMs work, so the step time does not
// shrink with the batch (measured: 7.0 ms per pass at 4,096, 2,048, 1,024 and
// 512 trajectories). Here every n-tile is shared by a 2-CTA cluster that SPLITS
// THE K DIMENSION: CTA r owns the complex columns / rows [40 r, 40 r + 40 + r)
// of the state — its "half" — and computes the partial products of ALL output
// rows over its half of the columns:
//   y_r = P[:, half_r] x[half_r].
// The half of y_r that belongs to the peer's rows is sent with st.async into
// the peer's partial buffer (DSMEM; the bytes complete on the peer's mbarrier),
// the own half is kept in registers, the peer's partial is added when it has
// landed, and the sum is the CTA's half of the next state — exactly the
// columns it needs for the next step, so the state never leaves the CTA.
//
// Per CTA and step: 20 m-tiles (8 real rows; complex rows 0..79) x 20 / 21
// k-steps (rank 0: complex columns 0..39; rank 1: 40..80, the last k-step
// holding column 80 and one zero column) x G n-tiles DMMAs, spread over the 4
// SM sub-partitions as exactly 5 m-tiles each (two warps per sub-partition;
// every warp computes its m-tiles of the PEER's rows first and ships them,
// then its own rows, so the transfer overlaps the own half of the step).
// Complex row 80 (real rows 160 / 161, a 21st m-tile would be 75% padding) is
// a DFMA dot product on warps 4..7 (two trajectories of each n-tile per warp,
// 16 k-slices per trajectory, shuffle-reduced). P's A fragments for the CTA's columns stay in REGISTERS
// for the whole kernel (<= 63 doubles per lane): no shared-memory traffic for
// P, only the state's B fragments (LDS.64, stride 84 = 4 mod 16 doubles:
// conflict-free).
//
// G n-tiles per cluster (1..4) with G = ceil(n-tiles / (SMs / 2)):
// 512 trajectories -> G = 1 on 64 clusters (128 SMs), 1,024 -> G = 2,
// 2,048 -> G = 4 (64 clusters). The per-step critical path is 5 G x 21 DMMAs
// per sub-partition (K1b-C at 4,096: 19 x 41).
//
// Synchronisation per step: one mbarrier per step parity receives the peer's
// partial (expect_tx by thread 0, complete_tx by the peer's st.async), then
// one CTA barrier publishes the new half-state. The peer cannot run two steps
// ahead (its step s + 1 needs this CTA's step s + 1 partial), so two partial
// buffers (by step parity) suffice.
//
// Replaces step_soa_kernel (proj/src/kernels_variants.cpp:26-41) inside
// evolve (proj/src/propagate.cpp:85-92), batched over trajectories.
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "internal.hpp"

namespace lbg {
namespace {

constexpr int KN = 81;      // n (config 2)
constexpr int KHALF = 40;   // complex rows / columns of rank 0's half (rank 1: 41)
constexpr int KSV = 84;     // doubles per trajectory row of a half-state (>= 82, = 4 mod 16)
constexpr int KPB = 42;     // complex rows per trajectory in a partial buffer
constexpr int KWARPS = 8;   // warps 0..3 own rows, 4..7 the peer's rows (+ row 80)
constexpr int KMAXG = 4;    // n-tiles per cluster

__host__ __device__ constexpr size_t ks_v_bytes(int G) { return size_t(8) * G * KSV * 8; }
__host__ __device__ constexpr size_t ks_pb_bytes(int G) { return size_t(8) * G * KPB * 16; }
__host__ __device__ constexpr size_t ks_smem_bytes(int G) {
  return 2 * ks_v_bytes(G) + 2 * ks_pb_bytes(G) + KPB * 16 + 16;
}

// Warp roles. Every warp first computes m-tiles of the PEER's rows and ships
// them, then m-tiles of its own rows, so the DSMEM transfer overlaps the own
// half of the step. Sub-partition q (warps q and q + 4) takes 3 remote + 2 own
// m-tiles for q < 2 and 2 + 3 for q >= 2 (5 each): warps 0, 1 = (2 remote, 1
// own), warps 2, 3 = (1, 2), warps 4..7 = (1, 1) + complex row 80.
//   remote m-tiles (of the peer's 10): SMSP offsets 0, 3, 6, 8
//   own m-tiles (of the CTA's 10):     SMSP offsets 0, 2, 4, 7
__device__ __forceinline__ int ks_nr(int w) { return w < 2 ? 2 : 1; }
__device__ __forceinline__ int ks_no(int w) { return (w == 2 || w == 3) ? 2 : 1; }
__device__ __forceinline__ int ks_r0(int w) {
  const int q = w & 3, base = q == 0 ? 0 : q == 1 ? 3 : q == 2 ? 6 : 8;
  return w < 4 ? base : base + ks_nr(q);
}
__device__ __forceinline__ int ks_o0(int w) {
  const int q = w & 3, base = q == 0 ? 0 : q == 1 ? 2 : q == 2 ? 4 : 7;
  return w < 4 ? base : base + ks_no(q);
}

struct KsCtx {
  const double2* p;     // P (n x n, AoS, global)
  double* va;           // current half-state  [8G][KSV]
  double* vb;           // next half-state
  double2* pb;          // local partial buffers [2][8G][KPB]
  unsigned pb_peer;     // the peer's partial buffers (shared::cluster)
  uint64_t* xbar;       // [2] mbarriers (step parity)
  unsigned bar_peer;    // the peer's xbar[0] (shared::cluster)
  unsigned in_bytes;    // bytes the peer sends per step
  const double2* prow;  // P[80][own columns] (shared)
  int rank, warp, lane;
};

// A fragments of P (NM m-tiles from global m-tile m0) over this CTA's KS k-steps
template <int NM, int KS>
__device__ __forceinline__ void ks_load_a(const KsCtx& c, const AFragLane& af, int m0, double (&a)[NM][KS]) {
  const double* pd = reinterpret_cast<const double*>(c.p);
#pragma unroll
  for (int mi = 0; mi < NM; ++mi)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int row = 4 * (m0 + mi) + af.di, col = 2 * (KHALF / 2 * c.rank + ks) + af.dj;
      a[mi][ks] = col < KN ? af.sign(pd[2 * (row * KN + col) + af.comp]) : 0.0;
    }
}

// acc[mi][g] = sum over the KS k-steps of A(mi) x B(g). With one or two
// accumulator chains per warp the DMMAs would be latency-bound (a dependent
// DMMA issues every ~26 cycles, the pipe takes one per 16 per sub-partition),
// so even and odd k-steps then accumulate separately and are added at the end.
// B fragments come from BR (registers, preloaded for the step) when G == 1,
// else from the half-state in shared memory.
// hook(0) / hook(1) run after the DMMAs of k-steps 1 and KS / 2: the DFMA row
// 80 (loads + FMAs, then the shuffle reduction) is interleaved with the DMMA
// stream there, so its latency chain hides under the DMMA issue.
template <int NM, int KS, int G, class Hook>
__device__ __forceinline__ void ks_mma(const double (&a)[NM][KS], const double* __restrict__ vrow,
                                       const double (&br)[G == 1 ? KS : 1], double (&acc)[NM][G][2], Hook&& hook) {
  constexpr int NA = NM * G <= 2 ? 2 : 1;
  double ac[NA][NM][G][2];
#pragma unroll
  for (int h = 0; h < NA; ++h)
#pragma unroll
    for (int mi = 0; mi < NM; ++mi)
#pragma unroll
      for (int g = 0; g < G; ++g) ac[h][mi][g][0] = ac[h][mi][g][1] = 0.0;
  if constexpr (G == 1) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
      for (int mi = 0; mi < NM; ++mi) dmma(ac[ks % NA][mi][0], a[mi][ks], br[ks]);
      if (ks == 1) hook(0);
      if (ks == KS / 2) hook(1);
    }
  } else {
    double b_cur[G];
#pragma unroll
    for (int g = 0; g < G; ++g) b_cur[g] = vrow[g * 8 * KSV];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      double b_nxt[G];
      const int kn = ks + 1 < KS ? ks + 1 : ks;  // last iteration reloads (harmless)
#pragma unroll
      for (int g = 0; g < G; ++g) b_nxt[g] = vrow[g * 8 * KSV + 4 * kn];
#pragma unroll
      for (int mi = 0; mi < NM; ++mi)
#pragma unroll
        for (int g = 0; g < G; ++g) dmma(ac[ks % NA][mi][g], a[mi][ks], b_cur[g]);
#pragma unroll
      for (int g = 0; g < G; ++g) b_cur[g] = b_nxt[g];
      if (ks == 1) hook(0);
      if (ks == KS / 2) hook(1);
    }
  }
#pragma unroll
  for (int mi = 0; mi < NM; ++mi)
#pragma unroll
    for (int g = 0; g < G; ++g) {
      acc[mi][g][0] = ac[0][mi][g][0];
      acc[mi][g][1] = ac[0][mi][g][1];
      if (NA == 2) {
        acc[mi][g][0] += ac[NA - 1][mi][g][0];
        acc[mi][g][1] += ac[NA - 1][mi][g][1];
      }
    }
}

// One warp's step loop: NR m-tiles of the peer's rows from global m-tile r0,
// NO of the own rows from o0, KS k-steps (20 on rank 0, 21 on rank 1);
// FRINGE: also complex row 80 (warps 4..7).
template <int NR, int NO, int KS, int G, bool FRINGE>
__device__ __forceinline__ void ks_steps(const KsCtx& c, int r0, int o0, int64_t steps) {
  const int lane = c.lane, rank = c.rank;
  const AFragLane af(lane);
  double ar[NR][KS], ao[NO][KS];  // P stays in registers for the whole kernel
  ks_load_a<NR, KS>(c, af, r0, ar);
  ks_load_a<NO, KS>(c, af, o0, ao);
  const int peer_base = KHALF * (1 - rank), own_base = KHALF * rank;  // first complex row of each half
  const int f = c.warp - 4;                 // fringe trajectories 2 f, 2 f + 1 of each n-tile
  const int tsel = lane >> 4, ksl = lane & 15;
  const int cnt = KHALF + rank;             // own complex columns
  double* va = c.va;
  double* vb = c.vb;
#pragma unroll 1
  for (int64_t s = 0; s < steps; ++s) {
    const int par = int(s & 1);
    if (threadIdx.x == 0) mbar_expect_tx(&c.xbar[par], c.in_bytes);
    const double* vrow = va + (lane >> 2) * KSV + (lane & 3);
    double br[G == 1 ? KS : 1];  // G == 1: the step's B fragments, shared by both halves
    if constexpr (G == 1) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) br[ks] = vrow[4 * ks];
    }
    const unsigned pbar = c.bar_peer + unsigned(par) * 8u;
    // complex row 80 over the own columns (FRINGE warps): 16 k-slices per
    // trajectory (3 columns per lane, branch-free), then a 16-lane shuffle
    // reduction; rank 0 computes it inside its remote phase and ships it,
    // rank 1 (its owner) inside its own phase
    double fre[FRINGE ? G : 1], fim[FRINGE ? G : 1];
    auto fringe = [&](int phase) {
      if constexpr (FRINGE) {
        if (phase == 0) {
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const double* x = va + (g * 8 + 2 * f + tsel) * KSV;
            double r1 = 0.0, r2 = 0.0, i1 = 0.0, i2 = 0.0;
#pragma unroll
            for (int it = 0; it < 3; ++it) {
              const int jl = ksl + 16 * it;
              if (jl < cnt) {
                const double2 pr = c.prow[jl];
                const double xr = x[2 * jl], xi = x[2 * jl + 1];
                r1 = fma(pr.x, xr, r1);
                r2 = fma(-pr.y, xi, r2);
                i1 = fma(pr.y, xr, i1);
                i2 = fma(pr.x, xi, i2);
              }
            }
            fre[g] = r1 + r2;
            fim[g] = i1 + i2;
          }
        } else {
#pragma unroll
          for (int g = 0; g < G; ++g)
#pragma unroll
            for (int off = 8; off >= 1; off >>= 1) {
              fre[g] += __shfl_xor_sync(0xffffffffu, fre[g], off);
              fim[g] += __shfl_xor_sync(0xffffffffu, fim[g], off);
            }
        }
      }
    };
    auto none = [](int) {};
    {  // the peer's rows first: ship the partials (complete_tx on the peer's mbarrier)
      double acc[NR][G][2];
      if (rank == 0)
        ks_mma<NR, KS, G>(ar, vrow, br, acc, fringe);
      else
        ks_mma<NR, KS, G>(ar, vrow, br, acc, none);
#pragma unroll
      for (int mi = 0; mi < NR; ++mi)
#pragma unroll
        for (int g = 0; g < G; ++g) {
          int coff;
          const double2 z = pair_complex(acc[mi][g], lane, coff);
          const int i = 4 * (r0 + mi) + (lane >> 3) - peer_base;
          const int t = g * 8 + coff;
          st_async_f64x2(c.pb_peer + unsigned(((par * 8 * G + t) * KPB + i) * 16), z, pbar);
        }
      if (FRINGE && rank == 0 && ksl == 0) {  // row 80 belongs to rank 1 (its local row 40)
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int t = g * 8 + 2 * f + tsel;
          st_async_f64x2(c.pb_peer + unsigned(((par * 8 * G + t) * KPB + KHALF) * 16), make_double2(fre[g], fim[g]),
                         pbar);
        }
      }
    }
    double acc[NO][G][2];  // the own rows, while the partials travel
    if (rank == 1)
      ks_mma<NO, KS, G>(ao, vrow, br, acc, fringe);
    else
      ks_mma<NO, KS, G>(ao, vrow, br, acc, none);
    mbar_wait_parity_cluster(&c.xbar[par], unsigned((s >> 1) & 1));  // the peer's partial has landed
    const double2* pbl = c.pb + par * 8 * G * KPB;
#pragma unroll
    for (int mi = 0; mi < NO; ++mi)
#pragma unroll
      for (int g = 0; g < G; ++g) {
        int coff;
        const double2 z = pair_complex(acc[mi][g], lane, coff);
        const int i = 4 * (o0 + mi) + (lane >> 3) - own_base;
        const int t = g * 8 + coff;
        const double2 q = pbl[t * KPB + i];
        *reinterpret_cast<double2*>(vb + t * KSV + 2 * i) = make_double2(z.x + q.x, z.y + q.y);
      }
    if (FRINGE && rank == 1 && ksl == 0) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int t = g * 8 + 2 * f + tsel;
        const double2 q = pbl[t * KPB + KHALF];
        *reinterpret_cast<double2*>(vb + t * KSV + 2 * KHALF) = make_double2(fre[g] + q.x, fim[g] + q.y);
      }
    }
    __syncthreads();  // the new half-state is complete; the old one may be overwritten next step
    double* tmp = va;
    va = vb;
    vb = tmp;
  }
}

template <int KS, int G>
__device__ __forceinline__ void ks_dispatch_ks(const KsCtx& c, int64_t steps) {
  const int w = c.warp;
  const int r0 = 10 * (1 - c.rank) + ks_r0(w), o0 = 10 * c.rank + ks_o0(w);
  if (w < 2)
    ks_steps<2, 1, KS, G, false>(c, r0, o0, steps);
  else if (w < 4)
    ks_steps<1, 2, KS, G, false>(c, r0, o0, steps);
  else
    ks_steps<1, 1, KS, G, true>(c, r0, o0, steps);
}

template <int G>
__device__ __forceinline__ void ks_dispatch(const KsCtx& c, int64_t steps) {
  if (c.rank == 0)
    ks_dispatch_ks<20, G>(c, steps);
  else
    ks_dispatch_ks<21, G>(c, steps);
}

template <Layout L, int G>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32 * KWARPS, 1)
    ksplit_cluster_kernel(const double2* __restrict__ p, double* __restrict__ x_re, double* __restrict__ x_im,
                          double* __restrict__ x_aos, int64_t batch, int64_t steps) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* va = reinterpret_cast<double*>(smem);
  double* vb = reinterpret_cast<double*>(smem + ks_v_bytes(G));
  double2* pb = reinterpret_cast<double2*>(smem + 2 * ks_v_bytes(G));
  double2* prow = reinterpret_cast<double2*>(smem + 2 * ks_v_bytes(G) + 2 * ks_pb_bytes(G));
  uint64_t* xbar = reinterpret_cast<uint64_t*>(smem + 2 * ks_v_bytes(G) + 2 * ks_pb_bytes(G) + KPB * 16);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned rank = cluster_ctarank(), peer = rank ^ 1u;
  const int64_t b0 = int64_t(blockIdx.x >> 1) * G * 8;  // first trajectory of the cluster
  const int base = KHALF * int(rank), cnt = KHALF + int(rank);

  // ---- stage the own half of each state (real form), zero padding; P row 80 ----
  for (int e = tid; e < 8 * G * KSV; e += blockDim.x) {
    const int t = e / KSV, r = e - t * KSV;
    const int64_t b = b0 + t;
    double v = 0.0;
    if (b < batch && r < 2 * cnt) {
      const int64_t col = base + (r >> 1);
      if (L == Layout::soa)
        v = (r & 1) ? x_im[b * KN + col] : x_re[b * KN + col];
      else
        v = x_aos[(b * KN + col) * 2 + (r & 1)];
    }
    va[e] = v;
    vb[e] = 0.0;
  }
  for (int j = tid; j < KPB; j += blockDim.x) prow[j] = j < cnt ? p[80 * KN + base + j] : make_double2(0.0, 0.0);
  if (tid == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(
          static_cast<unsigned>(__cvta_generic_to_shared(&xbar[b]))));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  cluster_sync_all();  // the peer's buffers and mbarriers exist before any remote store

  KsCtx c;
  c.p = p;
  c.va = va;
  c.vb = vb;
  c.pb = pb;
  c.pb_peer = mapa_shared(pb, peer);
  c.xbar = xbar;
  c.bar_peer = mapa_shared(&xbar[0], peer);
  // bytes the peer sends per step: the rows this CTA owns x 8 G trajectories x 16 B
  c.in_bytes = unsigned(cnt) * 8u * G * 16u;
  c.prow = prow;
  c.rank = int(rank);
  c.warp = warp;
  c.lane = lane;
  ks_dispatch<G>(c, steps);
  double* fin = (steps & 1) ? vb : va;

  cluster_sync_all();  // no CTA exits while its peer may still address its shared memory
  // ---- write back the own half ----
  for (int e = tid; e < 8 * G * 2 * cnt; e += blockDim.x) {
    const int t = e / (2 * cnt), r = e - t * 2 * cnt;
    const int64_t b = b0 + t;
    if (b >= batch) continue;
    const double v = fin[t * KSV + r];
    const int64_t col = base + (r >> 1);
    if (L == Layout::soa) {
      if (r & 1)
        x_im[b * KN + col] = v;
      else
        x_re[b * KN + col] = v;
    } else {
      x_aos[(b * KN + col) * 2 + (r & 1)] = v;
    }
  }
}

template <int G>
void launch_g(const double* p_dev, double* x_re, double* x_im, double* x_aos, int64_t batch, int64_t steps,
              Layout layout, cudaStream_t s) {
  const int64_t nt = (batch + 7) / 8, clusters = (nt + G - 1) / G;
  const dim3 grid(unsigned(2 * clusters));
  const size_t smem = ks_smem_bytes(G);
  const double2* p2 = reinterpret_cast<const double2*>(p_dev);
  if (layout == Layout::soa) {
    ensure_max_dyn_smem((const void*)ksplit_cluster_kernel<Layout::soa, G>, int(smem));
    ksplit_cluster_kernel<Layout::soa, G><<<grid, 32 * KWARPS, smem, s>>>(p2, x_re, x_im, nullptr, batch, steps);
  } else {
    ensure_max_dyn_smem((const void*)ksplit_cluster_kernel<Layout::aos, G>, int(smem));
    ksplit_cluster_kernel<Layout::aos, G><<<grid, 32 * KWARPS, smem, s>>>(p2, nullptr, nullptr, x_aos, batch, steps);
  }
  LBG_CHECK_LAUNCH("ksplit_cluster_kernel");
}

}  // namespace

// n-tiles per cluster for a batch (0 = more than KMAXG: the kernel does not apply)
int ksplit_group(std::size_t n, int64_t batch) {
  if (n != size_t(KN) || batch <= 0) return 0;
  const int64_t nt = (batch + 7) / 8, clusters = std::max(1, sm_count() / 2);
  const int64_t g = (nt + clusters - 1) / clusters;
  return g <= KMAXG ? int(g) : 0;
}

bool ksplit_supported(std::size_t n) { return n == size_t(KN); }

// per-step critical path in DMMA issue slots per sub-partition (x 41 k-steps
// units for K1b / K1b-C): 5 m-tiles x G n-tiles x 21 k-steps (+ the DFMA row),
// weighted by 4/3: measured, this kernel issues its DMMAs at 67-70% of the pipe
// at every G (the two-phase step, the exchange, the 3-vs-2 m-tile warps)
// against K1b's 94%, so equal slot counts are not equal times.
int64_t ksplit_cost(std::size_t n, int64_t batch) {
  const int g = ksplit_group(n, batch);
  return g ? (int64_t(5) * g * 21 + 2 * g) * 4 / 3 : INT64_MAX;
}

void launch_ksplit(const double* p_dev, std::size_t n, double* x_re, double* x_im, double* x_aos, int64_t batch,
                   int64_t steps, Layout layout, cudaStream_t s) {
  if (batch <= 0) return;
  if (n != size_t(KN)) throw invalid_argument("ksplit kernel needs n == 81");
  const int64_t nt = (batch + 7) / 8;
  // with more n-tiles than 4 per cluster slot the kernel still runs (in waves)
  const int g = std::max(1, ksplit_group(n, batch) ? ksplit_group(n, batch)
                                                   : int(std::min<int64_t>(KMAXG, nt)));
  switch (g) {
    case 1: return launch_g<1>(p_dev, x_re, x_im, x_aos, batch, steps, layout, s);
    case 2: return launch_g<2>(p_dev, x_re, x_im, x_aos, batch, steps, layout, s);
    case 3: return launch_g<3>(p_dev, x_re, x_im, x_aos, batch, steps, layout, s);
    default: return launch_g<4>(p_dev, x_re, x_im, x_aos, batch, steps, layout, s);
  }
}

}  // namespace lbg
