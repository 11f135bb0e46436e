// k_tiled.cu — K1c: shared-P propagation for any n with P streamed from L2
// (config 3: d = 27, n = 729, P = 8.5 MB, 1,024 trajectories, 200 steps), and
// the plain batched complex GEMM used by the GPU expm.
//
// One step is a complex GEMM  V_next (n x B) = P (n x n) * V (n x B).  P and both
// state buffers (2 x 12 MB at config 3) stay L2-resident (126 MB L2), so the
// bound is the DMMA pipe. The kernel is PERSISTENT (cooperative launch, all
// CTAs co-resident): per step a producer warp walks its CTA's stream-K range of
// (32x32 complex output tile, K chunk) iterations and streams each chunk into a
// 3-stage shared-memory ring with TWO 2-D tensor-map TMA copies (A box 32 rows
// x 34 complex, B box 32 rows x 36 complex: the box is 2 / 4 complex wider than
// the chunk so the TMA writes the padded, bank-conflict-free row strides
// directly; out-of-range rows / columns arrive zero-filled) signalled through
// mbarriers (complete_tx); the plain batched GEMM (expm) uses the same producer
// with the batch stacked as rows of one tensor. 8 consumer warps wait on the stage's "full" barrier, run the
// m8n8k4 DMMAs in real form (common.cuh), release the stage on its "empty"
// barrier and write finished tiles straight from registers to the other state
// buffer. No block-wide barrier in the main loop; one grid barrier per step
// (every output row needs every input row).
//
// Tile: 32 complex rows (64 real, 8 m-tiles) x 32 columns (4 n-tiles), K chunk
// 16 complex (8 k-steps); each consumer warp owns 2 m-tiles x 2 n-tiles.
// Shared strides SA = 2 (mod 8), SB = 4 (mod 8) complex make every fragment load
// bank-conflict free. Ragged edges are masked in registers (no smem zeroing).
//
// Replaces step_soa_kernel (proj/src/kernels_variants.cpp:26-41) inside
// evolve (proj/src/propagate.cpp:85-92), batched; the GEMM replaces
// lb::matmul (proj/src/complex_matrix.cpp:30-56) inside expm.
#include <cuda.h>  // CUtensorMap (driver types only; the encoder comes via cudaGetDriverEntryPoint)

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <map>
#include <mutex>

#include "common.cuh"
#include "internal.hpp"

namespace lbg {

namespace {

constexpr int BM = 32, BK = 32, STAGES = 2;  // default ring depth
constexpr int CWARPS = 8;  // default consumer warps (Geo<..., CW_>)
constexpr int SA = BK + 2;  // complex stride of A rows: 2 (mod 8), see header

// Tile geometry by tile width BN (complex columns): 32 for the expm GEMM, 16 for
// the stepper (twice the tiles per step -> half the step-tail granularity).
// Each consumer warp owns MI m8-tiles x NI n8-tiles; the 8 warps form a
// WM x WN grid. SB = BN + 4 = 4 (mod 8) keeps B fragment loads conflict free.
// REAL: the same engine on real matrices (density mode beyond n = 84): 64-row
// x BN tiles, K chunk 32, A stride 36 = 4 (mod 16) and B stride BN + 8 =
// 8 (mod 16) doubles (conflict-free m8n8k4 fragments), the same byte size per
// stage as the complex geometry.
template <int BN_, bool REAL_ = false, int BK_ = BK, int ST_ = STAGES, int CW_ = CWARPS, int BMC_ = BM,
          bool KS_ = false, int NI_ = 2>
struct Geo {
  static constexpr int ST = ST_;  // ring stages
  static constexpr int CW = CW_, NT = 32 * (CW_ + 1);  // consumer warps, threads (+ producer warp)
  static constexpr bool REAL = REAL_;
  // KS: warps w and w + CW / 2 compute the same output block over the even / odd
  // k-steps of every chunk and add at the end of the tile (exact-fit geometry)
  static constexpr bool KS = KS_;
  static constexpr int CWE = KS ? CW / 2 : CW;     // warps of the output grid
  static constexpr int CPX = REAL ? 1 : 2;         // doubles per element
  static constexpr int BMg = REAL ? 64 : BMC_;     // rows per tile
  static constexpr int BKg = BK_;                  // K chunk (elements)
  static constexpr int SAg = REAL ? BKg + 4 : SA;  // A row stride (elements)
  static constexpr int BN = BN_, NI = NI_, WN = BN_ / (8 * NI), WM = CWE / WN;
  static constexpr int MI = (REAL ? BMg / 8 : BMg / 4) / WM;
  static constexpr int SB = REAL ? BN_ + 8 : BN_ + 4;  // B row stride (elements)
  static constexpr int A_ELEMS = BMg * SAg * CPX / 2, B_ELEMS = BKg * SB * CPX / 2;  // double2 units
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t XCH_ELEMS = KS ? size_t(CWE) * 32 * MI * NI : 0;  // k-parity handoff (double2)
  static constexpr size_t kSmemBytes = size_t(ST) * STAGE_ELEMS * sizeof(double2) + 256 + XCH_ELEMS * 16;
  static_assert(WN * WM == CWE && MI * WM * (REAL ? 8 : 4) == BMg, "tile geometry");
  static_assert(!KS || (!REAL && CW % 2 == 0), "k-parity split: complex tiles, warp pairs");
  static_assert(REAL || BK_ == BK, "complex tiles use the global K chunk (SA and the B box follow BK)");
};

// ---- mbarrier / bulk-copy primitives (PTX) ----------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
#ifdef LBG_DEBUG_WATCHDOG
  {
    const long long t0 = clock64();
    while (true) {
      unsigned ok;
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(ok)
          : "r"(smem_u32(bar)), "r"(parity)
          : "memory");
      if (ok) return;
      if (clock64() - t0 > 4000000000ll) {
        printf("WATCHDOG block %d thread %d bar_off %u parity %u\n", blockIdx.x, threadIdx.x,
               smem_u32(bar) & 0xffffu, parity);
        return;
      }
    }
  }
#endif
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 2-D tensor-map TMA: box at coordinates {c0 (innermost, doubles), c1 (rows)}
__device__ __forceinline__ void tma_g2s_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

struct Ring {
  double2* data;   // STAGES x (A | B)
  uint64_t* full;  // STAGES
  uint64_t* empty; // STAGES
  int* hdr;        // STAGES x 4: tile id (-1 = end of step), k chunk, segment [lo, hi] chunks
  double2* xch;    // KS geometries: the odd-k warps' accumulators at the end of a tile
};

template <class G>
__device__ __forceinline__ Ring carve(unsigned char* smem) {
  Ring r;
  r.data = reinterpret_cast<double2*>(smem);
  unsigned char* tail = smem + size_t(G::ST) * G::STAGE_ELEMS * sizeof(double2);
  r.full = reinterpret_cast<uint64_t*>(tail);
  r.empty = r.full + G::ST;
  r.hdr = reinterpret_cast<int*>(r.empty + G::ST);
  r.xch = reinterpret_cast<double2*>(smem + size_t(G::ST) * G::STAGE_ELEMS * sizeof(double2) + 256);
  return r;
}

struct Problem {  // C (M x N) = A (M x K) * B (K x N), complex row-major
  const double2* A;
  long long lda;
  const double2* B;
  long long ldb;
  double2* C;
  long long ldc;
  int M, N, K;
};

template <int NST>
__device__ __forceinline__ void advance(int& stage, unsigned& phase) {
  if (++stage == NST) {
    stage = 0;
    phase ^= 1u;
  }
}

// Producer: one warp streams iterations [it0, it1) of the flattened
// (tile, K chunk) space into the ring (stream-K: a CTA's range may start or end
// inside a tile; the header tells the consumers which part of the tile it is).
// Same iteration space, one elected lane, two 2-D TMA copies per chunk. The
// boxes are SA / SB complex wide, so each smem row lands at the padded stride;
// rows >= M and columns >= K / N are zero-filled by the TMA unit.
template <class G>
__device__ __forceinline__ void produce_range_tma(const Ring& r, const Problem& p, const CUtensorMap* map_a,
                                                  const CUtensorMap* map_b, int tiles_m, long long it0,
                                                  long long it1, int& stage, unsigned& phase, int lane,
                                                  int a_row0 = 0, int b_row0 = 0) {
  constexpr int BN = G::BN, STAGE_ELEMS = G::STAGE_ELEMS;
  constexpr unsigned kBytes = unsigned(STAGE_ELEMS) * 16u;  // full boxes, OOB fill included
  constexpr int BK = G::BKg;
  const int nk = (p.K + BK - 1) / BK;
  for (long long it = it0; it < it1; ++it) {
    const int t = int(it / nk), kc = int(it - (long long)t * nk);
    const int m0 = (t % tiles_m) * G::BMg, n0 = (t / tiles_m) * BN;
    const long long tb = (long long)t * nk;
    const int lo = int(max(it0 - tb, 0ll)), hi = int(min(it1 - 1 - tb, (long long)nk - 1));
    mbar_wait(&r.empty[stage], phase ^ 1u);
    if (lane == 0) {
      double2* as = r.data + stage * STAGE_ELEMS;
      r.hdr[4 * stage] = t;
      r.hdr[4 * stage + 1] = kc;
      r.hdr[4 * stage + 2] = lo;
      r.hdr[4 * stage + 3] = hi;
      mbar_arrive_tx(&r.full[stage], kBytes);
      tma_g2s_2d(as, map_a, G::CPX * kc * BK, a_row0 + m0, &r.full[stage]);
      tma_g2s_2d(as + G::A_ELEMS, map_b, G::CPX * n0, b_row0 + kc * BK, &r.full[stage]);
    }
    __syncwarp();
    advance<G::ST>(stage, phase);
  }
}

template <class G>
__device__ __forceinline__ void produce_end(const Ring& r, int& stage, unsigned& phase, int lane) {
  mbar_wait(&r.empty[stage], phase ^ 1u);
  if (lane == 0) {
    r.hdr[4 * stage] = -1;
    mbar_arrive(&r.full[stage]);
  }
  advance<G::ST>(stage, phase);
}

// Producer for the exact-fit geometries (one whole tile per CTA and step, the
// same chunk sequence every step): the A parts (P, never written) of the next
// step's first chunks are issued as soon as their ring slots free up, BEFORE the
// grid barrier; after it only their B parts (the new state) remain to be
// issued. The slot's full barrier expects both (one expect_tx), so the
// consumers see no difference. npre_in: chunks of this step whose A part is
// already in flight (issued at the end of the previous step).
template <class G>
__device__ __forceinline__ int produce_tile_prefetch(const Ring& r, const Problem& p, const CUtensorMap* map_a,
                                                     const CUtensorMap* map_b, int tiles_m, int tile, int npre_in,
                                                     bool prefetch_next, int& stage, unsigned& phase,
                                                     int& pre_stage, unsigned& pre_phase, int lane) {
  constexpr int BN = G::BN, STAGE_ELEMS = G::STAGE_ELEMS, BK = G::BKg;
  constexpr unsigned kBytes = unsigned(STAGE_ELEMS) * 16u;
  const int nk = (p.K + BK - 1) / BK;
  const int m0 = (tile % tiles_m) * G::BMg, n0 = (tile / tiles_m) * BN;
  if (npre_in > 0) {  // back to the first slot that already holds this step's A part
    stage = pre_stage;
    phase = pre_phase;
  }
  for (int kc = 0; kc < nk; ++kc) {
    double2* as = r.data + stage * STAGE_ELEMS;
    if (kc >= npre_in) {
      mbar_wait(&r.empty[stage], phase ^ 1u);
      if (lane == 0) {
        r.hdr[4 * stage] = tile;
        r.hdr[4 * stage + 1] = kc;
        r.hdr[4 * stage + 2] = 0;
        r.hdr[4 * stage + 3] = nk - 1;
        mbar_arrive_tx(&r.full[stage], kBytes);
        tma_g2s_2d(as, map_a, G::CPX * kc * BK, m0, &r.full[stage]);
      }
    }
    if (lane == 0) tma_g2s_2d(as + G::A_ELEMS, map_b, G::CPX * n0, kc * BK, &r.full[stage]);
    __syncwarp();
    advance<G::ST>(stage, phase);
  }
  produce_end<G>(r, stage, phase, lane);
  if (!prefetch_next) return 0;
  const int npre = nk < G::ST ? nk : G::ST;
  pre_stage = stage;
  pre_phase = phase;
  for (int kc = 0; kc < npre; ++kc) {  // next step: header, expect_tx and the A part now
    mbar_wait(&r.empty[stage], phase ^ 1u);
    if (lane == 0) {
      double2* as = r.data + stage * STAGE_ELEMS;
      r.hdr[4 * stage] = tile;
      r.hdr[4 * stage + 1] = kc;
      r.hdr[4 * stage + 2] = 0;
      r.hdr[4 * stage + 3] = nk - 1;
      mbar_arrive_tx(&r.full[stage], kBytes);
      tma_g2s_2d(as, map_a, G::CPX * kc * BK, m0, &r.full[stage]);
    }
    __syncwarp();
    advance<G::ST>(stage, phase);
  }
  return npre;
}


// Consumer warps: run tiles until the end-of-step sentinel.
// Split tiles (stream-K): a tile cut between CTAs' ranges has a HEAD part
// (chunks from 0), possibly MIDDLE parts (a CTA whose whole range lies inside
// the tile) and a TAIL part (chunks up to nk-1). A TAIL or MIDDLE CTA reaches
// its part at the START of its range and publishes it (its own partial slot +
// epoch flag: a CTA publishes at most once per step); the HEAD CTA reaches its
// part at the END of its range, adds the published partials of the CTAs after
// it in CTA order (fixed order: deterministic) and stores the tile.
struct SplitK {
  double2* part;          // gridDim.x x (CW x 32 lanes x MI x NI) accumulator slots
  unsigned int* flags;    // gridDim.x, = epoch when that CTA's partial is published
  unsigned int epoch;
  long long work;         // (tile, K chunk) iterations per step
};
// the CTA whose stream-K range [work c / G, work (c+1) / G) holds iteration x
__device__ __forceinline__ unsigned cta_of_iter(long long x, long long work) {
  return unsigned(((x + 1) * (long long)gridDim.x - 1) / work);
}
template <int NTHREADS>
__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(NTHREADS) : "memory"); }

template <class G>
__device__ __forceinline__ void consume(const Ring& r, const Problem& p, int tiles_m, int& stage,
                                       unsigned& phase, int warp, int lane, const SplitK* sk) {
  constexpr int BN = G::BN, SB = G::SB, STAGE_ELEMS = G::STAGE_ELEMS, MI = G::MI, NI = G::NI;
  constexpr int BK = G::BKg;
  const AFragLane af(lane);
  const int wsub = G::KS ? warp % G::CWE : warp, kpar = G::KS ? warp / G::CWE : 0;
  const int wm = wsub / G::WN, wn = wsub % G::WN;
  const int nk = (p.K + BK - 1) / BK;
  const int gq = lane >> 2, tq = lane & 3;
  // fragment bases in doubles: complex real-form (common.cuh) or plain real
  const int a_off = G::REAL ? (wm * MI * 8 + gq) * G::SAg + tq
                            : 2 * ((wm * MI * 4 + af.di) * SA + af.dj) + af.comp;
  const int b_off = G::REAL ? tq * SB + wn * NI * 8 + gq
                            : 2 * (((lane & 3) >> 1) * SB + wn * NI * 8 + (lane >> 2)) + (lane & 1);
  double acc[MI][NI][2] = {};
  int m0 = 0, n0 = 0;
  while (true) {
    mbar_wait(&r.full[stage], phase);
    const int tile = r.hdr[4 * stage], kc = r.hdr[4 * stage + 1];
    const int lo = r.hdr[4 * stage + 2], hi = r.hdr[4 * stage + 3];
    if (tile < 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&r.empty[stage]);
      advance<G::ST>(stage, phase);
      return;
    }
    if (kc == lo) {
      m0 = (tile % tiles_m) * G::BMg;
      n0 = (tile / tiles_m) * BN;
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    }
    const double* ad = reinterpret_cast<const double*>(r.data + stage * STAGE_ELEMS) + a_off;
    const double* bd = reinterpret_cast<const double*>(r.data + stage * STAGE_ELEMS + G::A_ELEMS) + b_off;
    // rows >= M and k >= K arrive zero-filled by the TMA (the tensor maps end at
    // M rows / K columns of A and K rows of B): no masking in the inner loop
    if constexpr (G::REAL) {
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        double a[MI], b[NI];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) a[mi] = ad[mi * 8 * G::SAg + 4 * ks];
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) b[ni] = bd[4 * ks * SB + ni * 8];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
      }
    } else {
#pragma unroll
      for (int k2 = 0; k2 < BK / (G::KS ? 4 : 2); ++k2) {
        const int ks = G::KS ? 2 * k2 + kpar : k2;
        double a[MI], b[NI];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) a[mi] = af.sign(ad[2 * (mi * 4 * SA) + 4 * ks]);
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) b[ni] = bd[2 * (2 * ks * SB + ni * 8)];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&r.empty[stage]);
    advance<G::ST>(stage, phase);
    if (kc != hi) continue;
    if constexpr (G::KS) {  // odd-k warps hand their accumulators to the even-k warps
      double2* x = r.xch + (wsub * 32 + lane) * MI * NI;
      if (kpar)
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) x[mi * NI + ni] = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      consumer_bar<32 * G::CW>();
      if (kpar) {
        consumer_bar<32 * G::CW>();  // the xch slots are reused by the next tile
        continue;  // (KS geometries run one whole tile per CTA: no stream-K parts)
      }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          const double2 v = x[mi * NI + ni];
          acc[mi][ni][0] += v.x;
          acc[mi][ni][1] += v.y;
        }
      consumer_bar<32 * G::CW>();
    }
    constexpr int SLOT = G::CW * 32 * MI * NI;
    if (sk && lo > 0) {  // TAIL / MIDDLE part: publish the partial accumulators
      double2* dst = sk->part + (long long)blockIdx.x * SLOT;
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
          __stcg(dst + ((warp * MI + mi) * NI + ni) * 32 + lane, make_double2(acc[mi][ni][0], acc[mi][ni][1]));
      consumer_bar<32 * G::CW>();
      if (warp == 0 && lane == 0)  // release store: cumulative over the warps' partials (consumer barrier)
        asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(sk->flags + blockIdx.x), "r"(sk->epoch)
                     : "memory");
      continue;
    }
    if (sk && hi < nk - 1) {  // HEAD part: add the later parts' partials in CTA order, then store
      const unsigned c_last = cta_of_iter((long long)(tile + 1) * nk - 1, sk->work);
      if (warp == 0 && lane == 0) {
        for (unsigned c = blockIdx.x + 1; c <= c_last; ++c)
          while (true) {
            unsigned v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(sk->flags + c) : "memory");
            if (v == sk->epoch) break;
          }
      }
      consumer_bar<32 * G::CW>();
      // partials of up to kBatch contributors are loaded together (one L2
      // round trip per batch), then added in CTA order
      constexpr int kBatch = 4;
      for (unsigned c0 = blockIdx.x + 1; c0 <= c_last; c0 += kBatch) {
        double2 q[kBatch][MI][NI];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
          const double2* src = sk->part + (long long)(c0 + j) * SLOT;
#pragma unroll
          for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
              q[j][mi][ni] = c0 + j <= c_last ? __ldcg(src + ((warp * MI + mi) * NI + ni) * 32 + lane)
                                              : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int j = 0; j < kBatch; ++j)
          if (c0 + j <= c_last) {
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
              for (int ni = 0; ni < NI; ++ni) {
                acc[mi][ni][0] += q[j][mi][ni].x;
                acc[mi][ni][1] += q[j][mi][ni].y;
              }
          }
      }
    }
    if constexpr (G::REAL) {  // tile done: registers -> global (row g, columns 2t, 2t+1)
      double* C = reinterpret_cast<double*>(p.C);
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          const int i = m0 + (wm * MI + mi) * 8 + gq;
          const int col = n0 + (wn * NI + ni) * 8 + 2 * tq;
          if (i < p.M) {
            if (col < p.N) C[(long long)i * p.ldc + col] = acc[mi][ni][0];
            if (col + 1 < p.N) C[(long long)i * p.ldc + col + 1] = acc[mi][ni][1];
          }
        }
    } else {  // tile done: registers -> global
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          int coff;
          const double2 z = pair_complex(acc[mi][ni], lane, coff);
          const int i = m0 + (wm * MI + mi) * 4 + (lane >> 3);
          const int col = n0 + (wn * NI + ni) * 8 + coff;
          if (i < p.M && col < p.N) p.C[(long long)i * p.ldc + col] = z;
        }
    }
  }
}

template <class G>
__device__ __forceinline__ void init_ring(const Ring& r) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < G::ST; ++s) {
      mbar_init(&r.full[s], 1);
      mbar_init(&r.empty[s], G::CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
}

// ---- plain batched GEMM (expm): one tile per CTA -----------------------------
// A batch of matrices with stride n*n is one tensor of n*batch rows (stride 0:
// n rows); a box reaching past row n of matrix b reads rows of matrix b+1 —
// A rows >= n only feed outputs that are never stored, and B rows k >= n meet
// A columns k >= n, which the TMA zero-fills — so the product is exact.
// G complex (zgemm) or REAL (dgemm on matrices with leading dimension ld; the
// batch strides sa / sb / sc are in elements)
template <class G>
__global__ void __launch_bounds__(G::NT) gemm_kernel(const double2* __restrict__ A,
                                                       const double2* __restrict__ B,
                                                       double2* __restrict__ C, int n, int ld,
                                                       long long sa, long long sb, long long sc,
                                                       const __grid_constant__ CUtensorMap map_a,
                                                       const __grid_constant__ CUtensorMap map_b,
                                                       const int* __restrict__ cond, int cond_idx) {
  const int b = blockIdx.z, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // element offsets in units of double2: complex element = 1, real element = 1/2
  auto off = [&](long long e) { return G::REAL ? e / 2 : e; };
  if (cond && cond_idx >= *cond) {  // device-decided no-op product: C = A on this CTA's tile
    const int tm = (n + G::BMg - 1) / G::BMg, t = blockIdx.y * tm + blockIdx.x;
    const int m0 = (t % tm) * G::BMg, n0 = (t / tm) * G::BN;
    const double* src = reinterpret_cast<const double*>(A + off(b * sa));
    double* dst = reinterpret_cast<double*>(C + off(b * sc));
    constexpr int W = G::CPX;  // doubles per element
    for (int e = threadIdx.x; e < G::BMg * G::BN * W; e += blockDim.x) {
      const int i = m0 + e / (G::BN * W), jd = n0 * W + e % (G::BN * W);
      if (i < n && jd < n * W) dst[(long long)i * ld * W + jd] = src[(long long)i * ld * W + jd];
    }
    return;
  }
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const Ring r = carve<G>(smem_raw);
  init_ring<G>(r);
  const Problem p{A + off(b * sa), ld, B + off(b * sb), ld, C + off(b * sc), ld, n, n, n};
  const int tiles_m = (n + G::BMg - 1) / G::BMg;
  const int tile = blockIdx.y * tiles_m + blockIdx.x;
  int stage = 0;
  unsigned phase = 0;
  if (warp == G::CW) {
    const long long nk = (n + G::BKg - 1) / G::BKg;
    produce_range_tma<G>(r, p, &map_a, &map_b, tiles_m, tile * nk, (tile + 1) * nk, stage, phase, lane,
                         sa ? b * n : 0, sb ? b * n : 0);
    produce_end<G>(r, stage, phase, lane);
  } else {
    consume<G>(r, p, tiles_m, stage, phase, warp, lane, nullptr);
  }
}

// ---- persistent stepping ----------------------------------------------------
// 32-wide tiles: 16-wide halves the step-tail granularity but doubles the
// row copies per MMA and measured 2x slower at config 3 (copy-issue bound).
using StepGeo = Geo<32>;
// Exact-fit geometry for small batches: 20 complex rows (5 m-tiles) x 32
// trajectories, warp pair (w, w + 4) on n-tile w splitting the k-steps by
// parity, 4 stages (127 KB: one CTA per SM). At c3's 8-GPU share (n = 729,
// 128 trajectories) that is 37 x 4 = 148 tiles: one whole tile per SM per step,
// no stream-K parts and no fixups (the default 32 x 32 tiles: 92 tiles split
// several ways over 148 CTAs, the HEADs waiting on their contributors).
using StepGeoX = Geo<32, false, BK, 4, 8, 20, true, 1>;
using StepGeoR = Geo<32, true, 64>;  // real arithmetic (density mode); measured: <64,true,32> 11.2, <64,true,64> 8.34, this 8.32 ms at c3
struct StepCtl {
  unsigned int tile_ctr[2];
  unsigned int barrier;
  unsigned int pad;
};


template <class G>
__global__ void __launch_bounds__(G::NT) tiled_evolve_kernel(const double2* __restrict__ P, int n,
                                                               double2* v0, double2* v1,
                                                               int batch, int ldv, int64_t steps,
                                                               StepCtl* ctl, double2* part,
                                                               unsigned int* flags,
                                                               unsigned long long* trace,
                                                               const __grid_constant__ CUtensorMap map_p,
                                                               const __grid_constant__ CUtensorMap map_v0,
                                                               const __grid_constant__ CUtensorMap map_v1) {
  constexpr int BN = G::BN;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const Ring r = carve<G>(smem_raw);
  init_ring<G>(r);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = (n + G::BMg - 1) / G::BMg, tiles_n = (batch + BN - 1) / BN;
  const int ntiles = tiles_m * tiles_n;
  double2* cur = v0;
  double2* nxt = v1;
  int stage = 0;
  unsigned phase = 0;
  // stream-K: this CTA's fixed, contiguous share of the step's (tile, K chunk)
  // iterations; with grid > ntiles (small batches) a tile is split across
  // several CTAs (HEAD + MIDDLE + TAIL parts)
  const long long nk = (n + G::BKg - 1) / G::BKg, work = (long long)ntiles * nk;
  const long long it0 = work * blockIdx.x / gridDim.x, it1 = work * (blockIdx.x + 1) / gridDim.x;
  // trace (measurement only, LBG_TILED_TRACE): %globaltimer per step and CTA at
  // the step start and when each warp leaves its role, first kTraceSteps steps
  constexpr int kTraceSteps = 64;
  auto stamp = [&](int64_t s, int slot) {
    if (trace && s < kTraceSteps && lane == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[((size_t)s * gridDim.x + blockIdx.x) * (G::CW + 2) + slot] = t;
    }
  };
  int npre = 0;  // exact-fit producer: chunks of the step whose A part is already in flight,
  int pre_stage = 0;  // starting at this ring slot / phase
  unsigned pre_phase = 0;
  for (int64_t s = 0; s < steps; ++s) {
    const Problem p{P, n, cur, ldv, nxt, ldv, n, batch, n};
    if (warp == 0) stamp(s, 0);
    if (warp == G::CW) {
      // generic-proxy stores of the previous step -> async-proxy (bulk copy) reads
      asm volatile("fence.proxy.async.global;\n" ::: "memory");
      if constexpr (G::KS) {  // exact fit: it0 / it1 cover exactly the tile blockIdx.x
        npre = produce_tile_prefetch<G>(r, p, &map_p, (s & 1) ? &map_v1 : &map_v0, tiles_m, int(blockIdx.x), npre,
                                        s + 1 < steps, stage, phase, pre_stage, pre_phase, lane);
      } else {
        produce_range_tma<G>(r, p, &map_p, (s & 1) ? &map_v1 : &map_v0, tiles_m, it0, it1, stage, phase, lane);
        produce_end<G>(r, stage, phase, lane);
      }
      stamp(s, G::CW + 1);
    } else {
      const SplitK sk{part, flags, unsigned(s + 1), work};
      consume<G>(r, p, tiles_m, stage, phase, warp, lane, &sk);
      stamp(s, 1 + warp);
    }
    grid_barrier_sync(&ctl->barrier, unsigned(s + 1) * gridDim.x);
    double2* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
}

// layout conversion between the user's [b][k] (SoA / AoS) and V[k][b] (AoS)
template <Layout L, bool ToV>
__global__ void convert_kernel(double* x_re, double* x_im, double* x_aos, double2* v, int n,
                               int batch) {
  __shared__ double2 tile[32][33];
  const int kb = blockIdx.x * 32, bb = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  if (ToV) {
    for (int r = ty; r < 32; r += 8) {  // read x[b = bb + r][k = kb + tx]
      const int b = bb + r, k = kb + tx;
      double2 z = make_double2(0.0, 0.0);
      if (b < batch && k < n) {
        if (L == Layout::soa)
          z = make_double2(x_re[(long long)b * n + k], x_im[(long long)b * n + k]);
        else
          z = reinterpret_cast<const double2*>(x_aos)[(long long)b * n + k];
      }
      tile[r][tx] = z;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {  // write v[k = kb + r][b = bb + tx]
      const int k = kb + r, b = bb + tx;
      if (k < n && b < batch) v[(long long)k * batch + b] = tile[tx][r];
    }
  } else {
    for (int r = ty; r < 32; r += 8) {  // read v[k = kb + r][b = bb + tx]
      const int k = kb + r, b = bb + tx;
      tile[r][tx] = (k < n && b < batch) ? v[(long long)k * batch + b] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {  // write x[b = bb + r][k = kb + tx]
      const int b = bb + r, k = kb + tx;
      if (b < batch && k < n) {
        const double2 z = tile[tx][r];
        if (L == Layout::soa) {
          x_re[(long long)b * n + k] = z.x;
          x_im[(long long)b * n + k] = z.y;
        } else {
          reinterpret_cast<double2*>(x_aos)[(long long)b * n + k] = z;
        }
      }
    }
  }
}

template <bool ToV>
void convert(double* x_re, double* x_im, double* x_aos, double2* v, int n, int batch,
             Layout layout, cudaStream_t s) {
  const dim3 grid((n + 31) / 32, (batch + 31) / 32), block(32, 8);
  if (layout == Layout::soa)
    convert_kernel<Layout::soa, ToV><<<grid, block, 0, s>>>(x_re, x_im, x_aos, v, n, batch);
  else
    convert_kernel<Layout::aos, ToV><<<grid, block, 0, s>>>(x_re, x_im, x_aos, v, n, batch);
  LBG_CHECK_LAUNCH("convert_kernel");
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    check_cuda(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q),
               "cuTensorMapEncodeTiled entry point");
    if (q != cudaDriverEntryPointSuccess || !p) throw cuda_error("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// rows x cols complex row-major matrix viewed as FP64 [rows][2 cols]; the box
// is box_rows x box_cplx complex (box_cplx may exceed the chunk: padded stride)
CUtensorMap complex_map(const double2* base, size_t rows, size_t cols, unsigned box_rows, unsigned box_cplx) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(2 * cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(cols * sizeof(double2))};
  const cuuint32_t box[2] = {cuuint32_t(2 * box_cplx), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult rc = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double2*>(base), dims,
                                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(rc)) + ")");
  return m;
}

}  // namespace

int sm_count() {
  static std::mutex mu;
  static std::map<int, int>* counts = new std::map<int, int>;
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(mu);
  int& c = (*counts)[dev];
  if (c == 0) check_cuda(cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev), "sm count");
  return c;
}

template <class G>
size_t ntiles_of(size_t n, int64_t batch) {
  return ((n + G::BMg - 1) / G::BMg) * ((size_t(batch) + G::BN - 1) / G::BN);
}
template <class G>
constexpr size_t slot_of() {  // double2 per split tile
  return size_t(G::CW) * 32 * G::MI * G::NI;
}
// real rows must be 16-byte aligned for the TMA: even leading dimensions
inline size_t even(size_t x) { return x + (x & 1); }
template <class G>
size_t ldv_of(int64_t batch) {
  return G::REAL ? even(size_t(batch)) : size_t(batch);
}
// Persistent grid of the stepping engine. With at least as many tiles as
// resident slots (occupancy x SMs): every slot, stream-K splitting a tile
// between at most two CTAs. With fewer tiles (small batches: c3 at 128
// trajectories = 92 tiles): one CTA per SM and several-way tile splits (HEAD +
// MIDDLE + TAIL parts) instead of idle SMs — 1 CTA / SM measured 4.8 vs 5.0 ms
// for 3 / SM at c3 B = 128 (the three CTAs of an SM progress unevenly and the
// HEADs wait for the slowest contributor). With fewer iterations than
// kMinItersPerCta per SM: one CTA per tile, a whole multiple of the SM count
// when there are at least as many tiles as SMs.
template <class G>
int tiled_grid_of(size_t n, int64_t batch) {
  const auto kern = tiled_evolve_kernel<G>;
  ensure_max_dyn_smem((const void*)kern, int(G::kSmemBytes));
  int occ = 0;
  check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G::NT, G::kSmemBytes), "occupancy");
  const int sms = sm_count(), slots = std::max(1, occ * sms);
  const long long nt = (long long)ntiles_of<G>(n, batch), nk = ((long long)n + G::BKg - 1) / G::BKg;
  if constexpr (G::KS) return int(nt);  // exact fit: one whole tile per CTA (use_exact_fit: nt <= SMs)
  constexpr long long kMinItersPerCta = 3;
  int grid;
  if (nt >= slots) {
    grid = slots;
  } else if (nt < sms && nt * nk >= kMinItersPerCta * sms) {
    grid = sms;
  } else {
    grid = int(nt);
    if (grid >= sms) grid -= grid % sms;
  }
  return std::max(1, grid);
}
template <class G>
size_t aux_workspace_of(size_t n, int64_t batch) {
  const size_t g = size_t(tiled_grid_of<G>(n, batch));
  return align_up(sizeof(StepCtl)) + align_up(g * slot_of<G>() * sizeof(double2)) + align_up(g * sizeof(unsigned int));
}
template <class G>
size_t workspace_of(size_t n, int64_t batch) {
  const size_t vbytes = size_t(G::CPX) * 8 * n * ldv_of<G>(batch);
  return 2 * align_up(vbytes) + aux_workspace_of<G>(n, batch);
}

// the exact-fit geometry when its tiles fill 90-100% of the SMs and the default
// tiles would have to be split (fewer tiles than SMs)
bool use_exact_fit(size_t n, int64_t batch) {
  const long long sms = sm_count(), t = (long long)ntiles_of<StepGeoX>(n, batch);
  return t <= sms && 10 * t >= 9 * sms && (long long)ntiles_of<StepGeo>(n, batch) < sms;
}

size_t tiled_workspace(size_t n, int64_t batch) {
  return use_exact_fit(n, batch) ? std::max(workspace_of<StepGeo>(n, batch), workspace_of<StepGeoX>(n, batch))
                                 : workspace_of<StepGeo>(n, batch);
}
size_t tiled_real_workspace(size_t n, int64_t batch) {
  return workspace_of<StepGeoR>(n, batch) + align_up(8 * n * even(n));  // + an even-stride copy of P_R
}

// rows x cols real row-major matrix with leading dimension ld (even); box box_rows x box_cols
CUtensorMap real_map(const double* base, size_t rows, size_t cols, size_t ld, unsigned box_rows, unsigned box_cols) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(ld * sizeof(double))};
  const cuuint32_t box[2] = {cuuint32_t(box_cols), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult rc = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled failed (" + std::to_string(int(rc)) + ")");
  return m;
}

// real state layout conversion: x[b][k] (batch x n) <-> V[k][b]
template <bool ToV>
__global__ void convert_real_kernel(double* __restrict__ x, double* __restrict__ v, int n, int batch, int ldv) {
  __shared__ double tile[32][33];
  const int kb = blockIdx.x * 32, bb = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  if (ToV) {
    for (int r = ty; r < 32; r += 8) {
      const int b = bb + r, k = kb + tx;
      tile[r][tx] = (b < batch && k < n) ? x[(long long)b * n + k] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
      const int k = kb + r, b = bb + tx;
      if (k < n && b < batch) v[(long long)k * ldv + b] = tile[tx][r];
    }
  } else {
    for (int r = ty; r < 32; r += 8) {
      const int k = kb + r, b = bb + tx;
      tile[r][tx] = (k < n && b < batch) ? v[(long long)k * ldv + b] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
      const int b = bb + r, k = kb + tx;
      if (b < batch && k < n) x[(long long)b * n + k] = tile[tx][r];
    }
  }
}

// the persistent stream-K engine on caller-given state buffers: v0 holds V_0,
// step s reads V_s and writes V_{s+1} into the other buffer (v1 after an odd
// count). aux: aux_workspace_of<G>(n, batch) bytes.
template <class G>
void run_tiled_ext(const double* p_dev, size_t ldp, size_t n, int64_t batch, int64_t steps, double2* v0, double2* v1,
                   void* aux, cudaStream_t s) {
  const size_t ldv = ldv_of<G>(batch);
  StepCtl* ctl = static_cast<StepCtl*>(aux);
  const int grid = tiled_grid_of<G>(n, batch);
  double2* part = reinterpret_cast<double2*>(reinterpret_cast<char*>(ctl) + align_up(sizeof(StepCtl)));
  unsigned int* flags = reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(part) +
                                                        align_up(size_t(grid) * slot_of<G>() * sizeof(double2)));
  check_cuda(cudaMemsetAsync(flags, 0, size_t(grid) * sizeof(unsigned int), s), "memset flags");
  check_cuda(cudaMemsetAsync(ctl, 0, sizeof(StepCtl), s), "memset ctl");
  if (steps <= 0) return;
  const auto kern = tiled_evolve_kernel<G>;
  const double2* p2 = reinterpret_cast<const double2*>(p_dev);
  int ni = int(n), bi = int(batch), li = int(ldv);
  int64_t st = steps;
  // A = P (n x n), B = the state V[k][b] (n x batch); boxes BMg x SAg and BK x SB elements
  CUtensorMap map_p, map_v0, map_v1;
  if constexpr (G::REAL) {
    map_p = real_map(p_dev, n, n, ldp, G::BMg, G::SAg);
    map_v0 = real_map(reinterpret_cast<const double*>(v0), n, size_t(batch), ldv, G::BKg, G::SB);
    map_v1 = real_map(reinterpret_cast<const double*>(v1), n, size_t(batch), ldv, G::BKg, G::SB);
  } else {
    map_p = complex_map(p2, n, n, G::BMg, SA);
    map_v0 = complex_map(v0, n, size_t(batch), BK, G::SB);
    map_v1 = complex_map(v1, n, size_t(batch), BK, G::SB);
  }
  static const char* trace_path = std::getenv("LBG_TILED_TRACE");  // measurement only
  unsigned long long* trace = nullptr;
  const size_t trace_n = size_t(64) * grid * (G::CW + 2);
  if (trace_path) {
    check_cuda(cudaMalloc(&trace, trace_n * 8), "trace");
    check_cuda(cudaMemsetAsync(trace, 0, trace_n * 8, s), "trace");
  }
  void* args[] = {(void*)&p2,    (void*)&ni,    (void*)&v0,    (void*)&v1,     (void*)&bi,
                  (void*)&li,    (void*)&st,    (void*)&ctl,   (void*)&part,   (void*)&flags,
                  (void*)&trace, (void*)&map_p, (void*)&map_v0, (void*)&map_v1};
  check_cuda(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(G::NT), args, G::kSmemBytes, s),
             "tiled_evolve_kernel (cooperative)");
  note_launch();
  if (trace) {
    std::vector<unsigned long long> h(trace_n);
    check_cuda(cudaMemcpyAsync(h.data(), trace, trace_n * 8, cudaMemcpyDeviceToHost, s), "trace");
    check_cuda(cudaStreamSynchronize(s), "trace");
    cudaFree(trace);
    if (FILE* f = std::fopen(trace_path, "wb")) {
      const int hdr[3] = {grid, G::CW + 2, int(std::min<int64_t>(steps, 64))};
      std::fwrite(hdr, sizeof hdr, 1, f);
      std::fwrite(h.data(), 8, trace_n, f);
      std::fclose(f);
    }
  }
}

template <class G>
void run_tiled(const double* p_dev, size_t ldp, size_t n, int64_t batch, int64_t steps, void* work, cudaStream_t s) {
  char* w = static_cast<char*>(work);
  const size_t vbytes = size_t(G::CPX) * 8 * n * ldv_of<G>(batch);
  run_tiled_ext<G>(p_dev, ldp, n, batch, steps, reinterpret_cast<double2*>(w),
                   reinterpret_cast<double2*>(w + align_up(vbytes)), w + 2 * align_up(vbytes), s);
}

void launch_tiled_evolve(const double* p_dev, size_t n, double* x_re, double* x_im, double* x_aos,
                         int64_t batch, int64_t steps, Layout layout, void* work, cudaStream_t s) {
  if (batch <= 0) return;
  if (batch > (1ll << 30) || n > (1u << 20)) throw invalid_argument("tiled: shape too large");
  if (!work) throw invalid_argument("tiled: workspace required");
  double2* v0 = reinterpret_cast<double2*>(work);
  double2* v1 = reinterpret_cast<double2*>(static_cast<char*>(work) + align_up(sizeof(double2) * n * size_t(batch)));
  const int ni = int(n), bi = int(batch);
  convert<true>(x_re, x_im, x_aos, v0, ni, bi, layout, s);
  static const bool no_fit = std::getenv("LBG_TILED_NO_EXACT_FIT") != nullptr;  // A/B only
  if (!no_fit && use_exact_fit(n, batch))
    run_tiled<StepGeoX>(p_dev, n, n, batch, steps, work, s);
  else
    run_tiled<StepGeo>(p_dev, n, n, batch, steps, work, s);
  convert<false>(x_re, x_im, x_aos, (steps & 1) ? v1 : v0, ni, bi, layout, s);
}

// real: x (batch x n real, [b][k]) stepped in place by the real n x n P_R
void launch_tiled_evolve_real(const double* p_dev, size_t n, double* x, int64_t batch, int64_t steps, void* work,
                              cudaStream_t s) {
  if (batch <= 0) return;
  if (batch > (1ll << 30) || n > (1u << 20)) throw invalid_argument("tiled: shape too large");
  if (!work) throw invalid_argument("tiled: workspace required");
  const size_t ldv = ldv_of<StepGeoR>(batch), ldp = even(n);
  double* v0 = static_cast<double*>(work);
  double* v1 = reinterpret_cast<double*>(static_cast<char*>(work) + align_up(8 * n * ldv));
  const double* pt = p_dev;
  if (ldp != n) {  // odd n: an even-stride copy of P_R (TMA rows are 16-byte aligned)
    double* pp = reinterpret_cast<double*>(static_cast<char*>(work) + workspace_of<StepGeoR>(n, batch));
    check_cuda(cudaMemsetAsync(pp, 0, 8 * n * ldp, s), "memset");
    check_cuda(cudaMemcpy2DAsync(pp, ldp * 8, p_dev, n * 8, n * 8, n, cudaMemcpyDeviceToDevice, s), "P_R copy");
    pt = pp;
  }
  const int ni = int(n), bi = int(batch), li = int(ldv);
  const dim3 grid((ni + 31) / 32, (bi + 31) / 32), block(32, 8);
  convert_real_kernel<true><<<grid, block, 0, s>>>(x, v0, ni, bi, li);
  LBG_CHECK_LAUNCH("convert_real_kernel");
  run_tiled<StepGeoR>(pt, ldp, n, batch, steps, work, s);
  convert_real_kernel<false><<<grid, block, 0, s>>>(x, (steps & 1) ? v1 : v0, ni, bi, li);
  LBG_CHECK_LAUNCH("convert_real_kernel");
}

void launch_zgemm(const double* a, const double* b, double* c, int n, int batch, long long stride_a,
                  long long stride_b, long long stride_c, cudaStream_t s) {
  ensure_max_dyn_smem((const void*)gemm_kernel<Geo<32>>, int(Geo<32>::kSmemBytes));
  const long long nn = (long long)n * n;
  if ((stride_a != 0 && stride_a != nn) || (stride_b != 0 && stride_b != nn))
    throw invalid_argument("zgemm: batch strides must be 0 or n*n");
  const dim3 grid((n + BM - 1) / BM, (n + Geo<32>::BN - 1) / Geo<32>::BN, batch);
  const CUtensorMap map_a = complex_map(reinterpret_cast<const double2*>(a), size_t(n) * (stride_a ? batch : 1),
                                        size_t(n), BM, SA);
  const CUtensorMap map_b = complex_map(reinterpret_cast<const double2*>(b), size_t(n) * (stride_b ? batch : 1),
                                        size_t(n), BK, Geo<32>::SB);
  gemm_kernel<Geo<32>><<<grid, Geo<32>::NT, Geo<32>::kSmemBytes, s>>>(reinterpret_cast<const double2*>(a),
                                                                   reinterpret_cast<const double2*>(b),
                                                                   reinterpret_cast<double2*>(c), n, n, stride_a,
                                                                   stride_b, stride_c, map_a, map_b, nullptr, 0);
  LBG_CHECK_LAUNCH("zgemm_kernel");
}

// one complex GEMM C = A B (n x n, AoS, C distinct from A and B) on the
// persistent stream-K engine: a single product has n/32 x n/32 tiles, which
// one-tile-per-CTA launches quantise into partial waves (n = 729: 529 tiles on
// 444 slots = 2 waves at 60%); stream-K spreads them evenly.
size_t zgemm_stream_workspace(int n) { return aux_workspace_of<StepGeo>(size_t(n), n); }
void launch_zgemm_stream(const double* a, const double* b, double* c, int n, void* aux, cudaStream_t s) {
  run_tiled_ext<StepGeo>(a, size_t(n), size_t(n), n, 1, reinterpret_cast<double2*>(const_cast<double*>(b)),
                         reinterpret_cast<double2*>(c), aux, s);
}

// real batched GEMM C[b] = A[b] B[b] (n x n, leading dimension ld even, batch
// strides 0 or n*ld doubles)
void launch_dgemm(const double* a, const double* b, double* c, int n, int ld, int batch, long long stride_a,
                  long long stride_b, long long stride_c, cudaStream_t s, const int* cond, int cond_idx) {
  using G = StepGeoR;
  ensure_max_dyn_smem((const void*)gemm_kernel<G>, int(G::kSmemBytes));
  const long long nl = (long long)n * ld;
  if ((ld & 1) || ld < n) throw invalid_argument("dgemm: leading dimension must be even and >= n");
  if ((stride_a != 0 && stride_a != nl) || (stride_b != 0 && stride_b != nl) || (stride_c & 1))
    throw invalid_argument("dgemm: batch strides must be 0 or n*ld");
  const dim3 grid((n + G::BMg - 1) / G::BMg, (n + G::BN - 1) / G::BN, batch);
  const CUtensorMap map_a = real_map(a, size_t(n) * (stride_a ? batch : 1), size_t(n), size_t(ld), G::BMg, G::SAg);
  const CUtensorMap map_b = real_map(b, size_t(n) * (stride_b ? batch : 1), size_t(n), size_t(ld), G::BKg, G::SB);
  gemm_kernel<G><<<grid, G::NT, G::kSmemBytes, s>>>(reinterpret_cast<const double2*>(a),
                                                      reinterpret_cast<const double2*>(b),
                                                      reinterpret_cast<double2*>(c), n, ld, stride_a, stride_b,
                                                      stride_c, map_a, map_b, cond, cond_idx);
  LBG_CHECK_LAUNCH("dgemm_kernel");
}

}  // namespace lbg
