// common.cuh — shared device helpers for the sm_100a kernels.
//
// FP64 on sm_100a: tcgen05 has no f64 kind (ptxas rejects .kind::f64), so the
// FP64 tensor path is mma.sync ...f64 -> SASS DMMA.8x8x4 (measured 37.0 TF/s,
// profiles/r01_fp64_peaks.json; DFMA 34.1 TF/s).
//
// Complex GEMM on DMMA uses the exact real form of a complex product
// (no padding of the arithmetic, 4 real FMAs per complex MAC = 8 flops):
//   A'(2M x 2K):  A'[2i+a][2j+b] = a==b ? Re A_ij : (a==0 ? -Im A_ij : Im A_ij)
//   B'(2K x N):   B'[2j+b][n]    = b==0 ? Re B_jn : Im B_jn
//   C'(2M x N):   C'[2i+a][n]    = a==0 ? Re C_in : Im C_in
// With interleaved (AoS) complex storage B' and C' are the SAME bytes as B and
// C, so only the A fragment needs the sign/selection trick.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace lbg {

// ---- m8n8k4 f64 fragments (PTX ISA, mma.m8n8k4 .f64 layout) --------------
//   A (8x4 row): lane holds A[lane>>2][lane&3]
//   B (4x8 col): lane holds B[lane&3][lane>>2]
//   C (8x8):     lane holds C[lane>>2][2*(lane&3) + {0,1}]
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Per-lane constants of the real-form A fragment for complex storage.
struct AFragLane {
  int di;      // complex row offset within the m8 tile: lane >> 3        (0..3)
  int dj;      // complex col offset within the k4 step: (lane & 3) >> 1 (0..1)
  int comp;    // which double of the complex: ((lane >> 2) ^ lane) & 1
  unsigned hi_xor;  // 0x80000000 for (row re, col im): flips the sign bit (integer pipe)
  __device__ __forceinline__ AFragLane(int lane) {
    di = lane >> 3;
    dj = (lane & 3) >> 1;
    comp = ((lane >> 2) ^ lane) & 1;
    hi_xor = (((lane >> 2) & 1) == 0 && (lane & 1) == 1) ? 0x80000000u : 0u;
  }
  // apply the fragment sign without touching the FP64 pipe
  __device__ __forceinline__ double sign(double x) const {
    return __hiloint2double(__double2hiint(x) ^ int(hi_xor), __double2loint(x));
  }
};

// cp.async 16-byte copy global->shared, zero-filling when !pred.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Pair the two lanes of a C fragment that hold Re/Im of the same complex
// row (lane and lane^4), so each lane ends with one full complex value:
// lane with a==0 gets column 2t, lane with a==1 gets column 2t+1.
__device__ __forceinline__ double2 pair_complex(const double (&c)[2], int lane, int& col_off) {
  const int a = (lane >> 2) & 1;
  const double send = a ? c[0] : c[1];
  const double recv = __shfl_xor_sync(0xffffffffu, send, 4);
  col_off = 2 * (lane & 3) + a;
  return a ? make_double2(recv, c[1]) : make_double2(c[0], recv);
}


// Software grid barrier for cooperative (all-resident) launches: the arrival
// counter only grows (gridDim.x per barrier), so the target is compared
// wrap-safely — (int)(v - target) >= 0 stays correct after the 32-bit counter
// wraps (steps * grid >= 2^32), as long as fewer than 2^31 arrivals separate
// the fastest CTA from the target (one barrier's worth here).
__device__ __forceinline__ void grid_barrier_sync(unsigned int* bar, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // release-add after the CTA barrier (cumulativity carries the other warps'
    // stores; no full membar), acquire poll (no trailing fence needed)
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar) : "memory");
    while (true) {
      unsigned int v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
      if (int(v - target) >= 0) break;
    }
  }
  __syncthreads();
}

// ---- thread-block cluster / DSMEM primitives (PTX) ----------------------------
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// shared::cluster address of `local` in the shared memory of CTA `peer`
__device__ __forceinline__ unsigned mapa_shared(const void* local, unsigned peer) {
  unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(local)), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(peer));
  return r;
}
// asynchronous remote store that counts its 16 bytes on the receiver's mbarrier
__device__ __forceinline__ void st_async_f64x2(unsigned addr, double2 v, unsigned remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(addr),
               "d"(v.x), "d"(v.y), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(bar))),
               "r"(bytes)
               : "memory");
}
// wait for phase `parity` of a CTA-local mbarrier whose transaction bytes are
// the peers' st.async stores: the stores complete on this mbarrier, so the
// default (CTA-scope acquire) wait orders the reads of the landed bytes; an
// .acquire.cluster wait compiles to a CCTL.IVALL (L1 invalidate) per poll,
// measured as 25% of the stall samples of K1b-K.
__device__ __forceinline__ void mbar_wait_parity_cluster(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          static_cast<unsigned>(__cvta_generic_to_shared(bar))),
      "r"(parity)
      : "memory");
}

}  // namespace lbg
