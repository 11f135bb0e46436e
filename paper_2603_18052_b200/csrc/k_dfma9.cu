// k_dfma9.cu — K1a: shared-P batched propagation for n = d^2 = 9 (config 1).
//
// Regime (profiles/r01_fp64_peaks.json): 648 flops per
// trajectory-step on 144 B of state; far above the FP64 ridge, so the bound is
// the FP64 pipe. DMMA would pad the 18x18 real-form P to 24x20 (67.5% useful,
// <= 25 TF/s), so this kernel uses DFMA with P in the CONSTANT bank: ptxas
// lowers every P operand to a uniform register (LDCU.128 -> DFMA R, R, UR, R),
// one trajectory per thread keeps vec(rho) (18 doubles) in registers for all
// steps, and the only HBM traffic is one read and one write of the state.
// 324 DFMA per step = exactly the 8 d^4 = 648 algorithmic flops, no waste.
//
// Replaces the reference hot loop step_soa_kernel (proj/src/kernels_variants.cpp:26-41)
// driven by evolve (proj/src/propagate.cpp:85-92) for every trajectory.
#include <map>
#include <mutex>

#include "common.cuh"
#include "internal.hpp"

namespace lbg {

namespace {

constexpr int kSlots = 8;
__constant__ double2 c_p9[kSlots][81];

// SLOT is a template parameter so every P operand is a compile-time constant
// bank address (c[0x3][imm]) and ptxas keeps it out of the register file.
template <int SLOT, Layout L>
__global__ void __launch_bounds__(128) dfma9_kernel(double* __restrict__ x_re,
                                                    double* __restrict__ x_im,
                                                    double* __restrict__ x_aos, int64_t batch,
                                                    int64_t steps) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= batch) return;
  const double2* __restrict__ p = c_p9[SLOT];
  double vr[9], vi[9];
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    if (L == Layout::soa) {
      vr[j] = x_re[t * 9 + j];
      vi[j] = x_im[t * 9 + j];
    } else {
      const double2 z = reinterpret_cast<const double2*>(x_aos)[t * 9 + j];
      vr[j] = z.x;
      vi[j] = z.y;
    }
  }
  for (int64_t s = 0; s < steps; ++s) {
    double nr[9], ni[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      double ar = 0.0, ai = 0.0;
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        const double2 pij = p[i * 9 + j];
        ar = fma(pij.x, vr[j], ar);
        ar = fma(-pij.y, vi[j], ar);
        ai = fma(pij.x, vi[j], ai);
        ai = fma(pij.y, vr[j], ai);
      }
      nr[i] = ar;
      ni[i] = ai;
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      vr[i] = nr[i];
      vi[i] = ni[i];
    }
  }
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    if (L == Layout::soa) {
      x_re[t * 9 + j] = vr[j];
      x_im[t * 9 + j] = vi[j];
    } else {
      reinterpret_cast<double2*>(x_aos)[t * 9 + j] = make_double2(vr[j], vi[j]);
    }
  }
}

// Constant-bank slots: a slot is reused only after the kernel that last read
// it has finished (event wait), so concurrent streams never race on c_p9.
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

}  // namespace

void launch_dfma9(const double* /*unused*/, const double* p_dev, double* x_re, double* x_im,
                  double* x_aos, int64_t batch, int64_t steps, Layout layout, cudaStream_t s) {
  if (batch <= 0) return;
  SlotPool& sp = pool();
  std::lock_guard<std::mutex> lk(sp.mu);
  if (!sp.init) {
    for (auto& e : sp.ev) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    sp.init = true;
  }
  const int slot = sp.next;
  sp.next = (sp.next + 1) % kSlots;
  check_cuda(cudaStreamWaitEvent(s, sp.ev[slot], 0), "stream wait");
  check_cuda(cudaMemcpyToSymbolAsync(c_p9, p_dev, sizeof(double2) * 81,
                                     sizeof(double2) * 81 * slot, cudaMemcpyDeviceToDevice, s),
             "P -> constant bank");
  const int threads = 128;
  const unsigned blocks = static_cast<unsigned>((batch + threads - 1) / threads);
  switch (slot) {
#define LBG_SLOT(S)                                                                               \
  case S:                                                                                         \
    if (layout == Layout::soa)                                                                    \
      dfma9_kernel<S, Layout::soa><<<blocks, threads, 0, s>>>(x_re, x_im, nullptr, batch, steps); \
    else                                                                                          \
      dfma9_kernel<S, Layout::aos><<<blocks, threads, 0, s>>>(nullptr, nullptr, x_aos, batch, steps); \
    break;
    LBG_SLOT(0) LBG_SLOT(1) LBG_SLOT(2) LBG_SLOT(3) LBG_SLOT(4) LBG_SLOT(5) LBG_SLOT(6) LBG_SLOT(7)
#undef LBG_SLOT
  }
  LBG_CHECK_LAUNCH("dfma9_kernel");
  check_cuda(cudaEventRecord(sp.ev[slot], s), "event record");
}

}  // namespace lbg
