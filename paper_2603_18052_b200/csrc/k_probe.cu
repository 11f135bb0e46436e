// k_probe.cu — FP64 roofline denominators measured live on the current GPU.
// MEASURED_PEAKS.json carries HBM and bf16 peaks only, so bench.py calls
// lbg_fp64_peak() right before its timed region: a register-only DMMA loop
// (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4) and a DFMA loop (occupancy sweep),
// best of 3 by CUDA events. r02: DMMA 37.1, DFMA 36.8 TF/s at 1965 MHz; DMMA and
// DFMA share one FP64 pipe (tools/fp64_mixed.cu: any mix tops out at 36.9).
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "../../include/lbg.h"
#include "common.cuh"
#include "internal.hpp"

namespace lbg {
namespace {

__global__ void probe_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = k;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < 4; ++k) dmma(c[k], a, b);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 1234.5678) out[threadIdx.x] = s;
}

// 8 independent chains x 8 unrolled FMAs per loop trip with compile-time
// coefficients, so ptxas feeds the multiplier from a uniform register (DFMA R,
// R, UR, R) as the dfma9 stepper does: r02 measured 36.5-36.8 TF/s that way at
// one 512-thread CTA per SM (tools/fp64_mixed.cu), against 33.4-34.1 when all
// three operands come from the register file (runtime a, b).
__global__ void probe_dfma(double* out, int iters, double, double) {
  constexpr double a = 0.999, b = 1e-3;
  double acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], a, b);
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c];
  if (s == 1234.5678) out[threadIdx.x] = s;
}

// shared-memory read bandwidth: conflict-free 128-bit loads from a 32 KB buffer
__global__ void probe_lds(double* out, int iters) {
  __shared__ double2 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double2 v = buf[(idx + u * 64) & 2047];
      acc.x += v.x;
      acc.y += v.y;
    }
    idx = (idx + 37) & 2047;
  }
  if (acc.x == 12345.678) out[threadIdx.x] = acc.x + acc.y;
}

// L2 read bandwidth: an L2-resident buffer read repeatedly past L1 (ld.global.cg)
__global__ void probe_l2(const double2* __restrict__ src, size_t n, int reps, double* out) {
  double2 acc = make_double2(0, 0);
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      const double2 v = __ldcg(src + i);
      acc.x += v.x;
      acc.y += v.y;
    }
  if (acc.x == 12345.678) out[threadIdx.x] = acc.x + acc.y;
}

// HBM copy bandwidth (read + write bytes), buffers far larger than L2
__global__ void probe_copy(const double2* __restrict__ src, double2* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(dst + i, __ldcs(src + i));
}

}  // namespace
}  // namespace lbg

// The B200 ladder in the reference's 4-level machine-profile shape
// (roofline.hpp:27-36): L1 <- shared memory per SM, L2 <- L2, L3 <- HBM,
// DRAM <- host memory over PCIe (pinned H2D). Every figure is measured here.
extern "C" int lbg_measure_machine_profile(lbg_machine_profile* out) {
  using namespace lbg;
  if (!out) return LBG_EINVAL;
  try {
    std::memset(out, 0, sizeof *out);
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "device");
    cudaDeviceProp prop{};
    check_cuda(cudaGetDeviceProperties(&prop, dev), "properties");
    std::snprintf(out->name, sizeof out->name, "%.40s (%d SMs, sm_%d%d)", prop.name, prop.multiProcessorCount,
                  prop.major, prop.minor);
    double dmma = 0, dfma = 0;
    if (lbg_fp64_peak(&dmma, &dfma) != LBG_OK) throw cuda_error("fp64 peak probe failed");
    out->peak_gflops = std::max(dmma, dfma) * 1e3;
    cudaEvent_t e0, e1;
    check_cuda(cudaEventCreate(&e0), "event");
    check_cuda(cudaEventCreate(&e1), "event");
    auto best_ms = [&](auto launch) {
      float best = 1e30f;
      for (int r = 0; r < 4; ++r) {
        check_cuda(cudaEventRecord(e0), "record");
        launch();
        check_cuda(cudaEventRecord(e1), "record");
        check_cuda(cudaEventSynchronize(e1), "sync");
        float ms = 0;
        check_cuda(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
        if (r > 0) best = std::min(best, ms);
      }
      return double(best);
    };
    double* junk = nullptr;
    check_cuda(cudaMalloc(&junk, 1 << 16), "malloc");
    const int sms = sm_count();
    {  // shared memory
      const int blocks = sms * 4, threads = 512, iters = 4096;
      const double ms = best_ms([&] { probe_lds<<<blocks, threads>>>(junk, iters); });
      out->bandwidth_gbs[0] = 16.0 * 8 * double(iters) * blocks * threads / (ms * 1e-3) / 1e9;
    }
    {  // L2 (32 MB resident buffer)
      const size_t n = (size_t(32) << 20) / 16;
      double2* src = nullptr;
      check_cuda(cudaMalloc(&src, n * 16), "malloc");
      check_cuda(cudaMemset(src, 0, n * 16), "memset");
      const int reps = 20;
      const double ms = best_ms([&] { probe_l2<<<sms * 8, 512>>>(src, n, reps, junk); });
      out->bandwidth_gbs[1] = 16.0 * n * reps / (ms * 1e-3) / 1e9;
      cudaFree(src);
    }
    {  // HBM: copy 1 GiB -> 1 GiB
      const size_t n = (size_t(1) << 30) / 16;
      double2 *a = nullptr, *b = nullptr;
      check_cuda(cudaMalloc(&a, n * 16), "malloc");
      check_cuda(cudaMalloc(&b, n * 16), "malloc");
      check_cuda(cudaMemset(a, 0, n * 16), "memset");
      const double ms = best_ms([&] { probe_copy<<<sms * 8, 512>>>(a, b, n); });
      out->bandwidth_gbs[2] = 2.0 * 16.0 * n / (ms * 1e-3) / 1e9;
      cudaFree(a);
      cudaFree(b);
    }
    {  // host memory over PCIe: pinned H2D, 256 MiB
      const size_t bytes = size_t(256) << 20;
      void* h = nullptr;
      void* d = nullptr;
      check_cuda(cudaMallocHost(&h, bytes), "malloc host");
      check_cuda(cudaMalloc(&d, bytes), "malloc");
      std::memset(h, 0, bytes);
      const double ms = best_ms([&] { check_cuda(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice), "H2D"); });
      out->bandwidth_gbs[3] = double(bytes) / (ms * 1e-3) / 1e9;
      cudaFree(d);
      cudaFreeHost(h);
    }
    check_cuda(cudaGetLastError(), "probe");
    cudaFree(junk);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    out->capacity_bytes[0] = uint64_t(prop.sharedMemPerMultiprocessor);
    out->capacity_bytes[1] = uint64_t(prop.l2CacheSize);
    out->capacity_bytes[2] = uint64_t(prop.totalGlobalMem);
    return LBG_OK;
  } catch (const std::exception&) {
    return LBG_ECUDA;
  }
}

extern "C" int lbg_fp64_peak(double* dmma_tflops, double* dfma_tflops) {
  using namespace lbg;
  try {
    double* out = nullptr;
    check_cuda(cudaMalloc(&out, 4096), "malloc");
    cudaEvent_t e0, e1;
    check_cuda(cudaEventCreate(&e0), "event");
    check_cuda(cudaEventCreate(&e1), "event");
    const int blocks = sm_count() * 4, threads = 256, iters = 2048;
    auto best_of = [&](auto launch, double flops) {
      float best = 1e30f;
      for (int r = 0; r < 4; ++r) {
        check_cuda(cudaEventRecord(e0), "record");
        launch();
        check_cuda(cudaEventRecord(e1), "record");
        check_cuda(cudaEventSynchronize(e1), "sync");
        float ms = 0;
        check_cuda(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
        if (r > 0) best = std::min(best, ms);  // first launch is warm-up
      }
      return flops / (best * 1e-3) / 1e12;
    };
    *dmma_tflops = best_of([&] { probe_dmma<<<blocks, threads>>>(out, iters); },
                           2.0 * 256 * 16.0 * iters * blocks * (threads / 32));
    // occupancy sweep (r02: 4 x 256 threads per SM read 33.4-34.1 TF/s, below the 35.2 the
    // dfma9 stepper reaches; one 512-thread CTA per SM reads ~36.8, tools/fp64_mixed.cu)
    double best = 0.0;
    for (const int bpsm : {1, 2, 4}) {
      const int tb = bpsm == 1 ? 512 : 256, nb = sm_count() * bpsm;
      best = std::max(best, best_of([&] { probe_dfma<<<nb, tb>>>(out, iters, 0.999, 1e-3); },
                                    2.0 * 64 * double(iters) * nb * tb));
    }
    *dfma_tflops = best;
    check_cuda(cudaGetLastError(), "probe");
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return LBG_OK;
  } catch (const std::exception&) {
    return LBG_ECUDA;
  }
}
