// Do DMMA (mma.sync f64) and DFMA share one FP64 pipe on B200 (sm_100a)?
// One CTA per SM, 16 warps; warps with (warp / 4) < ndmma run a register-only
// DMMA loop, the others a register-only DFMA loop. If the pipes were separate,
// the mixed run would take max(T_dmma, T_dfma); if shared, about the sum.
// Prints one JSON line per layout.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mixed fp64_mixed.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); std::exit(1);} } while (0)

__device__ __forceinline__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) { c[k][0] = k; c[k][1] = -k; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// role per warp: warp w -> group g = w / 4 (each group has one warp per SMSP).
// groups [0, ndmma) run DMMA, groups [ndmma, ndmma + ndfma) DFMA, the rest idle.
__global__ void mixed(double* out, int ndmma, int ndfma, int it_dmma, int it_dfma) {
  int g = (threadIdx.x >> 5) >> 2;
  if (g < ndmma) dmma_loop(out, it_dmma);
  else if (g < ndmma + ndfma) dfma_loop(out, it_dfma, 0.999, 1e-3);
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto run = [&](int ndmma, int ndfma, int itm, int itf) {
    mixed<<<sms, 512>>>(out, ndmma, ndfma, itm, itf);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0)); mixed<<<sms, 512>>>(out, ndmma, ndfma, itm, itf);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
    }
    // flops: DMMA 16 mma x 512 flop per warp-iter; DFMA 64 fma x 2 flop x 32 lanes per warp-iter
    double fm = 2.0 * 8 * 8 * 4 * 16.0 * itm * 4.0 * ndmma * sms;
    double ff = 2.0 * 64 * 32.0 * itf * 4.0 * ndfma * sms;
    std::printf("{\"dmma_groups\": %d, \"dfma_groups\": %d, \"ms\": %.4f, \"dmma_tf\": %.2f, \"dfma_tf\": %.2f, \"total_tf\": %.2f}\n",
                ndmma, ndfma, best, fm / (best * 1e-3) / 1e12, ff / (best * 1e-3) / 1e12,
                (fm + ff) / (best * 1e-3) / 1e12);
  };
  const int itm = 4096, itf = 4096;
  run(2, 0, itm, itf);
  run(0, 2, itm, itf);
  run(2, 2, itm, itf);
  run(1, 1, itm, itf);
  run(4, 0, itm, itf);
  run(0, 4, itm, itf);
  run(2, 2, itm, itf / 2);
  run(2, 2, itm / 2, itf);
  return 0;
}
