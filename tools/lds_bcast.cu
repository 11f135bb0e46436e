// Shared-memory load cost by width and broadcast pattern on B200 (sm_100a).
// Each warp issues LDS of 4 / 8 / 16 bytes per lane with one of three address
// patterns: every lane the same address (full broadcast), 4 distinct addresses
// (lane & 3, the K3 column-block pattern), 32 distinct consecutive addresses.
// Prints loads per cycle per SM (warp-instructions) for each case; one
// wavefront per cycle is the shared-memory data path limit.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_bcast lds_bcast.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); std::exit(1);} } while (0)

constexpr int kIters = 2048, kUnroll = 16;

template <class T, int PAT>
__global__ void __launch_bounds__(512, 2) lds_kernel(double* out, int stride_hint) {
  __shared__ __align__(16) double buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i * 0.5;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int idx;  // element index in units of T
  if (PAT == 0) idx = 0;
  else if (PAT == 1) idx = (lane & 3) * stride_hint;
  else idx = lane;
  const T* base = reinterpret_cast<const T*>(buf) + (w & 7) * 64;
  unsigned x0 = 0, x1 = 0;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      // volatile asm so the loads are not merged or hoisted; integer XOR keeps the FP pipes idle
      const unsigned addr = (unsigned)__cvta_generic_to_shared(base + idx + u * 2);
      if constexpr (sizeof(T) == 4) {
        unsigned f;
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(f) : "r"(addr));
        x0 ^= f;
      } else if constexpr (sizeof(T) == 8) {
        unsigned f0, f1;
        asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(f0), "=r"(f1) : "r"(addr));
        x0 ^= f0; x1 ^= f1;
      } else {
        unsigned f0, f1, f2, f3;
        asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(f0), "=r"(f1), "=r"(f2), "=r"(f3) : "r"(addr));
        x0 ^= f0 ^ f2; x1 ^= f1 ^ f3;
      }
    }
  }
  if ((x0 ^ x1) == 0x12345u) out[threadIdx.x] = x0;
}

template <class T, int PAT>
void run(const char* name, int sms, double* out, float clock_ghz) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int threads = 512, blocks = sms * 2;
  lds_kernel<T, PAT><<<blocks, threads>>>(out, sizeof(T) == 16 ? 3 : 6);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  const int reps = getenv("ONCE") ? 0 : 5;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    lds_kernel<T, PAT><<<blocks, threads>>>(out, sizeof(T) == 16 ? 3 : 6);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
  }
  const double warp_loads_per_sm = double(kIters) * kUnroll * (threads / 32) * (blocks / sms);
  const double cycles = best * 1e-3 * clock_ghz * 1e9;
  std::printf("{\"case\": \"%s\", \"bytes\": %d, \"ms\": %.4f, \"warp_loads_per_cycle_per_sm\": %.3f}\n", name,
              (int)sizeof(T), best, warp_loads_per_sm / cycles);
}

struct B16 { double a, b; };

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int clk_khz = 0; CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  const float ghz = clk_khz * 1e-6f;
  double* out; CK(cudaMalloc(&out, 1 << 16));
  run<float, 0>("lds32_same", prop.multiProcessorCount, out, ghz);
  run<float, 1>("lds32_4addr", prop.multiProcessorCount, out, ghz);
  run<float, 2>("lds32_distinct", prop.multiProcessorCount, out, ghz);
  run<double, 0>("lds64_same", prop.multiProcessorCount, out, ghz);
  run<double, 1>("lds64_4addr", prop.multiProcessorCount, out, ghz);
  run<double, 2>("lds64_distinct", prop.multiProcessorCount, out, ghz);
  run<B16, 0>("lds128_same", prop.multiProcessorCount, out, ghz);
  run<B16, 1>("lds128_4addr", prop.multiProcessorCount, out, ghz);
  run<B16, 2>("lds128_distinct", prop.multiProcessorCount, out, ghz);
  std::printf("{\"clock_ghz\": %.3f}\n", ghz);
  return 0;
}
