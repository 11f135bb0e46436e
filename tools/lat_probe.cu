// Latency probes on the B200: dependent DFMA chain, DMMA chain, LDS round trip,
// STS->BAR->LDS, SHFL. One warp, clock64 around 1024 dependent ops.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* cyc, double a, double b) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = lane; sm[lane + 32] = lane;
  __syncthreads();
  double x = lane * 1e-3;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  double c[2] = {x, x}; double aa = a, bb = b;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c[0]), "+d"(c[1]) : "d"(aa), "d"(bb));
  long long t2 = clock64();
  int idx = lane;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) idx = (int)sm[idx & 31];
  long long t3 = clock64();
  double y = x;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { sm[lane] = y; __syncwarp(); y = sm[(lane + 1) & 31] + 1.0; }
  long long t4 = clock64();
  double z = x;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) z = __shfl_xor_sync(0xffffffffu, z, 1) + 1.0;
  long long t5 = clock64();
  double w = x;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) w = w + b;
  long long t6 = clock64();
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; }
  out[lane] = x + c[0] + c[1] + idx + y + z + w;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMallocManaged(&c, 64);
  probe<<<1, 32>>>(o, c, 0.999, 1e-3); cudaDeviceSynchronize();
  probe<<<1, 32>>>(o, c, 0.999, 1e-3); cudaDeviceSynchronize();
  printf("{\"dfma_lat\": %.1f, \"dmma_lat\": %.1f, \"lds_dep_lat\": %.1f, \"sts_syncwarp_lds_plus_dadd\": %.1f, \"shfl_plus_dadd\": %.1f, \"dadd_lat\": %.1f}\n",
         c[0] / 1024.0, c[1] / 1024.0, c[2] / 1024.0, c[3] / 1024.0, c[4] / 1024.0, c[5] / 1024.0);
  return 0;
}
