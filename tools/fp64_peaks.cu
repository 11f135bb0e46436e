// FP64 peak microbenchmarks for B200 (sm_100a): DFMA (register operands),
// DFMA with constant-bank operands (the d=3 shared-P regime), DMMA
// (mma.sync m8n8k4 f64), shared-memory LDS.128 bandwidth and L2 read bandwidth.
// Prints one JSON line. Used to pick each kernel's regime and as the FP64
// roofline denominator (MEASURED_PEAKS.json has no FP64 entry).
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); std::exit(1);} } while (0)

constexpr int kChains = 8;

__global__ void dfma_peak(double* out, int iters, double a, double b) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

struct PParam { double re[81]; double im[81]; };

// One trajectory per thread, P as a kernel parameter (constant bank 0).
__global__ void dfma_const_d3(const double* __restrict__ in, double* __restrict__ out,
                              long long batch, int steps, const PParam p) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= batch) return;
  double vr[9], vi[9];
#pragma unroll
  for (int j = 0; j < 9; ++j) { vr[j] = in[t * 18 + j]; vi[j] = in[t * 18 + 9 + j]; }
  for (int s = 0; s < steps; ++s) {
    double nr[9], ni[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      double ar = 0.0, ai = 0.0;
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        ar = fma(p.re[i * 9 + j], vr[j], ar);
        ar = fma(-p.im[i * 9 + j], vi[j], ar);
        ai = fma(p.re[i * 9 + j], vi[j], ai);
        ai = fma(p.im[i * 9 + j], vr[j], ai);
      }
      nr[i] = ar; ni[i] = ai;
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) { vr[i] = nr[i]; vi[i] = ni[i]; }
  }
#pragma unroll
  for (int j = 0; j < 9; ++j) { out[t * 18 + j] = vr[j]; out[t * 18 + 9 + j] = vi[j]; }
}

__global__ void dmma_peak(double* out, int iters) {
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

__global__ void dmma16_peak(double* out, int iters) {
  double a[4], b[2];
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = threadIdx.x * 1e-3 + k;
  b[0] = 1.0; b[1] = 0.5;
  double c[4][4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int q = 0; q < 4; ++q) c[k][q] = k + q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void lds_bw(double* out, int iters) {
  __shared__ double2 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      double2 v = buf[(idx + u * 64) & 2047];
      acc.x += v.x; acc.y += v.y;
    }
    idx = (idx + 37) & 2047;
  }
  if (acc.x == 12345.678) out[threadIdx.x] = acc.x + acc.y;
}

__global__ void l2_read(const double2* __restrict__ src, size_t n, int reps, double* out) {
  double2 acc = make_double2(0, 0);
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(src + i);
      acc.x += v.x; acc.y += v.y;
    }
  if (acc.x == 12345.678) out[threadIdx.x] = acc.x + acc.y;
}

template <class F>
float time_it(F f, int reps = 5) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 1 << 20));
  const int iters = 4096;

  // DFMA peak: occupancy sweep
  double dfma_best = 0;
  for (int bpsm : {4, 8, 16}) {
    int blocks = sms * bpsm, threads = 256;
    float ms = time_it([&] { dfma_peak<<<blocks, threads>>>(out, iters, 0.999, 1e-3); });
    double flops = 2.0 * kChains * 8 * (double)iters * blocks * threads;
    double tf = flops / (ms * 1e-3) / 1e12;
    std::fprintf(stderr, "dfma bpsm=%d %.3f ms %.2f TF\n", bpsm, ms, tf);
    if (tf > dfma_best) dfma_best = tf;
  }
  double dmma_best = 0;
  for (int bpsm : {4, 8, 16}) {
    int blocks = sms * bpsm, threads = 256;
    float ms = time_it([&] { dmma_peak<<<blocks, threads>>>(out, iters); });
    double flops = 2.0 * 8 * 8 * 4 * 16.0 * (double)iters * blocks * (threads / 32);
    double tf = flops / (ms * 1e-3) / 1e12;
    std::fprintf(stderr, "dmma m8n8k4 bpsm=%d %.3f ms %.2f TF\n", bpsm, ms, tf);
    if (tf > dmma_best) dmma_best = tf;
  }
  double dmma16_best = 0;
  for (int bpsm : {4, 8}) {
    int blocks = sms * bpsm, threads = 256;
    float ms = time_it([&] { dmma16_peak<<<blocks, threads>>>(out, iters); });
    double flops = 2.0 * 16 * 8 * 8 * 8.0 * (double)iters * blocks * (threads / 32);
    double tf = flops / (ms * 1e-3) / 1e12;
    std::fprintf(stderr, "dmma m16n8k8 bpsm=%d %.3f ms %.2f TF\n", bpsm, ms, tf);
    if (tf > dmma16_best) dmma16_best = tf;
  }
  // const-bank d=3 stepping
  long long batch = 1 << 20; int steps = 100;
  double *in, *o2;
  CK(cudaMalloc(&in, batch * 18 * 8)); CK(cudaMalloc(&o2, batch * 18 * 8));
  CK(cudaMemset(in, 0, batch * 18 * 8));
  PParam p; for (int i = 0; i < 81; ++i) { p.re[i] = 0.01 * i; p.im[i] = -0.003 * i; }
  double c1_best = 0;
  for (int threads : {128, 256}) {
    int blocks = (int)((batch + threads - 1) / threads);
    float ms = time_it([&] { dfma_const_d3<<<blocks, threads>>>(in, o2, batch, steps, p); });
    double tf = 648.0 * batch * steps / (ms * 1e-3) / 1e12;
    std::fprintf(stderr, "dfma_const_d3 threads=%d %.3f ms %.2f TF\n", threads, ms, tf);
    if (tf > c1_best) c1_best = tf;
  }
  // LDS bandwidth
  double lds_best = 0;
  {
    int blocks = sms * 4, threads = 512;
    float ms = time_it([&] { lds_bw<<<blocks, threads>>>(out, iters); });
    double bytes = 16.0 * 8 * (double)iters * blocks * threads;
    lds_best = bytes / (ms * 1e-3) / 1e9;
    std::fprintf(stderr, "lds.128 %.3f ms %.1f GB/s (%.1f B/clk/SM at %d MHz)\n", ms, lds_best,
                 lds_best * 1e9 / (sms * prop.clockRate * 1e3), prop.clockRate / 1000);
  }
  // L2 read bandwidth over a 32 MB buffer
  double l2_best = 0;
  {
    size_t n = (32u << 20) / 16; double2* src; CK(cudaMalloc(&src, n * 16)); CK(cudaMemset(src, 0, n * 16));
    int blocks = sms * 8, threads = 512, reps = 20;
    float ms = time_it([&] { l2_read<<<blocks, threads>>>(src, n, reps, out); });
    l2_best = 16.0 * n * reps / (ms * 1e-3) / 1e9;
    std::fprintf(stderr, "l2 read %.3f ms %.1f GB/s\n", ms, l2_best);
  }
  int clk_khz = 0; CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  std::printf("{\"dfma_tflops\": %.3f, \"dmma_m8n8k4_tflops\": %.3f, \"dmma_m16n8k8_tflops\": %.3f, "
              "\"dfma_const_d3_tflops\": %.3f, \"lds128_gbs\": %.1f, \"l2_read_gbs\": %.1f, \"sms\": %d, \"clock_mhz\": %d}\n",
              dfma_best, dmma_best, dmma16_best, c1_best, lds_best, l2_best, sms, clk_khz / 1000);
  return 0;
}
