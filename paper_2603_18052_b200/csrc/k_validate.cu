// k_validate.cu — the reference's invariant checks on the GPU
// (proj/src/validate.cpp:10-45, proj/include/lb/validate.hpp:20-31):
//   lbg_check_state      lb::check_state over a batch of host states (K6)
//   lbg_check_generator  lb::check_generator: trace annihilation of a generator
//
// check_generator draws `trials` states rho_t = lb::random_density(rng, dim) in
// sequence from the reference's fixed internal seed (lb::make_rng(kDefaultSeed),
// random.hpp:10-37; host_configs.cpp reproduces std::mt19937_64 +
// std::uniform_real_distribution and the i-k-j matmul), and asserts
// |Tr unvec(L vec(rho_t))| <= tol for every t. Only the d diagonal entries of
// unvec(L vec(rho)) enter the trace: row i (d + 1) of L dotted with vec(rho_t).
// One warp per trial: lane i < d accumulates that row over j in ascending order
// (the reference's matmul order), lane 0 adds the d entries in order.
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/lbg.h"
#include "internal.hpp"

namespace lbg {
namespace {

__global__ void generator_trace_kernel(const double2* __restrict__ l, const double2* __restrict__ rho, int d,
                                       int trials, double* __restrict__ abs_trace) {
  const int warp = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (warp >= trials) return;  // warp-uniform
  const int n = d * d;
  const double2* r = rho + size_t(warp) * n;
  double re = 0.0, im = 0.0;
  if (lane < d) {  // diagonal entry (lane, lane) of unvec(L vec(rho)): row lane * (d + 1) of L
    const double2* row = l + size_t(lane) * (d + 1) * n;
    for (int j = 0; j < n; ++j) {
      const double2 a = row[j], b = r[j];
      re = __dadd_rn(re, __dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)));
      im = __dadd_rn(im, __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
    }
  }
  double tr = 0.0, ti = 0.0;  // the trace in row order (validate.cpp:39-40)
  for (int i = 0; i < d; ++i) {
    tr += __shfl_sync(0xffffffffu, re, i);
    ti += __shfl_sync(0xffffffffu, im, i);
  }
  if (lane == 0) abs_trace[warp] = hypot(tr, ti);
}

// d > 32: one thread per trial walks the d diagonal rows in order
__global__ void generator_trace_serial_kernel(const double2* __restrict__ l, const double2* __restrict__ rho, int d,
                                              int trials, double* __restrict__ abs_trace) {
  const int t = int(blockIdx.x * blockDim.x + threadIdx.x);
  if (t >= trials) return;
  const int n = d * d;
  const double2* r = rho + size_t(t) * n;
  double tr = 0.0, ti = 0.0;
  for (int i = 0; i < d; ++i) {
    const double2* row = l + size_t(i) * (d + 1) * n;
    double sr = 0.0, si = 0.0;
    for (int j = 0; j < n; ++j) {
      const double2 a = row[j], b = r[j];
      sr = __dadd_rn(sr, __dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)));
      si = __dadd_rn(si, __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
    }
    tr += sr;
    ti += si;
  }
  abs_trace[t] = hypot(tr, ti);
}

struct Dev {
  void* p = nullptr;
  explicit Dev(size_t bytes) {
    if (bytes) check_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
  }
  ~Dev() {
    if (p) cudaFree(p);
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

thread_local std::string g_verr;

template <class F>
int vguard(F&& f) {
  try {
    f();
    return LBG_OK;
  } catch (const invalid_argument& e) {
    g_verr = e.what();
    return LBG_EINVAL;
  } catch (const cuda_error& e) {
    g_verr = e.what();
    (void)cudaGetLastError();
    return LBG_ECUDA;
  } catch (const std::exception& e) {
    g_verr = e.what();
    return LBG_ERUNTIME;
  }
}

__global__ void flag_nonfinite_kernel(const double* __restrict__ p, long long count, unsigned* __restrict__ flag) {
  bool bad = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    bad = bad || !isfinite(p[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

// flag |= 1 when the d x d complex matrix is not EXACTLY Hermitian (bitwise)
__global__ void flag_nonhermitian_kernel(const double2* __restrict__ m, long long d, unsigned* __restrict__ flag) {
  bool bad = false;
  for (long long e = threadIdx.x; e < d * d; e += blockDim.x) {
    const long long i = e / d, j = e - i * d;
    const double2 a = m[i * d + j], b = m[j * d + i];
    bad = bad || a.x != b.x || a.y != -b.y;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

}  // namespace

void launch_flag_nonhermitian(const double* m, long long d, unsigned* flag, cudaStream_t s) {
  if (d <= 0) return;
  flag_nonhermitian_kernel<<<1, 256, 0, s>>>(reinterpret_cast<const double2*>(m), d, flag);
  LBG_CHECK_LAUNCH("flag_nonhermitian_kernel");
}

// flag |= 1 when any of p[0 .. count) is NaN or infinite (stream-ordered)
void launch_flag_nonfinite(const double* p, long long count, unsigned* flag, cudaStream_t s) {
  if (count <= 0) return;
  const unsigned blocks = unsigned(std::min<long long>((count + 255) / 256, 148LL * 8));
  flag_nonfinite_kernel<<<blocks, 256, 0, s>>>(p, count, flag);
  LBG_CHECK_LAUNCH("flag_nonfinite_kernel");
}

}  // namespace lbg

using namespace lbg;

extern "C" {

const char* lbg_validate_last_error(void) { return g_verr.c_str(); }

int lbg_check_state(const double* rho, size_t d, int64_t batch, double* out3) {
  return vguard([&] {
    if (d == 0 || batch < 0 || !out3 || (batch > 0 && !rho)) throw invalid_argument("check_state: bad arguments");
    const size_t bytes = size_t(batch) * d * d * 16;
    Dev x(bytes), o(3 * 8);
    if (bytes) check_cuda(cudaMemcpy(x.p, rho, bytes, cudaMemcpyHostToDevice), "H2D");
    launch_check_state(static_cast<const double*>(x.p), d, batch, static_cast<double*>(o.p), nullptr);
    check_cuda(cudaMemcpy(out3, o.p, 3 * 8, cudaMemcpyDeviceToHost), "D2H");
  });
}

int lbg_check_generator(size_t dim, const double* l, size_t rows, size_t cols, size_t trials, double tol,
                        int* passed, double* worst) {
  return vguard([&] {
    if (rows != dim * dim || cols != dim * dim)  // validate.cpp:33-34
      throw invalid_argument("check_generator: matrix is not dim^2 x dim^2");
    if (!passed || (dim && !l)) throw invalid_argument("check_generator: null pointer");
    *passed = 1;
    if (worst) *worst = 0.0;
    if (trials == 0 || dim == 0) return;
    if (trials > (size_t(1) << 30)) throw invalid_argument("check_generator: too many trials");
    const size_t n = dim * dim;
    std::vector<double> states(size_t(trials) * n * 2), abs_tr(trials);
    if (lbg_random_density_batch(42, dim, int64_t(trials), states.data()) != LBG_OK)
      throw invalid_argument("check_generator: state generation failed");
    Dev dl(n * n * 16), dr(states.size() * 8), dt(trials * 8);
    check_cuda(cudaMemcpy(dl.p, l, n * n * 16, cudaMemcpyHostToDevice), "H2D L");
    check_cuda(cudaMemcpy(dr.p, states.data(), states.size() * 8, cudaMemcpyHostToDevice), "H2D states");
    const int t = int(trials), dd = int(dim);
    if (dim <= 32) {
      generator_trace_kernel<<<unsigned((t * 32 + 255) / 256), 256>>>(static_cast<const double2*>(dl.p),
                                                                      static_cast<const double2*>(dr.p), dd, t,
                                                                      static_cast<double*>(dt.p));
      LBG_CHECK_LAUNCH("generator_trace_kernel");
    } else {
      generator_trace_serial_kernel<<<unsigned((t + 127) / 128), 128>>>(static_cast<const double2*>(dl.p),
                                                                        static_cast<const double2*>(dr.p), dd, t,
                                                                        static_cast<double*>(dt.p));
      LBG_CHECK_LAUNCH("generator_trace_serial_kernel");
    }
    check_cuda(cudaMemcpy(abs_tr.data(), dt.p, trials * 8, cudaMemcpyDeviceToHost), "D2H");
    double w = 0.0;
    for (double a : abs_tr) {
      if (a > tol) *passed = 0;  // validate.cpp:41 (`abs(trace) > tol` fails the check)
      w = std::isnan(a) ? a : std::max(w, a);
    }
    if (worst) *worst = w;
  });
}

}  // extern "C"
