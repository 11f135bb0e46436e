// capi.cu — the extern "C" boundary (include/lbg.h). Validates arguments
// exactly where the reference throws (propagate.cpp:14-28,77-80; lindblad.cpp:25-33;
// expm.cpp:110-121), picks the kernel regime, and maps C++ exceptions to
// LBG_* status codes (no exception crosses the ABI).
#include <dlfcn.h>

#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/lbg.h"
#include "internal.hpp"

namespace lbg {

namespace {
thread_local std::string g_err;
thread_local int64_t g_launches = 0;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return LBG_OK;
  } catch (const lbg::invalid_argument& e) {
    g_err = e.what();
    return LBG_EINVAL;
  } catch (const lbg::cuda_error& e) {
    g_err = e.what();
    (void)cudaGetLastError();  // a non-sticky launch error must not surface in the next, unrelated call
    return LBG_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LBG_ERUNTIME;
  }
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// RAII device buffer for the host-pointer entry points
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) {
    if (bytes) check_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// reference is_hermitian (lindblad.cpp:13-20): relative 1e-12 on max |h|
bool is_hermitian(const double* h, size_t d) {
  double worst = 0.0, scale = 0.0;
  for (size_t i = 0; i < d; ++i)
    for (size_t j = 0; j < d; ++j) {
      const std::complex<double> a(h[2 * (i * d + j)], h[2 * (i * d + j) + 1]);
      const std::complex<double> b(h[2 * (j * d + i)], h[2 * (j * d + i) + 1]);
      worst = std::max(worst, std::abs(a - std::conj(b)));
      scale = std::max(scale, std::abs(a));
    }
  return scale == 0.0 ? worst == 0.0 : worst <= 1e-12 * scale;
}

// Regime selection: latency kernels for few trajectories,
// throughput kernels for batches. CTA / ROWSPLIT take the AoS layout only.
int choose_algo(size_t n, int64_t batch, int algo, Layout layout = Layout::aos) {
  if (algo != LBG_ALGO_AUTO) return algo;
  if (chain_supported(n) && batch <= 512) return LBG_ALGO_CHAIN;
  if (n == 9) return LBG_ALGO_DFMA9;
  if (layout == Layout::aos && cta_chain_supported(n) && batch <= 256) return LBG_ALGO_CTA;
  if (ksplit_supported(n) && ksplit_cost(n, batch) < std::min(cluster_cost(n, batch), smem81_cost(batch)))
    return LBG_ALGO_KSPLIT;
  if (cluster_preferred(n, batch)) return LBG_ALGO_CLUSTER;
  if (smem_supported(n)) return LBG_ALGO_SMEM;
  if (layout == Layout::aos && batch <= 2 && rowsplit_supported(n, batch)) return LBG_ALGO_ROWSPLIT;
  return LBG_ALGO_TILED;
}

void evolve_dev(const double* p, size_t n, double* x_re, double* x_im, double* x_aos, int64_t batch,
                int64_t steps, int algo, void* work, cudaStream_t s, Layout layout) {
  if (n == 0) throw invalid_argument("evolve: propagator must be non-empty");
  if (batch < 0 || steps < 0) throw invalid_argument("evolve: negative batch or steps");
  if (!p) throw invalid_argument("evolve: null propagator");
  if (batch == 0 || steps == 0) return;
  if (layout == Layout::soa && (!x_re || !x_im)) throw invalid_argument("evolve: null state");
  if (layout == Layout::aos && !x_aos) throw invalid_argument("evolve: null state");
  if (layout == Layout::soa && algo == LBG_ALGO_AUTO) {
    // the latency kernels take AoS: SoA callers in that regime are staged
    // through an interleaved copy in the workspace (lbg_evolve_workspace sizes it)
    const int a = choose_algo(n, batch, LBG_ALGO_AUTO, Layout::aos);
    if (a == LBG_ALGO_CTA || a == LBG_ALGO_ROWSPLIT) {
      if (!work) throw invalid_argument("evolve: workspace required");
      const size_t inner = a == LBG_ALGO_ROWSPLIT ? rowsplit_workspace(n, batch) : 0;
      double* stage = reinterpret_cast<double*>(static_cast<char*>(work) + ((inner + 255) & ~size_t(255)));
      const long long count = (long long)batch * (long long)n;
      launch_planes_to_aos(x_re, x_im, count, stage, s);
      evolve_dev(p, n, nullptr, nullptr, stage, batch, steps, a, work, s, Layout::aos);
      launch_aos_to_planes(stage, count, x_re, x_im, s);
      return;
    }
  }
  switch (choose_algo(n, batch, algo, layout)) {
    case LBG_ALGO_CHAIN:
      if (!chain_supported(n)) throw invalid_argument("evolve: chain kernel needs n <= 16");
      return launch_chain(p, n, x_re, x_im, x_aos, batch, steps, layout, s);
    case LBG_ALGO_DFMA9:
      if (n != 9) throw invalid_argument("evolve: dfma9 kernel needs n == 9");
      return launch_dfma9(nullptr, p, x_re, x_im, x_aos, batch, steps, layout, s);
    case LBG_ALGO_SMEM:
      if (!smem_supported(n)) throw invalid_argument("evolve: smem kernel needs n <= 84");
      return launch_smem(p, n, x_re, x_im, x_aos, batch, steps, layout, s);
    case LBG_ALGO_CLUSTER:
      if (!cluster_supported(n)) throw invalid_argument("evolve: cluster kernel needs n == 81");
      return launch_smem_cluster(p, x_re, x_im, x_aos, batch, steps, layout, s);
    case LBG_ALGO_KSPLIT:
      if (!ksplit_supported(n)) throw invalid_argument("evolve: ksplit kernel needs n == 81");
      return launch_ksplit(p, n, x_re, x_im, x_aos, batch, steps, layout, s);
    case LBG_ALGO_TILED:
      return launch_tiled_evolve(p, n, x_re, x_im, x_aos, batch, steps, layout, work, s);
    case LBG_ALGO_CTA:
      if (layout != Layout::aos) throw invalid_argument("evolve: cta kernel takes the AoS layout");
      return launch_cta_chain(p, n, x_aos, batch, steps, s);
    case LBG_ALGO_ROWSPLIT:
      if (layout != Layout::aos) throw invalid_argument("evolve: rowsplit kernel takes the AoS layout");
      return launch_rowsplit(p, n, x_aos, batch, steps, work, s);
    default:
      throw invalid_argument("evolve: unknown algo");
  }
}

}  // namespace

// AoS complex stepping with automatic kernel choice, for other launchers
// (the density mode's packed path, k_density.cu)
void evolve_dev_aos(const double* p, size_t n, double* x_aos, int64_t batch, int64_t steps, void* work,
                    cudaStream_t s) {
  evolve_dev(p, n, nullptr, nullptr, x_aos, batch, steps, LBG_ALGO_AUTO, work, s, Layout::aos);
}

namespace {

// ---- NCCL through dlopen (no link-time dependency) ----
struct Nccl {
  void* h = nullptr;
  int (*get_unique_id)(void*) = nullptr;
  int (*comm_init_rank)(void**, int, const void*, int) = nullptr;  // id passed by value: 128 B
  int (*comm_destroy)(void*) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  const char* (*error_string)(int) = nullptr;
};
typedef struct { char internal[128]; } NcclUniqueId;
typedef int (*CommInitRankFn)(void**, int, NcclUniqueId, int);

Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    x.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!x.h) return x;
    x.get_unique_id = reinterpret_cast<int (*)(void*)>(dlsym(x.h, "ncclGetUniqueId"));
    x.comm_destroy = reinterpret_cast<int (*)(void*)>(dlsym(x.h, "ncclCommDestroy"));
    x.all_reduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
        dlsym(x.h, "ncclAllReduce"));
    x.error_string = reinterpret_cast<const char* (*)(int)>(dlsym(x.h, "ncclGetErrorString"));
    return x;
  }();
  if (!n.h) throw cuda_error("libnccl.so.2 not loadable");
  return n;
}
void nccl_check(int rc, const char* what) {
  if (rc != 0)
    throw cuda_error(std::string(what) + ": " + (nccl().error_string ? nccl().error_string(rc) : "nccl error"));
}

}  // namespace

void note_launch(int n) { g_launches += n; }

__global__ void scale_kernel(double* x, size_t n, double s) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] *= s;
}
void launch_scale(double* x, size_t n, double s, cudaStream_t st) {
  if (n == 0) return;
  scale_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(x, n, s);
  LBG_CHECK_LAUNCH("scale_kernel");
}

void sync_event_spin(cudaEvent_t e, const char* what) {
  cudaError_t rc;
  while ((rc = cudaEventQuery(e)) == cudaErrorNotReady) {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  check_cuda(rc, what);
}
void sync_stream_spin(cudaStream_t s, const char* what) {
  thread_local std::map<int, cudaEvent_t>* evs = new std::map<int, cudaEvent_t>;  // per thread and device
  cudaEvent_t& e = (*evs)[current_device()];
  if (!e) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  check_cuda(cudaEventRecord(e, s), what);
  sync_event_spin(e, what);
}

int current_device() {
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "get device");
  return dev;
}

void ensure_max_dyn_smem(const void* fn, int bytes) {
  // the attribute is an upper bound: only ever raise it (launches of one
  // kernel with different sizes, in any order, all stay valid)
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int>* cur = new std::map<std::pair<const void*, int>, int>;
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(mu);
  int& have = (*cur)[{fn, dev}];
  if (bytes <= have) return;
  check_cuda(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "smem attr");
  have = bytes;
}

}  // namespace lbg

using namespace lbg;

extern "C" {

const char* lbg_last_error(void) { return g_err.c_str(); }
const char* lbg_version(void) { return "lbg 0.1 (sm_100a)"; }
int64_t lbg_launch_count(void) { return g_launches; }
void lbg_reset_launch_count(void) { g_launches = 0; }

// ---- raw step shims (kernels.hpp:22-24) ----
void lbg_step_soa(const double* p_re, const double* p_im, const double* v_re, const double* v_im,
                  double* out_re, double* out_im, size_t n) {
  const int rc = guarded([&] {
    std::vector<double> p(2 * n * n), v(2 * n), o(2 * n);
    for (size_t e = 0; e < n * n; ++e) {
      p[2 * e] = p_re[e];
      p[2 * e + 1] = p_im[e];
    }
    for (size_t e = 0; e < n; ++e) {
      v[2 * e] = v_re[e];
      v[2 * e + 1] = v_im[e];
    }
    DevBuf dp(p.size() * 8), dv(v.size() * 8), dout(o.size() * 8);
    check_cuda(cudaMemcpy(dp.p, p.data(), p.size() * 8, cudaMemcpyHostToDevice), "H2D");
    check_cuda(cudaMemcpy(dv.p, v.data(), v.size() * 8, cudaMemcpyHostToDevice), "H2D");
    launch_step_once(dp.as<double>(), dv.as<double>(), dout.as<double>(), n, nullptr);
    check_cuda(cudaMemcpy(o.data(), dout.p, o.size() * 8, cudaMemcpyDeviceToHost), "D2H");
    for (size_t e = 0; e < n; ++e) {
      out_re[e] = o[2 * e];
      out_im[e] = o[2 * e + 1];
    }
  });
  if (rc != LBG_OK) {
    std::fprintf(stderr, "lbg_step_soa: %s\n", g_err.c_str());
    std::abort();
  }
}

void lbg_step_aos(const double* p, const double* v, double* out, size_t n) {
  const int rc = guarded([&] {
    DevBuf dp(2 * n * n * 8), dv(2 * n * 8), dout(2 * n * 8);
    check_cuda(cudaMemcpy(dp.p, p, 2 * n * n * 8, cudaMemcpyHostToDevice), "H2D");
    check_cuda(cudaMemcpy(dv.p, v, 2 * n * 8, cudaMemcpyHostToDevice), "H2D");
    launch_step_once(dp.as<double>(), dv.as<double>(), dout.as<double>(), n, nullptr);
    check_cuda(cudaMemcpy(out, dout.p, 2 * n * 8, cudaMemcpyDeviceToHost), "D2H");
  });
  if (rc != LBG_OK) {
    std::fprintf(stderr, "lbg_step_aos: %s\n", g_err.c_str());
    std::abort();
  }
}

// ---- model assembly / propagator ----
int lbg_build_lindbladian_dev(size_t d, const double* h, size_t n_ops, const double* ops,
                              double* out, void* stream) {
  return guarded([&] {
    if (d == 0) throw invalid_argument("build_lindbladian: dimension must be positive");
    if (!h || !out || (n_ops && !ops)) throw invalid_argument("build_lindbladian: null pointer");
    launch_build_lindbladian(d, h, n_ops, ops, out, as_stream(stream));
  });
}

int lbg_build_lindbladian(size_t d, const double* h, size_t n_ops, const double* ops, double* out) {
  return guarded([&] {
    if (d == 0) throw invalid_argument("make_model: dimension must be positive");
    if (!is_hermitian(h, d)) throw invalid_argument("make_model: Hamiltonian is not Hermitian within 1e-12");
    const size_t n = d * d;
    DevBuf dh(2 * d * d * 8), dops(2 * n_ops * d * d * 8), dout(2 * n * n * 8);
    check_cuda(cudaMemcpy(dh.p, h, 2 * d * d * 8, cudaMemcpyHostToDevice), "H2D");
    if (n_ops) check_cuda(cudaMemcpy(dops.p, ops, 2 * n_ops * d * d * 8, cudaMemcpyHostToDevice), "H2D");
    launch_build_lindbladian(d, dh.as<double>(), n_ops, dops.as<double>(), dout.as<double>(), nullptr);
    check_cuda(cudaMemcpy(out, dout.p, 2 * n * n * 8, cudaMemcpyDeviceToHost), "D2H");
  });
}

size_t lbg_expm_workspace(size_t n) { return expm_workspace(n); }

int lbg_expm_dev(const double* a, size_t n, double dt, double* out, double* work, void* stream) {
  return guarded([&] {
    if (n == 0) throw invalid_argument("expm: matrix must be square and non-empty");
    if (!std::isfinite(dt)) throw invalid_argument("expm: dt must be finite");
    if (!a || !out || !work) throw invalid_argument("expm: null pointer");
    expm_dev(a, n, dt, out, work, as_stream(stream));
  });
}

int lbg_expm(const double* a, size_t n, double dt, double* out) {
  return guarded([&] {
    if (n == 0) throw invalid_argument("expm: matrix must be square and non-empty");
    if (!std::isfinite(dt)) throw invalid_argument("expm: dt must be finite");
    for (size_t e = 0; e < 2 * n * n; ++e)
      if (!std::isfinite(a[e])) throw invalid_argument("expm: non-finite entries in input");
    DevBuf da(2 * n * n * 8), dout(2 * n * n * 8), dw(lbg_expm_workspace(n));
    check_cuda(cudaMemcpy(da.p, a, 2 * n * n * 8, cudaMemcpyHostToDevice), "H2D");
    expm_dev(da.as<double>(), n, dt, dout.as<double>(), dw.as<double>(), nullptr);
    check_cuda(cudaMemcpy(out, dout.p, 2 * n * n * 8, cudaMemcpyDeviceToHost), "D2H");
  });
}

// ---- batched building blocks (lbg_assemble_batched / lbg_expm_batched) ----
int lbg_build_lindbladian_batched_dev(size_t d, const double* h, size_t n_ops, const double* ops, int64_t batch,
                                      double* out, void* stream) {
  return guarded([&] {
    if (d == 0) throw invalid_argument("build_lindbladian: dimension must be positive");
    if (batch < 0) throw invalid_argument("build_lindbladian: negative batch");
    if (batch == 0) return;
    if (!h || !out || (n_ops && !ops)) throw invalid_argument("build_lindbladian: null pointer");
    launch_build_lindbladian_batched(d, h, n_ops, ops, batch, out, as_stream(stream));
  });
}

size_t lbg_expm_batched_workspace(size_t n, int64_t batch) { return expm_batched_workspace(n, batch); }

int lbg_expm_batched_dev(const double* a, size_t n, int64_t batch, double dt, double* out, void* work,
                         void* stream) {
  return guarded([&] {
    if (n == 0) throw invalid_argument("expm: matrix must be square and non-empty");
    if (batch < 0) throw invalid_argument("expm: negative batch");
    if (!std::isfinite(dt)) throw invalid_argument("expm: dt must be finite");
    if (batch == 0) return;
    if (!a || !out || !work) throw invalid_argument("expm: null pointer");
    expm_batched_dev(a, n, batch, dt, out, work, as_stream(stream));
  });
}

// ---- batched shared-P propagation ----
size_t lbg_evolve_workspace(size_t n, int64_t batch, int algo) {
  if (n == 0 || batch <= 0) return 0;
  const int a = choose_algo(n, batch, algo);
  // SoA callers of the AoS-only latency kernels stage an interleaved copy
  const size_t stage = algo == LBG_ALGO_AUTO && (a == LBG_ALGO_CTA || a == LBG_ALGO_ROWSPLIT)
                           ? size_t(batch) * n * 16 : 0;
  switch (a) {
    case LBG_ALGO_TILED: return tiled_workspace(n, batch);
    case LBG_ALGO_ROWSPLIT:
      return rowsplit_supported(n, batch) ? ((rowsplit_workspace(n, batch) + 255) & ~size_t(255)) + stage : 0;
    default: return stage;
  }
}

int lbg_evolve_shared_p_soa_dev(const double* p, size_t n, double* x_re, double* x_im,
                                int64_t batch, int64_t steps, int algo, void* work, void* stream) {
  return guarded([&] {
    evolve_dev(p, n, x_re, x_im, nullptr, batch, steps, algo, work, as_stream(stream), Layout::soa);
  });
}

int lbg_evolve_shared_p_aos_dev(const double* p, size_t n, double* x, int64_t batch, int64_t steps,
                                int algo, void* work, void* stream) {
  return guarded([&] {
    evolve_dev(p, n, nullptr, nullptr, x, batch, steps, algo, work, as_stream(stream), Layout::aos);
  });
}

}  // extern "C"

namespace {
// 1-norm (max column sum) of a d x d complex matrix (interleaved doubles)
double norm1(const double* a, size_t d) {
  double best = 0.0;
  for (size_t c = 0; c < d; ++c) {
    double sum = 0.0;
    for (size_t r = 0; r < d; ++r) sum += std::hypot(a[2 * (r * d + c)], a[2 * (r * d + c) + 1]);
    best = std::max(best, sum);
  }
  return best;
}
// A-priori bound on the squarings the real-form GRAPE build needs (Taylor-16,
// theta = 0.79): ||L||_1 <= 2 max_j ||h0 + a_j hc||_1 + sum_k (||A_k||_1^2 +
// ||A_k^dag A_k||_1) by the Kronecker norm identity, and every real-form entry
// combines two complex entries, so ||L_R||_1 <= 2 ||L||_1.
int grape_squaring_bound(size_t d, const double* h0, const double* hc, const double* amps, int64_t segments,
                         size_t n_ops, const double* ops, double dt) {
  double hmax = 0.0;
  const double n0 = norm1(h0, d), nc = norm1(hc, d);
  for (int64_t j = 0; j < segments; ++j) hmax = std::max(hmax, n0 + std::fabs(amps[j]) * nc);
  double dis = 0.0;
  std::vector<double> ada(2 * d * d);
  for (size_t k = 0; k < n_ops; ++k) {
    const double* a = ops + k * 2 * d * d;
    for (size_t i = 0; i < d; ++i)
      for (size_t j = 0; j < d; ++j) {
        double re = 0.0, im = 0.0;  // (A^dag A)_ij = sum_r conj(A_ri) A_rj
        for (size_t r = 0; r < d; ++r) {
          const double xr = a[2 * (r * d + i)], xi = -a[2 * (r * d + i) + 1];
          const double yr = a[2 * (r * d + j)], yi = a[2 * (r * d + j) + 1];
          re += xr * yr - xi * yi;
          im += xr * yi + xi * yr;
        }
        ada[2 * (i * d + j)] = re;
        ada[2 * (i * d + j) + 1] = im;
      }
    const double na = norm1(a, d);
    dis += na * na + norm1(ada.data(), d);
  }
  const double bound = 2.0 * std::fabs(dt) * (2.0 * hmax + dis);
  if (!std::isfinite(bound)) throw invalid_argument("grape_chain: non-finite generator");
  const int sq = bound > 0.79 ? int(std::ceil(std::log2(bound / 0.79))) : 0;
  if (sq > 64) throw runtime_error("expm: norm requires more than 64 squarings");
  return sq;
}
}  // namespace

extern "C" {

size_t lbg_evolve_planes_workspace(size_t n, int64_t batch, int algo) {
  return ((n * n * 16 + 255) & ~size_t(255)) + lbg_evolve_workspace(n, batch, algo);
}

int lbg_evolve_shared_p_planes_dev(const double* p_re, const double* p_im, size_t n, double* x_re, double* x_im,
                                   int64_t batch, int64_t steps, int algo, void* work, void* stream) {
  return guarded([&] {
    if (!p_re || !p_im) throw invalid_argument("evolve: null propagator");
    if (!work) throw invalid_argument("evolve: workspace required");
    if (batch == 0 || steps == 0) return;
    cudaStream_t s = as_stream(stream);
    double* p = static_cast<double*>(work);
    launch_planes_to_aos(p_re, p_im, (long long)n * (long long)n, p, s);
    void* inner = static_cast<char*>(work) + ((n * n * 16 + 255) & ~size_t(255));
    evolve_dev(p, n, x_re, x_im, nullptr, batch, steps, algo, inner, s, Layout::soa);
  });
}

int lbg_evolve_shared_p(const double* p, size_t d, const double* rho0, int64_t batch, int64_t steps,
                        double* out, int algo) {
  return guarded([&] {
    if (steps < 0) throw invalid_argument("evolve: negative batch or steps");
    const size_t n = d * d;
    // the cooperative tile engine needs the whole device: one chunk, one stream
    const bool single = d > 0 && batch > 0 && choose_algo(n, batch, algo) == LBG_ALGO_TILED;
    host_evolve(p, d, rho0, batch, out, single, [&](int64_t chunk) { return lbg_evolve_workspace(n, chunk, algo); },
                [&](const double* dp, double* xc, int64_t nb, void* w, cudaStream_t s) {
                  evolve_dev(dp, n, nullptr, nullptr, xc, nb, steps, algo, w, s, Layout::aos);
                });
  });
}

int lbg_evolve_density(const double* p, size_t d, const double* rho0, int64_t batch, int64_t steps,
                       double* out) {
  return guarded([&] {
    if (steps < 0) throw invalid_argument("evolve: negative batch or steps");
    // beyond n = 84 the real tile engine (cooperative, the whole device) steps: one chunk, one stream
    const bool single = d > 0 && density_uses_tile_engine(d * d);
    host_evolve(p, d, rho0, batch, out, single, [&](int64_t chunk) { return density_workspace(d * d, chunk); },
                [&](const double* dp, double* xc, int64_t nb, void* w, cudaStream_t s) {
                  launch_density(dp, d, xc, nb, steps, kDensityAuto, w, s);
                });
  });
}

// ---- density-matrix mode (real coordinates) ----
size_t lbg_density_workspace(size_t n, int64_t batch) {
  return (n == 0 || batch <= 0) ? 0 : density_workspace(n, batch);
}

int lbg_evolve_density_dev(const double* p, size_t d, double* rho, int64_t batch, int64_t steps,
                           int mode, void* work, void* stream) {
  return guarded([&] {
    if (d == 0) throw invalid_argument("evolve: state dimension must be positive");
    if (batch < 0 || steps < 0) throw invalid_argument("evolve: negative batch or steps");
    if (batch == 0) return;
    if (!p || !rho || !work) throw invalid_argument("evolve: null pointer");
    launch_density(p, d, rho, batch, steps, mode, work, as_stream(stream));
  });
}

// ---- kernel benchmark harness (bench.cpp:70-158) ----
int lbg_run_bench(const lbg_bench_config* cfg, lbg_bench_result* out) {
  if (out) std::memset(out, 0, sizeof *out);
  const int rc = guarded([&] {
    if (!cfg || !out) throw invalid_argument("bench: null config or result");
    if (cfg->dim < 1) throw invalid_argument("bench: dim must be >= 1");
    if (cfg->reps < 1) throw invalid_argument("bench: reps must be >= 1");
    if (cfg->warmup < 0) throw invalid_argument("bench: warmup must be >= 0");
    if (cfg->variant == LBG_VARIANT_SIMD)
      throw lbg::runtime_error("bench: simd variant unavailable on this platform");
    if (cfg->variant != LBG_VARIANT_AOS && cfg->variant != LBG_VARIANT_SOA)
      throw invalid_argument("bench: unknown variant");
    const size_t d = cfg->dim, n = d * d;
    const int64_t batch = cfg->batch < 1 ? 1 : cfg->batch;
    std::vector<double> p(2 * n * n), v0(2 * n);
    if (lbg_bench_inputs(d, cfg->seed, p.data(), v0.data()) != LBG_OK)
      throw invalid_argument(lbg_bench_last_error());
    const Layout layout = cfg->variant == LBG_VARIANT_SOA ? Layout::soa : Layout::aos;
    // automatic regime; SoA inputs in the latency regime are staged to AoS (evolve_dev)
    const int algo = choose_algo(n, batch, LBG_ALGO_AUTO, Layout::aos);
    // state: AoS (batch x n complex) or SoA planes; every trajectory starts at v0
    std::vector<double> x0(size_t(batch) * 2 * n);
    for (int64_t b = 0; b < batch; ++b)
      for (size_t e = 0; e < n; ++e) {
        if (layout == Layout::aos) {
          x0[(size_t(b) * n + e) * 2] = v0[2 * e];
          x0[(size_t(b) * n + e) * 2 + 1] = v0[2 * e + 1];
        } else {
          x0[size_t(b) * n + e] = v0[2 * e];
          x0[size_t(batch) * n + size_t(b) * n + e] = v0[2 * e + 1];
        }
      }
    DevBuf dp(p.size() * 8), dx(x0.size() * 8), dw(std::max<size_t>(lbg_evolve_workspace(n, batch, LBG_ALGO_AUTO), 1));
    check_cuda(cudaMemcpy(dp.p, p.data(), p.size() * 8, cudaMemcpyHostToDevice), "H2D");
    check_cuda(cudaMemcpy(dx.p, x0.data(), x0.size() * 8, cudaMemcpyHostToDevice), "H2D");
    double* xa = dx.as<double>();
    double* xr = layout == Layout::soa ? xa : nullptr;
    double* xi = layout == Layout::soa ? xa + size_t(batch) * n : nullptr;
    auto run = [&](int64_t steps) {
      evolve_dev(dp.as<double>(), n, xr, xi, layout == Layout::aos ? xa : nullptr, batch, steps, LBG_ALGO_AUTO,
                 dw.p, nullptr, layout);
    };
    cudaEvent_t e0, e1;
    check_cuda(cudaEventCreate(&e0), "event");
    check_cuda(cudaEventCreate(&e1), "event");
    float ms = 0.f;
    try {
      run(cfg->warmup);  // bench.cpp:96-100 / 122-125: same chain, untimed
      check_cuda(cudaEventRecord(e0, nullptr), "event record");
      run(cfg->reps);
      check_cuda(cudaEventRecord(e1, nullptr), "event record");
      check_cuda(cudaEventSynchronize(e1), "event sync");
      check_cuda(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
    } catch (...) {
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      throw;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double block_ns = double(ms) * 1e6;
    const double resolution_ns = 500.0;  // CUDA event timer resolution
    if (resolution_ns > 0.1 * block_ns)  // bench.cpp:140-144
      throw lbg::runtime_error("bench: timer resolution (500 ns) exceeds 10% of the measured block; increase reps");
    std::vector<double> fin(2 * n);
    if (layout == Layout::aos) {
      check_cuda(cudaMemcpy(fin.data(), xa, 2 * n * 8, cudaMemcpyDeviceToHost), "D2H");
    } else {
      std::vector<double> re(n), im(n);
      check_cuda(cudaMemcpy(re.data(), xr, n * 8, cudaMemcpyDeviceToHost), "D2H");
      check_cuda(cudaMemcpy(im.data(), xi, n * 8, cudaMemcpyDeviceToHost), "D2H");
      for (size_t e = 0; e < n; ++e) {
        fin[2 * e] = re[e];
        fin[2 * e + 1] = im[e];
      }
    }
    std::complex<double> checksum{0.0, 0.0};  // bench.cpp:106,133: sum of the final vector
    for (size_t e = 0; e < n; ++e) checksum += std::complex<double>{fin[2 * e], fin[2 * e + 1]};
    const double d2 = double(d) * double(d), d4 = d2 * d2;
    out->ns_per_step = block_ns / double(cfg->reps);
    out->gflops = 8.0 * d4 / out->ns_per_step;
    out->gbs = (d4 + 2.0 * d2) * 16.0 / out->ns_per_step;
    out->checksum_re = checksum.real();
    out->checksum_im = checksum.imag();
    out->traj_steps_per_s = double(batch) * double(cfg->reps) / (block_ns * 1e-9);
    out->algo = algo;
  });
  if (rc != LBG_OK && out) {
    out->failed = 1;
    std::snprintf(out->error, sizeof out->error, "%s", g_err.c_str());
  }
  return rc;
}

// ---- per-trajectory sweep (config 4) ----
size_t lbg_sweep_workspace(size_t d, int64_t batch) {
  const size_t c = sweep_workspace(d, batch);
  if (ptm_small_supported(d)) return std::max(c, ptm_small_workspace(d, batch));
  return ptm_sweep_supported(d) ? std::max(c, ptm_sweep_workspace(batch)) : c;
}

int lbg_evolve_sweep_dev(size_t d, const double* h0, const double* hd, const double* hs, size_t n_ops,
                         const double* ops, const double* delta, const double* scale, double dt,
                         const double* rho0, int64_t batch, int64_t steps, double* pops,
                         double* ens_sum, int mode, void* work, void* stream) {
  return guarded([&] {
    if (d == 0) throw invalid_argument("sweep: dimension must be positive");
    if (batch < 0 || steps < 0) throw invalid_argument("sweep: negative batch or steps");
    if (!std::isfinite(dt)) throw invalid_argument("sweep: dt must be finite");
    if (!h0 || !hd || !hs || !delta || !scale || !rho0 || !pops || !ens_sum || (n_ops && !ops))
      throw invalid_argument("sweep: null pointer");
    if (!work) throw invalid_argument("sweep: workspace required");
    cudaStream_t s = as_stream(stream);
    if (batch == 0) return;
    bool real = false;
    if (mode != LBG_SWEEP_REAL && mode != LBG_SWEEP_AUTO && mode != LBG_SWEEP_COMPLEX)
      throw invalid_argument("sweep: unknown mode");
    {  // propagate.cpp:79-80: lb::evolve validates rho0 before any work (K6), and
       // lb::expm rejects a non-finite generator (expm.cpp:110-112): the model
       // terms and every (delta, s) are checked for NaN / Inf; the real form also
       // needs an exactly Hermitian rho0. One 32-byte D2H and one sync for all of it.
      double* dchk = nullptr;
      check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&dchk), 4 * sizeof(double), s), "malloc check");
      unsigned* flag = reinterpret_cast<unsigned*>(dchk + 3);  // [0] non-finite, [1] not Hermitian
      check_cuda(cudaMemsetAsync(flag, 0, 2 * sizeof(unsigned), s), "memset");
      launch_check_state(rho0, d, 1, dchk, s);
      const long long dd = (long long)(2 * d * d);
      for (const double* m : {h0, hd, hs}) launch_flag_nonfinite(m, dd, flag, s);
      launch_flag_nonfinite(ops, dd * (long long)n_ops, flag, s);
      launch_flag_nonfinite(delta, batch, flag, s);
      launch_flag_nonfinite(scale, batch, flag, s);
      const bool want_real = (mode == LBG_SWEEP_REAL || mode == LBG_SWEEP_AUTO) &&
                             (ptm_sweep_supported(d) || ptm_small_supported(d));
      if (want_real) launch_flag_nonhermitian(rho0, (long long)d, flag + 1, s);
      double chk[4];
      const cudaError_t e1 = cudaMemcpyAsync(chk, dchk, sizeof chk, cudaMemcpyDeviceToHost, s);
      const cudaError_t e2 = cudaFreeAsync(dchk, s);
      check_cuda(e1, "D2H check");
      check_cuda(e2, "free check");
      sync_stream_spin(s, "sync check");
      if (!(chk[0] <= 1e-8 && chk[1] <= 1e-8 && chk[2] >= -1e-8))
        throw invalid_argument("evolve: initial state fails physical-state checks");
      unsigned flags[2];
      std::memcpy(flags, &chk[3], sizeof flags);
      if (flags[0]) throw invalid_argument("sweep: non-finite entries in the model terms or sweep parameters");
      const bool herm = want_real && flags[1] == 0;
      if (mode == LBG_SWEEP_REAL && !herm)
        throw invalid_argument("sweep: real mode needs d in {2, 3, 9} and an exactly Hermitian rho0");
      real = herm && mode != LBG_SWEEP_COMPLEX;
    }
    if (real && ptm_small_supported(d))
      launch_ptm_sweep_small(d, h0, hd, hs, n_ops, ops, delta, scale, dt, rho0, batch, steps, pops, ens_sum, work, s);
    else if (real)
      launch_ptm_sweep(d, h0, hd, hs, n_ops, ops, delta, scale, dt, rho0, batch, steps, pops, ens_sum, work, s);
    else
      launch_sweep(d, h0, hd, hs, n_ops, ops, delta, scale, dt, rho0, batch, steps, pops, ens_sum, work, s);
  });
}

int lbg_grape_chain(size_t d, const double* h0, const double* hc, const double* amplitudes,
                    int64_t segments, int64_t steps_per_segment, double dt, size_t n_ops,
                    const double* ops, const double* rho0, double* out, double* build_ms,
                    double* chain_ms) {
  return guarded([&] {
    // propagate.cpp:116-118
    if (segments <= 0 || !amplitudes) throw invalid_argument("grape_chain: amplitudes are empty");
    if (d == 0 || !h0 || !hc || !rho0 || !out) throw invalid_argument("grape_chain: operator shapes do not conform");
    if (steps_per_segment < 0) throw invalid_argument("grape_chain: negative steps");
    if (!std::isfinite(dt)) throw invalid_argument("expm: dt must be finite");
    {  // lb::expm rejects a non-finite generator (expm.cpp:110-112)
      bool fin = true;
      for (size_t e = 0; e < 2 * d * d; ++e) fin = fin && std::isfinite(h0[e]) && std::isfinite(hc[e]);
      for (int64_t j = 0; j < segments; ++j) fin = fin && std::isfinite(amplitudes[j]);
      for (size_t e = 0; ops && e < 2 * n_ops * d * d; ++e) fin = fin && std::isfinite(ops[e]);
      if (!fin) throw invalid_argument("expm: non-finite entries in input");
    }
    // make_model's Hermiticity check on every segment Hamiltonian (lindblad.cpp:28-29)
    std::vector<double> h(2 * d * d);
    for (int64_t j = 0; j < segments; ++j) {
      for (size_t e = 0; e < 2 * d * d; ++e) h[e] = h0[e] + amplitudes[j] * hc[e];
      if (!is_hermitian(h.data(), d))
        throw invalid_argument("make_model: Hamiltonian is not Hermitian within 1e-12");
    }
    double chk[3];
    {
      DevBuf dr(2 * d * d * 8), dc(3 * 8);
      check_cuda(cudaMemcpy(dr.p, rho0, 2 * d * d * 8, cudaMemcpyHostToDevice), "H2D");
      launch_check_state(dr.as<double>(), d, 1, dc.as<double>(), nullptr);
      check_cuda(cudaMemcpy(chk, dc.p, sizeof chk, cudaMemcpyDeviceToHost), "D2H");
    }
    if (!(chk[0] <= 1e-8 && chk[1] <= 1e-8 && chk[2] >= -1e-8))
      throw invalid_argument("evolve: initial state fails physical-state checks");
    const size_t dd = d * d;
    // the real transfer-matrix form needs an exactly Hermitian rho0 (k_grape_real.cu)
    bool real = grape_real_supported(d) || ptm_grape_supported(d);
    for (size_t i = 0; real && i < d; ++i)
      for (size_t j = 0; j < d; ++j)
        real = real && rho0[2 * (i * d + j)] == rho0[2 * (j * d + i)] &&
               rho0[2 * (i * d + j) + 1] == -rho0[2 * (j * d + i) + 1];
    std::vector<double> zeros(size_t(segments), 0.0);
    DevBuf dh0(dd * 16), dhc(dd * 16), dz(dd * 16), dops(n_ops * dd * 16 + 16), damp(size_t(segments) * 8),
        dzs(size_t(segments) * 8), dx(dd * 16),
        dw(real ? (ptm_grape_supported(d) ? ptm_grape_workspace(segments) : grape_real_workspace(d, segments))
                : grape_workspace(d, segments));
    check_cuda(cudaMemcpy(dh0.p, h0, dd * 16, cudaMemcpyHostToDevice), "H2D");
    check_cuda(cudaMemcpy(dhc.p, hc, dd * 16, cudaMemcpyHostToDevice), "H2D");
    check_cuda(cudaMemset(dz.p, 0, dd * 16), "memset");
    if (n_ops) check_cuda(cudaMemcpy(dops.p, ops, n_ops * dd * 16, cudaMemcpyHostToDevice), "H2D");
    check_cuda(cudaMemcpy(damp.p, amplitudes, size_t(segments) * 8, cudaMemcpyHostToDevice), "H2D");
    check_cuda(cudaMemcpy(dzs.p, zeros.data(), size_t(segments) * 8, cudaMemcpyHostToDevice), "H2D");
    check_cuda(cudaMemcpy(dx.p, rho0, dd * 16, cudaMemcpyHostToDevice), "H2D");
    cudaEvent_t e0, e1, e2;
    check_cuda(cudaEventCreate(&e0), "event");
    check_cuda(cudaEventCreate(&e1), "event");
    check_cuda(cudaEventCreate(&e2), "event");
    check_cuda(cudaEventRecord(e0, nullptr), "event");
    if (real && ptm_grape_supported(d))
      launch_ptm_grape(dh0.as<double>(), dhc.as<double>(), dz.as<double>(), n_ops, dops.as<double>(),
                       damp.as<double>(), segments, steps_per_segment, dt, dx.as<double>(), dw.p, nullptr, e1);
    else if (real)
      launch_grape_real(d, dh0.as<double>(), dhc.as<double>(), dz.as<double>(), n_ops, dops.as<double>(),
                        damp.as<double>(), segments, steps_per_segment, dt, dx.as<double>(),
                        grape_squaring_bound(d, h0, hc, amplitudes, segments, n_ops, ops, dt), dw.p, nullptr, e1);
    else
      launch_grape(d, dh0.as<double>(), dhc.as<double>(), dz.as<double>(), n_ops, dops.as<double>(),
                   damp.as<double>(), dzs.as<double>(), segments, steps_per_segment, dt, dx.as<double>(), dw.p,
                   nullptr, e1);
    check_cuda(cudaEventRecord(e2, nullptr), "event");
    check_cuda(cudaEventSynchronize(e2), "sync");
    float b = 0.f, c = 0.f;
    check_cuda(cudaEventElapsedTime(&b, e0, e1), "elapsed");
    check_cuda(cudaEventElapsedTime(&c, e1, e2), "elapsed");
    if (build_ms) *build_ms = b;
    if (chain_ms) *chain_ms = c;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    check_cuda(cudaMemcpy(out, dx.p, dd * 16, cudaMemcpyDeviceToHost), "D2H");
  });
}

int lbg_check_state_batched_dev(const double* x, size_t d, int64_t batch, double* out3, void* stream) {
  return guarded([&] {
    if (d == 0 || batch < 0 || !out3) throw invalid_argument("check_state: bad arguments");
    launch_check_state(x, d, batch, out3, as_stream(stream));
  });
}

// ---- NCCL ----
int lbg_nccl_unique_id(void* id128) {
  return guarded([&] { nccl_check(nccl().get_unique_id(id128), "ncclGetUniqueId"); });
}

int lbg_nccl_comm_init(void** comm, int nranks, const void* id128, int rank) {
  return guarded([&] {
    auto fn = reinterpret_cast<CommInitRankFn>(dlsym(nccl().h, "ncclCommInitRank"));
    if (!fn) throw cuda_error("ncclCommInitRank missing");
    NcclUniqueId id;
    std::memcpy(id.internal, id128, 128);
    nccl_check(fn(comm, nranks, id, rank), "ncclCommInitRank");
  });
}

int lbg_nccl_comm_destroy(void* comm) {
  return guarded([&] { nccl_check(nccl().comm_destroy(comm), "ncclCommDestroy"); });
}

int lbg_ensemble_mean_dev(double* buf, size_t count, int64_t global_batch, void* comm, void* stream) {
  return guarded([&] {
    if (!buf || global_batch <= 0) throw invalid_argument("ensemble_mean: bad arguments");
    cudaStream_t s = as_stream(stream);
    // ncclFloat64 = 8, ncclSum = 0 (nccl.h); one rank: no communicator needed
    if (comm) nccl_check(nccl().all_reduce(buf, buf, count, 8, 0, comm, s), "ncclAllReduce");
    launch_scale(buf, count, 1.0 / double(global_batch), s);
  });
}

int lbg_allreduce_sum_dev(double* buf, size_t count, void* comm, void* stream) {
  return guarded([&] {
    if (!comm) throw invalid_argument("allreduce: null communicator");
    // ncclFloat64 = 8, ncclSum = 0 (nccl.h)
    nccl_check(nccl().all_reduce(buf, buf, count, 8, 0, comm, as_stream(stream)), "ncclAllReduce");
  });
}

}  // extern "C"
