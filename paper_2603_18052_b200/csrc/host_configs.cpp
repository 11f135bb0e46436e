// host_configs.cpp — host-side inputs of the engine (product code, C++):
// the BASELINE.json config models, seeded Ginibre initial states and the
// config-4 sweep parameters. Same construction spec as DESIGN.md "Configs";
// tests/test_host.py checks it bit-for-bit against the oracle's independent
// restatement (oracle/lbo.c) and against the reference's own primitives.
//
// Compiled with -ffp-contract=off so the host arithmetic rounds exactly like
// lb::matmul (proj/src/complex_matrix.cpp:30-56) on x86-64.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "../../include/lbg.h"

namespace {

using cplx = std::complex<double>;
using Mat = std::vector<cplx>;  // row-major d x d

constexpr double kTwoPi = 6.283185307179586;
constexpr double kGamma1 = 2e-5, kGammaPhi = 7e-6;

Mat eye(size_t d) {
  Mat m(d * d);
  for (size_t i = 0; i < d; ++i) m[i * d + i] = 1.0;
  return m;
}

// kron (complex_matrix.cpp:18-28)
Mat kron(const Mat& a, size_t da, const Mat& b, size_t db) {
  const size_t d = da * db;
  Mat out(d * d);
  for (size_t i = 0; i < da; ++i)
    for (size_t j = 0; j < da; ++j)
      for (size_t k = 0; k < db; ++k)
        for (size_t l = 0; l < db; ++l) out[(i * db + k) * d + j * db + l] = a[i * da + j] * b[k * db + l];
  return out;
}

// i-k-j matmul with the complex product spelled out (complex_matrix.cpp:41-54)
Mat matmul(const Mat& a, const Mat& b, size_t d) {
  std::vector<double> out(2 * d * d, 0.0);
  const double* bd = reinterpret_cast<const double*>(b.data());
  for (size_t i = 0; i < d; ++i) {
    double* crow = out.data() + 2 * i * d;
    for (size_t k = 0; k < d; ++k) {
      const double xr = a[i * d + k].real(), xi = a[i * d + k].imag();
      const double* brow = bd + 2 * k * d;
      for (size_t j = 0; j < d; ++j) {
        const double yr = brow[2 * j], yi = brow[2 * j + 1];
        crow[2 * j] += xr * yr - xi * yi;
        crow[2 * j + 1] += xr * yi + xi * yr;
      }
    }
  }
  Mat m(d * d);
  std::memcpy(static_cast<void*>(m.data()), out.data(), out.size() * sizeof(double));
  return m;
}

Mat dagger(const Mat& a, size_t d) {
  Mat out(d * d);
  for (size_t i = 0; i < d; ++i)
    for (size_t j = 0; j < d; ++j) out[j * d + i] = std::conj(a[i * d + j]);
  return out;
}

void add_real(Mat& acc, double c, const Mat& x) {
  for (size_t e = 0; e < acc.size(); ++e)
    acc[e] = cplx(acc[e].real() + c * x[e].real(), acc[e].imag() + c * x[e].imag());
}

size_t cfg_dim(int cfg) { return cfg == 3 ? 27 : (cfg == 2 || cfg == 4) ? 9 : (cfg == 0 || cfg == 1) ? 3 : 0; }

struct Ops {
  size_t d, nq;
  std::vector<Mat> a, ad, num;
};

Ops make_ops(size_t d) {
  Ops o;
  o.d = d;
  o.nq = d == 3 ? 1 : d == 9 ? 2 : 3;
  Mat a3(9);
  a3[0 * 3 + 1] = std::sqrt(1.0);
  a3[1 * 3 + 2] = std::sqrt(2.0);  // lowering_operator (lindblad.cpp:76-80)
  const Mat e3 = eye(3);
  for (size_t q = 0; q < o.nq; ++q) {
    Mat cur = q == 0 ? a3 : e3;
    size_t dim = 3;
    for (size_t f = 1; f < o.nq; ++f) {
      cur = kron(cur, dim, f == q ? a3 : e3, 3);
      dim *= 3;
    }
    o.a.push_back(cur);
    o.ad.push_back(dagger(cur, d));
    o.num.push_back(matmul(o.ad.back(), cur, d));
  }
  return o;
}

// H = sum_q (alpha_q/2) a^dag a^dag a a [+ Delta n_2] [+ delta (n_1 + n_2)]
//     + g sum_<pq> (a_p^dag a_q + a_p a_q^dag) + (s Omega / 2)(a_1 + a_1^dag)
void config_h(int cfg, double delta, double s, const Ops& o, Mat& h, bool with_delta, bool with_drive,
              bool with_static) {
  const size_t d = o.d;
  h.assign(d * d, 0.0);
  double alpha[3];
  if (o.nq == 1)
    alpha[0] = -kTwoPi * 0.3;
  else {
    alpha[0] = -kTwoPi * 0.30;
    alpha[1] = -kTwoPi * 0.28;
    alpha[2] = -kTwoPi * 0.32;
  }
  const double omega = kTwoPi * 0.02, g = kTwoPi * 0.005, detuning = kTwoPi * 0.1;
  if (with_static)
    for (size_t q = 0; q < o.nq; ++q)
      add_real(h, alpha[q] / 2.0, matmul(matmul(o.ad[q], o.ad[q], d), matmul(o.a[q], o.a[q], d), d));
  if (with_static && (cfg == 2 || cfg == 4)) add_real(h, detuning, o.num[1]);
  if (with_delta && cfg == 4) {
    add_real(h, delta, o.num[0]);
    add_real(h, delta, o.num[1]);
  }
  if (with_static)
    for (size_t q = 0; q + 1 < o.nq; ++q) {
      add_real(h, g, matmul(o.ad[q], o.a[q + 1], d));
      add_real(h, g, matmul(o.a[q], o.ad[q + 1], d));
    }
  if (with_drive) {
    const double drive = (s * omega) / 2.0;
    add_real(h, drive, o.a[0]);
    add_real(h, drive, o.ad[0]);
  }
}

void put(const Mat& m, double* out) { std::memcpy(out, m.data(), m.size() * sizeof(cplx)); }

uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Stream {
  uint64_t key;
  Stream(uint64_t seed, uint32_t cfg, uint64_t traj)
      : key(mix64(mix64(mix64(seed + 0x9E3779B97F4A7C15ull) ^ (uint64_t(cfg) + 0x632BE59BD9B4E019ull)) ^
                  (traj + 0xD6E8FEB86659FD93ull))) {}
  double uniform(uint64_t k) const {
    const uint64_t w = mix64(key + (k + 1) * 0x9E3779B97F4A7C15ull);
    return (double(w >> 11) + 0.5) * 0x1.0p-53;
  }
};

void ginibre(uint64_t seed, uint32_t cfg, uint64_t traj, size_t d, double* out) {
  const Stream st(seed, cfg, traj);
  Mat g(d * d);
  for (size_t p = 0; p < d * d; ++p) {
    const double u1 = st.uniform(2 * p), u2 = st.uniform(2 * p + 1);
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = kTwoPi * u2;
    g[p] = cplx(r * std::cos(th), r * std::sin(th));
  }
  const Mat rho = matmul(g, dagger(g, d), d);
  double tr = 0.0;
  for (size_t i = 0; i < d; ++i) tr += rho[i * d + i].real();
  const double* rd = reinterpret_cast<const double*>(rho.data());
  for (size_t e = 0; e < 2 * d * d; ++e) out[e] = rd[e] / tr;
}

template <class F>
void parallel(int64_t n, int threads, F&& body) {
  if (threads <= 1 || n < 1024) {
    body(int64_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back([&, t] { body(n * t / threads, n * (t + 1) / threads); });
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

int lbg_config_dims(int cfg, size_t* d, size_t* n_ops) {
  const size_t dim = cfg_dim(cfg);
  if (!dim) return LBG_EINVAL;
  *d = dim;
  *n_ops = dim == 3 ? 2 : dim == 9 ? 4 : 6;
  return LBG_OK;
}

int lbg_config_model(int cfg, double delta, double s, double* h, double* ops) {
  const size_t d = cfg_dim(cfg);
  if (!d) return LBG_EINVAL;
  const Ops o = make_ops(d);
  Mat hm;
  config_h(cfg, delta, s, o, hm, true, true, true);
  put(hm, h);
  const double c1 = std::sqrt(kGamma1), c2 = std::sqrt(2.0 * kGammaPhi);
  for (size_t q = 0; q < o.nq; ++q) {
    Mat l1(d * d), l2(d * d);
    for (size_t e = 0; e < d * d; ++e) {
      l1[e] = cplx(c1 * o.a[q][e].real(), c1 * o.a[q][e].imag());
      l2[e] = cplx(c2 * o.num[q][e].real(), c2 * o.num[q][e].imag());
    }
    put(l1, ops + 2 * (2 * q) * d * d);
    put(l2, ops + 2 * (2 * q + 1) * d * d);
  }
  return LBG_OK;
}

// Config 4's Hamiltonian as an affine family H(delta, s) = h0 + delta*hd + s*hs.
int lbg_config_sweep_terms(double* h0, double* hd, double* hs) {
  const Ops o = make_ops(9);
  Mat m;
  config_h(4, 0.0, 0.0, o, m, false, false, true);
  put(m, h0);
  config_h(4, 1.0, 0.0, o, m, true, false, false);
  put(m, hd);
  config_h(4, 0.0, 1.0, o, m, false, true, false);
  put(m, hs);
  return LBG_OK;
}

double lbg_uniform(uint64_t seed, uint32_t cfg, uint64_t traj, uint64_t k) {
  return Stream(seed, cfg, traj).uniform(k);
}

// rho0 of trajectories [first, first + count) of config cfg: (count, d, d) AoS
int lbg_ginibre_batch(uint64_t seed, uint32_t cfg, uint64_t first, int64_t count, size_t d, double* out,
                      int threads) {
  if (d == 0 || count < 0) return LBG_EINVAL;
  parallel(count, threads, [&](int64_t lo, int64_t hi) {
    for (int64_t b = lo; b < hi; ++b) ginibre(seed, cfg, first + uint64_t(b), d, out + 2 * d * d * size_t(b));
  });
  return LBG_OK;
}

// lb::random_density (random.hpp:31-37) drawn `count` times in sequence from
// lb::make_rng(seed) (random.hpp:12-14): G with std::uniform_real_distribution
// (-1, 1) re / im per element in row-major order (random.hpp:17-21), rho =
// G G^dag (i-k-j matmul), then (1 / tr) * rho in complex arithmetic.
int lbg_random_density_batch(uint64_t seed, size_t d, int64_t count, double* out) {
  if (d == 0 || count < 0 || (count && !out)) return LBG_EINVAL;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (int64_t t = 0; t < count; ++t) {
    Mat g(d * d);
    for (auto& z : g) {
      const double re = u(rng);
      const double im = u(rng);
      z = cplx{re, im};
    }
    const Mat rho = matmul(g, dagger(g, d), d);
    cplx tr{0.0, 0.0};
    for (size_t i = 0; i < d; ++i) tr += rho[i * d + i];
    const cplx inv = cplx{1.0, 0.0} / tr;
    for (size_t e = 0; e < d * d; ++e) {
      const cplx z = inv * rho[e];
      out[(size_t(t) * d * d + e) * 2] = z.real();
      out[(size_t(t) * d * d + e) * 2 + 1] = z.imag();
    }
  }
  return LBG_OK;
}

int lbg_sweep_params_batch(uint64_t seed, uint64_t first, int64_t count, double* delta, double* scale) {
  if (count < 0) return LBG_EINVAL;
  for (int64_t b = 0; b < count; ++b) {
    const Stream st(seed, 4, first + uint64_t(b));
    delta[b] = (kTwoPi * 0.005) * (2.0 * st.uniform(0) - 1.0);
    scale[b] = 0.9 + 0.2 * st.uniform(1);
  }
  return LBG_OK;
}

}  // extern "C"
