// ref_driver.cpp — drives the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libref.so)
// through its own public C++ API, and exposes a small extern "C" surface so
// Python (tests/, oracle/gen_golden.py, bench.py --impl reference) can call it.
//
// TEST / BASELINE INFRASTRUCTURE ONLY: the product never links this.
//
// Everything numeric here is a call into lb:: — lb::make_model,
// lb::build_lindbladian (lindblad.cpp:37-59), lb::expm (expm.cpp:109-134),
// lb::evolve (propagate.cpp:75-109) with Variant::soa and the native-fast
// profile (kernels.cpp:63-66, kernels_variants.cpp:26-41), lb::check_state
// (validate.cpp:10-30). The only code of ours is the batching over
// trajectories with std::thread (SPEC.md:326-327 allows concurrent kernel calls
// on disjoint outputs) and the config model construction, which uses lb::kron,
// lb::matmul, lb::dagger, lb::add_scaled, lb::lowering_operator.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "lb/bench.hpp"
#include "lb/complex_matrix.hpp"
#include "lb/expm.hpp"
#include "lb/kernels.hpp"
#include "lb/lindblad.hpp"
#include "lb/propagate.hpp"
#include "lb/random.hpp"
#include "lb/roofline.hpp"
#include "lb/model_io.hpp"
#include "lb/random.hpp"
#include <sstream>
#include "lb/validate.hpp"

using lb::cplx;
using lb::MatrixAoS;

namespace {

thread_local std::string g_err;

MatrixAoS from_buf(const double* p, std::size_t r, std::size_t c) {
    MatrixAoS m(r, c);
    std::memcpy(reinterpret_cast<double*>(m.data.data()), p, sizeof(double) * 2 * r * c);
    return m;
}
void to_buf(const MatrixAoS& m, double* p) {
    std::memcpy(p, reinterpret_cast<const double*>(m.data.data()), sizeof(double) * 2 * m.size());
}

constexpr double kTwoPi = 6.283185307179586;

MatrixAoS embed(const MatrixAoS& op3, std::size_t nq, std::size_t q) {
    const MatrixAoS eye = MatrixAoS::identity(3);
    MatrixAoS cur = q == 0 ? op3 : eye;
    for (std::size_t f = 1; f < nq; ++f) cur = lb::kron(cur, f == q ? op3 : eye);
    return cur;
}

// Config models of BASELINE.json built with the reference's own primitives
// (same term order as oracle/lbo.c lbo_config_model).
lb::LindbladModel config_model(int cfg, double delta, double s) {
    const std::size_t d = cfg == 3 ? 27 : (cfg == 2 || cfg == 4) ? 9 : 3;
    const std::size_t nq = d == 3 ? 1 : d == 9 ? 2 : 3;
    std::vector<double> alpha = nq == 1 ? std::vector<double>{-kTwoPi * 0.3}
                                        : std::vector<double>{-kTwoPi * 0.30, -kTwoPi * 0.28,
                                                              -kTwoPi * 0.32};
    const double omega = kTwoPi * 0.02, g = kTwoPi * 0.005, detuning = kTwoPi * 0.1;
    const MatrixAoS a3 = lb::lowering_operator(3);
    std::vector<MatrixAoS> a, ad, num;
    for (std::size_t q = 0; q < nq; ++q) {
        a.push_back(embed(a3, nq, q));
        ad.push_back(lb::dagger(a.back()));
        num.push_back(lb::matmul(ad.back(), a.back()));
    }
    MatrixAoS h(d, d);
    for (std::size_t q = 0; q < nq; ++q)
        lb::add_scaled(h, cplx{alpha[q] / 2.0, 0.0},
                       lb::matmul(lb::matmul(ad[q], ad[q]), lb::matmul(a[q], a[q])));
    if (cfg == 2 || cfg == 4) lb::add_scaled(h, cplx{detuning, 0.0}, num[1]);
    if (cfg == 4) {
        lb::add_scaled(h, cplx{delta, 0.0}, num[0]);
        lb::add_scaled(h, cplx{delta, 0.0}, num[1]);
    }
    for (std::size_t q = 0; q + 1 < nq; ++q) {
        lb::add_scaled(h, cplx{g, 0.0}, lb::matmul(ad[q], a[q + 1]));
        lb::add_scaled(h, cplx{g, 0.0}, lb::matmul(a[q], ad[q + 1]));
    }
    const double drive = (s * omega) / 2.0;
    lb::add_scaled(h, cplx{drive, 0.0}, a[0]);
    lb::add_scaled(h, cplx{drive, 0.0}, ad[0]);
    std::vector<MatrixAoS> ls;
    for (std::size_t q = 0; q < nq; ++q) {
        ls.push_back(cplx{std::sqrt(2e-5), 0.0} * a[q]);
        ls.push_back(cplx{std::sqrt(2.0 * 7e-6), 0.0} * num[q]);
    }
    return lb::make_model(std::move(h), std::move(ls));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

template <class F>
void parallel_for(std::int64_t n, int threads, F&& body) {
    if (threads <= 1 || n <= 1) {
        body(0, std::int64_t{0}, n);
        return;
    }
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(threads);
    for (int t = 0; t < threads; ++t) {
        const std::int64_t lo = n * t / threads, hi = n * (t + 1) / threads;
        pool.emplace_back([&, t, lo, hi] {
            try {
                body(t, lo, hi);
            } catch (...) {
                errs[t] = std::current_exception();
            }
        });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_hardware_threads() { return static_cast<int>(std::thread::hardware_concurrency()); }

int ref_config_model(int cfg, double delta, double s, double* h, double* ops) {
    return guarded([&] {
        const lb::LindbladModel m = config_model(cfg, delta, s);
        to_buf(m.hamiltonian, h);
        const std::size_t dd = m.dim * m.dim;
        for (std::size_t k = 0; k < m.collapse_ops.size(); ++k)
            to_buf(m.collapse_ops[k], ops + 2 * k * dd);
    });
}

int ref_build_lindbladian(std::size_t d, const double* h, std::size_t nops, const double* ops,
                          double* out) {
    return guarded([&] {
        std::vector<MatrixAoS> ls;
        for (std::size_t k = 0; k < nops; ++k) ls.push_back(from_buf(ops + 2 * k * d * d, d, d));
        const lb::Lindbladian l = lb::build_lindbladian(lb::make_model(from_buf(h, d, d), ls));
        to_buf(l.matrix, out);
    });
}

int ref_expm(const double* a, std::size_t n, double dt, double* out) {
    return guarded([&] { to_buf(lb::expm(from_buf(a, n, n), dt).matrix_aos, out); });
}

// P of config cfg (d^2 x d^2 interleaved) exactly as the reference builds it.
int ref_config_propagator(int cfg, double delta, double s, double* out) {
    return guarded([&] {
        const lb::Lindbladian l = lb::build_lindbladian(config_model(cfg, delta, s));
        to_buf(lb::expm(l.matrix, 0.1).matrix_aos, out);
    });
}

// One raw matvec through a named profile's kernel (kernels.hpp:22-24).
int ref_step_soa(const char* profile, const double* p_re, const double* p_im,
                 const double* v_re, const double* v_im, double* out_re, double* out_im,
                 std::size_t n) {
    const lb::KernelProfile* prof = lb::find_profile(profile);
    if (!prof) {
        g_err = "unknown profile";
        return 1;
    }
    prof->step_soa(p_re, p_im, v_re, v_im, out_re, out_im, n);
    return 0;
}

// evolve() over a batch: rho (B x d x d interleaved) -> out. Variant::soa,
// native-fast profile, `threads` std::threads over contiguous ranges.
// Returns wall seconds of the stepping region in *seconds.
int ref_evolve_batch(const double* p, std::size_t d, const double* rho0, std::int64_t batch,
                     std::size_t steps, double* out, int threads, double* seconds) {
    return guarded([&] {
        const std::size_t n = d * d, dd = d * d;
        lb::Propagator prop;
        prop.dim = d;
        prop.step = 0.1;
        prop.matrix_aos = from_buf(p, n, n);
        prop.matrix_soa = lb::to_soa(prop.matrix_aos);
        const lb::KernelProfile* prof = lb::find_profile("native-fast");
        const auto t0 = std::chrono::steady_clock::now();
        parallel_for(batch, threads, [&](int, std::int64_t lo, std::int64_t hi) {
            for (std::int64_t b = lo; b < hi; ++b) {
                const MatrixAoS r =
                    lb::evolve(prop, from_buf(rho0 + 2 * dd * b, d, d), steps, lb::Variant::soa, prof);
                to_buf(r, out + 2 * dd * b);
            }
        });
        if (seconds)
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// Config 4 through the reference, grape_chain style (propagate.cpp:138-143):
// per trajectory make_model + build_lindbladian + expm, then evolve(500) from
// |00><00|; writes populations (B x 9) and the ensemble SUM of rho (81 complex).
int ref_sweep_batch(const double* deltas, const double* scales, std::int64_t batch,
                    std::size_t steps, double* pops, double* ens_sum, int threads,
                    double* seconds) {
    return guarded([&] {
        const std::size_t d = 9;
        const lb::KernelProfile* prof = lb::find_profile("native-fast");
        std::vector<std::vector<double>> partial(std::max(threads, 1), std::vector<double>(2 * d * d, 0.0));
        const auto t0 = std::chrono::steady_clock::now();
        parallel_for(batch, threads, [&](int slot, std::int64_t lo, std::int64_t hi) {
            std::vector<double>& acc = partial[slot];
            MatrixAoS rho0(d, d);
            rho0(0, 0) = cplx{1.0, 0.0};
            for (std::int64_t b = lo; b < hi; ++b) {
                const lb::Lindbladian l =
                    lb::build_lindbladian(config_model(4, deltas[b], scales[b]));
                const lb::Propagator p = lb::expm(l.matrix, 0.1);
                const MatrixAoS r = lb::evolve(p, rho0, steps, lb::Variant::soa, prof);
                for (std::size_t i = 0; i < d; ++i) pops[b * d + i] = r(i, i).real();
                for (std::size_t e = 0; e < d * d; ++e) {
                    acc[2 * e] += r.data[e].real();
                    acc[2 * e + 1] += r.data[e].imag();
                }
            }
        });
        if (seconds)
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::fill(ens_sum, ens_sum + 2 * d * d, 0.0);
        for (const auto& acc : partial)
            for (std::size_t e = 0; e < 2 * d * d; ++e) ens_sum[e] += acc[e];
    });
}

// Inputs of the reference GRAPE benchmark exactly as cmd_grape draws them
// (commands.cpp:123-159): h0 = random_hermitian(rng(seed), d), dissipator
// 0.1 a, hc = (a + a^dag)/2, amplitudes U[-1,1] from the same rng, dt =
// auto_dt of the first segment's generator, rho0 = |d-1><d-1|.
int ref_grape_inputs(std::size_t d, std::size_t segments, std::uint64_t seed, double* h0,
                     double* hc, double* op, double* amps, double* dt, double* rho0) {
  return guarded([&] {
    auto rng = lb::make_rng(seed);
    const MatrixAoS h = lb::random_hermitian(rng, d);
    const MatrixAoS dis = cplx{0.1, 0.0} * lb::lowering_operator(d);
    const MatrixAoS a = lb::lowering_operator(d);
    const MatrixAoS c = cplx{0.5, 0.0} * (a + lb::dagger(a));
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    for (std::size_t j = 0; j < segments; ++j) amps[j] = u(rng);
    MatrixAoS h1 = h;
    lb::add_scaled(h1, cplx{amps[0], 0.0}, c);
    const double nrm = lb::one_norm(lb::build_lindbladian(lb::make_model(std::move(h1), {dis})).matrix);
    *dt = nrm > 0.0 ? 0.01 / nrm : 1.0;  // auto_dt, commands.cpp:38-41
    MatrixAoS r(d, d);
    r(d - 1, d - 1) = cplx{1.0, 0.0};
    to_buf(h, h0);
    to_buf(c, hc);
    to_buf(dis, op);
    to_buf(r, rho0);
  });
}

// lb::grape_chain (propagate.cpp:111-168) with the native-fast profile, SoA.
int ref_grape_chain(std::size_t d, const double* h0, const double* hc, const double* amps,
                    std::size_t segments, std::size_t steps, double dt, std::size_t n_ops,
                    const double* ops, const double* rho0, double* out, double* build_ms,
                    double* chain_ms) {
  return guarded([&] {
    std::vector<MatrixAoS> ls;
    for (std::size_t k = 0; k < n_ops; ++k) ls.push_back(from_buf(ops + 2 * k * d * d, d, d));
    const std::vector<double> a(amps, amps + segments);
    const lb::GrapeResult g = lb::grape_chain(from_buf(h0, d, d), from_buf(hc, d, d), a, steps, dt, ls,
                                              from_buf(rho0, d, d), lb::Variant::soa,
                                              lb::find_profile("native-fast"));
    to_buf(g.final_state, out);
    *build_ms = g.timings.build_ms;
    *chain_ms = g.timings.chain_ms;
  });
}

// lb::read_model (model_io.cpp:37-109) on a text buffer.
int ref_read_model(const char* text, std::size_t* d, std::size_t* nops, double* h, double* ops,
                   std::size_t cap) {
  return guarded([&] {
    std::istringstream is(text);
    const lb::LindbladModel m = lb::read_model(is);
    *d = m.dim;
    *nops = m.collapse_ops.size();
    if (h) to_buf(m.hamiltonian, h);
    if (ops)
      for (std::size_t k = 0; k < std::min(cap, m.collapse_ops.size()); ++k)
        to_buf(m.collapse_ops[k], ops + 2 * k * m.dim * m.dim);
  });
}

// lb::write_matrix (complex_matrix.cpp:166-177) into a buffer.
int ref_write_matrix(const double* a, std::size_t r, std::size_t c, char* buf, std::size_t cap,
                     std::size_t* len) {
  return guarded([&] {
    std::ostringstream os;
    lb::write_matrix(os, from_buf(a, r, c));
    const std::string s = os.str();
    *len = s.size();
    if (buf && cap > s.size()) std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int ref_check_state(const double* rho, std::size_t d, double tol, double* trace_err,
                    double* herm_err, double* min_diag) {
    return guarded([&] {
        const lb::ValidationReport r = lb::check_state(from_buf(rho, d, d), tol);
        *trace_err = r.trace_error;
        *herm_err = r.hermiticity_error;
        *min_diag = r.min_diagonal;
        if (!r.passed) throw std::runtime_error("check_state failed");
    });
}

// lb::check_generator (validate.cpp:32-45) on a caller-given generator matrix
int ref_check_generator(std::size_t dim, const double* l, std::size_t rows, std::size_t cols, std::size_t trials,
                        double tol, int* passed) {
  return guarded([&] {
    lb::Lindbladian g{dim, from_buf(l, rows, cols)};
    *passed = lb::check_generator(g, trials, tol) ? 1 : 0;
  });
}

// lb::random_density drawn `count` times from lb::make_rng(seed) (random.hpp:12-37):
// the state sequence lb::check_generator uses
int ref_random_density(std::uint64_t seed, std::size_t d, std::int64_t count, double* out) {
  return guarded([&] {
    auto rng = lb::make_rng(seed);
    for (std::int64_t t = 0; t < count; ++t) {
      const lb::MatrixAoS r = lb::random_density(rng, d);
      std::memcpy(out + std::size_t(t) * d * d * 2, r.data.data(), d * d * sizeof(lb::cplx));
    }
  });
}

// The benchmark harness's inputs exactly as lb::run_bench draws them
// (bench.cpp:81-86): lb::make_rng + lb::random_matrix, P scaled by 1/d^2.
int ref_bench_inputs(std::size_t dim, std::uint64_t seed, double* p, double* v0) {
  return guarded([&] {
    const std::size_t n = dim * dim;
    auto rng = lb::make_rng(seed);
    lb::MatrixAoS pm = lb::random_matrix(rng, n, n);
    const lb::cplx scale{1.0 / double(dim * dim), 0.0};
    for (auto& z : pm.data) z *= scale;
    const lb::VectorAoS v = lb::random_matrix(rng, n, 1);
    std::memcpy(p, pm.data.data(), n * n * sizeof(lb::cplx));
    std::memcpy(v0, v.data.data(), n * sizeof(lb::cplx));
  });
}

// lb::run_bench (bench.cpp:70-158): out = ns_per_step, gflops, gbs, checksum re, im
int ref_run_bench(std::size_t dim, int variant, std::size_t reps, std::size_t warmup, std::uint64_t seed,
                  const char* profile, double* out) {
  return guarded([&] {
    lb::BenchConfig c{dim, static_cast<lb::Variant>(variant), reps, warmup, seed, profile ? profile : ""};
    const lb::BenchResult r = lb::run_bench(c);
    out[0] = r.ns_per_step;
    out[1] = r.gflops;
    out[2] = r.gbs;
    out[3] = r.checksum.real();
    out[4] = r.checksum.imag();
  });
}

// lb::write_csv / lb::write_json (bench.cpp:202-248) of rows given as arrays:
// per row dims, variants, reps, warmups, failed flags, values[5] (ns, gflops,
// gbs, checksum re, im) and '\n'-separated error messages.
int ref_write_bench(int json, std::size_t count, const std::size_t* dims, const int* variants,
                    const std::size_t* reps, const std::size_t* warmups, const int* failed,
                    const double* values, const char* errors, const char* profile, const char* machine,
                    char* buf, std::size_t cap, std::size_t* len) {
  return guarded([&] {
    std::vector<lb::BenchResult> rows(count);
    std::string errs = errors ? errors : "";
    std::size_t pos = 0;
    for (std::size_t i = 0; i < count; ++i) {
      lb::BenchResult& r = rows[i];
      r.config.dim = dims[i];
      r.config.variant = static_cast<lb::Variant>(variants[i]);
      r.config.reps = reps[i];
      r.config.warmup = warmups[i];
      r.profile_name = profile;
      r.failed = failed[i] != 0;
      const std::size_t nl = errs.find('\n', pos);
      r.error = errs.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos);
      pos = nl == std::string::npos ? errs.size() : nl + 1;
      r.ns_per_step = values[5 * i];
      r.gflops = values[5 * i + 1];
      r.gbs = values[5 * i + 2];
      r.checksum = lb::cplx{values[5 * i + 3], values[5 * i + 4]};
    }
    std::ostringstream os;
    if (json)
      lb::write_json(os, rows, machine);
    else
      lb::write_csv(os, rows, machine);
    const std::string s = os.str();
    *len = s.size();
    if (buf && cap > s.size()) std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

// ---- roofline (roofline.cpp): profiles as peak + bw[4] + cap[3] arrays ----
static lb::MachineProfile prof_from(const char* name, double peak, const double* bw, const std::uint64_t* cap) {
  lb::MachineProfile m;
  m.name = name ? name : "";
  m.peak_gflops = peak;
  for (int i = 0; i < 4; ++i) m.bandwidth_gbs[i] = bw[i];
  for (int i = 0; i < 3; ++i) m.capacity_bytes[i] = cap[i];
  return m;
}

int ref_read_profile(const char* text, const char* name, double* peak, double* bw, std::uint64_t* cap) {
  return guarded([&] {
    std::istringstream is(text);
    const lb::MachineProfile m = lb::read_profile(is, name);
    *peak = m.peak_gflops;
    for (int i = 0; i < 4; ++i) bw[i] = m.bandwidth_gbs[i];
    for (int i = 0; i < 3; ++i) cap[i] = m.capacity_bytes[i];
  });
}

int ref_write_profile(const char* name, double peak, const double* bw, const std::uint64_t* cap, char* buf,
                      std::size_t capb, std::size_t* len) {
  return guarded([&] {
    std::ostringstream os;
    lb::write_profile(os, prof_from(name, peak, bw, cap));
    const std::string s = os.str();
    *len = s.size();
    if (buf && capb > s.size()) std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

// characterize -> place -> classify; out: flops, bytes, ai, placement, bound, attainable
int ref_roofline(std::size_t d, double peak, const double* bw, const std::uint64_t* cap, double* out) {
  return guarded([&] {
    const lb::MachineProfile m = prof_from("m", peak, bw, cap);
    const lb::KernelCharacter k = lb::place(lb::characterize(d), m);
    const lb::Classification c = lb::classify(k, m);
    out[0] = double(k.flops);
    out[1] = double(k.bytes);
    out[2] = k.ai;
    out[3] = double(static_cast<int>(*k.placement));
    out[4] = c.bound == lb::Bound::memory_bound ? 0.0 : 1.0;
    out[5] = c.attainable_gflops;
  });
}

}  // extern "C"
