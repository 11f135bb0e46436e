// dropin_gate.cpp — the drop-in boundary, exercised by the reference's OWN code.
//
// Builds a lb::KernelProfile whose raw step pointers are liblbg's C-ABI shims
// (include/lbg.h: lbg_step_aos / lbg_step_soa — exact StepAoSFn / StepSoAFn
// signatures, proj/include/lb/kernels.hpp:22-33) and hands it to the
// UNMODIFIED reference lb::evolve (propagate.cpp:75-109) and lb::grape_chain
// (propagate.cpp:111-168), compiled from /root/reference by oracle/Makefile
// into oracle/_ref/libref.so. Every step then runs on the B200. Results are
// compared with the reference's native-fast CPU profile, acceptance-style
// (proj/tests/acceptance.cpp): one PASS/FAIL line per criterion, exit code 1
// on any failure. Test infrastructure (built by __graft_entry__.build()).
#include <cmath>
#include <complex>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "lb/expm.hpp"
#include "lb/kernels.hpp"
#include "lb/lindblad.hpp"
#include "lb/propagate.hpp"
#include "lb/random.hpp"
#include "lb/validate.hpp"
#include "lbg.h"

using namespace lb;

namespace {

int g_fail = 0;

void criterion(const char* name, const std::function<std::string()>& body) {
  try {
    const std::string detail = body();
    std::printf("PASS %s: %s\n", name, detail.c_str());
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("FAIL %s: %s\n", name, e.what());
  }
  std::fflush(stdout);
}

void require(bool ok, const std::string& msg) {
  if (!ok) throw std::runtime_error(msg);
}

double max_diff(const MatrixAoS& a, const MatrixAoS& b) {
  double w = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) w = std::max(w, std::abs(a.data[i] - b.data[i]));
  return w;
}

// The whole integration a maintainer adds: two function pointers.
const KernelProfile& b200_profile() {
  static const KernelProfile p{"b200", reinterpret_cast<StepAoSFn>(&lbg_step_aos), &lbg_step_soa};
  return p;
}

char buf[256];

}  // namespace

int main() {
  const KernelProfile& gpu = b200_profile();
  const KernelProfile& cpu = default_profile();  // native-fast

  criterion("closed-form-damping", [&] {  // test_propagate.cpp:156-176 through the GPU profile
    const double gamma = 0.7, dt = 0.004;
    MatrixAoS l(2, 2);
    l(0, 1) = cplx{std::sqrt(gamma), 0.0};
    const Propagator p = expm(build_lindbladian(make_model(MatrixAoS(2, 2), {l})).matrix, dt);
    MatrixAoS rho0(2, 2);
    rho0(1, 1) = cplx{1.0, 0.0};
    double worst = 0.0;
    for (Variant v : {Variant::aos, Variant::soa}) {
      const MatrixAoS rho = evolve(p, rho0, 500, v, &gpu);
      const double err = std::abs(rho(1, 1).real() - std::exp(-gamma * 500 * dt));
      worst = std::max(worst, err);
      require(err < 1e-10, "excited population off by " + std::to_string(err));
      require(check_state(rho).passed, "state checks failed");
    }
    std::snprintf(buf, sizeof buf, "500 steps, aos+soa on the B200 profile, worst |err| %.2e", worst);
    return std::string(buf);
  });

  criterion("evolve-matches-native-fast", [&] {  // acceptance-style parity on the transmon preset
    const LindbladModel m = transmon_model(5e4, 1.0 / (4 * 7e-6), -2 * M_PI * 0.3, 2 * M_PI * 0.02);
    const Lindbladian L = build_lindbladian(m);
    const Propagator p = expm(L.matrix, 0.1);
    auto rng = make_rng(kDefaultSeed);
    double worst = 0.0;
    for (int t = 0; t < 4; ++t) {
      const MatrixAoS rho0 = random_density(rng, 3);
      const MatrixAoS a = evolve(p, rho0, 200, Variant::soa, &gpu);
      const MatrixAoS b = evolve(p, rho0, 200, Variant::soa, &cpu);
      worst = std::max(worst, max_diff(a, b));
    }
    require(worst <= 1e-10, "max |drho| " + std::to_string(worst));
    std::snprintf(buf, sizeof buf, "4 random states x 200 steps, max |drho| %.2e (tol 1e-10)", worst);
    return std::string(buf);
  });

  criterion("kernel-equivalence", [&] {  // acceptance.cpp:245-278 with the GPU kernel in the set
    double worst = 0.0;
    for (std::size_t d : {std::size_t{3}, std::size_t{9}, std::size_t{27}}) {
      auto rng = make_rng(kDefaultSeed + d);
      const std::size_t n = d * d;
      for (int trial = 0; trial < 3; ++trial) {
        const MatrixAoS p = random_matrix(rng, n, n);
        const VectorAoS v = random_matrix(rng, n, 1);
        const VectorAoS ref = step_aos(p, v, find_profile("baseline")->step_aos);
        const double scale = max_abs(ref);
        worst = std::max(worst, max_diff(step_aos(p, v, gpu.step_aos), ref) / scale);
        worst = std::max(worst, max_diff(from_soa(step_soa(to_soa(p), to_soa(v), gpu.step_soa)), ref) / scale);
      }
    }
    require(worst < 1e-12, "kernel divergence " + std::to_string(worst));
    std::snprintf(buf, sizeof buf, "d in {3,9,27}, worst rel diff %.2e", worst);
    return std::string(buf);
  });

  criterion("grape-chain-on-gpu", [&] {  // propagate.cpp:111-168 driving the GPU kernel
    auto rng = make_rng(31);
    const MatrixAoS h0 = random_hermitian(rng, 3), hc = random_hermitian(rng, 3);
    const std::vector<MatrixAoS> dis{cplx{0.2, 0} * lowering_operator(3)};
    MatrixAoS rho0(3, 3);
    rho0(2, 2) = cplx{1, 0};
    const std::vector<double> amps{0.8, -0.3, 0.5};
    const GrapeResult g = grape_chain(h0, hc, amps, 8, 0.002, dis, rho0, Variant::soa, &gpu);
    const GrapeResult c = grape_chain(h0, hc, amps, 8, 0.002, dis, rho0, Variant::soa, &cpu);
    const double err = max_diff(g.final_state, c.final_state);
    require(err <= 1e-12, "grape divergence " + std::to_string(err));
    std::snprintf(buf, sizeof buf, "3 segments x 8 steps, max |drho| %.2e", err);
    return std::string(buf);
  });

  if (g_fail) {
    std::printf("%d criterion(s) failed\n", g_fail);
    return 1;
  }
  std::printf("all criteria passed\n");
  return 0;
}
