// host_roofline.cpp — the reference's roofline model for the GPU ladder
// (host side; the measured profile comes from lbg_measure_machine_profile in
// k_probe.cu). Same formulas, same invariants and error messages, same text
// format as proj/src/roofline.cpp:44-182, so profiles and placements are
// interchangeable with the reference's tool.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>

#include "../../include/lbg.h"

namespace {

thread_local std::string g_roof_err;

std::string trim(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
  while (e > b && std::isspace(static_cast<unsigned char>(s[e - 1]))) --e;
  return s.substr(b, e - b);
}

template <class F>
int roof_guard(F&& f) {
  try {
    f();
    return LBG_OK;
  } catch (const std::invalid_argument& e) {
    g_roof_err = e.what();
    return LBG_EINVAL;
  } catch (const std::exception& e) {
    g_roof_err = e.what();
    return LBG_ERUNTIME;
  }
}

// roofline.cpp:44-60
void validate(const lbg_machine_profile& m) {
  if (!(m.peak_gflops > 0.0)) throw std::invalid_argument("machine profile: peak_gflops must be positive");
  for (double bw : m.bandwidth_gbs)
    if (!(bw > 0.0)) throw std::invalid_argument("machine profile: bandwidths must be positive");
  for (uint64_t cap : m.capacity_bytes)
    if (cap == 0) throw std::invalid_argument("machine profile: capacities must be positive");
  for (int i = 1; i < 4; ++i)
    if (!(m.bandwidth_gbs[i - 1] > m.bandwidth_gbs[i]))
      throw std::invalid_argument("machine profile: bandwidths must decrease strictly L1 > L2 > L3 > DRAM");
  for (int i = 1; i < 3; ++i)
    if (!(m.capacity_bytes[i - 1] < m.capacity_bytes[i]))
      throw std::invalid_argument("machine profile: capacities must increase strictly L1 < L2 < L3");
}

// std::ostream's default floating-point output (precision 6, %g)
std::string fmt_g(double x) {
  std::ostringstream os;
  os << x;
  return os.str();
}

}  // namespace

extern "C" {

const char* lbg_roofline_last_error(void) { return g_roof_err.c_str(); }

int lbg_validate_profile(const lbg_machine_profile* m) {
  return roof_guard([&] {
    if (!m) throw std::invalid_argument("machine profile: null");
    validate(*m);
  });
}

// roofline.cpp:62-74
int lbg_characterize(size_t d, lbg_kernel_character* out) {
  return roof_guard([&] {
    if (d < 1) throw std::invalid_argument("characterize: d must be >= 1");
    if (!out) throw std::invalid_argument("characterize: null output");
    const uint64_t d2 = uint64_t(d) * d, d4 = d2 * d2;
    out->dim = d;
    out->flops = 8 * d4;
    out->bytes = (d4 + 2 * d2) * 16;
    out->ai = double(out->flops) / double(out->bytes);
    out->working_set_bytes = out->bytes;
    out->placement = -1;
  });
}

// roofline.cpp:76-87
int lbg_place(lbg_kernel_character* k, const lbg_machine_profile* m) {
  return roof_guard([&] {
    if (!k || !m) throw std::invalid_argument("place: null argument");
    validate(*m);
    int level = 3;
    for (int i = 2; i >= 0; --i)
      if (k->working_set_bytes <= m->capacity_bytes[i]) level = i;
    k->placement = level;
  });
}

// roofline.cpp:89-91
int lbg_ridge_point(const lbg_machine_profile* m, int level, double* out) {
  return roof_guard([&] {
    if (!m || !out) throw std::invalid_argument("ridge_point: null argument");
    if (level < 0 || level > 3) throw std::invalid_argument("ridge_point: level out of range");
    *out = m->peak_gflops / m->bandwidth_gbs[level];
  });
}

// roofline.cpp:93-99
int lbg_classify(const lbg_kernel_character* k, const lbg_machine_profile* m, int* bound,
                 double* attainable_gflops) {
  return roof_guard([&] {
    if (!k || !m || !bound || !attainable_gflops) throw std::invalid_argument("classify: null argument");
    if (k->placement < 0 || k->placement > 3) throw std::invalid_argument("classify: placement is unset; call place()");
    const double bw = m->bandwidth_gbs[k->placement];
    *bound = k->ai < m->peak_gflops / bw ? LBG_MEMORY_BOUND : LBG_COMPUTE_BOUND;
    *attainable_gflops = std::fmin(m->peak_gflops, k->ai * bw);
  });
}

// roofline.cpp:172-182
int lbg_write_machine_profile(const lbg_machine_profile* m, char* buf, size_t cap, size_t* len) {
  return roof_guard([&] {
    if (!m || !len) throw std::invalid_argument("write_profile: null argument");
    std::string s = "# machine profile: " + std::string(m->name) + "\n";
    s += "peak_gflops = " + fmt_g(m->peak_gflops) + "\n";
    static const char* bw[] = {"bw_l1", "bw_l2", "bw_l3", "bw_dram"};
    for (int i = 0; i < 4; ++i) s += std::string(bw[i]) + " = " + fmt_g(m->bandwidth_gbs[i]) + "\n";
    static const char* cp[] = {"cap_l1", "cap_l2", "cap_l3"};
    for (int i = 0; i < 3; ++i) s += std::string(cp[i]) + " = " + std::to_string(m->capacity_bytes[i]) + "\n";
    *len = s.size();
    if (buf) {
      if (cap < s.size() + 1) throw std::invalid_argument("write_profile: buffer too small");
      std::memcpy(buf, s.c_str(), s.size() + 1);
    }
  });
}

// roofline.cpp:111-164
int lbg_read_machine_profile(const char* text, const char* name, lbg_machine_profile* out) {
  return roof_guard([&] {
    if (!out) throw std::invalid_argument("read_profile: null output");
    std::map<std::string, double> values;
    std::istringstream is(text ? text : "");
    std::string line;
    while (std::getline(is, line)) {
      const std::string st = trim(line);
      if (st.empty() || st[0] == '#') continue;
      const size_t eq = st.find('=');
      if (eq == std::string::npos) throw std::runtime_error("machine profile: expected 'key = value', got: " + st);
      const std::string key = trim(st.substr(0, eq)), value = trim(st.substr(eq + 1));
      double x = 0;
      try {
        size_t pos = 0;
        x = std::stod(value, &pos);
        if (pos != value.size()) throw std::invalid_argument(value);
      } catch (const std::exception&) {
        throw std::runtime_error("machine profile: bad numeric value for '" + key + "': " + value);
      }
      if (!values.emplace(key, x).second) throw std::runtime_error("machine profile: duplicate key: " + key);
    }
    static const char* const required[] = {"peak_gflops", "bw_l1", "bw_l2", "bw_l3",
                                           "bw_dram",     "cap_l1", "cap_l2", "cap_l3"};
    for (const char* key : required)
      if (!values.count(key)) throw std::runtime_error(std::string("machine profile: missing key: ") + key);
    for (const auto& kv : values) {
      bool known = false;
      for (const char* k : required) known = known || kv.first == k;
      if (!known) throw std::runtime_error("machine profile: unknown key: " + kv.first);
    }
    lbg_machine_profile m{};
    std::snprintf(m.name, sizeof m.name, "%s", name ? name : "");
    m.peak_gflops = values["peak_gflops"];
    m.bandwidth_gbs[0] = values["bw_l1"];
    m.bandwidth_gbs[1] = values["bw_l2"];
    m.bandwidth_gbs[2] = values["bw_l3"];
    m.bandwidth_gbs[3] = values["bw_dram"];
    static const char* cp[] = {"cap_l1", "cap_l2", "cap_l3"};
    for (int i = 0; i < 3; ++i) {
      const double c = values[cp[i]];
      if (c < 0 || c != double(uint64_t(c)))
        throw std::runtime_error(std::string("machine profile: ") + cp[i] +
                                 " must be a nonnegative integer byte count");
      m.capacity_bytes[i] = uint64_t(c);
    }
    validate(m);
    *out = m;
  });
}

}  // extern "C"
