// host_bench.cpp — the reference's kernel-benchmark inputs and report writers
// (host side; the timed GPU run is lbg_run_bench in capi.cu).
//
//   * inputs: P = random_matrix(rng, n, n) * (1/d^2), v0 = random_matrix(rng, n, 1)
//     from std::mt19937_64(seed) with std::uniform_real_distribution(-1, 1),
//     re then im per entry — proj/src/bench.cpp:81-86, include/lb/random.hpp:12-22.
//     Same standard library and no FP contraction: bit-identical to the reference.
//   * CSV: "# lindbench <UTC> machine-profile=<name>" header, the reference's
//     columns (%.6g timings, %.17g checksums, "# failed:" comment + nan row for a
//     failed config) — proj/src/bench.cpp:202-221 — then the GPU columns.
//   * JSON: the document of proj/src/bench.cpp:223-246 as nlohmann::json::dump(2)
//     prints it (keys in sorted order, shortest round-trip numbers, ".0" on
//     integral doubles, e+XX exponents), rows extended with the GPU keys.
#include <charconv>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <map>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lbg.h"

namespace {

thread_local std::string g_bench_err;

const char* variant_name(int v) {  // kernels.cpp to_string(Variant)
  switch (v) {
    case LBG_VARIANT_AOS: return "aos";
    case LBG_VARIANT_SOA: return "soa";
    case LBG_VARIANT_SIMD: return "simd";
    default: return "unknown";
  }
}

const char* algo_name(int a) {
  switch (a) {
    case LBG_ALGO_CHAIN: return "chain";
    case LBG_ALGO_DFMA9: return "dfma9";
    case LBG_ALGO_SMEM: return "smem";
    case LBG_ALGO_TILED: return "tiled";
    case LBG_ALGO_CTA: return "cta";
    case LBG_ALGO_ROWSPLIT: return "rowsplit";
    default: return "none";
  }
}

std::string timestamp_utc() {
  const std::time_t now = std::time(nullptr);
  std::tm tm{};
  gmtime_r(&now, &tm);
  char buf[32];
  std::strftime(buf, sizeof buf, "%Y-%m-%dT%H:%M:%SZ", &tm);
  return buf;
}

std::string fmt(const char* f, double x) {
  char buf[48];
  std::snprintf(buf, sizeof buf, f, x);
  return buf;
}

// nlohmann::json's double printing: shortest round-trip digits, then
// fixed notation for decimal exponents in (-4, 15], else d.ddde+XX.
std::string json_number(double x) {
  if (!std::isfinite(x)) return "null";
  if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
  char sci[64];
  const auto r = std::to_chars(sci, sci + sizeof sci, x, std::chars_format::scientific);
  const std::string s(sci, r.ptr);
  std::string out;
  size_t i = 0;
  if (s[0] == '-') {
    out += '-';
    i = 1;
  }
  const size_t epos = s.find('e');
  std::string digits;
  for (size_t k = i; k < epos; ++k)
    if (s[k] != '.') digits += s[k];
  const int k = int(digits.size());
  const int n = std::stoi(s.substr(epos + 1)) + 1;  // value = 0.d1d2...dk * 10^n
  if (k <= n && n <= 15) {
    out += digits + std::string(size_t(n - k), '0') + ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, size_t(n)) + "." + digits.substr(size_t(n));
  } else if (-4 < n && n <= 0) {
    out += "0." + std::string(size_t(-n), '0') + digits;
  } else {
    out += digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    int e = n - 1;
    out += 'e';
    out += e < 0 ? '-' : '+';
    e = e < 0 ? -e : e;
    char eb[8];
    std::snprintf(eb, sizeof eb, e < 10 ? "0%d" : "%d", e);
    out += eb;
  }
  return out;
}

std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", c);
          o += b;
        } else {
          o += char(c);
        }
    }
  }
  return o + "\"";
}

void emit(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (!len) throw std::invalid_argument("bench writer: null length pointer");
  *len = s.size();
  if (buf) {
    if (cap < s.size() + 1) throw std::invalid_argument("bench writer: buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  }
}

template <class F>
int bench_guard(F&& f) {
  try {
    f();
    return LBG_OK;
  } catch (const std::invalid_argument& e) {
    g_bench_err = e.what();
    return LBG_EINVAL;
  } catch (const std::exception& e) {
    g_bench_err = e.what();
    return LBG_ERUNTIME;
  }
}

}  // namespace

extern "C" {

const char* lbg_bench_last_error(void) { return g_bench_err.c_str(); }

int lbg_bench_inputs(size_t dim, uint64_t seed, double* p, double* v0) {
  return bench_guard([&] {
    if (dim < 1) throw std::invalid_argument("bench: dim must be >= 1");
    if (!p || !v0) throw std::invalid_argument("bench: null output");
    const size_t n = dim * dim;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    const std::complex<double> scale{1.0 / double(dim * dim), 0.0};
    for (size_t e = 0; e < n * n; ++e) {
      const double re = u(rng);
      const double im = u(rng);
      std::complex<double> z{re, im};
      z *= scale;
      p[2 * e] = z.real();
      p[2 * e + 1] = z.imag();
    }
    for (size_t e = 0; e < n; ++e) {
      const double re = u(rng);
      const double im = u(rng);
      v0[2 * e] = re;
      v0[2 * e + 1] = im;
    }
  });
}

int lbg_write_bench_csv(const lbg_bench_config* cfgs, const lbg_bench_result* res, size_t count,
                        const char* machine, char* buf, size_t cap, size_t* len) {
  return bench_guard([&] {
    if (count && (!cfgs || !res)) throw std::invalid_argument("bench writer: null rows");
    std::string s = "# lindbench " + timestamp_utc() + " machine-profile=" + (machine ? machine : "") + "\n";
    s += "profile,dim,variant,reps,warmup,ns_per_step,gflops,gbs,checksum_re,checksum_im,"
         "batch,algo,traj_steps_per_s\n";
    for (size_t i = 0; i < count; ++i) {
      const lbg_bench_config& c = cfgs[i];
      const lbg_bench_result& r = res[i];
      if (r.failed)
        s += "# failed: dim=" + std::to_string(c.dim) + " variant=" + variant_name(c.variant) + ": " +
             std::string(r.error) + "\n";
      s += "b200," + std::to_string(c.dim) + "," + variant_name(c.variant) + "," + std::to_string(c.reps) + "," +
           std::to_string(c.warmup) + ",";
      if (r.failed) {
        s += "nan,nan,nan,nan,nan,";
      } else {
        s += fmt("%.6g", r.ns_per_step) + "," + fmt("%.6g", r.gflops) + "," + fmt("%.6g", r.gbs) + "," +
             fmt("%.17g", r.checksum_re) + "," + fmt("%.17g", r.checksum_im) + ",";
      }
      s += std::to_string(c.batch < 1 ? 1 : c.batch) + "," + algo_name(r.algo) + "," +
           (r.failed ? std::string("nan") : fmt("%.6g", r.traj_steps_per_s)) + "\n";
    }
    emit(s, buf, cap, len);
  });
}

int lbg_write_bench_json(const lbg_bench_config* cfgs, const lbg_bench_result* res, size_t count,
                         const char* machine, char* buf, size_t cap, size_t* len) {
  return bench_guard([&] {
    if (count && (!cfgs || !res)) throw std::invalid_argument("bench writer: null rows");
    std::string s = "{\n  \"machine_profile\": " + json_string(machine ? machine : "") + ",\n  \"results\": ";
    if (count == 0) s += "[]";
    for (size_t i = 0; i < count; ++i) {
      const lbg_bench_config& c = cfgs[i];
      const lbg_bench_result& r = res[i];
      std::map<std::string, std::string> row;  // sorted keys, like nlohmann::json's std::map
      row["profile"] = json_string("b200");
      row["dim"] = std::to_string(c.dim);
      row["variant"] = json_string(variant_name(c.variant));
      row["reps"] = std::to_string(c.reps);
      row["warmup"] = std::to_string(c.warmup);
      row["batch"] = std::to_string(c.batch < 1 ? 1 : c.batch);
      row["algo"] = json_string(algo_name(r.algo));
      if (r.failed) {
        row["failed"] = "true";
        row["error"] = json_string(r.error);
      } else {
        row["ns_per_step"] = json_number(r.ns_per_step);
        row["gflops"] = json_number(r.gflops);
        row["gbs"] = json_number(r.gbs);
        row["checksum_re"] = json_number(r.checksum_re);
        row["checksum_im"] = json_number(r.checksum_im);
        row["traj_steps_per_s"] = json_number(r.traj_steps_per_s);
      }
      s += i == 0 ? "[\n    {\n" : ",\n    {\n";
      size_t k = 0;
      for (const auto& [key, val] : row)
        s += "      " + json_string(key) + ": " + val + (++k < row.size() ? ",\n" : "\n");
      s += "    }";
      if (i + 1 == count) s += "\n  ]";
    }
    s += ",\n  \"timestamp\": " + json_string(timestamp_utc()) + "\n}\n";
    emit(s, buf, cap, len);
  });
}

}  // extern "C"
