// host_io.cpp — model files and the matrix interchange format (host side).
//
// Restates, for the engine's C-ABI, the reference's text formats so a user of
// lindbench can bring their model files and dumped matrices unchanged:
//   * matrix interchange: header "complex-matrix <rows> <cols>", then one
//     "<re> <im>" pair per element, row-major, 17 significant digits (bit-exact
//     round trip) — proj/src/complex_matrix.cpp:166-188;
//   * model files: flat "key = value" text, '#' comments, keys dim /
//     hamiltonian / collapse (matrices on the following lines) or
//     preset = transmon with optional t1 / tphi / anharmonicity / drive_amp
//     ('inf' disables a channel) — proj/src/model_io.cpp:37-109, with the
//     transmon preset of proj/src/lindblad.cpp:82-100.
// Errors: malformed text -> LBG_ERUNTIME (std::runtime_error in the
// reference); an invalid model (non-Hermitian H) -> LBG_EINVAL.
#include <cctype>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <limits>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lbg.h"

namespace {

using cplx = std::complex<double>;
thread_local std::string g_io_err;

struct Mat {
  size_t rows = 0, cols = 0;
  std::vector<cplx> a;
};

struct bad_input : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct bad_model : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

std::string trim(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
  while (e > b && std::isspace(static_cast<unsigned char>(s[e - 1]))) --e;
  return s.substr(b, e - b);
}

Mat read_matrix(std::istream& is) {
  std::string tag;
  Mat m;
  if (!(is >> tag) || tag != "complex-matrix" || !(is >> m.rows >> m.cols))
    throw bad_input("read_matrix: expected 'complex-matrix <rows> <cols>' header");
  m.a.resize(m.rows * m.cols);
  for (auto& z : m.a) {
    double re = 0.0, im = 0.0;
    if (!(is >> re >> im)) throw bad_input("read_matrix: truncated matrix body");
    z = cplx(re, im);
  }
  return m;
}

double parse_number(const std::string& key, const std::string& value) {
  try {
    size_t pos = 0;
    const double x = std::stod(value, &pos);
    if (pos != value.size()) throw std::invalid_argument(value);
    return x;
  } catch (const std::exception&) {
    throw bad_input("model file: bad numeric value for '" + key + "': " + value);
  }
}

bool hermitian(const Mat& h) {  // lindblad.cpp:13-20, relative 1e-12
  double worst = 0.0, scale = 0.0;
  for (size_t i = 0; i < h.rows; ++i)
    for (size_t j = 0; j < h.cols; ++j) {
      worst = std::max(worst, std::abs(h.a[i * h.cols + j] - std::conj(h.a[j * h.cols + i])));
      scale = std::max(scale, std::abs(h.a[i * h.cols + j]));
    }
  return scale == 0.0 ? worst == 0.0 : worst <= 1e-12 * scale;
}

// three-level transmon preset (lindblad.cpp:82-100), same arithmetic order
void transmon(double t1, double tphi, double anharm, double drive, Mat& h, std::vector<Mat>& ops) {
  if (!(t1 > 0.0) || !(tphi > 0.0)) throw bad_model("transmon_model: t1 and tphi must be positive");
  const size_t d = 3;
  std::vector<cplx> a(9), ad(9);
  a[0 * 3 + 1] = std::sqrt(1.0);
  a[1 * 3 + 2] = std::sqrt(2.0);
  for (size_t i = 0; i < 3; ++i)
    for (size_t j = 0; j < 3; ++j) ad[j * 3 + i] = std::conj(a[i * 3 + j]);
  auto mm = [](const std::vector<cplx>& x, const std::vector<cplx>& y) {
    std::vector<double> o(18, 0.0);
    for (size_t i = 0; i < 3; ++i)
      for (size_t k = 0; k < 3; ++k) {
        const double xr = x[i * 3 + k].real(), xi = x[i * 3 + k].imag();
        for (size_t j = 0; j < 3; ++j) {
          const double yr = y[k * 3 + j].real(), yi = y[k * 3 + j].imag();
          o[2 * (i * 3 + j)] += xr * yr - xi * yi;
          o[2 * (i * 3 + j) + 1] += xr * yi + xi * yr;
        }
      }
    std::vector<cplx> r(9);
    for (size_t e = 0; e < 9; ++e) r[e] = cplx(o[2 * e], o[2 * e + 1]);
    return r;
  };
  h.rows = h.cols = d;
  h.a.assign(9, cplx());
  for (size_t e = 0; e < 9; ++e) h.a[e] = cplx{drive / 2.0, 0.0} * (a[e] + ad[e]);
  const std::vector<cplx> n4 = mm(mm(ad, ad), mm(a, a));
  for (size_t e = 0; e < 9; ++e) h.a[e] += cplx{anharm / 2.0, 0.0} * n4[e];
  ops.clear();
  if (std::isfinite(t1)) {
    Mat l{d, d, std::vector<cplx>(9)};
    for (size_t e = 0; e < 9; ++e) l.a[e] = cplx{std::sqrt(1.0 / t1), 0.0} * a[e];
    ops.push_back(l);
  }
  if (std::isfinite(tphi)) {
    const std::vector<cplx> num = mm(ad, a);
    Mat l{d, d, std::vector<cplx>(9)};
    for (size_t e = 0; e < 9; ++e) l.a[e] = cplx{std::sqrt(1.0 / (2.0 * tphi)), 0.0} * num[e];
    ops.push_back(l);
  }
}

void read_model(std::istream& is, Mat& h, std::vector<Mat>& ops) {
  std::optional<size_t> dim;
  std::optional<Mat> ham;
  std::vector<Mat> coll;
  bool preset = false;
  double t1 = 30e-6, tphi = 20e-6, anharm = -1.5e9, drive = 1.5e8;  // lindblad.hpp:42-45
  std::string line;
  while (std::getline(is, line)) {
    const std::string st = trim(line);
    if (st.empty() || st[0] == '#') continue;
    const size_t eq = st.find('=');
    if (eq == std::string::npos) throw bad_input("model file: expected 'key = value', got: " + st);
    const std::string key = trim(st.substr(0, eq)), value = trim(st.substr(eq + 1));
    if (key == "dim") {
      const double x = parse_number(key, value);
      if (x < 1 || x != static_cast<double>(static_cast<size_t>(x)))
        throw bad_input("model file: dim must be a positive integer");
      dim = static_cast<size_t>(x);
    } else if (key == "hamiltonian" || key == "collapse") {
      if (!value.empty()) throw bad_input("model file: matrix must start on the line after '" + key + " ='");
      if (key == "hamiltonian") {
        if (ham) throw bad_input("model file: duplicate hamiltonian");
        ham = read_matrix(is);
      } else {
        coll.push_back(read_matrix(is));
      }
    } else if (key == "preset") {
      if (value != "transmon") throw bad_input("model file: unknown preset: " + value);
      preset = true;
    } else if (key == "t1") {
      t1 = parse_number(key, value);
    } else if (key == "tphi") {
      tphi = parse_number(key, value);
    } else if (key == "anharmonicity") {
      anharm = parse_number(key, value);
    } else if (key == "drive_amp") {
      drive = parse_number(key, value);
    } else {
      throw bad_input("model file: unknown key: " + key);
    }
  }
  if (preset) {
    if (dim || ham || !coll.empty())
      throw bad_input("model file: preset = transmon excludes dim/hamiltonian/collapse keys");
    transmon(t1, tphi, anharm, drive, h, ops);
    return;
  }
  if (!dim) throw bad_input("model file: missing dim");
  if (!ham) throw bad_input("model file: missing hamiltonian");
  if (ham->rows != *dim || ham->cols != *dim) throw bad_input("model file: hamiltonian shape does not match dim");
  for (const auto& l : coll)
    if (l.rows != *dim || l.cols != *dim)
      throw bad_input("model file: collapse operator shape does not match dim");
  if (!hermitian(*ham)) throw bad_model("make_model: Hamiltonian is not Hermitian within 1e-12");
  h = std::move(*ham);
  ops = std::move(coll);
}

template <class F>
int io_guard(F&& f) {
  try {
    f();
    return LBG_OK;
  } catch (const std::invalid_argument& e) {
    g_io_err = e.what();
    return LBG_EINVAL;
  } catch (const std::exception& e) {
    g_io_err = e.what();
    return LBG_ERUNTIME;
  }
}

}  // namespace

extern "C" {

const char* lbg_io_last_error(void) { return g_io_err.c_str(); }

int lbg_write_matrix(const double* a, size_t rows, size_t cols, char* buf, size_t cap, size_t* len) {
  return io_guard([&] {
    std::string s = "complex-matrix " + std::to_string(rows) + " " + std::to_string(cols) + "\n";
    char tmp[64];
    for (size_t e = 0; e < rows * cols; ++e) {
      std::snprintf(tmp, sizeof tmp, "%.17g %.17g\n", a[2 * e], a[2 * e + 1]);
      s += tmp;
    }
    *len = s.size();
    if (buf) {
      if (cap < s.size() + 1) throw bad_input("write_matrix: buffer too small");
      std::memcpy(buf, s.c_str(), s.size() + 1);
    }
  });
}

int lbg_read_matrix(const char* text, size_t* rows, size_t* cols, double* out, size_t cap_elems) {
  return io_guard([&] {
    std::istringstream is(text ? text : "");
    const Mat m = read_matrix(is);
    *rows = m.rows;
    *cols = m.cols;
    if (out) {
      if (cap_elems < m.a.size()) throw bad_input("read_matrix: output too small");
      std::memcpy(out, m.a.data(), m.a.size() * sizeof(cplx));
    }
  });
}

int lbg_read_model(const char* text, size_t* d, size_t* n_ops, double* h, double* ops, size_t cap_ops) {
  return io_guard([&] {
    std::istringstream is(text ? text : "");
    Mat hm;
    std::vector<Mat> om;
    read_model(is, hm, om);
    *d = hm.rows;
    *n_ops = om.size();
    if (h) std::memcpy(h, hm.a.data(), hm.a.size() * sizeof(cplx));
    if (ops) {
      if (cap_ops < om.size()) throw bad_input("read_model: too many collapse operators for buffer");
      for (size_t k = 0; k < om.size(); ++k)
        std::memcpy(ops + 2 * k * hm.rows * hm.rows, om[k].a.data(), om[k].a.size() * sizeof(cplx));
    }
  });
}

}  // extern "C"
