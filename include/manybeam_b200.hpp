// manybeam_b200.hpp — C++ host mirror of the reference forward-model API over
// the C-ABI (manybeam_b200.h). Same names, argument meaning and error
// behaviour as /root/reference/proj/core/include/manybeam/*.hpp for the
// stepper path, so reference callers (driver.cpp:15-21, tests) switch by
// changing the namespace:
//
//   manybeam::RodSet::build            rods.hpp:23-47      -> mb_rods_build
//   manybeam::PotentialField::*        potential.hpp:35-61 -> mb_field
//   manybeam::StepperSpec::by_name     proposed.hpp:23-43  -> mb_stepper_by_name
//   manybeam::AngleGrid::validated     sweep.hpp:17-24
//   manybeam::rocking_curve            sweep.hpp:37-38     -> mb_rocking_curve
//   manybeam::curve_error              curve.hpp:38
//
// Errors are rethrown as the reference exception types (types.hpp:20-62);
// BreakdownError carries the step of the first failing row in row order
// (sweep.cpp:136-137). Header-only; link against libmanybeam_b200.so.
#pragma once

#include <array>
#include <cmath>
#include <complex>
#include <limits>
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <fstream>
#include <istream>
#include <memory>
#include <optional>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "manybeam_b200.h"

namespace manybeam::b200 {

using Complex = std::complex<double>;

struct Error : std::runtime_error {
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct ConfigError : Error { using Error::Error; };
struct SolverError : Error { using Error::Error; };
struct SingularMatrixError : SolverError { using SolverError::SolverError; };
struct BreakdownError : SolverError {
  BreakdownError(const std::string& m, std::size_t s) : SolverError(m), step(s) {}
  std::size_t step;
};
struct ConvergenceError : SolverError { using SolverError::SolverError; };
struct DomainError : SolverError { using SolverError::SolverError; };
struct CompareError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };

inline void check(int rc, std::size_t step = 0) {
  if (rc == MB_OK) return;
  const std::string msg = mb_last_error();
  switch (rc) {
    case MB_ERR_CONFIG: throw ConfigError(msg);
    case MB_ERR_SINGULAR: throw SingularMatrixError(msg);
    case MB_ERR_BREAKDOWN: throw BreakdownError(msg, step);
    case MB_ERR_CONVERGENCE: throw ConvergenceError(msg);
    case MB_ERR_DOMAIN: throw DomainError(msg);
    case MB_ERR_CUDA: throw DeviceError(msg);
    case MB_ERR_ARG: throw std::invalid_argument(msg);
    default: throw SolverError(msg);
  }
}

struct Vec2 {
  double x = 0, y = 0;
};

// rods.hpp:10-17
struct Lattice2D {
  Vec2 a1, a2;
};

// rods.hpp:23-47 (+ build_first extension)
class RodSet {
 public:
  static RodSet build(const Lattice2D& lat, double cutoff) { return make(lat, cutoff, 0); }
  static RodSet build_first(const Lattice2D& lat, int n) { return make(lat, 0.0, n); }
  // a rod set given as the reference's tables (rods.hpp:28-37): k[n][2],
  // m[n][2], diff[ndiff][2], diff_m[ndiff][2], diff_index[n*n]
  static RodSet from_tables(std::vector<double> k, std::vector<int> m, std::vector<double> diff,
                            std::vector<int> diff_m, std::vector<int> diff_index) {
    RodSet r;
    r.n_ = (int)(k.size() / 2);
    r.ndiff_ = (int)(diff.size() / 2);
    if (m.size() != k.size() || diff_m.size() != diff.size() || diff_index.size() != (std::size_t)r.n_ * r.n_)
      throw ConfigError("rods: inconsistent table sizes");
    r.k_ = std::move(k);
    r.m_ = std::move(m);
    r.diff_ = std::move(diff);
    r.diff_m_ = std::move(diff_m);
    r.diff_index_ = std::move(diff_index);
    return r;
  }
  int size() const { return n_; }
  int diff_count() const { return ndiff_; }
  Vec2 k(int i) const { return Vec2{k_[2 * i], k_[2 * i + 1]}; }
  std::array<int, 2> m(int i) const { return {m_[2 * i], m_[2 * i + 1]}; }
  int diff_index(int j, int k) const { return diff_index_[(std::size_t)j * n_ + k]; }
  mb_rods view() const {
    return mb_rods{n_, k_.data(), m_.data(), ndiff_, diff_.data(), diff_m_.data(), diff_index_.data()};
  }

 private:
  static RodSet make(const Lattice2D& lat, double cutoff, int first_n) {
    const mb_lattice l{{lat.a1.x, lat.a1.y}, {lat.a2.x, lat.a2.y}};
    RodSet r;
    check(mb_rods_build(&l, cutoff, first_n, &r.n_, &r.ndiff_, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0));
    r.k_.resize(2 * (std::size_t)r.n_);
    r.m_.resize(2 * (std::size_t)r.n_);
    r.diff_.resize(2 * (std::size_t)r.ndiff_);
    r.diff_m_.resize(2 * (std::size_t)r.ndiff_);
    r.diff_index_.resize((std::size_t)r.n_ * r.n_);
    check(mb_rods_build(&l, cutoff, first_n, &r.n_, &r.ndiff_, r.k_.data(), r.m_.data(), r.diff_.data(),
                        r.diff_m_.data(), r.diff_index_.data(), r.n_, r.ndiff_));
    return r;
  }
  int n_ = 0, ndiff_ = 0;
  std::vector<double> k_, diff_;
  std::vector<int> m_, diff_m_, diff_index_;
};

// potential.hpp:17-23
struct GaussianLayer {
  double z_center = 0.0, amplitude = 0.0, sigma_xy = 1.0, sigma_z = 1.0, absorption = 0.0;
};

// potential.hpp:35-61 (+ atoms extension)
class PotentialField {
 public:
  // bulk_period: the structure repeats below z_bottom with this period; the
  // solve is then seeded with the bulk reflection (compute_bulk_reflection_proposed)
  static PotentialField zero(double z_bottom, std::optional<double> bulk_period = {}) {
    PotentialField f;
    f.f_.kind = MB_FIELD_ZERO;
    f.f_.z_bottom = z_bottom;
    f.set_bulk(bulk_period);
    return f;
  }
  static PotentialField gaussian_layers(double z_bottom, const std::vector<GaussianLayer>& layers,
                                        std::optional<double> bulk_period = {}) {
    PotentialField f;
    f.f_.kind = MB_FIELD_GAUSSIAN_LAYERS;
    f.f_.z_bottom = z_bottom;
    f.set_bulk(bulk_period);
    for (const GaussianLayer& l : layers)
      f.d0_.insert(f.d0_.end(), {l.z_center, l.amplitude, l.sigma_xy, l.sigma_z, l.absorption});
    f.f_.nlayers = (int)layers.size();
    return f;
  }
  // entries: (dm, values per grid point)
  static PotentialField tabulated(double z_bottom, const std::vector<double>& z_grid,
                                  const std::vector<std::pair<std::array<int, 2>, std::vector<Complex>>>& entries,
                                  std::optional<double> bulk_period = {}) {
    PotentialField f;
    f.f_.kind = MB_FIELD_TABULATED;
    f.f_.z_bottom = z_bottom;
    f.set_bulk(bulk_period);
    f.d0_ = z_grid;
    for (const auto& e : entries) {
      f.i0_.push_back(e.first[0]);
      f.i0_.push_back(e.first[1]);
      if (e.second.size() != z_grid.size()) throw ConfigError("potential: tabulated entry sample count mismatch");
      for (const Complex& v : e.second) {
        f.d1_.push_back(v.real());
        f.d1_.push_back(v.imag());
      }
    }
    f.f_.ngrid = (int)z_grid.size();
    f.f_.nentries = (int)entries.size();
    return f;
  }
  struct Atom {
    double x, y, z;
    int species;
    double B;
  };
  static PotentialField atoms(double z_bottom, const std::vector<Atom>& atoms,
                              const std::vector<std::array<double, 4>>& ff_a,
                              const std::vector<std::array<double, 4>>& ff_b, double cell_area, double gamma_L,
                              double particle_sign, double absorption = 0.1,
                              std::optional<double> bulk_period = {}) {
    PotentialField f;
    f.f_.kind = MB_FIELD_ATOMS;
    f.f_.z_bottom = z_bottom;
    f.set_bulk(bulk_period);
    for (const Atom& a : atoms) {
      f.d0_.insert(f.d0_.end(), {a.x, a.y, a.z});
      f.i0_.push_back(a.species);
      f.d1_.push_back(a.B);
    }
    for (std::size_t s = 0; s < ff_a.size(); ++s) {
      f.d2_.insert(f.d2_.end(), ff_a[s].begin(), ff_a[s].end());
      f.d3_.insert(f.d3_.end(), ff_b[s].begin(), ff_b[s].end());
    }
    f.f_.natoms = (int)atoms.size();
    f.f_.nspecies = (int)ff_a.size();
    f.f_.cell_area = cell_area;
    f.f_.gamma_L = gamma_L;
    f.f_.particle_sign = particle_sign;
    f.f_.absorption = absorption;
    return f;
  }
  double z_bottom() const { return f_.z_bottom; }
  std::optional<double> bulk_period() const {
    return f_.has_bulk_period ? std::optional<double>(f_.bulk_period) : std::nullopt;
  }
  // C view; pointers refer to this object's storage
  mb_field view() const {
    mb_field v = f_;
    switch (f_.kind) {
      case MB_FIELD_GAUSSIAN_LAYERS:
        v.layers = d0_.data();
        break;
      case MB_FIELD_TABULATED:
        v.z_grid = d0_.data();
        v.entry_dm = i0_.data();
        v.entry_values = d1_.data();
        break;
      case MB_FIELD_ATOMS:
        v.atom_xyz = d0_.data();
        v.atom_species = i0_.data();
        v.atom_B = d1_.data();
        v.ff_a = d2_.data();
        v.ff_b = d3_.data();
        break;
      default:
        break;
    }
    return v;
  }

 private:
  void set_bulk(std::optional<double> p) {
    f_.has_bulk_period = p ? 1 : 0;
    f_.bulk_period = p ? *p : 0.0;
  }
  mb_field f_{};
  std::vector<double> d0_, d1_, d2_, d3_;
  std::vector<int> i0_;
};

// sweep.hpp:17-24, sweep.cpp:18-33
struct AngleGrid {
  std::vector<double> theta0, theta1;
  static AngleGrid validated(std::vector<double> t0, std::vector<double> t1) {
    if (t0.empty()) throw ConfigError("angle grid: theta0 list is empty");
    if (t1.empty()) throw ConfigError("angle grid: theta1 list is empty");
    for (double t : t0)
      if (!(t > 0.0 && t < 90.0)) throw ConfigError("angle grid: glancing angles must lie in (0, 90) degrees");
    for (std::size_t i = 1; i < t0.size(); ++i)
      if (!(t0[i] > t0[i - 1])) throw ConfigError("angle grid: theta0 must be strictly increasing");
    for (double t : t1)
      if (!std::isfinite(t)) throw ConfigError("angle grid: theta1 must be finite");
    return AngleGrid{std::move(t0), std::move(t1)};
  }
  long rows() const { return (long)(theta0.size() * theta1.size()); }
};

// sweep.hpp:26-32 for the stepper methods
struct SweepOptions {
  std::string method = "rk4";  // rk4 | sp4 | sp6 (conventional is not a device method)
  double dz = 0.01;
  long slices = 0;  // EXTENSION: fixed slice count
  double rhst_threshold = 1000.0;
  bool residual_check = true;
  bool fsal = false;
  int device = 0;
  std::vector<int> devices;  // EXTENSION: several GPUs behind one context (mb_context_create_multi)
};

// curve.hpp:19-31
struct RockingCurve {
  std::vector<double> theta0, theta1;
  std::vector<double> eta;  // rows x rods, row-major
  std::vector<Complex> rho;
  std::vector<mb_point_status> status;
  std::vector<std::string> rod_labels;  // "(m1;m2)" per rod (sweep.cpp:77-80)
  int rods = 0;
  std::string method;
  double dz = 0.0, rhst_threshold = 0.0;
  long rows() const { return (long)theta0.size(); }
  double eta_at(long r, int i) const { return eta[(std::size_t)r * rods + i]; }
};

// one device context per process and device, created on first use
inline mb_context* context(int device) {
  struct Holder {
    mb_context* c = nullptr;
    ~Holder() {
      if (c) mb_context_destroy(c);
    }
  };
  static thread_local std::vector<std::unique_ptr<Holder>> ctx;
  if ((int)ctx.size() <= device) ctx.resize((std::size_t)device + 1);
  if (!ctx[(std::size_t)device]) {
    auto h = std::make_unique<Holder>();
    check(mb_context_create(device, &h->c));
    ctx[(std::size_t)device] = std::move(h);
  }
  return ctx[(std::size_t)device]->c;
}

// a multi-device context per process and device list, created on first use
inline mb_context* context(const std::vector<int>& devices) {
  if (devices.empty()) return context(0);
  if (devices.size() == 1) return context(devices.front());
  struct Holder {
    std::vector<int> devs;
    mb_context* c = nullptr;
    ~Holder() {
      if (c) mb_context_destroy(c);
    }
  };
  static thread_local std::vector<std::unique_ptr<Holder>> ctx;
  for (auto& h : ctx)
    if (h->devs == devices) return h->c;
  auto h = std::make_unique<Holder>();
  h->devs = devices;
  check(mb_context_create_multi(devices.data(), (int)devices.size(), &h->c));
  ctx.push_back(std::move(h));
  return ctx.back()->c;
}

// sweep.hpp:37-38
inline RockingCurve rocking_curve(const PotentialField& field, const RodSet& rods, double gamma,
                                  const AngleGrid& grid, const SweepOptions& opts) {
  mb_stepper st{};
  check(mb_stepper_by_name(opts.method.c_str(), &st));
  const mb_options o{opts.dz, opts.slices, opts.rhst_threshold, opts.residual_check ? 1 : 0, opts.fsal ? 1 : 0, 0};
  RockingCurve c;
  c.rods = rods.size();
  const long rows = grid.rows();
  c.eta.assign((std::size_t)rows * c.rods, 0.0);
  c.rho.assign((std::size_t)rows * c.rods, Complex(0.0, 0.0));
  c.status.assign((std::size_t)rows, mb_point_status{});
  for (double t1 : grid.theta1)
    for (double t0 : grid.theta0) {
      c.theta0.push_back(t0);
      c.theta1.push_back(t1);
    }
  c.method = opts.method;
  c.dz = opts.dz;
  c.rhst_threshold = opts.rhst_threshold;
  for (int i = 0; i < rods.size(); ++i)
    c.rod_labels.push_back("(" + std::to_string(rods.m(i)[0]) + ";" + std::to_string(rods.m(i)[1]) + ")");
  const mb_field f = field.view();
  const mb_rods r = rods.view();
  mb_context* ctx = opts.devices.empty() ? context(opts.device) : context(opts.devices);
  const int rc = mb_rocking_curve(ctx, &f, &r, gamma, grid.theta0.data(), (int)grid.theta0.size(),
                                  grid.theta1.data(), (int)grid.theta1.size(), &st, &o, c.eta.data(),
                                  reinterpret_cast<double*>(c.rho.data()), c.status.data());
  std::size_t step = 0;
  for (const mb_point_status& s : c.status)
    if (s.code != MB_POINT_OK) {
      step = (std::size_t)s.step;
      break;
    }
  check(rc, step);
  return c;
}

// proposed.hpp:94-102 (SolveStats, solve_proposed): one beam direction,
// the state seeded with a caller-supplied R_init (n x n row-major; empty =
// zero, initial_state proposed.cpp:123-128) at z_bottom; returns rho0, the
// first column of R at the surface. Errors as the reference: "R_init has
// wrong dimensions" (SolverError, proposed.cpp:126), BreakdownError with the
// step for a nonfinite state, a failed RHST or a failed extraction.
struct SolveStats {
  long rhst_transforms = 0;
};

inline std::vector<Complex> solve_proposed(const PotentialField& field, const RodSet& rods, double gamma,
                                           double theta0_deg, double theta1_deg, const SweepOptions& opts,
                                           const std::vector<Complex>& R_init = {}, SolveStats* stats = nullptr) {
  const std::size_t n = (std::size_t)rods.size();
  if (!R_init.empty() && R_init.size() != n * n) throw SolverError("R_init has wrong dimensions");
  mb_stepper st{};
  check(mb_stepper_by_name(opts.method.c_str(), &st));
  if (st.algorithm == MB_STEP_CONVENTIONAL) throw ConfigError("solve_proposed: rk4, sp4 or sp6");
  const mb_options o{opts.dz, opts.slices, opts.rhst_threshold, opts.residual_check ? 1 : 0, opts.fsal ? 1 : 0, 0};
  const mb_field f = field.view();
  const mb_rods r = rods.view();
  const mb_pair pair{0, theta0_deg, theta1_deg};
  mb_context* ctx = context(opts.device);
  struct Guard {
    mb_plan* p = nullptr;
    ~Guard() {
      if (p) mb_plan_destroy(p);
    }
  } g;
  check(mb_plan_create_seeded(ctx, &r, &f, 1, gamma, &pair, 1, &st, &o,
                              R_init.empty() ? nullptr : reinterpret_cast<const double*>(R_init.data()),
                              R_init.empty() ? 0 : 1, &g.p));
  check(mb_plan_execute(g.p, nullptr));
  std::vector<double> eta(n);
  std::vector<Complex> rho(n);
  mb_point_status ps{};
  const int rc = mb_plan_results(g.p, eta.data(), reinterpret_cast<double*>(rho.data()), &ps);
  check(rc, (std::size_t)ps.step);
  if (stats) stats->rhst_transforms = ps.rhst_count;
  return rho;
}

// curve.cpp:22-41
inline double curve_error(const RockingCurve& cand, const RockingCurve& ref) {
  if (cand.rows() != ref.rows()) throw CompareError("curve_error: row count mismatch");
  if (cand.rods != ref.rods) throw CompareError("curve_error: rod count mismatch");
  for (long r = 0; r < cand.rows(); ++r)
    if (std::abs(cand.theta0[r] - ref.theta0[r]) > 1e-12 || std::abs(cand.theta1[r] - ref.theta1[r]) > 1e-12)
      throw CompareError("curve_error: angle grids differ");
  double num = 0.0, den = 0.0;
  for (long r = 0; r < cand.rows(); ++r) {
    double sn = 0.0, sd = 0.0;
    for (int i = 0; i < cand.rods; ++i) {
      const double d = cand.eta_at(r, i) - ref.eta_at(r, i);
      sn += d * d;
      sd += ref.eta_at(r, i) * ref.eta_at(r, i);
    }
    num = std::max(num, std::sqrt(sn));
    den = std::max(den, std::sqrt(sd));
  }
  if (num == 0.0) return 0.0;
  if (den == 0.0) return std::numeric_limits<double>::infinity();
  return num / den;
}


// ---- curve CSV: the reference's wire format (csvio.cpp:65-149, SURVEY §8f
// row 2): "# key: value" metadata, header theta0,theta1,eta(m1;m2)..., every
// number as %.14E, byte-deterministic for a given curve.
inline std::string format_full(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.14E", v);
  std::string s(buf);
  std::replace(s.begin(), s.end(), ',', '.');  // an embedding app's locale must not leak in
  return s;
}

inline void write_curve_csv(std::ostream& os, const RockingCurve& c) {
  os << "# manybeam-curve v1\n# method: " << c.method << "\n# dz: " << format_full(c.dz) << "\n";
  if (c.method != "conventional")
    os << "# rhst_threshold: " << (std::isinf(c.rhst_threshold) ? std::string("inf") : format_full(c.rhst_threshold))
       << "\n";
  os << "# rods: " << c.rods << "\ntheta0,theta1";
  for (const std::string& l : c.rod_labels) os << ",eta" << l;
  os << "\n";
  for (long r = 0; r < c.rows(); ++r) {
    os << format_full(c.theta0[(std::size_t)r]) << ',' << format_full(c.theta1[(std::size_t)r]);
    for (int i = 0; i < c.rods; ++i) os << ',' << format_full(c.eta_at(r, i));
    os << "\n";
  }
}

inline void write_curve_csv(const std::string& path, const RockingCurve& c) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw IoError("cannot open '" + path + "' for writing");
  write_curve_csv(os, c);
  os.flush();
  if (!os) throw IoError("write to '" + path + "' failed");
}

inline RockingCurve read_curve_csv(std::istream& is) {
  auto trim = [](const std::string& x) {
    const std::size_t a = x.find_first_not_of(" \t\r\n");
    if (a == std::string::npos) return std::string();
    return x.substr(a, x.find_last_not_of(" \t\r\n") - a + 1);
  };
  auto number = [](const std::string& f, const char* what) {
    if (f == "inf") return std::numeric_limits<double>::infinity();
    double v = 0.0;
    const auto [ptr, ec] = std::from_chars(f.data(), f.data() + f.size(), v, std::chars_format::general);
    if (ec != std::errc() || ptr != f.data() + f.size())
      throw IoError(std::string("curve csv: bad ") + what + " value '" + f + "'");
    return v;
  };
  RockingCurve c;
  std::string line;
  std::size_t ncols = 0;
  while (std::getline(is, line)) {
    const std::string t = trim(line);
    if (t.empty()) continue;
    if (t[0] == '#') {
      const std::size_t colon = t.find(':');
      if (colon == std::string::npos) continue;
      const std::string key = trim(t.substr(1, colon - 1)), val = trim(t.substr(colon + 1));
      if (key == "method") c.method = val;
      if (key == "dz") c.dz = number(val, "dz");
      if (key == "rhst_threshold") c.rhst_threshold = number(val, "threshold");
      continue;
    }
    std::vector<std::string> fields;
    for (std::size_t a = 0;;) {
      const std::size_t b = t.find(',', a);
      fields.push_back(trim(t.substr(a, b == std::string::npos ? std::string::npos : b - a)));
      if (b == std::string::npos) break;
      a = b + 1;
    }
    if (ncols == 0) {
      if (fields.size() < 3 || fields[0] != "theta0" || fields[1] != "theta1")
        throw IoError("curve csv: expected header starting with theta0,theta1");
      for (std::size_t i = 2; i < fields.size(); ++i) {
        if (fields[i].rfind("eta", 0) != 0) throw IoError("curve csv: intensity columns must be named eta(...)");
        c.rod_labels.push_back(fields[i].substr(3));
      }
      ncols = fields.size();
      continue;
    }
    if (fields.size() != ncols)
      throw IoError("curve csv: row has " + std::to_string(fields.size()) + " fields, expected " +
                    std::to_string(ncols));
    c.theta0.push_back(number(fields[0], "theta0"));
    c.theta1.push_back(number(fields[1], "theta1"));
    for (std::size_t i = 2; i < ncols; ++i) c.eta.push_back(number(fields[i], "eta"));
  }
  if (ncols == 0) throw IoError("curve csv: missing header row");
  if (c.theta0.empty()) throw IoError("curve csv: no data rows");
  c.rods = (int)ncols - 2;
  return c;
}

inline RockingCurve read_curve_csv(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw IoError("cannot open '" + path + "'");
  return read_curve_csv(is);
}

// the CLI's `compare a.csv b.csv` (main.cpp): curve_error of two stored curves
inline double compare_curve_files(const std::string& candidate, const std::string& reference) {
  return curve_error(read_curve_csv(candidate), read_curve_csv(reference));
}

}  // namespace manybeam::b200
