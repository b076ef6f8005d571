// ORACLE — TEST INFRASTRUCTURE ONLY (see mb_oracle.hpp header).
// Restatement of /root/reference/proj/core/src/*.cpp hot path; file:line
// citations are relative to /root/reference/proj.
#include "mb_oracle.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <string>
#include <exception>
#include <limits>
#include <map>
#include <memory>
#include <numeric>
#include <thread>

namespace mbo {

namespace {
constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kDegToRad = kPi / 180.0;
constexpr double kZTol = 1e-9;  // potential.cpp:15
}  // namespace

// ============================================================== dense
CMat CMat::identity(int n) {
  CMat I(n, n);
  for (int i = 0; i < n; ++i) I(i, i) = 1.0;
  return I;
}

bool CMat::all_finite() const {
  for (const cd& v : a)
    if (!std::isfinite(v.real()) || !std::isfinite(v.imag())) return false;
  return true;
}

double CMat::norm() const {
  double s = 0;
  for (const cd& v : a) s += v.real() * v.real() + v.imag() * v.imag();
  return std::sqrt(s);
}

// out = A * B (column-major, out(i,j) = sum_k A(i,k) B(k,j), k ascending)
void gemm(const CMat& A, const CMat& B, CMat& out) {
  const int m = A.r, n = B.c, K = A.c;
  out.r = m;
  out.c = n;
  out.a.assign((std::size_t)m * n, cd(0.0, 0.0));
  const double* a = reinterpret_cast<const double*>(A.a.data());
  const double* b = reinterpret_cast<const double*>(B.a.data());
  double* o = reinterpret_cast<double*>(out.a.data());
  for (int j = 0; j < n; ++j) {
    double* oc = o + 2 * (std::size_t)j * m;
    for (int k = 0; k < K; ++k) {
      const double br = b[2 * ((std::size_t)j * K + k)], bi = b[2 * ((std::size_t)j * K + k) + 1];
      const double* ac = a + 2 * (std::size_t)k * m;
      for (int i = 0; i < m; ++i) {
        const double ar = ac[2 * i], ai = ac[2 * i + 1];
        oc[2 * i] += ar * br - ai * bi;
        oc[2 * i + 1] += ar * bi + ai * br;
      }
    }
  }
}

CMat mul(const CMat& A, const CMat& B) {
  CMat o;
  gemm(A, B, o);
  return o;
}

// kernels.cpp:60-80. X A = B  <=>  A^T X^T = B^T; PartialPivLU of A^T with
// abs-score pivoting (Eigen scalar_score_coeff_op = abs), first maximum wins.
namespace {
// STUDY ONLY (MB_ORACLE_SOLVE=gj in the environment; never the default): the
// solve as Gauss-Jordan column elimination on [A; B] with the same pivot
// choice (first maximum of |A(k, j)| over j >= k), the form the device
// kernels use. Separates the elimination form's rounding from everything
// else in accuracy studies (tools/cfg3_accuracy.py).
bool study_gj() {
  static const bool on = [] {
    const char* e = std::getenv("MB_ORACLE_SOLVE");
    return e && std::string(e) == "gj";
  }();
  return on;
}

CMat gauss_jordan_right(const CMat& B, CMat A) {
  const int n = A.r, rhs = B.r;
  CMat X = B;
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::abs(A(k, k));
    for (int j = k + 1; j < n; ++j) {
      const double s = std::abs(A(k, j));
      if (s > best) {
        best = s;
        p = j;
      }
    }
    if (best == 0.0) throw SingularMatrixError("solve_right: exactly singular matrix (zero pivot)");
    if (p != k) {
      for (int i = 0; i < n; ++i) std::swap(A(i, k), A(i, p));
      for (int i = 0; i < rhs; ++i) std::swap(X(i, k), X(i, p));
    }
    const cd inv = 1.0 / A(k, k);
    for (int i = 0; i < n; ++i) A(i, k) *= inv;
    for (int i = 0; i < rhs; ++i) X(i, k) *= inv;
    for (int j = 0; j < n; ++j) {
      if (j == k) continue;
      const cd f = A(k, j);
      for (int i = 0; i < n; ++i) A(i, j) -= f * A(i, k);
      for (int i = 0; i < rhs; ++i) X(i, j) -= f * X(i, k);
    }
  }
  return X;
}
}  // namespace

CMat solve_right(const CMat& B, const CMat& A) {
  if (A.r != A.c) throw SolverError("solve_right: A must be square");
  if (B.c != A.r) throw SolverError("solve_right: dimension mismatch");
  if (!A.all_finite() || !B.all_finite()) throw SolverError("solve_right: nonfinite input");
  if (study_gj()) {
    CMat X = gauss_jordan_right(B, A);
    CMat XA = mul(X, A);
    for (std::size_t i = 0; i < XA.a.size(); ++i) XA.a[i] -= B.a[i];
    const double bnorm = B.norm();
    const double resid = XA.norm() / (bnorm > 0 ? bnorm : 1.0);
    if (!(resid <= 1e-10) || !X.all_finite())
      throw SingularMatrixError("solve_right: ill-conditioned system, relative residual " + std::to_string(resid));
    return X;
  }
  const int n = A.r;
  CMat M(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) M(i, j) = A(j, i);
  std::vector<int> perm(n);
  std::iota(perm.begin(), perm.end(), 0);
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::abs(M(k, k));
    for (int i = k + 1; i < n; ++i) {
      const double s = std::abs(M(i, k));
      if (s > best) {
        best = s;
        p = i;
      }
    }
    if (best != 0.0) {
      if (p != k) {
        for (int j = 0; j < n; ++j) std::swap(M(k, j), M(p, j));
        std::swap(perm[k], perm[p]);
      }
      const cd piv = M(k, k);
      for (int i = k + 1; i < n; ++i) M(i, k) /= piv;
      for (int j = k + 1; j < n; ++j) {
        const cd mkj = M(k, j);
        for (int i = k + 1; i < n; ++i) M(i, j) -= M(i, k) * mkj;
      }
    }
  }
  for (int i = 0; i < n; ++i)
    if (M(i, i) == cd(0.0, 0.0))
      throw SingularMatrixError("solve_right: exactly singular matrix (zero pivot)");
  // Y = M^-1 B^T (n x rhs), rhs = B.r
  const int rhs = B.r;
  CMat Y(n, rhs);
  for (int c = 0; c < rhs; ++c) {
    for (int i = 0; i < n; ++i) Y(i, c) = B(c, perm[i]);
    for (int i = 0; i < n; ++i) {  // unit lower
      cd s = Y(i, c);
      for (int j = 0; j < i; ++j) s -= M(i, j) * Y(j, c);
      Y(i, c) = s;
    }
    for (int i = n - 1; i >= 0; --i) {  // upper
      cd s = Y(i, c);
      for (int j = i + 1; j < n; ++j) s -= M(i, j) * Y(j, c);
      Y(i, c) = s / M(i, i);
    }
  }
  CMat X(rhs, n);
  for (int i = 0; i < rhs; ++i)
    for (int j = 0; j < n; ++j) X(i, j) = Y(j, i);
  const double bnorm = B.norm();
  CMat XA = mul(X, A);
  for (std::size_t i = 0; i < XA.a.size(); ++i) XA.a[i] -= B.a[i];
  const double resid = XA.norm() / (bnorm > 0 ? bnorm : 1.0);
  if (!(resid <= 1e-10) || !X.all_finite())
    throw SingularMatrixError("solve_right: ill-conditioned system, relative residual " +
                              std::to_string(resid));
  return X;
}

// kernels.cpp:82-99
double gershgorin_cond(const CMat& Q) {
  if (Q.r != Q.c) throw SolverError("gershgorin_cond: matrix must be square");
  const int n = Q.r;
  if (n == 0) return 1.0;
  double hi = 0.0, lo = std::numeric_limits<double>::infinity();
  for (int i = 0; i < n; ++i) {
    double r = 0.0;
    for (int j = 0; j < n; ++j)
      if (j != i) r += std::abs(Q(i, j));
    const double d = std::abs(Q(i, i));
    hi = std::max(hi, d + r);
    if (d - r <= 0.0) return std::numeric_limits<double>::infinity();
    lo = std::min(lo, d - r);
  }
  return hi / lo;
}

// ============================================================== lattice
// rods.cpp:14-22
Vec2 Lattice2D::b1() const {
  const double det = a1.x * a2.y - a1.y * a2.x;
  return Vec2{kTwoPi * a2.y / det, -kTwoPi * a2.x / det};
}
Vec2 Lattice2D::b2() const {
  const double det = a1.x * a2.y - a1.y * a2.x;
  return Vec2{-kTwoPi * a1.y / det, kTwoPi * a1.x / det};
}
static double vnorm(const Vec2& v) { return std::sqrt(v.x * v.x + v.y * v.y); }
// rods.cpp:24-30
void Lattice2D::validate() const {
  const double det = a1.x * a2.y - a1.y * a2.x;
  const double scale = vnorm(a1) * vnorm(a2);
  if (!(std::abs(det) > 1e-12 * std::max(scale, 1e-300)))
    throw ConfigError("lattice: basis vectors are degenerate (zero cell area)");
  if (!std::isfinite(a1.x) || !std::isfinite(a1.y) || !std::isfinite(a2.x) || !std::isfinite(a2.y))
    throw ConfigError("lattice: nonfinite basis");
}

namespace {
struct Rod {
  Vec2 k;
  Vec2i m;
};
// rods.cpp:50-66: enumerate |m_i| <= floor(cutoff |a_i| / 2pi + 1e-9), keep
// ||k|| <= cutoff, sort by (||k||, kx, ky) with exact comparisons
std::vector<Rod> enumerate_rods(const Lattice2D& lat, double cutoff) {
  const Vec2 b1 = lat.b1(), b2 = lat.b2();
  const int m1max = (int)std::floor(cutoff * vnorm(lat.a1) / kTwoPi + 1e-9);
  const int m2max = (int)std::floor(cutoff * vnorm(lat.a2) / kTwoPi + 1e-9);
  std::vector<Rod> rods;
  for (int m1 = -m1max; m1 <= m1max; ++m1)
    for (int m2 = -m2max; m2 <= m2max; ++m2) {
      const Vec2 k{m1 * b1.x + m2 * b2.x, m1 * b1.y + m2 * b2.y};
      if (vnorm(k) <= cutoff) rods.push_back({k, Vec2i{m1, m2}});
    }
  std::sort(rods.begin(), rods.end(), [](const Rod& p, const Rod& q) {
    const double np = vnorm(p.k), nq = vnorm(q.k);
    if (np != nq) return np < nq;
    if (p.k.x != q.k.x) return p.k.x < q.k.x;
    return p.k.y < q.k.y;
  });
  return rods;
}

// rods.cpp:67-94: copy rods, deduplicated integer difference table
void finish_rodset(RodSet& rs, const std::vector<Rod>& rods) {
  if (rods.empty() || rods.front().m.x != 0 || rods.front().m.y != 0)
    throw ConfigError("rod set does not contain the zero rod");
  const Vec2 b1 = rs.lattice.b1(), b2 = rs.lattice.b2();
  const int n = (int)rods.size();
  for (const Rod& r : rods) {
    rs.k.push_back(r.k);
    rs.m.push_back(r.m);
  }
  std::map<std::pair<int, int>, int> seen;
  rs.diff_index_.assign((std::size_t)n * n, -1);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      const Vec2i dm{rs.m[j].x - rs.m[k].x, rs.m[j].y - rs.m[k].y};
      auto key = std::make_pair(dm.x, dm.y);
      auto it = seen.find(key);
      int d;
      if (it == seen.end()) {
        d = (int)rs.diff.size();
        seen.emplace(key, d);
        rs.diff.push_back(Vec2{dm.x * b1.x + dm.y * b2.x, dm.x * b1.y + dm.y * b2.y});
        rs.diff_m.push_back(dm);
      } else {
        d = it->second;
      }
      rs.diff_index_[(std::size_t)j * n + k] = d;
    }
}
}  // namespace

// rods.cpp:32-96
RodSet RodSet::build(const Lattice2D& lat, double cutoff) {
  lat.validate();
  if (!(cutoff > 0.0) || !std::isfinite(cutoff))
    throw ConfigError("rod cutoff must be positive and finite");
  RodSet rs;
  rs.lattice = lat;
  rs.cutoff = cutoff;
  finish_rodset(rs, enumerate_rods(lat, cutoff));
  return rs;
}

// EXTENSION: first-n truncation. The cutoff grows until at least n rods are
// enumerated; the global sort order makes the prefix independent of the
// cutoff, so the first n rods are those of the reference order.
RodSet RodSet::build_first(const Lattice2D& lat, int n) {
  lat.validate();
  if (n < 1) throw ConfigError("rod count must be >= 1");
  const double bmin = std::min(vnorm(lat.b1()), vnorm(lat.b2()));
  double cutoff = 0.5 * bmin;
  std::vector<Rod> rods;
  for (;;) {
    rods = enumerate_rods(lat, cutoff);
    if ((int)rods.size() >= n) break;
    cutoff *= 1.25;
  }
  rods.resize((std::size_t)n);
  RodSet rs;
  rs.lattice = lat;
  rs.cutoff = vnorm(rods.back().k);
  finish_rodset(rs, rods);
  return rs;
}

// geometry.cpp:13-17
Vec2 project_incident(double gamma, double theta0_deg, double theta1_deg) {
  const double c0 = std::cos(theta0_deg * kDegToRad);
  const double t1 = theta1_deg * kDegToRad;
  return Vec2{gamma * c0 * std::cos(t1), gamma * c0 * std::sin(t1)};
}

// geometry.cpp:19-28
BeamGeometry::BeamGeometry(double g, double t0, double t1)
    : gamma(g), theta0_deg(t0), theta1_deg(t1) {
  if (!(gamma > 0.0) || !std::isfinite(gamma))
    throw ConfigError("beam: gamma must be positive and finite");
  if (!(t0 > 0.0 && t0 < 90.0))
    throw ConfigError("beam: theta0 must lie in (0, 90) degrees, got " + std::to_string(t0));
  if (!std::isfinite(t1)) throw ConfigError("beam: theta1 must be finite");
  b0 = project_incident(gamma, t0, t1);
  sin_theta0 = std::sin(t0 * kDegToRad);
}

// geometry.cpp:30-57
GammaMatrix GammaMatrix::build(const RodSet& rods, const BeamGeometry& beam) {
  const int n = rods.size();
  GammaMatrix g;
  g.gamma = beam.gamma;
  g.sin_theta0 = beam.sin_theta0;
  g.diag.resize(n);
  g.inv_diag.resize(n);
  g.gamma2.resize(n);
  g.propagating.resize(n);
  const double g2 = beam.gamma * beam.gamma;
  for (int i = 0; i < n; ++i) {
    const double px = beam.b0.x + rods.k[i].x, py = beam.b0.y + rods.k[i].y;
    const double par2 = px * px + py * py;
    const double d = g2 - par2;
    if (std::abs(d) < 1e-12)
      throw ConfigError("rod " + std::to_string(i) +
                        " emerges at grazing: |gamma^2 - ||b0+k||^2| = " + std::to_string(std::abs(d)));
    g.gamma2[i] = d;
    if (d > 0.0) {
      g.diag[i] = cd(std::sqrt(d), 0.0);
      g.propagating[i] = 1;
    } else {
      g.diag[i] = cd(0.0, std::sqrt(-d));
      g.propagating[i] = 0;
    }
    g.inv_diag[i] = 1.0 / g.diag[i];
  }
  return g;
}

// EXTENSION: CODATA m0 c^2 = 510998.95 eV, hc = 12398.419843320026 eV A.
BeamEnergy beam_from_energy(double e) {
  if (!(e > 0.0) || !std::isfinite(e)) throw ConfigError("beam: energy must be positive");
  const double mc2 = 510998.95, hc = 12398.419843320026;
  const double lambda = hc / std::sqrt(e * (e + 2.0 * mc2));
  return BeamEnergy{kTwoPi / lambda, 1.0 + e / mc2};
}

// ============================================================== potential
namespace {
void validate_bottom(double zb) {  // potential.cpp:17-20
  if (!(zb < 0.0) || !std::isfinite(zb))
    throw ConfigError("potential: z_bottom must be negative and finite");
}
void validate_period(double zb, const std::optional<double>& p) {  // potential.cpp:22-28
  if (!p) return;
  if (!(*p > 0.0) || !std::isfinite(*p))
    throw ConfigError("potential: bulk_period must be positive and finite");
  if (*p > -zb + kZTol) throw ConfigError("potential: bulk_period must not exceed |z_bottom|");
}
}  // namespace

PotentialField PotentialField::zero(double zb) {  // potential.cpp:32-38
  validate_bottom(zb);
  PotentialField f;
  f.kind = Kind::Zero;
  f.z_bottom = zb;
  return f;
}

PotentialField PotentialField::gaussian_layers(double zb, std::vector<GaussianLayer> layers,
                                               std::optional<double> period) {  // :40-59
  validate_bottom(zb);
  validate_period(zb, period);
  for (std::size_t i = 0; i < layers.size(); ++i) {
    const GaussianLayer& l = layers[i];
    const bool finite = std::isfinite(l.z_center) && std::isfinite(l.amplitude) &&
                        std::isfinite(l.sigma_xy) && std::isfinite(l.sigma_z) &&
                        std::isfinite(l.absorption);
    if (!finite || !(l.sigma_xy > 0.0) || !(l.sigma_z > 0.0) || l.absorption < 0.0)
      throw ConfigError("potential: layer " + std::to_string(i) +
                        " needs sigma_xy > 0, sigma_z > 0, absorption >= 0, finite values");
  }
  PotentialField f;
  f.kind = Kind::GaussianLayers;
  f.z_bottom = zb;
  f.bulk_period = period;
  f.layers = std::move(layers);
  return f;
}

PotentialField PotentialField::tabulated(double zb, std::vector<double> grid,
                                         std::vector<TabulatedEntry> entries,
                                         std::optional<double> period) {  // :61-88
  validate_bottom(zb);
  validate_period(zb, period);
  if (grid.size() < 2) throw ConfigError("potential: tabulated z_grid needs at least 2 points");
  for (std::size_t i = 0; i + 1 < grid.size(); ++i)
    if (!(grid[i] < grid[i + 1]))
      throw ConfigError("potential: tabulated z_grid must be strictly increasing");
  if (grid.front() > zb + kZTol || grid.back() < -kZTol)
    throw ConfigError("potential: tabulated z_grid must cover [z_bottom, 0]");
  for (const TabulatedEntry& e : entries) {
    if (e.values.size() != grid.size())
      throw ConfigError("potential: tabulated entry has wrong sample count");
    for (const cd& v : e.values)
      if (!std::isfinite(v.real()) || !std::isfinite(v.imag()))
        throw ConfigError("potential: tabulated entry has nonfinite sample");
  }
  PotentialField f;
  f.kind = Kind::Tabulated;
  f.z_bottom = zb;
  f.bulk_period = period;
  f.z_grid = std::move(grid);
  f.entries = std::move(entries);
  return f;
}

PotentialField PotentialField::atoms(double zb, AtomModel model, std::optional<double> period) {  // EXTENSION
  validate_bottom(zb);
  validate_period(zb, period);
  if (!(model.cell_area > 0.0)) throw ConfigError("atoms: cell area must be positive");
  for (const AtomSite& a : model.atoms) {
    if (a.species < 0 || a.species >= (int)model.species.size())
      throw ConfigError("atoms: species index out of range");
    if (!(a.B >= 0.0) || !std::isfinite(a.x) || !std::isfinite(a.y) || !std::isfinite(a.z))
      throw ConfigError("atoms: need finite positions and B >= 0");
    for (int i = 0; i < 4; ++i)
      if (!(model.species[a.species].b[i] + a.B > 0.0))
        throw ConfigError("atoms: form-factor widths b_i + B must be positive");
  }
  if (!(model.absorption >= 0.0)) throw ConfigError("atoms: absorption must be >= 0");
  PotentialField f;
  f.kind = Kind::Atoms;
  f.z_bottom = zb;
  f.bulk_period = period;
  f.model = std::move(model);
  return f;
}

// potential.cpp:90-150 (+ atoms extension)
BoundPotential::BoundPotential(const PotentialField& field, const RodSet& rods) {
  kind_ = field.kind;
  n_ = rods.size();
  ndiff_ = rods.diff_count();
  z_bottom_ = field.z_bottom;
  bulk_period_ = field.bulk_period;
  diff_index_ = rods.diff_index_;
  if (kind_ == PotentialField::Kind::GaussianLayers) {
    layers_ = field.layers;
    for (const GaussianLayer& l : layers_) {
      layer_amp_.push_back(cd(l.amplitude, l.amplitude * l.absorption));
      std::vector<double> lat((std::size_t)ndiff_);
      for (int d = 0; d < ndiff_; ++d) {
        const double sq = rods.diff[d].x * rods.diff[d].x + rods.diff[d].y * rods.diff[d].y;
        lat[d] = std::exp(-sq / (2.0 * l.sigma_xy * l.sigma_xy));
      }
      lateral_.push_back(std::move(lat));
    }
  } else if (kind_ == PotentialField::Kind::Tabulated) {
    z_grid_ = field.z_grid;
    std::map<std::pair<int, int>, const TabulatedEntry*> by_dm;
    for (const TabulatedEntry& e : field.entries) by_dm[{e.dm.x, e.dm.y}] = &e;
    samples_.resize(ndiff_);
    slopes_.resize(ndiff_);
    const std::size_t g = z_grid_.size();
    for (int d = 0; d < ndiff_; ++d) {
      auto it = by_dm.find({rods.diff_m[d].x, rods.diff_m[d].y});
      if (it == by_dm.end())
        throw ConfigError("potential: tabulated field lacks coefficient for rod difference (" +
                          std::to_string(rods.diff_m[d].x) + "," +
                          std::to_string(rods.diff_m[d].y) + ")");
      samples_[d] = it->second->values;
      std::vector<cd>& s = slopes_[d];
      s.resize(g);
      const std::vector<cd>& y = samples_[d];
      const std::vector<double>& z = z_grid_;
      if (g == 2) {
        s[0] = s[1] = (y[1] - y[0]) / (z[1] - z[0]);
      } else {  // potential.cpp:134-148
        for (std::size_t i = 1; i + 1 < g; ++i) {
          const double hl = z[i] - z[i - 1], hr = z[i + 1] - z[i];
          s[i] = ((y[i + 1] - y[i]) / hr * hl + (y[i] - y[i - 1]) / hl * hr) / (hl + hr);
        }
        {
          const double h0 = z[1] - z[0], h1 = z[2] - z[1];
          s[0] = -(2.0 * h0 + h1) / (h0 * (h0 + h1)) * y[0] + (h0 + h1) / (h0 * h1) * y[1] -
                 h0 / (h1 * (h0 + h1)) * y[2];
        }
        {
          const double h0 = z[g - 2] - z[g - 3], h1 = z[g - 1] - z[g - 2];
          s[g - 1] = h1 / (h0 * (h0 + h1)) * y[g - 3] - (h0 + h1) / (h0 * h1) * y[g - 2] +
                     (2.0 * h1 + h0) / (h1 * (h0 + h1)) * y[g - 1];
        }
      }
    }
  } else if (kind_ == PotentialField::Kind::Atoms) {
    // u(dg, z) = (s - i*alpha) * gamma_L * (4 pi / A) *
    //   sum_atoms exp(-i dg.rho_a) sum_i a_i (2 sqrt(pi) / sqrt(b')) exp(-b' |dg|^2 / 16 pi^2)
    //   * exp(-4 pi^2 (z - z_a)^2 / b'),   b' = b_i + B_a
    const AtomModel& M = field.model;
    const cd pre = cd(M.particle_sign, -M.absorption) * (M.gamma_L * 4.0 * kPi / M.cell_area);
    for (const AtomSite& at : M.atoms) {
      const Species& sp = M.species[at.species];
      for (int i = 0; i < 4; ++i) {
        const double bp = sp.b[i] + at.B;
        const double w = sp.a[i] * 2.0 * std::sqrt(kPi) / std::sqrt(bp);
        std::vector<cd> amp((std::size_t)ndiff_);
        for (int d = 0; d < ndiff_; ++d) {
          const double gx = rods.diff[d].x, gy = rods.diff[d].y;
          const double lat = std::exp(-bp * (gx * gx + gy * gy) / (16.0 * kPi * kPi));
          const double ph = -(gx * at.x + gy * at.y);
          amp[d] = pre * (w * lat) * cd(std::cos(ph), std::sin(ph));
        }
        term_z_.push_back(at.z);
        term_alpha_.push_back(4.0 * kPi * kPi / bp);
        term_amp_.push_back(std::move(amp));
      }
    }
  }
}

// potential.cpp:152-167
double BoundPotential::map_z(double z) const {
  if (z > kZTol || !std::isfinite(z))
    throw DomainError("potential evaluated above the surface: z = " + std::to_string(z));
  if (z > 0.0) z = 0.0;
  if (z >= z_bottom_) return z;
  if (z >= z_bottom_ - kZTol) return z_bottom_;
  if (!bulk_period_)
    throw DomainError("potential evaluated below z_bottom without a bulk period: z = " +
                      std::to_string(z));
  const double p = *bulk_period_;
  const double k = std::ceil((z_bottom_ - z) / p - 1e-12);
  double zm = z + k * p;
  if (zm < z_bottom_) zm += p;
  if (zm > z_bottom_ + p) zm = z_bottom_ + p;
  return std::min(zm, 0.0);
}

// potential.cpp:169-199 (+ atoms extension)
void BoundPotential::eval_coeffs(double z, std::vector<cd>& out) const {
  out.assign((std::size_t)ndiff_, cd(0.0, 0.0));
  const double zm = map_z(z);
  if (kind_ == PotentialField::Kind::Zero) return;
  if (kind_ == PotentialField::Kind::GaussianLayers) {
    for (std::size_t l = 0; l < layers_.size(); ++l) {
      const GaussianLayer& gl = layers_[l];
      const double dz = (zm - gl.z_center) / gl.sigma_z;
      const cd depth = layer_amp_[l] * std::exp(-0.5 * dz * dz);
      const std::vector<double>& lat = lateral_[l];
      for (int d = 0; d < ndiff_; ++d) out[d] += depth * lat[d];
    }
    return;
  }
  if (kind_ == PotentialField::Kind::Atoms) {
    for (std::size_t t = 0; t < term_z_.size(); ++t) {
      const double dz = zm - term_z_[t];
      const double g = std::exp(-term_alpha_[t] * dz * dz);
      const std::vector<cd>& amp = term_amp_[t];
      for (int d = 0; d < ndiff_; ++d) out[d] += amp[d] * g;
    }
    return;
  }
  const std::size_t g = z_grid_.size();
  std::size_t i =
      (std::size_t)(std::upper_bound(z_grid_.begin(), z_grid_.end(), zm) - z_grid_.begin());
  if (i == 0) i = 1;
  if (i >= g) i = g - 1;
  const double zl = z_grid_[i - 1], zr = z_grid_[i];
  const double h = zr - zl;
  const double t = std::clamp((zm - zl) / h, 0.0, 1.0);
  const double t2 = t * t, t3 = t2 * t;
  const double h00 = 2 * t3 - 3 * t2 + 1, h10 = t3 - 2 * t2 + t;
  const double h01 = -2 * t3 + 3 * t2, h11 = t3 - t2;
  for (int d = 0; d < ndiff_; ++d)
    out[d] = h00 * samples_[d][i - 1] + h10 * h * slopes_[d][i - 1] + h01 * samples_[d][i] +
             h11 * h * slopes_[d][i];
}

// potential.cpp:201-207
void BoundPotential::eval(double z, CMat& U) const {
  static thread_local std::vector<cd> coeffs;
  eval_coeffs(z, coeffs);
  U.r = U.c = n_;
  U.a.resize((std::size_t)n_ * n_);
  for (int k = 0; k < n_; ++k)
    for (int j = 0; j < n_; ++j) U(j, k) = coeffs[diff_index_[(std::size_t)j * n_ + k]];
}
CMat BoundPotential::eval(double z) const {
  CMat U;
  eval(z, U);
  return U;
}

// ============================================================== slicing
SlicingPlan SlicingPlan::with_count(double zb, long count) {  // slicing.hpp:17-23
  if (!(zb < 0.0) || !std::isfinite(zb))
    throw ConfigError("slicing: z_bottom must be negative and finite");
  if (count < 1) throw ConfigError("slicing: slice count must be >= 1");
  return SlicingPlan{zb, count, -zb / (double)count};
}
SlicingPlan SlicingPlan::with_target_dz(double zb, double dz) {  // slicing.hpp:25-31
  if (!(dz > 0.0) || !std::isfinite(dz)) throw ConfigError("slicing: dz must be positive");
  if (!(zb < 0.0) || !std::isfinite(zb))
    throw ConfigError("slicing: z_bottom must be negative and finite");
  const long count = std::max(1L, std::lround(-zb / dz));
  return with_count(zb, count);
}
StepWindow StepWindow::over(double z0, double z1, long count) {  // stages.hpp:20-23
  if (!(z0 < z1) || count < 1) throw SolverError("step window: need z0 < z1 and count >= 1");
  return StepWindow{z0, z1, count, (z1 - z0) / (double)count};
}

NodeSchedule midpoint_schedule() { return NodeSchedule{{0.5}}; }       // stages.cpp:8
NodeSchedule rk4_schedule() { return NodeSchedule{{0.0, 0.5, 1.0}}; }  // stages.cpp:10
NodeSchedule schedule_from_fracs(std::vector<double> raw) {            // stages.cpp:12-23
  for (double& f : raw) {
    if (std::abs(f) < 1e-12) f = 0.0;
    if (std::abs(f - 1.0) < 1e-12) f = 1.0;
  }
  std::sort(raw.begin(), raw.end());
  std::vector<double> uniq;
  for (double f : raw)
    if (uniq.empty() || f - uniq.back() > 1e-12) uniq.push_back(f);
  return NodeSchedule{std::move(uniq)};
}
double node_z(const StepWindow& w, long step, int node, const NodeSchedule& s) {  // :25-30
  const double f = s.frac[node];
  if (f == 0.0) return w.z(step);
  if (f == 1.0) return w.z(step + 1);
  return w.z(step) + f * w.h;
}

UTable::UTable(const BoundPotential& u, const StepWindow& w, const NodeSchedule& s)
    : sched_(s) {  // stages.cpp:32-47
  const int k = sched_.nodes();
  if (sched_.endpoint_pair()) {
    stride_ = k - 1;
    mats_.resize((std::size_t)(w.count * stride_ + 1));
    for (long i = 0; i < w.count; ++i)
      for (int m = 0; m < stride_; ++m)
        u.eval(node_z(w, i, m, sched_), mats_[(std::size_t)(i * stride_ + m)]);
    u.eval(node_z(w, w.count - 1, k - 1, sched_), mats_.back());
  } else {
    stride_ = k;
    mats_.resize((std::size_t)(w.count * k));
    for (long i = 0; i < w.count; ++i)
      for (int m = 0; m < k; ++m) u.eval(node_z(w, i, m, sched_), mats_[(std::size_t)(i * k + m)]);
  }
}
std::size_t UTable::bytes_estimate(int n, long steps, const NodeSchedule& s) {  // :53-57
  const long slots = s.endpoint_pair() ? steps * (s.nodes() - 1) + 1 : steps * (long)s.nodes();
  return (std::size_t)slots * (std::size_t)n * (std::size_t)n * sizeof(cd);
}

// ============================================================== steppers
// splitting_coefficients.cpp:13-77
namespace {
StepperSpec make_sp4() {
  const double b1 = 0.0829844064174052, b2 = 0.396309801498368, b3 = -0.0390563049223486;
  const double b4 = 1.0 - 2.0 * (b1 + b2 + b3);
  const double a1 = 0.245298957184271, a2 = 0.604872665711080;
  const double a3 = 0.5 - (a1 + a2);
  StepperSpec s;
  s.algorithm = StepAlgorithm::Splitting;
  s.name = "sp4";
  s.variant = SplitVariant::BAB;
  s.drift = {a1, a2, a3, a3, a2, a1};
  s.kick = {b1, b2, b3, b4, b3, b2, b1};
  s.validate();
  return s;
}
StepperSpec make_sp6() {
  const double b1 = 0.0414649985182624, b2 = 0.198128671918067, b3 = -0.0400061921041533;
  const double b4 = 0.0752539843015807, b5 = -0.0115113874206879;
  const double b6 = 0.5 - (b1 + b2 + b3 + b4 + b5);
  const double a1 = 0.123229775946271, a2 = 0.290553797799558, a3 = -0.127049212625417;
  const double a4 = -0.246331761062075, a5 = 0.357208872795928;
  const double a6 = 1.0 - 2.0 * (a1 + a2 + a3 + a4 + a5);
  StepperSpec s;
  s.algorithm = StepAlgorithm::Splitting;
  s.name = "sp6";
  s.variant = SplitVariant::BAB;
  s.drift = {a1, a2, a3, a4, a5, a6, a5, a4, a3, a2, a1};
  s.kick = {b1, b2, b3, b4, b5, b6, b6, b5, b4, b3, b2, b1};
  s.validate();
  return s;
}
StepperSpec make_rk4() {
  StepperSpec s;
  s.validate();
  return s;
}
}  // namespace

const StepperSpec& StepperSpec::rk4() { static const StepperSpec s = make_rk4(); return s; }
const StepperSpec& StepperSpec::sp4() { static const StepperSpec s = make_sp4(); return s; }
const StepperSpec& StepperSpec::sp6() { static const StepperSpec s = make_sp6(); return s; }

StepperSpec StepperSpec::splitting(std::string name, SplitVariant v, std::vector<double> drift,
                                   std::vector<double> kick) {  // proposed.cpp:12-22
  StepperSpec s;
  s.algorithm = StepAlgorithm::Splitting;
  s.name = std::move(name);
  s.variant = v;
  s.drift = std::move(drift);
  s.kick = std::move(kick);
  s.validate();
  return s;
}
const StepperSpec& StepperSpec::by_name(const std::string& name) {  // proposed.cpp:24-29
  if (name == "rk4") return rk4();
  if (name == "sp4") return sp4();
  if (name == "sp6") return sp6();
  throw ConfigError("unknown stepper '" + name + "' (expected rk4, sp4 or sp6)");
}
int StepperSpec::stages() const {  // proposed.cpp:31-34
  if (algorithm == StepAlgorithm::RK4) return 4;
  return variant == SplitVariant::BAB ? (int)drift.size() : (int)kick.size();
}
void StepperSpec::validate() const {  // proposed.cpp:36-60
  if (algorithm == StepAlgorithm::RK4) {
    if (rk_nodes.size() != 4 || rk_weights.size() != 4)
      throw ConfigError("stepper " + name + ": classical tableau needs 4 nodes and weights");
    const double sw = std::accumulate(rk_weights.begin(), rk_weights.end(), 0.0);
    if (std::abs(sw - 1.0) > 1e-13) throw ConfigError("stepper " + name + ": RK weights must sum to 1");
    return;
  }
  const std::size_t nd = drift.size(), nk = kick.size();
  const bool shape_ok = variant == SplitVariant::BAB ? (nk == nd + 1) : (nd == nk + 1);
  if (nd == 0 || nk == 0 || !shape_ok)
    throw ConfigError("stepper " + name + ": BAB needs s drifts and s+1 kicks, ABA the reverse");
  double sa = 0.0, sb = 0.0;
  for (double a : drift) {
    if (!std::isfinite(a)) throw ConfigError("stepper " + name + ": nonfinite drift coefficient");
    sa += a;
  }
  for (double b : kick) {
    if (!std::isfinite(b)) throw ConfigError("stepper " + name + ": nonfinite kick coefficient");
    sb += b;
  }
  if (std::abs(sa - 1.0) > 1e-13 || std::abs(sb - 1.0) > 1e-13)
    throw ConfigError("stepper " + name + ": drift and kick coefficients must each sum to 1");
}

// proposed.cpp:62-100
KickSchedule kick_schedule(const StepperSpec& spec) {
  if (spec.algorithm != StepAlgorithm::Splitting)
    throw SolverError("kick_schedule: not a splitting stepper");
  std::vector<double> fracs;
  if (spec.variant == SplitVariant::BAB) {
    double c = 0.0;
    fracs.push_back(0.0);
    for (double a : spec.drift) {
      c += a;
      fracs.push_back(c);
    }
  } else {
    double c = 0.0;
    for (std::size_t r = 0; r < spec.kick.size(); ++r) {
      c += spec.drift[r];
      fracs.push_back(c);
    }
  }
  KickSchedule ks;
  ks.nodes = schedule_from_fracs(fracs);
  for (double raw : fracs) {
    double f = raw;
    if (std::abs(f) < 1e-12) f = 0.0;
    if (std::abs(f - 1.0) < 1e-12) f = 1.0;
    int best = 0;
    double dist = std::numeric_limits<double>::infinity();
    for (int m = 0; m < ks.nodes.nodes(); ++m) {
      const double d = std::abs(ks.nodes.frac[m] - f);
      if (d < dist) {
        dist = d;
        best = m;
      }
    }
    ks.occ2node.push_back(best);
  }
  return ks;
}
NodeSchedule schedule_for(const StepperSpec& spec) {
  if (spec.algorithm == StepAlgorithm::RK4) return rk4_schedule();
  return kick_schedule(spec).nodes;
}

// proposed.cpp:107-112
void to_tau_rho(const GammaMatrix& g, const PropagationState& st, CMat& T, CMat& R) {
  const int n = st.Q.r, c = st.Q.c;
  T = CMat(n, c);
  R = CMat(n, c);
  const cd i1(0.0, 1.0);
  for (int j = 0; j < c; ++j)
    for (int i = 0; i < n; ++i) {
      const cd gq = g.diag[i] * st.Q(i, j), ip = i1 * st.P(i, j);
      T(i, j) = gq - ip;
      R(i, j) = gq + ip;
    }
}
// proposed.cpp:114-121
PropagationState from_tau_rho(const GammaMatrix& g, const CMat& T, const CMat& R, double z) {
  PropagationState st;
  const int n = T.r, c = T.c;
  st.Q = CMat(n, c);
  st.P = CMat(n, c);
  for (int j = 0; j < c; ++j)
    for (int i = 0; i < n; ++i) {
      st.Q(i, j) = 0.5 * (g.inv_diag[i] * (T(i, j) + R(i, j)));
      st.P(i, j) = cd(0.0, 0.5) * (T(i, j) - R(i, j));
    }
  st.z = z;
  return st;
}
// proposed.cpp:123-128
PropagationState initial_state(const GammaMatrix& g, const CMat& R_init, double z) {
  const int n = g.size();
  CMat R = R_init.size() == 0 ? CMat(n, n) : R_init;
  if (R.r != n || R.c != n) throw SolverError("R_init has wrong dimensions");
  return from_tau_rho(g, CMat::identity(n), R, z);
}

namespace {
// proposed.cpp:133-137: out = U X + diag(g2) X
void apply_w(const CMat& U, const RVec& g2, const CMat& X, CMat& out) {
  gemm(U, X, out);
  for (int j = 0; j < X.c; ++j)
    for (int i = 0; i < X.r; ++i) out(i, j) += g2[i] * X(i, j);
}
// a + s * b, elementwise
CMat axpy(const CMat& a, double s, const CMat& b) {
  CMat o = a;
  for (std::size_t i = 0; i < o.a.size(); ++i) o.a[i] += s * b.a[i];
  return o;
}
void negate(CMat& a) {
  for (cd& v : a.a) v = -v;
}
}  // namespace

// proposed.cpp:141-168
void rk4_step(PropagationState& st, double h, const CMat& U0, const CMat& Um, const CMat& U1,
              const RVec& g2) {
  const double h2 = 0.5 * h;
  CMat k1p, k2p, k3p, k4p, tmp;
  apply_w(U0, g2, st.Q, k1p);
  negate(k1p);
  const CMat& k1q = st.P;
  tmp = axpy(st.Q, h2, k1q);
  apply_w(Um, g2, tmp, k2p);
  negate(k2p);
  CMat k2q = axpy(st.P, h2, k1p);
  tmp = axpy(st.Q, h2, k2q);
  apply_w(Um, g2, tmp, k3p);
  negate(k3p);
  CMat k3q = axpy(st.P, h2, k2p);
  tmp = axpy(st.Q, h, k3q);
  apply_w(U1, g2, tmp, k4p);
  negate(k4p);
  CMat k4q = axpy(st.P, h, k3p);
  const double w = h / 6.0;
  for (std::size_t i = 0; i < st.Q.a.size(); ++i) {
    st.Q.a[i] += w * (k1q.a[i] + 2.0 * k2q.a[i] + 2.0 * k3q.a[i] + k4q.a[i]);
    st.P.a[i] += w * (k1p.a[i] + 2.0 * k2p.a[i] + 2.0 * k3p.a[i] + k4p.a[i]);
  }
}

// proposed.cpp:170-194
void splitting_step(PropagationState& st, double h, const StepperSpec& spec,
                    const std::vector<const CMat*>& U, const RVec& g2) {
  CMat wq;
  if (spec.variant == SplitVariant::BAB) {
    const std::size_t s = spec.drift.size();
    if (U.size() != s + 1) throw SolverError("splitting_step: kick matrix count mismatch");
    for (std::size_t r = 0; r < s; ++r) {
      apply_w(*U[r], g2, st.Q, wq);
      const double cb = h * spec.kick[r], ca = h * spec.drift[r];
      for (std::size_t i = 0; i < st.P.a.size(); ++i) st.P.a[i] -= cb * wq.a[i];
      for (std::size_t i = 0; i < st.Q.a.size(); ++i) st.Q.a[i] += ca * st.P.a[i];
    }
    apply_w(*U[s], g2, st.Q, wq);
    const double cb = h * spec.kick[s];
    for (std::size_t i = 0; i < st.P.a.size(); ++i) st.P.a[i] -= cb * wq.a[i];
  } else {
    const std::size_t s = spec.kick.size();
    if (U.size() != s) throw SolverError("splitting_step: kick matrix count mismatch");
    for (std::size_t r = 0; r < s; ++r) {
      const double ca = h * spec.drift[r], cb = h * spec.kick[r];
      for (std::size_t i = 0; i < st.Q.a.size(); ++i) st.Q.a[i] += ca * st.P.a[i];
      apply_w(*U[r], g2, st.Q, wq);
      for (std::size_t i = 0; i < st.P.a.size(); ++i) st.P.a[i] -= cb * wq.a[i];
    }
    const double ca = h * spec.drift[s];
    for (std::size_t i = 0; i < st.Q.a.size(); ++i) st.Q.a[i] += ca * st.P.a[i];
  }
}

// proposed.cpp:196-202
bool apply_rhst(PropagationState& st, double threshold) {
  const double xi = gershgorin_cond(st.Q);
  if (!(xi > threshold)) return false;
  st.P = solve_right(st.P, st.Q);
  st.Q = CMat::identity(st.Q.r);
  return true;
}

// proposed.cpp:204-208
CMat extract_reflection(const GammaMatrix& g, const PropagationState& st) {
  CMat T, R;
  to_tau_rho(g, st, T, R);
  return solve_right(R, T);
}

namespace {
// proposed.cpp:213-273
class StepDriver {
 public:
  StepDriver(const BoundPotential& u, const GammaMatrix& g, const StepperSpec& spec,
             const UTable* table)
      : u_(u), g_(g), spec_(spec), table_(table) {
    if (spec_.algorithm == StepAlgorithm::Splitting) {
      ks_ = kick_schedule(spec_);
      sched_ = ks_.nodes;
    } else {
      sched_ = rk4_schedule();
    }
    ring_.resize((std::size_t)sched_.nodes());
    kick_ptrs_.resize(ks_.occ2node.size());
  }
  const NodeSchedule& schedule() const { return sched_; }
  void advance(PropagationState& st, const StepWindow& w, long step) {
    const int K = sched_.nodes();
    node_.resize((std::size_t)K);
    for (int m = 0; m < K; ++m) {
      if (table_) {
        node_[(std::size_t)m] = &table_->at(step, m);
        continue;
      }
      const bool reuse_foot =
          m == 0 && sched_.endpoint_pair() && prev_step_ >= 0 && step == prev_step_ + 1;
      if (reuse_foot)
        std::swap(ring_.front(), ring_.back());
      else
        u_.eval(node_z(w, step, m, sched_), ring_[(std::size_t)m]);
      node_[(std::size_t)m] = &ring_[(std::size_t)m];
    }
    prev_step_ = step;
    if (spec_.algorithm == StepAlgorithm::RK4) {
      rk4_step(st, w.h, *node_[0], *node_[1], *node_[2], g_.gamma2);
    } else {
      for (std::size_t occ = 0; occ < ks_.occ2node.size(); ++occ)
        kick_ptrs_[occ] = node_[(std::size_t)ks_.occ2node[occ]];
      splitting_step(st, w.h, spec_, kick_ptrs_, g_.gamma2);
    }
  }
  void reset_window() { prev_step_ = -1; }

 private:
  const BoundPotential& u_;
  const GammaMatrix& g_;
  const StepperSpec& spec_;
  const UTable* table_;
  KickSchedule ks_;
  NodeSchedule sched_;
  std::vector<CMat> ring_;
  std::vector<const CMat*> kick_ptrs_, node_;
  long prev_step_ = -1;
};

// proposed.cpp:275-289
void run_window(StepDriver& driver, PropagationState& st, const StepWindow& w,
                const ProposedOptions& opts, SolveStats* stats, std::size_t step_offset) {
  for (long i = 0; i < w.count; ++i) {
    driver.advance(st, w, i);
    st.z = w.z(i + 1);
    if (!st.Q.all_finite() || !st.P.all_finite())
      throw BreakdownError("propagation state went nonfinite", step_offset + (std::size_t)i);
    try {
      if (apply_rhst(st, opts.rhst_threshold) && stats) ++stats->rhst_transforms;
    } catch (const SingularMatrixError& e) {
      throw BreakdownError(std::string("stabilizing transform: ") + e.what(),
                           step_offset + (std::size_t)i);
    }
  }
}
}  // namespace

// proposed.cpp:293-309
CVec solve_proposed(const BoundPotential& u, const GammaMatrix& g, const SlicingPlan& plan,
                    const StepperSpec& spec, const ProposedOptions& opts, const CMat& R_init,
                    const UTable* table, SolveStats* stats) {
  spec.validate();
  if (u.n() != g.size()) throw SolverError("potential and gamma dimensions disagree");
  const StepWindow w = StepWindow::of_plan(plan);
  StepDriver driver(u, g, spec, table);
  PropagationState st = initial_state(g, R_init, plan.z_bottom);
  run_window(driver, st, w, opts, stats, 0);
  try {
    const CMat R = extract_reflection(g, st);
    CVec col((std::size_t)R.r);
    for (int i = 0; i < R.r; ++i) col[i] = R(i, 0);
    return col;
  } catch (const SingularMatrixError& e) {
    throw BreakdownError(std::string("reflection extraction: ") + e.what(), (std::size_t)w.count);
  }
}

// proposed.cpp:311-342
CMat compute_bulk_reflection_proposed(const BoundPotential& u, const GammaMatrix& g, double dz,
                                      const StepperSpec& spec, const ProposedOptions& opts,
                                      const BulkOptions& bulk) {
  spec.validate();
  if (!u.bulk_period()) throw SolverError("bulk reflection needs a field with a bulk period");
  const double p = *u.bulk_period();
  const double ze = u.z_bottom();
  const long L = std::max(1L, std::lround(p / dz));
  const StepWindow w = StepWindow::over(ze - p, ze, L);
  StepDriver probe(u, g, spec, nullptr);
  UTable table(u, w, probe.schedule());
  StepDriver driver(u, g, spec, &table);
  PropagationState st = initial_state(g, CMat(), w.z0);
  CMat R;
  for (long m = 0; m < bulk.max_periods; ++m) {
    driver.reset_window();
    run_window(driver, st, w, opts, nullptr, (std::size_t)(m * L));
    CMat prev = R;
    try {
      R = extract_reflection(g, st);
    } catch (const SingularMatrixError& e) {
      throw BreakdownError(std::string("bulk reflection read: ") + e.what(), (std::size_t)m);
    }
    if (m > 0) {
      CMat d = R;
      for (std::size_t i = 0; i < d.a.size(); ++i) d.a[i] -= prev.a[i];
      if (d.norm() <= bulk.tol * std::max(1.0, R.norm())) return R;
    }
  }
  throw ConvergenceError("bulk reflection did not settle within " +
                         std::to_string(bulk.max_periods) + " periods");
}

// ============================================================== curve
// curve.cpp:8-20
RVec intensity(const CVec& rho0, const GammaMatrix& g) {
  const int n = (int)rho0.size();
  if (n != g.size()) throw DomainError("intensity: rho/Gamma size mismatch");
  RVec eta((std::size_t)n, 0.0);
  const double g0 = g.diag[0].real(), s0 = g.sin_theta0;
  for (int i = 0; i < n; ++i) {
    if (!g.propagating[i]) continue;
    eta[i] = std::norm(rho0[i]) * s0 * g0 / g.diag[i].real();
  }
  return eta;
}

// sweep.cpp:18-33
AngleGrid AngleGrid::validated(std::vector<double> t0, std::vector<double> t1) {
  if (t0.empty()) throw ConfigError("angle grid: theta0 list is empty");
  if (t1.empty()) throw ConfigError("angle grid: theta1 list is empty");
  for (double t : t0)
    if (!(t > 0.0 && t < 90.0))
      throw ConfigError("angle grid: glancing angles must lie in (0, 90) degrees");
  for (std::size_t i = 1; i < t0.size(); ++i)
    if (!(t0[i] > t0[i - 1])) throw ConfigError("angle grid: theta0 must be strictly increasing");
  for (double t : t1)
    if (!std::isfinite(t)) throw ConfigError("angle grid: theta1 must be finite");
  AngleGrid g;
  g.theta0 = std::move(t0);
  g.theta1 = std::move(t1);
  return g;
}

// sweep.cpp:54-143 (stepper methods only; bulk seed per row as :97-102)
RockingCurve rocking_curve(const PotentialField& field, const RodSet& rods, double gamma,
                           const AngleGrid& grid, const SweepOptions& opts) {
  const auto t_start = std::chrono::steady_clock::now();
  if (!(opts.dz > 0.0) || !std::isfinite(opts.dz))
    throw ConfigError("sweep: dz must be positive and finite");
  const StepperSpec& spec = StepperSpec::by_name(opts.method);
  const BoundPotential bound(field, rods);
  const SlicingPlan plan = opts.slices > 0 ? SlicingPlan::with_count(field.z_bottom, opts.slices)
                                           : SlicingPlan::with_target_dz(field.z_bottom, opts.dz);
  const long rows = grid.rows();
  const int n = rods.size();
  const NodeSchedule sched = schedule_for(spec);
  std::unique_ptr<UTable> table;
  if (rows > 1 && UTable::bytes_estimate(n, plan.count, sched) <= opts.table_budget_bytes)
    table = std::make_unique<UTable>(bound, StepWindow::of_plan(plan), sched);

  RockingCurve curve;
  curve.theta0.resize(rows);
  curve.theta1.resize(rows);
  curve.rods = n;
  curve.eta.assign((std::size_t)rows * n, 0.0);
  curve.rho.assign((std::size_t)rows * n, cd(0.0, 0.0));
  curve.rhst.assign((std::size_t)rows, 0);
  curve.method = opts.method;
  curve.dz = opts.dz;
  curve.rhst_threshold = opts.rhst_threshold;
  const long n_th0 = (long)grid.theta0.size();
  ProposedOptions popts;
  popts.rhst_threshold = opts.rhst_threshold;

  auto solve_row = [&](long row) {
    const double th1 = grid.theta1[(std::size_t)(row / n_th0)];
    const double th0 = grid.theta0[(std::size_t)(row % n_th0)];
    curve.theta0[(std::size_t)row] = th0;
    curve.theta1[(std::size_t)row] = th1;
    const BeamGeometry beam(gamma, th0, th1);
    const GammaMatrix gm = GammaMatrix::build(rods, beam);
    CMat R_init;
    if (bound.bulk_period())
      R_init = compute_bulk_reflection_proposed(bound, gm, opts.dz, spec, popts, BulkOptions{});
    SolveStats stats;
    const CVec rho0 = solve_proposed(bound, gm, plan, spec, popts, R_init, table.get(), &stats);
    const RVec eta = intensity(rho0, gm);
    for (int i = 0; i < n; ++i) {
      curve.eta[(std::size_t)row * n + i] = eta[i];
      curve.rho[(std::size_t)row * n + i] = rho0[i];
    }
    curve.rhst[(std::size_t)row] = stats.rhst_transforms;
  };

  int threads = opts.threads;
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  threads = (int)std::min<long>(threads, rows);
  if (threads <= 1) {
    for (long r = 0; r < rows; ++r) solve_row(r);
  } else {
    std::atomic<long> next{0};
    std::vector<std::exception_ptr> errors((std::size_t)rows);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&] {
        for (;;) {
          const long row = next.fetch_add(1, std::memory_order_relaxed);
          if (row >= rows) return;
          try {
            solve_row(row);
          } catch (...) {
            errors[(std::size_t)row] = std::current_exception();
          }
        }
      });
    for (auto& th : pool) th.join();
    for (long r = 0; r < rows; ++r)
      if (errors[(std::size_t)r]) std::rethrow_exception(errors[(std::size_t)r]);
  }
  curve.solve_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  return curve;
}

// curve.cpp:22-41
double curve_error(const RockingCurve& c, const RockingCurve& r) {
  if (c.rows() != r.rows()) throw CompareError("curve_error: row count mismatch");
  if (c.rods != r.rods) throw CompareError("curve_error: rod count mismatch");
  const double atol = 1e-12;
  for (long i = 0; i < c.rows(); ++i)
    if (std::abs(c.theta0[i] - r.theta0[i]) > atol || std::abs(c.theta1[i] - r.theta1[i]) > atol)
      throw CompareError("curve_error: angle grids differ");
  double num = 0.0, den = 0.0;
  for (long i = 0; i < c.rows(); ++i) {
    double sn = 0, sd = 0;
    for (int j = 0; j < c.rods; ++j) {
      const double dv = c.eta[(std::size_t)i * c.rods + j] - r.eta[(std::size_t)i * r.rods + j];
      sn += dv * dv;
      sd += r.eta[(std::size_t)i * r.rods + j] * r.eta[(std::size_t)i * r.rods + j];
    }
    num = std::max(num, std::sqrt(sn));
    den = std::max(den, std::sqrt(sd));
  }
  if (num == 0.0) return 0.0;
  if (den == 0.0) return std::numeric_limits<double>::infinity();
  return num / den;
}

}  // namespace mbo
