// ORACLE — TEST INFRASTRUCTURE ONLY. Not product code.
//
// CPU restatement of the reference forward-model hot path (arXiv 2306.00271,
// `manybeam` C++ project at /root/reference/proj). Only tests/, the
// __graft_entry__.smoke() checker and bench.py's cpu_baseline / --impl reference
// legs may load this. It is the checker, never the measured product path.
//
// Every function cites the reference file:line it restates (paths relative to
// /root/reference/proj). The reference depends on Eigen 3.3+ (absent here, no
// network); dense complex arithmetic is restated with plain loops: GEMM
// summation order and LU pivot scoring follow Eigen's semantics (abs-score
// partial pivoting on A^T, `kernels.cpp:60-80`) but not its blocking, so
// results agree with a real Eigen build to rounding only.
//
// Extensions that are NOT in the reference (shared with the product by
// convention, restated independently there):
//   * RodSet::build_first — first-N truncation of the reference sort key.
//   * Atom potential (Kind::Atoms) — SURVEY.md §8a row P0 formula.
//   * beam_from_energy — relativistic energy -> (gamma, gamma_L).
// Parity pinning: tests/test_oracle_*.py run the reference's own known-answer
// tests (closed forms, invariances) against this restatement.
#pragma once

#include <complex>
#include <cstddef>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace mbo {

using cd = std::complex<double>;

// ---------------------------------------------------------------- errors
// types.hpp:20-62
struct Error : std::runtime_error {
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct ConfigError : Error { using Error::Error; };
struct SolverError : Error { using Error::Error; };
struct SingularMatrixError : SolverError { using SolverError::SolverError; };
struct BreakdownError : SolverError {
  BreakdownError(const std::string& m, std::size_t s)
      : SolverError(m + " (step " + std::to_string(s) + ")"), step(s) {}
  std::size_t step;
};
struct ConvergenceError : SolverError { using SolverError::SolverError; };
struct DomainError : SolverError { using SolverError::SolverError; };
struct CompareError : Error { using Error::Error; };

// ---------------------------------------------------------------- dense
// Column-major complex matrix (types.hpp:11-14 convention).
struct CMat {
  int r = 0, c = 0;
  std::vector<cd> a;
  CMat() = default;
  CMat(int rows, int cols) : r(rows), c(cols), a((std::size_t)rows * cols) {}
  static CMat identity(int n);
  cd& operator()(int i, int j) { return a[(std::size_t)j * r + i]; }
  const cd& operator()(int i, int j) const { return a[(std::size_t)j * r + i]; }
  int size() const { return r * c; }
  bool all_finite() const;
  double norm() const;  // Frobenius, sqrt(squaredNorm) as Eigen
};
using CVec = std::vector<cd>;
using RVec = std::vector<double>;

void gemm(const CMat& A, const CMat& B, CMat& out);  // out = A*B
CMat mul(const CMat& A, const CMat& B);

// kernels.cpp:60-80 : X = B * inv(A) via PartialPivLU(A^T), zero-pivot check,
// residual gate 1e-10.
CMat solve_right(const CMat& B, const CMat& A);
// kernels.cpp:82-99
double gershgorin_cond(const CMat& Q);

// ---------------------------------------------------------------- lattice
struct Vec2 { double x = 0, y = 0; };
struct Vec2i { int x = 0, y = 0; };

// rods.hpp:9-17, rods.cpp:14-30
struct Lattice2D {
  Vec2 a1, a2;
  Vec2 b1() const;
  Vec2 b2() const;
  void validate() const;
};

// rods.hpp:23-47, rods.cpp:32-96
struct RodSet {
  static RodSet build(const Lattice2D& lat, double cutoff);
  // EXTENSION: the first `n` rods of the reference order (||k||, kx, ky),
  // diff table rebuilt on the truncated set.
  static RodSet build_first(const Lattice2D& lat, int n);
  int size() const { return (int)k.size(); }
  int diff_count() const { return (int)diff.size(); }
  int diff_index(int j, int kk) const { return diff_index_[(std::size_t)j * k.size() + kk]; }

  Lattice2D lattice;
  double cutoff = 0;
  std::vector<Vec2> k;
  std::vector<Vec2i> m;
  std::vector<Vec2> diff;
  std::vector<Vec2i> diff_m;
  std::vector<int> diff_index_;
};

// geometry.cpp:13-28
Vec2 project_incident(double gamma, double theta0_deg, double theta1_deg);
struct BeamGeometry {
  BeamGeometry(double gamma, double theta0_deg, double theta1_deg);
  double gamma, theta0_deg, theta1_deg;
  Vec2 b0;
  double sin_theta0;
};
// geometry.cpp:30-57
struct GammaMatrix {
  static GammaMatrix build(const RodSet& rods, const BeamGeometry& beam);
  int size() const { return (int)diag.size(); }
  CVec diag, inv_diag;
  RVec gamma2;
  std::vector<char> propagating;
  double gamma = 0, sin_theta0 = 0;
};

// EXTENSION: relativistic beam from kinetic energy (eV). gamma = 2 pi / lambda,
// lambda = hc / sqrt(E (E + 2 m0 c^2)); gamma_L = 1 + E / m0 c^2.
struct BeamEnergy { double gamma, gamma_L; };
BeamEnergy beam_from_energy(double energy_ev);

// ---------------------------------------------------------------- potential
// potential.hpp:17-23
struct GaussianLayer {
  double z_center = 0, amplitude = 0, sigma_xy = 1, sigma_z = 1, absorption = 0;
};
// potential.hpp:27-30
struct TabulatedEntry {
  Vec2i dm;
  std::vector<cd> values;
};
// EXTENSION: atom list with 4-Gaussian electron form
// factors, per-atom Debye-Waller B, absorptive imaginary part.
struct AtomSite {
  double x = 0, y = 0, z = 0;  // Cartesian, A
  int species = 0;
  double B = 0;  // Debye-Waller, A^2
};
struct Species {
  double a[4] = {0, 0, 0, 0};  // A
  double b[4] = {1, 1, 1, 1};  // A^2
};
struct AtomModel {
  std::vector<AtomSite> atoms;
  std::vector<Species> species;
  double cell_area = 1;     // A^2
  double gamma_L = 1;       // relativistic mass factor
  double particle_sign = 1; // +1 electron, -1 positron
  double absorption = 0.1;  // u = (sign - i*absorption) * V
};

// potential.hpp:35-61, potential.cpp:30-88 (+ Atoms extension)
class PotentialField {
 public:
  enum class Kind { Zero, GaussianLayers, Tabulated, Atoms };
  static PotentialField zero(double z_bottom);
  static PotentialField gaussian_layers(double z_bottom, std::vector<GaussianLayer> layers,
                                        std::optional<double> bulk_period = {});
  static PotentialField tabulated(double z_bottom, std::vector<double> z_grid,
                                  std::vector<TabulatedEntry> entries,
                                  std::optional<double> bulk_period = {});
  static PotentialField atoms(double z_bottom, AtomModel model, std::optional<double> bulk_period = {});
  Kind kind = Kind::Zero;
  double z_bottom = -1;
  std::optional<double> bulk_period;
  std::vector<GaussianLayer> layers;
  std::vector<double> z_grid;
  std::vector<TabulatedEntry> entries;
  AtomModel model;
};

// potential.hpp:67-100, potential.cpp:90-207
class BoundPotential {
 public:
  BoundPotential(const PotentialField& field, const RodSet& rods);
  int n() const { return n_; }
  int ndiff() const { return ndiff_; }
  double z_bottom() const { return z_bottom_; }
  const std::optional<double>& bulk_period() const { return bulk_period_; }
  void eval_coeffs(double z, std::vector<cd>& out) const;
  void eval(double z, CMat& U) const;
  CMat eval(double z) const;
  double map_z(double z) const;

 private:
  PotentialField::Kind kind_;
  int n_ = 0, ndiff_ = 0;
  double z_bottom_ = -1;
  std::optional<double> bulk_period_;
  std::vector<int> diff_index_;
  std::vector<GaussianLayer> layers_;
  std::vector<cd> layer_amp_;
  std::vector<std::vector<double>> lateral_;
  std::vector<double> z_grid_;
  std::vector<std::vector<cd>> samples_, slopes_;
  // atoms: per (atom, gaussian) term: complex lateral amplitude per diff
  std::vector<double> term_z_, term_alpha_;          // z_a, 4 pi^2 / b'
  std::vector<std::vector<cd>> term_amp_;            // [term][diff]
};

// ---------------------------------------------------------------- slicing
// slicing.hpp:12-35
struct SlicingPlan {
  double z_bottom = -1;
  long count = 1;
  double h = 1;
  static SlicingPlan with_count(double z_bottom, long count);
  static SlicingPlan with_target_dz(double z_bottom, double dz);
  double z(long i) const { return z_bottom * (double)(count - i) / (double)count; }
};
// stages.hpp:14-31
struct StepWindow {
  double z0 = -1, z1 = 0;
  long count = 1;
  double h = 1;
  static StepWindow over(double z0, double z1, long count);
  static StepWindow of_plan(const SlicingPlan& p) { return StepWindow{p.z_bottom, 0.0, p.count, p.h}; }
  double z(long i) const { return (z0 * (double)(count - i) + z1 * (double)i) / (double)count; }
};
// stages.hpp:37-45, stages.cpp:8-23
struct NodeSchedule {
  std::vector<double> frac;
  bool endpoint_pair() const { return frac.size() >= 2 && frac.front() == 0.0 && frac.back() == 1.0; }
  int nodes() const { return (int)frac.size(); }
};
NodeSchedule midpoint_schedule();
NodeSchedule rk4_schedule();
NodeSchedule schedule_from_fracs(std::vector<double> raw);
// stages.cpp:25-30
double node_z(const StepWindow& w, long step, int node, const NodeSchedule& s);
// stages.hpp:53-65, stages.cpp:32-57
class UTable {
 public:
  UTable(const BoundPotential& u, const StepWindow& w, const NodeSchedule& s);
  const CMat& at(long step, int node) const { return mats_[(std::size_t)(step * stride_ + node)]; }
  const NodeSchedule& schedule() const { return sched_; }
  static std::size_t bytes_estimate(int n, long steps, const NodeSchedule& s);

 private:
  NodeSchedule sched_;
  long stride_ = 0;
  std::vector<CMat> mats_;
};

// ---------------------------------------------------------------- steppers
enum class StepAlgorithm { RK4, Splitting };
enum class SplitVariant { ABA, BAB };
// proposed.hpp:23-43, proposed.cpp:12-60, splitting_coefficients.cpp:13-77
struct StepperSpec {
  StepAlgorithm algorithm = StepAlgorithm::RK4;
  std::string name = "rk4";
  SplitVariant variant = SplitVariant::BAB;
  std::vector<double> drift, kick;
  std::vector<double> rk_nodes{0.0, 0.5, 0.5, 1.0};
  std::vector<double> rk_weights{1.0 / 6, 1.0 / 3, 1.0 / 3, 1.0 / 6};
  static const StepperSpec& rk4();
  static const StepperSpec& sp4();
  static const StepperSpec& sp6();
  static StepperSpec splitting(std::string name, SplitVariant v, std::vector<double> drift,
                               std::vector<double> kick);
  static const StepperSpec& by_name(const std::string& name);
  int stages() const;
  void validate() const;
};
struct KickSchedule {
  NodeSchedule nodes;
  std::vector<int> occ2node;
};
KickSchedule kick_schedule(const StepperSpec& spec);  // proposed.cpp:62-100
NodeSchedule schedule_for(const StepperSpec& spec);   // proposed.cpp:102-105

struct PropagationState {
  CMat Q, P;
  double z = 0;
};
void to_tau_rho(const GammaMatrix& g, const PropagationState& st, CMat& T, CMat& R);
PropagationState from_tau_rho(const GammaMatrix& g, const CMat& T, const CMat& R, double z);
PropagationState initial_state(const GammaMatrix& g, const CMat& R_init, double z);
void rk4_step(PropagationState& st, double h, const CMat& U0, const CMat& Um, const CMat& U1,
              const RVec& gamma2);
void splitting_step(PropagationState& st, double h, const StepperSpec& spec,
                    const std::vector<const CMat*>& U_at_kicks, const RVec& gamma2);
bool apply_rhst(PropagationState& st, double threshold);
CMat extract_reflection(const GammaMatrix& g, const PropagationState& st);

struct ProposedOptions { double rhst_threshold = 1000.0; };
struct SolveStats { long rhst_transforms = 0; };
struct BulkOptions { long max_periods = 10000; double tol = 1e-12; };

// proposed.cpp:293-309
CVec solve_proposed(const BoundPotential& u, const GammaMatrix& g, const SlicingPlan& plan,
                    const StepperSpec& spec, const ProposedOptions& opts = {},
                    const CMat& R_init = CMat(), const UTable* table = nullptr,
                    SolveStats* stats = nullptr);
// proposed.cpp:311-342
CMat compute_bulk_reflection_proposed(const BoundPotential& u, const GammaMatrix& g, double dz,
                                      const StepperSpec& spec, const ProposedOptions& opts,
                                      const BulkOptions& bulk);

// ---------------------------------------------------------------- curve
// curve.cpp:8-20
RVec intensity(const CVec& rho0, const GammaMatrix& g);
// sweep.hpp:17-24, sweep.cpp:18-33
struct AngleGrid {
  std::vector<double> theta0, theta1;
  static AngleGrid validated(std::vector<double> theta0, std::vector<double> theta1);
  long rows() const { return (long)(theta0.size() * theta1.size()); }
};
// sweep.hpp:26-32 (method "conventional" is out of scope for the oracle)
struct SweepOptions {
  std::string method = "rk4";
  double dz = 0.01;
  long slices = 0;  // EXTENSION: >0 fixes the slice count (SlicingPlan::with_count)
  double rhst_threshold = 1000.0;
  int threads = 1;
  std::size_t table_budget_bytes = (std::size_t)1 << 30;
};
// curve.hpp:19-31
struct RockingCurve {
  std::vector<double> theta0, theta1;
  int rods = 0;
  std::vector<double> eta;  // row-major rows x rods
  std::vector<cd> rho;      // row-major rows x rods (EXTENSION: kept for parity)
  std::vector<long> rhst;   // per row RHST count (EXTENSION)
  std::string method;
  double dz = 0, rhst_threshold = 0, solve_seconds = 0;
  long rows() const { return (long)theta0.size(); }
};
// sweep.cpp:54-143
RockingCurve rocking_curve(const PotentialField& field, const RodSet& rods, double gamma,
                           const AngleGrid& grid, const SweepOptions& opts);
// curve.cpp:22-41
double curve_error(const RockingCurve& cand, const RockingCurve& ref);

}  // namespace mbo
