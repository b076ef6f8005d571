// manybeam_b200_ref.hpp — header-only adapters between the reference's own
// types (/root/reference/proj/core/include/manybeam/*.hpp, Eigen-based) and
// the B200 path, so a reference caller switches by calling
// manybeam::b200::rocking_curve with the SAME arguments as
// manybeam::rocking_curve (sweep.hpp:37-38):
//
//   #include <manybeam/sweep.hpp>          // the reference
//   #include <manybeam_b200_ref.hpp>       // -I<repo>/include, link libmanybeam_b200.so
//   manybeam::RockingCurve c = manybeam::b200::rocking_curve(field, rods, gamma, grid, opts);
//
// Errors arrive as the reference's exception types (types.hpp:20-62), a
// BreakdownError with the first failing row's step, as the reference
// rethrows worker errors in row order (sweep.cpp:136-137). Compiled and run
// against the reference sources by oracle/Makefile (_ref/tests/adapter_b200).
#pragma once

#include <manybeam/curve.hpp>
#include <manybeam/geometry.hpp>
#include <manybeam/potential.hpp>
#include <manybeam/proposed.hpp>
#include <manybeam/rods.hpp>
#include <manybeam/sweep.hpp>
#include <manybeam/types.hpp>

#include "manybeam_b200.hpp"

namespace manybeam::b200 {

// potential.hpp:35-61 -> mb_field (zero, gaussian layers, tabulated; bulk period)
inline PotentialField to_device(const manybeam::PotentialField& f) {
  using K = manybeam::PotentialField::Kind;
  switch (f.kind()) {
    case K::Zero:
      return PotentialField::zero(f.z_bottom(), f.bulk_period());
    case K::GaussianLayers: {
      std::vector<GaussianLayer> ls;
      for (const manybeam::GaussianLayer& l : f.layers())
        ls.push_back(GaussianLayer{l.z_center, l.amplitude, l.sigma_xy, l.sigma_z, l.absorption});
      return PotentialField::gaussian_layers(f.z_bottom(), ls, f.bulk_period());
    }
    case K::Tabulated: {
      std::vector<std::pair<std::array<int, 2>, std::vector<Complex>>> es;
      for (const manybeam::TabulatedEntry& e : f.entries()) es.push_back({{e.dm.x(), e.dm.y()}, e.values});
      return PotentialField::tabulated(f.z_bottom(), f.z_grid(), es, f.bulk_period());
    }
  }
  throw ConfigError("potential: unknown field kind");
}

// rods.hpp:23-47 -> the device rod tables, same order and difference table
inline RodSet to_device(const manybeam::RodSet& r) {
  const int n = r.size(), nd = r.diff_count();
  std::vector<double> k, diff;
  std::vector<int> m, diff_m, diff_index((std::size_t)n * n);
  for (int i = 0; i < n; ++i) {
    k.push_back(r.k(i).x());
    k.push_back(r.k(i).y());
    m.push_back(r.m(i).x());
    m.push_back(r.m(i).y());
  }
  for (int d = 0; d < nd; ++d) {
    diff.push_back(r.diff(d).x());
    diff.push_back(r.diff(d).y());
    diff_m.push_back(r.diff_m(d).x());
    diff_m.push_back(r.diff_m(d).y());
  }
  for (int j = 0; j < n; ++j)
    for (int q = 0; q < n; ++q) diff_index[(std::size_t)j * n + q] = r.diff_index(j, q);
  return RodSet::from_tables(std::move(k), std::move(m), std::move(diff), std::move(diff_m), std::move(diff_index));
}

// device curve -> curve.hpp:19-31 (same row and rod order; labels as sweep.cpp:77-80)
inline manybeam::RockingCurve from_device(const RockingCurve& c, const manybeam::RodSet& rods) {
  manybeam::RockingCurve out;
  out.theta0 = c.theta0;
  out.theta1 = c.theta1;
  out.eta = manybeam::RealMatrix::Zero(c.rows(), c.rods);
  for (long r = 0; r < c.rows(); ++r)
    for (int i = 0; i < c.rods; ++i) out.eta(r, i) = c.eta_at(r, i);
  for (int i = 0; i < rods.size(); ++i)
    out.rod_labels.push_back("(" + std::to_string(rods.m(i)(0)) + ";" + std::to_string(rods.m(i)(1)) + ")");
  out.method = c.method;
  out.dz = c.dz;
  out.rhst_threshold = c.method == "conventional" ? 0.0 : c.rhst_threshold;
  return out;
}

// device exception -> the reference's exception types (types.hpp:20-62)
template <class F>
auto with_reference_errors(F&& body) -> decltype(body()) {
  try {
    return body();
  } catch (const BreakdownError& e) {
    throw manybeam::BreakdownError(e.what(), e.step);
  } catch (const ConvergenceError& e) {
    throw manybeam::ConvergenceError(e.what());
  } catch (const DomainError& e) {
    throw manybeam::DomainError(e.what());
  } catch (const SingularMatrixError& e) {
    throw manybeam::SingularMatrixError(e.what());
  } catch (const SolverError& e) {
    throw manybeam::SolverError(e.what());
  } catch (const ConfigError& e) {
    throw manybeam::ConfigError(e.what());
  } catch (const CompareError& e) {
    throw manybeam::CompareError(e.what());
  } catch (const IoError& e) {
    throw manybeam::IoError(e.what());
  }
}

// sweep.hpp:37-38 on the device; the reference's exception types
inline manybeam::RockingCurve rocking_curve(const manybeam::PotentialField& field, const manybeam::RodSet& rods,
                                            double gamma, const manybeam::AngleGrid& grid,
                                            const manybeam::SweepOptions& opts, int device = 0) {
  return with_reference_errors([&] {
    SweepOptions o;
    o.method = opts.method;
    o.dz = opts.dz;
    o.rhst_threshold = opts.rhst_threshold;
    o.device = device;
    return from_device(rocking_curve(to_device(field), to_device(rods), gamma,
                                     AngleGrid::validated(grid.theta0, grid.theta1), o),
                       rods);
  });
}

// solve_proposed (proposed.hpp:98-102, proposed.cpp:293-309) on the device:
// rho0 for one beam from the state seeded with R_init (empty = zero) at
// plan.z_bottom, any StepperSpec (rk4, sp4, sp6 or a custom splitting). The
// reference call takes the BoundPotential and the GammaMatrix; the device
// builds both itself, so the adapter takes what they are built from (the
// field with its rods, and the beam). The UTable argument has no counterpart:
// the device's coefficient table always exists.
inline manybeam::ComplexVector solve_proposed(const manybeam::PotentialField& field, const manybeam::RodSet& rods,
                                              const manybeam::BeamGeometry& beam, const manybeam::SlicingPlan& plan,
                                              const manybeam::StepperSpec& spec,
                                              const manybeam::ProposedOptions& opts = {},
                                              const manybeam::ComplexMatrix& R_init = manybeam::ComplexMatrix(),
                                              manybeam::SolveStats* stats = nullptr, int device = 0) {
  return with_reference_errors([&] {
    spec.validate();
    const int n = rods.size();
    if (R_init.size() != 0 && (R_init.rows() != n || R_init.cols() != n))
      throw SolverError("R_init has wrong dimensions");  // proposed.cpp:126
    if (plan.z_bottom != field.z_bottom()) throw SolverError("slicing plan and field disagree on z_bottom");
    std::vector<double> seed;  // row-major interleaved (the C-ABI layout)
    if (R_init.size() != 0)
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          seed.push_back(R_init(i, j).real());
          seed.push_back(R_init(i, j).imag());
        }
    mb_stepper st{};
    if (spec.algorithm == manybeam::StepAlgorithm::RK4) {
      st.algorithm = MB_STEP_RK4;
      st.variant = MB_SPLIT_BAB;
    } else {
      st.algorithm = MB_STEP_SPLITTING;
      st.variant = spec.variant == manybeam::SplitVariant::ABA ? MB_SPLIT_ABA : MB_SPLIT_BAB;
      st.ndrift = (int)spec.drift.size();
      st.drift = spec.drift.data();
      st.nkick = (int)spec.kick.size();
      st.kick = spec.kick.data();
    }
    const mb_options o{plan.h, plan.count, opts.rhst_threshold, 1, 0, 0};
    const PotentialField df = to_device(field);
    const RodSet dr = to_device(rods);
    const mb_field f = df.view();
    const mb_rods r = dr.view();
    const mb_pair pair{0, beam.theta0_deg, beam.theta1_deg};
    struct Guard {
      mb_plan* p = nullptr;
      ~Guard() {
        if (p) mb_plan_destroy(p);
      }
    } g;
    check(mb_plan_create_seeded(context(device), &r, &f, 1, beam.gamma, &pair, 1, &st, &o,
                                seed.empty() ? nullptr : seed.data(), seed.empty() ? 0 : 1, &g.p));
    check(mb_plan_execute(g.p, nullptr));
    std::vector<double> eta((std::size_t)n);
    std::vector<Complex> rho((std::size_t)n);
    mb_point_status ps{};
    check(mb_plan_results(g.p, eta.data(), reinterpret_cast<double*>(rho.data()), &ps), (std::size_t)ps.step);
    if (stats) stats->rhst_transforms = ps.rhst_count;
    manybeam::ComplexVector out(n);
    for (int i = 0; i < n; ++i) out(i) = rho[(std::size_t)i];
    return out;
  });
}

}  // namespace manybeam::b200
