// ORACLE — TEST INFRASTRUCTURE ONLY. The reference's own types and fixtures
// (proj/tests/support/fields.hpp) driving the B200 path through
// include/manybeam_b200_ref.hpp, checked against the reference's
// manybeam::rocking_curve on the same arguments. Needs a GPU at run time.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <cmath>
#include <limits>

#include "manybeam/curve.hpp"
#include "manybeam/geometry.hpp"
#include "manybeam/proposed.hpp"
#include "manybeam/slicing.hpp"
#include "manybeam/sweep.hpp"
#include "manybeam_b200_ref.hpp"
#include "support/fields.hpp"

using namespace manybeam;

namespace {
AngleGrid grid69() {
  std::vector<double> t;
  for (int i = 1; i <= 69; ++i) t.push_back((double)i);
  return AngleGrid::validated(t, {0.0});
}
}  // namespace

TEST_CASE("the drop-in rocking_curve agrees with the reference on its own fixtures") {
  const RodSet rods = testfields::rods11();
  for (const char* method : {"rk4", "sp4", "sp6", "conventional"}) {
    SweepOptions o;
    o.method = method;
    o.dz = 0.05;
    o.threads = 0;
    const RockingCurve want = rocking_curve(testfields::layered_field(), rods, testfields::kGamma11, grid69(), o);
    const RockingCurve got =
        b200::rocking_curve(testfields::layered_field(), rods, testfields::kGamma11, grid69(), o);
    CHECK(got.rod_labels == want.rod_labels);
    CHECK(got.method == want.method);
    CHECK(curve_error(got, want) <= 1e-9);
  }
}

TEST_CASE("tabulated and bulk fields cross the adapter") {
  const RodSet rods = testfields::rods1();
  const PotentialField f = testfields::constant_field(Complex(-0.8, -0.2), -7.0);
  SweepOptions o;
  o.method = "sp6";
  o.dz = 0.01;
  const AngleGrid g = AngleGrid::validated({10.0, 30.0, 50.0}, {0.0});
  CHECK(curve_error(b200::rocking_curve(f, rods, 2.0, g, o), rocking_curve(f, rods, 2.0, g, o)) <= 1e-9);
  std::vector<GaussianLayer> layers{{-2.4, -0.22, 2.2, 1.6, 0.08}, {-6.0, -0.18, 2.2, 1.9, 0.08}};
  const PotentialField bulk = PotentialField::gaussian_layers(-10.0, layers, 5.0);
  o.dz = 0.05;
  const AngleGrid g2 = AngleGrid::validated({2.0, 7.0, 15.0}, {0.0});
  CHECK(curve_error(b200::rocking_curve(bulk, testfields::rods11(), testfields::kGamma11, g2, o),
                    rocking_curve(bulk, testfields::rods11(), testfields::kGamma11, g2, o)) <= 1e-8);
}

TEST_CASE("breakdown arrives as the reference's BreakdownError with a step") {
  std::vector<GaussianLayer> layers;
  for (int i = 0; i < 75; ++i) layers.push_back({-1.0 - 2.0 * i, -0.22, 2.2, 0.7, 0.08});
  const PotentialField deep = PotentialField::gaussian_layers(-150.0, layers);
  SweepOptions o;
  o.method = "sp6";
  o.dz = 0.02;
  o.rhst_threshold = std::numeric_limits<double>::infinity();
  bool caught = false;
  try {
    (void)b200::rocking_curve(deep, testfields::rods11(), testfields::kGamma11,
                              AngleGrid::validated({3.0, 5.0}, {0.0}), o);
  } catch (const BreakdownError& e) {
    caught = e.step > 0;
  }
  CHECK(caught);
}

TEST_CASE("the drop-in solve_proposed takes the reference's R_init") {
  const RodSet rods = testfields::rods11();
  const PotentialField field = testfields::layered_field();
  const BoundPotential bound(field, rods);
  const BeamGeometry beam(testfields::kGamma11, 7.0, 0.0);
  const GammaMatrix gm = GammaMatrix::build(rods, beam);
  const SlicingPlan plan = SlicingPlan::with_target_dz(field.z_bottom(), 0.02);
  const int n = rods.size();
  ComplexMatrix R(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) R(i, j) = Complex(0.03 * std::cos(1.0 + i + 2.0 * j), 0.02 * std::sin(0.5 + 3.0 * i - j));
  for (const char* method : {"rk4", "sp4", "sp6"}) {
    const StepperSpec& spec = StepperSpec::by_name(method);
    SolveStats want_stats, got_stats;
    const ComplexVector want = solve_proposed(bound, gm, plan, spec, {}, R, nullptr, &want_stats);
    const ComplexVector got = b200::solve_proposed(field, rods, beam, plan, spec, {}, R, &got_stats);
    CHECK(got_stats.rhst_transforms == want_stats.rhst_transforms);
    CHECK((got - want).norm() <= 1e-10 * want.norm());
    // an empty R_init is the unseeded solve
    const ComplexVector w0 = solve_proposed(bound, gm, plan, spec);
    const ComplexVector g0 = b200::solve_proposed(field, rods, beam, plan, spec);
    CHECK((g0 - w0).norm() <= 1e-10 * w0.norm());
    CHECK((want - w0).norm() > 1e-6 * w0.norm());
  }
  CHECK_THROWS_AS(b200::solve_proposed(field, rods, beam, plan, StepperSpec::sp6(), {}, ComplexMatrix(3, 3)),
                  SolverError);
}
