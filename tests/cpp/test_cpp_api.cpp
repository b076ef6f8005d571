// C++ host-API test, written like the reference's doctest suites
// (proj/tests/test_sweep.cpp, test_proposed.cpp) but against
// include/manybeam_b200.hpp. Exit code = number of failed checks.
// `--no-device` runs the host-only checks (CI without a GPU).
#include <cmath>
#include <cstdio>
#include <cstring>

#include "../../include/manybeam_b200.hpp"

using namespace manybeam::b200;
static int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      ++failures;                                                  \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
    }                                                              \
  } while (0)
#define CHECK_THROWS_AS(expr, T) \
  do {                           \
    bool hit = false;            \
    try {                        \
      (void)(expr);              \
    } catch (const T&) {         \
      hit = true;                \
    } catch (...) {              \
    }                            \
    CHECK(hit);                  \
  } while (0)

int main(int argc, char** argv) {
  const bool device = !(argc > 1 && std::strcmp(argv[1], "--no-device") == 0);
  // test_rods_geometry.cpp:39-45 : the canonical 11-rod set
  const Lattice2D rect{{2.0, 0.0}, {0.0, 2.6}};
  const RodSet rods = RodSet::build(rect, 5.0);
  CHECK(rods.size() == 11);
  CHECK(rods.m(0)[0] == 0 && rods.m(0)[1] == 0);
  for (int i = 1; i < rods.size(); ++i) {
    const double a = std::hypot(rods.k(i).x, rods.k(i).y), b = std::hypot(rods.k(i - 1).x, rods.k(i - 1).y);
    CHECK(a >= b);
  }
  CHECK_THROWS_AS(RodSet::build(Lattice2D{{1.0, 2.0}, {2.0, 4.0}}, 3.0), ConfigError);
  CHECK_THROWS_AS(AngleGrid::validated({3.0, 2.0}, {0.0}), ConfigError);
  CHECK(RodSet::build_first(Lattice2D{{3.84, 0.0}, {-1.92, 3.3255}}, 15).size() == 15);
  if (device) {
    // test_sweep.cpp:33-46 row order, test_sweep.cpp:48-61 determinism
    const PotentialField field = PotentialField::gaussian_layers(
        -10.0, {{-2.4, -0.22, 2.2, 1.6, 0.08}, {-6.0, -0.18, 2.2, 1.9, 0.08}});
    SweepOptions o;
    o.method = "sp4";
    o.dz = 0.02;
    const AngleGrid grid = AngleGrid::validated({4.0, 8.0, 12.0}, {0.0, 30.0});
    const RockingCurve a = rocking_curve(field, rods, 2.5, grid, o);
    const RockingCurve b = rocking_curve(field, rods, 2.5, grid, o);
    CHECK(a.rows() == 6 && a.theta0[3] == 4.0 && a.theta1[3] == 30.0);
    CHECK(curve_error(a, b) == 0.0);
    double worst = 0.0;
    for (long r = 0; r < a.rows(); ++r) {
      double s = 0.0;
      for (int i = 0; i < a.rods; ++i) s += a.eta_at(r, i);
      worst = std::max(worst, s);
    }
    CHECK(worst <= 1.0 + 1e-8 && worst > 0.0);  // acceptance.cpp:308-319
    // test_sweep.cpp:90-105: breakdown surfaces with its step
    std::vector<GaussianLayer> deep;
    for (int i = 0; i < 75; ++i) deep.push_back({-1.0 - 2.0 * i, -0.22, 2.2, 0.7, 0.08});
    SweepOptions off = o;
    off.method = "sp6";
    off.rhst_threshold = std::numeric_limits<double>::infinity();
    bool broke = false;
    try {
      rocking_curve(PotentialField::gaussian_layers(-150.0, deep), rods, 2.5, AngleGrid::validated({3.0}, {0.0}), off);
    } catch (const BreakdownError& e) {
      broke = e.step > 0;
    }
    CHECK(broke);
    CHECK_THROWS_AS(rocking_curve(field, rods, 2.5, grid, SweepOptions{"sp8"}), ConfigError);
  }
  std::printf("%s: %d failure(s)\n", device ? "device" : "host-only", failures);
  return failures;
}
