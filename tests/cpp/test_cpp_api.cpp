// C++ host-API test, written like the reference's doctest suites
// (proj/tests/test_sweep.cpp, test_proposed.cpp) but against
// include/manybeam_b200.hpp. Exit code = number of failed checks.
// `--no-device` runs the host-only checks (CI without a GPU).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>

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
  // `--rewrite in.csv out.csv`: read a curve CSV and write it back (byte
  // round trip against the Python writer, tests/test_cpp_api.py)
  if (argc == 4 && std::strcmp(argv[1], "--rewrite") == 0) {
    write_curve_csv(std::string(argv[3]), read_curve_csv(std::string(argv[2])));
    return 0;
  }
  const bool device = !(argc > 1 && std::strcmp(argv[1], "--no-device") == 0);
  {  // csvio.cpp:65-149 wire format
    RockingCurve c;
    c.theta0 = {0.5, 1.25};
    c.theta1 = {0.0, 0.0};
    c.rods = 2;
    c.rod_labels = {"(0;0)", "(1;-1)"};
    c.eta = {0.125, 3.0e-17, 1.0 / 3.0, 0.0};
    c.method = "sp6";
    c.dz = 0.01;
    c.rhst_threshold = std::numeric_limits<double>::infinity();
    std::ostringstream os;
    write_curve_csv(os, c);
    const std::string want =
        "# manybeam-curve v1\n# method: sp6\n# dz: 1.00000000000000E-02\n# rhst_threshold: inf\n# rods: 2\n"
        "theta0,theta1,eta(0;0),eta(1;-1)\n"
        "5.00000000000000E-01,0.00000000000000E+00,1.25000000000000E-01,3.00000000000000E-17\n"
        "1.25000000000000E+00,0.00000000000000E+00,3.33333333333333E-01,0.00000000000000E+00\n";
    CHECK(os.str() == want);
    std::istringstream is(os.str());
    const RockingCurve back = read_curve_csv(is);
    CHECK(back.rows() == 2 && back.rods == 2 && back.rod_labels[1] == "(1;-1)" && back.method == "sp6");
    CHECK(std::isinf(back.rhst_threshold) && back.dz == 0.01);
    CHECK(curve_error(back, c) <= 1e-15);
    std::istringstream bad("theta0,theta1,eta(0;0)\n1.0,2.0\n");
    CHECK_THROWS_AS(read_curve_csv(bad), IoError);
  }
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
    {  // a device curve through the wire format
      std::ostringstream os;
      write_curve_csv(os, a);
      std::istringstream is(os.str());
      const RockingCurve back = read_curve_csv(is);
      CHECK(back.rod_labels == a.rod_labels && curve_error(back, a) <= 1e-14);
    }
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
    {  // solve_proposed with R_init (proposed.hpp:98-102): zero R_init = the sweep's row
      SolveStats stats;
      const std::vector<Complex> rho0 = solve_proposed(field, rods, 2.5, 8.0, 0.0, o, {}, &stats);
      const std::vector<Complex> zero((std::size_t)(rods.size() * rods.size()), Complex(0.0, 0.0));
      const std::vector<Complex> rhoz = solve_proposed(field, rods, 2.5, 8.0, 0.0, o, zero);
      double d = 0.0, dz = 0.0;
      for (int i = 0; i < rods.size(); ++i) {
        d = std::max(d, std::abs(rho0[(std::size_t)i] - a.rho[(std::size_t)(1 * a.rods + i)]));
        dz = std::max(dz, std::abs(rhoz[(std::size_t)i] - rho0[(std::size_t)i]));
      }
      // the same pair in a 6-pair plan and alone; the zero-seeded solve runs the
      // seeded (BULK) instantiation of the kernel: rounding-level agreement
      if (!(d <= 1e-13 && dz <= 1e-13)) std::printf("solve_proposed: d = %.3e, dz = %.3e\n", d, dz);
      CHECK(d <= 1e-13 && dz <= 1e-13);
      CHECK(stats.rhst_transforms == a.status[1].rhst_count);
      std::vector<Complex> seeded = zero;
      for (int i = 0; i < rods.size(); ++i) seeded[(std::size_t)(i * rods.size() + i)] = Complex(0.2, -0.1);
      const std::vector<Complex> rhos = solve_proposed(field, rods, 2.5, 8.0, 0.0, o, seeded);
      CHECK(std::abs(rhos[0] - rho0[0]) > 1e-6);  // the substrate reflection reaches the surface
      CHECK_THROWS_AS(solve_proposed(field, rods, 2.5, 8.0, 0.0, o, std::vector<Complex>(5)), SolverError);
    }
  }
  std::printf("%s: %d failure(s)\n", device ? "device" : "host-only", failures);
  return failures;
}
