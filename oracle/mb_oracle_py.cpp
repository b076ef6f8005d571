// ORACLE — TEST INFRASTRUCTURE ONLY. pybind11 bindings of the CPU restatement
// (mb_oracle.hpp) so pytest can drive it the way the reference's doctest
// suites drive the C++ library.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cmath>
#include <cstring>

#include "mb_oracle.hpp"

namespace py = pybind11;
using namespace mbo;

namespace {

py::array_t<cd> to_np(const CMat& M) {
  py::array_t<cd> out({(py::ssize_t)M.r, (py::ssize_t)M.c});
  auto v = out.mutable_unchecked<2>();
  for (int i = 0; i < M.r; ++i)
    for (int j = 0; j < M.c; ++j) v(i, j) = M(i, j);
  return out;
}
CMat from_np(py::array_t<cd, py::array::forcecast> a) {
  if (a.ndim() == 1 && a.shape(0) == 0) return CMat();
  if (a.ndim() != 2) throw std::invalid_argument("expected a 2-D complex array");
  auto v = a.unchecked<2>();
  CMat M((int)a.shape(0), (int)a.shape(1));
  for (int i = 0; i < M.r; ++i)
    for (int j = 0; j < M.c; ++j) M(i, j) = v(i, j);
  return M;
}
template <class T>
py::array_t<T> vec_np(const std::vector<T>& v) {
  py::array_t<T> out((py::ssize_t)v.size());
  if (!v.empty()) std::memcpy(out.mutable_data(), v.data(), v.size() * sizeof(T));
  return out;
}
py::array_t<double> v2_np(const std::vector<Vec2>& v) {
  py::array_t<double> out({(py::ssize_t)v.size(), (py::ssize_t)2});
  auto w = out.mutable_unchecked<2>();
  for (std::size_t i = 0; i < v.size(); ++i) {
    w(i, 0) = v[i].x;
    w(i, 1) = v[i].y;
  }
  return out;
}
py::array_t<int> v2i_np(const std::vector<Vec2i>& v) {
  py::array_t<int> out({(py::ssize_t)v.size(), (py::ssize_t)2});
  auto w = out.mutable_unchecked<2>();
  for (std::size_t i = 0; i < v.size(); ++i) {
    w(i, 0) = v[i].x;
    w(i, 1) = v[i].y;
  }
  return out;
}
Lattice2D make_lattice(std::pair<double, double> a1, std::pair<double, double> a2) {
  Lattice2D l;
  l.a1 = Vec2{a1.first, a1.second};
  l.a2 = Vec2{a2.first, a2.second};
  return l;
}
std::optional<double> opt_period(py::object p) {
  if (p.is_none()) return std::nullopt;
  return p.cast<double>();
}

}  // namespace

PYBIND11_MODULE(mb_oracle, m) {
  m.doc() = "ORACLE (test infrastructure only): CPU restatement of the manybeam hot path";

  // ---- exceptions (types.hpp:20-62), derived types translated first
  static py::exception<Error> exc_error(m, "Error");
  static py::exception<ConfigError> exc_config(m, "ConfigError", exc_error.ptr());
  static py::exception<SolverError> exc_solver(m, "SolverError", exc_error.ptr());
  static py::exception<SingularMatrixError> exc_singular(m, "SingularMatrixError", exc_solver.ptr());
  static py::exception<BreakdownError> exc_breakdown(m, "BreakdownError", exc_solver.ptr());
  static py::exception<ConvergenceError> exc_conv(m, "ConvergenceError", exc_solver.ptr());
  static py::exception<DomainError> exc_domain(m, "DomainError", exc_solver.ptr());
  static py::exception<CompareError> exc_compare(m, "CompareError", exc_error.ptr());
  py::register_exception_translator([](std::exception_ptr p) {
    try {
      if (p) std::rethrow_exception(p);
    } catch (const BreakdownError& e) {
      py::object inst = py::reinterpret_borrow<py::object>(exc_breakdown.ptr())(e.what());
      inst.attr("step") = e.step;
      PyErr_SetObject(exc_breakdown.ptr(), inst.ptr());
    } catch (const SingularMatrixError& e) {
      PyErr_SetString(exc_singular.ptr(), e.what());
    } catch (const ConvergenceError& e) {
      PyErr_SetString(exc_conv.ptr(), e.what());
    } catch (const DomainError& e) {
      PyErr_SetString(exc_domain.ptr(), e.what());
    } catch (const SolverError& e) {
      PyErr_SetString(exc_solver.ptr(), e.what());
    } catch (const ConfigError& e) {
      PyErr_SetString(exc_config.ptr(), e.what());
    } catch (const CompareError& e) {
      PyErr_SetString(exc_compare.ptr(), e.what());
    } catch (const Error& e) {
      PyErr_SetString(exc_error.ptr(), e.what());
    }
  });

  // ---- dense kernels
  m.def("gershgorin_cond", [](py::array_t<cd, py::array::forcecast> Q) { return gershgorin_cond(from_np(Q)); });
  m.def("solve_right", [](py::array_t<cd, py::array::forcecast> B, py::array_t<cd, py::array::forcecast> A) {
    return to_np(solve_right(from_np(B), from_np(A)));
  });

  // ---- lattice / rods
  py::class_<Lattice2D>(m, "Lattice2D")
      .def(py::init(&make_lattice), py::arg("a1"), py::arg("a2"))
      .def("b1", [](const Lattice2D& l) { auto b = l.b1(); return std::make_pair(b.x, b.y); })
      .def("b2", [](const Lattice2D& l) { auto b = l.b2(); return std::make_pair(b.x, b.y); })
      .def("validate", &Lattice2D::validate);
  py::class_<RodSet>(m, "RodSet")
      .def_static("build", &RodSet::build, py::arg("lattice"), py::arg("cutoff"))
      .def_static("build_first", &RodSet::build_first, py::arg("lattice"), py::arg("n"))
      .def("size", &RodSet::size)
      .def("diff_count", &RodSet::diff_count)
      .def_readonly("cutoff", &RodSet::cutoff)
      .def_property_readonly("k", [](const RodSet& r) { return v2_np(r.k); })
      .def_property_readonly("m", [](const RodSet& r) { return v2i_np(r.m); })
      .def_property_readonly("diff", [](const RodSet& r) { return v2_np(r.diff); })
      .def_property_readonly("diff_m", [](const RodSet& r) { return v2i_np(r.diff_m); })
      .def_property_readonly("diff_index", [](const RodSet& r) {
        py::array_t<int> a({(py::ssize_t)r.size(), (py::ssize_t)r.size()});
        std::memcpy(a.mutable_data(), r.diff_index_.data(), r.diff_index_.size() * sizeof(int));
        return a;
      });

  // ---- geometry
  m.def("project_incident", [](double g, double t0, double t1) {
    auto b = project_incident(g, t0, t1);
    return std::make_pair(b.x, b.y);
  });
  py::class_<BeamGeometry>(m, "BeamGeometry")
      .def(py::init<double, double, double>(), py::arg("gamma"), py::arg("theta0_deg"), py::arg("theta1_deg") = 0.0)
      .def_readonly("gamma", &BeamGeometry::gamma)
      .def_readonly("sin_theta0", &BeamGeometry::sin_theta0)
      .def_property_readonly("b0", [](const BeamGeometry& b) { return std::make_pair(b.b0.x, b.b0.y); });
  py::class_<GammaMatrix>(m, "GammaMatrix")
      .def_static("build", &GammaMatrix::build)
      .def("size", &GammaMatrix::size)
      .def_property_readonly("diag", [](const GammaMatrix& g) { return vec_np(g.diag); })
      .def_property_readonly("inv_diag", [](const GammaMatrix& g) { return vec_np(g.inv_diag); })
      .def_property_readonly("gamma2", [](const GammaMatrix& g) { return vec_np(g.gamma2); })
      .def_property_readonly("propagating", [](const GammaMatrix& g) {
        std::vector<int> p(g.propagating.begin(), g.propagating.end());
        return vec_np(p);
      })
      .def_readonly("sin_theta0", &GammaMatrix::sin_theta0);
  m.def("beam_from_energy", [](double e) {
    auto b = beam_from_energy(e);
    return std::make_pair(b.gamma, b.gamma_L);
  });

  // ---- potential
  py::class_<PotentialField>(m, "PotentialField")
      .def_static("zero", &PotentialField::zero)
      .def_static(
          "gaussian_layers",
          [](double zb, std::vector<std::tuple<double, double, double, double, double>> layers, py::object period) {
            std::vector<GaussianLayer> ls;
            for (auto& t : layers)
              ls.push_back(GaussianLayer{std::get<0>(t), std::get<1>(t), std::get<2>(t), std::get<3>(t), std::get<4>(t)});
            return PotentialField::gaussian_layers(zb, std::move(ls), opt_period(period));
          },
          py::arg("z_bottom"), py::arg("layers"), py::arg("bulk_period") = py::none())
      .def_static(
          "tabulated",
          [](double zb, std::vector<double> grid, std::vector<std::pair<std::pair<int, int>, std::vector<cd>>> entries,
             py::object period) {
            std::vector<TabulatedEntry> es;
            for (auto& e : entries) es.push_back(TabulatedEntry{Vec2i{e.first.first, e.first.second}, e.second});
            return PotentialField::tabulated(zb, std::move(grid), std::move(es), opt_period(period));
          },
          py::arg("z_bottom"), py::arg("z_grid"), py::arg("entries"), py::arg("bulk_period") = py::none())
      .def_static(
          "atoms",
          [](double zb, py::array_t<double, py::array::forcecast> xyz, py::array_t<int, py::array::forcecast> species,
             py::array_t<double, py::array::forcecast> B, py::array_t<double, py::array::forcecast> ff_a,
             py::array_t<double, py::array::forcecast> ff_b, double cell_area, double gamma_L, double particle_sign,
             double absorption, py::object period) {
            AtomModel M;
            auto x = xyz.unchecked<2>();
            auto s = species.unchecked<1>();
            auto bb = B.unchecked<1>();
            for (py::ssize_t i = 0; i < xyz.shape(0); ++i)
              M.atoms.push_back(AtomSite{x(i, 0), x(i, 1), x(i, 2), s(i), bb(i)});
            auto fa = ff_a.unchecked<2>();
            auto fb = ff_b.unchecked<2>();
            for (py::ssize_t i = 0; i < ff_a.shape(0); ++i) {
              Species sp;
              for (int j = 0; j < 4; ++j) {
                sp.a[j] = fa(i, j);
                sp.b[j] = fb(i, j);
              }
              M.species.push_back(sp);
            }
            M.cell_area = cell_area;
            M.gamma_L = gamma_L;
            M.particle_sign = particle_sign;
            M.absorption = absorption;
            return PotentialField::atoms(zb, std::move(M), opt_period(period));
          },
          py::arg("z_bottom"), py::arg("xyz"), py::arg("species"), py::arg("B"), py::arg("ff_a"), py::arg("ff_b"),
          py::arg("cell_area"), py::arg("gamma_L"), py::arg("particle_sign"), py::arg("absorption"),
          py::arg("bulk_period") = py::none())
      .def_readonly("z_bottom", &PotentialField::z_bottom);
  py::class_<BoundPotential>(m, "BoundPotential")
      .def(py::init<const PotentialField&, const RodSet&>(), py::keep_alive<1, 2>())
      .def("n", &BoundPotential::n)
      .def("map_z", &BoundPotential::map_z)
      .def("eval", [](const BoundPotential& u, double z) { return to_np(u.eval(z)); })
      .def("eval_coeffs", [](const BoundPotential& u, double z) {
        std::vector<cd> c;
        u.eval_coeffs(z, c);
        return vec_np(c);
      });

  // ---- slicing / stages
  py::class_<SlicingPlan>(m, "SlicingPlan")
      .def_static("with_count", &SlicingPlan::with_count)
      .def_static("with_target_dz", &SlicingPlan::with_target_dz)
      .def_readonly("z_bottom", &SlicingPlan::z_bottom)
      .def_readonly("count", &SlicingPlan::count)
      .def_readonly("h", &SlicingPlan::h)
      .def("z", &SlicingPlan::z);
  py::class_<StepWindow>(m, "StepWindow")
      .def_static("over", &StepWindow::over)
      .def_static("of_plan", &StepWindow::of_plan)
      .def_readonly("count", &StepWindow::count)
      .def_readonly("h", &StepWindow::h)
      .def("z", &StepWindow::z);
  py::class_<NodeSchedule>(m, "NodeSchedule")
      .def_readonly("frac", &NodeSchedule::frac)
      .def("endpoint_pair", &NodeSchedule::endpoint_pair)
      .def("nodes", &NodeSchedule::nodes);
  m.def("midpoint_schedule", &midpoint_schedule);
  m.def("rk4_schedule", &rk4_schedule);
  m.def("schedule_from_fracs", &schedule_from_fracs);
  m.def("node_z", &node_z);
  py::class_<UTable>(m, "UTable")
      .def(py::init<const BoundPotential&, const StepWindow&, const NodeSchedule&>())
      .def("at", [](const UTable& t, long s, int n) { return to_np(t.at(s, n)); })
      .def_static("bytes_estimate", &UTable::bytes_estimate);

  // ---- steppers
  py::enum_<SplitVariant>(m, "SplitVariant").value("ABA", SplitVariant::ABA).value("BAB", SplitVariant::BAB);
  py::class_<StepperSpec>(m, "StepperSpec")
      .def_static("rk4", &StepperSpec::rk4, py::return_value_policy::copy)
      .def_static("sp4", &StepperSpec::sp4, py::return_value_policy::copy)
      .def_static("sp6", &StepperSpec::sp6, py::return_value_policy::copy)
      .def_static("by_name", &StepperSpec::by_name, py::return_value_policy::copy)
      .def_static("splitting", &StepperSpec::splitting)
      .def("validate", &StepperSpec::validate)
      .def("stages", &StepperSpec::stages)
      .def_readwrite("name", &StepperSpec::name)
      .def_readwrite("drift", &StepperSpec::drift)
      .def_readwrite("kick", &StepperSpec::kick)
      .def_readwrite("variant", &StepperSpec::variant)
      .def_property_readonly("is_rk4", [](const StepperSpec& s) { return s.algorithm == StepAlgorithm::RK4; });
  py::class_<KickSchedule>(m, "KickSchedule")
      .def_readonly("nodes", &KickSchedule::nodes)
      .def_readonly("occ2node", &KickSchedule::occ2node);
  m.def("kick_schedule", &kick_schedule);
  m.def("schedule_for", &schedule_for);

  py::class_<PropagationState>(m, "PropagationState")
      .def(py::init([](py::array_t<cd, py::array::forcecast> Q, py::array_t<cd, py::array::forcecast> P, double z) {
             PropagationState s;
             s.Q = from_np(Q);
             s.P = from_np(P);
             s.z = z;
             return s;
           }),
           py::arg("Q"), py::arg("P"), py::arg("z") = 0.0)
      .def_property_readonly("Q", [](const PropagationState& s) { return to_np(s.Q); })
      .def_property_readonly("P", [](const PropagationState& s) { return to_np(s.P); })
      .def_readonly("z", &PropagationState::z);
  m.def("initial_state", [](const GammaMatrix& g, py::array_t<cd, py::array::forcecast> R, double z) {
    return initial_state(g, from_np(R), z);
  });
  m.def("to_tau_rho", [](const GammaMatrix& g, const PropagationState& s) {
    CMat T, R;
    to_tau_rho(g, s, T, R);
    return std::make_pair(to_np(T), to_np(R));
  });
  m.def("from_tau_rho", [](const GammaMatrix& g, py::array_t<cd, py::array::forcecast> T,
                           py::array_t<cd, py::array::forcecast> R, double z) {
    return from_tau_rho(g, from_np(T), from_np(R), z);
  });
  m.def("rk4_step", [](PropagationState& st, double h, py::array_t<cd, py::array::forcecast> U0,
                       py::array_t<cd, py::array::forcecast> Um, py::array_t<cd, py::array::forcecast> U1,
                       std::vector<double> g2) {
    rk4_step(st, h, from_np(U0), from_np(Um), from_np(U1), g2);
  });
  m.def("splitting_step", [](PropagationState& st, double h, const StepperSpec& spec,
                             std::vector<py::array_t<cd, py::array::forcecast>> U, std::vector<double> g2) {
    std::vector<CMat> mats;
    for (auto& u : U) mats.push_back(from_np(u));
    std::vector<const CMat*> ptrs;
    for (auto& mm : mats) ptrs.push_back(&mm);
    splitting_step(st, h, spec, ptrs, g2);
  });
  m.def("apply_rhst", &apply_rhst);
  m.def("extract_reflection", [](const GammaMatrix& g, const PropagationState& s) {
    return to_np(extract_reflection(g, s));
  });
  m.def(
      "solve_proposed",
      [](const BoundPotential& u, const GammaMatrix& g, const SlicingPlan& plan, const StepperSpec& spec,
         double threshold, py::array_t<cd, py::array::forcecast> R_init, bool use_table) {
        ProposedOptions o;
        o.rhst_threshold = threshold;
        SolveStats st;
        std::unique_ptr<UTable> table;
        if (use_table) table = std::make_unique<UTable>(u, StepWindow::of_plan(plan), schedule_for(spec));
        CVec r = solve_proposed(u, g, plan, spec, o, from_np(R_init), table.get(), &st);
        return std::make_pair(vec_np(r), st.rhst_transforms);
      },
      py::arg("u"), py::arg("gamma"), py::arg("plan"), py::arg("spec"), py::arg("threshold") = 1000.0,
      py::arg("R_init") = py::array_t<cd>(0), py::arg("use_table") = false);
  m.def(
      "compute_bulk_reflection_proposed",
      [](const BoundPotential& u, const GammaMatrix& g, double dz, const StepperSpec& spec, double threshold,
         long max_periods, double tol) {
        ProposedOptions o;
        o.rhst_threshold = threshold;
        BulkOptions b;
        b.max_periods = max_periods;
        b.tol = tol;
        return to_np(compute_bulk_reflection_proposed(u, g, dz, spec, o, b));
      },
      py::arg("u"), py::arg("gamma"), py::arg("dz"), py::arg("spec"), py::arg("threshold") = 1000.0,
      py::arg("max_periods") = 10000, py::arg("tol") = 1e-12);

  // ---- curve / sweep
  m.def("intensity", [](py::array_t<cd, py::array::forcecast> rho, const GammaMatrix& g) {
    std::vector<cd> r(rho.data(), rho.data() + rho.size());
    return vec_np(intensity(r, g));
  });
  py::class_<AngleGrid>(m, "AngleGrid")
      .def_static("validated", &AngleGrid::validated)
      .def_readonly("theta0", &AngleGrid::theta0)
      .def_readonly("theta1", &AngleGrid::theta1)
      .def("rows", &AngleGrid::rows);
  py::class_<SweepOptions>(m, "SweepOptions")
      .def(py::init<>())
      .def_readwrite("method", &SweepOptions::method)
      .def_readwrite("dz", &SweepOptions::dz)
      .def_readwrite("slices", &SweepOptions::slices)
      .def_readwrite("rhst_threshold", &SweepOptions::rhst_threshold)
      .def_readwrite("threads", &SweepOptions::threads)
      .def_readwrite("table_budget_bytes", &SweepOptions::table_budget_bytes);
  py::class_<RockingCurve>(m, "RockingCurve")
      .def_readonly("theta0", &RockingCurve::theta0)
      .def_readonly("theta1", &RockingCurve::theta1)
      .def_readonly("method", &RockingCurve::method)
      .def_readonly("solve_seconds", &RockingCurve::solve_seconds)
      .def_property_readonly("eta", [](const RockingCurve& c) {
        py::array_t<double> a({(py::ssize_t)c.rows(), (py::ssize_t)c.rods});
        if (!c.eta.empty()) std::memcpy(a.mutable_data(), c.eta.data(), c.eta.size() * sizeof(double));
        return a;
      })
      .def_property_readonly("rho", [](const RockingCurve& c) {
        py::array_t<cd> a({(py::ssize_t)c.rows(), (py::ssize_t)c.rods});
        if (!c.rho.empty()) std::memcpy(a.mutable_data(), c.rho.data(), c.rho.size() * sizeof(cd));
        return a;
      })
      .def_property_readonly("rhst", [](const RockingCurve& c) { return vec_np(c.rhst); })
      .def("rows", &RockingCurve::rows);
  m.def("rocking_curve", &rocking_curve, py::call_guard<py::gil_scoped_release>());
  m.def("curve_error", &curve_error);
}
