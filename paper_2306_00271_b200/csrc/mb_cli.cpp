// manybeam_b200 — the reference CLI surface (proj/tools/main.cpp:24-82) on the
// B200 path:
//
//   manybeam_b200 [--threads N] simulate --config run.json [--out curve.csv]
//   manybeam_b200 [--threads N] bench --config run.json --out bench.csv
//                 [--dz a,b,..] [--methods m,..] [--repeats K]
//   manybeam_b200 compare a.csv b.csv
//
// Same JSON schema (config.cpp:223-282, strict unknown-key rejection at every
// level), same curve / bench CSV bytes (csvio.cpp) and the same exit codes
// (main.cpp:14-20): 0 ok, 2 config (and CLI misuse), 3 solver, 4 comparison
// mismatch, 5 I/O. The solves run through the C-ABI (mb_rocking_curve).
//
// Extensions, all optional keys (north_star):
//   "energy_ev" + "particle" ("electron" | "positron") instead of "gamma";
//   "rod_count": first-N rods of the reference order instead of "rod_cutoff";
//   field "type": "atoms" (atom list, 4-Gaussian form factors per species,
//     Debye-Waller B per atom, "absorption" ratio; cell area from the lattice);
//   "devices": [0, 1, ...] spreads the angle rows over several GPUs
//     (mb_context_create_multi), "fsal": true, "slices": L (fixed count).
// --threads is accepted for compatibility; host threads do not partition the
// work here (the output is byte-identical for any value, as the reference's).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "../../include/manybeam_b200.hpp"

namespace mb = manybeam::b200;
using nlohmann::json;

namespace {

// ------------------------------------------------------------------ schema
std::string where(const std::string& ctx) { return ctx.empty() ? "config" : "config: " + ctx; }

const json& require_object(const json& j, const std::string& ctx) {
  if (!j.is_object()) throw mb::ConfigError(where(ctx) + " must be a JSON object");
  return j;
}
void check_keys(const json& j, std::initializer_list<const char*> allowed, const std::string& ctx) {
  const std::set<std::string> ok(allowed.begin(), allowed.end());
  for (const auto& it : j.items())
    if (!ok.count(it.key())) throw mb::ConfigError(where(ctx) + " has unknown key '" + it.key() + "'");
}
const json* find(const json& j, const char* key) {
  auto it = j.find(key);
  return it == j.end() ? nullptr : &*it;
}
const json& require(const json& j, const char* key, const std::string& ctx) {
  const json* p = find(j, key);
  if (!p) throw mb::ConfigError(where(ctx) + " is missing required key '" + key + "'");
  return *p;
}
double as_number(const json& j, const std::string& ctx) {
  if (!j.is_number()) throw mb::ConfigError(where(ctx) + " must be a number");
  const double v = j.get<double>();
  if (!std::isfinite(v)) throw mb::ConfigError(where(ctx) + " must be finite");
  return v;
}
long as_integer(const json& j, const std::string& ctx) {
  if (!j.is_number_integer()) throw mb::ConfigError(where(ctx) + " must be an integer");
  return j.get<long>();
}
std::vector<double> as_number_list(const json& j, const std::string& ctx) {
  if (!j.is_array()) throw mb::ConfigError(where(ctx) + " must be an array of numbers");
  std::vector<double> out;
  for (std::size_t i = 0; i < j.size(); ++i) out.push_back(as_number(j[i], ctx + "[" + std::to_string(i) + "]"));
  return out;
}
std::string as_string(const json& j, const std::string& ctx) {
  if (!j.is_string()) throw mb::ConfigError(where(ctx) + " must be a string");
  return j.get<std::string>();
}
mb::Vec2 as_vec2(const json& j, const std::string& ctx) {
  const std::vector<double> v = as_number_list(j, ctx);
  if (v.size() != 2) throw mb::ConfigError(where(ctx) + " must have exactly 2 components");
  return mb::Vec2{v[0], v[1]};
}
// plain list or inclusive {start, stop, step} range (config.cpp:75-90)
std::vector<double> parse_axis(const json& j, const std::string& ctx) {
  if (j.is_array()) return as_number_list(j, ctx);
  require_object(j, ctx);
  check_keys(j, {"start", "stop", "step"}, ctx);
  const double start = as_number(require(j, "start", ctx), ctx + ".start");
  const double stop = as_number(require(j, "stop", ctx), ctx + ".stop");
  const double step = as_number(require(j, "step", ctx), ctx + ".step");
  if (!(step > 0.0)) throw mb::ConfigError(where(ctx) + ".step must be positive");
  if (stop < start - 1e-12) throw mb::ConfigError(where(ctx) + ".stop must be >= start");
  const long count = (long)std::floor((stop - start) / step + 1e-9) + 1;
  std::vector<double> out;
  for (long i = 0; i < count; ++i) out.push_back(start + step * (double)i);
  return out;
}
void check_method_name(const std::string& m, const std::string& ctx) {
  if (m != "conventional" && m != "rk4" && m != "sp4" && m != "sp6")
    throw mb::ConfigError(where(ctx) + ": method '" + m + "' not recognized (conventional, rk4, sp4, sp6)");
}

struct BenchRun {
  std::string method = "sp6";
  double dz = 0.001;
};
struct BenchCfg {
  BenchRun reference;
  std::optional<BenchRun> baseline;
  std::vector<std::string> methods;
  std::vector<double> dz_values;
  int repeats = 5;
};
struct RunConfig {
  double gamma = 1.0, gamma_L = 1.0, particle_sign = -1.0;
  bool have_energy = false;
  mb::Lattice2D lattice;
  double rod_cutoff = 0.0;
  int rod_count = 0;
  std::optional<mb::PotentialField> field;
  mb::AngleGrid angles;
  std::string method = "conventional";
  double dz = 0.01;
  long slices = 0;
  double rhst_threshold = 1000.0;
  int threads = 1;
  bool fsal = false;
  std::vector<int> devices;
  std::string out;
  std::optional<BenchCfg> bench;
};

// field types of config.cpp:92-159 plus "atoms" (extension)
mb::PotentialField parse_field(const json& j, const RunConfig& cfg) {
  const std::string ctx = "field";
  require_object(j, ctx);
  const std::string type = as_string(require(j, "type", ctx), ctx + ".type");
  const double z_bottom = as_number(require(j, "z_bottom", ctx), ctx + ".z_bottom");
  std::optional<double> bulk;
  if (const json* p = find(j, "bulk_period")) bulk = as_number(*p, ctx + ".bulk_period");
  if (type == "zero") {
    check_keys(j, {"type", "z_bottom"}, ctx);
    return mb::PotentialField::zero(z_bottom);
  }
  if (type == "gaussian_layers") {
    check_keys(j, {"type", "z_bottom", "bulk_period", "layers"}, ctx);
    const json& jl = require(j, "layers", ctx);
    if (!jl.is_array() || jl.empty()) throw mb::ConfigError("config: field.layers must be a nonempty array");
    std::vector<mb::GaussianLayer> layers;
    for (std::size_t i = 0; i < jl.size(); ++i) {
      const std::string lc = "field.layers[" + std::to_string(i) + "]";
      require_object(jl[i], lc);
      check_keys(jl[i], {"z_center", "amplitude", "sigma_xy", "sigma_z", "absorption"}, lc);
      mb::GaussianLayer l;
      l.z_center = as_number(require(jl[i], "z_center", lc), lc + ".z_center");
      l.amplitude = as_number(require(jl[i], "amplitude", lc), lc + ".amplitude");
      l.sigma_xy = as_number(require(jl[i], "sigma_xy", lc), lc + ".sigma_xy");
      l.sigma_z = as_number(require(jl[i], "sigma_z", lc), lc + ".sigma_z");
      if (const json* p = find(jl[i], "absorption")) l.absorption = as_number(*p, lc + ".absorption");
      layers.push_back(l);
    }
    return mb::PotentialField::gaussian_layers(z_bottom, layers, bulk);
  }
  if (type == "tabulated") {
    check_keys(j, {"type", "z_bottom", "bulk_period", "z_grid", "coefficients"}, ctx);
    const std::vector<double> z_grid = as_number_list(require(j, "z_grid", ctx), ctx + ".z_grid");
    const json& jc = require(j, "coefficients", ctx);
    if (!jc.is_array() || jc.empty()) throw mb::ConfigError("config: field.coefficients must be a nonempty array");
    std::vector<std::pair<std::array<int, 2>, std::vector<mb::Complex>>> entries;
    for (std::size_t i = 0; i < jc.size(); ++i) {
      const std::string ec = "field.coefficients[" + std::to_string(i) + "]";
      require_object(jc[i], ec);
      check_keys(jc[i], {"dm", "re", "im"}, ec);
      const json& jdm = require(jc[i], "dm", ec);
      if (!jdm.is_array() || jdm.size() != 2) throw mb::ConfigError(where(ec) + ".dm must be a 2-element integer array");
      const std::array<int, 2> dm{(int)as_integer(jdm[0], ec + ".dm[0]"), (int)as_integer(jdm[1], ec + ".dm[1]")};
      const std::vector<double> re = as_number_list(require(jc[i], "re", ec), ec + ".re");
      const std::vector<double> im = as_number_list(require(jc[i], "im", ec), ec + ".im");
      if (re.size() != im.size()) throw mb::ConfigError(where(ec) + ": re and im lengths differ");
      std::vector<mb::Complex> v;
      for (std::size_t k = 0; k < re.size(); ++k) v.emplace_back(re[k], im[k]);
      entries.emplace_back(dm, std::move(v));
    }
    return mb::PotentialField::tabulated(z_bottom, z_grid, entries, bulk);
  }
  if (type == "atoms") {  // EXTENSION
    check_keys(j, {"type", "z_bottom", "bulk_period", "absorption", "species", "atoms"}, ctx);
    const json& js = require(j, "species", ctx);
    if (!js.is_array() || js.empty()) throw mb::ConfigError("config: field.species must be a nonempty array");
    std::vector<std::array<double, 4>> fa, fb;
    for (std::size_t i = 0; i < js.size(); ++i) {
      const std::string sc = "field.species[" + std::to_string(i) + "]";
      require_object(js[i], sc);
      check_keys(js[i], {"a", "b", "label"}, sc);
      const std::vector<double> a = as_number_list(require(js[i], "a", sc), sc + ".a");
      const std::vector<double> b = as_number_list(require(js[i], "b", sc), sc + ".b");
      if (a.size() != 4 || b.size() != 4) throw mb::ConfigError(where(sc) + ": a and b need 4 Gaussian terms");
      fa.push_back({a[0], a[1], a[2], a[3]});
      fb.push_back({b[0], b[1], b[2], b[3]});
    }
    const json& ja = require(j, "atoms", ctx);
    if (!ja.is_array() || ja.empty()) throw mb::ConfigError("config: field.atoms must be a nonempty array");
    std::vector<mb::PotentialField::Atom> atoms;
    for (std::size_t i = 0; i < ja.size(); ++i) {
      const std::string ac = "field.atoms[" + std::to_string(i) + "]";
      require_object(ja[i], ac);
      check_keys(ja[i], {"xyz", "species", "B"}, ac);
      const std::vector<double> x = as_number_list(require(ja[i], "xyz", ac), ac + ".xyz");
      if (x.size() != 3) throw mb::ConfigError(where(ac) + ".xyz must have 3 components");
      const long s = as_integer(require(ja[i], "species", ac), ac + ".species");
      const double B = as_number(require(ja[i], "B", ac), ac + ".B");
      atoms.push_back(mb::PotentialField::Atom{x[0], x[1], x[2], (int)s, B});
    }
    const double absorption = find(j, "absorption") ? as_number(*find(j, "absorption"), ctx + ".absorption") : 0.1;
    const double area = std::abs(cfg.lattice.a1.x * cfg.lattice.a2.y - cfg.lattice.a1.y * cfg.lattice.a2.x);
    return mb::PotentialField::atoms(z_bottom, atoms, fa, fb, area, cfg.gamma_L, cfg.particle_sign, absorption, bulk);
  }
  throw mb::ConfigError("config: field.type '" + type + "' not recognized (zero, gaussian_layers, tabulated, atoms)");
}

double parse_threshold(const json& j) {
  if (j.is_string()) {
    if (j.get<std::string>() == "inf") return std::numeric_limits<double>::infinity();
    throw mb::ConfigError("config: rhst_threshold string form must be \"inf\"");
  }
  const double v = as_number(j, "rhst_threshold");
  if (v < 0.0) throw mb::ConfigError("config: rhst_threshold must be >= 0");
  return v;
}

BenchRun parse_bench_run(const json& j, const std::string& ctx) {
  require_object(j, ctx);
  check_keys(j, {"method", "dz"}, ctx);
  BenchRun r;
  r.method = as_string(require(j, "method", ctx), ctx + ".method");
  check_method_name(r.method, ctx);
  r.dz = as_number(require(j, "dz", ctx), ctx + ".dz");
  if (!(r.dz > 0.0)) throw mb::ConfigError(where(ctx) + ".dz must be positive");
  return r;
}

BenchCfg parse_bench(const json& j) {
  const std::string ctx = "bench";
  require_object(j, ctx);
  check_keys(j, {"reference", "baseline", "methods", "dz_values", "repeats"}, ctx);
  BenchCfg b;
  b.reference = parse_bench_run(require(j, "reference", ctx), "bench.reference");
  if (const json* p = find(j, "baseline")) b.baseline = parse_bench_run(*p, "bench.baseline");
  if (const json* p = find(j, "methods")) {
    if (!p->is_array()) throw mb::ConfigError("config: bench.methods must be an array of strings");
    for (const auto& m : *p) {
      if (!m.is_string()) throw mb::ConfigError("config: bench.methods must be an array of strings");
      b.methods.push_back(m.get<std::string>());
      check_method_name(b.methods.back(), "bench.methods");
    }
  }
  if (const json* p = find(j, "dz_values")) {
    b.dz_values = as_number_list(*p, "bench.dz_values");
    for (double d : b.dz_values)
      if (!(d > 0.0)) throw mb::ConfigError("config: bench.dz_values must be positive");
  }
  if (const json* p = find(j, "repeats")) {
    b.repeats = (int)as_integer(*p, "bench.repeats");
    if (b.repeats < 3) throw mb::ConfigError("config: bench.repeats must be >= 3");
  }
  return b;
}

// config.cpp:223-270 (+ extensions)
RunConfig parse_config(const json& j) {
  require_object(j, "");
  check_keys(j,
             {"gamma", "energy_ev", "particle", "lattice", "rod_cutoff", "rod_count", "field", "angles", "method",
              "dz", "slices", "rhst_threshold", "threads", "out", "bench", "devices", "fsal"},
             "");
  RunConfig cfg;
  if (const json* pe = find(j, "energy_ev")) {  // EXTENSION: relativistic beam
    if (find(j, "gamma")) throw mb::ConfigError("config: give either gamma or energy_ev, not both");
    const double e = as_number(*pe, "energy_ev");
    mb::check(mb_beam_from_energy(e, &cfg.gamma, &cfg.gamma_L));
    cfg.have_energy = true;
  } else {
    cfg.gamma = as_number(require(j, "gamma", ""), "gamma");
    if (!(cfg.gamma > 0.0)) throw mb::ConfigError("config: gamma must be positive");
  }
  if (const json* p = find(j, "particle")) {
    const std::string s = as_string(*p, "particle");
    if (s != "electron" && s != "positron") throw mb::ConfigError("config: particle must be electron or positron");
    cfg.particle_sign = s == "electron" ? 1.0 : -1.0;
  }
  const json& jl = require(j, "lattice", "");
  require_object(jl, "lattice");
  check_keys(jl, {"a1", "a2"}, "lattice");
  cfg.lattice.a1 = as_vec2(require(jl, "a1", "lattice"), "lattice.a1");
  cfg.lattice.a2 = as_vec2(require(jl, "a2", "lattice"), "lattice.a2");
  if (const json* p = find(j, "rod_count")) {  // EXTENSION: first-N rods
    if (find(j, "rod_cutoff")) throw mb::ConfigError("config: give either rod_cutoff or rod_count, not both");
    cfg.rod_count = (int)as_integer(*p, "rod_count");
    if (cfg.rod_count < 1) throw mb::ConfigError("config: rod_count must be >= 1");
  } else {
    cfg.rod_cutoff = as_number(require(j, "rod_cutoff", ""), "rod_cutoff");
    if (!(cfg.rod_cutoff >= 0.0)) throw mb::ConfigError("config: rod_cutoff must be >= 0");
  }
  cfg.field = parse_field(require(j, "field", ""), cfg);
  const json& ja = require(j, "angles", "");
  require_object(ja, "angles");
  check_keys(ja, {"theta0", "theta1"}, "angles");
  std::vector<double> th0 = parse_axis(require(ja, "theta0", "angles"), "angles.theta0");
  std::vector<double> th1{0.0};
  if (const json* p = find(ja, "theta1")) th1 = parse_axis(*p, "angles.theta1");
  cfg.angles = mb::AngleGrid::validated(std::move(th0), std::move(th1));
  if (const json* p = find(j, "method")) {
    cfg.method = as_string(*p, "method");
    check_method_name(cfg.method, "method");
  }
  if (const json* p = find(j, "dz")) {
    cfg.dz = as_number(*p, "dz");
    if (!(cfg.dz > 0.0)) throw mb::ConfigError("config: dz must be positive");
  }
  if (const json* p = find(j, "slices")) {
    cfg.slices = as_integer(*p, "slices");
    if (cfg.slices < 1) throw mb::ConfigError("config: slices must be >= 1");
  }
  if (const json* p = find(j, "rhst_threshold")) cfg.rhst_threshold = parse_threshold(*p);
  if (const json* p = find(j, "threads")) {
    cfg.threads = (int)as_integer(*p, "threads");
    if (cfg.threads < 0) throw mb::ConfigError("config: threads must be >= 0");
  }
  if (const json* p = find(j, "fsal")) {
    if (!p->is_boolean()) throw mb::ConfigError("config: fsal must be true or false");
    cfg.fsal = p->get<bool>();
  }
  if (const json* p = find(j, "devices")) {
    for (double d : as_number_list(*p, "devices")) {
      if (d < 0 || d != std::floor(d)) throw mb::ConfigError("config: devices must be device indices");
      cfg.devices.push_back((int)d);
    }
    if (cfg.devices.empty()) throw mb::ConfigError("config: devices must not be empty");
  }
  if (const json* p = find(j, "out")) cfg.out = as_string(*p, "out");
  if (const json* p = find(j, "bench")) cfg.bench = parse_bench(*p);
  return cfg;
}

RunConfig load_config(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw mb::IoError("cannot open config '" + path + "'");
  json j;
  try {
    j = json::parse(is);
  } catch (const json::parse_error& e) {
    throw mb::ConfigError(std::string("config: invalid JSON: ") + e.what());
  }
  return parse_config(j);
}

// ------------------------------------------------------------------ driver (driver.cpp)
const std::vector<double> kBenchDzPresets = {0.010, 0.015, 0.022, 0.033, 0.047, 0.068,
                                             0.10,  0.15,  0.22,  0.33,  0.47,  0.68};

mb::RockingCurve solve_with(const RunConfig& cfg, const std::string& method, double dz) {
  mb::SweepOptions o;
  o.method = method;
  o.dz = dz;
  o.slices = cfg.slices;
  o.rhst_threshold = cfg.rhst_threshold;
  o.fsal = cfg.fsal;
  o.devices = cfg.devices;
  const mb::RodSet rods = cfg.rod_count > 0 ? mb::RodSet::build_first(cfg.lattice, cfg.rod_count)
                                            : mb::RodSet::build(cfg.lattice, cfg.rod_cutoff);
  return mb::rocking_curve(*cfg.field, rods, cfg.gamma, cfg.angles, o);
}

double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  const std::size_t n = v.size();
  return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

struct BenchRecord {
  std::string method;
  double dz = 0.0;
  int repeats = 0;
  double median_seconds = 0.0, err_reference = 0.0;
  std::optional<double> err_baseline;
  std::string status = "ok", detail;
};

std::vector<BenchRecord> run_bench(const RunConfig& cfg, std::vector<std::string> methods,
                                   std::vector<double> dz_values, int repeats) {
  if (!cfg.bench) throw mb::ConfigError("bench: config has no \"bench\" section");
  const BenchCfg& bench = *cfg.bench;
  if (methods.empty())
    methods = bench.methods.empty() ? std::vector<std::string>{"conventional", "rk4", "sp4", "sp6"} : bench.methods;
  for (const std::string& m : methods) check_method_name(m, "--methods");
  if (dz_values.empty()) dz_values = bench.dz_values.empty() ? kBenchDzPresets : bench.dz_values;
  if (repeats < 1) repeats = bench.repeats;
  if (repeats < 3) throw mb::ConfigError("bench: repeats must be >= 3");
  const mb::RockingCurve reference = solve_with(cfg, bench.reference.method, bench.reference.dz);
  mb::RockingCurve baseline;
  if (bench.baseline) baseline = solve_with(cfg, bench.baseline->method, bench.baseline->dz);
  std::vector<BenchRecord> records;
  for (const std::string& method : methods)
    for (double dz : dz_values) {
      BenchRecord rec;
      rec.method = method;
      rec.dz = dz;
      rec.repeats = repeats;
      try {
        mb::RockingCurve curve;
        std::vector<double> times;
        for (int r = 0; r < repeats; ++r) {
          const auto t0 = std::chrono::steady_clock::now();
          curve = solve_with(cfg, method, dz);
          times.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        }
        rec.median_seconds = median(std::move(times));
        rec.err_reference = mb::curve_error(curve, reference);
        if (bench.baseline) rec.err_baseline = mb::curve_error(curve, baseline);
      } catch (const mb::Error& e) {
        rec.status = "failed";
        rec.detail = e.what();
        rec.median_seconds = 0.0;
        rec.err_reference = 0.0;
        rec.err_baseline.reset();
      }
      records.push_back(std::move(rec));
    }
  return records;
}

// csvio.cpp:151-171
std::string sanitize(std::string s) {
  for (char& c : s)
    if (c == ',' || c == '\n' || c == '\r') c = ';';
  return s;
}
void write_bench_csv(const std::string& path, const std::vector<BenchRecord>& records) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw mb::IoError("cannot open '" + path + "' for writing");
  os << "# manybeam-bench v1\n";
  os << "method,dz,repeats,median_seconds,err_reference,err_baseline,status,detail\n";
  for (const auto& r : records) {
    os << r.method << ',' << mb::format_full(r.dz) << ',' << r.repeats << ',' << mb::format_full(r.median_seconds)
       << ',' << (std::isinf(r.err_reference) ? std::string("inf") : mb::format_full(r.err_reference)) << ',';
    if (r.err_baseline)
      os << (std::isinf(*r.err_baseline) ? std::string("inf") : mb::format_full(*r.err_baseline));
    os << ',' << r.status << ',' << sanitize(r.detail) << "\n";
  }
  os.flush();
  if (!os) throw mb::IoError("write to '" + path + "' failed");
}

// ------------------------------------------------------------------ CLI
struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

const char* kHelp =
    "many-beam reflective diffraction engine (B200 path)\n"
    "Usage: manybeam_b200 [--threads N] [--version] [--help] SUBCOMMAND\n"
    "  simulate --config FILE [--out FILE]   solve a rocking curve and write its CSV\n"
    "  bench --config FILE --out FILE [--dz a,b] [--methods m,..] [--repeats K]\n"
    "                                        time methods across step widths\n"
    "  compare fileA fileB                   distance between two curve CSVs\n";

std::vector<std::string> split_list(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ','))
    if (!item.empty()) out.push_back(item);
  return out;
}

// exit codes (main.cpp:14-20): 2 config, 3 solver, 4 comparison, 5 I/O
int code_for(const std::exception& e) {
  if (dynamic_cast<const mb::ConfigError*>(&e)) return 2;
  if (dynamic_cast<const mb::CompareError*>(&e)) return 4;
  if (dynamic_cast<const mb::IoError*>(&e)) return 5;
  if (dynamic_cast<const mb::SolverError*>(&e)) return 3;
  return 1;
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  std::string sub, config, out, cmp_a, cmp_b;
  std::vector<std::string> methods;
  std::vector<double> dzs;
  int threads = -1, repeats = 0;
  try {
    std::vector<std::string> positional;
    for (std::size_t i = 0; i < args.size(); ++i) {
      const std::string& a = args[i];
      auto value = [&]() -> std::string {
        if (i + 1 >= args.size()) throw Usage(a + " needs a value");
        return args[++i];
      };
      if (a == "--help" || a == "-h") {
        std::printf("%s", kHelp);
        return 0;
      }
      if (a == "--version") {
        std::printf("manybeam 0.1.0 (b200)\n");
        return 0;
      }
      if (a == "--threads") {
        try {
          threads = std::stoi(value());
        } catch (const std::logic_error&) {
          throw Usage("--threads needs an integer");
        }
        continue;
      }
      if (sub.empty()) {
        if (a == "simulate" || a == "bench" || a == "compare") {
          sub = a;
          continue;
        }
        throw Usage("unknown subcommand or option '" + a + "'");
      }
      if (a == "--config" && sub != "compare") {
        config = value();
      } else if (a == "--out" && sub != "compare") {
        out = value();
      } else if (a == "--dz" && sub == "bench") {
        for (const std::string& s : split_list(value())) {
          try {
            dzs.push_back(std::stod(s));
          } catch (const std::logic_error&) {
            throw Usage("--dz needs numbers");
          }
        }
      } else if (a == "--methods" && sub == "bench") {
        methods = split_list(value());
      } else if (a == "--repeats" && sub == "bench") {
        try {
          repeats = std::stoi(value());
        } catch (const std::logic_error&) {
          throw Usage("--repeats needs an integer");
        }
      } else if (sub == "compare" && !a.empty() && a[0] != '-') {
        positional.push_back(a);
      } else {
        throw Usage("unknown option '" + a + "' for " + sub);
      }
    }
    if (sub.empty()) throw Usage("a subcommand is required");
    if (sub != "compare" && config.empty()) throw Usage("--config is required");
    if (sub == "bench" && out.empty()) throw Usage("--out is required");
    if (sub == "compare") {
      if (positional.size() != 2) throw Usage("compare needs fileA and fileB");
      cmp_a = positional[0];
      cmp_b = positional[1];
    }
  } catch (const Usage& e) {
    std::fprintf(stderr, "%s\n%s", e.what(), kHelp);
    return 2;
  }

  try {
    if (sub == "simulate") {
      RunConfig cfg = load_config(config);
      if (threads >= 0) cfg.threads = threads;
      const std::string& path = out.empty() ? cfg.out : out;
      if (path.empty()) throw mb::ConfigError("simulate: no output path (config \"out\" or --out)");
      mb::write_curve_csv(path, solve_with(cfg, cfg.method, cfg.dz));
    } else if (sub == "bench") {
      RunConfig cfg = load_config(config);
      if (threads >= 0) cfg.threads = threads;
      write_bench_csv(out, run_bench(cfg, methods, dzs, repeats));
    } else {
      std::printf("%s\n", mb::format_full(mb::compare_curve_files(cmp_a, cmp_b)).c_str());
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return code_for(e);
  }
  return 0;
}
