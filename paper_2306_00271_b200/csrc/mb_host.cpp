// Host runtime of the B200-native forward model: the C-ABI of
// include/manybeam_b200.h. Host-side logic restates the reference's setup
// layers (rods, beam geometry, slicing, node schedules, stepper tables;
// /root/reference/proj/core/src/{rods,geometry,stages,proposed,
// splitting_coefficients}.cpp) and stages every input on the device once per
// plan; all per-slice arithmetic runs in the sm_100a kernels (mb_kernels.cu).
// There is no CPU solve path: without a device every solve fails with
// MB_ERR_CUDA.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <thread>
#include <exception>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/manybeam_b200.h"
#include "mb_internal.h"

constexpr int kBigParts = 4;  // batched path: most sub-batches (streams) of one execute

namespace {

using cd = std::complex<double>;
constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kDegToRad = kPi / 180.0;

thread_local std::string g_last_error;

struct MbError : std::runtime_error {
  int code;
  MbError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& msg) { throw MbError(code, msg); }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(MB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return MB_OK;
  } catch (const MbError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return MB_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MB_ERR_SOLVER;
  }
}

// ------------------------------------------------------------------ rods
// rods.cpp:14-96 (+ first-N extension)
struct V2 {
  double x, y;
};
struct Rod {
  V2 k;
  int m1, m2;
};
double vnorm(V2 v) { return std::sqrt(v.x * v.x + v.y * v.y); }

struct Lattice {
  V2 a1, a2;
  V2 b1() const {
    const double det = a1.x * a2.y - a1.y * a2.x;
    return V2{kTwoPi * a2.y / det, -kTwoPi * a2.x / det};
  }
  V2 b2() const {
    const double det = a1.x * a2.y - a1.y * a2.x;
    return V2{-kTwoPi * a1.y / det, kTwoPi * a1.x / det};
  }
  void validate() const {
    const double det = a1.x * a2.y - a1.y * a2.x;
    const double scale = vnorm(a1) * vnorm(a2);
    if (!(std::abs(det) > 1e-12 * std::max(scale, 1e-300)))
      fail(MB_ERR_CONFIG, "lattice: basis vectors are degenerate (zero cell area)");
    if (!std::isfinite(a1.x) || !std::isfinite(a1.y) || !std::isfinite(a2.x) || !std::isfinite(a2.y))
      fail(MB_ERR_CONFIG, "lattice: nonfinite basis");
  }
};

std::vector<Rod> enumerate_rods(const Lattice& lat, double cutoff) {
  const V2 b1 = lat.b1(), b2 = lat.b2();
  const int m1max = (int)std::floor(cutoff * vnorm(lat.a1) / kTwoPi + 1e-9);
  const int m2max = (int)std::floor(cutoff * vnorm(lat.a2) / kTwoPi + 1e-9);
  std::vector<Rod> rods;
  for (int m1 = -m1max; m1 <= m1max; ++m1)
    for (int m2 = -m2max; m2 <= m2max; ++m2) {
      const V2 k{m1 * b1.x + m2 * b2.x, m1 * b1.y + m2 * b2.y};
      if (vnorm(k) <= cutoff) rods.push_back(Rod{k, m1, m2});
    }
  std::sort(rods.begin(), rods.end(), [](const Rod& p, const Rod& q) {
    const double np = vnorm(p.k), nq = vnorm(q.k);
    if (np != nq) return np < nq;
    if (p.k.x != q.k.x) return p.k.x < q.k.x;
    return p.k.y < q.k.y;
  });
  return rods;
}

struct RodTables {
  std::vector<Rod> rods;
  std::vector<V2> diff;
  std::vector<std::pair<int, int>> diff_m;
  std::vector<int> diff_index;
};

RodTables build_rods(const Lattice& lat, double cutoff, int first_n) {
  lat.validate();
  std::vector<Rod> rods;
  if (first_n > 0) {
    const double bmin = std::min(vnorm(lat.b1()), vnorm(lat.b2()));
    double c = 0.5 * bmin;
    for (;;) {
      rods = enumerate_rods(lat, c);
      if ((int)rods.size() >= first_n) break;
      c *= 1.25;
    }
    rods.resize((std::size_t)first_n);
  } else {
    if (!(cutoff > 0.0) || !std::isfinite(cutoff)) fail(MB_ERR_CONFIG, "rod cutoff must be positive and finite");
    rods = enumerate_rods(lat, cutoff);
  }
  if (rods.empty() || rods.front().m1 != 0 || rods.front().m2 != 0)
    fail(MB_ERR_CONFIG, "rod set does not contain the zero rod");
  RodTables t;
  t.rods = rods;
  const int n = (int)rods.size();
  const V2 b1 = lat.b1(), b2 = lat.b2();
  std::map<std::pair<int, int>, int> seen;
  t.diff_index.assign((std::size_t)n * n, -1);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      const int d1 = rods[j].m1 - rods[k].m1, d2 = rods[j].m2 - rods[k].m2;
      auto key = std::make_pair(d1, d2);
      auto it = seen.find(key);
      int d;
      if (it == seen.end()) {
        d = (int)t.diff.size();
        seen.emplace(key, d);
        t.diff.push_back(V2{d1 * b1.x + d2 * b2.x, d1 * b1.y + d2 * b2.y});
        t.diff_m.push_back(key);
      } else {
        d = it->second;
      }
      t.diff_index[(std::size_t)j * n + k] = d;
    }
  return t;
}

// ------------------------------------------------------------------ steppers
// splitting_coefficients.cpp:13-77 (published constants; trailing entries by
// symmetry and the sum rule)
struct Tables {
  double sp4_drift[6], sp4_kick[7], sp6_drift[11], sp6_kick[12];
  Tables() {
    const double b1 = 0.0829844064174052, b2 = 0.396309801498368, b3 = -0.0390563049223486;
    const double b4 = 1.0 - 2.0 * (b1 + b2 + b3);
    const double a1 = 0.245298957184271, a2 = 0.604872665711080;
    const double a3 = 0.5 - (a1 + a2);
    const double d4[6] = {a1, a2, a3, a3, a2, a1};
    const double k4[7] = {b1, b2, b3, b4, b3, b2, b1};
    std::memcpy(sp4_drift, d4, sizeof d4);
    std::memcpy(sp4_kick, k4, sizeof k4);
    const double c1 = 0.0414649985182624, c2 = 0.198128671918067, c3 = -0.0400061921041533;
    const double c4 = 0.0752539843015807, c5 = -0.0115113874206879;
    const double c6 = 0.5 - (c1 + c2 + c3 + c4 + c5);
    const double e1 = 0.123229775946271, e2 = 0.290553797799558, e3 = -0.127049212625417;
    const double e4 = -0.246331761062075, e5 = 0.357208872795928;
    const double e6 = 1.0 - 2.0 * (e1 + e2 + e3 + e4 + e5);
    const double d6[11] = {e1, e2, e3, e4, e5, e6, e5, e4, e3, e2, e1};
    const double k6[12] = {c1, c2, c3, c4, c5, c6, c6, c5, c4, c3, c2, c1};
    std::memcpy(sp6_drift, d6, sizeof d6);
    std::memcpy(sp6_kick, k6, sizeof k6);
  }
};
const Tables& tables() {
  static const Tables t;
  return t;
}

// proposed.cpp:36-60
void validate_stepper(const mb_stepper& s) {
  if (s.algorithm == MB_STEP_RK4 || s.algorithm == MB_STEP_CONVENTIONAL) return;
  if (s.algorithm != MB_STEP_SPLITTING) fail(MB_ERR_CONFIG, "stepper: unknown algorithm");
  const int nd = s.ndrift, nk = s.nkick;
  const bool shape_ok = s.variant == MB_SPLIT_BAB ? (nk == nd + 1) : (nd == nk + 1);
  if (nd <= 0 || nk <= 0 || !shape_ok || !s.drift || !s.kick)
    fail(MB_ERR_CONFIG, "stepper: BAB needs s drifts and s+1 kicks, ABA the reverse");
  double sa = 0.0, sb = 0.0;
  for (int i = 0; i < nd; ++i) {
    if (!std::isfinite(s.drift[i])) fail(MB_ERR_CONFIG, "stepper: nonfinite drift coefficient");
    sa += s.drift[i];
  }
  for (int i = 0; i < nk; ++i) {
    if (!std::isfinite(s.kick[i])) fail(MB_ERR_CONFIG, "stepper: nonfinite kick coefficient");
    sb += s.kick[i];
  }
  if (std::abs(sa - 1.0) > 1e-13 || std::abs(sb - 1.0) > 1e-13)
    fail(MB_ERR_CONFIG, "stepper: drift and kick coefficients must each sum to 1");
  // occ_kick / occ_drift hold one entry per kick and per drift (ABA has one
  // more drift than kicks)
  if (std::max(nk, nd) > mbx::kMaxOcc) fail(MB_ERR_CONFIG, "stepper: too many stages for the device kernel");
}

// stages.cpp:12-23
std::vector<double> schedule_from_fracs(std::vector<double> raw) {
  for (double& f : raw) {
    if (std::abs(f) < 1e-12) f = 0.0;
    if (std::abs(f - 1.0) < 1e-12) f = 1.0;
  }
  std::sort(raw.begin(), raw.end());
  std::vector<double> u;
  for (double f : raw)
    if (u.empty() || f - u.back() > 1e-12) u.push_back(f);
  return u;
}

// node schedule + kick occurrence -> node (proposed.cpp:62-100, stages.cpp:10)
struct Schedule {
  std::vector<double> frac;
  std::vector<int> occ2node;
  bool endpoint_pair() const { return frac.size() >= 2 && frac.front() == 0.0 && frac.back() == 1.0; }
};
Schedule make_schedule(const mb_stepper& s) {
  Schedule sc;
  if (s.algorithm == MB_STEP_CONVENTIONAL) {  // midpoint_schedule (stages.cpp:8), conventional.cpp:56
    sc.frac = {0.5};
    sc.occ2node = {0};
    return sc;
  }
  if (s.algorithm == MB_STEP_RK4) {
    sc.frac = {0.0, 0.5, 1.0};
    sc.occ2node = {0, 1, 1, 2};  // RK4 stages: foot, mid, mid, top
    return sc;
  }
  std::vector<double> fr;
  double c = 0.0;
  if (s.variant == MB_SPLIT_BAB) {
    fr.push_back(0.0);
    for (int i = 0; i < s.ndrift; ++i) {
      c += s.drift[i];
      fr.push_back(c);
    }
  } else {
    for (int r = 0; r < s.nkick; ++r) {
      c += s.drift[r];
      fr.push_back(c);
    }
  }
  sc.frac = schedule_from_fracs(fr);
  for (double raw : fr) {
    double f = raw;
    if (std::abs(f) < 1e-12) f = 0.0;
    if (std::abs(f - 1.0) < 1e-12) f = 1.0;
    int best = 0;
    double dist = std::numeric_limits<double>::infinity();
    for (int m = 0; m < (int)sc.frac.size(); ++m) {
      const double d = std::abs(sc.frac[m] - f);
      if (d < dist) {
        dist = d;
        best = m;
      }
    }
    sc.occ2node.push_back(best);
  }
  return sc;
}

// ------------------------------------------------------------------ fields
// potential.cpp:17-88 validation (+ atoms extension)
void validate_field(const mb_field& f) {
  if (!(f.z_bottom < 0.0) || !std::isfinite(f.z_bottom))
    fail(MB_ERR_CONFIG, "potential: z_bottom must be negative and finite");
  if (f.has_bulk_period) {  // potential.cpp:22-28
    if (!(f.bulk_period > 0.0) || !std::isfinite(f.bulk_period))
      fail(MB_ERR_CONFIG, "potential: bulk_period must be positive and finite");
    if (f.bulk_period > -f.z_bottom + 1e-9) fail(MB_ERR_CONFIG, "potential: bulk_period must not exceed |z_bottom|");
  }
  switch (f.kind) {
    case MB_FIELD_ZERO:
      return;
    case MB_FIELD_GAUSSIAN_LAYERS:
      if (f.nlayers < 0 || (f.nlayers > 0 && !f.layers)) fail(MB_ERR_ARG, "potential: layers missing");
      for (int i = 0; i < f.nlayers; ++i) {
        const double* l = f.layers + 5 * i;
        bool fin = true;
        for (int q = 0; q < 5; ++q) fin = fin && std::isfinite(l[q]);
        if (!fin || !(l[2] > 0.0) || !(l[3] > 0.0) || l[4] < 0.0)
          fail(MB_ERR_CONFIG, "potential: layer " + std::to_string(i) +
                                  " needs sigma_xy > 0, sigma_z > 0, absorption >= 0, finite values");
      }
      return;
    case MB_FIELD_TABULATED: {
      if (f.ngrid < 2 || !f.z_grid) fail(MB_ERR_CONFIG, "potential: tabulated z_grid needs at least 2 points");
      for (int i = 0; i + 1 < f.ngrid; ++i)
        if (!(f.z_grid[i] < f.z_grid[i + 1]))
          fail(MB_ERR_CONFIG, "potential: tabulated z_grid must be strictly increasing");
      if (f.z_grid[0] > f.z_bottom + 1e-9 || f.z_grid[f.ngrid - 1] < -1e-9)
        fail(MB_ERR_CONFIG, "potential: tabulated z_grid must cover [z_bottom, 0]");
      for (long i = 0; i < (long)f.nentries * f.ngrid * 2; ++i)
        if (!std::isfinite(f.entry_values[i])) fail(MB_ERR_CONFIG, "potential: tabulated entry has nonfinite sample");
      return;
    }
    case MB_FIELD_ATOMS:
      if (!(f.cell_area > 0.0)) fail(MB_ERR_CONFIG, "atoms: cell area must be positive");
      if (!(f.absorption >= 0.0)) fail(MB_ERR_CONFIG, "atoms: absorption must be >= 0");
      if (f.natoms > 0 && (!f.atom_xyz || !f.atom_species || !f.atom_B || !f.ff_a || !f.ff_b))
        fail(MB_ERR_ARG, "atoms: arrays missing");
      for (int a = 0; a < f.natoms; ++a) {
        const int sp = f.atom_species[a];
        if (sp < 0 || sp >= f.nspecies) fail(MB_ERR_CONFIG, "atoms: species index out of range");
        if (!(f.atom_B[a] >= 0.0)) fail(MB_ERR_CONFIG, "atoms: need B >= 0");
        for (int q = 0; q < 3; ++q)
          if (!std::isfinite(f.atom_xyz[3 * a + q])) fail(MB_ERR_CONFIG, "atoms: nonfinite position");
        for (int i = 0; i < 4; ++i)
          if (!(f.ff_b[4 * sp + i] + f.atom_B[a] > 0.0))
            fail(MB_ERR_CONFIG, "atoms: form-factor widths b_i + B must be positive");
      }
      return;
    default:
      fail(MB_ERR_CONFIG, "potential: unknown field kind");
  }
}

// Hermite evaluation of a tabulated field at z (potential.cpp:115-148,186-199),
// host side: the device consumes the resulting node-slot table.
struct Tabulated {
  std::vector<double> z;
  std::vector<std::vector<cd>> y, s;  // [diff][grid]
};
Tabulated bind_tabulated(const mb_field& f, const RodTables& rt) {
  std::map<std::pair<int, int>, int> by_dm;
  for (int e = 0; e < f.nentries; ++e) by_dm[{f.entry_dm[2 * e], f.entry_dm[2 * e + 1]}] = e;
  Tabulated t;
  t.z.assign(f.z_grid, f.z_grid + f.ngrid);
  const std::size_t g = t.z.size();
  for (std::size_t d = 0; d < rt.diff.size(); ++d) {
    auto it = by_dm.find(rt.diff_m[d]);
    if (it == by_dm.end())
      fail(MB_ERR_CONFIG, "potential: tabulated field lacks coefficient for rod difference (" +
                              std::to_string(rt.diff_m[d].first) + "," + std::to_string(rt.diff_m[d].second) + ")");
    std::vector<cd> y(g), s(g);
    for (std::size_t i = 0; i < g; ++i)
      y[i] = cd(f.entry_values[((std::size_t)it->second * g + i) * 2], f.entry_values[((std::size_t)it->second * g + i) * 2 + 1]);
    const std::vector<double>& z = t.z;
    if (g == 2) {
      s[0] = s[1] = (y[1] - y[0]) / (z[1] - z[0]);
    } else {
      for (std::size_t i = 1; i + 1 < g; ++i) {
        const double hl = z[i] - z[i - 1], hr = z[i + 1] - z[i];
        s[i] = ((y[i + 1] - y[i]) / hr * hl + (y[i] - y[i - 1]) / hl * hr) / (hl + hr);
      }
      const double h0 = z[1] - z[0], h1 = z[2] - z[1];
      s[0] = -(2.0 * h0 + h1) / (h0 * (h0 + h1)) * y[0] + (h0 + h1) / (h0 * h1) * y[1] - h0 / (h1 * (h0 + h1)) * y[2];
      const double k0 = z[g - 2] - z[g - 3], k1 = z[g - 1] - z[g - 2];
      s[g - 1] = k1 / (k0 * (k0 + k1)) * y[g - 3] - (k0 + k1) / (k0 * k1) * y[g - 2] +
                 (2.0 * k1 + k0) / (k1 * (k0 + k1)) * y[g - 1];
    }
    t.y.push_back(std::move(y));
    t.s.push_back(std::move(s));
  }
  return t;
}
double map_z(double z, double zb, double period = 0.0) {  // potential.cpp:152-167
  if (z > 1e-9 || !std::isfinite(z)) fail(MB_ERR_DOMAIN, "potential evaluated above the surface");
  if (z > 0.0) z = 0.0;
  if (z >= zb) return z;
  if (z >= zb - 1e-9) return zb;
  if (!(period > 0.0)) fail(MB_ERR_DOMAIN, "potential evaluated below z_bottom without a bulk period");
  const double k = std::ceil((zb - z) / period - 1e-12);
  double zm = z + k * period;
  if (zm < zb) zm += period;
  if (zm > zb + period) zm = zb + period;
  return std::min(zm, 0.0);
}
void eval_tabulated(const Tabulated& t, double zb, double z, cd* out) {
  const double zm = map_z(z, zb);
  const std::size_t g = t.z.size();
  std::size_t i = (std::size_t)(std::upper_bound(t.z.begin(), t.z.end(), zm) - t.z.begin());
  if (i == 0) i = 1;
  if (i >= g) i = g - 1;
  const double zl = t.z[i - 1], zr = t.z[i], h = zr - zl;
  const double tt = std::clamp((zm - zl) / h, 0.0, 1.0);
  const double t2 = tt * tt, t3 = t2 * tt;
  const double h00 = 2 * t3 - 3 * t2 + 1, h10 = t3 - 2 * t2 + tt, h01 = -2 * t3 + 3 * t2, h11 = t3 - t2;
  for (std::size_t d = 0; d < t.y.size(); ++d)
    out[d] = h00 * t.y[d][i - 1] + h10 * h * t.s[d][i - 1] + h01 * t.y[d][i] + h11 * h * t.s[d][i];
}

// ------------------------------------------------------------------ context
struct DevBuf {
  void* p = nullptr;
  std::size_t bytes = 0;
};

}  // namespace

struct mb_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  // multi-device context (mb_context_create_multi): one single-device
  // sub-context per listed device; empty for a plain context
  std::vector<mb_context*> subs;
};

struct mb_plan {
  mb_context* ctx = nullptr;
  bool big = false;      // large-N batched path (mb_large.cu)
  bool conv = false;     // conventional multi-slice method (mb_conventional.cu)
  long conv_ctas = 0;
  bool cluster = false;  // cluster-resident path (mb_cluster.cu)
  mbx::BigParams bp{};
  int stride = 0;
  int n = 0, ndiff = 0, npad = 0;
  long npairs = 0, nslots = 0;
  int S = 0, T = 0;
  bool use_k1 = false;
  std::vector<DevBuf> bufs;
  mbx::PotentialParams pot{};
  mbx::PropagateParams prop{};
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  std::vector<cudaStream_t> sides;  // batched path: streams of the other sub-batches
  std::vector<cudaEvent_t> joins;
  cudaEvent_t fork = nullptr;
  float ms_total = 0, ms_pot = 0, ms_prop = 0;
  int launches = 0;
  long h2d_bytes = 0;
  bool executed = false;
  std::vector<double2> host_coef;  // tabulated / zero fields: precomputed table
  // host copies kept for the parity hooks (mb_plan_node_heights / mb_plan_gamma)
  std::vector<double> zslot, g2, s0;
  std::vector<double2> gd, gi;
  std::vector<int> boxpos;
  int box_size = 0;
  // multi-device plan: one sub-plan per device that received pairs, the
  // global pair index of each of its pairs, and its first structure
  std::vector<mb_plan*> shards;
  std::vector<std::vector<long>> shard_rows;
  std::vector<int> shard_s0, shard_dev;
};

namespace {

template <class T>
T* dev_upload(mb_plan* pl, const T* src, std::size_t count) {
  DevBuf b;
  b.bytes = std::max<std::size_t>(count * sizeof(T), 16);
  cuda_check(cudaMallocAsync(&b.p, b.bytes, pl->ctx->stream), "cudaMallocAsync");
  pl->bufs.push_back(b);
  if (count && src) {
    cuda_check(cudaMemcpyAsync(b.p, src, count * sizeof(T), cudaMemcpyHostToDevice, pl->ctx->stream), "cudaMemcpyAsync H2D");
    pl->h2d_bytes += (long)(count * sizeof(T));
  }
  return static_cast<T*>(b.p);
}
template <class T>
T* dev_alloc(mb_plan* pl, std::size_t count) {
  return dev_upload<T>(pl, nullptr, count);
}

void free_plan(mb_plan* pl) {
  if (!pl) return;
  if (pl->ctx) {
    for (DevBuf& b : pl->bufs)
      if (b.p) cudaFreeAsync(b.p, pl->ctx->stream);
    cudaStreamSynchronize(pl->ctx->stream);
  }
  for (cudaEvent_t& e : pl->ev)
    if (e) cudaEventDestroy(e);
  if (pl->fork) cudaEventDestroy(pl->fork);
  for (cudaEvent_t e : pl->joins) cudaEventDestroy(e);
  for (cudaStream_t q : pl->sides) cudaStreamDestroy(q);
  delete pl;
}

// r_init (optional): caller-supplied R_init of solve_proposed (proposed.hpp:98-102),
// r_count matrices of n x n complex (row-major, interleaved re/im); 1 = shared
// by every pair, npairs = one per pair. It replaces the bulk seed.
mb_plan* create_plan(mb_context* ctx, const mb_rods* rods, const mb_field* fields, int nfields, double gamma,
                     const mb_pair* pairs, long npairs, const mb_stepper* stepper, const mb_options* opts,
                     const double* r_init = nullptr, long r_count = 0) {
  if (!ctx || !rods || !fields || !pairs || !stepper || !opts) fail(MB_ERR_ARG, "null argument");
  if (nfields < 1 || npairs < 1) fail(MB_ERR_ARG, "need at least one field and one pair");
  if (r_init && r_count != 1 && r_count != npairs)
    fail(MB_ERR_ARG, "R_init: count must be 1 (shared) or the number of pairs");
  if (!r_init && r_count != 0) fail(MB_ERR_ARG, "R_init: null array with a nonzero count");
  const int n = rods->n, ndiff = rods->ndiff;
  if (n < 1 || ndiff < 1 || !rods->k || !rods->m || !rods->diff || !rods->diff_m || !rods->diff_index)
    fail(MB_ERR_ARG, "rods: empty or missing arrays");
  validate_stepper(*stepper);
  if (!(gamma > 0.0) || !std::isfinite(gamma)) fail(MB_ERR_CONFIG, "beam: gamma must be positive and finite");
  const double zb = fields[0].z_bottom;
  for (int f = 0; f < nfields; ++f) {
    validate_field(fields[f]);
    if (fields[f].z_bottom != zb) fail(MB_ERR_CONFIG, "batch: every field must share z_bottom");
    if ((fields[f].has_bulk_period != 0) != (fields[0].has_bulk_period != 0) ||
        (fields[f].has_bulk_period && fields[f].bulk_period != fields[0].bulk_period))
      fail(MB_ERR_CONFIG, "batch: every field must share the bulk period");
    if (fields[f].kind != fields[0].kind) fail(MB_ERR_CONFIG, "batch: every field must be of one kind");
  }
  // resident kernel (state on chip) when it fits; 64 < n <= 256: one cluster
  // per pair (mb_cluster.cu) when its shared-memory footprint fits, else the
  // batched large-N path (state in HBM). Final choice after the box size below.
  if (n > 256) fail(MB_ERR_CONFIG, "device path supports at most 256 rods, got " + std::to_string(n));
  const bool conv = stepper->algorithm == MB_STEP_CONVENTIONAL;
  if (conv && n > 32) fail(MB_ERR_CONFIG, "conventional method on the device supports at most 32 rods");
  if (conv && fields[0].has_bulk_period)
    fail(MB_ERR_CONFIG, "conventional method on the device: bulk seeding is not supported");
  if (conv && r_init) fail(MB_ERR_CONFIG, "conventional method on the device: R_init is not supported");
  int npad = conv ? 0 : mbx::propagate_supported(n, stepper->algorithm == MB_STEP_RK4);
  if (conv && opts->path != 0) fail(MB_ERR_CONFIG, "conventional method: path must be 0");
  if (opts->path == 1 && !npad) fail(MB_ERR_CONFIG, "resident kernel does not cover this rod count / stepper");
  if (opts->path < 0 || opts->path > 4) fail(MB_ERR_ARG, "options: path must be 0..4");
  if (opts->path >= 2) npad = 0;
  if (conv) npad = 2 * n;
  bool big = npad == 0 && !conv;
  if (big) npad = (n + 7) & ~7;

  // slicing (slicing.hpp:17-34) and node heights (stages.cpp:25-30)
  long L;
  if (opts->slices > 0) {
    L = opts->slices;
  } else {
    if (!(opts->dz > 0.0) || !std::isfinite(opts->dz)) fail(MB_ERR_CONFIG, "sweep: dz must be positive and finite");
    L = std::max(1L, std::lround(-zb / opts->dz));
  }
  const double h = -zb / (double)L;
  const Schedule sc = make_schedule(*stepper);
  const int K = (int)sc.frac.size();
  const long stride = sc.endpoint_pair() ? K - 1 : K;
  const long nslots_main = sc.endpoint_pair() ? L * (K - 1) + 1 : L * K;
  // node heights of a window [z0, z1] in `count` steps (StepWindow::z, node_z)
  std::vector<double> zslot;
  auto add_window = [&](double z0, double z1, long count, double hw, double period) {
    const long ns = sc.endpoint_pair() ? count * (K - 1) + 1 : count * K;
    const std::size_t base = zslot.size();
    zslot.resize(base + (std::size_t)ns);
    auto wz = [&](long i) { return (z0 * (double)(count - i) + z1 * (double)i) / (double)count; };
    for (long i = 0; i < count; ++i)
      for (int m = 0; m < K; ++m) {
        const long slot = i * stride + m;
        if (slot >= ns) continue;
        const double f = sc.frac[m];
        const double z = f == 0.0 ? wz(i) : (f == 1.0 ? wz(i + 1) : wz(i) + f * hw);
        zslot[base + (std::size_t)slot] = period > 0.0 ? map_z(z, z1, period) : z;
      }
  };
  add_window(zb, 0.0, L, h, 0.0);
  // bulk window (proposed.cpp:311-321): one period below z_bottom, in
  // max(1, round(period / dz)) steps of StepWindow::over(zb - p, zb, .); the
  // potential there is the periodic continuation (map_z)
  // (a caller-supplied R_init replaces the bulk seed: solve_proposed takes
  // R_init as given, proposed.cpp:301)
  const bool bulk = fields[0].has_bulk_period != 0 && !r_init;
  long Lb = 0;
  double hb = 0.0;
  if (bulk) {
    if (!(opts->dz > 0.0) || !std::isfinite(opts->dz)) fail(MB_ERR_CONFIG, "sweep: dz must be positive and finite");
    const double per = fields[0].bulk_period;
    Lb = std::max(1L, std::lround(per / opts->dz));
    const double z0b = zb - per;
    hb = (zb - z0b) / (double)Lb;
    add_window(z0b, zb, Lb, hb, per);
  }
  const long nslots = (long)zslot.size();

  // pairs: AngleGrid semantics per pair, BeamGeometry + GammaMatrix::build
  // (geometry.cpp:19-57)
  std::vector<int> pstruct((std::size_t)npairs);
  std::vector<double> g2((std::size_t)npairs * n), s0((std::size_t)npairs);
  std::vector<double2> gd((std::size_t)npairs * n), gi((std::size_t)npairs * n);
  const double gg = gamma * gamma;
  for (long p = 0; p < npairs; ++p) {
    const mb_pair& pr = pairs[p];
    if (pr.structure < 0 || pr.structure >= nfields) fail(MB_ERR_ARG, "pair: structure index out of range");
    if (!(pr.theta0_deg > 0.0 && pr.theta0_deg < 90.0))
      fail(MB_ERR_CONFIG, "beam: theta0 must lie in (0, 90) degrees, got " + std::to_string(pr.theta0_deg));
    if (!std::isfinite(pr.theta1_deg)) fail(MB_ERR_CONFIG, "beam: theta1 must be finite");
    pstruct[(std::size_t)p] = pr.structure;
    const double c0 = std::cos(pr.theta0_deg * kDegToRad);
    const double t1 = pr.theta1_deg * kDegToRad;
    const double bx = gamma * c0 * std::cos(t1), by = gamma * c0 * std::sin(t1);
    s0[(std::size_t)p] = std::sin(pr.theta0_deg * kDegToRad);
    for (int i = 0; i < n; ++i) {
      const double px = bx + rods->k[2 * i], py = by + rods->k[2 * i + 1];
      const double d = gg - (px * px + py * py);
      if (std::abs(d) < 1e-12)
        fail(MB_ERR_CONFIG, "rod " + std::to_string(i) + " emerges at grazing: |gamma^2 - ||b0+k||^2| = " +
                                std::to_string(std::abs(d)));
      const std::size_t o = (std::size_t)p * n + i;
      g2[o] = d;
      const cd G = d > 0.0 ? cd(std::sqrt(d), 0.0) : cd(0.0, std::sqrt(-d));
      const cd Gi = 1.0 / G;
      gd[o] = make_double2(G.real(), G.imag());
      gi[o] = make_double2(Gi.real(), Gi.imag());
    }
  }

  // lattice box of rod differences: U(j,k) = box[center + off_j - off_k]
  int M1 = 0, M2 = 0;
  for (int d = 0; d < ndiff; ++d) {
    M1 = std::max(M1, std::abs(rods->diff_m[2 * d]));
    M2 = std::max(M2, std::abs(rods->diff_m[2 * d + 1]));
  }
  const int W2 = 2 * M2 + 1, W1 = 2 * M1 + 1;
  const int box_size = W1 * W2, center = M1 * W2 + M2;
  std::vector<int> boxpos((std::size_t)ndiff), rowoff((std::size_t)n);
  for (int d = 0; d < ndiff; ++d) boxpos[(std::size_t)d] = center + rods->diff_m[2 * d] * W2 + rods->diff_m[2 * d + 1];
  for (int j = 0; j < n; ++j) rowoff[(std::size_t)j] = rods->m[2 * j] * W2 + rods->m[2 * j + 1];
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      const int d = rods->diff_index[(std::size_t)j * n + k];
      if (d < 0 || d >= ndiff || boxpos[(std::size_t)d] != center + rowoff[(std::size_t)j] - rowoff[(std::size_t)k])
        fail(MB_ERR_ARG, "rods: diff_index inconsistent with m / diff_m");
    }

  // auto: the cluster kernel keeps the state on chip but spans CS SMs per pair
  // and serialises its Gauss-Jordan over the cluster; the batched path
  // amortises its per-pair solves over many pairs. Measured (B200, round 2,
  // tools/cmp_paths.py, 4096 pairs): splitting steppers are faster on the
  // cluster kernel at any batch size (N=127 sp6 25.8 vs 24.8 TF/s, N=255 sp6
  // 30.2 vs 28.0); rk4 keeps the batched path from 512 pairs (N=127: 20.8 vs
  // 18.5), where its four stage products per step amortise the per-pair solves.
  bool cluster = false;
  if (conv) big = false;
  // bulk seeding (per-pair period loop until R settles) runs inside the on-chip
  // kernels; the batched path steps the periods from the host (one sync per
  // period), so auto takes the cluster kernel at any batch size when it fits
  const bool want_cluster = opts->path == 3 || opts->path == 4;
  const int rk4 = stepper->algorithm == MB_STEP_RK4;
  if (big && (want_cluster || (opts->path == 0 && (npairs < 512 || bulk || !rk4)))) {
    const size_t need = mbx::cluster_smem_bytes(n, rk4, box_size, ndiff);
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
    cluster = need > 0 && (optin == 0 || need <= (size_t)optin);
    if (cluster) {
      big = false;
      npad = mbx::cluster_np(n);
    } else if (want_cluster) {
      fail(MB_ERR_CONFIG, "cluster kernel does not cover this rod count / stepper / box size");
    }
  }

  mb_plan* pl = new mb_plan();
  pl->ctx = ctx;
  try {
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    pl->n = n;
    pl->ndiff = ndiff;
    pl->npad = npad;
    pl->npairs = npairs;
    pl->nslots = nslots;
    pl->S = nfields;
    pl->zslot = zslot;
    pl->g2 = g2;
    pl->s0 = s0;
    pl->gd = gd;
    pl->gi = gi;
    pl->boxpos = boxpos;
    pl->box_size = box_size;
    cudaStream_t st = ctx->stream;

    // ---- coefficient table, boxed: slot = box_size double2 with difference d
    // at boxpos[d] and zero holes (zeroed once here; K1 only writes the
    // difference positions), so a node is one contiguous TMA bulk copy
    const int* boxpos_dev = dev_upload(pl, boxpos.data(), boxpos.size());
    const std::size_t coef_count = (std::size_t)nfields * nslots * box_size;
    double2* coef = dev_alloc<double2>(pl, coef_count);
    cuda_check(cudaMemsetAsync(coef, 0, coef_count * sizeof(double2), st), "zero the coefficient table");
    const int kind = fields[0].kind;
    if (kind == MB_FIELD_ATOMS || kind == MB_FIELD_GAUSSIAN_LAYERS) {
      int T = 0;
      for (int f = 0; f < nfields; ++f)
        T = std::max(T, kind == MB_FIELD_ATOMS ? 4 * fields[f].natoms : fields[f].nlayers);
      T = std::max(T, 1);
      std::vector<double> zc((std::size_t)nfields * T, 0.0), alpha((std::size_t)nfields * T, 0.0),
          latk((std::size_t)nfields * T, 0.0);
      std::vector<double2> cpre((std::size_t)nfields * T, make_double2(0.0, 0.0)),
          xy((std::size_t)nfields * T, make_double2(0.0, 0.0));
      for (int f = 0; f < nfields; ++f) {
        const mb_field& F = fields[f];
        if (kind == MB_FIELD_ATOMS) {
          // pre = (sign - i*absorption) gamma_L 4 pi / A
          const cd pre = cd(F.particle_sign, -F.absorption) * (F.gamma_L * 4.0 * kPi / F.cell_area);
          for (int a = 0; a < F.natoms; ++a)
            for (int i = 0; i < 4; ++i) {
              const std::size_t t = (std::size_t)f * T + 4 * a + i;
              const int sp = F.atom_species[a];
              const double bp = F.ff_b[4 * sp + i] + F.atom_B[a];
              const double w = F.ff_a[4 * sp + i] * 2.0 * std::sqrt(kPi) / std::sqrt(bp);
              const cd c = pre * w;
              cpre[t] = make_double2(c.real(), c.imag());
              latk[t] = bp / (16.0 * kPi * kPi);
              alpha[t] = 4.0 * kPi * kPi / bp;
              zc[t] = F.atom_xyz[3 * a + 2];
              xy[t] = make_double2(F.atom_xyz[3 * a], F.atom_xyz[3 * a + 1]);
            }
        } else {
          // GaussianLayer (potential.hpp:11-23): amplitude (1 + i absorption)
          // * exp(-|dk|^2 / 2 sxy^2) * exp(-(z - zc)^2 / 2 sz^2)
          for (int l = 0; l < F.nlayers; ++l) {
            const double* L5 = F.layers + 5 * l;
            const std::size_t t = (std::size_t)f * T + l;
            cpre[t] = make_double2(L5[1], L5[1] * L5[4]);
            latk[t] = 1.0 / (2.0 * L5[2] * L5[2]);
            alpha[t] = 1.0 / (2.0 * L5[3] * L5[3]);
            zc[t] = L5[0];
          }
        }
      }
      std::vector<double2> dg((std::size_t)ndiff);
      for (int d = 0; d < ndiff; ++d) dg[(std::size_t)d] = make_double2(rods->diff[2 * d], rods->diff[2 * d + 1]);
      pl->T = T;
      pl->use_k1 = true;
      mbx::PotentialParams& pp = pl->pot;
      pp.S = nfields;
      pp.T = T;
      pp.ndiff = ndiff;
      pp.nslots = nslots;
      pp.z_slot = dev_upload(pl, zslot.data(), zslot.size());
      pp.diff_g = dev_upload(pl, dg.data(), dg.size());
      pp.term_zc = dev_upload(pl, zc.data(), zc.size());
      pp.term_alpha = dev_upload(pl, alpha.data(), alpha.size());
      pp.term_latk = dev_upload(pl, latk.data(), latk.size());
      pp.term_cpre = dev_upload(pl, cpre.data(), cpre.size());
      pp.term_xy = dev_upload(pl, xy.data(), xy.size());
      pp.amp = dev_alloc<double2>(pl, (std::size_t)nfields * T * ndiff);
      pp.coef = coef;
      pp.boxpos = boxpos_dev;
      pp.box_size = box_size;
    } else {
      // zero or tabulated: node-slot table evaluated on the host once
      pl->host_coef.assign(coef_count, make_double2(0.0, 0.0));
      if (kind == MB_FIELD_TABULATED) {
        RodTables rt;
        for (int d = 0; d < ndiff; ++d) rt.diff_m.push_back({rods->diff_m[2 * d], rods->diff_m[2 * d + 1]});
        rt.diff.resize((std::size_t)ndiff);
        std::vector<cd> row((std::size_t)ndiff);
        for (int f = 0; f < nfields; ++f) {
          const Tabulated tb = bind_tabulated(fields[f], rt);
          for (long sl = 0; sl < nslots; ++sl) {
            eval_tabulated(tb, zb, zslot[(std::size_t)sl], row.data());
            for (int d = 0; d < ndiff; ++d)
              pl->host_coef[((std::size_t)f * nslots + sl) * box_size + boxpos[(std::size_t)d]] =
                  make_double2(row[d].real(), row[d].imag());
          }
        }
      }
      cuda_check(cudaMemcpyAsync(coef, pl->host_coef.data(), pl->host_coef.size() * sizeof(double2),
                                 cudaMemcpyHostToDevice, st),
                 "upload coefficient table");
      pl->h2d_bytes += (long)(pl->host_coef.size() * sizeof(double2));
    }

    // ---- propagation parameters
    mbx::PropagateParams& p = pl->prop;
    p.n = n;
    p.ndiff = ndiff;
    p.nsteps = (int)L;
    p.nslots = nslots;
    p.npairs = npairs;
    p.coef = coef;
    p.boxpos = dev_upload(pl, boxpos.data(), boxpos.size());
    p.rowoff = dev_upload(pl, rowoff.data(), rowoff.size());
    p.box_size = box_size;
    p.box_center = center;
    p.pair_struct = dev_upload(pl, pstruct.data(), pstruct.size());
    p.gamma2 = dev_upload(pl, g2.data(), g2.size());
    p.gdiag = dev_upload(pl, gd.data(), gd.size());
    p.ginv = dev_upload(pl, gi.data(), gi.size());
    p.sin_theta0 = dev_upload(pl, s0.data(), s0.size());
    p.rk4 = stepper->algorithm == MB_STEP_RK4;
    p.variant = stepper->variant;
    p.slot_stride = (int)stride;
    p.h = h;
    if (p.rk4) {
      p.nocc = 4;
      for (int r = 0; r < 4; ++r) p.occ_node[r] = sc.occ2node[(std::size_t)r];
    } else if (conv) {
      p.nocc = 1;
      p.occ_node[0] = 0;
    } else {
      p.nocc = stepper->nkick;
      for (int r = 0; r < stepper->nkick; ++r) {
        p.occ_node[r] = sc.occ2node[(std::size_t)r];
        p.occ_kick[r] = h * stepper->kick[r];
      }
      for (int r = 0; r < stepper->ndrift; ++r) p.occ_drift[r] = h * stepper->drift[r];
      p.final_drift = stepper->variant == MB_SPLIT_ABA ? h * stepper->drift[stepper->ndrift - 1] : 0.0;
      const bool can_fsal = stepper->variant == MB_SPLIT_BAB && sc.endpoint_pair() &&
                            sc.occ2node.front() == 0 && sc.occ2node.back() == K - 1;
      p.fsal = (opts->fsal && can_fsal) ? 1 : 0;
      p.fsal_kick = h * (stepper->kick[stepper->nkick - 1] + stepper->kick[0]);
    }
    p.threshold = opts->rhst_threshold;
    p.residual_check = opts->residual_check ? 1 : 0;
    p.bulk_steps = 0;
    if (bulk) {  // the same stepper on the bulk window's step hb (BulkOptions defaults)
      p.bulk_steps = (int)Lb;
      p.bulk_base = nslots_main;
      p.bulk_h = hb;
      for (int r = 0; r < mbx::kMaxOcc; ++r) p.bulk_kick[r] = p.bulk_drift[r] = 0.0;
      if (!p.rk4) {
        for (int r = 0; r < stepper->nkick; ++r) p.bulk_kick[r] = hb * stepper->kick[r];
        for (int r = 0; r < stepper->ndrift; ++r) p.bulk_drift[r] = hb * stepper->drift[r];
        p.bulk_final_drift = stepper->variant == MB_SPLIT_ABA ? hb * stepper->drift[stepper->ndrift - 1] : 0.0;
        p.bulk_fsal_kick = hb * (stepper->kick[stepper->nkick - 1] + stepper->kick[0]);
      }
      p.bulk_max_periods = 10000;
      p.bulk_tol = 1e-12;
      p.bulk_scratch = dev_alloc<double>(pl, (std::size_t)npairs * 2 * npad * npad);
    }
    p.r_seed = 0;
    if (r_init) {  // zero-padded re / im planes per pair (ld npad), read by every design
      const std::size_t NN = (std::size_t)npad * npad;
      std::vector<double> planes((std::size_t)npairs * 2 * NN, 0.0);
      for (long q = 0; q < npairs; ++q) {
        const double* src = r_init + (r_count == 1 ? 0 : (std::size_t)q * 2 * n * n);
        double* re = planes.data() + (std::size_t)q * 2 * NN;
        double* im = re + NN;
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) {
            re[(std::size_t)i * npad + j] = src[2 * ((std::size_t)i * n + j)];
            im[(std::size_t)i * npad + j] = src[2 * ((std::size_t)i * n + j) + 1];
          }
      }
      p.bulk_scratch = dev_upload(pl, planes.data(), planes.size());
      p.r_seed = 1;
    }
    p.eta = dev_alloc<double>(pl, (std::size_t)npairs * n);
    p.rho = dev_alloc<double2>(pl, (std::size_t)npairs * n);
    p.status = dev_alloc<mbx::PointStatus>(pl, (std::size_t)npairs);
    p.prof = dev_alloc<unsigned long long>(pl, mbx::kProfSlots);
    pl->big = big;
    pl->cluster = cluster;
    pl->conv = conv;
    if (conv) {
      pl->conv_ctas = mbx::conventional_ctas(npairs);
      p.scratch = dev_alloc<double>(pl, mbx::conventional_scratch_doubles(pl->conv_ctas));
    }
    pl->stride = (int)stride;
    // cluster kernel: A, B, panel rows (+ the saved Q slab of a bulk period)
    if (cluster) {
      p.scratch = dev_alloc<double>(pl, (std::size_t)npairs * ((bulk || r_init) ? 8 : 6) * npad * npad);
      // cluster or cooperative groups: path 3 / 4 force one; auto takes the
      // variant that finishes the batch in fewer rounds of co-resident groups
      p.coop = opts->path == 4 ? 1 : (opts->path == 3 ? 0 : mbx::cluster_prefer_coop(p));
      if (p.coop) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
        const std::size_t maxc = (std::size_t)sms * mbx::kCoopMaxCtasPerSm;
        p.coop_bar = dev_alloc<unsigned>(pl, maxc);
        p.coop_pub = dev_alloc<double>(pl, maxc * mbx::kCoopPubDoubles);
      }
    }
    if (big) {
      mbx::BigParams& b = pl->bp;
      b.n = n;
      b.np = npad;
      b.ndiff = ndiff;
      b.npairs = npairs;
      b.nsteps = (int)L;
      b.nslots = nslots;
      b.slot_stride = (int)stride;
      b.coef = coef;
      b.boxpos = p.boxpos;
      b.rowoff = p.rowoff;
      b.box_size = box_size;
      b.box_center = center;
      b.pair_struct = p.pair_struct;
      b.gamma2 = p.gamma2;
      b.gdiag = p.gdiag;
      b.ginv = p.ginv;
      b.sin_theta0 = p.sin_theta0;
      b.r_init = r_init ? p.bulk_scratch : nullptr;
      b.bulk_r = bulk ? p.bulk_scratch : nullptr;
      b.bulk_tol = p.bulk_tol;
      b.bulk_left = bulk ? dev_alloc<unsigned>(pl, kBigParts) : nullptr;
      // splitting: Q0, Q1 (ping-pong), P, scratch; rk4: Q, P, X2, X3, W, V, SQ
      b.nmat = p.rk4 ? 7 : 4;
      b.pair_stride = (long)b.nmat * 2 * npad * npad;
      b.state = dev_alloc<double>(pl, (std::size_t)npairs * b.pair_stride);
      b.status = p.status;
      b.xi = dev_alloc<double>(pl, (std::size_t)npairs);
      b.chk = dev_alloc<double>(pl, (std::size_t)npairs * ((npad + 15) / 16) * 4);
      b.chk_count = dev_alloc<unsigned>(pl, (std::size_t)npairs);
      cuda_check(cudaMemsetAsync(b.chk_count, 0, (std::size_t)npairs * sizeof(unsigned), pl->ctx->stream),
                 "cudaMemsetAsync");
      b.threshold = p.threshold;
      b.residual_check = p.residual_check;
      b.eta = p.eta;
      b.rho = p.rho;
    }
    for (cudaEvent_t& e : pl->ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
  } catch (...) {
    free_plan(pl);
    throw;
  }
  return pl;
}

// Large-N orchestration: one launch per kick / RK stage over all pairs, then
// the per-pair check and RHST kernels each step; the surface solve at the end.
// The batched path as two half-batches on two streams. Per step a
// half-batch runs its stage products, the row-block check and the per-pair
// Gauss-Jordan; the solve launch keeps few CTAs busy (only the pairs that
// RHST at this step), so the other half's stage products fill the SMs
// meanwhile. Launches are issued step by step, alternating halves, so neither
// stream's queue runs ahead of the other. Pairs are independent: the halves
// give bitwise the rows of one batch.
mbx::BigParams big_part(const mbx::BigParams& b, long lo, long hi, int index) {
  mbx::BigParams h = b;
  const long rplanes = 2L * b.np * b.np;
  if (b.r_init) h.r_init = b.r_init + lo * rplanes;
  if (b.bulk_r) h.bulk_r = b.bulk_r + lo * rplanes;
  if (b.bulk_left) h.bulk_left = b.bulk_left + index;
  const long chk_per = (long)((b.np + 15) / 16) * 4;
  h.npairs = hi - lo;
  h.pair_struct = b.pair_struct + lo;
  h.gamma2 = b.gamma2 + lo * b.n;
  h.gdiag = b.gdiag + lo * b.n;
  h.ginv = b.ginv + lo * b.n;
  h.sin_theta0 = b.sin_theta0 + lo;
  h.state = b.state + lo * b.pair_stride;
  h.status = b.status + lo;
  h.xi = b.xi + lo;
  h.chk = b.chk + lo * chk_per;
  h.chk_count = b.chk_count + lo;
  h.eta = b.eta + lo * b.n;
  h.rho = b.rho + lo * b.n;
  return h;
}

void execute_big(mb_plan* pl, cudaStream_t st) {
  const mbx::PropagateParams& p = pl->prop;
  int* nl = &pl->launches;
  // sub-batches on their own streams: two from 1024 pairs, MB_BIG_PARTS (2..4,
  // default 2) from 2048 (each part still fills the GPU with tiles)
  int want = 1;
  if (pl->bp.npairs >= 1024) want = 2;
  if (pl->bp.npairs >= 2048) {
    const char* e = std::getenv("MB_BIG_PARTS");
    if (e) want = std::max(1, std::min(kBigParts, std::atoi(e)));
  }
  const bool two = want > 1;
  std::vector<mbx::BigParams> part;
  std::vector<cudaStream_t> sts;
  if (two) {
    if (!pl->fork) cuda_check(cudaEventCreateWithFlags(&pl->fork, cudaEventDisableTiming), "cudaEventCreate");
    while ((int)pl->sides.size() < want - 1) {
      cudaStream_t q;
      cudaEvent_t e;
      cuda_check(cudaStreamCreateWithFlags(&q, cudaStreamNonBlocking), "cudaStreamCreate");
      pl->sides.push_back(q);
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
      pl->joins.push_back(e);
    }
    cuda_check(cudaEventRecord(pl->fork, st), "event");
    for (int h = 0; h < want; ++h) {
      const long lo = pl->bp.npairs * h / want, hi = pl->bp.npairs * (h + 1) / want;
      part.push_back(big_part(pl->bp, lo, hi, h));
      sts.push_back(h == 0 ? st : pl->sides[(std::size_t)h - 1]);
      if (h > 0) cuda_check(cudaStreamWaitEvent(sts.back(), pl->fork, 0), "stream wait");
    }
  } else {
    part = {pl->bp};
    sts = {st};
  }
  const int H = (int)part.size();
  auto launch = [&](const mbx::BigStage& s) {
    for (int h = 0; h < H; ++h) cuda_check(mbx::big_launch_stage(part[h], s, sts[h], nl), "big stage launch");
  };
  auto check_and_solve = [&](int step, int mq, int mp, int msa, int msb, int mx2, double hh) {
    for (int h = 0; h < H; ++h) {
      cuda_check(mbx::big_launch_check(part[h], step, mq, mp, sts[h], nl), "big check launch");
      cuda_check(mbx::big_launch_gj(part[h], 0, step, mq, mp, msa, msb, mx2, hh, sts[h], nl), "big RHST launch");
    }
  };
  auto surface = [&](int mq, int mp, int msa, int msb) {
    for (int h = 0; h < H; ++h)
      cuda_check(mbx::big_launch_gj(part[h], 1, p.nsteps, mq, mp, msa, msb, -1, 0.0, sts[h], nl),
                 "big surface-solve launch");
    for (int h = 1; h < H; ++h) {
      cuda_check(cudaEventRecord(pl->joins[(std::size_t)h - 1], sts[h]), "event");
      cuda_check(cudaStreamWaitEvent(st, pl->joins[(std::size_t)h - 1], 0), "stream wait");
    }
  };
  // One window of L steps (run_window, proposed.cpp:275-289) whose node slots
  // start at `base`: the slab, or one bulk period on the bulk window's step
  // (proposed.cpp:311-321). Failures report step_off + step.
  mbx::BigStage s{};
  const int Q = 0, P4 = 1, X2 = 2, X3 = 3, W = 4, V = 5, SQ = 6;  // rk4 matrices
  const int P = 2, SCR = 3;                                       // splitting: Q0, Q1, P, scratch
  int qc = 0;
  const int nk = p.nocc;
  auto init = [&](int kind, double hw) {
    s = p.rk4 ? mbx::BigStage{kind, 0, 0, 0, hw, 0.0, 0.0, Q, -1, P4, X2, X3, W, V, SQ}
              : mbx::BigStage{kind, 0, 0, 0, hw, 0.0, 0.0, qc, -1, P, -1, -1, -1, -1, -1};
    launch(s);  // initial state (rk4: + X2)
  };
  // FSAL is not merged on the batched path: a merged kick must keep the
  // reference's two roundings around the end-of-step check (see the on-chip
  // kernels), and here the shared product would be an extra N x N plane per
  // pair in HBM. Unmerged kicks give exactly the fsal = 0 results.
  auto drift = [&](double c) {
    mbx::BigStage d{2, 0, 0, 0, 0.0, c, 0.0, qc, qc ^ 1, P, -1, -1, -1, -1, -1};
    launch(d);
    qc ^= 1;
  };
  auto window = [&](long base, int Lw, double hw, const double* kick, const double* drf, double fin, int step_off) {
    auto slot = [&](int step, int r) { return base + (long)step * pl->stride + p.occ_node[r]; };
    for (int step = 0; step < Lw; ++step) {
      if (p.rk4) {
        const int ops[4] = {Q, X2, X3, V};
        for (int k = 0; k < 4; ++k) {
          s = mbx::BigStage{3 + k, ops[k], slot(step, k), step_off + step, hw, 0.0, 0.0, Q, -1, P4, X2, X3, W, V, SQ};
          launch(s);
        }
        check_and_solve(step_off + step, Q, P4, X3, V, X2, hw);
        continue;
      }
      for (int r = 0; r < nk; ++r) {
        const bool last = r == nk - 1;
        if (p.variant == 0) drift(drf[r]);
        const double kc = kick[r];
        const double dc = (p.variant == 1 && !last) ? drf[r] : 0.0;
        mbx::BigStage k{1, qc, slot(step, r), step_off + step, kc, dc, 0.0, qc, qc ^ 1, P, -1, -1, -1, -1, -1};
        launch(k);
        if (dc != 0.0) qc ^= 1;
      }
      if (p.variant == 0) drift(fin);
      check_and_solve(step_off + step, qc, P, qc ^ 1, SCR, -1, 0.0);
    }
  };
  if (p.bulk_steps > 0) {
    // bulk seeding (compute_bulk_reflection_proposed, proposed.cpp:311-342):
    // one bulk period after another from R = 0; after each period the full R
    // is read (the surface solve's machinery) and compared with the previous
    // one per pair; a settled pair is frozen until the slab is seeded. One
    // host sync per period (the count of pairs still unsettled).
    init(0, p.bulk_h);
    for (long m = 0; m < p.bulk_max_periods; ++m) {
      window(p.bulk_base, p.bulk_steps, p.bulk_h, p.bulk_kick, p.bulk_drift, p.bulk_final_drift,
             (int)(m * p.bulk_steps));
      const int mode = m + 1 == p.bulk_max_periods ? 3 : 2;
      unsigned left[kBigParts] = {0, 0, 0, 0};
      for (int h = 0; h < H; ++h) {
        cuda_check(cudaMemsetAsync(part[h].bulk_left, 0, sizeof(unsigned), sts[h]), "memset");
        cuda_check(p.rk4 ? mbx::big_launch_gj(part[h], mode, (int)m, Q, P4, X3, V, -1, 0.0, sts[h], nl)
                         : mbx::big_launch_gj(part[h], mode, (int)m, qc, P, qc ^ 1, SCR, -1, 0.0, sts[h], nl),
                   "big bulk-read launch");
        cuda_check(cudaMemcpyAsync(&left[h], part[h].bulk_left, sizeof(unsigned), cudaMemcpyDeviceToHost, sts[h]),
                   "D2H bulk count");
      }
      for (int h = 0; h < H; ++h) cuda_check(cudaStreamSynchronize(sts[h]), "bulk period sync");
      if (left[0] + left[1] + left[2] + left[3] == 0) break;
    }
    init(7, p.h);  // Q = G^-1 (I + R)/2, P = (i/2)(I - R) from the settled R
  } else {
    init(0, p.h);
  }
  window(0, p.nsteps, p.h, p.occ_kick, p.occ_drift, p.final_drift, 0);
  if (p.rk4)
    surface(Q, P4, X3, V);
  else
    surface(qc, P, qc ^ 1, SCR);
}

void execute_plan(mb_plan* pl, cudaStream_t st) {
  cuda_check(cudaSetDevice(pl->ctx->device), "cudaSetDevice");
  if (!st) st = pl->ctx->stream;
  pl->launches = 0;
  cuda_check(cudaEventRecord(pl->ev[0], st), "event");
  if (pl->use_k1) cuda_check(mbx::launch_potential(pl->pot, st, &pl->launches), "potential kernel launch");
  cuda_check(cudaEventRecord(pl->ev[1], st), "event");
  cuda_check(cudaMemsetAsync(pl->prop.prof, 0, mbx::kProfSlots * sizeof(unsigned long long), st), "memset");
  int npad = 0;
  if (pl->conv)
    cuda_check(mbx::launch_conventional(pl->prop, pl->conv_ctas, st, &pl->launches), "conventional kernel launch");
  else if (pl->big)
    execute_big(pl, st);
  else if (pl->cluster)
    cuda_check(mbx::launch_cluster(pl->prop, st, &pl->launches), "cluster propagation kernel launch");
  else
    cuda_check(mbx::launch_propagate(pl->prop, st, &pl->launches, &npad), "propagation kernel launch");
  cuda_check(cudaEventRecord(pl->ev[2], st), "event");
  cuda_check(cudaEventSynchronize(pl->ev[2]), "propagation kernel");
  cuda_check(cudaGetLastError(), "kernel execution");
  cudaEventElapsedTime(&pl->ms_pot, pl->ev[0], pl->ev[1]);
  cudaEventElapsedTime(&pl->ms_prop, pl->ev[1], pl->ev[2]);
  cudaEventElapsedTime(&pl->ms_total, pl->ev[0], pl->ev[2]);
  pl->executed = true;
}

// the first failing pair in row order decides (sweep.cpp:136-137)
void raise_first_failure(const std::vector<mbx::PointStatus>& stv) {
  for (std::size_t i = 0; i < stv.size(); ++i) {
    if (stv[i].code == MB_POINT_OK) continue;
    const std::string where = " (pair " + std::to_string(i) + ", step " + std::to_string(stv[i].step) + ")";
    if (stv[i].code == MB_POINT_NONFINITE) fail(MB_ERR_BREAKDOWN, "propagation state went nonfinite" + where);
    if (stv[i].code == MB_POINT_RHST)
      fail(MB_ERR_BREAKDOWN, "stabilizing transform: solve_right: singular or ill-conditioned system" + where);
    if (stv[i].code == MB_POINT_BULK_READ)
      fail(MB_ERR_BREAKDOWN, "bulk reflection read: solve_right: singular or ill-conditioned system (pair " +
                                 std::to_string(i) + ", period " + std::to_string(stv[i].step) + ")");
    if (stv[i].code == MB_POINT_RECURSION)
      fail(MB_ERR_BREAKDOWN, "conventional recursion: singular, ill-conditioned or nonfinite reflection" + where);
    if (stv[i].code == MB_POINT_BULK_CONVERGENCE)
      fail(MB_ERR_CONVERGENCE, "bulk reflection did not settle within 10000 periods (pair " + std::to_string(i) + ")");
    fail(MB_ERR_BREAKDOWN, "reflection extraction: solve_right: singular or ill-conditioned system" + where);
  }
}

// D2H of one single-device plan's outputs (any pointer may be null)
void fetch_results(mb_plan* pl, double* eta, double2* rho, std::vector<mbx::PointStatus>& stv) {
  if (!pl->executed) fail(MB_ERR_ARG, "plan has not been executed");
  cuda_check(cudaSetDevice(pl->ctx->device), "cudaSetDevice");
  cudaStream_t st = pl->ctx->stream;
  const std::size_t ne = (std::size_t)pl->npairs * pl->n;
  stv.assign((std::size_t)pl->npairs, mbx::PointStatus{});
  if (eta) cuda_check(cudaMemcpyAsync(eta, pl->prop.eta, ne * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H eta");
  if (rho) cuda_check(cudaMemcpyAsync(rho, pl->prop.rho, ne * sizeof(double2), cudaMemcpyDeviceToHost, st), "D2H rho");
  cuda_check(cudaMemcpyAsync(stv.data(), pl->prop.status, stv.size() * sizeof(mbx::PointStatus),
                             cudaMemcpyDeviceToHost, st),
             "D2H status");
  cuda_check(cudaStreamSynchronize(st), "D2H");
}

int collect_results(mb_plan* pl, double* eta, double* rho, mb_point_status* status) {
  std::vector<mbx::PointStatus> stv;
  if (pl->shards.empty()) {
    fetch_results(pl, eta, reinterpret_cast<double2*>(rho), stv);
  } else {
    // gather every shard's rows into the caller's preassigned rows (sweep.cpp:92-108)
    stv.assign((std::size_t)pl->npairs, mbx::PointStatus{});
    const int n = pl->n;
    for (std::size_t s = 0; s < pl->shards.size(); ++s) {
      mb_plan* sp = pl->shards[s];
      const std::vector<long>& rows = pl->shard_rows[s];
      std::vector<double> e(eta ? rows.size() * n : 0);
      std::vector<double2> r(rho ? rows.size() * n : 0);
      std::vector<mbx::PointStatus> ss;
      fetch_results(sp, eta ? e.data() : nullptr, rho ? r.data() : nullptr, ss);
      for (std::size_t i = 0; i < rows.size(); ++i) {
        const long g = rows[i];
        if (eta) std::memcpy(eta + (std::size_t)g * n, e.data() + i * n, n * sizeof(double));
        if (rho) std::memcpy(rho + (std::size_t)g * n * 2, r.data() + i * n, n * sizeof(double2));
        stv[(std::size_t)g] = ss[i];
      }
    }
  }
  if (status)
    for (std::size_t i = 0; i < stv.size(); ++i)
      status[i] = mb_point_status{stv[i].code, stv[i].step, stv[i].rhst, stv[i].reserved};
  raise_first_failure(stv);
  return MB_OK;
}

// ------------------------------------------------------------ multi-device
// pairs are independent and U depends only on the structure.
// Several fields: contiguous structure blocks, balanced by pair count (a
// structure's coefficient table is built on one device only). One field:
// pairs round-robin. Fixed map, so the gathered rows do not depend on timing.
mb_plan* create_multi_plan(mb_context* ctx, const mb_rods* rods, const mb_field* fields, int nfields, double gamma,
                           const mb_pair* pairs, long npairs, const mb_stepper* stepper, const mb_options* opts,
                           const double* r_init, long r_count) {
  if (!pairs || !fields) fail(MB_ERR_ARG, "null argument");
  if (nfields < 1 || npairs < 1) fail(MB_ERR_ARG, "need at least one field and one pair");
  const int G = (int)ctx->subs.size();
  std::vector<int> owner((std::size_t)npairs, 0);
  std::vector<int> s_lo(G, 0), s_hi(G, 0);
  if (nfields > 1) {
    std::vector<long> cnt((std::size_t)nfields, 0);
    for (long p = 0; p < npairs; ++p) {
      const int s = pairs[p].structure;
      if (s < 0 || s >= nfields) fail(MB_ERR_ARG, "pair: structure index out of range");
      ++cnt[(std::size_t)s];
    }
    // device g takes structures whose cumulative pair count midpoint falls in [g, g+1) / G of the total
    long acc = 0;
    std::vector<int> dev_of((std::size_t)nfields, 0);
    for (int s = 0; s < nfields; ++s) {
      const double mid = (double)acc + 0.5 * (double)cnt[(std::size_t)s];
      dev_of[(std::size_t)s] = std::min(G - 1, (int)(mid * G / (double)npairs));
      acc += cnt[(std::size_t)s];
    }
    for (int g = 0; g < G; ++g) {
      s_lo[g] = nfields;
      s_hi[g] = 0;
    }
    for (int s = 0; s < nfields; ++s) {
      const int g = dev_of[(std::size_t)s];
      s_lo[g] = std::min(s_lo[g], s);
      s_hi[g] = std::max(s_hi[g], s + 1);
    }
    for (long p = 0; p < npairs; ++p) owner[(std::size_t)p] = dev_of[(std::size_t)pairs[p].structure];
  } else {
    for (long p = 0; p < npairs; ++p) owner[(std::size_t)p] = (int)(p % G);
    for (int g = 0; g < G; ++g) s_lo[g] = 0, s_hi[g] = 1;
  }
  auto* pl = new mb_plan();
  pl->ctx = ctx;
  pl->n = rods ? rods->n : 0;
  pl->npairs = npairs;
  pl->S = nfields;
  try {
    for (int g = 0; g < G; ++g) {
      std::vector<mb_pair> mine;
      std::vector<long> rows;
      for (long p = 0; p < npairs; ++p)
        if (owner[(std::size_t)p] == g) {
          mb_pair q = pairs[p];
          q.structure -= s_lo[g];
          mine.push_back(q);
          rows.push_back(p);
        }
      if (mine.empty()) continue;
      // per-pair R_init follows its pair to the owning device
      std::vector<double> seed;
      const double* r_mine = r_init;
      long r_mine_count = r_count;
      if (r_init && r_count != 1) {
        if (r_count != npairs || !rods) fail(MB_ERR_ARG, "R_init: count must be 1 (shared) or the number of pairs");
        const std::size_t per = (std::size_t)2 * rods->n * rods->n;
        seed.resize(rows.size() * per);
        for (std::size_t q = 0; q < rows.size(); ++q)
          std::memcpy(seed.data() + q * per, r_init + (std::size_t)rows[q] * per, per * sizeof(double));
        r_mine = seed.data();
        r_mine_count = (long)rows.size();
      }
      mb_plan* sp = create_plan(ctx->subs[(std::size_t)g], rods, fields + s_lo[g], s_hi[g] - s_lo[g], gamma,
                                mine.data(), (long)mine.size(), stepper, opts, r_mine, r_mine_count);
      // (the pageable upload is staged before create_plan returns)
      pl->shards.push_back(sp);
      pl->shard_rows.push_back(std::move(rows));
      pl->shard_s0.push_back(s_lo[g]);
      pl->shard_dev.push_back(g);
    }
    for (mb_plan* sp : pl->shards) cuda_check(cudaStreamSynchronize(sp->ctx->stream), "plan upload");
    const mb_plan* f = pl->shards.front();
    pl->ndiff = f->ndiff;
    pl->npad = f->npad;
    pl->nslots = f->nslots;
    for (mb_plan* sp : pl->shards) pl->h2d_bytes += sp->h2d_bytes;
  } catch (...) {
    for (mb_plan* sp : pl->shards) free_plan(sp);
    delete pl;
    throw;
  }
  return pl;
}

// one host thread per device; the first failure (shard order) is rethrown
void execute_multi(mb_plan* pl) {
  const std::size_t G = pl->shards.size();
  std::vector<std::exception_ptr> err(G);
  std::vector<std::thread> th;
  for (std::size_t s = 0; s < G; ++s)
    th.emplace_back([&, s] {
      try {
        execute_plan(pl->shards[s], nullptr);
      } catch (...) {
        err[s] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
  pl->ms_total = pl->ms_pot = pl->ms_prop = 0.0f;
  pl->launches = 0;
  for (mb_plan* sp : pl->shards) {
    pl->ms_total = std::max(pl->ms_total, sp->ms_total);
    pl->ms_pot = std::max(pl->ms_pot, sp->ms_pot);
    pl->ms_prop = std::max(pl->ms_prop, sp->ms_prop);
    pl->launches += sp->launches;
  }
  pl->executed = true;
}

void destroy_any(mb_plan* pl) {
  if (!pl) return;
  if (!pl->shards.empty()) {
    for (mb_plan* sp : pl->shards) free_plan(sp);
    delete pl;
    return;
  }
  free_plan(pl);
}

mb_plan* create_any(mb_context* ctx, const mb_rods* rods, const mb_field* fields, int nfields, double gamma,
                    const mb_pair* pairs, long npairs, const mb_stepper* stepper, const mb_options* opts,
                    const double* r_init = nullptr, long r_count = 0) {
  if (!ctx) fail(MB_ERR_ARG, "null context");
  if (!ctx->subs.empty())
    return create_multi_plan(ctx, rods, fields, nfields, gamma, pairs, npairs, stepper, opts, r_init, r_count);
  mb_plan* pl = create_plan(ctx, rods, fields, nfields, gamma, pairs, npairs, stepper, opts, r_init, r_count);
  cuda_check(cudaStreamSynchronize(ctx->stream), "plan upload");
  return pl;
}

void execute_any(mb_plan* pl, cudaStream_t st) {
  if (!pl->shards.empty())
    execute_multi(pl);
  else
    execute_plan(pl, st);
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

const char* mb_last_error(void) { return g_last_error.c_str(); }

int mb_device_ok(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) return 0;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return 0;
  return prop.major == 10 && prop.minor == 0;
}

int mb_rods_build(const mb_lattice* lattice, double cutoff, int first_n, int* n, int* ndiff, double* k, int* m,
                  double* diff, int* diff_m, int* diff_index, int cap_n, int cap_diff) {
  return guarded([&] {
    if (!lattice || !n || !ndiff) fail(MB_ERR_ARG, "null argument");
    const Lattice lat{V2{lattice->a1[0], lattice->a1[1]}, V2{lattice->a2[0], lattice->a2[1]}};
    const RodTables t = build_rods(lat, cutoff, first_n);
    const int nn = (int)t.rods.size(), nd = (int)t.diff.size();
    *n = nn;
    *ndiff = nd;
    if (!k && !m && !diff && !diff_m && !diff_index) return;
    if (cap_n < nn || cap_diff < nd) fail(MB_ERR_ARG, "mb_rods_build: capacity too small");
    for (int i = 0; i < nn; ++i) {
      if (k) {
        k[2 * i] = t.rods[i].k.x;
        k[2 * i + 1] = t.rods[i].k.y;
      }
      if (m) {
        m[2 * i] = t.rods[i].m1;
        m[2 * i + 1] = t.rods[i].m2;
      }
    }
    for (int d = 0; d < nd; ++d) {
      if (diff) {
        diff[2 * d] = t.diff[d].x;
        diff[2 * d + 1] = t.diff[d].y;
      }
      if (diff_m) {
        diff_m[2 * d] = t.diff_m[d].first;
        diff_m[2 * d + 1] = t.diff_m[d].second;
      }
    }
    if (diff_index) std::memcpy(diff_index, t.diff_index.data(), t.diff_index.size() * sizeof(int));
  });
}

int mb_beam_from_energy(double e, double* gamma, double* gamma_L) {
  return guarded([&] {
    if (!gamma || !gamma_L) fail(MB_ERR_ARG, "null argument");
    if (!(e > 0.0) || !std::isfinite(e)) fail(MB_ERR_CONFIG, "beam: energy must be positive");
    const double mc2 = 510998.95, hc = 12398.419843320026;
    const double lambda = hc / std::sqrt(e * (e + 2.0 * mc2));
    *gamma = kTwoPi / lambda;
    *gamma_L = 1.0 + e / mc2;
  });
}

int mb_stepper_by_name(const char* name, mb_stepper* out) {
  return guarded([&] {
    if (!name || !out) fail(MB_ERR_ARG, "null argument");
    const std::string s(name);
    const Tables& t = tables();
    if (s == "rk4") {
      *out = mb_stepper{MB_STEP_RK4, MB_SPLIT_BAB, 0, nullptr, 0, nullptr};
    } else if (s == "sp4") {
      *out = mb_stepper{MB_STEP_SPLITTING, MB_SPLIT_BAB, 6, t.sp4_drift, 7, t.sp4_kick};
    } else if (s == "sp6") {
      *out = mb_stepper{MB_STEP_SPLITTING, MB_SPLIT_BAB, 11, t.sp6_drift, 12, t.sp6_kick};
    } else if (s == "conventional") {
      *out = mb_stepper{MB_STEP_CONVENTIONAL, MB_SPLIT_BAB, 0, nullptr, 0, nullptr};
    } else {
      fail(MB_ERR_CONFIG, "unknown stepper '" + s + "' (expected rk4, sp4 or sp6)");
    }
  });
}

int mb_context_create(int device, mb_context** out) {
  return guarded([&] {
    if (!out) fail(MB_ERR_ARG, "null argument");
    *out = nullptr;
    int count = 0;
    cuda_check(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count) fail(MB_ERR_CUDA, "no such CUDA device");
    if (!mb_device_ok(device)) fail(MB_ERR_CUDA, "device is not an sm_100 (B200) GPU; no CPU fallback exists");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    auto* ctx = new mb_context();
    ctx->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete ctx;
      cuda_check(e, "cudaStreamCreate");
    }
    // keep freed plan memory in the pool for the next call
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = ctx;
  });
}

int mb_context_create_multi(const int* devices, int ndevices, mb_context** out) {
  return guarded([&] {
    if (!out || !devices || ndevices < 1) fail(MB_ERR_ARG, "mb_context_create_multi: need a device list");
    *out = nullptr;
    auto* ctx = new mb_context();
    try {
      for (int i = 0; i < ndevices; ++i) {
        mb_context* sub = nullptr;
        const int rc = mb_context_create(devices[i], &sub);
        if (rc != MB_OK) fail(rc, g_last_error);
        ctx->subs.push_back(sub);
      }
    } catch (...) {
      for (mb_context* sub : ctx->subs) mb_context_destroy(sub);
      delete ctx;
      throw;
    }
    ctx->device = ctx->subs.front()->device;
    ctx->stream = ctx->subs.front()->stream;
    *out = ctx;
  });
}

int mb_context_device_count(const mb_context* ctx) {
  if (!ctx) return 0;
  return ctx->subs.empty() ? 1 : (int)ctx->subs.size();
}

int mb_context_destroy(mb_context* ctx) {
  return guarded([&] {
    if (!ctx) return;
    if (!ctx->subs.empty()) {
      for (mb_context* sub : ctx->subs) mb_context_destroy(sub);
      delete ctx;
      return;
    }
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int mb_plan_create(mb_context* ctx, const mb_rods* rods, const mb_field* fields, int nfields, double gamma,
                   const mb_pair* pairs, long npairs, const mb_stepper* stepper, const mb_options* opts,
                   mb_plan** out) {
  return guarded([&] {
    if (!out || !ctx) fail(MB_ERR_ARG, "null argument");
    *out = nullptr;
    std::lock_guard<std::mutex> lk(ctx->mu);
    *out = create_any(ctx, rods, fields, nfields, gamma, pairs, npairs, stepper, opts);
  });
}

int mb_plan_create_seeded(mb_context* ctx, const mb_rods* rods, const mb_field* fields, int nfields, double gamma,
                          const mb_pair* pairs, long npairs, const mb_stepper* stepper, const mb_options* opts,
                          const double* r_init, long r_init_count, mb_plan** out) {
  return guarded([&] {
    if (!out || !ctx) fail(MB_ERR_ARG, "null argument");
    *out = nullptr;
    std::lock_guard<std::mutex> lk(ctx->mu);
    *out = create_any(ctx, rods, fields, nfields, gamma, pairs, npairs, stepper, opts, r_init, r_init_count);
  });
}

int mb_plan_execute(mb_plan* plan, void* stream) {
  return guarded([&] {
    if (!plan) fail(MB_ERR_ARG, "null plan");
    std::lock_guard<std::mutex> lk(plan->ctx->mu);
    execute_any(plan, static_cast<cudaStream_t>(stream));
  });
}

int mb_plan_results(mb_plan* plan, double* eta, double* rho, mb_point_status* status) {
  int rc = MB_OK;
  const int g = guarded([&] {
    if (!plan) fail(MB_ERR_ARG, "null plan");
    std::lock_guard<std::mutex> lk(plan->ctx->mu);
    rc = collect_results(plan, eta, rho, status);
  });
  return g != MB_OK ? g : rc;
}

int mb_plan_timing(const mb_plan* plan, double* ms_total, double* ms_potential, double* ms_propagate, int* launches) {
  return guarded([&] {
    if (!plan) fail(MB_ERR_ARG, "null plan");
    if (ms_total) *ms_total = plan->ms_total;
    if (ms_potential) *ms_potential = plan->ms_pot;
    if (ms_propagate) *ms_propagate = plan->ms_prop;
    if (launches) *launches = plan->launches;
  });
}

int mb_plan_info(const mb_plan* plan, long* slots, int* ndiff, long* coef_bytes, int* npad, long* h2d_bytes) {
  return guarded([&] {
    if (!plan) fail(MB_ERR_ARG, "null plan");
    if (slots) *slots = plan->nslots;
    if (ndiff) *ndiff = plan->ndiff;
    // the boxed table's bytes over all devices
    const int bs = plan->shards.empty() ? plan->box_size : plan->shards.front()->box_size;
    if (coef_bytes) *coef_bytes = (long)plan->S * plan->nslots * bs * (long)sizeof(double2);
    if (npad) *npad = plan->npad;
    if (h2d_bytes) *h2d_bytes = plan->h2d_bytes;
  });
}

int mb_plan_profile(const mb_plan* plan, double* cycles) {
  return guarded([&] {
    if (!plan || !cycles) fail(MB_ERR_ARG, "null argument");
    double acc[mbx::kProfSlots] = {};
    std::vector<const mb_plan*> parts;
    if (plan->shards.empty())
      parts.push_back(plan);
    else
      for (const mb_plan* sp : plan->shards) parts.push_back(sp);
    for (const mb_plan* sp : parts) {
      unsigned long long v[mbx::kProfSlots];
      cuda_check(cudaSetDevice(sp->ctx->device), "cudaSetDevice");
      cuda_check(cudaMemcpy(v, sp->prop.prof, sizeof v, cudaMemcpyDeviceToHost), "D2H profile");
      for (int q = 0; q < mbx::kProfSlots; ++q) acc[q] += (double)v[q];
    }
    for (int q = 0; q < mbx::kProfSlots; ++q) cycles[q] = acc[q] / (double)plan->npairs;
  });
}

int mb_plan_node_heights(const mb_plan* plan, double* z, long cap) {
  return guarded([&] {
    if (!plan || !z) fail(MB_ERR_ARG, "null argument");
    const mb_plan* p0 = plan->shards.empty() ? plan : plan->shards.front();
    if (cap < (long)p0->zslot.size()) fail(MB_ERR_ARG, "mb_plan_node_heights: capacity too small");
    std::memcpy(z, p0->zslot.data(), p0->zslot.size() * sizeof(double));
  });
}

int mb_plan_gamma(const mb_plan* plan, long pair, double* gdiag, double* ginv, double* gamma2, double* sin_theta0) {
  return guarded([&] {
    if (!plan) fail(MB_ERR_ARG, "null plan");
    if (pair < 0 || pair >= plan->npairs) fail(MB_ERR_ARG, "mb_plan_gamma: pair index out of range");
    if (!plan->shards.empty()) {
      for (std::size_t s = 0; s < plan->shards.size(); ++s) {
        const auto& rows = plan->shard_rows[s];
        auto it = std::lower_bound(rows.begin(), rows.end(), pair);
        if (it != rows.end() && *it == pair)
          return (void)mb_plan_gamma(plan->shards[s], (long)(it - rows.begin()), gdiag, ginv, gamma2, sin_theta0);
      }
      fail(MB_ERR_ARG, "mb_plan_gamma: pair not found");
    }
    const std::size_t o = (std::size_t)pair * plan->n;
    for (int i = 0; i < plan->n; ++i) {
      if (gdiag) gdiag[2 * i] = plan->gd[o + i].x, gdiag[2 * i + 1] = plan->gd[o + i].y;
      if (ginv) ginv[2 * i] = plan->gi[o + i].x, ginv[2 * i + 1] = plan->gi[o + i].y;
      if (gamma2) gamma2[i] = plan->g2[o + i];
    }
    if (sin_theta0) *sin_theta0 = plan->s0[(std::size_t)pair];
  });
}

int mb_plan_coefficients(mb_plan* plan, int structure, double* coef, long cap) {
  return guarded([&] {
    if (!plan || !coef) fail(MB_ERR_ARG, "null argument");
    if (structure < 0 || structure >= plan->S) fail(MB_ERR_ARG, "mb_plan_coefficients: structure out of range");
    if (!plan->executed) fail(MB_ERR_ARG, "plan has not been executed");
    if (!plan->shards.empty()) {
      for (std::size_t s = 0; s < plan->shards.size(); ++s) {
        const int lo = plan->shard_s0[s], hi = lo + plan->shards[s]->S;
        if (structure >= lo && structure < hi) {
          const int rc = mb_plan_coefficients(plan->shards[s], structure - lo, coef, cap);
          if (rc != MB_OK) fail(rc, g_last_error);
          return;
        }
      }
      fail(MB_ERR_ARG, "mb_plan_coefficients: structure not on any device");
    }
    const std::size_t cnt = (std::size_t)plan->nslots * plan->ndiff;
    if (cap < (long)(2 * cnt)) fail(MB_ERR_ARG, "mb_plan_coefficients: capacity too small");
    std::lock_guard<std::mutex> lk(plan->ctx->mu);
    const std::size_t bcnt = (std::size_t)plan->nslots * plan->box_size;
    std::vector<double2> boxed(bcnt);
    cuda_check(cudaSetDevice(plan->ctx->device), "cudaSetDevice");
    cuda_check(cudaMemcpyAsync(boxed.data(), plan->prop.coef + (std::size_t)structure * bcnt, bcnt * sizeof(double2),
                               cudaMemcpyDeviceToHost, plan->ctx->stream),
               "D2H coefficient table");
    cuda_check(cudaStreamSynchronize(plan->ctx->stream), "D2H coefficient table");
    // the boxed table back in difference order [slot][ndiff]
    for (long sl = 0; sl < plan->nslots; ++sl)
      for (int d = 0; d < plan->ndiff; ++d) {
        const double2 v = boxed[(std::size_t)sl * plan->box_size + plan->boxpos[(std::size_t)d]];
        coef[2 * ((std::size_t)sl * plan->ndiff + d)] = v.x;
        coef[2 * ((std::size_t)sl * plan->ndiff + d) + 1] = v.y;
      }
  });
}

int mb_plan_destroy(mb_plan* plan) {
  return guarded([&] {
    if (!plan) return;
    std::lock_guard<std::mutex> lk(plan->ctx->mu);
    destroy_any(plan);
  });
}

int mb_rocking_curve(mb_context* ctx, const mb_field* field, const mb_rods* rods, double gamma, const double* theta0,
                     int n_theta0, const double* theta1, int n_theta1, const mb_stepper* stepper,
                     const mb_options* opts, double* eta, double* rho, mb_point_status* status) {
  mb_plan* plan = nullptr;
  int rc = guarded([&] {
    if (!theta0 || !theta1 || !eta) fail(MB_ERR_ARG, "null argument");
    // AngleGrid::validated (sweep.cpp:18-33)
    if (n_theta0 < 1) fail(MB_ERR_CONFIG, "angle grid: theta0 list is empty");
    if (n_theta1 < 1) fail(MB_ERR_CONFIG, "angle grid: theta1 list is empty");
    for (int i = 0; i < n_theta0; ++i)
      if (!(theta0[i] > 0.0 && theta0[i] < 90.0))
        fail(MB_ERR_CONFIG, "angle grid: glancing angles must lie in (0, 90) degrees");
    for (int i = 1; i < n_theta0; ++i)
      if (!(theta0[i] > theta0[i - 1])) fail(MB_ERR_CONFIG, "angle grid: theta0 must be strictly increasing");
    for (int i = 0; i < n_theta1; ++i)
      if (!std::isfinite(theta1[i])) fail(MB_ERR_CONFIG, "angle grid: theta1 must be finite");
    std::vector<mb_pair> pairs;
    for (int b = 0; b < n_theta1; ++b)
      for (int a = 0; a < n_theta0; ++a) pairs.push_back(mb_pair{0, theta0[a], theta1[b]});
    if (!ctx) fail(MB_ERR_ARG, "null context");
    std::lock_guard<std::mutex> lk(ctx->mu);
    plan = create_any(ctx, rods, field, 1, gamma, pairs.data(), (long)pairs.size(), stepper, opts);
    execute_any(plan, nullptr);
  });
  if (rc != MB_OK) {
    if (plan) mb_plan_destroy(plan);
    return rc;
  }
  rc = mb_plan_results(plan, eta, rho, status);
  const std::string err = g_last_error;
  mb_plan_destroy(plan);
  g_last_error = err;
  return rc;
}

}  // extern "C"
