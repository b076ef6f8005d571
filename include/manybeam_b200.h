/*
 * manybeam_b200 — C-ABI of the B200-native forward model (matrix-ODE
 * propagation + RHST + surface boundary solve -> rocking-curve intensities).
 *
 * Drop-in boundary for the reference C++ library `manybeam`
 * (/root/reference/proj, arXiv 2306.00271). Every entry point names the
 * reference interface it replaces. Plain C types only: no torch, no C++, no
 * exceptions across the ABI. All arithmetic on the device path is FP64
 * (complex128 as interleaved re/im doubles, layout-compatible with
 * std::complex<double> / cuDoubleComplex).
 *
 * Error model (reference types.hpp:20-62 -> status codes): every function
 * returns MB_OK or one of the MB_ERR_* codes below; mb_last_error() returns a
 * thread-local message. Per-point failures (BreakdownError with a step index)
 * are reported in mb_point_status; the first failing point in row order
 * decides the call's return code, as the reference rethrows worker errors in
 * row order (sweep.cpp:136-137).
 *
 * There is NO CPU fallback: without a usable sm_100 device every solve
 * returns MB_ERR_CUDA.
 */
#ifndef MANYBEAM_B200_H
#define MANYBEAM_B200_H

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (types.hpp:20-62) ---------------------------------- */
#define MB_OK 0
#define MB_ERR_CONFIG 1      /* ConfigError */
#define MB_ERR_SOLVER 2      /* SolverError (generic) */
#define MB_ERR_SINGULAR 3    /* SingularMatrixError */
#define MB_ERR_BREAKDOWN 4   /* BreakdownError{step} */
#define MB_ERR_CONVERGENCE 5 /* ConvergenceError */
#define MB_ERR_DOMAIN 6      /* DomainError */
#define MB_ERR_CUDA 7        /* device / runtime failure, no device */
#define MB_ERR_ARG 8         /* null pointer, bad size, capacity too small */

/* per-point breakdown causes (proposed.cpp:280-287, 303-308) */
#define MB_POINT_OK 0
#define MB_POINT_NONFINITE 1   /* "propagation state went nonfinite" */
#define MB_POINT_RHST 2        /* "stabilizing transform: ..." (zero pivot or residual > 1e-10) */
#define MB_POINT_EXTRACTION 3  /* "reflection extraction: ..." (zero pivot) */
#define MB_POINT_BULK_READ 4   /* "bulk reflection read: ..." (BreakdownError, step = period) */
#define MB_POINT_BULK_CONVERGENCE 5 /* ConvergenceError: bulk R did not settle (proposed.cpp:338-341) */
#define MB_POINT_RECURSION 6   /* conventional method: "conventional recursion: ..." (conventional.cpp:67-74) */

typedef struct mb_context mb_context;
typedef struct mb_plan mb_plan;

/* ---- geometry / rods (rods.hpp:9-47, rods.cpp:14-96) ------------------ */
typedef struct {
  double a1[2]; /* direct basis, A */
  double a2[2];
} mb_lattice;

/* Rod set in the reference order (||k||, kx, ky), zero rod first, plus the
 * deduplicated difference table. Caller-owned arrays:
 *   k[n][2] (1/A), m[n][2], diff[ndiff][2] (1/A), diff_m[ndiff][2],
 *   diff_index[n*n] with diff_index[j*n+k] = index of k_j - k_k (rods.hpp:37). */
typedef struct {
  int n;
  const double* k;
  const int* m;
  int ndiff;
  const double* diff;
  const int* diff_m;
  const int* diff_index;
} mb_rods;

/* RodSet::build (rods.cpp:32-96) when first_n <= 0; otherwise the first-N
 * truncation of the same order (EXTENSION, SURVEY.md finding 4; `cutoff` is
 * ignored). Two-call pattern: with null output arrays only *n and *ndiff are
 * written; with arrays of capacity cap_n / cap_diff they are filled.
 * Returns MB_ERR_ARG when a capacity is too small (sizes still written). */
int mb_rods_build(const mb_lattice* lattice, double cutoff, int first_n, int* n, int* ndiff,
                  double* k, int* m, double* diff, int* diff_m, int* diff_index, int cap_n,
                  int cap_diff);

/* ---- potential fields (potential.hpp:11-61) --------------------------- */
#define MB_FIELD_ZERO 0
#define MB_FIELD_GAUSSIAN_LAYERS 1 /* GaussianLayer list, potential.hpp:17-23 */
#define MB_FIELD_TABULATED 2       /* cubic-Hermite table, potential.cpp:169-199 */
#define MB_FIELD_ATOMS 3           /* EXTENSION: atoms + 4-Gaussian form factors */

typedef struct {
  int kind;
  double z_bottom; /* A, < 0 */
  int has_bulk_period; /* bulk seed R_init per pair (compute_bulk_reflection_proposed,
                          proposed.cpp:311-342), every N <= 256 and stepper: inside
                          the resident (N <= 64) and cluster kernels (64 < N <= 256;
                          rk4 up to N = 128), on the batched path otherwise (bulk
                          periods stepped from the host). A caller-supplied R_init
                          (mb_plan_create_seeded) replaces it. */
  double bulk_period;
  /* MB_FIELD_GAUSSIAN_LAYERS: layers[nlayers][5] = z_center, amplitude,
   * sigma_xy, sigma_z, absorption */
  int nlayers;
  const double* layers;
  /* MB_FIELD_TABULATED: z_grid[ngrid]; entry_dm[nentries][2];
   * entry_values[nentries][ngrid][2] (re, im) */
  int ngrid;
  const double* z_grid;
  int nentries;
  const int* entry_dm;
  const double* entry_values;
  /* MB_FIELD_ATOMS: atom_xyz[natoms][3] Cartesian A, atom_species[natoms],
   * atom_B[natoms] (Debye-Waller, A^2); ff_a/ff_b[nspecies][4] (A, A^2).
   * u(dg, z) = (particle_sign - i*absorption) * gamma_L * (4 pi / cell_area)
   *   * sum_a e^{-i dg.rho_a} sum_i a_i (2 sqrt(pi)/sqrt(b')) e^{-b'|dg|^2/16pi^2}
   *   * e^{-4 pi^2 (z - z_a)^2 / b'},  b' = b_i + B_a */
  int natoms;
  const double* atom_xyz;
  const int* atom_species;
  const double* atom_B;
  int nspecies;
  const double* ff_a;
  const double* ff_b;
  double cell_area;
  double gamma_L;
  double particle_sign; /* +1 electron, -1 positron */
  double absorption;
} mb_field;

/* EXTENSION: relativistic beam from kinetic energy (eV):
 * gamma = 2 pi / lambda (1/A), gamma_L = 1 + E / m0 c^2. */
int mb_beam_from_energy(double energy_ev, double* gamma, double* gamma_L);

/* ---- stepper (proposed.hpp:23-43, splitting_coefficients.cpp) -------- */
#define MB_STEP_RK4 0
#define MB_STEP_SPLITTING 1
#define MB_STEP_CONVENTIONAL 2 /* the multi-slice method (conventional.cpp:50-78): Pade-13
                                  slice exponentials + reflection recursion; N <= 32,
                                  no bulk seed; the other mb_stepper fields are unused */
#define MB_SPLIT_ABA 0
#define MB_SPLIT_BAB 1
typedef struct {
  int algorithm;
  int variant;
  int ndrift;
  const double* drift;
  int nkick;
  const double* kick;
} mb_stepper;

/* StepperSpec::by_name (proposed.cpp:24-29): "rk4", "sp4", "sp6"; and the
 * sweep's method name "conventional" (sweep.cpp:41-50) as MB_STEP_CONVENTIONAL.
 * The coefficient arrays point to library-owned static storage. */
int mb_stepper_by_name(const char* name, mb_stepper* out);

/* ---- solve options (sweep.hpp:26-32, proposed.hpp:90-92) --------------- */
typedef struct {
  double dz;             /* target slice width, SlicingPlan::with_target_dz */
  long slices;           /* EXTENSION: >0 fixes the count (SlicingPlan::with_count) */
  double rhst_threshold; /* strict '>' trigger, +inf disables (proposed.cpp:198) */
  int residual_check;    /* 1: solve_right's 1e-10 residual gate on every RHST (kernels.cpp:75-79) */
  int fsal;              /* 1: merge the last kick of a step with the next step's first
                            (same node height; exact in exact arithmetic). 0 = reference op order */
  int path;              /* 0 auto, 1 on-chip resident kernel (N <= 64),
                            2 batched large-N kernels (state in HBM, N <= 256),
                            3 cluster-resident kernel (64 < N <= 256, one CTA cluster per pair),
                            4 the same kernel as persistent cooperative CTA groups exchanging
                              through L2 (64 < N <= 256; auto picks 3 or 4 by co-residency) */
} mb_options;

/* one (structure, glancing angle) point */
typedef struct {
  int structure;
  double theta0_deg;
  double theta1_deg;
} mb_pair;

typedef struct {
  int code;        /* MB_POINT_* */
  int step;        /* BreakdownError::step */
  int rhst_count;  /* SolveStats::rhst_transforms */
  int rhst_pivoting; /* EXTENSION: transforms whose Q was not strictly row-dominant
                        (Gershgorin estimate +inf), i.e. needed a pivoting solve */
} mb_point_status;

/* ---- context ----------------------------------------------------------- */
/* One context per device; owns streams and a grow-only device arena reused
 * across calls. Thread-safe per context (calls serialize on an internal lock). */
int mb_context_create(int device, mb_context** out);
/* Several devices behind one context (the reference's
 * rocking_curve spreads its rows over the machine, sweep.cpp:111-138). A plan
 * made on it splits its pairs over the devices with a fixed map: contiguous
 * structure blocks balanced by pair count when it has several fields (each
 * structure's coefficient table is built on one device only), pairs
 * round-robin when it has one. mb_plan_execute runs every device's share on
 * its own host thread; mb_plan_results gathers the rows into the caller's
 * arrays in pair order, so the output does not depend on the device count.
 * A device may be listed twice (two shards on one GPU, separate streams).
 * Timing reports the slowest device; launches are summed. */
int mb_context_create_multi(const int* devices, int ndevices, mb_context** out);
/* devices behind a context (1 for mb_context_create) */
int mb_context_device_count(const mb_context* ctx);
int mb_context_destroy(mb_context* ctx);
const char* mb_last_error(void);
/* 1 when the library was built for sm_100a and a matching device is present */
int mb_device_ok(int device);

/* ---- batched solve (plan / execute split, cuFFT-style) ----------------
 * Replaces the per-row loop of rocking_curve (sweep.cpp:89-138) with one
 * device pass over all (structure, angle) pairs. Every field shares one rod
 * set, gamma, z_bottom and slicing. */
int mb_plan_create(mb_context* ctx, const mb_rods* rods, const mb_field* fields, int nfields,
                   double gamma, const mb_pair* pairs, long npairs, const mb_stepper* stepper,
                   const mb_options* opts, mb_plan** out);
/* The same with a caller-supplied R_init: solve_proposed(u, gamma, plan, spec,
 * opts, R_init, ...) (proposed.hpp:98-102; initial_state, proposed.cpp:123-128:
 * T = I, R = R_init at z_bottom). r_init holds r_init_count matrices of
 * n x n complex128, row-major, interleaved (re, im): count 1 = one R_init
 * shared by every pair, count npairs = one per pair (pair order). It is used
 * as given, so a field's bulk period is NOT solved for (the reference's
 * solve_row passes its bulk R the same way, sweep.cpp:96-101). Null r_init
 * with count 0 is mb_plan_create. Every design takes it (resident, cluster /
 * cooperative, batched, any device count); MB_STEP_CONVENTIONAL does not
 * (MB_ERR_CONFIG). A wrong count is MB_ERR_ARG ("R_init has wrong
 * dimensions", proposed.cpp:126). */
int mb_plan_create_seeded(mb_context* ctx, const mb_rods* rods, const mb_field* fields, int nfields,
                          double gamma, const mb_pair* pairs, long npairs, const mb_stepper* stepper,
                          const mb_options* opts, const double* r_init, long r_init_count,
                          mb_plan** out);
/* K1 (slice-potential coefficients) + K2 (propagation, RHST, extraction,
 * intensity). Inputs already device-resident; stream 0 = context stream. */
int mb_plan_execute(mb_plan* plan, void* cuda_stream);
/* D2H of eta[npairs][n], optional rho[npairs][n][2], optional status[npairs].
 * Returns the first failing pair's code (row order). */
int mb_plan_results(mb_plan* plan, double* eta, double* rho, mb_point_status* status);
/* timing of the last execute (CUDA events on the execute stream): total,
 * potential kernel, propagation kernel, in milliseconds; kernel launches */
int mb_plan_timing(const mb_plan* plan, double* ms_total, double* ms_potential,
                   double* ms_propagate, int* launches);
/* node slots of the coefficient table, its device bytes, the padded kernel
 * size and the host->device bytes the plan uploaded */
int mb_plan_info(const mb_plan* plan, long* slots, int* ndiff, long* coef_bytes, int* npad, long* h2d_bytes);
/* per-CTA average SM cycles by kernel phase (table wait, GEMM, kick epilogue,
 * finite check, Gershgorin, RHST, surface solve, prologue) of the last
 * execute; all zero unless the library was built with MB_PROFILE */
int mb_plan_profile(const mb_plan* plan, double* cycles16);
/* EXTENSION (parity hooks; no reference counterpart): host copies of what
 * mb_plan_create built, so tests can compare them with the reference.
 *   node heights z[slots] in coefficient-table slot order (stages.cpp:25-47;
 *     slab window then, with a bulk period, the mapped bulk window);
 *   per pair Gamma[n][2], 1/Gamma[n][2], Gamma^2[n] and sin(theta0)
 *     (GammaMatrix::build, geometry.cpp:30-57; any output may be null);
 *   after an execute, the K1 coefficient table of one structure,
 *     coef[slots][ndiff][2] (BoundPotential::eval_coeffs per node,
 *     potential.cpp:169-199, plus the atom extension). cap counts doubles. */
int mb_plan_node_heights(const mb_plan* plan, double* z, long cap);
int mb_plan_gamma(const mb_plan* plan, long pair, double* gdiag, double* ginv, double* gamma2, double* sin_theta0);
int mb_plan_coefficients(mb_plan* plan, int structure, double* coef, long cap);
int mb_plan_destroy(mb_plan* plan);

/* rocking_curve (sweep.hpp:37-38, sweep.cpp:54-143), stepper methods:
 * rows are theta1-major with theta0 inner (sweep.cpp:90-91). eta[rows][n]. */
int mb_rocking_curve(mb_context* ctx, const mb_field* field, const mb_rods* rods, double gamma,
                     const double* theta0, int n_theta0, const double* theta1, int n_theta1,
                     const mb_stepper* stepper, const mb_options* opts, double* eta, double* rho,
                     mb_point_status* status);

#ifdef __cplusplus
}
#endif
#endif /* MANYBEAM_B200_H */
