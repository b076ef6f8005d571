// Internal structures shared by the host runtime (mb_host.cpp) and the sm_100a
// kernels (mb_kernels.cu). Not part of the public ABI.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace mbx {

constexpr int kProfSlots = 16;  // MB_PROFILE phase slots
constexpr int kMaxOcc = 32;  // kick occurrences (or RK stages) per step
constexpr int MB_POINT_RECURSION_CODE = 6;  // = MB_POINT_RECURSION (conventional method)

// Point status on the device (mirrors mb_point_status)
struct PointStatus {
  int code, step, rhst, reserved;  // reserved: RHSTs that took the pivoting solve
};

// ---- K1: slice-potential coefficients --------------------------------------
// coef[s][slot][d] = sum_t amp[s][t][d] * exp(-alpha[s][t] * (z[slot] - zc[s][t])^2)
// amp[s][t][d]     = cpre[s][t] * lat * e^{-i g_d . rho_t}   (atoms)
//                  = cpre[s][t] * lat                         (gaussian layers)
// lat              = exp(-lat_k[s][t] * |g_d|^2)
struct PotentialParams {
  int S, T, ndiff;
  long nslots;
  const double* z_slot;   // [nslots]
  const double2* diff_g;  // [ndiff] (gx, gy), 1/A
  const double* term_zc;  // [S*T]
  const double* term_alpha;
  const double* term_latk;
  const double2* term_cpre;  // complex prefactor
  const double2* term_xy;    // in-plane position (atoms) or (0,0)
  double2* amp;              // [S][T][ndiff] scratch
  // boxed table: coef[s][slot][box_size], difference d at position boxpos[d],
  // holes zero (set once at plan creation): one node = one contiguous block
  // that the propagation kernels stage with a single TMA bulk copy
  double2* coef;             // [S][nslots][box_size]
  const int* boxpos;         // [ndiff]
  int box_size;
};

// ---- K2: propagation + RHST + extraction + intensity -----------------------
struct PropagateParams {
  int n, ndiff;
  int nsteps;
  long nslots;
  long npairs;
  // coefficient table, boxed: node slot = box_size double2 (holes zero)
  const double2* coef;     // [S][nslots][box_size]
  const int* boxpos;       // [ndiff] -> position inside the box
  const int* rowoff;       // [n] -> m1*W2 + m2 (box row offset of rod j)
  int box_size, box_center;
  // pairs
  const int* pair_struct;     // [npairs]
  const double* gamma2;       // [npairs][n]  Gamma^2 (real)
  const double2* gdiag;       // [npairs][n]  Gamma
  const double2* ginv;        // [npairs][n]  1/Gamma
  const double* sin_theta0;   // [npairs]
  // stepper
  int rk4;                    // 1 = classical RK4
  int variant;                // splitting: 0 ABA, 1 BAB
  int nocc;                   // table occurrences per step (RK4: 4 stages)
  int slot_stride;            // slots per step
  int occ_node[kMaxOcc];      // node index within the step per occurrence
  double occ_kick[kMaxOcc];   // h * b_r per kick occurrence (splitting)
  double occ_drift[kMaxOcc];  // h * a_r (BAB: after kick r; ABA: before kick r)
  double final_drift;         // ABA: trailing drift h * a_s
  double fsal_kick;           // BAB + fsal: merged coefficient h*(b_s + b_0)
  int fsal;
  double h;
  double threshold;
  int residual_check;
  // outputs
  double* eta;                // [npairs][n]
  double2* rho;               // [npairs][n]
  PointStatus* status;        // [npairs]
  unsigned long long* prof;   // [8] phase cycles (MB_PROFILE builds), may be null
  double* scratch;            // cluster kernel: per pair 6 NP^2 doubles (8 with a bulk period)
  // bulk seeding (proposed.cpp:311-342), resident and cluster kernels; bulk_steps = 0: none
  int bulk_steps;             // steps per bulk period
  long bulk_base;             // first table slot of the bulk window
  double bulk_h, bulk_final_drift, bulk_fsal_kick;
  double bulk_kick[kMaxOcc], bulk_drift[kMaxOcc];
  long bulk_max_periods;
  double bulk_tol;
  double* bulk_scratch;       // per pair 2 NP^2 doubles: the previous period's R
  // caller-supplied R_init (solve_proposed's R_init, proposed.hpp:98-102,
  // initial_state proposed.cpp:123-128): bulk_scratch holds it per pair as
  // zero-padded re / im planes (row-major, ld NP) and the slab starts from
  // Q = G^-1 (I + R)/2, P = (i/2)(I - R); no bulk window runs
  int r_seed;
  // cluster kernel, cooperative variant (COOP): persistent groups of coop_cs
  // co-resident CTAs exchanging through L2 instead of DSMEM
  int coop;                   // 1: cooperative grid, 0: one thread-block cluster per pair
  int coop_cs;                // CTAs per group (set by the launcher)
  unsigned* coop_bar;         // [groups] barrier counters (zeroed by the launcher)
  double* coop_pub;           // per CTA published arrays (kCoopPubDoubles each)
};

// upper bounds for the cooperative cluster variant's buffers
constexpr int kCoopMaxCtasPerSm = 4;
constexpr int kCoopPubDoubles = 2 * 256 + 8 + 2 * (3 * 32 + 1) + 2;

// ---- large-N batched path (mb_large.cu): state in HBM, one launch per kick
// or RK stage over all (pair, tile) work items, per-pair check and
// Gauss-Jordan kernels. Matrix m of pair p: re plane at
// state + p*pair_stride + m*2*np*np, im plane right after (row-major, ld np).
struct BigParams {
  int n, np, ndiff;
  long npairs;
  int nsteps;
  long nslots;
  int slot_stride;
  const double2* coef;
  const int* boxpos;
  const int* rowoff;
  int box_size, box_center;
  const int* pair_struct;
  const double* gamma2;
  const double2* gdiag;
  const double2* ginv;
  const double* sin_theta0;
  double* state;
  int nmat;
  long pair_stride;  // doubles per pair
  PointStatus* status;
  double* xi;  // per pair: Gershgorin estimate of the last check, -1 = nonfinite
  double* chk;               // [npairs][ceil(np/16)][4] check partials
  unsigned* chk_count;       // [npairs] arrival counters (zeroed at plan creation)
  double threshold;
  int residual_check;
  double* eta;
  double2* rho;
  const double* r_init;  // caller-supplied R_init per pair (2 np^2 doubles: re, im planes) or null
  // bulk seeding on the batched path (proposed.cpp:311-342): the previous
  // period's R per pair (same plane layout), the stopping tolerance and the
  // count of pairs that have not settled after the last bulk read
  double* bulk_r;
  double bulk_tol;
  unsigned* bulk_left;
};
// PointStatus::code of a pair whose bulk R has settled: frozen (every kernel
// skips code != 0) until the slab is seeded from it; never leaves the device
constexpr int kBulkSettled = 100;

// one tiled-GEMM launch: acc = U(slot) * M[op]; epilogue `kind`
struct BigStage {
  int kind;   // 0 init, 1 kick(+drift), 2 drift, 3..6 rk4 stage 1..4, 7 slab seeded from the settled bulk R
  int op;     // operand matrix of the GEMM
  long slot;  // node slot of U (box table)
  int step;
  double c0, c1, c2;  // kick / drift / stage coefficients
  // matrix indices
  int mq, mqn, mp, mx2, mx3, mw, mv, msq;
};

cudaError_t big_launch_stage(const BigParams& p, const BigStage& s, cudaStream_t st, int* launches);
cudaError_t big_launch_check(const BigParams& p, int step, int mq, int mp, cudaStream_t st, int* launches);
// mode 0: RHST on (A = mq, B = mp) with saves (msa, msb); mode 1: surface solve
// with scratch (msa, msb)
cudaError_t big_launch_gj(const BigParams& p, int mode, int step, int mq, int mp, int msa, int msb, int mx2,
                          double h, cudaStream_t st, int* launches);

// conventional multi-slice method (mb_conventional.cu), N <= 32
size_t conventional_scratch_doubles(long ctas);
long conventional_ctas(long npairs);
cudaError_t launch_conventional(const PropagateParams& p, long ctas, cudaStream_t st, int* launches);

// launchers (mb_kernels.cu)
cudaError_t launch_potential(const PotentialParams& p, cudaStream_t st, int* launches);
// returns cudaErrorInvalidValue when no kernel variant covers n / stepper
cudaError_t launch_propagate(const PropagateParams& p, cudaStream_t st, int* launches, int* npad);
int propagate_supported(int n, int rk4);  // padded size or 0
// cluster-resident kernel (mb_cluster.cu) for 64 < n <= 256
int cluster_np(int n);  // padded row count (128 / 256) or 0
size_t cluster_smem_bytes(int n, int rk4, int box_size, int ndiff);
// 1 when the cooperative variant finishes the batch in fewer rounds of
// co-resident pair groups than thread-block clusters do (GPC packing)
int cluster_prefer_coop(const PropagateParams& p);
cudaError_t launch_cluster(const PropagateParams& p, cudaStream_t st, int* launches);

}  // namespace mbx
