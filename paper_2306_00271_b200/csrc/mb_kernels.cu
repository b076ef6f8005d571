// sm_100a kernels of the B200-native forward model.
//
//   K1  potential_amp_kernel / potential_coef_kernel
//       slice-potential coefficients u(dg, z_slot) for every node slot of the
//       slicing plan (replaces BoundPotential::eval_coeffs + UTable,
//       /root/reference/proj/core/src/potential.cpp:169-207, stages.cpp:32-47).
//   K2  propagate_kernel<Cfg, RK4>
//       one CTA per (structure, angle) pair; the economical state [Q; P]
//       stays on chip for all slices (proposed.cpp:275-289). Per kick / RK
//       stage the complex product U*X runs on the FP64 tensor pipe
//       (mma.sync m8n8k4 f64 -> DMMA.8x8x4) with U gathered on the fly from the
//       node's compact coefficient table staged in shared memory (cp.async),
//       so no N x N U matrix ever touches HBM. Fused: Gershgorin estimate and
//       RHST (kernels.cpp:82-99, proposed.cpp:196-202) as an in-CTA
//       Gauss-Jordan column elimination with partial pivoting plus the 1e-10
//       residual gate of solve_right (kernels.cpp:60-80); the surface solve
//       R T^-1 (proposed.cpp:204-208) with the same machinery; intensity
//       (curve.cpp:8-20).
#include <cuda_runtime.h>

#include <cstdint>

#include "mb_device.cuh"
#include "mb_internal.h"
#include "mb_tiles.cuh"

namespace mbx {

// ============================================================== helpers
// MB_PROFILE builds (make prof) accumulate per-phase SM cycles of thread 0 of
// every CTA: 0 table wait+barrier, 1 GEMM, 2 kick epilogue, 3 RHST Gauss-Jordan,
// 4 Gershgorin, 5 RHST, 6 surface solve, 7 prologue.
#ifdef MB_PROFILE
#define PROF_MARK(slot)                             \
  do {                                              \
    const long long _t = clock64();                 \
    prof_acc[slot] += _t - prof_t;                  \
    prof_t = _t;                                    \
  } while (0)
#else
#define PROF_MARK(slot) \
  do {                  \
  } while (0)
#endif
// ============================================================== K1
// amp[s][t][d] = cpre * exp(-latk |g|^2) * exp(-i g.xy)
__global__ void potential_amp_kernel(const __grid_constant__ PotentialParams p) {
  const long total = (long)p.S * p.T * p.ndiff;
  for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
       idx += (long)gridDim.x * blockDim.x) {
    const int d = (int)(idx % p.ndiff);
    const long st = idx / p.ndiff;  // s*T + t
    const double2 g = p.diff_g[d];
    const double lat = exp(-p.term_latk[st] * (g.x * g.x + g.y * g.y));
    const double2 xy = p.term_xy[st];
    const double ph = -(g.x * xy.x + g.y * xy.y);
    double sn, cs;
    sincos(ph, &sn, &cs);
    const double2 c = p.term_cpre[st];
    const double2 cl = make_double2(c.x * lat, c.y * lat);
    p.amp[idx] = cmul(cl, make_double2(cs, sn));
  }
}

// coef[s][slot][boxpos[d]] = sum_t amp[s][t][d] * exp(-alpha_t (z_slot - zc_t)^2)
// grid: (structure x slot blocks of kSlotTile) folded into gridDim.x; threads
// over d. The z-Gaussians of the slot tile are staged in shared memory in
// chunks of kTermChunk terms (fixed 32 KB, any atom count); every amp element
// is read once per tile and reused kSlotTile times from registers, the sums
// stay in registers across chunks.
constexpr int kSlotTile = 16, kTermChunk = 256;
__global__ void __launch_bounds__(128) potential_coef_kernel(const __grid_constant__ PotentialParams p) {
  __shared__ double zg[kTermChunk * kSlotTile];  // [t in chunk][kSlotTile]
  const long tiles = (p.nslots + kSlotTile - 1) / kSlotTile;
  const int s = (int)(blockIdx.x / tiles);
  const long slot0 = (long)(blockIdx.x % tiles) * kSlotTile;
  const int nsl = (int)min((long)kSlotTile, p.nslots - slot0);
  const double2* amp = p.amp + (long)s * p.T * p.ndiff;
  // d loop outside so each thread keeps its sums across the term chunks
  const int dlim = (p.ndiff + blockDim.x - 1) / blockDim.x * blockDim.x;
  for (int d0 = 0; d0 < dlim; d0 += blockDim.x) {
    const int d = d0 + threadIdx.x;
    double re[kSlotTile], im[kSlotTile];
#pragma unroll
    for (int q = 0; q < kSlotTile; ++q) re[q] = im[q] = 0.0;
    for (int t0 = 0; t0 < p.T; t0 += kTermChunk) {
      const int tn = min(kTermChunk, p.T - t0);
      __syncthreads();
      for (int i = threadIdx.x; i < tn * kSlotTile; i += blockDim.x) {
        const int t = t0 + i / kSlotTile, q = i % kSlotTile;
        double v = 0.0;
        if (q < nsl) {
          const double dz = p.z_slot[slot0 + q] - p.term_zc[(long)s * p.T + t];
          v = exp(-p.term_alpha[(long)s * p.T + t] * dz * dz);
        }
        zg[i] = v;
      }
      __syncthreads();
      if (d < p.ndiff)
        for (int t = 0; t < tn; ++t) {
          const double2 a = amp[(long)(t0 + t) * p.ndiff + d];
#pragma unroll
          for (int q = 0; q < kSlotTile; ++q) {
            const double g = zg[t * kSlotTile + q];
            re[q] = fma(a.x, g, re[q]);
            im[q] = fma(a.y, g, im[q]);
          }
        }
    }
    if (d < p.ndiff) {
      double2* out = p.coef + ((long)s * p.nslots + slot0) * p.box_size + p.boxpos[d];
#pragma unroll
      for (int q = 0; q < kSlotTile; ++q)
        if (q < nsl) out[(long)q * p.box_size] = make_double2(re[q], im[q]);
    }
  }
}

cudaError_t launch_potential(const PotentialParams& p, cudaStream_t st, int* launches) {
  const long total = (long)p.S * p.T * p.ndiff;
  if (total > 0) {
    const int blocks = (int)min((total + 255) / 256, (long)148 * 16);
    potential_amp_kernel<<<blocks, 256, 0, st>>>(p);
    ++*launches;
  }
  const long blocks = (long)p.S * ((p.nslots + kSlotTile - 1) / kSlotTile);
  if (blocks > 0x7fffffffL) return cudaErrorInvalidConfiguration;
  potential_coef_kernel<<<(unsigned)blocks, 128, 0, st>>>(p);
  ++*launches;
  return cudaGetLastError();
}

// ============================================================== K2

// B <- B * A^-1 on the n x n blocks (A destroyed): Gauss-Jordan column
// elimination with partial pivoting on row k of A. This is Eigen's
// PartialPivLU of A^T (kernels.cpp:66-71: row pivoting of A^T = column
// pivoting here, first maximum wins) fused with the substitution. Warp 0
// updates row k+1 of A first and immediately computes the next pivot (the
// only serial chain); every warp then updates the remaining rows in batches.
// One barrier per pivot step. Returns false on an exactly zero pivot
// (kernels.cpp:68-71).
template <class C, int RB_ = 0>
__device__ bool gauss_jordan(double* Ar, double* Ai, double* Br, double* Bi, double2* fv /*[2][NP]*/, int n,
                             Scratch& sc, int warp, int lane, long long* pa = nullptr) {
#ifdef MB_PROFILE
  long long t_prev = clock64();
#define GJ_MARK(q)                    \
  do {                                \
    if (pa) {                         \
      const long long _t = clock64(); \
      pa[q] += _t - t_prev;           \
      t_prev = _t;                    \
    }                                 \
  } while (0)
#else
#define GJ_MARK(q) \
  do {             \
  } while (0)
#endif
  constexpr int NQ = (C::NP + 31) / 32;
  constexpr int RB = RB_ ? RB_ : (NQ == 1 ? 8 : 4);  // rows per batch (register budget: P stays live)
  if (n == 0) return true;
  if (warp == 0) {
    double2 a[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int j = lane + 32 * q;
      a[q] = j < C::NP ? make_double2(Ar[sw<C::NP>(0, j)], Ai[sw<C::NP>(0, j)]) : make_double2(0.0, 0.0);
    }
    gj_pivot<C>(a, 0, n, fv, sc, 0, lane);
  }
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const int slot = k & 1;
    if (!(sc.pivval[slot] > 0.0)) return false;
    const int p = sc.piv[slot];
    const double2 inv = sc.inv[slot];
    const double2* f = fv + slot * C::NP;
    double2 fj[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int j = lane + 32 * q;
      fj[q] = j < C::NP ? f[j] : make_double2(0.0, 0.0);
    }
    GJ_MARK(11);
    if (warp == 0 && k + 1 < n) {  // critical chain: row k+1, then the next pivot
      const int rows[1] = {k + 1};
      const bool isA[1] = {true};
      double2 row[1][NQ];
      gj_rows<C, 1>(Ar, Ai, Br, Bi, rows, isA, k, p, inv, fj, row, lane);
      GJ_MARK(8);
      gj_pivot<C>(row[0], k + 1, n, fv + (slot ^ 1) * C::NP, sc, slot ^ 1, lane);
      GJ_MARK(9);
    }
    // remaining rows: A rows k+2..n-1, B rows 0..n-1, over the warps that are
    // not on the pivot chain
    constexpr int W0 = C::NW > 1 ? 1 : 0, NWP = C::NW - W0;
    const int nA = n > k + 2 ? n - k - 2 : 0, total = nA + n;
    for (int t0 = warp - W0; t0 >= 0 && t0 < total; t0 += RB * NWP) {
      int rows[RB];
      bool isA[RB];
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        const int t = t0 + u * NWP;
        isA[u] = t < nA;
        rows[u] = t >= total ? -1 : (t < nA ? k + 2 + t : t - nA);
      }
      double2 row[RB][NQ];
      gj_rows<C, RB>(Ar, Ai, Br, Bi, rows, isA, k, p, inv, fj, row, lane);
    }
    GJ_MARK(10);
    __syncthreads();
  }
  return true;
#undef GJ_MARK
}

// ---------------------------------------------------------------- blocked,
// pivot-free Gauss-Jordan for strictly row-diagonally-dominant A (finite
// Gershgorin estimate). Then A^T is column-diagonally dominant, partial
// pivoting on A^T (the reference's PartialPivLU, kernels.cpp:66) selects the
// diagonal at every step and every Schur complement stays dominant, so the
// pivot sequence is the identity: this computes the same elimination with the
// bulk of the work as DMMA tiles. Panels of 8 rows of A: T = (A_pp)^-1 by
// warp 0, then every warp owns whole 8-row blocks of [A; B] and applies
// X[:, panel] <- X[:, panel] T and X[:, rest] -= X[:, panel] A[panel, rest].
struct PanelScratch {
  double rr[8 * 64], ri[8 * 64];  // -A[panel rows][:] with the panel columns zeroed
  double tr[64], ti[64];          // T = A_pp^-1, row-major [k][n]
  int fail;
  int vfail;  // VERIFY: a pivot would leave the diagonal
};

// 8x8 complex tile product: c += A[r0.., k0..k0+7] (swizzled NP plane) x
// B (8 x ldb plane, swizzled rows 0..7) at columns c0..c0+7
template <class C>
__device__ __forceinline__ void tile_k8(double (&c)[4], const double* Ar, const double* Ai, int r0, int k0,
                                        const double* Br, const double* Bi, int c0, int lane, bool b_small) {
#pragma unroll
  for (int kb = 0; kb < 2; ++kb) {
    const int ao = sw<C::NP>(r0 + (lane >> 2), k0 + kb * 4 + (lane & 3));
    const double ar = Ar[ao], ai = Ai[ao];
    const int k = kb * 4 + (lane & 3);
    const int bo = b_small ? k * 8 + (lane >> 2) : sw<C::NP>(k, c0 + (lane >> 2));
    const double br = Br[bo], bi = Bi[bo];
    dmma(c[0], c[1], ar, br);
    dmma(c[2], c[3], ar, bi);
    dmma(c[0], c[1], dneg(ai), bi);
    dmma(c[2], c[3], ai, br);
  }
}

// VERIFY: used when the Gershgorin estimate is not finite. Partial pivoting
// may then leave the diagonal, but it rarely does (cfg1: 45 of the 50
// non-dominant RHSTs per point keep every pivot on the diagonal; cfg2: all).
// Warp 0 replays each panel's eliminations on the panel's full rows and
// checks the pivot rule of the unblocked elimination at every step: the
// diagonal must be a first maximum of |a_kj|^2 over j >= k. The first failed
// check (or zero pivot) returns false, and the caller redoes the solve with
// partial pivoting from the saved Q and P.
template <class C, bool VERIFY = false>
__device__ bool gauss_jordan_dominant(double* Ar, double* Ai, double* Br, double* Bi, int n, PanelScratch& ps,
                                      int tid, int warp, int lane) {
  constexpr int NP = C::NP;
  static_assert(NP <= 64, "panel scratch sized for NP <= 64");
  const int nbB = (n + 7) >> 3;
  for (int k0 = 0; k0 < n; k0 += 8) {
    const int bsz = min(8, n - k0);
    // (1) -A[panel rows][:] with the panel columns zeroed (rank-8 operand)
    for (int w = tid; w < 8 * NP; w += C::NT) {
      const int i = w / NP, c = w % NP;
      const bool keep = i < bsz && (c < k0 || c >= k0 + 8);
      const int o = sw<NP>(k0 + i, c);
      ps.rr[sw<NP>(i, c)] = keep ? -Ar[o] : 0.0;
      ps.ri[sw<NP>(i, c)] = keep ? -Ai[o] : 0.0;
    }
    // (2) warp 0: T = A_pp^-1 (row-operation Gauss-Jordan on [A_pp | I]; the
    // padded block of a partial panel is the identity)
    // the pivot-rule replay (VERIFY) runs on warp 1 next to warp 0's inverse
    constexpr int VW = C::NW > 1 ? 1 : 0;
    if (VERIFY && warp == VW) {
      int bad = 0;
      {
        constexpr int NQ = (NP + 31) / 32;
        double2 R[8][NQ];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const int j = lane + 32 * q;
            R[i][q] = (i < bsz && j < NP) ? make_double2(Ar[sw<NP>(k0 + i, j)], Ai[sw<NP>(k0 + i, j)])
                                          : make_double2(0.0, 0.0);
          }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (t < bsz) {  // predicated, not break: R stays in registers
          const int k = k0 + t;
          double vmax = 0.0, vkk = 0.0;
          double2 rk = make_double2(0.0, 0.0);
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const int j = lane + 32 * q;
            const double v = R[t][q].x * R[t][q].x + R[t][q].y * R[t][q].y;
            if (j > k && j < n) vmax = fmax(vmax, v);
            if (q == (k >> 5)) {
              vkk = v;
              rk = R[t][q];
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
          vkk = __shfl_sync(0xffffffffu, vkk, k & 31);
          rk = make_double2(__shfl_sync(0xffffffffu, rk.x, k & 31), __shfl_sync(0xffffffffu, rk.y, k & 31));
          bad |= !(vkk >= vmax && vkk > 0.0);  // NaN fails too
          double r;
          asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(vkk));
          r = r * fma(-vkk, r, 2.0);
          r = r * fma(-vkk, r, 2.0);
          const double2 inv = make_double2(rk.x * r, -rk.y * r);
#pragma unroll
          for (int i = t + 1; i < 8; ++i) {
            if (i < bsz) {
            double2 xi = R[i][0];
#pragma unroll
            for (int q = 1; q < NQ; ++q)
              if (q == (k >> 5)) xi = R[i][q];
            xi = make_double2(__shfl_sync(0xffffffffu, xi.x, k & 31), __shfl_sync(0xffffffffu, xi.y, k & 31));
            const double2 x = cmul(xi, inv);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              const int j = lane + 32 * q;
              const double2 f = R[t][q];
              const double2 nv =
                  make_double2(R[i][q].x - (f.x * x.x - f.y * x.y), R[i][q].y - (f.x * x.y + f.y * x.x));
              R[i][q] = (j == k) ? x : nv;
            }
            }
          }
          }
        }
      }
      if (lane == 0) ps.vfail = bad;
    }
    if (warp == 0) {
      int bad = 0;
      const int col = lane & 15;  // lanes 0..7: A_pp columns, 8..15: identity columns
      double2 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (col < 8) {
          const bool real = i < bsz && col < bsz;
          const int o = sw<NP>(k0 + i, k0 + col);
          v[i] = real ? make_double2(Ar[o], Ai[o]) : make_double2(i == col ? 1.0 : 0.0, 0.0);
        } else {
          v[i] = make_double2(i == col - 8 ? 1.0 : 0.0, 0.0);
        }
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const double2 piv = make_double2(__shfl_sync(0xffffffffu, v[t].x, t), __shfl_sync(0xffffffffu, v[t].y, t));
        double2 f[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          f[i] = make_double2(__shfl_sync(0xffffffffu, v[i].x, t), __shfl_sync(0xffffffffu, v[i].y, t));
        const double m2 = piv.x * piv.x + piv.y * piv.y;
        bad |= !(m2 > 0.0);
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(m2));
        r = r * fma(-m2, r, 2.0);
        r = r * fma(-m2, r, 2.0);
        const double2 inv = make_double2(piv.x * r, -piv.y * r);
        const double2 vt = cmul(v[t], inv);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i == t) continue;
          v[i].x -= f[i].x * vt.x - f[i].y * vt.y;
          v[i].y -= f[i].x * vt.y + f[i].y * vt.x;
        }
        v[t] = vt;
      }
      if (lane >= 8 && lane < 16) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          ps.tr[i * 8 + (lane - 8)] = v[i].x;
          ps.ti[i * 8 + (lane - 8)] = v[i].y;
        }
      }
      if (lane == 0) ps.fail = bad;
    }
    __syncthreads();
    if (ps.fail || (VERIFY && ps.vfail)) return false;
    // (3)+(4): whole 8-row blocks per warp: A rows >= k0+8 (future panels),
    // B rows < n
    const int nbA = (NP - k0 - 8) >> 3;
    for (int rb = warp; rb < nbA + nbB; rb += C::NW) {
      const bool isA = rb < nbA;
      double* Xr = isA ? Ar : Br;
      double* Xi = isA ? Ai : Bi;
      const int r0 = isA ? k0 + 8 + 8 * rb : 8 * (rb - nbA);
      double c[4] = {0.0, 0.0, 0.0, 0.0};
      tile_k8<C>(c, Xr, Xi, r0, k0, ps.tr, ps.ti, 0, lane, true);  // X_panel T
      __syncwarp();
      {
        const int o = sw<NP>(r0 + (lane >> 2), k0 + 2 * (lane & 3));
        *reinterpret_cast<double2*>(Xr + o) = make_double2(c[0], c[1]);
        *reinterpret_cast<double2*>(Xi + o) = make_double2(c[2], c[3]);
      }
      __syncwarp();
      for (int cb = 0; cb < NP / 8; ++cb) {
        if (cb * 8 == k0) continue;
        const int c0 = cb * 8;
        const int o = sw<NP>(r0 + (lane >> 2), c0 + 2 * (lane & 3));
        const double2 xr = *reinterpret_cast<const double2*>(Xr + o);
        const double2 xi = *reinterpret_cast<const double2*>(Xi + o);
        double d[4] = {xr.x, xr.y, xi.x, xi.y};
        tile_k8<C>(d, Xr, Xi, r0, k0, ps.rr, ps.ri, c0, lane, false);
        *reinterpret_cast<double2*>(Xr + o) = make_double2(d[0], d[1]);
        *reinterpret_cast<double2*>(Xi + o) = make_double2(d[2], d[3]);
      }
    }
    __syncthreads();
  }
  return true;
}

// identity on the n x n block, zero elsewhere
template <class C>
__device__ void set_identity(double* Xr, double* Xi, int n, int tid) {
  for (int w = tid; w < C::NP * C::NP; w += C::NT) {
    const int r = w / C::NP, c = w % C::NP;
    Xr[sw<C::NP>(r, c)] = (r == c && r < n) ? 1.0 : 0.0;
    Xi[sw<C::NP>(r, c)] = 0.0;
  }
}

// solve_right residual gate (kernels.cpp:73-79): ||X A0 - B0||_F / ||B0||_F <= 1e-10.
// X dense in (Xr, Xi), A0 dense in (Or, Oi); B0 element (mb, nb, q) of the
// calling thread is produced by `b0`.
template <class C, class F>
__device__ bool residual_ok(const double* Or, const double* Oi, const double* Xr, const double* Xi, F&& b0,
                            double (&acc)[C::MB][C::NB][4], const Own<C>& own, int n, Scratch& sc, int warp,
                            int lane) {
  gemm_dense<C>(acc, Xr, Xi, Or, Oi, own.row0, own.col0, lane, (n + 3) & ~3);
  double rn = 0.0, bn = 0.0, bad = 0.0;
#pragma unroll
  for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < C::NB; ++nb)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double t = b0(mb, nb, q);
        const double d = acc[mb][nb][q] - t;
        rn += d * d;
        bn += t * t;
        if (!isfinite(acc[mb][nb][q])) bad = 1.0;
      }
  rn = warp_sum(rn);
  bn = warp_sum(bn);
  bad = warp_sum(bad);
  if (lane == 0) {
    sc.red_a[warp] = rn;
    sc.red_b[warp] = bn;
    sc.red_i[warp] = bad > 0.0;
  }
  __syncthreads();
  double R = 0.0, Bn = 0.0;
  int B = 0;
#pragma unroll
  for (int w = 0; w < C::NW; ++w) {
    R += sc.red_a[w];
    Bn += sc.red_b[w];
    B |= sc.red_i[w];
  }
  __syncthreads();
  const double bnorm = sqrt(Bn);
  const double resid = sqrt(R) / (bnorm > 0.0 ? bnorm : 1.0);
  return (resid <= 1e-10) && !B;
}

template <class C, bool RK4, bool BULK>
__global__ void __launch_bounds__(C::NT, C::MINB) propagate_kernel(const __grid_constant__ PropagateParams p) {
  constexpr int NP = C::NP, MB = C::MB, NB = C::NB;
  extern __shared__ __align__(16) unsigned char smem[];
  // planes: splitting uses X0/X1 as ping-pong Q buffers (the free one is the
  // RHST scratch) and X2 for the residual gate's saved copy; RK4 uses
  // X0 = Q, X1 = X2/X4 (scratch at step end), X2 = X3 (saved copy).
  double* const base = reinterpret_cast<double*>(smem);
  double* const Xr[3] = {base, base + 2 * NP * NP, base + 4 * NP * NP};
  double* const Xi[3] = {base + NP * NP, base + 3 * NP * NP, base + 5 * NP * NP};
  // per column group (the WM warps sharing one column range) two box buffers:
  // the groups only meet at the end-of-step check, so each syncs on its own
  // named barrier and overlaps its epilogue with the other group's GEMM
  double2* boxes = reinterpret_cast<double2*>(reinterpret_cast<double*>(smem) + 6 * NP * NP);
  double2* fv = boxes + 2 * C::WN * p.box_size;  // [2][NP]
  double* g2s = reinterpret_cast<double*>(fv + 2 * NP);  // [NP]
  // Gershgorin row sums alias the Gauss-Jordan multipliers (never live together)
  static_assert(C::WN <= 2, "rsum/dsum alias fv");
  static_assert(sizeof(PanelScratch) >= 2 * C::WN * NP * sizeof(double), "rsum/dsum alias the panel scratch");
  double* rsum = reinterpret_cast<double*>(fv);  // [WN][NP]
  double* dsum = rsum + C::WN * NP;              // [WN][NP]
  int* soff = reinterpret_cast<int*>(g2s + NP);  // [NP]
  Scratch* sc = reinterpret_cast<Scratch*>(soff + NP);
  PanelScratch* ps = reinterpret_cast<PanelScratch*>(sc + 1);
  // runtime-indexed stepper tables in shared memory (not the param space)
  double* okick = reinterpret_cast<double*>(ps + 1);  // [kMaxOcc]
  double* odrift = okick + kMaxOcc;                   // [kMaxOcc]
  double* bkick = odrift + kMaxOcc;                   // [kMaxOcc] bulk window (h_bulk)
  double* bdrift = bkick + kMaxOcc;                   // [kMaxOcc]
  int* onode = reinterpret_cast<int*>(bdrift + kMaxOcc);
  // TMA: one box-full mbarrier per box buffer (2 per column group)
  unsigned long long* const tbar = reinterpret_cast<unsigned long long*>(onode + kMaxOcc);  // [2 WN]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = p.n;
  const long pair = blockIdx.x;
  const int wm = warp / C::WN, wn = warp % C::WN;
  Own<C> own{wm * C::TM, wn * C::TN, lane};
  const double2* coef = p.coef + (long)p.pair_struct[pair] * p.nslots * p.box_size;
  const int gtid = wm * 32 + lane;  // thread index inside the column group
  constexpr int GNT = C::NT / C::WN;
  auto group_sync = [&]() __attribute__((always_inline)) {
    if constexpr (C::WN == 1)
      __syncthreads();
    else
      asm volatile("bar.sync %0, %1;" ::"r"(1 + wn), "r"(GNT) : "memory");
  };
  const int kmax = (n + 3) & ~3;
#ifdef MB_PROFILE
  long long prof_t = clock64(), prof_acc[kProfSlots] = {};
#endif

  // current / next Q planes (pointer swap, never a runtime-indexed array)
  double* Ar = Xr[0];
  double* Ai = Xi[0];
  double* Nr = Xr[1];
  double* Ni = Xi[1];
  // splitting: X2 holds the re+im sum planes of the two Q buffers (GEMM B-side
  // 3M operand); the RHST borrows them as its saved-Q pair and rebuilds them
  double* As = Xr[2];
  double* Ns = Xi[2];
  constexpr bool XS = !RK4 && NP >= 64;  // measured: a small gain at NP = 64 only
  for (int i = tid; i < kMaxOcc; i += C::NT) {
    okick[i] = p.occ_kick[i];
    odrift[i] = p.occ_drift[i];
    bkick[i] = p.bulk_kick[i];
    bdrift[i] = p.bulk_drift[i];
    onode[i] = p.occ_node[i];
  }
  // box holes (positions no rod difference maps to) are read for the padded
  // k in [n, kmax) and multiplied by zero rows of X: the boxed table carries
  // them as zeros, so every staged box is complete
  if (tid == 0) {
    for (int i = 0; i < 2 * C::WN; ++i) mbar_init(tbar + i, 1);
    mbar_fence_init();
  }
  for (int i = tid; i < NP; i += C::NT) {
    soff[i] = i < n ? p.rowoff[i] : 0;
    g2s[i] = i < n ? p.gamma2[pair * n + i] : 0.0;
  }
  // initial_state (proposed.cpp:123-128) with R_init = 0:
  // Q = diag(ginv)/2, P = (i/2) I on the n x n block, zero padding.
  for (int w = tid; w < NP * NP; w += C::NT) {
    Ar[w] = 0.0;
    Ai[w] = 0.0;
  }
  __syncthreads();
  for (int i = tid; i < n; i += C::NT) {
    const double2 gi = p.ginv[pair * n + i];
    Ar[sw<NP>(i, i)] = 0.5 * gi.x;
    Ai[sw<NP>(i, i)] = 0.5 * gi.y;
  }
  double P[MB][NB][4];
#pragma unroll
  for (int mb = 0; mb < MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = own.r(mb), c = own.c(nb) + e;
        P[mb][nb][e] = 0.0;
        P[mb][nb][2 + e] = (r == c && r < n) ? 0.5 : 0.0;
      }
  int raddr[MB];
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) {
    const int r = own.r(mb);
    raddr[mb] = r < n ? p.box_center + p.rowoff[r] : -1;
  }

  double acc[MB][NB][4];
  // rk4 K-sum in registers where they allow it (narrow tiles); at NP = 64 the
  // sum is folded into the Q plane stage by stage instead (stage-2 epilogue)
  constexpr bool SQR = RK4 && NP <= 32;
  double SQ[SQR ? MB : 1][SQR ? NB : 1][4];

  // the propagation window: the slab (main) or one bulk period (bulk seeding,
  // proposed.cpp:311-342); its node slots start at wbase in the table
  // (BULK = false: every window parameter is the slab's, read from the
  // parameter space; the bulk machinery compiles away)
  bool bulk_phase = BULK && p.bulk_steps > 0;
  auto WL = [&]() __attribute__((always_inline)) -> int { return (BULK && bulk_phase) ? p.bulk_steps : p.nsteps; };
  auto wbase = [&]() __attribute__((always_inline)) -> long { return (BULK && bulk_phase) ? p.bulk_base : 0L; };
  auto wh = [&]() __attribute__((always_inline)) -> double { return (BULK && bulk_phase) ? p.bulk_h : p.h; };
  auto wfin = [&]() __attribute__((always_inline)) -> double { return (BULK && bulk_phase) ? p.bulk_final_drift : p.final_drift; };
  auto wkick = [&](int r) __attribute__((always_inline)) -> double { return (BULK && bulk_phase) ? bkick[r] : okick[r]; };
  auto wdrift = [&](int r) __attribute__((always_inline)) -> double { return (BULK && bulk_phase) ? bdrift[r] : odrift[r]; };
  // table pipeline: slot of occurrence (step, r) = base + step*stride + node
  auto slot_of = [&](int step, int r) __attribute__((always_inline)) -> long { return wbase() + (long)step * p.slot_stride + onode[r]; };
  // TMA staging: the group's first thread arms the buffer's mbarrier with the
  // byte count and issues one cp.async.bulk of the node's box; every thread
  // of the group waits on the phase before reading. pend / ph: per buffer,
  // a copy in flight / the parity to wait for (group-uniform).
  double2* const bufA = boxes + (2 * wn) * p.box_size;
  unsigned long long* const barA = tbar + 2 * wn;
  const unsigned box_bytes = (unsigned)p.box_size * (unsigned)sizeof(double2);
  unsigned pend = 0u, ph = 0u;
  auto issue = [&](double2* dst, long slot) __attribute__((always_inline)) {
    const int b = dst == bufA ? 0 : 1;
    if (gtid == 0) {
      mbar_expect_tx(barA + b, box_bytes);
      bulk_g2s(dst, coef + slot * p.box_size, box_bytes, barA + b);
    }
    pend |= 1u << b;
  };
  auto wait_box = [&](double2* buf) __attribute__((always_inline)) {
    const int b = buf == bufA ? 0 : 1;
    if ((pend >> b) & 1u) {
      mbar_wait(barA + b, (ph >> b) & 1u);
      ph ^= 1u << b;
      pend &= ~(1u << b);
    }
  };
  double2* cur = bufA;
  double2* nxt = bufA + p.box_size;
  __syncthreads();  // barriers initialised
  long cur_slot = -1;

  int rhst = 0, npiv = 0;
  int code = 0, fail_step = 0;
  const int nocc = p.nocc;
  const bool fsal = !RK4 && p.fsal && p.variant == 1;
  // FSAL (BAB): the last kick of a step and the first kick of the next share
  // the node height and Q, hence one product W = (U + G^2) Q. Both
  // subtractions run separately with the reference's rounding around the
  // end-of-step check (P1 = P - k_last W is what the check and an RHST see);
  // after an RHST the first kick uses Q = I, W = U + G^2 from the node's box
  // (U I is exact in the reference). Bitwise the results of fsal = 0.
  double2* mbox = bufA;
  bool qident = false;  // BAB without FSAL: this step's first kick sees Q = I (an RHST just ran)


  // Barrier that publishes the previous phase's shared-memory writes and the
  // table of occurrence (step, r); prefetches the next occurrence's table.
  auto begin_occ = [&](int nstep, int nr) __attribute__((always_inline)) -> double2* {
    PROF_MARK(2);
    wait_box(cur);
    group_sync();  // every warp of the group is done with nxt (its previous box)
    PROF_MARK(0);
    if (nstep < WL()) {
      const long ns = slot_of(nstep, nr);
      if (ns != cur_slot) issue(nxt, ns);
    }
    return cur;
  };
  auto end_occ = [&](int nstep, int nr) __attribute__((always_inline)) {
    if (nstep < WL()) {
      const long ns = slot_of(nstep, nr);
      if (ns != cur_slot) {
        double2* t = cur;
        cur = nxt;
        nxt = t;
        cur_slot = ns;
      }
    }
  };

#define FOR_BLK _Pragma("unroll") for (int mb = 0; mb < MB; ++mb) _Pragma("unroll") for (int nb = 0; nb < NB; ++nb)
  // splitting drift into the other Q buffer: Qn = Q + c P (own elements); no
  // write-after-read hazard with warps still reading Q in their GEMM.
  auto drift_swap = [&](double c) __attribute__((always_inline)) {
    FOR_BLK {
      double q0[4];
      own.ld(Ar, Ai, mb, nb, q0);
#pragma unroll
      for (int q = 0; q < 4; ++q) q0[q] = drift_ref(q0[q], c, P[mb][nb][q]);
      own.st(Nr, Ni, mb, nb, q0);
      if constexpr (XS)
        *reinterpret_cast<double2*>(Ns + sw<NP>(own.r(mb), own.c(nb))) = make_double2(q0[0] + q0[2], q0[1] + q0[3]);
    }
    double* t = Ar;
    Ar = Nr;
    Nr = t;
    t = Ai;
    Ai = Ni;
    Ni = t;
    t = As;
    As = Ns;
    Ns = t;
  };
  // a kick against Q = I (right after an RHST): W = U + G^2 straight from the
  // node's box, as the reference's U * I is exact (no 3M rounding of U)
  auto ukick = [&](const double2* ubox, double kf) __attribute__((always_inline)) {
    FOR_BLK {
      const int r = own.r(mb);
      const double g2 = g2s[r];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = own.c(nb) + e;
        double2 u = make_double2(0.0, 0.0);
        if (r < n && c < n) u = ubox[raddr[mb] - soff[c]];
        P[mb][nb][e] = kick_ref(P[mb][nb][e], kf, u.x, g2, (r == c && r < n) ? 1.0 : 0.0);
        P[mb][nb][2 + e] = kick_ref(P[mb][nb][2 + e], kf, u.y, g2, 0.0);
      }
    }
  };  // sum plane of the current Q (splitting); after the initial state and RHST
  auto rebuild_sum = [&]() __attribute__((always_inline)) {
    if constexpr (XS)
      for (int w = tid; w < NP * NP; w += C::NT) As[w] = Ar[w] + Ai[w];
  };
  rebuild_sum();
  __syncthreads();
  PROF_MARK(7);
  // one pass over the current window (run_window, proposed.cpp:275-289);
  // failures set code / fail_step (step numbers offset by step_off)
  // Windows (run_window, proposed.cpp:275-289): with a bulk period, one bulk
  // period after another (compute_bulk_reflection_proposed, proposed.cpp:
  // 311-342) until R settles, then the slab from the seeded state; each window
  // ends with extract_reflection (proposed.cpp:204-208). One inline loop: the
  // window, extraction and bulk logic stay in registers (no outlined calls).
  long period = 0;
  double* const Rr = BULK ? p.bulk_scratch + pair * 2 * NP * NP : nullptr;  // previous R
  double* const Ri = BULK ? Rr + NP * NP : nullptr;
  // the slab's initial state comes from R (Rr, Ri): the settled bulk R, or a
  // caller-supplied R_init (p.r_seed; solve_proposed's R_init, proposed.cpp:301)
  bool seed = BULK && p.r_seed != 0;
  for (;;) {
  if (BULK && seed) {
    // ---- seeded slab: Q = G^-1 (I + R) / 2, P = (i/2)(I - R) (proposed.cpp:114-128)
    FOR_BLK {
      const int r = own.r(mb);
      const double2 gi = r < n ? p.ginv[pair * n + r] : make_double2(0.0, 0.0);
      const int o = r * NP + own.c(nb);
      const double2 rr = *reinterpret_cast<const double2*>(Rr + o);
      const double2 ri = *reinterpret_cast<const double2*>(Ri + o);
      double q0[4];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = own.c(nb) + e;
        const double dlt = (r == c && r < n) ? 1.0 : 0.0;
        const double re = (e ? rr.y : rr.x), im = (e ? ri.y : ri.x);
        const double ar = 0.5 * (dlt + re), ai = 0.5 * im;  // (I + R) / 2
        q0[e] = gi.x * ar - gi.y * ai;
        q0[2 + e] = gi.x * ai + gi.y * ar;
        P[mb][nb][e] = 0.5 * im;  // (i/2)(I - R) = Im(R)/2 + i (1 - Re R)/2
        P[mb][nb][2 + e] = 0.5 * (dlt - re);
      }
      own.st(Ar, Ai, mb, nb, q0);
    }
    __syncthreads();
    rebuild_sum();
    __syncthreads();
    seed = false;
  }
  const bool main = !bulk_phase;
  const int L = WL();
  const int step_off = (int)(period * L);
  cur_slot = slot_of(0, 0);
  issue(cur, cur_slot);
  qident = false;
  for (int step = 0; step < L; ++step) {
    if constexpr (RK4) {
      // ---------------- classical RK4 (proposed.cpp:141-168), restructured:
      // Qnew = Q + hP + h^2/6 (K1+K2+K3), Pnew = P + h/6 (K1 + 2K2 + 2K3 + K4),
      // X2 = Q + h/2 P, X3 = X2 + h^2/4 K1, X4 = Q + hP + h^2/2 K2, K = -(U+G^2) X
      const double h = wh();
      double *Qr = Xr[0], *Qi = Xi[0], *Yr = Xr[1], *Yi = Xi[1], *Zr = Xr[2], *Zi = Xi[2];
      FOR_BLK {  // Y = X2 = Q + h/2 P
        double v[4];
        own.ld(Qr, Qi, mb, nb, v);
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] += (0.5 * h) * P[mb][nb][q];
        own.st(Yr, Yi, mb, nb, v);
      }
      // stage 1 (foot) on Q
      double2* box = begin_occ(step, 1);
      gemm_box<C>(acc, box, soff, raddr, Qr, Qi, own.col0, lane, kmax);
      PROF_MARK(1);
      end_occ(step, 1);
      FOR_BLK {
        double q0[4], x2[4];
        own.ld(Qr, Qi, mb, nb, q0);
        own.ld(Yr, Yi, mb, nb, x2);
        const double g2 = g2s[own.r(mb)];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double K = -(acc[mb][nb][q] + g2 * q0[q]);
          acc[mb][nb][q] = K;
          if constexpr (SQR) SQ[mb][nb][q] = K;
          x2[q] += (0.25 * h * h) * K;  // X3
        }
        own.st(Zr, Zi, mb, nb, x2);
      }
      group_sync();  // every warp of the group finished reading Q in the stage-1 GEMM
      FOR_BLK {
        double q0[4];
        own.ld(Qr, Qi, mb, nb, q0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          q0[q] += h * P[mb][nb][q];  // Qbase = Q + hP
          P[mb][nb][q] += (h / 6.0) * acc[mb][nb][q];
        }
        own.st(Qr, Qi, mb, nb, q0);
      }
      // stage 2 (mid) on X2 (Y)
      box = begin_occ(step, 2);
      gemm_box<C>(acc, box, soff, raddr, Yr, Yi, own.col0, lane, kmax);
      PROF_MARK(1);
      end_occ(step, 2);
      FOR_BLK {
        double x2[4];
        own.ld(Yr, Yi, mb, nb, x2);
        const double g2 = g2s[own.r(mb)];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double K = -(acc[mb][nb][q] + g2 * x2[q]);
          acc[mb][nb][q] = K;
          if constexpr (SQR) SQ[mb][nb][q] += K;
          P[mb][nb][q] += (h / 3.0) * K;
        }
      }
      group_sync();  // every warp of the group finished reading Y
      // Y = X4 = Qbase + h^2/2 K2; Q = Qbase + h^2/6 (K1 + K2), with
      // h^2/6 K1 = 2/3 (X3 - X2) read back from the planes (no K-sum registers;
      // the rounding is one ulp of |X3|, the size of the Q update's own)
      // (braces matter: a _Pragma directly under an if/else is not a safe body)
      if constexpr (SQR) {
        FOR_BLK {
          double qb[4];
          own.ld(Qr, Qi, mb, nb, qb);
#pragma unroll
          for (int q = 0; q < 4; ++q) qb[q] += (0.5 * h * h) * acc[mb][nb][q];
          own.st(Yr, Yi, mb, nb, qb);
        }
      } else {
        FOR_BLK {
          double qb[4], x2[4], x3[4], x4[4];
          own.ld(Qr, Qi, mb, nb, qb);
          own.ld(Yr, Yi, mb, nb, x2);
          own.ld(Zr, Zi, mb, nb, x3);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            x4[q] = qb[q] + (0.5 * h * h) * acc[mb][nb][q];
            qb[q] += (h * h / 6.0) * acc[mb][nb][q] + (2.0 / 3.0) * (x3[q] - x2[q]);
          }
          own.st(Yr, Yi, mb, nb, x4);
          own.st(Qr, Qi, mb, nb, qb);
        }
      }
      // stage 3 (mid) on X3 (Z)
      box = begin_occ(step, 3);
      gemm_box<C>(acc, box, soff, raddr, Zr, Zi, own.col0, lane, kmax);
      PROF_MARK(1);
      end_occ(step, 3);
      FOR_BLK {
        double x3[4];
        own.ld(Zr, Zi, mb, nb, x3);
        const double g2 = g2s[own.r(mb)];
        if constexpr (SQR) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double K = -(acc[mb][nb][q] + g2 * x3[q]);
            SQ[mb][nb][q] += K;
            P[mb][nb][q] += (h / 3.0) * K;
          }
        } else {
          double qb[4];
          own.ld(Qr, Qi, mb, nb, qb);  // no GEMM reads Q until the next step
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double K = -(acc[mb][nb][q] + g2 * x3[q]);
            qb[q] += (h * h / 6.0) * K;
            P[mb][nb][q] += (h / 3.0) * K;
          }
          own.st(Qr, Qi, mb, nb, qb);
        }
      }
      // stage 4 (top) on X4 (Y)
      box = begin_occ(step + 1, 0);
      gemm_box<C>(acc, box, soff, raddr, Yr, Yi, own.col0, lane, kmax);
      PROF_MARK(1);
      end_occ(step + 1, 0);
      FOR_BLK {
        double x4[4];
        own.ld(Yr, Yi, mb, nb, x4);
        const double g2 = g2s[own.r(mb)];
#pragma unroll
        for (int q = 0; q < 4; ++q) P[mb][nb][q] += (h / 6.0) * -(acc[mb][nb][q] + g2 * x4[q]);
        if constexpr (SQR) {
          double qb[4];
          own.ld(Qr, Qi, mb, nb, qb);
#pragma unroll
          for (int q = 0; q < 4; ++q) qb[q] += (h * h / 6.0) * SQ[mb][nb][q];
          own.st(Qr, Qi, mb, nb, qb);
        }
      }
    } else {
      // ---------------- splitting (proposed.cpp:170-194)
      // BAB: nocc = s+1 kicks, drift after kicks 0..s-1; ABA: nocc = s kicks,
      // a drift before every kick plus a trailing drift.
      int r0 = 0;
      if (fsal && step > 0) {
        // kick 0 of this step was merged into the previous step's last kick
        // (same node height); its drift still runs.
        drift_swap(wdrift(0));
        r0 = 1;
      }
      for (int r = r0; r < nocc; ++r) {
        const bool last = (r == nocc - 1);
        const int nstep = last ? step + 1 : step;
        const int nr = last ? (fsal ? 1 : 0) : r + 1;
        if (p.variant == 0) drift_swap(wdrift(r));  // ABA: drift before kick r
        double2* box = begin_occ(nstep, nr);
        if (qident) {  // r == 0 right after an RHST: no product needed
          ukick(box, wkick(r));
          end_occ(nstep, nr);
          qident = false;
        } else {
        gemm_box<C, XS>(acc, box, soff, raddr, Ar, Ai, own.col0, lane, kmax, As);
        PROF_MARK(1);
        end_occ(nstep, nr);
        if (last) mbox = box;  // FSAL: node of the next step's first kick
        const double kc = wkick(r);
        FOR_BLK {  // acc <- W = U Q + G^2 Q (kept for an FSAL-merged next kick)
          double q0[4];
          own.ld(Ar, Ai, mb, nb, q0);
          const double g2 = g2s[own.r(mb)];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[mb][nb][q] = w_ref(acc[mb][nb][q], g2, q0[q]);
            P[mb][nb][q] = sub_ref(P[mb][nb][q], kc, acc[mb][nb][q]);
          }
        }
        }
        if (p.variant == 1 && !last) drift_swap(wdrift(r));  // BAB: drift after kick r
      }
      if (p.variant == 0) drift_swap(wfin());  // ABA trailing drift
    }

    // ---------------- end of step: finite check, Gershgorin, RHST
    // (proposed.cpp:279-287)
    PROF_MARK(2);
    double* Sr = RK4 ? Xr[1] : Nr;  // free scratch plane pair
    double* Si = RK4 ? Xi[1] : Ni;
    // row-sum buffers alternate by step (the Gauss-Jordan multipliers / the
    // blocked solve's panel scratch, both idle here): the check has one
    // CTA-wide barrier, and a warp still folding step k's sums must not see
    // a column group of step k+1 overwrite them
    double* const rsb = (step & 1) ? reinterpret_cast<double*>(ps) : rsum;
    const double xi =
        finite_and_gershgorin<C>(Ar, Ai, P, own, n, rsb, rsb + (dsum - rsum), *sc, tid, warp, lane);
    PROF_MARK(4);
    if (xi < 0.0) {
      code = 1;
      fail_step = step_off + step;
      break;
    }
    if (fsal && step + 1 < L && !(xi > p.threshold)) {  // the next step's first kick, shared W
      const double kf = wkick(0);
      FOR_BLK {
#pragma unroll
        for (int q = 0; q < 4; ++q) P[mb][nb][q] = sub_ref(P[mb][nb][q], kf, acc[mb][nb][q]);
      }
    }
    if (xi > p.threshold) {
      // P <- P Q^-1, Q <- I (proposed.cpp:196-202)
      double* Or = Xr[2];  // saved Q for the residual gate
      double* Oi = Xi[2];
      const bool dominant = isfinite(xi);
      FOR_BLK {
        double v[4];
        if (p.residual_check || !dominant) {  // saved Q: residual gate, pivoting fallback
          own.ld(Ar, Ai, mb, nb, v);
          own.st(Or, Oi, mb, nb, v);
        }
        own.st(Sr, Si, mb, nb, P[mb][nb]);
      }
      __syncthreads();
      PROF_MARK(5);
      // finite estimate = strict row dominance: pivot-free blocked solve
      // (identical pivot sequence). Otherwise the same blocked solve with the
      // pivot rule checked panel by panel, and partial pivoting from the
      // saved Q and P when a pivot would leave the diagonal.
      bool ok;
      if (dominant) {
        ok = gauss_jordan_dominant<C>(Ar, Ai, Sr, Si, n, *ps, tid, warp, lane);
      } else {
        ok = gauss_jordan_dominant<C, true>(Ar, Ai, Sr, Si, n, *ps, tid, warp, lane);
        if (!ok) {
          FOR_BLK {
            double v[4];
            own.ld(Or, Oi, mb, nb, v);
            own.st(Ar, Ai, mb, nb, v);
            own.st(Sr, Si, mb, nb, P[mb][nb]);
          }
          __syncthreads();
#ifdef MB_PROFILE
          ok = gauss_jordan<C, RK4 ? 4 : 0>(Ar, Ai, Sr, Si, fv, n, *sc, warp, lane, tid == 0 ? prof_acc : nullptr);
          prof_t = clock64();
#else
          ok = gauss_jordan<C, RK4 ? 4 : 0>(Ar, Ai, Sr, Si, fv, n, *sc, warp, lane);
#endif
        }
      }
      PROF_MARK(3);
      if (ok && p.residual_check)
        ok = residual_ok<C>(Or, Oi, Sr, Si, [&](int mb, int nb, int q) __attribute__((always_inline)) { return P[mb][nb][q]; }, acc, own, n, *sc,
                            warp, lane);
      if (!ok) {
        code = 2;
        fail_step = step_off + step;
        break;
      }
      own.load(Sr, Si, P);
      __syncthreads();
      set_identity<C>(Ar, Ai, n, tid);
      __syncthreads();
      rebuild_sum();
      if (main) {  // SolveStats counts the slab solve only (proposed.cpp:328)
        ++rhst;
        if (!isfinite(xi)) ++npiv;
      }
      if (fsal && step + 1 < L)
        ukick(mbox, wkick(0));  // the next step's first kick, Q = I
      else
        qident = !RK4 && p.variant == 1;  // BAB: the next step opens with a kick on Q = I
      __syncthreads();
    }
    PROF_MARK(5);
  }
  wait_box(bufA);  // no copy may stay in flight past the window
  wait_box(bufA + p.box_size);
  __syncthreads();
  if (code) break;

  // ---------------- extract_reflection (proposed.cpp:204-208): X = R T^-1
  // with T = G Q - i P, R = G Q + i P; X lands in (Er, Ei). In the bulk phase
  // the state Q is put back afterwards (the next period continues from it).
  double* const Er = RK4 ? Xr[1] : Nr;
  double* const Ei = RK4 ? Xi[1] : Ni;
  {
    double* Or = Xr[2];  // saved Q: T and R are rebuilt bit-identically for the residual gate
    double* Oi = Xi[2];
    // T = G Q - i P, R = G Q + i P  (i*P = (-pi, pr)), own elements
    auto tr = [&](int mb, int nb, const double (&q0)[4], double (&t)[4], double (&rr)[4]) __attribute__((always_inline)) {
      const int r = own.r(mb);
      const double2 g = r < n ? p.gdiag[pair * n + r] : make_double2(0.0, 0.0);
#pragma unroll
      for (int e = 0; e < 2; ++e)
        tau_rho_ref(g, q0[e], q0[2 + e], P[mb][nb][e], P[mb][nb][2 + e], t[e], t[2 + e], rr[e], rr[2 + e]);
    };
    __syncthreads();
    FOR_BLK {
      double q0[4], t[4], rr[4];
      own.ld(Ar, Ai, mb, nb, q0);
      tr(mb, nb, q0, t, rr);
      own.st(Or, Oi, mb, nb, q0);
      own.st(Ar, Ai, mb, nb, t);
      own.st(Er, Ei, mb, nb, rr);
    }
    __syncthreads();
    bool ok = gauss_jordan<C, RK4 ? 4 : 0>(Ar, Ai, Er, Ei, fv, n, *sc, warp, lane);
    if (ok && p.residual_check) {
      FOR_BLK {  // A <- T0 (the solver destroyed it)
        double q0[4], t[4], rr[4];
        own.ld(Or, Oi, mb, nb, q0);
        tr(mb, nb, q0, t, rr);
        own.st(Ar, Ai, mb, nb, t);
      }
      __syncthreads();
      ok = residual_ok<C>(
          Ar, Ai, Er, Ei,
          [&](int mb, int nb, int q) __attribute__((always_inline)) {
            double q0[4], t[4], rr[4];
            own.ld(Or, Oi, mb, nb, q0);
            tr(mb, nb, q0, t, rr);
            return rr[q];
          },
          acc, own, n, *sc, warp, lane);
    }
    if (!ok) {
      code = bulk_phase ? 4 : 3;  // "bulk reflection read: ..." / "reflection extraction: ..."
      fail_step = bulk_phase ? (int)period : L;
      break;
    }
    if (BULK && bulk_phase) {
      FOR_BLK {
        double q0[4];
        own.ld(Or, Oi, mb, nb, q0);
        own.st(Ar, Ai, mb, nb, q0);
      }
      __syncthreads();
      rebuild_sum();
      __syncthreads();
    }
  }
  if (!(BULK && bulk_phase)) {
    // intensity (curve.cpp:8-20)
    const double s0 = p.sin_theta0[pair];
    const double g0 = p.gdiag[pair * n].x;
    for (int i = tid; i < n; i += C::NT) {
      const int o = sw<NP>(i, 0);
      const double2 rho = make_double2(Er[o], Ei[o]);
      const double2 gi = p.gdiag[pair * n + i];
      const bool prop = gi.y == 0.0;  // geometry.cpp:46-50: propagating rods have real Gamma
      p.rho[pair * n + i] = rho;
      p.eta[pair * n + i] = prop ? (rho.x * rho.x + rho.y * rho.y) * s0 * g0 / gi.x : 0.0;
    }
    break;
  }
  if constexpr (BULK) {
  // ---- bulk: ||R - R_prev||_F <= tol max(1, ||R||_F) (proposed.cpp:334-339)
  {
    double dn = 0.0, rn = 0.0;
    FOR_BLK {
      double x[4];
      own.ld(Er, Ei, mb, nb, x);
      const int o = own.r(mb) * NP + own.c(nb);
      const double2 pr = *reinterpret_cast<const double2*>(Rr + o);
      const double2 pi = *reinterpret_cast<const double2*>(Ri + o);
      if (period > 0) {
        const double d0 = x[0] - pr.x, d1 = x[1] - pr.y, d2 = x[2] - pi.x, d3 = x[3] - pi.y;
        dn += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
      }
      rn += x[0] * x[0] + x[1] * x[1] + x[2] * x[2] + x[3] * x[3];
      *reinterpret_cast<double2*>(Rr + o) = make_double2(x[0], x[1]);
      *reinterpret_cast<double2*>(Ri + o) = make_double2(x[2], x[3]);
    }
    dn = warp_sum(dn);
    rn = warp_sum(rn);
    if (lane == 0) {
      sc->red_a[warp] = dn;
      sc->red_b[warp] = rn;
    }
    __syncthreads();
    double D = 0.0, Rn = 0.0;
#pragma unroll
    for (int w = 0; w < C::NW; ++w) {
      D += sc->red_a[w];
      Rn += sc->red_b[w];
    }
    __syncthreads();
    if (!(period > 0 && sqrt(D) <= p.bulk_tol * fmax(1.0, sqrt(Rn)))) {
      if (++period >= p.bulk_max_periods) {
        code = 5;  // ConvergenceError: the bulk R did not settle
        fail_step = (int)period;
        break;
      }
      continue;
    }
  }
  // settled: the slab starts from the seeded state (top of the loop)
  seed = true;
  bulk_phase = false;
  period = 0;
  }
  }
  PROF_MARK(6);
#ifdef MB_PROFILE
  if (tid == 0 && p.prof)
    for (int q = 0; q < kProfSlots; ++q) atomicAdd(p.prof + q, (unsigned long long)prof_acc[q]);
#endif
  if (tid == 0) {
    PointStatus st;
    st.code = code;
    st.step = fail_step;
    st.rhst = rhst;
    st.reserved = npiv;
    p.status[pair] = st;
  }
}

// ============================================================== dispatch
template <class C, bool RK4>
static size_t smem_bytes(const PropagateParams& p) {
  const int np = C::NP;
  size_t b = (size_t)6 * np * np * sizeof(double);
  b += 2 * (size_t)C::WN * p.box_size * sizeof(double2);  // per column group
  b += 2 * (size_t)np * sizeof(double2);              // fv
  b += (size_t)np * sizeof(double);                   // g2s (rsum/dsum alias fv)
  b += (size_t)np * sizeof(int);                      // soff
  b += sizeof(Scratch) + sizeof(PanelScratch) + 16;
  b += (size_t)kMaxOcc * (4 * sizeof(double) + sizeof(int));  // stepper tables (main, bulk)
  b += 2 * (size_t)C::WN * sizeof(unsigned long long);         // TMA box barriers
  return b;
}

template <class C, bool RK4>
static cudaError_t launch_cfg(const PropagateParams& p, cudaStream_t st) {
  const size_t smem = smem_bytes<C, RK4>(p);
  auto kern = (p.bulk_steps > 0 || p.r_seed) ? propagate_kernel<C, RK4, true> : propagate_kernel<C, RK4, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)p.npairs, C::NT, smem, st>>>(p);
  return cudaGetLastError();
}

// splitting keeps P + acc (+ drift temporaries) in registers: wide tiles, one
// CTA bound; rk4 at NP <= 32 (P, SQ, acc) fits 128 registers with narrower
// tiles and gains resident CTAs per SM; rk4 at NP = 64 runs the splitting
// tile (C64) with the K-sum folded into the Q plane (16 warps spill)
// tile variants (WM, WN, CTAs/SM) selectable at build time for tuning sweeps
// (round-1 sweep on B200, tools/sweep.py cfg2 + cfg4 N=15/31: 4 warps x 3
// CTAs/SM at NP=32 beat 8 warps x 2 by 12% for rk4 and 3% for sp6; round 2:
// splitting at NP=32 takes 2 CTAs/SM, since its 3-CTA register cap (170)
// spilled the reference-rounding epilogue: N=31 sp6 14.9K -> 17.9K points/s)
#ifndef MB_C32_WM
#define MB_C32_WM 2
#define MB_C32_WN 2
#define MB_C32_MINB 2
#endif
#ifndef MB_C32R_WM
#define MB_C32R_WM 2
#define MB_C32R_WN 2
#define MB_C32R_MINB 3
#endif
#ifndef MB_C16_WM
#define MB_C16_WM 1
#define MB_C16_WN 2
#define MB_C16_MINB 4
#endif
#ifndef MB_C16R_WM
#define MB_C16R_WM 2
#define MB_C16R_WN 2
#define MB_C16R_MINB 4
#endif
using C16 = Cfg<16, MB_C16_WM, MB_C16_WN, MB_C16_MINB, true>;
using C32 = Cfg<32, MB_C32_WM, MB_C32_WN, MB_C32_MINB, true>;
using C16R = Cfg<16, MB_C16R_WM, MB_C16R_WN, MB_C16R_MINB, true>;  // 4 warps, 8x8 tiles, 4 CTAs/SM
using C32R = Cfg<32, MB_C32R_WM, MB_C32R_WN, MB_C32R_MINB, true>;  // 4 warps, 16x16 tiles, 3 CTAs/SM
using C64 = Cfg<64, 4, 2, 1, true>;

int propagate_supported(int n, int rk4) {
  if (n <= 16) return 16;
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  return 0;
}

cudaError_t launch_propagate(const PropagateParams& p, cudaStream_t st, int* launches, int* npad) {
  const int np = propagate_supported(p.n, p.rk4);
  *npad = np;
  cudaError_t e = cudaErrorInvalidValue;
  if (np == 16) e = p.rk4 ? launch_cfg<C16R, true>(p, st) : launch_cfg<C16, false>(p, st);
  if (np == 32) e = p.rk4 ? launch_cfg<C32R, true>(p, st) : launch_cfg<C32, false>(p, st);
  if (np == 64) e = p.rk4 ? launch_cfg<C64, true>(p, st) : launch_cfg<C64, false>(p, st);
  if (e == cudaSuccess) ++*launches;
  return e;
}

}  // namespace mbx
