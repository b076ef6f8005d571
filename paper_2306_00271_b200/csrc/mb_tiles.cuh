// Tile machinery shared by the resident kernel (mb_kernels.cu) and the
// cluster kernel (mb_cluster.cu): tile configuration, swizzled planes, DMMA
// complex products (3M), the box-gathered propagation GEMM and the
// Gauss-Jordan pivot / row-update primitives.
#pragma once

#include <cuda_runtime.h>

#include "mb_device.cuh"

namespace mbx {

// Tile configuration: NP = padded rod count; WM x WN warps; each warp owns a
// (NP/WM) x (NP/WN) complex tile = MB x NB blocks of 8x8 (DMMA C fragments).
template <int NP_, int WM_, int WN_, int MINB_ = 1, bool M3_ = false>
struct Cfg {
  static constexpr int NP = NP_, WM = WM_, WN = WN_, MINB = MINB_;  // MINB: resident CTAs per SM
  static constexpr bool M3 = M3_;  // propagation GEMM as 3 real products (see gemm_box)
  static constexpr int NW = WM * WN, NT = NW * 32;
  static constexpr int TM = NP / WM, TN = NP / WN;
  static constexpr int MB = TM / 8, NB = TN / 8;
  static_assert(TM % 8 == 0 && TN % 8 == 0, "tile must be a multiple of 8");
};

// swizzled row-major plane: element (r, c) of an NP x NP matrix (NP >= 16).
// Row r's columns are XORed with x_r = 0, 8, 4, 12 for r & 3 = 0..3:
//  - DMMA B fragments (8-byte loads, 4 consecutive rows x 4 columns per
//    16-lane phase) and dense A fragments (rows x 4 k) see four distinct
//    column offsets mod 16, i.e. disjoint bank sets;
//  - own-element double2 accesses (rows r, r+1 x 8 columns per 8-lane phase)
//    see x_r and x_{r+1} differ in bit 3, so the two rows fill the low and
//    high halves of the 128-byte bank window.
// Both patterns are conflict-free without padding.
template <int NP>
__device__ __forceinline__ int sw(int r, int c) {
  return r * NP + (c ^ (((r & 1) << 3) | ((r & 2) << 1)));
}

// own-element accessors: v[mb][nb][0..3] = re(r,c), re(r,c+1), im(r,c), im(r,c+1)
template <class C>
struct Own {
  int row0, col0, lane;
  __device__ __forceinline__ int r(int mb) const { return row0 + mb * 8 + (lane >> 2); }
  __device__ __forceinline__ int c(int nb) const { return col0 + nb * 8 + 2 * (lane & 3); }
  __device__ __forceinline__ void ld(const double* Xr, const double* Xi, int mb, int nb, double (&v)[4]) const {
    const int o = sw<C::NP>(r(mb), c(nb));
    const double2 a = *reinterpret_cast<const double2*>(Xr + o);
    const double2 b = *reinterpret_cast<const double2*>(Xi + o);
    v[0] = a.x;
    v[1] = a.y;
    v[2] = b.x;
    v[3] = b.y;
  }
  __device__ __forceinline__ void st(double* Xr, double* Xi, int mb, int nb, const double (&v)[4]) const {
    const int o = sw<C::NP>(r(mb), c(nb));
    *reinterpret_cast<double2*>(Xr + o) = make_double2(v[0], v[1]);
    *reinterpret_cast<double2*>(Xi + o) = make_double2(v[2], v[3]);
  }
  __device__ __forceinline__ void load(const double* Xr, const double* Xi, double (&v)[C::MB][C::NB][4]) const {
#pragma unroll
    for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
      for (int nb = 0; nb < C::NB; ++nb) {
        const int o = sw<C::NP>(r(mb), c(nb));
        const double2 a = *reinterpret_cast<const double2*>(Xr + o);
        const double2 b = *reinterpret_cast<const double2*>(Xi + o);
        v[mb][nb][0] = a.x;
        v[mb][nb][1] = a.y;
        v[mb][nb][2] = b.x;
        v[mb][nb][3] = b.y;
      }
  }
  __device__ __forceinline__ void store(double* Xr, double* Xi, const double (&v)[C::MB][C::NB][4]) const {
#pragma unroll
    for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
      for (int nb = 0; nb < C::NB; ++nb) {
        const int o = sw<C::NP>(r(mb), c(nb));
        *reinterpret_cast<double2*>(Xr + o) = make_double2(v[mb][nb][0], v[mb][nb][1]);
        *reinterpret_cast<double2*>(Xi + o) = make_double2(v[mb][nb][2], v[mb][nb][3]);
      }
  }
};

template <class C>
__device__ __forceinline__ void zero(double (&v)[C::MB][C::NB][4]) {
#pragma unroll
  for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < C::NB; ++nb)
#pragma unroll
      for (int q = 0; q < 4; ++q) v[mb][nb][q] = 0.0;
}

// complex 8x8x4 block products: re += ar*br - ai*bi, im += ar*bi + ai*br.
// Issue order keeps the two updates of one accumulator 2*MB*NB DMMAs apart so
// the DMMA latency is hidden (back-to-back dependent DMMAs stall the warp).
template <class C>
__device__ __forceinline__ void cmma(double (&acc)[C::MB][C::NB][4], const double (&ar)[C::MB],
                                     const double (&ai)[C::MB], const double (&an)[C::MB], const double (&br)[C::NB],
                                     const double (&bi)[C::NB]) {
#pragma unroll
  for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < C::NB; ++nb) dmma(acc[mb][nb][0], acc[mb][nb][1], ar[mb], br[nb]);
#pragma unroll
  for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < C::NB; ++nb) dmma(acc[mb][nb][2], acc[mb][nb][3], ar[mb], bi[nb]);
#pragma unroll
  for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < C::NB; ++nb) dmma(acc[mb][nb][0], acc[mb][nb][1], an[mb], bi[nb]);
#pragma unroll
  for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < C::NB; ++nb) dmma(acc[mb][nb][2], acc[mb][nb][3], ai[mb], br[nb]);
}

// acc = U * X, U gathered from the node's box table: U(j,k) = box[raddr_j - off_k]
// (raddr_j = center + off_j, or -1 for padded rows -> 0). X rows k >= n are zero
// by construction, so padded columns of U need no mask.
//
// C::M3: the complex product as three real DMMA products (the 3M scheme of
// zgemm3m): T1 = Ur Xr, T2 = Ui Xi, T3 = (Ur+Ui)(Xr+Xi); re = T1 - T2,
// im = T3 - T1 - T2. 24 instead of 32 DMMAs per 8x8 block-k step; the sums are
// one DADD per fragment. Normwise error stays O(eps |U| |X|) (Higham, "Stability
// of a method for multiplying complex matrices with three real matrix
// multiplications", 1992), which is the bound the propagation needs.
// Xs (XS = true): a plane holding Xr + Xi, kept by the writer of X, so the
// B-side sums cost a shared load instead of a DADD on the FP64 pipe that the
// DMMAs occupy.
template <class C, bool XS = false>
__device__ __forceinline__ void gemm_box(double (&acc)[C::MB][C::NB][4], const double2* __restrict__ box,
                                         const int* __restrict__ soff, const int (&raddr)[C::MB],
                                         const double* __restrict__ Xr, const double* __restrict__ Xi,
                                         int col0, int lane, int kmax, const double* __restrict__ Xs = nullptr) {
  const int kl = lane & 3, cl = lane >> 2;
  if constexpr (C::M3) {
    double t1[C::MB][C::NB][2], t2[C::MB][C::NB][2], t3[C::MB][C::NB][2];
#pragma unroll
    for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
      for (int nb = 0; nb < C::NB; ++nb)
#pragma unroll
        for (int e = 0; e < 2; ++e) t1[mb][nb][e] = t2[mb][nb][e] = t3[mb][nb][e] = 0.0;
#pragma unroll 2
    for (int k0 = 0; k0 < kmax; k0 += 4) {
      const int k = k0 + kl;
      const int offk = soff[k];
      double ar[C::MB], ai[C::MB], as[C::MB];
#pragma unroll
      for (int mb = 0; mb < C::MB; ++mb) {
        double2 a = make_double2(0.0, 0.0);
        if (raddr[mb] >= 0) a = box[raddr[mb] - offk];
        ar[mb] = a.x;
        ai[mb] = a.y;
        as[mb] = a.x + a.y;
      }
      double br[C::NB], bi[C::NB], bs[C::NB];
#pragma unroll
      for (int nb = 0; nb < C::NB; ++nb) {
        const int o = sw<C::NP>(k, col0 + nb * 8 + cl);
        br[nb] = Xr[o];
        bi[nb] = Xi[o];
        if constexpr (XS)
          bs[nb] = Xs[o];
        else
          bs[nb] = br[nb] + bi[nb];
      }
#pragma unroll
      for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < C::NB; ++nb) dmma(t1[mb][nb][0], t1[mb][nb][1], ar[mb], br[nb]);
#pragma unroll
      for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < C::NB; ++nb) dmma(t2[mb][nb][0], t2[mb][nb][1], ai[mb], bi[nb]);
#pragma unroll
      for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < C::NB; ++nb) dmma(t3[mb][nb][0], t3[mb][nb][1], as[mb], bs[nb]);
    }
#pragma unroll
    for (int mb = 0; mb < C::MB; ++mb)
#pragma unroll
      for (int nb = 0; nb < C::NB; ++nb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          acc[mb][nb][e] = t1[mb][nb][e] - t2[mb][nb][e];
          acc[mb][nb][2 + e] = (t3[mb][nb][e] - t1[mb][nb][e]) - t2[mb][nb][e];
        }
    return;
  }
  zero<C>(acc);
#pragma unroll 2
  for (int k0 = 0; k0 < kmax; k0 += 4) {
    const int k = k0 + kl;
    const int offk = soff[k];
    double ar[C::MB], ai[C::MB], an[C::MB];
#pragma unroll
    for (int mb = 0; mb < C::MB; ++mb) {
      double2 a = make_double2(0.0, 0.0);
      if (raddr[mb] >= 0) a = box[raddr[mb] - offk];
      ar[mb] = a.x;
      ai[mb] = a.y;
      an[mb] = dneg(a.y);
    }
    double br[C::NB], bi[C::NB];
#pragma unroll
    for (int nb = 0; nb < C::NB; ++nb) {
      const int o = sw<C::NP>(k, col0 + nb * 8 + cl);
      br[nb] = Xr[o];
      bi[nb] = Xi[o];
    }
    cmma<C>(acc, ar, ai, an, br, bi);
  }
}

// acc = A * X with a dense A in shared memory (residual gate of solve_right)
template <class C>
__device__ __forceinline__ void gemm_dense(double (&acc)[C::MB][C::NB][4], const double* __restrict__ Ar,
                                           const double* __restrict__ Ai, const double* __restrict__ Xr,
                                           const double* __restrict__ Xi, int row0, int col0, int lane,
                                           int kmax) {
  zero<C>(acc);
  const int kl = lane & 3, cl = lane >> 2;
  for (int k0 = 0; k0 < kmax; k0 += 4) {
    const int k = k0 + kl;
    double ar[C::MB], ai[C::MB], an[C::MB];
#pragma unroll
    for (int mb = 0; mb < C::MB; ++mb) {
      const int o = sw<C::NP>(row0 + mb * 8 + cl, k);
      ar[mb] = Ar[o];
      ai[mb] = Ai[o];
      an[mb] = dneg(ai[mb]);
    }
    double br[C::NB], bi[C::NB];
#pragma unroll
    for (int nb = 0; nb < C::NB; ++nb) {
      const int o = sw<C::NP>(k, col0 + nb * 8 + cl);
      br[nb] = Xr[o];
      bi[nb] = Xi[o];
    }
    cmma<C>(acc, ar, ai, an, br, bi);
  }
}

// shared scratch for the block-level reductions / Gauss-Jordan
struct Scratch {
  double red_a[32], red_b[32];
  int red_i[32];
  int piv[2];
  double pivval[2];
  double2 inv[2];
};

__device__ __forceinline__ double inf_d() { return __longlong_as_double(0x7ff0000000000000LL); }

// End-of-step check on own elements, fused (proposed.cpp:279-287 +
// kernels.cpp:82-99): returns -1 if Q or P holds a nonfinite value, else the
// Gershgorin estimate max_i(|q_ii| + r_i) / min_i(|q_ii| - r_i) (+inf when
// some |q_ii| - r_i <= 0). Row sums are reduced in the accumulator layout:
// quad shuffles, then the WN column-warps through shared memory.
template <class C>
__device__ double finite_and_gershgorin(const double* Qr, const double* Qi, const double (&P)[C::MB][C::NB][4],
                                        const Own<C>& own, int n, double* rsum /*[WN][NP]*/,
                                        double* dsum /*[WN][NP]*/, Scratch& sc, int tid, int warp, int lane) {
  int bad = 0;
  double rs[C::MB], dg[C::MB];
#pragma unroll
  for (int mb = 0; mb < C::MB; ++mb) {
    rs[mb] = 0.0;
    dg[mb] = 0.0;
    const int r = own.r(mb);
#pragma unroll
    for (int nb = 0; nb < C::NB; ++nb) {
      double q[4];
      own.ld(Qr, Qi, mb, nb, q);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = own.c(nb) + e;
        bad |= !isfinite(q[e]) || !isfinite(q[2 + e]) || !isfinite(P[mb][nb][e]) || !isfinite(P[mb][nb][2 + e]);
        const double a = sqrt(q[e] * q[e] + q[2 + e] * q[2 + e]);
        if (c == r)
          dg[mb] = a;
        else if (c < n)
          rs[mb] += a;
      }
    }
    rs[mb] += __shfl_xor_sync(0xffffffffu, rs[mb], 1);
    rs[mb] += __shfl_xor_sync(0xffffffffu, rs[mb], 2);
    dg[mb] += __shfl_xor_sync(0xffffffffu, dg[mb], 1);
    dg[mb] += __shfl_xor_sync(0xffffffffu, dg[mb], 2);
    if ((lane & 3) == 0) {
      const int wn = own.col0 / C::TN;
      rsum[wn * C::NP + r] = rs[mb];
      dsum[wn * C::NP + r] = dg[mb];
    }
  }
  bad = __syncthreads_or(bad);
  if (bad) return -1.0;
  // every warp folds all rows itself (max / min / or are order-free and the
  // per-row sums keep their column-group order), so no second barrier
  double hi = 0.0, lo = inf_d();
  int nd = 0;
  for (int i = lane; i < n; i += 32) {
    double r = 0.0, d = 0.0;
#pragma unroll
    for (int w = 0; w < C::WN; ++w) {
      r += rsum[w * C::NP + i];
      d += dsum[w * C::NP + i];
    }
    hi = fmax(hi, d + r);
    if (d - r <= 0.0) nd = 1;
    lo = fmin(lo, d - r);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    nd |= __shfl_xor_sync(0xffffffffu, nd, o);
  }
  (void)sc;
  (void)tid;
  (void)warp;
  if (n == 0) return 1.0;
  if (nd) return inf_d();
  return hi / lo;
}

// Pivot of row k for the Gauss-Jordan step: first maximum of |A[k][j]| over
// j >= k (Eigen's abs score; compared as |a|^2, which orders identically up to
// ties within one rounding), multipliers f_j of the post-swap row, 1/pivot.
// `a` holds the lane's row-k elements (j = lane + 32 q).
template <class C>
__device__ __forceinline__ void gj_pivot(const double2 (&a)[(C::NP + 31) / 32], int k, int n, double2* fv,
                                         Scratch& sc, int slot, int lane) {
  constexpr int NQ = (C::NP + 31) / 32;
  // lane-local first maximum of |a|^2 (q ascending = j ascending)
  double best = -1.0;
  int bj = n;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int j = lane + 32 * q;
    const double v = a[q].x * a[q].x + a[q].y * a[q].y;
    if (j >= k && j < n && v > best) {
      best = v;
      bj = j;
    }
  }
  // warp maximum: 32-bit key (float(|a|^2) bits are monotone for v >= 0; -1
  // maps to 0), exact double comparison only among lanes tied on the key
  const unsigned key = best < 0.0 ? 0u : __float_as_uint(__double2float_ru(best)) + 1u;
  const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
  const unsigned tied = __ballot_sync(0xffffffffu, key == kmax);
  if (__popc(tied) > 1) {
    double b = key == kmax ? best : -1.0;
    int jj = key == kmax ? bj : n;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, b, o);
      const int oj = __shfl_xor_sync(0xffffffffu, jj, o);
      if (ob > b || (ob == b && oj < jj)) {
        b = ob;
        jj = oj;
      }
    }
    best = b;
    bj = jj;
  } else {
    const int src = __ffs(tied) - 1;
    best = __shfl_sync(0xffffffffu, best, src);
    bj = __shfl_sync(0xffffffffu, bj, src);
  }
  const int p = bj;
  double2 akk = make_double2(0.0, 0.0), akp = make_double2(0.0, 0.0);
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double2 x = make_double2(__shfl_sync(0xffffffffu, a[q].x, k & 31), __shfl_sync(0xffffffffu, a[q].y, k & 31));
    const double2 y = make_double2(__shfl_sync(0xffffffffu, a[q].x, p & 31), __shfl_sync(0xffffffffu, a[q].y, p & 31));
    if (q == (k >> 5)) akk = x;
    if (q == (p >> 5)) akp = y;
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int j = lane + 32 * q;
    if (j < C::NP) fv[j] = (j == k || j >= n) ? make_double2(0.0, 0.0) : (j == p ? akk : a[q]);
  }
  if (lane == 0) {
    sc.piv[slot] = p;
    sc.pivval[slot] = best;
    // 1/|pivot|^2: RCP64H seed + two Newton steps (inverse by multiplication,
    // like any reciprocal-scaled elimination; rounding-level only)
    double r;
#ifdef MB_EXACT_RCP
    r = 1.0 / best;  // accuracy study build: IEEE division
#else
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(best));
    r = r * fma(-best, r, 2.0);
    r = r * fma(-best, r, 2.0);
#endif
    sc.inv[slot] = best > 0.0 ? make_double2(akp.x * r, -akp.y * r) : make_double2(0.0, 0.0);
  }
}

// Gauss-Jordan row update: X[i][:] for the elimination of column k with
// pivot column p (new column k = X[i][p] * inv; column p takes old column k).
// Branch-free (clamped rows, value selects, predicated stores) so the loads of
// all RB rows issue before any arithmetic.
template <class C, int RB>
__device__ __forceinline__ void gj_rows(double* Ar, double* Ai, double* Br, double* Bi, const int (&rows)[RB],
                                        const bool (&isA)[RB], int k, int p, double2 inv,
                                        const double2 (&fj)[(C::NP + 31) / 32], double2 (&row)[RB][(C::NP + 31) / 32],
                                        int lane) {
  constexpr int NQ = (C::NP + 31) / 32;
  double2 xv[RB], ok_[RB];
  int base[RB];
  double* pr[RB];
  double* pi[RB];
#pragma unroll
  for (int u = 0; u < RB; ++u) {
    const int i = rows[u] < 0 ? 0 : rows[u];
    pr[u] = isA[u] ? Ar : Br;
    pi[u] = isA[u] ? Ai : Bi;
    base[u] = i;
    xv[u] = make_double2(pr[u][sw<C::NP>(i, p)], pi[u][sw<C::NP>(i, p)]);
    ok_[u] = make_double2(pr[u][sw<C::NP>(i, k)], pi[u][sw<C::NP>(i, k)]);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int j = (lane + 32 * q) & (C::NP - 1);
      row[u][q] = make_double2(pr[u][sw<C::NP>(i, j)], pi[u][sw<C::NP>(i, j)]);
    }
  }
  __syncwarp();
#pragma unroll
  for (int u = 0; u < RB; ++u) {
    const double2 x = cmul(xv[u], inv);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int j = lane + 32 * q;
      const double2 v = (j == p) ? ok_[u] : row[u][q];
      double2 nv = make_double2(v.x - (fj[q].x * x.x - fj[q].y * x.y), v.y - (fj[q].x * x.y + fj[q].y * x.x));
      nv = (j == k) ? x : nv;
      row[u][q] = nv;
      if (rows[u] >= 0 && j < C::NP) {
        const int o = sw<C::NP>(base[u], j);
        pr[u][o] = nv.x;
        pi[u][o] = nv.y;
      }
    }
  }
}

}  // namespace mbx
