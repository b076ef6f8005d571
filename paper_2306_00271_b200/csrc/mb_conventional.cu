// K5: the conventional multi-slice method on the device (
// reference conventional.cpp:9-78 with kernels.cpp:25-80). It is the method
// the paper replaces and serves as the cross-method check of the stepper path
// (acceptance.cpp:164-178: conventional vs sp6 within 1e-8).
//
// Per (structure, angle) pair, one CTA walks the L slices in order:
//   A = h * [[UG + iG, UG], [-UG, -UG - iG]],  UG = (i/2) U(z_mid) G^-1
//       (slice_coefficient, conventional.cpp:9-22; U gathered from the boxed
//        K1 table at the slice midpoint);
//   E = exp(A)  (Pade-13 scaling and squaring, kernels.cpp:25-58: 1-norm
//       scaling power, A2/A4/A6, U/V polynomials, (V-U) X = (V+U) by
//       partial-pivoting LU, s squarings);
//   R <- (Z + W R)(X + Y R)^-1  (reflect_update, conventional.cpp:35-37, by
//       solve_right: LU of the transpose with partial pivoting, zero-pivot
//       check, residual gate 1e-10, kernels.cpp:60-80).
// Then rho = R[:, 0] and the intensities (curve.cpp:8-20). Breakdown is
// reported with the slice index (conventional.cpp:67-74).
//
// Sizes: 2N <= 64 (N <= 32). Matrices are row-major complex (double2) in a
// per-CTA global scratch (L2-resident); GEMM operands and the LU work matrix
// are staged in shared memory. Arithmetic is plain FP64 (DFMA): this path is
// a correctness cross-check, not the hot path.
#include <cuda_runtime.h>

#include "mb_device.cuh"
#include "mb_internal.h"

namespace mbx {
namespace {

constexpr int KNT = 256;   // threads per CTA
constexpr int KMAX = 64;   // 2N bound
constexpr int KSZ = KMAX * KMAX;

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double cabs2(double2 a) { return hypot(a.x, a.y); }
// Eigen SSE pdiv: a * conj(b) / |b|^2
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double s = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / s, (a.y * b.x - a.x * b.y) / s);
}
__device__ __forceinline__ bool cfinite(double2 a) { return isfinite(a.x) && isfinite(a.y); }

// C[m x n] = A[m x k] B[k x n], all row-major with leading dimension KMAX,
// k-sum in order 0..k-1; operands staged in shared memory (sa, sb)
__device__ void cta_gemm(double2* C, const double2* A, const double2* B, int m, int n, int k, double2* sa,
                         double2* sb) {
  for (int w = threadIdx.x; w < m * k; w += KNT) sa[(w / k) * KMAX + w % k] = A[(w / k) * KMAX + w % k];
  for (int w = threadIdx.x; w < k * n; w += KNT) sb[(w / n) * KMAX + w % n] = B[(w / n) * KMAX + w % n];
  __syncthreads();
  for (int w = threadIdx.x; w < m * n; w += KNT) {
    const int i = w / n, j = w % n;
    double re = 0.0, im = 0.0;
    for (int q = 0; q < k; ++q) {
      const double2 a = sa[i * KMAX + q], b = sb[q * KMAX + j];
      re += a.x * b.x - a.y * b.y;
      im += a.x * b.y + a.y * b.x;
    }
    C[i * KMAX + j] = make_double2(re, im);
  }
  __syncthreads();
}

struct LuScratch {
  int piv[KMAX];
  double best[KNT / 32];
  int bidx[KNT / 32];
  int zero;
};

// In-place partial-pivoting LU of the m x m matrix `a` (shared memory), as
// Eigen's PartialPivLU unblocked_lu: pivot = first max |a_ik| over i >= k,
// row swap, column scaled by the pivot, rank-1 update. piv[k] = swapped row.
// Sets ls.zero when a pivot is exactly zero (kernels.cpp:68-71).
__device__ void cta_lu(double2* a, int m, LuScratch& ls) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) ls.zero = 0;
  __syncthreads();
  for (int k = 0; k < m; ++k) {
    // first maximum of |a_ik|, i >= k (warp 0: m <= 64)
    if (warp == 0) {
      double bv = -1.0;
      int bi = m;
      for (int i = k + lane; i < m; i += 32) {
        const double v = cabs2(a[i * KMAX + k]);
        if (v > bv) {
          bv = v;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        ls.piv[k] = bi;
        ls.best[0] = bv;
        if (!(bv != 0.0) && !ls.zero) ls.zero = 1;
      }
    }
    __syncthreads();
    const int p = ls.piv[k];
    const bool nz = ls.best[0] != 0.0;
    if (nz && p != k)
      for (int j = tid; j < m; j += KNT) {
        const double2 t = a[k * KMAX + j];
        a[k * KMAX + j] = a[p * KMAX + j];
        a[p * KMAX + j] = t;
      }
    __syncthreads();
    if (nz) {
      const double2 pv = a[k * KMAX + k];
      for (int i = k + 1 + tid; i < m; i += KNT) a[i * KMAX + k] = cdiv(a[i * KMAX + k], pv);
    }
    __syncthreads();
    const int r = m - k - 1;
    for (int w = tid; w < r * r; w += KNT) {
      const int i = k + 1 + w / r, j = k + 1 + w % r;
      const double2 l = a[i * KMAX + k], u = a[k * KMAX + j], v = a[i * KMAX + j];
      a[i * KMAX + j] = make_double2(v.x - (l.x * u.x - l.y * u.y), v.y - (l.x * u.y + l.y * u.x));
    }
    __syncthreads();
  }
}

// b (m x ncol, shared memory) <- LU^-1 P b: row permutation, unit-lower
// forward and upper back substitution; columns in parallel
__device__ void cta_lu_solve(const double2* a, const LuScratch& ls, double2* b, int m, int ncol) {
  for (int k = 0; k < m; ++k) {
    const int p = ls.piv[k];
    if (p != k && p < m)
      for (int j = threadIdx.x; j < ncol; j += KNT) {
        const double2 t = b[k * KMAX + j];
        b[k * KMAX + j] = b[p * KMAX + j];
        b[p * KMAX + j] = t;
      }
    __syncthreads();
  }
  for (int j = threadIdx.x; j < ncol; j += KNT) {
    for (int i = 0; i < m; ++i) {
      double2 s = b[i * KMAX + j];
      for (int q = 0; q < i; ++q) {
        const double2 l = a[i * KMAX + q], x = b[q * KMAX + j];
        s = make_double2(s.x - (l.x * x.x - l.y * x.y), s.y - (l.x * x.y + l.y * x.x));
      }
      b[i * KMAX + j] = s;
    }
    for (int i = m - 1; i >= 0; --i) {
      double2 s = b[i * KMAX + j];
      for (int q = i + 1; q < m; ++q) {
        const double2 u = a[i * KMAX + q], x = b[q * KMAX + j];
        s = make_double2(s.x - (u.x * x.x - u.y * x.y), s.y - (u.x * x.y + u.y * x.x));
      }
      b[i * KMAX + j] = cdiv(s, a[i * KMAX + i]);
    }
  }
  __syncthreads();
}

__device__ double cta_reduce_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < KNT / 32; ++w) s += red[w];
  __syncthreads();
  return s;
}

__device__ double cta_reduce_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < KNT / 32; ++w) s = fmax(s, red[w]);
  __syncthreads();
  return s;
}

// Pade(13,13) coefficients and the unscaled 1-norm bound (kernels.cpp:11-22)
__constant__ double kPade13[14] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                                   1187353796428800.0,  129060195264000.0,   10559470521600.0,
                                   670442572800.0,      33522128640.0,       1323241920.0,
                                   40840800.0,          960960.0,            16380.0,
                                   182.0,               1.0};
constexpr double kTheta13 = 5.371920351148152;

struct ConvSmem {
  double2 sa[KSZ];
  double2 sb[KSZ];
  LuScratch ls;
  double red[KNT / 32];
  int flag;
};

__global__ void __launch_bounds__(KNT, 1) conventional_kernel(const __grid_constant__ PropagateParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ConvSmem& S = *reinterpret_cast<ConvSmem*>(smem_raw);
  const int n = p.n, m2 = 2 * n, tid = threadIdx.x;
  // per-CTA scratch: A, A2, A4, A6, U, V, T (2N x 2N each), R, R2 (N x N in the same stride)
  double2* W = reinterpret_cast<double2*>(p.scratch) + (long)blockIdx.x * 9 * KSZ;
  double2 *Am = W, *A2 = W + KSZ, *A4 = W + 2 * KSZ, *A6 = W + 3 * KSZ, *Um = W + 4 * KSZ, *Vm = W + 5 * KSZ,
          *Tm = W + 6 * KSZ, *Rm = W + 7 * KSZ, *Bm = W + 8 * KSZ;
  for (long pair = blockIdx.x; pair < p.npairs; pair += gridDim.x) {
    const double2* coef = p.coef + (long)p.pair_struct[pair] * p.nslots * p.box_size;
    const double2* gd = p.gdiag + pair * n;
    const double2* gi = p.ginv + pair * n;
    for (int w = tid; w < n * n; w += KNT) Rm[(w / n) * KMAX + w % n] = make_double2(0.0, 0.0);  // seed_or_zero
    int code = 0, fail_step = 0;
    for (int step = 0; step < p.nsteps && !code; ++step) {
      // ---- A = h * slice_coefficient(U_mid, G)
      const double2* box = coef + (long)step * p.slot_stride * p.box_size;
      const double h = p.h;
      for (int w = tid; w < m2 * m2; w += KNT) {
        const int r = w / m2, c = w % m2, j = r % n, k = c % n;
        const double2 u = box[p.box_center + p.rowoff[j] - p.rowoff[k]];
        const double2 ug0 = cmul(u, gi[k]);                          // U * G^-1 (column scaling)
        const double2 ug = make_double2(-0.5 * ug0.y, 0.5 * ug0.x);  // (i/2) (.)
        double2 v;
        if (r < n && c < n) {
          v = ug;
          if (j == k) v = cadd(v, make_double2(-gd[j].y, gd[j].x));  // + i G
        } else if (r < n) {
          v = ug;
        } else if (c < n) {
          v = make_double2(-ug.x, -ug.y);
        } else {
          v = make_double2(-ug.x, -ug.y);
          if (j == k) v = csub(v, make_double2(-gd[j].y, gd[j].x));  // - i G
        }
        Am[r * KMAX + c] = cscale(h, v);
      }
      __syncthreads();
      // ---- matrix_exponential (kernels.cpp:25-58)
      double colmax = 0.0;
      for (int c = tid; c < m2; c += KNT) {
        double sum = 0.0;
        for (int r = 0; r < m2; ++r) sum += cabs2(Am[r * KMAX + c]);
        colmax = fmax(colmax, sum);
      }
      const double norm1 = cta_reduce_max(colmax, S.red);
      int sq = 0;
      if (norm1 > kTheta13) sq = (int)ceil(log2(norm1 / kTheta13));
      const double scl = exp2(-(double)sq);
      for (int w = tid; w < m2 * m2; w += KNT) Am[(w / m2) * KMAX + w % m2] = cscale(scl, Am[(w / m2) * KMAX + w % m2]);
      __syncthreads();
      cta_gemm(A2, Am, Am, m2, m2, m2, S.sa, S.sb);
      cta_gemm(A4, A2, A2, m2, m2, m2, S.sa, S.sb);
      cta_gemm(A6, A4, A2, m2, m2, m2, S.sa, S.sb);
      for (int w = tid; w < m2 * m2; w += KNT) {  // T = b13 A6 + b11 A4 + b9 A2
        const int o = (w / m2) * KMAX + w % m2;
        Tm[o] = cadd(cadd(cscale(kPade13[13], A6[o]), cscale(kPade13[11], A4[o])), cscale(kPade13[9], A2[o]));
      }
      __syncthreads();
      cta_gemm(Um, A6, Tm, m2, m2, m2, S.sa, S.sb);
      for (int w = tid; w < m2 * m2; w += KNT) {  // U += b7 A6 + b5 A4 + b3 A2 + b1 I
        const int r = w / m2, c = w % m2, o = r * KMAX + c;
        double2 t = cadd(cadd(cscale(kPade13[7], A6[o]), cscale(kPade13[5], A4[o])), cscale(kPade13[3], A2[o]));
        t = cadd(t, make_double2(r == c ? kPade13[1] : 0.0, 0.0));
        Um[o] = cadd(Um[o], t);
      }
      __syncthreads();
      cta_gemm(Tm, Am, Um, m2, m2, m2, S.sa, S.sb);  // U = A U  (into T)
      for (int w = tid; w < m2 * m2; w += KNT) {     // U <- T; T = b12 A6 + b10 A4 + b8 A2
        const int o = (w / m2) * KMAX + w % m2;
        Um[o] = Tm[o];
        Tm[o] = cadd(cadd(cscale(kPade13[12], A6[o]), cscale(kPade13[10], A4[o])), cscale(kPade13[8], A2[o]));
      }
      __syncthreads();
      cta_gemm(Vm, A6, Tm, m2, m2, m2, S.sa, S.sb);
      for (int w = tid; w < m2 * m2; w += KNT) {  // V += b6 A6 + b4 A4 + b2 A2 + b0 I
        const int r = w / m2, c = w % m2, o = r * KMAX + c;
        double2 t = cadd(cadd(cscale(kPade13[6], A6[o]), cscale(kPade13[4], A4[o])), cscale(kPade13[2], A2[o]));
        t = cadd(t, make_double2(r == c ? kPade13[0] : 0.0, 0.0));
        Vm[o] = cadd(Vm[o], t);
      }
      __syncthreads();
      // (V - U) E = (V + U)
      for (int w = tid; w < m2 * m2; w += KNT) {
        const int o = (w / m2) * KMAX + w % m2;
        S.sa[o] = csub(Vm[o], Um[o]);
        S.sb[o] = cadd(Vm[o], Um[o]);
      }
      __syncthreads();
      cta_lu(S.sa, m2, S.ls);
      cta_lu_solve(S.sa, S.ls, S.sb, m2, m2);
      for (int w = tid; w < m2 * m2; w += KNT) Am[(w / m2) * KMAX + w % m2] = S.sb[(w / m2) * KMAX + w % m2];
      __syncthreads();
      for (int s = 0; s < sq; ++s) {  // R = R * R
        cta_gemm(Tm, Am, Am, m2, m2, m2, S.sa, S.sb);
        for (int w = tid; w < m2 * m2; w += KNT) Am[(w / m2) * KMAX + w % m2] = Tm[(w / m2) * KMAX + w % m2];
        __syncthreads();
      }
      // E blocks: X = E[0:n,0:n], Y = E[0:n,n:], Z = E[n:,0:n], W = E[n:,n:]
      // ---- reflect_update: R <- solve_right(Z + W R, X + Y R)
      cta_gemm(Tm, Am + n * KMAX + n, Rm, n, n, n, S.sa, S.sb);  // W R
      cta_gemm(Um, Am + n, Rm, n, n, n, S.sa, S.sb);             // Y R
      for (int w = tid; w < n * n; w += KNT) {
        const int r = w / n, c = w % n, o = r * KMAX + c;
        Bm[o] = cadd(Am[(n + r) * KMAX + c], Tm[o]);  // B = Z + W R
        Vm[o] = cadd(Am[o], Um[o]);                   // A' = X + Y R
      }
      __syncthreads();
      // X A' = B  <=>  A'^T X^T = B^T (kernels.cpp:66-72)
      for (int w = tid; w < n * n; w += KNT) {
        const int r = w / n, c = w % n;
        S.sa[c * KMAX + r] = Vm[r * KMAX + c];
        S.sb[c * KMAX + r] = Bm[r * KMAX + c];
      }
      if (tid == 0) S.flag = 0;
      __syncthreads();
      cta_lu(S.sa, n, S.ls);
      bool singular = S.ls.zero != 0;
      for (int i = tid; i < n; i += KNT)
        if (S.sa[i * KMAX + i].x == 0.0 && S.sa[i * KMAX + i].y == 0.0) S.flag = 1;
      __syncthreads();
      singular = singular || S.flag;
      if (!singular) {
        cta_lu_solve(S.sa, S.ls, S.sb, n, n);
        for (int w = tid; w < n * n; w += KNT) {  // X = (X^T)^T -> T
          const int r = w / n, c = w % n;
          Tm[r * KMAX + c] = S.sb[c * KMAX + r];
        }
        __syncthreads();
        // residual gate ||X A' - B||_F / ||B||_F <= 1e-10 and X finite
        cta_gemm(Um, Tm, Vm, n, n, n, S.sa, S.sb);
        double rn = 0.0, bn = 0.0, bad = 0.0;
        for (int w = tid; w < n * n; w += KNT) {
          const int o = (w / n) * KMAX + w % n;
          const double2 d = csub(Um[o], Bm[o]);
          rn += d.x * d.x + d.y * d.y;
          bn += Bm[o].x * Bm[o].x + Bm[o].y * Bm[o].y;
          if (!cfinite(Tm[o])) bad = 1.0;
        }
        rn = cta_reduce_sum(rn, S.red);
        bn = cta_reduce_sum(bn, S.red);
        bad = cta_reduce_max(bad, S.red);
        const double bnorm = sqrt(bn);
        const double resid = sqrt(rn) / (bnorm > 0.0 ? bnorm : 1.0);
        if (p.residual_check && !(resid <= 1e-10)) singular = true;
        if (bad > 0.0) singular = true;
      }
      if (singular) {
        code = MB_POINT_RECURSION_CODE;
        fail_step = step;
        break;
      }
      double nonfinite = 0.0;
      for (int w = tid; w < n * n; w += KNT) {
        const int o = (w / n) * KMAX + w % n;
        Rm[o] = Tm[o];
        if (!cfinite(Tm[o])) nonfinite = 1.0;
      }
      nonfinite = cta_reduce_max(nonfinite, S.red);
      if (nonfinite > 0.0) {
        code = MB_POINT_RECURSION_CODE;
        fail_step = step;
      }
      __syncthreads();
    }
    // rho = R[:, 0]; eta (curve.cpp:8-20)
    if (!code) {
      const double g0 = p.gdiag[pair * n].x, s0 = p.sin_theta0[pair];
      for (int i = tid; i < n; i += KNT) {
        const double2 r = Rm[i * KMAX];
        p.rho[pair * n + i] = r;
        const double2 gdi = p.gdiag[pair * n + i];
        p.eta[pair * n + i] = p.gamma2[pair * n + i] > 0.0 ? (r.x * r.x + r.y * r.y) * s0 * g0 / gdi.x : 0.0;
      }
    }
    if (tid == 0) {
      PointStatus st;
      st.code = code;
      st.step = fail_step;
      st.rhst = 0;
      st.reserved = 0;
      p.status[pair] = st;
    }
    __syncthreads();
  }
}

}  // namespace

size_t conventional_scratch_doubles(long ctas) { return (size_t)ctas * 9 * KSZ * 2; }

long conventional_ctas(long npairs) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return npairs < sms ? npairs : sms;
}

cudaError_t launch_conventional(const PropagateParams& p, long ctas, cudaStream_t st, int* launches) {
  if (2 * p.n > KMAX) return cudaErrorInvalidValue;
  const size_t smem = sizeof(ConvSmem);
  cudaError_t e = cudaFuncSetAttribute(conventional_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  conventional_kernel<<<(unsigned)ctas, KNT, smem, st>>>(p);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace mbx
