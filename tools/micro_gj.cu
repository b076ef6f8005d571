// Microbenchmark (tools only): cycles of the Gauss-Jordan pivot search
// gj_pivot<C> (mb_tiles.cuh) at NP = 256 for one warp, in a dependent chain
// (each step's row depends on the previous pivot), as in the panel
// factorisation of the cluster kernel. Also times the pieces.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../paper_2306_00271_b200/csrc micro_gj.cu -o micro_gj
#include <cstdio>

#include "mb_tiles.cuh"

using namespace mbx;

struct C256 {
  static constexpr int NP = 256;
};

template <int MODE>
__global__ void k(double2* out, long long* cyc, int n, int steps) {
  __shared__ double2 fv[2 * 256];
  __shared__ Scratch sc;
  const int lane = threadIdx.x & 31;
  constexpr int NQ = 8;
  double2 a[NQ];
  for (int q = 0; q < NQ; ++q) a[q] = make_double2(1.0 + 0.01 * (lane + 32 * q), 0.5 - 0.003 * q);
  __syncwarp();
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    const int kk = s % 128;
    if (MODE == 0) {
      gj_pivot<C256>(a, kk, n, fv + (s & 1) * 256, sc, s & 1, lane);
    } else if (MODE == 1) {  // lane-local max + warp reduction only
      double best = -1.0;
      int bj = n;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int j = lane + 32 * q;
        const double v = a[q].x * a[q].x + a[q].y * a[q].y;
        if (j >= kk && j < n && v > best) {
          best = v;
          bj = j;
        }
      }
      const unsigned key = best < 0.0 ? 0u : __float_as_uint(__double2float_ru(best)) + 1u;
      const unsigned km = __reduce_max_sync(0xffffffffu, key);
      const unsigned tied = __ballot_sync(0xffffffffu, key == km);
      const int src = __ffs(tied) - 1;
      bj = __shfl_sync(0xffffffffu, bj, src);
      if (lane == 0) sc.piv[s & 1] = bj;
    } else {  // reciprocal only
      if (lane == 0) {
        double r;
        const double b = a[0].x + 1.0;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
        r = r * fma(-b, r, 2.0);
        r = r * fma(-b, r, 2.0);
        sc.inv[s & 1] = make_double2(r, r);
      }
    }
    __syncwarp();
    // make the next row depend on this step's result
    const int p = sc.piv[s & 1] & 255;
    const double2 iv = sc.inv[s & 1];
#pragma unroll
    for (int q = 0; q < NQ; ++q) a[q].x += 1e-9 * (double)((p + q) & 7) + 0.0 * iv.x;
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x] = (t1 - t0) / steps;
  out[threadIdx.x] = a[0];
}

int main() {
  double2* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double2));
  cudaMalloc(&cyc, 64 * sizeof(long long));
  long long h[1];
  const char* names[3] = {"gj_pivot (full)", "local max + CREDUX + pick", "rcp + 2 Newton"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<1, 32>>>(out, cyc, 199, 4096);
      if (mode == 1) k<1><<<1, 32>>>(out, cyc, 199, 4096);
      if (mode == 2) k<2><<<1, 32>>>(out, cyc, 199, 4096);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    printf("%-28s %lld cycles/step\n", names[mode], h[0]);
  }
  return 0;
}
