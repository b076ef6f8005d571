// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64 -> DMMA.8x8x4)
// and DFMA throughput at several warps/SM. Output: one JSON line per case plus a
// summary line. Used to fill the FP64 roofline denominator (MEASURED_PEAKS.json
// has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int j = 0; j < CHAINS; j++) { c[j][0] = 0; c[j][1] = 0; }
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < CHAINS; j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; j++) s += c[j][0] + c[j][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[CHAINS];
#pragma unroll
  for (int j = 0; j < CHAINS; j++) c[j] = j * 1e-3;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < CHAINS; j++) c[j] = fma(c[j], b, a);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; j++) s += c[j];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\":\"%s\",\"sms\":%d,\"smem_optin\":%zu,\"smem_per_sm\":%zu,\"regs_per_sm\":%d,\"clock_khz\":%d,\"l2\":%d}\n",
         p.name, p.multiProcessorCount, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor,
         p.regsPerMultiprocessor, clk, p.l2CacheSize);
  double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  double best_dmma = 0, best_dfma = 0;
  for (int warps : {4, 8, 16, 32}) {
    for (int rep = 0; rep < 2; rep++) {
      const int iters = 20000;
      // DMMA: 8 chains x 512 flop per warp-instruction
      dmma_loop<8><<<sms * 2, warps * 32 / 2>>>(out, 100); // warm
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_loop<8><<<sms * 2, warps * 32 / 2>>>(out, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = (double)sms * 2 * (warps / 2) * iters * 8 * 512.0;
      double tf = fl / (ms * 1e-3) / 1e12;
      if (tf > best_dmma) best_dmma = tf;
      printf("{\"case\":\"dmma\",\"warps_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", warps, ms, tf);
      // DFMA: 8 chains x 2 flop x 32 lanes per warp-instruction
      dfma_loop<8><<<sms * 2, warps * 32 / 2>>>(out, 100);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_loop<8><<<sms * 2, warps * 32 / 2>>>(out, iters * 4);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      fl = (double)sms * 2 * (warps / 2) * 32 * iters * 4 * 8 * 2.0;
      tf = fl / (ms * 1e-3) / 1e12;
      if (tf > best_dfma) best_dfma = tf;
      printf("{\"case\":\"dfma\",\"warps_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.2f}\n", warps, ms, tf);
    }
  }
  printf("{\"summary\":true,\"fp64_dmma_tflops\":%.2f,\"fp64_dfma_tflops\":%.2f}\n", best_dmma, best_dfma);
  return 0;
}
