// Device helpers shared by the sm_100a kernels (mb_kernels.cu, mb_large.cu).
#pragma once

#include <cuda_runtime.h>

namespace mbx {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double dneg(double x) {
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)0x8000000000000000ULL);
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier.
// Stages one node's coefficient box (box_size x 16 B, holes already zero in
// the boxed table) into shared memory in a single transaction.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make initialised mbarriers visible to the async proxy (and the cluster)
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// global -> own shared memory, bytes % 16 == 0, both addresses 16-B aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// global -> the same shared offset in every CTA of ctamask (cluster launch
// only); completes on the mbarrier at the same offset in each of them
__device__ __forceinline__ void bulk_g2s_multicast(void* dst, const void* src, unsigned bytes,
                                                   unsigned long long* bar, unsigned short ctamask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
      "%4;\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(ctamask)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// arrive on the mbarrier at the same shared offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(unsigned long long* bar, unsigned rank) {
  asm volatile(
      "{\n .reg .b32 ra;\n"
      " mapa.shared::cluster.u32 ra, %0, %1;\n"
      " mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}
// wait on a cluster-scope phase (remote arrivals with release.cluster)
__device__ __forceinline__ void mbar_wait_cluster(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAITC_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Splitting kick / drift with the reference's rounding (proposed.cpp:133-137,
// 180-193): apply_w forms out = U X, then out += G^2 X (product, then sum),
// then P -= (h b) out; a drift is Q += (h a) P. Each operation rounds once,
// as the reference's Eigen expressions do on x86-64 without FMA; the _rn
// intrinsics are never contracted into FMAs. The conditioning of deep slabs
// (cfg3) amplifies a contracted epilogue's different rounding to ~5e-8 in eta.
__device__ __forceinline__ double w_ref(double uq, double g2, double q) { return __dadd_rn(uq, __dmul_rn(g2, q)); }
__device__ __forceinline__ double sub_ref(double p, double c, double w) { return __dsub_rn(p, __dmul_rn(c, w)); }
__device__ __forceinline__ double kick_ref(double p, double c, double uq, double g2, double q) {
  return sub_ref(p, c, w_ref(uq, g2, q));
}
__device__ __forceinline__ double drift_ref(double q, double c, double p) { return __dadd_rn(q, __dmul_rn(c, p)); }
// to_tau_rho (proposed.cpp:108-113) with the reference's rounding:
// G Q (complex product, two rounded products and one rounded sum per part),
// T = G Q - i P, R = G Q + i P (i P = (-pi, pr) exactly).
__device__ __forceinline__ void tau_rho_ref(double2 g, double qr, double qi, double pr, double pi, double& tr,
                                            double& ti, double& rr, double& ri) {
  const double gqr = __dsub_rn(__dmul_rn(g.x, qr), __dmul_rn(g.y, qi));
  const double gqi = __dadd_rn(__dmul_rn(g.x, qi), __dmul_rn(g.y, qr));
  tr = __dadd_rn(gqr, pi);
  ti = __dsub_rn(gqi, pr);
  rr = __dsub_rn(gqr, pi);
  ri = __dadd_rn(gqi, pr);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// complex helpers on (re, im) pairs
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cinv(double2 a) {  // 1/a with scaling (Smith)
  if (fabs(a.x) >= fabs(a.y)) {
    const double r = a.y / a.x, d = a.x + a.y * r;
    return make_double2(1.0 / d, -r / d);
  }
  const double r = a.x / a.y, d = a.y + a.x * r;
  return make_double2(r / d, -1.0 / d);
}


}  // namespace mbx
