// K2c host side: variant choice (cluster vs cooperative groups), shared-memory
// sizing and launch of the cluster-resident propagation kernel (mb_cluster.cuh).
#include "mb_cluster.cuh"

namespace mbx {

cudaError_t cluster_dispatch_128(const PropagateParams& p, cudaStream_t st, int mode, int* groups_out);
cudaError_t cluster_dispatch_256(const PropagateParams& p, cudaStream_t st, int mode, int* groups_out);

// slab width per padded size: NP=256 -> 16 columns (CS <= 16); NP=128 -> 32
// for splitting (CS <= 4), 16 for rk4 (its third slab plane does not fit at 32)
static int cluster_sw(int np, int rk4) { return np == 128 && !rk4 ? MB_SW128 : 16; }

size_t cluster_smem_bytes(int n, int rk4, int box_size, int ndiff) {
  if (n <= 64 || n > 256) return 0;
  const int np = n <= 128 ? 128 : 256;
  return cluster_layout(np, cluster_sw(np, rk4), rk4 ? 3 : 2, box_size, ndiff).total;
}

int cluster_np(int n) { return n <= 64 || n > 256 ? 0 : (n <= 128 ? 128 : 256); }

// mode 0: one thread-block cluster per pair; 1: cooperative groups.
// groups_out != nullptr: only report how many groups run concurrently
// (the instantiations live in mb_cluster_128.cu / mb_cluster_256.cu so they
// compile in parallel)
static cudaError_t dispatch(const PropagateParams& p, cudaStream_t st, int mode, int* groups_out) {
  return p.n <= 128 ? cluster_dispatch_128(p, st, mode, groups_out) : cluster_dispatch_256(p, st, mode, groups_out);
}

int cluster_prefer_coop(const PropagateParams& p) {
  int gcl = 0, gco = 0;
  PropagateParams q = p;
  q.coop_bar = nullptr;
  if (dispatch(q, nullptr, 0, &gcl) != cudaSuccess) gcl = 0;
  if (dispatch(q, nullptr, 1, &gco) != cudaSuccess) gco = 0;
  cudaGetLastError();
  if (gco <= 0) return 0;
  if (gcl <= 0) return 1;
  const long rcl = (p.npairs + gcl - 1) / gcl, rco = (p.npairs + gco - 1) / gco;
  return rco < rcl ? 1 : 0;
}

cudaError_t launch_cluster(const PropagateParams& p, cudaStream_t st, int* launches) {
  const cudaError_t e = dispatch(p, st, p.coop ? 1 : 0, nullptr);
  if (e == cudaSuccess) ++*launches;
  return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace mbx
