// K2c instantiations for NP = 128 (see mb_cluster.cuh).
#include "mb_cluster.cuh"

namespace mbx {

cudaError_t cluster_dispatch_128(const PropagateParams& p, cudaStream_t st, int mode, int* groups_out) {
  constexpr int S = MB_SW128;
  return p.rk4 ? launch_cfg<CCfg<128, 16>, true>(p, st, (p.n + 15) / 16, mode, groups_out)
               : launch_cfg<CCfg<128, S>, false>(p, st, (p.n + S - 1) / S, mode, groups_out);
}

}  // namespace mbx
