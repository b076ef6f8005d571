// K2c instantiations for NP = 256 (see mb_cluster.cuh).
#include "mb_cluster.cuh"

namespace mbx {

cudaError_t cluster_dispatch_256(const PropagateParams& p, cudaStream_t st, int mode, int* groups_out) {
  const int cs = (p.n + 15) / 16;
  return p.rk4 ? launch_cfg<CCfg<256, 16>, true>(p, st, cs, mode, groups_out)
               : launch_cfg<CCfg<256, 16>, false>(p, st, cs, mode, groups_out);
}

}  // namespace mbx
