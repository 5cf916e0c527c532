// complex128 instantiations of the hopping kernels (split out for parallel builds)
#include "dirac_kernels.cuh"

namespace b200wd {
void launch_hop_c128(const HopParams& p, cudaStream_t st) { launch_hop<double, 1>(p, st); }
void launch_pack_c128(const HopParams& p, void* lam, void* chi, cudaStream_t st) {
  launch_pack<double, 1>(p, lam, chi, st);
}
}  // namespace b200wd
