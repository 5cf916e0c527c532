// complex128 instantiations of the hopping kernels (split out for parallel builds)
#include "dirac_kernels.cuh"

namespace b200wd {
void launch_hop_c128(const HopParams& p, cudaStream_t st) { launch_hop<double, 1>(p, st); }
void launch_pack_c128(const HopParams& p, void* lam, void* chi, cudaStream_t st) {
  launch_pack<double, 1>(p, lam, chi, st);
}
void launch_clover_apply_c128(int64_t n, int b, const void* M, const void* x, void* out, cudaStream_t st) {
  const int64_t total = n * b;
  clover_apply_kernel<double><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
      n, b, static_cast<const cx<double>*>(M), static_cast<const cx<double>*>(x), static_cast<cx<double>*>(out));
}
}  // namespace b200wd
