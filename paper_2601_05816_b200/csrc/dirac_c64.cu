// complex64 instantiations of the hopping kernels (2 rhs per thread, 128-bit
// loads, when the rhs count is even)
#include "dirac_kernels.cuh"

namespace b200wd {
void launch_hop_c64(const HopParams& p, cudaStream_t st) {
  if (p.b % 2 == 0) launch_hop<float, 2>(p, st);
  else launch_hop<float, 1>(p, st);
}
void launch_pack_c64(const HopParams& p, void* lam, void* chi, cudaStream_t st) {
  if (p.b % 2 == 0) launch_pack<float, 2>(p, lam, chi, st);
  else launch_pack<float, 1>(p, lam, chi, st);
}
void launch_clover_apply_c64(int64_t n, int b, const void* M, const void* x, void* out, cudaStream_t st) {
  const int64_t total = n * b;
  clover_apply_kernel<float><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
      n, b, static_cast<const cx<float>*>(M), static_cast<const cx<float>*>(x), static_cast<cx<float>*>(out));
}
}  // namespace b200wd
