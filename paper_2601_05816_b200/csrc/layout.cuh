// Device storage layouts (see include/b200wd.h).
//
// Spinor block field with s components, n sites (n % 8 == 0), b rhs:
//   element (site, k, r) at  (((site >> 3) * s + k) * 8 + (site & 7)) * b + r
// i.e. blocks of 8 sites; inside a block, component k of the 8 sites is one
// contiguous run of 8*b complex numbers ("site-blocked component planes").
// rhs is innermost, a warp's load of one component over consecutive
// (site, rhs) pairs is contiguous and line-aligned for every b, and the
// distance between the components of one site is the compile-time constant
// 8*b, so the 12 loads of a neighbour spinor are one address + immediates.
//
// Links, 4 directions x 9 entries per site:
//   element (site, mu, e) at  ((site >> 3) * 36 + mu * 9 + e) * 8 + (site & 7)
#pragma once
#include <stdint.h>

namespace b200wd {

constexpr int kSiteBlock = 8;

__host__ __device__ __forceinline__ int64_t spinor_elem(int64_t site, int k, int r, int s, int b) {
  return ((((site >> 3) * s + k) << 3) + (site & 7)) * (int64_t)b + r;
}
// element of (site, k=0, r=0)
__host__ __device__ __forceinline__ int64_t spinor_base(int64_t site, int s, int b) {
  return (((site >> 3) * s * 8) + (site & 7)) * (int64_t)b;
}
__host__ __device__ __forceinline__ int64_t link_base(int64_t site) { return (site >> 3) * 288 + (site & 7); }

}  // namespace b200wd
