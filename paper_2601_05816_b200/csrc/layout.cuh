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
// Links, 4 directions x 9 entries per site, direction-major:
//   element (site, mu, e) at  ((mu * nblk + (site >> 3)) * 9 + e) * 8 + (site & 7),  nblk = n / 8
// so one direction's links of consecutive site blocks are one contiguous run
// (a single bulk copy per hop tile, whatever the number of blocks).
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
// element of (site, mu, e=0); entry e is at +8*e
__host__ __device__ __forceinline__ int64_t link_base(int64_t site, int mu, int64_t nblk) {
  return (mu * nblk + (site >> 3)) * 72 + (site & 7);
}

// Site-local clover blocks: 2 x 21 packed complex per site,
//   element (site, q) at ((site >> 3) * 42 + q) * 8 + (site & 7),  q = 21*block + idx
__host__ __device__ __forceinline__ int64_t clover_base(int64_t site) { return (site >> 3) * 336 + (site & 7); }

}  // namespace b200wd
