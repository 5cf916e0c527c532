// Boundary layout conversions between the reference's host storage orders
// (fields.py:48-137, 156-161) and the device layouts documented in
// include/b200wd.h, plus the parity split/merge of oddeven.py:72-95.
#include "capi.cuh"
#include "common.cuh"
#include "layout.cuh"

namespace b200wd {

template <typename C> __device__ __forceinline__ C from_c128(double2 v);
template <> __device__ __forceinline__ double2 from_c128<double2>(double2 v) { return v; }
template <> __device__ __forceinline__ float2 from_c128<float2>(double2 v) {
  return make_float2((float)v.x, (float)v.y);
}
__device__ __forceinline__ double2 to_c128(double2 v) { return v; }
__device__ __forceinline__ double2 to_c128(float2 v) { return make_double2(v.x, v.y); }

// device element i (site-blocked planes, layout.cuh) <-> reference offset
template <typename C, bool IMPORT>
__global__ void spinor_convert_kernel(const void* __restrict__ in, void* __restrict__ out, int layout, int64_t n,
                                      int s, int b) {
  // device storage is padded to a whole number of 8-site blocks; padding
  // sites are written as zeros on import and skipped on export
  const int64_t total = ((n + 7) / 8) * 8 * s * b;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    // i = (((blk * s + k) * 8 + lo) * b + r
    const int r = (int)(i % b);
    int64_t q = i / b;
    const int lo = (int)(q & 7);
    q >>= 3;
    const int k = (int)(q % s);
    const int64_t x = (q / s) * 8 + lo;
    if (x >= n) {
      if (IMPORT) static_cast<C*>(out)[i] = from_c128<C>(make_double2(0.0, 0.0));
      continue;
    }
    const int64_t ref = layout == 1 ? (x * b + r) * s + k : (x * s + k) * b + r;  // fields.py:53-64
    if (IMPORT) {
      static_cast<C*>(out)[i] = from_c128<C>(__ldg(static_cast<const double2*>(in) + ref));
    } else {
      static_cast<double2*>(out)[ref] = to_c128(__ldg(static_cast<const C*>(in) + i));
    }
  }
}

// (n,4,3,3) row-major -> direction-major site-blocked link planes (layout.cuh)
template <typename C>
__global__ void gauge_import_kernel(const double2* __restrict__ in, C* __restrict__ out, int64_t n) {
  const int64_t total = n * 36;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    // i = ((mu * nblk + blk) * 9 + e) * 8 + lo
    const int64_t nblk = n >> 3;
    const int lo = (int)(i & 7);
    int64_t q = i >> 3;
    const int e = (int)(q % 9);
    q /= 9;
    const int64_t blk = q % nblk;
    const int mu = (int)(q / nblk);
    const int64_t x = blk * 8 + lo;
    out[i] = from_c128<C>(__ldg(in + x * 36 + mu * 9 + e));
  }
}

// (n, 2, 21) packed clover blocks -> site-blocked (layout.cuh clover_base)
template <typename C>
__global__ void clover_import_kernel(const double2* __restrict__ in, C* __restrict__ out, int64_t n) {
  const int64_t total = n * 42;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int lo = (int)(i & 7);
    const int64_t q = i >> 3;
    const int e = (int)(q % 42);
    const int64_t x = (q / 42) * 8 + lo;
    out[i] = from_c128<C>(__ldg(in + x * 42 + e));
  }
}

// full <-> parity fields; cb = site >> 1 (oddeven.py:62-65 ordering)
template <typename C, bool SPLIT>
__global__ void parity_kernel(C* __restrict__ full, C* __restrict__ even, C* __restrict__ odd, int64_t n, int s,
                              int b, int X, int Y, int Z, int par0) {
  const int64_t total = n * s * b;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i % b);
    int64_t q = i / b;
    const int lo = (int)(q & 7);
    q >>= 3;
    const int k = (int)(q % s);
    const int64_t site = (q / s) * 8 + lo;
    const int z = (int)(site % Z);
    int64_t c = site / Z;
    const int y = (int)(c % Y);
    c /= Y;
    const int x = (int)(c % X);
    const int t = (int)(c / X);
    const int par = (t + x + y + z + par0) & 1;
    C* half = par ? odd : even;
    const int64_t hi = spinor_elem(site >> 1, k, r, s, b);
    if (SPLIT) half[hi] = full[i];
    else full[i] = half[hi];
  }
}

static dim3 grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return dim3((unsigned)g);
}

}  // namespace b200wd

using namespace b200wd;

extern "C" int b200wd_spinor_import(const void* src_c128, int32_t layout, int64_t n_sites, int32_t s, int32_t b,
                                    void* dst, int32_t dtype, void* stream) {
  B200WD_REQUIRE(layout == 1 || layout == 2, "layout must be 1 (rhs-major) or 2 (component-major), got %d", layout);
  B200WD_REQUIRE(n_sites >= 1 && s >= 1 && b >= 1, "bad field shape n=%lld s=%d b=%d", (long long)n_sites, s, b);
  B200WD_REQUIRE(src_c128 && dst, "NULL pointer");
  const int64_t total = ((n_sites + 7) / 8) * 8 * s * b;
  if (dtype == B200WD_C128)
    spinor_convert_kernel<double2, true><<<grid_for(total), 256, 0, as_stream(stream)>>>(src_c128, dst, layout,
                                                                                          n_sites, s, b);
  else if (dtype == B200WD_C64)
    spinor_convert_kernel<float2, true><<<grid_for(total), 256, 0, as_stream(stream)>>>(src_c128, dst, layout,
                                                                                         n_sites, s, b);
  else
    B200WD_REQUIRE(false, "unknown dtype %d", dtype);
  return check_launch("b200wd_spinor_import");
}

extern "C" int b200wd_spinor_export(const void* src, int32_t dtype, int64_t n_sites, int32_t s, int32_t b,
                                    void* dst_c128, int32_t layout, void* stream) {
  B200WD_REQUIRE(layout == 1 || layout == 2, "layout must be 1 or 2, got %d", layout);
  B200WD_REQUIRE(n_sites >= 1 && s >= 1 && b >= 1, "bad field shape");
  B200WD_REQUIRE(src && dst_c128, "NULL pointer");
  const int64_t total = ((n_sites + 7) / 8) * 8 * s * b;
  if (dtype == B200WD_C128)
    spinor_convert_kernel<double2, false><<<grid_for(total), 256, 0, as_stream(stream)>>>(src, dst_c128, layout,
                                                                                           n_sites, s, b);
  else if (dtype == B200WD_C64)
    spinor_convert_kernel<float2, false><<<grid_for(total), 256, 0, as_stream(stream)>>>(src, dst_c128, layout,
                                                                                          n_sites, s, b);
  else
    B200WD_REQUIRE(false, "unknown dtype %d", dtype);
  return check_launch("b200wd_spinor_export");
}

extern "C" int b200wd_gauge_import(const void* src_c128, int64_t n_sites, void* dst, int32_t dtype, void* stream) {
  B200WD_REQUIRE(n_sites >= 1 && n_sites % 8 == 0 && src_c128 && dst, "bad gauge import arguments (n=%lld)",
                 (long long)n_sites);
  const int64_t total = n_sites * 36;
  if (dtype == B200WD_C128)
    gauge_import_kernel<double2><<<grid_for(total), 256, 0, as_stream(stream)>>>(
        static_cast<const double2*>(src_c128), static_cast<double2*>(dst), n_sites);
  else if (dtype == B200WD_C64)
    gauge_import_kernel<float2><<<grid_for(total), 256, 0, as_stream(stream)>>>(
        static_cast<const double2*>(src_c128), static_cast<float2*>(dst), n_sites);
  else
    B200WD_REQUIRE(false, "unknown dtype %d", dtype);
  return check_launch("b200wd_gauge_import");
}

extern "C" int b200wd_clover_import(const void* src_c128, int64_t n_sites, void* dst, int32_t dtype, void* stream) {
  B200WD_REQUIRE(n_sites >= 8 && n_sites % 8 == 0 && src_c128 && dst, "bad clover import arguments (n=%lld)",
                 (long long)n_sites);
  const int64_t total = n_sites * 42;
  if (dtype == B200WD_C128)
    clover_import_kernel<double2><<<grid_for(total), 256, 0, as_stream(stream)>>>(
        static_cast<const double2*>(src_c128), static_cast<double2*>(dst), n_sites);
  else if (dtype == B200WD_C64)
    clover_import_kernel<float2><<<grid_for(total), 256, 0, as_stream(stream)>>>(
        static_cast<const double2*>(src_c128), static_cast<float2*>(dst), n_sites);
  else
    B200WD_REQUIRE(false, "unknown dtype %d", dtype);
  return check_launch("b200wd_clover_import");
}

static int parity_common(const b200wd_lattice* lat, int32_t dtype, int32_t s, int32_t b, void* full, void* even,
                         void* odd, bool split, void* stream) {
  B200WD_REQUIRE(lat && full && even && odd, "NULL pointer");
  B200WD_REQUIRE(s >= 1 && b >= 1, "bad field shape");
  for (int d = 0; d < 4; ++d) B200WD_REQUIRE(lat->dims[d] >= 2 && lat->dims[d] % 2 == 0, "bad extent");
  const int64_t n = (int64_t)lat->dims[0] * lat->dims[1] * lat->dims[2] * lat->dims[3];
  const int64_t total = n * s * b;
  const int par0 = lat->t_origin & 1;
  cudaStream_t st = as_stream(stream);
  if (dtype == B200WD_C128) {
    auto f = static_cast<double2*>(full);
    auto e = static_cast<double2*>(even);
    auto o = static_cast<double2*>(odd);
    if (split)
      parity_kernel<double2, true><<<grid_for(total), 256, 0, st>>>(f, e, o, n, s, b, lat->dims[1], lat->dims[2],
                                                                    lat->dims[3], par0);
    else
      parity_kernel<double2, false><<<grid_for(total), 256, 0, st>>>(f, e, o, n, s, b, lat->dims[1], lat->dims[2],
                                                                     lat->dims[3], par0);
  } else if (dtype == B200WD_C64) {
    auto f = static_cast<float2*>(full);
    auto e = static_cast<float2*>(even);
    auto o = static_cast<float2*>(odd);
    if (split)
      parity_kernel<float2, true><<<grid_for(total), 256, 0, st>>>(f, e, o, n, s, b, lat->dims[1], lat->dims[2],
                                                                   lat->dims[3], par0);
    else
      parity_kernel<float2, false><<<grid_for(total), 256, 0, st>>>(f, e, o, n, s, b, lat->dims[1], lat->dims[2],
                                                                    lat->dims[3], par0);
  } else {
    B200WD_REQUIRE(false, "unknown dtype %d", dtype);
  }
  return check_launch(split ? "b200wd_parity_split" : "b200wd_parity_merge");
}

extern "C" int b200wd_parity_split(const b200wd_lattice* lat, int32_t dtype, int32_t s, int32_t b, const void* full,
                                   void* even, void* odd, void* stream) {
  return parity_common(lat, dtype, s, b, const_cast<void*>(full), even, odd, true, stream);
}

extern "C" int b200wd_parity_merge(const b200wd_lattice* lat, int32_t dtype, int32_t s, int32_t b, const void* even,
                                   const void* odd, void* full, void* stream) {
  return parity_common(lat, dtype, s, b, full, const_cast<void*>(even), const_cast<void*>(odd), false, stream);
}
