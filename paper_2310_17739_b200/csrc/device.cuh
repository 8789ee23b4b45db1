// Device-side helpers shared by the sm_100a kernels in device.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace nsb {
namespace dev {

// acc += m * x  (complex, four explicit FMAs)
__device__ __forceinline__ void cmac(double2& acc, const double2 m, const double2 x) {
  acc.x = fma(m.x, x.x, acc.x);
  acc.x = fma(-m.y, x.y, acc.x);
  acc.y = fma(m.x, x.y, acc.y);
  acc.y = fma(m.y, x.x, acc.y);
}

__device__ __forceinline__ double2 cmul(const double2 m, const double2 x) {
  double2 r;
  r.x = fma(m.x, x.x, -m.y * x.y);
  r.y = fma(m.x, x.y, m.y * x.x);
  return r;
}

// insert a zero bit at position `pos` of index i
__device__ __forceinline__ uint64_t insert_zero(uint64_t i, int pos) {
  const uint64_t lo = i & ((uint64_t(1) << pos) - 1);
  return ((i >> pos) << (pos + 1)) | lo;
}

// shared-memory slot of tile-local amplitude l: XOR swizzle of the 16-byte
// slot (bits 0..2) with bits 3..11 so strided group accesses spread banks
__device__ __forceinline__ int swz(int l) { return l ^ (((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7); }

}  // namespace dev
}  // namespace nsb
