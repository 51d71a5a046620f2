// Row-access helpers shared by the row kernels (fc_rows.cu, fc_backward.cu).
#pragma once

#include "fc_internal.cuh"

namespace fc {

// 16-byte units of a row; lg = log2(upr) when upr is a power of two
struct Units {
  int upr;
  int lg;
  __device__ __forceinline__ int row(int u) const { return lg >= 0 ? (u >> lg) : (u / upr); }
};

inline Units units_for(int width) {
  Units un;
  un.upr = width / 4 > 0 ? width / 4 : 1;
  un.lg = (un.upr & (un.upr - 1)) == 0 ? __builtin_ctz(un.upr) : -1;
  return un;
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

template <bool VEC>
__device__ __forceinline__ void copy_row(float* __restrict__ dst, const float* __restrict__ src, int w, int gl, int G) {
  if (VEC) {
    for (int c = gl * 4; c < w; c += G * 4)
      *reinterpret_cast<float4*>(dst + c) = *reinterpret_cast<const float4*>(src + c);
  } else {
    for (int c = gl; c < w; c += G) dst[c] = src[c];
  }
}

// bag b spans occurrences [s, e): offsets == NULL means one occurrence per bag;
// otherwise torch.nn.functional.embedding_bag's layout (include_last_offset or not)
template <typename OffT>
__device__ __forceinline__ void bag_bounds(const OffT* off, int64_t b, int64_t nbags, int64_t n, int incl, int64_t& s,
                                           int64_t& e) {
  if (off == nullptr) {
    s = b;
    e = b + 1;
    return;
  }
  s = (int64_t)off[b];
  e = (incl || b + 1 < nbags) ? (int64_t)off[b + 1] : n;
}

inline size_t align16(size_t b) { return (b + 15) & ~size_t(15); }

inline int key_bits_for(int64_t u) {
  int b = 1;
  while ((int64_t(1) << b) < u) ++b;
  return b;
}

}  // namespace fc
