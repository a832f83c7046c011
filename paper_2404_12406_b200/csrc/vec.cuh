// 8-element vector load / store helpers shared by the elementwise kernels
// (16 bytes for 16-bit types, two float4 for float32).
#pragma once

#include "common.cuh"

namespace ms {

template <typename T>
__device__ __forceinline__ void ld8(const T* p, float (&v)[8], bool vec) {
  if (vec) {
    if constexpr (sizeof(T) == 2) {
      uint4 u = *reinterpret_cast<const uint4*>(p);
      const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = IO<T>::ld(e + j);
    } else {
      float4 a = *reinterpret_cast<const float4*>(p);
      float4 b = *reinterpret_cast<const float4*>(p + 4);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = IO<T>::ld(p + j);
  }
}

template <typename T>
__device__ __forceinline__ void st8(T* p, const float (&v)[8], bool vec) {
  if (vec) {
    if constexpr (sizeof(T) == 2) {
      uint4 u;
      T* e = reinterpret_cast<T*>(&u);
#pragma unroll
      for (int j = 0; j < 8; ++j) e[j] = IO<T>::cvt(v[j]);
      *reinterpret_cast<uint4*>(p) = u;
    } else {
      *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = IO<T>::cvt(v[j]);
  }
}

#define MS_DT_DISPATCH(dt, ...)                                    \
  switch (dt) {                                                    \
    case MS_F32: { using T = float; __VA_ARGS__; } break;          \
    case MS_BF16: { using T = __nv_bfloat16; __VA_ARGS__; } break; \
    case MS_F16: { using T = __half; __VA_ARGS__; } break;         \
    default: set_error("bad dtype %d", dt); return MS_ERR_DTYPE;   \
  }

}  // namespace ms
