// ReLU with a bit-packed mask and MaxPool2d with a 1-byte window-argmax map:
// the reference's MemSave ReLU / MaxPool storage (rules.py:98-101, :108-109;
// saved.py:53-71 BitMask, saved.py:111-125 IndexMap) and kernels
// (numpy_impl.py:54-78, numba_impl.py:78-106).  Both are HBM-bound.
//
// ReLU: y = max(x, 0); mask bit i = (x_i > 0) (ties at 0 -> 0, SPEC.md "ReLU at
//   exactly 0 -> mask bit 0"); dx = g where the bit is set.  8 elements per
//   thread-step = one mask byte; y/dx may alias x/g (in-place).
// MaxPool2d: the argmax is stored as the window-local offset r*kw + s (one
//   byte) instead of the reference's 4-byte flat index; ties keep the first
//   occurrence in row-major window order (numpy_impl.py:60-69), padding is
//   -inf.  Backward is a gather: every input element checks the <= ceil(k/s)^2
//   windows that contain it, so no atomics and a fully written dx.
#include <type_traits>
#include "misc.cuh"
#include "vec.cuh"

namespace ms {
namespace {

int grid_for(int64_t work) {
  int64_t b = (work + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (b > cap) b = cap;
  return (int)(b > 0 ? b : 1);
}

// ---------------------------------------------------------------- ReLU
// Each thread handles RELU_UNR groups of 8 elements per iteration, loads first
// (memory-level parallelism), then computes and stores.
constexpr int RELU_UNR = 4;

template <typename T>
__device__ __forceinline__ uint32_t relu8(float (&v)[8]) {
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const bool pos = !(v[j] <= 0.f);  // x > 0, and NaN propagates like torch.relu
    bits |= (pos ? 1u : 0u) << j;
    v[j] = pos ? v[j] : 0.f;
  }
  return bits;
}

// y = relu(x [+ b]); b (nullable) is the residual operand of a fused add + ReLU
template <typename T>
__global__ void __launch_bounds__(256) relu_fwd_kernel(int64_t n, const T* x, T* y,
                                                       uint8_t* __restrict__ mask, bool vec,
                                                       const T* b = nullptr) {
  const int64_t full = n / 8;  // complete groups
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g0 < full;
       g0 += stride * RELU_UNR) {
    float v[RELU_UNR][8];
#pragma unroll
    for (int u = 0; u < RELU_UNR; ++u) {
      const int64_t gi = g0 + u * stride;
      if (gi < full) ld8<T>(x + gi * 8, v[u], vec);
    }
    if (b) {
      float w[RELU_UNR][8];
#pragma unroll
      for (int u = 0; u < RELU_UNR; ++u) {
        const int64_t gi = g0 + u * stride;
        if (gi < full) ld8<T>(b + gi * 8, w[u], vec);
      }
#pragma unroll
      for (int u = 0; u < RELU_UNR; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j) v[u][j] += w[u][j];
    }
#pragma unroll
    for (int u = 0; u < RELU_UNR; ++u) {
      const int64_t gi = g0 + u * stride;
      if (gi >= full) continue;
      const uint32_t bits = relu8<T>(v[u]);
      st8<T>(y + gi * 8, v[u], vec);
      if (mask) mask[gi] = static_cast<uint8_t>(bits);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && full * 8 < n) {  // tail group
    const int64_t e = full * 8;
    uint32_t bits = 0;
    for (int j = 0; e + j < n; ++j) {
      const float a = IO<T>::ld(x + e + j) + (b ? IO<T>::ld(b + e + j) : 0.f);
      const bool pos = !(a <= 0.f);
      bits |= (pos ? 1u : 0u) << j;
      y[e + j] = IO<T>::cvt(pos ? a : 0.f);
    }
    if (mask) mask[full] = static_cast<uint8_t>(bits);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) relu_bwd_kernel(int64_t n, const T* g,
                                                       const uint8_t* __restrict__ mask, T* dx,
                                                       bool vec) {
  const int64_t full = n / 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g0 < full;
       g0 += stride * RELU_UNR) {
    float v[RELU_UNR][8];
    uint32_t bits[RELU_UNR];
#pragma unroll
    for (int u = 0; u < RELU_UNR; ++u) {
      const int64_t gi = g0 + u * stride;
      if (gi < full) {
        ld8<T>(g + gi * 8, v[u], vec);
        bits[u] = mask[gi];
      }
    }
#pragma unroll
    for (int u = 0; u < RELU_UNR; ++u) {
      const int64_t gi = g0 + u * stride;
      if (gi >= full) continue;
#pragma unroll
      for (int j = 0; j < 8; ++j) v[u][j] = (bits[u] >> j) & 1u ? v[u][j] : 0.f;
      st8<T>(dx + gi * 8, v[u], vec);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && full * 8 < n) {
    const int64_t e = full * 8;
    const uint32_t bits = mask[full];
    for (int j = 0; e + j < n; ++j)
      dx[e + j] = IO<T>::cvt((bits >> j) & 1u ? IO<T>::ld(g + e + j) : 0.f);
  }
}

// ---------------------------------------------------------------- MaxPool2d
constexpr int MAXPOOL_FUSED_C = 512;  // channels of the fused-epilogue scale table

struct PoolDims {
  int n, c, h, w, oh, ow, kh, kw, sh, sw, ph, pw;
};

// NHWC, 8 channels per thread (C % 8 == 0, 16-byte aligned)
template <typename T>
__global__ void __launch_bounds__(256) maxpool_fwd_nhwc8(PoolDims d, const T* __restrict__ x,
                                                         T* __restrict__ y,
                                                         uint8_t* __restrict__ idx) {
  // 32-bit index math: the host routes tensors with >= 2^31 vector groups to
  // the generic kernel
  const int G = d.c >> 3;
  const int total = d.n * d.oh * d.ow * G;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int pix = t / G;
    const int g = t - pix * G;
    const int ow = pix % d.ow;
    const int nh = pix / d.ow;
    const int oh = nh % d.oh;
    const int n = nh / d.oh;
    float best[8];
    uint32_t arg[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      best[j] = -INFINITY;
      arg[j] = 0;
    }
    bool first = true;
    const T* xn = x + (int64_t)n * d.h * d.w * d.c + g * 8;
    for (int r = 0; r < d.kh; ++r) {
      const int ih = oh * d.sh - d.ph + r;
      if (ih < 0 || ih >= d.h) continue;
      for (int s = 0; s < d.kw; ++s) {
        const int iw = ow * d.sw - d.pw + s;
        if (iw < 0 || iw >= d.w) continue;
        float v[8];
        ld8<T>(xn + ((int64_t)ih * d.w + iw) * d.c, v, true);
        const uint32_t k = r * d.kw + s;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (first || v[j] > best[j] || (v[j] != v[j] && best[j] == best[j])) {
            best[j] = v[j];
            arg[j] = k;
          }
        }
        first = false;
      }
    }
    const int64_t o = (int64_t)pix * d.c + g * 8;
    st8<T>(y + o, best, true);
    if (idx) {
      uint2 u;
      u.x = arg[0] | (arg[1] << 8) | (arg[2] << 16) | (arg[3] << 24);
      u.y = arg[4] | (arg[5] << 8) | (arg[6] << 16) | (arg[7] << 24);
      *reinterpret_cast<uint2*>(idx + o) = u;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) maxpool_bwd_nhwc8(PoolDims d, const T* __restrict__ g,
                                                         const uint8_t* __restrict__ idx,
                                                         T* __restrict__ dx) {
  const int G = d.c >> 3;
  const int total = d.n * d.h * d.w * G;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int pix = t / G;
    const int gg = t - pix * G;
    const int iw = pix % d.w;
    const int nh = pix / d.w;
    const int ih = nh % d.h;
    const int n = nh / d.h;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // windows (oh, ow) with oh*sh - ph <= ih <= oh*sh - ph + kh - 1
    const int oh_lo = max(0, (ih + d.ph - d.kh + d.sh) / d.sh);
    const int oh_hi = min(d.oh - 1, (ih + d.ph) / d.sh);
    const int ow_lo = max(0, (iw + d.pw - d.kw + d.sw) / d.sw);
    const int ow_hi = min(d.ow - 1, (iw + d.pw) / d.sw);
    const int64_t nbase = (int64_t)n * d.oh * d.ow;
    for (int oh = oh_lo; oh <= oh_hi; ++oh) {
      const int r = ih + d.ph - oh * d.sh;
      if (r < 0 || r >= d.kh) continue;
      for (int ow = ow_lo; ow <= ow_hi; ++ow) {
        const int s = iw + d.pw - ow * d.sw;
        if (s < 0 || s >= d.kw) continue;
        const uint32_t k = r * d.kw + s;
        const int64_t o = (nbase + (int64_t)oh * d.ow + ow) * d.c + gg * 8;
        const uint2 u = *reinterpret_cast<const uint2*>(idx + o);
        // skip the gradient load when no lane of this window picked (ih, iw)
        const uint32_t kk = k * 0x01010101u;
        const uint32_t hx = u.x ^ kk, hy = u.y ^ kk;
        const bool any = ((hx - 0x01010101u) & ~hx & 0x80808080u) ||
                         ((hy - 0x01010101u) & ~hy & 0x80808080u);
        if (!any) continue;
        float gv[8];
        ld8<T>(g + o, gv, true);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t a = ((j < 4 ? u.x : u.y) >> (8 * (j & 3))) & 0xFFu;
          if (a == k) acc[j] += gv[j];
        }
      }
    }
    st8<T>(dx + (int64_t)pix * d.c + gg * 8, acc, true);
  }
}

// The ResNet/VGG stem pool (3x3, stride 2, pad 1), NHWC, 8 channels per
// thread, 2-D grid (blockIdx.y = image row, x = (column, channel group)) so no
// per-element division.  Window (oh, ow) covers rows 2oh-1 .. 2oh+1, so input
// row 2i is only in window row i (tap r = 1) and row 2i+1 in rows i (r = 2) and
// i+1 (r = 0); the same holds for columns.
template <typename T>
__global__ void __launch_bounds__(256) maxpool_fwd_k3s2p1(PoolDims d, const T* __restrict__ x,
                                                          T* __restrict__ y,
                                                          uint8_t* __restrict__ idx) {
  const int G = d.c >> 3;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d.ow * G) return;
  const int ow = t / G;
  const int gg = t - ow * G;
  const int n = blockIdx.y / d.oh;
  const int oh = blockIdx.y - n * d.oh;
  const T* xn = x + (int64_t)n * d.h * d.w * d.c + gg * 8;
  const int64_t o = (((int64_t)n * d.oh + oh) * d.ow + ow) * d.c + gg * 8;
  if constexpr (sizeof(T) == 2) {
    // packed 16-bit: the window max by NaN-propagating HMNMX2, then the argmax as
    // the first in-range tap equal to it (or the first NaN) -- the same answer as
    // the r-major "first, then strictly greater" scan, at ~1/3 of the instructions
    using T2 = typename std::conditional<std::is_same<T, __half>::value, __half2,
                                         __nv_bfloat162>::type;
    uint4 raw[9];
    bool in[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int ih = 2 * oh - 1 + k / 3, iw = 2 * ow - 1 + k % 3;
      in[k] = ih >= 0 && ih < d.h && iw >= 0 && iw < d.w;
      raw[k] = in[k] ? __ldg(reinterpret_cast<const uint4*>(xn + ((int64_t)ih * d.w + iw) * d.c))
                     : make_uint4(0u, 0u, 0u, 0u);
    }
    uint32_t mx[4], yv[4], ag[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      T2 m = *reinterpret_cast<const T2*>(reinterpret_cast<const uint32_t*>(&raw[4]) + q);
#pragma unroll
      for (int k = 0; k < 9; ++k)  // tap 4 (the window centre) is always in range
        if (k != 4 && in[k])
          m = __hmax2_nan(m, *reinterpret_cast<const T2*>(reinterpret_cast<const uint32_t*>(&raw[k]) + q));
      mx[q] = *reinterpret_cast<uint32_t*>(&m);
      yv[q] = 0u;
      ag[q] = 0u;
    }
#pragma unroll
    for (int k = 8; k >= 0; --k) {
      if (!in[k]) continue;
      const uint32_t kk = (uint32_t)k | ((uint32_t)k << 16);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t vw = reinterpret_cast<const uint32_t*>(&raw[k])[q];
        const T2 v2 = *reinterpret_cast<const T2*>(&vw);
        const T2 m2 = *reinterpret_cast<const T2*>(&mx[q]);
        const uint32_t hit = __heq2_mask(v2, m2) | __hneu2_mask(v2, v2);
        yv[q] = (yv[q] & ~hit) | (vw & hit);
        ag[q] = (ag[q] & ~hit) | (kk & hit);
      }
    }
    *reinterpret_cast<uint4*>(y + o) = make_uint4(yv[0], yv[1], yv[2], yv[3]);
    if (idx) {
      uint2 u;  // 16-bit args (channel pairs) -> one byte per channel
      u.x = (ag[0] & 0xFFu) | ((ag[0] >> 8) & 0xFF00u) | ((ag[1] & 0xFFu) << 16) |
            ((ag[1] >> 16) << 24);
      u.y = (ag[2] & 0xFFu) | ((ag[2] >> 8) & 0xFF00u) | ((ag[3] & 0xFFu) << 16) |
            ((ag[3] >> 16) << 24);
      *reinterpret_cast<uint2*>(idx + o) = u;
    }
    return;
  }
  float best[8];
  uint32_t arg[8];
  bool first = true;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    const int ih = 2 * oh - 1 + r;
    if (ih < 0 || ih >= d.h) continue;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int iw = 2 * ow - 1 + s;
      if (iw < 0 || iw >= d.w) continue;
      float v[8];
      ld8<T>(xn + ((int64_t)ih * d.w + iw) * d.c, v, true);
      const uint32_t k = r * 3 + s;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (first || v[j] > best[j] || (v[j] != v[j] && best[j] == best[j])) {
          best[j] = v[j];
          arg[j] = k;
        }
      }
      first = false;
    }
  }
  st8<T>(y + o, best, true);
  if (idx) {
    uint2 u;
    u.x = arg[0] | (arg[1] << 8) | (arg[2] << 16) | (arg[3] << 24);
    u.y = arg[4] | (arg[5] << 8) | (arg[6] << 16) | (arg[7] << 24);
    *reinterpret_cast<uint2*>(idx + o) = u;
  }
}

// 2x2 / stride 2 / no padding (VGG): every tap is in range; packed 16-bit max
// and first-equal argmax as in maxpool_fwd_k3s2p1.  2-D grid: blockIdx.y = n*oh.
template <typename T>
__global__ void __launch_bounds__(256) maxpool_fwd_k2s2(PoolDims d, const T* __restrict__ x,
                                                        T* __restrict__ y,
                                                        uint8_t* __restrict__ idx) {
  using T2 = typename std::conditional<std::is_same<T, __half>::value, __half2,
                                       __nv_bfloat162>::type;
  const int G = d.c >> 3;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d.ow * G) return;
  const int ow = t / G;
  const int gg = t - ow * G;
  const int n = blockIdx.y / d.oh;
  const int oh = blockIdx.y - n * d.oh;
  const T* xn = x + ((int64_t)n * d.h + 2 * oh) * d.w * d.c + gg * 8;
  uint4 raw[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    raw[k] = __ldg(reinterpret_cast<const uint4*>(xn + ((int64_t)(k >> 1) * d.w + 2 * ow + (k & 1)) *
                                                           d.c));
  uint32_t yv[4], ag[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    T2 m = *reinterpret_cast<const T2*>(reinterpret_cast<const uint32_t*>(&raw[0]) + q);
#pragma unroll
    for (int k = 1; k < 4; ++k)
      m = __hmax2_nan(m, *reinterpret_cast<const T2*>(reinterpret_cast<const uint32_t*>(&raw[k]) + q));
    yv[q] = 0u;
    ag[q] = 0u;
#pragma unroll
    for (int k = 3; k >= 0; --k) {  // the last write wins: the first equal tap (or NaN)
      const uint32_t vw = reinterpret_cast<const uint32_t*>(&raw[k])[q];
      const T2 v2 = *reinterpret_cast<const T2*>(&vw);
      const uint32_t hit = __heq2_mask(v2, m) | __hneu2_mask(v2, v2);
      const uint32_t kk = (uint32_t)k | ((uint32_t)k << 16);
      yv[q] = (yv[q] & ~hit) | (vw & hit);
      ag[q] = (ag[q] & ~hit) | (kk & hit);
    }
  }
  const int64_t o = (((int64_t)n * d.oh + oh) * d.ow + ow) * d.c + gg * 8;
  *reinterpret_cast<uint4*>(y + o) = make_uint4(yv[0], yv[1], yv[2], yv[3]);
  if (idx) {
    uint2 u;
    u.x = (ag[0] & 0xFFu) | ((ag[0] >> 8) & 0xFF00u) | ((ag[1] & 0xFFu) << 16) |
          ((ag[1] >> 16) << 24);
    u.y = (ag[2] & 0xFFu) | ((ag[2] >> 8) & 0xFF00u) | ((ag[3] & 0xFFu) << 16) |
          ((ag[3] >> 16) << 24);
    *reinterpret_cast<uint2*>(idx + o) = u;
  }
}

// add g[j] to acc[j] for the channels whose window argmax is tap k
template <typename T>
__device__ __forceinline__ void route8(float (&acc)[8], const uint2 u, const float (&gv)[8],
                                       uint32_t k) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t a = ((j < 4 ? u.x : u.y) >> (8 * (j & 3))) & 0xFFu;
    if (a == k) acc[j] += gv[j];
  }
}

// Backward of the 3x3/2/1 pool: one thread per 2x2 input block (rows 2i, 2i+1,
// cols 2j, 2j+1) x 8 channels reads the <= 4 windows (i..i+1) x (j..j+1) once
// and writes the 4 input pixels (two 2-pixel runs), every dx element exactly once.
template <typename T>
__global__ void __launch_bounds__(256, 4) maxpool_bwd_k3s2p1(PoolDims d, const T* __restrict__ g,
                                                          const uint8_t* __restrict__ idx,
                                                          T* __restrict__ dx,
                                                          const uint8_t* __restrict__ keep,
                                                          const BnFold in_bn) {
  // keep (nullable): the bit mask of the ReLU that produced x, and in_bn.var
  // (nullable) the eval-BN before it: dx = keep ? dx * s : 0 (their backward)
  __shared__ float s_sc[MAXPOOL_FUSED_C];
  if (in_bn.var) {
    for (int c = threadIdx.x; c < d.c; c += blockDim.x) {
      float s, t_;
      bn_fold(in_bn, c, s, t_);
      s_sc[c] = s;
    }
    __syncthreads();
  }
  const int G = d.c >> 3;
  const int jn = (d.w + 1) >> 1;
  const int in = (d.h + 1) >> 1;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= jn * G) return;
  const int j = t / G;
  const int gg = t - j * G;
  const int n = blockIdx.y / in;
  const int i = blockIdx.y - n * in;
  const int h0 = 2 * i, w0 = 2 * j;
  // the producer ReLU's keep bits of the 4 output pixels, loaded with the
  // windows (one memory round trip per thread instead of two)
  uint32_t kb4[2][2] = {{0xFFu, 0xFFu}, {0xFFu, 0xFFu}};
  if (keep) {
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
        if (h0 + a < d.h && w0 + b < d.w)
          kb4[a][b] = __ldg(keep + (((int64_t)n * d.h + h0 + a) * d.w + w0 + b) * G + gg);
  }
  float gv[2][2][8];
  uint2 u[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int oh = i + a, ow = j + b;
      if (oh < d.oh && ow < d.ow) {
        const int64_t o = (((int64_t)n * d.oh + oh) * d.ow + ow) * d.c + gg * 8;
        u[a][b] = __ldg(reinterpret_cast<const uint2*>(idx + o));
        ld8<T>(g + o, gv[a][b], true);
      } else {
        u[a][b] = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);  // matches no tap
#pragma unroll
        for (int q = 0; q < 8; ++q) gv[a][b][q] = 0.f;
      }
    }
  // taps: window (i, j) -> input (2i + r - 1, 2j + s - 1), k = 3r + s
  float o00[8] = {0, 0, 0, 0, 0, 0, 0, 0}, o01[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  float o10[8] = {0, 0, 0, 0, 0, 0, 0, 0}, o11[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  route8<T>(o00, u[0][0], gv[0][0], 4);  // (2i,   2j  ) <- (i, j) r1 s1
  route8<T>(o01, u[0][0], gv[0][0], 5);  // (2i,   2j+1) <- (i, j) r1 s2
  route8<T>(o01, u[0][1], gv[0][1], 3);  //                (i, j+1) r1 s0
  route8<T>(o10, u[0][0], gv[0][0], 7);  // (2i+1, 2j  ) <- (i, j) r2 s1
  route8<T>(o10, u[1][0], gv[1][0], 1);  //                (i+1, j) r0 s1
  route8<T>(o11, u[0][0], gv[0][0], 8);  // (2i+1, 2j+1) <- (i, j) r2 s2
  route8<T>(o11, u[0][1], gv[0][1], 6);  //                (i, j+1) r2 s0
  route8<T>(o11, u[1][0], gv[1][0], 2);  //                (i+1, j) r0 s2
  route8<T>(o11, u[1][1], gv[1][1], 0);  //                (i+1, j+1) r0 s0
  if (keep || in_bn.var) {
    auto fin = [&](float (&o)[8], uint32_t kb) {
      if (keep) {
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = ((kb >> q) & 1u) ? o[q] : 0.f;
      }
      if (in_bn.var) {
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] *= s_sc[gg * 8 + q];
      }
    };
    fin(o00, kb4[0][0]);
    fin(o01, kb4[0][1]);
    fin(o10, kb4[1][0]);
    fin(o11, kb4[1][1]);
  }
  T* base = dx + ((int64_t)n * d.h + h0) * d.w * d.c + gg * 8;
  st8<T>(base + (int64_t)w0 * d.c, o00, true);
  if (w0 + 1 < d.w) st8<T>(base + (int64_t)(w0 + 1) * d.c, o01, true);
  if (h0 + 1 < d.h) {
    T* b1 = base + (int64_t)d.w * d.c;
    st8<T>(b1 + (int64_t)w0 * d.c, o10, true);
    if (w0 + 1 < d.w) st8<T>(b1 + (int64_t)(w0 + 1) * d.c, o11, true);
  }
}

// generic (any layout via strides, scalar)
struct S4 {
  int64_t n, c, h, w;
};

template <typename T>
__global__ void maxpool_fwd_generic(PoolDims d, const T* __restrict__ x, S4 xs, T* __restrict__ y,
                                    S4 ys, uint8_t* __restrict__ idx) {
  const int64_t total = (int64_t)d.n * d.c * d.oh * d.ow;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = t;
    const int ow = p % d.ow; p /= d.ow;
    const int oh = p % d.oh; p /= d.oh;
    const int c = p % d.c;
    const int n = (int)(p / d.c);
    float best = -INFINITY;
    uint32_t arg = 0;
    bool first = true;
    for (int r = 0; r < d.kh; ++r) {
      const int ih = oh * d.sh - d.ph + r;
      if (ih < 0 || ih >= d.h) continue;
      for (int s = 0; s < d.kw; ++s) {
        const int iw = ow * d.sw - d.pw + s;
        if (iw < 0 || iw >= d.w) continue;
        const float v = IO<T>::ld(x + n * xs.n + c * xs.c + ih * xs.h + iw * xs.w);
        if (first || v > best || (v != v && best == best)) {
          best = v;
          arg = r * d.kw + s;
        }
        first = false;
      }
    }
    const int64_t o = n * ys.n + c * ys.c + oh * ys.h + ow * ys.w;
    y[o] = IO<T>::cvt(best);
    if (idx) idx[o] = (uint8_t)arg;
  }
}

template <typename T>
__global__ void maxpool_bwd_generic(PoolDims d, const T* __restrict__ g, S4 gs,
                                    const uint8_t* __restrict__ idx, T* __restrict__ dx, S4 xs) {
  const int64_t total = (int64_t)d.n * d.c * d.h * d.w;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = t;
    const int iw = p % d.w; p /= d.w;
    const int ih = p % d.h; p /= d.h;
    const int c = p % d.c;
    const int n = (int)(p / d.c);
    float acc = 0.f;
    const int oh_lo = max(0, (ih + d.ph - d.kh + d.sh) / d.sh);
    const int oh_hi = min(d.oh - 1, (ih + d.ph) / d.sh);
    const int ow_lo = max(0, (iw + d.pw - d.kw + d.sw) / d.sw);
    const int ow_hi = min(d.ow - 1, (iw + d.pw) / d.sw);
    for (int oh = oh_lo; oh <= oh_hi; ++oh) {
      const int r = ih + d.ph - oh * d.sh;
      if (r < 0 || r >= d.kh) continue;
      for (int ow = ow_lo; ow <= ow_hi; ++ow) {
        const int s = iw + d.pw - ow * d.sw;
        if (s < 0 || s >= d.kw) continue;
        const int64_t o = n * gs.n + c * gs.c + oh * gs.h + ow * gs.w;
        if (idx[o] == (uint8_t)(r * d.kw + s)) acc += IO<T>::ld(g + o);
      }
    }
    dx[n * xs.n + c * xs.c + ih * xs.h + iw * xs.w] = IO<T>::cvt(acc);
  }
}

S4 strides_of(int layout, int64_t c, int64_t h, int64_t w) {
  if (layout == MS_NHWC) return S4{h * w * c, 1, w * c, c};
  return S4{c * h * w, h * w, w, 1};
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ---------------------------------------------------------------- GELU
// Elementwise GELU (erf form) and its VJP, the unfused halves of a Linear ->
// GELU pair (the forward is normally fused into the GEMM epilogue).  The erf
// makes them issue-bound rather than HBM-bound: GELU_UNR groups of 8 per
// thread (loads first) keep the registers low enough for full occupancy.
constexpr int GELU_UNR = 1;
template <typename T, bool BWD>
__global__ void __launch_bounds__(256) gelu_kernel(int64_t n, const T* __restrict__ a,
                                                   const T* __restrict__ pre, T* __restrict__ y,
                                                   bool vec) {
  const int64_t groups = (n + 7) / 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g0 < groups;
       g0 += stride * GELU_UNR) {
    float v[GELU_UNR][8], x[GELU_UNR][8];
#pragma unroll
    for (int u = 0; u < GELU_UNR; ++u) {
      const int64_t gi = g0 + u * stride;
      if (gi >= groups) continue;
      const bool full = gi * 8 + 8 <= n;
      if (full) {
        ld8<T>(a + gi * 8, v[u], vec);
        if (BWD) ld8<T>(pre + gi * 8, x[u], vec);
      } else {
        for (int j = 0; j < 8; ++j) {
          v[u][j] = gi * 8 + j < n ? IO<T>::ld(a + gi * 8 + j) : 0.f;
          if (BWD) x[u][j] = gi * 8 + j < n ? IO<T>::ld(pre + gi * 8 + j) : 0.f;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < GELU_UNR; ++u) {
      const int64_t gi = g0 + u * stride;
      if (gi >= groups) continue;
#pragma unroll
      if constexpr (BWD) {
        gelu_grad_n<8>(x[u], v[u]);
      } else {
        gelu_n<8>(v[u]);  // the GEMM epilogue's evaluation (bit-identical to erff)
      }
      if (gi * 8 + 8 <= n) {
        st8<T>(y + gi * 8, v[u], vec);
      } else {
        for (int j = 0; j < 8 && gi * 8 + j < n; ++j) y[gi * 8 + j] = IO<T>::cvt(v[u][j]);
      }
    }
  }
}

}  // namespace

namespace {
template <typename T>
__global__ void __launch_bounds__(256) add_kernel(int64_t n, T* __restrict__ y,
                                                  const T* __restrict__ r, bool vec) {
  const int64_t groups = (n + 7) / 8;
  for (int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < groups;
       gi += (int64_t)gridDim.x * blockDim.x) {
    if (gi * 8 + 8 <= n) {
      float a[8], b[8];
      ld8<T>(y + gi * 8, a, vec);
      ld8<T>(r + gi * 8, b, vec);
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] += b[j];
      st8<T>(y + gi * 8, a, vec);
    } else {
      for (int64_t e = gi * 8; e < n; ++e) y[e] = IO<T>::cvt(IO<T>::ld(y + e) + IO<T>::ld(r + e));
    }
  }
}
}  // namespace

ms_status add_inplace(int64_t n, int dt, void* y, const void* r, cudaStream_t st) {
  if (n <= 0) return MS_OK;
  const bool vec = al16(y) && al16(r);
  MS_DT_DISPATCH(dt, (add_kernel<T><<<grid_for((n + 7) / 8), 256, 0, st>>>(n, (T*)y, (const T*)r,
                                                                          vec)));
  count_launch();
  return launch_status("add_kernel");
}

ms_status gelu_fwd(int64_t n, int dt, const void* x, void* y, cudaStream_t st) {
  if (n <= 0) return MS_OK;
  const bool vec = al16(x) && al16(y);
  MS_DT_DISPATCH(dt, (gelu_kernel<T, false><<<grid_for((n + 7) / 8), 256, 0, st>>>(
                         n, (const T*)x, nullptr, (T*)y, vec)));
  count_launch();
  return launch_status("gelu_kernel");
}

ms_status gelu_bwd(int64_t n, int dt, const void* g, const void* pre, void* dx, cudaStream_t st) {
  if (n <= 0) return MS_OK;
  const bool vec = al16(g) && al16(pre) && al16(dx);
  MS_DT_DISPATCH(dt, (gelu_kernel<T, true><<<grid_for((n + 7) / 8), 256, 0, st>>>(
                         n, (const T*)g, (const T*)pre, (T*)dx, vec)));
  count_launch();
  return launch_status("gelu_bwd_kernel");
}

}  // namespace ms

using namespace ms;

extern "C" ms_status ms_gelu_fwd(int64_t numel, int32_t dt, const void* x, void* y,
                                 void* stream) {
  MS_CHECK_ARG(numel >= 0 && x && y, MS_ERR_SHAPE, "gelu: bad arguments");
  if (numel == 0) return MS_OK;
  MS_TRY(bind_device(y));
  return gelu_fwd(numel, dt, x, y, (cudaStream_t)stream);
}

extern "C" ms_status ms_gelu_bwd(int64_t numel, int32_t dt, const void* g, const void* pre,
                                 void* dx, void* stream) {
  MS_CHECK_ARG(numel >= 0 && g && pre && dx, MS_ERR_SHAPE, "gelu bwd: bad arguments");
  if (numel == 0) return MS_OK;
  MS_TRY(bind_device(dx));
  return gelu_bwd(numel, dt, g, pre, dx, (cudaStream_t)stream);
}

extern "C" ms_status ms_relu_fwd(int64_t numel, int32_t dt, const void* x, void* y,
                                 void* mask_or_null, void* stream) {
  MS_CHECK_ARG(numel >= 0 && x && y, MS_ERR_SHAPE, "relu: bad arguments");
  if (numel == 0) return MS_OK;
  MS_TRY(bind_device(y));
  cudaStream_t st = (cudaStream_t)stream;
  const bool vec = al16(x) && al16(y);
  MS_DT_DISPATCH(dt, relu_fwd_kernel<T><<<grid_for((numel + 31) / 32), 256, 0, st>>>(
                         numel, (const T*)x, (T*)y, (uint8_t*)mask_or_null, vec));
  count_launch();
  return launch_status("relu_fwd_kernel");
}

extern "C" ms_status ms_add_relu_fwd(int64_t numel, int32_t dt, const void* a, const void* b,
                                     void* y, void* mask_or_null, void* stream) {
  MS_CHECK_ARG(numel >= 0 && a && b && y, MS_ERR_SHAPE, "add_relu: bad arguments");
  if (numel == 0) return MS_OK;
  MS_TRY(bind_device(y));
  cudaStream_t st = (cudaStream_t)stream;
  const bool vec = al16(a) && al16(b) && al16(y);
  MS_DT_DISPATCH(dt, relu_fwd_kernel<T><<<grid_for((numel + 31) / 32), 256, 0, st>>>(
                         numel, (const T*)a, (T*)y, (uint8_t*)mask_or_null, vec, (const T*)b));
  count_launch();
  return launch_status("add_relu_fwd_kernel");
}

extern "C" ms_status ms_relu_bwd(int64_t numel, int32_t dt, const void* g, const void* mask,
                                 void* dx, void* stream) {
  MS_CHECK_ARG(numel >= 0 && g && mask && dx, MS_ERR_SHAPE, "relu bwd: bad arguments");
  if (numel == 0) return MS_OK;
  MS_TRY(bind_device(dx));
  cudaStream_t st = (cudaStream_t)stream;
  const bool vec = al16(g) && al16(dx);
  MS_DT_DISPATCH(dt, relu_bwd_kernel<T><<<grid_for((numel + 31) / 32), 256, 0, st>>>(
                         numel, (const T*)g, (const uint8_t*)mask, (T*)dx, vec));
  count_launch();
  return launch_status("relu_bwd_kernel");
}

static ms_status pool_dims(const ms_pool_desc* p, PoolDims& d) {
  MS_CHECK_ARG(p && p->n >= 0 && p->c > 0 && p->h > 0 && p->w > 0 && p->kh > 0 && p->kw > 0 &&
                   p->stride_h > 0 && p->stride_w > 0 && p->pad_h >= 0 && p->pad_w >= 0,
               MS_ERR_SHAPE, "maxpool: bad geometry");
  MS_CHECK_ARG(p->kh * p->kw <= 256, MS_ERR_UNSUPPORTED, "maxpool: window larger than 256");
  MS_CHECK_ARG(2 * p->pad_h <= p->kh && 2 * p->pad_w <= p->kw, MS_ERR_SHAPE,
               "maxpool: padding must be at most half the window");
  d = PoolDims{(int)p->n, (int)p->c, (int)p->h, (int)p->w, 0, 0, p->kh, p->kw, p->stride_h,
               p->stride_w, p->pad_h, p->pad_w};
  d.oh = (int)((p->h + 2 * p->pad_h - p->kh) / p->stride_h + 1);
  d.ow = (int)((p->w + 2 * p->pad_w - p->kw) / p->stride_w + 1);
  MS_CHECK_ARG(d.oh > 0 && d.ow > 0, MS_ERR_SHAPE, "maxpool: empty output");
  return MS_OK;
}

// the 3x3/2/1 specialisation; grid.y = n * rows must fit the 65535 limit
static bool is_k3s2p1(const PoolDims& d) {
  return d.kh == 3 && d.kw == 3 && d.sh == 2 && d.sw == 2 && d.ph == 1 && d.pw == 1 &&
         (int64_t)d.n * d.oh <= 65535 && (int64_t)d.n * ((d.h + 1) / 2) <= 65535 &&
         d.oh == (d.h + 1) / 2 && d.ow == (d.w + 1) / 2;
}

extern "C" int64_t ms_maxpool2d_out_h(const ms_pool_desc* p) {
  return (p->h + 2 * p->pad_h - p->kh) / p->stride_h + 1;
}
extern "C" int64_t ms_maxpool2d_out_w(const ms_pool_desc* p) {
  return (p->w + 2 * p->pad_w - p->kw) / p->stride_w + 1;
}

extern "C" ms_status ms_maxpool2d_fwd(const ms_pool_desc* p, const void* x, void* y,
                                      void* idx_or_null, void* stream) {
  PoolDims d;
  MS_TRY(pool_dims(p, d));
  if (d.n == 0) return MS_OK;
  MS_TRY(bind_device(y));
  cudaStream_t st = (cudaStream_t)stream;
  const int dt = p->dtype;
  if (p->layout == MS_NHWC && d.c % 8 == 0 && al16(x) && al16(y) &&
      (!idx_or_null || (reinterpret_cast<uintptr_t>(idx_or_null) & 7) == 0) &&
      (int64_t)d.n * d.h * d.w * (d.c / 8) < (1ll << 31)) {
    if (is_k3s2p1(d)) {
      const dim3 grid((unsigned)((d.ow * (d.c / 8) + 255) / 256), (unsigned)(d.n * d.oh));
      MS_DT_DISPATCH(dt, maxpool_fwd_k3s2p1<T><<<grid, 256, 0, st>>>(d, (const T*)x, (T*)y,
                                                                     (uint8_t*)idx_or_null));
    } else {
      const int64_t work = (int64_t)d.n * d.oh * d.ow * (d.c / 8);
      if (dtype_size(dt) == 2 && d.kh == 2 && d.kw == 2 && d.sh == 2 && d.sw == 2 && d.ph == 0 &&
          d.pw == 0) {
        const dim3 grid((unsigned)((d.ow * (d.c / 8) + 255) / 256), (unsigned)(d.n * d.oh));
        if (dt == MS_BF16)
          maxpool_fwd_k2s2<__nv_bfloat16><<<grid, 256, 0, st>>>(
              d, (const __nv_bfloat16*)x, (__nv_bfloat16*)y, (uint8_t*)idx_or_null);
        else
          maxpool_fwd_k2s2<__half><<<grid, 256, 0, st>>>(d, (const __half*)x, (__half*)y,
                                                          (uint8_t*)idx_or_null);
      } else {
        MS_DT_DISPATCH(dt, maxpool_fwd_nhwc8<T><<<grid_for(work), 256, 0, st>>>(
                               d, (const T*)x, (T*)y, (uint8_t*)idx_or_null));
      }
    }
  } else {
    const int64_t work = (int64_t)d.n * d.c * d.oh * d.ow;
    MS_DT_DISPATCH(dt, maxpool_fwd_generic<T><<<grid_for(work), 256, 0, st>>>(
                           d, (const T*)x, strides_of(p->layout, d.c, d.h, d.w), (T*)y,
                           strides_of(p->layout, d.c, d.oh, d.ow), (uint8_t*)idx_or_null));
  }
  count_launch();
  return launch_status("maxpool_fwd");
}

static ms_status maxpool_bwd_impl(const ms_pool_desc* p, const void* g, const void* idx,
                                  const uint8_t* keep, const BnFold& in_bn, void* dx,
                                  void* stream) {
  PoolDims d;
  MS_TRY(pool_dims(p, d));
  MS_CHECK_ARG(g && idx && dx, MS_ERR_SHAPE, "maxpool bwd: null tensor");
  if (d.n == 0) return MS_OK;
  MS_TRY(bind_device(dx));
  cudaStream_t st = (cudaStream_t)stream;
  const int dt = p->dtype;
  const bool fast = p->layout == MS_NHWC && d.c % 8 == 0 && al16(g) && al16(dx) &&
                    (reinterpret_cast<uintptr_t>(idx) & 7) == 0 &&
                    (int64_t)d.n * d.h * d.w * (d.c / 8) < (1ll << 31);
  MS_CHECK_ARG((!keep && !in_bn.var) || (fast && is_k3s2p1(d) && d.c <= MAXPOOL_FUSED_C),
               MS_ERR_UNSUPPORTED,
               "maxpool bwd: the fused ReLU/BN backward needs the NHWC 3x3/2/1 kernel, C <= %d",
               MAXPOOL_FUSED_C);
  if (fast) {
    if (is_k3s2p1(d)) {
      const dim3 grid((unsigned)((((d.w + 1) / 2) * (d.c / 8) + 255) / 256),
                      (unsigned)(d.n * ((d.h + 1) / 2)));
      MS_DT_DISPATCH(dt, maxpool_bwd_k3s2p1<T><<<grid, 256, 0, st>>>(
                             d, (const T*)g, (const uint8_t*)idx, (T*)dx, keep, in_bn));
    } else {
      const int64_t work = (int64_t)d.n * d.h * d.w * (d.c / 8);
      MS_DT_DISPATCH(dt, maxpool_bwd_nhwc8<T><<<grid_for(work), 256, 0, st>>>(
                             d, (const T*)g, (const uint8_t*)idx, (T*)dx));
    }
  } else {
    const int64_t work = (int64_t)d.n * d.c * d.h * d.w;
    MS_DT_DISPATCH(dt, maxpool_bwd_generic<T><<<grid_for(work), 256, 0, st>>>(
                           d, (const T*)g, strides_of(p->layout, d.c, d.oh, d.ow),
                           (const uint8_t*)idx, (T*)dx, strides_of(p->layout, d.c, d.h, d.w)));
  }
  count_launch();
  return launch_status("maxpool_bwd");
}

extern "C" ms_status ms_maxpool2d_bwd(const ms_pool_desc* p, const void* g, const void* idx,
                                      void* dx, void* stream) {
  return maxpool_bwd_impl(p, g, idx, nullptr, BnFold{}, dx, stream);
}

extern "C" ms_status ms_maxpool2d_relu_bwd(const ms_pool_desc* p, const void* g, const void* idx,
                                           const void* keep, const void* in_var,
                                           const void* in_weight, int32_t in_pdtype,
                                           double in_eps, void* dx, void* stream) {
  BnFold bn;
  bn.var = in_var;
  bn.w = in_weight;
  bn.pdt = in_pdtype;
  bn.eps = (float)in_eps;
  return maxpool_bwd_impl(p, g, idx, static_cast<const uint8_t*>(keep), bn, dx, stream);
}
