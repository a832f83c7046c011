// CUDA-core (SIMT) kernels: the float32 path (rtol 1e-5 needs fp32 products
// with wide accumulation, which the 16-bit tensor-core kernels cannot give)
// and the general path for geometries the tcgen05 kernels do not cover
// (unaligned channel counts, NCHW 16-bit activations).  All accumulate in
// float64 for float32 operands and in float32 for 16-bit operands.
#include "simt.cuh"

namespace ms {

template <typename T> struct Acc { using type = float; };
template <> struct Acc<float> { using type = double; };

// ------------------------------------------------------------------ GEMM
// C[m, n] = sum_k A(m, k) * B(k, n) (+ bias[n]); A(m,k) = A[m*sam + k*sak],
// B(k,n) = B[k*sbk + n*sbn]; C row-major with pitch ldc.
template <typename T>
__global__ void __launch_bounds__(256) simt_gemm_kernel(int M, int N, int K, const T* __restrict__ A,
                                                        int64_t sam, int64_t sak,
                                                        const T* __restrict__ B, int64_t sbk,
                                                        int64_t sbn, const T* __restrict__ bias,
                                                        T* __restrict__ C, int64_t ldc) {
  using AT = typename Acc<T>::type;
  constexpr int TM = 64, TN = 64, TK = 16;
  __shared__ float As[TK][TM + 1];
  __shared__ float Bs[TK][TN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  AT acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int idx = threadIdx.x; idx < TM * TK; idx += 256) {
      const int mm = idx / TK, kk = idx % TK;
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? IO<T>::ld(A + m * sam + k * sak) : 0.f;
    }
    for (int idx = threadIdx.x; idx < TN * TK; idx += 256) {
      const int nn = idx % TN, kk = idx / TN;
      const int n = n0 + nn, k = k0 + kk;
      Bs[kk][nn] = (n < N && k < K) ? IO<T>::ld(B + k * sbk + n * sbn) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += static_cast<AT>(a[i]) * static_cast<AT>(b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= N) continue;
      AT v = acc[i][j];
      if (bias) v += static_cast<AT>(IO<T>::ld(bias + n));
      C[m * ldc + n] = IO<T>::cvt(static_cast<float>(v));
    }
  }
}

// Skinny outputs with a long reduction (e.g. a 2-class head: M = 64, N = 2,
// K = 768): one warp per output element, lanes split K, shuffle reduction.
// The 64 x 64 tile kernel would run one block down the whole K.
template <typename T>
__global__ void __launch_bounds__(256) simt_dot_kernel(int M, int N, int K, const T* __restrict__ A,
                                                       int64_t sam, int64_t sak,
                                                       const T* __restrict__ B, int64_t sbk,
                                                       int64_t sbn, const T* __restrict__ bias,
                                                       T* __restrict__ C, int64_t ldc) {
  using AT = typename Acc<T>::type;
  const int64_t o = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (o >= (int64_t)M * N) return;
  const int m = (int)(o / N), n = (int)(o % N);
  const T* a = A + m * sam;
  const T* b = B + n * sbn;
  AT acc = 0;
  for (int k = lane; k < K; k += 32)
    acc += static_cast<AT>(IO<T>::ld(a + k * sak)) * static_cast<AT>(IO<T>::ld(b + k * sbk));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) {
    if (bias) acc += static_cast<AT>(IO<T>::ld(bias + n));
    C[m * ldc + n] = IO<T>::cvt(static_cast<float>(acc));
  }
}

ms_status simt_gemm(int dt, int M, int N, int K, const void* A, int64_t sam, int64_t sak,
                    const void* B, int64_t sbk, int64_t sbn, const void* bias, void* C,
                    int64_t ldc, cudaStream_t st) {
  if (M <= 0 || N <= 0) return MS_OK;
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  if ((int64_t)grid.x * grid.y < 16 && K >= 256 && (int64_t)M * N <= (1 << 16)) {
    const unsigned blocks = (unsigned)(((int64_t)M * N + 7) / 8);
    switch (dt) {
      case MS_F32:
        simt_dot_kernel<float><<<blocks, 256, 0, st>>>(M, N, K, (const float*)A, sam, sak,
                                                       (const float*)B, sbk, sbn,
                                                       (const float*)bias, (float*)C, ldc);
        break;
      case MS_BF16:
        simt_dot_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
            M, N, K, (const __nv_bfloat16*)A, sam, sak, (const __nv_bfloat16*)B, sbk, sbn,
            (const __nv_bfloat16*)bias, (__nv_bfloat16*)C, ldc);
        break;
      case MS_F16:
        simt_dot_kernel<__half><<<blocks, 256, 0, st>>>(M, N, K, (const __half*)A, sam, sak,
                                                        (const __half*)B, sbk, sbn,
                                                        (const __half*)bias, (__half*)C, ldc);
        break;
      default:
        set_error("simt_gemm: bad dtype %d", dt);
        return MS_ERR_DTYPE;
    }
    count_launch(1, KF_SIMT);
    return launch_status("simt_dot_kernel");
  }
  switch (dt) {
    case MS_F32:
      simt_gemm_kernel<float><<<grid, 256, 0, st>>>(M, N, K, (const float*)A, sam, sak,
                                                    (const float*)B, sbk, sbn, (const float*)bias,
                                                    (float*)C, ldc);
      break;
    case MS_BF16:
      simt_gemm_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
          M, N, K, (const __nv_bfloat16*)A, sam, sak, (const __nv_bfloat16*)B, sbk, sbn,
          (const __nv_bfloat16*)bias, (__nv_bfloat16*)C, ldc);
      break;
    case MS_F16:
      simt_gemm_kernel<__half><<<grid, 256, 0, st>>>(M, N, K, (const __half*)A, sam, sak,
                                                     (const __half*)B, sbk, sbn,
                                                     (const __half*)bias, (__half*)C, ldc);
      break;
    default:
      set_error("simt_gemm: bad dtype %d", dt);
      return MS_ERR_DTYPE;
  }
  count_launch(1, KF_SIMT);
  return launch_status("simt_gemm_kernel");
}

// ------------------------------------------------------------------ direct conv
// Activation index: n*sn + c*sc + h*sh + w*sw ; weight: k*wk + c*wc + r*wr + s*ws.
struct Strides4 {
  int64_t n, c, h, w;
};

template <typename T>
__global__ void direct_conv_fwd_kernel(ConvDims d, const T* __restrict__ x, Strides4 xs,
                                       const T* __restrict__ w, Strides4 wsd,
                                       const T* __restrict__ bias, T* __restrict__ y,
                                       Strides4 ys) {
  using AT = typename Acc<T>::type;
  const int64_t total = (int64_t)d.n * d.k * d.oh * d.ow;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int ow = t % d.ow; t /= d.ow;
    const int oh = t % d.oh; t /= d.oh;
    const int k = t % d.k; t /= d.k;
    const int n = (int)t;
    AT acc = 0;
    for (int c = 0; c < d.c; ++c) {
      for (int r = 0; r < d.r; ++r) {
        const int ih = oh * d.sh - d.ph + r;
        if (ih < 0 || ih >= d.h) continue;
        for (int s = 0; s < d.s; ++s) {
          const int iw = ow * d.sw - d.pw + s;
          if (iw < 0 || iw >= d.w) continue;
          acc += static_cast<AT>(IO<T>::ld(x + n * xs.n + c * xs.c + ih * xs.h + iw * xs.w)) *
                 static_cast<AT>(IO<T>::ld(w + k * wsd.n + c * wsd.c + r * wsd.h + s * wsd.w));
        }
      }
    }
    if (bias) acc += static_cast<AT>(IO<T>::ld(bias + k));
    y[n * ys.n + k * ys.c + oh * ys.h + ow * ys.w] = IO<T>::cvt(static_cast<float>(acc));
  }
}

template <typename T>
__global__ void direct_conv_dx_kernel(ConvDims d, const T* __restrict__ g, Strides4 gs,
                                      const T* __restrict__ w, Strides4 wsd, T* __restrict__ dx,
                                      Strides4 xs) {
  using AT = typename Acc<T>::type;
  const int64_t total = (int64_t)d.n * d.c * d.h * d.w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int iw = t % d.w; t /= d.w;
    const int ih = t % d.h; t /= d.h;
    const int c = t % d.c; t /= d.c;
    const int n = (int)t;
    AT acc = 0;
    for (int r = 0; r < d.r; ++r) {
      const int a = ih + d.ph - r;
      if (a < 0 || a % d.sh) continue;
      const int oh = a / d.sh;
      if (oh >= d.oh) continue;
      for (int s = 0; s < d.s; ++s) {
        const int b = iw + d.pw - s;
        if (b < 0 || b % d.sw) continue;
        const int ow = b / d.sw;
        if (ow >= d.ow) continue;
        for (int k = 0; k < d.k; ++k)
          acc += static_cast<AT>(IO<T>::ld(g + n * gs.n + k * gs.c + oh * gs.h + ow * gs.w)) *
                 static_cast<AT>(IO<T>::ld(w + k * wsd.n + c * wsd.c + r * wsd.h + s * wsd.w));
      }
    }
    dx[n * xs.n + c * xs.c + ih * xs.h + iw * xs.w] = IO<T>::cvt(static_cast<float>(acc));
  }
}

// One block per (k, c) weight pair and pixel slice; each thread accumulates
// the r*s taps in float64 and the block adds its partials into `acc` (f64).
template <typename T>
__global__ void __launch_bounds__(256) direct_conv_dw_kernel(ConvDims d, const T* __restrict__ x,
                                                             Strides4 xs, const T* __restrict__ g,
                                                             Strides4 gs, double* __restrict__ acc,
                                                             int64_t pix_per_block) {
  constexpr int MAXT = 49;
  const int kc = blockIdx.x;
  const int k = kc / d.c, c = kc % d.c;
  const int taps = d.r * d.s;
  double part[MAXT];
#pragma unroll
  for (int i = 0; i < MAXT; ++i) part[i] = 0.0;
  const int64_t P = (int64_t)d.n * d.oh * d.ow;
  const int64_t p_begin = blockIdx.y * pix_per_block;
  const int64_t p_end = min(P, p_begin + pix_per_block);
  for (int64_t p = p_begin + threadIdx.x; p < p_end; p += blockDim.x) {
    int64_t t = p;
    const int ow = t % d.ow; t /= d.ow;
    const int oh = t % d.oh; t /= d.oh;
    const int n = (int)t;
    const double gv = (double)IO<T>::ld(g + n * gs.n + k * gs.c + oh * gs.h + ow * gs.w);
#pragma unroll
    for (int tap = 0; tap < MAXT; ++tap) {
      if (tap >= taps) break;
      const int r = tap / d.s, s = tap % d.s;
      const int ih = oh * d.sh - d.ph + r, iw = ow * d.sw - d.pw + s;
      if (ih < 0 || ih >= d.h || iw < 0 || iw >= d.w) continue;
      part[tap] += gv * (double)IO<T>::ld(x + n * xs.n + c * xs.c + ih * xs.h + iw * xs.w);
    }
  }
  __shared__ double red[8];
  for (int tap = 0; tap < taps; ++tap) {
    double v = part[tap < MAXT ? tap : 0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
      atomicAdd(acc + ((int64_t)k * d.c + c) * taps + tap, s);
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void f64_to_weight_kernel(ConvDims d, const double* __restrict__ acc, T* __restrict__ dw,
                                     Strides4 wsd) {
  const int64_t total = (int64_t)d.k * d.c * d.r * d.s;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int s = t % d.s; t /= d.s;
    const int r = t % d.r; t /= d.r;
    const int c = t % d.c; t /= d.c;
    const int k = (int)t;
    dw[k * wsd.n + c * wsd.c + r * wsd.h + s * wsd.w] = IO<T>::cvt((float)acc[i]);
  }
}

static Strides4 act_strides(const ConvDims& d, int layout, bool out) {
  const int64_t C = out ? d.k : d.c, H = out ? d.oh : d.h, W = out ? d.ow : d.w;
  if (layout == MS_NHWC) return Strides4{H * W * C, 1, W * C, C};
  return Strides4{C * H * W, H * W, W, 1};
}
static Strides4 wt_strides(const ConvDims& d, int wlayout) {
  if (wlayout == MS_NHWC) return Strides4{(int64_t)d.r * d.s * d.c, 1, (int64_t)d.s * d.c, d.c};
  return Strides4{(int64_t)d.c * d.r * d.s, (int64_t)d.r * d.s, d.s, 1};
}

static int grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)(b < cap ? (b > 0 ? b : 1) : cap);
}

#define MS_DT_DISPATCH(dt, ...)                                    \
  switch (dt) {                                                    \
    case MS_F32: { using T = float; __VA_ARGS__; } break;          \
    case MS_BF16: { using T = __nv_bfloat16; __VA_ARGS__; } break; \
    case MS_F16: { using T = __half; __VA_ARGS__; } break;         \
    default: set_error("bad dtype %d", dt); return MS_ERR_DTYPE;   \
  }

ms_status simt_conv_fwd(const ConvDims& d, int dt, int layout, int wlayout, const void* x,
                        const void* w, const void* bias, void* y, cudaStream_t st) {
  const int64_t total = (int64_t)d.n * d.k * d.oh * d.ow;
  MS_DT_DISPATCH(dt, direct_conv_fwd_kernel<T><<<grid_for(total), 256, 0, st>>>(
                         d, (const T*)x, act_strides(d, layout, false), (const T*)w,
                         wt_strides(d, wlayout), (const T*)bias, (T*)y,
                         act_strides(d, layout, true)));
  count_launch(1, KF_SIMT);
  return launch_status("direct_conv_fwd_kernel");
}

ms_status simt_conv_dx(const ConvDims& d, int dt, int layout, int wlayout, const void* g,
                       const void* w, void* dx, cudaStream_t st) {
  const int64_t total = (int64_t)d.n * d.c * d.h * d.w;
  MS_DT_DISPATCH(dt, direct_conv_dx_kernel<T><<<grid_for(total), 256, 0, st>>>(
                         d, (const T*)g, act_strides(d, layout, true), (const T*)w,
                         wt_strides(d, wlayout), (T*)dx, act_strides(d, layout, false)));
  count_launch(1, KF_SIMT);
  return launch_status("direct_conv_dx_kernel");
}

size_t simt_conv_dw_workspace(const ConvDims& d) {
  return sizeof(double) * (size_t)d.k * d.c * d.r * d.s;
}

ms_status simt_conv_dw(const ConvDims& d, int dt, int layout, int wlayout, const void* x,
                       const void* g, void* dw, void* ws, size_t ws_bytes, cudaStream_t st) {
  MS_CHECK_ARG(d.r * d.s <= 49, MS_ERR_UNSUPPORTED, "simt conv dW supports kernels up to 7x7");
  MS_CHECK_ARG(ws != nullptr && ws_bytes >= simt_conv_dw_workspace(d), MS_ERR_WORKSPACE,
               "simt conv dW workspace too small");
  double* acc = static_cast<double*>(ws);
  cudaMemsetAsync(acc, 0, simt_conv_dw_workspace(d), st);
  const int64_t P = (int64_t)d.n * d.oh * d.ow;
  const int64_t kc = (int64_t)d.k * d.c;
  // enough blocks to fill the GPU a few times over
  int64_t splits = ((int64_t)num_sms() * 8 + kc - 1) / kc;
  int64_t per = (P + splits - 1) / splits;
  per = ((per + 255) / 256) * 256;
  if (per < 1024) per = 1024;
  splits = (P + per - 1) / per;
  dim3 grid((unsigned)kc, (unsigned)splits);
  MS_DT_DISPATCH(dt, direct_conv_dw_kernel<T><<<grid, 256, 0, st>>>(
                         d, (const T*)x, act_strides(d, layout, false), (const T*)g,
                         act_strides(d, layout, true), acc, per);
                 f64_to_weight_kernel<T><<<grid_for(kc * d.r * d.s), 256, 0, st>>>(
                     d, acc, (T*)dw, wt_strides(d, wlayout)));
  count_launch(2, KF_SIMT);
  return launch_status("direct_conv_dw_kernel");
}

}  // namespace ms
