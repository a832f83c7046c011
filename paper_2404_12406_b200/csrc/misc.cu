// Bandwidth helpers: bias-gradient reductions, fp32 -> output dtype casts,
// conv weight repacks and the channel-pad copy used by the tcgen05 conv path.
#include "misc.cuh"

namespace ms {

// ------------------------------------------------------------------ column sums
// Row-major [rows][cols]; each thread owns 8 consecutive columns (16-byte loads
// for 16-bit data) and strides over rows; warps reduce through smem; one fp32
// atomic per column per block.
template <typename T>
__global__ void __launch_bounds__(256) colsum_kernel(int64_t rows, int64_t cols, const T* __restrict__ g,
                                                    float* __restrict__ acc, int64_t rows_per_block,
                                                    void* out, int odt, unsigned* ticket) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c0 = (blockIdx.x * 32 + lane) * 8;
  float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t r_begin = blockIdx.y * rows_per_block;
  const int64_t r_end = min(rows, r_begin + rows_per_block);
  if (c0 < cols) {
    const bool vec = (c0 + 8 <= cols) && (cols % 8 == 0) && sizeof(T) == 2;
    int64_t r = r_begin + warp;
    if (vec) {  // 4 rows per iteration: four independent 16-byte loads in flight
      for (; r + 24 < r_end; r += 32) {
        uint4 u[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = __ldg(reinterpret_cast<const uint4*>(g + (r + 8 * q) * cols + c0));
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const T* e = reinterpret_cast<const T*>(&u[q]);
#pragma unroll
          for (int j = 0; j < 8; ++j) s[j] += IO<T>::ld(e + j);
        }
      }
    }
    for (; r < r_end; r += 8) {
      const T* p = g + r * cols + c0;
      if (vec) {
        uint4 u = *reinterpret_cast<const uint4*>(p);
        const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j] += IO<T>::ld(e + j);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (c0 + j < cols) s[j] += IO<T>::ld(p + j);
      }
    }
  }
  __shared__ float red[8][256 + 8];
#pragma unroll
  for (int j = 0; j < 8; ++j) red[warp][lane * 8 + j] = s[j];
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += 256) {
    float v = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += red[w][i];
    const int64_t c = blockIdx.x * 256 + i;
    if (c < cols) atomicAdd(acc + c, v);
  }
  // the last block converts the sums to the output dtype (no separate launch;
  // the ticket is zeroed with the accumulators)
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (last) {
    __threadfence();
    for (int64_t c = threadIdx.x; c < cols; c += 256) store_from_float(out, odt, c, __ldcg(acc + c));
  }
}

// NCHW planes: block (plane chunk) reduces hw contiguous elements of one (n, c)
template <typename T>
__global__ void __launch_bounds__(256) planesum_kernel(int64_t n, int64_t c, int64_t hw,
                                                       const T* __restrict__ g, float* __restrict__ acc) {
  const int64_t plane = blockIdx.x;  // n*c planes
  const int64_t ch = plane % c;
  const T* p = g + plane * hw;
  float s = 0;
  for (int64_t i = threadIdx.x; i < hw; i += 256) s += IO<T>::ld(p + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ float red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0;
    for (int i = 0; i < 8; ++i) t += red[i];
    atomicAdd(acc + ch, t);
  }
}

template <typename T>
__global__ void f32_to_kernel(const float* __restrict__ src, T* __restrict__ dst, int64_t count,
                              const T* __restrict__ bias, int64_t bias_period) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = src[i];
    if (bias) v += IO<T>::ld(bias + (i % bias_period));
    dst[i] = IO<T>::cvt(v);
  }
}

static int grid_1d(int64_t total, int per_thread = 1) {
  int64_t b = (total / per_thread + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 32;
  if (b < 1) b = 1;
  return (int)(b < cap ? b : cap);
}

#define MS_DT_DISPATCH(dt, ...)                                    \
  switch (dt) {                                                    \
    case MS_F32: { using T = float; __VA_ARGS__; } break;          \
    case MS_BF16: { using T = __nv_bfloat16; __VA_ARGS__; } break; \
    case MS_F16: { using T = __half; __VA_ARGS__; } break;         \
    default: set_error("bad dtype %d", dt); return MS_ERR_DTYPE;   \
  }

// [cols] fp32 accumulators, then the finalize ticket
size_t colsum_workspace(int64_t cols) { return sizeof(float) * (size_t)cols + 16; }

ms_status f32_to(const float* src, void* dst, int dt, int64_t count, const void* bias,
                 int64_t bias_period, cudaStream_t st) {
  if (count <= 0) return MS_OK;
  MS_DT_DISPATCH(dt, f32_to_kernel<T><<<grid_1d(count), 256, 0, st>>>(
                         src, (T*)dst, count, (const T*)bias, bias_period > 0 ? bias_period : 1));
  count_launch();
  return launch_status("f32_to_kernel");
}

ms_status colsum(int64_t rows, int64_t cols, int dt, const void* g, void* db, int odt, void* ws,
                 cudaStream_t st) {
  float* acc = static_cast<float*>(ws);
  unsigned* ticket = reinterpret_cast<unsigned*>(acc + cols);
  cudaMemsetAsync(acc, 0, colsum_workspace(cols), st);
  const int64_t gx = (cols + 255) / 256;
  int64_t gy = ((int64_t)num_sms() * 4 + gx - 1) / gx;
  int64_t per = (rows + gy - 1) / gy;
  if (per < 64) per = 64;
  gy = (rows + per - 1) / per;
  if (gy < 1) gy = 1;
  dim3 grid((unsigned)gx, (unsigned)gy);
  MS_DT_DISPATCH(dt, colsum_kernel<T><<<grid, 256, 0, st>>>(rows, cols, (const T*)g, acc, per, db,
                                                             odt, ticket));
  count_launch();
  return launch_status("colsum_kernel");
}

ms_status planesum(int64_t n, int64_t c, int64_t hw, int dt, const void* g, void* db, int odt,
                   void* ws, cudaStream_t st) {
  float* acc = static_cast<float*>(ws);
  cudaMemsetAsync(acc, 0, sizeof(float) * c, st);
  MS_DT_DISPATCH(dt, planesum_kernel<T><<<(unsigned)(n * c), 256, 0, st>>>(n, c, hw, (const T*)g, acc));
  count_launch();
  MS_TRY(launch_status("planesum_kernel"));
  return f32_to(acc, db, odt, c, nullptr, 1, st);
}

// ------------------------------------------------------------------ repacks
// Forward weight [k][tap][cpad] (K-major rows for the B operand) from OIHW/OHWI.
template <typename T>
__global__ void repack_fprop_kernel(int K, int C, int R, int S, int cpad, int wlayout,
                                    const T* __restrict__ w, T* __restrict__ out) {
  const int64_t total = (int64_t)K * R * S * cpad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int c = t % cpad; t /= cpad;
    const int tap = t % (R * S); t /= (R * S);
    const int k = (int)t;
    const int r = tap / S, s = tap % S;
    T v = IO<T>::cvt(0.f);
    if (c < C)
      v = wlayout == MS_NHWC ? w[(((int64_t)k * R + r) * S + s) * C + c]
                             : w[(((int64_t)k * C + c) * R + r) * S + s];
    out[i] = v;
  }
}

// Input-VJP weight [c][tap][kpad] from OIHW/OHWI (B operand of the dgrad GEMM).
// kvar (nullable): multiply output-channel k by kw[k] / sqrt(kvar[k] + eps) -- a
// following eval-BatchNorm's scale folded into the input-VJP weight
// As a 32 x 32 tile transpose through shared memory: reads run along c
// (contiguous in OHWI), writes along k; one tap per blockIdx.z.
template <typename T>
__global__ void repack_dgrad_tiled_kernel(int K, int C, int RS, int kpad, int wlayout,
                                          const T* __restrict__ w, T* __restrict__ out,
                                          const void* kvar, const void* kw, int pdt, float eps) {
  __shared__ float tile[32][33];
  const int k0 = blockIdx.x * 32, c0 = blockIdx.y * 32, tap = blockIdx.z;
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + ty + 8 * i, c = c0 + tx;
    float v = 0.f;
    if (k < K && c < C) {
      v = IO<T>::ld(w + (wlayout == MS_NHWC ? ((int64_t)k * RS + tap) * C + c
                                            : ((int64_t)k * C + c) * RS + tap));
      if (kvar)
        v *= (kw ? load_as_float(kw, pdt, k) : 1.f) / sqrtf(load_as_float(kvar, pdt, k) + eps);
    }
    tile[ty + 8 * i][tx] = v;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = c0 + ty + 8 * i, k = k0 + tx;
    if (c < C && k < kpad)
      out[((int64_t)c * RS + tap) * kpad + k] = IO<T>::cvt(tile[tx][ty + 8 * i]);
  }
}

// Scatter input-VJP weight [(tap, c)][kpad] (row = one output column of the
// dY x W GEMM) from OIHW/OHWI.
template <typename T>
__global__ void repack_scatter_kernel(int K, int C, int R, int S, int kpad, int wlayout,
                                      const T* __restrict__ w, T* __restrict__ out) {
  const int64_t total = (int64_t)R * S * C * kpad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int k = t % kpad; t /= kpad;
    const int c = t % C; t /= C;
    const int tap = (int)t;
    const int r = tap / S, s = tap % S;
    T v = IO<T>::cvt(0.f);
    if (k < K)
      v = wlayout == MS_NHWC ? w[(((int64_t)k * R + r) * S + s) * C + c]
                             : w[(((int64_t)k * C + c) * R + r) * S + s];
    out[i] = v;
  }
}

// Row-segment stem weights [k][r][32]: element s*4 + c of row r = w[k][c][r][s]
template <typename T>
__global__ void repack_rowseg_kernel(int K, int C, int R, int S, int cpx, int wlayout,
                                     const T* __restrict__ w, T* __restrict__ out) {
  const int64_t total = (int64_t)K * R * 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int e = i % 32;
    const int r = (i / 32) % R;
    const int k = (int)(i / (32 * R));
    const int s = e / cpx, c = e % cpx;
    T v = IO<T>::cvt(0.f);
    if (s < S && c < C)
      v = wlayout == MS_NHWC ? w[(((int64_t)k * R + r) * S + s) * C + c]
                             : w[(((int64_t)k * C + c) * R + r) * S + s];
    out[i] = v;
  }
}

// [n][h][w][c<=CPX] -> [n][h][wp][CPX] with pw zero pixels on the left and
// zeros on the right up to wp (the row-segment conv's padded activation copy)
template <typename T, int CPX>
__global__ void pad_rowseg_kernel(int N, int H, int W, int C, int pw, int wp,
                                  const T* __restrict__ x, T* __restrict__ out) {
  const int64_t total = (int64_t)N * H * wp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int j = i % wp;
    const int64_t nh = i / wp;
    const int src = j - pw;
    T v[CPX];
#pragma unroll
    for (int c = 0; c < CPX; ++c)
      v[c] = (src >= 0 && src < W && c < C) ? x[(nh * W + src) * C + c] : IO<T>::cvt(0.f);
    T* o = out + i * CPX;
    if constexpr (sizeof(T) == 2 && CPX == 4) {
      uint2 u;
      T* e = reinterpret_cast<T*>(&u);
#pragma unroll
      for (int c = 0; c < 4; ++c) e[c] = v[c];
      *reinterpret_cast<uint2*>(o) = u;
    } else if constexpr (sizeof(T) == 2 && CPX == 8) {
      uint4 u;
      T* e = reinterpret_cast<T*>(&u);
#pragma unroll
      for (int c = 0; c < 8; ++c) e[c] = v[c];
      *reinterpret_cast<uint4*>(o) = u;
    } else {
#pragma unroll
      for (int c = 0; c < CPX; ++c) o[c] = v[c];
    }
  }
}

// fp32 [k][tap][c] accumulator -> weight gradient in OIHW/OHWI, dtype T
template <typename T>
__global__ void wgrad_finalize_kernel(int K, int C, int R, int S, int wlayout,
                                      const float* __restrict__ acc, T* __restrict__ dw) {
  const int64_t total = (int64_t)K * R * S * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = i;
    const int c = t % C; t /= C;
    const int tap = t % (R * S); t /= (R * S);
    const int k = (int)t;
    const int r = tap / S, s = tap % S;
    const int64_t o = wlayout == MS_NHWC ? i : (((int64_t)k * C + c) * R + r) * S + s;
    dw[o] = IO<T>::cvt(acc[i]);
  }
}

// NHWC channel pad: [p][c] -> [p][cpad] (zeros in c..cpad)
template <typename T>
__global__ void pad_channels_kernel(int64_t pixels, int c, int cpad, const T* __restrict__ x,
                                    T* __restrict__ out) {
  const int64_t total = pixels * cpad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ch = i % cpad;
    const int64_t p = i / cpad;
    out[i] = ch < c ? x[p * c + ch] : IO<T>::cvt(0.f);
  }
}

ms_status repack_fprop(int dt, int K, int C, int R, int S, int cpad, int wlayout, const void* w,
                       void* out, cudaStream_t st) {
  const int64_t total = (int64_t)K * R * S * cpad;
  MS_DT_DISPATCH(dt, repack_fprop_kernel<T><<<grid_1d(total), 256, 0, st>>>(
                         K, C, R, S, cpad, wlayout, (const T*)w, (T*)out));
  count_launch();
  return launch_status("repack_fprop_kernel");
}

ms_status repack_dgrad(int dt, int K, int C, int R, int S, int kpad, int wlayout, const void* w,
                       void* out, cudaStream_t st, const void* kvar, const void* kw, int pdt,
                       float eps) {
  const dim3 grid((unsigned)((kpad + 31) / 32), (unsigned)((C + 31) / 32), (unsigned)(R * S));
  MS_DT_DISPATCH(dt, repack_dgrad_tiled_kernel<T><<<grid, dim3(32, 8), 0, st>>>(
                         K, C, R * S, kpad, wlayout, (const T*)w, (T*)out, kvar, kw, pdt, eps));
  count_launch();
  return launch_status("repack_dgrad_tiled_kernel");
}

ms_status repack_scatter(int dt, int K, int C, int R, int S, int kpad, int wlayout, const void* w,
                         void* out, cudaStream_t st) {
  const int64_t total = (int64_t)R * S * C * kpad;
  MS_DT_DISPATCH(dt, repack_scatter_kernel<T><<<grid_1d(total), 256, 0, st>>>(
                         K, C, R, S, kpad, wlayout, (const T*)w, (T*)out));
  count_launch();
  return launch_status("repack_scatter_kernel");
}

ms_status repack_rowseg(int dt, int K, int C, int R, int S, int cpx, int wlayout, const void* w,
                        void* out,
                        cudaStream_t st) {
  const int64_t total = (int64_t)K * R * 32;
  MS_DT_DISPATCH(dt, repack_rowseg_kernel<T><<<grid_1d(total), 256, 0, st>>>(
                         K, C, R, S, cpx, wlayout, (const T*)w, (T*)out));
  count_launch();
  return launch_status("repack_rowseg_kernel");
}

ms_status pad_rowseg(int dt, int N, int H, int W, int C, int pw, int wp, int cpx, const void* x,
                     void* out,
                     cudaStream_t st) {
  const int64_t total = (int64_t)N * H * wp;
  if (cpx == 8) {
    MS_DT_DISPATCH(dt, (pad_rowseg_kernel<T, 8><<<grid_1d(total), 256, 0, st>>>(
                           N, H, W, C, pw, wp, (const T*)x, (T*)out)));
  } else {
    MS_DT_DISPATCH(dt, (pad_rowseg_kernel<T, 4><<<grid_1d(total), 256, 0, st>>>(
                           N, H, W, C, pw, wp, (const T*)x, (T*)out)));
  }
  count_launch();
  return launch_status("pad_rowseg_kernel");
}

ms_status wgrad_finalize(int dt, int K, int C, int R, int S, int wlayout, const float* acc,
                         void* dw, cudaStream_t st) {
  const int64_t total = (int64_t)K * R * S * C;
  MS_DT_DISPATCH(dt, wgrad_finalize_kernel<T><<<grid_1d(total), 256, 0, st>>>(
                         K, C, R, S, wlayout, acc, (T*)dw));
  count_launch();
  return launch_status("wgrad_finalize_kernel");
}

ms_status pad_channels(int dt, int64_t pixels, int c, int cpad, const void* x, void* out,
                       cudaStream_t st) {
  const int64_t total = pixels * cpad;
  MS_DT_DISPATCH(dt, pad_channels_kernel<T><<<grid_1d(total), 256, 0, st>>>(
                         pixels, c, cpad, (const T*)x, (T*)out));
  count_launch();
  return launch_status("pad_channels_kernel");
}

}  // namespace ms
