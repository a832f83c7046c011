// float32 3x3 stride-1 convolution for few channels (the Fig. 1 network:
// 8 -> 8 channels), NCHW.  float32 at rtol 1e-5 rules out
// TF32 tensor cores, and an 8-deep contraction is too narrow for them anyway,
// so this is a CUDA-core (FFMA) kernel tiled through shared memory:
//   block = 16 x 64 output pixels x all K channels; thread = 1 row x 4 columns x
//   K channels (4K accumulators); input tile (C x 18 x 66) and weights in smem.
// dX of a stride-1 conv is the same kernel on dY with W'[c][k][2-r][2-s]
// (transposed, flipped), loaded into smem in that order (numpy_impl.py:27-38).
// dW: block reduces its tile's pixels for all K*C*9 taps in float64, then one
// float64 atomic per tap (numpy_impl.py:41-51).
#include "misc.cuh"

namespace ms {
namespace {

constexpr int TH = 16, TW = 64;  // output tile per block
constexpr int PX = 4;            // output columns per thread

template <int C, int K, bool FLIP>
__global__ void __launch_bounds__(256) conv3x3_small_kernel(int N, int H, int W, int pad,
                                                            const float* __restrict__ x,
                                                            const float* __restrict__ w,
                                                            float* __restrict__ y) {
  // FLIP: x is dY (K_in = C channels here means dY channels), weights are read
  // as W'[co][ci][r][s] = W[ci][co][2-r][2-s] with W given as [C_in_of_fwd=K][...]
  __shared__ float s_in[C][TH + 2][TW + 2];
  __shared__ float s_w[K][C][9];
  const int tiles_w = (W + TW - 1) / TW, tiles_h = (H + TH - 1) / TH;
  const int n = blockIdx.x / (tiles_w * tiles_h);
  const int rem = blockIdx.x - n * tiles_w * tiles_h;
  const int h0 = (rem / tiles_w) * TH, w0 = (rem % tiles_w) * TW;
  for (int i = threadIdx.x; i < K * C * 9; i += 256) {
    const int t = i % 9, c = (i / 9) % C, k = i / (9 * C);
    float v;
    if (!FLIP) v = w[(k * C + c) * 9 + t];             // W[k][c][r][s]
    else v = w[(c * K + k) * 9 + (8 - t)];              // W[c][k][2-r][2-s]
    s_w[k][c][t] = v;
  }
  const float* xn = x + (int64_t)n * C * H * W;
  for (int i = threadIdx.x; i < C * (TH + 2) * (TW + 2); i += 256) {
    const int cc = i % (TW + 2);
    const int rr = (i / (TW + 2)) % (TH + 2);
    const int c = i / ((TW + 2) * (TH + 2));
    const int ih = h0 - pad + rr, iw = w0 - pad + cc;
    s_in[c][rr][cc] = (ih >= 0 && ih < H && iw >= 0 && iw < W) ? xn[((int64_t)c * H + ih) * W + iw]
                                                                 : 0.f;
  }
  __syncthreads();
  const int tr = threadIdx.x / (TW / PX), tc = (threadIdx.x % (TW / PX)) * PX;
  float acc[K][PX];
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int j = 0; j < PX; ++j) acc[k][j] = 0.f;
#pragma unroll 1
  for (int c = 0; c < C; ++c) {
    float in[3][PX + 2];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int j = 0; j < PX + 2; ++j) in[r][j] = s_in[c][tr + r][tc + j];
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          const float wv = s_w[k][c][r * 3 + s];
#pragma unroll
          for (int j = 0; j < PX; ++j) acc[k][j] = fmaf(wv, in[r][j + s], acc[k][j]);
        }
    }
  }
  const int oh = h0 + tr;
  if (oh >= H) return;
  float* yn = y + (int64_t)n * K * H * W;
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int j = 0; j < PX; ++j) {
      const int ow = w0 + tc + j;
      if (ow < W) yn[((int64_t)k * H + oh) * W + ow] = acc[k][j];
    }
}

constexpr int DTH = 8;  // dW tile height (static smem <= 48 KB)

// dW[k][c][r][s] = sum_{n,h,w} dY[n][k][h][w] * X[n][c][h+r-pad][w+s-pad]
template <int C, int K>
__global__ void __launch_bounds__(256) conv3x3_small_dw_kernel(int N, int H, int W, int pad,
                                                               const float* __restrict__ x,
                                                               const float* __restrict__ g,
                                                               double* __restrict__ acc) {
  __shared__ float s_in[C][DTH + 2][TW + 2];
  __shared__ float s_g[K][DTH][TW];
  const int tiles_w = (W + TW - 1) / TW, tiles_h = (H + DTH - 1) / DTH;
  const int n = blockIdx.x / (tiles_w * tiles_h);
  const int rem = blockIdx.x - n * tiles_w * tiles_h;
  const int h0 = (rem / tiles_w) * DTH, w0 = (rem % tiles_w) * TW;
  const float* xn = x + (int64_t)n * C * H * W;
  const float* gn = g + (int64_t)n * K * H * W;
  for (int i = threadIdx.x; i < C * (DTH + 2) * (TW + 2); i += 256) {
    const int cc = i % (TW + 2);
    const int rr = (i / (TW + 2)) % (DTH + 2);
    const int c = i / ((TW + 2) * (DTH + 2));
    const int ih = h0 - pad + rr, iw = w0 - pad + cc;
    s_in[c][rr][cc] = (ih >= 0 && ih < H && iw >= 0 && iw < W) ? xn[((int64_t)c * H + ih) * W + iw]
                                                                 : 0.f;
  }
  for (int i = threadIdx.x; i < K * DTH * TW; i += 256) {
    const int cc = i % TW, rr = (i / TW) % DTH, k = i / (TW * DTH);
    const int oh = h0 + rr, ow = w0 + cc;
    s_g[k][rr][cc] = (oh < H && ow < W) ? gn[((int64_t)k * H + oh) * W + ow] : 0.f;
  }
  __syncthreads();
  // outputs (k, c, t) distributed over the threads
  for (int o = threadIdx.x; o < K * C * 9; o += 256) {
    const int t = o % 9, c = (o / 9) % C, k = o / (9 * C);
    const int r = t / 3, s = t % 3;
    double sum = 0.0;
#pragma unroll 4
    for (int rr = 0; rr < DTH; ++rr) {
      float part = 0.f;
#pragma unroll 8
      for (int cc = 0; cc < TW; ++cc) part = fmaf(s_g[k][rr][cc], s_in[c][rr + r][cc + s], part);
      sum += part;
    }
    atomicAdd(acc + o, sum);
  }
}

template <int C, int K>
ms_status launch_small(bool flip, int N, int H, int W, int pad, const float* x, const float* w,
                       float* y, cudaStream_t st) {
  const int blocks = N * ((H + TH - 1) / TH) * ((W + TW - 1) / TW);
  if (flip) conv3x3_small_kernel<C, K, true><<<blocks, 256, 0, st>>>(N, H, W, pad, x, w, y);
  else conv3x3_small_kernel<C, K, false><<<blocks, 256, 0, st>>>(N, H, W, pad, x, w, y);
  count_launch(1, KF_SIMT);
  return launch_status("conv3x3_small_kernel");
}

__global__ void f64_to_f32_kernel(const double* a, float* b, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (float)a[i];
}

}  // namespace

// Returns MS_ERR_UNSUPPORTED when the geometry is not the specialised one.
bool conv3x3_tf32_applies(const ConvDims& d, int layout, int wlayout, int pass);
ms_status conv3x3_tf32(int pass, const ConvDims& d, const void* a, const void* b, void* out,
                       cudaStream_t st);
size_t conv3x3_c8_dw_workspace(const ConvDims& d);
ms_status conv3x3_c8_dw(const ConvDims& d, const void* x, const void* g, void* dw, void* ws,
                        size_t ws_bytes, cudaStream_t st);

size_t small_conv_fp32_workspace(const ConvDims& d, int pass) {
  if (pass == MS_CONV_DW && conv3x3_tf32_applies(d, MS_NCHW, MS_NCHW, MS_CONV_DW))
    return conv3x3_c8_dw_workspace(d);
  return pass == MS_CONV_DW ? sizeof(double) * 576 : 0;
}

ms_status small_conv_fp32(int pass, const ConvDims& d, int layout, int wlayout, const void* a,
                          const void* b, void* out, void* ws, size_t ws_bytes, cudaStream_t st) {
  // tensor cores (3xTF32) for fwd / dX, the CUDA-core partial-sum kernel for dW
  if (conv3x3_tf32_applies(d, layout, wlayout, pass)) {
    if (pass == MS_CONV_DW) return conv3x3_c8_dw(d, a, b, out, ws, ws_bytes, st);
    return conv3x3_tf32(pass, d, a, b, out, st);
  }
  const bool ok = layout == MS_NCHW && wlayout == MS_NCHW && d.r == 3 && d.s == 3 && d.sh == 1 &&
                  d.sw == 1 && d.ph == 1 && d.pw == 1 && d.c == 8 && d.k == 8;
  if (!ok) return MS_ERR_UNSUPPORTED;
  if (pass == MS_CONV_FWD)
    return launch_small<8, 8>(false, d.n, d.h, d.w, d.ph, (const float*)a, (const float*)b,
                              (float*)out, st);
  if (pass == MS_CONV_DX) {  // size-preserving: the transposed conv also pads by 1
    return launch_small<8, 8>(true, d.n, d.oh, d.ow, 1, (const float*)a, (const float*)b,
                              (float*)out, st);
  }
  // weight gradient: a = x, b = dY
  MS_CHECK_ARG(ws && ws_bytes >= sizeof(double) * 576, MS_ERR_WORKSPACE, "small dw workspace");
  double* acc = static_cast<double*>(ws);
  cudaMemsetAsync(acc, 0, sizeof(double) * 576, st);
  const int blocks = d.n * ((d.h + DTH - 1) / DTH) * ((d.w + TW - 1) / TW);
  conv3x3_small_dw_kernel<8, 8><<<blocks, 256, 0, st>>>(d.n, d.h, d.w, d.ph, (const float*)a,
                                                         (const float*)b, acc);
  f64_to_f32_kernel<<<3, 256, 0, st>>>(acc, (float*)out, 576);
  count_launch(2, KF_SIMT);
  return launch_status("conv3x3_small_dw_kernel");
}

}  // namespace ms
