#pragma once

#include "host.cuh"

namespace ms {

struct ConvDims {
  int n, c, h, w;    // input
  int k, r, s;       // output channels, kernel
  int oh, ow;        // output spatial
  int sh, sw, ph, pw;
};

ms_status simt_gemm(int dt, int M, int N, int K, const void* A, int64_t sam, int64_t sak,
                    const void* B, int64_t sbk, int64_t sbn, const void* bias, void* C,
                    int64_t ldc, cudaStream_t st);

ms_status simt_conv_fwd(const ConvDims& d, int dt, int layout, int wlayout, const void* x,
                        const void* w, const void* bias, void* y, cudaStream_t st);
ms_status simt_conv_dx(const ConvDims& d, int dt, int layout, int wlayout, const void* g,
                       const void* w, void* dx, cudaStream_t st);
size_t simt_conv_dw_workspace(const ConvDims& d);
ms_status simt_conv_dw(const ConvDims& d, int dt, int layout, int wlayout, const void* x,
                       const void* g, void* dw, void* ws, size_t ws_bytes, cudaStream_t st);

// specialised float32 3x3/1 conv for 8 -> 8 channels, NCHW (smallconv.cu);
// MS_ERR_UNSUPPORTED when the geometry does not match
ms_status small_conv_fp32(int pass, const ConvDims& d, int layout, int wlayout, const void* a,
                          const void* b, void* out, void* ws, size_t ws_bytes, cudaStream_t st);
size_t small_conv_fp32_workspace(const ConvDims& d, int pass);

// reductions / elementwise helpers (misc.cu)
size_t colsum_workspace(int64_t cols);
// db[c] = sum_r g[r*ld + c] (row-major [rows][cols]) -> dtype `odt`
ms_status colsum(int64_t rows, int64_t cols, int dt, const void* g, void* db, int odt, void* ws,
                 cudaStream_t st);
// db[c] = sum over n, hw of g[n][c][hw] (NCHW planes)
ms_status planesum(int64_t n, int64_t c, int64_t hw, int dt, const void* g, void* db, int odt,
                   void* ws, cudaStream_t st);
// out[i] = (dtype) f32[i]
ms_status f32_to(const float* src, void* dst, int dt, int64_t count, const void* bias,
                 int64_t bias_period, cudaStream_t st);

}  // namespace ms
