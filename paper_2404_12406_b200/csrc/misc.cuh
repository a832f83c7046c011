#pragma once

#include "simt.cuh"

namespace ms {

ms_status repack_fprop(int dt, int K, int C, int R, int S, int cpad, int wlayout, const void* w,
                       void* out, cudaStream_t st);
ms_status repack_dgrad(int dt, int K, int C, int R, int S, int kpad, int wlayout, const void* w,
                       void* out, cudaStream_t st, const void* kvar = nullptr,
                       const void* kw = nullptr, int pdt = 0, float eps = 0.f);
ms_status repack_scatter(int dt, int K, int C, int R, int S, int kpad, int wlayout, const void* w,
                         void* out, cudaStream_t st);
ms_status repack_rowseg(int dt, int K, int C, int R, int S, int cpx, int wlayout, const void* w,
                        void* out, cudaStream_t st);
ms_status pad_rowseg(int dt, int N, int H, int W, int C, int pw, int wp, int cpx, const void* x,
                     void* out, cudaStream_t st);
ms_status wgrad_finalize(int dt, int K, int C, int R, int S, int wlayout, const float* acc,
                         void* dw, cudaStream_t st);
ms_status pad_channels(int dt, int64_t pixels, int c, int cpad, const void* x, void* out,
                       cudaStream_t st);

// 3-channel 7x7 stride-2 pad-3 stem input-VJP with register col2im (stem_dgrad.cu)
bool stem_dgrad_ok(int dt, int layout, int c, int r, int s, int sh, int sw, int ph, int pw,
                   int64_t ow, int64_t k);
ms_status stem_dgrad(int dt, int n, int h, int w, int p, int q, int k, const void* dy,
                     const void* wt, void* dx, cudaStream_t st);

// <= 4-channel 7x7 stride-2 pad-3 stem forward reading overlapping input rows in
// place (stem_dgrad.cu); xp = pad_rowseg output, wb = stem_fprop_weight_bytes(k)
bool stem_fprop_ok(int dt, int layout, int c, int r, int s, int sh, int sw, int ph, int pw,
                   int64_t ow, int64_t k);
size_t stem_fprop_weight_bytes(int k);
ms_status stem_fprop(int dt, int n, int h, int wp, int p, int q, int k, int c, int wlayout,
                     const void* xp, const void* w, void* wb, const void* bias, void* y,
                     cudaStream_t st, const BnFold& bn = BnFold{}, int relu = 0,
                     uint8_t* mask = nullptr);

// 3x3/1/1 64->64-channel convolution, halo-tiled (conv3x3.cu); transpose = 1 is
// the input-VJP of the same conv (x = dY, y = dX)
bool conv3x3_halo_ok(int dt, int layout, int c, int k, int r, int s, int sh, int sw, int ph,
                     int pw, int w);
size_t conv3x3_halo_workspace();
ms_status conv3x3_halo(int dt, int n, int h, int w, int wlayout, int transpose, const void* x,
                       const void* wt, void* ws, void* y, const BnFold& bn, const void* bias, const void* resid, int relu, uint8_t* mask,
                       const void* ks_var, const void* ks_w, int ks_pdt, float ks_eps,
                       cudaStream_t st, const uint8_t* keep_in = nullptr, int bn_post = 0);

// elementwise GELU (erf form) and its VJP dx = g * gelu'(pre) (misc.cu)
ms_status gelu_fwd(int64_t n, int dt, const void* x, void* y, cudaStream_t st);
ms_status gelu_bwd(int64_t n, int dt, const void* g, const void* pre, void* dx, cudaStream_t st);

// y += r elementwise (16-bit: rounded once, as torch's add)
ms_status add_inplace(int64_t n, int dt, void* y, const void* r, cudaStream_t st);

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }
inline size_t align256(size_t v) { return (v + 255) & ~static_cast<size_t>(255); }

}  // namespace ms
