/*
 * memsave_b200.h — C ABI of the B200 (sm_100a) selective-save layer kernels.
 *
 * This is the drop-in boundary for the hot path of arxiv 2404.12406
 * ("Lowering PyTorch's Memory Consumption for Selective Differentiation").
 * Each entry point replaces one kernel-level operation of the reference
 * (`/root/reference/pkg/src/leantape`, a CPU numpy/numba restatement of the
 * paper) or one VJP that the reference specifies.  The save
 * decision itself (which of X / W is kept for backward) stays in the caller:
 * these functions only compute, and each backward product is a separate entry
 * point so the caller launches exactly the products that were requested.
 *
 *   ms_conv2d_fwd   ← leantape.kernels.conv2d_fwd   (kernels/__init__.py:26,
 *                      numba_impl.py:109-116, numpy_impl.py:12-24)
 *   ms_conv2d_dx    ← leantape.kernels.conv2d_dx    (kernels/__init__.py:27,
 *                      numba_impl.py:119-124, numpy_impl.py:27-38)
 *   ms_conv2d_dw    ← leantape.kernels.conv2d_dw    (kernels/__init__.py:28,
 *                      numba_impl.py:127-132, numpy_impl.py:41-51)
 *   ms_linear_fwd / ms_linear_dx / ms_linear_dw / ms_bias_grad
 *                   ← forward_linear and its VJPs
 *   ms_bn_eval_fwd / ms_bn_eval_bwd
 *                   ← forward_batchnorm2d, Eval mode
 *
 * Conventions (mirroring the reference kernel boundary):
 *   - plain device pointers and sizes; no framework types in any signature;
 *   - outputs are allocated by the CALLER (the reference allocates fresh
 *     outputs itself; here the caller does it so that its allocator sees every
 *     byte) and fully overwritten; inputs are read-only;
 *   - every call is asynchronous and stream-ordered on `stream` (a
 *     cudaStream_t passed as void*; NULL = legacy default stream); no host
 *     synchronisation, no device allocation, re-entrant;
 *   - workspaces are sized by the matching *_workspace() query and passed in;
 *   - there is no CPU path: host pointers are an error of the caller;
 *   - errors return a non-zero ms_status; ms_last_error() gives a message.
 */
#ifndef MEMSAVE_B200_H
#define MEMSAVE_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MS_API __attribute__((visibility("default")))
#else
#define MS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MS_OK = 0,
  MS_ERR_SHAPE = 1,       /* inconsistent or non-positive sizes          */
  MS_ERR_DTYPE = 2,       /* unsupported dtype combination               */
  MS_ERR_ALIGN = 3,       /* pointer / stride alignment not met          */
  MS_ERR_UNSUPPORTED = 4, /* geometry outside what the kernels implement */
  MS_ERR_LAUNCH = 5,      /* CUDA launch / driver error                  */
  MS_ERR_WORKSPACE = 6    /* workspace missing or too small              */
} ms_status;

typedef enum { MS_F32 = 0, MS_BF16 = 1, MS_F16 = 2 } ms_dtype;

/* activation layout; for weights MS_NCHW means OIHW, MS_NHWC means OHWI */
typedef enum { MS_NCHW = 0, MS_NHWC = 1 } ms_layout;

typedef enum { MS_CONV_FWD = 0, MS_CONV_DX = 1, MS_CONV_DW = 2 } ms_conv_pass;

/* 2-d cross-correlation geometry (OH = (H+2p-kh)//s+1). */
typedef struct {
  int64_t n, c, h, w;   /* input batch, channels, height, width        */
  int64_t k, r, s;      /* output channels, kernel height, kernel width */
  int32_t stride_h, stride_w;
  int32_t pad_h, pad_w;
  int32_t layout;       /* ms_layout of x / y / dx / dy                */
  int32_t wlayout;      /* ms_layout of w / dw                         */
  int32_t dtype;        /* ms_dtype of every tensor operand            */
} ms_conv_desc;

/* ------------------------------------------------------------ conv2d */
MS_API int64_t ms_conv2d_out_h(const ms_conv_desc* d);
MS_API int64_t ms_conv2d_out_w(const ms_conv_desc* d);
/* bytes of device workspace the given pass needs (0 = none) */
MS_API size_t ms_conv2d_workspace(const ms_conv_desc* d, int32_t pass);
/* y = conv(x, w) (+ bias[k] if bias != NULL; bias has dtype d->dtype) */
MS_API ms_status ms_conv2d_fwd(const ms_conv_desc* d, const void* x, const void* w, const void* bias,
                        void* y, void* ws, size_t ws_bytes, void* stream);
/* dx = conv2d input-VJP of dy with w (transpose convolution) */
MS_API ms_status ms_conv2d_dx(const ms_conv_desc* d, const void* dy, const void* w, void* dx, void* ws,
                       size_t ws_bytes, void* stream);
/* dw = conv2d weight-VJP of dy with x; dw has layout d->wlayout and dtype d->dtype */
MS_API ms_status ms_conv2d_dw(const ms_conv_desc* d, const void* x, const void* dy, void* dw, void* ws,
                       size_t ws_bytes, void* stream);
/* db[k] = sum of dy over n, oh, ow (dy in d->layout, db in d->dtype);
 * ws_bytes >= ms_bias_grad_workspace(0, d->k, d->dtype) */
MS_API ms_status ms_conv2d_db(const ms_conv_desc* d, const void* dy, void* db, void* ws,
                       size_t ws_bytes, void* stream);

/* ------------------------------------------------------------ linear
 * x: [M, K] row-major, w: [N, K] row-major, y/dy: [M, N] row-major.      */
MS_API size_t ms_linear_workspace(int64_t M, int64_t N, int64_t K, int32_t dtype, int32_t pass);
MS_API ms_status ms_linear_fwd(int64_t M, int64_t N, int64_t K, int32_t dtype, const void* x,
                        const void* w, const void* bias, void* y, void* ws, size_t ws_bytes,
                        void* stream);
/* Linear -> GELU (erf form, torch gelu approximate='none') in one call: pre =
 * x·wᵀ + b (kept: it is what the GELU's VJP reads) and y = gelu(pre), the GELU
 * applied to the rounded pre in the GEMM epilogue (tcgen05 path) or by a second
 * launch (other paths).  ws as ms_linear_workspace(M, N, K, dtype, 0).  Replaces
 * the pair forward_linear (kernels/__init__.py:26-28) + the consumer's GELU.  */
MS_API ms_status ms_linear_gelu_fwd(int64_t M, int64_t N, int64_t K, int32_t dtype,
                             const void* x, const void* w, const void* bias, void* pre,
                             void* y, void* ws, size_t ws_bytes, void* stream);
/* Linear -> dropout -> + residual (a transformer block's output projection)
 * in one call: y = r + dropout_p(x·wᵀ + b), each intermediate rounded to
 * `dtype` as the separate launches round it, the mask drawn exactly as
 * ms_dropout_fwd(numel = M*N, seed, stream_id, p, generator) draws it (so
 * ms_dropout_bwd replays it for the VJP).  p = 0: y = r + (x·wᵀ + b).  r: [M, N]
 * like y (y must not alias r).  ws as ms_linear_workspace(M, N, K, dtype, 0).  */
MS_API ms_status ms_linear_dropout_add_fwd(int64_t M, int64_t N, int64_t K, int32_t dtype,
                                    const void* x, const void* w, const void* bias,
                                    const void* r, double p, uint64_t seed, uint64_t stream_id,
                                    int32_t generator, void* y, void* ws, size_t ws_bytes,
                                    void* stream);
MS_API ms_status ms_linear_dx(int64_t M, int64_t N, int64_t K, int32_t dtype, const void* dy,
                       const void* w, void* dx, void* ws, size_t ws_bytes, void* stream);
MS_API ms_status ms_linear_dw(int64_t M, int64_t N, int64_t K, int32_t dtype, const void* x,
                       const void* dy, void* dw, void* ws, size_t ws_bytes, void* stream);
/* db[c] = sum_r g[r, c] for a row-major [rows, cols] matrix */
MS_API size_t ms_bias_grad_workspace(int64_t rows, int64_t cols, int32_t dtype);
MS_API ms_status ms_bias_grad(int64_t rows, int64_t cols, int32_t dtype, const void* g, void* db,
                       void* ws, size_t ws_bytes, void* stream);

/* GELU (erf form) and its VJP dx = g * gelu'(pre), elementwise over numel  */
MS_API ms_status ms_gelu_fwd(int64_t numel, int32_t dtype, const void* x, void* y, void* stream);
MS_API ms_status ms_gelu_bwd(int64_t numel, int32_t dtype, const void* g, const void* pre,
                      void* dx, void* stream);

/* ------------------------------------------------------------ batchnorm2d (eval)
 * x/y/dy/dx: [n, c, hw] (MS_NCHW) or [n, hw, c] (MS_NHWC) in `dtype`.
 * mean/var/weight/bias/dw/db: [c] in `pdtype`; weight/bias may be NULL
 * (affine=False).  dw needs x; dx needs only weight and var.  */
MS_API size_t ms_bn_eval_workspace(int64_t n, int64_t c, int64_t hw, int32_t layout);
MS_API ms_status ms_bn_eval_fwd(int64_t n, int64_t c, int64_t hw, int32_t layout, int32_t dtype,
                         int32_t pdtype, const void* x, const void* mean, const void* var,
                         const void* weight, const void* bias, double eps, void* y, void* ws,
                         size_t ws_bytes, void* stream);
MS_API ms_status ms_bn_eval_bwd(int64_t n, int64_t c, int64_t hw, int32_t layout, int32_t dtype,
                         int32_t pdtype, const void* dy, const void* x_or_null, const void* mean,
                         const void* var, const void* weight, double eps, void* dx_or_null,
                         void* dw_or_null, void* db_or_null, void* ws, size_t ws_bytes,
                         void* stream);

/* BN-eval -> ReLU in one pass, for BN layers whose affine is trainable (so the
 * conv cannot absorb them): y = max(x*s + t, 0) with the ReLU bit mask (NHWC,
 * 16-bit, C % 8 == 0, C <= 2048; x [n*hw][c]).  The backward applies the mask
 * to dy and then the BN-eval VJP (dx, dw, db as requested; x needed for dw).
 * Saved set = the union of the two rows (rules.py:84-87, 98-101).
 * MS_ERR_UNSUPPORTED outside that layout.                                   */
MS_API ms_status ms_bn_eval_relu_fwd(int64_t n, int64_t c, int64_t hw, int32_t dtype,
                                     int32_t pdtype, const void* x, const void* mean,
                                     const void* var, const void* weight_or_null,
                                     const void* bias_or_null, double eps, void* y,
                                     void* mask_or_null, void* stream);
MS_API ms_status ms_bn_eval_relu_bwd(int64_t n, int64_t c, int64_t hw, int32_t dtype,
                                     int32_t pdtype, const void* dy, const void* mask,
                                     const void* x_or_null, const void* mean, const void* var,
                                     const void* weight_or_null, double eps, void* dx_or_null,
                                     void* dw_or_null, void* db_or_null, void* ws,
                                     size_t ws_bytes, void* stream);
/* The same with the residual add of a bottleneck block between BN and ReLU:
 * y = max(bf16(x*s + t) + residual, 0) (the BN output rounded as the unfused
 * chain stores it).  The backward also writes dy * keep to dresidual (the add's
 * gradient for its other operand), in the same pass.                        */
MS_API ms_status ms_bn_eval_add_relu_fwd(int64_t n, int64_t c, int64_t hw, int32_t dtype,
                                         int32_t pdtype, const void* x, const void* residual,
                                         const void* mean, const void* var,
                                         const void* weight_or_null, const void* bias_or_null,
                                         double eps, void* y, void* mask_or_null, void* stream);
MS_API ms_status ms_bn_eval_add_relu_bwd(int64_t n, int64_t c, int64_t hw, int32_t dtype,
                                         int32_t pdtype, const void* dy, const void* mask,
                                         const void* x_or_null, const void* mean,
                                         const void* var, const void* weight_or_null, double eps,
                                         void* dx_or_null, void* dresidual_or_null,
                                         void* dw_or_null, void* db_or_null, void* ws,
                                         size_t ws_bytes, void* stream);

/* ------------------------------------------------------------ relu (bit mask)
 * MemSave ReLU (rules.py:98-101, saved.py:53-71): y = max(x, 0) over a dense
 * buffer of `numel` elements (any memory format: the mask follows storage
 * order); mask bit i = (x_i > 0), ceil(numel/8) bytes, bit j of byte i/8.
 * y may alias x; dx may alias g.                                            */
MS_API ms_status ms_relu_fwd(int64_t numel, int32_t dtype, const void* x, void* y,
                             void* mask_or_null, void* stream);
MS_API ms_status ms_relu_bwd(int64_t numel, int32_t dtype, const void* g, const void* mask,
                             void* dx, void* stream);

/* y = relu(a + b) with the ReLU's bit mask: the residual add of a ResNet block
 * fused with the ReLU that follows it (backward = ms_relu_bwd, whose result is
 * the gradient of both a and b).  y may alias a or b.                       */
MS_API ms_status ms_add_relu_fwd(int64_t numel, int32_t dtype, const void* a, const void* b,
                                 void* y, void* mask_or_null, void* stream);

/* ------------------------------------------------------------ conv2d + batchnorm2d(eval) [+ relu]
 * The conv -> eval-BN (-> ReLU) chain of a frozen-normalisation network in one
 * launch: the BN affine y = conv*s + t (s = w/sqrt(var+eps), t = b - mean*s)
 * and the ReLU (keep bits to mask, as ms_relu_fwd) run in the conv's tcgen05
 * epilogue; nothing is materialised between the three layers.  The saved set
 * is the union of the three layers' rows (conv: W iff x needs a grad; BN with
 * frozen parameters: nothing; ReLU: the bit mask).  16-bit NHWC, K % 8 == 0
 * (MS_ERR_UNSUPPORTED otherwise: the caller runs the three layers).
 * Workspace: ms_conv2d_bn_workspace(d).  Backward: ms_bn_relu_bwd then
 * ms_conv2d_dx / ms_conv2d_dw.                                              */
MS_API size_t ms_conv2d_bn_workspace(const ms_conv_desc* d);
MS_API ms_status ms_conv2d_bn_fwd(const ms_conv_desc* d, const void* x, const void* w,
                                  const void* bias_or_null, const void* bn_mean,
                                  const void* bn_var, const void* bn_weight_or_null,
                                  const void* bn_bias_or_null, int32_t bn_pdtype, double eps,
                                  const void* residual_or_null, int32_t relu, void* y,
                                  void* mask_or_null, void* ws, size_t ws_bytes, void* stream);
/* residual_or_null: a tensor shaped like y added after the BN affine and before
 * the ReLU (the conv -> BN -> add -> ReLU join of a ResNet block).  bn_mean =
 * bn_var = NULL: no BN, i.e. conv [+ bias] -> ReLU (VGG).                   */
/* dX of a conv inside a fused chain, everything in the dgrad epilogue:
 *   dx = [keep ? (dgrad(dy, W * s) + addend) : 0] * s_in
 * s = w/sqrt(var+eps) of a following eval-BN without ReLU (bn_var = NULL: 1),
 * folded into the repacked dgrad weight so dY is used as is;
 * addend_or_null: shaped like dx, the gradient x receives from its other
 * consumer (identity / downsample branch of a ResNet block);
 * keep_or_null: the bit mask of the ReLU that produced x (1 bit per element,
 * storage order, 4-byte aligned) -- that ReLU's backward;
 * s_in = in_weight/sqrt(in_var+in_eps) of the eval-BN before that ReLU
 * (in_var = NULL: 1).  The three replace separate passes over dx (the
 * engine's gradient sum, ms_relu_bwd / ms_bn_relu_bwd).
 * Workspace: ms_conv2d_workspace(d, MS_CONV_DX).  MS_ERR_UNSUPPORTED outside
 * the tcgen05 dgrad (16-bit NHWC, phase GEMM or 3x3 halo kernel).           */
MS_API ms_status ms_conv2d_bn_dx(const ms_conv_desc* d, const void* dy, const void* w,
                                 const void* bn_var_or_null, const void* bn_weight_or_null,
                                 int32_t bn_pdtype, double eps, const void* addend_or_null,
                                 const void* keep_or_null, const void* in_var_or_null,
                                 const void* in_weight_or_null, int32_t in_pdtype,
                                 double in_eps, void* dx, void* ws, size_t ws_bytes,
                                 void* stream);
/* dx = g * keep * w/sqrt(var+eps) per channel (NHWC, C % 8 == 0, 16-bit);
 * mask_or_null = NULL for a conv -> BN chain without ReLU.                  */
MS_API ms_status ms_bn_relu_bwd(int64_t numel, int64_t c, int32_t dtype, int32_t pdtype,
                                const void* g, const void* mask_or_null, const void* mean,
                                const void* var, const void* weight_or_null, double eps,
                                void* dx, void* stream);

/* ------------------------------------------------------------ maxpool2d (index map)
 * MemSave MaxPool2d (rules.py:108-109, saved.py:111-125, kernels
 * numpy_impl.py:54-78): the argmax is kept as the window-local offset
 * r*kw + s in one byte per output element (the reference keeps a 4-byte flat
 * index); first occurrence wins ties; padding is -inf.                      */
typedef struct {
  int64_t n, c, h, w;
  int32_t kh, kw, stride_h, stride_w, pad_h, pad_w;
  int32_t layout; /* ms_layout of x / y / g / dx / idx */
  int32_t dtype;
} ms_pool_desc;
MS_API int64_t ms_maxpool2d_out_h(const ms_pool_desc* p);
MS_API int64_t ms_maxpool2d_out_w(const ms_pool_desc* p);
MS_API ms_status ms_maxpool2d_fwd(const ms_pool_desc* p, const void* x, void* y,
                                  void* idx_or_null, void* stream);
MS_API ms_status ms_maxpool2d_bwd(const ms_pool_desc* p, const void* g, const void* idx,
                                  void* dx, void* stream);
/* The same, with the backward of the ReLU [+ eval-BN] that produced x applied
 * before the store: dx = keep ? dx * s_in : 0 (keep: that ReLU's bit mask in
 * storage order; s_in = in_weight/sqrt(in_var+in_eps), in_var = NULL: 1) --
 * replaces a separate ms_relu_bwd / ms_bn_relu_bwd pass over dx.
 * MS_ERR_UNSUPPORTED outside the NHWC 3x3/2/1 kernel (C % 8 == 0, C <= 512). */
MS_API ms_status ms_maxpool2d_relu_bwd(const ms_pool_desc* p, const void* g, const void* idx,
                                       const void* keep, const void* in_var_or_null,
                                       const void* in_weight_or_null, int32_t in_pdtype,
                                       double in_eps, void* dx, void* stream);

/* ------------------------------------------------------------ conv_transpose2d
 * ConvTranspose2d forward (rules.py:68-71; SPEC.md forward_conv_transpose2d:
 * "forward equals conv2d's input-VJP with the same kernel"): `d` describes
 * the equivalent conv2d, whose INPUT is y ([n][c][h][w], c = out channels of
 * the transposed conv) and whose OUTPUT is x ([n][k][oh][ow]); w is
 * [k][c][r][s] (= the ConvTranspose2d weight [C_in][C_out][kh][kw]).  bias
 * ([c], nullable) is added in the same pass.  Workspace: ms_conv2d_workspace(d,
 * MS_CONV_DX).  dX and dW of the transposed conv are ms_conv2d_fwd(d, g, w) and
 * ms_conv2d_dw(d, g, x).                                                    */
MS_API ms_status ms_conv_transpose2d_fwd(const ms_conv_desc* d, const void* x, const void* w,
                                         const void* bias_or_null, void* y, void* ws,
                                         size_t ws_bytes, void* stream);

/* ------------------------------------------------------------ dropout (RNG replay)
 * MemSave Dropout (rules.py:103-106, saved.py:91-108 RngSeed; SPEC.md
 * forward_dropout): the keep mask is a pure function of (seed, stream_id, p,
 * element index); kept elements are scaled by 1/(1-p).  Backward regenerates
 * the same mask: nothing O(numel) is stored.  Generators:
 *   MS_RNG_PHILOX4X32      Philox4x32-10 (Random123), key = seed, counter =
 *                          (block, stream_id); element 4j+i kept iff word i of
 *                          block j >= ceil(p * 2^32).  Near HBM speed.
 *   MS_RNG_PHILOX4X64_REF  the reference generator leantape.core.Rng(seed,
 *                          stream_id).uniform() (core.py:100-124; numpy
 *                          Philox4x64-10 keyed [seed, stream_id]); element i
 *                          kept iff U_i >= p: bit-identical to the reference's
 *                          mask (seeds < 2^63).  ~4x the integer work.
 * mask_or_null receives the keep flags at one byte per element (the NAIVE
 * StoreMask convention, tests).  y may alias x; dx may alias g; 0 <= p < 1. */
typedef enum { MS_RNG_PHILOX4X32 = 0, MS_RNG_PHILOX4X64_REF = 1 } ms_rng;
MS_API ms_status ms_dropout_fwd(int64_t numel, int32_t dtype, const void* x, void* y,
                                uint64_t seed, uint64_t stream_id, double p, int32_t generator,
                                void* mask_or_null, void* stream);
MS_API ms_status ms_dropout_bwd(int64_t numel, int32_t dtype, const void* g, void* dx,
                                uint64_t seed, uint64_t stream_id, double p, int32_t generator,
                                void* stream);

/* ------------------------------------------------------------ layernorm
 * LayerNorm over the last dimension (rules.py:89-96; SPEC.md forward_layernorm):
 * x is [rows][dim] row-major; w / b ([dim], dtype of x) may be NULL; mean and
 * rstd are fp32 [rows] (the "stats" the rule saves; NULL in inference).
 * Backward products are independent: dx, dw, db may each be NULL.  dw / db
 * need the workspace sized by ms_layernorm_workspace.                       */
MS_API size_t ms_layernorm_workspace(int64_t rows, int64_t dim, int32_t dtype);
MS_API ms_status ms_layernorm_fwd(int64_t rows, int64_t dim, int32_t dtype, const void* x,
                                  const void* w_or_null, const void* b_or_null, double eps,
                                  void* y, float* mean_or_null, float* rstd_or_null,
                                  void* stream);
MS_API ms_status ms_layernorm_bwd(int64_t rows, int64_t dim, int32_t dtype, const void* g,
                                  const void* x, const float* mean, const float* rstd,
                                  const void* w_or_null, void* dx_or_null, void* dw_or_null,
                                  void* db_or_null, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------ misc */
MS_API const char* ms_status_string(int32_t status);
MS_API const char* ms_last_error(void);
MS_API int32_t ms_version(void);
/* number of kernels this library has launched since load (all threads) */
MS_API int64_t ms_launch_count(void);
/* launches by kernel family: [0] tcgen05 GEMM/implicit-GEMM, [1] SIMT (CUDA-core)
 * GEMM/conv, [2] batchnorm, [3] reductions / casts / repacks */
MS_API void ms_launch_stats(int64_t* out4);
/* Caller contract for the calling thread: `device_plus_one` = d + 1 declares
 * that CUDA device d owns every operand of the following calls (the PyTorch op
 * layer passes the tensors' device), so entry points skip their per-call
 * pointer-attribute query and only make d current; 0 (default) restores the
 * query.  ctypes / FFI callers need not care. */
MS_API void ms_set_device_bound(int32_t device_plus_one);

#ifdef __cplusplus
}
#endif
#endif /* MEMSAVE_B200_H */
