// PyTorch custom-op layer over the C ABI (include/memsave_b200.h):
// TORCH_LIBRARY(memsave) defines one functional op per kernel-level entry
// point, implemented for the CUDA key (allocate the outputs from the caching
// allocator, call the C ABI on the current stream under a device guard) and
// for the Meta key (the same allocations, no launch), so the ops are visible to
// FakeTensor / torch.compile / torch.export and to CUDA-graph capture.
//
// The save decision for Linear is made here, in a C++ autograd Function
// (memsave::linear, Autograd key): at forward time X is kept only if W requires
// a gradient and W only if X does (reference rules.py:133-141), and backward
// calls only the requested products -- without the per-call cost of a Python
// autograd.Function (Linear is the most frequent memsave op in the transformer
// steps).  The other layers decide in the autograd.Functions of functional.py.
// Reference anchors: leantape.kernels.conv2d_fwd / conv2d_dx / conv2d_dw
// (kernels/__init__.py:26-28), the Linear and BN-eval VJPs
// and the autograd primitive the paper wraps them in.
#include <ATen/ATen.h>
#include <ATen/core/dispatch/Dispatcher.h>
#include <ATen/cuda/CUDAContext.h>
#include <c10/cuda/CUDAGuard.h>
#include <torch/csrc/autograd/custom_function.h>
#include <torch/library.h>

#include <optional>
#include <tuple>
#include <vector>

#include "memsave_b200.h"

namespace {

using at::IntArrayRef;
using at::Tensor;
using OptT = std::optional<Tensor>;

int dtc(at::ScalarType s) {
  switch (s) {
    case at::kFloat: return MS_F32;
    case at::kBFloat16: return MS_BF16;
    case at::kHalf: return MS_F16;
    default: TORCH_CHECK(false, "memsave: unsupported dtype ", s,
                         "; expected float32, bfloat16 or float16");
  }
  return -1;
}

bool has(const OptT& t) { return t.has_value() && t->defined(); }
const void* cp(const Tensor& t) { return t.defined() && t.numel() ? t.const_data_ptr() : nullptr; }
const void* cp(const OptT& t) { return has(t) ? cp(*t) : nullptr; }
void* mp(const Tensor& t) { return t.defined() && t.numel() ? t.data_ptr() : nullptr; }

// device guard + current stream; tells the library the device is already bound
struct Launch {
  c10::cuda::CUDAGuard guard;
  void* stream;
  explicit Launch(const Tensor& t)
      : guard(t.device()), stream(at::cuda::getCurrentCUDAStream(t.device().index()).stream()) {
    ms_set_device_bound((int32_t)t.device().index() + 1);
  }
  ~Launch() { ms_set_device_bound(0); }
};

void ok(ms_status s, const char* what) {
  TORCH_CHECK(s == MS_OK, "memsave::", what, " failed: ", ms_status_string(s), ": ",
              ms_last_error());
}

Tensor wsp(size_t nb, const Tensor& like) {
  return nb ? at::empty({(int64_t)nb}, like.options().dtype(at::kByte)) : Tensor();
}

at::MemoryFormat mfmt(int64_t layout) {
  return layout == MS_NHWC ? at::MemoryFormat::ChannelsLast : at::MemoryFormat::Contiguous;
}

Tensor empty4(IntArrayRef shape, const Tensor& like, int64_t layout) {
  return at::empty(shape, like.options().memory_format(mfmt(layout)));
}

Tensor nothing(const Tensor& like) { return at::empty({0}, like.options()); }

Tensor as_dtype(const OptT& t, at::ScalarType s) {
  if (!has(t)) return Tensor();
  return t->to(s).contiguous();
}

Tensor mask_for(int64_t numel, const Tensor& like, bool want) {
  return at::empty({want ? (numel + 7) / 8 : 0}, like.options().dtype(at::kByte));
}

ms_conv_desc conv_desc(IntArrayRef xs, IntArrayRef ws, IntArrayRef stride, IntArrayRef pad,
                       int64_t layout, int64_t wlayout, int dt) {
  TORCH_CHECK(xs.size() == 4 && ws.size() == 4, "conv2d: expected 4-d input and weight");
  TORCH_CHECK(ws[1] == xs[1], "conv2d: input channels ", xs[1], " != weight channels ", ws[1],
              " (groups unsupported)");
  ms_conv_desc d;
  d.n = xs[0];
  d.c = xs[1];
  d.h = xs[2];
  d.w = xs[3];
  d.k = ws[0];
  d.r = ws[2];
  d.s = ws[3];
  d.stride_h = (int32_t)stride[0];
  d.stride_w = (int32_t)stride[1];
  d.pad_h = (int32_t)pad[0];
  d.pad_w = (int32_t)pad[1];
  d.layout = (int32_t)layout;
  d.wlayout = (int32_t)wlayout;
  d.dtype = dt;
  return d;
}

std::vector<int64_t> conv_out(const ms_conv_desc& d) {
  const int64_t oh = (d.h + 2 * d.pad_h - d.r) / d.stride_h + 1;
  const int64_t ow = (d.w + 2 * d.pad_w - d.s) / d.stride_w + 1;
  TORCH_CHECK(oh > 0 && ow > 0, "conv2d: empty output");
  return {d.n, d.k, oh, ow};
}

ms_pool_desc pool_desc(IntArrayRef xs, IntArrayRef k, IntArrayRef s, IntArrayRef p,
                       int64_t layout, int dt) {
  ms_pool_desc d;
  d.n = xs[0];
  d.c = xs[1];
  d.h = xs[2];
  d.w = xs[3];
  d.kh = (int32_t)k[0];
  d.kw = (int32_t)k[1];
  d.stride_h = (int32_t)s[0];
  d.stride_w = (int32_t)s[1];
  d.pad_h = (int32_t)p[0];
  d.pad_w = (int32_t)p[1];
  d.layout = (int32_t)layout;
  d.dtype = dt;
  return d;
}

// ================================================================ linear
Tensor linear_fwd(const Tensor& x, const Tensor& w, const OptT& b) {
  const int64_t N = w.size(0), K = w.size(1);
  TORCH_CHECK(x.size(-1) == K, "linear: input last dim ", x.size(-1), " != in_features ", K);
  auto shape = x.sizes().vec();
  shape.back() = N;
  Tensor y = at::empty(shape, x.options());
  if (x.is_meta()) return y;
  Tensor x2 = x.reshape({-1, K}).contiguous(), wc = w.contiguous();
  Tensor bb = as_dtype(b, x.scalar_type());
  const int64_t M = x2.size(0);
  const int dt = dtc(x.scalar_type());
  Launch L(x);
  const size_t nb = ms_linear_workspace(M, N, K, dt, 0);
  Tensor ws = wsp(nb, x);
  ok(ms_linear_fwd(M, N, K, dt, cp(x2), cp(wc), cp(bb), mp(y), mp(ws), nb, L.stream),
     "linear_fwd");
  return y;
}

Tensor linear_dx(const Tensor& g, const Tensor& w, IntArrayRef x_shape) {
  const int64_t N = g.size(-1), K = w.size(1);
  Tensor dx = at::empty(x_shape, g.options());
  if (g.is_meta()) return dx;
  Tensor g2 = g.reshape({-1, N}).contiguous(), wc = w.contiguous();
  const int64_t M = g2.size(0);
  const int dt = dtc(g.scalar_type());
  Launch L(g);
  const size_t nb = ms_linear_workspace(M, N, K, dt, 1);
  Tensor ws = wsp(nb, g);
  ok(ms_linear_dx(M, N, K, dt, cp(g2), cp(wc), mp(dx), mp(ws), nb, L.stream), "linear_dx");
  return dx;
}

Tensor linear_dw(const Tensor& x, const Tensor& g) {
  const int64_t N = g.size(-1), K = x.size(-1);
  Tensor dw = at::empty({N, K}, g.options());
  if (g.is_meta()) return dw;
  Tensor x2 = x.reshape({-1, K}).contiguous(), g2 = g.reshape({-1, N}).contiguous();
  const int64_t M = g2.size(0);
  const int dt = dtc(g.scalar_type());
  Launch L(g);
  const size_t nb = ms_linear_workspace(M, N, K, dt, 2);
  Tensor ws = wsp(nb, g);
  ok(ms_linear_dw(M, N, K, dt, cp(x2), cp(g2), mp(dw), mp(ws), nb, L.stream), "linear_dw");
  return dw;
}

// pre = x·wᵀ + b and y = gelu(pre) in one GEMM (GELU in the epilogue)
std::tuple<Tensor, Tensor> linear_gelu_fwd(const Tensor& x, const Tensor& w, const OptT& b) {
  const int64_t N = w.size(0), K = w.size(1);
  TORCH_CHECK(x.size(-1) == K, "linear_gelu: input last dim ", x.size(-1), " != in_features ", K);
  auto shape = x.sizes().vec();
  shape.back() = N;
  Tensor pre = at::empty(shape, x.options()), y = at::empty(shape, x.options());
  if (x.is_meta()) return {pre, y};
  Tensor x2 = x.reshape({-1, K}).contiguous(), wc = w.contiguous();
  Tensor bb = as_dtype(b, x.scalar_type());
  const int64_t M = x2.size(0);
  const int dt = dtc(x.scalar_type());
  Launch L(x);
  const size_t nb = ms_linear_workspace(M, N, K, dt, 0);
  Tensor ws = wsp(nb, x);
  ok(ms_linear_gelu_fwd(M, N, K, dt, cp(x2), cp(wc), cp(bb), mp(pre), mp(y), mp(ws), nb,
                        L.stream),
     "linear_gelu_fwd");
  return {pre, y};
}

// y = r + dropout_p(x·wᵀ + b) in one GEMM (dropout and the add in the epilogue)
Tensor linear_dropout_add_fwd(const Tensor& x, const Tensor& w, const OptT& b, const Tensor& r,
                              double p, int64_t seed, int64_t stream_id, int64_t gen) {
  const int64_t N = w.size(0), K = w.size(1);
  TORCH_CHECK(x.size(-1) == K, "linear_dropout_add: input last dim ", x.size(-1),
              " != in_features ", K);
  auto shape = x.sizes().vec();
  shape.back() = N;
  TORCH_CHECK(r.sizes().vec() == shape && r.scalar_type() == x.scalar_type(),
              "linear_dropout_add: residual ", r.sizes(), " does not match the output ",
              c10::IntArrayRef(shape));
  Tensor y = at::empty(shape, x.options());
  if (x.is_meta()) return y;
  Tensor x2 = x.reshape({-1, K}).contiguous(), wc = w.contiguous(), rc = r.contiguous();
  Tensor bb = as_dtype(b, x.scalar_type());
  const int64_t M = x2.size(0);
  const int dt = dtc(x.scalar_type());
  Launch L(x);
  const size_t nb = ms_linear_workspace(M, N, K, dt, 0);
  Tensor ws = wsp(nb, x);
  ok(ms_linear_dropout_add_fwd(M, N, K, dt, cp(x2), cp(wc), cp(bb), cp(rc), p, (uint64_t)seed,
                               (uint64_t)stream_id, (int32_t)gen, mp(y), mp(ws), nb, L.stream),
     "linear_dropout_add_fwd");
  return y;
}

Tensor gelu_fwd(const Tensor& x) {
  Tensor xc = x.contiguous();
  Tensor y = at::empty_like(xc);
  if (x.is_meta()) return y;
  Launch L(x);
  ok(ms_gelu_fwd(xc.numel(), dtc(x.scalar_type()), cp(xc), mp(y), L.stream), "gelu_fwd");
  return y;
}

// dx = g * gelu'(pre)
Tensor gelu_bwd(const Tensor& g, const Tensor& pre) {
  TORCH_CHECK(g.sizes() == pre.sizes() && g.scalar_type() == pre.scalar_type(),
              "gelu_bwd: gradient and pre-activation differ in shape or dtype");
  Tensor gc = g.contiguous(), pc = pre.contiguous();
  Tensor dx = at::empty_like(gc);
  if (g.is_meta()) return dx;
  Launch L(g);
  ok(ms_gelu_bwd(gc.numel(), dtc(g.scalar_type()), cp(gc), cp(pc), mp(dx), L.stream), "gelu_bwd");
  return dx;
}

// db[c] = sum_r g[r, c] over g viewed [rows, cols]
Tensor bias_grad(const Tensor& g, int64_t cols) {
  Tensor db = at::empty({cols}, g.options());
  if (g.is_meta()) return db;
  Tensor g2 = g.reshape({-1, cols}).contiguous();
  const int dt = dtc(g.scalar_type());
  Launch L(g);
  const size_t nb = ms_bias_grad_workspace(g2.size(0), cols, dt);
  Tensor ws = wsp(nb, g);
  ok(ms_bias_grad(g2.size(0), cols, dt, cp(g2), mp(db), mp(ws), nb, L.stream), "bias_grad");
  return db;
}

// ================================================================ conv2d
Tensor conv2d_fwd(const Tensor& x, const Tensor& w, const OptT& b, IntArrayRef stride,
                  IntArrayRef padding, int64_t layout, int64_t wlayout) {
  const int dt = dtc(x.scalar_type());
  ms_conv_desc d = conv_desc(x.sizes(), w.sizes(), stride, padding, layout, wlayout, dt);
  Tensor y = empty4(conv_out(d), x, layout);
  if (x.is_meta()) return y;
  Tensor bb = as_dtype(b, x.scalar_type());
  Launch L(x);
  const size_t nb = ms_conv2d_workspace(&d, MS_CONV_FWD);
  Tensor ws = wsp(nb, x);
  ok(ms_conv2d_fwd(&d, cp(x), cp(w), cp(bb), mp(y), mp(ws), nb, L.stream), "conv2d_fwd");
  return y;
}

Tensor conv2d_dx(const Tensor& g, const Tensor& w, IntArrayRef x_shape, IntArrayRef stride,
                 IntArrayRef padding, int64_t layout, int64_t wlayout) {
  const int dt = dtc(g.scalar_type());
  ms_conv_desc d = conv_desc(x_shape, w.sizes(), stride, padding, layout, wlayout, dt);
  Tensor dx = empty4(x_shape, g, layout);
  if (g.is_meta()) return dx;
  Launch L(g);
  const size_t nb = ms_conv2d_workspace(&d, MS_CONV_DX);
  Tensor ws = wsp(nb, g);
  ok(ms_conv2d_dx(&d, cp(g), cp(w), mp(dx), mp(ws), nb, L.stream), "conv2d_dx");
  return dx;
}

Tensor conv2d_dw(const Tensor& x, const Tensor& g, IntArrayRef w_shape, IntArrayRef stride,
                 IntArrayRef padding, int64_t layout, int64_t wlayout) {
  const int dt = dtc(g.scalar_type());
  ms_conv_desc d = conv_desc(x.sizes(), w_shape, stride, padding, layout, wlayout, dt);
  Tensor dw = empty4(w_shape, g, wlayout);
  if (g.is_meta()) return dw;
  Launch L(g);
  const size_t nb = ms_conv2d_workspace(&d, MS_CONV_DW);
  Tensor ws = wsp(nb, g);
  ok(ms_conv2d_dw(&d, cp(x), cp(g), mp(dw), mp(ws), nb, L.stream), "conv2d_dw");
  return dw;
}

Tensor conv2d_db(const Tensor& g, IntArrayRef x_shape, IntArrayRef w_shape, IntArrayRef stride,
                 IntArrayRef padding, int64_t layout, int64_t wlayout) {
  const int dt = dtc(g.scalar_type());
  ms_conv_desc d = conv_desc(x_shape, w_shape, stride, padding, layout, wlayout, dt);
  Tensor db = at::empty({d.k}, g.options());
  if (g.is_meta()) return db;
  Launch L(g);
  const size_t nb = ms_bias_grad_workspace(0, d.k, dt);  // fp32 sums + finalize ticket
  Tensor ws = wsp(nb, g);
  ok(ms_conv2d_db(&d, cp(g), mp(db), mp(ws), nb, L.stream), "conv2d_db");
  return db;
}

// forward of ConvTranspose2d = the input-VJP of the conv2d with input conv_x_shape
Tensor conv_transpose2d_fwd(const Tensor& x, const Tensor& w, const OptT& b,
                            IntArrayRef conv_x_shape, IntArrayRef stride, IntArrayRef padding,
                            int64_t layout, int64_t wlayout) {
  const int dt = dtc(x.scalar_type());
  ms_conv_desc d = conv_desc(conv_x_shape, w.sizes(), stride, padding, layout, wlayout, dt);
  Tensor y = empty4(conv_x_shape, x, layout);
  if (x.is_meta()) return y;
  Tensor bb = as_dtype(b, x.scalar_type());
  Launch L(x);
  const size_t nb = ms_conv2d_workspace(&d, MS_CONV_DX);
  Tensor ws = wsp(nb, x);
  ok(ms_conv_transpose2d_fwd(&d, cp(x), cp(w), cp(bb), mp(y), mp(ws), nb, L.stream),
     "conv_transpose2d_fwd");
  return y;
}

// ================================================================ batchnorm2d (eval)
Tensor bn_eval_fwd(const Tensor& x, const Tensor& mean, const Tensor& var, const OptT& w,
                   const OptT& b, double eps, int64_t layout) {
  Tensor y = at::empty_like(x);
  if (x.is_meta()) return y;
  const auto pdt = var.scalar_type();
  Tensor m = mean.to(pdt).contiguous(), v = var.contiguous();
  Tensor wt = as_dtype(w, pdt), bt = as_dtype(b, pdt);
  Launch L(x);
  ok(ms_bn_eval_fwd(x.size(0), x.size(1), x.size(2) * x.size(3), (int32_t)layout,
                    dtc(x.scalar_type()), dtc(pdt), cp(x), cp(m), cp(v), cp(wt), cp(bt), eps,
                    mp(y), nullptr, 0, L.stream),
     "bn_eval_fwd");
  return y;
}

// returns (dx, dwdb): dwdb is [2, C] in the statistics dtype (row 0 = dW, row 1 =
// db; allocated iff either is requested), unrequested products are empty
std::tuple<Tensor, Tensor> bn_eval_bwd(const Tensor& g, const OptT& x, const Tensor& mean,
                                       const Tensor& var, const OptT& w, double eps,
                                       int64_t layout, bool need_dx, bool need_dw,
                                       bool need_db) {
  const int64_t c = g.size(1);
  const auto pdt = var.scalar_type();
  Tensor dx = need_dx ? at::empty_like(g) : nothing(g);
  Tensor dwdb = at::empty({(need_dw || need_db) ? 2 : 0, c}, g.options().dtype(pdt));
  if (g.is_meta()) return {dx, dwdb};
  TORCH_CHECK(!need_dw || has(x), "bn_eval_bwd: dW needs the saved input");
  Tensor m = mean.to(pdt).contiguous(), v = var.contiguous(), wt = as_dtype(w, pdt);
  const int64_t n = g.size(0), hw = g.size(2) * g.size(3);
  Launch L(g);
  const size_t nb = (need_dw || need_db) ? ms_bn_eval_workspace(n, c, hw, (int32_t)layout) : 0;
  Tensor ws = wsp(nb, g);
  char* base = (need_dw || need_db) ? (char*)dwdb.data_ptr() : nullptr;
  const size_t row = (size_t)c * dwdb.element_size();
  ok(ms_bn_eval_bwd(n, c, hw, (int32_t)layout, dtc(g.scalar_type()), dtc(pdt), cp(g),
                    need_dw ? cp(x) : nullptr, cp(m), cp(v), cp(wt), eps,
                    need_dx ? mp(dx) : nullptr, need_dw ? (void*)base : nullptr,
                    need_db ? (void*)(base + row) : nullptr, mp(ws), nb, L.stream),
     "bn_eval_bwd");
  return {dx, dwdb};
}

// relu(bn(x) [+ residual]) in one pass (NHWC 16-bit); (y, keep bit mask)
std::tuple<Tensor, Tensor> bn_relu_fwd(const Tensor& x, const OptT& residual, const Tensor& mean,
                                       const Tensor& var, const OptT& w, const OptT& b,
                                       double eps, bool want_mask) {
  Tensor y = at::empty_like(x);
  Tensor mask = mask_for(x.numel(), x, want_mask);
  if (x.is_meta()) return {y, mask};
  const auto pdt = var.scalar_type();
  Tensor m = mean.to(pdt).contiguous(), v = var.contiguous();
  Tensor wt = as_dtype(w, pdt), bt = as_dtype(b, pdt);
  const int64_t n = x.size(0), c = x.size(1), hw = x.size(2) * x.size(3);
  Launch L(x);
  if (has(residual)) {
    TORCH_CHECK(residual->sizes() == x.sizes() && residual->scalar_type() == x.scalar_type(),
                "bn+add+relu: residual must match the BN input's shape and dtype");
    ok(ms_bn_eval_add_relu_fwd(n, c, hw, dtc(x.scalar_type()), dtc(pdt), cp(x), cp(residual),
                               cp(m), cp(v), cp(wt), cp(bt), eps, mp(y),
                               want_mask ? mp(mask) : nullptr, L.stream),
       "bn_eval_add_relu_fwd");
  } else {
    ok(ms_bn_eval_relu_fwd(n, c, hw, dtc(x.scalar_type()), dtc(pdt), cp(x), cp(m), cp(v), cp(wt),
                           cp(bt), eps, mp(y), want_mask ? mp(mask) : nullptr, L.stream),
       "bn_eval_relu_fwd");
  }
  return {y, mask};
}

// backward of relu(bn(x) [+ r]): (dx, dr, dwdb[2, C])
std::tuple<Tensor, Tensor, Tensor> bn_add_relu_bwd(const Tensor& g, const Tensor& mask,
                                                   const OptT& x, const Tensor& mean,
                                                   const Tensor& var, const OptT& w, double eps,
                                                   bool need_dx, bool need_dr, bool need_dw,
                                                   bool need_db) {
  const int64_t c = g.size(1);
  const auto pdt = var.scalar_type();
  Tensor dx = need_dx ? at::empty_like(g) : nothing(g);
  Tensor dr = need_dr ? at::empty_like(g) : nothing(g);
  Tensor dwdb = at::empty({(need_dw || need_db) ? 2 : 0, c}, g.options().dtype(pdt));
  if (g.is_meta()) return {dx, dr, dwdb};
  TORCH_CHECK(!need_dw || has(x), "bn_add_relu_bwd: dW needs the saved input");
  Tensor m = mean.to(pdt).contiguous(), v = var.contiguous(), wt = as_dtype(w, pdt);
  const int64_t n = g.size(0), hw = g.size(2) * g.size(3);
  Launch L(g);
  const size_t nb = (need_dw || need_db) ? ms_bn_eval_workspace(n, c, hw, MS_NHWC) : 0;
  Tensor ws = wsp(nb, g);
  char* base = (need_dw || need_db) ? (char*)dwdb.data_ptr() : nullptr;
  const size_t row = (size_t)c * dwdb.element_size();
  ok(ms_bn_eval_add_relu_bwd(n, c, hw, dtc(g.scalar_type()), dtc(pdt), cp(g), cp(mask),
                             need_dw ? cp(x) : nullptr, cp(m), cp(v), cp(wt), eps,
                             need_dx ? mp(dx) : nullptr, need_dr ? mp(dr) : nullptr,
                             need_dw ? (void*)base : nullptr,
                             need_db ? (void*)(base + row) : nullptr, mp(ws), nb, L.stream),
     "bn_eval_add_relu_bwd");
  return {dx, dr, dwdb};
}

// g * keep * w/sqrt(var+eps) per channel (NHWC, C = g.size(1)); keep nullable
Tensor bn_relu_bwd(const Tensor& g, const OptT& keep, const Tensor& mean, const Tensor& var,
                   const OptT& w, double eps) {
  Tensor out = at::empty_like(g);
  if (g.is_meta()) return out;
  Launch L(g);
  ok(ms_bn_relu_bwd(g.numel(), g.size(1), dtc(g.scalar_type()), dtc(mean.scalar_type()), cp(g),
                    cp(keep), cp(mean), cp(var), cp(w), eps, mp(out), L.stream),
     "bn_relu_bwd");
  return out;
}

// ================================================================ relu / add+relu (bit mask)
std::tuple<Tensor, Tensor> relu_fwd(const Tensor& x, bool want_mask) {
  Tensor y = at::empty_like(x);
  Tensor mask = mask_for(x.numel(), x, want_mask);
  if (x.is_meta()) return {y, mask};
  Launch L(x);
  ok(ms_relu_fwd(x.numel(), dtc(x.scalar_type()), cp(x), mp(y), want_mask ? mp(mask) : nullptr,
                 L.stream),
     "relu_fwd");
  return {y, mask};
}

Tensor relu_fwd_(Tensor& x, bool want_mask) {
  Tensor mask = mask_for(x.numel(), x, want_mask);
  if (x.is_meta()) return mask;
  Launch L(x);
  ok(ms_relu_fwd(x.numel(), dtc(x.scalar_type()), cp(x), mp(x), want_mask ? mp(mask) : nullptr,
                 L.stream),
     "relu_fwd_");
  return mask;
}

Tensor relu_bwd(const Tensor& g, const Tensor& mask) {
  Tensor dx = at::empty_like(g);
  if (g.is_meta()) return dx;
  Launch L(g);
  ok(ms_relu_bwd(g.numel(), dtc(g.scalar_type()), cp(g), cp(mask), mp(dx), L.stream),
     "relu_bwd");
  return dx;
}

std::tuple<Tensor, Tensor> add_relu_fwd(const Tensor& a, const Tensor& b, bool want_mask) {
  Tensor y = at::empty_like(a);
  Tensor mask = mask_for(a.numel(), a, want_mask);
  if (a.is_meta()) return {y, mask};
  Launch L(a);
  ok(ms_add_relu_fwd(a.numel(), dtc(a.scalar_type()), cp(a), cp(b), mp(y),
                     want_mask ? mp(mask) : nullptr, L.stream),
     "add_relu_fwd");
  return {y, mask};
}

// ================================================================ maxpool2d (index map)
std::tuple<Tensor, Tensor> maxpool2d_fwd(const Tensor& x, IntArrayRef kernel, IntArrayRef stride,
                                         IntArrayRef padding, int64_t layout, bool want_idx) {
  ms_pool_desc d = pool_desc(x.sizes(), kernel, stride, padding, layout, dtc(x.scalar_type()));
  const int64_t oh = (d.h + 2 * d.pad_h - d.kh) / d.stride_h + 1;
  const int64_t ow = (d.w + 2 * d.pad_w - d.kw) / d.stride_w + 1;
  Tensor y = empty4({d.n, d.c, oh, ow}, x, layout);
  Tensor idx = want_idx ? at::empty({d.n, d.c, oh, ow},
                                    x.options().dtype(at::kByte).memory_format(mfmt(layout)))
                        : at::empty({0}, x.options().dtype(at::kByte));
  if (x.is_meta()) return {y, idx};
  Launch L(x);
  ok(ms_maxpool2d_fwd(&d, cp(x), mp(y), want_idx ? mp(idx) : nullptr, L.stream),
     "maxpool2d_fwd");
  return {y, idx};
}

Tensor maxpool2d_bwd(const Tensor& g, const Tensor& idx, IntArrayRef x_shape, IntArrayRef kernel,
                     IntArrayRef stride, IntArrayRef padding, int64_t layout) {
  ms_pool_desc d = pool_desc(x_shape, kernel, stride, padding, layout, dtc(g.scalar_type()));
  Tensor dx = empty4(x_shape, g, layout);
  if (g.is_meta()) return dx;
  Launch L(g);
  ok(ms_maxpool2d_bwd(&d, cp(g), cp(idx), mp(dx), L.stream), "maxpool2d_bwd");
  return dx;
}

// the pool backward with the producer ReLU [+ eval-BN]'s backward at the store;
// geometries the fused kernel does not cover run as the two passes
Tensor maxpool2d_relu_bwd(const Tensor& g, const Tensor& idx, const Tensor& keep,
                          const OptT& in_mean, const OptT& in_var, const OptT& in_w,
                          double in_eps, IntArrayRef x_shape, IntArrayRef kernel,
                          IntArrayRef stride, IntArrayRef padding, int64_t layout) {
  ms_pool_desc d = pool_desc(x_shape, kernel, stride, padding, layout, dtc(g.scalar_type()));
  Tensor dx = empty4(x_shape, g, layout);
  if (g.is_meta()) return dx;
  Launch L(g);
  const int pdt = has(in_var) ? dtc(in_var->scalar_type()) : 0;
  ms_status s = ms_maxpool2d_relu_bwd(&d, cp(g), cp(idx), cp(keep), cp(in_var), cp(in_w), pdt,
                                      in_eps, mp(dx), L.stream);
  if (s == MS_OK) return dx;
  TORCH_CHECK(s == MS_ERR_UNSUPPORTED, "memsave::maxpool2d_relu_bwd failed: ",
              ms_status_string(s), ": ", ms_last_error());
  ok(ms_maxpool2d_bwd(&d, cp(g), cp(idx), mp(dx), L.stream), "maxpool2d_bwd");
  Tensor out = at::empty_like(dx);
  if (has(in_var)) {
    ok(ms_bn_relu_bwd(dx.numel(), dx.size(1), dtc(dx.scalar_type()), pdt, cp(dx), cp(keep),
                      cp(in_mean), cp(in_var), cp(in_w), in_eps, mp(out), L.stream),
       "bn_relu_bwd");
  } else {
    ok(ms_relu_bwd(dx.numel(), dtc(dx.scalar_type()), cp(dx), cp(keep), mp(out), L.stream),
       "relu_bwd");
  }
  return out;
}

// ================================================================ dropout (RNG replay)
Tensor dropout_fwd(const Tensor& x, double p, int64_t seed, int64_t stream_id, int64_t gen) {
  Tensor y = at::empty_like(x);
  if (x.is_meta()) return y;
  Launch L(x);
  ok(ms_dropout_fwd(x.numel(), dtc(x.scalar_type()), cp(x), mp(y), (uint64_t)seed,
                    (uint64_t)stream_id, p, (int32_t)gen, nullptr, L.stream),
     "dropout_fwd");
  return y;
}

void dropout_fwd_(Tensor& x, double p, int64_t seed, int64_t stream_id, int64_t gen) {
  if (x.is_meta()) return;
  Launch L(x);
  ok(ms_dropout_fwd(x.numel(), dtc(x.scalar_type()), cp(x), mp(x), (uint64_t)seed,
                    (uint64_t)stream_id, p, (int32_t)gen, nullptr, L.stream),
     "dropout_fwd_");
}

Tensor dropout_bwd(const Tensor& g, double p, int64_t seed, int64_t stream_id, int64_t gen) {
  Tensor dx = at::empty_like(g);
  if (g.is_meta()) return dx;
  Launch L(g);
  ok(ms_dropout_bwd(g.numel(), dtc(g.scalar_type()), cp(g), mp(dx), (uint64_t)seed,
                    (uint64_t)stream_id, p, (int32_t)gen, L.stream),
     "dropout_bwd");
  return dx;
}

// ================================================================ layernorm
// x contiguous [rows, dim] (any leading shape); (y, mean, rstd) with the fp32
// per-row statistics only when want_stats
std::tuple<Tensor, Tensor, Tensor> layernorm_fwd(const Tensor& x, const OptT& w, const OptT& b,
                                                 double eps, int64_t dim, bool want_stats) {
  const int64_t rows = dim ? x.numel() / dim : 0;
  Tensor y = at::empty_like(x);
  auto f32 = x.options().dtype(at::kFloat);
  Tensor mean = at::empty({want_stats ? rows : 0}, f32);
  Tensor rstd = at::empty({want_stats ? rows : 0}, f32);
  if (x.is_meta()) return {y, mean, rstd};
  Tensor wt = as_dtype(w, x.scalar_type()), bt = as_dtype(b, x.scalar_type());
  Launch L(x);
  ok(ms_layernorm_fwd(rows, dim, dtc(x.scalar_type()), cp(x), cp(wt), cp(bt), eps, mp(y),
                      want_stats ? mean.data_ptr<float>() : nullptr,
                      want_stats ? rstd.data_ptr<float>() : nullptr, L.stream),
     "layernorm_fwd");
  return {y, mean, rstd};
}

std::tuple<Tensor, Tensor, Tensor> layernorm_bwd(const Tensor& g, const Tensor& x,
                                                 const Tensor& mean, const Tensor& rstd,
                                                 const OptT& w, int64_t dim, bool need_dx,
                                                 bool need_dw, bool need_db) {
  const int64_t rows = dim ? g.numel() / dim : 0;
  Tensor dx = need_dx ? at::empty_like(g) : nothing(g);
  Tensor dw = at::empty({need_dw ? dim : 0}, g.options());
  Tensor db = at::empty({need_db ? dim : 0}, g.options());
  if (g.is_meta()) return {dx, dw, db};
  const int dt = dtc(g.scalar_type());
  Launch L(g);
  const size_t nb = (need_dw || need_db) ? ms_layernorm_workspace(rows, dim, dt) : 0;
  Tensor ws = wsp(nb, g);
  ok(ms_layernorm_bwd(rows, dim, dt, cp(g), cp(x), mean.const_data_ptr<float>(),
                      rstd.const_data_ptr<float>(), cp(w), need_dx ? mp(dx) : nullptr,
                      need_dw ? mp(dw) : nullptr, need_db ? mp(db) : nullptr, mp(ws), nb,
                      L.stream),
     "layernorm_bwd");
  return {dx, dw, db};
}

// ================================================================ fused conv chains
// relu?(bn?(conv(x) + bias) [+ residual]) in one tcgen05 launch: (y, keep mask)
std::tuple<Tensor, Tensor> conv2d_bn_fwd(const Tensor& x, const Tensor& w, const OptT& bias,
                                         const OptT& mean, const OptT& var, const OptT& bn_w,
                                         const OptT& bn_b, double eps, const OptT& residual,
                                         bool relu, bool want_mask, IntArrayRef stride,
                                         IntArrayRef padding, int64_t layout, int64_t wlayout) {
  const int dt = dtc(x.scalar_type());
  ms_conv_desc d = conv_desc(x.sizes(), w.sizes(), stride, padding, layout, wlayout, dt);
  auto oshape = conv_out(d);
  Tensor y = empty4(oshape, x, layout);
  Tensor mask = mask_for(oshape[0] * oshape[1] * oshape[2] * oshape[3], x, relu && want_mask);
  if (x.is_meta()) return {y, mask};
  Tensor bb = as_dtype(bias, x.scalar_type());
  Tensor res = has(residual) ? (layout == MS_NHWC
                                    ? residual->contiguous(at::MemoryFormat::ChannelsLast)
                                    : residual->contiguous())
                             : Tensor();
  if (res.defined())
    TORCH_CHECK(res.sizes() == y.sizes(), "conv2d_bn_fwd: residual shape ", res.sizes(),
                " != output shape ", y.sizes());
  Launch L(x);
  const size_t nb = ms_conv2d_bn_workspace(&d);
  Tensor ws = wsp(nb, x);
  ok(ms_conv2d_bn_fwd(&d, cp(x), cp(w), cp(bb), cp(mean), cp(var), cp(bn_w), cp(bn_b),
                      has(mean) ? dtc(mean->scalar_type()) : dt, eps, cp(res), relu ? 1 : 0,
                      mp(y), (relu && want_mask) ? mp(mask) : nullptr, mp(ws), nb, L.stream),
     "conv2d_bn_fwd");
  return {y, mask};
}

// dX of a conv inside a fused chain with everything in the dgrad epilogue:
//   dx = [keep ? dgrad(g, W * s) + addend : 0] * s_in
// s = bn_w / sqrt(var + eps) of the BN after the conv (bn_var null: none);
// keep / s_in = the backward of the ReLU [+ BN] that produced x.  Geometries the
// fused epilogue does not cover run as the separate passes (same result).
Tensor conv2d_bn_dx(const Tensor& g, const Tensor& w, const OptT& bn_var, const OptT& bn_w,
                    double eps, const OptT& addend, const OptT& keep, const OptT& in_mean,
                    const OptT& in_var, const OptT& in_w, double in_eps, IntArrayRef x_shape,
                    IntArrayRef stride, IntArrayRef padding, int64_t layout, int64_t wlayout) {
  const int dt = dtc(g.scalar_type());
  ms_conv_desc d = conv_desc(x_shape, w.sizes(), stride, padding, layout, wlayout, dt);
  Tensor dx = empty4(x_shape, g, layout);
  if (g.is_meta()) return dx;
  Tensor add = has(addend) ? (layout == MS_NHWC
                                  ? addend->contiguous(at::MemoryFormat::ChannelsLast)
                                  : addend->contiguous())
                           : Tensor();
  Launch L(g);
  const size_t nb = ms_conv2d_workspace(&d, MS_CONV_DX);
  Tensor ws = wsp(nb, g);
  const int in_pdt = has(in_var) ? dtc(in_var->scalar_type()) : dt;
  ms_status s = ms_conv2d_bn_dx(&d, cp(g), cp(w), cp(bn_var), cp(bn_w),
                                has(bn_var) ? dtc(bn_var->scalar_type()) : dt, eps, cp(add),
                                cp(keep), cp(in_var), cp(in_w), in_pdt, in_eps, mp(dx), mp(ws),
                                nb, L.stream);
  if (s == MS_OK) return dx;
  TORCH_CHECK(s == MS_ERR_UNSUPPORTED, "memsave::conv2d_bn_dx failed: ", ms_status_string(s),
              ": ", ms_last_error());
  // the separate passes: BN scale folded into a weight copy (weight-sized), dgrad,
  // addend, ReLU [+ BN] backward
  Tensor wk = w;
  if (has(bn_var)) {
    Tensor sc = at::rsqrt(bn_var->to(at::kFloat) + eps);
    if (has(bn_w)) sc = sc * bn_w->to(at::kFloat);
    wk = (w.to(at::kFloat) * sc.view({-1, 1, 1, 1})).to(w.scalar_type());
    wk = wlayout == MS_NHWC ? wk.contiguous(at::MemoryFormat::ChannelsLast) : wk.contiguous();
  }
  ok(ms_conv2d_dx(&d, cp(g), cp(wk), mp(dx), mp(ws), nb, L.stream), "conv2d_dx");
  if (add.defined()) dx.add_(add);
  if (!has(keep)) return dx;
  Tensor out = at::empty_like(dx);
  if (has(in_var)) {
    ok(ms_bn_relu_bwd(dx.numel(), dx.size(1), dt, in_pdt, cp(dx), cp(keep), cp(in_mean),
                      cp(in_var), cp(in_w), in_eps, mp(out), L.stream),
       "bn_relu_bwd");
  } else {
    ok(ms_relu_bwd(dx.numel(), dt, cp(dx), cp(keep), mp(out), L.stream), "relu_bwd");
  }
  return out;
}

// ------------------------------------------------ Linear with C++ autograd
template <typename Sig>
c10::TypedOperatorHandle<Sig> op_handle(const char* name) {
  return c10::Dispatcher::singleton().findSchemaOrThrow(name, "").typed<Sig>();
}

struct LinearFn : public torch::autograd::Function<LinearFn> {
  static Tensor forward(torch::autograd::AutogradContext* ctx, const Tensor& x, const Tensor& w,
                        const OptT& b) {
    // MemSave rule (rules.py:133-141): X iff W needs a grad, W iff X does;
    // the bias needs nothing (rules.py:134-135)
    const bool x_rg = x.requires_grad(), w_rg = w.requires_grad();
    ctx->save_for_backward({w_rg ? x : Tensor(), x_rg ? w : Tensor()});
    ctx->saved_data["x_shape"] = x.sizes().vec();
    // a None bias is not an input variable of the node (needs_input_grad has 2 slots)
    ctx->saved_data["has_b"] = has(b);
    static auto fwd = op_handle<Tensor(const Tensor&, const Tensor&, const OptT&)>(
        "memsave::linear_fwd");
    at::AutoDispatchBelowADInplaceOrView guard;
    return fwd.call(x, w, b);
  }
  static torch::autograd::variable_list backward(torch::autograd::AutogradContext* ctx,
                                                 torch::autograd::variable_list grads) {
    static auto dx_op =
        op_handle<Tensor(const Tensor&, const Tensor&, IntArrayRef)>("memsave::linear_dx");
    static auto dw_op = op_handle<Tensor(const Tensor&, const Tensor&)>("memsave::linear_dw");
    static auto db_op = op_handle<Tensor(const Tensor&, int64_t)>("memsave::bias_grad");
    const auto saved = ctx->get_saved_variables();
    const Tensor& gy = grads[0];
    Tensor dx, dw, db;
    // db first: dY was just written by the previous backward op and is still in
    // L2, and the bias reduction writes almost nothing, so the dX / dW GEMMs
    // that follow find dY there too
    if (ctx->saved_data["has_b"].toBool() && ctx->needs_input_grad(2))
      db = db_op.call(gy, gy.size(-1));
    if (ctx->needs_input_grad(0)) {
      TORCH_CHECK(saved[1].defined(), "MissingSavedValue: linear dX needs 'w' but the storage "
                                      "rule did not keep it");
      dx = dx_op.call(gy, saved[1], ctx->saved_data["x_shape"].toIntVector());
    }
    if (ctx->needs_input_grad(1)) {
      TORCH_CHECK(saved[0].defined(), "MissingSavedValue: linear dW needs 'x' but the storage "
                                      "rule did not keep it");
      dw = dw_op.call(saved[0], gy);
    }
    return {dx, dw, db};
  }
};

// Linear -> GELU as one node: the saved set is the union of the two layers'
// rules -- X iff W needs a grad, W iff X does (rules.py:133-141), and the GELU's
// input (the pre-activation), which its VJP reads under every policy
struct LinearGeluFn : public torch::autograd::Function<LinearGeluFn> {
  static Tensor forward(torch::autograd::AutogradContext* ctx, const Tensor& x, const Tensor& w,
                        const OptT& b) {
    const bool x_rg = x.requires_grad(), w_rg = w.requires_grad();
    static auto fwd = op_handle<std::tuple<Tensor, Tensor>(const Tensor&, const Tensor&,
                                                           const OptT&)>("memsave::linear_gelu_fwd");
    Tensor pre, y;
    {
      at::AutoDispatchBelowADInplaceOrView guard;
      std::tie(pre, y) = fwd.call(x, w, b);
    }
    ctx->save_for_backward({w_rg ? x : Tensor(), x_rg ? w : Tensor(), pre});
    ctx->saved_data["x_shape"] = x.sizes().vec();
    ctx->saved_data["has_b"] = has(b);
    return y;
  }
  static torch::autograd::variable_list backward(torch::autograd::AutogradContext* ctx,
                                                 torch::autograd::variable_list grads) {
    static auto gb_op = op_handle<Tensor(const Tensor&, const Tensor&)>("memsave::gelu_bwd");
    static auto dx_op =
        op_handle<Tensor(const Tensor&, const Tensor&, IntArrayRef)>("memsave::linear_dx");
    static auto dw_op = op_handle<Tensor(const Tensor&, const Tensor&)>("memsave::linear_dw");
    static auto db_op = op_handle<Tensor(const Tensor&, int64_t)>("memsave::bias_grad");
    const auto saved = ctx->get_saved_variables();
    const Tensor gz = gb_op.call(grads[0].contiguous(), saved[2]);  // dL/d pre
    Tensor dx, dw, db;
    if (ctx->saved_data["has_b"].toBool() && ctx->needs_input_grad(2))
      db = db_op.call(gz, gz.size(-1));
    if (ctx->needs_input_grad(0)) {
      TORCH_CHECK(saved[1].defined(), "MissingSavedValue: linear dX needs 'w' but the storage "
                                      "rule did not keep it");
      dx = dx_op.call(gz, saved[1], ctx->saved_data["x_shape"].toIntVector());
    }
    if (ctx->needs_input_grad(1)) {
      TORCH_CHECK(saved[0].defined(), "MissingSavedValue: linear dW needs 'x' but the storage "
                                      "rule did not keep it");
      dw = dw_op.call(saved[0], gz);
    }
    return {dx, dw, db};
  }
};

// Linear -> dropout -> + residual as one node: the saved set is the Linear's
// rule (rules.py:133-141) plus the dropout's 16-byte RNG key (rules.py:103-106,
// kept as node data, not a tensor); the add saves nothing (rules.py:116-117)
struct LinearDropoutAddFn : public torch::autograd::Function<LinearDropoutAddFn> {
  static Tensor forward(torch::autograd::AutogradContext* ctx, const Tensor& x, const Tensor& w,
                        const OptT& b, const Tensor& r, double p, int64_t seed, int64_t stream_id,
                        int64_t gen) {
    const bool x_rg = x.requires_grad(), w_rg = w.requires_grad();
    static auto fwd = op_handle<Tensor(const Tensor&, const Tensor&, const OptT&, const Tensor&,
                                       double, int64_t, int64_t, int64_t)>(
        "memsave::linear_dropout_add_fwd");
    Tensor y;
    {
      at::AutoDispatchBelowADInplaceOrView guard;
      y = fwd.call(x, w, b, r, p, seed, stream_id, gen);
    }
    ctx->save_for_backward({w_rg ? x : Tensor(), x_rg ? w : Tensor()});
    ctx->saved_data["x_shape"] = x.sizes().vec();
    ctx->saved_data["has_b"] = has(b);
    ctx->saved_data["p"] = p;
    ctx->saved_data["seed"] = seed;
    ctx->saved_data["stream"] = stream_id;
    ctx->saved_data["gen"] = gen;
    return y;
  }
  static torch::autograd::variable_list backward(torch::autograd::AutogradContext* ctx,
                                                 torch::autograd::variable_list grads) {
    static auto drop_op = op_handle<Tensor(const Tensor&, double, int64_t, int64_t, int64_t)>(
        "memsave::dropout_bwd");
    static auto dx_op =
        op_handle<Tensor(const Tensor&, const Tensor&, IntArrayRef)>("memsave::linear_dx");
    static auto dw_op = op_handle<Tensor(const Tensor&, const Tensor&)>("memsave::linear_dw");
    static auto db_op = op_handle<Tensor(const Tensor&, int64_t)>("memsave::bias_grad");
    const auto saved = ctx->get_saved_variables();
    const bool has_b = ctx->saved_data["has_b"].toBool();
    const int ir = has_b ? 3 : 2;  // input slot of r (a None bias is not an input)
    const Tensor gy = grads[0].contiguous();
    const double p = ctx->saved_data["p"].toDouble();
    Tensor dx, dw, db, dr;
    if (ctx->needs_input_grad(ir)) dr = gy;  // the add passes the gradient through
    const bool lin = ctx->needs_input_grad(0) || ctx->needs_input_grad(1) ||
                     (has_b && ctx->needs_input_grad(2));
    if (lin) {
      // the mask replayed from its key (dropout's VJP), then the Linear's VJPs
      const Tensor gz = p > 0.0 ? drop_op.call(gy, p, ctx->saved_data["seed"].toInt(),
                                               ctx->saved_data["stream"].toInt(),
                                               ctx->saved_data["gen"].toInt())
                                : gy;
      if (has_b && ctx->needs_input_grad(2)) db = db_op.call(gz, gz.size(-1));
      if (ctx->needs_input_grad(0)) {
        TORCH_CHECK(saved[1].defined(), "MissingSavedValue: linear dX needs 'w' but the storage "
                                        "rule did not keep it");
        dx = dx_op.call(gz, saved[1], ctx->saved_data["x_shape"].toIntVector());
      }
      if (ctx->needs_input_grad(1)) {
        TORCH_CHECK(saved[0].defined(), "MissingSavedValue: linear dW needs 'x' but the storage "
                                        "rule did not keep it");
        dw = dw_op.call(saved[0], gz);
      }
    }
    return {dx, dw, db, dr, Tensor(), Tensor(), Tensor(), Tensor()};
  }
};

void check_linear(const Tensor& x, const Tensor& w, const OptT& b) {
  for (const Tensor* t : {&x, &w, has(b) ? &*b : nullptr}) {
    if (!t) continue;
    TORCH_CHECK(t->is_cuda() || t->is_meta(), "memsave_b200.linear: tensors must be on a CUDA "
                "device (got ", t->device(), "); this implementation has no CPU path");
  }
  TORCH_CHECK(w.dim() == 2 && x.dim() >= 1 && x.size(-1) == w.size(1), "linear: input last dim ",
              x.size(-1), " != in_features ", w.size(-1));
  TORCH_CHECK(x.scalar_type() == w.scalar_type(), "linear: input dtype ", x.scalar_type(),
              " != weight dtype ", w.scalar_type());
}

Tensor linear_autograd(const Tensor& x, const Tensor& w, const OptT& b) {
  check_linear(x, w, b);
  return LinearFn::apply(x, w, b);
}

Tensor linear_noautograd(const Tensor& x, const Tensor& w, const OptT& b) {
  check_linear(x, w, b);
  return linear_fwd(x, w, b);
}

Tensor linear_dropout_add_autograd(const Tensor& x, const Tensor& w, const OptT& b,
                                   const Tensor& r, double p, int64_t seed, int64_t stream_id,
                                   int64_t gen) {
  check_linear(x, w, b);
  TORCH_CHECK(r.is_cuda() || r.is_meta(), "memsave_b200.linear_dropout_add: residual must be on "
              "a CUDA device; this implementation has no CPU path");
  return LinearDropoutAddFn::apply(x, w, b, r, p, seed, stream_id, gen);
}

Tensor linear_dropout_add_noautograd(const Tensor& x, const Tensor& w, const OptT& b,
                                     const Tensor& r, double p, int64_t seed, int64_t stream_id,
                                     int64_t gen) {
  check_linear(x, w, b);
  return linear_dropout_add_fwd(x, w, b, r, p, seed, stream_id, gen);
}

Tensor linear_gelu_autograd(const Tensor& x, const Tensor& w, const OptT& b) {
  check_linear(x, w, b);
  return LinearGeluFn::apply(x, w, b);
}

Tensor linear_gelu_noautograd(const Tensor& x, const Tensor& w, const OptT& b) {
  check_linear(x, w, b);
  return std::get<1>(linear_gelu_fwd(x, w, b));
}

}  // namespace

TORCH_LIBRARY(memsave, m) {
  m.def("linear(Tensor x, Tensor w, Tensor? b) -> Tensor");
  m.def("linear_fwd(Tensor x, Tensor w, Tensor? b) -> Tensor");
  m.def("linear_dx(Tensor g, Tensor w, int[] x_shape) -> Tensor");
  m.def("linear_gelu(Tensor x, Tensor w, Tensor? b) -> Tensor");
  m.def("linear_dropout_add(Tensor x, Tensor w, Tensor? b, Tensor r, float p, int seed, "
        "int stream_id, int gen) -> Tensor");
  m.def("linear_dropout_add_fwd(Tensor x, Tensor w, Tensor? b, Tensor r, float p, int seed, "
        "int stream_id, int gen) -> Tensor");
  m.def("linear_gelu_fwd(Tensor x, Tensor w, Tensor? b) -> (Tensor, Tensor)");
  m.def("gelu_fwd(Tensor x) -> Tensor");
  m.def("gelu_bwd(Tensor g, Tensor pre) -> Tensor");
  m.def("linear_dw(Tensor x, Tensor g) -> Tensor");
  m.def("bias_grad(Tensor g, int cols) -> Tensor");
  m.def("conv2d_fwd(Tensor x, Tensor w, Tensor? b, int[] stride, int[] padding, int layout, "
        "int wlayout) -> Tensor");
  m.def("conv2d_dx(Tensor g, Tensor w, int[] x_shape, int[] stride, int[] padding, int layout, "
        "int wlayout) -> Tensor");
  m.def("conv2d_dw(Tensor x, Tensor g, int[] w_shape, int[] stride, int[] padding, int layout, "
        "int wlayout) -> Tensor");
  m.def("conv2d_db(Tensor g, int[] x_shape, int[] w_shape, int[] stride, int[] padding, "
        "int layout, int wlayout) -> Tensor");
  m.def("conv_transpose2d_fwd(Tensor x, Tensor w, Tensor? b, int[] conv_x_shape, int[] stride, "
        "int[] padding, int layout, int wlayout) -> Tensor");
  m.def("bn_eval_fwd(Tensor x, Tensor mean, Tensor var, Tensor? w, Tensor? b, float eps, "
        "int layout) -> Tensor");
  m.def("bn_eval_bwd(Tensor g, Tensor? x, Tensor mean, Tensor var, Tensor? w, float eps, "
        "int layout, bool need_dx, bool need_dw, bool need_db) -> (Tensor, Tensor)");
  m.def("bn_relu_fwd(Tensor x, Tensor? residual, Tensor mean, Tensor var, Tensor? w, "
        "Tensor? b, float eps, bool want_mask) -> (Tensor, Tensor)");
  m.def("bn_add_relu_bwd(Tensor g, Tensor mask, Tensor? x, Tensor mean, Tensor var, Tensor? w, "
        "float eps, bool need_dx, bool need_dr, bool need_dw, bool need_db) "
        "-> (Tensor, Tensor, Tensor)");
  m.def("bn_relu_bwd(Tensor g, Tensor? keep, Tensor mean, Tensor var, Tensor? w, float eps) "
        "-> Tensor");
  m.def("relu_fwd(Tensor x, bool want_mask) -> (Tensor, Tensor)");
  m.def("relu_fwd_(Tensor(a!) x, bool want_mask) -> Tensor");
  m.def("relu_bwd(Tensor g, Tensor mask) -> Tensor");
  m.def("add_relu_fwd(Tensor a, Tensor b, bool want_mask) -> (Tensor, Tensor)");
  m.def("maxpool2d_fwd(Tensor x, int[] kernel, int[] stride, int[] padding, int layout, "
        "bool want_idx) -> (Tensor, Tensor)");
  m.def("maxpool2d_bwd(Tensor g, Tensor idx, int[] x_shape, int[] kernel, int[] stride, "
        "int[] padding, int layout) -> Tensor");
  m.def("maxpool2d_relu_bwd(Tensor g, Tensor idx, Tensor keep, Tensor? in_mean, Tensor? in_var, "
        "Tensor? in_w, float in_eps, int[] x_shape, int[] kernel, int[] stride, int[] padding, "
        "int layout) -> Tensor");
  m.def("dropout_fwd(Tensor x, float p, int seed, int stream_id, int gen) -> Tensor");
  m.def("dropout_fwd_(Tensor(a!) x, float p, int seed, int stream_id, int gen) -> ()");
  m.def("dropout_bwd(Tensor g, float p, int seed, int stream_id, int gen) -> Tensor");
  m.def("layernorm_fwd(Tensor x, Tensor? w, Tensor? b, float eps, int dim, bool want_stats) "
        "-> (Tensor, Tensor, Tensor)");
  m.def("layernorm_bwd(Tensor g, Tensor x, Tensor mean, Tensor rstd, Tensor? w, int dim, "
        "bool need_dx, bool need_dw, bool need_db) -> (Tensor, Tensor, Tensor)");
  m.def("conv2d_bn_fwd(Tensor x, Tensor w, Tensor? bias, Tensor? mean, Tensor? var, "
        "Tensor? bn_w, Tensor? bn_b, float eps, Tensor? residual, bool relu, bool want_mask, "
        "int[] stride, int[] padding, int layout, int wlayout) -> (Tensor, Tensor)");
  m.def("conv2d_bn_dx(Tensor g, Tensor w, Tensor? bn_var, Tensor? bn_w, float eps, "
        "Tensor? addend, Tensor? keep, Tensor? in_mean, Tensor? in_var, Tensor? in_w, "
        "float in_eps, int[] x_shape, int[] stride, int[] padding, int layout, int wlayout) "
        "-> Tensor");
}

#define MS_IMPLS(m)                                          \
  m.impl("linear_fwd", &linear_fwd);                         \
  m.impl("linear_dx", &linear_dx);                           \
  m.impl("linear_gelu_fwd", &linear_gelu_fwd);               \
  m.impl("linear_dropout_add_fwd", &linear_dropout_add_fwd); \
  m.impl("gelu_fwd", &gelu_fwd);                             \
  m.impl("gelu_bwd", &gelu_bwd);                             \
  m.impl("linear_dw", &linear_dw);                           \
  m.impl("bias_grad", &bias_grad);                           \
  m.impl("conv2d_fwd", &conv2d_fwd);                         \
  m.impl("conv2d_dx", &conv2d_dx);                           \
  m.impl("conv2d_dw", &conv2d_dw);                           \
  m.impl("conv2d_db", &conv2d_db);                           \
  m.impl("conv_transpose2d_fwd", &conv_transpose2d_fwd);     \
  m.impl("bn_eval_fwd", &bn_eval_fwd);                       \
  m.impl("bn_eval_bwd", &bn_eval_bwd);                       \
  m.impl("bn_relu_fwd", &bn_relu_fwd);                       \
  m.impl("bn_add_relu_bwd", &bn_add_relu_bwd);               \
  m.impl("bn_relu_bwd", &bn_relu_bwd);                       \
  m.impl("relu_fwd", &relu_fwd);                             \
  m.impl("relu_fwd_", &relu_fwd_);                           \
  m.impl("relu_bwd", &relu_bwd);                             \
  m.impl("add_relu_fwd", &add_relu_fwd);                     \
  m.impl("maxpool2d_fwd", &maxpool2d_fwd);                   \
  m.impl("maxpool2d_bwd", &maxpool2d_bwd);                   \
  m.impl("maxpool2d_relu_bwd", &maxpool2d_relu_bwd);         \
  m.impl("dropout_fwd", &dropout_fwd);                       \
  m.impl("dropout_fwd_", &dropout_fwd_);                     \
  m.impl("dropout_bwd", &dropout_bwd);                       \
  m.impl("layernorm_fwd", &layernorm_fwd);                   \
  m.impl("layernorm_bwd", &layernorm_bwd);                   \
  m.impl("conv2d_bn_fwd", &conv2d_bn_fwd);                   \
  m.impl("conv2d_bn_dx", &conv2d_bn_dx)

TORCH_LIBRARY_IMPL(memsave, CUDA, m) {
  MS_IMPLS(m);
  m.impl("linear", &linear_noautograd);
  m.impl("linear_gelu", &linear_gelu_noautograd);
  m.impl("linear_dropout_add", &linear_dropout_add_noautograd);
}
TORCH_LIBRARY_IMPL(memsave, Meta, m) {
  MS_IMPLS(m);
  m.impl("linear", &linear_noautograd);
  m.impl("linear_gelu", &linear_gelu_noautograd);
  m.impl("linear_dropout_add", &linear_dropout_add_noautograd);
}
TORCH_LIBRARY_IMPL(memsave, Autograd, m) {
  m.impl("linear", &linear_autograd);
  m.impl("linear_gelu", &linear_gelu_autograd);
  m.impl("linear_dropout_add", &linear_dropout_add_autograd);
}
// CPU tensors reach the autograd kernel too (then fail loudly in check_linear)
