// Conv2d forward / input-VJP / weight-VJP entry points (the C-ABI boundary for
// leantape.kernels.conv2d_fwd/dx/dw, kernels/__init__.py:26-28).
//
// 16-bit NHWC activations run as implicit GEMMs on the tcgen05 kernel:
//   fwd : A = im2col(x) through a TMA im2col tensor map (padding = OOB zero
//         fill, stride = traversal stride), B = weight [k][tap][c] (OHWI used
//         in place when C % 64 == 0, otherwise a zero-padded repack)
//   dx  : one GEMM per stride phase (h % sh, w % sw) — only the taps whose
//         parity matches contribute, so no zero MACs; A = im2col(dy) with a
//         per-phase bounding box, B = weight repacked [c][tap][k]
//   dw  : A = dyᵀ (MN-major tiles of dy), B = im2col(x)ᵀ (MN-major), one tile
//         set per tap, split-K over output pixels with fp32 red.add, then a
//         cast/layout pass into OIHW or OHWI
// float32, NCHW 16-bit and channel counts that are not multiples of 8 run on
// the SIMT direct kernels (simt.cu).
#include <algorithm>
#include <cstdlib>

#include "misc.cuh"

namespace ms {
namespace {

bool is16(int dt) { return dt == MS_BF16 || dt == MS_F16; }

ConvDims dims_of(const ms_conv_desc* d) {
  ConvDims c;
  c.n = (int)d->n; c.c = (int)d->c; c.h = (int)d->h; c.w = (int)d->w;
  c.k = (int)d->k; c.r = (int)d->r; c.s = (int)d->s;
  c.sh = d->stride_h; c.sw = d->stride_w; c.ph = d->pad_h; c.pw = d->pad_w;
  c.oh = (int)((d->h + 2 * d->pad_h - d->r) / d->stride_h + 1);
  c.ow = (int)((d->w + 2 * d->pad_w - d->s) / d->stride_w + 1);
  return c;
}

ms_status validate(const ms_conv_desc* d) {
  MS_CHECK_ARG(d != nullptr, MS_ERR_SHAPE, "conv: null descriptor");
  MS_CHECK_ARG(d->n >= 0 && d->c > 0 && d->h > 0 && d->w > 0 && d->k > 0 && d->r > 0 && d->s > 0,
               MS_ERR_SHAPE, "conv: non-positive dimension");
  MS_CHECK_ARG(d->stride_h > 0 && d->stride_w > 0 && d->pad_h >= 0 && d->pad_w >= 0, MS_ERR_SHAPE,
               "conv: invalid stride/padding");
  MS_CHECK_ARG(d->h + 2 * d->pad_h >= d->r && d->w + 2 * d->pad_w >= d->s, MS_ERR_SHAPE,
               "conv: kernel larger than padded input");
  MS_CHECK_ARG(d->dtype == MS_F32 || d->dtype == MS_BF16 || d->dtype == MS_F16, MS_ERR_DTYPE,
               "conv: bad dtype %d", d->dtype);
  MS_CHECK_ARG(d->n * d->c * d->h * d->w < (1ll << 31) &&
                   d->n * d->k * (d->h + 2 * d->pad_h) * (d->w + 2 * d->pad_w) < (1ll << 33),
               MS_ERR_UNSUPPORTED, "conv: tensor too large for 32-bit tile indexing");
  return MS_OK;
}

// ----------------------------------------------------------------- planning
struct ConvPlan {
  bool tc = false;
  int cpad8 = 0;        // fwd: channel count of the (possibly padded) activation
  bool pad_x = false;   // fwd: activation is channel-padded into ws
  bool repack = false;  // fwd: weight repacked into ws
  int cpad = 0;         // fwd: per-tap weight pitch (multiple of 64)
  int kpad = 0;         // dx: per-tap pitch of the repacked weight
  bool c8 = false;      // fwd: 8-channel im2col variant
  bool rowseg = false;  // fwd: <=4-ch stride-2 / <=8-ch stride-1 row-segment loads
  int xw_pad = 0;       // rowseg: padded width of the channel-padded activation copy
  int cpx = 4;          // rowseg: channels per padded pixel (16 B between windows)
  bool band = false;    // dx: <8-channel input gradient (the stem), band col2im
  bool stem = false;    // dx: the 3-channel 7x7/2 stem, register col2im (stem_dgrad.cu)
  bool halo3 = false;   // fwd / dx: 3x3/1/1 64->64 halo-tiled kernel (conv3x3.cu)
  int band_h = 16;
  size_t ws_pad = 0, ws_w = 0, ws_acc = 0;
  size_t ws = 0;
};

bool tc_ok(const ms_conv_desc* d) {
  return is16(d->dtype) && d->layout == MS_NHWC && d->r <= 64 && d->s <= 64 &&
         d->pad_h < 64 && d->pad_w < 64;
}

// Row-segment stem forward: one A row = S*4 consecutive elements of a
// 4-channel input row; consecutive output pixels start sw*8 bytes apart, which
// TMA needs to be a multiple of 16 (stride 2).  Checked once against the driver.
// row-segment loads apply when consecutive output pixels' input windows start
// 16 bytes apart in a channel-padded copy: <= 4 channels at stride 2 (the 7x7
// stem) or <= 8 channels at stride 1 (VGG's first 3x3), one kernel row <= 32
// elements (64 bytes)
int rowseg_cpx(const ms_conv_desc* d) {
  if (d->c <= 4 && d->stride_w == 2 && d->s * 4 <= 32) return 4;
  if (d->c <= 8 && d->stride_w == 1 && d->s * 8 <= 32) return 8;
  return 0;
}

bool rowseg_ok(const ms_conv_desc* d, const ConvDims& c) {
  (void)c;
  if (!rowseg_cpx(d)) return false;
  static int cached = -1;
  if (cached < 0) {
    CUtensorMap m;
    const uint64_t dims[4] = {32, 112, 224, 2};
    const uint64_t str[3] = {16, 232 * 8, 224ull * 232 * 8};
    const uint32_t box[4] = {32, BM, 1, 1};
    cached = make_tmap_nd(&m, MS_BF16, reinterpret_cast<void*>(0x100000), 4, dims, str, box, 64) ==
                     MS_OK
                 ? 1
                 : 0;
  }
  return cached == 1;
}

ConvPlan plan(const ms_conv_desc* d, int pass, bool dx_bias = false) {
  ConvPlan p;
  const ConvDims c = dims_of(d);
  const size_t es = dtype_size(d->dtype);
  const int64_t taps = (int64_t)d->r * d->s;
  if (!tc_ok(d)) {
    if (pass == MS_CONV_DW) {
      size_t w = simt_conv_dw_workspace(c);
      if (d->dtype == MS_F32) {
        const size_t s = small_conv_fp32_workspace(c, pass);
        if (s > w) w = s;
      }
      p.ws = align256(w);
    }
    return p;
  }
  if (pass == MS_CONV_FWD) {
    p.tc = true;
    if (conv3x3_halo_ok(d->dtype, d->layout, (int)d->c, (int)d->k, (int)d->r, (int)d->s,
                        d->stride_h, d->stride_w, d->pad_h, d->pad_w, (int)d->w)) {
      p.halo3 = true;
      p.ws = conv3x3_halo_workspace();
      return p;
    }
    if (rowseg_ok(d, c)) {
      p.rowseg = true;
      p.cpx = rowseg_cpx(d);
      // the last window reads 64 bytes = 64 / (2 cpx) pixels from its start
      p.xw_pad = (int)std::max<int64_t>(d->w + 2 * d->pad_w,
                                        (int64_t)(c.ow - 1) * d->stride_w + 32 / p.cpx);
      if (p.cpx == 8 && d->stride_w == 1) p.xw_pad = (p.xw_pad + 7) / 8 * 8;  // 128-B row chunks
      p.ws_pad = align256(es * (size_t)d->n * d->h * p.xw_pad * p.cpx);
      p.ws_w = align256(es * (size_t)d->k * d->r * 32);
      p.ws = p.ws_pad + p.ws_w;
      return p;
    }
    p.cpad8 = (int)(d->c < 8 ? 8 : round_up(d->c, 8));
    p.pad_x = p.cpad8 != d->c;
    p.c8 = p.cpad8 == 8;
    p.cpad = p.c8 ? 8 : (int)round_up(p.cpad8, 64);
    p.repack = !(d->wlayout == MS_NHWC && d->c % 64 == 0);
    if (p.pad_x) p.ws_pad = align256(es * (size_t)d->n * d->h * d->w * p.cpad8);
    if (p.repack) p.ws_w = align256(es * (size_t)d->k * taps * p.cpad);
    p.ws = p.ws_pad + p.ws_w;
  } else if (pass == MS_CONV_DX) {
    if (d->k % 8 != 0) return p;  // SIMT
    static const bool env_band = getenv("MS_STEM_BAND") != nullptr;  // A/B against the band kernel
    if (!dx_bias && !env_band &&
        stem_dgrad_ok(d->dtype, d->layout, (int)d->c, (int)d->r, (int)d->s, d->stride_h,
                      d->stride_w, d->pad_h, d->pad_w, c.ow, d->k)) {
      p.tc = true;
      p.stem = true;
      p.kpad = (int)d->k;
      p.ws_w = align256(es * (size_t)taps * d->c * p.kpad);
      p.ws = p.ws_w;
      return p;
    }
    if (!dx_bias && d->c == BAND_C && d->r == BAND_R && d->s == BAND_S && d->stride_w == BAND_SW &&
        d->stride_h == BAND_SW && c.ow <= BM && (int64_t)BAND_WINDOWS * BAND_WIN * 4 <= BAND_WINDOW_BYTES) {
      // the 3-channel 7x7/2 stem: per dX-row band, dY-row x W GEMM + col2im
      p.tc = true;
      p.band = true;
      p.band_h = BAND_H;
      p.kpad = (int)round_up(d->k, 64);
      p.ws_w = align256(es * (size_t)taps * d->c * p.kpad);
      p.ws = p.ws_w;
      return p;
    }
    if (conv3x3_halo_ok(d->dtype, d->layout, (int)d->k, (int)d->c, (int)d->r, (int)d->s,
                        d->stride_h, d->stride_w, d->pad_h, d->pad_w, (int)d->w)) {
      p.tc = true;
      p.halo3 = true;
      p.kpad = (int)round_up(d->k, 64);  // the phase-GEMM fallback (with a bias) uses it
      p.ws = std::max(conv3x3_halo_workspace(), align256(es * (size_t)d->c * taps * p.kpad));
      return p;
    }
    if (d->stride_h > 2 || d->stride_w > 2) return p;  // SIMT
    p.tc = true;
    p.kpad = (int)round_up(d->k, 64);
    p.ws_w = align256(es * (size_t)d->c * taps * p.kpad);
    p.ws = p.ws_w;
  } else {
    if (d->k % 8 != 0 || d->c % 8 != 0) {
      p.ws = align256(simt_conv_dw_workspace(c));
      return p;
    }
    p.tc = true;
    p.ws_acc = align256(sizeof(float) * (size_t)d->k * taps * d->c);
    p.ws = p.ws_acc;
  }
  return p;
}

// 1x1, stride 1, no padding: output pixel m reads input pixel m only
bool is_pointwise(const ConvDims& c) {
  static const bool off = getenv("MS_CONV1X1_IM2COL") != nullptr;  // A/B switch
  return !off && c.r == 1 && c.s == 1 && c.sh == 1 && c.sw == 1 && c.ph == 0 && c.pw == 0 &&
         c.oh == c.h && c.ow == c.w;
}

GemmArgs base_args(int dt) {
  GemmArgs g{};
  g.ab_fmt = dt == MS_BF16 ? 1 : 0;
  g.splits = 1;
  g.taps = 1;
  g.nphases = 1;
  return g;
}

ConvShape shape_of(const ConvDims& c, int C, int H, int W, int cblocks, int wpitch, int outH,
                   int outW) {
  ConvShape s{};
  s.N = c.n; s.H = H; s.W = W; s.C = C;
  s.P = c.oh; s.Q = c.ow; s.R = c.r; s.S = c.s;
  s.sh = c.sh; s.sw = c.sw; s.ph = c.ph; s.pw = c.pw;
  s.cblocks = cblocks; s.wrow_cpad = wpitch; s.outH = outH; s.outW = outW;
  return s;
}

// ----------------------------------------------------------------- forward
// optional epilogue fusion of a following eval-BatchNorm (+ ReLU with its mask)
struct Fuse {
  BnFold bn;
  int relu = 0;
  uint8_t* mask = nullptr;
  const void* resid = nullptr;
};

void apply_fuse(EpiParams& e, const Fuse* f) {
  if (!f) return;
  e.bn = f->bn;
  e.relu = f->relu;
  e.mask = f->mask;
  e.resid = f->resid;
}

ms_status fwd_rowseg(const ms_conv_desc* d, const ConvPlan& p, const void* x, const void* w,
                     const void* bias, void* y, void* ws, cudaStream_t st,
                     const Fuse* f = nullptr) {
  const ConvDims c = dims_of(d);
  const int dt = d->dtype;
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  void* x4 = wsb;
  void* wr = wsb + p.ws_pad;
  MS_TRY(pad_rowseg(dt, c.n, c.h, c.w, c.c, c.pw, p.xw_pad, p.cpx, x, x4, st));
  static const bool env_im2col = getenv("MS_STEM_IM2COL") != nullptr;  // A/B switch
  if (!env_im2col && (!f || !f->resid) && p.cpx == 4 &&
      stem_fprop_ok(dt, d->layout, c.c, c.r, c.s, c.sh, c.sw, c.ph, c.pw, c.ow, c.k) &&
      stem_fprop_weight_bytes(c.k) <= p.ws_w)
    return stem_fprop(dt, c.n, c.h, p.xw_pad, c.oh, c.ow, c.k, c.c, d->wlayout, x4, w, wr, bias, y,
                      st, f ? f->bn : BnFold{}, f ? f->relu : 0, f ? f->mask : nullptr);
  MS_TRY(repack_rowseg(dt, c.k, c.c, c.r, c.s, p.cpx, d->wlayout, w, wr, st));
  GemmArgs g = base_args(dt);
  g.M = c.n * c.oh * c.ow;
  g.N = c.k;
  const int bn = c.k <= 32 ? 32 : (c.k <= 64 ? 64 : (c.k <= 128 ? 128 : 256));
  const int segs = (int)((c.ow + BM - 1) / BM);  // 128-pixel segments per output row
  g.n_blocks = (c.k + bn - 1) / bn;
  g.num_tiles = c.n * c.oh * segs * g.n_blocks;
  g.cv = shape_of(c, p.cpx, c.h, p.xw_pad, 1, 32, c.oh, c.ow);
  g.cv.band_sub = segs;
  g.epi = EpiParams{y, c.k, dt, 0, bias, dt};
  apply_fuse(g.epi, f);
  TmapPack tm;
  const size_t es = dtype_size(dt);
  const uint64_t dims[4] = {32, (uint64_t)c.ow, (uint64_t)c.h, (uint64_t)c.n};
  const uint64_t str[3] = {(uint64_t)c.sw * p.cpx * es, (uint64_t)p.xw_pad * p.cpx * es,
                           (uint64_t)c.h * p.xw_pad * p.cpx * es};
  const uint32_t box[4] = {32, BM, 1, 1};
  if (p.cpx == 8 && c.sw == 1 && p.xw_pad % 8 == 0) {
    // contiguous row segments: [64 elements = 8 px][xw_pad / 8][H][N], 17 chunks per box
    const uint64_t d8[4] = {64, (uint64_t)p.xw_pad / 8, (uint64_t)c.h, (uint64_t)c.n};
    const uint64_t s8[3] = {128, (uint64_t)p.xw_pad * 8 * es, (uint64_t)c.h * p.xw_pad * 8 * es};
    const uint32_t b8[4] = {64, ROWSEG8_A_TX / 128, 1, 1};
    MS_TRY(make_tmap_nd(&tm.a[0], dt, x4, 4, d8, s8, b8, 0));
    g.rowseg8 = 1;
  } else {
    MS_TRY(make_tmap_nd(&tm.a[0], dt, x4, 4, dims, str, box, 64));
  }
  tm.a[1] = tm.a[2] = tm.a[3] = tm.a[0];
  const uint64_t wd[2] = {(uint64_t)c.r * 32, (uint64_t)c.k};
  const uint64_t ws2[1] = {(uint64_t)c.r * 32 * es};
  const uint32_t wb[2] = {32, (uint32_t)bn};
  MS_TRY(make_tmap_nd(&tm.b, dt, wr, 2, wd, ws2, wb, 64));
  // epilogue TMA stores through [N*OH][OW][K]: a 32-pixel x 32-channel chunk per
  // warp, the pixel tail of a row's last segment clipped by the map
  if (dt != MS_F32 && (reinterpret_cast<uintptr_t>(y) & 15) == 0 && (c.k * es) % 16 == 0) {
    const uint64_t yd[3] = {(uint64_t)c.k, (uint64_t)c.ow, (uint64_t)c.n * c.oh};
    const uint64_t ys[2] = {(uint64_t)c.k * es, (uint64_t)c.ow * c.k * es};
    const uint32_t yb[3] = {32, 32, 1};
    MS_TRY(make_tmap_nd(&tm.c, dt, y, 3, yd, ys, yb, 64));
    g.tma_store = 1;
  }
  return launch_umma(bn, 0, 0, LOAD_CONV_FPROP_ROWSEG, tm, g, st);
}

ms_status fwd_tc(const ms_conv_desc* d, const ConvPlan& p, const void* x, const void* w,
                 const void* bias, void* y, void* ws, cudaStream_t st, const Fuse* f = nullptr) {
  if (p.rowseg) return fwd_rowseg(d, p, x, w, bias, y, ws, st, f);
  if (p.halo3)
    return conv3x3_halo(d->dtype, (int)d->n, (int)d->h, (int)d->w, d->wlayout, 0, x, w, ws, y,
                        f ? f->bn : BnFold{}, bias, f ? f->resid : nullptr, f ? f->relu : 0, f ? f->mask : nullptr, nullptr,
                        nullptr, 0, 0.f, st);
  const ConvDims c = dims_of(d);
  const int dt = d->dtype;
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  const void* xsrc = x;
  if (p.pad_x) {
    MS_TRY(pad_channels(dt, (int64_t)c.n * c.h * c.w, c.c, p.cpad8, x, wsb, st));
    xsrc = wsb;
  }
  const void* wsrc = w;
  if (p.repack) {
    MS_TRY(repack_fprop(dt, c.k, c.c, c.r, c.s, p.cpad, d->wlayout, w, wsb + p.ws_pad, st));
    wsrc = wsb + p.ws_pad;
  }
  const int64_t M = (int64_t)c.n * c.oh * c.ow;
  GemmArgs g = base_args(dt);
  g.M = (int)M;
  g.N = c.k;
  const int m_tiles = (int)((M + BM - 1) / BM);
  const TilePick tp = pick_tiles(m_tiles, c.k, !p.c8, false);
  if (is_pointwise(c) && !p.c8 && d->layout == MS_NHWC) {
    // 1x1 / stride 1 / pad 0 over NHWC pixels is a plain GEMM: tiled TMA rows of
    // x instead of im2col boxes, and the GEMM epilogue (TMA stores + fusion)
    const int bn = tp.bn;
    g.m_blocks = (m_tiles + tp.cl - 1) / tp.cl;
    g.n_blocks = (c.k + bn - 1) / bn;
    g.k_blocks = p.cpad / BK;
    g.kb_per_split = g.k_blocks;
    g.num_tiles = g.m_blocks * g.n_blocks;
    g.epi = EpiParams{y, c.k, dt, 0, bias, dt};
    apply_fuse(g.epi, f);
    TmapPack tm;
    MS_TRY(make_tmap_2d(&tm.a[0], dt, xsrc, p.cpad8, M, p.cpad8, BK, BM));
    tm.a[1] = tm.a[2] = tm.a[3] = tm.a[0];
    MS_TRY(make_tmap_2d(&tm.b, dt, wsrc, p.cpad, c.k, p.cpad, BK, bn / tp.cl));
    MS_TRY(setup_tma_store(tm, g, dt, y, M, c.k, c.k));
    return launch_umma(bn, 0, 0, LOAD_GEMM, tm, g, st, tp.cl);
  }
  const int bn = tp.bn;
  g.m_blocks = (m_tiles + tp.cl - 1) / tp.cl;  // pairs of M tiles when clustered
  g.n_blocks = (c.k + bn - 1) / bn;
  g.num_tiles = g.m_blocks * g.n_blocks;
  g.k_blocks = (c.r * c.s + 7) / 8;  // C8 variant: 8 taps per k-block
  g.cv = shape_of(c, p.cpad8, c.h, c.w, p.c8 ? 1 : p.cpad / 64, p.cpad, c.oh, c.ow);
  g.epi = EpiParams{y, c.k, dt, 0, bias, dt};
  apply_fuse(g.epi, f);
  TmapPack tm;
  const int lower[2] = {-c.pw, -c.ph};
  const int upper[2] = {c.pw - (c.s - 1), c.ph - (c.r - 1)};
  MS_TRY(make_tmap_im2col(&tm.a[0], dt, xsrc, c.n, c.h, c.w, p.cpad8, lower, upper, c.sw, c.sh,
                          p.c8 ? 8 : 64, BM, !p.c8));
  tm.a[1] = tm.a[2] = tm.a[3] = tm.a[0];
  const int64_t wrow = (int64_t)c.r * c.s * p.cpad;
  MS_TRY(make_tmap_2d(&tm.b, dt, wsrc, wrow, c.k, wrow, BK, bn / tp.cl));
  MS_TRY(setup_tma_store(tm, g, dt, y, M, c.k, c.k));
  return launch_umma(bn, 0, 0, p.c8 ? LOAD_CONV_FPROP_C8 : LOAD_CONV_FPROP, tm, g, st, tp.cl);
}

// ----------------------------------------------------------------- input-VJP
ms_status dx_band(const ms_conv_desc* d, const ConvPlan& p, const void* dy, const void* w,
                  void* dx, void* ws, cudaStream_t st) {
  const ConvDims c = dims_of(d);
  const int dt = d->dtype;
  void* wt = ws;
  MS_TRY(repack_scatter(dt, c.k, c.c, c.r, c.s, p.kpad, d->wlayout, w, wt, st));
  const int ncols = c.r * c.s * c.c;
  const int bn = 160;  // band kernel is specialised to 7*7*3 = 147 columns
  GemmArgs g = base_args(dt);
  g.M = c.n * c.oh * c.ow;
  g.N = ncols;
  g.n_blocks = 1;
  g.k_blocks = p.kpad / 64;
  g.cv = shape_of(c, c.k, c.oh, c.ow, p.kpad / 64, p.kpad, c.h, c.w);
  g.cv.outC = c.c;
  g.cv.band_h = p.band_h;
  g.cv.band_sub = (p.band_h + c.r - 2) / c.sh + 1;
  g.cv.bands_per_img = (c.h + p.band_h - 1) / p.band_h;
  g.num_tiles = c.n * g.cv.bands_per_img;
  g.epi = EpiParams{dx, 0, dt, 0, nullptr, 0};
  TmapPack tm;
  const size_t es = dtype_size(dt);
  const uint64_t dims[4] = {(uint64_t)c.k, (uint64_t)c.ow, (uint64_t)c.oh, (uint64_t)c.n};
  const uint64_t str[3] = {(uint64_t)c.k * es, (uint64_t)c.ow * c.k * es,
                           (uint64_t)c.oh * c.ow * c.k * es};
  const uint32_t box[4] = {64, BM, 1, 1};
  MS_TRY(make_tmap_nd(&tm.a[0], dt, dy, 4, dims, str, box, 128));
  tm.a[1] = tm.a[2] = tm.a[3] = tm.a[0];
  MS_TRY(make_tmap_2d(&tm.b, dt, wt, p.kpad, ncols, p.kpad, BK, bn));
  return launch_umma(bn, 0, 0, LOAD_CONV_DGRAD_BAND, tm, g, st);
}

struct KScale {  // an eval-BN scale w/sqrt(var+eps) folded into the dgrad weight
  const void* var = nullptr;
  const void* weight = nullptr;
  int pdt = 0;
  float eps = 0.f;
};

// epilogue work of an input-VJP: dx = keep ? (dgrad + addend) : 0, times the
// producer BN's scale when in_bn.var is set
struct DxFuse {
  const void* addend = nullptr;
  const uint8_t* keep = nullptr;
  BnFold in_bn;
  bool any() const { return addend || keep || in_bn.var; }
};

ms_status dx_tc(const ms_conv_desc* d, const ConvPlan& p, const void* dy, const void* w, void* dx,
                void* ws, cudaStream_t st, const void* bias = nullptr,
                const KScale* ks = nullptr, const DxFuse* xf = nullptr) {
  const ConvDims c = dims_of(d);
  const int dt = d->dtype;
  MS_CHECK_ARG(!xf || !xf->any() || (!p.band && !p.stem), MS_ERR_UNSUPPORTED,
               "conv dx: no fused epilogue in the stem / band kernels");
  const DxFuse none;
  if (!xf) xf = &none;
  if (p.band) return dx_band(d, p, dy, w, dx, ws, st);
  if (p.halo3 && !bias)  // the input-VJP is the same 3x3 conv of dY with W transposed + flipped
    return conv3x3_halo(d->dtype, (int)d->n, (int)d->h, (int)d->w, d->wlayout, 1, dy, w, ws, dx,
                        xf->in_bn, nullptr, xf->addend, 0, nullptr, ks ? ks->var : nullptr,
                        ks ? ks->weight : nullptr, ks ? ks->pdt : 0, ks ? ks->eps : 0.f, st,
                        xf->keep, xf->in_bn.var != nullptr);
  if (p.stem) {
    MS_TRY(repack_scatter(dt, c.k, c.c, c.r, c.s, p.kpad, d->wlayout, w, ws, st));
    return stem_dgrad(dt, c.n, c.h, c.w, c.oh, c.ow, c.k, dy, ws, dx, st);
  }
  void* wd = ws;
  MS_TRY(repack_dgrad(dt, c.k, c.c, c.r, c.s, p.kpad, d->wlayout, w, wd, st,
                      ks ? ks->var : nullptr, ks ? ks->weight : nullptr, ks ? ks->pdt : 0,
                      ks ? ks->eps : 0.f));
  GemmArgs g = base_args(dt);
  g.N = c.c;
  const TilePick tp = pick_tiles((int64_t)c.n * c.h * c.w / BM + 1, c.c, true, false);
  const int bn = tp.bn;
  g.n_blocks = (c.c + bn - 1) / bn;
  if (is_pointwise(c) && d->layout == MS_NHWC) {
    // 1x1 / stride 1: dX[px][c] = dY[px][k] . W'[c][k] (the repacked, BN-scaled
    // weight) as a plain GEMM with the fused dgrad epilogue
    const int64_t M = (int64_t)c.n * c.h * c.w;
    const int m_tiles = (int)((M + BM - 1) / BM);
    g.M = (int)M;
    g.m_blocks = (m_tiles + tp.cl - 1) / tp.cl;
    g.k_blocks = p.kpad / BK;
    g.kb_per_split = g.k_blocks;
    g.num_tiles = g.m_blocks * g.n_blocks;
    g.epi = EpiParams{dx, c.c, dt, 0, bias, dt};
    g.epi.resid = xf->addend;
    g.epi.keep_in = xf->keep;
    g.epi.bn = xf->in_bn;
    g.epi.bn_post = xf->in_bn.var != nullptr;
    TmapPack tm;
    MS_TRY(make_tmap_2d(&tm.a[0], dt, dy, c.k, M, c.k, BK, BM));
    tm.a[1] = tm.a[2] = tm.a[3] = tm.a[0];
    MS_TRY(make_tmap_2d(&tm.b, dt, wd, p.kpad, c.c, p.kpad, BK, bn / tp.cl));
    MS_TRY(setup_tma_store(tm, g, dt, dx, M, c.c, c.c));
    return launch_umma(bn, 0, 0, LOAD_GEMM, tm, g, st, tp.cl);
  }
  g.cv = shape_of(c, c.k, c.oh, c.ow, p.kpad / 64, p.kpad, c.h, c.w);
  TmapPack tm;
  int np = 0, tiles = 0;
  for (int ph = 0; ph < c.sh; ++ph) {
    for (int pw = 0; pw < c.sw; ++pw) {
      PhaseInfo P{};
      P.ph = ph;
      P.pw = pw;
      P.Hp = (c.h - ph + c.sh - 1) / c.sh;
      P.Wp = (c.w - pw + c.sw - 1) / c.sw;
      if (P.Hp <= 0 || P.Wp <= 0) continue;
      P.r0 = (ph + c.ph) % c.sh;
      P.s0 = (pw + c.pw) % c.sw;
      P.nr = P.r0 < c.r ? (c.r - P.r0 + c.sh - 1) / c.sh : 0;
      P.ns = P.s0 < c.s ? (c.s - P.s0 + c.sw - 1) / c.sw : 0;
      const int dh0 = (ph + c.ph - P.r0) / c.sh;
      const int dw0 = (pw + c.pw - P.s0) / c.sw;
      P.Lh = P.nr > 0 ? dh0 - (P.nr - 1) : 0;
      P.Lw = P.ns > 0 ? dw0 - (P.ns - 1) : 0;
      P.m_total = c.n * P.Hp * P.Wp;
      P.m_blocks = ((P.m_total + BM - 1) / BM + tp.cl - 1) / tp.cl;  // pairs when clustered
      P.tile_begin = tiles;
      tiles += P.m_blocks * g.n_blocks;
      if (P.nr > 0 && P.ns > 0) {
        const int lower[2] = {P.Lw, P.Lh};
        const int upper[2] = {P.Lw + P.Wp - c.ow, P.Lh + P.Hp - c.oh};
        MS_TRY(make_tmap_im2col(&tm.a[np], dt, dy, c.n, c.oh, c.ow, c.k, lower, upper, 1, 1, 64,
                                BM));
      } else if (np > 0) {
        tm.a[np] = tm.a[0];
      } else {
        const int lower[2] = {0, 0};
        const int upper[2] = {0, 0};
        MS_TRY(make_tmap_im2col(&tm.a[np], dt, dy, c.n, c.oh, c.ow, c.k, lower, upper, 1, 1, 64,
                                BM));
      }
      g.phase[np++] = P;
    }
  }
  g.nphases = np;
  g.num_tiles = tiles;
  g.epi = EpiParams{dx, c.c, dt, 0, bias, dt};  // bias: conv_transpose2d forward
  g.epi.resid = xf->addend;                      // dx = dgrad + addend (tee'd input)
  g.epi.keep_in = xf->keep;
  g.epi.bn = xf->in_bn;
  g.epi.bn_post = xf->in_bn.var != nullptr;
  const int64_t wrow = (int64_t)c.r * c.s * p.kpad;
  MS_TRY(make_tmap_2d(&tm.b, dt, wd, wrow, c.c, wrow, BK, bn / tp.cl));
  return launch_umma(bn, 0, 0, LOAD_CONV_DGRAD, tm, g, st, tp.cl);
}

// ----------------------------------------------------------------- weight-VJP
ms_status dw_tc(const ms_conv_desc* d, const ConvPlan& p, const void* x, const void* dy, void* dw,
                void* ws, cudaStream_t st) {
  const ConvDims c = dims_of(d);
  const int dt = d->dtype;
  float* acc = static_cast<float*>(ws);
  const int taps = c.r * c.s;
  cudaMemsetAsync(acc, 0, sizeof(float) * (size_t)c.k * taps * c.c, st);
  const int64_t P = (int64_t)c.n * c.oh * c.ow;
  GemmArgs g = base_args(dt);
  g.M = c.k;
  g.N = c.c;
  g.m_blocks = (c.k + BM - 1) / BM;
  int bn = c.c <= 64 ? 64 : (c.c <= 128 ? 128 : 256);
  g.n_blocks = (c.c + bn - 1) / bn;
  g.taps = taps;
  g.k_blocks = (int)((P + BK - 1) / BK);
  const int64_t base_tiles = (int64_t)g.m_blocks * g.n_blocks * taps;
  int64_t splits = (2 * (int64_t)num_sms() + base_tiles - 1) / base_tiles;
  if (splits > g.k_blocks / 2) splits = g.k_blocks / 2;
  if (splits < 1) splits = 1;
  g.kb_per_split = (int)((g.k_blocks + splits - 1) / splits);
  g.splits = (g.k_blocks + g.kb_per_split - 1) / g.kb_per_split;
  g.num_tiles = (int)(base_tiles * g.splits);
  g.cv = shape_of(c, c.c, c.h, c.w, (c.c + 63) / 64, 0, c.oh, c.ow);
  g.epi = EpiParams{acc, (int64_t)taps * c.c, MS_F32, 1, nullptr, 0};
  TmapPack tm;
  MS_TRY(make_tmap_2d(&tm.a[0], dt, dy, c.k, P, c.k, 64, BK));
  tm.a[1] = tm.a[2] = tm.a[3] = tm.a[0];
  const int lower[2] = {-c.pw, -c.ph};
  const int upper[2] = {c.pw - (c.s - 1), c.ph - (c.r - 1)};
  MS_TRY(make_tmap_im2col(&tm.b, dt, x, c.n, c.h, c.w, c.c, lower, upper, c.sw, c.sh, 64, BK));
  MS_TRY(launch_umma(bn, 1, 1, LOAD_CONV_WGRAD, tm, g, st));
  return wgrad_finalize(dt, c.k, c.c, c.r, c.s, d->wlayout, acc, dw, st);
}

// y[n, c, ...] += bias[c] (NCHW planes or NHWC rows)
template <typename T>
__global__ void add_channel_bias_kernel(int64_t total, int64_t c, int64_t hw, int nhwc, T* y,
                                        const T* bias) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ch = nhwc ? i % c : (i / hw) % c;
    y[i] = IO<T>::cvt(IO<T>::ld(y + i) + IO<T>::ld(bias + ch));
  }
}

ms_status add_channel_bias(int dt, int layout, int64_t n, int64_t c, int64_t hw, void* y,
                           const void* bias, cudaStream_t st) {
  const int64_t total = n * c * hw;
  if (total == 0) return MS_OK;
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  const int nhwc = layout == MS_NHWC;
  switch (dt) {
    case MS_F32:
      add_channel_bias_kernel<float><<<(unsigned)blocks, 256, 0, st>>>(total, c, hw, nhwc,
                                                                      (float*)y, (const float*)bias);
      break;
    case MS_BF16:
      add_channel_bias_kernel<__nv_bfloat16><<<(unsigned)blocks, 256, 0, st>>>(
          total, c, hw, nhwc, (__nv_bfloat16*)y, (const __nv_bfloat16*)bias);
      break;
    default:
      add_channel_bias_kernel<__half><<<(unsigned)blocks, 256, 0, st>>>(
          total, c, hw, nhwc, (__half*)y, (const __half*)bias);
  }
  count_launch();
  return launch_status("add_channel_bias");
}

}  // namespace
}  // namespace ms

using namespace ms;

extern "C" int64_t ms_conv2d_out_h(const ms_conv_desc* d) {
  return (d->h + 2 * d->pad_h - d->r) / d->stride_h + 1;
}
extern "C" int64_t ms_conv2d_out_w(const ms_conv_desc* d) {
  return (d->w + 2 * d->pad_w - d->s) / d->stride_w + 1;
}

extern "C" size_t ms_conv2d_workspace(const ms_conv_desc* d, int32_t pass) {
  if (validate(d) != MS_OK) return 0;
  return plan(d, pass).ws;
}

extern "C" ms_status ms_conv2d_fwd(const ms_conv_desc* d, const void* x, const void* w,
                                   const void* bias, void* y, void* ws, size_t ws_bytes,
                                   void* stream) {
  MS_TRY(validate(d));
  MS_TRY(bind_device(y));
  if (d->n == 0) return MS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  ConvPlan p = plan(d, MS_CONV_FWD);
  MS_CHECK_ARG(ws_bytes >= p.ws && (p.ws == 0 || ws), MS_ERR_WORKSPACE,
               "conv fwd: workspace %zu < %zu", ws_bytes, p.ws);
  if (p.tc) return fwd_tc(d, p, x, w, bias, y, ws, st);
  if (d->dtype == MS_F32 && !bias) {
    const ms_status s = small_conv_fp32(MS_CONV_FWD, dims_of(d), d->layout, d->wlayout, x, w, y,
                                        ws, ws_bytes, st);
    if (s != MS_ERR_UNSUPPORTED) return s;
  }
  return simt_conv_fwd(dims_of(d), d->dtype, d->layout, d->wlayout, x, w, bias, y, st);
}

extern "C" ms_status ms_conv2d_dx(const ms_conv_desc* d, const void* dy, const void* w, void* dx,
                                  void* ws, size_t ws_bytes, void* stream) {
  MS_TRY(validate(d));
  MS_TRY(bind_device(dx));
  if (d->n == 0) return MS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  ConvPlan p = plan(d, MS_CONV_DX);
  MS_CHECK_ARG(ws_bytes >= p.ws && (p.ws == 0 || ws), MS_ERR_WORKSPACE,
               "conv dx: workspace %zu < %zu", ws_bytes, p.ws);
  if (p.tc) return dx_tc(d, p, dy, w, dx, ws, st);
  if (d->dtype == MS_F32) {
    const ms_status s = small_conv_fp32(MS_CONV_DX, dims_of(d), d->layout, d->wlayout, dy, w, dx,
                                        ws, ws_bytes, st);
    if (s != MS_ERR_UNSUPPORTED) return s;
  }
  return simt_conv_dx(dims_of(d), d->dtype, d->layout, d->wlayout, dy, w, dx, st);
}

extern "C" ms_status ms_conv2d_dw(const ms_conv_desc* d, const void* x, const void* dy, void* dw,
                                  void* ws, size_t ws_bytes, void* stream) {
  MS_TRY(validate(d));
  MS_TRY(bind_device(dw));
  cudaStream_t st = (cudaStream_t)stream;
  ConvPlan p = plan(d, MS_CONV_DW);
  MS_CHECK_ARG(ws_bytes >= p.ws && (p.ws == 0 || ws), MS_ERR_WORKSPACE,
               "conv dw: workspace %zu < %zu", ws_bytes, p.ws);
  if (d->n == 0) {
    return cudaMemsetAsync(dw, 0, dtype_size(d->dtype) * d->k * d->c * d->r * d->s, st) ==
                   cudaSuccess
               ? MS_OK
               : MS_ERR_LAUNCH;
  }
  if (p.tc) return dw_tc(d, p, x, dy, dw, ws, st);
  if (d->dtype == MS_F32) {
    const ms_status s = small_conv_fp32(MS_CONV_DW, dims_of(d), d->layout, d->wlayout, x, dy, dw,
                                        ws, ws_bytes, st);
    if (s != MS_ERR_UNSUPPORTED) return s;
  }
  return simt_conv_dw(dims_of(d), d->dtype, d->layout, d->wlayout, x, dy, dw, ws, ws_bytes, st);
}

extern "C" ms_status ms_conv2d_db(const ms_conv_desc* d, const void* dy, void* db, void* ws,
                                  size_t ws_bytes, void* stream) {
  MS_TRY(validate(d));
  MS_TRY(bind_device(db));
  MS_CHECK_ARG(ws && ws_bytes >= colsum_workspace(d->k), MS_ERR_WORKSPACE,
               "conv db: workspace too small");
  const ConvDims c = dims_of(d);
  cudaStream_t st = (cudaStream_t)stream;
  if (d->layout == MS_NHWC)
    return colsum((int64_t)c.n * c.oh * c.ow, c.k, d->dtype, dy, db, d->dtype, ws, st);
  return planesum(c.n, c.k, (int64_t)c.oh * c.ow, d->dtype, dy, db, d->dtype, ws, st);
}

extern "C" ms_status ms_conv_transpose2d_fwd(const ms_conv_desc* d, const void* x, const void* w,
                                             const void* bias, void* y, void* ws,
                                             size_t ws_bytes, void* stream) {
  // the input-VJP of the conv2d `d` (whose input is y, output x), plus a bias
  // per conv-input channel fused into the tcgen05 epilogue
  MS_TRY(validate(d));
  MS_TRY(bind_device(y));
  if (d->n == 0) return MS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  ConvPlan p = plan(d, MS_CONV_DX, bias != nullptr);
  MS_CHECK_ARG(ws_bytes >= p.ws && (p.ws == 0 || ws), MS_ERR_WORKSPACE,
               "conv_transpose2d fwd: workspace %zu < %zu", ws_bytes, p.ws);
  if (p.tc) return dx_tc(d, p, x, w, y, ws, st, bias);
  ms_status s = MS_ERR_UNSUPPORTED;
  if (d->dtype == MS_F32)
    s = small_conv_fp32(MS_CONV_DX, dims_of(d), d->layout, d->wlayout, x, w, y, ws, ws_bytes, st);
  if (s == MS_ERR_UNSUPPORTED)
    s = simt_conv_dx(dims_of(d), d->dtype, d->layout, d->wlayout, x, w, y, st);
  MS_TRY(s);
  if (bias) MS_TRY(add_channel_bias(d->dtype, d->layout, d->n, d->c, d->h * d->w, y, bias, st));
  return MS_OK;
}

// ----------------------------------------------------------------- conv + BN-eval (+ ReLU)
extern "C" size_t ms_conv2d_bn_workspace(const ms_conv_desc* d) {
  if (validate(d) != MS_OK) return 0;
  return plan(d, MS_CONV_FWD).ws;
}

extern "C" ms_status ms_conv2d_bn_fwd(const ms_conv_desc* d, const void* x, const void* w,
                                      const void* bias, const void* bn_mean, const void* bn_var,
                                      const void* bn_weight, const void* bn_bias,
                                      int32_t bn_pdtype, double eps, const void* residual,
                                      int32_t relu, void* y, void* mask_or_null, void* ws,
                                      size_t ws_bytes, void* stream) {
  MS_TRY(validate(d));
  MS_TRY(bind_device(y));
  MS_CHECK_ARG((bn_mean && bn_var) || (!bn_mean && !bn_var), MS_ERR_SHAPE,
               "conv+bn: give both running statistics (or neither for conv [+ relu] only)");
  if (d->n == 0) return MS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  ConvPlan p = plan(d, MS_CONV_FWD);
  MS_CHECK_ARG(p.tc && d->k % 8 == 0, MS_ERR_UNSUPPORTED,
               "conv+bn fusion needs the tcgen05 path (16-bit NHWC) and K %% 8 == 0");
  MS_CHECK_ARG(ws_bytes >= p.ws && (p.ws == 0 || ws), MS_ERR_WORKSPACE,
               "conv+bn: workspace %zu < %zu", ws_bytes, p.ws);
  Fuse f;
  if (bn_mean) {  // folded per channel inside the conv epilogue (BnFold)
    f.bn.mean = bn_mean;
    f.bn.var = bn_var;
    f.bn.w = bn_weight;
    f.bn.b = bn_bias;
    f.bn.pdt = bn_pdtype;
    f.bn.eps = (float)eps;
  }
  f.relu = relu;
  f.mask = static_cast<uint8_t*>(mask_or_null);
  f.resid = residual;
  MS_CHECK_ARG(!residual || (reinterpret_cast<uintptr_t>(residual) & 15) == 0, MS_ERR_ALIGN,
               "conv+bn: residual must be 16-byte aligned");
  return fwd_tc(d, p, x, w, bias, y, ws, st, &f);
}

extern "C" ms_status ms_conv2d_bn_dx(const ms_conv_desc* d, const void* dy, const void* w,
                                     const void* bn_var, const void* bn_weight, int32_t bn_pdtype,
                                     double eps, const void* addend, const void* keep,
                                     const void* in_var, const void* in_weight, int32_t in_pdtype,
                                     double in_eps, void* dx, void* ws, size_t ws_bytes,
                                     void* stream) {
  MS_TRY(validate(d));
  MS_TRY(bind_device(dx));
  if (d->n == 0) return MS_OK;
  ConvPlan p = plan(d, MS_CONV_DX, /*dx_bias=*/true);  // the generic phase GEMM, no band kernel
  MS_CHECK_ARG(p.tc && !p.stem && !p.band, MS_ERR_UNSUPPORTED,
               "conv+bn dx: the folded-scale / addend path needs the tcgen05 dgrad");
  MS_CHECK_ARG(ws_bytes >= p.ws && (p.ws == 0 || ws), MS_ERR_WORKSPACE,
               "conv+bn dx: workspace %zu < %zu", ws_bytes, p.ws);
  MS_CHECK_ARG(!addend || (reinterpret_cast<uintptr_t>(addend) & 15) == 0, MS_ERR_ALIGN,
               "conv+bn dx: addend must be 16-byte aligned");
  MS_CHECK_ARG(!keep || (reinterpret_cast<uintptr_t>(keep) & 3) == 0, MS_ERR_ALIGN,
               "conv+bn dx: keep mask must be 4-byte aligned");
  DxFuse xf;
  xf.addend = addend;
  xf.keep = static_cast<const uint8_t*>(keep);
  xf.in_bn.var = in_var;
  xf.in_bn.w = in_weight;
  xf.in_bn.pdt = in_pdtype;
  xf.in_bn.eps = (float)in_eps;
  KScale ks;
  ks.var = bn_var;
  ks.weight = bn_weight;
  ks.pdt = bn_pdtype;
  ks.eps = (float)eps;
  return dx_tc(d, p, dy, w, dx, ws, (cudaStream_t)stream, nullptr, bn_var ? &ks : nullptr, &xf);
}
