// 3x3 / stride-1 / pad-1 convolution with 64 -> 64 channels (ResNet layer1)
// as a halo-tiled tcgen05 kernel: forward, and the input-VJP as the same
// convolution of dY with the transposed, flipped kernel.
//
// The im2col implicit GEMM stages every input pixel 9 times through shared
// memory (one 128-pixel box per tap); with N = 64 output channels that is
// ~3x the 128 B/clk an SM's shared memory delivers, so the tensor core idles.
// Here a tile is 2 output rows of one image (M = 128 = 2 x 64: the row pitch
// is 64 pixels, W <= 62 of them real).  The tile's 4 input rows (the halo,
// pixels -1 .. 62, OOB zeros) are loaded once by TMA with the 128-byte
// swizzle; the A operand of tap (r, s) is the same buffer started (r*64 + s)
// rows later -- a swizzled K-major operand whose start is not 1024-byte
// aligned (the hardware swizzles by absolute address, like TMA did).
// The 9 weight taps ([64 n][64 c], 72 KB) stay resident in shared memory.
// Per tile: 32 KB of TMA traffic instead of 216 KB, 36 MMAs of 128x64x16.
// Epilogue: 4 warps (TMEM lane quarters = 32 output pixels of one row), the
// same fused eval-BN / residual / ReLU + bit mask as the generic kernel, TMA
// stores through a 3-D map [N*H][W][K] that clips the pitch padding.
#include <cstdlib>

#include "misc.cuh"

namespace ms {
namespace {

constexpr int H3_C = 64;                    // reduction channels (one 128-B row)
constexpr int H3_N = 64;                    // output channels (UMMA N)
constexpr int H3_B = 9 * H3_N * 128;        // 9 taps x [64 n][64 c]
constexpr int H3_EPI = 8;  // warps per epilogue group: 2 per TMEM lane quarter, 32 ch each
constexpr int H3_ACC = 4;                   // TMEM accumulators (4 x 64 columns) in flight

// Tile geometry.  WIDE = 0 (rows of <= 62 pixels): 2 output rows at a 64-pixel
// pitch.  WIDE = 1 (any width, VGG's 224): 1 output row segment of 128
// pixels; its 130-pixel halo rows sit at a 136-pixel pitch (1024-byte aligned
// TMA destinations), so tap (r, s) still reads rows r*136 + s .. + 127.
template <int WIDE>
struct H3Geo {
  static constexpr int ROWS = WIDE ? 1 : 2;            // output rows per tile
  static constexpr int SEG = WIDE ? 128 : 64;          // tile pixels per output row
  static constexpr int P = WIDE ? 136 : 64;            // halo row pitch in pixels
  static constexpr int BOXW = WIDE ? 130 : 64;         // halo pixels loaded per row
  static constexpr int HALO = (ROWS + 2) * P * 128;    // bytes per stage
  static constexpr int STAGES = 2;
  // epilogue groups: 2 alternate tiles (16 warps) where the smem allows it, so
  // the fused epilogue (residual / addend / masks) keeps pace with the MMAs
  static constexpr int NG = WIDE ? 1 : 2;
  static constexpr int EPI = NG * H3_EPI;
  static constexpr int THREADS = 64 + 32 * EPI;
  static constexpr int STG = EPI * 2 * 2048;  // TMA-store staging, 2 x (32 px x 32 ch) per warp
  static constexpr int SMEM = H3_B + STAGES * HALO + STG + 1024 + 256;
};

struct H3Args {
  int N, H, W;        // activation (input == output spatial size)
  int tiles_per_img;  // ceil(H / ROWS) row tiles per image
  int segs;           // WIDE: 128-pixel segments per row (else 1)
  int units;
  int dt;
  void* y;
  BnFold bn;           // fused eval-BN (bn.var nullable)
  const void* bias;    // conv bias (nullable)
  const void* resid;   // residual, shaped like y (nullable)
  int relu;
  uint8_t* mask;
  const uint8_t* keep_in;  // dgrad: the producer ReLU's mask, applied after resid
  int bn_post;             // dgrad: then scale by the producer BN's s (bn)
  int dbg;                 // profiling (MS_H3_DBG): 1 = every tap reads the s = 0 rows
};

// SW128 K-major descriptor whose start may sit at any 128-byte row of a
// 1024-byte swizzle atom.  Measured on B200: the tensor core applies the
// 128-byte XOR pattern from the absolute shared-memory address bits, exactly
// as TMA wrote it, so the base-offset field stays 0 (setting it to the row
// phase double-applies the shift; tests/test_gpu_parity.py halo cases).
__device__ __forceinline__ uint64_t desc_sw128_rows(uint32_t saddr) {
  return make_smem_desc(saddr, 16, 1024, LAYOUT_SWIZZLE_128B);
}

template <typename T, int WIDE>
__global__ void __launch_bounds__(H3Geo<WIDE>::THREADS, 1)
    conv3x3_halo_kernel(const __grid_constant__ CUtensorMap tma_x,
                        const __grid_constant__ CUtensorMap tma_w,
                        const __grid_constant__ CUtensorMap tma_y,
                        const __grid_constant__ H3Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // aligned by an offset from the shared array (keeps the accesses STS / LDS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  using G = H3Geo<WIDE>;
  constexpr int H3_ROWS = G::ROWS, H3_P = G::P, H3_HALO = G::HALO, H3_STAGES = G::STAGES;
  uint8_t* sB = smem;
  uint8_t* ring = smem + H3_B;
  uint8_t* staging = ring + H3_STAGES * H3_HALO;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + G::STG);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + H3_STAGES;
  uint64_t* tfull_bar = bars + 2 * H3_STAGES;
  uint64_t* tempty_bar = bars + 2 * H3_STAGES + H3_ACC;
  uint64_t* b_bar = bars + 2 * H3_STAGES + 2 * H3_ACC;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * H3_STAGES + 2 * H3_ACC + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < H3_STAGES; ++i) {
      mbar_init(smem_u32(&full_bar[i]), 1);
      mbar_init(smem_u32(&empty_bar[i]), 1);
    }
    for (int i = 0; i < H3_ACC; ++i) {
      mbar_init(smem_u32(&tfull_bar[i]), 1);
      mbar_init(smem_u32(&tempty_bar[i]), H3_EPI);  // one group drains each tile
    }
    mbar_init(smem_u32(b_bar), 1);
    fence_mbar_init();
    tma_prefetch_desc(&tma_x);
    tma_prefetch_desc(&tma_w);
    tma_prefetch_desc(&tma_y);
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_holder), H3_ACC * H3_N);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ============================ TMA producer ============================
    {  // whole warp (uniform coordinates), an elect.sync lane issues
      const uint32_t bb = smem_u32(b_bar);
      if (elect_one()) {
        mbar_arrive_expect_tx(bb, H3_B);
        for (int t = 0; t < 9; ++t) tma_load_2d(smem_u32(sB + t * 8192), &tma_w, bb, 0, t * H3_N);
      }
      __syncwarp();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
        const int n = u / (a.tiles_per_img * a.segs);
        const int rem = u - n * (a.tiles_per_img * a.segs);
        const int i0 = (rem / a.segs) * H3_ROWS;
        const int x0 = (rem - (rem / a.segs) * a.segs) * G::SEG;
        mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
        const uint32_t fb = smem_u32(&full_bar[stage]);
        const uint32_t sh = smem_u32(ring + stage * H3_HALO);
        if (elect_one()) {
          mbar_arrive_expect_tx(fb, (H3_ROWS + 2) * G::BOXW * 128);
#pragma unroll
          for (int rr = 0; rr < H3_ROWS + 2; ++rr)  // input rows i0-1 .., pixels x0-1 ..
            tma_load_4d(sh + rr * H3_P * 128, &tma_x, fb, 0, x0 - 1, i0 - 1 + rr, n);
        }
        __syncwarp();
        if (++stage == H3_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    // whole warp: descriptors in uniform registers; an elect.sync lane issues
    // the 36 MMAs of a tile back to back (no per-MMA ELECT / R2UR waterfall)
    {
      const uint32_t idesc = make_idesc_f16(a.dt == MS_BF16 ? 1 : 0, BM, H3_N, 0, 0);
      const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
      const uint32_t ring_u = smem_u32(ring), sB_u = smem_u32(sB);
      mbar_wait(smem_u32(b_bar), 0);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int u = blockIdx.x; u < a.units; u += gridDim.x, ++local) {
        const int acc = local % H3_ACC;
        mbar_wait(smem_u32(&tempty_bar[acc]), ((local / H3_ACC) & 1) ^ 1);
        mbar_wait(smem_u32(&full_bar[stage]), phase);
        tc_fence_after();
        const uint32_t dcol = tmem_u + acc * H3_N;
        const uint32_t sh = ring_u + stage * H3_HALO;
        if (elect_one()) {
#pragma unroll
          for (int t = 0; t < 9; ++t) {
            const int r = t / 3, s = t - (t / 3) * 3;
            // output pixel m' = i*64 + j reads halo row (i + r)*64 + (j + s)
            const uint32_t arow = sh + (r * H3_P + (a.dbg & 1 ? 0 : s)) * 128;
            const uint32_t brow = sB_u + t * 8192;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_f16(dcol, desc_sw128_rows(arow + k * 32),
                       make_smem_desc(brow + k * 32, 16, 1024, LAYOUT_SWIZZLE_128B), idesc,
                       (t > 0 || k > 0) ? 1u : 0u);
          }
          umma_commit(smem_u32(&empty_bar[stage]));
          umma_commit(smem_u32(&tfull_bar[acc]));
        }
        __syncwarp();
        if (++stage == H3_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ============================ epilogue ============================
    // 8 warps: warp w drains TMEM lane quarter w % 4 (its pixels) and channel half
    // (w - 2) / 4 -- twice the warps of one per quarter, so the fused epilogue
    // (BN affine, residual / addend, masks) keeps up with the 36-MMA tiles
    const int quarter = static_cast<int>(warp & 3);
    const int ew = static_cast<int>(warp) - 2;
    const int grp = ew / H3_EPI;           // epilogue group: tiles grp, grp + NG, ...
    const int c0 = ((ew % H3_EPI) >> 2) * 32;  // this warp's 32 output channels
    const int rw = static_cast<int>(lane);
    const int ti = WIDE ? 0 : quarter >> 1;           // output row within the tile
    const int j0 = WIDE ? quarter * 32 : (quarter & 1) * 32;  // first pixel of the warp's 32
    const int j = j0 + rw;
    int local = grp;  // the CTA's tile sequence number (accumulator ring position)
    uint32_t nst = 0;
    float bs0 = 1.f, bt0 = 0.f;  // eval-BN affine of channel c0 + lane
    if (a.bn.var) bn_fold(a.bn, c0 + rw, bs0, bt0);
    for (int u = blockIdx.x + grp * gridDim.x; u < a.units;
         u += G::NG * gridDim.x, local += G::NG) {
      const int n = u / (a.tiles_per_img * a.segs);
      const int rem = u - n * (a.tiles_per_img * a.segs);
      const int oh = (rem / a.segs) * H3_ROWS + ti;
      const int x0 = (rem - (rem / a.segs) * a.segs) * G::SEG;
      const bool row_ok = oh < a.H;
      const bool valid = row_ok && x0 + j < a.W;
      const int64_t pix = (static_cast<int64_t>(n) * a.H + oh) * a.W + x0 + j;
      const int buf = local % H3_ACC;
      mbar_wait(smem_u32(&tfull_bar[buf]), (local / H3_ACC) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((static_cast<uint32_t>(quarter) * 32u) << 16) + buf * H3_N;
      uint32_t v0[32];
      tmem_ld_32x32b_x32(taddr + c0, v0);
      tmem_ld_wait_regs(v0);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&tempty_bar[buf]));
      {
        float f[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) f[q] = __uint_as_float(v0[q]);
        if (a.bias) {
#pragma unroll
          for (int q = 0; q < 32; ++q) f[q] += IO<T>::ld(static_cast<const T*>(a.bias) + c0 + q);
        }
        if (a.bn.var && !a.bn_post) {  // lane j holds channel c0 + j's folded BN affine
#pragma unroll
          for (int q = 0; q < 32; ++q)
            f[q] = f[q] * __shfl_sync(0xffffffffu, bs0, q) + __shfl_sync(0xffffffffu, bt0, q);
        }
        if (a.resid && valid) {
          const uint4* r4 = reinterpret_cast<const uint4*>(static_cast<const T*>(a.resid) +
                                                           pix * H3_N + c0);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 u4 = __ldg(r4 + q);
            const T* e = reinterpret_cast<const T*>(&u4);
#pragma unroll
            for (int h = 0; h < 8; ++h) f[q * 8 + h] += IO<T>::ld(e + h);
          }
        }
        if (a.keep_in) {
          const uint32_t kb =
              valid ? __ldg(reinterpret_cast<const uint32_t*>(a.keep_in) + ((pix * H3_N + c0) >> 5))
                    : 0u;
#pragma unroll
          for (int q = 0; q < 32; ++q) f[q] = ((kb >> q) & 1u) ? f[q] : 0.f;
        }
        if (a.bn_post) {
#pragma unroll
          for (int q = 0; q < 32; ++q) f[q] *= __shfl_sync(0xffffffffu, bs0, q);
        }
        if (a.relu) {
          uint32_t bits = 0;
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const bool pos = !(f[q] <= 0.f);
            bits |= (pos ? 1u : 0u) << q;
            f[q] = pos ? f[q] : 0.f;
          }
          if (a.mask && valid) reinterpret_cast<uint32_t*>(a.mask)[(pix * H3_N + c0) >> 5] = bits;
        }
        // stage 32 pixels x 32 channels (64-byte rows, 64-byte swizzle), one TMA store
        uint8_t* sb = staging + (ew * 2 + (nst & 1)) * 2048;
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 pk;
          pk.x = pack2<T>(f[8 * q], f[8 * q + 1]);
          pk.y = pack2<T>(f[8 * q + 2], f[8 * q + 3]);
          pk.z = pack2<T>(f[8 * q + 4], f[8 * q + 5]);
          pk.w = pack2<T>(f[8 * q + 6], f[8 * q + 7]);
          *reinterpret_cast<uint4*>(sb + rw * 64 + ((q ^ ((rw >> 1) & 3)) << 4)) = pk;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && row_ok) {
          tma_store_3d(&tma_y, smem_u32(sb), c0, x0 + j0, n * a.H + oh);
          bulk_commit();
        }
        ++nst;
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, H3_ACC * H3_N);
  }
}

// [tap][n][c] K-major weight tiles: fwd n = out channel k, c = in channel;
// dgrad (transpose) n = in channel c, c = out channel k, taps flipped.
// kvar (nullable, dgrad): scale out-channel k by kw[k]/sqrt(kvar[k]+eps).
template <typename T>
__global__ void repack_h3_kernel(int wlayout, int transpose, const T* __restrict__ w,
                                 T* __restrict__ out, const void* kvar, const void* kw, int pdt,
                                 float eps) {
  const int total = 9 * H3_N * H3_C;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int cc = i % H3_C, nn = (i / H3_C) % H3_N, t = i / (H3_C * H3_N);
    int k, c, r, s;
    if (!transpose) {
      k = nn; c = cc; r = t / 3; s = t % 3;
    } else {
      k = cc; c = nn; r = 2 - t / 3; s = 2 - t % 3;
    }
    T v = wlayout == MS_NHWC ? w[((k * 3 + r) * 3 + s) * H3_C + c]
                             : w[((k * H3_C + c) * 3 + r) * 3 + s];
    if (kvar) {
      const float sc = (kw ? load_as_float(kw, pdt, k) : 1.f) /
                       sqrtf(load_as_float(kvar, pdt, k) + eps);
      v = IO<T>::cvt(IO<T>::ld(&v) * sc);
    }
    out[i] = v;
  }
}

}  // namespace

bool conv3x3_halo_ok(int dt, int layout, int c, int k, int r, int s, int sh, int sw, int ph,
                     int pw, int w) {
  static const bool off = getenv("MS_NO_HALO3") != nullptr;  // A/B switch
  return !off && (dt == MS_BF16 || dt == MS_F16) && layout == MS_NHWC && c == H3_C &&
         k == H3_N && r == 3 && s == 3 && sh == 1 && sw == 1 && ph == 1 && pw == 1;
}

size_t conv3x3_halo_workspace() { return align256((size_t)9 * H3_N * H3_C * 2); }

// x [N][H][W][64] -> y [N][H][W][64] (NHWC); transpose = 1: the input-VJP (x = dY,
// y = dX, weights transposed and flipped, optional folded BN scale in ks_*)
ms_status conv3x3_halo(int dt, int n, int h, int w, int wlayout, int transpose, const void* x,
                       const void* wt, void* ws, void* y, const BnFold& bn, const void* bias, const void* resid, int relu, uint8_t* mask,
                       const void* ks_var, const void* ks_w, int ks_pdt, float ks_eps,
                       cudaStream_t st, const uint8_t* keep_in, int bn_post) {
  const int total = 9 * H3_N * H3_C;
  if (dt == MS_BF16)
    repack_h3_kernel<__nv_bfloat16><<<(total + 255) / 256, 256, 0, st>>>(
        wlayout, transpose, (const __nv_bfloat16*)wt, (__nv_bfloat16*)ws, ks_var, ks_w, ks_pdt,
        ks_eps);
  else
    repack_h3_kernel<__half><<<(total + 255) / 256, 256, 0, st>>>(
        wlayout, transpose, (const __half*)wt, (__half*)ws, ks_var, ks_w, ks_pdt, ks_eps);
  count_launch();
  MS_TRY(launch_status("repack_h3"));
  const size_t es = dtype_size(dt);
  CUtensorMap tx, tw, ty;
  const bool wide = w + 2 > H3Geo<0>::P;  // rows wider than 62 pixels: 128-pixel segments
  {
    const uint64_t dims[4] = {(uint64_t)H3_C, (uint64_t)w, (uint64_t)h, (uint64_t)n};
    const uint64_t str[3] = {H3_C * es, (uint64_t)w * H3_C * es, (uint64_t)h * w * H3_C * es};
    const uint32_t box[4] = {64, (uint32_t)(wide ? H3Geo<1>::BOXW : H3Geo<0>::BOXW), 1, 1};
    MS_TRY(make_tmap_nd(&tx, dt, x, 4, dims, str, box, 128));
  }
  MS_TRY(make_tmap_2d(&tw, dt, ws, H3_C, 9 * H3_N, H3_C, 64, H3_N));
  {
    const uint64_t dims[3] = {(uint64_t)H3_N, (uint64_t)w, (uint64_t)n * h};
    const uint64_t str[2] = {H3_N * es, (uint64_t)w * H3_N * es};
    const uint32_t box[3] = {32, 32, 1};
    MS_TRY(make_tmap_nd(&ty, dt, y, 3, dims, str, box, 64));
  }
  H3Args a{};
  a.N = n; a.H = h; a.W = w;
  const int rows = wide ? H3Geo<1>::ROWS : H3Geo<0>::ROWS;
  a.tiles_per_img = (h + rows - 1) / rows;
  a.segs = wide ? (w + H3Geo<1>::SEG - 1) / H3Geo<1>::SEG : 1;
  a.units = n * a.tiles_per_img * a.segs;
  {
    static const int env_dbg = [] {
      const char* e = getenv("MS_H3_DBG");
      return e ? atoi(e) : 0;
    }();
    a.dbg = env_dbg;
  }
  a.dt = dt; a.y = y; a.bn = bn; a.bias = bias; a.resid = resid;
  a.relu = relu; a.mask = mask; a.keep_in = keep_in; a.bn_post = bn_post;
  const int grid = a.units < num_sms() ? a.units : num_sms();
  auto go = [&](auto kern, int smem, int threads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<grid, threads, smem, st>>>(tx, tw, ty, a);
  };
  if (dt == MS_BF16) {
    if (wide) go(conv3x3_halo_kernel<__nv_bfloat16, 1>, H3Geo<1>::SMEM, H3Geo<1>::THREADS);
    else go(conv3x3_halo_kernel<__nv_bfloat16, 0>, H3Geo<0>::SMEM, H3Geo<0>::THREADS);
  } else {
    if (wide) go(conv3x3_halo_kernel<__half, 1>, H3Geo<1>::SMEM, H3Geo<1>::THREADS);
    else go(conv3x3_halo_kernel<__half, 0>, H3Geo<0>::SMEM, H3Geo<0>::THREADS);
  }
  count_launch(1, KF_UMMA);
  return launch_status("conv3x3_halo_kernel");
}

}  // namespace ms
