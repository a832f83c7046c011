// Input-VJP of the 3-channel 7x7 / stride-2 / pad-3 stem convolution (the
// ResNet stem), as one warp-specialised tcgen05 kernel with a register
// col2im -- the dominant launch of the ResNet-18 input-only step.
//
// Scatter form (numba_impl.py:36-54): dX[n, 2*oh-3+r, 2*ow-3+s, c] +=
// sum_k dY[n, oh, ow, k] W[k, c, r, s].  Per dY row the tensor core computes
// P[ow][(r, s, c)] = dY[oh, ow, :] . W[:, c, r, s]  (M = 128 pixels, N = 160 >=
// 147 columns, K = 64 channels), then the epilogue scatters P into dX without
// atomics or shared-memory read-modify-writes:
//
//  * columns: lane q (dY pixel ow = q) owns dX columns 2q and 2q+1.  Column 2q
//    receives s = 5, 3, 1 from pixels q-1, q, q+1, column 2q+1 receives s = 6,
//    4, 2, 0 from pixels q-1 .. q+2, gathered with warp shuffles.  A 32-lane
//    segment therefore owns the 29 pixels of lanes 1..29; the 128-row tile is
//    4 segments starting 29 pixels apart (4 TMA boxes of 32 pixels, padding
//    pixels are TMA out-of-bounds zeros), covering rows of up to 116 pixels.
//  * rows: dY row oh adds to dX rows 2oh-3 .. 2oh+3; a lane keeps those 7 rows
//    x 2 columns x 3 channels in registers, and after row oh the dX rows 2oh-3
//    and 2oh-2 are complete and go straight to global memory.  A work unit is
//    32 dX rows of one image: dY rows 16b-1 .. 16b+17 (3 warm-up rows).
//
// dY is read once from HBM (411 MB at ResNet-18 b256) and dX written once;
// the weight tile (160 x K) stays in shared memory for the whole launch.
#include "misc.cuh"

namespace ms {
namespace {

constexpr int SD_C = 3, SD_R = 7, SD_S = 7;
constexpr int SD_N = 160;     // 147 (tap, channel) columns padded to a UMMA N
constexpr int SD_SEG = 29;    // dY pixels owned per 32-lane segment
constexpr int SD_SEGS = 4;    // segments per 128-row tile
constexpr int SD_BAND = 16;   // dY rows (32 dX rows) owned per work unit
constexpr int SD_STAGES = 6;
constexpr int SD_EPI = 4;
constexpr int SD_THREADS = 64 + 32 * SD_EPI;
constexpr int SD_A_BYTES = BM * 128;       // 128 pixels x 64 channels (bf16)
constexpr int SD_B_KB_BYTES = SD_N * 128;  // 160 rows x 64 channels per k-block

struct StemDgradArgs {
  int N, H, W;     // dX
  int P, Q, K;     // dY rows, columns, channels
  int kblocks;     // K / 64
  int bands;       // work units per image
  int units;
  void* dx;
  int dt;          // MS_BF16 / MS_F16
};

__host__ __device__ constexpr int sd_smem_bytes(int kblocks) {
  return kblocks * SD_B_KB_BYTES + SD_STAGES * SD_A_BYTES + 1024 + 256;
}

template <typename T>
__global__ void __launch_bounds__(SD_THREADS, 1)
    stem_dgrad_kernel(const __grid_constant__ CUtensorMap tma_dy,
                      const __grid_constant__ CUtensorMap tma_w,
                      const __grid_constant__ StemDgradArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sB = smem;
  uint8_t* ring = smem + a.kblocks * SD_B_KB_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + SD_STAGES * SD_A_BYTES);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + SD_STAGES;
  uint64_t* tfull_bar = bars + 2 * SD_STAGES;
  uint64_t* tempty_bar = bars + 2 * SD_STAGES + 2;
  uint64_t* b_bar = bars + 2 * SD_STAGES + 4;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * SD_STAGES + 5);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < SD_STAGES; ++i) {
      mbar_init(smem_u32(&full_bar[i]), 1);
      mbar_init(smem_u32(&empty_bar[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&tfull_bar[i]), 1);
      mbar_init(smem_u32(&tempty_bar[i]), SD_EPI);  // one arrival per epilogue warp
    }
    mbar_init(smem_u32(b_bar), 1);
    fence_mbar_init();
    tma_prefetch_desc(&tma_dy);
    tma_prefetch_desc(&tma_w);
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_holder), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int rows_per_unit = SD_BAND + 3;

  if (warp == 0) {
    // ============================ TMA producer ============================
    {  // whole warp (uniform operands), an elect.sync lane issues
      const uint32_t bb = smem_u32(b_bar);
      if (elect_one()) {
        mbar_arrive_expect_tx(bb, a.kblocks * SD_B_KB_BYTES);
        for (int kb = 0; kb < a.kblocks; ++kb)
          tma_load_2d(smem_u32(sB + kb * SD_B_KB_BYTES), &tma_w, bb, kb * 64, 0);
      }
      __syncwarp();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
        const int n = u / a.bands, b = u - (u / a.bands) * a.bands;
        for (int i = 0; i < rows_per_unit; ++i) {
          const int oh = SD_BAND * b - 1 + i;  // rows outside [0, P) load zeros
          for (int kb = 0; kb < a.kblocks; ++kb) {
            mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
            const uint32_t fb = smem_u32(&full_bar[stage]);
            const uint32_t sA = smem_u32(ring + stage * SD_A_BYTES);
            if (elect_one()) {
              mbar_arrive_expect_tx(fb, SD_A_BYTES);
#pragma unroll
              for (int w = 0; w < SD_SEGS; ++w)
                tma_load_4d(sA + w * 4096, &tma_dy, fb, kb * 64, SD_SEG * w - 1, oh, n);
            }
            __syncwarp();
            if (++stage == SD_STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    {  // whole warp: descriptors in uniform registers; an elect.sync lane issues
      const uint32_t idesc = make_idesc_f16(a.dt == MS_BF16 ? 1 : 0, BM, SD_N, 0, 0);
      const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
      mbar_wait(smem_u32(b_bar), 0);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
        for (int i = 0; i < rows_per_unit; ++i, ++local) {
          const int acc = local & 1;
          mbar_wait(smem_u32(&tempty_bar[acc]), ((local >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t dcol = tmem_u + acc * SD_N;
          for (int kb = 0; kb < a.kblocks; ++kb) {
            mbar_wait(smem_u32(&full_bar[stage]), phase);
            tc_fence_after();
            const uint32_t sA = smem_u32(ring + stage * SD_A_BYTES);
            const uint32_t sBk = smem_u32(sB + kb * SD_B_KB_BYTES);
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint64_t ad = make_smem_desc(sA + k * 32, 16, 1024, LAYOUT_SWIZZLE_128B);
                const uint64_t bd = make_smem_desc(sBk + k * 32, 16, 1024, LAYOUT_SWIZZLE_128B);
                umma_f16(dcol, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
              }
              umma_commit(smem_u32(&empty_bar[stage]));
            }
            __syncwarp();
            if (++stage == SD_STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (elect_one()) umma_commit(smem_u32(&tfull_bar[acc]));
          __syncwarp();
        }
      }
    }
  } else {
    // ============================ epilogue ============================
    const int seg = static_cast<int>(warp & 3);  // TMEM lane quarter = pixel segment
    const int l = static_cast<int>(lane);
    const int q = SD_SEG * seg - 1 + l;           // dY column of this lane
    const bool owner = l >= 1 && l <= SD_SEG && q < a.Q;
    const uint32_t taddr = tmem_base + ((static_cast<uint32_t>(seg) * 32u) << 16);
    T* dx = static_cast<T*>(a.dx);
    const bool pairs = (a.W & 1) == 0;  // 3-element column pairs start 4-byte aligned
    int local = 0;
    for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
      const int n = u / a.bands, b = u - (u / a.bands) * a.bands;
      const int h0 = 2 * SD_BAND * b;
      float acc[SD_R][6];
#pragma unroll
      for (int r = 0; r < SD_R; ++r)
#pragma unroll
        for (int j = 0; j < 6; ++j) acc[r][j] = 0.f;
      for (int i = 0; i < rows_per_unit; ++i, ++local) {
        const int oh = SD_BAND * b - 1 + i;
        const int buf = local & 1;
        mbar_wait(smem_u32(&tfull_bar[buf]), (local >> 1) & 1);
        tc_fence_after();
        uint32_t p[5][32];
#pragma unroll
        for (int j = 0; j < 5; ++j) tmem_ld_32x32b_x32(taddr + buf * SD_N + 32 * j, p[j]);
#pragma unroll
        for (int j = 0; j < 5; ++j) tmem_ld_wait_regs(p[j]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&tempty_bar[buf]));  // TMEM free for row i+2
        // gather the 7 x 2 x 3 contributions of this dY row to the lane's columns
#define SD_P(r, s, c) __uint_as_float(p[(((r) * SD_S + (s)) * SD_C + (c)) >> 5][(((r) * SD_S + (s)) * SD_C + (c)) & 31])
#pragma unroll
        for (int r = 0; r < SD_R; ++r) {
#pragma unroll
          for (int c = 0; c < SD_C; ++c) {
            const float ev = __shfl_up_sync(0xffffffffu, SD_P(r, 5, c), 1) + SD_P(r, 3, c) +
                             __shfl_down_sync(0xffffffffu, SD_P(r, 1, c), 1);
            const float od = __shfl_up_sync(0xffffffffu, SD_P(r, 6, c), 1) + SD_P(r, 4, c) +
                             __shfl_down_sync(0xffffffffu, SD_P(r, 2, c), 1) +
                             __shfl_down_sync(0xffffffffu, SD_P(r, 0, c), 2);
            acc[r][c] += ev;
            acc[r][3 + c] += od;
          }
        }
#undef SD_P
        // dX rows 2oh-3 and 2oh-2 are complete: store the owned ones
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int h = 2 * oh - 3 + r;
          if (owner && h >= h0 && h < h0 + 2 * SD_BAND && h < a.H) {
            const int64_t o = ((static_cast<int64_t>(n) * a.H + h) * a.W + 2 * q) * SD_C;
            if (pairs) {
              uint32_t* o32 = reinterpret_cast<uint32_t*>(dx + o);
              o32[0] = pack2<T>(acc[r][0], acc[r][1]);
              o32[1] = pack2<T>(acc[r][2], acc[r][3]);
              o32[2] = pack2<T>(acc[r][4], acc[r][5]);
            } else {
              for (int j = 0; j < 6; ++j)
                if (2 * q + j / 3 < a.W) dx[o + j] = IO<T>::cvt(acc[r][j]);
            }
          }
        }
#pragma unroll
        for (int r = 0; r < SD_R - 2; ++r)
#pragma unroll
          for (int j = 0; j < 6; ++j) acc[r][j] = acc[r + 2][j];
#pragma unroll
        for (int j = 0; j < 6; ++j) acc[SD_R - 2][j] = acc[SD_R - 1][j] = 0.f;
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace

bool stem_dgrad_ok(int dt, int layout, int c, int r, int s, int sh, int sw, int ph, int pw,
                   int64_t ow, int64_t k) {
  return (dt == MS_BF16 || dt == MS_F16) && layout == MS_NHWC && c == SD_C && r == SD_R &&
         s == SD_S && sh == 2 && sw == 2 && ph == 3 && pw == 3 && ow <= SD_SEG * SD_SEGS &&
         k % 64 == 0 && k <= 256;
}

// dy [n][P][Q][K] NHWC, wt = repack_scatter output [147][kpad=K] K-major, dx NHWC
ms_status stem_dgrad(int dt, int n, int h, int w, int p, int q, int k, const void* dy,
                     const void* wt, void* dx, cudaStream_t st) {
  const size_t es = dtype_size(dt);
  StemDgradArgs a{};
  a.N = n; a.H = h; a.W = w; a.P = p; a.Q = q; a.K = k;
  a.kblocks = k / 64;
  a.bands = (h + 2 * SD_BAND - 1) / (2 * SD_BAND);
  a.units = n * a.bands;
  a.dx = dx;
  a.dt = dt;
  CUtensorMap tdy, tw;
  const uint64_t dims[4] = {(uint64_t)k, (uint64_t)q, (uint64_t)p, (uint64_t)n};
  const uint64_t str[3] = {(uint64_t)k * es, (uint64_t)q * k * es, (uint64_t)p * q * k * es};
  const uint32_t box[4] = {64, 32, 1, 1};
  MS_TRY(make_tmap_nd(&tdy, dt, dy, 4, dims, str, box, 128));
  MS_TRY(make_tmap_2d(&tw, dt, wt, k, SD_R * SD_S * SD_C, k, BK, SD_N));
  const int smem = sd_smem_bytes(a.kblocks);
  if (dt == MS_BF16) {
    auto kern = stem_dgrad_kernel<__nv_bfloat16>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = a.units < num_sms() ? a.units : num_sms();
    kern<<<grid, SD_THREADS, smem, st>>>(tdy, tw, a);
  } else {
    auto kern = stem_dgrad_kernel<__half>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = a.units < num_sms() ? a.units : num_sms();
    kern<<<grid, SD_THREADS, smem, st>>>(tdy, tw, a);
  }
  count_launch(1, KF_UMMA);
  return launch_status("stem_dgrad_kernel");
}


// ============================================================================
// Forward of the same stem (<= 4-channel 7x7 / stride 2 / pad 3 convolution)
// with the A operand read straight out of the input rows -- no im2col.
//
// In a 4-channel copy of the input padded by 3 pixels on the left, the K-slice
// of output pixel ow for kernel row r (7 taps x 4 channels, 56 B, padded to
// K = 32) starts at byte 16*ow of input row 2*oh-3+r.  A K-major no-swizzle
// UMMA operand whose 8x16 B core matrices are 16 B apart along K (LBO = 16) and
// 128 B apart along M (SBO = 128) describes exactly these overlapping rows, so
// each input row is copied once per output row with one 1.8 KB bulk copy and
// the tensor core reads the overlapping windows in place (the im2col variant
// moves 4x the bytes through TMA).  The weight tile (7 x 32 x K) stays in
// shared memory for the whole launch.  Output row tiles: M = 128 >= OW.
// ============================================================================
namespace {

constexpr int SF_R = 7;
constexpr int SF_SLOT = 2176;              // one padded input row (>= 16*127 + 64 bytes)
constexpr int SF_STAGE = SF_R * SF_SLOT;   // the 7 input rows of one output row
constexpr int SF_STAGES = 6;
constexpr int SF_EPI = 4;   // warps per epilogue group (one per TMEM lane quarter)
constexpr int SF_NG = 2;    // epilogue groups, draining alternate output rows
constexpr int SF_ACC = 4;   // TMEM accumulators in flight (4 x K <= 512 columns)
constexpr int SF_THREADS = 64 + 32 * SF_EPI * SF_NG;

struct StemFpropArgs {
  int N, H, Wp;    // padded 4-channel input: [N][H][Wp][4]
  int P, Q, K;     // output rows, columns, channels
  int units;       // N * P output rows
  void* y;         // [N][P][Q][K]
  const void* bias;
  int dt;
  const void* xp;  // padded input
  const void* wb;  // weights in core-matrix layout [r][kg 4][K][8]
  BnFold bn;           // fused eval-BN (bn.var nullable): y = conv * s[k] + t[k]
  int relu;            // fused ReLU; keep bits to mask (1 bit per element, NHWC order)
  uint8_t* mask;
};

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
      : "memory");
}

constexpr int SF_STG = SF_EPI * SF_NG * 2 * 4096;  // per epilogue warp: 2 x (32 px x 128 B), SW128
constexpr int SF_AFF = 2 * 128 * 4;         // fused eval-BN scale / shift (K <= 128)

template <typename T>
__global__ void __launch_bounds__(SF_THREADS, 1)
    stem_fprop_kernel(const __grid_constant__ StemFpropArgs a,
                      const __grid_constant__ CUtensorMap tma_y) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int b_bytes = SF_R * 4 * a.K * 16;
  uint8_t* stg = smem;                         // TMA-store staging (1024-aligned)
  uint8_t* sB = smem + SF_STG;
  uint8_t* zero_row = sB + b_bytes;            // out-of-range input rows read zeros
  uint8_t* ring = zero_row + SF_SLOT;
  float* s_aff = reinterpret_cast<float*>(ring + SF_STAGES * SF_STAGE);  // [scale K][shift K]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + SF_STAGES * SF_STAGE + SF_AFF);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + SF_STAGES;
  uint64_t* tfull_bar = bars + 2 * SF_STAGES;
  uint64_t* tempty_bar = bars + 2 * SF_STAGES + SF_ACC;
  uint64_t* b_bar = bars + 2 * SF_STAGES + 2 * SF_ACC;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * SF_STAGES + 2 * SF_ACC + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  for (int i = threadIdx.x; i < SF_SLOT / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(zero_row)[i] = 0u;
  if (a.bn.var)
    for (int i = threadIdx.x; i < a.K; i += blockDim.x) bn_fold(a.bn, i, s_aff[i], s_aff[a.K + i]);
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < SF_STAGES; ++i) {
      mbar_init(smem_u32(&full_bar[i]), 1);
      mbar_init(smem_u32(&empty_bar[i]), 1);
    }
    for (int i = 0; i < SF_ACC; ++i) {
      mbar_init(smem_u32(&tfull_bar[i]), 1);
      mbar_init(smem_u32(&tempty_bar[i]), SF_EPI);  // one group drains each row
    }
    mbar_init(smem_u32(b_bar), 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_holder), SF_ACC * 128);
  fence_proxy_async_smem();  // the zero row is read by the tensor core (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const uint32_t row_bytes = static_cast<uint32_t>(a.Wp) * 8u;

  if (warp == 0) {
    // ============================ bulk-copy producer ============================
    {  // whole warp (uniform operands), an elect.sync lane issues
      if (elect_one()) {
        mbar_arrive_expect_tx(smem_u32(b_bar), b_bytes);
        bulk_g2s(smem_u32(sB), a.wb, b_bytes, smem_u32(b_bar));
      }
      __syncwarp();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
        const int n = u / a.P, oh = u - (u / a.P) * a.P;
        mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
        const uint32_t fb = smem_u32(&full_bar[stage]);
        int rows = 0;
        for (int r = 0; r < SF_R; ++r) {
          const int h = 2 * oh - 3 + r;
          rows += (h >= 0 && h < a.H) ? 1 : 0;
        }
        if (elect_one()) {
          mbar_arrive_expect_tx(fb, rows * row_bytes);
          for (int r = 0; r < SF_R; ++r) {
            const int h = 2 * oh - 3 + r;
            if (h >= 0 && h < a.H) {
              const uint8_t* src = static_cast<const uint8_t*>(a.xp) +
                                   (static_cast<int64_t>(n) * a.H + h) * row_bytes;
              bulk_g2s(smem_u32(ring + stage * SF_STAGE + r * SF_SLOT), src, row_bytes, fb);
            }
          }
        }
        __syncwarp();
        if (++stage == SF_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    {  // whole warp: descriptors in uniform registers; an elect.sync lane issues
      const uint32_t idesc = make_idesc_f16(a.dt == MS_BF16 ? 1 : 0, BM, a.K, 0, 0);
      const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
      mbar_wait(smem_u32(b_bar), 0);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int u = blockIdx.x; u < a.units; u += gridDim.x, ++local) {
        const int oh = u - (u / a.P) * a.P;
        const int acc = local % SF_ACC;
        mbar_wait(smem_u32(&tempty_bar[acc]), ((local / SF_ACC) & 1) ^ 1);
        mbar_wait(smem_u32(&full_bar[stage]), phase);
        tc_fence_after();
        const uint32_t dcol = tmem_u + acc * a.K;
        uint64_t ads[2 * SF_R], bds[2 * SF_R];
#pragma unroll
        for (int r = 0; r < SF_R; ++r) {
          const int h = 2 * oh - 3 + r;
          const uint32_t arow = (h >= 0 && h < a.H)
                                    ? smem_u32(ring + stage * SF_STAGE + r * SF_SLOT)
                                    : smem_u32(zero_row);
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            // A: rows 16 B apart, K core matrices 16 B apart (overlapping windows)
            ads[2 * r + half] = make_smem_desc(arow + half * 32, 16, 128, LAYOUT_SWIZZLE_NONE);
            // B: [r][kg][K][8]: K core matrices 16*K B apart, 8-row groups 128 B apart
            bds[2 * r + half] = make_smem_desc(smem_u32(sB) + (r * 4 + 2 * half) * a.K * 16,
                                               a.K * 16, 128, LAYOUT_SWIZZLE_NONE);
          }
        }
        if (elect_one()) {
#pragma unroll
          for (int i = 0; i < 2 * SF_R; ++i) umma_f16(dcol, ads[i], bds[i], idesc, i ? 1u : 0u);
          umma_commit(smem_u32(&empty_bar[stage]));
          umma_commit(smem_u32(&tfull_bar[acc]));
        }
        __syncwarp();
        if (++stage == SF_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ============================ epilogue ============================
    // thread = output pixel (TMEM lane); 64-channel rows staged in shared memory
    // with the 128-byte swizzle and written by one TMA store per 32 pixels
    // (a 3-D map [N*P][Q][K] clips the pixels past Q)
    const int quarter = static_cast<int>(warp & 3);
    const int ew = static_cast<int>(warp) - 2;
    const int grp = ew / SF_EPI;  // this group drains output rows grp, grp + SF_NG, ...
    const int rw = static_cast<int>(lane);
    int local = grp;
    uint32_t nst = 0;
    for (int u = blockIdx.x + grp * gridDim.x; u < a.units;
         u += SF_NG * gridDim.x, local += SF_NG) {
      const int buf = local % SF_ACC;
      mbar_wait(smem_u32(&tfull_bar[buf]), (local / SF_ACC) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((static_cast<uint32_t>(quarter) * 32u) << 16) + buf * a.K;
#pragma unroll 1
      for (int c0 = 0; c0 < a.K; c0 += 64) {
        uint32_t v0[32], v1[32];
        tmem_ld_32x32b_x32(taddr + c0, v0);
        tmem_ld_32x32b_x32(taddr + c0 + 32, v1);
        tmem_ld_wait_regs(v0);
        tmem_ld_wait_regs(v1);
        if (c0 + 64 >= a.K) {  // accumulator drained: release it to the next row's MMAs
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&tempty_bar[buf]));
        }
        uint8_t* sb = stg + (ew * 2 + (nst & 1)) * 4096;
        if (lane == 0) bulk_wait_read<1>();  // the store issued 2 chunks ago has read sb
        __syncwarp();
        const int ow = quarter * 32 + rw;
        uint64_t keep = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float f[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int ch = q * 8 + j;
            f[j] = __uint_as_float(ch < 32 ? v0[ch] : v1[ch - 32]);
            if (a.bias) f[j] += IO<T>::ld(static_cast<const T*>(a.bias) + c0 + ch);
            if (a.bn.var) f[j] = f[j] * s_aff[c0 + ch] + s_aff[a.K + c0 + ch];
            if (a.relu) {
              const bool pos = !(f[j] <= 0.f);
              keep |= (pos ? 1ull : 0ull) << ch;
              f[j] = pos ? f[j] : 0.f;
            }
          }
          uint4 pk;
          pk.x = pack2<T>(f[0], f[1]);
          pk.y = pack2<T>(f[2], f[3]);
          pk.z = pack2<T>(f[4], f[5]);
          pk.w = pack2<T>(f[6], f[7]);
          *reinterpret_cast<uint4*>(sb + rw * 128 + ((q ^ (rw & 7)) << 4)) = pk;
        }
        if (a.relu && a.mask && ow < a.Q)  // 64 channels = 8 mask bytes (K % 64 == 0)
          reinterpret_cast<uint64_t*>(a.mask)[((static_cast<int64_t>(u) * a.Q + ow) * a.K + c0) >> 6] =
              keep;
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&tma_y, smem_u32(sb), c0, quarter * 32, u);
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
    tmem_dealloc(tmem_base, SF_ACC * 128);
  }
}

// [r][kg][K][8]: element j of row n in k-group kg = w[n][c][r][s], k = 8kg + j = 4s + c
template <typename T>
__global__ void repack_stem_fprop_kernel(int K, int C, int R, int S, int wlayout, const T* w,
                                         T* out) {
  const int total = R * 4 * K * 8;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int j = i % 8, n = (i / 8) % K, kg = (i / (8 * K)) % 4, r = i / (32 * K);
    const int k = kg * 8 + j, s = k / 4, c = k % 4;
    T v = IO<T>::cvt(0.f);
    if (s < S && c < C)
      v = wlayout == MS_NHWC ? w[(((int64_t)n * R + r) * S + s) * C + c]
                             : w[(((int64_t)n * C + c) * R + r) * S + s];
    out[i] = v;
  }
}

}  // namespace

bool stem_fprop_ok(int dt, int layout, int c, int r, int s, int sh, int sw, int ph, int pw,
                   int64_t ow, int64_t k) {
  return (dt == MS_BF16 || dt == MS_F16) && layout == MS_NHWC && c <= 4 && r == SF_R && s == 7 &&
         sh == 2 && sw == 2 && ph == 3 && pw == 3 && ow <= BM && k % 64 == 0 && k <= 128;
}

size_t stem_fprop_weight_bytes(int k) { return (size_t)SF_R * 4 * k * 16; }

// xp: pad_rowseg output [n][h][wp][4]; wb: workspace of stem_fprop_weight_bytes(k)
ms_status stem_fprop(int dt, int n, int h, int wp, int p, int q, int k, int c, int wlayout,
                     const void* xp, const void* w, void* wb, const void* bias, void* y,
                     cudaStream_t st, const BnFold& bn, int relu, uint8_t* mask) {
  const int total = SF_R * 4 * k * 8;
  const int blocks = (total + 255) / 256;
  if (dt == MS_BF16)
    repack_stem_fprop_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
        k, c, SF_R, 7, wlayout, (const __nv_bfloat16*)w, (__nv_bfloat16*)wb);
  else
    repack_stem_fprop_kernel<__half><<<blocks, 256, 0, st>>>(k, c, SF_R, 7, wlayout,
                                                             (const __half*)w, (__half*)wb);
  count_launch();
  MS_TRY(launch_status("repack_stem_fprop"));
  StemFpropArgs a{};
  a.N = n; a.H = h; a.Wp = wp; a.P = p; a.Q = q; a.K = k;
  a.units = n * p;
  a.y = y; a.bias = bias; a.dt = dt; a.xp = xp; a.wb = wb;
  a.bn = bn; a.relu = relu; a.mask = mask;
  const int smem =
      SF_STG + (int)stem_fprop_weight_bytes(k) + SF_SLOT + SF_STAGES * SF_STAGE + SF_AFF + 1024 +
      256;
  const int grid = a.units < num_sms() ? a.units : num_sms();
  CUtensorMap ty;
  const size_t es = dtype_size(dt);
  const uint64_t dims[3] = {(uint64_t)k, (uint64_t)q, (uint64_t)n * p};
  const uint64_t str[2] = {(uint64_t)k * es, (uint64_t)q * k * es};
  const uint32_t box[3] = {64, 32, 1};
  MS_TRY(make_tmap_nd(&ty, dt, y, 3, dims, str, box, 128));
  if (dt == MS_BF16) {
    auto kern = stem_fprop_kernel<__nv_bfloat16>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<grid, SF_THREADS, smem, st>>>(a, ty);
  } else {
    auto kern = stem_fprop_kernel<__half>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<grid, SF_THREADS, smem, st>>>(a, ty);
  }
  count_launch(1, KF_UMMA);
  return launch_status("stem_fprop_kernel");
}

}  // namespace ms
