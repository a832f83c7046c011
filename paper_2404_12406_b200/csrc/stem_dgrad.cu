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
    if (lane == 0) {
      const uint32_t bb = smem_u32(b_bar);
      mbar_arrive_expect_tx(bb, a.kblocks * SD_B_KB_BYTES);
      for (int kb = 0; kb < a.kblocks; ++kb)
        tma_load_2d(smem_u32(sB + kb * SD_B_KB_BYTES), &tma_w, bb, kb * 64, 0);
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
            mbar_arrive_expect_tx(fb, SD_A_BYTES);
#pragma unroll
            for (int w = 0; w < SD_SEGS; ++w)
              tma_load_4d(sA + w * 4096, &tma_dy, fb, kb * 64, SD_SEG * w - 1, oh, n);
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
    if (lane == 0) {
      const uint32_t idesc = make_idesc_f16(a.dt == MS_BF16 ? 1 : 0, BM, SD_N, 0, 0);
      mbar_wait(smem_u32(b_bar), 0);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
        for (int i = 0; i < rows_per_unit; ++i, ++local) {
          const int acc = local & 1;
          mbar_wait(smem_u32(&tempty_bar[acc]), ((local >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t dcol = tmem_base + acc * SD_N;
          for (int kb = 0; kb < a.kblocks; ++kb) {
            mbar_wait(smem_u32(&full_bar[stage]), phase);
            tc_fence_after();
            const uint32_t sA = smem_u32(ring + stage * SD_A_BYTES);
            const uint32_t sBk = smem_u32(sB + kb * SD_B_KB_BYTES);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ad = make_smem_desc(sA + k * 32, 16, 1024, LAYOUT_SWIZZLE_128B);
              const uint64_t bd = make_smem_desc(sBk + k * 32, 16, 1024, LAYOUT_SWIZZLE_128B);
              umma_f16(dcol, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
            }
            umma_commit(smem_u32(&empty_bar[stage]));
            if (++stage == SD_STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit(smem_u32(&tfull_bar[acc]));
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

}  // namespace ms
