// Warp-specialised, persistent tcgen05 GEMM / implicit-GEMM kernel (sm_100a).
//
// One kernel template serves every dense contraction of the hot path:
//   LOAD_GEMM        Linear fwd (X·Wᵀ), dX (dY·W), dW (dYᵀ·X)
//   LOAD_CONV_FPROP  Conv2d forward, A = im2col(x) via TMA im2col mode   numpy_impl.py:12-24
//   LOAD_CONV_DGRAD  Conv2d input-VJP, stride phases, A = im2col(dy)     numpy_impl.py:27-38
//   LOAD_CONV_WGRAD  Conv2d weight-VJP, A = dyᵀ, B = im2col(x)ᵀ, split-K numpy_impl.py:41-51
//
// CTA = 6 warps, 1 CTA per SM, grid = min(tiles, #SMs), static round-robin tiles.
//   warp 0      TMA producer (one lane): fills a STAGES-deep smem ring
//   warp 1      TMEM allocator + MMA issuer (one lane): tcgen05.mma 128xBNx16
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> (bias) -> global
// Accumulators are double-buffered in TMEM (2 x BN fp32 columns) so the
// epilogue of tile i overlaps the main loop of tile i+1.
// Operand tiles are 128-byte-swizzled (TMA SWIZZLE_128B == UMMA SWIZZLE_128B);
// K-major tiles are [rows][64 elems]; MN-major tiles are [64 k-rows][64 elems]
// blocks placed 8 KiB apart along MN.
#pragma once

#include "common.cuh"

namespace ms {

enum : int {
  LOAD_GEMM = 0,
  LOAD_CONV_FPROP = 1,
  LOAD_CONV_DGRAD = 2,
  LOAD_CONV_WGRAD = 3,
  LOAD_CONV_FPROP_C8 = 4,    // 8-channel activations: 8 taps x 8 ch per k-block, no swizzle
  LOAD_CONV_DGRAD_SCATTER = 5  // tiny-Cin input-VJP: dY rows x (tap,c) GEMM + col2im scatter
};
constexpr int SCATTER_REGION_BYTES = 32 * 1024;

constexpr int BM = 128;        // UMMA M (cta_group::1)
constexpr int BK = 64;         // K elements per stage (128 bytes of bf16)
constexpr int UMMA_K = 16;     // K per tcgen05.mma for 16-bit inputs
constexpr int EPI_WARPS = 4;
constexpr int GEMM_THREADS = 64 + 32 * EPI_WARPS;

struct ConvShape {
  int N, H, W, C;    // TMA source activation (x for fprop/wgrad, dy for dgrad)
  int P, Q;          // output spatial dims of the conv (OH, OW)
  int R, S;
  int sh, sw, ph, pw;
  int cblocks;       // 64-channel blocks of the contraction channel dim
  int wrow_cpad;     // per-tap channel pitch of the repacked weight (multiple of 64)
  int outH, outW;    // dgrad: dX spatial dims (for the phase row mapping)
};

struct PhaseInfo {   // one stride phase of the input-VJP (dgrad)
  int Hp, Wp;        // phase grid: dX rows h = sh*i + ph, cols w = sw*j + pw
  int Lh, Lw;        // im2col start offset (lower corner) in dY coordinates
  int nr, ns;        // taps contributing to this phase
  int r0, s0;        // first contributing tap
  int ph, pw;
  int m_total;       // N * Hp * Wp
  int m_blocks;
  int tile_begin;    // first tile index of this phase
};

struct EpiParams {
  void* out;
  int64_t ldc;       // elements between consecutive output rows
  int out_dtype;     // ms_dtype
  int atomic;        // 1: fp32 red.add into out (split-K / wgrad workspace)
  const void* bias;  // per-column bias (nullable)
  int bias_dtype;
};

struct GemmArgs {
  int M, N;          // output rows / cols of the GEMM view
  int m_blocks, n_blocks;
  int k_blocks;      // k-blocks along the full reduction (GEMM / WGRAD)
  int splits, kb_per_split;
  int taps;          // WGRAD: R*S
  int num_tiles;
  int ab_fmt;        // 1 = bf16, 0 = fp16
  ConvShape cv;
  int nphases;
  PhaseInfo phase[4];
  EpiParams epi;
};

struct TmapPack {
  CUtensorMap a[4];  // A operand (per dgrad phase; a[0] otherwise)
  CUtensorMap b;     // B operand
};

struct TileInfo {
  int m0;            // first output row of the tile (phase-local for dgrad)
  int nb;            // n-block index (n0 = nb * BN)
  int kb_begin, kb_end;
  int phase;         // dgrad: stride phase
  int tap;           // wgrad: kernel tap r*S+s
};

template <int MODE>
__device__ __forceinline__ TileInfo decode_tile(const GemmArgs& g, int t) {
  TileInfo ti;
  ti.phase = 0;
  ti.tap = 0;
  if constexpr (MODE == LOAD_CONV_DGRAD) {
    int p = 0;
#pragma unroll 1
    for (int i = 1; i < g.nphases; ++i)
      if (t >= g.phase[i].tile_begin) p = i;
    const PhaseInfo& P = g.phase[p];
    const int lt = t - P.tile_begin;
    ti.phase = p;
    ti.m0 = (lt % P.m_blocks) * BM;
    ti.nb = lt / P.m_blocks;
    ti.kb_begin = 0;
    ti.kb_end = P.nr * P.ns * g.cv.cblocks;
  } else if constexpr (MODE == LOAD_CONV_DGRAD_SCATTER) {
    // one tile = one dY row (n, oh): rows ow in [0, Q) of the [N*P*Q][K] matrix
    const int row = t / g.n_blocks;
    ti.nb = t - row * g.n_blocks;
    ti.m0 = row;  // row index (n*P + oh); the A coordinate is row*Q
    ti.kb_begin = 0;
    ti.kb_end = g.k_blocks;
  } else {
    const int mb = t % g.m_blocks;
    int rest = t / g.m_blocks;
    ti.m0 = mb * BM;
    ti.nb = rest % g.n_blocks;
    rest /= g.n_blocks;
    if constexpr (MODE == LOAD_CONV_WGRAD) {
      ti.tap = rest % g.taps;
      const int split = rest / g.taps;
      ti.kb_begin = split * g.kb_per_split;
      ti.kb_end = min(g.k_blocks, ti.kb_begin + g.kb_per_split);
    } else if constexpr (MODE == LOAD_CONV_FPROP) {
      ti.kb_begin = 0;
      ti.kb_end = g.cv.R * g.cv.S * g.cv.cblocks;
    } else if constexpr (MODE == LOAD_CONV_FPROP_C8) {
      ti.kb_begin = 0;
      ti.kb_end = g.k_blocks;
    } else {
      const int split = rest;
      ti.kb_begin = split * g.kb_per_split;
      ti.kb_end = min(g.k_blocks, ti.kb_begin + g.kb_per_split);
    }
  }
  return ti;
}

template <int BN, int A_MN, int B_MN, int MODE>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EXTRA = MODE == LOAD_CONV_DGRAD_SCATTER ? SCATTER_REGION_BYTES : 0;
  static constexpr int STAGES_MAX = (200 * 1024 - EXTRA) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_MAX > 8 ? 8 : STAGES_MAX;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EXTRA + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN, int A_MN, int B_MN, int MODE>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    umma_gemm_kernel(const __grid_constant__ TmapPack tm, const __grid_constant__ GemmArgs g) {
  using Cfg = GemmCfg<BN, A_MN, B_MN, MODE>;
  constexpr int STAGES = Cfg::STAGES;
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the SWIZZLE_128B atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* ring = smem;
  float* region = reinterpret_cast<float*>(smem + STAGES * Cfg::STAGE_BYTES);  // scatter mode
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::EXTRA);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + STAGES;
  uint64_t* tfull_bar = bars + 2 * STAGES;
  uint64_t* tempty_bar = bars + 2 * STAGES + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(smem_u32(&full_bar[i]), 1);
      mbar_init(smem_u32(&empty_bar[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&tfull_bar[i]), 1);
      mbar_init(smem_u32(&tempty_bar[i]), EPI_WARPS * 32);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tm.b);
    tma_prefetch_desc(&tm.a[0]);
  }
  if constexpr (MODE == LOAD_CONV_DGRAD_SCATTER)
    for (int i = threadIdx.x; i < SCATTER_REGION_BYTES / 4; i += blockDim.x) region[i] = 0.f;
  if (warp == 1) tmem_alloc(smem_u32(tmem_holder), Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < g.num_tiles; t += gridDim.x) {
        TileInfo ti = decode_tile<MODE>(g, t);
        const int n0 = ti.nb * BN;
        // per-tile conv coordinates
        int cn = 0, ch = 0, cw = 0;
        const CUtensorMap* amap = &tm.a[0];
        if constexpr (MODE == LOAD_CONV_FPROP || MODE == LOAD_CONV_FPROP_C8) {
          const int pq = g.cv.P * g.cv.Q;
          cn = ti.m0 / pq;
          int rem = ti.m0 - cn * pq;
          int oh = rem / g.cv.Q, ow = rem - (rem / g.cv.Q) * g.cv.Q;
          ch = oh * g.cv.sh - g.cv.ph;
          cw = ow * g.cv.sw - g.cv.pw;
        } else if constexpr (MODE == LOAD_CONV_DGRAD) {
          const PhaseInfo& P = g.phase[ti.phase];
          const int hw = P.Hp * P.Wp;
          cn = ti.m0 / hw;
          int rem = ti.m0 - cn * hw;
          int i = rem / P.Wp, j = rem - (rem / P.Wp) * P.Wp;
          ch = i + P.Lh;
          cw = j + P.Lw;
          amap = &tm.a[ti.phase];
        }
        for (int kb = ti.kb_begin; kb < ti.kb_end; ++kb) {
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
          const uint32_t fb = smem_u32(&full_bar[stage]);
          const uint32_t sA = smem_u32(ring + stage * Cfg::STAGE_BYTES);
          const uint32_t sB = sA + Cfg::A_BYTES;
          mbar_arrive_expect_tx(fb, Cfg::STAGE_BYTES);
          if constexpr (MODE == LOAD_GEMM) {
            const int k0 = kb * BK;
            if constexpr (A_MN) {
              tma_load_2d(sA, &tm.a[0], fb, ti.m0, k0);
              tma_load_2d(sA + 8192, &tm.a[0], fb, ti.m0 + 64, k0);
            } else {
              tma_load_2d(sA, &tm.a[0], fb, k0, ti.m0);
            }
            if constexpr (B_MN) {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) tma_load_2d(sB + j * 8192, &tm.b, fb, n0 + 64 * j, k0);
            } else {
              tma_load_2d(sB, &tm.b, fb, k0, n0);
            }
          } else if constexpr (MODE == LOAD_CONV_FPROP) {
            const int tap = kb / g.cv.cblocks;
            const int cb = kb - tap * g.cv.cblocks;
            const int r = tap / g.cv.S, s = tap - (tap / g.cv.S) * g.cv.S;
            tma_load_im2col_4d(sA, amap, fb, cb * 64, cw, ch, cn, (uint16_t)s, (uint16_t)r);
            tma_load_2d(sB, &tm.b, fb, tap * g.cv.wrow_cpad + cb * 64, n0);
          } else if constexpr (MODE == LOAD_CONV_FPROP_C8) {
            // 8 taps x 8 channels; each tap is one 128-pixel x 16-byte im2col box
            const int taps = g.cv.R * g.cv.S;
#pragma unroll 1
            for (int j = 0; j < 8; ++j) {
              const int tap = kb * 8 + j;
              if (tap < taps) {
                const int r = tap / g.cv.S, s = tap - (tap / g.cv.S) * g.cv.S;
                tma_load_im2col_4d(sA + j * 2048, amap, fb, 0, cw, ch, cn, (uint16_t)s,
                                   (uint16_t)r);
              } else {  // past the last tap: an all-out-of-bounds box loads zeros
                tma_load_im2col_4d(sA + j * 2048, amap, fb, 0, cw, ch, g.cv.N, 0, 0);
              }
            }
            tma_load_2d(sB, &tm.b, fb, kb * BK, n0);
          } else if constexpr (MODE == LOAD_CONV_DGRAD_SCATTER) {
            tma_load_2d(sA, &tm.a[0], fb, kb * BK, ti.m0 * g.cv.Q);
            tma_load_2d(sB, &tm.b, fb, kb * BK, n0);
          } else if constexpr (MODE == LOAD_CONV_DGRAD) {
            const PhaseInfo& P = g.phase[ti.phase];
            const int cb = kb % g.cv.cblocks;
            const int tt = kb / g.cv.cblocks;
            const int ts = tt % P.ns, tr = tt / P.ns;
            const int r = P.r0 + g.cv.sh * tr, s = P.s0 + g.cv.sw * ts;
            tma_load_im2col_4d(sA, amap, fb, cb * 64, cw, ch, cn, (uint16_t)(P.ns - 1 - ts),
                               (uint16_t)(P.nr - 1 - tr));
            tma_load_2d(sB, &tm.b, fb, (r * g.cv.S + s) * g.cv.wrow_cpad + cb * 64, n0);
          } else {  // LOAD_CONV_WGRAD: K = output pixels
            const int p0 = kb * BK;
            const int pq = g.cv.P * g.cv.Q;
            const int pn = p0 / pq;
            const int rem = p0 - pn * pq;
            const int oh = rem / g.cv.Q, ow = rem - (rem / g.cv.Q) * g.cv.Q;
            const int tap = ti.tap;
            const int r = tap / g.cv.S, s = tap - (tap / g.cv.S) * g.cv.S;
            tma_load_2d(sA, &tm.a[0], fb, ti.m0, p0);
            tma_load_2d(sA + 8192, &tm.a[0], fb, ti.m0 + 64, p0);
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_im2col_4d(sB + j * 8192, &tm.b, fb, n0 + 64 * j, ow * g.cv.sw - g.cv.pw,
                                 oh * g.cv.sh - g.cv.ph, pn, (uint16_t)s, (uint16_t)r);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    if (lane == 0) {
      const uint32_t idesc = make_idesc_f16(g.ab_fmt, BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = blockIdx.x; t < g.num_tiles; t += gridDim.x, ++local) {
        TileInfo ti = decode_tile<MODE>(g, t);
        const int acc = local & 1;
        const uint32_t use = static_cast<uint32_t>(local >> 1);
        mbar_wait(smem_u32(&tempty_bar[acc]), (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem_base + acc * BN;
        if (ti.kb_end <= ti.kb_begin) {
          mbar_arrive(smem_u32(&tfull_bar[acc]));  // empty reduction: epilogue writes zeros
          continue;
        }
        for (int kb = ti.kb_begin; kb < ti.kb_end; ++kb) {
          mbar_wait(smem_u32(&full_bar[stage]), phase);
          tc_fence_after();
          const uint32_t sA = smem_u32(ring + stage * Cfg::STAGE_BYTES);
          const uint32_t sB = sA + Cfg::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            uint64_t ad, bd;
            if constexpr (MODE == LOAD_CONV_FPROP_C8)  // core matrices 8 rows x 16 B, no swizzle
              ad = make_smem_desc(sA + k * 4096, 2048, 128, LAYOUT_SWIZZLE_NONE);
            else if constexpr (A_MN) ad = make_smem_desc(sA + k * 2048, 8192, 1024, LAYOUT_SWIZZLE_128B);
            else ad = make_smem_desc(sA + k * 32, 16, 1024, LAYOUT_SWIZZLE_128B);
            if constexpr (B_MN) bd = make_smem_desc(sB + k * 2048, 8192, 1024, LAYOUT_SWIZZLE_128B);
            else bd = make_smem_desc(sB + k * 32, 16, 1024, LAYOUT_SWIZZLE_128B);
            umma_f16(dcol, ad, bd, idesc, (kb > ti.kb_begin || k > 0) ? 1u : 0u);
          }
          umma_commit(smem_u32(&empty_bar[stage]));  // frees the smem slot when MMAs retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(smem_u32(&tfull_bar[acc]));  // accumulator ready for the epilogue
      }
    }
  } else {
    // ============================ epilogue ============================
    const uint32_t quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    int local = 0;
    const EpiParams& e = g.epi;
    for (int t = blockIdx.x; t < g.num_tiles; t += gridDim.x, ++local) {
      TileInfo ti = decode_tile<MODE>(g, t);
      const int n0 = ti.nb * BN;
      const int acc = local & 1;
      const uint32_t use = static_cast<uint32_t>(local >> 1);
      mbar_wait(smem_u32(&tfull_bar[acc]), use & 1);
      tc_fence_after();
      const bool zero = ti.kb_end <= ti.kb_begin;

      if constexpr (MODE == LOAD_CONV_DGRAD_SCATTER) {
        // Tile = dY row (nn, oh); TMEM lane `row` = output pixel ow of that row;
        // column j = (tap, ci).  Accumulate dX contributions of the whole row in
        // a shared-memory window (R dX rows x region width x C), then flush the
        // window to the fp32 dX accumulator with red.add (windows of adjacent
        // rows overlap, so the flush must be atomic).
        const int nn = ti.m0 / g.cv.P, oh = ti.m0 - (ti.m0 / g.cv.P) * g.cv.P;
        const int C = g.cv.C, S = g.cv.S;
        const int RW = (g.cv.Q - 1) * g.cv.sw + S;
        const int ow = row;
        const bool rvalid = ow < g.cv.Q;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + ((quarter * 32u) << 16) + acc * BN + c, r);
          tmem_ld_wait();
          if (rvalid) {
            // (tap, ci) of the chunk's first column, then walk forward
            int col = n0 + c;
            int tap = col / C, ci = col - tap * C;
            int rr = tap / S, ss = tap - rr * S;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (col < g.N)
                atomicAdd(&region[(rr * RW + ow * g.cv.sw + ss) * C + ci], __uint_as_float(r[j]));
              ++col;
              if (++ci == C) {
                ci = 0;
                if (++ss == S) {
                  ss = 0;
                  ++rr;
                }
              }
            }
          }
        }
        tc_fence_before();
        mbar_arrive(smem_u32(&tempty_bar[acc]));  // TMEM is free once values are in smem
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int total = g.cv.R * RW * C;
        float* outp = static_cast<float*>(e.out);
        const int tid = (static_cast<int>(warp) - 2) * 32 + static_cast<int>(lane);
        for (int i = tid; i < total; i += EPI_WARPS * 32) {
          const int ci = i % C;
          const int rest = i / C;
          const int cc = rest % RW, rr = rest / RW;
          const int h = oh * g.cv.sh - g.cv.ph + rr, w = cc - g.cv.pw;
          const float v = region[i];
          region[i] = 0.f;
          if (h >= 0 && h < g.cv.outH && w >= 0 && w < g.cv.outW && v != 0.f)
            red_add_f32(outp + ((static_cast<int64_t>(nn) * g.cv.outH + h) * g.cv.outW + w) * C + ci,
                        v);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        continue;
      }

      // ---- output row address
      const int m = ti.m0 + row;
      bool valid;
      int64_t orow;
      int ncols = g.N;
      if constexpr (MODE == LOAD_CONV_DGRAD) {
        const PhaseInfo& P = g.phase[ti.phase];
        valid = m < P.m_total;
        const int hw = P.Hp * P.Wp;
        const int nn = m / hw;
        const int rem = m - nn * hw;
        const int i = rem / P.Wp, j = rem - (rem / P.Wp) * P.Wp;
        const int h = g.cv.sh * i + P.ph, w = g.cv.sw * j + P.pw;
        orow = (static_cast<int64_t>(nn) * g.cv.outH + h) * g.cv.outW + w;
      } else if constexpr (MODE == LOAD_CONV_WGRAD) {
        valid = m < g.M;
        orow = m;
        ncols = g.N;  // Cin
      } else {
        valid = m < g.M;
        orow = m;
      }
      int64_t col_base = n0;
      if constexpr (MODE == LOAD_CONV_WGRAD) col_base += static_cast<int64_t>(ti.tap) * g.N;

#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        if (!zero) {
          tmem_ld_32x32b_x32(tmem_base + ((quarter * 32u) << 16) + acc * BN + c, r);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = 0u;
        }
        const int nc = n0 + c;  // first column of this chunk in GEMM-N space
        if (!valid || nc >= ncols) continue;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (e.bias != nullptr) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (nc + j < ncols) v[j] += load_as_float(e.bias, e.bias_dtype, nc + j);
        }
        const int64_t off = orow * e.ldc + col_base + c;
        const bool full = (nc + 32 <= ncols);
        if (e.atomic) {
          float* o = static_cast<float*>(e.out) + off;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (full || nc + j < ncols) red_add_f32(o + j, v[j]);
        } else if (e.out_dtype == MS_F32) {
          float* o = static_cast<float*>(e.out) + off;
          if (full && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
            for (int j = 0; j < 32; ++j)
              if (nc + j < ncols) o[j] = v[j];
          }
        } else {
          uint16_t* o = static_cast<uint16_t*>(e.out) + off;
          if (full && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
            uint32_t p[16];
            if (e.out_dtype == MS_BF16) {
#pragma unroll
              for (int j = 0; j < 16; ++j) p[j] = pack2<__nv_bfloat16>(v[2 * j], v[2 * j + 1]);
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j) p[j] = pack2<__half>(v[2 * j], v[2 * j + 1]);
            }
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              *reinterpret_cast<uint4*>(o + 2 * j) = make_uint4(p[j], p[j + 1], p[j + 2], p[j + 3]);
          } else {
            for (int j = 0; j < 32; ++j)
              if (nc + j < ncols) store_from_float(e.out, e.out_dtype, off + j, v[j]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(smem_u32(&tempty_bar[acc]));
    }
  }

  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace ms
