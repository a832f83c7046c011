// Warp-specialised, persistent tcgen05 GEMM / implicit-GEMM kernel (sm_100a).
//
// One kernel template serves every dense contraction of the hot path:
//   LOAD_GEMM         Linear fwd (X·Wᵀ), dX (dY·W), dW (dYᵀ·X)
//   LOAD_CONV_FPROP   Conv2d forward, A = im2col(x) via TMA im2col mode    numpy_impl.py:12-24
//   LOAD_CONV_DGRAD   Conv2d input-VJP, stride phases, A = im2col(dy)      numpy_impl.py:27-38
//   LOAD_CONV_WGRAD   Conv2d weight-VJP, A = dyᵀ, B = im2col(x)ᵀ, split-K  numpy_impl.py:41-51
//   LOAD_CONV_FPROP_C8    forward for 8-channel activations (8 taps per k-block)
//   LOAD_CONV_FPROP_ROWSEG forward for <=4-channel stride-2 stems: one k-block per
//                     kernel row, A = overlapping input-row segments (4-D TMA)
//   LOAD_GEMM_3XTF32  float32 GEMM (Linear fwd / dX / dW at fp32) on kind::tf32:
//                     A and B arrive as hi / lo planes (K-major), and each k-step
//                     issues hi*hi + hi*lo + lo*hi (3xTF32, ~fp32 accuracy)
//   LOAD_CONV_DGRAD_BAND  input-VJP for <8-channel inputs (the stem's dX): per band
//                     of dX rows, GEMM dY-row x W[(tap,c)] then a col2im into
//                     warp-private shared windows (no atomics), direct store
//
// CTA = 6 warps, 1 CTA per SM, grid = min(tiles, #SMs), static round-robin tiles.
//   warp 0      TMA producer (one lane): fills a STAGES-deep smem ring
//   warp 1      TMEM allocator + MMA issuer (one lane): tcgen05.mma 128xBNx16
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> (bias) -> global
// Accumulators are double-buffered in TMEM (2 x BN fp32 columns) so the
// epilogue of one accumulation overlaps the main loop of the next.
#pragma once

#include "common.cuh"
#include "rng.cuh"

namespace ms {

enum : int {
  LOAD_GEMM = 0,
  LOAD_CONV_FPROP = 1,
  LOAD_CONV_DGRAD = 2,
  LOAD_CONV_WGRAD = 3,
  LOAD_CONV_FPROP_C8 = 4,
  LOAD_CONV_FPROP_ROWSEG = 6,
  LOAD_CONV_DGRAD_BAND = 7,
  LOAD_GEMM_3XTF32 = 8
};
constexpr int BAND_WINDOWS = 8;  // one private col2im window per epilogue warp
constexpr int BAND_WINDOW_BYTES = 112 * 1024;
// The band input-VJP is specialised to the ResNet/VGG-style stem geometry so
// that every accumulator column's (kernel row, kernel col, channel) is a
// compile-time constant: C = 3 input channels, 7x7 kernel, stride 2.
constexpr int BAND_C = 3, BAND_R = 7, BAND_S = 7, BAND_SW = 2, BAND_H = 16;
constexpr int BAND_WC = 31 * BAND_SW + BAND_S;       // window columns of 32 dY pixels (69)
constexpr int BAND_WH = (BAND_WC + 1) / 2;           // per parity plane (35)
constexpr int BAND_ROWF = BAND_C * 2 * BAND_WH;      // floats per window row (210)
constexpr int BAND_WIN = BAND_H * BAND_ROWF;         // floats per window (3360)
template <int V> struct IntC { static constexpr int value = V; };

constexpr int BM = 128;        // UMMA M (cta_group::1)
constexpr int ROWSEG8_A_TX = (BM + 8) * 16;  // rowseg8: one staged segment (136 px x 16 B)
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
  int outH, outW;    // dgrad: dX spatial dims (phase row mapping, band windows)
  int outC;          // band dgrad: dX channels
  int band_h;        // band dgrad: dX rows owned per band
  int band_sub;      // band dgrad: dY rows per band
  int bands_per_img; // band dgrad
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
  // fused eval-BatchNorm + ReLU (conv forward): v = v * s[col] + t[col] (bn.var
  // != nullptr), then v = max(v, 0) with the keep bit of every element written to
  // mask (1 bit per element in storage order, as ms_relu_fwd)
  BnFold bn;
  int relu;
  uint8_t* mask;       // nullable
  const void* resid;   // nullable: residual added after the affine, before the ReLU
                       // (same dtype / pitch as out)
  // input-VJP of a conv whose input came out of a ReLU [after an eval-BN]: after
  // the addend (resid), v = keep ? v : 0 with keep_in the producer's bit mask
  // (storage order), then v *= s[col] when bn_post (bn = the producer's BN)
  const uint8_t* keep_in;
  int bn_post;
  // fused GELU (Linear -> GELU): out keeps the pre-activation (what the GELU's
  // backward reads) and act_out receives gelu(pre) of the ROUNDED pre, exactly
  // what a separate gelu launch would read and write (same dtype / pitch)
  void* act_out;
  // Linear -> dropout -> + residual (a transformer block's output projection):
  // the linear output is rounded to the storage type, dropped with the mask the
  // dropout kernels draw for the same (seed, stream, element) and rounded
  // again, then resid is added -- bit for bit the three separate launches
  // (round_lin: round before the residual add even without dropout)
  DropEpi drop;
  int round_lin;
};

struct GemmArgs {
  int M, N;          // output rows / cols of the GEMM view
  int m_blocks, n_blocks;
  int k_blocks;      // k-blocks along the full reduction (GEMM / WGRAD / C8 / BAND)
  int splits, kb_per_split;
  int taps;          // WGRAD: R*S
  int num_tiles;
  int ab_fmt;        // 1 = bf16, 0 = fp16
  int tma_store;     // 1: epilogue stages 32x32 chunks in smem and stores them by TMA
  // GEMM tail split: tiles [full_tiles, tiles) -- those of the last, partial wave
  // -- run as tail_splits K-slices of tail_kbps k-blocks each; every slice stores
  // its fp32 partial tile densely in tail_ws ([unit][CL*BM][BN]) and a finalize
  // pass sums them (tail_splits = 0: off)
  int full_tiles, tail_splits, tail_kbps;
  float* tail_ws;
  // GEMM raster order: 0 = M-blocks fastest (concurrent tiles share B), 1 =
  // N-blocks fastest (they share A: A streams from HBM once when B fits in L2)
  int n_fastest;
  // profiling switch (MS_GEMM_DBG, GEMM mode only): bit 0 drops the epilogue's
  // stores, bit 1 also its TMEM loads -- isolates the main loop's feed rate;
  // fused GELU: bit 2 skips its arithmetic, bit 3 its second output
  int dbg;
  // LOAD_CONV_FPROP_ROWSEG with 8-channel stride-1 rows: stage each input row
  // segment once ([136 px][8 ch], 16 B per pixel, no swizzle) and read tap pairs
  // at 16-byte-shifted descriptor starts (LBO = 16 B: the next K core matrix is
  // the next pixel) instead of 128 overlapping 64-byte windows per k-block
  int rowseg8;
  ConvShape cv;
  int nphases;
  PhaseInfo phase[4];
  EpiParams epi;
};

struct TmapPack {
  CUtensorMap a[4];  // A operand (per dgrad phase; a[0] otherwise)
  CUtensorMap b;     // B operand
  CUtensorMap c;     // output (GEMM / conv fwd, 16-bit): box {32 cols, 32 rows}, SW64
  CUtensorMap c2;    // second output of a fused GELU (EpiParams::act_out), as c
};

// 32 consecutive 16-bit outputs of one row from fp32 (vector stores when the
// chunk is whole and 16-byte aligned, else the first `left` elements)
__device__ __forceinline__ void store_row32(void* out, int dt, int64_t off, const float (&v)[32],
                                            bool full, int left) {
  uint16_t* o = static_cast<uint16_t*>(out) + off;
  if (full && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
    uint32_t p[16];
    if (dt == MS_BF16) {
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
#pragma unroll
    for (int j = 0; j < 32; ++j)  // constant indices: v stays in registers
      if (j < left) store_from_float(out, dt, off + j, v[j]);
  }
}

#ifndef GELU_ILP
#define GELU_ILP 4  // erf evaluations interleaved by the fused GELU epilogue
#endif

struct TileInfo {
  int m0;            // first output row of the tile (phase-local for dgrad; row id
                     // n*P+oh for ROWSEG; band id n*bands+b for BAND)
  int nb;            // n-block index (n0 = nb * BN)
  int kb_begin, kb_end;
  int phase;         // dgrad: stride phase
  int tap;           // wgrad: kernel tap r*S+s
  int nsub;          // accumulations in this tile (BAND: dY rows; otherwise 1)
  int unit;          // GEMM tail split: slice index (>= 0) of a tail tile, else -1
};

__device__ __forceinline__ int floor_div(int a, int b) {
  return a >= 0 ? a / b : -((-a + b - 1) / b);
}

template <int MODE, int CL = 1>
__device__ __forceinline__ TileInfo decode_tile(const GemmArgs& g, int t, int crank = 0) {
  TileInfo ti;
  ti.phase = 0;
  ti.tap = 0;
  ti.nsub = 1;
  ti.unit = -1;
  if constexpr (MODE == LOAD_CONV_DGRAD) {
    int p = 0;
#pragma unroll 1
    for (int i = 1; i < g.nphases; ++i)
      if (t >= g.phase[i].tile_begin) p = i;
    const PhaseInfo& P = g.phase[p];
    const int lt = t - P.tile_begin;
    ti.phase = p;
    ti.m0 = (CL * (lt % P.m_blocks) + crank) * BM;  // CL == 2: m_blocks counts pairs
    ti.nb = lt / P.m_blocks;
    ti.kb_begin = 0;
    ti.kb_end = P.nr * P.ns * g.cv.cblocks;
  } else if constexpr (MODE == LOAD_CONV_FPROP_ROWSEG) {
    // tile = 128 output pixels (segment ti.tap) of output row n*P + oh; rows
    // wider than 128 pixels take cv.band_sub segments
    const int rs = t / g.n_blocks;
    ti.nb = t - rs * g.n_blocks;
    const int row = rs / g.cv.band_sub;
    ti.tap = rs - row * g.cv.band_sub;
    ti.m0 = row;  // n*P + oh
    ti.kb_begin = 0;
    ti.kb_end = g.cv.R;
  } else if constexpr (MODE == LOAD_CONV_DGRAD_BAND) {
    const int band = t / g.n_blocks;
    ti.nb = t - band * g.n_blocks;
    ti.m0 = band;  // n*bands_per_img + b
    ti.kb_begin = 0;
    ti.kb_end = g.k_blocks;
    ti.nsub = g.cv.band_sub;
  } else {
    int split_t = 0;
    if constexpr (MODE == LOAD_GEMM) {
      if (g.tail_splits > 0 && t >= g.full_tiles) {  // K-slice of a last-wave tile
        ti.unit = t - g.full_tiles;
        split_t = ti.unit % g.tail_splits;
        t = g.full_tiles + ti.unit / g.tail_splits;
      }
    }
    int mb, rest;
    if ((MODE == LOAD_GEMM || MODE == LOAD_GEMM_3XTF32) && g.n_fastest) {
      ti.nb = t % g.n_blocks;
      rest = t / g.n_blocks;
      mb = rest % g.m_blocks;
      rest /= g.m_blocks;
    } else {
      mb = t % g.m_blocks;  // CL == 2: m_blocks counts pairs of M tiles
      rest = t / g.m_blocks;
      ti.nb = rest % g.n_blocks;
      rest /= g.n_blocks;
    }
    ti.m0 = (CL * mb + crank) * BM;
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
    } else if (ti.unit >= 0) {
      ti.kb_begin = split_t * g.tail_kbps;
      ti.kb_end = min(g.k_blocks, ti.kb_begin + g.tail_kbps);
    } else {
      const int split = rest;
      ti.kb_begin = split * g.kb_per_split;
      ti.kb_end = min(g.k_blocks, ti.kb_begin + g.kb_per_split);
    }
  }
  return ti;
}

// band dgrad: first dY row contributing to dX rows [h0, h0 + band_h)
__device__ __forceinline__ int band_first_row(const ConvShape& cv, int h0) {
  return -floor_div(-(h0 + cv.ph - cv.R + 1), cv.sh);  // ceil((h0+ph-R+1)/sh)
}

constexpr int pow2_cols(int c) {
  return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

template <int BN, int A_MN, int B_MN, int MODE, int CL = 1>
struct GemmCfg {
  static constexpr int KBYTES = MODE == LOAD_CONV_FPROP_ROWSEG ? 64 : 128;  // K bytes per row
  // k-blocks per pipeline stage: 2 for CTA pairs and N = 64 single tiles, whose
  // 4-MMA k-blocks (64 clk per MMA at N = 128) are too short to amortise one
  // barrier round trip and one TMA batch per k-block (layer-2 conv 0.081 ->
  // 0.066 ms); wgrad / stem / C8 modes keep 1
  static constexpr int KS =
      MODE == LOAD_CONV_FPROP_ROWSEG ? 4  // a whole 3x3 window (3 kernel rows) per stage
      : (((CL == 2 && BN <= 256) || (CL == 1 && BN == 64)) &&
         (MODE == LOAD_CONV_FPROP || MODE == LOAD_CONV_DGRAD || MODE == LOAD_GEMM))
          ? 2
          : 1;
  static constexpr int A_SUB = BM * KBYTES;          // one k-block of A
  static constexpr int B_SUB = BN / CL * KBYTES;     // this CTA's share of one k-block of B
  static constexpr int PARTS = MODE == LOAD_GEMM_3XTF32 ? 2 : 1;  // hi / lo planes
  static constexpr int A_BYTES = KS * A_SUB * PARTS;
  static constexpr int B_BYTES = KS * B_SUB * PARTS;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EXTRA = MODE == LOAD_CONV_DGRAD_BAND ? BAND_WINDOW_BYTES : 0;
  // TMA-store staging: 4 epilogue warps x 4 buffers x (32 rows x 64 B)
  static constexpr bool CAN_TMA_STORE = MODE == LOAD_GEMM || MODE == LOAD_CONV_FPROP ||
                                        MODE == LOAD_CONV_FPROP_C8 ||
                                        MODE == LOAD_CONV_FPROP_ROWSEG;
  // epilogue warps: 8 (two per TMEM lane quarter, each draining half of the
  // columns) so a second warp per SM sub-partition hides TMEM-load / store
  // latency; the band dgrad has its own 8-window layout
  static constexpr int EPI = MODE == LOAD_CONV_DGRAD_BAND ? BAND_WINDOWS : (BN >= 64 ? 8 : 4);
  static constexpr int EPI_H = MODE == LOAD_CONV_DGRAD_BAND ? 1 : EPI / 4;  // warps per quarter
  // BN = 64: the two warps of a TMEM lane quarter take alternate TILES (all 64
  // columns each) instead of half the columns of every tile, so two tiles' fused
  // epilogues are in flight (a 64-column tile's epilogue is latency-bound: VGG
  // conv1_1 wrote 1.9 TB/s with one tile at a time)
  static constexpr bool TILE_ALT = BN == 64 && CL == 1 && MODE != LOAD_CONV_DGRAD_BAND && EPI == 8;
  static constexpr int COL_SPLIT = TILE_ALT ? 1 : EPI_H;  // warps sharing one tile's columns
  static constexpr int STG_BUFS = 4 / EPI_H;
  static constexpr int STG = CAN_TMA_STORE ? EPI * STG_BUFS * 2048 : 0;
  static constexpr int SMEM_MAX = 227 * 1024;
  static constexpr int STAGES_MAX = (SMEM_MAX - 1280 - EXTRA - STG) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_MAX > 8 ? 8 : STAGES_MAX;
  // TMEM accumulators in flight: 4 when they fit the 512 columns (BN <= 128),
  // so epilogue jitter does not stall the MMAs; the band dgrad keeps 2
  static constexpr int NACC = (MODE != LOAD_CONV_DGRAD_BAND && 4 * BN <= 512) ? 4 : 2;
  static constexpr int TMEM_COLS = pow2_cols(NACC * BN);
  static constexpr int SMEM_BYTES =
      STAGES * STAGE_BYTES + STG + EXTRA + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int THREADS = 64 + 32 * EPI;
};

// CL = 2: a CTA pair (cluster of 2 on one TPC) computes a 256 x BN tile with
// tcgen05.mma.cta_group::2 (M = 256).  Each CTA TMA-loads its own 128 rows of A
// and half of the B tile into its smem, signalling the even CTA's full barrier;
// the even CTA alone issues the MMAs, whose commits arrive on both CTAs' empty /
// accumulator-full barriers.  Each CTA's epilogue drains its own TMEM lanes and
// releases the accumulator on the even CTA's barrier.  Per SM this halves the B
// bytes staged through shared memory per FLOP (the 1-CTA 128x256 tile is smem-
// bandwidth bound at ~2/3 of tensor peak).
template <int BN, int A_MN, int B_MN, int MODE, int CL = 1>
__global__ void __launch_bounds__(GemmCfg<BN, A_MN, B_MN, MODE, CL>::THREADS, 1)
    umma_gemm_kernel(const __grid_constant__ TmapPack tm, const __grid_constant__ GemmArgs g) {
  using Cfg = GemmCfg<BN, A_MN, B_MN, MODE, CL>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int KMMA = Cfg::KBYTES / 32;  // tcgen05.mma (K=16) per stage
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");
  static_assert(MODE != LOAD_CONV_DGRAD_BAND || BN == 160, "band dgrad is specialised to BN=160");
  static_assert(MODE != LOAD_GEMM_3XTF32 || (CL == 1 && Cfg::KS == 1), "3xTF32: 1 CTA, 1 k-block");
  static_assert(CL == 1 || MODE == LOAD_GEMM || MODE == LOAD_CONV_FPROP ||
                    MODE == LOAD_CONV_DGRAD,
                "CTA pairs are implemented for GEMM and im2col conv fprop / dgrad");
  static_assert(CL == 1 || (BN / CL) % 16 == 0, "pair: B half must be a multiple of 16 rows");
  // a follow-up launched with programmatic stream serialization (the last-wave
  // K-split finalize) may be scheduled now: its blocks wait in
  // griddepcontrol.wait until this grid has finished, so only the launch
  // latency overlaps (no effect on launches without the attribute)
  pdl_trigger();
  const int crank = CL > 1 ? static_cast<int>(cluster_ctarank()) : 0;
  const int t_first = static_cast<int>(blockIdx.x) / CL;
  const int t_step = static_cast<int>(gridDim.x) / CL;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the swizzle atoms, by an offset from the shared
  // array (an integer round trip would make the pointer generic: the staging
  // and band-window accesses would compile to generic ST/LD instead of STS/LDS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;
  uint8_t* staging = smem + STAGES * Cfg::STAGE_BYTES;  // TMA-store chunks (1024-aligned)
  float* region = reinterpret_cast<float*>(staging + Cfg::STG);  // band windows
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(staging + Cfg::STG + Cfg::EXTRA);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + STAGES;
  constexpr int NACC = Cfg::NACC;
  uint64_t* tfull_bar = bars + 2 * STAGES;
  uint64_t* tempty_bar = bars + 2 * STAGES + NACC;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 2 * NACC);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(smem_u32(&full_bar[i]), 1);
      mbar_init(smem_u32(&empty_bar[i]), 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(smem_u32(&tfull_bar[i]), 1);
      // CL = 2: one arrival per epilogue warp of both CTAs (on the even CTA's barrier)
      mbar_init(smem_u32(&tempty_bar[i]),
                CL == 1 ? (Cfg::TILE_ALT ? 4 : Cfg::EPI) * 32 : CL * Cfg::EPI);
    }
    fence_mbar_init();
    tma_prefetch_desc(&tm.b);
    tma_prefetch_desc(&tm.a[0]);
  }
  if constexpr (MODE == LOAD_CONV_DGRAD_BAND)
    for (int i = threadIdx.x; i < BAND_WINDOW_BYTES / 4; i += blockDim.x) region[i] = 0.f;
  if (warp == 1) {
    if constexpr (CL == 1) tmem_alloc(smem_u32(tmem_holder), Cfg::TMEM_COLS);
    else tmem_alloc_cg2(smem_u32(tmem_holder), Cfg::TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync();  // peer barriers initialised before any remote signal
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  pdl_wait();  // the prologue above may overlap the previous kernel (launch_pdl)

  if (warp == 0) {
    // ============================ TMA producer ============================
    {  // whole warp: uniform tile / stage arithmetic; an elect.sync lane issues
      int stage = 0;
      uint32_t phase = 0;
      for (int t = t_first; t < g.num_tiles; t += t_step) {
        TileInfo ti = decode_tile<MODE, CL>(g, t, crank);
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
        } else if constexpr (MODE == LOAD_CONV_FPROP_ROWSEG) {
          cn = ti.m0 / g.cv.P;
          const int oh = ti.m0 - cn * g.cv.P;
          ch = oh * g.cv.sh - g.cv.ph;
        } else if constexpr (MODE == LOAD_CONV_DGRAD_BAND) {
          cn = ti.m0 / g.cv.bands_per_img;
          const int b = ti.m0 - cn * g.cv.bands_per_img;
          ch = band_first_row(g.cv, b * g.cv.band_h);  // first dY row of the band
        }
        for (int sub = 0; sub < ti.nsub; ++sub) {
          for (int kb0 = ti.kb_begin; kb0 < ti.kb_end; kb0 += Cfg::KS) {
            const int nkb = min(Cfg::KS, ti.kb_end - kb0);
            mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
            // CL = 2: both CTAs' loads complete on the even CTA's full barrier
            const uint32_t fb = CL == 1 ? smem_u32(&full_bar[stage])
                                        : mapa_shared(smem_u32(&full_bar[stage]), 0);
            const uint32_t sA0 = smem_u32(ring + stage * Cfg::STAGE_BYTES);
            // one k-block's TMA loads into (sA, sB)
            auto issue = [&](const int kb, const uint32_t sA, const uint32_t sB) {
              if constexpr (MODE == LOAD_GEMM) {
                const int k0 = kb * BK;
                if constexpr (CL > 1) {
                  if constexpr (A_MN) {
                    tma_load_2d_cg2(sA, &tm.a[0], fb, ti.m0, k0);
                    tma_load_2d_cg2(sA + 8192, &tm.a[0], fb, ti.m0 + 64, k0);
                  } else {
                    tma_load_2d_cg2(sA, &tm.a[0], fb, k0, ti.m0);
                  }
                  const int nh = n0 + crank * (BN / CL);  // this CTA's half of the B tile
                  if constexpr (B_MN) {
  #pragma unroll
                    for (int j = 0; j < BN / CL / 64; ++j)
                      tma_load_2d_cg2(sB + j * 8192, &tm.b, fb, nh + 64 * j, k0);
                  } else {
                    tma_load_2d_cg2(sB, &tm.b, fb, k0, nh);
                  }
                } else {
                  if constexpr (A_MN) {
                    tma_load_2d(sA, &tm.a[0], fb, ti.m0, k0);
                    tma_load_2d(sA + 8192, &tm.a[0], fb, ti.m0 + 64, k0);
                  } else {
                    tma_load_2d(sA, &tm.a[0], fb, k0, ti.m0);
                  }
                }
                if constexpr (CL > 1) {
                } else if constexpr (B_MN) {
  #pragma unroll
                  for (int j = 0; j < BN / 64; ++j)
                    tma_load_2d(sB + j * 8192, &tm.b, fb, n0 + 64 * j, k0);
                } else {
                  tma_load_2d(sB, &tm.b, fb, k0, n0);
                }
              } else if constexpr (MODE == LOAD_GEMM_3XTF32) {
                // 128-byte rows = 32 fp32; a[0] / a[1] = A hi / lo, b / a[2] = B hi / lo
                const int k0 = kb * 32;
                tma_load_2d(sA, &tm.a[0], fb, k0, ti.m0);
                tma_load_2d(sA + Cfg::A_SUB, &tm.a[1], fb, k0, ti.m0);
                tma_load_2d(sB, &tm.b, fb, k0, n0);
                tma_load_2d(sB + Cfg::B_SUB, &tm.a[2], fb, k0, n0);
              } else if constexpr (MODE == LOAD_CONV_FPROP) {
                const int tap = kb / g.cv.cblocks;
                const int cb = kb - tap * g.cv.cblocks;
                const int r = tap / g.cv.S, s = tap - (tap / g.cv.S) * g.cv.S;
                if constexpr (CL > 1) {
                  tma_load_im2col_4d_cg2(sA, amap, fb, cb * 64, cw, ch, cn, (uint16_t)s, (uint16_t)r);
                  tma_load_2d_cg2(sB, &tm.b, fb, tap * g.cv.wrow_cpad + cb * 64,
                                  n0 + crank * (BN / CL));
                } else {
                  tma_load_im2col_4d(sA, amap, fb, cb * 64, cw, ch, cn, (uint16_t)s, (uint16_t)r);
                  tma_load_2d(sB, &tm.b, fb, tap * g.cv.wrow_cpad + cb * 64, n0);
                }
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
              } else if constexpr (MODE == LOAD_CONV_FPROP_ROWSEG) {
                // k-block = kernel row r: 128 overlapping segments of one input row
                // (rowseg8: the contiguous segment, 17 x 128-byte chunks)
                if (g.rowseg8) tma_load_4d(sA, amap, fb, 0, ti.tap * (BM / 8), ch + kb, cn);
                else tma_load_4d(sA, amap, fb, 0, ti.tap * BM, ch + kb, cn);
                tma_load_2d(sB, &tm.b, fb, kb * 32, n0);
              } else if constexpr (MODE == LOAD_CONV_DGRAD_BAND) {
                // one full dY row (Q pixels, 64 channels); rows outside [0, P) load zeros
                tma_load_4d(sA, amap, fb, kb * BK, 0, ch + sub, cn);
                tma_load_2d(sB, &tm.b, fb, kb * BK, n0);
              } else if constexpr (MODE == LOAD_CONV_DGRAD) {
                const PhaseInfo& P = g.phase[ti.phase];
                const int cb = kb % g.cv.cblocks;
                const int tt = kb / g.cv.cblocks;
                const int ts = tt % P.ns, tr = tt / P.ns;
                const int r = P.r0 + g.cv.sh * tr, s = P.s0 + g.cv.sw * ts;
                if constexpr (CL > 1) {
                  tma_load_im2col_4d_cg2(sA, amap, fb, cb * 64, cw, ch, cn,
                                         (uint16_t)(P.ns - 1 - ts), (uint16_t)(P.nr - 1 - tr));
                  tma_load_2d_cg2(sB, &tm.b, fb, (r * g.cv.S + s) * g.cv.wrow_cpad + cb * 64,
                                  n0 + crank * (BN / CL));
                } else {
                  tma_load_im2col_4d(sA, amap, fb, cb * 64, cw, ch, cn, (uint16_t)(P.ns - 1 - ts),
                                     (uint16_t)(P.nr - 1 - tr));
                  tma_load_2d(sB, &tm.b, fb, (r * g.cv.S + s) * g.cv.wrow_cpad + cb * 64, n0);
                }
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
            };
            if (elect_one()) {
              if (crank == 0)
                mbar_arrive_expect_tx(
                    smem_u32(&full_bar[stage]),
                    CL * nkb *
                        ((MODE == LOAD_CONV_FPROP_ROWSEG && g.rowseg8 ? ROWSEG8_A_TX : Cfg::A_SUB) +
                         Cfg::B_SUB) *
                        Cfg::PARTS);
              for (int j = 0; j < nkb; ++j)
                issue(kb0 + j, sA0 + j * Cfg::A_SUB, sA0 + Cfg::A_BYTES + j * Cfg::B_SUB);
            }
            __syncwarp();
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    // The whole warp runs the loop, so the tile / stage arithmetic and the smem
    // descriptors are warp-uniform (uniform registers), and an elect.sync lane
    // issues.  (A lane-0-only loop makes the compiler wrap every tcgen05.mma in
    // an ELECT / R2UR.BROADCAST waterfall -- as long as an N = 128 MMA itself.)
    if (crank == 0) {
      const uint32_t idesc = make_idesc_f16(g.ab_fmt, BM * CL, BN, A_MN, B_MN);
      const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
      const uint32_t ring_u = smem_u32(ring);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = t_first; t < g.num_tiles; t += t_step) {
        TileInfo ti = decode_tile<MODE, CL>(g, t, crank);
        for (int sub = 0; sub < ti.nsub; ++sub, ++local) {
          const int acc = local % NACC;
          const uint32_t use = static_cast<uint32_t>(local / NACC);
          if constexpr (CL == 1) mbar_wait(smem_u32(&tempty_bar[acc]), (use & 1) ^ 1);
          else mbar_wait_cluster(smem_u32(&tempty_bar[acc]), (use & 1) ^ 1);
          tc_fence_after();
          const uint32_t dcol = tmem_u + acc * BN;
          if (ti.kb_end <= ti.kb_begin) {
            // empty reduction: the epilogue writes zeros
            if (elect_one()) {
              if constexpr (CL == 1) {
                mbar_arrive(smem_u32(&tfull_bar[acc]));
              } else {
                for (int c = 0; c < CL; ++c)
                  mbar_arrive_cluster(mapa_shared(smem_u32(&tfull_bar[acc]), c));
              }
            }
            __syncwarp();
            continue;
          }
          for (int kb0 = ti.kb_begin; kb0 < ti.kb_end; kb0 += Cfg::KS) {
            const int nkb = min(Cfg::KS, ti.kb_end - kb0);
            mbar_wait(smem_u32(&full_bar[stage]), phase);
            tc_fence_after();
            uint64_t ads[Cfg::KS * KMMA], bds[Cfg::KS * KMMA];
#pragma unroll
            for (int kk = 0; kk < Cfg::KS * KMMA; ++kk) {
              const int k = kk % KMMA, jsub = kk / KMMA;
              const uint32_t sA = ring_u + stage * Cfg::STAGE_BYTES + jsub * Cfg::A_SUB;
              const uint32_t sB = ring_u + stage * Cfg::STAGE_BYTES + Cfg::A_BYTES +
                                  jsub * Cfg::B_SUB;
              uint64_t ad, bd;
              if constexpr (MODE == LOAD_CONV_FPROP_C8)  // core matrices 8 rows x 16 B
                ad = make_smem_desc(sA + k * 4096, 2048, 128, LAYOUT_SWIZZLE_NONE);
              else if constexpr (MODE == LOAD_CONV_FPROP_ROWSEG)  // 64-byte rows
                ad = g.rowseg8 ? make_smem_desc(sA + k * 32, 16, 128, LAYOUT_SWIZZLE_NONE)
                               : make_smem_desc(sA + k * 32, 16, 512, LAYOUT_SWIZZLE_64B);
              else if constexpr (A_MN)
                ad = make_smem_desc(sA + k * 2048, 8192, 1024, LAYOUT_SWIZZLE_128B);
              else
                ad = make_smem_desc(sA + k * 32, 16, 1024, LAYOUT_SWIZZLE_128B);
              if constexpr (MODE == LOAD_CONV_FPROP_ROWSEG)
                bd = make_smem_desc(sB + k * 32, 16, 512, LAYOUT_SWIZZLE_64B);
              else if constexpr (B_MN)
                bd = make_smem_desc(sB + k * 2048, 8192, 1024, LAYOUT_SWIZZLE_128B);
              else
                bd = make_smem_desc(sB + k * 32, 16, 1024, LAYOUT_SWIZZLE_128B);
              ads[kk] = ad;
              bds[kk] = bd;
            }
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < Cfg::KS * KMMA; ++kk) {
                if (kk / KMMA < nkb) {
                  const uint32_t accum = (kb0 > ti.kb_begin || kk > 0) ? 1u : 0u;
                  if constexpr (MODE == LOAD_GEMM_3XTF32) {
                    // hi*hi + hi*lo + lo*hi (descriptor start +A_SUB / +B_SUB = lo plane)
                    const uint64_t a_lo = ads[kk] + (uint64_t)(Cfg::A_SUB >> 4);
                    const uint64_t b_lo = bds[kk] + (uint64_t)(Cfg::B_SUB >> 4);
                    umma_tf32(dcol, ads[kk], bds[kk], idesc, accum);
                    umma_tf32(dcol, ads[kk], b_lo, idesc, 1u);
                    umma_tf32(dcol, a_lo, bds[kk], idesc, 1u);
                  } else if constexpr (CL == 1) {
                    umma_f16(dcol, ads[kk], bds[kk], idesc, accum);
                  } else {
                    umma_f16_cg2(dcol, ads[kk], bds[kk], idesc, accum);
                  }
                }
              }
              // frees the smem slot (in both CTAs of a pair) when the MMAs retire
              if constexpr (CL > 1)
                umma_commit_cg2_mc(smem_u32(&empty_bar[stage]), (1u << CL) - 1);
              else
                umma_commit(smem_u32(&empty_bar[stage]));
            }
            __syncwarp();
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          // accumulator ready for the epilogue (of both CTAs of a pair)
          if (elect_one()) {
            if constexpr (CL > 1) umma_commit_cg2_mc(smem_u32(&tfull_bar[acc]), (1u << CL) - 1);
            else umma_commit(smem_u32(&tfull_bar[acc]));
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ============================ epilogue ============================
    const uint32_t quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    int local = 0;
    uint32_t stg_count = 0;  // TMA-store staging buffer parity
    const EpiParams& e = g.epi;
    // eval-BN fold of this warp's columns, hoisted out of the tile loop when the
    // columns never change (one N-block): the four parameter loads and the rsqrt
    // otherwise sit on every tile's epilogue critical path
    constexpr int NCH = (BN / Cfg::COL_SPLIT + 31) / 32;
    float hs[NCH], ht[NCH];
    const bool bn_hoist = MODE != LOAD_CONV_DGRAD_BAND && e.bn.var != nullptr && g.n_blocks == 1;
    if (bn_hoist) {
      const int c_lo0 =
          (Cfg::COL_SPLIT == 1 ? 0 : ((static_cast<int>(warp) - 2) >> 2)) * (BN / Cfg::COL_SPLIT);
#pragma unroll
      for (int ci = 0; ci < NCH; ++ci) {
        hs[ci] = 1.f;
        ht[ci] = 0.f;
        const int col = c_lo0 + ci * 32 + static_cast<int>(lane);
        if (col < g.N) bn_fold(e.bn, col, hs[ci], ht[ci]);
      }
    }
    for (int t = t_first; t < g.num_tiles; t += t_step) {
      TileInfo ti = decode_tile<MODE, CL>(g, t, crank);
      const int n0 = ti.nb * BN;

      if constexpr (MODE == LOAD_CONV_DGRAD_BAND) {
        // ---- band of dX rows [h0, h0 + BAND_H) of image nn.  Thread = dY pixel
        // ow = its TMEM lane.  Each epilogue warp owns a private window covering
        // its 32 pixels, stored as [row][ci][x parity][x/2] so that for a fixed
        // accumulator column the 32 lanes touch 32 consecutive floats.
        const ConvShape& cv = g.cv;
        const int nn = ti.m0 / cv.bands_per_img;
        const int h0 = (ti.m0 - nn * cv.bands_per_img) * BAND_H;
        const int oh0 = band_first_row(cv, h0);
        const int ew = static_cast<int>(warp) - 2;  // 0..7
        const int half = ew >> 2;                   // which chunks of 32 columns
        // window index = half*4 + TMEM lane quarter (the flush relies on it)
        // volatile: lane l's column (s+2) aliases lane l+1's column s, so the
        // per-column read-modify-writes must stay in program order (the warp
        // executes them in lockstep; the compiler must not batch them).
        volatile float* win = region + (half * 4 + static_cast<int>(quarter)) * BAND_WIN +
                              static_cast<int>(lane);
        const int ow = row;
        for (int sub = 0; sub < ti.nsub; ++sub, ++local) {
          const int acc = local % NACC;
          const uint32_t use = static_cast<uint32_t>(local / NACC);
          mbar_wait(smem_u32(&tfull_bar[acc]), use & 1);
          tc_fence_after();
          const int oh = oh0 + sub;
          const bool rvalid = ow < cv.Q && oh >= 0 && oh < cv.P;
          const int hbase = oh * cv.sh - cv.ph - h0;  // window row of kernel row 0
          auto chunk = [&](auto cc) {
            constexpr int c = decltype(cc)::value;
            uint32_t r[32];
            tmem_ld_32x32b_x32(tmem_base + ((quarter * 32u) << 16) + acc * BN + c, r);
            tmem_ld_wait();
            if (!rvalid) return;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = c + j;  // compile-time after unrolling
              if (col < BAND_R * BAND_S * BAND_C) {
                const int tap = col / BAND_C, ci = col % BAND_C;
                const int rr = tap / BAND_S, ss = tap % BAND_S;
                const int hh = hbase + rr;
                if (static_cast<unsigned>(hh) < static_cast<unsigned>(BAND_H))
                  win[hh * BAND_ROWF + (ci * 2 + (ss & 1)) * BAND_WH + (ss >> 1)] +=
                      __uint_as_float(r[j]);
              }
            }
          };
          if (half == 0) {
            chunk(IntC<0>{});
            chunk(IntC<64>{});
            chunk(IntC<128>{});
          } else {
            chunk(IntC<32>{});
            chunk(IntC<96>{});
          }
          tc_fence_before();
          mbar_arrive(smem_u32(&tempty_bar[acc]));
        }
        // ---- flush: sum the warp windows covering each dX pixel, store dX directly
        constexpr int NT = BAND_WINDOWS * 32;
        asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
        const int tid = ew * 32 + static_cast<int>(lane);
        const int rows = min(BAND_H, cv.outH - h0);
        const int per_row = cv.outW * BAND_C;
        for (int hh = 0; hh < rows; ++hh) {
          const int64_t obase = ((static_cast<int64_t>(nn) * cv.outH + h0 + hh) * cv.outW) * BAND_C;
          for (int i = tid; i < per_row; i += NT) {
            const int w = i / BAND_C, ci = i - (i / BAND_C) * BAND_C;
            const int xg = w + cv.pw;  // window column for quarter 0
            float v = 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int x = xg - 32 * q * BAND_SW;
              if (x >= 0 && x < BAND_WC) {
                const int o = hh * BAND_ROWF + (ci * 2 + (x & 1)) * BAND_WH + (x >> 1);
                v += region[q * BAND_WIN + o] + region[(q + 4) * BAND_WIN + o];
              }
            }
            store_from_float(e.out, e.out_dtype, obase + i, v);
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
        for (int i = tid; i < BAND_WINDOWS * BAND_WIN; i += NT) region[i] = 0.f;
        asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
      } else {
        const int acc = local % NACC;
        const uint32_t use = static_cast<uint32_t>(local / NACC);
        ++local;
        // TILE_ALT: warps 2-5 take the CTA's even tiles, warps 6-9 the odd ones
        if (Cfg::TILE_ALT && (((local - 1) & 1) != ((static_cast<int>(warp) - 2) >> 2))) continue;
        const bool tail = ti.unit >= 0;  // fp32 partial of a K-sliced last-wave tile
        const bool tma_st = Cfg::CAN_TMA_STORE && g.tma_store && !tail;
        const int ncols = g.N;
        // this warp drains columns [c_lo, c_lo + BN / COL_SPLIT) of the accumulator
        constexpr int WCOLS = BN / Cfg::COL_SPLIT;
        const int c_lo = (Cfg::COL_SPLIT == 1 ? 0 : ((static_cast<int>(warp) - 2) >> 2)) * WCOLS;
        // 16-bit bias of this warp's columns, fetched before the accumulator wait
        // so its latency overlaps the main loop: lane j holds columns 8j .. 8j + 7
        // (a K-sliced tile adds the bias in its first slice only)
        const bool bias_vec = e.bias != nullptr && e.bias_dtype != MS_F32 && (ncols & 7) == 0 &&
                              (reinterpret_cast<uintptr_t>(e.bias) & 15) == 0 &&
                              ti.kb_begin == 0;
        uint4 bq = make_uint4(0u, 0u, 0u, 0u);
        if (bias_vec) {
          const int bc = n0 + c_lo + 8 * static_cast<int>(lane);
          if (static_cast<int>(lane) < WCOLS / 8 && bc < ncols)
            bq = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(e.bias) + bc));
        }
        mbar_wait(smem_u32(&tfull_bar[acc]), use & 1);
        tc_fence_after();
        const bool zero = ti.kb_end <= ti.kb_begin;

        // ---- output row address
        const int m = ti.m0 + row;
        bool valid;
        int64_t orow;
        if constexpr (MODE == LOAD_CONV_DGRAD) {
          const PhaseInfo& P = g.phase[ti.phase];
          valid = m < P.m_total;
          const int hw = P.Hp * P.Wp;
          const int nn = m / hw;
          const int rem = m - nn * hw;
          const int i = rem / P.Wp, j = rem - (rem / P.Wp) * P.Wp;
          const int h = g.cv.sh * i + P.ph, w = g.cv.sw * j + P.pw;
          orow = (static_cast<int64_t>(nn) * g.cv.outH + h) * g.cv.outW + w;
        } else if constexpr (MODE == LOAD_CONV_FPROP_ROWSEG) {
          const int q = ti.tap * BM + row;
          valid = q < g.cv.Q;
          orow = static_cast<int64_t>(ti.m0) * g.cv.Q + q;
        } else {
          valid = m < g.M;
          orow = m;
        }
        int64_t col_base = n0;
        if constexpr (MODE == LOAD_CONV_WGRAD) col_base += static_cast<int64_t>(ti.tap) * g.N;

        const uint32_t taddr = tmem_base + ((quarter * 32u) << 16) + acc * BN;
        // residual / addend chunk and producer-ReLU keep bits of chunk cc, loaded
        // one chunk ahead: their global-load latency overlaps the previous
        // chunk's work instead of serialising every chunk (fused dgrad epilogues
        // read an addend and a mask per 32 columns)
        uint4 rnx[4];
        bool rnx_ok = false, knx_ok = false;
        uint32_t knx = 0;
        auto prefetch = [&](int cc) {
          const int cpf = c_lo + cc * 32;
          rnx_ok = knx_ok = false;
          if (!valid || tail || n0 + cpf + 32 > ncols) return;
          const int64_t el = orow * e.ldc + col_base + cpf;
          if (e.resid != nullptr) {
            const uint16_t* r16 = static_cast<const uint16_t*>(e.resid) + el;
            if ((reinterpret_cast<uintptr_t>(r16) & 15) == 0) {
              rnx_ok = true;
#pragma unroll
              for (int q = 0; q < 4; ++q) rnx[q] = __ldg(reinterpret_cast<const uint4*>(r16) + q);
            }
          }
          if (e.keep_in != nullptr && (el & 31) == 0) {
            knx_ok = true;
            knx = __ldg(reinterpret_cast<const uint32_t*>(e.keep_in) + (el >> 5));
          }
        };
        prefetch(0);
#pragma unroll 1
        for (int ci = 0; ci < WCOLS / 32; ++ci) {
          const int c = c_lo + ci * 32;
          uint32_t r[32];
          // eval-BN affine: lane j folds column n0 + c + j (loads overlap the TMEM read)
          float bs = 1.f, bt = 0.f;
          if (bn_hoist) {
#pragma unroll
            for (int q = 0; q < NCH; ++q)
              if (q == ci) {
                bs = hs[q];
                bt = ht[q];
              }
          } else if (e.bn.var != nullptr && n0 + c + static_cast<int>(lane) < ncols) {
            bn_fold(e.bn, n0 + c + static_cast<int>(lane), bs, bt);
          }
          // this chunk's prefetched residual / keep bits; start the next chunk's
          uint4 rpre[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) rpre[q] = rnx[q];
          const bool rpre_ok = rnx_ok, kpre_ok = knx_ok;
          const uint32_t kpre = knx;
          if (ci + 1 < WCOLS / 32) prefetch(ci + 1);
          __syncwarp();  // tcgen05.ld / wait are warp-collective: reconverge invalid rows
          if (MODE == LOAD_GEMM && (g.dbg & 2)) continue;
          if (!zero) {
            tmem_ld_32x32b_x32(taddr + c, r);
            tmem_ld_wait_regs(r);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = 0u;
          }
          const int nc = n0 + c;  // first column of this chunk in GEMM-N space
          if (nc >= ncols) continue;  // warp-uniform
          if (MODE == LOAD_GEMM && (g.dbg & 1)) continue;
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          const bool full = (nc + 32 <= ncols);
          if (bias_vec) {  // full-warp shuffles: before any per-row exit
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int src = ci * 4 + q;  // lane holding columns c + 8q .. + 7
              const uint32_t w4[4] = {__shfl_sync(0xffffffffu, bq.x, src),
                                      __shfl_sync(0xffffffffu, bq.y, src),
                                      __shfl_sync(0xffffffffu, bq.z, src),
                                      __shfl_sync(0xffffffffu, bq.w, src)};
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                float lo, hi;
                if (e.bias_dtype == MS_BF16) {
                  lo = __uint_as_float(w4[h] << 16);
                  hi = __uint_as_float(w4[h] & 0xFFFF0000u);
                } else {
                  lo = __half2float(__ushort_as_half((unsigned short)(w4[h] & 0xFFFF)));
                  hi = __half2float(__ushort_as_half((unsigned short)(w4[h] >> 16)));
                }
                v[q * 8 + 2 * h] += lo;
                v[q * 8 + 2 * h + 1] += hi;
              }
            }
          } else if (e.bias != nullptr && ti.kb_begin == 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (nc + j < ncols) v[j] += load_as_float(e.bias, e.bias_dtype, nc + j);
          }
          if (tail) {  // dense fp32 partial [unit][CL*BM][BN], summed by the finalize pass
            if (valid) {
              float* o = g.tail_ws +
                         ((static_cast<int64_t>(ti.unit) * CL + crank) * BM + row) * BN + c;
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            }
            continue;
          }
          if (e.round_lin) {
            auto round_all = [&]() {
              if (e.out_dtype == MS_BF16) {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __bfloat162float(__float2bfloat16_rn(v[j]));
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __half2float(__float2half_rn(v[j]));
              }
            };
            round_all();  // the Linear's output as stored
            if (e.drop.on) {
              // elements el .. el + 31 of the output (el % 4 == 0: N and the
              // pitch are multiples of 4): Philox blocks el/4 .. el/4 + 7
              const int64_t el = orow * e.ldc + col_base + c;
              const uint32_t kb = keep_n32<8>(static_cast<uint64_t>(el) >> 2, e.drop.stream,
                                              e.drop.keys, e.drop.thr);
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = ((kb >> j) & 1u) ? v[j] * e.drop.scale : 0.f;
              round_all();  // the dropout's output as stored
            }
          }
          if (e.bn.var != nullptr && !e.bn_post) {  // folded eval-BN: per-column affine
#pragma unroll
            for (int j = 0; j < 32; ++j)
              v[j] = v[j] * __shfl_sync(0xffffffffu, bs, j) + __shfl_sync(0xffffffffu, bt, j);
          }
          if (e.resid != nullptr && valid) {  // fused residual join of a ResNet block
            const int64_t el = orow * e.ldc + col_base + c;
            const uint16_t* r16 = static_cast<const uint16_t*>(e.resid) + el;
            if (rpre_ok) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint4 u = rpre[q];
                const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                  float lo, hi;
                  if (e.out_dtype == MS_BF16) {
                    lo = __uint_as_float(w4[h] << 16);
                    hi = __uint_as_float(w4[h] & 0xFFFF0000u);
                  } else {
                    lo = __half2float(__ushort_as_half((unsigned short)(w4[h] & 0xFFFF)));
                    hi = __half2float(__ushort_as_half((unsigned short)(w4[h] >> 16)));
                  }
                  v[q * 8 + 2 * h] += lo;
                  v[q * 8 + 2 * h + 1] += hi;
                }
              }
            } else {
              for (int j = 0; j < 32; ++j)
                if (nc + j < ncols) v[j] += load_as_float(e.resid, e.out_dtype, el + j);
            }
          }
          if (e.keep_in != nullptr) {  // the producer ReLU's backward
            uint32_t kb = kpre_ok ? kpre : 0u;
            if (valid && !kpre_ok) {
              const int64_t el = orow * e.ldc + col_base + c;
              if (full && (el & 31) == 0) {
                kb = __ldg(reinterpret_cast<const uint32_t*>(e.keep_in) + (el >> 5));
              } else {
                for (int j = 0; j < 32 && nc + j < ncols; ++j)
                  kb |= ((e.keep_in[(el + j) >> 3] >> ((el + j) & 7)) & 1u) << j;
              }
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = ((kb >> j) & 1u) ? v[j] : 0.f;
          }
          if (e.bn_post) {  // the producer BN's scale (all lanes: warp-uniform)
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] *= __shfl_sync(0xffffffffu, bs, j);
          }
          if (e.relu) {
            uint32_t bits = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const bool pos = !(v[j] <= 0.f);  // NaN propagates, as ms_relu_fwd
              bits |= (pos ? 1u : 0u) << j;
              v[j] = pos ? v[j] : 0.f;
            }
            if (e.mask != nullptr && valid) {
              const int64_t el = orow * e.ldc + col_base + c;  // first element of the chunk
              if (full && (el & 31) == 0) {
                reinterpret_cast<uint32_t*>(e.mask)[el >> 5] = bits;
              } else {
                for (int j = 0; j < 32 && nc + j < ncols; j += 8)
                  e.mask[(el + j) >> 3] = static_cast<uint8_t>(bits >> j);
              }
            }
          }
          // fused GELU: after the pre-activation is stored, v becomes gelu(v rounded)
          // in place (no second array: the 32 independent evaluations keep the
          // registers to interleave) and is stored to act_out the same way
          const bool act = e.act_out != nullptr && !(g.dbg & 8);
          auto to_act = [&]() {
            if (g.dbg & 4) return;
            // dtype branch outside the element loop: branch-free bodies let the
            // compiler interleave the 32 independent erf evaluations
            if (e.out_dtype == MS_BF16) {
              // round to bf16 (nearest-even) with integer ops instead of the
              // quarter-rate conversion unit, which MUFU.EX2 also needs
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const uint32_t b = __float_as_uint(v[j]);
                v[j] = __uint_as_float((b + 0x7fffu + ((b >> 16) & 1u)) & 0xffff0000u);
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __half2float(__float2half_rn(v[j]));
            }
#pragma unroll
            for (int j0 = 0; j0 < 32; j0 += GELU_ILP) {
              float q[GELU_ILP];
#pragma unroll
              for (int k = 0; k < GELU_ILP; ++k) q[k] = v[j0 + k];
              gelu_n<GELU_ILP>(q);
#pragma unroll
              for (int k = 0; k < GELU_ILP; ++k) v[j0 + k] = q[k];
            }
          };
          if (!valid && !tma_st) continue;
          if constexpr (Cfg::CAN_TMA_STORE) {
            if (tma_st) {
              // pack, stage this warp's 32 rows x 32 columns (64-byte rows, 64B swizzle),
              // and let one lane store the chunk with TMA (clips the M / N tails)
              const int ew = static_cast<int>(warp) - 2;
              static_assert(Cfg::STG_BUFS >= 2, "staging ring");
#pragma unroll 1
              for (int pass = 0; pass < (act ? 2 : 1); ++pass) {
                if (pass == 1) to_act();
                uint32_t p[16];
                if (e.out_dtype == MS_BF16) {
#pragma unroll
                  for (int j = 0; j < 16; ++j) p[j] = pack2<__nv_bfloat16>(v[2 * j], v[2 * j + 1]);
                } else {
#pragma unroll
                  for (int j = 0; j < 16; ++j) p[j] = pack2<__half>(v[2 * j], v[2 * j + 1]);
                }
                uint8_t* stg = staging + (ew * Cfg::STG_BUFS + (stg_count % Cfg::STG_BUFS)) * 2048;
                // the store issued STG_BUFS chunks ago has finished reading this buffer
                if (lane == 0) bulk_wait_read<Cfg::STG_BUFS - 1>();
                __syncwarp();
                const int rw = static_cast<int>(lane);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  *reinterpret_cast<uint4*>(stg + rw * 64 + ((q ^ ((rw >> 1) & 3)) << 4)) =
                      make_uint4(p[4 * q], p[4 * q + 1], p[4 * q + 2], p[4 * q + 3]);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                  if constexpr (MODE == LOAD_CONV_FPROP_ROWSEG)  // [row][pixel][ch]: clips q >= Q
                    tma_store_3d(&tm.c, smem_u32(stg), nc,
                                 ti.tap * BM + static_cast<int>(quarter) * 32, ti.m0);
                  else
                    tma_store_2d(pass ? &tm.c2 : &tm.c, smem_u32(stg), nc,
                                 ti.m0 + static_cast<int>(quarter) * 32);
                  bulk_commit();
                }
                ++stg_count;
              }
              continue;
            }
          }
          const int64_t off = orow * e.ldc + col_base + c;
          if (e.atomic) {
            float* o = static_cast<float*>(e.out) + off;
            if (full && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
#pragma unroll
              for (int j = 0; j < 32; j += 4) red_add_v4_f32(o + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (full || nc + j < ncols) red_add_f32(o + j, v[j]);
            }
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
            store_row32(e.out, e.out_dtype, off, v, full, ncols - nc);
            if (act) {
              to_act();
              store_row32(e.act_out, e.out_dtype, off, v, full, ncols - nc);
            }
          }
        }
        tc_fence_before();
        if constexpr (CL == 1) {
          mbar_arrive(smem_u32(&tempty_bar[acc]));
        } else {  // one arrival per warp on the even CTA's barrier
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty_bar[acc]), 0));
        }
      }
    }
  }

  if constexpr (Cfg::CAN_TMA_STORE)
    if (warp >= 2 && lane == 0) bulk_wait_all();  // TMA stores complete before exit
  __syncthreads();
  if constexpr (CL > 1) cluster_sync();  // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CL == 1) tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    else tmem_dealloc_cg2(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace ms
