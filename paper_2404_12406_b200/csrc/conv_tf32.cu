// float32 3x3 / stride 1 / pad 1 convolution with 8 input channels on the
// tcgen05 tensor cores (kind::tf32) at float32 accuracy: the Fig. 1 network
// (8 -> 8 channels, NCHW; reference numpy_impl.py:12-38).
//
// 3xTF32: every operand is split exactly into hi = x with the low 13 mantissa
// bits cleared (representable in tf32) and lo = x - hi (exact in fp32), and
//   x * w  ~=  hi_x * hi_w + hi_x * lo_w + lo_x * hi_w
// (the dropped lo*lo term and the tf32 rounding of lo are ~2^-21 relative), so
// 27 MMAs (9 taps x 3 products, M = 128 pixels, N = 16 >= K_out, K = 8
// channels) accumulate one output row segment in fp32 in TMEM.
//
// The A operand (pixels x channels, tap-shifted) lives in TENSOR MEMORY: each
// of the 128 threads owns one output pixel (= one TMEM lane), reads its 3x3x8
// input neighbourhood from three staged input rows in shared memory, splits it
// and stores hi / lo for the 9 taps with tcgen05.st (144 columns).  The MMAs then
// read A from TMEM (the "TS" form) and only the 512-byte weight tiles from
// shared memory, so a K = 8 MMA is not paced by a 4 KB shared-memory A fetch.
// Input rows arrive by TMA (3-D box [8 ch][1 row][136 px] of the NCHW tensor,
// zero fill outside the image = the padding); a CTA walks down a strip of rows
// so each input row is loaded once per strip and serves three output rows.
//
// dX of the same conv is this kernel on dY with the transposed, flipped weights
// W'[c][k][2-r][2-s] (numpy_impl.py:27-38).  dW is a CUDA-core reduction with
// per-block fp32 partials reduced in a fixed order in fp64 (deterministic,
// numpy_impl.py:41-51).
#include "misc.cuh"

namespace ms {
namespace {

constexpr int T3_M = 128;            // output pixels per tile (a row segment)
constexpr int T3_N = 16;             // MMA N: output channels padded to 16
constexpr int T3_C = 8;              // input channels = one tf32 K step
constexpr int T3_LW = 136;           // staged pixels per input row (w0-4 .. w0+131): the
                                     // innermost TMA coordinate must stay 16-byte aligned
constexpr int T3_ROWB = T3_C * T3_LW * 4;  // bytes of one staged row
constexpr int T3_SLOTS = 8;          // input-row ring
constexpr int T3_R = 8;              // output rows per work unit
constexpr int T3_ACC0 = 0;           // TMEM columns: 2 accumulators x 16
constexpr int T3_A0 = 32;            // then A: tap t, part q (hi/lo) at 32 + (2t+q)*8
constexpr int T3_TMEM = 256;         // 2 CTAs per SM share the 512 columns
constexpr int T3_THREADS = 128;
constexpr int T3_SMEM = 96 * 1024;   // > 1/3 of the SM: at most 2 CTAs (TMEM) per SM

struct T3Args {
  int N, H, W, K;        // K = real output channels (<= 16)
  int segs, chunks;      // row segments per row, row chunks per image
  int units;             // N * chunks * segs
  const float* w;        // weights [K][8][3][3] (fwd) or [8][K][3][3] (flip)
  int flip;
  float* y;              // [N][K][H][W]
};

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* tmap, uint32_t bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tmem_st_x8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// D[tmem] (+)= A[tmem] * B[smem], kind::tf32
__device__ __forceinline__ void umma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ float tf32_hi(float v) {
  return __uint_as_float(__float_as_uint(v) & 0xffffe000u);
}

// unit u -> (image, row chunk, segment)
__device__ __forceinline__ void unit_coords(const T3Args& a, int u, int& n, int& h0, int& rows,
                                            int& w0) {
  const int seg = u % a.segs;
  const int rest = u / a.segs;
  const int chunk = rest % a.chunks;
  n = rest / a.chunks;
  h0 = chunk * T3_R;
  rows = min(T3_R, a.H - h0);
  w0 = seg * T3_M;
}

__global__ void __launch_bounds__(T3_THREADS) conv3x3_tf32_kernel(const __grid_constant__
                                                                  CUtensorMap tx, T3Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  float* ring = reinterpret_cast<float*>(smem);                       // [SLOTS][8][136]
  uint8_t* sB = smem + T3_SLOTS * T3_ROWB;                             // 18 x 512 B
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + 18 * 512);         // [SLOTS]
  uint64_t* mma_bar = full + T3_SLOTS;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(mma_bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;

  // ---- weights -> 18 B tiles (tap t, part q): [N=16][K=8] tf32, K-major, no
  // swizzle, two planes of 4 channels (LBO = 256 B), 8-row groups 128 B apart
  for (int i = tid; i < 9 * T3_N * T3_C; i += T3_THREADS) {
    const int c = i % T3_C, n = (i / T3_C) % T3_N, t = i / (T3_C * T3_N);
    float v = 0.f;
    if (n < a.K) {
      v = a.flip ? a.w[((c * a.K + n) * 9) + (8 - t)]   // W[c][k][2-r][2-s]
                 : a.w[((n * T3_C + c) * 9) + t];       // W[k][c][r][s]
    }
    const float hi = tf32_hi(v);
    const int off = (c >> 2) * 256 + n * 16 + (c & 3) * 4;
    *reinterpret_cast<float*>(sB + (2 * t) * 512 + off) = hi;
    *reinterpret_cast<float*>(sB + (2 * t + 1) * 512 + off) = v - hi;
  }
  if (tid == 0) {
    for (int i = 0; i < T3_SLOTS; ++i) mbar_init(smem_u32(&full[i]), 1);
    mbar_init(smem_u32(mma_bar), 1);
    fence_mbar_init();
    tma_prefetch_desc(&tx);
  }
  if (warp == 0) tmem_alloc(smem_u32(tmem_holder), T3_TMEM);
  fence_proxy_async_smem();  // the B tiles are read by the tensor core (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  const uint32_t idesc = make_idesc_f16(2, T3_M, T3_N, 0, 0);  // tf32 x tf32 -> f32

  // the CTA's stream of input rows: unit k (k-th of this CTA) contributes rows
  // h0-1 .. h0+rows, entry e of the stream sits in ring slot e % SLOTS
  auto entry_of = [&](int e, int& uidx, int& j) {
    // walk units (few per CTA); e counts rows across this CTA's units
    int u = blockIdx.x;
    while (u < a.units) {
      int n, h0, rows, w0;
      unit_coords(a, u, n, h0, rows, w0);
      if (e < rows + 2) {
        uidx = u;
        j = e;
        return;
      }
      e -= rows + 2;
      u += gridDim.x;
    }
    uidx = -1;
    j = 0;
  };
  int total = 0;
  for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
    int n, h0, rows, w0;
    unit_coords(a, u, n, h0, rows, w0);
    total += rows + 2;
  }
  int issued = 0;
  auto issue_upto = [&](int limit) {  // thread 0: loads for entries < limit
    while (issued < limit && issued < total) {
      int u, j;
      entry_of(issued, u, j);
      int n, h0, rows, w0;
      unit_coords(a, u, n, h0, rows, w0);
      const int slot = issued % T3_SLOTS;
      const uint32_t bar = smem_u32(&full[slot]);
      mbar_arrive_expect_tx(bar, T3_ROWB);
      tma_load_3d(smem_u32(ring) + slot * T3_ROWB, &tx, bar, w0 - 4, h0 - 1 + j, n * T3_C);
      ++issued;
    }
  };
  if (tid == 0) issue_upto(T3_SLOTS);

  int base = 0;      // stream entry of the current unit's row h0-1
  int tile = 0;      // tiles issued by this CTA
  int pn = 0, ph = 0, pw0 = 0;  // previous tile's output coordinates
  auto epilogue = [&](int t) {
    // wait for tile t's MMAs; its accumulator -> y (thread = pixel)
    mbar_wait(smem_u32(mma_bar), t & 1);
    tc_fence_after();
    uint32_t r[16];
    tmem_ld_x16(tmem + lane_base + T3_ACC0 + (t & 1) * T3_N, r);
    tmem_ld_wait();
    const int w = pw0 + tid;
    if (w < a.W) {
      float* yo = a.y + ((int64_t)pn * a.K * a.H + ph) * a.W + w;
#pragma unroll
      for (int k = 0; k < T3_N; ++k)
        if (k < a.K) yo[(int64_t)k * a.H * a.W] = __uint_as_float(r[k]);
    }
  };
  for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
    int n, h0, rows, w0;
    unit_coords(a, u, n, h0, rows, w0);
    for (int t = 0; t < rows; ++t) {
      // rows h0-1+t .. h0+1+t = stream entries base+t .. base+t+2
      if (tile > 0) epilogue(tile - 1);  // also frees the A columns of tile-1
      for (int q = 0; q < 3; ++q) {
        const int e = base + t + q;
        mbar_wait(smem_u32(&full[e % T3_SLOTS]), (e / T3_SLOTS) & 1);
      }
      // ---- build A: thread tid = pixel w0 + tid; tap (r, s) reads input column
      // w0 + tid + s - 1 = staged index tid + s + 3
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const float* row = ring + ((base + t + r) % T3_SLOTS) * (T3_C * T3_LW);
#pragma unroll
        for (int s = 0; s < 3; ++s) {
          uint32_t hi[8], lo[8];
#pragma unroll
          for (int c = 0; c < T3_C; ++c) {
            const float v = row[c * T3_LW + tid + s + 3];
            const float h = tf32_hi(v);
            hi[c] = __float_as_uint(h);
            lo[c] = __float_as_uint(v - h);
          }
          const int tap = r * 3 + s;
          tmem_st_x8(tmem + lane_base + T3_A0 + (2 * tap) * 8, hi);
          tmem_st_x8(tmem + lane_base + T3_A0 + (2 * tap + 1) * 8, lo);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncthreads();
      if (warp == 0) {
        tc_fence_after();
        if (elect_one()) {
          const uint32_t d = tmem + T3_ACC0 + (tile & 1) * T3_N;
          const uint32_t b0 = smem_u32(sB);
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const uint32_t ahi = tmem + T3_A0 + (2 * tap) * 8;
            const uint32_t alo = tmem + T3_A0 + (2 * tap + 1) * 8;
            const uint64_t bhi = make_smem_desc(b0 + (2 * tap) * 512, 256, 128,
                                                LAYOUT_SWIZZLE_NONE);
            const uint64_t blo = make_smem_desc(b0 + (2 * tap + 1) * 512, 256, 128,
                                                LAYOUT_SWIZZLE_NONE);
            umma_tf32_ts(d, ahi, bhi, idesc, tap ? 1u : 0u);
            umma_tf32_ts(d, ahi, blo, idesc, 1u);
            umma_tf32_ts(d, alo, bhi, idesc, 1u);
          }
          umma_commit(smem_u32(mma_bar));
        }
        __syncwarp();
        if (tid == 0) {
          // entry base+t (row h0-1+t) is no longer needed: refill the ring
          int freed = base + t + 1;
          if (t == rows - 1) freed = base + rows + 2;
          issue_upto(freed + T3_SLOTS);
        }
      }
      pn = n;
      ph = h0 + t;
      pw0 = w0;
      ++tile;
    }
    base += rows + 2;
  }
  if (tile > 0) epilogue(tile - 1);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, T3_TMEM);
}

// ---------------------------------------------------------------- dW (CUDA cores)
// dW[k][c][r][s] = sum_{n,h,w} dY[n][k][h][w] * X[n][c][h+r-1][w+s-1].
// Block = (image, 8-row chunk); warp w = input channel c, lane = a column
// pair; 72 fp32 accumulators (8 k x 9 taps) per thread, reduced across the warp
// by shuffles, written as the block's partial; a second kernel sums the
// partials in a fixed order in fp64.
constexpr int DW_ROWS = 8;

template <int K>
__global__ void __launch_bounds__(256) conv3x3_c8_dw_partial(int N, int H, int W,
                                                             const float* __restrict__ x,
                                                             const float* __restrict__ g,
                                                             float* __restrict__ part) {
  const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunks = (H + DW_ROWS - 1) / DW_ROWS;
  const int n = blockIdx.x / chunks, h0 = (blockIdx.x % chunks) * DW_ROWS;
  const float* xc = x + ((int64_t)n * T3_C + c) * H * W;
  const float* gn = g + (int64_t)n * K * H * W;
  float acc[K][9];
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int t = 0; t < 9; ++t) acc[k][t] = 0.f;
  for (int h = h0; h < min(H, h0 + DW_ROWS); ++h) {
    for (int w = 2 * lane; w < W; w += 64) {
      // x[c][h+r-1][w-1 .. w+2] (zero outside the image)
      float xv[3][4];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const int ih = h + r - 1;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int iw = w - 1 + j;
          xv[r][j] = (ih >= 0 && ih < H && iw >= 0 && iw < W) ? __ldg(xc + (int64_t)ih * W + iw)
                                                              : 0.f;
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const float* gk = gn + ((int64_t)k * H + h) * W + w;
        const float g0 = __ldg(gk);
        const float g1 = (w + 1 < W) ? __ldg(gk + 1) : 0.f;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int s = 0; s < 3; ++s)
            acc[k][r * 3 + s] = fmaf(g1, xv[r][s + 1], fmaf(g0, xv[r][s], acc[k][r * 3 + s]));
      }
    }
  }
  // reduce across the warp (fixed order), lane 0 writes the block partial
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      float v = acc[k][t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) part[(size_t)blockIdx.x * (K * T3_C * 9) + (k * T3_C + c) * 9 + t] = v;
    }
}

__global__ void dw_partials_sum(const float* __restrict__ part, int blocks, int outs,
                                float* __restrict__ dw) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= outs) return;
  double s = 0.0;
  for (int b = 0; b < blocks; ++b) s += (double)part[(size_t)b * outs + o];
  dw[o] = (float)s;
}

}  // namespace

bool conv3x3_tf32_applies(const ConvDims& d, int layout, int wlayout, int pass) {
  if (layout != MS_NCHW || wlayout != MS_NCHW) return false;
  if (d.r != 3 || d.s != 3 || d.sh != 1 || d.sw != 1 || d.ph != 1 || d.pw != 1) return false;
  static const bool off = [] {
    const char* e = getenv("MS_FP32_CONV");
    return e && e[0] == 's';  // "simt": the CUDA-core kernels
  }();
  if (off) return false;
  // fwd: C = 8 inputs, K <= 16 outputs; dX: the roles swap
  const int cin = pass == MS_CONV_DX ? d.k : d.c, cout = pass == MS_CONV_DX ? d.c : d.k;
  if (pass == MS_CONV_DW) return d.c == 8 && (d.k == 8);
  return cin == T3_C && cout >= 1 && cout <= T3_N && d.w % 4 == 0;
}

size_t conv3x3_c8_dw_workspace(const ConvDims& d) {
  const int chunks = (d.h + DW_ROWS - 1) / DW_ROWS;
  return sizeof(float) * (size_t)d.n * chunks * d.k * T3_C * 9;
}

// fwd (x, w -> y) or dX (a = dY, b = W -> out = dX) on the tensor cores
ms_status conv3x3_tf32(int pass, const ConvDims& d, const void* a, const void* b, void* out,
                       cudaStream_t st) {
  const bool dx = pass == MS_CONV_DX;
  // the conv actually computed: input a [N][8][H][W] -> out [N][K][H][W]
  const int H = dx ? d.oh : d.h, W = dx ? d.ow : d.w;
  const int K = dx ? d.c : d.k;
  CUtensorMap tx;
  const uint64_t dims[3] = {(uint64_t)W, (uint64_t)H, (uint64_t)d.n * T3_C};
  const uint64_t str[2] = {(uint64_t)W * 4, (uint64_t)W * H * 4};
  const uint32_t box[3] = {T3_LW, 1, T3_C};
  MS_TRY(make_tmap_nd(&tx, MS_F32, a, 3, dims, str, box, 0));
  T3Args args;
  args.N = d.n;
  args.H = H;
  args.W = W;
  args.K = K;
  args.segs = (W + T3_M - 1) / T3_M;
  args.chunks = (H + T3_R - 1) / T3_R;
  args.units = d.n * args.chunks * args.segs;
  args.w = static_cast<const float*>(b);
  args.flip = dx ? 1 : 0;
  args.y = static_cast<float*>(out);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv3x3_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         T3_SMEM);
    attr = true;
  }
  int grid = 2 * num_sms();
  if (grid > args.units) grid = args.units;
  conv3x3_tf32_kernel<<<grid, T3_THREADS, T3_SMEM, st>>>(tx, args);
  count_launch(1, KF_UMMA);
  return launch_status("conv3x3_tf32_kernel");
}

ms_status conv3x3_c8_dw(const ConvDims& d, const void* x, const void* g, void* dw, void* ws,
                        size_t ws_bytes, cudaStream_t st) {
  MS_CHECK_ARG(ws && ws_bytes >= conv3x3_c8_dw_workspace(d), MS_ERR_WORKSPACE,
               "conv3x3 c8 dW workspace too small");
  const int chunks = (d.h + DW_ROWS - 1) / DW_ROWS;
  const int blocks = d.n * chunks;
  float* part = static_cast<float*>(ws);
  conv3x3_c8_dw_partial<8><<<blocks, 256, 0, st>>>(d.n, d.h, d.w, (const float*)x,
                                                   (const float*)g, part);
  const int outs = d.k * T3_C * 9;
  dw_partials_sum<<<(outs + 127) / 128, 128, 0, st>>>(part, blocks, outs, (float*)dw);
  count_launch(2, KF_SIMT);
  return launch_status("conv3x3_c8_dw");
}

}  // namespace ms
