// float32 3x3 / stride 1 / pad 1 convolution with 8 input and <= 8 output
// channels on the tcgen05 tensor cores (kind::tf32) at float32 accuracy: the
// Fig. 1 network (8 -> 8 channels, NCHW; reference
// numpy_impl.py:12-38).
//
// 3xTF32: every operand is split exactly into hi = x with the low 13 mantissa
// bits cleared (representable in tf32) and lo = x - hi (exact in fp32), and
//   x * w  ~=  hi_x * hi_w + hi_x * lo_w + lo_x * hi_w
// (the dropped lo*lo term and the tf32 rounding of lo are ~2^-21 relative).
//
// GEMM view.  A work unit is a strip of R = 8 output rows x 128 output pixels
// of one image.  The CTA walks the strip's R + 2 input rows once.  For input
// row i and kernel column s the A operand is the 128 x 8 tile
//   A_s[p][c] = x[c][i][w0 + p + s - 1]
// read straight from shared memory: rows are staged as [hi|lo][c/4][px][c%4]
// (16 bytes per pixel per half), so the three column shifts s are three
// descriptor start addresses 16 bytes apart -- nothing is replicated.  One MMA
// (M = 128, N = 48, K = 8) multiplies A_s by the weights of all three kernel
// rows r at once, [W_hi(r,s) | W_lo(r,s)] for r = 0..2, and writes the three
// 16-column groups of the output rows o = i+1, i, i-1 (r = i - o + 1).  The
// accumulators are laid out in TENSOR MEMORY so that consecutive input rows
// hit overlapping groups: output row o lives at column 16*(h0 + R + 1 - o) of
// the strip's region, so the MMA for input row i starts at the group of o =
// i + 1.  Output row o is complete after input row o + 1 -- a "rolling"
// accumulation with 6 MMAs (3 s x {A_hi, A_lo}) per input row and the A tile
// fetched from shared memory 6 times per 128 pixels (24 KB, vs 9 taps x 3
// products x 4 KB for one MMA per tap).  Group layout: columns 0-7 collect
// A_hi*W_hi + A_lo*W_hi, columns 8-15 A_hi*W_lo; y = sum of the two halves.
//
// Warp roles (14 warps, one CTA per SM):
//   warp 0     TMA producer: two [8 ch][5 rows][136 px] boxes per unit, 7 in flight (3-D box of the NCHW
//              tensor from w0 - 4, 16-byte aligned; zero fill = the padding)
//   warp 1     TMEM allocator + MMA issuer
//   warps 2-9  converters: raw row -> hi / lo planes in the MMA's K-major layout
//              (one (pixel, 4-channel half) task per thread and row)
//   warps 10-13 epilogue: tcgen05.ld of a finished output row -> y (coalesced
//              128-byte rows per channel); the region is zeroed after its strip
// Two TMEM regions (2 x 192 of the 512 columns) alternate between strips, so
// the epilogue of one strip overlaps the MMAs of the next.
//
// dX of the same conv is this kernel on dY with the transposed, flipped weights
// W'[c][k][2-r][2-s] (numpy_impl.py:27-38).  dW is a CUDA-core reduction with
// per-block fp32 partials reduced in a fixed order in fp64 (deterministic,
// numpy_impl.py:41-51).
#include <cstdlib>

#include "misc.cuh"

namespace ms {
namespace {

constexpr int T3_M = 128;              // output pixels per unit (one A tile)
constexpr int T3_C = 8;                // input channels = one tf32 K step
constexpr int T3_KO = 8;               // output channels (<= 8)
constexpr int T3_R = 8;                // output rows per unit (strip)
constexpr int T3_LW = 136;             // staged pixels per input row (w0-4 .. w0+131): the
                                       // innermost TMA coordinate must stay 16-byte aligned
constexpr int T3_ROWS = T3_R + 2;            // input rows per unit
constexpr int T3_HROWS = T3_ROWS / 2;        // rows per TMA box (half a unit)
constexpr int T3_RAWB = T3_C * T3_HROWS * T3_LW * 4;  // raw box [8 ch][5 rows][136 px] fp32
constexpr int T3_HALFB = T3_LW * 16;          // one 4-channel plane [136 px][4] (2176 B)
constexpr int T3_PARTB = 2 * T3_HALFB;        // hi (or lo) of a row (4352 B)
constexpr int T3_SPLB = 2 * T3_PARTB;         // hi + lo (8704 B)
constexpr int T3_RAWS = 6;                    // raw ring of half-unit boxes (152 KB in flight
                                              // per SM).  TMA cost is per box row: multi-row
                                              // boxes stream ~3x faster than [136][1][8] rows
constexpr int T3_SLOTS = 8;                   // split ring (rows, power of 2)
constexpr int T3_N = 48;                      // MMA N: 3 kernel rows x 16-column groups
constexpr int T3_BTILE = T3_N * T3_C * 4;     // one B tile (1536 B)
constexpr int T3_REGION = 16 * (T3_R + 4);    // TMEM columns per strip region (192)
constexpr int T3_ACCQ = 2;                    // acc-full barriers: one per strip region
constexpr int T3_CONV_WARPS = 8;              // converter warps: T3_GROUPS groups of 2
constexpr int T3_GROUPS = T3_CONV_WARPS / 2;  // (power of 2)
constexpr int T3_EPI_W0 = 2 + T3_CONV_WARPS;   // first epilogue warp
constexpr int T3_THREADS = 32 * (T3_EPI_W0 + 4);
constexpr int T3_OFF_SPL = T3_RAWS * T3_RAWB;
constexpr int T3_OFF_B = T3_OFF_SPL + T3_SLOTS * T3_SPLB;
constexpr int T3_OFF_BAR = T3_OFF_B + 6 * T3_BTILE;
// barriers: raw_full, raw_empty, spl_full, spl_empty [SLOTS]; acc_full [ACCQ];
// region_free [2]; then the TMEM address holder
constexpr int T3_PAIRS = T3_SLOTS / 2;         // split slots are released in pairs (one
                                              // tcgen05.commit per two rows)
static_assert(T3_SLOTS % 2 == 0, "pairs");
constexpr int T3_NBAR = 2 * T3_RAWS + T3_SLOTS + T3_PAIRS + T3_ACCQ + 2;
constexpr int T3_SMEM_USED = T3_OFF_BAR + T3_NBAR * 8 + 16;
// more than half the SM's shared memory: exactly one CTA (and one 512-column
// TMEM allocation) per SM
constexpr int T3_SMEM = 220 * 1024;
static_assert(T3_SMEM_USED <= T3_SMEM, "smem");

struct T3Args {
  int N, H, W, K;        // K = real output channels (<= 8)
  int segs, chunks;      // 128-pixel segments per row, R-row strips per image
  int units;             // N * chunks * segs
  const float* w;        // weights [K][8][3][3] (fwd) or [8][K][3][3] (flip)
  int flip;
  float* y;              // [N][K][H][W]
  int dbg;               // profiling (MS_TF32_DBG): 1 no conversion, 2 no MMAs, 4 no stores,
                         // 8 TMA stream only (converters release boxes; MMA / epilogue idle),
                         // 32 no proxy fence
};

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* tmap, uint32_t bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tmem_st_zero_x32(uint32_t taddr) {
  const uint32_t z = 0u;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
      "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(
          taddr),
      "r"(z)
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
// D[tmem] (+)= A[smem] * B[smem], kind::tf32
__device__ __forceinline__ void umma_tf32_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// mbarrier wait without a suspend-time hint: the hand-offs of this pipeline
// (TMA -> converters -> MMA -> epilogue) are short and latency-bound, so waiters
// poll instead of sleeping (bounded, like mbar_wait)
__device__ __forceinline__ void mbar_arrive_cnt(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void spin_wait(uint32_t bar, uint32_t parity) {
  uint32_t spins = 0;
  while (true) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t"
        "}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    if (ok) return;
    if (++spins > MS_WATCHDOG_SPINS) {
      printf("memsave_b200: conv3x3_tf32 mbarrier watchdog (block %d thread %d)\n", blockIdx.x,
             threadIdx.x);
      __trap();
    }
  }
}

__device__ __forceinline__ float tf32_hi(float v) {
  return __uint_as_float(__float_as_uint(v) & 0xffffe000u);
}

// unit u -> (image, strip, segment)
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

__global__ void __launch_bounds__(T3_THREADS, 1)
    conv3x3_tf32_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ T3Args a) {
  // (no manual re-alignment: the operands need 16-byte alignment only, and a
  // pointer derived from the __shared__ symbol keeps ld/st.shared addressing)
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* raw = smem;
  uint8_t* spl = smem + T3_OFF_SPL;
  uint8_t* sB = smem + T3_OFF_B;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T3_OFF_BAR);
  uint64_t* raw_full = bars;
  uint64_t* raw_empty = bars + T3_RAWS;
  uint64_t* spl_full = bars + 2 * T3_RAWS;
  uint64_t* spl_empty = spl_full + T3_SLOTS;  // [PAIRS]
  uint64_t* acc_full = spl_empty + T3_PAIRS;
  uint64_t* region_free = acc_full + T3_ACCQ;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(region_free + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- B tiles.  Tile (s, part): part 0 multiplies A_hi, part 1 A_lo.  Row nn of
  // the N = 48 rows: group r = nn / 16, j = nn % 16: j < 8 -> W_hi(r, s)[k = j],
  // j >= 8 -> (part 0) W_lo(r, s)[k = j - 8] / (part 1) 0.  K-major tf32, no
  // swizzle: core matrices of 8 rows x 16 B, SBO = 128 B, LBO = 48 * 16 B.
  // (zero the tiles, then one weight per thread, scattered to its 3 slots: a
  // single round of independent global loads instead of a dependent chain)
  for (int i = tid; i < 6 * T3_BTILE / 16; i += T3_THREADS)
    reinterpret_cast<float4*>(sB)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  const int nw = a.K * T3_C * 9;  // <= 576 < 2 x T3_THREADS
  float wv[2] = {0.f, 0.f};
#pragma unroll
  for (int q = 0; q < 2; ++q)
    if (tid + q * T3_THREADS < nw) wv[q] = __ldg(a.w + tid + q * T3_THREADS);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int i = tid + q * T3_THREADS;
    if (i >= nw) break;
    int k, c, t;
    if (a.flip) {  // w = W[c][k][r'][s'] with tap t = 8 - (r' * 3 + s')
      c = i / (a.K * 9);
      k = (i / 9) % a.K;
      t = 8 - i % 9;
    } else {       // w = W[k][c][r][s]
      k = i / (T3_C * 9);
      c = (i / 9) % T3_C;
      t = i % 9;
    }
    const int r = t / 3, s = t % 3;
    const float hi = tf32_hi(wv[q]), lo = wv[q] - hi;
    auto put = [&](int tile, int nn, float v) {
      const int off = (c >> 2) * (T3_N * 16) + (nn >> 3) * 128 + (nn & 7) * 16 + (c & 3) * 4;
      *reinterpret_cast<float*>(sB + tile * T3_BTILE + off) = v;
    };
    put(2 * s, r * 16 + k, hi);          // A_hi x W_hi
    put(2 * s, r * 16 + 8 + k, lo);      // A_hi x W_lo
    put(2 * s + 1, r * 16 + k, hi);      // A_lo x W_hi
  }
  if (tid == 0) {
    for (int i = 0; i < T3_RAWS; ++i) {
      mbar_init(smem_u32(&raw_full[i]), 1);
      mbar_init(smem_u32(&raw_empty[i]), 2 * T3_HROWS);  // 2 warps x rows per box
    }
    for (int i = 0; i < T3_SLOTS; ++i) mbar_init(smem_u32(&spl_full[i]), 2);  // the row's 2 warps
    for (int i = 0; i < T3_PAIRS; ++i) mbar_init(smem_u32(&spl_empty[i]), 1);
    for (int i = 0; i < T3_ACCQ; ++i) mbar_init(smem_u32(&acc_full[i]), 1);
    mbar_init(smem_u32(&region_free[0]), 4);
    mbar_init(smem_u32(&region_free[1]), 4);
    fence_mbar_init();
    tma_prefetch_desc(&tx);
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_holder), 512);
  fence_proxy_async_smem();  // the B tiles are read by the tensor core (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ============================ TMA producer ============================
    int hs = 0;  // half-unit boxes issued
    for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
      int n, h0, rows, w0;
      unit_coords(a, u, n, h0, rows, w0);
      for (int half = 0; half < 2; ++half, ++hs) {
        const int slot = hs % T3_RAWS;
        spin_wait(smem_u32(&raw_empty[slot]), ((hs / T3_RAWS) & 1) ^ 1);
        if (elect_one()) {
          const uint32_t bar = smem_u32(&raw_full[slot]);
          mbar_arrive_expect_tx(bar, T3_RAWB);
          tma_load_3d(smem_u32(raw + slot * T3_RAWB), &tx, bar, w0 - 4, h0 - 1 + half * T3_HROWS,
                      n * T3_C);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    if (a.dbg & 8) goto done;
    const uint32_t idesc = make_idesc_f16(2, T3_M, T3_N, 0, 0);  // tf32 x tf32 -> f32
    const uint32_t spl_u = smem_u32(spl), b_u = smem_u32(sB);
    int e = 0, lu = 0;
    for (int u = blockIdx.x; u < a.units; u += gridDim.x, ++lu) {
      int n, h0, rows, w0;
      unit_coords(a, u, n, h0, rows, w0);
      const int reg = lu & 1;
      // the region was zeroed by the epilogue (initially, or after strip lu - 2)
      spin_wait(smem_u32(&region_free[reg]), (lu >> 1) & 1);
      tc_fence_after();
      const uint32_t region = tmem + reg * 256;
      for (int j = 0; j < rows + 2; ++j, ++e) {
        const int slot = e % T3_SLOTS;
        spin_wait(smem_u32(&spl_full[slot]), (e / T3_SLOTS) & 1);
        tc_fence_after();
        // input row i = h0 - 1 + j feeds output rows i + 1, i, i - 1 = the three
        // groups starting at that of o = i + 1
        const uint32_t d = region + 16u * static_cast<uint32_t>(T3_R + 1 - j);
        if (elect_one()) {
#pragma unroll
          for (int s = 0; s < 3 && !(a.dbg & 2); ++s) {
#pragma unroll
            for (int part = 0; part < 2; ++part) {
              const uint32_t sa = spl_u + slot * T3_SPLB + part * T3_PARTB + (3 + s) * 16;
              const uint64_t ad = make_smem_desc(sa, T3_HALFB, 128, LAYOUT_SWIZZLE_NONE);
              const uint64_t bd = make_smem_desc(b_u + (2 * s + part) * T3_BTILE, T3_N * 16, 128,
                                                 LAYOUT_SWIZZLE_NONE);
              umma_tf32_ss(d, ad, bd, idesc, 1u);
            }
          }
          // every second row: free the pair of staged rows; after the strip's
          // last row: its accumulators are complete
          if (e & 1) umma_commit(smem_u32(&spl_empty[(e >> 1) % T3_PAIRS]));
          if (j == rows + 1) umma_commit(smem_u32(&acc_full[reg]));
        }
        __syncwarp();
      }
    }
  } else if (warp < T3_EPI_W0) {
    // ============================ converters ============================
    if (a.dbg & 64) {  // profiling: one thread consumes the boxes (TMA stream only)
      if (warp == 2 && lane == 0) {
        int hs = 0;
        for (int u = blockIdx.x; u < a.units; u += gridDim.x)
          for (int half = 0; half < 2; ++half, ++hs) {
            spin_wait(smem_u32(&raw_full[hs % T3_RAWS]), (hs / T3_RAWS) & 1);
            mbar_arrive_cnt(smem_u32(&raw_empty[hs % T3_RAWS]), 2 * T3_HROWS);
          }
      }
      goto done;
    }
    // Rows are converted by T3_GROUPS groups of 2 warps, group g taking rows e
    // with e % T3_GROUPS == g: a single group walking every row made the row
    // loop's serial latency (~250-450 cycles per row, one warp's dependent
    // chain) the kernel's critical path (MS_TF32_DBG=256 cycle counters).
    // The MMA reads staged pixels 3 .. 132 (A rows p + s + 3): 130 pixels x 2
    // channel halves = 260 tasks over the group's 64 threads.
    constexpr int GT = 64, NPX = T3_M + 2, TASKS = 2 * NPX;
    const int grp = (warp - 2) >> 1;
    const int gt = tid - 64 - grp * GT;
    int e0 = 0, lu = 0;  // first row of the unit, unit counter
    for (int u = blockIdx.x; u < a.units; u += gridDim.x, ++lu) {
      int n, h0, rows, w0;
      unit_coords(a, u, n, h0, rows, w0);
      const int nrow = rows + 2;
      for (int j = (grp - e0) & (T3_GROUPS - 1); j < nrow; j += T3_GROUPS) {
        const int e = e0 + j;
        const int half = j >= T3_HROWS ? 1 : 0, jj = j - half * T3_HROWS;
        const int hs = 2 * lu + half, rs = hs % T3_RAWS;
        const int slot = e & (T3_SLOTS - 1), pair = (e >> 1) & (T3_PAIRS - 1);
        spin_wait(smem_u32(&raw_full[rs]), (hs / T3_RAWS) & 1);
        if (!(a.dbg & 8)) spin_wait(smem_u32(&spl_empty[pair]), ((e / T3_SLOTS) & 1) ^ 1);
        const float* rr = reinterpret_cast<const float*>(raw + rs * T3_RAWB) + jj * T3_LW;
        uint8_t* ss = spl + slot * T3_SPLB;
        if (!(a.dbg & 1)) {
#pragma unroll
          for (int q = 0; q < (TASKS + GT - 1) / GT; ++q) {
            const int t = gt + q * GT;
            if (t < TASKS) {
              const int hf = t >= NPX ? 1 : 0;
              const int px = 3 + t - hf * NPX;
              float hv[4], lv[4];
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const float v = rr[(hf * 4 + c) * T3_HROWS * T3_LW + px];
                hv[c] = tf32_hi(v);
                lv[c] = v - hv[c];
              }
              *reinterpret_cast<float4*>(ss + hf * T3_HALFB + px * 16) =
                  make_float4(hv[0], hv[1], hv[2], hv[3]);
              *reinterpret_cast<float4*>(ss + T3_PARTB + hf * T3_HALFB + px * 16) =
                  make_float4(lv[0], lv[1], lv[2], lv[3]);
            }
          }
        }
        if (!(a.dbg & 32)) fence_proxy_async_smem();  // generic-proxy writes -> tensor-core reads
        __syncwarp();
        if (lane == 0) {
          if (!(a.dbg & 128)) mbar_arrive(smem_u32(&spl_full[slot]));
          // raw_empty counts 2 warps x T3_HROWS rows per box; the box's last row
          // also arrives for the rows a short strip does not have
          const bool last = jj == T3_HROWS - 1 || j == nrow - 1;
          mbar_arrive_cnt(smem_u32(&raw_empty[rs]), last ? T3_HROWS - jj : 1);
          if (j == nrow - 1 && nrow <= T3_HROWS) {  // the unread second box of a short strip
            const int hs2 = 2 * lu + 1, rs2 = hs2 % T3_RAWS;
            spin_wait(smem_u32(&raw_full[rs2]), (hs2 / T3_RAWS) & 1);
            mbar_arrive_cnt(smem_u32(&raw_empty[rs2]), T3_HROWS);
          }
        }
      }
      e0 += nrow;
    }
  } else {
    // ============================ epilogue ============================
    if (a.dbg & 8) goto done;
    const uint32_t quarter = warp & 3;  // TMEM lane quarter this warp may access
    const uint32_t lane_base = (quarter * 32u) << 16;
    const int p = static_cast<int>(quarter) * 32 + lane;  // pixel (TMEM lane / A row)
    // zero both regions (TMEM is undefined at allocation), then release them
    for (int c = 0; c < 2 * 256; c += 32) tmem_st_zero_x32(tmem + lane_base + c);
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(smem_u32(&region_free[0]));
      mbar_arrive(smem_u32(&region_free[1]));
    }
    int lu = 0;
    for (int u = blockIdx.x; u < a.units; u += gridDim.x, ++lu) {
      int n, h0, rows, w0;
      unit_coords(a, u, n, h0, rows, w0);
      const int reg = lu & 1;
      const uint32_t region = tmem + lane_base + reg * 256;
      const int w = w0 + p;
      spin_wait(smem_u32(&acc_full[reg]), (lu >> 1) & 1);  // the strip's rows are complete
      for (int q = 0; q < rows; ++q) {
        tc_fence_after();
        uint32_t r[16];
        tmem_ld_x16(region + 16u * static_cast<uint32_t>(T3_R + 1 - q), r);
        tmem_ld_wait();
        if (w < a.W && !(a.dbg & 4)) {
          float* yo = a.y + ((static_cast<int64_t>(n) * a.K * a.H + h0 + q) * a.W + w);
#pragma unroll
          for (int k = 0; k < T3_KO; ++k)
            if (k < a.K)
              yo[static_cast<int64_t>(k) * a.H * a.W] =
                  __uint_as_float(r[k]) + __uint_as_float(r[8 + k]);
        }
      }
      // strip drained: zero the region for strip lu + 2 and release it
      for (int c = 0; c < T3_REGION; c += 32) tmem_st_zero_x32(region + c);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&region_free[reg]));
    }
  }
done:
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- dW (CUDA cores)
// dW[k][c][r][s] = sum_{n,h,w} dY[n][k][h][w] * X[n][c][h+r-1][w+s-1].
// Persistent blocks (2 per SM) walk units of (image, 4-row strip, 256-pixel
// segment).  A unit's 6 input rows and 4 dY rows (8 channels each) are staged in
// shared memory with a skewed pitch (one pad word per 8 pixels), so lane l's run
// of 8 consecutive pixels [8l, 8l + 8) hits 32 distinct banks.  Warp = input
// channel c; each thread keeps the 72 (8 k x 9 taps) sums of its pixels in
// registers across all of the block's units, sliding a 3 x 3 window of X along
// its run (per pixel: 3 + 8 shared loads for 72 FMAs).  The block's sums are
// reduced across the warp by shuffles and written as its partial; a second
// kernel adds the partials in a fixed order in fp64 (deterministic for a given
// grid).
constexpr int DW_L = 8;                    // pixels per lane
constexpr int DW_SEG = 32 * DW_L;          // pixels per segment
constexpr int DW_RB = 4;                   // dY rows per unit
constexpr int DW_XN = DW_SEG + 2;          // staged X pixels (w0-1 .. w0+256)
constexpr int DW_XP = DW_XN + DW_XN / 8 + 1;   // skewed pitch (words)
constexpr int DW_GP = DW_SEG + DW_SEG / 8;     // skewed pitch of a dY row
constexpr int DW_SMEM = ((DW_RB + 2) * T3_C * DW_XP + DW_RB * T3_C * DW_GP) * 4;
constexpr int DW_BLOCKS_PER_SM = 2;

__device__ __forceinline__ int dw_skew(int p) { return p + (p >> 3); }

template <int K>
__global__ void __launch_bounds__(256, DW_BLOCKS_PER_SM)
    conv3x3_c8_dw_partial(int N, int H, int W, const float* __restrict__ x,
                          const float* __restrict__ g, float* __restrict__ part) {
  extern __shared__ float dsm[];
  float* sx = dsm;                                  // [(row * 8 + c) * XP + skew(p)]
  float* sg = dsm + (DW_RB + 2) * T3_C * DW_XP;     // [(row * 8 + k) * GP + skew(p)]
  const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int strips = (H + DW_RB - 1) / DW_RB, segs = (W + DW_SEG - 1) / DW_SEG;
  const int units = N * strips * segs;
  const int64_t plane = (int64_t)H * W;
  float acc[K][9];
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int t = 0; t < 9; ++t) acc[k][t] = 0.f;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int seg = u % segs, rest = u / segs;
    const int strip = rest % strips, n = rest / strips;
    const int h0 = strip * DW_RB, w0 = seg * DW_SEG;
    __syncthreads();  // the previous unit's reads are done
    // stage X rows h0-1 .. h0+RB (zero outside the image): warp = (row, channel)
    for (int rc = c; rc < (DW_RB + 2) * T3_C; rc += 8) {
      const int row = rc / T3_C, ch = rc % T3_C, ih = h0 - 1 + row;
      const bool rin = ih >= 0 && ih < H;
      const float* src = x + (n * T3_C + ch) * plane + (int64_t)(rin ? ih : 0) * W;
      float* dst = sx + rc * DW_XP;
      for (int p = lane; p < DW_XN; p += 32) {
        const int iw = w0 - 1 + p;
        dst[dw_skew(p)] = (rin && iw >= 0 && iw < W) ? __ldg(src + iw) : 0.f;
      }
    }
    for (int rk = c; rk < DW_RB * K; rk += 8) {
      const int row = rk / K, k = rk % K, oh = h0 + row;
      const bool rin = oh < H;
      const float* src = g + (n * K + k) * plane + (int64_t)(rin ? oh : 0) * W;
      float* dst = sg + rk * DW_GP;
      for (int p = lane; p < DW_SEG; p += 32) {
        const int iw = w0 + p;
        dst[dw_skew(p)] = (rin && iw < W) ? __ldg(src + iw) : 0.f;
      }
    }
    __syncthreads();
    const int p0 = lane * DW_L;
#pragma unroll 1
    for (int rr = 0; rr < DW_RB; ++rr) {
      const float* xr = sx + (rr * T3_C + c) * DW_XP;  // row rr of the 3 = input row h-1
      const float* gr = sg + rr * K * DW_GP;
      float xw[3][3];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        xw[r][0] = xr[r * T3_C * DW_XP + dw_skew(p0)];
        xw[r][1] = xr[r * T3_C * DW_XP + dw_skew(p0 + 1)];
      }
#pragma unroll
      for (int j = 0; j < DW_L; ++j) {
#pragma unroll
        for (int r = 0; r < 3; ++r) xw[r][2] = xr[r * T3_C * DW_XP + dw_skew(p0 + j + 2)];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const float gv = gr[k * DW_GP + dw_skew(p0 + j)];
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int s = 0; s < 3; ++s) acc[k][r * 3 + s] = fmaf(gv, xw[r][s], acc[k][r * 3 + s]);
        }
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          xw[r][0] = xw[r][1];
          xw[r][1] = xw[r][2];
        }
      }
    }
  }
  // reduce across the warp, lane 0 writes the block partial
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

// dW for rows of at most 256 pixels (the Fig. 1 shape), staged by TMA and
// double-buffered: one persistent CTA of 16 warps per SM walks units of (image,
// 4-row strip).  A unit's X rows h0-1 .. h0+4 and dY rows h0 .. h0+3 (8
// channels, whole rows, zero fill outside the image) arrive as two boxes while
// the previous unit is reduced.  Warp = (input channel c, pixel half); lane l
// takes pixels l + 32 j (conflict-free shared loads, no padding), 72 fp32
// accumulators (8 k x 9 taps) per thread; two output rows are processed
// together so each X value loaded serves both (12 + 16 shared loads per 144
// FMAs).  Each warp's sums are reduced by shuffles into its own partial slot.
constexpr int DW2_RB = 4;                       // dY rows per unit
constexpr int DW2_W = 256;                      // staged row width (max W)
constexpr int DW2_XB = T3_C * (DW2_RB + 2) * DW2_W * 4;   // X box bytes (48 KB)
constexpr int DW2_GB = T3_C * DW2_RB * DW2_W * 4;         // dY box bytes (32 KB)
constexpr int DW2_STAGE = DW2_XB + DW2_GB;
constexpr int DW2_SMEM = 2 * DW2_STAGE + 64;
constexpr int DW2_THREADS = 512;

template <int K>
__global__ void __launch_bounds__(DW2_THREADS, 1)
    conv3x3_c8_dw_tma(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tg,
                      int N, int H, int W, float* __restrict__ part) {
  extern __shared__ __align__(1024) uint8_t dsm2[];
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm2 + 2 * DW2_STAGE);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = warp & 7, jh = warp >> 3;
  const int strips = (H + DW2_RB - 1) / DW2_RB;
  const int units = N * strips;
  if (tid == 0) {
    mbar_init(smem_u32(&full[0]), 1);
    mbar_init(smem_u32(&full[1]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int u, int stg) {
    const int n = u / strips, h0 = (u % strips) * DW2_RB;
    const uint32_t bar = smem_u32(&full[stg]);
    uint8_t* base = dsm2 + stg * DW2_STAGE;
    mbar_arrive_expect_tx(bar, DW2_STAGE);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(base)),
        "l"(reinterpret_cast<uint64_t>(&tx)), "r"(bar), "r"(0), "r"(h0 - 1), "r"(n * T3_C)
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(base + DW2_XB)),
        "l"(reinterpret_cast<uint64_t>(&tg)), "r"(bar), "r"(0), "r"(h0), "r"(n * K)
        : "memory");
  };
  if (tid == 0) {
    if ((int)blockIdx.x < units) issue(blockIdx.x, 0);
    if ((int)(blockIdx.x + gridDim.x) < units) issue(blockIdx.x + gridDim.x, 1);
  }
  float acc[K][9];
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int t = 0; t < 9; ++t) acc[k][t] = 0.f;
  int it = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x, ++it) {
    const int stg = it & 1;
    spin_wait(smem_u32(&full[stg]), (it >> 1) & 1);
    const float* xs = reinterpret_cast<const float*>(dsm2 + stg * DW2_STAGE);  // [c][6][256]
    const float* gs = reinterpret_cast<const float*>(dsm2 + stg * DW2_STAGE + DW2_XB);  // [k][4][256]
#pragma unroll 1
    for (int rp = 0; rp < DW2_RB; rp += 2) {
#pragma unroll 1
      for (int j = 4 * jh; j < 4 * jh + 4; ++j) {
        const int px = lane + 32 * j;
        if (px >= W) break;  // warp-uniform (W is a multiple of 32 or the tail is idle)
        float xv[4][3];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float* xr = xs + (c * (DW2_RB + 2) + rp + q) * DW2_W;
          xv[q][0] = px > 0 ? xr[px - 1] : 0.f;
          xv[q][1] = xr[px];
          xv[q][2] = px + 1 < DW2_W ? xr[px + 1] : 0.f;
        }
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const float gv = gs[(k * DW2_RB + rp + rr) * DW2_W + px];
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
              for (int s = 0; s < 3; ++s)
                acc[k][r * 3 + s] = fmaf(gv, xv[rr + r][s], acc[k][r * 3 + s]);
          }
        }
      }
    }
    __syncthreads();  // every warp is done with this stage
    if (tid == 0 && u + 2 * (int)gridDim.x < units) issue(u + 2 * gridDim.x, stg);
  }
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      float v = acc[k][t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0)
        part[((size_t)blockIdx.x * 2 + jh) * (K * T3_C * 9) + (k * T3_C + c) * 9 + t] = v;
    }
}

// out[o] = sum over partial slots b of part[b][o], in a fixed order: warp per
// output, lane l adds slots l, l + 32, ... in fp64, then a fixed shuffle tree
__global__ void dw_partials_sum(const float* __restrict__ part, int blocks, int outs,
                                float* __restrict__ dw) {
  const int o = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (o >= outs) return;
  double s = 0.0;
  for (int b = lane; b < blocks; b += 32) s += (double)part[(size_t)b * outs + o];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) dw[o] = (float)s;
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
  return cin == T3_C && cout >= 1 && cout <= T3_KO && d.w % 4 == 0;
}

static bool dw_tma_ok(const ConvDims& d) { return d.w <= DW2_W && d.w % 4 == 0; }

// partial slots written by the dW kernel (the fixed-order fp64 sum reads them all)
static int dw_slots(const ConvDims& d) {
  if (dw_tma_ok(d)) {
    const int units = d.n * ((d.h + DW2_RB - 1) / DW2_RB);
    return 2 * (units < num_sms() ? units : num_sms());
  }
  const int units = d.n * ((d.h + DW_RB - 1) / DW_RB) * ((d.w + DW_SEG - 1) / DW_SEG);
  const int g = DW_BLOCKS_PER_SM * num_sms();
  return units < g ? units : g;
}

size_t conv3x3_c8_dw_workspace(const ConvDims& d) {
  return sizeof(float) * (size_t)dw_slots(d) * d.k * T3_C * 9;
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
  const uint32_t box[3] = {T3_LW, T3_HROWS, T3_C};
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
  static const int env_dbg = [] {
    const char* e = getenv("MS_TF32_DBG");
    return e ? atoi(e) : 0;
  }();
  args.dbg = env_dbg;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv3x3_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         T3_SMEM);
    attr = true;
  }
  int grid = num_sms();
  if (grid > args.units) grid = args.units;
  conv3x3_tf32_kernel<<<grid, T3_THREADS, T3_SMEM, st>>>(tx, args);
  count_launch(1, KF_UMMA);
  return launch_status("conv3x3_tf32_kernel");
}

ms_status conv3x3_c8_dw(const ConvDims& d, const void* x, const void* g, void* dw, void* ws,
                        size_t ws_bytes, cudaStream_t st) {
  MS_CHECK_ARG(ws && ws_bytes >= conv3x3_c8_dw_workspace(d), MS_ERR_WORKSPACE,
               "conv3x3 c8 dW workspace too small");
  const int slots = dw_slots(d);
  float* part = static_cast<float*>(ws);
  if (dw_tma_ok(d)) {
    CUtensorMap tx, tg;
    const uint64_t dims_x[3] = {(uint64_t)d.w, (uint64_t)d.h, (uint64_t)d.n * T3_C};
    const uint64_t dims_g[3] = {(uint64_t)d.w, (uint64_t)d.h, (uint64_t)d.n * d.k};
    const uint64_t str[2] = {(uint64_t)d.w * 4, (uint64_t)d.w * d.h * 4};
    const uint32_t box_x[3] = {DW2_W, DW2_RB + 2, T3_C}, box_g[3] = {DW2_W, DW2_RB, 8};
    MS_TRY(make_tmap_nd(&tx, MS_F32, x, 3, dims_x, str, box_x, 0));
    MS_TRY(make_tmap_nd(&tg, MS_F32, g, 3, dims_g, str, box_g, 0));
    static bool attr2 = false;
    if (!attr2) {
      cudaFuncSetAttribute(conv3x3_c8_dw_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           DW2_SMEM);
      attr2 = true;
    }
    conv3x3_c8_dw_tma<8><<<slots / 2, DW2_THREADS, DW2_SMEM, st>>>(tx, tg, d.n, d.h, d.w, part);
  } else {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(conv3x3_c8_dw_partial<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           DW_SMEM);
      attr = true;
    }
    conv3x3_c8_dw_partial<8><<<slots, 256, DW_SMEM, st>>>(d.n, d.h, d.w, (const float*)x,
                                                          (const float*)g, part);
  }
  const int outs = d.k * T3_C * 9;
  dw_partials_sum<<<(outs + 7) / 8, 256, 0, st>>>(part, slots, outs, (float*)dw);
  count_launch(2, KF_SIMT);
  return launch_status("conv3x3_c8_dw");
}

}  // namespace ms
