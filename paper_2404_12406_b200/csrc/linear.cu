// Fully-connected layer: Z = X·Wᵀ + b, dX = G·W, dW = Gᵀ·X,
// db = Σ G.  16-bit operands with 16-byte-aligned rows run on the tcgen05
// kernel (A/B K-major or MN-major straight from the row-major tensors, no
// transposes); float32 and unaligned shapes run on the SIMT kernel.
#include <cstdlib>

#include "misc.cuh"
#include "rng.cuh"

namespace ms {

namespace {

bool is16(int dt) { return dt == MS_BF16 || dt == MS_F16; }
bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

struct LinPlan {
  bool tc = false;
  bool tf32 = false;  // float32 on the tensor cores (3xTF32, LOAD_GEMM_3XTF32)
  int cl = 1;   // 2: B tile multicast across a CTA pair on adjacent M tiles
  int bn = 0;
  int splits = 1;
  int kb_per_split = 0;
  int m_blocks = 0, n_blocks = 0, k_blocks = 0;
  // last-wave K split (GemmArgs::tail_splits): tiles >= full_tiles run as
  // tail_splits slices of tail_kbps k-blocks; partials in ws, then finalize
  int full_tiles = 0, tail_splits = 0, tail_kbps = 0;
  size_t ws = 0;
};

// rows x cols output, contraction red; b_mn: B operand MN-major (BN >= 64).
// Tile shape from pick_tiles (single-CTA or CTA-pair); split-K when the output
// tiles cannot fill the GPU.
LinPlan plan_gemm(int64_t rows, int64_t cols, int64_t red, bool b_mn, bool allow_split) {
  LinPlan p;
  p.tc = true;
  p.m_blocks = (int)((rows + BM - 1) / BM);
  const int sms = num_sms();
  const TilePick tp = pick_tiles(p.m_blocks, cols, true, b_mn);
  p.bn = tp.bn;
  p.cl = tp.cl;
  p.n_blocks = (int)((cols + p.bn - 1) / p.bn);
  p.k_blocks = (int)((red + BK - 1) / BK);
  const int64_t tiles = (int64_t)((p.m_blocks + p.cl - 1) / p.cl) * p.n_blocks;
  const int64_t slots = p.cl == 2 ? pair_slots() : sms;
  p.splits = 1;
  if (allow_split && tiles * 2 <= slots && p.k_blocks >= 8) {
    // split-K into fp32 (red.add): as many slices as fit in ONE wave
    int64_t s = slots / tiles;
    const int64_t cap = p.k_blocks / 4;
    if (s > cap) s = cap;
    if (s < 1) s = 1;
    p.splits = (int)s;
  }
  p.kb_per_split = (p.k_blocks + p.splits - 1) / p.splits;
  p.splits = (p.k_blocks + p.kb_per_split - 1) / p.kb_per_split;
  if (p.splits > 1) {
    p.ws = align256(sizeof(float) * (size_t)rows * cols);
    return p;
  }
  // The last wave of a persistent launch is partly idle when tiles % slots != 0
  // (or the only wave, when tiles < slots).  Its r tiles are split into S
  // K-slices (r*S units): the tail then costs ceil(r*S / slots) / S tile-times
  // instead of one.  Pick S in 2..8 when that saves >= 15% of a tile-time and
  // every slice keeps >= 16 k-blocks.
  static const bool env_off = getenv("MS_GEMM_NO_TAIL_SPLIT") != nullptr;
  const int64_t r = tiles % slots;
  if (allow_split && !env_off && r > 0) {
    double best = 1.0;
    int bs = 0;
    for (int s = 2; s <= 8; ++s) {
      if (p.k_blocks / s < 16) break;  // short slices: the fp32 partials cost more
      const double cost = (double)((r * s + slots - 1) / slots) / s;
      if (cost < best - 0.15) {
        best = cost;
        bs = s;
      }
    }
    if (bs) {
      p.full_tiles = (int)(tiles - r);
      p.tail_splits = bs;
      p.tail_kbps = (p.k_blocks + bs - 1) / bs;
      p.tail_splits = (p.k_blocks + p.tail_kbps - 1) / p.tail_kbps;
      p.ws = align256(sizeof(float) * (size_t)r * p.tail_splits * p.cl * BM * p.bn);
    }
  }
  return p;
}

// 8 consecutive 16-bit outputs (one 16-byte store when vec, else the first left)
template <typename T>
__device__ __forceinline__ void store8(T* o, const float (&v)[8], bool vec, int left) {
  if (vec) {
    uint4 u;
    u.x = pack2<T>(v[0], v[1]);
    u.y = pack2<T>(v[2], v[3]);
    u.z = pack2<T>(v[4], v[5]);
    u.w = pack2<T>(v[6], v[7]);
    *reinterpret_cast<uint4*>(o) = u;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < left) o[j] = IO<T>::cvt(v[j]);
  }
}

// out[rows of tail tile i] = sum of its tail_splits fp32 partials (bias already
// added by slice 0), rounded once to the output dtype
template <typename T>
__global__ void tail_finalize_kernel(const float* __restrict__ ws, T* __restrict__ out,
                                     int64_t ldc, int rows, int cols, int m_blocks, int n_blocks,
                                     int n_fastest, int full_tiles, int splits, int tile_rows,
                                     int bn, T* __restrict__ act_out,
                                     const T* __restrict__ resid, const __grid_constant__ DropEpi drop,
                                     int round_lin) {
  // launched as a programmatic dependent of the GEMM: wait for its partials
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = blockIdx.y;  // tail tile
  const int tile = full_tiles + i;
  const int mb = n_fastest ? (tile / n_blocks) % m_blocks : tile % m_blocks;
  const int nb = n_fastest ? tile % n_blocks : (tile / m_blocks) % n_blocks;
  const int m0 = mb * tile_rows;
  const int n0 = nb * bn;
  const int per_row = bn / 8;
  const size_t tile_elems = (size_t)tile_rows * bn;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tile_rows * per_row;
       e += gridDim.x * blockDim.x) {
    const int r = e / per_row, c = (e - r * per_row) * 8;
    if (m0 + r >= rows || n0 + c >= cols) continue;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int s = 0; s < splits; ++s) {
      const float4* p = reinterpret_cast<const float4*>(
          ws + ((size_t)i * splits + s) * tile_elems + (size_t)r * bn + c);
      const float4 a = __ldg(p), b = __ldg(p + 1);
      acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
      acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
    }
    const int64_t off = (int64_t)(m0 + r) * ldc + n0 + c;
    const bool vec = n0 + c + 8 <= cols && ((reinterpret_cast<uintptr_t>(out + off) & 15) == 0);
    if (round_lin) {  // the epilogue's Linear -> dropout -> + residual, same roundings
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = IO<T>::ld_val(IO<T>::cvt(acc[j]));
      if (drop.on) {  // off % 4 == 0: Philox blocks off/4, off/4 + 1
        const uint32_t kb = keep_n32<2>(static_cast<uint64_t>(off) >> 2, drop.stream, drop.keys,
                                        drop.thr);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          acc[j] = ((kb >> j) & 1u) ? IO<T>::ld_val(IO<T>::cvt(acc[j] * drop.scale)) : 0.f;
      }
      if (resid) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (n0 + c + j < cols) acc[j] += IO<T>::ld(resid + off + j);
      }
    }
    store8(out + off, acc, vec, cols - n0 - c);
    if (act_out) {  // fused GELU of the rounded pre-activation
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = gelu_erf(IO<T>::ld_val(IO<T>::cvt(acc[j])));
      store8(act_out + off, acc, vec, cols - n0 - c);
    }
  }
}

// float32: hi / lo planes of both operands, K-major, pitch rounded to 16 bytes
constexpr int TF32_BN = 128;
constexpr int TF32_KB_PER_SLICE = 8;  // 8 k-blocks of 32 = 256 products per TMEM accumulation
int64_t tf32_pitch(int64_t red) { return (red + 3) / 4 * 4; }
size_t tf32_ws(int64_t rows, int64_t cols, int64_t red) {
  const int64_t ld = tf32_pitch(red);
  return 2 * align256(sizeof(float) * (size_t)rows * ld) + 2 * align256(sizeof(float) * (size_t)cols * ld);
}

LinPlan plan_linear(int64_t M, int64_t N, int64_t K, int dt, int pass) {
  LinPlan p;
  if (dt == MS_F32 && M > 0 && N > 0 && K > 0) {
    // output rows x cols, reduction red of this pass
    const int64_t rows = pass == 2 ? N : M, cols = pass == 0 ? N : K,
                  red = pass == 0 ? K : (pass == 1 ? N : M);
    static const bool env_off = getenv("MS_FP32_LINEAR") && getenv("MS_FP32_LINEAR")[0] == 's';
    // small products stay on the CUDA cores (the split pre-pass would dominate)
    if (!env_off && rows >= 64 && cols >= 32 && (double)rows * cols * red >= (double)(1 << 24)) {
      p.tf32 = true;
      p.bn = TF32_BN;
      p.ws = tf32_ws(rows, cols, red);
    }
    return p;
  }
  if (!is16(dt) || K % 8 || N % 8 || M <= 0 || N <= 0 || K <= 0) return p;  // SIMT
  if (pass == 0) return plan_gemm(M, N, K, false, true);
  if (pass == 1) return plan_gemm(M, K, N, true, true);
  return plan_gemm(N, K, M, true, true);
}

// act_out: fused GELU output (EpiParams::act_out); resid / drop: a fused
// dropout + residual add after the bias (EpiParams::drop, round_lin; the tail
// finalize applies them to K-split last-wave tiles)
ms_status run_gemm(const LinPlan& p0, int dt, int a_mn, int b_mn, const CUtensorMap& ta,
                   const CUtensorMap& tb, int64_t rows, int64_t cols, void* out, int64_t ldc,
                   const void* bias, void* ws, size_t ws_bytes, cudaStream_t st,
                   void* act_out = nullptr, const void* resid = nullptr,
                   const DropEpi* drop = nullptr) {
  const LinPlan& p = p0;
  const bool post = resid != nullptr || drop != nullptr;
  TmapPack tm;
  tm.a[0] = ta;
  tm.a[1] = ta;
  tm.a[2] = ta;
  tm.a[3] = ta;
  tm.b = tb;
  GemmArgs g{};
  g.M = (int)rows;
  g.N = (int)cols;
  g.m_blocks = (p.m_blocks + p.cl - 1) / p.cl;  // pairs of M tiles when clustered
  g.n_blocks = p.n_blocks;
  g.k_blocks = p.k_blocks;
  g.splits = p.splits;
  g.kb_per_split = p.kb_per_split;
  g.taps = 1;
  g.num_tiles = g.m_blocks * p.n_blocks * p.splits;
  g.ab_fmt = dt == MS_BF16 ? 1 : 0;
  g.nphases = 1;
  {
    static const int env_dbg = [] {
      const char* e = getenv("MS_GEMM_DBG");
      return e ? atoi(e) : 0;
    }();
    g.dbg = env_dbg;
  }
  // N-blocks fastest when B (cols x red) fits well inside L2 and A does not: the
  // concurrent tiles then share their A rows and A streams from HBM once
  {
    static const int env_r = [] {
      const char* e = getenv("MS_GEMM_RASTER");  // A/B: 0 = M fastest, 1 = N fastest
      return e ? atoi(e) : -1;
    }();
    const double a_bytes = 2.0 * rows * (double)p.k_blocks * BK;
    const double b_bytes = 2.0 * cols * (double)p.k_blocks * BK;
    g.n_fastest = env_r >= 0 ? env_r
                             : (p.n_blocks > 1 && b_bytes <= 32e6 && a_bytes > b_bytes ? 1 : 0);
  }
  if (p.splits > 1) {
    MS_CHECK_ARG(!post, MS_ERR_UNSUPPORTED, "linear: split-K with a fused dropout / residual");
    MS_CHECK_ARG(ws && ws_bytes >= p.ws, MS_ERR_WORKSPACE, "linear: split-K workspace too small");
    cudaMemsetAsync(ws, 0, sizeof(float) * rows * cols, st);
    g.epi = EpiParams{ws, cols, MS_F32, 1, nullptr, 0};
    MS_TRY(launch_umma(p.bn, a_mn, b_mn, LOAD_GEMM, tm, g, st, p.cl));
    MS_CHECK_ARG(ldc == cols, MS_ERR_UNSUPPORTED, "linear: split-K needs dense output");
    MS_TRY(f32_to(static_cast<const float*>(ws), out, dt, rows * cols, bias, cols, st));
    return act_out ? gelu_fwd(rows * cols, dt, out, act_out, st) : MS_OK;
  }
  g.epi = EpiParams{out, ldc, dt, 0, bias, dt};
  g.epi.act_out = act_out;
  if (post) {
    g.epi.resid = resid;
    if (drop) g.epi.drop = *drop;
    g.epi.round_lin = 1;
  }
  MS_TRY(setup_tma_store(tm, g, dt, out, rows, cols, ldc));
  if (p.tail_splits > 0) {
    MS_CHECK_ARG(ws && ws_bytes >= p.ws, MS_ERR_WORKSPACE,
                 "linear: tail-split workspace %zu < %zu", ws_bytes, p.ws);
    g.full_tiles = p.full_tiles;
    g.tail_splits = p.tail_splits;
    g.tail_kbps = p.tail_kbps;
    g.tail_ws = static_cast<float*>(ws);
    const int tail = g.num_tiles - p.full_tiles;
    g.num_tiles = p.full_tiles + tail * p.tail_splits;
    MS_TRY(launch_umma(p.bn, a_mn, b_mn, LOAD_GEMM, tm, g, st, p.cl));
    const int tile_rows = BM * p.cl;
    const dim3 grid((unsigned)((tile_rows * (p.bn / 8) + 255) / 256), (unsigned)tail);
    // programmatic dependent launch: scheduled while the GEMM still runs (its
    // blocks wait in griddepcontrol.wait), so the launch latency is hidden
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (dt == MS_BF16)
      e = cudaLaunchKernelEx(&cfg, tail_finalize_kernel<__nv_bfloat16>,
                             static_cast<const float*>(ws), static_cast<__nv_bfloat16*>(out), ldc,
                             (int)rows, (int)cols, g.m_blocks, g.n_blocks, g.n_fastest,
                             p.full_tiles, p.tail_splits, tile_rows, p.bn,
                             static_cast<__nv_bfloat16*>(act_out),
                             static_cast<const __nv_bfloat16*>(resid), g.epi.drop,
                             g.epi.round_lin);
    else
      e = cudaLaunchKernelEx(&cfg, tail_finalize_kernel<__half>, static_cast<const float*>(ws),
                             static_cast<__half*>(out), ldc, (int)rows, (int)cols, g.m_blocks,
                             g.n_blocks, g.n_fastest, p.full_tiles, p.tail_splits, tile_rows,
                             p.bn, static_cast<__half*>(act_out),
                             static_cast<const __half*>(resid), g.epi.drop, g.epi.round_lin);
    count_launch();
    MS_CHECK_ARG(e == cudaSuccess, MS_ERR_LAUNCH, "tail_finalize_kernel: %s",
                 cudaGetErrorString(e));
    return launch_status("tail_finalize_kernel");
  }
  return launch_umma(p.bn, a_mn, b_mn, LOAD_GEMM, tm, g, st, p.cl);
}

// hi / lo tf32 planes of a float32 operand: element (r, c) = src[r * sr + c * sc]
// -> hi[r][c], lo[r][c] (pitch ld), hi = v with the low 13 mantissa bits cleared
// (exact in tf32), lo = v - hi (exact in fp32).  32 x 32 tiles through shared
// memory, so both a row-major and a transposed source are read coalesced.
__global__ void __launch_bounds__(256) split_tf32_kernel(int64_t R, int64_t C, const float* __restrict__ src,
                                                         int64_t sr, int64_t sc, float* __restrict__ hi,
                                                         float* __restrict__ lo, int64_t ld) {
  __shared__ float t[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const bool c_fast = sc == 1;  // source contiguous along c (else along r)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int a = ty + 8 * i;  // slow index within the tile
    const int64_t r = c_fast ? r0 + a : r0 + tx, c = c_fast ? c0 + tx : c0 + a;
    const float v = (r < R && c < C) ? __ldg(src + r * sr + c * sc) : 0.f;
    if (c_fast) t[a][tx] = v;
    else t[tx][a] = v;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int a = ty + 8 * i;
    const int64_t r = r0 + a, c = c0 + tx;
    if (r < R && c < C) {
      const float v = t[a][tx];
      const float h = __uint_as_float(__float_as_uint(v) & 0xffffe000u);
      hi[r * ld + c] = h;
      lo[r * ld + c] = v - h;
    }
  }
}

// out[rows][cols] (pitch ldc, fp32) = A . B^T (+ bias), A(r, k) = a[r*ar + k*ak],
// B(n, k) = b[n*br + k*bk], on the tcgen05 kind::tf32 kernel (3xTF32)
ms_status run_tf32(int64_t rows, int64_t cols, int64_t red, const float* a, int64_t ar, int64_t ak,
                   const float* b, int64_t br, int64_t bk, float* out, int64_t ldc,
                   const float* bias, void* ws, size_t ws_bytes, cudaStream_t st) {
  MS_CHECK_ARG(ws && ws_bytes >= tf32_ws(rows, cols, red), MS_ERR_WORKSPACE,
               "linear fp32: workspace %zu < %zu", ws_bytes, tf32_ws(rows, cols, red));
  const int64_t ld = tf32_pitch(red);
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  float* a_hi = reinterpret_cast<float*>(w8);
  float* a_lo = reinterpret_cast<float*>(w8 + align256(sizeof(float) * rows * ld));
  float* b_hi = reinterpret_cast<float*>(w8 + 2 * align256(sizeof(float) * rows * ld));
  float* b_lo = reinterpret_cast<float*>(w8 + 2 * align256(sizeof(float) * rows * ld) +
                                         align256(sizeof(float) * cols * ld));
  split_tf32_kernel<<<dim3((unsigned)((red + 31) / 32), (unsigned)((rows + 31) / 32)), 256, 0, st>>>(
      rows, red, a, ar, ak, a_hi, a_lo, ld);
  split_tf32_kernel<<<dim3((unsigned)((red + 31) / 32), (unsigned)((cols + 31) / 32)), 256, 0, st>>>(
      cols, red, b, br, bk, b_hi, b_lo, ld);
  count_launch(2);
  MS_TRY(launch_status("split_tf32_kernel"));
  TmapPack tm;
  MS_TRY(make_tmap_2d(&tm.a[0], MS_F32, a_hi, red, rows, ld, 32, BM));
  MS_TRY(make_tmap_2d(&tm.a[1], MS_F32, a_lo, red, rows, ld, 32, BM));
  MS_TRY(make_tmap_2d(&tm.b, MS_F32, b_hi, red, cols, ld, 32, TF32_BN));
  MS_TRY(make_tmap_2d(&tm.a[2], MS_F32, b_lo, red, cols, ld, 32, TF32_BN));
  tm.a[3] = tm.a[0];
  GemmArgs g{};
  g.M = (int)rows;
  g.N = (int)cols;
  g.m_blocks = (int)((rows + BM - 1) / BM);
  g.n_blocks = (int)((cols + TF32_BN - 1) / TF32_BN);
  g.k_blocks = (int)((red + 31) / 32);
  // The tensor core's fp32 accumulation of a long reduction drifts past the
  // fp32 bar (norm-wise 3e-5 at K = 2048-4096, measured): every tile
  // accumulates at most 256 products of the reduction in TMEM, and the slices
  // are added into the zeroed fp32 output with red.add.
  g.kb_per_split = TF32_KB_PER_SLICE;
  g.splits = (g.k_blocks + g.kb_per_split - 1) / g.kb_per_split;
  g.taps = 1;
  g.num_tiles = g.m_blocks * g.n_blocks * g.splits;
  g.ab_fmt = 2;  // tf32
  g.nphases = 1;
  g.n_fastest = g.n_blocks > 1 && cols * red <= 4 * 1024 * 1024 && rows > cols ? 1 : 0;
  if (g.splits > 1) {
    MS_CHECK_ARG(cudaMemset2DAsync(out, sizeof(float) * ldc, 0, sizeof(float) * cols, rows, st) ==
                     cudaSuccess,
                 MS_ERR_LAUNCH, "linear fp32: memset failed");
  }
  g.epi = EpiParams{out, ldc, MS_F32, g.splits > 1 ? 1 : 0, bias, MS_F32};
  return launch_umma(TF32_BN, 0, 0, LOAD_GEMM_3XTF32, tm, g, st, 1);
}

}  // namespace
}  // namespace ms

using namespace ms;

extern "C" size_t ms_linear_workspace(int64_t M, int64_t N, int64_t K, int32_t dtype,
                                      int32_t pass) {
  return plan_linear(M, N, K, dtype, pass).ws;
}

extern "C" ms_status ms_linear_fwd(int64_t M, int64_t N, int64_t K, int32_t dt, const void* x,
                                   const void* w, const void* bias, void* y, void* ws,
                                   size_t ws_bytes, void* stream) {
  MS_TRY(bind_device(y));
  cudaStream_t st = (cudaStream_t)stream;
  MS_CHECK_ARG(M >= 0 && N > 0 && K > 0, MS_ERR_SHAPE, "linear: bad shape");
  if (M == 0) return MS_OK;
  LinPlan p = plan_linear(M, N, K, dt, 0);
  if (p.tc && al16(x) && al16(w) && al16(y)) {
    CUtensorMap ta, tb;
    MS_TRY(make_tmap_2d(&ta, dt, x, K, M, K, BK, BM));
    MS_TRY(make_tmap_2d(&tb, dt, w, K, N, K, BK, p.bn / p.cl));  // each CTA loads BN/cl rows
    return run_gemm(p, dt, 0, 0, ta, tb, M, N, y, N, bias, ws, ws_bytes, st);
  }
  if (p.tf32)  // y[m,n] = sum_k x[m,k] w[n,k]
    return run_tf32(M, N, K, (const float*)x, K, 1, (const float*)w, K, 1, (float*)y, N,
                    (const float*)bias, ws, ws_bytes, st);
  // y[m,n] = sum_k x[m,k] w[n,k]
  return simt_gemm(dt, (int)M, (int)N, (int)K, x, K, 1, w, 1, K, bias, y, N, st);
}

extern "C" ms_status ms_linear_gelu_fwd(int64_t M, int64_t N, int64_t K, int32_t dt,
                                        const void* x, const void* w, const void* bias, void* pre,
                                        void* y, void* ws, size_t ws_bytes, void* stream) {
  MS_TRY(bind_device(y));
  cudaStream_t st = (cudaStream_t)stream;
  MS_CHECK_ARG(M >= 0 && N > 0 && K > 0, MS_ERR_SHAPE, "linear_gelu: bad shape");
  MS_CHECK_ARG(pre != nullptr && y != nullptr && pre != y, MS_ERR_SHAPE,
               "linear_gelu: needs distinct pre-activation and output buffers");
  if (M == 0) return MS_OK;
  LinPlan p = plan_linear(M, N, K, dt, 0);
  if (p.tc && al16(x) && al16(w) && al16(pre) && al16(y)) {  // GELU in the GEMM epilogue
    CUtensorMap ta, tb;
    MS_TRY(make_tmap_2d(&ta, dt, x, K, M, K, BK, BM));
    MS_TRY(make_tmap_2d(&tb, dt, w, K, N, K, BK, p.bn / p.cl));
    return run_gemm(p, dt, 0, 0, ta, tb, M, N, pre, N, bias, ws, ws_bytes, st, y);
  }
  MS_TRY(ms_linear_fwd(M, N, K, dt, x, w, bias, pre, ws, ws_bytes, stream));
  return gelu_fwd(M * N, dt, pre, y, st);
}

extern "C" ms_status ms_linear_dropout_add_fwd(int64_t M, int64_t N, int64_t K, int32_t dt,
                                               const void* x, const void* w, const void* bias,
                                               const void* resid, double p, uint64_t seed,
                                               uint64_t stream_id, int32_t gen, void* y, void* ws,
                                               size_t ws_bytes, void* stream) {
  MS_TRY(bind_device(y));
  cudaStream_t st = (cudaStream_t)stream;
  MS_CHECK_ARG(M >= 0 && N > 0 && K > 0 && resid != nullptr && y != resid, MS_ERR_SHAPE,
               "linear_dropout_add: bad arguments");
  MS_CHECK_ARG(p >= 0.0 && p < 1.0, MS_ERR_SHAPE, "linear_dropout_add: p must be in [0, 1)");
  if (M == 0) return MS_OK;
  LinPlan pl = plan_linear(M, N, K, dt, 0);
  const bool drop = p > 0.0;
  // the epilogue draws the default generator's bits for whole 4-element blocks
  if (pl.tc && pl.splits == 1 && N % 4 == 0 && al16(x) && al16(w) && al16(y) && al16(resid) &&
      (!drop || gen == MS_RNG_PHILOX4X32)) {
    CUtensorMap ta, tb;
    MS_TRY(make_tmap_2d(&ta, dt, x, K, M, K, BK, BM));
    MS_TRY(make_tmap_2d(&tb, dt, w, K, N, K, BK, pl.bn / pl.cl));
    DropEpi d{};
    if (drop) {
      d.keys = philox32_keys(seed);
      d.stream = stream_id;
      d.thr = static_cast<uint64_t>(ceil(p * 4294967296.0));
      d.scale = static_cast<float>(1.0 / (1.0 - p));
      d.on = 1;
    }
    return run_gemm(pl, dt, 0, 0, ta, tb, M, N, y, N, bias, ws, ws_bytes, st, nullptr, resid,
                    drop ? &d : nullptr);
  }
  // the three launches
  MS_TRY(ms_linear_fwd(M, N, K, dt, x, w, bias, y, ws, ws_bytes, stream));
  if (drop) MS_TRY(ms_dropout_fwd(M * N, dt, y, y, seed, stream_id, p, gen, nullptr, stream));
  return add_inplace(M * N, dt, y, resid, st);
}

extern "C" ms_status ms_linear_dx(int64_t M, int64_t N, int64_t K, int32_t dt, const void* dy,
                                  const void* w, void* dx, void* ws, size_t ws_bytes,
                                  void* stream) {
  MS_TRY(bind_device(dx));
  cudaStream_t st = (cudaStream_t)stream;
  MS_CHECK_ARG(M >= 0 && N > 0 && K > 0, MS_ERR_SHAPE, "linear dx: bad shape");
  if (M == 0) return MS_OK;
  LinPlan p = plan_linear(M, N, K, dt, 1);
  if (p.tc && al16(dy) && al16(w) && al16(dx)) {
    CUtensorMap ta, tb;
    MS_TRY(make_tmap_2d(&ta, dt, dy, N, M, N, BK, BM));  // A = dY [M][N], K-major
    MS_TRY(make_tmap_2d(&tb, dt, w, K, N, K, 64, BK));   // B = W [N][K], MN-major
    return run_gemm(p, dt, 0, 1, ta, tb, M, K, dx, K, nullptr, ws, ws_bytes, st);
  }
  if (p.tf32)  // dx[m,k] = sum_n dy[m,n] w[n,k]: A = dY, B(k, n) = w[n*K + k]
    return run_tf32(M, K, N, (const float*)dy, N, 1, (const float*)w, 1, K, (float*)dx, K,
                    nullptr, ws, ws_bytes, st);
  // dx[m,k] = sum_n dy[m,n] w[n,k]
  return simt_gemm(dt, (int)M, (int)K, (int)N, dy, N, 1, w, K, 1, nullptr, dx, K, st);
}

extern "C" ms_status ms_linear_dw(int64_t M, int64_t N, int64_t K, int32_t dt, const void* x,
                                  const void* dy, void* dw, void* ws, size_t ws_bytes,
                                  void* stream) {
  MS_TRY(bind_device(dw));
  cudaStream_t st = (cudaStream_t)stream;
  MS_CHECK_ARG(M >= 0 && N > 0 && K > 0, MS_ERR_SHAPE, "linear dw: bad shape");
  if (M == 0) return cudaMemsetAsync(dw, 0, dtype_size(dt) * N * K, st) == cudaSuccess
                         ? MS_OK
                         : MS_ERR_LAUNCH;
  LinPlan p = plan_linear(M, N, K, dt, 2);
  if (p.tc && al16(dy) && al16(x) && al16(dw)) {
    CUtensorMap ta, tb;
    MS_TRY(make_tmap_2d(&ta, dt, dy, N, M, N, 64, BK));  // A = dYᵀ, MN-major
    MS_TRY(make_tmap_2d(&tb, dt, x, K, M, K, 64, BK));   // B = X, MN-major
    return run_gemm(p, dt, 1, 1, ta, tb, N, K, dw, K, nullptr, ws, ws_bytes, st);
  }
  if (p.tf32)  // dw[n,k] = sum_m dy[m,n] x[m,k]: A(n, m) = dy[m*N + n], B(k, m) = x[m*K + k]
    return run_tf32(N, K, M, (const float*)dy, 1, N, (const float*)x, 1, K, (float*)dw, K,
                    nullptr, ws, ws_bytes, st);
  // dw[n,k] = sum_m dy[m,n] x[m,k]
  return simt_gemm(dt, (int)N, (int)K, (int)M, dy, 1, N, x, K, 1, nullptr, dw, K, st);
}

extern "C" size_t ms_bias_grad_workspace(int64_t rows, int64_t cols, int32_t dtype) {
  (void)rows;
  (void)dtype;
  return colsum_workspace(cols);
}

extern "C" ms_status ms_bias_grad(int64_t rows, int64_t cols, int32_t dt, const void* g, void* db,
                                  void* ws, size_t ws_bytes, void* stream) {
  MS_TRY(bind_device(db));
  MS_CHECK_ARG(rows >= 0 && cols > 0, MS_ERR_SHAPE, "bias grad: bad shape");
  MS_CHECK_ARG(ws && ws_bytes >= colsum_workspace(cols), MS_ERR_WORKSPACE,
               "bias grad: workspace too small");
  return colsum(rows, cols, dt, g, db, dt, ws, (cudaStream_t)stream);
}
