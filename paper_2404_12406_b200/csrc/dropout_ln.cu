// Dropout with RNG replay and LayerNorm.
//
// Dropout (rules.py:103-106 MEMSAVE row, saved.py:91-108 RngSeed, SPEC.md
// forward_dropout): the keep mask is a pure function of (seed, stream, element
// index), so backward regenerates it instead of reading a stored mask.  Two
// counter-based generators:
//
// MS_RNG_PHILOX4X32 (default): Philox4x32-10 (Salmon et al., Random123; the
// generator curand and torch use), key = seed (lo, hi words), counter = (j lo,
// j hi, stream lo, stream hi) for the block j of elements 4j .. 4j+3; element
// 4j + i is kept iff word_i >= ceil(p * 2^32).  32-bit multiplies make it ~4x
// cheaper than the 64-bit generator below, so it runs near HBM speed.
//
// MS_RNG_PHILOX4X64_REF: the reference's own generator,
// leantape.core.Rng(seed, stream).uniform()
// (core.py:100-124) is numpy's Philox4x64-10 keyed [seed, stream] with a
// 256-bit counter that is incremented before each 4-word block, and
// Generator.random() maps a 64-bit word u to (u >> 11) * 2^-53.  Element i
// therefore uses word i % 4 of block (i / 4) + 1 and is kept iff
// U_i >= p  <=>  (u >> 11) >= ceil(p * 2^53), so the mask here is bit-identical
// to the reference's for the same (seed, stream, p).  Kept elements are scaled
// by 1 / (1 - p) (SPEC.md DropoutConfig).
//
// LayerNorm over the last dimension (rules.py:89-96, SPEC.md forward_layernorm):
// y = (x - mean) * rstd * w + b with fp32 statistics; the saved set is
// {x, mean/rstd, w} under both policies.  Backward:
//   dx = rstd * (g w - mean_j(g w) - xhat * mean_j(g w xhat)),
//   dw = sum_rows g xhat,  db = sum_rows g   (launched only when requested).
// One warp per row; rows up to 2048 elements live in registers (8 per lane per
// 256-column slab), longer or unaligned rows take a block-per-row loop.
#include "misc.cuh"
#include "rng.cuh"
#include "vec.cuh"

namespace ms {
namespace {

// ---------------------------------------------------------------- Philox4x64-10
// Round keys (k0 + r*W0, k1 + r*W1) are the same for every element: the host
// precomputes them (kernel parameters, read from the constant bank).
struct PhiloxKeys {
  uint64_t k[10][2];
};

// hi:lo = a * b, 64 x 64 -> 128 bits as four 32x32->64 multiply-adds (each
// one IMAD.WIDE; the 64-bit addends never overflow): about half the IMADs of
// __umul64hi plus a separate 64-bit multiply
__device__ __forceinline__ void mul128(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32);
  const uint32_t b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  const uint64_t t = (uint64_t)a0 * b0;
  const uint64_t u = (uint64_t)a1 * b0 + (t >> 32);
  const uint64_t v = (uint64_t)a0 * b1 + (uint32_t)u;
  lo = (v << 32) | (uint32_t)t;
  hi = (uint64_t)a1 * b1 + (u >> 32) + (v >> 32);
}

// Philox4x32-10: rng.cuh (shared with the GEMM epilogue's fused dropout)

struct DropoutKeys {
  PhiloxKeys k64;    // MS_RNG_PHILOX4X64_REF
  Philox32Keys k32;  // MS_RNG_PHILOX4X32
  uint64_t stream;
};

// NB Philox blocks in lockstep (independent dependency chains for ILP):
// block blk0 + b -> bits 4b .. 4b+3
template <int NB>
__device__ __forceinline__ uint32_t keep_n(uint64_t blk0, const PhiloxKeys& K, uint64_t thr) {
  constexpr uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  uint64_t c[NB][4];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    c[b][0] = blk0 + b;
    c[b][1] = c[b][2] = c[b][3] = 0ull;
  }
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      uint64_t hi0, lo0, hi1, lo1;
      mul128(M0, c[b][0], hi0, lo0);
      mul128(M1, c[b][2], hi1, lo1);
      const uint64_t n0 = hi1 ^ c[b][1] ^ K.k[r][0], n2 = hi0 ^ c[b][3] ^ K.k[r][1];
      c[b][0] = n0;
      c[b][1] = lo1;
      c[b][2] = n2;
      c[b][3] = lo0;
    }
  }
  uint32_t bits = 0;
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int j = 0; j < 4; ++j) bits |= ((c[b][j] >> 11) >= thr ? 1u : 0u) << (4 * b + j);
  return bits;
}

// y = keep ? x * scale : 0 over groups of 16 elements (four Philox blocks);
// mask (optional, 1 byte per element) receives the keep flags.
template <int GEN, int NB>
__device__ __forceinline__ uint32_t keep_blocks(uint64_t blk, const DropoutKeys& K, uint64_t thr) {
  if constexpr (GEN == MS_RNG_PHILOX4X64_REF) return keep_n<NB>(blk + 1, K.k64, thr);
  else return keep_n32<NB>(blk, K.stream, K.k32, thr);
}

template <typename T, int GEN>
__global__ void __launch_bounds__(256) dropout_kernel(int64_t n, const T* x, T* y,
                                                      const __grid_constant__ DropoutKeys K,
                                                      uint64_t thr, float scale,
                                                      uint8_t* __restrict__ mask, bool vec) {
  const int64_t full = n / 16;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < full; gi += stride) {
    float v[2][8];
    ld8<T>(x + gi * 16, v[0], vec);
    ld8<T>(x + gi * 16 + 8, v[1], vec);
    const uint32_t bits = keep_blocks<GEN, 4>(4 * gi, K, thr);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[h][j] = (bits >> (8 * h + j)) & 1u ? v[h][j] * scale : 0.f;
      st8<T>(y + gi * 16 + 8 * h, v[h], vec);
    }
    if (mask) {
      if (vec) {
        uint4 m;
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          w[q] = ((bits >> (4 * q)) & 1u) | ((bits >> (4 * q + 1)) & 1u) << 8 |
                 ((bits >> (4 * q + 2)) & 1u) << 16 | ((bits >> (4 * q + 3)) & 1u) << 24;
        m.x = w[0]; m.y = w[1]; m.z = w[2]; m.w = w[3];
        *reinterpret_cast<uint4*>(mask + gi * 16) = m;
      } else {
        for (int j = 0; j < 16; ++j) mask[gi * 16 + j] = (bits >> j) & 1u;
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // tail elements
    for (int64_t e = full * 16; e < n; ++e) {
      const uint32_t b = keep_blocks<GEN, 1>(static_cast<uint64_t>(e / 4), K, thr);
      const bool keep = (b >> (e % 4)) & 1u;
      y[e] = IO<T>::cvt(keep ? IO<T>::ld(x + e) * scale : 0.f);
      if (mask) mask[e] = keep ? 1 : 0;
    }
  }
}

int grid_for(int64_t work, int per_sm = 16) {
  int64_t b = (work + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * per_sm;
  if (b > cap) b = cap;
  return (int)(b > 0 ? b : 1);
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

ms_status dropout_launch(int64_t numel, int dt, const void* x, void* y, uint64_t seed,
                         uint64_t stream_id, double p, int gen, void* mask, cudaStream_t st) {
  MS_CHECK_ARG(numel >= 0, MS_ERR_SHAPE, "dropout: negative numel");
  MS_CHECK_ARG(p >= 0.0 && p < 1.0, MS_ERR_SHAPE, "dropout: p must be in [0, 1), got %g", p);
  MS_CHECK_ARG(gen == MS_RNG_PHILOX4X32 || gen == MS_RNG_PHILOX4X64_REF, MS_ERR_UNSUPPORTED,
               "dropout: unknown generator %d", gen);
  if (numel == 0) return MS_OK;
  // 64-bit reference generator: keep iff (u >> 11) >= ceil(p * 2^53) (p * 2^53
  // is exact in double); 32-bit generator: keep iff u >= ceil(p * 2^32)
  const uint64_t thr = static_cast<uint64_t>(
      ceil(p * (gen == MS_RNG_PHILOX4X64_REF ? 9007199254740992.0 : 4294967296.0)));
  const float scale = static_cast<float>(1.0 / (1.0 - p));
  const bool vec = al16(x) && al16(y) && (!mask || (reinterpret_cast<uintptr_t>(mask) & 15) == 0);
  DropoutKeys K;
  uint64_t k0 = seed, k1 = stream_id;
  for (int r = 0; r < 10; ++r) {  // Weyl key schedule
    K.k64.k[r][0] = k0;
    K.k64.k[r][1] = k1;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  K.k32 = philox32_keys(seed);
  K.stream = stream_id;
  const int grid = grid_for(numel / 16 + 1);
  if (gen == MS_RNG_PHILOX4X64_REF) {
    MS_DT_DISPATCH(dt, (dropout_kernel<T, MS_RNG_PHILOX4X64_REF><<<grid, 256, 0, st>>>(
                           numel, (const T*)x, (T*)y, K, thr, scale, (uint8_t*)mask, vec)));
  } else {
    MS_DT_DISPATCH(dt, (dropout_kernel<T, MS_RNG_PHILOX4X32><<<grid, 256, 0, st>>>(
                           numel, (const T*)x, (T*)y, K, thr, scale, (uint8_t*)mask, vec)));
  }
  count_launch();
  return launch_status("dropout");
}

// ---------------------------------------------------------------- LayerNorm
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int LN_WARPS = 8;

// KV slabs of 256 columns (8 per lane) held in registers
template <int KV> struct LnRows {  // rows per warp (2 halves the resident warps: slower)
  static constexpr int BWD = 1;
};

template <typename T, int KV>
__global__ void __launch_bounds__(LN_WARPS * 32) ln_fwd_vec(int64_t rows, int D, const T* x,
                                                            const T* w, const T* b, float eps,
                                                            T* y, float* mean, float* rstd) {
  // one row per warp; w / b are read after the reductions so few registers are
  // live and many warps per SM keep HBM busy (measured faster than prefetching)
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * LN_WARPS + (threadIdx.x >> 5);
  if (row >= rows) return;
  const T* xr = x + row * D;
  float v[KV][8];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    const int col = (k * 32 + lane) * 8;
    if (col < D) {
      ld8<T>(xr + col, v[k], true);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[k][j];
    }
  }
  const float mu = warp_sum(s) / D;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    const int col = (k * 32 + lane) * 8;
    if (col < D) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float d = v[k][j] - mu;
        q += d * d;
      }
    }
  }
  const float r = rsqrtf(warp_sum(q) / D + eps);
  T* yr = y + row * D;
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    const int col = (k * 32 + lane) * 8;
    if (col < D) {
      float wv[8], bv[8];
      if (w) ld8<T>(w + col, wv, true);
      if (b) ld8<T>(b + col, bv, true);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float o = (v[k][j] - mu) * r;
        if (w) o *= wv[j];
        if (b) o += bv[j];
        v[k][j] = o;
      }
      st8<T>(yr + col, v[k], true);
    }
  }
  if (lane == 0) {
    if (mean) mean[row] = mu;
    if (rstd) rstd[row] = r;
  }
}

// input-VJP only (frozen w / b: BERT's LayerNorms), LN_RPW rows per warp, all
// loads issued up front; rows of <= 768 elements are held to 4 resident blocks
// per SM (32 warps, 96 KB of loads in flight): 40 -> 36 us at 32768 x 768
template <typename T, int KV>
__global__ void __launch_bounds__(LN_WARPS * 32, KV <= 3 ? 4 : 1) ln_bwd_dx_vec(int64_t rows, int D, const T* g,
                                                               const T* x, const float* mean,
                                                               const float* rstd, const T* w,
                                                               T* dx) {
  constexpr int LN_RPW = LnRows<KV>::BWD;
  const int lane = threadIdx.x & 31;
  const int64_t row0 = ((int64_t)blockIdx.x * LN_WARPS + (threadIdx.x >> 5)) * LN_RPW;
  if (row0 >= rows) return;
  float xv[LN_RPW][KV][8], gv[LN_RPW][KV][8], wv[KV][8];
  float mu[LN_RPW], rs[LN_RPW];
#pragma unroll
  for (int rr = 0; rr < LN_RPW; ++rr) {
    const int64_t row = row0 + rr < rows ? row0 + rr : row0;
    mu[rr] = mean[row];
    rs[rr] = rstd[row];
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int col = (k * 32 + lane) * 8;
      if (col < D) {
        ld8<T>(x + row * D + col, xv[rr][k], true);
        ld8<T>(g + row * D + col, gv[rr][k], true);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    const int col = (k * 32 + lane) * 8;
    if (col < D && w) {
      ld8<T>(w + col, wv[k], true);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) wv[k][j] = 1.f;
    }
  }
#pragma unroll
  for (int rr = 0; rr < LN_RPW; ++rr) {
    const int64_t row = row0 + rr;
    if (row >= rows) break;
    float a = 0.f, c = 0.f;
#pragma unroll
    for (int k = 0; k < KV; ++k)
      if ((k * 32 + lane) * 8 < D)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          xv[rr][k][j] = (xv[rr][k][j] - mu[rr]) * rs[rr];
          const float gw = gv[rr][k][j] * wv[k][j];
          gv[rr][k][j] = gw;
          a += gw;
          c += gw * xv[rr][k][j];
        }
    const float ma = warp_sum(a) / D, mc = warp_sum(c) / D;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int col = (k * 32 + lane) * 8;
      if (col < D) {
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = rs[rr] * (gv[rr][k][j] - ma - xv[rr][k][j] * mc);
        st8<T>(dx + row * D + col, o, true);
      }
    }
  }
}

__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

// any D / alignment: one block per row, three passes over the row
template <typename T>
__global__ void __launch_bounds__(256) ln_fwd_generic(int64_t rows, int D, const T* x, const T* w,
                                                      const T* b, float eps, T* y, float* mean,
                                                      float* rstd) {
  __shared__ float red[8];
  const int64_t row = blockIdx.x;
  const T* xr = x + row * D;
  float s = 0.f;
  for (int i = threadIdx.x; i < D; i += blockDim.x) s += IO<T>::ld(xr + i);
  const float mu = block_sum(s, red) / D;
  float q = 0.f;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    const float d = IO<T>::ld(xr + i) - mu;
    q += d * d;
  }
  const float r = rsqrtf(block_sum(q, red) / D + eps);
  T* yr = y + row * D;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    float o = (IO<T>::ld(xr + i) - mu) * r;
    if (w) o *= IO<T>::ld(w + i);
    if (b) o += IO<T>::ld(b + i);
    yr[i] = IO<T>::cvt(o);
  }
  if (threadIdx.x == 0) {
    if (mean) mean[row] = mu;
    if (rstd) rstd[row] = r;
  }
}

// backward, one warp per row (grid-stride over rows).  dw / db partial sums:
// in registers for rows of <= 1024 16-bit elements (KV <= 4); for longer rows
// (KV > 4) the partials live in per-warp shared-memory slices (each lane owns
// its 8-column chunks, so no atomics) and the weight row is read from shared
// memory, which keeps the row's x-hat and g in registers without spilling.
// The per-warp partials are reduced per block and added into the workspace with
// one fp32 atomic per column per block.
template <int KV>
struct LnBwdSmem {
  static constexpr bool PS = KV > 4;  // partials + weight row in shared memory
};

template <typename T, int KV, bool WANTP>
__global__ void __launch_bounds__(LN_WARPS * 32) ln_bwd_vec(int64_t rows, int D, const T* g,
                                                            const T* x, const float* mean,
                                                            const float* rstd, const T* w, T* dx,
                                                            float* dw_acc, float* db_acc) {
  // shared memory: register partials -> sacc[2][D];
  //                smem partials    -> part[LN_WARPS][2][D], then wrow[D]
  extern __shared__ float sacc[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr bool wantp = WANTP;
  constexpr bool ps = WANTP && LnBwdSmem<KV>::PS;
  float* part = sacc + (size_t)wid * 2 * D;       // this warp's [2][D] slice (ps)
  float* wrow = sacc + (size_t)LN_WARPS * 2 * D;  // weight row (ps)
  if constexpr (ps) {
    for (int i = threadIdx.x; i < LN_WARPS * 2 * D; i += blockDim.x) sacc[i] = 0.f;
    for (int i = threadIdx.x; i < D; i += blockDim.x) wrow[i] = w ? IO<T>::ld(w + i) : 1.f;
    __syncthreads();
  } else if constexpr (wantp) {
    for (int i = threadIdx.x; i < 2 * D; i += blockDim.x) sacc[i] = 0.f;
    __syncthreads();
  }
  float wv[ps ? 1 : KV][8];
  float pw[ps ? 1 : KV][8], pb[ps ? 1 : KV][8];
  if constexpr (!ps) {
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int col = (k * 32 + lane) * 8;
      if (col < D && w) {
        ld8<T>(w + col, wv[k], true);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) wv[k][j] = 1.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) pw[k][j] = pb[k][j] = 0.f;
    }
  }
  auto wget = [&](int k, int j) -> float {
    if constexpr (ps) return wrow[(k * 32 + lane) * 8 + j];
    else return wv[k][j];
  };
  const int64_t step = (int64_t)gridDim.x * LN_WARPS;
  for (int64_t row = (int64_t)blockIdx.x * LN_WARPS + wid; row < rows; row += step) {
    const float mu = mean[row], r = rstd[row];
    float xh[KV][8], gv[KV][8];
    float a = 0.f, c = 0.f;
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int col = (k * 32 + lane) * 8;
      if (col < D) {
        ld8<T>(x + row * D + col, xh[k], true);
        ld8<T>(g + row * D + col, gv[k], true);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          xh[k][j] = (xh[k][j] - mu) * r;
          const float gw = gv[k][j] * wget(k, j);
          a += gw;
          c += gw * xh[k][j];
        }
        if constexpr (ps) {
          float4* pw4 = reinterpret_cast<float4*>(part + col);
          float4* pb4 = reinterpret_cast<float4*>(part + D + col);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float4 u = pw4[h], v = pb4[h];
            u.x += gv[k][4 * h] * xh[k][4 * h];
            u.y += gv[k][4 * h + 1] * xh[k][4 * h + 1];
            u.z += gv[k][4 * h + 2] * xh[k][4 * h + 2];
            u.w += gv[k][4 * h + 3] * xh[k][4 * h + 3];
            v.x += gv[k][4 * h];
            v.y += gv[k][4 * h + 1];
            v.z += gv[k][4 * h + 2];
            v.w += gv[k][4 * h + 3];
            pw4[h] = u;
            pb4[h] = v;
          }
        } else if constexpr (wantp) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            pw[k][j] += gv[k][j] * xh[k][j];
            pb[k][j] += gv[k][j];
          }
        }
      }
    }
    if (dx) {
      const float ma = warp_sum(a) / D, mc = warp_sum(c) / D;
#pragma unroll
      for (int k = 0; k < KV; ++k) {
        const int col = (k * 32 + lane) * 8;
        if (col < D) {
          float o[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] = r * (gv[k][j] * wget(k, j) - ma - xh[k][j] * mc);
          st8<T>(dx + row * D + col, o, true);
        }
      }
    }
  }
  if constexpr (ps) {
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * D; i += blockDim.x) {
      float t = 0.f;
#pragma unroll
      for (int q = 0; q < LN_WARPS; ++q) t += sacc[(size_t)q * 2 * D + i];
      float* dst = i < D ? dw_acc : db_acc;
      if (dst) atomicAdd(&dst[i < D ? i : i - D], t);
    }
  } else if constexpr (wantp) {
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int col = (k * 32 + lane) * 8;
      if (col < D) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          atomicAdd(&sacc[col + j], pw[k][j]);
          atomicAdd(&sacc[D + col + j], pb[k][j]);
        }
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < D; i += blockDim.x) {
      if (dw_acc) atomicAdd(&dw_acc[i], sacc[i]);
      if (db_acc) atomicAdd(&db_acc[i], sacc[D + i]);
    }
  }
}

// any D / alignment: one block per row
template <typename T>
__global__ void __launch_bounds__(256) ln_bwd_generic(int64_t rows, int D, const T* g, const T* x,
                                                      const float* mean, const float* rstd,
                                                      const T* w, T* dx, float* dw_acc,
                                                      float* db_acc) {
  __shared__ float red[8];
  const int64_t row = blockIdx.x;
  const float mu = mean[row], r = rstd[row];
  const T* xr = x + row * D;
  const T* gr = g + row * D;
  float a = 0.f, c = 0.f;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    const float xh = (IO<T>::ld(xr + i) - mu) * r;
    const float gv = IO<T>::ld(gr + i);
    const float gw = gv * (w ? IO<T>::ld(w + i) : 1.f);
    a += gw;
    c += gw * xh;
    if (dw_acc) atomicAdd(&dw_acc[i], gv * xh);
    if (db_acc) atomicAdd(&db_acc[i], gv);
  }
  const float ma = block_sum(a, red) / D, mc = block_sum(c, red) / D;
  if (!dx) return;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    const float xh = (IO<T>::ld(xr + i) - mu) * r;
    const float gw = IO<T>::ld(gr + i) * (w ? IO<T>::ld(w + i) : 1.f);
    dx[row * D + i] = IO<T>::cvt(r * (gw - ma - xh * mc));
  }
}

// KV slabs for the register path (0 = generic)
int ln_kv(int64_t D, int dt, const void* const* ptrs, int nptr) {
  if (D % 8 != 0 || D > 2048) return 0;
  for (int i = 0; i < nptr; ++i)
    if (ptrs[i] && !al16(ptrs[i])) return 0;
  (void)dt;
  const int kv = (int)((D + 255) / 256);
  return kv <= 4 ? kv : (kv <= 6 ? 6 : 8);
}

#define MS_KV_SWITCH(kv, ...)              \
  switch (kv) {                            \
    case 1: { constexpr int KV = 1; __VA_ARGS__; } break; \
    case 2: { constexpr int KV = 2; __VA_ARGS__; } break; \
    case 3: { constexpr int KV = 3; __VA_ARGS__; } break; \
    case 4: { constexpr int KV = 4; __VA_ARGS__; } break; \
    case 6: { constexpr int KV = 6; __VA_ARGS__; } break; \
    default: { constexpr int KV = 8; __VA_ARGS__; } break; \
  }

}  // namespace
}  // namespace ms

using namespace ms;

extern "C" ms_status ms_dropout_fwd(int64_t numel, int32_t dtype, const void* x, void* y,
                                    uint64_t seed, uint64_t stream_id, double p,
                                    int32_t generator, void* mask_or_null, void* stream) {
  MS_TRY(bind_device(y));
  return dropout_launch(numel, dtype, x, y, seed, stream_id, p, generator, mask_or_null,
                        (cudaStream_t)stream);
}

extern "C" ms_status ms_dropout_bwd(int64_t numel, int32_t dtype, const void* g, void* dx,
                                    uint64_t seed, uint64_t stream_id, double p,
                                    int32_t generator, void* stream) {
  MS_TRY(bind_device(dx));
  // dx = g * mask / (1 - p): the same map as the forward, with the mask replayed
  return dropout_launch(numel, dtype, g, dx, seed, stream_id, p, generator, nullptr,
                        (cudaStream_t)stream);
}

extern "C" size_t ms_layernorm_workspace(int64_t rows, int64_t dim, int32_t dtype) {
  (void)rows;
  (void)dtype;
  return (size_t)(2 * dim * sizeof(float) + 255) & ~(size_t)255;
}

extern "C" ms_status ms_layernorm_fwd(int64_t rows, int64_t dim, int32_t dt, const void* x,
                                      const void* w, const void* b, double eps, void* y,
                                      float* mean, float* rstd, void* stream) {
  MS_TRY(bind_device(y));
  MS_CHECK_ARG(rows >= 0 && dim > 0 && dim < (1ll << 31), MS_ERR_SHAPE, "layernorm: bad shape");
  if (rows == 0) return MS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const void* ps[4] = {x, y, w, b};
  const int kv = ln_kv(dim, dt, ps, 4);
  const int D = (int)dim;
  if (kv > 0) {
    MS_DT_DISPATCH(dt, MS_KV_SWITCH(kv, (ln_fwd_vec<T, KV><<<
                           (unsigned)((rows + LN_WARPS - 1) / LN_WARPS), LN_WARPS * 32, 0, st>>>(
                                            rows, D, (const T*)x, (const T*)w, (const T*)b,
                                            (float)eps, (T*)y, mean, rstd))));
  } else {
    MS_CHECK_ARG(rows < (1ll << 31), MS_ERR_UNSUPPORTED, "layernorm: too many rows");
    MS_DT_DISPATCH(dt, (ln_fwd_generic<T><<<(unsigned)rows, 256, 0, st>>>(
                           rows, D, (const T*)x, (const T*)w, (const T*)b, (float)eps, (T*)y,
                           mean, rstd)));
  }
  count_launch();
  return launch_status("layernorm_fwd");
}

extern "C" ms_status ms_layernorm_bwd(int64_t rows, int64_t dim, int32_t dt, const void* g,
                                      const void* x, const float* mean, const float* rstd,
                                      const void* w, void* dx, void* dw, void* db, void* ws,
                                      size_t ws_bytes, void* stream) {
  MS_TRY(bind_device(g));
  MS_CHECK_ARG(rows >= 0 && dim > 0 && dim < (1ll << 31), MS_ERR_SHAPE, "layernorm: bad shape");
  MS_CHECK_ARG(x && mean && rstd, MS_ERR_SHAPE, "layernorm bwd: x / mean / rstd required");
  cudaStream_t st = (cudaStream_t)stream;
  const bool wantp = dw || db;
  float* acc = static_cast<float*>(ws);
  if (wantp) {
    MS_CHECK_ARG(ws && ws_bytes >= ms_layernorm_workspace(rows, dim, dt), MS_ERR_WORKSPACE,
                 "layernorm bwd: workspace too small");
    if (cudaMemsetAsync(acc, 0, 2 * dim * sizeof(float), st) != cudaSuccess)
      return launch_status("layernorm memset");
  }
  if (rows > 0 && (dx || wantp)) {
    const void* ps[4] = {g, x, w, dx};
    const int kv = ln_kv(dim, dt, ps, 4);
    const int D = (int)dim;
    float* dwa = dw ? acc : nullptr;
    float* dba = db ? acc + dim : nullptr;
    if (kv > 0) {
      int64_t grid = (rows + LN_WARPS - 1) / LN_WARPS;
      if (wantp && grid > (int64_t)num_sms() * 4) grid = num_sms() * 4;  // amortise the atomics
      if (grid > (1ll << 30)) grid = 1ll << 30;
      if (wantp) {
        MS_DT_DISPATCH(dt, MS_KV_SWITCH(kv, ({
          const size_t smem = LnBwdSmem<KV>::PS ? (size_t)(LN_WARPS * 2 + 1) * D * sizeof(float)
                                                : (size_t)2 * D * sizeof(float);
          auto kern = ln_bwd_vec<T, KV, true>;
          if (smem > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          int64_t gr = grid;
          if (LnBwdSmem<KV>::PS && gr > (int64_t)num_sms()) gr = num_sms();  // 1 block / SM
          kern<<<(unsigned)gr, LN_WARPS * 32, smem, st>>>(rows, D, (const T*)g, (const T*)x,
                                                          mean, rstd, (const T*)w, (T*)dx, dwa,
                                                          dba);
        })));
      } else {
        MS_DT_DISPATCH(dt, MS_KV_SWITCH(kv, (ln_bwd_dx_vec<T, KV><<<
                               (unsigned)((rows + LN_WARPS * LnRows<KV>::BWD - 1) /
                                          (LN_WARPS * LnRows<KV>::BWD)),
                               LN_WARPS * 32, 0, st>>>(
                                                rows, D, (const T*)g, (const T*)x, mean, rstd,
                                                (const T*)w, (T*)dx))));
      }
    } else {
      MS_CHECK_ARG(rows < (1ll << 31), MS_ERR_UNSUPPORTED, "layernorm: too many rows");
      MS_DT_DISPATCH(dt, (ln_bwd_generic<T><<<(unsigned)rows, 256, 0, st>>>(
                             rows, D, (const T*)g, (const T*)x, mean, rstd, (const T*)w, (T*)dx,
                             dwa, dba)));
    }
    count_launch();
    MS_TRY(launch_status("layernorm_bwd"));
  }
  if (dw) MS_TRY(f32_to(acc, dw, dt, dim, nullptr, 0, st));
  if (db) MS_TRY(f32_to(acc + dim, db, dt, dim, nullptr, 0, st));
  return MS_OK;
}
