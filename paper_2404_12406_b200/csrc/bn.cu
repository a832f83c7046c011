// BatchNorm2d in eval mode: y = x*scale_c + shift_c with
// scale_c = w_c/sqrt(var_c+eps), shift_c = b_c - mean_c*scale_c.
// Backward: dx = g*scale_c (iff requested), dw_c = sum g*(x-mean_c)*invstd_c
// (iff requested; the only consumer of x), db_c = sum g.
// HBM-bound: 16-byte vector loads/stores, per-channel constants in smem, one
// pass over g (and x iff dw is requested), fp32 per-block channel partials
// reduced with shared atomics and one global atomic per channel per block.
#include "misc.cuh"

namespace ms {

struct BnParams {
  const void* mean;
  const void* var;
  const void* weight;  // nullable (affine=False)
  const void* bias;    // nullable
  int pdtype;
  float eps;
};

__device__ __forceinline__ void bn_channel_consts(const BnParams& p, int c, float& scale,
                                                  float& shift, float& invstd, float& mean) {
  const float v = load_as_float(p.var, p.pdtype, c);
  mean = load_as_float(p.mean, p.pdtype, c);
  invstd = 1.0f / sqrtf(v + p.eps);
  const float w = p.weight ? load_as_float(p.weight, p.pdtype, c) : 1.0f;
  const float b = p.bias ? load_as_float(p.bias, p.pdtype, c) : 0.0f;
  scale = w * invstd;
  shift = b - mean * scale;
}

template <typename T, int VEC>
struct Vec {
  static constexpr int BYTES = VEC * sizeof(T);
};

template <typename T, int VEC>
__device__ __forceinline__ void load_vec(const T* p, float (&v)[VEC]) {
  if constexpr (VEC * sizeof(T) == 16) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int j = 0; j < VEC; ++j) v[j] = IO<T>::ld(e + j);
  } else {
#pragma unroll
    for (int j = 0; j < VEC; ++j) v[j] = IO<T>::ld(p + j);
  }
}
template <typename T, int VEC>
__device__ __forceinline__ void store_vec(T* p, const float (&v)[VEC]) {
  if constexpr (VEC * sizeof(T) == 16) {
    uint4 u;
    T* e = reinterpret_cast<T*>(&u);
#pragma unroll
    for (int j = 0; j < VEC; ++j) e[j] = IO<T>::cvt(v[j]);
    *reinterpret_cast<uint4*>(p) = u;
  } else {
#pragma unroll
    for (int j = 0; j < VEC; ++j) p[j] = IO<T>::cvt(v[j]);
  }
}

// ---------------------------------------------------------------- forward
// NHWC requires C % VEC == 0; NCHW requires hw % VEC == 0 (host checks, else VEC=1)
template <typename T, int VEC>
__global__ void __launch_bounds__(256) bn_fwd_kernel(int64_t total, int C, int64_t hw, int layout,
                                                     BnParams p, const T* __restrict__ x,
                                                     T* __restrict__ y) {
  extern __shared__ float sh[];
  float* s_scale = sh;
  float* s_shift = sh + C;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float sc, sf, inv, mu;
    bn_channel_consts(p, c, sc, sf, inv, mu);
    s_scale[c] = sc;
    s_shift[c] = sf;
  }
  __syncthreads();
  const int64_t nvec = total / VEC;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * VEC;
    float v[VEC];
    load_vec<T, VEC>(x + e, v);
    if (layout == MS_NHWC) {
      const int c0 = (int)(e % C);
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = v[j] * s_scale[c0 + j] + s_shift[c0 + j];
    } else {
      const int c = (int)((e / hw) % C);
      const float sc = s_scale[c], sf = s_shift[c];
#pragma unroll
      for (int j = 0; j < VEC; ++j) v[j] = v[j] * sc + sf;
    }
    store_vec<T, VEC>(y + e, v);
  }
}

// ---------------------------------------------------------------- backward
template <typename T, int VEC>
__global__ void __launch_bounds__(256) bn_bwd_kernel(int64_t total, int C, int64_t hw, int layout,
                                                     BnParams p, const T* __restrict__ g,
                                                     const T* __restrict__ x, T* __restrict__ dx,
                                                     float* __restrict__ acc_dw,
                                                     float* __restrict__ acc_db) {
  extern __shared__ float sh[];
  float* s_scale = sh;
  float* s_inv = sh + C;
  float* s_mean = sh + 2 * C;
  float* s_dw = sh + 3 * C;
  float* s_db = sh + 4 * C;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float sc, sf, inv, mu;
    bn_channel_consts(p, c, sc, sf, inv, mu);
    s_scale[c] = sc;
    s_inv[c] = inv;
    s_mean[c] = mu;
    s_dw[c] = 0.f;
    s_db[c] = 0.f;
  }
  __syncthreads();
  const bool want_dw = acc_dw != nullptr, want_db = acc_db != nullptr, want_dx = dx != nullptr;
  const int64_t nvec = total / VEC;
  // Per-thread partials; NHWC threads keep a fixed channel group when the
  // grid stride is a multiple of C/VEC (host arranges it), otherwise flush.
  float pdw[VEC], pdb[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) pdw[j] = pdb[j] = 0.f;
  int cur_c = -1;
  auto flush = [&](int c0) {
    if (c0 < 0) return;
    if (layout == MS_NHWC) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        if (want_dw) atomicAdd(&s_dw[c0 + j], pdw[j]);
        if (want_db) atomicAdd(&s_db[c0 + j], pdb[j]);
      }
    } else {
      float a = 0.f, b = 0.f;
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        a += pdw[j];
        b += pdb[j];
      }
      if (want_dw) atomicAdd(&s_dw[c0], a);
      if (want_db) atomicAdd(&s_db[c0], b);
    }
#pragma unroll
    for (int j = 0; j < VEC; ++j) pdw[j] = pdb[j] = 0.f;
  };
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * VEC;
    const int c0 = layout == MS_NHWC ? (int)(e % C) : (int)((e / hw) % C);
    if (c0 != cur_c) {
      flush(cur_c);
      cur_c = c0;
    }
    float gv[VEC];
    load_vec<T, VEC>(g + e, gv);
    if (want_dx) {
      float o[VEC];
#pragma unroll
      for (int j = 0; j < VEC; ++j) o[j] = gv[j] * s_scale[layout == MS_NHWC ? c0 + j : c0];
      store_vec<T, VEC>(dx + e, o);
    }
    if (want_db) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) pdb[j] += gv[j];
    }
    if (want_dw) {
      float xv[VEC];
      load_vec<T, VEC>(x + e, xv);
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        const int c = layout == MS_NHWC ? c0 + j : c0;
        pdw[j] += gv[j] * (xv[j] - s_mean[c]) * s_inv[c];
      }
    }
  }
  flush(cur_c);
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    if (want_dw) atomicAdd(acc_dw + c, s_dw[c]);
    if (want_db) atomicAdd(acc_db + c, s_db[c]);
  }
}

// ---------------------------------------------------------------- NHWC fast paths
// Thread (rl, grp): channel group grp (VEC channels) of rows rl, rl+RPB, ...;
// per-channel constants live in registers, each thread keeps UNR 16-byte
// loads in flight (memory-level parallelism for HBM).
constexpr int BN_UNR = 4;
constexpr int BN_FWD_UNR = 6;  // 8 spilled under the 3-block register cap
constexpr int BN_BWD_UNR = 4, BN_BWD_UNR_DW = 5;

template <typename T, int VEC, bool RES = false, int U = BN_FWD_UNR>
__global__ void __launch_bounds__(256, RES ? 2 : 3) bn_fwd_nhwc_kernel(int64_t rows, int C, BnParams p,
                                                          const T* __restrict__ x,
                                                          T* __restrict__ y,
                                                          uint8_t* __restrict__ relu_mask = nullptr,
                                                          int relu = 0,
                                                          const T* __restrict__ resid = nullptr) {
  // relu: y = max(bn(x) [+ resid], 0) and (when relu_mask) its keep bits, one
  // byte per 8 channels of a pixel (storage order, as ms_relu_fwd; VEC == 8)
  const int G = C / VEC;
  const int rpb = 256 / G;
  const int tid = threadIdx.x;
  if (tid >= rpb * G) return;
  const int grp = tid % G, rl = tid / G;
  float sc[VEC], sf[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    float inv, mu;
    bn_channel_consts(p, grp * VEC + j, sc[j], sf[j], inv, mu);
  }
  // raw 16-byte loads held packed (4 registers per row, not 8 floats), so
  // BN_FWD_UNR rows per operand are in flight per thread before any store
  static_assert(VEC * sizeof(T) == 16, "bn_fwd_nhwc: 16-byte vectors");
  const int64_t step = (int64_t)gridDim.x * rpb;
  for (int64_t r0 = (int64_t)blockIdx.x * rpb + rl; r0 < rows; r0 += step * U) {
    uint4 raw[U], rraw[RES ? U : 1];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * step;
      if (r < rows) {
        raw[u] = __ldcs(reinterpret_cast<const uint4*>(x + r * C + grp * VEC));
        if constexpr (RES)
          rraw[u] = __ldcs(reinterpret_cast<const uint4*>(resid + r * C + grp * VEC));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * step;
      if (r < rows) {
        const T* xe = reinterpret_cast<const T*>(&raw[u]);
        const T* re = reinterpret_cast<const T*>(&rraw[RES ? u : 0]);
        float v[VEC];
        uint32_t bits = 0;
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          v[j] = IO<T>::ld(xe + j) * sc[j] + sf[j];
          if constexpr (RES) {
            // round the BN output first: the unfused chain adds two stored tensors
            T t = IO<T>::cvt(v[j]);
            v[j] = IO<T>::ld(&t) + IO<T>::ld(re + j);
          }
          if (relu) {
            const bool pos = !(v[j] <= 0.f);  // NaN propagates, as ms_relu_fwd
            bits |= (pos ? 1u : 0u) << j;
            v[j] = pos ? v[j] : 0.f;
          }
        }
        store_vec<T, VEC>(y + r * C + grp * VEC, v);
        if (relu_mask) relu_mask[(r * C + grp * VEC) / 8] = static_cast<uint8_t>(bits);
      }
    }
  }
}

template <typename T, int VEC, bool WANT_DW, int U = (WANT_DW ? BN_BWD_UNR_DW : BN_BWD_UNR)>
__global__ void __launch_bounds__(256, WANT_DW ? 2 : 3) bn_bwd_nhwc_kernel(int64_t rows, int C, BnParams p,
                                                          const T* __restrict__ g,
                                                          const T* __restrict__ x,
                                                          T* __restrict__ dx,
                                                          float* __restrict__ acc_dw,
                                                          float* __restrict__ acc_db,
                                                          const uint8_t* __restrict__ keep = nullptr,
                                                          T* __restrict__ gkeep = nullptr,
                                                          void* dw_out = nullptr,
                                                          void* db_out = nullptr,
                                                          unsigned* ticket = nullptr) {
  // keep (nullable, VEC == 8): the following ReLU's mask, g := keep ? g : 0 first;
  // gkeep (nullable): that masked g stored too (the residual operand's gradient)
  __shared__ float s_dw[2048], s_db[2048];
  const int G = C / VEC;
  const int rpb = 256 / G;
  const int tid = threadIdx.x;
  for (int c = tid; c < C; c += 256) s_dw[c] = s_db[c] = 0.f;
  __syncthreads();
  const bool want_dw = WANT_DW, want_db = acc_db != nullptr, want_dx = dx != nullptr;
  if (tid < rpb * G) {
    const int grp = tid % G, rl = tid / G;
    float sc[VEC], inv[VEC], mu[VEC], pdw[VEC], pdb[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      float sf;
      bn_channel_consts(p, grp * VEC + j, sc[j], sf, inv[j], mu[j]);
      pdw[j] = pdb[j] = 0.f;
    }
    const int64_t step = (int64_t)gridDim.x * rpb;
    // raw 16-byte loads held packed until used (see bn_fwd_nhwc_kernel)
    static_assert(VEC * sizeof(T) == 16, "bn_bwd_nhwc: 16-byte vectors");
    for (int64_t r0 = (int64_t)blockIdx.x * rpb + rl; r0 < rows; r0 += step * U) {
      uint4 graw[U], xraw[WANT_DW ? U : 1];
      uint32_t kb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t r = r0 + u * step;
        kb[u] = 0xffu;
        if (r < rows) {
          graw[u] = __ldcs(reinterpret_cast<const uint4*>(g + r * C + grp * VEC));
          if constexpr (WANT_DW)
            xraw[u] = __ldcs(reinterpret_cast<const uint4*>(x + r * C + grp * VEC));
          if (keep) kb[u] = keep[(r * C + grp * VEC) / 8];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t r = r0 + u * step;
        if (r >= rows) continue;
        const T* ge = reinterpret_cast<const T*>(&graw[u]);
        const T* xe = reinterpret_cast<const T*>(&xraw[WANT_DW ? u : 0]);
        float gv[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) gv[j] = ((kb[u] >> j) & 1u) ? IO<T>::ld(ge + j) : 0.f;
        if (gkeep) store_vec<T, VEC>(gkeep + r * C + grp * VEC, gv);
        if (want_dx) {
          float o[VEC];
#pragma unroll
          for (int j = 0; j < VEC; ++j) o[j] = gv[j] * sc[j];
          store_vec<T, VEC>(dx + r * C + grp * VEC, o);
        }
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          pdb[j] += gv[j];
          if constexpr (WANT_DW) pdw[j] += gv[j] * (IO<T>::ld(xe + j) - mu[j]) * inv[j];
        }
      }
    }
    if (want_dw || want_db) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        if (want_dw) atomicAdd(&s_dw[grp * VEC + j], pdw[j]);
        if (want_db) atomicAdd(&s_db[grp * VEC + j], pdb[j]);
      }
    }
  }
  if (want_dw || want_db) {
    __syncthreads();
    for (int c = tid; c < C; c += 256) {
      if (want_dw) atomicAdd(acc_dw + c, s_dw[c]);
      if (want_db) atomicAdd(acc_db + c, s_db[c]);
    }
    if (ticket) {
      // the last block to finish converts the fp32 sums to the parameter dtype
      // (no separate f32_to launch; the ticket is zeroed with the accumulators)
      __shared__ bool last;
      __threadfence();
      __syncthreads();
      if (tid == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
      __syncthreads();
      if (last) {
        __threadfence();
        for (int c = tid; c < C; c += 256) {
          if (want_dw) store_from_float(dw_out, p.pdtype, c, __ldcg(acc_dw + c));
          if (want_db) store_from_float(db_out, p.pdtype, c, __ldcg(acc_db + c));
        }
      }
    }
  }
}

#define MS_DT_DISPATCH(dt, ...)                                    \
  switch (dt) {                                                    \
    case MS_F32: { using T = float; __VA_ARGS__; } break;          \
    case MS_BF16: { using T = __nv_bfloat16; __VA_ARGS__; } break; \
    case MS_F16: { using T = __half; __VA_ARGS__; } break;         \
    default: set_error("bad dtype %d", dt); return MS_ERR_DTYPE;   \
  }

static bool can_vec(int64_t c, int64_t hw, int layout, int vec, const void* a, const void* b,
                    const void* d) {
  auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (!al(a) || (b && !al(b)) || (d && !al(d))) return false;
  return layout == MS_NHWC ? (c % vec == 0) : (hw % vec == 0);
}

// NHWC: choose a grid whose thread stride is a multiple of C/VEC so that each
// thread keeps one channel group for the whole sweep.
static int bn_grid(int64_t nvec, int64_t C, int layout, int vec) {
  int64_t blocks = (int64_t)num_sms() * 4;
  if (layout == MS_NHWC) {
    const int64_t groups = C / vec;
    // total threads = blocks*256 -> make it a multiple of `groups`
    int64_t a = groups, b = 256;
    while (b) { const int64_t t = a % b; a = b; b = t; }
    const int64_t lcm_blocks = groups / a;
    if (lcm_blocks > 0) blocks = ((blocks + lcm_blocks - 1) / lcm_blocks) * lcm_blocks;
  }
  const int64_t need = (nvec + 255) / 256;
  if (blocks > need) blocks = need > 0 ? need : 1;
  return (int)blocks;
}

// rows of an NHWC tensor, G channel groups per row: 256/G rows per block pass
// occ: resident blocks per SM of the kernel (its __launch_bounds__ minimum,
// which its register count meets exactly).  One wave: every thread loops over
// rows, so the per-channel constants and the dW/db block reduction (2C global
// atomics per block) are paid once per resident block, not once per 4 rows.
// dW/db accumulators (ws = [dw | db], fp32) to the parameter dtype: one
// launch when the caller's outputs are adjacent too (the host's (2, C) buffer)
static ms_status store_dw_db(const float* acc_dw, const float* acc_db, void* dw, void* db,
                             int pdtype, int64_t c, cudaStream_t st) {
  if (dw && db && acc_db == acc_dw + c &&
      static_cast<char*>(db) == static_cast<char*>(dw) + c * dtype_size(pdtype))
    return f32_to(acc_dw, dw, pdtype, 2 * c, nullptr, 1, st);
  if (dw) MS_TRY(f32_to(acc_dw, dw, pdtype, c, nullptr, 1, st));
  if (db) MS_TRY(f32_to(acc_db, db, pdtype, c, nullptr, 1, st));
  return MS_OK;
}

static int bn_fwd_unr() {
  static const int u = [] {
    const char* e = getenv("MS_BN_FWD_UNR");
    return e && atoi(e) == 4 ? 4 : BN_FWD_UNR;
  }();
  return u;
}

static int nhwc_grid(int64_t rows, int64_t G, int occ, int unr = BN_UNR) {
  static const int waves = [] {
    const char* e = getenv("MS_BN_WAVES");
    return e ? atoi(e) : 1;
  }();
  const int64_t rpb = 256 / G;
  int64_t need = (rows + rpb * unr - 1) / (rpb * unr);
  const int64_t cap = (int64_t)num_sms() * occ * (waves > 0 ? waves : 1);
  if (need > cap) need = cap;
  return (int)(need > 0 ? need : 1);
}

// [dw | db] fp32 accumulators, then the finalize ticket of bn_bwd_nhwc_kernel
size_t bn_eval_workspace_bytes(int64_t c) { return sizeof(float) * 2 * (size_t)c + 16; }

ms_status bn_eval_fwd(int64_t n, int64_t c, int64_t hw, int layout, int dt, const BnParams& p,
                      const void* x, void* y, cudaStream_t st) {
  const int64_t total = n * c * hw;
  if (total == 0) return MS_OK;
  MS_CHECK_ARG(c <= 8192, MS_ERR_UNSUPPORTED, "batchnorm: C=%lld > 8192", (long long)c);
  const size_t smem = sizeof(float) * 2 * c;
  MS_DT_DISPATCH(dt, {
    constexpr int V = 16 / sizeof(T);
    if (layout == MS_NHWC && can_vec(c, hw, layout, V, x, y, nullptr) && c / V <= 256) {
      const int64_t rows = n * hw;
      if (bn_fwd_unr() == 4)
        bn_fwd_nhwc_kernel<T, V, false, 4><<<nhwc_grid(rows, c / V, 3, 4), 256, 0, st>>>(
            rows, (int)c, p, (const T*)x, (T*)y);
      else
        bn_fwd_nhwc_kernel<T, V><<<nhwc_grid(rows, c / V, 3, BN_FWD_UNR), 256, 0, st>>>(
            rows, (int)c, p, (const T*)x, (T*)y);
    } else if (can_vec(c, hw, layout, V, x, y, nullptr)) {
      bn_fwd_kernel<T, V><<<bn_grid(total / V, c, layout, V), 256, smem, st>>>(
          total, (int)c, hw, layout, p, (const T*)x, (T*)y);
    } else {
      bn_fwd_kernel<T, 1><<<bn_grid(total, c, layout, 1), 256, smem, st>>>(
          total, (int)c, hw, layout, p, (const T*)x, (T*)y);
    }
  });
  count_launch(1, KF_BN);
  return launch_status("bn_fwd_kernel");
}

// BN-eval -> ReLU in one pass (NHWC, 16-bit, C % 8 == 0, C <= 2048): the
// chain kept unfused around the conv when BN's affine is trainable
ms_status bn_relu_eval_fwd(int64_t n, int64_t c, int64_t hw, int dt, const BnParams& p,
                           const void* x, const void* resid, void* y, uint8_t* mask,
                           cudaStream_t st) {
  const int64_t rows = n * hw;
  MS_CHECK_ARG(dtype_size(dt) == 2 && c % 8 == 0 && c <= 2048, MS_ERR_UNSUPPORTED,
               "bn+relu: 16-bit NHWC with C %% 8 == 0 only");
  if (rows == 0) return MS_OK;
  auto go = [&](auto tag) {
    using T = decltype(tag);
    const bool u4 = bn_fwd_unr() == 4;
    const int gr = nhwc_grid(rows, c / 8, resid ? 2 : 3, u4 ? 4 : BN_FWD_UNR);
    if (resid && u4)
      bn_fwd_nhwc_kernel<T, 8, true, 4><<<gr, 256, 0, st>>>(
          rows, (int)c, p, (const T*)x, (T*)y, mask, 1, (const T*)resid);
    else if (resid)
      bn_fwd_nhwc_kernel<T, 8, true><<<gr, 256, 0, st>>>(
          rows, (int)c, p, (const T*)x, (T*)y, mask, 1, (const T*)resid);
    else if (u4)
      bn_fwd_nhwc_kernel<T, 8, false, 4><<<gr, 256, 0, st>>>(
          rows, (int)c, p, (const T*)x, (T*)y, mask, 1);
    else
      bn_fwd_nhwc_kernel<T, 8><<<gr, 256, 0, st>>>(rows, (int)c, p, (const T*)x, (T*)y, mask, 1);
  };
  if (dt == MS_BF16) go(__nv_bfloat16{});
  else go(__half{});
  count_launch(1, KF_BN);
  return launch_status("bn_fwd_nhwc_kernel (relu)");
}

ms_status bn_relu_eval_bwd(int64_t n, int64_t c, int64_t hw, int dt, const BnParams& p,
                           const void* g, const uint8_t* keep, const void* x, void* dx,
                           void* dresid, void* dw, void* db, void* ws, size_t ws_bytes,
                           cudaStream_t st) {
  const int64_t rows = n * hw;
  MS_CHECK_ARG(dtype_size(dt) == 2 && c % 8 == 0 && c <= 2048 && keep, MS_ERR_UNSUPPORTED,
               "bn+relu bwd: 16-bit NHWC with C %% 8 == 0 and a mask only");
  MS_CHECK_ARG(!(dw && !x), MS_ERR_SHAPE, "bn+relu bwd: dw requested without x");
  float* acc_dw = nullptr;
  float* acc_db = nullptr;
  if (dw || db) {
    MS_CHECK_ARG(ws && ws_bytes >= bn_eval_workspace_bytes(c), MS_ERR_WORKSPACE,
                 "bn+relu bwd workspace too small");
    cudaMemsetAsync(ws, 0, bn_eval_workspace_bytes(c), st);
    if (dw) acc_dw = static_cast<float*>(ws);
    if (db) acc_db = static_cast<float*>(ws) + c;
  }
  if (rows > 0 && (dx || dresid || dw || db)) {
    auto go = [&](auto tag) {
      using T = decltype(tag);
      unsigned* tk = (dw || db) ? reinterpret_cast<unsigned*>(static_cast<float*>(ws) + 2 * c)
                                : nullptr;
      if (dw)
        bn_bwd_nhwc_kernel<T, 8, true><<<nhwc_grid(rows, c / 8, 2, BN_BWD_UNR_DW), 256, 0, st>>>(
            rows, (int)c, p, (const T*)g, (const T*)x, (T*)dx, acc_dw, acc_db, keep,
            (T*)dresid, dw, db, tk);
      else
        bn_bwd_nhwc_kernel<T, 8, false><<<nhwc_grid(rows, c / 8, 3, BN_BWD_UNR), 256, 0, st>>>(
            rows, (int)c, p, (const T*)g, (const T*)x, (T*)dx, acc_dw, acc_db, keep,
            (T*)dresid, dw, db, tk);
    };
    if (dt == MS_BF16) go(__nv_bfloat16{});
    else go(__half{});
    count_launch(1, KF_BN);
    MS_TRY(launch_status("bn_bwd_nhwc_kernel (relu)"));
    return MS_OK;  // dW / db converted by the kernel's last block
  }
  return store_dw_db(acc_dw, acc_db, dw, db, p.pdtype, c, st);
  return MS_OK;
}

ms_status bn_eval_bwd(int64_t n, int64_t c, int64_t hw, int layout, int dt, const BnParams& p,
                      const void* g, const void* x, void* dx, void* dw, void* db, void* ws,
                      size_t ws_bytes, cudaStream_t st) {
  const int64_t total = n * c * hw;
  MS_CHECK_ARG(c <= 8192, MS_ERR_UNSUPPORTED, "batchnorm: C=%lld > 8192", (long long)c);
  MS_CHECK_ARG(!(dw && !x), MS_ERR_SHAPE, "batchnorm bwd: dw requested without x");
  float* acc_dw = nullptr;
  float* acc_db = nullptr;
  if (dw || db) {
    MS_CHECK_ARG(ws && ws_bytes >= bn_eval_workspace_bytes(c), MS_ERR_WORKSPACE,
                 "batchnorm bwd workspace too small");
    cudaMemsetAsync(ws, 0, bn_eval_workspace_bytes(c), st);
    if (dw) acc_dw = static_cast<float*>(ws);
    if (db) acc_db = static_cast<float*>(ws) + c;
  }
  bool fused_store = false;  // dW / db converted by the NHWC kernel's last block
  if (total > 0 && (dx || dw || db)) {
    const size_t smem = sizeof(float) * 5 * c;
    MS_DT_DISPATCH(dt, {
      constexpr int V = 16 / sizeof(T);
      if (layout == MS_NHWC && can_vec(c, hw, layout, V, g, dw ? x : nullptr, dx) &&
          c / V <= 256 && c <= 2048) {
        const int64_t rows = n * hw;
        unsigned* tk = (dw || db) ? reinterpret_cast<unsigned*>(static_cast<float*>(ws) + 2 * c)
                                  : nullptr;
        if (dw)
          bn_bwd_nhwc_kernel<T, V, true><<<nhwc_grid(rows, c / V, 2, BN_BWD_UNR_DW), 256, 0, st>>>(
              rows, (int)c, p, (const T*)g, (const T*)x, (T*)dx, acc_dw, acc_db, nullptr,
              nullptr, dw, db, tk);
        else
          bn_bwd_nhwc_kernel<T, V, false><<<nhwc_grid(rows, c / V, 3, BN_BWD_UNR), 256, 0, st>>>(
              rows, (int)c, p, (const T*)g, (const T*)x, (T*)dx, acc_dw, acc_db, nullptr,
              nullptr, dw, db, tk);
        fused_store = true;
      } else if (can_vec(c, hw, layout, V, g, dw ? x : nullptr, dx)) {
        bn_bwd_kernel<T, V><<<bn_grid(total / V, c, layout, V), 256, smem, st>>>(
            total, (int)c, hw, layout, p, (const T*)g, (const T*)x, (T*)dx, acc_dw, acc_db);
      } else {
        bn_bwd_kernel<T, 1><<<bn_grid(total, c, layout, 1), 256, smem, st>>>(
            total, (int)c, hw, layout, p, (const T*)g, (const T*)x, (T*)dx, acc_dw, acc_db);
      }
    });
    count_launch(1, KF_BN);
    MS_TRY(launch_status("bn_bwd_kernel"));
  }
  if (fused_store) return MS_OK;
  return store_dw_db(acc_dw, acc_db, dw, db, p.pdtype, c, st);
  return MS_OK;
}

}  // namespace ms

// ---------------------------------------------------------------- C ABI
extern "C" size_t ms_bn_eval_workspace(int64_t n, int64_t c, int64_t hw, int32_t layout) {
  (void)n;
  (void)hw;
  (void)layout;
  return ms::bn_eval_workspace_bytes(c);
}

extern "C" ms_status ms_bn_eval_fwd(int64_t n, int64_t c, int64_t hw, int32_t layout, int32_t dtype,
                                    int32_t pdtype, const void* x, const void* mean,
                                    const void* var, const void* weight, const void* bias,
                                    double eps, void* y, void* ws, size_t ws_bytes, void* stream) {
  MS_TRY(ms::bind_device(y));
  (void)ws;
  (void)ws_bytes;
  MS_CHECK_ARG(n >= 0 && c > 0 && hw >= 0, MS_ERR_SHAPE, "batchnorm: bad shape");
  MS_CHECK_ARG(x && y && mean && var, MS_ERR_SHAPE, "batchnorm: null tensor");
  ms::BnParams p{mean, var, weight, bias, pdtype, (float)eps};
  return ms::bn_eval_fwd(n, c, hw, layout, dtype, p, x, y, (cudaStream_t)stream);
}

extern "C" ms_status ms_bn_eval_bwd(int64_t n, int64_t c, int64_t hw, int32_t layout,
                                    int32_t dtype, int32_t pdtype, const void* dy,
                                    const void* x_or_null, const void* mean, const void* var,
                                    const void* weight, double eps, void* dx_or_null,
                                    void* dw_or_null, void* db_or_null, void* ws, size_t ws_bytes,
                                    void* stream) {
  MS_TRY(ms::bind_device(dy));
  MS_CHECK_ARG(n >= 0 && c > 0 && hw >= 0, MS_ERR_SHAPE, "batchnorm: bad shape");
  MS_CHECK_ARG(dy && mean && var, MS_ERR_SHAPE, "batchnorm bwd: null tensor");
  ms::BnParams p{mean, var, weight, nullptr, pdtype, (float)eps};
  return ms::bn_eval_bwd(n, c, hw, layout, dtype, p, dy, x_or_null, dx_or_null, dw_or_null,
                         db_or_null, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" ms_status ms_bn_eval_relu_fwd(int64_t n, int64_t c, int64_t hw, int32_t dtype,
                                         int32_t pdtype, const void* x, const void* mean,
                                         const void* var, const void* weight, const void* bias,
                                         double eps, void* y, void* mask_or_null, void* stream) {
  MS_TRY(ms::bind_device(y));
  MS_CHECK_ARG(n >= 0 && c > 0 && hw >= 0, MS_ERR_SHAPE, "bn+relu: bad shape");
  MS_CHECK_ARG(x && y && mean && var, MS_ERR_SHAPE, "bn+relu: null tensor");
  ms::BnParams p{mean, var, weight, bias, pdtype, (float)eps};
  return ms::bn_relu_eval_fwd(n, c, hw, dtype, p, x, nullptr, y,
                              static_cast<uint8_t*>(mask_or_null), (cudaStream_t)stream);
}

extern "C" ms_status ms_bn_eval_add_relu_fwd(int64_t n, int64_t c, int64_t hw, int32_t dtype,
                                             int32_t pdtype, const void* x, const void* residual,
                                             const void* mean, const void* var,
                                             const void* weight, const void* bias, double eps,
                                             void* y, void* mask_or_null, void* stream) {
  MS_TRY(ms::bind_device(y));
  MS_CHECK_ARG(n >= 0 && c > 0 && hw >= 0, MS_ERR_SHAPE, "bn+add+relu: bad shape");
  MS_CHECK_ARG(x && residual && y && mean && var, MS_ERR_SHAPE, "bn+add+relu: null tensor");
  ms::BnParams p{mean, var, weight, bias, pdtype, (float)eps};
  return ms::bn_relu_eval_fwd(n, c, hw, dtype, p, x, residual, y,
                              static_cast<uint8_t*>(mask_or_null), (cudaStream_t)stream);
}

extern "C" ms_status ms_bn_eval_relu_bwd(int64_t n, int64_t c, int64_t hw, int32_t dtype,
                                         int32_t pdtype, const void* dy, const void* mask,
                                         const void* x_or_null, const void* mean, const void* var,
                                         const void* weight, double eps, void* dx_or_null,
                                         void* dw_or_null, void* db_or_null, void* ws,
                                         size_t ws_bytes, void* stream) {
  MS_TRY(ms::bind_device(dy));
  MS_CHECK_ARG(n >= 0 && c > 0 && hw >= 0, MS_ERR_SHAPE, "bn+relu bwd: bad shape");
  MS_CHECK_ARG(dy && mask && mean && var, MS_ERR_SHAPE, "bn+relu bwd: null tensor");
  ms::BnParams p{mean, var, weight, nullptr, pdtype, (float)eps};
  return ms::bn_relu_eval_bwd(n, c, hw, dtype, p, dy, static_cast<const uint8_t*>(mask),
                              x_or_null, dx_or_null, nullptr, dw_or_null, db_or_null, ws,
                              ws_bytes, (cudaStream_t)stream);
}

extern "C" ms_status ms_bn_eval_add_relu_bwd(int64_t n, int64_t c, int64_t hw, int32_t dtype,
                                             int32_t pdtype, const void* dy, const void* mask,
                                             const void* x_or_null, const void* mean,
                                             const void* var, const void* weight, double eps,
                                             void* dx_or_null, void* dresidual_or_null,
                                             void* dw_or_null, void* db_or_null, void* ws,
                                             size_t ws_bytes, void* stream) {
  MS_TRY(ms::bind_device(dy));
  MS_CHECK_ARG(n >= 0 && c > 0 && hw >= 0, MS_ERR_SHAPE, "bn+add+relu bwd: bad shape");
  MS_CHECK_ARG(dy && mask && mean && var, MS_ERR_SHAPE, "bn+add+relu bwd: null tensor");
  ms::BnParams p{mean, var, weight, nullptr, pdtype, (float)eps};
  return ms::bn_relu_eval_bwd(n, c, hw, dtype, p, dy, static_cast<const uint8_t*>(mask),
                              x_or_null, dx_or_null, dresidual_or_null, dw_or_null, db_or_null,
                              ws, ws_bytes, (cudaStream_t)stream);
}

// ---------------------------------------------------------------- BN-eval + ReLU backward
// dx = g * keep * scale_c for the fused conv + BN-eval (+ ReLU) forward
// (NHWC, C % 8 == 0): one mask byte = 8 consecutive channels of one pixel
namespace ms {
namespace {
template <typename T>
__global__ void __launch_bounds__(256) bn_relu_bwd_kernel(int64_t groups, int C, BnParams p,
                                                          const T* __restrict__ g,
                                                          const uint8_t* __restrict__ mask,
                                                          T* __restrict__ dx) {
  extern __shared__ float s_scale[];
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float sc, sf, inv, mu;
    bn_channel_consts(p, c, sc, sf, inv, mu);
    s_scale[c] = sc;
  }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g0 < groups;
       g0 += stride * BN_UNR) {
    float v[BN_UNR][8];
    uint32_t bits[BN_UNR];
#pragma unroll
    for (int u = 0; u < BN_UNR; ++u) {
      const int64_t gi = g0 + u * stride;
      if (gi < groups) {
        load_vec<T, 8>(g + gi * 8, v[u]);
        bits[u] = mask ? mask[gi] : 0xFFu;
      }
    }
#pragma unroll
    for (int u = 0; u < BN_UNR; ++u) {
      const int64_t gi = g0 + u * stride;
      if (gi >= groups) continue;
      const int c0 = (int)((gi * 8) % C);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[u][j] = (bits[u] >> j) & 1u ? v[u][j] * s_scale[c0 + j] : 0.f;
      store_vec<T, 8>(dx + gi * 8, v[u]);
    }
  }
}
}  // namespace
}  // namespace ms

extern "C" ms_status ms_bn_relu_bwd(int64_t numel, int64_t c, int32_t dtype, int32_t pdtype,
                                    const void* g, const void* mask_or_null, const void* mean,
                                    const void* var, const void* weight, double eps, void* dx,
                                    void* stream) {
  MS_TRY(ms::bind_device(dx));
  MS_CHECK_ARG(numel >= 0 && c > 0 && c % 8 == 0 && c <= 8192 && numel % c == 0, MS_ERR_SHAPE,
               "bn_relu_bwd: NHWC with C %% 8 == 0 required");
  MS_CHECK_ARG(dtype == MS_BF16 || dtype == MS_F16, MS_ERR_DTYPE, "bn_relu_bwd: 16-bit only");
  MS_CHECK_ARG(((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(dx)) & 15) == 0,
               MS_ERR_ALIGN, "bn_relu_bwd: 16-byte alignment");
  if (numel == 0) return MS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  ms::BnParams p{mean, var, weight, nullptr, pdtype, (float)eps};
  const int64_t groups = numel / 8;
  int64_t blocks = (groups + 255) / 256;
  if (blocks > (int64_t)ms::num_sms() * 8) blocks = (int64_t)ms::num_sms() * 8;
  const size_t smem = sizeof(float) * c;
  if (dtype == MS_BF16)
    ms::bn_relu_bwd_kernel<__nv_bfloat16><<<(unsigned)blocks, 256, smem, st>>>(
        groups, (int)c, p, (const __nv_bfloat16*)g, (const uint8_t*)mask_or_null,
        (__nv_bfloat16*)dx);
  else
    ms::bn_relu_bwd_kernel<__half><<<(unsigned)blocks, 256, smem, st>>>(
        groups, (int)c, p, (const __half*)g, (const uint8_t*)mask_or_null, (__half*)dx);
  ms::count_launch(1, ms::KF_BN);
  return ms::launch_status("bn_relu_bwd");
}
