// Host plumbing: status/error strings, SM count cache, tensor-map encoders,
// umma_gemm dispatch.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>

#include "host.cuh"

namespace ms {

std::atomic<int64_t> g_launches{0};
std::atomic<int64_t> g_family[KF_COUNT];

static thread_local char t_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_err, sizeof(t_err), fmt, ap);
  va_end(ap);
}

const char* last_error() { return t_err; }

ms_status launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return MS_ERR_LAUNCH;
  }
  return MS_OK;
}

static thread_local int t_device_bound = 0;
void set_device_bound(int on) { t_device_bound = on; }

ms_status bind_device(const void* p) {
  if (t_device_bound > 0) {
    // ms_set_device_bound(dev + 1): the caller named the device; no pointer query.
    // cudaSetDevice still runs: it makes the device's primary context current on
    // this thread (an autograd worker thread may have none yet, and the tensor-map
    // encoders are driver calls)
    if (cudaSetDevice(t_device_bound - 1) != cudaSuccess) {
      set_error("cudaSetDevice(%d) failed", t_device_bound - 1);
      cudaGetLastError();
      return MS_ERR_LAUNCH;
    }
    return MS_OK;
  }
  // The autograd engine calls backward on its own device thread, where neither
  // this library's runtime nor the driver API has a current context yet: bind
  // the device that owns the operand before any driver call (tensor-map
  // encoding) or launch.
  int dev = -1;
  if (p != nullptr) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeDevice)
      dev = a.device;
    else
      cudaGetLastError();
  }
  if (dev < 0) cudaGetDevice(&dev);
  if (cudaSetDevice(dev) != cudaSuccess) {
    set_error("cudaSetDevice(%d) failed", dev);
    cudaGetLastError();
    return MS_ERR_LAUNCH;
  }
  return MS_OK;
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

// ------------------------------------------------------------------ tensor maps
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                       const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                       const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion,
                                       CUtensorMapFloatOOBfill);
typedef CUresult (*PFN_encodeIm2col_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                        const cuuint64_t*, const cuuint64_t*, const int*,
                                        const int*, cuuint32_t, cuuint32_t, const cuuint32_t*,
                                        CUtensorMapInterleave, CUtensorMapSwizzle,
                                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t g_encode_tiled = nullptr;
static PFN_encodeIm2col_t g_encode_im2col = nullptr;
static int g_driver_version = 0;

static ms_status resolve_driver() {
  static std::once_flag once;
  static ms_status st = MS_OK;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr) {
      st = MS_ERR_LAUNCH;
      return;
    }
    g_encode_tiled = reinterpret_cast<PFN_encodeTiled_t>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr) {
      st = MS_ERR_LAUNCH;
      return;
    }
    g_encode_im2col = reinterpret_cast<PFN_encodeIm2col_t>(fn);
    cudaDriverGetVersion(&g_driver_version);
  });
  if (st != MS_OK) set_error("could not resolve cuTensorMapEncode* driver entry points");
  return st;
}

ms_status make_tmap_2d(CUtensorMap* m, int dt, const void* base, uint64_t inner, uint64_t outer,
                       uint64_t ld, uint32_t box_inner, uint32_t box_outer) {
  MS_TRY(resolve_driver());
  const size_t es = dtype_size(dt);
  MS_CHECK_ARG((reinterpret_cast<uintptr_t>(base) & 15) == 0, MS_ERR_ALIGN,
               "tensor base %p not 16-byte aligned", base);
  MS_CHECK_ARG((ld * es) % 16 == 0, MS_ERR_ALIGN, "row pitch %llu elems not a multiple of 16 B",
               (unsigned long long)ld);
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * es};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode_tiled(m, tma_dtype(dt), 2, const_cast<void*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MS_CHECK_ARG(r == CUDA_SUCCESS, MS_ERR_LAUNCH,
               "cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu ld=%llu box=%ux%u", (int)r,
               (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)ld,
               box_inner, box_outer);
  return MS_OK;
}

ms_status make_tmap_nd(CUtensorMap* m, int dt, const void* base, int rank, const uint64_t* dims,
                       const uint64_t* strides_bytes, const uint32_t* box, int swizzle) {
  MS_TRY(resolve_driver());
  MS_CHECK_ARG((reinterpret_cast<uintptr_t>(base) & 15) == 0, MS_ERR_ALIGN,
               "tensor base %p not 16-byte aligned", base);
  cuuint64_t d[5];
  cuuint64_t s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i + 1 < rank) s[i] = strides_bytes[i];
  }
  const CUtensorMapSwizzle sw = swizzle == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = g_encode_tiled(m, tma_dtype(dt), rank, const_cast<void*>(base), d, s, b, e,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MS_CHECK_ARG(r == CUDA_SUCCESS, MS_ERR_LAUNCH, "cuTensorMapEncodeTiled (rank %d) failed (%d)",
               rank, (int)r);
  return MS_OK;
}

ms_status make_tmap_im2col(CUtensorMap* m, int dt, const void* base, int n, int h, int w, int c,
                           const int lower[2], const int upper[2], int stride_w, int stride_h,
                           uint32_t channels, uint32_t pixels, bool swizzle128) {
  MS_TRY(resolve_driver());
  const size_t es = dtype_size(dt);
  MS_CHECK_ARG((reinterpret_cast<uintptr_t>(base) & 15) == 0, MS_ERR_ALIGN,
               "activation base %p not 16-byte aligned", base);
  MS_CHECK_ARG((c * es) % 16 == 0, MS_ERR_ALIGN, "channels*%zu must be a multiple of 16 B", es);
  cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)c * es, (cuuint64_t)c * w * es, (cuuint64_t)c * w * h * es};
  cuuint32_t estr[4] = {1, (cuuint32_t)stride_w, (cuuint32_t)stride_h, 1};
  CUresult r = g_encode_im2col(m, tma_dtype(dt), 4, const_cast<void*>(base), dims, strides, lower,
                               upper, channels, pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MS_CHECK_ARG(r == CUDA_SUCCESS, MS_ERR_LAUNCH,
               "cuTensorMapEncodeIm2col failed (%d): nhwc=%d,%d,%d,%d lower=(%d,%d) upper=(%d,%d) "
               "stride=(%d,%d) box=%ux%u",
               (int)r, n, h, w, c, lower[0], lower[1], upper[0], upper[1], stride_w, stride_h,
               channels, pixels);
  // Driver <= 13.1 mis-encodes one descriptor bit for small im2col tensors
  // (same workaround as CUTLASS make_im2col_tma_copy_desc).
  const uint64_t bytes = (uint64_t)n * h * w * c * es;
  if (g_driver_version <= 13010 && bytes < 131072)
    reinterpret_cast<uint64_t*>(m)[1] &= ~(1ull << 21);
  return MS_OK;
}

ms_status setup_tma_store(TmapPack& tm, GemmArgs& g, int dt, void* out, int64_t rows,
                          int64_t cols, int64_t ldc) {
  g.tma_store = 0;
  static const bool disabled = [] {
    const char* e = getenv("MS_TMA_STORE");
    return e && atoi(e) == 0;
  }();
  if (disabled || dt == MS_F32 || (reinterpret_cast<uintptr_t>(out) & 15) || (ldc * 2) % 16 ||
      rows <= 0 || cols <= 0)
    return MS_OK;
  const uint64_t dims[2] = {(uint64_t)cols, (uint64_t)rows};
  const uint64_t strides[1] = {(uint64_t)ldc * 2};
  const uint32_t box[2] = {32, 32};
  MS_TRY(make_tmap_nd(&tm.c, dt, out, 2, dims, strides, box, 64));
  if (g.epi.act_out) {
    if (reinterpret_cast<uintptr_t>(g.epi.act_out) & 15) return MS_OK;  // direct stores
    MS_TRY(make_tmap_nd(&tm.c2, dt, g.epi.act_out, 2, dims, strides, box, 64));
  }
  g.tma_store = 1;
  return MS_OK;
}

// programmatic dependent launch of the GEMM / conv kernels (MS_PDL=0: off)
static bool use_pdl() {
  static const bool on = [] {
    const char* e = getenv("MS_PDL");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

// ------------------------------------------------------------------ dispatch
template <int BN, int A_MN, int B_MN, int MODE, int CL = 1>
static ms_status launch_t(const TmapPack& tm, const GemmArgs& g, cudaStream_t st) {
  auto kern = umma_gemm_kernel<BN, A_MN, B_MN, MODE, CL>;
  constexpr int smem = GemmCfg<BN, A_MN, B_MN, MODE, CL>::SMEM_BYTES;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int sms = num_sms();
  if (g.num_tiles <= 0) return MS_OK;
  if constexpr (CL == 1) {
    const int grid = g.num_tiles < sms ? g.num_tiles : sms;
    const cudaError_t e = use_pdl()
        ? launch_pdl(kern, dim3(grid), dim3(GemmCfg<BN, A_MN, B_MN, MODE, CL>::THREADS), smem, st,
                     tm, g)
        : (kern<<<grid, GemmCfg<BN, A_MN, B_MN, MODE, CL>::THREADS, smem, st>>>(tm, g),
           cudaSuccess);
    if (e != cudaSuccess) {
      set_error("cudaLaunchKernelEx: %s", cudaGetErrorString(e));
      return MS_ERR_LAUNCH;
    }
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(GemmCfg<BN, A_MN, B_MN, MODE, CL>::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // persistent grid = the clusters that can be co-resident (GPCs with an odd
    // SM count leave one SM out of the pairs), not #SMs / 2
    static int max_clusters = 0;
    if (max_clusters == 0) {
      cfg.gridDim = dim3(sms / CL * CL);
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        n = sms / CL;
      }
      max_clusters = n;
    }
    const int clusters = g.num_tiles < max_clusters ? g.num_tiles : max_clusters;
    cfg.gridDim = dim3(clusters * CL);
    cfg.numAttrs = use_pdl() ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tm, g);
    if (e != cudaSuccess) {
      set_error("cudaLaunchKernelEx (cluster %d): %s", CL, cudaGetErrorString(e));
      return MS_ERR_LAUNCH;
    }
  }
  count_launch(1, KF_UMMA);
  return launch_status("umma_gemm_kernel");
}

#define MS_BN_SWITCH(A, B, M)                                   \
  switch (bn) {                                                 \
    case 32: return launch_t<32, A, B, M>(tm, g, st);           \
    case 64: return launch_t<64, A, B, M>(tm, g, st);           \
    case 128: return launch_t<128, A, B, M>(tm, g, st);         \
    case 192: return launch_t<192, A, B, M>(tm, g, st);         \
    case 256: return launch_t<256, A, B, M>(tm, g, st);         \
    default: break;                                             \
  }

ms_status launch_umma(int bn, int a_mn, int b_mn, int mode, const TmapPack& tm,
                      const GemmArgs& g, cudaStream_t st, int g_cluster) {
  if ((b_mn || mode == LOAD_CONV_WGRAD) && bn < 64) {
    set_error("launch_umma: MN-major B needs BN >= 64");
    return MS_ERR_UNSUPPORTED;
  }
  if (g_cluster == 2) {
    switch (bn) {
#define MS_CL2(BNV)                                                                       \
  case BNV:                                                                               \
    if (mode == LOAD_GEMM && !a_mn && !b_mn) return launch_t<BNV, 0, 0, LOAD_GEMM, 2>(tm, g, st); \
    if (mode == LOAD_GEMM && !a_mn && b_mn) return launch_t<BNV, 0, 1, LOAD_GEMM, 2>(tm, g, st);  \
    if (mode == LOAD_GEMM && a_mn && b_mn) return launch_t<BNV, 1, 1, LOAD_GEMM, 2>(tm, g, st);   \
    if (mode == LOAD_CONV_FPROP) return launch_t<BNV, 0, 0, LOAD_CONV_FPROP, 2>(tm, g, st);       \
    if (mode == LOAD_CONV_DGRAD) return launch_t<BNV, 0, 0, LOAD_CONV_DGRAD, 2>(tm, g, st);       \
    break;
      MS_CL2(128)
      MS_CL2(256)
#undef MS_CL2
      default: break;
    }
    set_error("launch_umma: no CTA-pair variant (bn=%d mode=%d)", bn, mode);
    return MS_ERR_UNSUPPORTED;
  }
  if (mode == LOAD_GEMM) {
    if (!a_mn && !b_mn) { MS_BN_SWITCH(0, 0, LOAD_GEMM) }
    if (!a_mn && b_mn) { MS_BN_SWITCH(0, 1, LOAD_GEMM) }
    if (a_mn && b_mn) { MS_BN_SWITCH(1, 1, LOAD_GEMM) }
  } else if (mode == LOAD_GEMM_3XTF32) {
    switch (bn) {
      case 128: return launch_t<128, 0, 0, LOAD_GEMM_3XTF32>(tm, g, st);
      default: break;
    }
  } else if (mode == LOAD_CONV_FPROP) {
    MS_BN_SWITCH(0, 0, LOAD_CONV_FPROP)
  } else if (mode == LOAD_CONV_DGRAD) {
    MS_BN_SWITCH(0, 0, LOAD_CONV_DGRAD)
  } else if (mode == LOAD_CONV_FPROP_C8) {
    MS_BN_SWITCH(0, 0, LOAD_CONV_FPROP_C8)
  } else if (mode == LOAD_CONV_FPROP_ROWSEG) {
    MS_BN_SWITCH(0, 0, LOAD_CONV_FPROP_ROWSEG)
  } else if (mode == LOAD_CONV_DGRAD_BAND) {
    if (bn == 160) return launch_t<160, 0, 0, LOAD_CONV_DGRAD_BAND>(tm, g, st);
  } else if (mode == LOAD_CONV_WGRAD) {
    switch (bn) {
      case 64: return launch_t<64, 1, 1, LOAD_CONV_WGRAD>(tm, g, st);
      case 192: return launch_t<192, 1, 1, LOAD_CONV_WGRAD>(tm, g, st);
      case 128: return launch_t<128, 1, 1, LOAD_CONV_WGRAD>(tm, g, st);
      case 256: return launch_t<256, 1, 1, LOAD_CONV_WGRAD>(tm, g, st);
      default: break;
    }
  }
  set_error("launch_umma: unsupported (bn=%d a_mn=%d b_mn=%d mode=%d)", bn, a_mn, b_mn, mode);
  return MS_ERR_UNSUPPORTED;
}

int pick_bn(int64_t other_tiles, int64_t ncols) {
  if (ncols <= 32) return 32;
  if (ncols <= 64) return 64;
  // Persistent CTAs take tiles round-robin, so a launch costs about
  // ceil(tiles / #SMs) tile-times; a tile costs ~ (BN + 64) column-units (the
  // constant is the per-tile epilogue / pipeline overhead).  Pick the cheapest.
  static const int cands[] = {256, 192, 128, 64};
  int best = 256;
  double best_cost = 1e30;
  for (int bn : cands) {
    if (bn > 128 && ncols <= 128) continue;
    const int64_t tiles = other_tiles * ((ncols + bn - 1) / bn);
    const int64_t waves = (tiles + num_sms() - 1) / num_sms();
    const double cost = (double)waves * (bn + 64);
    if (cost < best_cost * 0.97) {  // prefer the larger tile on near-ties
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

int pair_slots() {
  static int n = 0;
  if (n == 0) {
    auto kern = umma_gemm_kernel<256, 0, 0, LOAD_GEMM, 2>;
    constexpr int smem = GemmCfg<256, 0, 0, LOAD_GEMM, 2>::SMEM_BYTES;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(GemmCfg<256, 0, 0, LOAD_GEMM, 2>::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.gridDim = dim3(num_sms() / 2 * 2);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, kern, &cfg) != cudaSuccess || c <= 0) {
      cudaGetLastError();
      c = num_sms() / 2;
    }
    n = c;
  }
  return n;
}

TilePick pick_tiles(int64_t m_blocks, int64_t cols, bool allow_pair, bool b_mn) {
  static const int env_cl = [] {
    const char* e = getenv("MS_GEMM_CLUSTER");
    return e ? atoi(e) : 2;
  }();
  static const int env_bn = [] {
    const char* e = getenv("MS_GEMM_BN");
    return e ? atoi(e) : 0;
  }();
  // A persistent launch costs about ceil(tiles / slots) tile-times; a tile-time
  // ~ (BN + 64) column-units (the constant is the per-tile epilogue / pipeline
  // overhead), and a pair tile is ~0.7x a single tile per SM (half the B bytes
  // staged through shared memory).  The pair splits B in halves of BN/2 rows,
  // which the hardware accepts for BN in {128, 256} (96- and 32-row halves hang
  // the MMA), so those are the only pair widths.
  static const TilePick cands[] = {{2, 256}, {2, 128}, {1, 256}, {1, 192},
                                   {1, 128}, {1, 64},  {1, 32}};
  const int sms = num_sms();
  double best = 1e30;
  TilePick pick{1, 0};
  for (const TilePick& c : cands) {
    if (c.cl == 2 && (!allow_pair || env_cl != 2 || m_blocks < 2)) continue;
    if (env_bn && c.bn != env_bn) continue;
    if (b_mn && c.bn < 64) continue;
    if (c.bn > 128 && cols <= 128) continue;
    if (c.bn > 64 && cols <= 32) continue;
    if (c.bn > 32 && cols <= 16) continue;
    const int64_t mt = (m_blocks + c.cl - 1) / c.cl;
    const int64_t tiles = mt * ((cols + c.bn - 1) / c.bn);
    const int64_t slots = sms / c.cl;
    const int64_t waves = (tiles + slots - 1) / slots;
    const double cost = (double)waves * (c.bn + 64) * (c.cl == 2 ? 0.7 : 1.0);
    if (cost < best * 0.97) {  // candidates are ordered large-first: prefer them on near-ties
      best = cost;
      pick = c;
    }
  }
  if (pick.bn == 0) pick = TilePick{1, env_bn ? env_bn : (b_mn ? 64 : 32)};
  return pick;
}

}  // namespace ms
