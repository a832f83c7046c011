// Host-side helpers: TMA tensor-map encoding (driver entry points resolved at
// run time, so the library does not link libcuda), GEMM launch dispatch, and
// the launch counter behind ms_launch_count().
#pragma once

#include <atomic>

#include "umma_gemm.cuh"

namespace ms {

// launch counters by kernel family (ms_launch_stats)
enum KernelFamily : int { KF_UMMA = 0, KF_SIMT = 1, KF_BN = 2, KF_MISC = 3, KF_COUNT = 4 };
extern std::atomic<int64_t> g_launches;
extern std::atomic<int64_t> g_family[KF_COUNT];
inline void count_launch(int n = 1, int family = KF_MISC) {
  g_launches.fetch_add(n, std::memory_order_relaxed);
  g_family[family].fetch_add(n, std::memory_order_relaxed);
}

inline CUtensorMapDataType tma_dtype(int dt) {
  return dt == MS_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                       : (dt == MS_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                       : CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
}

// 2-D row-major matrix [outer][inner] with row pitch `ld` elements,
// box {box_inner, box_outer}, 128-byte swizzle, OOB -> zero.
ms_status make_tmap_2d(CUtensorMap* m, int dt, const void* base, uint64_t inner, uint64_t outer,
                       uint64_t ld, uint32_t box_inner, uint32_t box_outer);

// General tiled tensor map: dims[0] innermost, strides in bytes for dims 1..rank-1.
// swizzle: 0 none, 64, 128 (bytes).
ms_status make_tmap_nd(CUtensorMap* m, int dt, const void* base, int rank, const uint64_t* dims,
                       const uint64_t* strides_bytes, const uint32_t* box, int swizzle);

// NHWC activation [n][h][w][c] as an im2col tensor map.
//   lower/upper: pixel bounding-box corners {w, h}; strides: traversal {w, h}
ms_status make_tmap_im2col(CUtensorMap* m, int dt, const void* base, int n, int h, int w, int c,
                           const int lower[2], const int upper[2], int stride_w, int stride_h,
                           uint32_t channels, uint32_t pixels, bool swizzle128 = true);

// Epilogue through TMA stores when the output is 16-bit, 16-byte aligned and
// densely pitched (sets g.tma_store and tm.c; MS_TMA_STORE=0 disables).
ms_status setup_tma_store(TmapPack& tm, GemmArgs& g, int dt, void* out, int64_t rows,
                          int64_t cols, int64_t ldc);

// Runs umma_gemm_kernel<BN, A_MN, B_MN, MODE, cluster> with BN chosen at run
// time.  cluster = 2: CTA-pair tiles (tcgen05 cta_group::2, 256 x BN; g.m_blocks
// / PhaseInfo::m_blocks then count pairs of 128-row M tiles).
ms_status launch_umma(int bn, int a_mn, int b_mn, int mode, const TmapPack& tm,
                      const GemmArgs& g, cudaStream_t st, int cluster = 1);

// Single-CTA BN for `m_tiles_times_other` 128-row tiles over `ncols` columns.
int pick_bn(int64_t m_tiles_times_other, int64_t ncols);

// Tile shape for a persistent launch over m_blocks 128-row tiles x ncols:
// single-CTA 128 x BN (BN in 32..256) or CTA-pair 256 x BN (BN in {128, 256})
// by a wave-quantisation cost model.  MS_GEMM_CLUSTER=1 / MS_GEMM_BN=<n>
// override it (tuning and debugging).
struct TilePick {
  int cl, bn;
};
TilePick pick_tiles(int64_t m_blocks, int64_t ncols, bool allow_pair, bool mn_major_b);
// co-resident CTA-pair clusters of the persistent GEMM (one CTA per SM; GPCs
// with an odd SM count leave an SM out of the pairs)
int pair_slots();

}  // namespace ms
