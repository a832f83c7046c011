// Probe: TMA streaming throughput of NCHW fp32 row boxes [bw px][bh rows][8 ch]
// (3-D map W x H x N*8), S-slot ring, one producer lane, one consumer warp.
// usage: tma_rows bw bh slots
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(bar), "r"(par) : "memory");
}

__global__ void k(const __grid_constant__ CUtensorMap tx, int bw, int bh, int slots, int bytes,
                  int units, int segs, int hb, int N, int spinners, int kmode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + slots * bytes);
  uint64_t* empty = full + slots;
  if (threadIdx.x == 0) {
    for (int i = 0; i < slots; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int e = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++e) {
      const int s = e % slots;
      wait(su32(&empty[s]), ((e / slots) & 1) ^ 1);
      const int seg = u % segs, hh = (u / segs) % hb, n = u / segs / hb;
      if (kmode) {  // the Fig.1 kernel's pattern: box u = half (u & 1) of unit u / 2
        const int uu = u >> 1, half = u & 1;
        const int sg = uu % 2, ch = (uu / 2) % 32, nn = uu / 64;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(bytes));
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(smem + s * bytes)),
            "l"(reinterpret_cast<uint64_t>(&tx)), "r"(su32(&full[s])), "r"(sg * 128 - 4), "r"(ch * 8 - 1 + 5 * half), "r"(nn * 8)
            : "memory");
        continue;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(bytes));
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(smem + s * bytes)),
          "l"(reinterpret_cast<uint64_t>(&tx)), "r"(su32(&full[s])), "r"(seg * 128 - 4), "r"(hh * (bh > 2 ? bh - 2 : bh) - 1), "r"(n * 8)
          : "memory");
    }
  } else if (threadIdx.x >= 64 && (threadIdx.x >> 5) < 2 + spinners) {
    // extra warps poll the same full barriers (all lanes), like converter warps
    int e = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++e) wait(su32(&full[e % slots]), (e / slots) & 1);
  } else if (threadIdx.x == 32) {
    int e = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++e) {
      const int s = e % slots;
      wait(su32(&full[s]), (e / slots) & 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])));
    }
  }
}

int main(int argc, char** argv) {
  const int bw = atoi(argv[1]), bh = atoi(argv[2]), slots = atoi(argv[3]);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int N = argc > 4 ? atoi(argv[4]) : 32, C = 8, H = 256, W = 256;
  float* x;
  cudaMalloc(&x, sizeof(float) * N * C * H * W);
  { float* h = (float*)malloc(sizeof(float) * N * C * H * W); for (size_t i = 0; i < (size_t)N * C * H * W; ++i) h[i] = (float)(i % 977) * 0.37f; cudaMemcpy(x, h, sizeof(float) * N * C * H * W, cudaMemcpyHostToDevice); free(h); }
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N * C};
  cuuint64_t str[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 8}, e[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, str, box, e,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int bytes = bw * bh * 8 * 4;
  const int step = bh > 2 ? bh - 2 : bh;  // overlapping row windows (bh-2 new rows)
  const int segs = 2, hb = (H + step - 1) / step;
  const int kmode = argc > 7 ? atoi(argv[7]) : 0;
  const int units = kmode ? N * 2 * 32 * 2 : N * segs * hb;
  const int smem = argc > 6 ? atoi(argv[6]) * 1024 : slots * bytes + 2 * slots * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int spin = argc > 5 ? atoi(argv[5]) : 0;
  const int thr = 64 + 32 * spin;
  k<<<148, thr, smem>>>(m, bw, bh, slots, bytes, units, segs, hb, N, spin, kmode);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) k<<<148, thr, smem>>>(m, bw, bh, slots, bytes, units, segs, hb, N, spin, kmode);
  cudaEventRecord(b);
  cudaError_t err = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 10;
  const double tot = (double)units * bytes;
  const double uniq = (double)N * C * H * W * 4;
  printf("spin %d box %dx%dx8 (%d B) slots %d: enc=%d %s  %.1f us  box %.0f GB/s, unique %.0f GB/s\n", spin, bw, bh, bytes, slots,
         (int)r, cudaGetErrorString(err), ms * 1e3, tot / ms / 1e6, uniq / ms / 1e6);
  return 0;
}
