// Probe: 3-D fp32 TMA row loads like conv3x3_tf32_kernel (box [132][1][8]).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap tx, int c0, int c1, int c2, int bytes, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8 * 4224 + 18 * 512);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(smem)),
        "l"(reinterpret_cast<uint64_t>(&tx)), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(su32(bar)));
    }
    float s = 0.f;
    for (int i = 0; i < bytes / 4; ++i) s += reinterpret_cast<float*>(smem)[i];
    out[0] = s;
  }
}

int main(int argc, char** argv) {
  int only = argc > 1 ? atoi(argv[1]) : -1; int idx = -1;
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int N = 2, C = 8, H = 20, W = 36;
  float* x; float* out;
  cudaMalloc(&x, sizeof(float) * N * C * H * W);
  cudaMalloc(&out, 4);
  cudaMemset(x, 0, sizeof(float) * N * C * H * W);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  struct V { unsigned bw, bc; int c0, c1, c2; const char* name; } vs[] = {
      {128, 8, 0, 0, 0, "box128 origin"}, {132, 8, 0, 0, 0, "box132 origin"},
      {132, 8, -1, -1, 0, "box132 neg"}, {32, 8, 0, 0, 0, "box32 origin"},
      {132, 1, 0, 0, 0, "box132 c1"}, {36, 8, 0, 0, 0, "box36 (=W)"}};
  for (auto& v : vs) {
    if (++idx != only && only >= 0) continue;
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N * C};
    cuuint64_t str[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
    cuuint32_t box[3] = {v.bw, 1, v.bc}, e[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, str, box, e,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 128, 96 * 1024>>>(m, v.c0, v.c1, v.c2, v.bw * v.bc * 4, out);
    cudaError_t e2 = cudaDeviceSynchronize();
    printf("%-16s encode=%d run=%s\n", v.name, (int)r, cudaGetErrorString(e2));
    if (e2 != cudaSuccess) return 1;
  }
  return 0;
}
