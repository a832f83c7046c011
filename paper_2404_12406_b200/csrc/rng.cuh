// Philox4x32-10 keep masks of the default dropout generator (MS_RNG_PHILOX4X32),
// shared by the dropout kernels (dropout_ln.cu) and the GEMM epilogue that
// fuses a Linear's dropout (umma_gemm.cuh): element 4j + i of a tensor is kept
// iff word i of Philox4x32-10(counter = (j lo, j hi, stream lo, stream hi),
// key = seed) is >= thr = ceil(p * 2^32) -- the same bits whichever kernel
// draws them, so a backward can replay a mask a fused forward drew.
#pragma once

#include "common.cuh"

namespace ms {

struct Philox32Keys {
  uint32_t k[10][2];  // Weyl key schedule: round r = (seed lo + r*W0, seed hi + r*W1)
};

inline Philox32Keys philox32_keys(uint64_t seed) {
  Philox32Keys K;
  uint32_t q0 = (uint32_t)seed, q1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    K.k[r][0] = q0;
    K.k[r][1] = q1;
    q0 += 0x9E3779B9u;
    q1 += 0xBB67AE85u;
  }
  return K;
}

// keep bits of elements 4*blk0 .. 4*(blk0 + NB) - 1 (bit 4b + i = element
// 4(blk0 + b) + i); NB blocks in lockstep for ILP
template <int NB>
__device__ __forceinline__ uint32_t keep_n32(uint64_t blk0, uint64_t stream,
                                             const Philox32Keys& K, uint64_t thr) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  uint32_t c[NB][4];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const uint64_t j = blk0 + b;
    c[b][0] = (uint32_t)j;
    c[b][1] = (uint32_t)(j >> 32);
    c[b][2] = (uint32_t)stream;
    c[b][3] = (uint32_t)(stream >> 32);
  }
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const uint32_t hi0 = __umulhi(M0, c[b][0]), lo0 = M0 * c[b][0];
      const uint32_t hi1 = __umulhi(M1, c[b][2]), lo1 = M1 * c[b][2];
      const uint32_t n0 = hi1 ^ c[b][1] ^ K.k[r][0], n2 = hi0 ^ c[b][3] ^ K.k[r][1];
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
    for (int j = 0; j < 4; ++j) bits |= ((uint64_t)c[b][j] >= thr ? 1u : 0u) << (4 * b + j);
  return bits;
}

// a Linear's dropout fused into its GEMM epilogue (EpiParams::drop)
struct DropEpi {
  Philox32Keys keys;
  uint64_t stream;
  uint64_t thr;   // keep iff word >= thr
  float scale;    // 1 / (1 - p)
  int on;
};

}  // namespace ms
