// pm1.cuh — packed bits -> +-1 int8 operands for the kind::i8 tensor-core MMAs.
#pragma once
#include <cstdint>

namespace btnn_gpu {

// Sign-replicating byte permute: prmt.b32 in its default mode honours bit 3 of each
// selector nibble (replicate the msb of the selected byte); CUDA's __byte_perm masks the
// selector to 3 bits, so it cannot be used here.
__device__ __forceinline__ uint32_t prmt_sign(uint32_t x) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(r) : "r"(x));
  return r;
}
// 32 bits -> 8 words of 4 int8 each: word s byte k = (bit 8k+7-s) ? -1 : +1. Operand K index
// kappa = 4s + k of the word holds bit 8k + 7 - s: a fixed permutation of K, harmless as long
// as both operands of a dot product use it.
__device__ __forceinline__ void expand_word(uint32_t w, uint32_t* o) {
#pragma unroll
  for (int s = 0; s < 8; ++s) o[s] = prmt_sign(w << s) | 0x01010101u;
}

// 32 bits -> 8 words of 4 {0,1} bytes in the same K order as expand_word: byte k of word s =
// bit 8k + 7 - s. Paired with a +-1 operand, sum(a * b01) = sum over b's set bits of a, and
// the +-1 dot follows as sum(a) - 2 sum(a * b01).
__device__ __forceinline__ void expand_word01(uint32_t w, uint32_t* o) {
#pragma unroll
  for (int s = 0; s < 8; ++s) o[s] = (w >> (7 - s)) & 0x01010101u;
}

}  // namespace btnn_gpu
