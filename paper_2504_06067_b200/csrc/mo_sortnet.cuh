// Batcher odd-even merge sorting networks on N = 2, 4, 8, 16 unsigned keys (ascending), as
// straight-line compare-exchanges so every index is static (no local-memory arrays).  Generated from
// the textbook iteration (p = 1, 2, 4, ...; k = p, p/2, ..., 1; pairs (i + j, i + j + k) inside the same
// 2p-block) and checked by the 0-1 principle; callers pad to N with all-ones keys and the compiler
// folds the comparators that only touch padding.
#pragma once
#include <cstdint>

namespace mo {

__device__ __forceinline__ void sortnet_ce(uint32_t& a, uint32_t& b) {
  const uint32_t lo = min(a, b), hi = max(a, b);
  a = lo;
  b = hi;
}

template <int N>
__device__ __forceinline__ void sortnet(uint32_t* k);

template <>
__device__ __forceinline__ void sortnet<2>(uint32_t* k) {   // 1 comparators
  sortnet_ce(k[0], k[1]);
}

template <>
__device__ __forceinline__ void sortnet<4>(uint32_t* k) {   // 5 comparators
  sortnet_ce(k[0], k[1]); sortnet_ce(k[2], k[3]); sortnet_ce(k[0], k[2]); sortnet_ce(k[1], k[3]);
  sortnet_ce(k[1], k[2]);
}

template <>
__device__ __forceinline__ void sortnet<8>(uint32_t* k) {   // 19 comparators
  sortnet_ce(k[0], k[1]); sortnet_ce(k[2], k[3]); sortnet_ce(k[4], k[5]); sortnet_ce(k[6], k[7]);
  sortnet_ce(k[0], k[2]); sortnet_ce(k[1], k[3]); sortnet_ce(k[4], k[6]); sortnet_ce(k[5], k[7]);
  sortnet_ce(k[1], k[2]); sortnet_ce(k[5], k[6]); sortnet_ce(k[0], k[4]); sortnet_ce(k[1], k[5]);
  sortnet_ce(k[2], k[6]); sortnet_ce(k[3], k[7]); sortnet_ce(k[2], k[4]); sortnet_ce(k[3], k[5]);
  sortnet_ce(k[1], k[2]); sortnet_ce(k[3], k[4]); sortnet_ce(k[5], k[6]);
}

template <>
__device__ __forceinline__ void sortnet<16>(uint32_t* k) {   // 63 comparators
  sortnet_ce(k[0], k[1]); sortnet_ce(k[2], k[3]); sortnet_ce(k[4], k[5]); sortnet_ce(k[6], k[7]);
  sortnet_ce(k[8], k[9]); sortnet_ce(k[10], k[11]); sortnet_ce(k[12], k[13]); sortnet_ce(k[14], k[15]);
  sortnet_ce(k[0], k[2]); sortnet_ce(k[1], k[3]); sortnet_ce(k[4], k[6]); sortnet_ce(k[5], k[7]);
  sortnet_ce(k[8], k[10]); sortnet_ce(k[9], k[11]); sortnet_ce(k[12], k[14]); sortnet_ce(k[13], k[15]);
  sortnet_ce(k[1], k[2]); sortnet_ce(k[5], k[6]); sortnet_ce(k[9], k[10]); sortnet_ce(k[13], k[14]);
  sortnet_ce(k[0], k[4]); sortnet_ce(k[1], k[5]); sortnet_ce(k[2], k[6]); sortnet_ce(k[3], k[7]);
  sortnet_ce(k[8], k[12]); sortnet_ce(k[9], k[13]); sortnet_ce(k[10], k[14]); sortnet_ce(k[11], k[15]);
  sortnet_ce(k[2], k[4]); sortnet_ce(k[3], k[5]); sortnet_ce(k[10], k[12]); sortnet_ce(k[11], k[13]);
  sortnet_ce(k[1], k[2]); sortnet_ce(k[3], k[4]); sortnet_ce(k[5], k[6]); sortnet_ce(k[9], k[10]);
  sortnet_ce(k[11], k[12]); sortnet_ce(k[13], k[14]); sortnet_ce(k[0], k[8]); sortnet_ce(k[1], k[9]);
  sortnet_ce(k[2], k[10]); sortnet_ce(k[3], k[11]); sortnet_ce(k[4], k[12]); sortnet_ce(k[5], k[13]);
  sortnet_ce(k[6], k[14]); sortnet_ce(k[7], k[15]); sortnet_ce(k[4], k[8]); sortnet_ce(k[5], k[9]);
  sortnet_ce(k[6], k[10]); sortnet_ce(k[7], k[11]); sortnet_ce(k[2], k[4]); sortnet_ce(k[3], k[5]);
  sortnet_ce(k[6], k[8]); sortnet_ce(k[7], k[9]); sortnet_ce(k[10], k[12]); sortnet_ce(k[11], k[13]);
  sortnet_ce(k[1], k[2]); sortnet_ce(k[3], k[4]); sortnet_ce(k[5], k[6]); sortnet_ce(k[7], k[8]);
  sortnet_ce(k[9], k[10]); sortnet_ce(k[11], k[12]); sortnet_ce(k[13], k[14]);
}

}  // namespace mo
