// Counter-based RNG and keyed permutations (device side).
//
// Pins (mirrored by oracle/manyobj_ref/rng.py):
//   Philox4x32-10, key = (seed_lo, seed_hi), counter = (idx_lo, idx_hi, generation, stream)
//   u01(x) = (x >> 8) * 2^-24
//   permutation of [0,n): swap-or-not network, 32 + 2*bitlen(n-1) rounds,
//   round r: K_r = (x0 | x1 << 32) % n, S_r = x2 of Philox(r, n, generation, stream).
// SPEC.md:33-37 (SeedableRng), :67-75 (shuffle_rows), PAPER.md:153 (pre-shuffle).
#pragma once
#include <stdint.h>

namespace mo {

enum Stream : uint32_t {
  STREAM_INIT = 1,
  STREAM_MATING = 2,
  STREAM_SBX = 3,
  STREAM_PM = 4,
  STREAM_POP_SHUFFLE = 5,
  STREAM_REF_SHUFFLE = 6,
  STREAM_HV = 7,   // Monte-Carlo hypervolume samples (metrics, not the generation)
};
constexpr uint32_t PAIR_SLOT = 0xffffffffu;
constexpr int MAX_SHUFFLE_ROUNDS = 32 + 2 * 32;

struct U4 {
  uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ U4 philox4x32(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                  uint64_t seed) {
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return U4{c0, c1, c2, c3};
}

__host__ __device__ __forceinline__ float u01(uint32_t x) {
  return (float)(x >> 8) * (1.0f / 16777216.0f);
}

__host__ __device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}

__host__ __device__ __forceinline__ int bitlen(uint32_t v) {
  int b = 0;
  while (v) {
    ++b;
    v >>= 1;
  }
  return b;
}

__host__ __device__ __forceinline__ int shuffle_rounds(uint32_t n) {
  return 32 + 2 * bitlen(n > 1 ? n - 1 : 1);
}

// Round keys of the keyed permutation of [0, n).
struct ShuffleKeys {
  uint32_t n;
  int rounds;
  uint32_t K[MAX_SHUFFLE_ROUNDS];
  uint32_t S[MAX_SHUFFLE_ROUNDS];
};

__host__ __device__ inline void make_shuffle_keys(ShuffleKeys& sk, uint32_t n, uint64_t seed,
                                                  uint32_t generation, uint32_t stream) {
  sk.n = n;
  sk.rounds = shuffle_rounds(n);
  for (int r = 0; r < sk.rounds; ++r) {
    U4 x = philox4x32((uint32_t)r, n, generation, stream, seed);
    uint64_t k64 = (uint64_t)x.x | ((uint64_t)x.y << 32);
    sk.K[r] = n ? (uint32_t)(k64 % n) : 0u;
    sk.S[r] = x.z;
  }
}

// x' = (k - x) mod n with k, x < n: 32-bit wrap-around then + n when k < x (same value as the signed form)
__device__ __forceinline__ uint32_t sn_round(uint32_t x, uint32_t n, uint32_t k, uint32_t s) {
  uint32_t xpu = k - x;
  if (k < x) xpu += n;
  uint32_t xh = x > xpu ? x : xpu;
  return (lowbias32(xh ^ s) & 1u) ? xpu : x;
}

// Shuffled position of item x (keys in shared or global memory).  The round chain is the latency of a
// shuffle (~74 dependent rounds); unrolling lets the key loads of later rounds issue early.
__device__ __forceinline__ uint32_t prp(uint32_t x, const uint32_t* K, const uint32_t* S, int rounds,
                                        uint32_t n) {
  if (n <= 1) return x;
#pragma unroll 4
  for (int r = 0; r < rounds; ++r) x = sn_round(x, n, K[r], S[r]);
  return x;
}

// Item placed at shuffled position p.
__device__ __forceinline__ uint32_t prp_inv(uint32_t p, const uint32_t* K, const uint32_t* S, int rounds,
                                            uint32_t n) {
  if (n <= 1) return p;
#pragma unroll 4
  for (int r = rounds - 1; r >= 0; --r) p = sn_round(p, n, K[r], S[r]);
  return p;
}

// Block-cooperative load of shuffle keys into shared memory (call by all threads, then __syncthreads()).
__device__ __forceinline__ void load_shuffle_keys_smem(uint32_t* shK, uint32_t* shS, int* shRounds, uint32_t n,
                                                       uint64_t seed, uint32_t generation, uint32_t stream) {
  int rounds = shuffle_rounds(n);
  for (int r = threadIdx.x; r < rounds; r += blockDim.x) {
    U4 x = philox4x32((uint32_t)r, n, generation, stream, seed);
    uint64_t k64 = (uint64_t)x.x | ((uint64_t)x.y << 32);
    shK[r] = n ? (uint32_t)(k64 % n) : 0u;
    shS[r] = x.z;
  }
  if (threadIdx.x == 0) *shRounds = rounds;
}

}  // namespace mo
