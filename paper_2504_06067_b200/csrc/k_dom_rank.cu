// Dominance bit-matrix by per-objective rank masks (K1, engine path for m = 2..16).
//
// Reference: dominance.dominance_matrix, the input of non_dominated_sort
// (SPEC.md:196-204).  Same output as k_dom_tile_sorted (k_dominance.cu) -- the dominated-major
// bit-matrix over presorted positions plus hasdom -- with far fewer instructions per pair.
//
// For a 256-row block I of the S-presorted rows and one objective k, the set {i in I : a_ik <= b}
// is the prefix of I's rows sorted by objective k whose length c is the number of values <= b.
// So per block and objective we precompute (k_dom_tables):
//   * the sorted values in Eytzinger (BFS) order, 511 slots padded with NaN -> c by 9 branch-free
//     probes, conflict-free in shared memory (level t of the tree is 2^t contiguous words);
//   * the 257 prefix masks P_k[c] (256 bits = 8 words each).
// Then, for a row j, the 256 bits "a_i <= b_j in every objective" are AND_k P_k[c_k(j)]: m searches
// and m x 8 word ANDs for 256 pairs instead of 256 m-long compare chains (about 1.6 instructions per
// pair at m = 10 instead of ~11).  In S-separated tiles (max S(I) < min S(J)) that weak relation is
// already "i dominates j" (S differs, so the rows differ).  Tiles with overlapping S ranges (the
// diagonal) also need the reverse relation: {i : a_ik >= b} = complement of the strict prefix
// P_k[#{a < b}], giving both dominance directions with the exact compare semantics of the pairwise
// kernel (IEEE <=, -0 == +0; a row with a NaN objective dominates nothing and is dominated by
// nothing).
//
// k_dom_rank: persistent grid over items (I block, run of J blocks).  The CTA pulls block I's m
// tables (m x 10,272 B) into shared memory with ONE bulk TMA copy (cp.async.bulk + mbarrier), then
// sweeps its J blocks, one row j per thread: b_j from FS (L2), m Eytzinger searches (unrolled across
// the m objectives for ILP), the mask ANDs, 8 words stored to row j.  Reverse-direction words of the
// overlapping tiles are transposed through warp ballots and shared memory.
#include <cuda_runtime.h>

#include <cstdlib>

#include "mo_common.cuh"
#include "k_dominance_args.cuh"
#include "mo_async.cuh"
#include "mo_sortnet.cuh"

namespace mo {

constexpr int DR_BLK = 256;                        // rows per block (= the bit-matrix tile)
constexpr int DR_EYT = 512;                        // Eytzinger slots (1..511 used)
constexpr int DR_MASKS = DR_BLK + 1;               // prefix masks c = 0..256
constexpr int DR_TBL_WORDS = DR_EYT + DR_MASKS * 8;
constexpr int DR_TBL_BYTES = DR_TBL_WORDS * 4;     // 10,272 (16-byte multiple)
static_assert(DR_TBL_BYTES % 32 == 0, "bulk copies move 16-byte multiples; prefix-mask slot pairs are 32-byte aligned");

__host__ __device__ inline int64_t dom_rank_blocks(int64_t R) { return (R + DR_BLK - 1) / DR_BLK; }

// 16-byte half h of prefix mask c: swizzled so that 8 lanes loading random masks spread over all 8
// bank groups of a 128-bit shared-memory phase
__device__ __forceinline__ int mask_slot(int c, int h) { return 2 * c + (h ^ ((c >> 2) & 1)); }

// ------------------------------------------------------------------ tables
// grid (nb, M): block bi, objective k.  vmask[bi*8 + w]: rows of block bi that exist and have no NaN.
// M = 0: runtime m (the wide-m path, m > 16)
template <int M>
__global__ void __launch_bounds__(DR_BLK) k_dom_tables(const float* __restrict__ FS, int R,
                                                        uint32_t* __restrict__ tables, uint32_t* __restrict__ vmask,
                                                        int m_rt, uint32_t* __restrict__ tsum) {
  pdl_wait();
  const int m = M > 0 ? M : m_rt;
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
    vmask[(int64_t)gridDim.x * 8] = 0u;   // k_dom_rank's chunk counter (in the tables' slack)
  if (tsum && blockIdx.y == 0) {   // this generation's tile summary of block bi's rows starts empty
    const int64_t TW = tsum_words(R);
    const int64_t r0 = (int64_t)blockIdx.x * DR_BLK, r1 = min((int64_t)R, r0 + DR_BLK);
    for (int64_t e = r0 * TW + threadIdx.x; e < r1 * TW; e += DR_BLK) tsum[e] = 0u;
  }
  __shared__ uint32_t sKey[DR_BLK];
  __shared__ int sIdx[DR_BLK];
  const int bi = blockIdx.x, k = blockIdx.y, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int i = bi * DR_BLK + t;
  const float x = i < R ? FS[(int64_t)i * m + k] : __int_as_float(0x7fc00000);
  sKey[t] = x != x ? 0xffffffffu : f2ord(__fadd_rn(x, 0.0f));   // NaN last; -0 -> +0
  sIdx[t] = t;
  if (k == 0) {
    bool ok = i < R;
    if (ok)
      for (int q = 0; q < m; ++q) {
        const float v = FS[(int64_t)i * m + q];
        ok = ok && v == v;
      }
    const uint32_t bal = __ballot_sync(MO_FULL, ok);
    if (lane == 0) vmask[(int64_t)bi * 8 + warp] = bal;
  }
  // bitonic sort of (key, idx), ascending, one element per thread: strides < 32 exchange through warp
  // shuffles, only the 6 stages with stride >= 32 go through shared memory (12 barriers instead of 36).
  // Ties may land in any order: every count c the sweep looks up (#{a <= b}, #{a < b}) ends on a
  // tie-group boundary, where the prefix P[c] does not depend on the order inside the group.
  uint32_t key = sKey[t];
  int idx = t;
#pragma unroll
  for (int size = 2; size <= DR_BLK; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      uint32_t ok;
      int oi;
      if (stride >= 32) {
        __syncthreads();   // previous readers of sKey / sIdx are done
        sKey[t] = key;
        sIdx[t] = idx;
        __syncthreads();
        ok = sKey[t ^ stride];
        oi = sIdx[t ^ stride];
      } else {
        ok = __shfl_xor_sync(MO_FULL, key, stride);
        oi = __shfl_xor_sync(MO_FULL, idx, stride);
      }
      const bool up = (t & size) == 0, lower = (t & stride) == 0;
      const uint32_t lo = lower ? key : ok, hi = lower ? ok : key;
      if (up ? lo > hi : lo < hi) {   // both partners decide on the same (lo, hi): they swap together
        key = ok;
        idx = oi;
      }
    }
  }
  __syncthreads();
  sKey[t] = key;
  sIdx[t] = idx;
  __syncthreads();
  uint32_t* tab = tables + ((int64_t)bi * m + k) * DR_TBL_WORDS;
  // Eytzinger: node n at depth d holds sorted position ((2 (n - 2^d) + 1) << (8 - d)) - 1
  for (int n = t; n < DR_EYT; n += DR_BLK) {
    float v = __int_as_float(0x7fc00000);
    if (n >= 1) {
      const int d = 31 - __clz(n);
      const int pos = ((2 * (n - (1 << d)) + 1) << (8 - d)) - 1;
      if (pos < DR_BLK && sKey[pos] != 0xffffffffu) v = ord2f(sKey[pos]);
    }
    tab[n] = __float_as_uint(v);
  }
  // prefix masks: warp w builds word w of P[0..256] by an inclusive OR-scan over the sorted order
  uint32_t* P = tab + DR_EYT;
  uint32_t carry = 0;
  for (int q = 0; q < DR_BLK / 32; ++q) {
    const int s = q * 32 + lane;
    const int idx = sIdx[s];
    uint32_t v = (idx >> 5) == warp ? 1u << (idx & 31) : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(MO_FULL, v, o);
      if (lane >= o) v |= y;
    }
    v |= carry;
    const int c = s + 1;   // P[c] = first c sorted rows
    P[mask_slot(c, warp >> 2) * 4 + (warp & 3)] = v;
    carry = __shfl_sync(MO_FULL, v, 31);
  }
  if (lane == 0) P[mask_slot(0, warp >> 2) * 4 + (warp & 3)] = 0u;
  pdl_trigger();
}

// ---------------------------------------------------------------- main sweep

struct DomRankArgs {
  const float* FS;
  const float* blkmin;
  const float* blkmax;
  const int* wend;
  const uint32_t* tables;
  const uint32_t* vmask;
  uint32_t* bits;
  uint8_t* hasdom;
  int R, nb, ch;           // rows, blocks, J blocks per item
  int64_t W;               // words per bit-matrix row
  int64_t items;
  uint32_t* tsum;          // nullable: tile summary (then zero word blocks are not stored)
  int64_t TW;
  int ordered_and;         // S-separated tiles: AND the prefixes shortest first with early exit
  uint32_t two;            // 2, opaque to the compiler (see dr_search)
  int64_t pairs;           // k_dom_rank<M>: tiles of the block upper triangle (row-major), chunks of ch
  unsigned* next;          // k_dom_rank<M>: chunk counter (zeroed by k_dom_tables)
};

// store the 8 words of block `blk` of row `row` (always without a summary; with one, only when nonzero,
// flagging the block); hasdom[row] = 1 when nonzero
__device__ __forceinline__ void dr_store(const DomRankArgs& a, int row, int blk, const uint32_t* v) {
  const bool nz = (v[0] | v[1] | v[2] | v[3] | v[4] | v[5] | v[6] | v[7]) != 0u;
  if (!a.tsum || nz) {
    uint4* dst = reinterpret_cast<uint4*>(a.bits + (int64_t)row * a.W + (int64_t)blk * 8);
    dst[0] = make_uint4(v[0], v[1], v[2], v[3]);
    dst[1] = make_uint4(v[4], v[5], v[6], v[7]);
  }
  if (nz) {
    a.hasdom[row] = 1;
    if (a.tsum) atomicOr(a.tsum + (int64_t)row * a.TW + (blk >> 5), 1u << (blk & 31));
  }
}

// items of block row bi: ceil((nb - bi) / ch); G(n) = sum_{x=1..n} ceil(x / ch)
__device__ __forceinline__ int64_t dr_G(int64_t n, int ch) {
  const int64_t q = n / ch, r = n % ch;
  return ch * q * (q + 1) / 2 + r * (q + 1);
}
__device__ __forceinline__ void dr_decode(int64_t t, int nb, int ch, int& bi, int& bj0, int& bj1) {
  const int64_t Gn = dr_G(nb, ch);
  int lo = 0, hi = nb - 1;   // largest bi with cum(bi) = Gn - G(nb - bi) <= t
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (Gn - dr_G(nb - mid, ch) <= t) lo = mid;
    else hi = mid - 1;
  }
  bi = lo;
  const int64_t off = t - (Gn - dr_G(nb - bi, ch));
  bj0 = bi + (int)off * ch;
  bj1 = min(nb, bj0 + ch);
}

// The m Eytzinger searches of one row, returned as shared addresses ad[k] = base + 4 node[k] with
// node[k] = 512 + #{values of objective k <= b[k]} (STRICT: < b[k]).  The walk carries the addresses, so a probe is one load, one compare, one
// select of two constants and one multiply-add: ad' = 2 ad - base + 4 [go] = base + 4 (2 node + go);
// the per-objective table offset k * DR_TBL_BYTES folds into the load's immediate.  `two` (= 2) comes
// from the kernel arguments so that ptxas keeps the multiply-add on the FMA pipe (IMAD) instead of an
// ALU IADD3: the sweep is ALU-pipe bound, and the compare and select already sit there.
template <int M, bool STRICT>
__device__ __forceinline__ void dr_search(uint32_t base, uint32_t two, const float* b, uint32_t* ad) {
  const uint32_t c0 = 0u - base, c1 = 4u - base;
#pragma unroll
  for (int k = 0; k < M; ++k) ad[k] = base + 4u;
#pragma unroll
  for (int s = 0; s < 9; ++s) {
#pragma unroll
    for (int k = 0; k < M; ++k) {
      float e;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(e) : "r"(ad[k] + (uint32_t)(k * DR_TBL_BYTES)));
      if (STRICT)
        asm("{\n\t.reg .pred p;\n\tsetp.lt.f32 p, %1, %2;\n\t@p mad.lo.u32 %0, %0, %3, %4;\n\t"
            "@!p mad.lo.u32 %0, %0, %3, %5;\n\t}"
            : "+r"(ad[k]) : "f"(e), "f"(b[k]), "r"(two), "r"(c1), "r"(c0));
      else
        asm("{\n\t.reg .pred p;\n\tsetp.le.f32 p, %1, %2;\n\t@p mad.lo.u32 %0, %0, %3, %4;\n\t"
            "@!p mad.lo.u32 %0, %0, %3, %5;\n\t}"
            : "+r"(ad[k]) : "f"(e), "f"(b[k]), "r"(two), "r"(c1), "r"(c0));
    }
  }
}

// tile t of the row-major upper block triangle (row bi holds tiles (bi, bi..nb-1), offset
// off(bi) = bi nb - bi (bi - 1) / 2) -> block row bi and the J run [bj0, bj1) up to the row end or t1
__device__ __forceinline__ void dr_tile_decode(int64_t t, int64_t t1, int nb, int& bi, int& bj0, int& bj1) {
  int lo = 0, hi = nb - 1;   // largest bi with off(bi) <= t
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((int64_t)mid * nb - (int64_t)mid * (mid - 1) / 2 <= t) lo = mid;
    else hi = mid - 1;
  }
  bi = lo;
  bj0 = bi + (int)(t - ((int64_t)bi * nb - (int64_t)bi * (bi - 1) / 2));
  bj1 = (int)min((int64_t)nb, (int64_t)bj0 + (t1 - t));
}

// le = AND_k P_k[c_k] (c_k = node[k] - DR_EYT, from the search addresses): a_i <= b_j (INV: the
// complement of the strict prefixes, a_i >= b_j) in every objective
template <int M, bool INV>
__device__ __forceinline__ void dr_and_all(const uint32_t* sTab, uint32_t base, const uint32_t* ad, uint32_t* le) {
#pragma unroll
  for (int k = 0; k < M; ++k) {
    const int c = (int)((ad[k] - base) >> 2) - DR_EYT;
    const uint4* P = reinterpret_cast<const uint4*>(sTab + k * DR_TBL_WORDS + DR_EYT);
    const uint4 h0 = P[mask_slot(c, 0)], h1 = P[mask_slot(c, 1)];
    if (INV) {
      le[0] &= ~h0.x; le[1] &= ~h0.y; le[2] &= ~h0.z; le[3] &= ~h0.w;
      le[4] &= ~h1.x; le[5] &= ~h1.y; le[6] &= ~h1.z; le[7] &= ~h1.w;
    } else {
      le[0] &= h0.x; le[1] &= h0.y; le[2] &= h0.z; le[3] &= h0.w;
      le[4] &= h1.x; le[5] &= h1.y; le[6] &= h1.z; le[7] &= h1.w;
    }
  }
}

__host__ __device__ constexpr int dr_pow2(int m) { return m <= 1 ? 1 : 2 * dr_pow2((m + 1) / 2); }

// The same set for S-separated tiles, where only le is needed and ~96 % of the (row, block) results
// are empty (C3): the prefixes are ANDed shortest first and a lane stops once its AND is empty, so the
// later mask gathers run with fewer active lanes -- fewer shared-memory wavefronts and bank conflicts.
// Sort keys are c << 18 | (byte offset of half 0 of P_k[c] in the tables), so the loop needs no
// swizzle arithmetic: half 1 sits at offset ^ 16 (mask_slot pairs the slots 2c, 2c + 1 and every table
// starts on a 32-byte boundary).  Batcher's odd-even merge network over the keys padded to a power of
// two with all-ones keys (the compiler folds the comparators that touch padding): 32 comparators at
// m = 10 instead of 45 for odd-even transposition; the sweep is ALU-pipe bound.
template <int M>
__device__ __forceinline__ void dr_and_shortest_first(uint32_t sbase, const uint32_t* ad, uint32_t* out) {
  constexpr int N = dr_pow2(M);
  uint32_t key[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    if (k < M) {
      // q = ad - base - 2048 = 4c: c << 18 | 16 slot0 = q (2^16 + 8) + (q & 16) with slot0 = 2c + ((c >> 2) & 1)
      // (mask_slot), and the table offset K has bit 4 clear -- one IADD, one LOP3, one IMAD
      const uint32_t q = ad[k] - (sbase + DR_EYT * 4u);
      key[k] = q * 65544u + ((q & 16u) | (uint32_t)(k * DR_TBL_BYTES + DR_EYT * 4));
    } else {
      key[k] = 0xffffffffu;
    }
  }
  sortnet<N>(key);
  bool nz = (key[0] >> 18) != 0u;   // an empty prefix empties the AND
  const uint32_t ones = nz ? 0xffffffffu : 0u;
  uint32_t le[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) le[w] = ones;
#pragma unroll
  for (int s = 0; s < M; ++s) {
    if (nz) {
      const uint32_t off = key[s] & 0x3ffffu;
      uint4 h0, h1;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(h0.x), "=r"(h0.y), "=r"(h0.z), "=r"(h0.w) : "r"(sbase + off));
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(h1.x), "=r"(h1.y), "=r"(h1.z), "=r"(h1.w) : "r"(sbase + (off ^ 16u)));
      le[0] &= h0.x; le[1] &= h0.y; le[2] &= h0.z; le[3] &= h0.w;
      le[4] &= h1.x; le[5] &= h1.y; le[6] &= h1.z; le[7] &= h1.w;
      // the shortest prefix alone (c >= 1) is never empty; from the second objective on, stop at empty
      if (s > 0) nz = (le[0] | le[1] | le[2] | le[3] | le[4] | le[5] | le[6] | le[7]) != 0u;
    }
  }
#pragma unroll
  for (int w = 0; w < 8; ++w) out[w] = le[w];   // zero whenever the walk stopped early
}

template <int M>
__global__ void __launch_bounds__(DR_BLK, 2) k_dom_rank(DomRankArgs a) {
  pdl_wait();
  extern __shared__ __align__(128) uint32_t sTab[];   // M tables of block I
  __shared__ __align__(8) uint64_t sBar;
  __shared__ uint32_t sT[DR_BLK * 9];                  // reverse-direction words (row i, J word w)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) mbar_init(&sBar, 1);
  __syncthreads();
  unsigned parity = 0;
  __shared__ int sChunk;
  int cur_bi = -1;   // block whose tables are in sTab
  for (;;) {
    __syncthreads();   // the previous chunk is done with sTab / sT / sChunk
    if (tid == 0) sChunk = (int)atomicAdd(a.next, 1u);
    __syncthreads();
    const int64_t chunk = sChunk;
    if (chunk >= a.items) break;
    // chunks are taken from the END of the row-major tile order first: the short block rows at the
    // end (a diagonal tile and a table load every few tiles) are the costliest per tile
    const int64_t t0 = (a.items - 1 - chunk) * a.ch, t1 = min(a.pairs, t0 + a.ch);
    for (int64_t t = t0; t < t1;) {
      int bi, bj0, bj1;
      dr_tile_decode(t, t1, a.nb, bi, bj0, bj1);
      t += bj1 - bj0;
      const bool load = bi != cur_bi;   // CTA-uniform
      if (load) {
        __syncthreads();   // everyone is done with the previous block's tables
        if (tid == 0) {
          mbar_expect_tx(&sBar, (unsigned)(M * DR_TBL_BYTES));
          bulk_g2s(sTab, a.tables + (int64_t)bi * M * DR_TBL_WORDS, (unsigned)(M * DR_TBL_BYTES), &sBar);
        }
      }
      uint32_t vI[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) vI[w] = __ldg(a.vmask + (int64_t)bi * 8 + w);
      const float smaxI = __ldg(a.blkmax + bi);
      const int i0 = bi * DR_BLK;
      // first J row's objectives while the tables land
      float bnext[M];
      {
        const int j = bj0 * DR_BLK + tid;
#pragma unroll
        for (int k = 0; k < M; ++k) bnext[k] = j < a.R ? __ldg(a.FS + (int64_t)j * M + k) : 0.0f;
      }
      if (load) {
        mbar_wait(&sBar, parity);
        parity ^= 1u;
        cur_bi = bi;
      }
      for (int bj = bj0; bj < bj1; ++bj) {
        const int j = bj * DR_BLK + tid;
        float b[M];
        bool jnan = false;
#pragma unroll
        for (int k = 0; k < M; ++k) {
          b[k] = bnext[k];
          jnan = jnan || (b[k] != b[k]);
        }
        if (bj + 1 < bj1) {   // prefetch the next J block's row
          const int jn = j + DR_BLK;
#pragma unroll
          for (int k = 0; k < M; ++k) bnext[k] = jn < a.R ? __ldg(a.FS + (int64_t)jn * M + k) : 0.0f;
        }
        const bool fast = bi < bj && smaxI < __ldg(a.blkmin + bj);   // CTA-uniform
        // weak relation a_i <= b_j in every objective: AND of the prefix masks
        const uint32_t sbase = smem_addr(sTab);
        uint32_t ad[M];
        dr_search<M, false>(sbase, a.two, b, ad);
        uint32_t out[8], le[8];
        const bool ordered = fast && M >= 4 && a.ordered_and;   // CTA-uniform
        if (ordered) {
          dr_and_shortest_first<M>(sbase, ad, out);
        } else {
#pragma unroll
          for (int w = 0; w < 8; ++w) le[w] = 0xffffffffu;
          dr_and_all<M, false>(sTab, sbase, ad, le);
        }
        if (fast && !ordered) {
#pragma unroll
          for (int w = 0; w < 8; ++w) out[w] = le[w];
        } else if (!fast) {
          // reverse weak relation a_i >= b_j: complement of the strict prefix #{a_i < b_j}
          uint32_t nd[M];
          dr_search<M, true>(sbase, a.two, b, nd);
          uint32_t ge[8];
#pragma unroll
          for (int w = 0; w < 8; ++w) ge[w] = jnan ? 0u : vI[w];
          dr_and_all<M, true>(sTab, sbase, nd, ge);
#pragma unroll
          for (int w = 0; w < 8; ++w) out[w] = le[w] & ~ge[w];   // i dominates j
          if (bi != bj) {
            // j dominates i: transpose the per-j masks into rows i (word bj*8 + warp) by ballots
            const bool jok = j < a.R;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
              const uint32_t rev = jok ? (ge[w] & ~le[w]) : 0u;
              uint32_t mine = 0;
#pragma unroll
              for (int b2 = 0; b2 < 32; ++b2) {
                const uint32_t bal = __ballot_sync(MO_FULL, (rev >> b2) & 1u);
                mine = lane == b2 ? bal : mine;
              }
              sT[(w * 32 + lane) * 9 + warp] = mine;   // row i = w*32 + lane, word warp of block bj
            }
          }
        }
        if (j < a.R) dr_store(a, j, bi, out);
        if (fast && !a.tsum) {
          // rows i of I's last S bucket may share it with rows of J: their words of block bj lie below
          // wend and are read by the peel, so they must hold zeros (no j of a fast tile dominates an i)
          const int ilast = min(a.R, i0 + DR_BLK) - 1;
          if (__ldg(a.wend + ilast) > bj * 8) {
            const int i = i0 + tid;
            if (i < a.R && __ldg(a.wend + i) > bj * 8) {
              uint4* dst = reinterpret_cast<uint4*>(a.bits + (int64_t)i * a.W + (int64_t)bj * 8);
              dst[0] = make_uint4(0u, 0u, 0u, 0u);
              dst[1] = make_uint4(0u, 0u, 0u, 0u);
            }
          }
        } else if (!fast && bi != bj) {
          __syncthreads();
          const int i = i0 + tid;
          if (i < a.R) {
            uint32_t sw[8];
#pragma unroll
            for (int w = 0; w < 8; ++w) sw[w] = sT[tid * 9 + w];
            dr_store(a, i, bj, sw);
          }
          __syncthreads();
        }
      }
    }
  }
  pdl_trigger();
}

// ------------------------------------------------------------ wide m (m > 16)
//
// The same rank-mask relation for any m (Appendix D: m up to 512): the m tables of block I do
// not fit in shared memory, so each (I, J) tile walks the objectives in chunks of DRW_MC tables (one
// bulk copy per chunk) and keeps the running AND of the prefix masks -- le (a_i <= b_j) and ge
// (a_i >= b_j) -- in registers.  Output identical to k_dom_rank (same words, hasdom, zeroed straddle
// words); objectives are visited in ascending order, so no result depends on the chunking.
constexpr int DRW_MC = 8;

__global__ void __launch_bounds__(DR_BLK) k_dom_rank_wide(DomRankArgs a, int m) {
  pdl_wait();
  extern __shared__ __align__(128) uint32_t sTab[];   // DRW_MC tables of block I
  __shared__ __align__(8) uint64_t sBar;
  __shared__ uint32_t sT[DR_BLK * 9];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) mbar_init(&sBar, 1);
  __syncthreads();
  unsigned parity = 0;
  for (int64_t item = blockIdx.x; item < a.items; item += gridDim.x) {
    int bi, bj0, bj1;
    dr_decode(item, a.nb, a.ch, bi, bj0, bj1);
    uint32_t vI[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) vI[w] = __ldg(a.vmask + (int64_t)bi * 8 + w);
    const float smaxI = __ldg(a.blkmax + bi);
    const int i0 = bi * DR_BLK;
    for (int bj = bj0; bj < bj1; ++bj) {
      const int j = bj * DR_BLK + tid;
      const bool fast = bi < bj && smaxI < __ldg(a.blkmin + bj);   // CTA-uniform
      uint32_t le[8], ge[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        le[w] = 0xffffffffu;
        ge[w] = vI[w];
      }
      bool jnan = false;
      for (int k0 = 0; k0 < m; k0 += DRW_MC) {
        const int mc = min(DRW_MC, m - k0);
        __syncthreads();   // everyone is done with the previous chunk / item
        if (tid == 0) {
          mbar_expect_tx(&sBar, (unsigned)(mc * DR_TBL_BYTES));
          bulk_g2s(sTab, a.tables + ((int64_t)bi * m + k0) * DR_TBL_WORDS, (unsigned)(mc * DR_TBL_BYTES), &sBar);
        }
        float b[DRW_MC];
#pragma unroll
        for (int q = 0; q < DRW_MC; ++q) {
          b[q] = (j < a.R && q < mc) ? __ldg(a.FS + (int64_t)j * m + k0 + q) : 0.0f;
          jnan = jnan || (b[q] != b[q]);
        }
        mbar_wait(&sBar, parity);
        parity ^= 1u;
#pragma unroll
        for (int q = 0; q < DRW_MC; ++q) {
          if (q < mc) {
            const uint32_t* tab = sTab + q * DR_TBL_WORDS;
            int node = 1, nd = 1;
#pragma unroll
            for (int st = 0; st < 9; ++st) {
              const float e = __uint_as_float(tab[node]);
              node = 2 * node + (e <= b[q] ? 1 : 0);
              if (!fast) {
                const float e2 = __uint_as_float(tab[nd]);
                nd = 2 * nd + (e2 < b[q] ? 1 : 0);
              }
            }
            const uint4* P = reinterpret_cast<const uint4*>(tab + DR_EYT);
            {
              const int c = node - DR_EYT;
              const uint4 h0 = P[mask_slot(c, 0)], h1 = P[mask_slot(c, 1)];
              le[0] &= h0.x; le[1] &= h0.y; le[2] &= h0.z; le[3] &= h0.w;
              le[4] &= h1.x; le[5] &= h1.y; le[6] &= h1.z; le[7] &= h1.w;
            }
            if (!fast) {
              const int c = nd - DR_EYT;
              const uint4 h0 = P[mask_slot(c, 0)], h1 = P[mask_slot(c, 1)];
              ge[0] &= ~h0.x; ge[1] &= ~h0.y; ge[2] &= ~h0.z; ge[3] &= ~h0.w;
              ge[4] &= ~h1.x; ge[5] &= ~h1.y; ge[6] &= ~h1.z; ge[7] &= ~h1.w;
            }
          }
        }
      }
      uint32_t out[8];
      if (fast) {
#pragma unroll
        for (int w = 0; w < 8; ++w) out[w] = le[w];
      } else {
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          if (jnan) ge[w] = 0u;
          out[w] = le[w] & ~ge[w];
        }
        if (bi != bj) {
          const bool jok = j < a.R;
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            const uint32_t rev = jok ? (ge[w] & ~le[w]) : 0u;
            uint32_t mine = 0;
#pragma unroll
            for (int b2 = 0; b2 < 32; ++b2) {
              const uint32_t bal = __ballot_sync(MO_FULL, (rev >> b2) & 1u);
              mine = lane == b2 ? bal : mine;
            }
            sT[(w * 32 + lane) * 9 + warp] = mine;
          }
        }
      }
      if (j < a.R) dr_store(a, j, bi, out);
      if (fast && !a.tsum) {
        const int ilast = min(a.R, i0 + DR_BLK) - 1;
        if (__ldg(a.wend + ilast) > bj * 8) {
          const int i = i0 + tid;
          if (i < a.R && __ldg(a.wend + i) > bj * 8) {
            uint4* dst = reinterpret_cast<uint4*>(a.bits + (int64_t)i * a.W + (int64_t)bj * 8);
            dst[0] = make_uint4(0u, 0u, 0u, 0u);
            dst[1] = make_uint4(0u, 0u, 0u, 0u);
          }
        }
      } else if (!fast && bi != bj) {
        __syncthreads();
        const int i = i0 + tid;
        if (i < a.R) {
          uint32_t sw[8];
#pragma unroll
          for (int w = 0; w < 8; ++w) sw[w] = sT[tid * 9 + w];
          dr_store(a, i, bj, sw);
        }
      }
    }
  }
  pdl_trigger();
}

static int launch_dom_rank_wide(const float* FS, const float* blkmin, const float* blkmax, const int* wend,
                                int64_t R, int m, uint32_t* bits, uint8_t* hasdom, uint32_t* tables, cudaStream_t s,
                                uint32_t* tsum) {
  const int nb = (int)dom_rank_blocks(R);
  uint32_t* vmask = tables + (int64_t)nb * m * DR_TBL_WORDS;
  MO_TRY(launch_ex(k_dom_tables<0>, dim3(nb, m), dim3(DR_BLK), 0, s, false, g_mo_pdl, FS, (int)R, tables, vmask, m,
                   tsum));
  const size_t smem = (size_t)DRW_MC * DR_TBL_BYTES;
  static int per_sm = -1, sms = 0;
  if (per_sm < 0) {
    if (cudaFuncSetAttribute(k_dom_rank_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return MO_ERR_CUDA;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dom_rank_wide, DR_BLK, smem);
    if (per_sm < 1) per_sm = 1;
  }
  DomRankArgs a;
  a.FS = FS;
  a.blkmin = blkmin;
  a.blkmax = blkmax;
  a.wend = wend;
  a.tables = tables;
  a.vmask = vmask;
  a.bits = bits;
  a.hasdom = hasdom;
  a.tsum = tsum;
  a.TW = tsum_words(R);
  a.ordered_and = getenv("MO_DOM_PLAIN_AND") == nullptr;   // A/B switch for measurements
  a.R = (int)R;
  a.nb = nb;
  a.ch = 1;   // one (I, J) tile per item: every tile re-streams block I's m tables anyway
  a.W = words_per_row(R);
  a.items = (int64_t)nb * (nb + 1) / 2;
  const int64_t slots = (int64_t)sms * per_sm;
  const int64_t grid = a.items < slots ? a.items : slots;
  return launch_ex(k_dom_rank_wide, dim3((unsigned)grid), dim3(DR_BLK), smem, s, false, g_mo_pdl, a, m);
}

size_t dom_rank_tables_bytes(int64_t R, int m) {
  const int64_t nb = dom_rank_blocks(R);
  return (size_t)nb * (size_t)m * DR_TBL_BYTES + (size_t)nb * 8 * 4 + 256;
}

// resident CTAs of k_dom_rank<M> per SM (attributes set once per instantiation)
template <int M>
static int dom_rank_slots(size_t smem, int64_t& slots) {
  static int per_sm = -1, sms = 0;
  if (per_sm < 0) {
    if (cudaFuncSetAttribute(k_dom_rank<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return MO_ERR_CUDA;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dom_rank<M>, DR_BLK, smem);
    if (per_sm < 1) per_sm = 1;
  }
  slots = (int64_t)sms * per_sm;
  return MO_OK;
}

template <int M>
static int launch_dom_rank_mg(DomRankArgs a, cudaStream_t s) {
  const size_t smem = (size_t)M * DR_TBL_BYTES;
  int64_t slots = 0;
  if (const int e = dom_rank_slots<M>(smem, slots)) return e;
  // equal chunks of consecutive tiles, ~12 per resident CTA, pulled from a counter: a chunk
  // re-loads block I's tables (M x 10 KB) only where it enters a new block row, and the dynamic
  // schedule keeps the SMs evenly loaded (static round-robin over per-row runs of 1..ch tiles left SMs
  // 40 % idle)
  int64_t ch = ceil_div(a.pairs, 12 * slots);
  ch = ch < 2 ? 2 : ch;
  a.ch = (int)ch;
  a.items = ceil_div(a.pairs, ch);
  const int64_t grid = a.items < slots ? a.items : slots;
  return launch_ex(k_dom_rank<M>, dim3((unsigned)grid), dim3(DR_BLK), smem, s, false, g_mo_pdl, a);
}

template <int M>
static int launch_dom_rank_m(const float* FS, const float* blkmin, const float* blkmax, const int* wend, int64_t R,
                             uint32_t* bits, uint8_t* hasdom, uint32_t* tables, cudaStream_t s, uint32_t* tsum) {
  const int nb = (int)dom_rank_blocks(R);
  uint32_t* vmask = tables + (int64_t)nb * M * DR_TBL_WORDS;
  MO_TRY(launch_ex(k_dom_tables<M>, dim3(nb, M), dim3(DR_BLK), 0, s, false, g_mo_pdl, FS, (int)R, tables, vmask, M,
                   tsum));
  DomRankArgs a;
  a.FS = FS;
  a.blkmin = blkmin;
  a.blkmax = blkmax;
  a.wend = wend;
  a.tables = tables;
  a.vmask = vmask;
  a.bits = bits;
  a.hasdom = hasdom;
  a.tsum = tsum;
  a.TW = tsum_words(R);
  a.ordered_and = getenv("MO_DOM_PLAIN_AND") == nullptr;   // A/B switch for measurements
  a.two = 2u;
  a.R = (int)R;
  a.nb = nb;
  a.W = words_per_row(R);
  a.pairs = (int64_t)nb * (nb + 1) / 2;
  a.next = vmask + (int64_t)nb * 8;
  return launch_dom_rank_mg<M>(a, s);
}

int launch_dom_rank(const float* FS, const float* blkmin, const float* blkmax, const int* wend, int64_t R, int m,
                    uint32_t* bits, uint8_t* hasdom, uint32_t* tables, cudaStream_t s, uint32_t* tsum) {
  if (R <= 0) return MO_OK;
  if (R > (1ll << 31) - 1 - DR_BLK) return MO_ERR_PARAM;
  switch (m) {
#define MO_DR_CASE(MM) \
  case MM: return launch_dom_rank_m<MM>(FS, blkmin, blkmax, wend, R, bits, hasdom, tables, s, tsum);
    MO_DR_CASE(2) MO_DR_CASE(3) MO_DR_CASE(4) MO_DR_CASE(5) MO_DR_CASE(6) MO_DR_CASE(7) MO_DR_CASE(8)
    MO_DR_CASE(9) MO_DR_CASE(10) MO_DR_CASE(11) MO_DR_CASE(12) MO_DR_CASE(13) MO_DR_CASE(14) MO_DR_CASE(15)
    MO_DR_CASE(16)
#undef MO_DR_CASE
    default:
      if (m > 16 && m <= MO_MAX_M)
        return launch_dom_rank_wide(FS, blkmin, blkmax, wend, R, m, bits, hasdom, tables, s, tsum);
      return MO_ERR_PARAM;
  }
}

}  // namespace mo
