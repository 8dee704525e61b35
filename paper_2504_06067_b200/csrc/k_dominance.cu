// Dominance bit-matrix (K1 dom_tile) and front peeling (K2 front_peel).
//
// Reference: dominance.dominance_matrix, non_dominated_sort
// (SPEC.md:196-204), split_fronts; design SPEC.md:220-223.
//
// Layout ("dominated-major"): row j of `bits` (W = round_up(R,256)/32 words)
// holds bit i set iff F[i] dominates F[j], i.e. the dominators of j.
//
// K1: one CTA per 256x256 block pair (bi <= bj, upper block triangle).  Lane
// = one j; the CTA walks the 256 i's of block bi from shared memory.  For each
// unordered pair one FSETP-OR chain per direction gives both "i dom j" (packed
// per lane into the word of row j) and "j dom i" (a warp ballot = the word of
// row i), so each unordered pair is compared once.  Rows j of the tile get 32
// contiguous bytes (8 words) from registers; rows i get 32 bytes from smem.
//
// K2: persistent cooperative kernel.  Front k = unranked rows whose every
// dominator is ranked.  Each row keeps a resume word: words before it are
// known to contain only ranked dominators, and the ranked set only grows, so
// across all fronts every word of a row is read once plus one re-check per
// front.  Eight lanes scan one row 128 bytes at a time.
#include "mo_chains.cuh"
#include <cstdlib>

#include "mo_common.cuh"
#include "mo_grid.cuh"
#include "k_dominance_args.cuh"

namespace mo {

constexpr int DOM_TILE = 256;

__device__ __forceinline__ void tri_decode(int64_t t, int& bi, int& bj) {
  int64_t b = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((b + 1) * (b + 2) / 2 <= t) ++b;
  while (b * (b + 1) / 2 > t) --b;
  bj = (int)b;
  bi = (int)(t - b * (b + 1) / 2);
}

template <int M>
__global__ void __launch_bounds__(DOM_TILE) k_dom_tile(const float* __restrict__ F, int R,
                                                       const uint8_t* __restrict__ valid,
                                                       uint32_t* __restrict__ bits, int64_t W) {
  constexpr int MP = (M + 3) & ~3;
  __shared__ __align__(16) float sFi[DOM_TILE * MP];
  __shared__ uint32_t sB2[DOM_TILE * 9];  // row i of the tile, 8 words (+1 pad)
  __shared__ uint8_t sVi[DOM_TILE];
  int bi, bj;
  tri_decode(blockIdx.x, bi, bj);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i0 = bi * DOM_TILE, j0 = bj * DOM_TILE;

  // stage the i-block (AoS, padded to MP) and its validity
  for (int e = tid; e < DOM_TILE * MP; e += DOM_TILE) {
    int r = e / MP, k = e - r * MP;
    int i = i0 + r;
    sFi[e] = (k < M && i < R) ? F[(int64_t)i * M + k] : 0.0f;
  }
  {
    int i = i0 + tid;
    sVi[tid] = (i < R) && (valid == nullptr || valid[i]);
  }
  const int j = j0 + tid;
  const bool vj = (j < R) && (valid == nullptr || valid[j]);
  float fj[M];
#pragma unroll
  for (int k = 0; k < M; ++k) fj[k] = vj ? F[(int64_t)j * M + k] : 0.0f;
  __syncthreads();

  uint32_t accw[8];
#pragma unroll 1
  for (int c = 0; c < 8; ++c) {
    uint32_t acc = 0, mybal = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
      const int ii = c * 32 + b;
      const float* fi = sFi + ii * MP;
      bool lt = false, gt = false;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        lt |= fi[k] < fj[k];
        gt |= fi[k] > fj[k];
      }
      const bool both = vj && sVi[ii];
      const bool idomj = both && lt && !gt;
      const bool jdomi = both && gt && !lt;
      const uint32_t bal = __ballot_sync(MO_FULL, jdomi);
      acc |= (uint32_t)idomj << b;
      mybal = (lane == b) ? bal : mybal;
    }
    accw[c] = acc;
    sB2[(c * 32 + lane) * 9 + warp] = mybal;
  }
  // rows j of the tile: words [bi*8, bi*8+8) from registers
  if (j < R) {
    uint4* dst = reinterpret_cast<uint4*>(bits + (int64_t)j * W + (int64_t)bi * 8);
    dst[0] = make_uint4(accw[0], accw[1], accw[2], accw[3]);
    dst[1] = make_uint4(accw[4], accw[5], accw[6], accw[7]);
  }
  if (bi != bj) {
    __syncthreads();
    const int i = i0 + tid;
    if (i < R) {
      const uint32_t* s = sB2 + tid * 9;
      uint4* dst = reinterpret_cast<uint4*>(bits + (int64_t)i * W + (int64_t)bj * 8);
      dst[0] = make_uint4(s[0], s[1], s[2], s[3]);
      dst[1] = make_uint4(s[4], s[5], s[6], s[7]);
    }
  }
}

// Generic-m variant (m > 10): objectives of j in shared memory as well.
__global__ void __launch_bounds__(DOM_TILE) k_dom_tile_generic(const float* __restrict__ F, int R, int M,
                                                               const uint8_t* __restrict__ valid,
                                                               uint32_t* __restrict__ bits, int64_t W) {
  extern __shared__ float dyn[];
  float* sFi = dyn;                       // DOM_TILE * M
  float* sFj = dyn + DOM_TILE * M;        // DOM_TILE * M (transposed: k-major)
  __shared__ uint32_t sB2[DOM_TILE * 9];
  __shared__ uint8_t sVi[DOM_TILE];
  int bi, bj;
  tri_decode(blockIdx.x, bi, bj);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i0 = bi * DOM_TILE, j0 = bj * DOM_TILE;
  for (int e = tid; e < DOM_TILE * M; e += DOM_TILE) {
    int r = e / M, k = e - r * M;
    sFi[e] = (i0 + r < R) ? F[(int64_t)(i0 + r) * M + k] : 0.0f;
    sFj[k * DOM_TILE + r] = (j0 + r < R) ? F[(int64_t)(j0 + r) * M + k] : 0.0f;
  }
  sVi[tid] = (i0 + tid < R) && (valid == nullptr || valid[i0 + tid]);
  const int j = j0 + tid;
  const bool vj = (j < R) && (valid == nullptr || valid[j]);
  __syncthreads();
  uint32_t accw[8];
  for (int c = 0; c < 8; ++c) {
    uint32_t acc = 0, mybal = 0;
    for (int b = 0; b < 32; ++b) {
      const int ii = c * 32 + b;
      bool lt = false, gt = false;
      for (int k = 0; k < M; ++k) {
        float a = sFi[ii * M + k], bb = sFj[k * DOM_TILE + tid];
        lt |= a < bb;
        gt |= a > bb;
      }
      const bool both = vj && sVi[ii];
      const uint32_t bal = __ballot_sync(MO_FULL, both && gt && !lt);
      acc |= (uint32_t)(both && lt && !gt) << b;
      mybal = (lane == b) ? bal : mybal;
    }
    accw[c] = acc;
    sB2[(c * 32 + lane) * 9 + warp] = mybal;
  }
  if (j < R) {
    uint4* dst = reinterpret_cast<uint4*>(bits + (int64_t)j * W + (int64_t)bi * 8);
    dst[0] = make_uint4(accw[0], accw[1], accw[2], accw[3]);
    dst[1] = make_uint4(accw[4], accw[5], accw[6], accw[7]);
  }
  if (bi != bj) {
    __syncthreads();
    const int i = i0 + tid;
    if (i < R) {
      const uint32_t* s = sB2 + tid * 9;
      uint4* dst = reinterpret_cast<uint4*>(bits + (int64_t)i * W + (int64_t)bj * 8);
      dst[0] = make_uint4(s[0], s[1], s[2], s[3]);
      dst[1] = make_uint4(s[4], s[5], s[6], s[7]);
    }
  }
}

// ---------------------------------------------------------------- sorted path
//
// Engine path (mo_step): rows are presorted by S = FP32 left-to-right sum of
// their objectives.  S is monotone under component-wise <= (rounding is
// monotone), so j dominates i only if S_j <= S_i.  In an off-diagonal tile
// (bi < bj) with max S(bi) < min S(bj) no lane j can dominate any i
// and, S differing, "i dominates j" reduces to an m-long FSETP.LE AND chain:
// m compares per unordered pair instead of 2m plus ballots.  Tiles touching an
// S tie and the diagonal tiles run the symmetric code above.  The rows of bits
// are then indexed by sorted position; words past a row's S-tie group are
// never written (the peel is bounded by wend[p]).  hasdom[p] = 1 iff row p
// has at least one dominator, so front 0 needs no scan at all.

constexpr int DOMS_THREADS = DOM_TILE / 2;  // two j columns per thread

template <int NW>
__device__ __forceinline__ void store_words(uint32_t* dst, const uint32_t* w) {
  if (NW % 4 == 0) {
#pragma unroll
    for (int c = 0; c < NW; c += 4) reinterpret_cast<uint4*>(dst)[c / 4] = make_uint4(w[c], w[c + 1], w[c + 2], w[c + 3]);
  } else {
#pragma unroll
    for (int c = 0; c < NW; c += 2) reinterpret_cast<uint2*>(dst)[c / 2] = make_uint2(w[c], w[c + 1]);
  }
}

// TI = i rows per tile (256 or 128): a (256-row i block, 256-row j block) pair is split into 256/TI
// tiles of TI i rows each -- the same work in more, shorter CTAs, which shrinks the last partial wave
// (C2: 3,160 tiles of 256 = 2.1 waves -> 6,320 of 128).
template <int M, int TI>
__global__ void __launch_bounds__(DOMS_THREADS) k_dom_tile_sorted(const float* __restrict__ FS,
                                                                  const float* __restrict__ blkmin,
                                                                  const float* __restrict__ blkmax,
                                                                  const int* __restrict__ wend, int R,
                                                                  uint32_t* __restrict__ bits, int64_t W,
                                                                  uint8_t* __restrict__ hasdom) {
  pdl_wait();
  constexpr int MP = (M + 3) & ~3;
  constexpr int HALVES = DOM_TILE / TI;   // tiles per block pair
  constexpr int NW = TI / 32;             // words of a j row written by this tile
  __shared__ __align__(16) float sFi[TI * MP];
  __shared__ uint32_t sB2[TI * 9];
  int bi, bj;
  tri_decode(blockIdx.x / HALVES, bi, bj);
  const int h = blockIdx.x % HALVES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int i0 = bi * DOM_TILE + h * TI, j0 = bj * DOM_TILE;
  // rows past R are padded with +FLT_MAX: they dominate nothing and are never stored
  for (int e = tid; e < TI * MP; e += DOMS_THREADS) {
    int r = e / MP, k = e - r * MP;
    int i = i0 + r;
    sFi[e] = (k < M && i < R) ? FS[(int64_t)i * M + k] : 3.402823466e38f;
  }
  const int ja = j0 + tid, jb = j0 + tid + DOMS_THREADS;
  float fa[M], fb[M];
#pragma unroll
  for (int k = 0; k < M; ++k) {
    fa[k] = ja < R ? FS[(int64_t)ja * M + k] : 3.402823466e38f;
    fb[k] = jb < R ? FS[(int64_t)jb * M + k] : 3.402823466e38f;
  }
  const bool fast = (bi < bj) && (__ldg(blkmax + bi) < __ldg(blkmin + bj));
  __syncthreads();
  uint32_t wa[NW], wb[NW];
  if (fast) {
    // m-long setp.le.and chains + predicated OR.  (A sign-of-difference variant -- m FADD on the FMA
    // pipe + LOP3 + funnel shift -- measured no faster: the tile is issue-bound, not ALU-bound.)
#pragma unroll 1
    for (int c = 0; c < NW; ++c) {
      uint32_t acca = 0, accb = 0;
#pragma unroll
      for (int b = 0; b < 32; ++b) {
        const float* fi = sFi + (c * 32 + b) * MP;
        float v[M];
#pragma unroll
        for (int k = 0; k < M; ++k) v[k] = fi[k];
        Chain<M>::le(v, fa, acca, 1u << b);
        Chain<M>::le(v, fb, accb, 1u << b);
      }
      wa[c] = acca;
      wb[c] = accb;
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < NW; ++c) {
      uint32_t acca = 0, accb = 0, bala = 0, balb = 0;
#pragma unroll
      for (int b = 0; b < 32; ++b) {
        const float* fi = sFi + (c * 32 + b) * MP;
        float v[M];
#pragma unroll
        for (int k = 0; k < M; ++k) v[k] = fi[k];
        const uint32_t x = Chain<M>::sym(v, fa, acca, 1u << b);
        const uint32_t y = Chain<M>::sym(v, fb, accb, 1u << b);
        bala = (lane == b) ? x : bala;
        balb = (lane == b) ? y : balb;
      }
      wa[c] = acca;
      wb[c] = accb;
      sB2[(c * 32 + lane) * 9 + warp] = bala;
      sB2[(c * 32 + lane) * 9 + warp + 4] = balb;
    }
  }
  uint32_t anya = 0, anyb = 0;
#pragma unroll
  for (int c = 0; c < NW; ++c) {
    anya |= wa[c];
    anyb |= wb[c];
  }
  if (ja < R) {
    store_words<NW>(bits + (int64_t)ja * W + (int64_t)(i0 / 32), wa);
    if (anya) hasdom[ja] = 1;
  }
  if (jb < R) {
    store_words<NW>(bits + (int64_t)jb * W + (int64_t)(i0 / 32), wb);
    if (anyb) hasdom[jb] = 1;
  }
  if (fast) {
    // rows i of the last S bucket of bi may share it with rows of bj: their
    // words of block bj lie below wend and are read by the peel, so they must
    // hold zeros (no j of a fast tile dominates an i) rather than stale bits
    const int ilast = min(R, i0 + TI) - 1;
    if (ilast >= i0 && __ldg(wend + ilast) > bj * 8) {
      for (int r = tid; r < TI; r += DOMS_THREADS) {
        const int i = i0 + r;
        if (i < R && __ldg(wend + i) > bj * 8) {
          uint4* dst = reinterpret_cast<uint4*>(bits + (int64_t)i * W + (int64_t)bj * 8);
          dst[0] = make_uint4(0u, 0u, 0u, 0u);
          dst[1] = make_uint4(0u, 0u, 0u, 0u);
        }
      }
    }
  }
  if (!fast && bi != bj) {
    __syncthreads();
    for (int r = tid; r < TI; r += DOMS_THREADS) {
      const int i = i0 + r;
      if (i < R) {
        const uint32_t* sw = sB2 + r * 9;
        uint4* dst = reinterpret_cast<uint4*>(bits + (int64_t)i * W + (int64_t)bj * 8);
        dst[0] = make_uint4(sw[0], sw[1], sw[2], sw[3]);
        dst[1] = make_uint4(sw[4], sw[5], sw[6], sw[7]);
        if ((sw[0] | sw[1] | sw[2] | sw[3] | sw[4] | sw[5] | sw[6] | sw[7]) != 0u) hasdom[i] = 1;
      }
    }
  }
  pdl_trigger();   // multi-wave grid: let the peel's CTAs in only as this CTA retires
}

int64_t words_per_row(int64_t R) { return round_up(R, DOM_TILE) / 32; }

int launch_dom_tile(const float* F, int64_t R, int m, const uint8_t* valid, uint32_t* bits, cudaStream_t s) {
  if (R <= 0) return MO_OK;
  if (m < 1 || R > (1ll << 31) - 1) return MO_ERR_PARAM;
  const int64_t W = words_per_row(R);
  const int64_t nb = W / 8;
  const int64_t tiles = nb * (nb + 1) / 2;
  if (tiles > 0x7fffffffll) return MO_ERR_PARAM;
  dim3 grid((unsigned)tiles);
  switch (m) {
#define MO_DOM_CASE(MM) \
  case MM: k_dom_tile<MM><<<grid, DOM_TILE, 0, s>>>(F, (int)R, valid, bits, W); break;
    MO_DOM_CASE(1)
    MO_DOM_CASE(2)
    MO_DOM_CASE(3)
    MO_DOM_CASE(4)
    MO_DOM_CASE(5)
    MO_DOM_CASE(6)
    MO_DOM_CASE(7)
    MO_DOM_CASE(8)
    MO_DOM_CASE(9)
    MO_DOM_CASE(10)
#undef MO_DOM_CASE
    default: {
      size_t smem = (size_t)2 * DOM_TILE * m * sizeof(float);
      if (smem > 200 * 1024) return MO_ERR_PARAM;
      cudaFuncSetAttribute(k_dom_tile_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_dom_tile_generic<<<grid, DOM_TILE, smem, s>>>(F, (int)R, m, valid, bits, W);
    }
  }
  MO_CHECK_LAUNCH();
  return MO_OK;
}


int launch_dom_tile_sorted(const float* FS, const float* blkmin, const float* blkmax, const int* wend, int64_t R,
                           int m, uint32_t* bits, uint8_t* hasdom, cudaStream_t s, bool clear_hasdom) {
  if (R <= 0) return MO_OK;
  const int64_t W = words_per_row(R);
  const int64_t nb = W / 8;
  const int64_t pairs = nb * (nb + 1) / 2;
  // 128-row i tiles: 256-row tiles leave a ragged last wave on small grids (C2: 0.105 -> 0.095 ms;
  // 64-row tiles measured the same as 128)
  constexpr int TI = 128;
  const int64_t tiles = pairs * (DOM_TILE / TI);
  if (tiles > 0x7fffffffll) return MO_ERR_PARAM;
  if (clear_hasdom && cudaMemsetAsync(hasdom, 0, (size_t)R, s) != cudaSuccess) return MO_ERR_CUDA;
  dim3 grid((unsigned)tiles);
  switch (m) {
#define MO_DOMS_CASE(MM) \
  case MM:                                                                                                  \
    MO_TRY(launch_ex(k_dom_tile_sorted<MM, TI>, grid, dim3(DOMS_THREADS), 0, s, false, g_mo_pdl, FS, blkmin,    \
                     blkmax, wend, (int)R, bits, W, hasdom));                                                 \
    break;
    MO_DOMS_CASE(2)
    MO_DOMS_CASE(3)
    MO_DOMS_CASE(4)
    MO_DOMS_CASE(5)
    MO_DOMS_CASE(6)
    MO_DOMS_CASE(7)
    MO_DOMS_CASE(8)
    MO_DOMS_CASE(9)
    MO_DOMS_CASE(10)
    MO_DOMS_CASE(11)
    MO_DOMS_CASE(12)
    MO_DOMS_CASE(13)
    MO_DOMS_CASE(14)
    MO_DOMS_CASE(15)
    MO_DOMS_CASE(16)
#undef MO_DOMS_CASE
    default:
      return MO_ERR_PARAM;
  }
  MO_CHECK_LAUNCH();
  return MO_OK;
}

// ---------------------------------------------------------------- presort
//
// k_presort (persistent, all SMs): S_i = ((f_i0 + f_i1) + ...) in FP32 and
// key_i = ord(S_i); rows are bucketed by a 16-bit quantisation of key_i over
// [min key, max key] (monotone in S), i.e. one counting-sort pass:
//   P0 S, key, key range      P1 bucket histogram     P2 bucket starts (scan)
//   P3 scatter rows to FS/SS  P4 wend + per-256-row block min/max of S.
// Order inside a bucket is arbitrary (the bit layout may differ run to run,
// the ranks cannot: fronts are a function of the point set).  Because buckets
// are S-ordered, a row's dominators lie at earlier positions or in its own
// bucket, so wend[p] = one past the word of its bucket's last position, and a
// tile (bi < bj) is free of reverse dominance when max S(bi) < min S(bj).
constexpr int PRESORT_THREADS = 512;

__global__ void __launch_bounds__(PRESORT_THREADS) k_presort(PresortArgs a) {
  pdl_wait();
  __shared__ int sh[40];
  __shared__ unsigned sMin, sMax;
  __shared__ int sWcnt[(PRESORT_THREADS / 32) * 256], sRun[256], sOff[256];
  const int tid = threadIdx.x, lane = tid & 31;
  const int gtid = blockIdx.x * blockDim.x + tid, gthreads = gridDim.x * blockDim.x;
  const int R = a.R, m = a.m;
  const int NB = presort_buckets(R);
  // row loops of P0 / P3: wide rows (m > 16) are dealt round-robin over the CTAs (row b + G t) so the
  // strided row reads spread over every SM's L1 instead of the first few CTAs'
  const int rstart = m > 16 ? (int)blockIdx.x + (int)gridDim.x * tid : gtid;
  trace_mark(a.trace, 0);
  // P0: sums, keys, key range; clear bucket counts and fill cursors
  if (tid == 0) {
    sMin = 0xffffffffu;
    sMax = 0u;
  }
  for (int q = gtid; q < NB; q += gthreads) {
    a.valB[q] = 0;
    a.fill[q] = 0;
  }
  __syncthreads();
  unsigned kmin = 0xffffffffu, kmax = 0u;
  for (int i = rstart; i < R; i += gthreads) {
    const float* f = a.F + (int64_t)i * m;
    float s = f[0];
    for (int k = 1; k < m; ++k) s = __fadd_rn(s, f[k]);
    const uint32_t key = f2ord(s);
    a.keyB[i] = key;
    kmin = min(kmin, key);
    kmax = max(kmax, key);
  }
  kmin = warp_min_u32(kmin);
  kmax = warp_max_u32(kmax);
  if (lane == 0) {
    atomicMin(&sMin, kmin);
    atomicMax(&sMax, kmax);
  }
  __syncthreads();
  if (tid == 0) {
    atomicMax(&a.ctl[0], ~sMin);   // ~min: 0 is the neutral value (no reset node needed)
    atomicMax(&a.ctl[1], sMax);
  }
  grid_sync(a.g.bar);
  trace_mark(a.trace, 1);
  // P1: bucket of every row + histogram
  const uint32_t lo = ~__ldcg(a.ctl), hi = __ldcg(a.ctl + 1);
  const uint64_t span = (uint64_t)(hi - lo) + 1ull;
  for (int i = gtid; i < R; i += gthreads) {
    const uint32_t key = __ldcg(a.keyB + i);
    const uint32_t q = (uint32_t)(((uint64_t)(key - lo) * (uint64_t)NB) / span);
    a.keyA[i] = q;
    if (a.stable) a.valA[i] = i;
    atomicAdd(&a.valB[q], 1);
  }
  grid_sync(a.g.bar);
  trace_mark(a.trace, 2);
  // P2: exclusive scan of the bucket counts -> bucket starts (in fill[] to keep counts)
  grid_scan(
      a.g, NB, [&](int64_t q) { return __ldcg(a.valB + q); },
      [&](int64_t q, int pre) {
        // atomic path: valB[q] becomes the bucket END (its count is not needed any more), so P3 can
        // write wend and the block S bounds itself (no P3 -> P4 barrier)
        if (!a.stable) a.valB[q] = pre + __ldcg(a.valB + q);
        a.fill[q] = pre;
      },
      sh);
  grid_sync(a.g.bar);
  trace_mark(a.trace, 3);
  // every block has read the key range (P1): restore its neutral values for the next launch
  if (gtid == 0) {
    a.ctl[0] = 0u;
    a.ctl[1] = 0u;
  }
  if (a.hasdom)
    for (int p = gtid; p < R; p += gthreads) a.hasdom[p] = 0;
  // P3: scatter rows into their buckets
  if (a.stable) {
    // (bucket, row) pairs sorted by bucket, rows ascending inside a bucket
    grid_radix_pass(a.g, R, 0, a.keyA, a.valA, a.tkey, a.tval, sWcnt, sRun, sOff, sh);
    grid_radix_pass(a.g, R, 8, a.tkey, a.tval, a.keyA, a.valA, sWcnt, sRun, sOff, sh);
    for (int pos = gtid; pos < R; pos += gthreads) {
      const int i = __ldcg(a.valA + pos);
      a.perm[pos] = i;
      a.SS[pos] = ord2f(__ldcg(a.keyB + i));
      for (int k = 0; k < m; ++k) a.FS[(int64_t)pos * m + k] = __fadd_rn(a.F[(int64_t)i * m + k], 0.0f);  // -0 -> +0
    }
    // bucket ends for P4 (the atomic path leaves fill[q] at the end of bucket q)
    for (int q = gtid; q < NB; q += gthreads) a.fill[q] += __ldcg(a.valB + q);
    grid_sync(a.g.bar);
    // keyA was overwritten by the sorted keys: restore row -> bucket for P4
    for (int pos = gtid; pos < R; pos += gthreads) a.tkey[__ldcg(a.valA + pos)] = __ldcg(a.keyA + pos);
    grid_sync(a.g.bar);
  } else {
    for (int i = rstart; i < R; i += gthreads) {
      const uint32_t q = __ldcg(a.keyA + i);
      const int pos = atomicAdd(&a.fill[q], 1);
      a.perm[pos] = i;
      a.SS[pos] = ord2f(__ldcg(a.keyB + i));
      for (int k = 0; k < m; ++k) a.FS[(int64_t)pos * m + k] = __fadd_rn(a.F[(int64_t)i * m + k], 0.0f);  // -0 -> +0
      // P4 folded in: wend from the bucket end; the 256-row block S range from the key range of the
      // buckets at the block's first / last position (conservative: the fast-tile test max S(bi) <
      // min S(bj) stays sound, adjacent blocks sharing a bucket are simply not fast)
      a.wend[pos] = (__ldcg(a.valB + q) - 1) / 32 + 1;
      if ((pos & 255) == 0) {
        const uint64_t kmin = (uint64_t)q * span;
        a.blkmin[pos >> 8] = ord2f(lo + (uint32_t)((kmin + NB - 1) / NB));
      }
      if ((pos & 255) == 255 || pos == R - 1) {
        const uint64_t kmax = ((uint64_t)q + 1) * span;
        a.blkmax[pos >> 8] = ord2f(lo + (uint32_t)((kmax + NB - 1) / NB) - 1u);
      }
    }
    trace_mark(a.trace, 4);
    trace_mark(a.trace, 5);
    return;
  }
  grid_sync(a.g.bar);
  const uint32_t* rowq = a.stable ? a.tkey : a.keyA;
  trace_mark(a.trace, 4);
  // P4: wend (after P3 fill[q] = end of bucket q) and per-256-row S range
  for (int p = gtid; p < R; p += gthreads) {
    const int i = __ldcg(a.perm + p);
    const uint32_t q = __ldcg(rowq + i);
    const int last = __ldcg(a.fill + q) - 1;
    a.wend[p] = last / 32 + 1;
  }
  const int nblk = (R + 255) / 256;
  for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
    float mn = 3.402823466e38f, mx = -3.402823466e38f;
    for (int p = b * 256 + tid; p < min(R, b * 256 + 256); p += blockDim.x) {
      const float v = __ldcg(a.SS + p);
      mn = fminf(mn, v);
      mx = fmaxf(mx, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(MO_FULL, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(MO_FULL, mx, o));
    }
    __shared__ float wmn[PRESORT_THREADS / 32], wmx[PRESORT_THREADS / 32];
    if (lane == 0) {
      wmn[tid >> 5] = mn;
      wmx[tid >> 5] = mx;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < PRESORT_THREADS / 32; ++w) {
        mn = fminf(mn, wmn[w]);
        mx = fmaxf(mx, wmx[w]);
      }
      a.blkmin[b] = fminf(mn, wmn[0]);
      a.blkmax[b] = fmaxf(mx, wmx[0]);
    }
    __syncthreads();
  }
  trace_mark(a.trace, 5);
}

// k_presort_small: the same counting sort for R <= PS_MAXR rows in ONE 1024-thread CTA with the keys and
// bucket counters in shared memory -- no grid barriers (the multi-CTA version spends most of its ~22 us at
// C2 in six of them).  Buckets: min(presort_buckets(R), PS_MAXNB); as in k_presort the order inside a
// bucket is arbitrary and only S-monotonicity of the buckets matters.  Row state in shared memory:
// key (P0) -> bucket (P1) -> (bucket << 15 | position) (P3).
constexpr int PS_THREADS = 1024;
constexpr int PS_MAXR = 32768;
constexpr int PS_MAXNB = 16384;

size_t presort_small_smem(int R) {
  const int nb = presort_buckets(R) < PS_MAXNB ? presort_buckets(R) : PS_MAXNB;
  return (size_t)R * 4 + (size_t)nb * 4;
}

__global__ void __launch_bounds__(PS_THREADS, 1) k_presort_small(PresortArgs a) {
  pdl_wait();
  extern __shared__ uint32_t ps_smem[];
  __shared__ unsigned sMin, sMax;
  __shared__ int sh[40];
  const int R = a.R, m = a.m, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NB = presort_buckets(R) < PS_MAXNB ? presort_buckets(R) : PS_MAXNB;
  uint32_t* sKQ = ps_smem;
  int* sCnt = reinterpret_cast<int*>(ps_smem + R);
  trace_mark(a.trace, 0);
  if (tid == 0) {
    sMin = 0xffffffffu;
    sMax = 0u;
  }
  for (int q = tid; q < NB; q += PS_THREADS) sCnt[q] = 0;
  if (a.hasdom)
    for (int p = tid; p < R; p += PS_THREADS) a.hasdom[p] = 0;
  __syncthreads();
  // P0: S, key, key range
  unsigned kmin = 0xffffffffu, kmax = 0u;
#pragma unroll 4
  for (int i = tid; i < R; i += PS_THREADS) {
    const float* f = a.F + (int64_t)i * m;
    float sm = f[0];
    for (int k = 1; k < m; ++k) sm = __fadd_rn(sm, f[k]);
    const uint32_t key = f2ord(sm);
    sKQ[i] = key;
    kmin = min(kmin, key);
    kmax = max(kmax, key);
  }
  kmin = warp_min_u32(kmin);
  kmax = warp_max_u32(kmax);
  if (lane == 0) {
    atomicMin(&sMin, kmin);
    atomicMax(&sMax, kmax);
  }
  __syncthreads();
  trace_mark(a.trace, 1);
  // P1: bucket + histogram (shared-memory atomics)
  const uint32_t lo = sMin;
  const uint64_t span = (uint64_t)(sMax - lo) + 1ull;
  for (int i = tid; i < R; i += PS_THREADS) {
    const uint32_t q = (uint32_t)(((uint64_t)(sKQ[i] - lo) * (uint64_t)NB) / span);
    sKQ[i] = q;
    atomicAdd(&sCnt[q], 1);
  }
  __syncthreads();
  trace_mark(a.trace, 2);
  // P2: exclusive scan of the counts (NB is a multiple of PS_THREADS: consecutive runs per thread)
  {
    const int per = NB / PS_THREADS, q0 = tid * per;
    int run = 0;
    for (int q = q0; q < q0 + per; ++q) run += sCnt[q];
    int total;
    int pre = block_excl_scan(run, sh, &total);
    for (int q = q0; q < q0 + per; ++q) {
      const int c = sCnt[q];
      sCnt[q] = pre;
      pre += c;
    }
  }
  __syncthreads();
  trace_mark(a.trace, 3);
  // P3: scatter (after it sCnt[q] = end of bucket q)
#pragma unroll 2
  for (int i = tid; i < R; i += PS_THREADS) {
    const uint32_t q = sKQ[i];
    const int pos = atomicAdd(&sCnt[q], 1);
    sKQ[i] = (q << 15) | (uint32_t)pos;
    const float* f = a.F + (int64_t)i * m;
    float* fs = a.FS + (int64_t)pos * m;
    float sm = f[0];
    fs[0] = __fadd_rn(sm, 0.0f);   // -0 -> +0
    for (int k = 1; k < m; ++k) {
      const float v = f[k];
      sm = __fadd_rn(sm, v);
      fs[k] = __fadd_rn(v, 0.0f);
    }
    a.perm[pos] = i;
    a.SS[pos] = sm;                // == ord2f(key): the same FP32 sum
  }
  __syncthreads();
  trace_mark(a.trace, 4);
  // P4: wend, then per-256-row S range (SS written above by this CTA)
  for (int i = tid; i < R; i += PS_THREADS) {
    const uint32_t v = sKQ[i];
    a.wend[v & 0x7fffu] = (sCnt[v >> 15] - 1) / 32 + 1;
  }
  const int nblk = (R + 255) / 256;
  for (int b = warp; b < nblk; b += PS_THREADS / 32) {
    float mn = 3.402823466e38f, mx = -3.402823466e38f;
    for (int p = b * 256 + lane; p < min(R, b * 256 + 256); p += 32) {
      const float v = a.SS[p];
      mn = fminf(mn, v);
      mx = fmaxf(mx, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(MO_FULL, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(MO_FULL, mx, o));
    }
    if (lane == 0) {
      a.blkmin[b] = mn;
      a.blkmax[b] = mx;
    }
  }
  trace_mark(a.trace, 5);
}

int launch_presort(const PresortArgs& args, cudaStream_t s) {
  static int maxb = 0;
  if (!maxb) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_presort, PRESORT_THREADS, 0);
    maxb = sms * (per > 0 ? (per > 1 ? 1 : per) : 1);
  }
  static int small_max = -1;
  if (small_max < 0) {   // crossover (rows) below which the single-CTA presort wins; MO_PRESORT_SMALL_MAX overrides
    const char* e = getenv("MO_PRESORT_SMALL_MAX");
    small_max = e ? atoi(e) : 2048;
    if (small_max > PS_MAXR) small_max = PS_MAXR;
  }
  // (and wide rows: the one-CTA version reads R x m strided values through a single SM)
  if (!args.stable && args.R <= small_max && (int64_t)args.R * args.m <= 32768) {
    static bool attr = false;
    if (!attr) {
      if (cudaFuncSetAttribute(k_presort_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)presort_small_smem(PS_MAXR)) != cudaSuccess)
        return MO_ERR_CUDA;
      attr = true;
    }
    return launch_ex(k_presort_small, dim3(1), dim3(PS_THREADS), presort_small_smem(args.R), s, false,
                     g_mo_pdl && args.in_step, args);
  }
  const int NB = presort_buckets(args.R);
  // rows drive the grid (a CTA per 128 rows: C2's bucket scan wants ~all SMs); a tiny population keeps
  // one or two CTAs so its grid barriers stay cheap (C1: 8 -> 2 CTAs, 0.116 -> 0.106 ms/generation)
  const int64_t by_rows = ceil_div((int64_t)args.R, (int64_t)(PRESORT_THREADS / 2));
  const int64_t by_buckets = ceil_div((int64_t)NB, (int64_t)(PRESORT_THREADS * 4));
  int blocks = (int)(by_rows > by_buckets ? by_rows : by_buckets);
  if (args.m > 16) blocks = (int)ceil_div((int64_t)args.R, (int64_t)8);   // wide rows: ~8 rows per CTA
  if (blocks > maxb) blocks = maxb;
  if (blocks < 1) blocks = 1;
  if (!args.in_step) {
    if (cudaMemsetAsync(args.g.bar, 0, 2 * sizeof(unsigned), s) != cudaSuccess) return MO_ERR_CUDA;
    if (cudaMemsetAsync(args.ctl, 0, 2 * sizeof(unsigned), s) != cudaSuccess) return MO_ERR_CUDA;
  }
  return launch_ex(k_presort, dim3(blocks), dim3(PRESORT_THREADS), 0, s, true, g_mo_pdl && args.in_step, args);
}

// ------------------------------------------------------------------ peeling

struct PeelArgs {
  const uint32_t* bits;
  int R;
  int64_t W;
  const uint8_t* valid;    // nullable (per row, position space)
  int64_t stop_at;
  int* ranks;              // output, original row order
  int* info;
  int* resume;
  uint32_t* ranked;
  int* front_sizes;
  unsigned* bar;
  // sorted engine path (all nullable): position -> row map, rows' "has any
  // dominator" flags, exclusive word bound of each row's possible dominators,
  // and the position-space rank scratch
  const int* perm;
  const uint8_t* hasdom;
  const int* wend;
  int* rank_pos;
  unsigned long long* trace;  // nullable phase trace (slots 8..11)
  // nullable tile summary (k_dom_rank): only flagged 256-bit word blocks were stored; resume[] then
  // counts word blocks instead of words
  const uint32_t* tsum;
  int64_t TW;
};

constexpr int PEEL_THREADS = 256;

// Phase A of one row with a tile summary: 8 lanes (l8) walk row j's summary words from block `t0`
// (8 summary words = 256 blocks per step); each lane tests its flagged blocks (2 x uint4 of the
// dominators' words against the ranked mask) in ascending order and stops at its first unranked
// dominator; the group keeps the smallest such block.  Returns the first blocking block, or -1 when
// every flagged block below tlim holds ranked dominators only.
__device__ __forceinline__ int64_t peel_row_summary(const PeelArgs& a, int64_t j, bool active, int64_t t0,
                                                    int64_t tlim, int l8, uint32_t gmask) {
  int64_t blocked_at = -1;
  int64_t sw0 = t0 >> 5;
  for (;;) {
    const bool scanning = active && blocked_at < 0 && (sw0 << 5) < tlim;
    if (__ballot_sync(MO_FULL, scanning) == 0) break;
    uint32_t f = 0;
    if (scanning) {
      const int64_t swi = sw0 + l8;
      if ((swi << 5) < tlim) {
        f = __ldcg(a.tsum + j * a.TW + swi);
        if (swi == (t0 >> 5)) f &= 0xffffffffu << (t0 & 31);              // blocks before the resume block
        const int64_t rem = tlim - (swi << 5);
        if (rem < 32) f &= (1u << rem) - 1u;
      }
    }
    // the group's 8 summary words in block order; the 8 lanes split each nonzero word's flagged blocks
    // (dense rows: up to 4 blocks per lane per word, in parallel), and the first word with an unranked
    // dominator ends the scan at its smallest such block
    int64_t hit = INT64_MAX;
    for (int k = 0; k < 8; ++k) {
      const uint32_t wk = __shfl_sync(MO_FULL, f, k, 8);
      if (wk == 0u || hit != INT64_MAX) continue;   // uniform within the 8-lane group
      const int nbits = __popc(wk);
      int64_t tmin = INT64_MAX;
      for (int r = l8; r < nbits; r += 8) {
        const int bpos = (int)__fns(wk, 0, r + 1);
        const int64_t t = ((sw0 + k) << 5) + bpos;
        const uint4* bw = reinterpret_cast<const uint4*>(a.bits + j * a.W + t * 8);
        const uint4* rw = reinterpret_cast<const uint4*>(a.ranked + t * 8);
        const uint4 b0 = __ldg(bw), b1 = __ldg(bw + 1);
        const uint4 r0 = __ldcg(rw), r1 = __ldcg(rw + 1);
        const uint32_t h = (b0.x & ~r0.x) | (b0.y & ~r0.y) | (b0.z & ~r0.z) | (b0.w & ~r0.w) |
                           (b1.x & ~r1.x) | (b1.y & ~r1.y) | (b1.z & ~r1.z) | (b1.w & ~r1.w);
        if (h && t < tmin) tmin = t;
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        const int64_t ot = __shfl_xor_sync(gmask, tmin, o, 8);
        tmin = ot < tmin ? ot : tmin;
      }
      hit = tmin;
    }
    if (scanning) {
      if (hit != INT64_MAX)
        blocked_at = hit;
      else
        sw0 += 8;
    }
  }
  return blocked_at;
}

__global__ void __launch_bounds__(PEEL_THREADS) k_front_peel(PeelArgs a) {
  pdl_wait();
  __shared__ int sCount[PEEL_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  const int gthreads = gridDim.x * blockDim.x;
  const int gtid = blockIdx.x * blockDim.x + tid;
  const int R = a.R;
  const int64_t W = a.W;
  const int nwords_used = (R + 31) / 32;
  int* rk = a.perm ? a.rank_pos : a.ranks;   // ranks indexed by bit-matrix row
  trace_mark(a.trace, 8);

  // prologue: ranks / resume / ranked mask (invalid rows count as ranked so they never block).
  // pre0 (all rows valid, hasdom from the tile kernel): front 0 is found here too -- its rows are the
  // ones without a dominator, a per-row test on the same thread-to-row mapping -- and counted into a
  // spare slot of front_sizes, so the first barrier publishes it (one barrier less per generation)
  const bool pre0 = a.valid == nullptr && a.hasdom != nullptr;
  int* fs0 = a.front_sizes + R + 3;   // zero at entry; reset by the last block after every read
  int nvalid_local = 0, ready0 = 0;
  for (int j = gtid; j < R; j += gthreads) {
    bool v = a.valid == nullptr || a.valid[j];
    int r = v ? MO_RANK_UNRANKED : MO_RANK_DROPPED;
    if (pre0 && a.hasdom[j] == 0) {
      r = 0;
      ready0++;
    }
    rk[j] = r;
    a.resume[j] = 0;
    nvalid_local += v;
  }
  if (pre0) {
    ready0 = warp_sum(ready0);
    if (lane == 0) sCount[wib] = ready0;
    __syncthreads();
    if (tid == 0) {
      int s0 = 0;
      for (int w = 0; w < PEEL_THREADS / 32; ++w) s0 += sCount[w];
      if (s0) atomicAdd(fs0, s0);
    }
    if (gtid == 0) a.front_sizes[2] = 0;   // front 1's counter (phase A of front 0 is skipped)
  }
  for (int64_t w = gtid; w < W; w += gthreads) {
    uint32_t m = 0;
    if (w < nwords_used) {
      for (int b = 0; b < 32; ++b) {
        int64_t j = w * 32 + b;
        bool ranked = (j >= R) || (a.valid != nullptr && !a.valid[j]);
        m |= (uint32_t)ranked << b;
      }
    } else {
      m = 0xffffffffu;
    }
    a.ranked[w] = m;
  }
  nvalid_local = warp_sum(nvalid_local);
  if (!pre0 && lane == 0) atomicAdd(&a.front_sizes[0], nvalid_local);
  if (!pre0 && gtid == 0) a.front_sizes[1] = 0;
  grid_sync(a.bar);
  trace_mark(a.trace, 9);
  const int nvalid = pre0 ? R : __ldcg(a.front_sizes);
  const int64_t target = a.stop_at > 0 ? a.stop_at : (int64_t)nvalid;
  if (a.stop_at > 0 && nvalid < a.stop_at) {
    grid_sync(a.bar);            // everyone has read front_sizes[0]
    if (gtid == 0) {
      a.info[MO_INFO_ERROR] = MO_ERR_INFEASIBLE;
      if (a.info[MO_INFO_ERROR_FIRST] == 0) a.info[MO_INFO_ERROR_FIRST] = MO_ERR_INFEASIBLE;
      a.info[MO_INFO_L] = -1;
      a.front_sizes[0] = 0;      // neutral for the next launch (no memset node)
      if (pre0) *fs0 = 0;
    }
    return;
  }

  const int gwarp = gtid >> 5, nwarps = gthreads >> 5;
  const int g8 = lane >> 3, l8 = lane & 7;
  const uint32_t gmask = 0xffu << (lane & ~7);
  int64_t cum = 0;
  int k = 0;
  for (;;) {
    // ---- phase A: find front k
    int ready_local = 0;
    if (k == 0 && pre0) {
      // found in the prologue
    } else if (k == 0 && a.hasdom) {
      // front 0 = rows without any dominator, known from the tile kernel
      for (int j = gtid; j < R; j += gthreads) {
        if (rk[j] == MO_RANK_UNRANKED && a.hasdom[j] == 0) {
          rk[j] = 0;
          ready_local++;
        }
      }
    } else if (a.tsum) {
      for (int rb = gwarp * 4; rb < R; rb += nwarps * 4) {
        const int j = rb + g8;
        const bool active = (j < R) && (__ldcg(rk + j) == MO_RANK_UNRANKED);
        const int64_t tlim = active ? ((int64_t)a.wend[j] + 7) / 8 : 0;
        const int64_t t0 = active ? (int64_t)a.resume[j] : 0;
        const int64_t bl = peel_row_summary(a, j, active, t0, tlim, l8, gmask);
        if (active && l8 == 0) {
          if (bl >= 0) {
            a.resume[j] = (int)bl;
          } else {
            rk[j] = k;
            ready_local++;
          }
        }
      }
    } else {
      for (int rb = gwarp * 4; rb < R; rb += nwarps * 4) {
        const int j = rb + g8;
        bool active = (j < R) && (__ldcg(rk + j) == MO_RANK_UNRANKED);
        const int64_t wlim = (active && a.wend) ? (int64_t)a.wend[j] : W;
        int64_t base = active ? (int64_t)a.resume[j] : W;
        bool blocked = false;
        for (;;) {
          const bool scanning = active && !blocked && base < wlim;
          if (__ballot_sync(MO_FULL, scanning) == 0) break;
          bool hit = false;
          if (scanning) {
            const int64_t idx = base + l8 * 4;
            if (idx < wlim) {
              uint4 b4 = __ldg(reinterpret_cast<const uint4*>(a.bits + (int64_t)j * W + idx));
              uint4 r4 = __ldcg(reinterpret_cast<const uint4*>(a.ranked + idx));
              uint32_t h = b4.x & ~r4.x;
              if (idx + 1 < wlim) h |= b4.y & ~r4.y;
              if (idx + 2 < wlim) h |= b4.z & ~r4.z;
              if (idx + 3 < wlim) h |= b4.w & ~r4.w;
              hit = h != 0u;
            }
          }
          const uint32_t hb = __ballot_sync(MO_FULL, hit);
          if (scanning) {
            if (hb & gmask)
              blocked = true;
            else
              base += 32;
          }
        }
        if (active && l8 == 0) {
          if (blocked) {
            a.resume[j] = (int)base;
          } else {
            rk[j] = k;
            ready_local++;
          }
        }
      }
    }
    int fk;
    if (k == 0 && pre0) {
      fk = __ldcg(fs0);
      if (gtid == 0) a.front_sizes[1] = fk;   // the front-size record later readers use
    } else {
      ready_local = warp_sum(ready_local);
      if (lane == 0) sCount[wib] = ready_local;
      __syncthreads();
      if (tid == 0) {
        int s = 0;
        for (int w = 0; w < PEEL_THREADS / 32; ++w) s += sCount[w];
        if (s) atomicAdd(&a.front_sizes[k + 1], s);
      }
      if (gtid == 0) a.front_sizes[k + 2] = 0;
      grid_sync(a.bar);
      // ---- phase B: decide, then publish front k into the ranked mask
      fk = __ldcg(a.front_sizes + k + 1);
    }
    cum += fk;
    const bool done = (cum >= target) || (fk == 0);
    if (done) {
      for (int j = gtid; j < R; j += gthreads) {
        int r = __ldcg(rk + j);
        if (r == MO_RANK_UNRANKED) {
          r = MO_RANK_DROPPED;
          if (!a.perm) rk[j] = r;
        }
        if (a.perm) a.ranks[a.perm[j]] = r;
      }
      if (gtid == 0) {
        const int64_t sel = cum - fk;
        a.info[MO_INFO_L] = k;
        a.info[MO_INFO_SELECTED] = (int)sel;
        a.info[MO_INFO_K] = a.stop_at > 0 ? (int)(a.stop_at - sel) : fk;
        a.info[MO_INFO_NFRONTS] = k + 1;
        a.info[MO_INFO_FL_SIZE] = fk;
        a.info[MO_INFO_SKIPPED] = (a.stop_at > 0 && sel + fk == a.stop_at) ? 1 : 0;
        a.info[MO_INFO_ERROR] = 0;
        if (!pre0) a.front_sizes[0] = 0;    // read by every block after the prologue barrier, long passed
      }
      // pre0: every block has read fs0 before getting here; the last one restores its neutral value
      if (pre0 && grid_last(a.bar) && tid == 0) *fs0 = 0;
      trace_mark(a.trace, 10);
      return;
    }
    for (int64_t w = gwarp; w < nwords_used; w += nwarps) {
      const int64_t j = w * 32 + lane;
      const bool in = (j < R) && (__ldcg(rk + j) == k);
      const uint32_t m = __ballot_sync(MO_FULL, in);
      if (lane == 0 && m) a.ranked[w] |= m;
    }
    grid_sync(a.bar);
    if (k == 0 && pre0 && gtid == 0) *fs0 = 0;   // every block read it before this barrier
    ++k;
  }
}

int peel_grid_blocks() {
  static int blocks = 0;
  if (blocks == 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_front_peel, PEEL_THREADS, 0);
    if (per > 4) per = 4;
    blocks = sms * (per > 0 ? per : 1);
  }
  return blocks;
}

int launch_front_peel(const uint32_t* bits, int64_t R, const uint8_t* valid, int64_t stop_at, int* ranks,
                      int* info, int* resume, uint32_t* ranked, int* front_sizes, unsigned* bar,
                      const int* perm, const uint8_t* hasdom, const int* wend, int* rank_pos,
                      unsigned long long* trace, cudaStream_t s, bool in_step, const uint32_t* tsum) {
  if (R <= 0) return MO_ERR_PARAM;
  if (tsum && !wend) return MO_ERR_PARAM;
  PeelArgs a{bits, (int)R, words_per_row(R), valid, stop_at, ranks, info, resume, ranked, front_sizes, bar,
             perm, hasdom, wend, rank_pos, trace, tsum, tsum_words(R)};
  if (!in_step) {
    if (cudaMemsetAsync(front_sizes, 0, 2 * sizeof(int), s) != cudaSuccess) return MO_ERR_CUDA;
    if (cudaMemsetAsync(front_sizes + R + 3, 0, sizeof(int), s) != cudaSuccess) return MO_ERR_CUDA;
    if (cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), s) != cudaSuccess) return MO_ERR_CUDA;
  }
  int blocks = peel_grid_blocks();
  // two grid barriers per front: ~32 rows per warp keeps the barriers cheap
  int needed = (int)ceil_div(R, (PEEL_THREADS / 32) * 32);
  if (blocks > needed) blocks = needed < 1 ? 1 : needed;
  return launch_ex(k_front_peel, dim3(blocks), dim3(PEEL_THREADS), 0, s, true, g_mo_pdl && in_step, a);
}

}  // namespace mo
