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
#include "mo_common.cuh"

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

// ------------------------------------------------------------------ peeling

struct PeelArgs {
  const uint32_t* bits;
  int R;
  int64_t W;
  const uint8_t* valid;
  int64_t stop_at;
  int* ranks;
  int* info;
  int* resume;
  uint32_t* ranked;
  int* front_sizes;
  unsigned* bar;
};

constexpr int PEEL_THREADS = 256;

__global__ void __launch_bounds__(PEEL_THREADS) k_front_peel(PeelArgs a) {
  __shared__ int sCount[PEEL_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  const int gthreads = gridDim.x * blockDim.x;
  const int gtid = blockIdx.x * blockDim.x + tid;
  const int R = a.R;
  const int64_t W = a.W;
  const int nwords_used = (R + 31) / 32;

  // prologue: ranks / resume / ranked mask (invalid rows count as ranked so they never block)
  int nvalid_local = 0;
  for (int j = gtid; j < R; j += gthreads) {
    bool v = a.valid == nullptr || a.valid[j];
    a.ranks[j] = v ? MO_RANK_UNRANKED : MO_RANK_DROPPED;
    a.resume[j] = 0;
    nvalid_local += v;
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
  // valid-row count -> front_sizes[-1] slot (front_sizes[0] of the array is reserved)
  nvalid_local = warp_sum(nvalid_local);
  if (lane == 0) atomicAdd(&a.front_sizes[0], nvalid_local);
  if (gtid == 0) a.front_sizes[1] = 0;
  grid_sync(a.bar);
  const int nvalid = __ldcg(a.front_sizes);
  const int64_t target = a.stop_at > 0 ? a.stop_at : (int64_t)nvalid;
  if (a.stop_at > 0 && nvalid < a.stop_at) {
    if (gtid == 0) {
      a.info[MO_INFO_ERROR] = MO_ERR_INFEASIBLE;
      a.info[MO_INFO_L] = -1;
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
    for (int rb = gwarp * 4; rb < R; rb += nwarps * 4) {
      const int j = rb + g8;
      bool active = (j < R) && (__ldcg(a.ranks + j) == MO_RANK_UNRANKED);
      int64_t base = active ? (int64_t)a.resume[j] : W;
      bool blocked = false;
      for (;;) {
        const bool scanning = active && !blocked && base < W;
        if (__ballot_sync(MO_FULL, scanning) == 0) break;
        bool hit = false;
        if (scanning) {
          const int64_t idx = base + l8 * 4;
          if (idx < W) {
            uint4 b4 = __ldg(reinterpret_cast<const uint4*>(a.bits + (int64_t)j * W + idx));
            uint4 r4 = __ldcg(reinterpret_cast<const uint4*>(a.ranked + idx));
            hit = ((b4.x & ~r4.x) | (b4.y & ~r4.y) | (b4.z & ~r4.z) | (b4.w & ~r4.w)) != 0u;
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
          a.ranks[j] = k;
          ready_local++;
        }
      }
    }
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
    const int fk = __ldcg(a.front_sizes + k + 1);
    cum += fk;
    const bool done = (cum >= target) || (fk == 0);
    if (done) {
      for (int j = gtid; j < R; j += gthreads)
        if (__ldcg(a.ranks + j) == MO_RANK_UNRANKED) a.ranks[j] = MO_RANK_DROPPED;
      if (gtid == 0) {
        const int64_t sel = cum - fk;
        a.info[MO_INFO_L] = k;
        a.info[MO_INFO_SELECTED] = (int)sel;
        a.info[MO_INFO_K] = a.stop_at > 0 ? (int)(a.stop_at - sel) : fk;
        a.info[MO_INFO_NFRONTS] = k + 1;
        a.info[MO_INFO_FL_SIZE] = fk;
        a.info[MO_INFO_SKIPPED] = (a.stop_at > 0 && sel + fk == a.stop_at) ? 1 : 0;
        a.info[MO_INFO_ERROR] = 0;
      }
      return;
    }
    for (int64_t w = gwarp; w < nwords_used; w += nwarps) {
      const int64_t j = w * 32 + lane;
      const bool in = (j < R) && (__ldcg(a.ranks + j) == k);
      const uint32_t m = __ballot_sync(MO_FULL, in);
      if (lane == 0 && m) a.ranked[w] |= m;
    }
    grid_sync(a.bar);
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
                      cudaStream_t s) {
  if (R <= 0) return MO_ERR_PARAM;
  PeelArgs a{bits, (int)R, words_per_row(R), valid, stop_at, ranks, info, resume, ranked, front_sizes, bar};
  if (cudaMemsetAsync(front_sizes, 0, 2 * sizeof(int), s) != cudaSuccess) return MO_ERR_CUDA;
  if (cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), s) != cudaSuccess) return MO_ERR_CUDA;
  int blocks = peel_grid_blocks();
  int needed = (int)ceil_div(R, (PEEL_THREADS / 32) * 4);
  if (blocks > needed) blocks = needed < 1 ? 1 : needed;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(PEEL_THREADS);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, k_front_peel, a) != cudaSuccess) return MO_ERR_CUDA;
  MO_CHECK_LAUNCH();
  return MO_OK;
}

}  // namespace mo
