// Normalisation (K3), association (K4) and niche selection (K5-K9).
//
// Reference: niche.normalize_objectives SPEC.md:331-339, perpendicular_distance
// _matrix :340-348, associate :349-357, niche_counts :358-366,
// nearest_selection :367-375, build_cache :376-384, batched_random_selection
// :385-393; Alg. 2 PAPER.md:157-191.  Pins: DESIGN.md "Pinned semantics" and
// oracle/manyobj_ref/niche.py (same arithmetic, same tie-breaks).
//
// k_prep      (persistent): running ideal, keyed shuffles of rows and
//             reference points, candidate list (rank <= l), ASF extreme
//             points, FP64 hyperplane solve -> FP32 intercepts.
// k_assoc<M>  (rows x reference-split grid): canonical FP32 key
//             t = ((f0*z0 + f1*z1) + ...) against zhat in shuffled order,
//             running (max t, first position), merged across splits with a
//             64-bit atomicMax of (ord(t), ~position).  D is never stored.
// k_assoc_final: pi = perm_ref[p*], d = sqrt(sum (f - t z)^2).
// k_select    (persistent): nearest selection (64-bit atomicMin of
//             (d, position)), closed-form water-filling of the Alg. 2 loop,
//             the cache table as per-point buckets whose take_j smallest
//             shuffled positions are promoted, and the stable survivor
//             compaction.  (Niche counts are warp-aggregated atomics fused
//             into k_assoc_final.)
#include <cuda_bf16.h>

#include "mo_common.cuh"
#include "mo_grid.cuh"
#include "mo_rng.cuh"
#include "k_niche_args.cuh"
#include "mo_prologue.cuh"

namespace mo {

constexpr int MAXM = 64;
constexpr float ASF_EPS = 1e-6f;
constexpr double DEGENERATE = 1e-10;

// ---------------------------------------------------------------- prep



__device__ __forceinline__ void atomic_min_f(float* addr, float v) {
  if (v >= 0.0f)
    atomicMin(reinterpret_cast<int*>(addr), __float_as_int(v));
  else
    atomicMax(reinterpret_cast<unsigned*>(addr), __float_as_uint(v));
}

// E b = 1 with partial pivoting, FP64, every operation separately rounded
// (library built with -fmad=false).  Mirrors oracle niche.gauss_solve.
// A (m x m, row-major) and rhs are overwritten; rhs returns b.
__device__ void gauss_solve(double* A, double* rhs, int m, int* singular) {
  for (int c = 0; c < m; ++c) {
    int p = c;
    double best = fabs(A[c * m + c]);
    for (int r = c + 1; r < m; ++r)
      if (fabs(A[r * m + c]) > best) {
        best = fabs(A[r * m + c]);
        p = r;
      }
    if (best == 0.0) {
      *singular = 1;
      return;
    }
    if (p != c) {
      for (int q = 0; q < m; ++q) {
        double t = A[c * m + q];
        A[c * m + q] = A[p * m + q];
        A[p * m + q] = t;
      }
      double t = rhs[c];
      rhs[c] = rhs[p];
      rhs[p] = t;
    }
    for (int r = c + 1; r < m; ++r) {
      double f = A[r * m + c] / A[c * m + c];
      for (int q = c; q < m; ++q) A[r * m + q] = A[r * m + q] - f * A[c * m + q];
      rhs[r] = rhs[r] - f * rhs[c];
    }
  }
  for (int c = m - 1; c >= 0; --c) {
    double s = rhs[c];
    for (int q = c + 1; q < m; ++q) s = s - A[c * m + q] * rhs[q];
    rhs[c] = s / A[c * m + c];
  }
  *singular = 0;
}

// gauss_solve with one warp (m <= 32): lane r owns row r.  Same operations on the same elements as
// the one-thread version (pivot = first row with the strictly largest |A[r][c]|; each lane updates its
// own row from the unchanged pivot row), so the solution is bit-identical; only the schedule differs.
// Called by all 32 lanes of one warp; result in rhs, *singular set by lane 0.
__device__ void gauss_solve_warp(double* A, double* rhs, int m, int* singular) {
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < m; ++c) {
    double v = (lane >= c && lane < m) ? fabs(A[lane * m + c]) : -1.0;
    int p = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double vo = __shfl_xor_sync(MO_FULL, v, o);
      const int po = __shfl_xor_sync(MO_FULL, p, o);
      if (vo > v || (vo == v && po < p)) {
        v = vo;
        p = po;
      }
    }
    if (v == 0.0) {
      if (lane == 0) *singular = 1;
      return;
    }
    if (p != c) {
      if (lane < m) {
        const double t = A[c * m + lane];
        A[c * m + lane] = A[p * m + lane];
        A[p * m + lane] = t;
      }
      if (lane == 0) {
        const double t = rhs[c];
        rhs[c] = rhs[p];
        rhs[p] = t;
      }
    }
    __syncwarp();
    if (lane > c && lane < m) {
      const double f = A[lane * m + c] / A[c * m + c];
      for (int q = c; q < m; ++q) A[lane * m + q] = A[lane * m + q] - f * A[c * m + q];
      rhs[lane] = rhs[lane] - f * rhs[c];
    }
    __syncwarp();
  }
  if (lane == 0) {
    for (int c = m - 1; c >= 0; --c) {
      double s = rhs[c];
      for (int q = c + 1; q < m; ++q) s = s - A[c * m + q] * rhs[q];
      rhs[c] = s / A[c * m + c];
    }
    *singular = 0;
  }
  __syncwarp();
}

// gauss_solve with a whole block (wide m, 32 < m <= MO_MAX_M): the same operations on the same elements
// as the one-thread version -- pivot = first row with the strictly largest |A[r][c]|; every multiplier
// f_r = A[r][c] / A[c][c] is taken from the unchanged column before the rows are updated; each element
// A[r][q] - f_r * A[c][q] and rhs[r] - f_r * rhs[c] is rounded once per operation (-fmad=false) -- so
// the solution is bit-identical; back substitution forms the products in parallel and subtracts them
// in the sequential order (q ascending) on one thread.  sF: shared scratch of m doubles.
__device__ void gauss_solve_block(double* A, double* rhs, int m, int* singular, double* sF) {
  __shared__ double sV[32];
  __shared__ int sP[32];
  __shared__ int sPiv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = (blockDim.x + 31) >> 5;
  for (int c = 0; c < m; ++c) {
    double v = -1.0;
    int p = 0x7fffffff;
    for (int r = c + tid; r < m; r += blockDim.x) {
      const double x = fabs(A[(int64_t)r * m + c]);
      if (x > v) {
        v = x;
        p = r;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double vo = __shfl_xor_sync(MO_FULL, v, o);
      const int po = __shfl_xor_sync(MO_FULL, p, o);
      if (vo > v || (vo == v && po < p)) {
        v = vo;
        p = po;
      }
    }
    if (lane == 0) {
      sV[warp] = v;
      sP[warp] = p;
    }
    __syncthreads();
    if (tid == 0) {
      double bv = sV[0];
      int bp = sP[0];
      for (int q = 1; q < nw; ++q)
        if (sV[q] > bv || (sV[q] == bv && sP[q] < bp)) {
          bv = sV[q];
          bp = sP[q];
        }
      sPiv = bv == 0.0 ? -1 : bp;
    }
    __syncthreads();
    const int piv = sPiv;
    if (piv < 0) {
      if (tid == 0) *singular = 1;
      __syncthreads();
      return;
    }
    if (piv != c) {
      for (int q = tid; q < m; q += blockDim.x) {
        const double t = A[(int64_t)c * m + q];
        A[(int64_t)c * m + q] = A[(int64_t)piv * m + q];
        A[(int64_t)piv * m + q] = t;
      }
      if (tid == 0) {
        const double t = rhs[c];
        rhs[c] = rhs[piv];
        rhs[piv] = t;
      }
      __syncthreads();
    }
    const double acc = A[(int64_t)c * m + c];
    for (int r = c + 1 + tid; r < m; r += blockDim.x) sF[r] = A[(int64_t)r * m + c] / acc;
    __syncthreads();
    const int cols = m - c;
    const int64_t cells = (int64_t)(m - c - 1) * cols;
    for (int64_t e = tid; e < cells; e += blockDim.x) {
      const int r = c + 1 + (int)(e / cols), q = c + (int)(e % cols);
      A[(int64_t)r * m + q] = A[(int64_t)r * m + q] - sF[r] * A[(int64_t)c * m + q];
    }
    for (int r = c + 1 + tid; r < m; r += blockDim.x) rhs[r] = rhs[r] - sF[r] * rhs[c];
    __syncthreads();
  }
  for (int c = m - 1; c >= 0; --c) {
    for (int q = c + 1 + tid; q < m; q += blockDim.x) sF[q] = A[(int64_t)c * m + q] * rhs[q];
    __syncthreads();
    if (tid == 0) {
      double s = rhs[c];
      for (int q = c + 1; q < m; ++q) s = s - sF[q];
      rhs[c] = s / A[(int64_t)c * m + c];
    }
    __syncthreads();
  }
  if (tid == 0) *singular = 0;
  __syncthreads();
}

// phase 1 of k_prep for runtime m (wide m > 16): the same keys and column maxima as prep_extremes<M>.
// The ASF of axis ax is max(ft[ax], max_{k != ax} q[k]) (fmaxf: exact, NaN-ignoring, order-free), so
// one pass finds the largest q (first index) and the largest q outside its index and every axis takes
// one of them.  A warp per candidate row (coalesced row reads, the top-2 merged across lanes), the
// column maxima and complemented keys reduced in shared memory (scratch: k_prep's not yet used system
// buffer), one atomic per CTA and axis.
__device__ __forceinline__ void prep_extremes_rt(const PrepArgs& a, int R, int l, bool build_cand, int m,
                                                 double* scratch) {
  const int tid = threadIdx.x, lane = tid & 31, nwb = blockDim.x >> 5;
  uint32_t* sCol = reinterpret_cast<uint32_t*>(scratch);                       // MO_MAX_M
  unsigned long long* sKey = reinterpret_cast<unsigned long long*>(scratch + MO_MAX_M / 2);
  for (int k = tid; k < m; k += blockDim.x) {
    sCol[k] = 0u;
    sKey[k] = 0ull;
  }
  __syncthreads();
  const float QNAN = __int_as_float(0x7fc00000);
  for (int row = blockIdx.x * nwb + (tid >> 5); row < R; row += gridDim.x * nwb) {   // warp-uniform
    const int r = a.ranks[row];
    if (!(r >= 0 && r <= l)) continue;
    if (build_cand && lane == 0) a.cand[atomicAdd(a.ctl, 1)] = row;   // candidate order is immaterial
    const float* f = a.F + (int64_t)row * m;
    const int pp = __ldcg(a.pos_pop + row);
    float t1 = QNAN, t2 = QNAN;   // largest q (first index i1) and the largest q at any other index
    int i1 = 0x7fffffff;
    for (int k = lane; k < m; k += 32) {
      const float q = __fdiv_rn(__fsub_rn(f[k], __ldcg(a.ideal + k)), ASF_EPS);
      if (q > t1 || t1 != t1) {
        if (q == q) {
          t2 = t1;
          t1 = q;
          i1 = k;
        }
      } else {
        t2 = fmaxf(t2, q);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float b1 = __shfl_xor_sync(MO_FULL, t1, o), b2 = __shfl_xor_sync(MO_FULL, t2, o);
      const int bi = __shfl_xor_sync(MO_FULL, i1, o);
      if (b1 != b1) continue;                       // nothing on the other side
      if (t1 != t1 || b1 > t1 || (b1 == t1 && bi < i1)) {
        t2 = t1 != t1 ? b2 : fmaxf(b2, fmaxf(t2, t1));
        t1 = b1;
        i1 = bi;
      } else {
        t2 = fmaxf(t2, fmaxf(b2, b1));
      }
    }
    for (int k = lane; k < m; k += 32) {
      const float ft = __fsub_rn(f[k], __ldcg(a.ideal + k));
      const uint32_t c = f2ord(ft);
      if (c) atomicMax(&sCol[k], c);
      const float sv = fmaxf(ft, k == i1 ? t2 : t1);
      const unsigned long long key = ((unsigned long long)f2ord(sv) << 32) | (uint32_t)pp;
      atomicMax(&sKey[k], ~key);
    }
  }
  __syncthreads();
  for (int k = tid; k < m; k += blockDim.x) {
    if (sCol[k]) atomicMax(&a.colmax[k], sCol[k]);
    if (sKey[k]) atomicMax(&a.ext_key[k], sKey[k]);
  }
}

// phase 1 of k_prep for m = M (register arrays): ASF extreme-point keys and column maxima of the
// translated candidate rows (rank in [0, l]).  Each thread keeps its best key per axis and its column
// maxima across its rows; warp, then block reductions (shared memory) leave one atomic per CTA per
// axis / column -- per-warp atomics on these 2M addresses serialised at C3 (6k warps x 2M atomics).
// The keys are stored complemented (atomicMax of ~key: 0 is neutral, so a zeroed workspace needs no
// reset node; phase 2 restores 0 after reading).  build_cand: also append the candidates to cand
// (engine path: phase 0's list pass and its grid barrier are folded in here), one atomic per CTA and
// row chunk.
template <int M>
__device__ __forceinline__ void prep_extremes(const PrepArgs& a, int R, int l, int gthreads, bool build_cand,
                                              double* scratch) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  // scratch: k_prep's (not yet used) system buffer -- 8 warps x M keys, 8 x M column maxima, counters
  unsigned long long (*sKey)[M] = reinterpret_cast<unsigned long long (*)[M]>(scratch);
  uint32_t (*sCol)[M] = reinterpret_cast<uint32_t (*)[M]>(scratch + 8 * M);
  int* sCnt = reinterpret_cast<int*>(scratch + 16 * M);
  int& sBase = sCnt[8];
  float idl[M];
#pragma unroll
  for (int k = 0; k < M; ++k) idl[k] = __ldcg(a.ideal + k);
  unsigned long long best[M];
  uint32_t cmax[M];
#pragma unroll
  for (int k = 0; k < M; ++k) {
    best[k] = ~0ull;
    cmax[k] = 0u;
  }
  for (int base = blockIdx.x * blockDim.x; base < R; base += gthreads) {   // uniform trip count
    const int row = base + tid;
    const bool act = row < R && a.ranks[row] >= 0 && a.ranks[row] <= l;
    if (build_cand) {   // candidate order is immaterial: one atomic per CTA and chunk
      const unsigned bal = __ballot_sync(MO_FULL, act);
      if (lane == 0) sCnt[warp] = __popc(bal);
      __syncthreads();
      if (tid == 0) {
        int tot = 0;
        for (int w = 0; w < nw; ++w) {
          const int c = sCnt[w];
          sCnt[w] = tot;
          tot += c;
        }
        sBase = tot ? atomicAdd(a.ctl, tot) : 0;
      }
      __syncthreads();
      if (act) a.cand[sBase + sCnt[warp] + __popc(bal & ((1u << lane) - 1u))] = row;
      __syncthreads();   // sCnt / sBase are rewritten by the next chunk
    }
    if (act) {
      const int pp = __ldcg(a.pos_pop + row);
      float ft[M], q[M];
#pragma unroll
      for (int k = 0; k < M; ++k) {
        ft[k] = __fsub_rn(a.F[(int64_t)row * M + k], idl[k]);
        q[k] = __fdiv_rn(ft[k], ASF_EPS);
        cmax[k] = max(cmax[k], f2ord(ft[k]));
      }
#pragma unroll
      for (int ax = 0; ax < M; ++ax) {
        float s = ft[ax];  // w_ax,ax = 1: f / 1 is exact
#pragma unroll
        for (int k = 0; k < M; ++k)
          if (k != ax) s = fmaxf(s, q[k]);
        const unsigned long long key = ((unsigned long long)f2ord(s) << 32) | (uint32_t)pp;
        best[ax] = key < best[ax] ? key : best[ax];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < M; ++k) {
    const unsigned long long kv = warp_min_u64(best[k]);
    const uint32_t cv = warp_max_u32(cmax[k]);
    if (lane == 0) {
      sKey[warp][k] = kv;
      sCol[warp][k] = cv;
    }
  }
  __syncthreads();
  if (tid < M) {
    unsigned long long kv = ~0ull;
    uint32_t cv = 0u;
    for (int w = 0; w < nw; ++w) {
      kv = sKey[w][tid] < kv ? sKey[w][tid] : kv;
      cv = max(cv, sCol[w][tid]);
    }
    if (kv != ~0ull) atomicMax(&a.ext_key[tid], ~kv);
    if (cv) atomicMax(&a.colmax[tid], cv);
  }
}

__global__ void __launch_bounds__(256) k_prep(PrepArgs a) {
  pdl_wait();
  __shared__ uint32_t sKp[MAX_SHUFFLE_ROUNDS], sSp[MAX_SHUFFLE_ROUNDS], sKr[MAX_SHUFFLE_ROUNDS],
      sSr[MAX_SHUFFLE_ROUNDS];
  __shared__ int sRp, sRr;
  __shared__ float sMin0[MAXM];
  __shared__ double sA[MAXM * MAXM];
  __shared__ double sRhs0[MAXM];
  const int tid = threadIdx.x, lane = tid & 31;
  const int gtid = blockIdx.x * blockDim.x + tid, gthreads = gridDim.x * blockDim.x;
  const int R = a.R, m = a.m, w = a.w;
  // m > MAXM (wide): the system lives in global memory (a.solveA) and sA's shared bytes hold the
  // per-objective vectors instead (MO_MAX_M doubles each)
  static_assert(MAXM * MAXM >= 3 * MO_MAX_M, "wide-m scratch must fit in sA");
  const bool big = m > MAXM;
  float* sMin = big ? reinterpret_cast<float*>(sA) : sMin0;
  double* sRhs = big ? sA : sRhs0;
  if (__ldcg(a.info + MO_INFO_ERROR) != 0) return;
  const int l = __ldcg(a.info + MO_INFO_L);
  const bool skipped = __ldcg(a.info + MO_INFO_SKIPPED) != 0;
  trace_mark(a.trace, 16);

  // ---- phase 0: running ideal over all R rows (A-4), shuffles, candidate list
  for (int k = tid; k < m; k += blockDim.x) sMin[k] = __int_as_float(0x7f800000);
  const uint32_t gen = a.gen_ptr ? __ldcg(a.gen_ptr) : a.gen;
  __syncthreads();
  if (a.mode == PREP_FULL && !a.ideal_done) {
    // column minima: per column, strided rows, warp reduction, one smem atomic per warp
    for (int k = 0; k < m; ++k) {
      float v = __int_as_float(0x7f800000);
      for (int i = gtid; i < R; i += gthreads) v = fminf(v, a.F[(int64_t)i * m + k]);
      for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(MO_FULL, v, o));
      if (lane == 0) atomic_min_f(&sMin[k], v);
    }
    __syncthreads();
    for (int k = tid; k < m; k += blockDim.x) atomic_min_f(&a.ideal[k], sMin[k]);
  }
  if (skipped) return;
  if (!a.pro_done) {
    if (a.mode == PREP_PERMS) {   // op-level niche_select: shuffles + niche state only
      PrepArgs b = a;
      b.akey = nullptr;
      gen_prologue(b, gen, gtid, gthreads, sKp, sSp, &sRp, sKr, sSr, &sRr);
      return;
    }
    gen_prologue(a, gen, gtid, gthreads, sKp, sSp, &sRp, sKr, sSr, &sRr);
  }
  // engine path (ideal and positions final at launch): the candidate list is built inside phase 1
  const bool fused = a.mode == PREP_FULL && a.ideal_done && a.pro_done;
  if (!fused) {
    for (int base = blockIdx.x * blockDim.x; base < R; base += gthreads) {   // uniform trip count
      const int i = base + tid;
      const bool c = i < R && a.ranks[i] >= 0 && a.ranks[i] <= l;
      const int slot = warp_alloc(a.ctl, c ? 1 : 0);          // candidate order is immaterial
      if (c) a.cand[slot] = i;
    }
    if (a.mode != PREP_FULL) return;
    for (int k = gtid; k < m; k += gthreads) {
      a.ext_key[k] = 0ull;
      a.colmax[k] = 0u;
    }
    grid_sync(a.bar);
  }
  trace_mark(a.trace, 17);

  // ---- phase 1: ASF extreme points + column maxima of translated candidates
  switch (m) {
#define MO_PX_CASE(MM) \
  case MM: prep_extremes<MM>(a, R, l, gthreads, fused, sA); break;
    MO_PX_CASE(1) MO_PX_CASE(2) MO_PX_CASE(3) MO_PX_CASE(4) MO_PX_CASE(5) MO_PX_CASE(6) MO_PX_CASE(7)
    MO_PX_CASE(8) MO_PX_CASE(9) MO_PX_CASE(10) MO_PX_CASE(11) MO_PX_CASE(12) MO_PX_CASE(13) MO_PX_CASE(14)
    MO_PX_CASE(15) MO_PX_CASE(16)
#undef MO_PX_CASE
    default: prep_extremes_rt(a, R, l, fused, m, sA);   // wide m (launch_prep: m <= MO_MAX_M)
  }
  if (big) {
    // m > 64: the m x m system lives in global memory; every block loads a slice of it (one more grid
    // barrier) instead of the last block alone -- a single CTA's load -> store round trips over 262K
    // values took ~0.3 ms at m = 512
    grid_sync(a.bar);
    int* sRowX = reinterpret_cast<int*>(sA + 3 * MO_MAX_M);   // after rhs / fallbacks / solve scratch
    for (int r = tid; r < m; r += blockDim.x) {
      const unsigned long long ck = __ldcg(a.ext_key + r);   // complemented key; 0 = no candidate
      sRowX[r] = ck ? __ldcg(a.perm_pop + (uint32_t)(~ck & 0xffffffffull)) : 0;
    }
    __syncthreads();
    for (int e = gtid; e < m * m; e += gthreads) {
      const int r = e / m, c = e - r * m;
      a.solveA[e] = (double)__fsub_rn(__ldg(a.F + (int64_t)sRowX[r] * m + c), __ldcg(a.ideal + c));
    }
  }
  // phase 2 runs in the last block to finish phase 1
  if (!grid_last(a.bar)) return;
  trace_mark_any(a.trace, 18);
  const int ncand = __ldcg(a.ctl);

  // ---- phase 2: hyperplane solve (one warp) on the extreme rows loaded by the block,
  //      per-component fallbacks
  {
    __shared__ double sFb0[MAXM], sGF0[MAXM];
    double* sFb = big ? sA + MO_MAX_M : sFb0;
    double* A = big ? a.solveA : sA;
    if (!big) {   // (m > 64: loaded by every block before grid_last)
      for (int e = tid; e < m * m; e += blockDim.x) {
        const int r = e / m, c = e - r * m;
        const unsigned long long ck = __ldcg(a.ext_key + r);   // complemented key; 0 = no candidate
        const int row = ck ? __ldcg(a.perm_pop + (uint32_t)(~ck & 0xffffffffull)) : 0;
        A[e] = (double)__fsub_rn(a.F[(int64_t)row * m + c], __ldcg(a.ideal + c));
      }
    }
    for (int k = tid; k < m; k += blockDim.x) {
      const double mx = (double)ord2f(__ldcg(a.colmax + k));
      sFb[k] = mx > DEGENERATE ? mx : 1.0;
      sRhs[k] = 1.0;
    }
    __syncthreads();
    trace_mark_any(a.trace, 20);
    for (int k = tid; k < m; k += blockDim.x) {   // every reader of this generation's keys is done:
      a.ext_key[k] = 0ull;                        // neutral values for the next launch
      a.colmax[k] = 0u;
    }
    __shared__ int sSing;
    if (tid == 0) sSing = ncand == 0 ? 1 : 0;
    __syncthreads();
    if (ncand != 0) {
      if (m <= 32) {
        if (tid < 32) gauss_solve_warp(A, sRhs, m, &sSing);
      } else {
        // multipliers: sGF0 when the system is in shared memory (m <= 64), else sA after sRhs / sFb
        gauss_solve_block(A, sRhs, m, &sSing, big ? sA + 2 * MO_MAX_M : sGF0);
      }
    }
    __syncthreads();
    trace_mark_any(a.trace, 21);
    if (tid < 32) {   // one lane per component (m <= 32 here; larger m loops), same arithmetic per k
      bool fin = true;
      for (int k = tid; k < m; k += 32) fin = fin && isfinite(sRhs[k]);
      const bool bad = sSing != 0 || !__all_sync(MO_FULL, fin);
      for (int k = tid; k < m; k += 32) {
        double ak;
        if (bad) {
          ak = sFb[k];
        } else {
          ak = 1.0 / sRhs[k];
          if (!(isfinite(ak) && ak > DEGENERATE)) ak = sFb[k];
        }
        a.icpt[k] = ak;
        a.a32[k] = __double2float_rn(ak);
        if (a.icpt_out) a.icpt_out[k] = ak;
      }
      if (tid == 0) a.info[MO_INFO_SINGULAR] = bad ? 1 : 0;
    }
  }
  trace_mark_any(a.trace, 19);
}

// ---------------------------------------------------------- association

constexpr int ASSOC_THREADS = 256;
// candidate rows per thread (registers) and rows per item
template <int M>
struct AssocShape {
  static constexpr int RB = 4;   // (2 rows at m = 10: fewer registers but slower, C3 10.0 -> 10.6 ms)
  static constexpr int ROWS = ASSOC_THREADS * RB;
};
constexpr int ASSOC_PTILE = 256;                   // reference points staged per smem tile

template <int M>
__device__ __forceinline__ float canon_dot(const float* f, const float* z) {
  float t = __fmul_rn(f[0], z[0]);
#pragma unroll
  for (int k = 1; k < M; ++k) t = __fadd_rn(t, __fmul_rn(f[k], z[k]));
  return t;
}

// rows x reference-split grid.  Thread: AssocShape<M>::RB candidate rows in registers;
// the block streams its reference range through shared memory (shuffled
// order) two points per step; strict '>' keeps the first maximum, and the
// splits merge through a 64-bit atomicMax of (ord(t), ~position).
template <int M>
__device__ __forceinline__ void assoc_item(const AssocArgs& a, int ncand, int rbase, int p0, int p1, float* sz) {
  constexpr int MP = (M + 3) & ~3;
  if (p0 >= p1) return;
  const int tid = threadIdx.x;
  float fn[AssocShape<M>::RB][M];
  int rows[AssocShape<M>::RB];
#pragma unroll
  for (int r = 0; r < AssocShape<M>::RB; ++r) {
    const int c = rbase + r * ASSOC_THREADS + tid;
    rows[r] = c < ncand ? __ldcg(a.cand + c) : -1;
    const int row = rows[r] < 0 ? 0 : rows[r];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      float v = a.F[(int64_t)row * M + k];
      if (a.ideal) v = __fsub_rn(v, a.ideal[k]);
      if (a.a32) v = __fdiv_rn(v, a.a32[k]);
      fn[r][k] = v;
    }
  }
  float best[AssocShape<M>::RB];
  int bp[AssocShape<M>::RB];
#pragma unroll
  for (int r = 0; r < AssocShape<M>::RB; ++r) {
    best[r] = -__int_as_float(0x7f800000);
    bp[r] = p0;
  }
  for (int t0 = p0; t0 < p1; t0 += ASSOC_PTILE) {
    const int tn = min(ASSOC_PTILE, p1 - t0);
    __syncthreads();
    for (int e = tid; e < ASSOC_PTILE * MP; e += ASSOC_THREADS) {
      const int p = e / MP, k = e - p * MP;
      sz[e] = (k < M && p < tn) ? a.zs[(int64_t)(t0 + p) * M + k] : -__int_as_float(0x7f800000);
    }
    __syncthreads();
    // pairs of reference points; a padded point (-inf direction) never wins a strict '>'
    for (int p = 0; p < tn; p += 2) {
      float z0[M], z1[M];
#pragma unroll
      for (int k = 0; k < M; ++k) {
        z0[k] = sz[p * MP + k];
        z1[k] = sz[(p + 1) * MP + k];
      }
#pragma unroll
      for (int r = 0; r < AssocShape<M>::RB; ++r) {
        const float ta = canon_dot<M>(fn[r], z0);
        const float tb = canon_dot<M>(fn[r], z1);
        if (ta > best[r]) {
          best[r] = ta;
          bp[r] = t0 + p;
        }
        if (tb > best[r]) {
          best[r] = tb;
          bp[r] = t0 + p + 1;
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < AssocShape<M>::RB; ++r) {
    if (rows[r] >= 0) {
      const unsigned long long key = ((unsigned long long)f2ord(best[r]) << 32) | (uint32_t)(0xffffffffu - (uint32_t)bp[r]);
      atomicMax(&a.akey[rows[r]], key);
    }
  }
}

template <int M>
__global__ void __launch_bounds__(ASSOC_THREADS) k_assoc(AssocArgs a) {
  pdl_wait();
  constexpr int MP = (M + 3) & ~3;
  __shared__ __align__(16) float sz[ASSOC_PTILE * MP];
  if (__ldcg(a.info + MO_INFO_ERROR) != 0) return;
  if (__ldcg(a.info + MO_INFO_SKIPPED) != 0) return;
  const int ncand = __ldcg(a.ctl);
  // persistent schedule sized on the device from the real candidate count:
  // (row block, reference split) items spread over exactly gridDim.x blocks
  constexpr int ROWS = AssocShape<M>::ROWS;
  const int nrb = (ncand + ROWS - 1) / ROWS;
  if (nrb == 0) return;
  const int wr = a.zend - a.zbeg;
  if (wr <= 0) return;
  // ~4 items per CTA so the last wave is short (items are long: 1024 rows x a slice of the points)
  int splits = (4 * (int)gridDim.x + nrb - 1) / nrb;
  const int maxsplit = (wr + 63) / 64;
  splits = splits < 1 ? 1 : (splits > maxsplit ? maxsplit : splits);
  const int psplit = (wr + splits - 1) / splits;
  const int items = nrb * splits;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int p0 = a.zbeg + (item % splits) * psplit;
    assoc_item<M>(a, ncand, (item / splits) * ROWS, p0, min(a.zend, p0 + psplit), sz);
  }
}


// Wide m (16 < m <= MO_MAX_M): the same canonical keys, tie rule and atomicMax merge as k_assoc with a
// runtime objective count.  Item = (16 candidate rows, a split of the reference positions); the rows'
// normalised objectives sit in shared memory (read as broadcasts), each thread walks the split's points
// p = p0 + tid, p0 + tid + 256, ... (ascending, strict '>': its first maximum) reading the objective-major
// directions zsT[k * w + p] (coalesced), 16 running keys in registers.
constexpr int ASSOCW_ROWS = 16;

__global__ void __launch_bounds__(ASSOC_THREADS) k_assoc_wide(AssocArgs a, int m) {
  pdl_wait();
  extern __shared__ float sFw[];   // ASSOCW_ROWS x m
  __shared__ int sRow[ASSOCW_ROWS];
  if (__ldcg(a.info + MO_INFO_ERROR) != 0) return;
  if (__ldcg(a.info + MO_INFO_SKIPPED) != 0) return;
  const int ncand = __ldcg(a.ctl);
  const int nrt = (ncand + ASSOCW_ROWS - 1) / ASSOCW_ROWS;
  const int wr = a.zend - a.zbeg;
  if (nrt == 0 || wr <= 0) return;
  int splits = (4 * (int)gridDim.x + nrt - 1) / nrt;
  const int maxsplit = (wr + ASSOC_THREADS - 1) / ASSOC_THREADS;
  splits = splits < 1 ? 1 : (splits > maxsplit ? maxsplit : splits);
  const int psplit = (wr + splits - 1) / splits;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int item = blockIdx.x; item < nrt * splits; item += gridDim.x) {
    const int rbase = (item / splits) * ASSOCW_ROWS;
    const int p0 = a.zbeg + (item % splits) * psplit, p1 = min(a.zend, p0 + psplit);
    __syncthreads();   // previous item done with sFw / sRow
    if (tid < ASSOCW_ROWS) sRow[tid] = rbase + tid < ncand ? __ldcg(a.cand + rbase + tid) : -1;
    for (int e = tid; e < ASSOCW_ROWS * m; e += ASSOC_THREADS) {
      const int r = e / m, k = e - r * m;
      const int c = rbase + r;
      float v = 0.0f;
      if (c < ncand) {
        const int row = __ldcg(a.cand + c);
        v = a.F[(int64_t)row * m + k];
        if (a.ideal) v = __fsub_rn(v, a.ideal[k]);
        if (a.a32) v = __fdiv_rn(v, a.a32[k]);
      }
      sFw[e] = v;
    }
    __syncthreads();
    float best[ASSOCW_ROWS];
    int bp[ASSOCW_ROWS];
#pragma unroll
    for (int r = 0; r < ASSOCW_ROWS; ++r) {
      best[r] = -__int_as_float(0x7f800000);
      bp[r] = p0;
    }
    for (int p = p0 + tid; p < p1; p += ASSOC_THREADS) {
      float t[ASSOCW_ROWS];
      {
        const float z = __ldg(a.zsT + p);
#pragma unroll
        for (int r = 0; r < ASSOCW_ROWS; ++r) t[r] = __fmul_rn(sFw[r * m], z);
      }
      for (int k = 1; k < m; ++k) {
        const float z = __ldg(a.zsT + (int64_t)k * a.w + p);
#pragma unroll
        for (int r = 0; r < ASSOCW_ROWS; ++r) t[r] = __fadd_rn(t[r], __fmul_rn(sFw[r * m + k], z));
      }
#pragma unroll
      for (int r = 0; r < ASSOCW_ROWS; ++r)
        if (t[r] > best[r]) {
          best[r] = t[r];
          bp[r] = p;
        }
    }
#pragma unroll
    for (int r = 0; r < ASSOCW_ROWS; ++r) {
      unsigned long long key = ((unsigned long long)f2ord(best[r]) << 32) | (uint32_t)(0xffffffffu - (uint32_t)bp[r]);
      key = warp_max_u64(key);
      if (lane == 0 && sRow[r] >= 0) atomicMax(&a.akey[sRow[r]], key);
    }
  }
}

// ------------------------------------------------- lattice-pruned association
//
// Single-layer Das-Dennis sets (z = k/H, k integer, sum k = H) at m <= 5: the
// direction with the largest key t = f.zhat lies near the simplex projection
// u = f / sum(f).  A group of LPR lanes evaluates the canonical key (same
// arithmetic and tie-break as assoc_item) on the lattice points with
// |k_i - u_i H| < r for i < m-1, reading the directions from a static copy
// in lattice order (zl) and their shuffled positions from lat_pos (scattered
// by k_prep every generation), so no load depends on another.  The winner is
// then certified: every point outside the box has ||z - u|| >= r/H, and the
// distance from u to the line through z is >= ||z - u|| / (sqrt(m) ||z||)
// (the line crosses the simplex plane at angle acos(1 / (sqrt(m) ||z||))),
// so sin(angle) >= (r/H) / (sqrt(m) ||u||) with ||z|| <= 1; its FP32 key is
// then <= ||f|| cos(angle) (1 + (m + 2) 2^-24) -- every term is nonnegative,
// so the m roundings of products / sums and the FP32 rounding of zhat move a
// key by at most (m + 1) 2^-24 relative.  A winner above that bound is the
// global argmax, ties included; rows that fail (or f = 0) go to a fallback
// list for the full-scan k_assoc.  Exact: the result equals the full scan
// bit for bit; the certificate only decides where it is computed.
template <int M, int LPR>
__global__ void __launch_bounds__(256) k_assoc_lattice(AssocArgs a) {
  pdl_wait();
  if (__ldcg(a.info + MO_INFO_ERROR) != 0) return;
  if (__ldcg(a.info + MO_INFO_SKIPPED) != 0) return;
  const int ncand = __ldcg(a.ctl);
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = gt / LPR, sub = gt % LPR;
  if ((gt & ~31) / LPR >= ncand) return;       // whole warp idle (no lane of it has a row)
  const bool live = c < ncand;                   // idle groups still join the warp shuffles
  const int row = live ? __ldcg(a.cand + c) : __ldcg(a.cand);
  const int H = a.lat_H, r = a.lat_r;
  float fn[M];
  double s = 0.0, nn = 0.0;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    float v = a.F[(int64_t)row * M + k];
    if (a.ideal) v = __fsub_rn(v, a.ideal[k]);
    if (a.a32) v = __fdiv_rn(v, a.a32[k]);
    fn[k] = v;
    s += (double)v;
    nn += (double)v * (double)v;
  }
  bool ok = live && s > 0.0 && isfinite(s);
#pragma unroll
  for (int k = 0; k < M; ++k) ok = ok && fn[k] >= 0.0f;
  // rows the box cannot serve (f = 0, non-finite) go straight to the fallback list
  if (live && !ok && sub == 0) {
    a.fb_cand[atomicAdd(a.fb_ctl, 1)] = row;
    atomicAdd(const_cast<int*>(a.info) + MO_INFO_ASSOC_FALLBACK, 1);
  }
  bool done = !ok;   // group-uniform
  // per-row FP64 constants of the box and the certificate, hoisted out of the radius loop: x_k = f_k * H/s;
  // sin >= (r/H) / (sqrt(m) ||u||) = r * s / (H sqrt(m) ||f||) with u = f/s (rounding here is ~1e-16
  // relative, far inside the 1e-6 radius margin and the 2^-24 key slack of the bound)
  const double hs = ok ? (double)H / s : 0.0;
  const double sn = sqrt(nn);
  const double c_se = ok ? s / ((double)H * sqrt((double)M) * sn) : 0.0;
  // radius r, then r+1 for the rows whose certificate failed; the rare rest goes to the sliced full scan
  // (a (2r+4)^(m-1) box walked by one group is a latency-bound straggler that holds the whole grid) --
  // unless the reference set is so large that a full-scan row costs more than 64 such boxes, where the
  // third radius r+2 is tried in the group first
  int box3 = 1;
#pragma unroll
  for (int k = 0; k < M - 1; ++k) box3 *= 2 * (r + 2);
  const int tries = (int64_t)box3 * 64 < (int64_t)a.w ? 3 : 2;
  for (int it = 0; it < tries; ++it) {
    if (__all_sync(MO_FULL, done)) break;
    const int rr = r + it;
    float best = -__int_as_float(0x7f800000);
    int bp = 0x7fffffff;
    // the box (lo, extent per coordinate) is computed once per group, by its leader, in FP64, and broadcast
    int lo[M], ext[M];
    float inv[M];
    int total = 0;
    if (sub == 0 && !done) {
      total = 1;
#pragma unroll
      for (int k = 0; k < M - 1; ++k) {
        const double x = (double)fn[k] * hs;
        lo[k] = max(0, (int)floor(x - (double)rr) + 1);
        const int hi = min(H, (int)ceil(x + (double)rr) - 1);
        ext[k] = max(0, hi - lo[k] + 1);
        total *= ext[k];
      }
    }
    total = __shfl_sync(MO_FULL, total, 0, LPR);
#pragma unroll
    for (int k = 0; k < M - 1; ++k) {
      lo[k] = __shfl_sync(MO_FULL, lo[k], 0, LPR);
      ext[k] = __shfl_sync(MO_FULL, ext[k], 0, LPR);
      inv[k] = ext[k] > 0 ? 1.0f / (float)ext[k] : 0.0f;
    }
#pragma unroll 2
    for (int q = sub; q < total; q += LPR) {
      int rem = q, rest, idx = 0;
      int kv[M];  // mixed-radix decode of the box index, k_{m-2} fastest; (rem + .5) / ext is exact in
                  // FP32 for these small operands, so no integer division
#pragma unroll
      for (int k = M - 2; k >= 0; --k) {
        const int qk = (int)(((float)rem + 0.5f) * inv[k]);
        kv[k] = lo[k] + (rem - qk * ext[k]);
        rem = qk;
      }
      rest = H;
#pragma unroll
      for (int k = 0; k < M - 1; ++k) {
        rest -= kv[k];
        idx = idx * (H + 1) + kv[k];
      }
      if (rest < 0) continue;
      const int p = __ldg(a.lat_pos + idx);
      const float t = canon_dot<M>(fn, a.lat_z + (int64_t)idx * M);   // (lat_pos -> zs measured slower)
      if (t > best || (t == best && p < bp)) {
        best = t;
        bp = p;
      }
    }
    // group reduction: max key, lowest position on ties
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) {
      const float tb = __shfl_xor_sync(MO_FULL, best, o);
      const int pb = __shfl_xor_sync(MO_FULL, bp, o);
      if (tb > best || (tb == best && pb < bp)) {
        best = tb;
        bp = pb;
      }
    }
    int cert = 0;
    if (sub == 0 && !done) {
      double se = ((double)rr - 1e-6) * c_se;
      se = se < 1.0 ? se : 1.0;
      const double bound = sn * sqrt(1.0 - se * se) * (1.0 + (M + 2) * 5.9604644775390625e-8);
      cert = bp != 0x7fffffff && (double)best > bound;
      if (cert)
        a.akey[row] = ((unsigned long long)f2ord(best) << 32) | (uint32_t)(0xffffffffu - (uint32_t)bp);
    }
    const int cert_g = __shfl_sync(MO_FULL, cert, 0, LPR);   // every lane joins (no short circuit)
    done = done || cert_g != 0;
  }
  if (!done && sub == 0) {
    a.fb_cand[atomicAdd(a.fb_ctl, 1)] = row;
    atomicAdd(const_cast<int*>(a.info) + MO_INFO_ASSOC_FALLBACK, 1);
  }
}

// Full scan for the few rows the lattice certificate rejected: items = (row, slice of the shard's
// reference range sized so the items cover the grid's warps, >= 32 points); a warp per item, lanes stride the slice in shuffled order with the
// canonical key and a strict '>' (first maximum per lane), a warp reduction (max key, lowest position),
// and an atomicMax merge of the slices into akey -- many short independent scans instead of a few long
// latency-bound ones.
template <int M>
__global__ void __launch_bounds__(256) k_assoc_fallback(AssocArgs a) {
  pdl_wait();
  if (__ldcg(a.info + MO_INFO_ERROR) != 0) return;
  if (__ldcg(a.info + MO_INFO_SKIPPED) != 0) return;
  const int nfb = __ldcg(a.fb_ctl);
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  // slice the reference range so that the items cover the grid's warps (a handful of rows -> one
  // 32-point slice per warp; many rows -> longer slices); at least 32 points per slice
  const int range = a.zend - a.zbeg;
  const int per_row = max(1, nwarps / max(nfb, 1));
  const int SLICE = max(32, ((range + per_row - 1) / per_row + 31) & ~31);
  const int nslice = (range + SLICE - 1) / SLICE;
  for (int it = warp; it < nfb * nslice; it += nwarps) {
    const int c = it / nslice, sl = it - c * nslice;
    const int row = __ldcg(a.fb_cand + c);
    const int p0 = a.zbeg + sl * SLICE, p1 = min(a.zend, p0 + SLICE);
    float fn[M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      float v = a.F[(int64_t)row * M + k];
      if (a.ideal) v = __fsub_rn(v, a.ideal[k]);
      if (a.a32) v = __fdiv_rn(v, a.a32[k]);
      fn[k] = v;
    }
    float best = -__int_as_float(0x7f800000);
    int bp = 0x7fffffff;
#pragma unroll 4
    for (int p = p0 + lane; p < p1; p += 32) {
      const float t = canon_dot<M>(fn, a.zs + (int64_t)p * M);
      if (t > best) {
        best = t;
        bp = p;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float tb = __shfl_xor_sync(MO_FULL, best, o);
      const int pb = __shfl_xor_sync(MO_FULL, bp, o);
      if (tb > best || (tb == best && pb < bp)) {
        best = tb;
        bp = pb;
      }
    }
    if (lane == 0 && bp != 0x7fffffff)
      atomicMax(&a.akey[row], ((unsigned long long)f2ord(best) << 32) | (uint32_t)(0xffffffffu - (uint32_t)bp));
  }
}

// ------------------------------------------- association: tensor-core filter + exact FP32 keys
//
// The full-scan association (no lattice) is a GEMM, Fn (rows x m) x Zhat^T (m x w), followed by a row
// argmax of the canonical FP32 key.  k_assoc_hmma evaluates the dots on the tensor cores as a FILTER and
// the canonical key only where it can matter:
//   * the m <= 16 coordinates are padded to K = 16 and split into bf16 hi + lo parts (x = hi + lo +
//     O(2^-17 |x|)); three m16n8k16 bf16 MMAs with FP32 accumulation (hi.hi + hi.lo + lo.hi) give
//     t~ with |t~ - t| <= 2^-13 sum_k |f_k z_k| <= 2^-13 ||f|| for the canonical key t (products of
//     bf16 are exact in FP32; <= 48 accumulations; the dropped lo.lo and residual terms) -- the filter
//     uses eps = 2^-12 ||f||, twice that;
//   * a reference is a candidate when t~ >= (running max of t~ seen by this lane) - 2 eps; the exact
//     argmax j* and every exact tie satisfy t~ >= T* - eps >= max t~ - 2 eps, so each is a candidate
//     when it is reached; candidates get the canonical key (ord(t) << 32 | ~position), the same
//     atomicMax merge as the FP32 scan -> bit-identical association;
//   * rows with ||f|| = 0 or non-finite values (every reference ties / no order) go to the sliced
//     full scan (fb_cand), like the lattice rejects.
// Layout: a warp owns 16 candidate rows (A fragments in registers for the whole sweep) and walks a chunk
// of 8-reference tiles; the 8 warps of a CTA take 8 row tiles of the SAME chunk so the fragment stream
// (544 B per tile: hi, lo, reference indices) is read once per CTA from L2 and hit in L1 by the other warps.  mma.sync
// (HMMA) rather than tcgen05: K = 16 is a single MMA step and the work is the per-element filter and
// running max on the accumulators, which needs them in registers anyway.
constexpr int HMMA_WARPS = 8;

__device__ __forceinline__ uint32_t bf16x2_bits(float lo_k, float hi_k) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo_k, hi_k);
  return *reinterpret_cast<const uint32_t*>(&v);
}

__device__ __forceinline__ void split_bf16(float x, float& h, float& l) {
  h = __bfloat162float(__float2bfloat16_rn(x));
  l = __fsub_rn(x, h);
}

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// fragments of tile t (refs 8t..8t+7, static order): lane L holds ref n = L / 4 and k pairs (2(L%4), +1),
// (2(L%4) + 8, +9): [t][0..31] hi parts, [t][32..63] lo parts
constexpr int HMMA_TS = 68;   // uint2 per packed tile: 32 hi + 32 lo fragments, then 8 int32 reference indices

__global__ void k_pack_refs(const float* __restrict__ zhat, int64_t w, int m, const int32_t* __restrict__ order,
                            uint2* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t ntiles = (w + 7) / 8;
  if (e >= ntiles * 32) return;
  const int64_t t = e >> 5;
  const int lane = (int)(e & 31), tg = lane & 3, n = lane >> 2;
  const int64_t q = t * 8 + n;                       // packed column
  const int64_t j = q < w ? (order ? (int64_t)order[q] : q) : -1;
  float v[4], h[4], l[4];
  const int ks[4] = {2 * tg, 2 * tg + 1, 2 * tg + 8, 2 * tg + 9};
  for (int c = 0; c < 4; ++c) {
    v[c] = (j >= 0 && ks[c] < m) ? zhat[j * m + ks[c]] : 0.0f;
    split_bf16(v[c], h[c], l[c]);
  }
  out[t * HMMA_TS + lane] = make_uint2(bf16x2_bits(h[0], h[1]), bf16x2_bits(h[2], h[3]));
  out[t * HMMA_TS + 32 + lane] = make_uint2(bf16x2_bits(l[0], l[1]), bf16x2_bits(l[2], l[3]));
  if (tg == 0) reinterpret_cast<int32_t*>(out + t * HMMA_TS + 64)[n] = (int32_t)j;
}

template <int M>
__device__ __forceinline__ void hmma_load_fn(const AssocArgs& a, int row, float (&fn)[M]) {
#pragma unroll
  for (int k = 0; k < M; ++k) {
    float v = a.F[(int64_t)row * M + k];
    if (a.ideal) v = __fsub_rn(v, a.ideal[k]);
    if (a.a32) v = __fdiv_rn(v, a.a32[k]);
    fn[k] = v;
  }
}

// exact canonical keys of the candidates among the step's filter values of one row (packed columns
// 2tg, 2tg + 1 of tiles t .. t+U-1; the reference index of a column is stored after the tile's fragments);
// fn: the row's normalised objectives (shared memory, written once per item)
template <int M, int U>
__device__ __forceinline__ void hmma_exact(const AssocArgs& a, const float* fn, const float (&v)[U][2], int t, int tg,
                                           float thr, unsigned long long& best) {
  uint32_t mask = 0;
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int e = 0; e < 2; ++e) mask |= (v[u][e] >= thr ? 1u : 0u) << (2 * u + e);
  while (mask) {
    const int b = __ffs(mask) - 1;
    mask &= mask - 1;
    const int j = __ldg(reinterpret_cast<const int*>(a.zfrag + (int64_t)(t + (b >> 1)) * HMMA_TS + 64) +
                        2 * tg + (b & 1));
    if (j < 0) continue;
    const int p = __ldg(a.pos_ref + j);
    float f[M];
#pragma unroll
    for (int k = 0; k < M; ++k) f[k] = fn[k];
    const float tk = canon_dot<M>(f, a.zs + (int64_t)p * M);
    const unsigned long long key = ((unsigned long long)f2ord(tk) << 32) | (uint32_t)(0xffffffffu - (uint32_t)p);
    best = key > best ? key : best;
  }
}

constexpr int HMMA_U = 8;   // tiles per filter step

// one filter step over U tiles t .. t+U-1: 3U independent MMAs (fragment loads issued first), one max per
// row; rows whose step maximum reaches (running max - 2 eps) get their candidates' exact keys (rare after
// the first steps)
template <int M, int U, bool WARM>
__device__ __forceinline__ void hmma_step(const AssocArgs& a, int t, int lane, int tg, const uint32_t (&ah)[4],
                                          const uint32_t (&al)[4], const bool (&act)[2], const float* fn0,
                                          const float* fn1, const float (&marg)[2], float& mx0, float& mx1,
                                          unsigned long long& best0, unsigned long long& best1) {
  uint2 bh[U], bl[U];
  const uint2* fr = a.zfrag + (int64_t)t * HMMA_TS + lane;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    bh[u] = __ldg(fr + u * HMMA_TS);
    bl[u] = __ldg(fr + u * HMMA_TS + 32);
  }
  float v0[U][2], v1[U][2];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    float c[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    mma_bf16_16816(c, ah, bh[u].x, bh[u].y);
    mma_bf16_16816(c, ah, bl[u].x, bl[u].y);
    mma_bf16_16816(c, al, bh[u].x, bh[u].y);
    v0[u][0] = c[0];   // row gid, packed columns 2tg, 2tg + 1 of tile t + u
    v0[u][1] = c[1];
    v1[u][0] = c[2];   // row gid + 8
    v1[u][1] = c[3];
  }
  float s0 = fmaxf(v0[0][0], v0[0][1]), s1 = fmaxf(v1[0][0], v1[0][1]);
#pragma unroll
  for (int u = 1; u < U; ++u) {
    s0 = fmaxf(s0, fmaxf(v0[u][0], v0[u][1]));
    s1 = fmaxf(s1, fmaxf(v1[u][0], v1[u][1]));
  }
  if (!WARM) {
    const float th0 = mx0 - marg[0], th1 = mx1 - marg[1];
    if (act[0] && s0 >= th0) hmma_exact<M, U>(a, fn0, v0, t, tg, th0, best0);
    if (act[1] && s1 >= th1) hmma_exact<M, U>(a, fn1, v1, t, tg, th1, best1);
  }
  // the quad's four lanes see disjoint columns of the same rows: share the step maxima, so a new record
  // triggers one exact pass per row rather than one per lane
  s0 = fmaxf(s0, __shfl_xor_sync(MO_FULL, s0, 1));
  s1 = fmaxf(s1, __shfl_xor_sync(MO_FULL, s1, 1));
  s0 = fmaxf(s0, __shfl_xor_sync(MO_FULL, s0, 2));
  s1 = fmaxf(s1, __shfl_xor_sync(MO_FULL, s1, 2));
  mx0 = fmaxf(mx0, s0);
  mx1 = fmaxf(mx1, s1);
}

template <int M>
__global__ void __launch_bounds__(HMMA_WARPS * 32) k_assoc_hmma(AssocArgs a, int chunks) {
  pdl_wait();
  if (__ldcg(a.info + MO_INFO_ERROR) != 0) return;
  if (__ldcg(a.info + MO_INFO_SKIPPED) != 0) return;
  const int ncand = __ldcg(a.ctl);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gid = lane >> 2, tg = lane & 3;
  const int nrt = (ncand + 15) / 16;                    // 16-row tiles
  const int ngrp = (nrt + HMMA_WARPS - 1) / HMMA_WARPS;  // CTA items: 8 row tiles x one chunk
  const int ntiles = (a.w + 7) / 8;
  const int per_chunk = (ntiles + chunks - 1) / chunks;
  __shared__ float sFn[HMMA_WARPS][16][M];
  for (int item = blockIdx.x; item < ngrp * chunks; item += gridDim.x) {
    const int grp = item / chunks, ch = item - grp * chunks;
    const int rt = grp * HMMA_WARPS + warp;
    const int t0 = ch * per_chunk, t1 = min(ntiles, t0 + per_chunk);
    if (rt >= nrt || t0 >= t1) continue;   // warp-uniform
    // the lane's two rows: gid and gid + 8 of the tile
    int row[2];
    bool act[2];
    float marg[2];
    uint32_t ah[4], al[4];
    float av[2][4];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int c = rt * 16 + gid + 8 * r;
      act[r] = c < ncand;
      row[r] = act[r] ? __ldcg(a.cand + c) : 0;
      float fn[M];
      hmma_load_fn<M>(a, row[r], fn);
      __syncwarp();
      if (tg == 0)
#pragma unroll
        for (int k = 0; k < M; ++k) sFn[warp][gid + 8 * r][k] = fn[k];
      float nn = 0.0f;
      bool fin = true;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        fin = fin && isfinite(fn[k]);
        nn = fmaf(fn[k], fn[k], nn);
      }
      const float norm = sqrtf(nn);
      const bool ok = fin && norm > 1e-30f && isfinite(norm);   // (tiny rows: bf16 subnormal flushes)
      if (act[r] && !ok) {
        if (ch == 0 && tg == 0) {
          a.fb_cand[atomicAdd(a.fb_ctl, 1)] = row[r];
          atomicAdd(const_cast<int*>(a.info) + MO_INFO_ASSOC_FALLBACK, 1);
        }
        act[r] = false;
      }
      marg[r] = act[r] ? ldexpf(norm, -11) : 0.0f;    // 2 eps
      // A-fragment coordinates of this lane: k = 2tg, 2tg+1, 2tg+8, 2tg+9 (0 past m or for idle rows)
#pragma unroll
      for (int q = 0; q < 4; ++q) av[r][q] = 0.0f;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const float v = act[r] ? fn[k] : 0.0f;
        if (k == 2 * tg) av[r][0] = v;
        if (k == 2 * tg + 1) av[r][1] = v;
        if (k == 2 * tg + 8) av[r][2] = v;
        if (k == 2 * tg + 9) av[r][3] = v;
      }
    }
    {
      float h[2][4], l[2][4];
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) split_bf16(av[r][q], h[r][q], l[r][q]);
      // a0: (row gid, k 2tg..+1), a1: (row gid+8, same k), a2: (row gid, k +8), a3: (row gid+8, k +8)
      ah[0] = bf16x2_bits(h[0][0], h[0][1]);
      ah[1] = bf16x2_bits(h[1][0], h[1][1]);
      ah[2] = bf16x2_bits(h[0][2], h[0][3]);
      ah[3] = bf16x2_bits(h[1][2], h[1][3]);
      al[0] = bf16x2_bits(l[0][0], l[0][1]);
      al[1] = bf16x2_bits(l[1][0], l[1][1]);
      al[2] = bf16x2_bits(l[0][2], l[0][3]);
      al[3] = bf16x2_bits(l[1][2], l[1][3]);
    }
    __syncwarp();
    if (!__any_sync(MO_FULL, act[0] || act[1])) continue;
    const float* fn0 = sFn[warp][gid];
    const float* fn1 = sFn[warp][gid + 8];
    float mx0 = -__int_as_float(0x7f800000), mx1 = mx0;
    unsigned long long best0 = 0ull, best1 = 0ull;
    // filter steps of HMMA_U tiles: 3U independent MMAs, then one max per row; the (rare after the first
    // steps) rows whose step maximum reaches the running max - 2 eps get their candidates' exact keys
    const int tfull = t0 + (t1 - t0) / HMMA_U * HMMA_U;
    // warm-up: the filter maxima of the first steps (packed order is a fixed random permutation of the
    // references, so a few steps already sit near the row's maximum) shared across the quad; any value
    // actually seen is a valid running maximum, so the sweep below starts with a tight threshold and
    // evaluates few exact keys
    {
      const int tw = min(tfull, t0 + 4 * HMMA_U);
      for (int t = t0; t < tw; t += HMMA_U)
        hmma_step<M, HMMA_U, true>(a, t, lane, tg, ah, al, act, fn0, fn1, marg, mx0, mx1, best0, best1);
    }
    for (int t = t0; t < tfull; t += HMMA_U)
      hmma_step<M, HMMA_U, false>(a, t, lane, tg, ah, al, act, fn0, fn1, marg, mx0, mx1, best0, best1);
    for (int t = tfull; t < t1; ++t)
      hmma_step<M, 1, false>(a, t, lane, tg, ah, al, act, fn0, fn1, marg, mx0, mx1, best0, best1);
    // the four lanes of a quad hold the same two rows: max key, then one atomic per row
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const unsigned long long b0 = __shfl_xor_sync(MO_FULL, best0, o);
      const unsigned long long b1 = __shfl_xor_sync(MO_FULL, best1, o);
      best0 = b0 > best0 ? b0 : best0;
      best1 = b1 > best1 ? b1 : best1;
    }
    if (tg == 0) {
      if (act[0] && best0) atomicMax(&a.akey[row[0]], best0);
      if (act[1] && best1) atomicMax(&a.akey[row[1]], best1);
    }
  }
}

template <int M>   // m = M: register arrays (the runtime-m version kept fn[] on the stack)
__global__ void k_assoc_final(AssocFinalArgs a) {
  pdl_wait();
  if (__ldcg(a.info + MO_INFO_ERROR) != 0) return;
  if (__ldcg(a.info + MO_INFO_SKIPPED) != 0) return;
  const int ncand = __ldcg(a.ctl);
  const int base = blockIdx.x * blockDim.x;
  if (base >= ncand) return;  // whole block idle (uniform)
  const int c = base + threadIdx.x;
  const bool act = c < ncand;
  constexpr int m = M;
  const int row = act ? __ldcg(a.cand + c) : 0;
  float fn[M];
  if (act) {
#pragma unroll
    for (int k = 0; k < m; ++k) {
      float v = a.F[(int64_t)row * m + k];
      if (a.ideal) v = __fsub_rn(v, a.ideal[k]);
      if (a.a32) v = __fdiv_rn(v, a.a32[k]);
      fn[k] = v;
      if (a.Fn_out) a.Fn_out[(int64_t)row * m + k] = v;
    }
  }
  if (a.fn_only) return;
  int j = 0;
  if (act) {
    const unsigned long long key = __ldcg(a.akey + row);
    const int p = (int)(0xffffffffu - (uint32_t)(key & 0xffffffffull));
    const float* z = a.zs + (int64_t)p * m;
    float t = __fmul_rn(fn[0], z[0]);
#pragma unroll
    for (int k = 1; k < m; ++k) t = __fadd_rn(t, __fmul_rn(fn[k], z[k]));
    float s2 = 0.0f;
#pragma unroll
    for (int k = 0; k < m; ++k) {
      const float e = __fsub_rn(fn[k], __fmul_rn(t, z[k]));
      s2 = k == 0 ? __fmul_rn(e, e) : __fadd_rn(s2, __fmul_rn(e, e));
    }
    j = a.perm_ref[p];
    a.pi[row] = j;
    a.d[row] = __fsqrt_rn(s2);
  }
  if (a.ranks) {  // niche counts, warp-aggregated
    const int l = __ldcg(a.info + MO_INFO_L);
    const int r = act ? a.ranks[row] : -1;
    warp_agg_add(a.rho, j, act && r < l);
    warp_agg_add(a.rho_p, j, act && r == l);
  }
}

// k_assoc_final for runtime m (wide m > 16): identical arithmetic, objectives re-read from F (L1)
// Wide m: a warp per candidate row -- Fn_k and the direction z_k staged by the lanes (coalesced) in a
// per-warp shared-memory slice, then lane 0 runs the same sequential FP32 folds (t, then s2) as
// k_assoc_final<M>, so the results are bit-identical while the loads and divides are spread over 32
// lanes.
constexpr int AFW_WARPS = 4;
__global__ void __launch_bounds__(AFW_WARPS * 32) k_assoc_final_rt(AssocFinalArgs a) {
  __shared__ float sF[AFW_WARPS][MO_MAX_M], sZ[AFW_WARPS][MO_MAX_M];
  pdl_wait();
  if (__ldcg(a.info + MO_INFO_ERROR) != 0) return;
  if (__ldcg(a.info + MO_INFO_SKIPPED) != 0) return;
  const int ncand = __ldcg(a.ctl);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int m = a.m;
  float* fw = sF[w];
  float* zw = sZ[w];
  const int l = a.ranks ? __ldcg(a.info + MO_INFO_L) : 0;
  for (int c = blockIdx.x * AFW_WARPS + w; c < ncand; c += gridDim.x * AFW_WARPS) {   // warp-uniform
    const int row = __ldcg(a.cand + c);
    for (int k = lane; k < m; k += 32) {
      float v = a.F[(int64_t)row * m + k];
      if (a.ideal) v = __fsub_rn(v, a.ideal[k]);
      if (a.a32) v = __fdiv_rn(v, a.a32[k]);
      fw[k] = v;
      if (a.Fn_out) a.Fn_out[(int64_t)row * m + k] = v;
    }
    if (a.fn_only) continue;
    const unsigned long long key = __ldcg(a.akey + row);
    const int p = (int)(0xffffffffu - (uint32_t)(key & 0xffffffffull));
    for (int k = lane; k < m; k += 32) zw[k] = a.zs[(int64_t)p * m + k];
    __syncwarp();
    if (lane == 0) {
      float t = __fmul_rn(fw[0], zw[0]);
      for (int k = 1; k < m; ++k) t = __fadd_rn(t, __fmul_rn(fw[k], zw[k]));
      float s2 = 0.0f;
      for (int k = 0; k < m; ++k) {
        const float e = __fsub_rn(fw[k], __fmul_rn(t, zw[k]));
        s2 = k == 0 ? __fmul_rn(e, e) : __fadd_rn(s2, __fmul_rn(e, e));
      }
      const int j = a.perm_ref[p];
      a.pi[row] = j;
      a.d[row] = __fsqrt_rn(s2);
      if (a.ranks) {
        const int r = a.ranks[row];
        if (r < l) atomicAdd(a.rho + j, 1);
        if (r == l) atomicAdd(a.rho_p + j, 1);
      }
    }
    __syncwarp();   // the slices are rewritten by the next row
  }
}

// --------------------------------------------------------------- select



constexpr int SELECT_THREADS = 512;
constexpr int SEL_BIG = 1024;   // partial buckets above this many candidates are selected block-wide

__device__ __forceinline__ int warp_bitonic_asc(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int o = __shfl_xor_sync(MO_FULL, v, j);
      const bool up = (lane & k) == 0, lower = (lane & j) == 0;
      v = (lower == up) ? min(v, o) : max(v, o);
    }
  return v;
}

// Niche selection after association (Alg. 2 lines 5-26).
//   P0 (op-level only) niche counts
//   P1 nearest-candidate keys of empty niches; M0 = #empty niches
//   P2 M0 > k: promote the nearest of the first k empty niches in shuffled
//      reference order (done).  Else promote every empty niche's nearest,
//      post-nearest counts, level histogram of [rho_j, rho_j + c_j)
//   P3 every block: water level L* = min{L : T(L) >= k'} and `need`
//   P4 marked points at L*, first `need` in shuffled reference order
//   P5 take_j; buckets for partially taken points
//   P6 cache members: all taken, or bucketed by position
//   P7 per bucket: the take_j smallest shuffled positions (warp bitonic /
//      threshold search) -- equal to the cursor order of the cache table
//   P8 survivors: stable compaction in merged-row order
__global__ void __launch_bounds__(SELECT_THREADS) k_select(SelectArgs a) {
  pdl_wait();
  __shared__ int sh[40];
  __shared__ int sHist[2][LVL_BINS];
  __shared__ int sRes[4];
  __shared__ int sSel[(SELECT_THREADS / 32) * 256];   // per-warp radix bins of the P7 top-t select
  const int tid = threadIdx.x, lane = tid & 31;
  const int gtid = blockIdx.x * blockDim.x + tid, gthreads = gridDim.x * blockDim.x;
  const int gwarp = gtid >> 5, nwarps = gthreads >> 5;
  const int R = a.R, w = a.w;
  int* plist = reinterpret_cast<int*>(a.near_key);   // P5 -> P7 list of partially taken points
  if (a.reset_ctl && gtid == 0) *a.reset_ctl = 0;   // k_assoc_final (the last reader) has completed
  if (__ldcg(a.info + MO_INFO_ERROR) != 0) return;
  const int l = __ldcg(a.info + MO_INFO_L);
  const int k = __ldcg(a.info + MO_INFO_K);
  const bool skipped = __ldcg(a.info + MO_INFO_SKIPPED) != 0;
  int kept_nearest = 0, level = -1;
  trace_mark(a.trace, 24);

  if (!skipped) {
    if (a.count_inside) {
      for (int base = blockIdx.x * blockDim.x; base < R; base += gthreads) {
        const int i = base + tid;
        const int r = i < R ? a.ranks[i] : MO_RANK_DROPPED;
        const bool c = (r >= 0) && (r <= l);
        const int j = c ? __ldcg(a.pi + i) : 0;
        warp_agg_add(a.rho, j, c && r < l);
        warp_agg_add(a.rho_p, j, c && r == l);
      }
      grid_sync(a.g.bar);
    }
    // ---- P1
    for (int i = gtid; i < R; i += gthreads) {
      if (a.ranks[i] != l) continue;
      const int j = __ldcg(a.pi + i);
      if (__ldcg(a.rho + j) != 0) continue;
      const unsigned long long key = ((unsigned long long)f2ord(__ldcg(a.d + i)) << 32) | (uint32_t)a.pos_pop[i];
      atomicMin(&a.near_key[j], key);
    }
    {
      int e = 0;
      for (int j = gtid; j < w; j += gthreads) e += (__ldcg(a.rho + j) == 0) & (__ldcg(a.rho_p + j) > 0);
      e = warp_sum(e);
      if (lane == 0 && e) atomicAdd(&a.sctl[SCTL_M0], e);
    }
    grid_sync(a.g.bar);
    trace_mark(a.trace, 25);
    const int M0 = __ldcg(a.sctl + SCTL_M0);
    int k_rem = 0;
    if (M0 > k) {
      // ---- P2 (truncated): the first k empty niches in shuffled reference order
      grid_scan(
          a.g, w,
          [&](int64_t p) {
            const int j = a.perm_ref[p];
            return (int)((__ldcg(a.rho + j) == 0) & (__ldcg(a.rho_p + j) > 0));
          },
          [&](int64_t p, int pre) {
            if (pre >= k) return;
            const int j = a.perm_ref[p];
            a.prom[a.perm_pop[(uint32_t)(__ldcg(a.near_key + j) & 0xffffffffull)]] = 1;
          },
          sh);
      kept_nearest = k;
      grid_sync(a.g.bar);
    } else {
      // ---- P2: all empty niches take their nearest; post-nearest counts; level histogram
      for (int q = tid; q < 2 * LVL_BINS; q += blockDim.x) (&sHist[0][0])[q] = 0;
      __syncthreads();
      int maxe = 0;   // largest end level rho_j + c_j of an active niche (bounds the water level)
      for (int j = gtid; j < w; j += gthreads) {
        int r = __ldcg(a.rho + j), c = __ldcg(a.rho_p + j);
        if (c == 0) continue;
        if (r == 0) {
          a.prom[a.perm_pop[(uint32_t)(__ldcg(a.near_key + j) & 0xffffffffull)]] = 1;
          r = 1;
          c -= 1;
          a.rho[j] = r;
          a.rho_p[j] = c;
        }
        if (c == 0) continue;
        maxe = max(maxe, r + c);
        if (r < LVL_BINS) atomicAdd(&sHist[0][r], 1);
        if (r + c < LVL_BINS) atomicAdd(&sHist[1][r + c], 1);
      }
      maxe = (int)warp_max_u32((uint32_t)maxe);
      if (lane == 0 && maxe >= LVL_BINS) atomicMax(&a.sctl[SCTL_MAXE], maxe);
      __syncthreads();
      for (int q = tid; q < 2 * LVL_BINS; q += blockDim.x) {
        const int v = (&sHist[0][0])[q];
        if (v) atomicAdd(a.lvl + q, v);
      }
      kept_nearest = M0;
      k_rem = k - M0;
      grid_sync(a.g.bar);
    }
    trace_mark(a.trace, 26);
    if (k_rem > 0) {
      // ---- P3: L* from the level histogram, redundantly in every block (no barrier)
      if (tid < 32) {
        long long carryA = 0, carryT = 0, Lstar = -1, before = 0;
        for (int base = 0; base < LVL_BINS && Lstar < 0; base += 32) {
          const int q = base + lane;
          long long x = (long long)__ldcg(a.lvl + q) - (long long)__ldcg(a.lvl + LVL_BINS + q);
          for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(MO_FULL, x, o);
            if (lane >= o) x += t;
          }
          long long A = x + carryA;  // active points at level q
          long long y = A;
          for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(MO_FULL, y, o);
            if (lane >= o) y += t;
          }
          const long long T = y + carryT;  // takes once level q is processed
          const unsigned hit = __ballot_sync(MO_FULL, T >= k_rem);
          if (hit) {
            const int f = __ffs(hit) - 1;
            Lstar = base + f;
            before = __shfl_sync(MO_FULL, T - A, f);
          }
          carryA = __shfl_sync(MO_FULL, A, 31);
          carryT = __shfl_sync(MO_FULL, T, 31);
        }
        if (lane == 0) {
          sRes[0] = (int)Lstar;
          sRes[1] = (int)before;
          sRes[2] = (int)carryT;   // takes below level LVL_BINS (when the level lies beyond the window)
        }
      }
      __syncthreads();
      int L = sRes[0];
      long long before = sRes[1];
      if (L < 0) {
        // level beyond the histogram window (a few crowded niches, e.g. DTLZ3 m = 10 late in a run):
        // grid-cooperative 32-ary search for X = min{x : U(x) >= k'} with U(x) = sum_j clamp(x - rho_j,
        // 0, c_j) the takes below level x; lane i of every warp evaluates candidate x_i, each warp
        // streams 32 niches per coalesced load and broadcasts them by shuffles; one global accumulator
        // per candidate (three rotating sets of 32), one grid barrier per pass, ~log32(max level) passes.
        // Then L* = X - 1 and before = U(X - 1).
        __shared__ unsigned long long sAcc[32];
        __shared__ long long sSearch[3];
        unsigned long long* acc = reinterpret_cast<unsigned long long*>(a.lvl + 2 * LVL_BINS);
        long long lo = LVL_BINS + 1, hi = __ldcg(a.sctl + SCTL_MAXE), Ulo = sRes[2];
        for (int pass = 0; lo < hi; ++pass) {
          unsigned long long* cur = acc + (pass % 3) * 32;
          if (blockIdx.x == 0 && tid < 32) acc[((pass + 1) % 3) * 32 + tid] = 0ull;   // next pass's set
          if (tid < 32) sAcc[tid] = 0ull;
          __syncthreads();
          const long long x = lo + (hi - lo) * lane / 32;
          unsigned long long part = 0;
          for (int base = gwarp * 32; base < w; base += nwarps * 32) {
            const int j = base + lane;
            const int c = j < w ? __ldcg(a.rho_p + j) : 0;
            const int r = c > 0 ? __ldcg(a.rho + j) : 0;
#pragma unroll 8
            for (int q = 0; q < 32; ++q) {
              const int cq = __shfl_sync(MO_FULL, c, q), rq = __shfl_sync(MO_FULL, r, q);
              const long long t0 = x - rq;
              part += t0 <= 0 ? 0ull : (unsigned long long)(t0 > cq ? cq : t0);
            }
          }
          if (part) atomicAdd(&sAcc[lane], part);
          __syncthreads();
          if (tid < 32 && sAcc[tid]) atomicAdd(cur + tid, sAcc[tid]);
          grid_sync(a.g.bar);
          if (tid < 32) {
            const long long u = (long long)__ldcg(cur + tid);
            const unsigned ge = __ballot_sync(MO_FULL, u >= k_rem);   // a suffix of the lanes (U, x_i monotone)
            const int f = ge ? __ffs(ge) - 1 : 32;
            const long long xf = __shfl_sync(MO_FULL, x, f & 31);
            const long long xp = __shfl_sync(MO_FULL, x, (f + 31) & 31);   // x_{f-1} (x_31 when f = 32)
            const long long up = __shfl_sync(MO_FULL, u, (f + 31) & 31);
            if (tid == 0) {
              long long nlo = lo, nhi = hi, nU = Ulo;
              if (f < 32) nhi = xf;
              if (f > 0) {
                nlo = xp + 1;
                nU = up;
              }
              sSearch[0] = nlo;
              sSearch[1] = nhi;
              sSearch[2] = nU;
            }
          }
          __syncthreads();
          lo = sSearch[0];
          hi = sSearch[1];
          Ulo = sSearch[2];
          __syncthreads();
        }
        L = (int)(lo - 1);
        before = Ulo;
      }
      const int need = (int)(k_rem - before);
      level = L;
      trace_mark(a.trace, 27);
      // ---- P4: marked at L*, keep the first `need` in shuffled reference order
      grid_scan(
          a.g, w,
          [&](int64_t p) {
            const int j = a.perm_ref[p];
            const int c = __ldcg(a.rho_p + j);
            const int r = __ldcg(a.rho + j);
            return (int)(c > 0 && r <= L && (long long)L < (long long)r + c);
          },
          [&](int64_t p, int pre) {
            if (pre < need) a.kept[a.perm_ref[p]] = 1;
          },
          sh);
      grid_sync(a.g.bar);
      trace_mark(a.trace, 28);
      // ---- P5: take_j; bucket storage for partially taken points
      for (int base = blockIdx.x * blockDim.x; base < w; base += gthreads) {   // uniform trip count
        const int j = base + threadIdx.x;
        const int c = j < w ? __ldcg(a.rho_p + j) : 0;
        int t = 0;
        if (c > 0) {
          const long long t0 = (long long)L - __ldcg(a.rho + j);
          t = (int)(t0 < 0 ? 0 : (t0 > c ? c : t0)) + __ldcg(a.kept + j);
          a.take[j] = t;
        }
        const bool part = c > 0 && t > 0 && t < c;
        const int off = warp_alloc(&a.sctl[SCTL_ALLOC], part ? c : 0);   // bucket order is immaterial
        if (part) a.bstart[j] = off;
        // the partially taken points, listed for P7 (near_key is dead after P2 and reset by the prologue)
        const int slot = warp_alloc(&a.sctl[SCTL_NPART], part ? 1 : 0);
        if (part) plist[slot] = j;
      }
      grid_sync(a.g.bar);
      trace_mark(a.trace, 29);
      // ---- P6: cache members (F_l minus the nearest-promoted)
      for (int i = gtid; i < R; i += gthreads) {
        if (a.ranks[i] != l || __ldcg(a.prom + i)) continue;
        const int j = __ldcg(a.pi + i);
        const int t = __ldcg(a.take + j);
        if (t == 0) continue;
        if (t >= __ldcg(a.rho_p + j)) {
          a.prom[i] = 1;
        } else {
          const int slot = __ldcg(a.bstart + j) + atomicAdd(&a.fill[j], 1);
          a.bucket[slot] = a.pos_pop[i];
        }
      }
      grid_sync(a.g.bar);
      trace_mark(a.trace, 30);
      // ---- P7: the take_j smallest shuffled positions of every partial bucket (warp per point)
      const int npart = __ldcg(a.sctl + SCTL_NPART);
      for (int e = gwarp; e < npart; e += nwarps) {
        const int j = __ldcg(plist + e);
        const int t = __ldcg(a.take + j), c = __ldcg(a.rho_p + j);
        if (c > SEL_BIG) continue;   // crowded niche: a whole block below
        const int* bk = a.bucket + __ldcg(a.bstart + j);
        if (c <= 32) {
          int v = lane < c ? __ldcg(bk + lane) : 0x7fffffff;
          v = warp_bitonic_asc(v);
          if (lane < t) a.prom[a.perm_pop[v]] = 1;
        } else {
          // the t-th smallest of the c distinct positions (< R) by an 8-bit-digit radix select in this
          // warp's shared-memory bins: ceil(log2(R) / 8) passes over the bucket instead of a binary
          // search of log2(R) passes (crowded niches hold thousands of candidates late in a run)
          int* bins = sSel + (tid >> 5) * 256;
          const int nbits = 32 - __clz(max(R - 1, 1));
          int prefix = 0, need = t;
          for (int shift = nbits; shift > 0;) {
            const int b = min(8, shift);
            shift -= b;
            const int hiShift = shift + b;   // bits >= hiShift are fixed in prefix
#pragma unroll
            for (int q = 0; q < 8; ++q) bins[lane * 8 + q] = 0;
            __syncwarp();
            for (int q = lane; q < c; q += 32) {
              const int v = __ldcg(bk + q);
              if (hiShift >= 31 || (v >> hiShift) == (prefix >> hiShift))
                atomicAdd(&bins[(v >> shift) & ((1 << b) - 1)], 1);
            }
            __syncwarp();
            int cnt[8], sum = 0;   // lane owns bins [8 lane, 8 lane + 8)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              cnt[q] = bins[lane * 8 + q];
              sum += cnt[q];
            }
            int incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int y = __shfl_up_sync(MO_FULL, incl, o);
              if (lane >= o) incl += y;
            }
            const unsigned hit = __ballot_sync(MO_FULL, incl >= need);
            const int fl = __ffs(hit) - 1;   // the lane whose bins reach `need` (always exists)
            int digit = 0, below = 0;
            if (lane == fl) {
              int run = incl - sum;
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                if (run + cnt[q] >= need) {
                  digit = lane * 8 + q;
                  below = run;
                  break;
                }
                run += cnt[q];
              }
            }
            digit = __shfl_sync(MO_FULL, digit, fl);
            below = __shfl_sync(MO_FULL, below, fl);
            prefix |= digit << shift;
            need -= below;
            __syncwarp();
          }
          for (int q = lane; q < c; q += 32) {
            const int v = __ldcg(bk + q);
            if (v <= prefix) a.prom[a.perm_pop[v]] = 1;
          }
        }
      }
      // crowded niches (> SEL_BIG bucketed candidates): the same radix select by a whole block, the
      // candidates of 512 reference points at a time compacted through shared memory
      {
        int* bins = &sHist[0][0];          // free after P2
        int* list = &sHist[1][0];
        __shared__ int sNbig, sDigit, sBelow;
        for (int base = blockIdx.x * SELECT_THREADS; base < npart; base += gridDim.x * SELECT_THREADS) {
          if (tid == 0) sNbig = 0;
          __syncthreads();
          if (base + tid < npart) {
            const int j = __ldcg(plist + base + tid);
            if (__ldcg(a.rho_p + j) > SEL_BIG) list[atomicAdd(&sNbig, 1)] = j;
          }
          __syncthreads();
          const int nbig = sNbig;
          for (int e = 0; e < nbig; ++e) {
            const int j = list[e];
            const int t = __ldcg(a.take + j), c = __ldcg(a.rho_p + j);
            const int* bk = a.bucket + __ldcg(a.bstart + j);
            const int nbits = 32 - __clz(max(R - 1, 1));
            int prefix = 0, need = t;
            for (int shift = nbits; shift > 0;) {
              const int b = min(8, shift);
              shift -= b;
              const int hiShift = shift + b;
              if (tid < 256) bins[tid] = 0;
              __syncthreads();
              for (int q = tid; q < c; q += SELECT_THREADS) {
                const int v = __ldcg(bk + q);
                if (hiShift >= 31 || (v >> hiShift) == (prefix >> hiShift))
                  atomicAdd(&bins[(v >> shift) & ((1 << b) - 1)], 1);
              }
              __syncthreads();
              if (tid < 32) {
                int cnt[8], sum = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                  cnt[q] = bins[lane * 8 + q];
                  sum += cnt[q];
                }
                int incl = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                  const int y = __shfl_up_sync(MO_FULL, incl, o);
                  if (lane >= o) incl += y;
                }
                const unsigned hit = __ballot_sync(MO_FULL, incl >= need);
                const int fl = __ffs(hit) - 1;
                if (lane == fl) {
                  int run = incl - sum;
#pragma unroll
                  for (int q = 0; q < 8; ++q) {
                    if (run + cnt[q] >= need) {
                      sDigit = lane * 8 + q;
                      sBelow = run;
                      break;
                    }
                    run += cnt[q];
                  }
                }
              }
              __syncthreads();
              prefix |= sDigit << shift;
              need -= sBelow;
              __syncthreads();
            }
            for (int q = tid; q < c; q += SELECT_THREADS) {
              const int v = __ldcg(bk + q);
              if (v <= prefix) a.prom[a.perm_pop[v]] = 1;
            }
          }
          __syncthreads();   // list / sNbig reuse
        }
      }
      grid_sync(a.g.bar);
      trace_mark(a.trace, 31);
    }
  }
  // ---- P8: survivors = fronts < l + promoted (or fronts <= l when niching was skipped);
  //          promoted rank = l - 1 (A-8); stable compaction in merged-row order (A-9)
  // wide rows (d + m >= 64, e.g. PAPER Appendix D d = 1000): the emitting thread only records the slot
  // and the block's warps copy its chunk's survivors row by row, coalesced
  const bool wide_copy = a.X_next && a.dvars + a.m >= 64;
  auto survives = [&](int64_t i) {
    const int r = a.ranks[i];
    return skipped ? (r >= 0 && r <= l) : ((r >= 0 && r < l) || __ldcg(a.prom + i) != 0);
  };
  const int nsurv = grid_scan(
      a.g, R, [&](int64_t i) { return (int)survives(i); },
      [&](int64_t i, int pre) {
        // survivor `pre` <- merged row i, copied by the emitting thread (the rows are L2-resident; no
        // barrier + second pass for a separate gather)
        if (wide_copy) {
          a.bucket[i] = pre;   // bucket (P6 / P7) is dead here
        } else if (a.X_next) {
          const int d = a.dvars, mm = a.m;
          const float* xs = a.XR + i * d;
          float* xd = a.X_next + (int64_t)pre * d;
          for (int v = 0; v < d; ++v) xd[v] = xs[v];
          for (int k = 0; k < mm; ++k) a.F_next[(int64_t)pre * mm + k] = a.FR[i * mm + k];
        }
      },
      sh);
  if (wide_copy) {
    // this block's chunk of the scan, SELECT_THREADS rows at a time: its survivors listed in shared
    // memory (sSel is free after P7), then the (row, element) space copied by the whole block
    __shared__ int sNl;
    const int64_t chunk = ceil_div((int64_t)R, (int64_t)gridDim.x);
    const int64_t lo = min((int64_t)blockIdx.x * chunk, (int64_t)R), hi = min(lo + chunk, (int64_t)R);
    const int d = a.dvars, mm = a.m, rowlen = a.dvars + a.m;
    for (int64_t w0 = lo; w0 < hi; w0 += SELECT_THREADS) {
      if (tid == 0) sNl = 0;
      __syncthreads();   // (first window: the slot records of this chunk are visible block-wide)
      const int64_t e = w0 + tid;
      if (e < hi && survives(e)) sSel[atomicAdd(&sNl, 1)] = (int)e;
      __syncthreads();
      const int nl = sNl;
      for (int t = tid; t < nl * rowlen; t += SELECT_THREADS) {   // nl <= 512: fits in int
        const int li = t / rowlen, v = t - li * rowlen;
        const int64_t i = sSel[li];
        const int64_t dst = __ldcg(a.bucket + i);
        if (v < d) a.X_next[dst * d + v] = a.XR[i * d + v];
        else a.F_next[dst * mm + (v - d)] = a.FR[i * mm + (v - d)];
      }
      __syncthreads();
    }
  }
  trace_mark(a.trace, 35);
  // No grid barrier after the P8 compaction scan: other blocks may still be in grid_scan's second
  // pass re-reading ranks[] of their chunks while this loop rewrites promoted rows to l-1.  That is
  // benign only because the P8 predicate of a promoted row is true through `prom` whatever its rank
  // (r = l or l-1 both select it); a predicate that depends on the rank value of a promoted row
  // would need the barrier back.
  for (int i = gtid; i < R; i += gthreads) {
    const int r = a.ranks[i];
    const bool pr = !skipped && __ldcg(a.prom + i) != 0;
    const bool s = skipped ? (r >= 0 && r <= l) : ((r >= 0 && r < l) || pr);
    if (a.selected) a.selected[i] = s;
    if (pr) a.ranks[i] = l - 1;
  }
  if (gtid == 0) {
    a.info[MO_INFO_NEAREST] = kept_nearest;
    a.info[MO_INFO_LEVEL] = level;
    a.info[MO_INFO_SURVIVORS] = nsurv;
    if (a.gen_ptr) *a.gen_ptr += 1u;
  }
  trace_mark(a.trace, 36);
}

// ------------------------------------------------------------- launchers

static int coop_blocks(const void* fn, int threads, int cap_per_sm) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, 0);
  if (per > cap_per_sm) per = cap_per_sm;
  return sms * (per > 0 ? per : 1);
}

template <class Args>
static int launch_coop(void (*fn)(Args), int blocks, int threads, Args args, cudaStream_t s) {
  return launch_ex(fn, dim3(blocks), dim3(threads), 0, s, true, g_mo_pdl, args);
}

int prep_grid_blocks() {
  static int b = 0;
  if (!b) b = coop_blocks((const void*)k_prep, 256, 2);
  return b;
}
int select_grid_blocks() {
  static int b = 0;
  if (!b) b = coop_blocks((const void*)k_select, SELECT_THREADS, 1);
  return b;
}

int launch_prep(const PrepArgs& a, cudaStream_t s) {
  // phase 1 (extreme points): register arrays for m <= 16 (MO_PX_CASE), the runtime-m pass above; m > MAXM
  // needs the global system buffer
  if (a.m < 1 || a.m > MO_MAX_M || (a.mode == PREP_FULL && a.m > MAXM && !a.solveA)) return MO_ERR_PARAM;
  if (!a.in_step) {
    if (cudaMemsetAsync(a.ctl, 0, sizeof(int), s) != cudaSuccess) return MO_ERR_CUDA;
    if (cudaMemsetAsync(a.bar, 0, 2 * sizeof(unsigned), s) != cudaSuccess) return MO_ERR_CUDA;
  }
  int blocks = prep_grid_blocks();
  int need = (int)ceil_div((int64_t)(a.R > a.w ? a.R : a.w), 256);
  if (a.m > 16) need = (int)ceil_div((int64_t)a.R, (int64_t)32);   // wide m: a warp per row, ~4 rows per warp
  if (blocks > need) blocks = need < 1 ? 1 : need;
  return launch_coop(k_prep, blocks, 256, a, s);
}

int launch_assoc(const AssocArgs& a, int m, int64_t R, cudaStream_t s) {
  if (R <= 0) return MO_OK;
  static int capacity = 0;
  if (!capacity) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_assoc<5>, ASSOC_THREADS, 0);
    capacity = sms * (per > 0 ? per : 1);
  }
  AssocArgs b = a;
  dim3 grid(capacity);
  switch (m) {
#define MO_AS_CASE(MM) \
  case MM: MO_TRY(launch_ex(k_assoc<MM>, grid, dim3(ASSOC_THREADS), 0, s, false, g_mo_pdl, b)); break;
    MO_AS_CASE(1)
    MO_AS_CASE(2)
    MO_AS_CASE(3)
    MO_AS_CASE(4)
    MO_AS_CASE(5)
    MO_AS_CASE(6)
    MO_AS_CASE(7)
    MO_AS_CASE(8)
    MO_AS_CASE(9)
    MO_AS_CASE(10)
    MO_AS_CASE(11)
    MO_AS_CASE(12)
    MO_AS_CASE(13)
    MO_AS_CASE(14)
    MO_AS_CASE(15)
    MO_AS_CASE(16)
#undef MO_AS_CASE
    default: {
      if (m > MO_MAX_M || !a.zsT) return MO_ERR_PARAM;
      const size_t smem = (size_t)ASSOCW_ROWS * m * sizeof(float);
      static bool attr = false;
      if (!attr) {
        if (cudaFuncSetAttribute(k_assoc_wide, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 ASSOCW_ROWS * MO_MAX_M * (int)sizeof(float)) != cudaSuccess)
          return MO_ERR_CUDA;
        attr = true;
      }
      MO_TRY(launch_ex(k_assoc_wide, grid, dim3(ASSOC_THREADS), smem, s, false, g_mo_pdl, b, m));
    }
  }
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int launch_pack_refs(const float* zhat, int64_t w, int m, const int32_t* order, uint2* out, cudaStream_t s) {
  if (w < 1 || m < 1 || m > 16) return MO_ERR_PARAM;
  const int64_t n = (w + 7) / 8 * 32;
  k_pack_refs<<<(unsigned)ceil_div(n, (int64_t)256), 256, 0, s>>>(zhat, w, m, order, out);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

// tensor-core filtered full scan + the sliced FP32 scan for its rejects (zero / non-finite rows)
int launch_assoc_hmma(const AssocArgs& a, int m, int64_t R, cudaStream_t s) {
  if (R <= 0) return MO_OK;
  if (!a.zfrag || m < 2 || m > 16 || a.zbeg != 0 || a.zend != a.w) return MO_ERR_PARAM;
  if (!a.in_step) {
    if (cudaMemsetAsync(a.fb_ctl, 0, sizeof(int), s) != cudaSuccess) return MO_ERR_CUDA;
    if (cudaMemsetAsync(const_cast<int*>(a.info) + MO_INFO_ASSOC_FALLBACK, 0, sizeof(int), s) != cudaSuccess)
      return MO_ERR_CUDA;
  }
  static int sms = 0, per = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_assoc_hmma<16>, HMMA_WARPS * 32, 0);
  }
  // chunks of the reference range: enough CTA items (8 row tiles x chunk) for ~4 waves of 2 CTAs per SM
  // at the worst-case candidate count R, each chunk >= 64 tiles
  const int64_t grp = ceil_div(ceil_div(R, (int64_t)16), (int64_t)HMMA_WARPS);
  const int64_t ntiles = ceil_div((int64_t)a.w, (int64_t)8);
  int64_t chunks = ceil_div((int64_t)sms * 16, grp);
  if (chunks > ntiles / 64) chunks = ntiles / 64;
  if (chunks < 1) chunks = 1;
  const dim3 grid((unsigned)(sms * (per > 1 ? per : 2))), blk(HMMA_WARPS * 32);
  switch (m) {
#define MO_HM_CASE(MM) \
  case MM: MO_TRY(launch_ex(k_assoc_hmma<MM>, grid, blk, 0, s, false, g_mo_pdl, a, (int)chunks)); break;
    MO_HM_CASE(2) MO_HM_CASE(3) MO_HM_CASE(4) MO_HM_CASE(5) MO_HM_CASE(6) MO_HM_CASE(7) MO_HM_CASE(8)
    MO_HM_CASE(9) MO_HM_CASE(10) MO_HM_CASE(11) MO_HM_CASE(12) MO_HM_CASE(13) MO_HM_CASE(14)
    MO_HM_CASE(15) MO_HM_CASE(16)
#undef MO_HM_CASE
    default: return MO_ERR_PARAM;
  }
  return launch_assoc_fallback(a, m, s);
}

// the sliced FP32 full scan of the rows a filtered association appended to fb_cand
int launch_assoc_fallback(const AssocArgs& a, int m, cudaStream_t s) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const dim3 fg((unsigned)sms), fb(256);
  switch (m) {
#define MO_FB_CASE(MM) \
  case MM: return launch_ex(k_assoc_fallback<MM>, fg, fb, 0, s, false, g_mo_pdl, a);
    MO_FB_CASE(2) MO_FB_CASE(3) MO_FB_CASE(4) MO_FB_CASE(5) MO_FB_CASE(6) MO_FB_CASE(7) MO_FB_CASE(8)
    MO_FB_CASE(9) MO_FB_CASE(10) MO_FB_CASE(11) MO_FB_CASE(12) MO_FB_CASE(13) MO_FB_CASE(14)
    MO_FB_CASE(15) MO_FB_CASE(16)
#undef MO_FB_CASE
    default: return MO_ERR_PARAM;
  }
}

int launch_assoc_lattice(const AssocArgs& a, int m, int64_t R, cudaStream_t s) {
  if (R <= 0) return MO_OK;
  if (!a.in_step) {
    if (cudaMemsetAsync(a.fb_ctl, 0, sizeof(int), s) != cudaSuccess) return MO_ERR_CUDA;
    if (cudaMemsetAsync(const_cast<int*>(a.info) + MO_INFO_ASSOC_FALLBACK, 0, sizeof(int), s) != cudaSuccess)
      return MO_ERR_CUDA;
  }
  // lanes per candidate row: enough to cover the box with few points each
  switch (m) {
    case 2: MO_TRY(launch_ex(k_assoc_lattice<2, 1>, dim3((unsigned)ceil_div(R, 256)), dim3(256), 0, s, false, g_mo_pdl, a)); break;
    case 3: MO_TRY(launch_ex(k_assoc_lattice<3, 8>, dim3((unsigned)ceil_div(R * 8, 256)), dim3(256), 0, s, false, g_mo_pdl, a)); break;
    case 4: MO_TRY(launch_ex(k_assoc_lattice<4, 32>, dim3((unsigned)ceil_div(R * 32, 256)), dim3(256), 0, s, false, g_mo_pdl, a)); break;
    case 5: MO_TRY(launch_ex(k_assoc_lattice<5, 16>, dim3((unsigned)ceil_div(R * 16, 256)), dim3(256), 0, s, false, g_mo_pdl, a)); break;
    default: return MO_ERR_PARAM;
  }
  // fallback rows: a warp-per-row full scan over this launch's reference range
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const dim3 fg((unsigned)sms), fb(256);
  switch (m) {
    case 2: return launch_ex(k_assoc_fallback<2>, fg, fb, 0, s, false, g_mo_pdl, a);
    case 3: return launch_ex(k_assoc_fallback<3>, fg, fb, 0, s, false, g_mo_pdl, a);
    case 4: return launch_ex(k_assoc_fallback<4>, fg, fb, 0, s, false, g_mo_pdl, a);
    case 5: return launch_ex(k_assoc_fallback<5>, fg, fb, 0, s, false, g_mo_pdl, a);
    default: return MO_ERR_PARAM;
  }
}

int launch_assoc_final(const AssocFinalArgs& a, int64_t R, cudaStream_t s) {
  if (R <= 0) return MO_OK;
  const dim3 grid((unsigned)ceil_div(R, 128)), blk(128);
  switch (a.m) {
#define MO_AF_CASE(MM) \
  case MM: return launch_ex(k_assoc_final<MM>, grid, blk, 0, s, false, g_mo_pdl, a);
    MO_AF_CASE(1) MO_AF_CASE(2) MO_AF_CASE(3) MO_AF_CASE(4) MO_AF_CASE(5) MO_AF_CASE(6) MO_AF_CASE(7)
    MO_AF_CASE(8) MO_AF_CASE(9) MO_AF_CASE(10) MO_AF_CASE(11) MO_AF_CASE(12) MO_AF_CASE(13) MO_AF_CASE(14)
    MO_AF_CASE(15) MO_AF_CASE(16)
#undef MO_AF_CASE
    default:
      if (a.m > MO_MAX_M) return MO_ERR_PARAM;
      return launch_ex(k_assoc_final_rt, dim3((unsigned)ceil_div(R, (int64_t)AFW_WARPS)), dim3(AFW_WARPS * 32), 0, s,
                       false, g_mo_pdl, a);
  }
}

int launch_select(const SelectArgs& a, cudaStream_t s) {
  if (!a.in_step && cudaMemsetAsync(a.g.bar, 0, 2 * sizeof(unsigned), s) != cudaSuccess) return MO_ERR_CUDA;
  int blocks = select_grid_blocks();
  // ~128 rows per CTA (one CTA per SM at C2): the phases are latency-bound, and more CTAs in flight beat
  // the extra barrier arrivals (C2: 64 -> 44 us, rows/CTA 1024 -> 128)
  const int64_t rows = a.R > a.w ? a.R : a.w;
  int need = (int)ceil_div(rows, (int64_t)128);
  // C1-sized: one CTA, every grid barrier is a __syncthreads (not for wide rows: the survivor copy;
  // measured: R = 184 10.2k -> 11.8k generations/s, but R = 2,000 ~10 % slower than 16 CTAs)
  if (rows <= 512 && a.dvars + a.m < 64) need = 1;
  // wide rows: enough CTAs for the survivor copy (~32K copied values per CTA)
  if (a.X_next && a.dvars + a.m >= 64) {
    const int64_t copy = ceil_div((int64_t)a.n * (a.dvars + a.m), (int64_t)32768);
    if (copy > need) need = (int)copy;
  }
  if (blocks > need) blocks = need < 1 ? 1 : need;
  return launch_coop(k_select, blocks, SELECT_THREADS, a, s);
}

}  // namespace mo
