// Streamed / row-sharded non-dominated sort (no bit-matrix in memory).
//
// Reference: dominance.non_dominated_sort + split_fronts,
// dominance_matrix.  Same ranks as the bit-matrix path
// (k_dominance.cu); this one is for populations whose R^2/8-byte bit-matrix
// does not fit (C4: R = 2M -> 500 GB) and for sharding across GPUs
// (north_star: rows of the dominance relation split across the GPUs of a
// box, per-front masks all-gathered over NVLink).
//
// Rows live in presort position space (k_presort: S-ordered buckets, so the
// dominators of position p sit at positions < wend[p] * 32).  Position blocks
// of 256 rows are dealt round-robin to the G shards (block b -> shard b % G,
// local index b / G), which balances the triangular work.  A shard owns the
// dominated rows j of its blocks:
//
//   begin     cnt[j] = #dominators of j       (k_stream_tiles, COUNT)
//             front 0 = owned rows with cnt 0 (k_stream_mark -> mask_local)
//   front k   host all-gathers mask_local -> mask_full (NCCL; G = 1: alias)
//             k_stream_apply: rank_pos = k for the front, ordered front list
//             fl (position order), |F_k|, cumulative size, split decision
//             cnt[j] -= #dominators of j in F_k  (k_stream_tiles, DEC)
//             front k+1 = owned unranked rows with cnt 0
//   end       ranks in row order
//
// Count-decrement is bounded: sum_k |F_k| x R pairs <= the R^2/2 triangle
// (only F_k rows before j in position order are compared), so a generation
// costs at most two triangle sweeps of m-compare chains and O(R) memory.
// Every kernel checks ctl[SC_DONE] first, so the host may run ahead of the
// split decision (it polls info[MO_INFO_NFRONTS] every few fronts).
// Work is a device-planned queue: k_stream_plan counts the (row block, i
// chunk) items of every owned block from wend / the front list, and the
// persistent k_stream_tiles CTAs pull items with one atomic each.
//
// Two position spaces.  "Slab" (m > 10): k_presort's S-ordered buckets --
// dominators precede (triangle), S-separated tiles need only the <= chain.
// "Boxed" (m <= 10): k_presort_morton's Morton order of the quantised
// objectives makes every 256-row block compact in objective space, so an
// ordered block pair (i block, j block) is usually decided by the two
// bounding boxes alone: some min_i[k] > max_j[k] -> no i dominates any j;
// max_i <= min_j everywhere and < somewhere -> every i dominates every j
// (count += |block|); only "mixed" pairs are computed row by row.  Every
// ordered pair is visited (no triangle) but at C4 (m = 3, R = 2M) only a few
// per cent are mixed.  The front-list chunks of DEC carry boxes too.
#include "mo_chains.cuh"
#include "mo_common.cuh"
#include "mo_grid.cuh"
#include "k_stream_args.cuh"

namespace mo {

constexpr int ST_THREADS = STREAM_BLK / 2;   // two j columns per thread
// k_stream_fused: big CTAs (the sweep is warp-centric) so its grid barriers have few participants
constexpr int FUSED_THREADS = 512;
constexpr int PLAN_THREADS = 1024;
constexpr int APPLY_THREADS = 512;
enum { MODE_COUNT = 0, MODE_DEC = 1 };

__device__ __forceinline__ int owned_block(const StreamArgs& a, int t) { return t * a.G + a.g; }
__device__ __forceinline__ int nblocks(int R) { return (R + STREAM_BLK - 1) / STREAM_BLK; }
// first position after every possible dominator of the rows of block b
__device__ __forceinline__ int block_bend(const StreamArgs& a, int b) {
  const int last = min(a.R, (b + 1) * STREAM_BLK) - 1;
  return min(a.R, __ldg(a.wend + last) * 32);
}

__global__ void k_stream_reset(StreamArgs a) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  for (int p = gt; p < a.R; p += gs) {
    a.rank_pos[p] = MO_RANK_UNRANKED;
    a.cnt[p] = 0;
  }
  for (int t = gt; t < a.T; t += gs) {
    const int b = owned_block(a, t);
    a.ucnt[t] = max(0, min(a.R, (b + 1) * STREAM_BLK) - b * STREAM_BLK);
  }
  if (gt < SC_COUNT) a.ctl[gt] = 0;
  if (gt < MO_INFO_COUNT) a.info[gt] = 0;
  if (a.stats && gt < 4) a.stats[gt] = 0;
}

// Work items of owned block t: (j block, chunk of CHUNK i blocks / front-list entries).
template <int MODE>
__device__ __forceinline__ int block_items(const StreamArgs& a, int t, int fln) {
  const int nb = nblocks(a.R);
  const int b = owned_block(a, t);
  if (b >= nb) return 0;
  if (a.boxed) {
    if (MODE == MODE_COUNT) return (nb + STREAM_CHUNK - 1) / STREAM_CHUNK;
    if (__ldcg(a.ucnt + t) == 0) return 0;
    return (fln + STREAM_BLK * STREAM_CHUNK - 1) / (STREAM_BLK * STREAM_CHUNK);
  }
  const int bend = block_bend(a, b);
  if (MODE == MODE_COUNT) {
    const int nib = (bend + STREAM_BLK - 1) / STREAM_BLK;
    return (nib + STREAM_CHUNK - 1) / STREAM_CHUNK;
  }
  if (__ldcg(a.ucnt + t) == 0) return 0;
  int lo = 0, hi = fln;  // fl entries with position < bend
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldcg(a.fl + mid) < bend) lo = mid + 1; else hi = mid;
  }
  return (lo + STREAM_BLK * STREAM_CHUNK - 1) / (STREAM_BLK * STREAM_CHUNK);
}

// Boxed mode: every owned block has the same number of items (no bound per block), so items decode
// as (t, c) = (item / per, item % per) without a plan search; blocks with nothing to do are skipped
// when their item comes up.
template <int MODE>
__host__ __device__ __forceinline__ int boxed_items_per_block(int nb, int fln) {
  return MODE == MODE_COUNT ? (nb + STREAM_CHUNK - 1) / STREAM_CHUNK
                            : (fln + STREAM_BLK * STREAM_CHUNK - 1) / (STREAM_BLK * STREAM_CHUNK);
}

// One CTA: items per owned block, exclusive prefix into plan[0..T].
template <int MODE>
__global__ void __launch_bounds__(PLAN_THREADS) k_stream_plan(StreamArgs a) {
  __shared__ int sh[40];
  const int tid = threadIdx.x;
  const bool done = __ldcg(a.ctl + SC_DONE) != 0;
  const int fln = __ldcg(a.ctl + SC_FLN);
  if (a.boxed) {
    if (tid == 0) {
      a.ctl[SC_ITEMS] = done ? 0 : a.T * boxed_items_per_block<MODE>(nblocks(a.R), fln);
      a.ctl[SC_WORK] = 0;
    }
    return;
  }
  const int per = (a.T + PLAN_THREADS - 1) / PLAN_THREADS;
  const int t0 = min(a.T, tid * per), t1 = min(a.T, t0 + per);
  int mine = 0;
  for (int t = t0; t < t1; ++t) {
    const int items = done ? 0 : block_items<MODE>(a, t, fln);
    a.plan[t] = items;  // temporarily the count
    mine += items;
  }
  int total;
  int pre = block_excl_scan(mine, sh, &total);
  for (int t = t0; t < t1; ++t) {
    const int c = a.plan[t];
    a.plan[t] = pre;
    pre += c;
  }
  if (tid == 0) {
    a.plan[a.T] = total;
    a.ctl[SC_ITEMS] = total;
    a.ctl[SC_WORK] = 0;
  }
}

// Persistent tiles: item = (owned block t, chunk c).  COUNT: i over the
// position blocks [c*CHUNK, ...) below the block's bound; DEC: i over the
// front list entries [c*CHUNK*256, ...) below the bound.  Thread = 2 rows j;
// i rows staged in shared memory.  Fast tiles (every S_i < every S_j) need
// only the m-long <= chain; others the full dominance chain (also rejects
// i == j).  Counts accumulate with a predicated FADD (FMA pipe, exact below
// 2^24) and land with one atomic per row per item.
// The work loop of the tile sweep, shared by k_stream_tiles (one launch per
// sweep) and k_stream_fused (all sweeps of a generation in one launch).
// Items are pulled from `counter`; the item index is the counter value minus
// `base`.  Arrays written earlier in the same fused launch (plan, fl, flmax,
// flbox) are read through L2 (__ldcg).
// Read-only-during-the-launch data through L1 (__ldg); data written earlier in the same fused launch
// through L2 (__ldcg).
template <bool FUSED, class T>
__device__ __forceinline__ T ldx(const T* p) {
  if (FUSED) return __ldcg(p);
  return __ldg(p);
}

// Warp-centric: a work item is (owned j block t, chunk c of i rows, quarter wq of the block's 256 j
// rows); each warp pulls its own items and stages its 32-row i groups in a private shared-memory slice
// with __syncwarp -- no CTA barriers, so warps whose boxes skip most groups never wait for busy ones.
// Lane = 2 adjacent j rows; the warp owns 64 j rows (one j box).
template <int M, int MODE, bool FUSED>
__device__ __forceinline__ void tiles_run(const StreamArgs& a, float* sFw, int items, int fln, int* counter,
                                          int base) {
  constexpr int MP = (M + 3) & ~3;
  const int lane = threadIdx.x & 31;
  float* sF = sFw + (threadIdx.x >> 5) * 32 * MP;   // this warp's 32-row staging slice
  const float PINF = __int_as_float(0x7f800000);
  const int nbk = nblocks(a.R);
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(counter, 1) - base;
    item = __shfl_sync(MO_FULL, item, 0);
    if (item >= 4 * items) break;
    const int wq = item & 3;
    item >>= 2;
    int t, c;
    if (a.boxed) {
      const int per = boxed_items_per_block<MODE>(nbk, fln);
      t = item / per;
      c = item - t * per;
      if (owned_block(a, t) >= nbk) continue;
      if (MODE == MODE_DEC && ldx<FUSED>(a.ucnt + t) == 0) continue;
    } else {
      int lo = 0, hi = a.T;  // largest t with plan[t] <= item
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (ldx<FUSED>(a.plan + mid) <= item) lo = mid; else hi = mid;
      }
      t = lo;
      c = item - ldx<FUSED>(a.plan + t);
    }
    const int bj = owned_block(a, t);
    const int j0 = bj * STREAM_BLK;
    const int ja = j0 + 64 * wq + 2 * lane, jb = ja + 1;
    if (j0 + 64 * wq >= a.R) continue;
    float fa[M], fb[M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      fa[k] = ja < a.R ? __ldg(a.FS + (int64_t)ja * M + k) : PINF;
      fb[k] = jb < a.R ? __ldg(a.FS + (int64_t)jb * M + k) : PINF;
    }
    const float jmin = __ldg(a.blkmin + bj);
    float wjmn[M], wjmx[M];  // bounding box of this warp's 64 j rows (boxed mode)
    float wjS = 0.0f;        // min S over them
    if (a.boxed) {
      const int q = (j0 + 64 * wq) / 32;
      const int q2 = min(q + 1, (a.R - 1) / 32);
#pragma unroll
      for (int k = 0; k < M; ++k) {
        wjmn[k] = fminf(__ldg(a.blkbox32 + (int64_t)q * 2 * M + k), __ldg(a.blkbox32 + (int64_t)q2 * 2 * M + k));
        wjmx[k] = fmaxf(__ldg(a.blkbox32 + (int64_t)q * 2 * M + M + k),
                        __ldg(a.blkbox32 + (int64_t)q2 * 2 * M + M + k));
      }
      wjS = fminf(__ldg(a.blkS32 + (int64_t)q * 2), __ldg(a.blkS32 + (int64_t)q2 * 2));
    }
    const int bend = a.boxed ? a.R : block_bend(a, bj);
    int e0, e1;  // i range: positions (COUNT) or front-list entries (DEC)
    if (MODE == MODE_COUNT) {
      e0 = c * STREAM_CHUNK * STREAM_BLK;
      e1 = min(bend, e0 + STREAM_CHUNK * STREAM_BLK);
      e1 = (e1 + STREAM_BLK - 1) / STREAM_BLK * STREAM_BLK;  // whole blocks (rows >= bend cannot dominate)
      e1 = min(e1, a.R);
    } else {
      e0 = c * STREAM_CHUNK * STREAM_BLK;
      e1 = min(fln, e0 + STREAM_CHUNK * STREAM_BLK);
    }
    float ca = 0.0f, cb = 0.0f;   // predicated-FADD counts
    unsigned long long nfast = 0, nfull = 0;   // (i, j) pairs evaluated by this lane (measurement)
    int na = 0, nb2 = 0;          // box "all" counts
    for (int s0 = e0; s0 < e1; s0 += STREAM_BLK) {
      const int nv = min(STREAM_BLK, e1 - s0);
      if (a.boxed) {  // block-pair classification from the 256-level bounding boxes
        const float* ib = (MODE == MODE_COUNT ? a.blkbox : a.flbox) + (int64_t)(s0 / STREAM_BLK) * 2 * M;
        const float* jb2 = a.blkbox + (int64_t)bj * 2 * M;
        bool none = false, all = true, strict = false;
#pragma unroll
        for (int k = 0; k < M; ++k) {
          const float imn = ldx<FUSED>(ib + k), imx = ldx<FUSED>(ib + M + k);
          const float jmn = __ldg(jb2 + k), jmx = __ldg(jb2 + M + k);
          none |= imn > jmx;
          all &= imx <= jmn;
          strict |= imx < jmn;
        }
        if (none) continue;
        if (all && strict) {
          na += nv;
          nb2 += nv;
          continue;
        }
      }
      const float imax = MODE == MODE_COUNT ? __ldg(a.blkmax + s0 / STREAM_BLK) : ldx<FUSED>(a.flmax + s0 / STREAM_BLK);
      const bool fast = (MODE == MODE_COUNT && !a.boxed ? (s0 / STREAM_BLK < bj) : true) && imax < jmin;
      for (int g0 = 0; g0 < nv; g0 += 32) {
        const int gn = min(32, nv - g0);
        if (a.boxed) {  // 32 i rows (their box) against this warp's 64 j rows
          const float* ib = (MODE == MODE_COUNT ? a.blkbox32 : a.flbox32) + (int64_t)((s0 + g0) / 32) * 2 * M;
          bool none = false, all = true, strict = false;
#pragma unroll
          for (int k = 0; k < M; ++k) {
            const float imn = ldx<FUSED>(ib + k), imx = ldx<FUSED>(ib + M + k);
            none |= imn > wjmx[k];
            all &= imx <= wjmn[k];
            strict |= imx < wjmn[k];
          }
          if (none) continue;
          if (all && strict) {
            na += gn;
            nb2 += gn;
            continue;
          }
        }
        // stage the group: lane l loads i row g0 + l (pads: +inf, never <= a finite row)
        {
          int src = -1;
          if (lane < gn) src = MODE == MODE_COUNT ? s0 + g0 + lane : ldx<FUSED>(a.fl + s0 + g0 + lane);
          __syncwarp();
#pragma unroll
          for (int k = 0; k < MP; ++k)
            sF[lane * MP + k] = (src >= 0 && k < M) ? __ldg(a.FS + (int64_t)src * M + k) : PINF;
          __syncwarp();
        }
        const int gn8 = (gn + 7) & ~7;
        // S-separated at the (32 i, 64 j) level: the <= chain suffices
        const bool fast32 = fast || (a.boxed && ldx<FUSED>((MODE == MODE_COUNT ? a.blkS32 : a.flS32) +
                                                           (int64_t)((s0 + g0) / 32) * 2 + 1) < wjS);
        if (fast32) {
          nfast += 2 * gn8;
          for (int i = 0; i < gn8; i += 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              float v[M];
#pragma unroll
              for (int k = 0; k < M; ++k) v[k] = sF[(i + u) * MP + k];
              Chain<M>::le_cnt(v, fa, ca);
              Chain<M>::le_cnt(v, fb, cb);
            }
          }
        } else {
          nfull += 2 * gn8;
          for (int i = 0; i < gn8; i += 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              float v[M];
#pragma unroll
              for (int k = 0; k < M; ++k) v[k] = sF[(i + u) * MP + k];
              Chain<M>::dom_cnt(v, fa, ca);
              Chain<M>::dom_cnt(v, fb, cb);
            }
          }
        }
      }
    }
    if (a.stats) {   // executed pairs, for the roofline (one atomic per warp and item)
      nfast = warp_sum(nfast);
      nfull = warp_sum(nfull);
      if (lane == 0) {
        if (nfast) atomicAdd(a.stats + (MODE == MODE_COUNT ? 0 : 2), nfast);
        if (nfull) atomicAdd(a.stats + (MODE == MODE_COUNT ? 1 : 3), nfull);
      }
    }
    const int ia = (int)ca + na, ib = (int)cb + nb2;
    if (ja < a.R && ia) atomicAdd(a.cnt + ja, MODE == MODE_COUNT ? ia : -ia);
    if (jb < a.R && ib) atomicAdd(a.cnt + jb, MODE == MODE_COUNT ? ib : -ib);
  }
}

template <int M, int MODE>
__global__ void __launch_bounds__(ST_THREADS) k_stream_tiles(StreamArgs a) {
  constexpr int MP = (M + 3) & ~3;
  __shared__ __align__(16) float sFw[(ST_THREADS / 32) * 32 * MP];
  tiles_run<M, MODE, false>(a, sFw, __ldcg(a.ctl + SC_ITEMS), MODE == MODE_DEC ? __ldcg(a.ctl + SC_FLN) : 0,
                            a.ctl + SC_WORK, 0);
}

// Owned unranked rows with no unranked dominator left -> local mask slice.
__global__ void k_stream_mark(StreamArgs a) {
  if (__ldcg(a.ctl + SC_DONE) != 0) return;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t)a.T * (STREAM_BLK / 32);
  if (gw >= nw) return;
  const int t = (int)(gw / (STREAM_BLK / 32)), w8 = (int)(gw % (STREAM_BLK / 32));
  const int p = owned_block(a, t) * STREAM_BLK + w8 * 32 + lane;
  const bool in = p < a.R && __ldcg(a.rank_pos + p) == MO_RANK_UNRANKED && __ldcg(a.cnt + p) == 0;
  const uint32_t word = __ballot_sync(MO_FULL, in);
  if (lane == 0) a.mask_local[gw] = word;
}

// Front k from the gathered mask: ranks, ordered front list, split decision.
__global__ void __launch_bounds__(APPLY_THREADS) k_stream_apply(StreamArgs a, int k) {
  __shared__ int sh[40];
  __shared__ float sMax[APPLY_THREADS / 32], sMin[APPLY_THREADS / 32];
  if (__ldcg(a.ctl + SC_DONE) != 0) return;  // set only after the last barrier below
  const int nb = nblocks(a.R);
  const int64_t N = (int64_t)nb * (STREAM_BLK / 32);
  auto word = [&](int64_t e) -> uint32_t {
    const int b = (int)(e / (STREAM_BLK / 32)), w8 = (int)(e % (STREAM_BLK / 32));
    return __ldcg(a.mask_full + ((int64_t)(b % a.G) * a.T + b / a.G) * (STREAM_BLK / 32) + w8);
  };
  const int fk = grid_scan(
      a.gc, N, [&](int64_t e) { return __popc(word(e)); },
      [&](int64_t e, int pre) {
        uint32_t wv = word(e);
        const int b = (int)(e / (STREAM_BLK / 32));
        const int base = (int)(e * 32);
        if (b % a.G == a.g) atomicSub(a.ucnt + b / a.G, __popc(wv));
        int r = pre;
        while (wv) {
          const int bit = __ffs(wv) - 1;
          wv &= wv - 1;
          a.fl[r++] = base + bit;
          a.rank_pos[base + bit] = k;
        }
      },
      sh);
  grid_sync(a.gc.bar);
  // max S per 256-entry block of the front list (fast-tile test of DEC)
  const int nq = (fk + STREAM_BLK - 1) / STREAM_BLK;
  for (int q = blockIdx.x; q < nq; q += gridDim.x) {
    const int e = q * STREAM_BLK + (int)threadIdx.x;
    const bool act = threadIdx.x < STREAM_BLK && e < fk;
    const int p = act ? __ldcg(a.fl + e) : 0;
    float v = act ? __ldg(a.SS + p) : -__int_as_float(0x7f800000);
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(MO_FULL, v, o));
    if ((threadIdx.x & 31) == 0) sMax[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      float mx = sMax[0];
      for (int w = 1; w < APPLY_THREADS / 32; ++w) mx = fmaxf(mx, sMax[w]);
      a.flmax[q] = mx;
    }
    __syncthreads();
    if (a.boxed) {
      {  // S range of every 32-entry group (the warp-level <= test of the DEC sweep)
        const float sv = act ? __ldg(a.SS + p) : 0.0f;
        float mn = act ? sv : __int_as_float(0x7f800000), mx = act ? sv : -__int_as_float(0x7f800000);
        for (int o = 16; o > 0; o >>= 1) {
          mn = fminf(mn, __shfl_xor_sync(MO_FULL, mn, o));
          mx = fmaxf(mx, __shfl_xor_sync(MO_FULL, mx, o));
        }
        if ((threadIdx.x & 31) == 0 && threadIdx.x < STREAM_BLK) {
          const int64_t q32 = (int64_t)q * (STREAM_BLK / 32) + (threadIdx.x >> 5);
          a.flS32[q32 * 2] = mn;
          a.flS32[q32 * 2 + 1] = mx;
        }
      }
      for (int k = 0; k < a.m; ++k) {
        const float f = act ? __ldg(a.FS + (int64_t)p * a.m + k) : 0.0f;
        float mn = act ? f : __int_as_float(0x7f800000), mx = act ? f : -__int_as_float(0x7f800000);
        for (int o = 16; o > 0; o >>= 1) {
          mn = fminf(mn, __shfl_xor_sync(MO_FULL, mn, o));
          mx = fmaxf(mx, __shfl_xor_sync(MO_FULL, mx, o));
        }
        if ((threadIdx.x & 31) == 0 && threadIdx.x < STREAM_BLK) {
          const int64_t q32 = (int64_t)q * (STREAM_BLK / 32) + (threadIdx.x >> 5);
          a.flbox32[q32 * 2 * a.m + k] = mn;
          a.flbox32[q32 * 2 * a.m + a.m + k] = mx;
        }
        if ((threadIdx.x & 31) == 0) {
          sMax[threadIdx.x >> 5] = mx;
          sMin[threadIdx.x >> 5] = mn;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          float a0 = sMin[0], a1 = sMax[0];
          for (int w = 1; w < APPLY_THREADS / 32; ++w) {
            a0 = fminf(a0, sMin[w]);
            a1 = fmaxf(a1, sMax[w]);
          }
          a.flbox[(int64_t)q * 2 * a.m + k] = a0;
          a.flbox[(int64_t)q * 2 * a.m + a.m + k] = a1;
        }
        __syncthreads();
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t sel = __ldcg(a.ctl + SC_CUM);
    const int64_t cum = sel + fk;
    a.ctl[SC_CUM] = (int)cum;
    a.ctl[SC_FLN] = fk;
    if (cum >= a.stop_at || fk == 0) {
      a.info[MO_INFO_L] = k;
      a.info[MO_INFO_SELECTED] = (int)sel;
      a.info[MO_INFO_K] = (int)(a.stop_at - sel);
      a.info[MO_INFO_FL_SIZE] = fk;
      a.info[MO_INFO_SKIPPED] = (sel + fk == a.stop_at) ? 1 : 0;
      a.info[MO_INFO_ERROR] = (cum < a.stop_at) ? MO_ERR_INFEASIBLE : 0;
      if (cum < a.stop_at && a.info[MO_INFO_ERROR_FIRST] == 0) a.info[MO_INFO_ERROR_FIRST] = MO_ERR_INFEASIBLE;
      __threadfence();
      a.info[MO_INFO_NFRONTS] = k + 1;
      a.ctl[SC_DONE] = k + 1;
    }
  }
}

__global__ void k_stream_end(StreamArgs a) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  for (int p = gt; p < a.R; p += gs) {
    const int r = __ldcg(a.rank_pos + p);
    a.ranks[__ldg(a.perm + p)] = r == MO_RANK_UNRANKED ? MO_RANK_DROPPED : r;
  }
}

// ------------------------------------------------- single-GPU fused sweep loop
//
// k_stream_fused: the whole streamed sort of one generation (G = 1) in one
// cooperative launch -- reset, dominator counts, front 0, then per front:
// ordered front list from the mask (grid scan), chunk ranges / boxes, the
// DEC plan (per-block item counts + grid scan), the DEC sweep, the next mask
// -- with grid barriers instead of host round trips, so a generation is one
// graph-capturable mo_step.  Work items are pulled from one counter that
// keeps counting across sweeps: every CTA overshoots each sweep exactly once,
// so sweep s starts at base_s = sum_{r<s} (items_r + gridDim.x).

// grid_scan that calls emit(e, prefix) for EVERY e (zero values included).
template <class ValueF, class EmitF>
__device__ int grid_scan_all(GridCtx& g, int64_t N, ValueF value, EmitF emit, int* sh) {
  const int G = gridDim.x, b = blockIdx.x;
  int* part = g.part + g.parity * (G + 1);
  g.parity ^= 1;
  const int64_t chunk = ceil_div(N, (int64_t)G);
  const int64_t lo = min((int64_t)b * chunk, N), hi = min(lo + chunk, N);
  int cnt = 0;
  for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) cnt += value(e);
  int tot;
  block_excl_scan(cnt, sh, &tot);
  if (threadIdx.x == 0) part[b] = tot;
  grid_sync(g.bar);
  int pre = 0, all = 0;
  for (int q = threadIdx.x; q < G; q += blockDim.x) {
    const int v = __ldcg(part + q);
    all += v;
    if (q < b) pre += v;
  }
  int offset, total;
  block_excl_scan(pre, sh, &offset);
  block_excl_scan(all, sh, &total);
  for (int64_t base = lo; base < hi; base += blockDim.x) {
    const int64_t e = base + threadIdx.x;
    const int v = (e < hi) ? value(e) : 0;
    int t;
    const int p = block_excl_scan(v, sh, &t);
    if (e < hi) emit(e, offset + p);
    offset += t;
  }
  return total;
}

// plan[t] = exclusive prefix of the items of owned block t; returns the total (all CTAs).
__device__ __noinline__ int plan_all(const StreamArgs& a, GridCtx& g, int mode, int fln, int* sh) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  if (a.boxed) {   // uniform items per block, no plan (the caller's barrier publishes earlier writes)
    grid_sync(g.bar);
    return a.T * (mode == MODE_COUNT ? boxed_items_per_block<MODE_COUNT>(nblocks(a.R), fln)
                                     : boxed_items_per_block<MODE_DEC>(nblocks(a.R), fln));
  }
  for (int t = gt; t < a.T; t += gs)
    a.plan[t] = mode == MODE_COUNT ? block_items<MODE_COUNT>(a, t, fln) : block_items<MODE_DEC>(a, t, fln);
  grid_sync(g.bar);
  const int total = grid_scan_all(
      g, a.T, [&](int64_t t) { return __ldcg(a.plan + t); }, [&](int64_t t, int pre) { a.plan[t] = pre; }, sh);
  grid_sync(g.bar);   // every prefix written before any CTA searches the plan
  return total;
}

__device__ void mark_all(const StreamArgs& a) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)a.T * (STREAM_BLK / 32);
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t gw = w0; gw < nw; gw += ws) {
    const int t = (int)(gw / (STREAM_BLK / 32)), w8 = (int)(gw % (STREAM_BLK / 32));
    const int p = owned_block(a, t) * STREAM_BLK + w8 * 32 + lane;
    const bool in = p < a.R && __ldcg(a.rank_pos + p) == MO_RANK_UNRANKED && __ldcg(a.cnt + p) == 0;
    const uint32_t word = __ballot_sync(MO_FULL, in);
    if (lane == 0) a.mask_local[gw] = word;
  }
}

// max S and (boxed) bounding boxes of every 256- and 32-entry chunk of fl[0, fk)
template <int M>
__device__ void chunk_boxes(const StreamArgs& a, int fk, float* sRedMin, float* sRedMax) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int bd = blockDim.x, nw = bd >> 5;
  const int nq = (fk + STREAM_BLK - 1) / STREAM_BLK;
  for (int q = blockIdx.x; q < nq; q += gridDim.x) {
    int p[2];
    bool act[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {   // chunk entry tid + bd*u: warp w covers the 32-group w + nw*u
      const int el = tid + bd * u, e = q * STREAM_BLK + el;
      act[u] = el < STREAM_BLK && e < fk;
      p[u] = act[u] ? __ldcg(a.fl + e) : 0;
    }
    for (int k = -1; k < (a.boxed ? M : 0); ++k) {
      float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        float gmn = __int_as_float(0x7f800000), gmx = -__int_as_float(0x7f800000);
        if (act[u]) {
          const float v = k < 0 ? __ldg(a.SS + p[u]) : __ldg(a.FS + (int64_t)p[u] * M + k);
          gmn = v;
          gmx = v;
        }
        for (int o = 16; o > 0; o >>= 1) {
          gmn = fminf(gmn, __shfl_xor_sync(MO_FULL, gmn, o));
          gmx = fmaxf(gmx, __shfl_xor_sync(MO_FULL, gmx, o));
        }
        if (lane == 0 && wid + nw * u < STREAM_BLK / 32) {
          const int64_t q32 = (int64_t)q * (STREAM_BLK / 32) + wid + nw * u;
          if (k >= 0) {
            a.flbox32[q32 * 2 * M + k] = gmn;
            a.flbox32[q32 * 2 * M + M + k] = gmx;
          } else if (a.boxed) {
            a.flS32[q32 * 2] = gmn;
            a.flS32[q32 * 2 + 1] = gmx;
          }
        }
        mn = fminf(mn, gmn);
        mx = fmaxf(mx, gmx);
      }
      if (lane == 0) {
        sRedMin[wid] = mn;
        sRedMax[wid] = mx;
      }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < nw; ++w) {
          mn = fminf(mn, sRedMin[w]);
          mx = fmaxf(mx, sRedMax[w]);
        }
        if (k < 0) {
          a.flmax[q] = mx;
        } else {
          a.flbox[(int64_t)q * 2 * M + k] = mn;
          a.flbox[(int64_t)q * 2 * M + M + k] = mx;
        }
      }
      __syncthreads();
    }
  }
}

__device__ __noinline__ int apply_front_local(const StreamArgs& a, GridCtx& g, int64_t N, int k, int* sh) {
  return grid_scan(
      g, N, [&](int64_t e) { return __popc(__ldcg(a.mask_local + e)); },
      [&](int64_t e, int pre) {
        uint32_t wv = __ldcg(a.mask_local + e);
        const int base_p = (int)(e * 32);
        atomicSub(a.ucnt + (int)(e / (STREAM_BLK / 32)), __popc(wv));
        int r = pre;
        while (wv) {
          const int bit = __ffs(wv) - 1;
          wv &= wv - 1;
          a.fl[r++] = base_p + bit;
          a.rank_pos[base_p + bit] = k;
        }
      },
      sh);
}

template <int M>
__global__ void __launch_bounds__(FUSED_THREADS, 2) k_stream_fused(StreamArgs a) {
  constexpr int MP = (M + 3) & ~3;
  __shared__ __align__(16) float sFw[(FUSED_THREADS / 32) * 32 * MP];
  __shared__ int sh[40];
  __shared__ float sRedMin[FUSED_THREADS / 32], sRedMax[FUSED_THREADS / 32];
  GridCtx g = a.gc;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  const int R = a.R;
  // reset
  for (int p = gt; p < R; p += gs) {
    a.rank_pos[p] = MO_RANK_UNRANKED;
    a.cnt[p] = 0;
  }
  for (int t = gt; t < a.T; t += gs) {
    const int b = owned_block(a, t);
    a.ucnt[t] = max(0, min(R, (b + 1) * STREAM_BLK) - b * STREAM_BLK);
  }
  if (gt < MO_INFO_COUNT && gt != MO_INFO_ASSOC_FALLBACK) a.info[gt] = 0;
  if (gt == 0) a.ctl[SC_WORK] = 0;
  if (a.stats && gt < 4) a.stats[gt] = 0;
  grid_sync(g.bar);
  // dominator counts, front 0
  int base = 0;
  int items = plan_all(a, g, MODE_COUNT, 0, sh);
  tiles_run<M, MODE_COUNT, true>(a, sFw, items, 0, a.ctl + SC_WORK, base);
  base += 4 * items + (int)gridDim.x * (FUSED_THREADS / 32);   // every warp overshoots once
  grid_sync(g.bar);
  mark_all(a);
  grid_sync(g.bar);
  const int nb = nblocks(R);
  const int64_t N = (int64_t)nb * (STREAM_BLK / 32);
  int64_t cum = 0;
  for (int k = 0;; ++k) {
    // front k: ordered list, ranks, unranked counts per block (mask_full aliases mask_local, G = 1)
    const int fk = apply_front_local(a, g, N, k, sh);
    const int64_t sel = cum;
    cum += fk;
    if (cum >= a.stop_at || fk == 0) {
      if (gt == 0) {
        a.info[MO_INFO_L] = k;
        a.info[MO_INFO_SELECTED] = (int)sel;
        a.info[MO_INFO_K] = (int)(a.stop_at - sel);
        a.info[MO_INFO_FL_SIZE] = fk;
        a.info[MO_INFO_SKIPPED] = (sel + fk == a.stop_at) ? 1 : 0;
        a.info[MO_INFO_ERROR] = (cum < a.stop_at) ? MO_ERR_INFEASIBLE : 0;
      if (cum < a.stop_at && a.info[MO_INFO_ERROR_FIRST] == 0) a.info[MO_INFO_ERROR_FIRST] = MO_ERR_INFEASIBLE;
        a.info[MO_INFO_NFRONTS] = k + 1;
      }
      break;
    }
    grid_sync(g.bar);            // fl / rank_pos / ucnt of front k visible
    chunk_boxes<M>(a, fk, sRedMin, sRedMax);
    items = plan_all(a, g, MODE_DEC, fk, sh);  // (its first barrier also publishes the chunk boxes)
    tiles_run<M, MODE_DEC, true>(a, sFw, items, fk, a.ctl + SC_WORK, base);
    base += 4 * items + (int)gridDim.x * (FUSED_THREADS / 32);
    grid_sync(g.bar);
    mark_all(a);
    grid_sync(g.bar);
  }
  grid_sync(g.bar);              // every rank_pos write of the last front done
  for (int p = gt; p < R; p += gs) {
    const int r = __ldcg(a.rank_pos + p);
    a.ranks[__ldg(a.perm + p)] = r == MO_RANK_UNRANKED ? MO_RANK_DROPPED : r;
  }
}

// ------------------------------------------------------------ Morton presort
//
// Boxed mode position space.  P0 per-coordinate min / max (ordered-uint
// atomics) and row sums S; P1 Morton key of the quantised objectives
// (b = 30 / m bits per coordinate, interleaved most significant first) and
// row ids; P2 four stable 8-bit radix passes (ties keep row order, so every
// shard derives the same positions); P3 gather FS / SS / perm; P4 per-block
// S range and bounding box.
constexpr int MORTON_THREADS = 512;

__global__ void __launch_bounds__(MORTON_THREADS) k_presort_morton(MortonArgs a) {
  __shared__ int sh[40];
  __shared__ int sWcnt[(MORTON_THREADS / 32) * 256], sRun[256], sOff[256];
  __shared__ unsigned sMn[16], sMx[16];
  __shared__ float sRed[2][MORTON_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31;
  const int gtid = blockIdx.x * blockDim.x + tid, gthreads = gridDim.x * blockDim.x;
  const int R = a.R, m = a.m;
  if (tid < 16) {
    sMn[tid] = 0xffffffffu;
    sMx[tid] = 0u;
  }
  __syncthreads();
  for (int k = 0; k < m; ++k) {
    unsigned mn = 0xffffffffu, mx = 0u;
    for (int i = gtid; i < R; i += gthreads) {
      const unsigned o = f2ord(a.F[(int64_t)i * m + k]);
      mn = min(mn, o);
      mx = max(mx, o);
    }
    mn = warp_min_u32(mn);
    mx = warp_max_u32(mx);
    if (lane == 0) {
      atomicMin(&sMn[k], mn);
      atomicMax(&sMx[k], mx);
    }
  }
  __syncthreads();
  if (tid < m) {
    atomicMin(&a.cbox[tid], sMn[tid]);
    atomicMax(&a.cbox[16 + tid], sMx[tid]);
  }
  grid_sync(a.g.bar);
  // P1: Morton keys
  const int bits = 30 / m;
  const float levels = (float)((1u << bits) - 1u);
  float lo[16], sc[16];
  for (int k = 0; k < m; ++k) {
    lo[k] = ord2f(__ldcg(a.cbox + k));
    const float hi = ord2f(__ldcg(a.cbox + 16 + k));
    sc[k] = hi > lo[k] ? levels / (hi - lo[k]) : 0.0f;
  }
  for (int i = gtid; i < R; i += gthreads) {
    uint32_t q[16];
    for (int k = 0; k < m; ++k) {
      float v = (a.F[(int64_t)i * m + k] - lo[k]) * sc[k];
      v = fminf(fmaxf(v, 0.0f), levels);
      q[k] = (uint32_t)v;
    }
    uint32_t key = 0;
    for (int b = bits - 1; b >= 0; --b)
      for (int k = 0; k < m; ++k) key = (key << 1) | ((q[k] >> b) & 1u);
    a.keyA[i] = key;
    a.valA[i] = i;
  }
  grid_sync(a.g.bar);
  // P2: stable radix sort by key (4 x 8 bits), result back in keyA / valA
  grid_radix_pass(a.g, R, 0, a.keyA, a.valA, a.tkey, a.tval, sWcnt, sRun, sOff, sh);
  grid_radix_pass(a.g, R, 8, a.tkey, a.tval, a.keyA, a.valA, sWcnt, sRun, sOff, sh);
  grid_radix_pass(a.g, R, 16, a.keyA, a.valA, a.tkey, a.tval, sWcnt, sRun, sOff, sh);
  grid_radix_pass(a.g, R, 24, a.tkey, a.tval, a.keyA, a.valA, sWcnt, sRun, sOff, sh);
  // P3: gather
  for (int p = gtid; p < R; p += gthreads) {
    const int i = __ldcg(a.valA + p);
    a.perm[p] = i;
    const float* f = a.F + (int64_t)i * m;
    float s = f[0];
    a.FS[(int64_t)p * m] = __fadd_rn(f[0], 0.0f);  // -0 -> +0 (canonical zero in the sorted rows)
    for (int k = 1; k < m; ++k) {
      s = __fadd_rn(s, f[k]);
      a.FS[(int64_t)p * m + k] = __fadd_rn(f[k], 0.0f);
    }
    a.SS[p] = s;
  }
  grid_sync(a.g.bar);
  // P4: per-block S range and bounding box
  const int nblk = (R + STREAM_BLK - 1) / STREAM_BLK;
  for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
    const int p = b * STREAM_BLK + tid;
    const bool act = tid < STREAM_BLK && p < R;
    for (int k = -1; k < m; ++k) {
      float v = 0.0f;
      if (act) v = k < 0 ? __ldcg(a.SS + p) : __ldcg(a.FS + (int64_t)p * m + k);
      float mn = act ? v : __int_as_float(0x7f800000), mx = act ? v : -__int_as_float(0x7f800000);
      for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(MO_FULL, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(MO_FULL, mx, o));
      }
      if (lane == 0 && tid < STREAM_BLK) {
        const int64_t q32 = (int64_t)b * (STREAM_BLK / 32) + (tid >> 5);
        if (k >= 0) {
          a.blkbox32[q32 * 2 * m + k] = mn;
          a.blkbox32[q32 * 2 * m + m + k] = mx;
        } else {
          a.blkS32[q32 * 2] = mn;
          a.blkS32[q32 * 2 + 1] = mx;
        }
      }
      if (lane == 0) {
        sRed[0][tid >> 5] = mn;
        sRed[1][tid >> 5] = mx;
      }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < MORTON_THREADS / 32; ++w) {
          mn = fminf(mn, sRed[0][w]);
          mx = fmaxf(mx, sRed[1][w]);
        }
        if (k < 0) {
          a.blkmin[b] = mn;
          a.blkmax[b] = mx;
        } else {
          a.blkbox[(int64_t)b * 2 * m + k] = mn;
          a.blkbox[(int64_t)b * 2 * m + m + k] = mx;
        }
      }
      __syncthreads();
    }
  }
}

int launch_presort_morton(const MortonArgs& a, cudaStream_t s) {
  static int maxb = 0;
  if (!maxb) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_presort_morton, MORTON_THREADS, 0);
    maxb = sms * (per > 0 ? 1 : 1);
  }
  if (a.R < 1 || a.m < 1 || a.m > 16) return MO_ERR_PARAM;
  int blocks = (int)ceil_div(a.R, MORTON_THREADS * 4);
  if (blocks > maxb) blocks = maxb;
  if (blocks < 1) blocks = 1;
  if (cudaMemsetAsync(a.g.bar, 0, 2 * sizeof(unsigned), s) != cudaSuccess) return MO_ERR_CUDA;
  if (cudaMemsetAsync(a.cbox, 0xff, 16 * sizeof(unsigned), s) != cudaSuccess) return MO_ERR_CUDA;
  if (cudaMemsetAsync(a.cbox + 16, 0, 16 * sizeof(unsigned), s) != cudaSuccess) return MO_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(MORTON_THREADS);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, k_presort_morton, a) != cudaSuccess) return MO_ERR_CUDA;
  MO_CHECK_LAUNCH();
  return MO_OK;
}

// ------------------------------------------------------------- launchers

template <int MODE>
static int launch_tiles(const StreamArgs& a, cudaStream_t s) {
  static int per[17][2];
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  switch (a.m) {
#define MO_ST_CASE(MM)                                                                          \
  case MM: {                                                                                    \
    if (!per[MM][MODE]) {                                                                       \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per[MM][MODE], k_stream_tiles<MM, MODE>,   \
                                                    ST_THREADS, 0);                             \
      if (per[MM][MODE] < 1) per[MM][MODE] = 1;                                                 \
    }                                                                                           \
    k_stream_tiles<MM, MODE><<<sms * per[MM][MODE], ST_THREADS, 0, s>>>(a);                     \
    break;                                                                                      \
  }
    MO_ST_CASE(2)
    MO_ST_CASE(3)
    MO_ST_CASE(4)
    MO_ST_CASE(5)
    MO_ST_CASE(6)
    MO_ST_CASE(7)
    MO_ST_CASE(8)
    MO_ST_CASE(9)
    MO_ST_CASE(10)
    MO_ST_CASE(11)
    MO_ST_CASE(12)
    MO_ST_CASE(13)
    MO_ST_CASE(14)
    MO_ST_CASE(15)
    MO_ST_CASE(16)
#undef MO_ST_CASE
    default:
      return MO_ERR_PARAM;
  }
  MO_CHECK_LAUNCH();
  return MO_OK;
}

static int mark_launch(const StreamArgs& a, cudaStream_t s) {
  const int64_t threads = (int64_t)a.T * STREAM_BLK;
  k_stream_mark<<<(unsigned)ceil_div(threads, 256), 256, 0, s>>>(a);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int launch_stream_begin(StreamArgs a, cudaStream_t s) {
  if (a.R < 1 || a.G < 1 || a.g < 0 || a.g >= a.G || a.m < 2 || a.m > 16) return MO_ERR_PARAM;
  int64_t rb = ceil_div(a.R > a.T ? a.R : a.T, 256);
  k_stream_reset<<<(unsigned)(rb > 4096 ? 4096 : rb), 256, 0, s>>>(a);
  MO_CHECK_LAUNCH();
  k_stream_plan<MODE_COUNT><<<1, PLAN_THREADS, 0, s>>>(a);
  MO_CHECK_LAUNCH();
  MO_TRY(launch_tiles<MODE_COUNT>(a, s));
  return mark_launch(a, s);
}

int launch_stream_front(StreamArgs a, int k, cudaStream_t s) {
  static int blocks = 0;
  if (!blocks) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_stream_apply, APPLY_THREADS, 0);
    blocks = sms * (per > 1 ? 1 : (per > 0 ? per : 1));
  }
  if (cudaMemsetAsync(a.gc.bar, 0, 2 * sizeof(unsigned), s) != cudaSuccess) return MO_ERR_CUDA;
  a.gc.parity = 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(APPLY_THREADS);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, k_stream_apply, a, k) != cudaSuccess) return MO_ERR_CUDA;
  MO_CHECK_LAUNCH();
  k_stream_plan<MODE_DEC><<<1, PLAN_THREADS, 0, s>>>(a);
  MO_CHECK_LAUNCH();
  MO_TRY(launch_tiles<MODE_DEC>(a, s));
  return mark_launch(a, s);
}

int launch_stream_fused(StreamArgs a, cudaStream_t s) {
  if (a.G != 1) return MO_ERR_PARAM;
  static int blocks[17];
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaMemsetAsync(a.gc.bar, 0, 2 * sizeof(unsigned), s) != cudaSuccess) return MO_ERR_CUDA;
  a.gc.parity = 0;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(FUSED_THREADS);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaSuccess;
  switch (a.m) {
#define MO_SF_CASE(MM)                                                                            \
  case MM: {                                                                                      \
    if (!blocks[MM]) {                                                                            \
      int per = 0;                                                                                \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_stream_fused<MM>, FUSED_THREADS, 0);     \
      per = per > 2 ? 2 : (per < 1 ? 1 : per);   /* few barrier participants */        \
      blocks[MM] = sms * per;                                                                     \
    }                                                                                             \
    cfg.gridDim = dim3(blocks[MM]);                                                               \
    e = cudaLaunchKernelEx(&cfg, k_stream_fused<MM>, a);                                          \
    break;                                                                                        \
  }
    MO_SF_CASE(2)
    MO_SF_CASE(3)
    MO_SF_CASE(4)
    MO_SF_CASE(5)
    MO_SF_CASE(6)
    MO_SF_CASE(7)
    MO_SF_CASE(8)
    MO_SF_CASE(9)
    MO_SF_CASE(10)
    MO_SF_CASE(11)
    MO_SF_CASE(12)
    MO_SF_CASE(13)
    MO_SF_CASE(14)
    MO_SF_CASE(15)
    MO_SF_CASE(16)
#undef MO_SF_CASE
    default:
      return MO_ERR_PARAM;
  }
  if (e != cudaSuccess) return MO_ERR_CUDA;
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int launch_stream_end(StreamArgs a, cudaStream_t s) {
  unsigned blocks = (unsigned)ceil_div(a.R, 256);
  if (blocks > 4096) blocks = 4096;
  k_stream_end<<<blocks, 256, 0, s>>>(a);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

}  // namespace mo
