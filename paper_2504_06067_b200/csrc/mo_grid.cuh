// Grid-wide primitives for persistent cooperative kernels: chunked stable
// scans/compactions and a stable LSD radix-sort pass.  Every block of the grid
// must call these with identical arguments (they contain grid barriers).
#pragma once
#include "mo_common.cuh"

namespace mo {

struct GridCtx {
  unsigned* bar;  // {count, gen}
  int* part;      // >= 2 * (gridDim.x + 1) ints: double-buffered block partials
  int* hist;      // >= 256 * gridDim.x ints (radix)
  int parity;     // which half of `part` the next grid_scan uses (same on every block)
};

// Stable exclusive scan of value(e) over e in [0, N) in ascending e.  Calls
// emit(e, prefix) for every e with value(e) != 0.  Returns the grand total.
// `sh` must hold >= 34 ints of shared memory.  One internal grid barrier.
template <class ValueF, class EmitF>
__device__ int grid_scan(GridCtx& g, int64_t N, ValueF value, EmitF emit, int* sh) {
  const int G = gridDim.x, b = blockIdx.x;
  // alternate halves of `part`: a fast block may enter the next scan and write
  // its partial while a slow block still reads this scan's partials
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
  // offset = sum of parts of earlier blocks; total = sum of all parts
  int pre = 0, all = 0;
  for (int q = threadIdx.x; q < G; q += blockDim.x) {
    int v = __ldcg(part + q);
    all += v;
    if (q < b) pre += v;
  }
  int dummy;
  int s1 = block_excl_scan(pre, sh, &dummy);
  (void)s1;
  int offset = dummy;
  block_excl_scan(all, sh, &dummy);
  int total = dummy;
  for (int64_t base = lo; base < hi; base += blockDim.x) {
    int64_t e = base + threadIdx.x;
    int v = (e < hi) ? value(e) : 0;
    int t;
    int p = block_excl_scan(v, sh, &t);
    if (v) emit(e, offset + p);
    offset += t;
  }
  return total;
}

// One stable LSD radix pass (8-bit digit at `shift`) of N (key, val) pairs
// from (kin, vin) to (kout, vout).  Block b owns a contiguous chunk; warp w of
// the block owns a contiguous sub-segment of that chunk and scatters it in
// order, 32 keys at a time, ranking equal digits with __match_any_sync against
// its own running counters -- no block barrier inside the scatter.  Shared
// memory: `wcnt` >= (blockDim/32)*256 ints, `off` >= 256 ints.  Two grid
// barriers per pass.
__device__ inline void grid_radix_pass(GridCtx& g, int N, int shift, const uint32_t* kin, const int* vin,
                                       uint32_t* kout, int* vout, int* wcnt, int* run, int* off, int* sh) {
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nw = blockDim.x >> 5;
  const int chunk = (int)ceil_div(N, G);
  const int lo = min(b * chunk, N), hi = min(lo + chunk, N);
  const int seg = (int)ceil_div(hi - lo, nw);
  const int wlo = min(lo + wid * seg, hi), whi = min(wlo + seg, hi);
  int* my = wcnt + wid * 256;
  // 1. per-warp digit histogram of its sub-segment
  for (int q = lane; q < 256; q += 32) my[q] = 0;
  __syncwarp();
  for (int base = wlo; base < whi; base += 32) {
    const int e = base + lane;
    const bool act = e < whi;
    const int dg = act ? (int)((__ldcg(kin + e) >> shift) & 255u) : 256 + lane;
    const unsigned peers = __match_any_sync(MO_FULL, dg);
    if (act && (peers & ((1u << lane) - 1u)) == 0) my[dg] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // block histogram -> hist[d * G + b]
  for (int d = tid; d < 256; d += blockDim.x) {
    int t = 0;
    for (int q = 0; q < nw; ++q) t += wcnt[q * 256 + d];
    g.hist[d * G + b] = t;
  }
  grid_sync(g.bar);
  // 2. base of (digit d, this block) = totals of smaller digits + earlier blocks of digit d
  for (int d = tid; d < 256; d += blockDim.x) {
    int pre = 0, tot = 0;
    for (int q = 0; q < G; ++q) {
      int v = __ldcg(g.hist + d * G + q);
      tot += v;
      if (q < b) pre += v;
    }
    off[d] = pre;
    run[d] = tot;
  }
  __syncthreads();
  if (tid < 32) {  // exclusive scan of the 256 digit totals by one warp (8 per lane)
    int v[8], s = 0;
    for (int q = 0; q < 8; ++q) {
      v[q] = run[lane * 8 + q];
      s += v[q];
    }
    int x = s;
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(MO_FULL, x, o);
      if (lane >= o) x += t;
    }
    int ex = x - s;
    for (int q = 0; q < 8; ++q) {
      off[lane * 8 + q] += ex;
      ex += v[q];
    }
  }
  __syncthreads();
  // per-warp running base: off[d] + counts of earlier warps of this block
  for (int d = tid; d < 256; d += blockDim.x) {
    int r = off[d];
    for (int q = 0; q < nw; ++q) {
      const int c = wcnt[q * 256 + d];
      wcnt[q * 256 + d] = r;
      r += c;
    }
  }
  __syncthreads();
  // 3. stable scatter of the warp's sub-segment
  for (int base = wlo; base < whi; base += 32) {
    const int e = base + lane;
    const bool act = e < whi;
    const uint32_t key = act ? __ldcg(kin + e) : 0u;
    const int val = act ? __ldcg(vin + e) : 0;
    const int dg = act ? (int)((key >> shift) & 255u) : 256 + lane;
    const unsigned peers = __match_any_sync(MO_FULL, dg);
    const unsigned below = peers & ((1u << lane) - 1u);
    if (act) {
      const int pos = my[dg] + __popc(below);
      kout[pos] = key;
      vout[pos] = val;
    }
    __syncwarp();
    if (act && below == 0) my[dg] += __popc(peers);
    __syncwarp();
  }
  grid_sync(g.bar);
  (void)sh;
}

}  // namespace mo
