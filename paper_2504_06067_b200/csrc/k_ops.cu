// Op-level entry points of the reference's per-op API -- batchcore, niche
// and variation -- each a short chain of small kernels.
//
// These are NOT the engine hot path: mo_step fuses the same stages (k_vary_eval, k_assoc_final,
// k_select).  They exist so that a caller of the reference's per-op functions finds them on the
// device with the reference's argument meaning and output order, and so that SPEC.md's worked
// examples can be run through the GPU (tests/test_gpu_ops.py).  Index/count outputs are int64 and
// follow the oracle's order exactly (oracle/manyobj_ref/niche.py:157-278).  Scans and sorts use CUB
// (CUDA toolkit headers); the caller sizes the workspace with mo_ops_workspace_bytes.
#include <cub/cub.cuh>

#include "mo_common.cuh"
#include "mo_rng.cuh"
#include "mo_variation.cuh"

namespace mo {

constexpr int OPS_THREADS = 256;
constexpr int64_t I64_INF = 0x7fffffff;                  // SPEC "infinity" count marker (2^31 - 1)

static unsigned ops_blocks(int64_t n) {
  int64_t b = ceil_div(n > 0 ? n : 1, OPS_THREADS);
  return (unsigned)(b < 4096 ? b : 4096);
}
#define MO_GRID_LOOP(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// ------------------------------------------------------------------ batchcore

__global__ void k_step_mask(const double* x, int64_t n, int8_t* out) {
  MO_GRID_LOOP(i, n) out[i] = x[i] > 0.0 ? 1 : 0;
}

struct ArgMin {
  double v;
  int64_t i;   // -1: no valid slot
};
__device__ __forceinline__ ArgMin argmin_better(ArgMin a, ArgMin b) {
  if (a.i < 0) return b;
  if (b.i < 0) return a;
  return (b.v < a.v || (b.v == a.v && b.i < a.i)) ? b : a;
}
__device__ ArgMin block_argmin(ArgMin x) {
  __shared__ double sv[32];
  __shared__ long long si[32];
  for (int o = 16; o > 0; o >>= 1) {
    ArgMin y{__shfl_xor_sync(MO_FULL, x.v, o), (int64_t)__shfl_xor_sync(MO_FULL, (long long)x.i, o)};
    x = argmin_better(x, y);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    sv[wid] = x.v;
    si[wid] = x.i;
  }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    x = lane < nw ? ArgMin{sv[lane], (int64_t)si[lane]} : ArgMin{0.0, -1};
    for (int o = 16; o > 0; o >>= 1) {
      ArgMin y{__shfl_xor_sync(MO_FULL, x.v, o), (int64_t)__shfl_xor_sync(MO_FULL, (long long)x.i, o)};
      x = argmin_better(x, y);
    }
  }
  return x;   // valid in warp 0
}

__global__ void k_argmin_partial(const double* v, const uint8_t* valid, int64_t n, ArgMin* part) {
  ArgMin x{0.0, -1};
  MO_GRID_LOOP(i, n) {
    if (valid && !valid[i]) continue;
    x = argmin_better(x, ArgMin{v[i], i});
  }
  x = block_argmin(x);
  if (threadIdx.x == 0) part[blockIdx.x] = x;
}
__global__ void k_argmin_final(const ArgMin* part, int np, int64_t* out) {
  ArgMin x{0.0, -1};
  for (int b = threadIdx.x; b < np; b += blockDim.x) x = argmin_better(x, part[b]);
  x = block_argmin(x);
  if (threadIdx.x == 0) *out = x.i;
}

__global__ void k_fill_i64(int64_t* p, int64_t n, int64_t v) {
  MO_GRID_LOOP(i, n) p[i] = v;
}

__global__ void k_segment_count(const int64_t* labels, const uint8_t* valid, int64_t n, int64_t segments,
                                unsigned long long* counts, int* status) {
  MO_GRID_LOOP(i, n) {
    if (valid && !valid[i]) continue;
    const int64_t b = labels[i];
    if (b < 0 || b >= segments) {
      atomicExch(status, MO_ERR_BOUNDS);
      continue;
    }
    atomicAdd(counts + b, 1ull);
  }
}

// -------------------------------------------------------------------- niche

// associate(D, valid): one warp per row, first minimum (lowest column) -- oracle niche.py:157
__global__ void k_associate_matrix(const double* D, const uint8_t* valid, int64_t R, int64_t w, int64_t* pi,
                                   double* d) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < R; r += warps) {
    if (valid && !valid[r]) {
      if (lane == 0) {
        pi[r] = -1;
        d[r] = __longlong_as_double(0x7ff8000000000000ll);
      }
      continue;
    }
    ArgMin x{0.0, -1};
    for (int64_t j = lane; j < w; j += 32) x = argmin_better(x, ArgMin{D[r * w + j], j});
    for (int o = 16; o > 0; o >>= 1) {
      ArgMin y{__shfl_xor_sync(MO_FULL, x.v, o), (int64_t)__shfl_xor_sync(MO_FULL, (long long)x.i, o)};
      x = argmin_better(x, y);
    }
    if (lane == 0) {
      pi[r] = x.i;
      d[r] = x.v;
    }
  }
}

// niche_counts(pi, ranks, l, w): rho over rank < l (l > 0), rho' over rank == l, rho = INF where
// rho' == 0 -- oracle niche.py:200
__global__ void k_niche_count(const int64_t* pi, const int64_t* ranks, int64_t R, int64_t l, int64_t w,
                              unsigned long long* rho, unsigned long long* rho_p) {
  MO_GRID_LOOP(i, R) {
    const int64_t r = ranks[i], j = pi[i];
    if (j < 0 || j >= w) continue;
    if (r == l) atomicAdd(rho_p + j, 1ull);
    else if (l > 0 && r < l) atomicAdd(rho + j, 1ull);
  }
}
__global__ void k_niche_count_finish(int64_t* rho, const int64_t* rho_p, int64_t w) {
  MO_GRID_LOOP(j, w) if (rho_p[j] == 0) rho[j] = I64_INF;
}

// nearest_selection: per empty point (rho == 0) the F_l candidate with the smallest (d, shuffled
// position) -- oracle niche.py:218
__global__ void k_near_keys(const int64_t* pi, const float* d, const int64_t* ranks, const int64_t* rho,
                            const int64_t* pos_pop, int64_t R, int64_t l, int64_t w, unsigned long long* keys) {
  MO_GRID_LOOP(i, R) {
    if (ranks[i] != l) continue;
    const int64_t j = pi[i];
    if (j < 0 || j >= w || rho[j] != 0) continue;
    const unsigned long long key = ((unsigned long long)f2ord(d[i] + 0.0f) << 32) | (uint32_t)pos_pop[i];
    atomicMin(keys + j, key);
  }
}
__global__ void k_near_rows(const int64_t* pi, const float* d, const int64_t* ranks, const int64_t* rho,
                            const int64_t* pos_pop, int64_t R, int64_t l, int64_t w,
                            const unsigned long long* keys, int64_t* chosen) {
  MO_GRID_LOOP(i, R) {
    if (ranks[i] != l) continue;
    const int64_t j = pi[i];
    if (j < 0 || j >= w || rho[j] != 0) continue;
    const unsigned long long key = ((unsigned long long)f2ord(d[i] + 0.0f) << 32) | (uint32_t)pos_pop[i];
    if (key == keys[j]) chosen[j] = i;   // positions are unique: exactly one row per point
  }
}
// flags of the empty points, in point order (fj) and in shuffled-reference order (fp)
__global__ void k_near_flags(const int64_t* rho, const int64_t* pos_ref, int64_t w, int* fj, int* fp) {
  MO_GRID_LOOP(j, w) {
    const int e = rho[j] == 0;
    fj[j] = e;
    fp[pos_ref[j]] = e;
  }
}
// kept = all empties in ascending point order when they fit in k, else the first k by position
// (oracle _first_k_by_pos); promoted[t] = chosen[kept_t]; counts updated
__global__ void k_near_emit(const int* fj, const int* sj, const int* sp, const int64_t* pos_ref, int64_t w, int64_t k,
                            const int64_t* chosen, int64_t* rho, int64_t* rho_p, int64_t* promoted,
                            int64_t* n_promoted) {
  const int64_t E = w ? (int64_t)sj[w - 1] + fj[w - 1] : 0;
  const bool by_pos = E > k;
  MO_GRID_LOOP(j, w) {
    if (!fj[j] || k <= 0) continue;
    int64_t t;
    if (by_pos) {
      const int64_t p = pos_ref[j];
      t = sp[p];
      if (t >= k) continue;
    } else {
      t = sj[j];
    }
    promoted[t] = chosen[j];
    rho[j] = 1;
    const int64_t c = rho_p[j] - 1;
    rho_p[j] = c;
    if (c == 0) rho[j] = I64_INF;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_promoted = k <= 0 ? 0 : (E < k ? E : k);
}

// build_cache: F_l candidates (minus `exclude`) grouped by point, shuffled population order inside a
// point (oracle niche.py:239): 64-bit keys (pi, pos_pop) radix-sorted, rows recovered through the
// inverse population permutation
__global__ void k_cache_keys(const int64_t* pi, const int64_t* ranks, const uint8_t* exclude,
                             const int64_t* pos_pop, int64_t R, int64_t l, int64_t w, unsigned long long* keys,
                             int64_t* inv_pop) {
  MO_GRID_LOOP(i, R) {
    inv_pop[pos_pop[i]] = i;
    const int64_t j = pi[i];
    const bool c = ranks[i] == l && !(exclude && exclude[i]) && j >= 0 && j < w;
    keys[i] = c ? (((unsigned long long)j << 32) | (uint32_t)pos_pop[i]) : ~0ull;
  }
}
__device__ __forceinline__ int64_t lower_bound_u64(const unsigned long long* a, int64_t n, unsigned long long v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__global__ void k_cache_emit(const unsigned long long* sorted, const int64_t* inv_pop, int64_t R, int64_t w,
                             int64_t* offsets, int64_t* cand) {
  MO_GRID_LOOP(j, w + 1) offsets[j] = lower_bound_u64(sorted, R, (unsigned long long)j << 32);
  MO_GRID_LOOP(t, R) {
    const unsigned long long key = sorted[t];
    if (key != ~0ull) cand[t] = inv_pop[(uint32_t)key];
  }
}

// batched_random_selection (Alg. 2 lines 15-26, oracle niche.py:254) in its closed form (water-fill,
// oracle niche.py:279; loop == water-fill is tested in tests/test_oracle_props.py), one block.  Every
// take is emitted as (level, order key) -> row and sorted so the output order is the loop's: level by
// level, points ascending inside a level, except the truncated last level, which keeps the first
// marked points in shuffled reference order.
constexpr int BRS_THREADS = 1024;

__device__ int64_t block_sum_i64(int64_t v, int64_t* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MO_FULL, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  int64_t t = 0;
  for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += sh[q];
  return t;
}
__device__ int64_t block_min_i64(int64_t v, int64_t* sh) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, (int64_t)__shfl_xor_sync(MO_FULL, (long long)v, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  int64_t t = sh[0];
  for (int q = 1; q < (int)(blockDim.x >> 5); ++q) t = min(t, sh[q]);
  return t;
}
__device__ int64_t block_max_i64(int64_t v, int64_t* sh) { return -block_min_i64(-v, sh); }

__global__ void __launch_bounds__(BRS_THREADS) k_brs(const int64_t* offsets, const int64_t* cand, const int64_t* rho,
                                                      const int64_t* rho_p, int64_t w, int64_t k,
                                                      const int64_t* pos_ref, int64_t* inv_ref,
                                                      unsigned long long* ekey, int64_t* erow, int64_t* info) {
  __shared__ int64_t sh[32];
  __shared__ int64_t sScan[BRS_THREADS];
  const int tid = threadIdx.x;
  for (int64_t j = tid; j < w; j += blockDim.x) inv_ref[pos_ref[j]] = j;
  const int64_t big = (int64_t)1 << 62;
  int64_t lo_v = big, hi_v = -big;
  for (int64_t j = tid; j < w; j += blockDim.x)
    if (rho[j] < I64_INF) {
      lo_v = min(lo_v, rho[j]);
      hi_v = max(hi_v, rho[j] + rho_p[j]);
    }
  const int64_t rmin = block_min_i64(lo_v, sh);
  int64_t hi = block_max_i64(hi_v, sh);
  if (k <= 0) {
    if (tid == 0) info[0] = info[1] = info[2] = 0;
    return;
  }
  auto T = [&](int64_t L) {
    int64_t s = 0;
    for (int64_t j = tid; j < w; j += blockDim.x)
      if (rho[j] < I64_INF) {
        int64_t t = L + 1 - rho[j];
        t = t < 0 ? 0 : (t > rho_p[j] ? rho_p[j] : t);
        s += t;
      }
    return block_sum_i64(s, sh);
  };
  if (rmin == big || T(hi) < k) {
    if (tid == 0) {
      info[0] = 0;
      info[1] = 0;
      info[2] = MO_ERR_INFEASIBLE;
    }
    return;
  }
  int64_t lo = rmin;
  while (lo < hi) {   // L* = min{L : T(L) >= k}
    const int64_t mid = (lo + hi) >> 1;
    if (T(mid) >= k) hi = mid;
    else lo = mid + 1;
  }
  const int64_t L = lo;
  // base takes below L* and the marked points at L*
  int64_t bsum = 0, msum = 0;
  for (int64_t j = tid; j < w; j += blockDim.x)
    if (rho[j] < I64_INF) {
      int64_t b = L - rho[j];
      b = b < 0 ? 0 : (b > rho_p[j] ? rho_p[j] : b);
      bsum += b;
      msum += (rho[j] <= L && L < rho[j] + rho_p[j]) ? 1 : 0;
    }
  const int64_t need = k - block_sum_i64(bsum, sh);
  const int64_t M = block_sum_i64(msum, sh);
  const bool trunc = M > need;
  // pass over shuffled positions: rank of each marked point among marked (position order); emit
  // this point's takes at the running offset of the emission scan
  __shared__ int64_t sCarryM, sCarryE;
  if (tid == 0) sCarryM = sCarryE = 0;
  __syncthreads();
  for (int64_t p0 = 0; p0 < w; p0 += blockDim.x) {
    const int64_t p = p0 + tid;
    int64_t j = -1, take = 0, mk = 0, base = 0;
    if (p < w) {
      j = inv_ref[p];
      if (rho[j] < I64_INF) {
        base = L - rho[j];
        base = base < 0 ? 0 : (base > rho_p[j] ? rho_p[j] : base);
        mk = (rho[j] <= L && L < rho[j] + rho_p[j]) ? 1 : 0;
      }
    }
    // inclusive scan of mk over the block (marked rank in position order)
    sScan[tid] = mk;
    __syncthreads();
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {
      const int64_t add = tid >= o ? sScan[tid - o] : 0;
      __syncthreads();
      sScan[tid] += add;
      __syncthreads();
    }
    const int64_t mrank = sCarryM + sScan[tid] - mk;
    const int64_t keep = mk && (!trunc || mrank < need) ? 1 : 0;
    take = base + keep;
    __syncthreads();
    sScan[tid] = take;
    __syncthreads();
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {
      const int64_t add = tid >= o ? sScan[tid - o] : 0;
      __syncthreads();
      sScan[tid] += add;
      __syncthreads();
    }
    int64_t e = sCarryE + sScan[tid] - take;
    for (int64_t c = 0; c < take; ++c, ++e) {
      const int64_t lev = rho[j] + c;
      const uint32_t ord = (trunc && lev == L) ? (uint32_t)p : (uint32_t)j;
      ekey[e] = ((unsigned long long)(lev - rmin) << 32) | ord;
      erow[e] = cand[offsets[j] + c];
    }
    // carries: marked and emitted totals of this chunk
    int64_t cm = block_sum_i64(mk, sh), ce = block_sum_i64(take, sh);
    if (tid == 0) {
      sCarryM += cm;
      sCarryE += ce;
    }
    __syncthreads();
  }
  if (tid == 0) {
    info[0] = sCarryE;   // == k
    info[1] = 0;         // iterations: counted after the sort (k_brs_levels)
    info[2] = 0;
  }
}
__global__ void k_brs_levels(const unsigned long long* keys, int64_t k, int64_t* info) {
  int64_t c = 0;
  for (int64_t t = threadIdx.x; t < k; t += blockDim.x) c += (t == 0 || (keys[t] >> 32) != (keys[t - 1] >> 32));
  __shared__ int64_t sh[32];
  c = block_sum_i64(c, sh);
  if (threadIdx.x == 0) info[1] = c;
}

// ----------------------------------------------------------------- variation

// sbx_pair over a batch of pairs, FP64 (oracle variation.py:46).  u given: SBX on every variable (the
// oracle's sbx_pair); u == NULL: the engine's draws -- Bernoulli(p_c) per pair from
// Philox(q, PAIR_SLOT, g, SBX), u_v from Philox(q, v, g, SBX).
__global__ void k_sbx(const double* P1, const double* P2, int64_t npairs, int d, const double* u, double eta,
                      float p_c, double lo, double hi, int clamp, uint64_t seed, uint32_t gen, double* C1,
                      double* C2) {
  MO_GRID_LOOP(e, npairs * d) {
    const int64_t q = e / d;
    const int v = (int)(e - q * d);
    const double x1 = P1[e], x2 = P2[e];
    double uu;
    if (u) {
      uu = u[e];
    } else {
      if (!(u01(philox4x32((uint32_t)q, PAIR_SLOT, gen, STREAM_SBX, seed).x) < p_c)) {
        C1[e] = x1;
        C2[e] = x2;
        continue;
      }
      uu = (double)u01(philox4x32((uint32_t)q, (uint32_t)v, gen, STREAM_SBX, seed).x);
    }
    const double b = sbx_beta(uu, eta);
    double c1 = 0.5 * ((1.0 + b) * x1 + (1.0 - b) * x2);
    double c2 = 0.5 * ((1.0 - b) * x1 + (1.0 + b) * x2);
    if (clamp) {
      c1 = clamp_to(c1, lo, hi);
      c2 = clamp_to(c2, lo, hi);
    }
    C1[e] = c1;
    C2[e] = c2;
  }
}

// polynomial_mutation, FP64 (oracle variation.py:57): u given -> mutate where flag (all when flag ==
// NULL); u == NULL -> the engine's draws (flag = u01(Philox(i, v, g, PM).x) < p_m, u = .y)
__global__ void k_pm(const double* X, int64_t n, int d, const double* u, const uint8_t* flag, double eta, float p_m,
                     double lo, double hi, uint64_t seed, uint32_t gen, double* out) {
  MO_GRID_LOOP(e, n * d) {
    const int64_t i = e / d;
    const int v = (int)(e - i * d);
    const double x = X[e];
    double uu;
    bool f;
    if (u) {
      uu = u[e];
      f = flag ? flag[e] != 0 : true;
    } else {
      const U4 r = philox4x32((uint32_t)i, (uint32_t)v, gen, STREAM_PM, seed);
      f = u01(r.x) < p_m;
      uu = (double)u01(r.y);
    }
    out[e] = f ? clamp_to(pm_apply(x, uu, eta, lo, hi), lo, hi) : x;
  }
}

}  // namespace mo

using namespace mo;

// ------------------------------------------------------------------ C-ABI

namespace {
struct OpsLayout {
  size_t a, b, c, d, e, f, cub, total;
};
size_t cub_bytes(int64_t R, int64_t w) {
  size_t s1 = 0, s2 = 0, s3 = 0;
  const int64_t n = R > w ? R : w;
  cub::DeviceRadixSort::SortKeys((void*)nullptr, s1, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                 (int)(n > 0 ? n : 1));
  cub::DeviceRadixSort::SortPairs((void*)nullptr, s2, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const int64_t*)nullptr, (int64_t*)nullptr,
                                  (int)(n > 0 ? n : 1));
  cub::DeviceScan::ExclusiveSum((void*)nullptr, s3, (const int*)nullptr, (int*)nullptr, (int)(w > 0 ? w : 1));
  size_t s = s1 > s2 ? s1 : s2;
  return s > s3 ? s : s3;
}
OpsLayout ops_layout(int64_t R, int64_t w) {
  const int64_t n = (R > w ? R : w) + 1;
  OpsLayout L;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o += (size_t)round_up((int64_t)bytes, 256);
    return at;
  };
  L.a = take(8 * n);   // keys / ArgMin partials
  L.b = take(8 * n);   // sorted keys
  L.c = take(8 * n);   // inverse permutation / chosen
  L.d = take(8 * n);   // rows (sort values)
  L.e = take(4 * n);   // flags
  L.f = take(4 * n);   // scans
  L.cub = take(cub_bytes(R, w));
  L.total = o;
  return L;
}
template <typename T>
T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}
}  // namespace

extern "C" {

int mo_ops_workspace_bytes(int64_t R, int64_t w, size_t* bytes) {
  if (R < 0 || w < 0 || !bytes) return MO_ERR_PARAM;
  *bytes = ops_layout(R, w).total;
  return MO_OK;
}

int mo_step_mask(const double* x, int64_t n, int8_t* out, void* stream_) {
  if (n < 0 || (n && (!x || !out))) return MO_ERR_PARAM;
  if (n == 0) return MO_OK;
  k_step_mask<<<ops_blocks(n), OPS_THREADS, 0, (cudaStream_t)stream_>>>(x, n, out);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int mo_masked_argmin(const double* values, const uint8_t* valid, int64_t n, int64_t* out, void* workspace,
                     size_t workspace_bytes, void* stream_) {
  if (n < 0 || !out || (n && !values)) return MO_ERR_PARAM;
  OpsLayout L = ops_layout(n, 1);
  if (!workspace || workspace_bytes < L.total) return MO_ERR_PARAM;
  cudaStream_t s = (cudaStream_t)stream_;
  const unsigned nb = n ? (ops_blocks(n) < 1024 ? ops_blocks(n) : 1024) : 1;
  ArgMin* part = at<ArgMin>(workspace, L.a);
  k_argmin_partial<<<nb, OPS_THREADS, 0, s>>>(values, valid, n, part);
  k_argmin_final<<<1, OPS_THREADS, 0, s>>>(part, (int)nb, out);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int mo_segment_count(const int64_t* labels, const uint8_t* valid, int64_t n, int64_t segments, int64_t* counts,
                     int32_t* status, void* stream_) {
  if (n < 0 || segments < 0 || !status || (segments && !counts) || (n && !labels)) return MO_ERR_PARAM;
  cudaStream_t s = (cudaStream_t)stream_;
  if (cudaMemsetAsync(status, 0, sizeof(int32_t), s) != cudaSuccess) return MO_ERR_CUDA;
  if (segments) k_fill_i64<<<ops_blocks(segments), OPS_THREADS, 0, s>>>(counts, segments, 0);
  if (n)
    k_segment_count<<<ops_blocks(n), OPS_THREADS, 0, s>>>(labels, valid, n, segments,
                                                          reinterpret_cast<unsigned long long*>(counts), status);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int mo_associate_matrix(const double* D, const uint8_t* valid, int64_t R, int64_t w, int64_t* pi, double* d,
                        void* stream_) {
  if (R < 0 || w < 1 || (R && (!D || !pi || !d))) return MO_ERR_PARAM;
  if (R == 0) return MO_OK;
  const int64_t blocks = ceil_div(R, OPS_THREADS / 32);
  k_associate_matrix<<<(unsigned)(blocks < 8192 ? blocks : 8192), OPS_THREADS, 0, (cudaStream_t)stream_>>>(
      D, valid, R, w, pi, d);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int mo_niche_counts(const int64_t* pi, const int64_t* ranks, int64_t R, int64_t l, int64_t w, int64_t* rho,
                    int64_t* rho_p, void* stream_) {
  if (R < 0 || w < 1 || !rho || !rho_p || (R && (!pi || !ranks))) return MO_ERR_PARAM;
  cudaStream_t s = (cudaStream_t)stream_;
  k_fill_i64<<<ops_blocks(w), OPS_THREADS, 0, s>>>(rho, w, 0);
  k_fill_i64<<<ops_blocks(w), OPS_THREADS, 0, s>>>(rho_p, w, 0);
  if (R)
    k_niche_count<<<ops_blocks(R), OPS_THREADS, 0, s>>>(pi, ranks, R, l, w,
                                                        reinterpret_cast<unsigned long long*>(rho),
                                                        reinterpret_cast<unsigned long long*>(rho_p));
  k_niche_count_finish<<<ops_blocks(w), OPS_THREADS, 0, s>>>(rho, rho_p, w);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int mo_nearest_selection(const int64_t* pi, const float* d, const int64_t* ranks, int64_t R, int64_t l,
                         int64_t* rho, int64_t* rho_p, int64_t w, int64_t k, const int64_t* pos_pop,
                         const int64_t* pos_ref, int64_t* promoted, int64_t* n_promoted, void* workspace,
                         size_t workspace_bytes, void* stream_) {
  if (R < 0 || w < 1 || !rho || !rho_p || !pos_ref || !promoted || !n_promoted ||
      (R && (!pi || !d || !ranks || !pos_pop)))
    return MO_ERR_PARAM;
  OpsLayout L = ops_layout(R, w);
  if (!workspace || workspace_bytes < L.total) return MO_ERR_PARAM;
  cudaStream_t s = (cudaStream_t)stream_;
  unsigned long long* keys = at<unsigned long long>(workspace, L.a);
  int64_t* chosen = at<int64_t>(workspace, L.c);
  int* fj = at<int>(workspace, L.e);                      // empty flags / their scan, point order
  int* sj = at<int>(workspace, L.f);
  int* fp = at<int>(workspace, L.b);                      // the same in shuffled-reference order
  int* sp = fp + w;                                       //  (region b holds 8(w+1) bytes)
  if (cudaMemsetAsync(keys, 0xff, sizeof(unsigned long long) * (size_t)w, s) != cudaSuccess) return MO_ERR_CUDA;
  if (R) {
    k_near_keys<<<ops_blocks(R), OPS_THREADS, 0, s>>>(pi, d, ranks, rho, pos_pop, R, l, w, keys);
    k_near_rows<<<ops_blocks(R), OPS_THREADS, 0, s>>>(pi, d, ranks, rho, pos_pop, R, l, w, keys, chosen);
  }
  k_near_flags<<<ops_blocks(w), OPS_THREADS, 0, s>>>(rho, pos_ref, w, fj, fp);
  size_t tb = workspace_bytes - L.cub;
  void* tmp = at<void>(workspace, L.cub);
  if (cub::DeviceScan::ExclusiveSum(tmp, tb, fj, sj, (int)w, s) != cudaSuccess) return MO_ERR_CUDA;
  tb = workspace_bytes - L.cub;
  if (cub::DeviceScan::ExclusiveSum(tmp, tb, fp, sp, (int)w, s) != cudaSuccess) return MO_ERR_CUDA;
  k_near_emit<<<ops_blocks(w), OPS_THREADS, 0, s>>>(fj, sj, sp, pos_ref, w, k, chosen, rho, rho_p, promoted,
                                                     n_promoted);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int mo_build_cache(const int64_t* pi, const int64_t* ranks, int64_t R, int64_t l, int64_t w, const int64_t* pos_pop,
                   const uint8_t* exclude, int64_t* offsets, int64_t* cand, void* workspace, size_t workspace_bytes,
                   void* stream_) {
  if (R < 0 || w < 1 || !offsets || (R && (!pi || !ranks || !pos_pop || !cand))) return MO_ERR_PARAM;
  OpsLayout L = ops_layout(R, w);
  if (!workspace || workspace_bytes < L.total) return MO_ERR_PARAM;
  cudaStream_t s = (cudaStream_t)stream_;
  if (R == 0) {
    k_fill_i64<<<ops_blocks(w + 1), OPS_THREADS, 0, s>>>(offsets, w + 1, 0);
    MO_CHECK_LAUNCH();
    return MO_OK;
  }
  unsigned long long* keys = at<unsigned long long>(workspace, L.a);
  unsigned long long* sorted = at<unsigned long long>(workspace, L.b);
  int64_t* inv = at<int64_t>(workspace, L.c);
  k_cache_keys<<<ops_blocks(R), OPS_THREADS, 0, s>>>(pi, ranks, exclude, pos_pop, R, l, w, keys, inv);
  size_t tb = workspace_bytes - L.cub;
  if (cub::DeviceRadixSort::SortKeys(at<void>(workspace, L.cub), tb, keys, sorted, (int)R, 0, 64, s) != cudaSuccess)
    return MO_ERR_CUDA;
  k_cache_emit<<<ops_blocks(R > w + 1 ? R : w + 1), OPS_THREADS, 0, s>>>(sorted, inv, R, w, offsets, cand);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int mo_batched_random_selection(const int64_t* offsets, const int64_t* cand, const int64_t* rho, const int64_t* rho_p,
                                int64_t w, int64_t k, const int64_t* pos_ref, int64_t* taken, int64_t* info,
                                void* workspace, size_t workspace_bytes, void* stream_) {
  if (w < 1 || k < 0 || !offsets || !rho || !rho_p || !pos_ref || !info || (k && (!cand || !taken)))
    return MO_ERR_PARAM;
  OpsLayout L = ops_layout(k, w);
  if (!workspace || workspace_bytes < L.total) return MO_ERR_PARAM;
  cudaStream_t s = (cudaStream_t)stream_;
  unsigned long long* ekey = at<unsigned long long>(workspace, L.a);
  unsigned long long* skey = at<unsigned long long>(workspace, L.b);
  int64_t* inv = at<int64_t>(workspace, L.c);
  int64_t* erow = at<int64_t>(workspace, L.d);
  k_brs<<<1, BRS_THREADS, 0, s>>>(offsets, cand, rho, rho_p, w, k, pos_ref, inv, ekey, erow, info);
  MO_CHECK_LAUNCH();
  if (k) {
    size_t tb = workspace_bytes - L.cub;
    if (cub::DeviceRadixSort::SortPairs(at<void>(workspace, L.cub), tb, ekey, skey, erow, taken, (int)k, 0, 64, s) !=
        cudaSuccess)
      return MO_ERR_CUDA;
    k_brs_levels<<<1, 1024, 0, s>>>(skey, k, info);
    MO_CHECK_LAUNCH();
  }
  return MO_OK;
}

int mo_sbx_pairs(const double* P1, const double* P2, int64_t npairs, int32_t d, const double* u, double eta_c,
                 float p_c, double lo, double hi, int32_t clamp, uint64_t seed, uint32_t generation, double* C1,
                 double* C2, void* stream_) {
  if (npairs < 0 || d < 1 || !(eta_c > 0.0) || (npairs && (!P1 || !P2 || !C1 || !C2))) return MO_ERR_PARAM;
  if (npairs == 0) return MO_OK;
  k_sbx<<<ops_blocks(npairs * d), OPS_THREADS, 0, (cudaStream_t)stream_>>>(P1, P2, npairs, d, u, eta_c, p_c, lo, hi,
                                                                           clamp, seed, generation, C1, C2);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int mo_polynomial_mutation(const double* X, int64_t n, int32_t d, const double* u, const uint8_t* flag, double eta_m,
                           float p_m, double lo, double hi, uint64_t seed, uint32_t generation, double* out,
                           void* stream_) {
  if (n < 0 || d < 1 || !(eta_m > 0.0) || !(hi > lo) || (n && (!X || !out))) return MO_ERR_PARAM;
  if (n == 0) return MO_OK;
  k_pm<<<ops_blocks(n * d), OPS_THREADS, 0, (cudaStream_t)stream_>>>(X, n, d, u, flag, eta_m, p_m, lo, hi, seed,
                                                                      generation, out);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

}  // extern "C"
