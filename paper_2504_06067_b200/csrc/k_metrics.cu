// Quality indicators on the GPU (metrics module; SURVEY.md
// 8(f) item 1): IGD and Monte-Carlo hypervolume.
//
// IGD: mean over reference points of the Euclidean distance
// to the nearest front member.  k_igd_min: a 2-D grid of (reference tile,
// front split); a thread keeps IGD_RPT reference points in FP64 registers
// and streams its split of the front through shared memory (FP64), then
// merges its minimum squared distances with a 64-bit atomicMin on the bit
// patterns (non-negative doubles order like their bits), so the result does
// not depend on the split count or scheduling.  k_igd_sum: one block adds
// sqrt(min) in a fixed order (per-thread strided partials, fixed tree) -- the
// value is deterministic run to run.
//
// HV (m > 3 branch): Monte-Carlo with a counter-based
// (Philox) sample stream over the box [lower, ref]; a sample counts when some
// retained front point weakly dominates it.  Per-block hit counts are summed
// in fixed order; hv = box volume * hits / samples.
//
// HV exact (m <= 3 branch; m = 1, 2 are padded to m = 3
// with a zero coordinate and a unit reference extent, which multiplies the
// volume by exactly 1): slab decomposition along the third objective.
// k_hv_rank ranks the retained rows (F <= ref) in (f1, f2, row) order and in
// (f3, row) order by tiled all-pairs counting (no sort library; deterministic
// dense positions) and scatters them; k_hv_slab gives slab k = [z_(k),
// z_(k+1)) the 2-D staircase area of the rows with z-rank <= k, swept in
// (f1, f2) order in FP64 (area += (r1 - x) * max(0, ymin - y)), times its
// thickness; the slabs are added in a fixed order.  O(n^2) work, all of it
// parallel: ~ms at n = 10^5.
#include "mo_common.cuh"
#include "mo_rng.cuh"

namespace mo {

constexpr int IGD_THREADS = 256;
constexpr int IGD_RPT = 2;          // reference points per thread
constexpr int IGD_FTILE = 256;      // front rows per shared-memory tile
constexpr int IGD_MAXM = 16;

template <int M>
__global__ void __launch_bounds__(IGD_THREADS) k_igd_min(const float* __restrict__ front, int64_t nf,
                                                         const float* __restrict__ ref, int64_t nr,
                                                         int64_t fsplit, unsigned long long* __restrict__ dmin) {
  constexpr int m = M;
  __shared__ double sF[IGD_FTILE * M];
  const int64_t r0 = ((int64_t)blockIdx.x * IGD_THREADS + threadIdx.x) * IGD_RPT;
  double rv[IGD_RPT][M];
  double best[IGD_RPT];
#pragma unroll
  for (int q = 0; q < IGD_RPT; ++q) {
    best[q] = __longlong_as_double(0x7ff0000000000000ll);
#pragma unroll
    for (int k = 0; k < m; ++k) rv[q][k] = (r0 + q < nr) ? (double)ref[(r0 + q) * m + k] : 0.0;
  }
  const int64_t f0 = (int64_t)blockIdx.y * fsplit, f1 = min(nf, f0 + fsplit);
  for (int64_t t0 = f0; t0 < f1; t0 += IGD_FTILE) {
    const int tn = (int)min((int64_t)IGD_FTILE, f1 - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < tn * m; e += IGD_THREADS) sF[e] = (double)front[t0 * m + e];
    __syncthreads();
    for (int i = 0; i < tn; ++i) {
#pragma unroll
      for (int q = 0; q < IGD_RPT; ++q) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < m; ++k) {
          const double d = __dsub_rn(sF[i * m + k], rv[q][k]);
          s = __dadd_rn(s, __dmul_rn(d, d));
        }
        best[q] = fmin(best[q], s);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < IGD_RPT; ++q)
    if (r0 + q < nr) atomicMin(dmin + r0 + q, (unsigned long long)__double_as_longlong(best[q]));
}

constexpr int SUM_THREADS = 1024;

__global__ void __launch_bounds__(SUM_THREADS) k_igd_sum(const unsigned long long* __restrict__ dmin, int64_t nr,
                                                         double* __restrict__ out) {
  __shared__ double sh[SUM_THREADS];
  double s = 0.0;
  for (int64_t r = threadIdx.x; r < nr; r += SUM_THREADS) s = __dadd_rn(s, sqrt(__longlong_as_double((long long)dmin[r])));
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = SUM_THREADS / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sh[0] / (double)nr;
}

// ------------------------------------------------------------------- HV (MC)

constexpr int HV_THREADS = 256;
constexpr int HV_SPT = 4;      // samples per thread

template <int M>
__global__ void __launch_bounds__(HV_THREADS) k_hv_mc(const float* __restrict__ front, int64_t nf,
                                                      const double* __restrict__ lower,
                                                      const double* __restrict__ upper, int64_t samples,
                                                      uint64_t seed, unsigned long long* __restrict__ hits) {
  constexpr int m = M;
  __shared__ float sF[IGD_FTILE * M];
  __shared__ int sCnt[HV_THREADS / 32];
  const int64_t s0 = ((int64_t)blockIdx.x * HV_THREADS + threadIdx.x) * HV_SPT;
  double x[HV_SPT][M];
  bool hit[HV_SPT];
#pragma unroll
  for (int q = 0; q < HV_SPT; ++q) {
    hit[q] = s0 + q >= samples;  // padding samples never count (cleared below)
#pragma unroll
    for (int k = 0; k < m; k += 4) {
      // Philox counter (sample_lo, sample_hi, k/4, STREAM_HV): four 24-bit uniforms in [0,1)
      const U4 w = philox4x32((uint32_t)(s0 + q), (uint32_t)((s0 + q) >> 32), (uint32_t)(k / 4), STREAM_HV, seed);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (k + u >= m) break;
        const double t = (double)(ws[u] >> 8) * (1.0 / 16777216.0);
        x[q][k + u] = lower[k + u] + t * (upper[k + u] - lower[k + u]);
      }
    }
  }
  for (int64_t t0 = 0; t0 < nf; t0 += IGD_FTILE) {
    const int tn = (int)min((int64_t)IGD_FTILE, nf - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < tn * m; e += HV_THREADS) sF[e] = front[t0 * m + e];
    __syncthreads();
    for (int i = 0; i < tn; ++i) {
#pragma unroll
      for (int q = 0; q < HV_SPT; ++q) {
        bool dom = true;
#pragma unroll
        for (int k = 0; k < m; ++k) dom = dom && ((double)sF[i * m + k] <= x[q][k]);
        hit[q] = hit[q] || dom;
      }
    }
  }
  int c = 0;
#pragma unroll
  for (int q = 0; q < HV_SPT; ++q) c += (s0 + q < samples) && hit[q];
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0) sCnt[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < HV_THREADS / 32; ++w) t += sCnt[w];
    hits[blockIdx.x] = (unsigned long long)t;
  }
}

__global__ void k_hv_sum(const unsigned long long* __restrict__ hits, int64_t nblk, unsigned long long* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long t = 0;
    for (int64_t b = 0; b < nblk; ++b) t += hits[b];
    out[0] = t;
  }
}

// ------------------------------------------------------------------ HV (exact)

constexpr int HVX_THREADS = 256;

struct HvExactWs {
  double2* xy;      // [nf] retained rows in (x, y, row) order
  int32_t* zr;      // [nf] their z-ranks
  double* zs;       // [nf] z values in (z, row) order
  double* slab;     // [nf]
  int32_t* nv;      // retained count
};

__device__ __forceinline__ void hv_row(const float* F, int m, int64_t i, double& x, double& y, double& z) {
  x = (double)F[i * m];
  y = m > 1 ? (double)F[i * m + 1] : 0.0;
  z = m > 2 ? (double)F[i * m + 2] : 0.0;
}

__global__ void __launch_bounds__(HVX_THREADS) k_hv_rank(const float* __restrict__ F, int64_t nf, int m,
                                                         const double* __restrict__ ref, HvExactWs w) {
  __shared__ double sX[HVX_THREADS], sY[HVX_THREADS], sZ[HVX_THREADS];
  __shared__ int sV[HVX_THREADS];
  const double r0 = ref[0], r1 = m > 1 ? ref[1] : 1.0, r2 = m > 2 ? ref[2] : 1.0;
  const int64_t i = (int64_t)blockIdx.x * HVX_THREADS + threadIdx.x;
  double x = 0, y = 0, z = 0;
  bool vi = false;
  if (i < nf) {
    hv_row(F, m, i, x, y, z);
    vi = x <= r0 && y <= r1 && z <= r2;
  }
  int px = 0, pz = 0;
  for (int64_t t0 = 0; t0 < nf; t0 += HVX_THREADS) {
    __syncthreads();
    const int64_t j = t0 + threadIdx.x;
    double a = 0, b = 0, c = 0;
    bool vj = false;
    if (j < nf) {
      hv_row(F, m, j, a, b, c);
      vj = a <= r0 && b <= r1 && c <= r2;
    }
    sX[threadIdx.x] = a; sY[threadIdx.x] = b; sZ[threadIdx.x] = c; sV[threadIdx.x] = vj;
    __syncthreads();
    const int tn = (int)min((int64_t)HVX_THREADS, nf - t0);
    for (int q = 0; q < tn; ++q) {
      if (!sV[q]) continue;
      const int64_t jj = t0 + q;
      const double a2 = sX[q], b2 = sY[q], c2 = sZ[q];
      px += (a2 < x) || (a2 == x && (b2 < y || (b2 == y && jj < i)));
      pz += (c2 < z) || (c2 == z && jj < i);
    }
  }
  if (vi) {
    w.xy[px] = make_double2(x, y);
    w.zr[px] = pz;
    w.zs[pz] = z;
    atomicAdd(w.nv, 1);
  }
}

__global__ void __launch_bounds__(HVX_THREADS) k_hv_slab(int m, const double* __restrict__ ref, HvExactWs w) {
  __shared__ double2 sXY[HVX_THREADS];
  __shared__ int sZR[HVX_THREADS];
  const int nv = *w.nv;
  if ((int64_t)blockIdx.x * HVX_THREADS >= nv) return;  // uniform per block
  const double r0 = ref[0], r1 = m > 1 ? ref[1] : 1.0, r2 = m > 2 ? ref[2] : 1.0;
  const int k = blockIdx.x * HVX_THREADS + threadIdx.x;
  double thick = 0.0;
  if (k < nv) thick = (k + 1 < nv ? w.zs[k + 1] : r2) - w.zs[k];
  double area = 0.0, ymin = r1;
  const bool busy = __syncthreads_or(thick > 0.0);
  if (!busy) {
    if (k < nv) w.slab[k] = 0.0;
    return;
  }
  for (int t0 = 0; t0 < nv; t0 += HVX_THREADS) {
    __syncthreads();
    if (t0 + (int)threadIdx.x < nv) {
      sXY[threadIdx.x] = w.xy[t0 + threadIdx.x];
      sZR[threadIdx.x] = w.zr[t0 + threadIdx.x];
    }
    __syncthreads();
    const int tn = min(HVX_THREADS, nv - t0);
    if (thick > 0.0) {
      for (int q = 0; q < tn; ++q) {
        const double2 p = sXY[q];
        if (sZR[q] <= k && p.y < ymin) {
          area = __fma_rn(r0 - p.x, ymin - p.y, area);
          ymin = p.y;
        }
      }
    }
  }
  if (k < nv) w.slab[k] = thick > 0.0 ? area * thick : 0.0;
}

__global__ void __launch_bounds__(SUM_THREADS) k_hv_exact_sum(HvExactWs w, double* __restrict__ out) {
  __shared__ double sh[SUM_THREADS];
  const int nv = *w.nv;
  double s = 0.0;
  for (int r = threadIdx.x; r < nv; r += SUM_THREADS) s = __dadd_rn(s, w.slab[r]);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int q = SUM_THREADS / 2; q > 0; q >>= 1) {
    if ((int)threadIdx.x < q) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + q]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sh[0];
}

static HvExactWs hv_exact_layout(void* ws, int64_t nf) {
  char* p = reinterpret_cast<char*>(ws);
  HvExactWs w;
  w.xy = reinterpret_cast<double2*>(p);
  p += (size_t)nf * 16;
  w.zs = reinterpret_cast<double*>(p);
  p += (size_t)nf * 8;
  w.slab = reinterpret_cast<double*>(p);
  p += (size_t)nf * 8;
  w.zr = reinterpret_cast<int32_t*>(p);
  p += (size_t)((nf + 1) & ~1ll) * 4;
  w.nv = reinterpret_cast<int32_t*>(p);
  return w;
}

}  // namespace mo

using namespace mo;

extern "C" {

size_t mo_igd_workspace_bytes(int64_t nr) { return nr > 0 ? (size_t)nr * 8 : 8; }

int mo_igd(const float* front, int64_t nf, const float* ref, int64_t nr, int32_t m, double* out, void* workspace,
           size_t workspace_bytes, void* stream_) {
  if (nf < 1 || nr < 1) return MO_ERR_EMPTY;
  if (m < 1 || m > IGD_MAXM || !front || !ref || !out || !workspace) return MO_ERR_PARAM;
  if (workspace_bytes < mo_igd_workspace_bytes(nr)) return MO_ERR_PARAM;
  cudaStream_t s = (cudaStream_t)stream_;
  unsigned long long* dmin = reinterpret_cast<unsigned long long*>(workspace);
  if (cudaMemsetAsync(dmin, 0x7f, (size_t)nr * 8, s) != cudaSuccess) return MO_ERR_CUDA;  // large positive
  const int64_t rblocks = ceil_div(nr, (int64_t)IGD_THREADS * IGD_RPT);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // split the front so the grid covers every SM a few times
  int64_t splits = ceil_div((int64_t)sms * 4, rblocks);
  splits = splits < 1 ? 1 : (splits > 65535 ? 65535 : splits);
  const int64_t fsplit = ceil_div(nf, splits);
  splits = ceil_div(nf, fsplit);
  if (rblocks > 0x7fffffff) return MO_ERR_PARAM;
  const dim3 grid((unsigned)rblocks, (unsigned)splits);
  switch (m) {
#define MO_IGD_CASE(MM) \
  case MM: k_igd_min<MM><<<grid, IGD_THREADS, 0, s>>>(front, nf, ref, nr, fsplit, dmin); break;
    MO_IGD_CASE(1) MO_IGD_CASE(2) MO_IGD_CASE(3) MO_IGD_CASE(4) MO_IGD_CASE(5) MO_IGD_CASE(6) MO_IGD_CASE(7)
    MO_IGD_CASE(8) MO_IGD_CASE(9) MO_IGD_CASE(10) MO_IGD_CASE(11) MO_IGD_CASE(12) MO_IGD_CASE(13)
    MO_IGD_CASE(14) MO_IGD_CASE(15) MO_IGD_CASE(16)
#undef MO_IGD_CASE
    default: return MO_ERR_PARAM;
  }
  MO_CHECK_LAUNCH();
  k_igd_sum<<<1, SUM_THREADS, 0, s>>>(dmin, nr, out);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

size_t mo_hv_mc_workspace_bytes(int64_t samples) {
  return (size_t)(ceil_div(samples, (int64_t)HV_THREADS * HV_SPT) + 1) * 8;
}

int mo_hv_mc(const float* front, int64_t nf, int32_t m, const double* lower, const double* upper, int64_t samples,
             uint64_t seed, unsigned long long* hits_out, void* workspace, size_t workspace_bytes, void* stream_) {
  if (m < 1 || m > IGD_MAXM || samples < 1 || !lower || !upper || !hits_out) return MO_ERR_PARAM;
  if (workspace_bytes < mo_hv_mc_workspace_bytes(samples) || !workspace) return MO_ERR_PARAM;
  cudaStream_t s = (cudaStream_t)stream_;
  const int64_t blocks = ceil_div(samples, (int64_t)HV_THREADS * HV_SPT);
  unsigned long long* hits = reinterpret_cast<unsigned long long*>(workspace);
  if (nf < 1) return cudaMemsetAsync(hits_out, 0, 8, s) == cudaSuccess ? MO_OK : MO_ERR_CUDA;
  if (blocks > 0x7fffffff) return MO_ERR_PARAM;
  switch (m) {
#define MO_HV_CASE(MM) \
  case MM: k_hv_mc<MM><<<(unsigned)blocks, HV_THREADS, 0, s>>>(front, nf, lower, upper, samples, seed, hits); break;
    MO_HV_CASE(1) MO_HV_CASE(2) MO_HV_CASE(3) MO_HV_CASE(4) MO_HV_CASE(5) MO_HV_CASE(6) MO_HV_CASE(7)
    MO_HV_CASE(8) MO_HV_CASE(9) MO_HV_CASE(10) MO_HV_CASE(11) MO_HV_CASE(12) MO_HV_CASE(13)
    MO_HV_CASE(14) MO_HV_CASE(15) MO_HV_CASE(16)
#undef MO_HV_CASE
    default: return MO_ERR_PARAM;
  }
  MO_CHECK_LAUNCH();
  k_hv_sum<<<1, 32, 0, s>>>(hits, blocks, hits_out);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

size_t mo_hv_exact_workspace_bytes(int64_t nf) {
  const int64_t n = nf > 0 ? nf : 1;
  return (size_t)n * 32 + (size_t)((n + 1) & ~1ll) * 4 + 16;
}

int mo_hv_exact(const float* front, int64_t nf, int32_t m, const double* ref, double* out, void* workspace,
                size_t workspace_bytes, void* stream_) {
  if (m < 1 || m > 3 || nf < 0 || !ref || !out) return MO_ERR_PARAM;
  if (nf > 0x7ffffffe || (nf > 0 && (!front || !workspace || workspace_bytes < mo_hv_exact_workspace_bytes(nf))))
    return MO_ERR_PARAM;
  cudaStream_t s = (cudaStream_t)stream_;
  if (nf == 0) return cudaMemsetAsync(out, 0, 8, s) == cudaSuccess ? MO_OK : MO_ERR_CUDA;
  HvExactWs w = hv_exact_layout(workspace, nf);
  if (cudaMemsetAsync(w.nv, 0, 4, s) != cudaSuccess) return MO_ERR_CUDA;
  const unsigned blocks = (unsigned)ceil_div(nf, (int64_t)HVX_THREADS);
  k_hv_rank<<<blocks, HVX_THREADS, 0, s>>>(front, nf, m, ref, w);
  MO_CHECK_LAUNCH();
  k_hv_slab<<<blocks, HVX_THREADS, 0, s>>>(m, ref, w);
  MO_CHECK_LAUNCH();
  k_hv_exact_sum<<<1, SUM_THREADS, 0, s>>>(w, out);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

}  // extern "C"
