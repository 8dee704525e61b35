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

}  // extern "C"
