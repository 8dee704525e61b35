// Fused variation + evaluation: mating pool -> SBX -> clamp -> PM -> clamp -> DTLZ.
//
// Reference ops: variation.mating_pool, sbx_pair (:258-266),
// polynomial_mutation (:267-275), clamp (:295), problems.dtlz_eval (:520-528).
// One thread per mating pair q: parents a = perm[2q], b = perm[2q+1] of the
// keyed MATING permutation; children are written to rows 2q and 2q+1.
// Draws: pair Bernoulli(p_c) = Philox(q, PAIR_SLOT, g, SBX).x, SBX u_v =
// Philox(q, v, g, SBX).x, PM flag/draw = Philox(i, v, g, PM).x/.y.  The
// arithmetic is FP64 (oracle order), children are rounded to FP32 once after
// SBX+clamp and once after PM+clamp.
#include <string.h>

#include "mo_common.cuh"
#include "mo_dtlz.cuh"
#include "mo_rng.cuh"
#include "mo_prologue.cuh"
#include "mo_variation.cuh"

namespace mo {



// One block = ppb <= VARY_PAIRS mating pairs, VARY_THREADS threads.  Phase 1: one
// thread per pair draws the parents (keyed MATING permutation) into shared
// memory.  Phase 2: one thread per (pair, variable) runs SBX + clamp + PM +
// clamp and writes both children.  Phase 3: one thread per (child,
// objective) evaluates DTLZ in FP64 and lowers the block's column minima.
constexpr int VARY_PAIRS = 16;
constexpr int VARY_THREADS = 256;
#ifndef MO_VARY_FACTOR_M
#define MO_VARY_FACTOR_M 5
#endif

__global__ void __launch_bounds__(VARY_THREADS) k_vary_eval(int problem, const float* __restrict__ X, int n, int d,
                                                            int m, uint64_t seed, uint32_t gen_val,
                                                            const uint32_t* gen_ptr, mo_var_cfg cfg,
                                                            float* __restrict__ Xo, float* __restrict__ Fo,
                                                            float* __restrict__ ideal, int* __restrict__ domain_flag,
                                                            PrepArgs pro, int pro_blocks, int ppb) {
  pdl_wait();
  __shared__ uint32_t shK[MAX_SHUFFLE_ROUNDS], shS[MAX_SHUFFLE_ROUNDS];
  __shared__ int shR;
  if ((int)blockIdx.x < pro_blocks) {   // first CTAs (scheduled first): the generation prologue
    __shared__ uint32_t shK2[MAX_SHUFFLE_ROUNDS], shS2[MAX_SHUFFLE_ROUNDS];
    __shared__ int shR2;
    if (blockIdx.x == 0) trace_mark_any(pro.trace, 46);
    const uint32_t g = gen_ptr ? *gen_ptr : gen_val;
    const int gtid = (int)blockIdx.x * VARY_THREADS + (int)threadIdx.x, gthreads = pro_blocks * VARY_THREADS;
    gen_prologue(pro, g, gtid, gthreads, shK, shS, &shR, shK2, shS2, &shR2);
    if (pro.mate) {
      // next generation's mating parents (off this generation's critical path)
      const uint32_t gn = g + 1u;
      __syncthreads();
      load_shuffle_keys_smem(shK2, shS2, &shR2, (uint32_t)n, seed, gn, STREAM_MATING);
      __syncthreads();
      int* buf = pro.mate + 16 + (int64_t)(gn & 1u) * n;
      int* tag = pro.mate + 4 * (gn & 1u);
      // continue the prologue's index space (rows, reference points, then mating slots) so that the
      // slots go to threads that had no row / reference item when the grid covers all three
      const int off = (pro.R + pro.w) % gthreads;
      for (int q = (gtid - off + gthreads) % gthreads; q < n; q += gthreads)
        buf[q] = (int)prp_inv((uint32_t)q, shK2, shS2, shR2, (uint32_t)n);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(pro.mate + 8, 1) == pro_blocks - 1) {   // last prologue CTA: publish
          pro.mate[8] = 0;
          tag[1] = (int)(uint32_t)seed;
          tag[2] = (int)(uint32_t)(seed >> 32);
          tag[3] = n;
          __threadfence();
          tag[0] = (int)~gn;                                   // written last: the validity flag
        }
      }
    }
    if (blockIdx.x == 0) trace_mark_any(pro.trace, 45);
    return;
  }
  const bool tb = (int)blockIdx.x == pro_blocks;   // traced vary block
  if (tb) trace_mark_any(pro.trace, 40);
  const int vblock = (int)blockIdx.x - pro_blocks;
  __shared__ float shMin[16];
  __shared__ int shA[VARY_PAIRS], shB[VARY_PAIRS];
  __shared__ uint8_t shCross[VARY_PAIRS];
  const uint32_t gen = gen_ptr ? *gen_ptr : gen_val;
  // parents precomputed by the previous generation's prologue CTAs, when their tag matches
  const int* mtag = pro.mate ? pro.mate + 4 * (gen & 1u) : nullptr;
  const int* mbuf = (mtag && __ldcg(mtag) == (int)~gen && __ldcg(mtag + 1) == (int)(uint32_t)seed &&
                     __ldcg(mtag + 2) == (int)(uint32_t)(seed >> 32) && __ldcg(mtag + 3) == n)
                        ? pro.mate + 16 + (int64_t)(gen & 1u) * n : nullptr;
  if (!mbuf) load_shuffle_keys_smem(shK, shS, &shR, (uint32_t)n, seed, gen, STREAM_MATING);
  if (threadIdx.x < 16) shMin[threadIdx.x] = __int_as_float(0x7f800000);
  __syncthreads();
  const int npairs = n / 2;
  const int q0 = vblock * ppb;
  const int tid = threadIdx.x;
  // the two parents of a pair on two threads (each inverse shuffle is ~74 dependent rounds)
  if (tid < 2 * ppb && q0 + (tid >> 1) < npairs) {
    const int ql = tid >> 1, q = q0 + ql;
    const uint32_t slot = 2u * q + (uint32_t)(tid & 1);
    const int par = mbuf ? __ldcg(mbuf + slot) : (int)prp_inv(slot, shK, shS, shR, (uint32_t)n);
    if (tid & 1) {
      shB[ql] = par;
    } else {
      shA[ql] = par;
      shCross[ql] = u01(philox4x32((uint32_t)q, PAIR_SLOT, gen, STREAM_SBX, seed).x) < cfg.p_c;
    }
  }
  __syncthreads();
  if (tb) trace_mark_any(pro.trace, 41);
  const float p_m = cfg.p_m < 0.0f ? 1.0f / (float)d : cfg.p_m;
  const double eta_c = (double)cfg.eta_c, eta_m = (double)cfg.eta_m;
  const int npb = min(ppb, npairs - q0);
  const int tasks = npb * d;
  for (int e = tid; e < tasks; e += VARY_THREADS) {
    const int ql = e / d, v = e - ql * d;
    const int q = q0 + ql;
    const float y1 = X[(int64_t)shA[ql] * d + v], y2 = X[(int64_t)shB[ql] * d + v];
    float o1 = y1, o2 = y2;
    if (shCross[ql]) {
      const double x1 = (double)y1, x2 = (double)y2;
      const double u = (double)u01(philox4x32((uint32_t)q, (uint32_t)v, gen, STREAM_SBX, seed).x);
      const double be = sbx_beta(u, eta_c);
      o1 = (float)clamp01(0.5 * ((1.0 + be) * x1 + (1.0 - be) * x2));
      o2 = (float)clamp01(0.5 * ((1.0 - be) * x1 + (1.0 + be) * x2));
    }
    const U4 r1 = philox4x32((uint32_t)(2 * q), (uint32_t)v, gen, STREAM_PM, seed);
    const U4 r2 = philox4x32((uint32_t)(2 * q + 1), (uint32_t)v, gen, STREAM_PM, seed);
    if (u01(r1.x) < p_m) o1 = (float)clamp01(pm_apply((double)o1, (double)u01(r1.y), eta_m));
    if (u01(r2.x) < p_m) o2 = (float)clamp01(pm_apply((double)o2, (double)u01(r2.y), eta_m));
    Xo[(int64_t)(2 * q) * d + v] = o1;
    Xo[(int64_t)(2 * q + 1) * d + v] = o2;
  }
  __syncthreads();
  if (tb) trace_mark_any(pro.trace, 42);
  // Phase 3a: g of every child by a group of 8 lanes (strided partial sums + the pinned xor
  // butterfly, = dtlz_g), and the domain check; 256 threads = 32 children x 8 lanes
  static_assert(VARY_THREADS == 2 * VARY_PAIRS * G_LANES, "one 8-lane group per child");
  __shared__ double shG[2 * VARY_PAIRS];
  const int nch = 2 * npb;
  {
    const int cl = tid / G_LANES, l = tid % G_LANES;
    double p = 0.0;
    bool ok = true;
    if (cl < nch) {
      const float* x = Xo + (int64_t)(2 * q0 + cl) * d;
      p = dtlz_g_partial(problem, x, d, m, l);
      if (domain_flag)
        for (int v = l; v < d; v += G_LANES) ok = ok && (x[v] >= 0.0f) && (x[v] <= 1.0f);
    }
    p = p + __shfl_xor_sync(MO_FULL, p, 4, G_LANES);
    p = p + __shfl_xor_sync(MO_FULL, p, 2, G_LANES);
    p = p + __shfl_xor_sync(MO_FULL, p, 1, G_LANES);
    if (cl < nch && l == 0) shG[cl] = dtlz_g_finish(problem, p, d - m + 1);
    if (!ok) atomicOr(domain_flag, 1);
  }
  __syncthreads();
  if (tb) trace_mark_any(pro.trace, 43);
  // Phase 3b: one thread per (child, objective) for small m; from MO_VARY_FACTOR_M objectives on, the
  // factors of the running prefix products by all threads, then one thread per child folds them
  // (O(m) transcendentals per child instead of O(m^2), bit-identical)
  if (m >= MO_VARY_FACTOR_M && problem != 7) {
    // the factors (cos, sin or x, 1 - x of the first m-1 variables) of 32 variables at a time for every
    // child by all threads, then one thread per child extends its running prefix product over them
    __shared__ double shC[2 * VARY_PAIRS][32], shS[2 * VARY_PAIRS][32];
    double P = 0.0;
    const int cl0 = tid;   // the child this thread folds (tid < nch)
    if (cl0 < nch) P = problem == 1 ? 0.5 * (1.0 + shG[cl0]) : 1.0 + shG[cl0];
    for (int t0 = 0; t0 < m - 1; t0 += 32) {
      const int cw = min(32, m - 1 - t0);   // variables in this chunk
      for (int e = tid; e < nch * cw; e += VARY_THREADS) {
        const int cl = e / cw, u = e - cl * cw;
        double cf, sf;
        dtlz_factors(problem, Xo + (int64_t)(2 * q0 + cl) * d, t0 + u, shG[cl], cf, sf);
        shC[cl][u] = cf;
        shS[cl][u] = sf;
      }
      __syncthreads();
      if (cl0 < nch) {
        const int child = 2 * q0 + cl0;
        float* fo = Fo + (int64_t)child * m;
        for (int u = 0; u < 32 && t0 + u < m - 1; ++u) {
          const int j = m - 1 - (t0 + u);
          const float f = (float)(P * shS[cl0][u]);
          P = P * shC[cl0][u];
          fo[j] = f;
          if (ideal) {
            if (j < 16) atomic_min_float(&shMin[j], f);
            else atomic_min_float(&ideal[j], f);
          }
        }
        if (t0 + 32 >= m - 1) {   // last chunk: f_0 = the full product
          const float f = (float)P;
          fo[0] = f;
          if (ideal) atomic_min_float(&shMin[0], f);
        }
      }
      __syncthreads();
    }
  } else if (m > 16) {
    for (int cl = tid; cl < nch; cl += VARY_THREADS) {
      const int child = 2 * q0 + cl;
      float* fo = Fo + (int64_t)child * m;
      dtlz_eval_prefix(problem, Xo + (int64_t)child * d, m, shG[cl], [&](int j, float f) {
        fo[j] = f;
        if (ideal) {
          if (j < 16) atomic_min_float(&shMin[j], f);
          else atomic_min_float(&ideal[j], f);
        }
      });
    }
  }
  const int etasks = (m > 16 || (m >= MO_VARY_FACTOR_M && problem != 7)) ? 0 : nch * m;
  for (int e = tid; e < etasks; e += VARY_THREADS) {
    const int cl = e / m, j = e - cl * m;
    const int child = 2 * q0 + cl;
    const float* x = Xo + (int64_t)child * d;
    const float f = dtlz_eval_obj(problem, x, m, j, shG[cl]);
    Fo[(int64_t)child * m + j] = f;
    if (ideal) {
      if (j < 16) atomic_min_float(&shMin[j], f);
      else atomic_min_float(&ideal[j], f);
    }
  }
  if (ideal) {
    __syncthreads();
    if (tid < m && tid < 16) atomic_min_float(&ideal[tid], shMin[tid]);
  }
  if (tb) {
    __syncthreads();
    trace_mark_any(pro.trace, 44);
  }
}

__global__ void k_init_population(float* __restrict__ X, int64_t n, int d, uint64_t seed) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * d) return;
  int64_t i = t / d;
  int v = (int)(t - i * d);
  X[t] = u01(philox4x32((uint32_t)i, (uint32_t)v, 0u, STREAM_INIT, seed).x);
}

__global__ void k_dtlz_eval(int problem, const float* __restrict__ X, int64_t n, int d, int m,
                            float* __restrict__ F, int* __restrict__ domain_flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool ok = dtlz_eval_row(problem, X + i * d, d, m, F + i * m);
  if (!ok && domain_flag) atomicOr(domain_flag, 1);
}

__global__ void k_min_rows(const float* __restrict__ F, int64_t R, int m, float* __restrict__ ideal) {
  // column minima of F into ideal (running minimum); one thread per (row, column)
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= R * m) return;
  atomic_min_float(&ideal[t % m], F[t]);
}

int launch_vary_eval(int problem, const float* X, int64_t n, int d, int m, uint64_t seed, uint32_t gen,
                     const uint32_t* gen_ptr, const mo_var_cfg& cfg, float* Xo, float* Fo, float* ideal,
                     int* domain_flag, cudaStream_t s, const PrepArgs* pro) {
  if (n <= 0 || (n & 1) || d < m || m < 2) return MO_ERR_PARAM;
  if (problem < MO_DTLZ1 || problem > MO_DTLZ7) return MO_ERR_PARAM;
  const int pairs = (int)(n / 2);
  // pairs per block: 16, fewer when that would leave SMs idle (small n: spread the (pair, variable)
  // work; every block also pays the mating-shuffle keys, so no fewer than needed)
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int ppb = (int)ceil_div(pairs, 2 * (int64_t)sms);
  ppb = ppb < 1 ? 1 : (ppb > VARY_PAIRS ? VARY_PAIRS : ppb);
  const int vblocks = (int)ceil_div(pairs, ppb);
  int pblocks = 0;
  PrepArgs p;
  memset(&p, 0, sizeof(p));
  if (pro) {
    p = *pro;
    // one shuffle item (row, reference point or next generation's mating slot: ~74 dependent rounds)
    // per thread: the prologue CTAs are the kernel's critical path when they loop
    const int64_t items = (int64_t)pro->R + pro->w + (pro->mate ? n : 0);
    pblocks = (int)ceil_div(items, (int64_t)VARY_THREADS);
    pblocks = pblocks < 1 ? 1 : (pblocks > 296 ? 296 : pblocks);
  }
  k_vary_eval<<<(unsigned)(vblocks + pblocks), VARY_THREADS, 0, s>>>(problem, X, (int)n, d, m, seed, gen, gen_ptr,
                                                                     cfg, Xo, Fo, ideal, domain_flag, p, pblocks, ppb);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int launch_init_population(float* X, int64_t n, int d, uint64_t seed, cudaStream_t s) {
  if (n <= 0 || d <= 0) return MO_ERR_PARAM;
  int64_t tot = n * d;
  k_init_population<<<(unsigned)ceil_div(tot, 256), 256, 0, s>>>(X, n, d, seed);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int launch_dtlz_eval(int problem, const float* X, int64_t n, int d, int m, float* F, int* domain_flag,
                     cudaStream_t s) {
  if (n < 0 || d < m || m < 2) return MO_ERR_PARAM;
  if (problem < MO_DTLZ1 || problem > MO_DTLZ7) return MO_ERR_PARAM;
  if (n == 0) return MO_OK;
  k_dtlz_eval<<<(unsigned)ceil_div(n, 128), 128, 0, s>>>(problem, X, n, d, m, F, domain_flag);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

int launch_min_rows(const float* F, int64_t R, int m, float* ideal, cudaStream_t s) {
  if (R <= 0) return MO_OK;
  k_min_rows<<<(unsigned)ceil_div(R * m, 256), 256, 0, s>>>(F, R, m, ideal);
  MO_CHECK_LAUNCH();
  return MO_OK;
}

}  // namespace mo
