// Association on the 5th-generation tensor cores: tcgen05.mma (FP16 x FP16 -> FP32 in TMEM) as the
// FILTER of the full-scan argmax, exact canonical FP32 keys only where they can matter.
//
// Reference: niche.associate with the pinned key of DESIGN.md section 2 -- pi(f) =
// argmax_j t_j, t_j = ((f0 z0 + f1 z1) + ...) in separately rounded FP32, ties -> lowest shuffled
// position.  Same contract as k_assoc / k_assoc_hmma (k_niche.cu): the winner of every candidate row is
// merged into akey[row] with a 64-bit atomicMax of (ord(t) << 32 | ~position), bit-identical results.
//
// Filter (per row): with the exact power-of-two row scale 2^e putting max_k |f_k| in [1/2, 1) and FP16
// hi/lo splits x = h(x) + l(x) + O(2^-22 |x|) of f / 2^e and of z, the K dimension carries the three
// partial products side by side -- A = [h(f) | h(f) | l(f)], B = [h(z) | l(z) | h(z)], K = 3m padded to a
// multiple of 16 (one K16 tcgen05.mma step per 16) -- so t~ = sum h.h + h.l + l.h accumulates in FP32
// TMEM with |t~ - t/2^e| <= 2^-18.5 ||f/2^e|| (the dropped l.l and split residuals 2^-20, subnormal
// terms 2^-22, FP32 accumulation of <= 48 terms 2^-19, the canonical key's own rounding 2^-20).  eps =
// 2^-16 ||f/2^e|| (> 5x margin): the exact argmax j* and every exact tie satisfy t~ >= T* - eps >= max t~ -
// 2 eps, so a column is a candidate when t~ >= (running max of this thread's t~) - 2 eps.  Candidates are
// buffered in shared memory (value, column) and pruned against the final running max before their
// canonical keys are computed (a full buffer is pruned, then evaluated); rows with ||f|| = 0 or
// non-finite values go to the sliced FP32 fallback (fb_cand), as in the bf16 mma.sync filter.
//
// CTA (one per SM, warp-specialised, persistent over an equal contiguous share of the (256 candidate
// rows, reference tile) units, walked as segments of consecutive reference tiles of one row pair):
//   warp 0        producer: 1-D bulk copies (cp.async.bulk + mbarrier complete_tx) of the pre-packed
//                 reference tiles (128 directions x KS K16 steps of FP16, UMMA K-major no-swizzle
//                 core-matrix layout, 4 KB per step) into a shared-memory ring (a warm-up prefix of
//                 UA_WARM tiles is streamed twice: running maxima first, candidates after);
//   warp 1        TMEM owner (alloc 512 columns / dealloc) and MMA issuer: per reference tile and row
//                 tile KS tcgen05.mma.cta_group::1.kind::f16 M128 N128 K16 (the two row tiles share the
//                 B tile), tcgen05.commit to the ring slot's empty barrier and to the accumulator
//                 buffer's full barrier; two accumulator buffers (2 x 2 x 128 columns);
//   warps 2..17   epilogue in two groups of 8: group g takes the tiles whose running counter is g mod 2
//                 (TMEM buffer g), so the two groups' per-tile chains (mbarrier wait -> tcgen05.ld ->
//                 release -> FMNMX3 trees) overlap; a warp covers its TMEM lane quarter (warp % 4) and a
//                 64-column half of both row tiles, one row tile at a time (64 live values).
// Running maxima are seeded with the key of the reference point nearest to the row's simplex
// projection (ua_guess: the divisions of the Das-Dennis / two-layer set), so there is no warm-up pass
// and new maxima -- each one a candidate record -- are rare; without divisions an UA_WARM-tile warm-up
// pass runs first.  Measured at C3 (MO_UMMA_DEBUG timing modes): 2.29 ms with per-element candidates
// -> 1.57 ms (chunk records, one reference chunk per item, two groups, lattice seeds); the candidate
// work left is ~0.14 ms, the rest is the per-tile chain.  N = 64 with four buffers and two CTAs per SM
// measured slower.
#include <cuda_fp16.h>
#include <stdlib.h>
#include <cuda_runtime.h>

#include "mo_async.cuh"
#include "mo_common.cuh"
#include "k_niche_args.cuh"

namespace mo {

constexpr int UA_N = 128;                        // references per B tile (MMA N)
constexpr int UA_NBUF = 2;                       // accumulator buffers (2 row tiles x 128 columns each)
constexpr int UA_ROWS = 256;                     // candidate rows per item: two M = 128 row tiles
constexpr int UA_STEP_BYTES = UA_N * 16 * 2;     // 4 KB: 128 directions x K16 FP16 (one MMA K step)
constexpr int UA_A_STEP = 128 * 16 * 2;          // 4 KB: 128 rows x K16 FP16
constexpr int UA_GROUPS = 2;                     // epilogue groups: group g takes the tiles with counter % 2 == g
constexpr int UA_EPI_WARPS = 8 * UA_GROUPS;   // 10 warps: <= 3 per SM sub-partition, 168 registers each
constexpr int UA_EPI = UA_EPI_WARPS * 32;
constexpr int UA_THREADS = 64 + UA_EPI;
constexpr int UA_TMEM_COLS = 512;                // 2 buffers x 2 row tiles x 128 columns
constexpr int UA_NB = 4;                         // candidate chunks buffered per (thread, row tile)
constexpr int UA_RING_BYTES = 96 * 1024;
constexpr int UA_WARM = 32;                      // warm-up tiles per item (running maxima before candidates)
__host__ __device__ constexpr int ua_ks(int m) { return (3 * m + 15) / 16; }   // K16 steps for K = 3m
__host__ __device__ constexpr size_t ua_smem(int ks) {                         // > 114 KB: 1 CTA/SM
  return 1024 + 2 * (size_t)ks * UA_A_STEP + UA_RING_BYTES + 2 * (size_t)UA_NB * UA_EPI * 12;
}

// byte offset of element (row n, k) in a K-major no-swizzle tile of 8-row x 16-byte core matrices:
// LBO (next core matrix along K) = 128 B, SBO (next 8-row group) = 256 B
__host__ __device__ __forceinline__ int ua_off(int n, int k) { return (n >> 3) * 256 + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2; }

__device__ __forceinline__ uint64_t ua_desc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(128u >> 4) << 16;   // leading byte offset
  d |= (uint64_t)(256u >> 4) << 32;   // stride byte offset
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
  return d;                           // base offset 0, layout type 0 = SWIZZLE_NONE
}

// kind::f16 instruction descriptor: A = B = F16 (0), D = F32 (1), both K-major, N = 128, M = 128
constexpr uint32_t UA_IDESC = (1u << 4) | ((uint32_t)(UA_N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ void ua_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(UA_IDESC), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void ua_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void ua_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// 32 consecutive FP32 columns of this thread's TMEM lane (no wait: call ua_ld_wait before reading r)
__device__ __forceinline__ void ua_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void ua_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// max of 32 FP32 bit patterns as a depth-4 FMNMX3 tree (a serial chain would be 16 dependent ops)
__device__ __forceinline__ float max32(const uint32_t (&u)[32]) {
  float l1[11];
#pragma unroll
  for (int i = 0; i < 10; ++i)
    l1[i] = fmax3(__uint_as_float(u[3 * i]), __uint_as_float(u[3 * i + 1]), __uint_as_float(u[3 * i + 2]));
  l1[10] = fmaxf(__uint_as_float(u[30]), __uint_as_float(u[31]));
  const float a = fmax3(l1[0], l1[1], l1[2]), b = fmax3(l1[3], l1[4], l1[5]), c = fmax3(l1[6], l1[7], l1[8]);
  const float d = fmaxf(l1[9], l1[10]);
  return fmaxf(fmax3(a, b, c), d);
}

template <int M>
__device__ __forceinline__ float ua_canon_dot(const float (&f)[M], const float* z) {
  float t = __fmul_rn(f[0], __ldg(z));
#pragma unroll
  for (int k = 1; k < M; ++k) t = __fadd_rn(t, __fmul_rn(f[k], __ldg(z + k)));
  return t;
}

// packed reference tiles: [ntiles][KS x 4 KB] FP16 fragments (K position k' = part * m + kk: part 0 and 2
// hold h(z_kk), part 1 l(z_kk); zero past 3m), then colref[ntiles * 128] (reference index of every packed
// column, -1 = padding); `order` = packed column -> reference (a fixed random permutation)
__global__ void k_pack_refs_f16(const float* __restrict__ zhat, int64_t w, int m, const int32_t* __restrict__ order,
                                uint8_t* __restrict__ out) {
  const int ks = ua_ks(m), kt = 16 * ks;
  const int64_t ntiles = (w + UA_N - 1) / UA_N;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ntiles * UA_N * kt) return;
  const int64_t q = e / kt;   // packed column
  const int kp = (int)(e - q * kt);
  const int64_t j = q < w ? (order ? (int64_t)order[q] : q) : -1;
  __half v = __float2half_rn(0.0f);
  if (j >= 0 && kp < 3 * m) {
    const int part = kp / m, kk = kp - part * m;
    const float z = zhat[j * m + kk];
    const __half h = __float2half_rn(z);
    v = part == 1 ? __float2half_rn(__fsub_rn(z, __half2float(h))) : h;
  }
  const int64_t t = q / UA_N;
  const int n = (int)(q - t * UA_N);
  *reinterpret_cast<__half*>(out + (t * ks + kp / 16) * UA_STEP_BYTES + ua_off(n, kp & 15)) = v;
  if (kp == 0) reinterpret_cast<int32_t*>(out + ntiles * ks * UA_STEP_BYTES)[q] = (int32_t)j;
}

size_t pack_refs_f16_bytes(int64_t w, int m) {
  const int64_t ntiles = (w + UA_N - 1) / UA_N;
  return (size_t)ntiles * ((size_t)ua_ks(m) * UA_STEP_BYTES + UA_N * 4);
}

int launch_pack_refs_f16(const float* zhat, int64_t w, int m, const int32_t* order, void* out, cudaStream_t s) {
  if (w < 1 || m < 1 || m > 16 || !zhat || !out) return MO_ERR_PARAM;
  const int64_t n = (w + UA_N - 1) / UA_N * UA_N * 16 * ua_ks(m);
  k_pack_refs_f16<<<(unsigned)ceil_div(n, (int64_t)256), 256, 0, s>>>(zhat, w, m, order,
                                                                      static_cast<uint8_t*>(out));
  MO_CHECK_LAUNCH();
  return MO_OK;
}

template <int M>
__device__ __forceinline__ void ua_load_fn(const AssocArgs& a, int row, float (&fn)[M]) {
#pragma unroll
  for (int k = 0; k < M; ++k) {
    float v = a.F[(int64_t)row * M + k];
    if (a.ideal) v = __fsub_rn(v, a.ideal[k]);
    if (a.a32) v = __fdiv_rn(v, a.a32[k]);
    fn[k] = v;
  }
}

// canonical keys of the packed columns col0 + i, i in the bitmask `qm` (the columns of a 32-column chunk
// that were within 2 eps of the running maximum when the chunk was seen), for candidate row `row`
// (objectives re-read: only chunks still within 2 eps of the row's final running maximum get here)
template <int M>
__device__ __forceinline__ void ua_exact_cols(const AssocArgs& a, const int32_t* colref, int row, int col0,
                                              uint32_t qm, unsigned long long& best) {
  float fn[M];
  ua_load_fn<M>(a, row, fn);
  while (qm) {
    const int i = __ffs(qm) - 1;
    qm &= qm - 1u;
    const int j = __ldg(colref + col0 + i);
    if (j < 0) continue;
    const int p = __ldg(a.pos_ref + j);
    const float tk = ua_canon_dot<M>(fn, a.zs + (int64_t)p * M);
    const unsigned long long key = ((unsigned long long)f2ord(tk) << 32) | (uint32_t)(0xffffffffu - (uint32_t)p);
    best = key > best ? key : best;
  }
}

// Seed of a row's running maximum: the exact key (FP64) of the reference point nearest to the row's
// simplex projection u = f / sum(f) on the outer lattice (z = p / Ho) and on the inner layer (z = q /
// (2 Hi) + 1 / (2m)) of the Das-Dennis / two-layer set -- a point that exists in the set, so its
// canonical FP32 key is >= this value - 2^-18 ||f|| (FP32 rounding of the key and of the stored unit
// direction), and its filter value >= that / 2^e - eps: a valid running maximum from the first tile on
// (no warm-up pass, few new maxima later).  Returns 0 when unknown (f not finite / zero sum).
template <int M>
__device__ double ua_lattice_round(const double (&v)[M], int H, int (&p)[M]) {
  int sum = 0;
  double fr[M];
#pragma unroll
  for (int k = 0; k < M; ++k) {
    const double fl = floor(v[k]);
    p[k] = (int)fl;
    fr[k] = v[k] - fl;
    sum += p[k];
  }
  const int rem = H - sum;   // 0 <= rem < M: give +1 to the rem largest fractional parts
#pragma unroll
  for (int k = 0; k < M; ++k) {
    int rank = 0;
#pragma unroll
    for (int k2 = 0; k2 < M; ++k2) rank += (fr[k2] > fr[k]) || (fr[k2] == fr[k] && k2 < k);
    p[k] += rank < rem ? 1 : 0;
  }
  return 0.0;
}

template <int M>
__device__ double ua_guess(const float (&f)[M], int Ho, int Hi) {
  double S = 0.0;
#pragma unroll
  for (int k = 0; k < M; ++k) S += (double)f[k];
  if (!(S > 0.0) || !isfinite(S)) return 0.0;
  double best = 0.0;
  {
    double v[M];
    int p[M];
#pragma unroll
    for (int k = 0; k < M; ++k) v[k] = fmax(0.0, (double)f[k]) / S * Ho;
    ua_lattice_round<M>(v, Ho, p);
    double dot = 0.0, nn = 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const double z = (double)p[k] / Ho;
      dot += (double)f[k] * z;
      nn += z * z;
    }
    if (nn > 0.0) best = fmax(best, dot / sqrt(nn));
  }
  if (Hi > 0) {
    double v[M], sv = 0.0;
    int q[M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      v[k] = fmax(0.0, (2.0 * (double)f[k] / S - 1.0 / M) * Hi);
      sv += v[k];
    }
    if (sv > 0.0) {
#pragma unroll
      for (int k = 0; k < M; ++k) v[k] = v[k] * Hi / sv;
      ua_lattice_round<M>(v, Hi, q);
      double dot = 0.0, nn = 0.0;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const double z = (double)q[k] / (2.0 * Hi) + 1.0 / (2.0 * M);
        dot += (double)f[k] * z;
        nn += z * z;
      }
      if (nn > 0.0) best = fmax(best, dot / sqrt(nn));
    }
  }
  return best;
}

// next segment of a CTA's unit range: row tile pair rti, reference tiles [t0, t1); advances u
__device__ __forceinline__ void ua_segment(int64_t& u, int64_t u_end, int ntiles, int& rti, int& t0, int& t1) {
  rti = (int)(u / ntiles);
  t0 = (int)(u - (int64_t)rti * ntiles);
  t1 = (int)min((int64_t)ntiles, (int64_t)t0 + (u_end - u));
  u += t1 - t0;
}

template <int M>
__global__ void __launch_bounds__(UA_THREADS, 1) k_assoc_umma(AssocArgs a, int dbg) {
  constexpr int KS = ua_ks(M);
  constexpr int TILE = KS * UA_STEP_BYTES;          // one packed reference tile
  constexpr int ATILE = KS * UA_A_STEP;             // one row tile of A
  constexpr int STAGES = UA_RING_BYTES / TILE;
  pdl_wait();
  extern __shared__ __align__(1024) uint8_t ua_dyn[];
  __shared__ __align__(8) uint64_t sFull[STAGES], sEmpty[STAGES], sTFull[UA_NBUF], sTEmpty[UA_NBUF], sAReady;
  __shared__ uint32_t sTmem;
  if (__ldcg(a.info + MO_INFO_ERROR) != 0) return;
  if (__ldcg(a.info + MO_INFO_SKIPPED) != 0) return;
  const int ncand = __ldcg(a.ctl);
  const int nrt = (ncand + UA_ROWS - 1) / UA_ROWS;
  const int ntiles = (a.w + UA_N - 1) / UA_N;
  // this CTA's equal, contiguous share of the nrt x ntiles (row tile pair, reference tile) units,
  // walked as segments (row tile pair, reference tiles [t0, t1)); a row tile pair split between CTAs
  // merges its keys by the atomicMax below
  const int64_t units = (int64_t)nrt * ntiles;
  const int64_t u_begin = units * blockIdx.x / gridDim.x, u_end = units * (blockIdx.x + 1) / gridDim.x;
  if (u_begin >= u_end) return;   // CTA-uniform, before any barrier / TMEM use
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ua_dyn) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = base;                              // 2 row tiles x KS steps
  uint8_t* sB = base + 2 * ATILE;                  // ring
  float* sCV = reinterpret_cast<float*>(sB + UA_RING_BYTES);   // candidate chunks: max t~ [rt][NB][thread]
  int* sCC = reinterpret_cast<int*>(sCV + 2 * UA_NB * UA_EPI); // candidate chunks: first packed column
  uint32_t* sCM = reinterpret_cast<uint32_t*>(sCC + 2 * UA_NB * UA_EPI);   // qualifying columns of the chunk
  const uint8_t* tiles = static_cast<const uint8_t*>(a.zumma);
  const int32_t* colref = reinterpret_cast<const int32_t*>(tiles + (int64_t)ntiles * TILE);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&sFull[s], 1);
      mbar_init(&sEmpty[s], 1);
    }
    for (int b = 0; b < UA_NBUF; ++b) {
      mbar_init(&sTFull[b], 1);
      mbar_init(&sTEmpty[b], UA_EPI / UA_GROUPS);   // buffer b is drained by group b
    }
    mbar_init(&sAReady, UA_EPI);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&sTmem)),
                 "r"(UA_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sTmem;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int s = 0;
      unsigned ph = 0;
      for (int64_t u = u_begin; u < u_end;) {
        int rti, t0, t1;
        ua_segment(u, u_end, ntiles, rti, t0, t1);
        const int wu = a.ref_Ho > 0 ? 0 : min(UA_WARM, t1 - t0);
        for (int ti = 0; ti < wu + (t1 - t0); ++ti) {
          const int t = ti < wu ? t0 + ti : t0 + ti - wu;
          mbar_wait(&sEmpty[s], ph ^ 1u);
          mbar_expect_tx(&sFull[s], TILE);
          bulk_g2s(sB + (size_t)s * TILE, tiles + (int64_t)t * TILE, TILE, &sFull[s]);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int s = 0;
      unsigned ph = 0, aph = 0;
      int buf = 0;
      unsigned tph = 0;
      const uint32_t abase = smem_addr(sA), bbase = smem_addr(sB);
      for (int64_t u = u_begin; u < u_end;) {
        int rti, t0, t1;
        ua_segment(u, u_end, ntiles, rti, t0, t1);
        mbar_wait(&sAReady, aph);
        aph ^= 1u;
        tc_fence_after();
        const int wu = a.ref_Ho > 0 ? 0 : min(UA_WARM, t1 - t0);
        for (int ti = 0; ti < wu + (t1 - t0); ++ti) {
          mbar_wait(&sFull[s], ph);
          mbar_wait(&sTEmpty[buf], tph ^ 1u);
          tc_fence_after();
#pragma unroll
          for (int rt = 0; rt < 2; ++rt)
#pragma unroll
            for (int k = 0; k < KS; ++k)
              if (!(dbg & 2))   // debug timing: 2 = no MMA issue (commits only)
              ua_mma(tmem + (uint32_t)(buf * 2 + rt) * UA_N, ua_desc(abase + (uint32_t)(rt * ATILE + k * UA_A_STEP)),
                     ua_desc(bbase + (uint32_t)(s * TILE + k * UA_STEP_BYTES)), k > 0 ? 1u : 0u);
          ua_commit(&sEmpty[s]);
          ua_commit(&sTFull[buf]);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1u;
          }
          if (++buf == UA_NBUF) {
            buf = 0;
            tph ^= 1u;
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int et = threadIdx.x - 64;        // 0 .. UA_EPI-1
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int grp = (warp - 2) >> 3;        // tiles with global counter % UA_GROUPS == grp (its own buffer)
    const int cgp = ((warp - 2) >> 2) & 1;  // 64-column half of every 128-column accumulator
    const int r = q * 32 + lane;            // row within each row tile
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    int gt = 0;                             // tiles of all items so far (the MMA issuer's buffer counter)
    for (int64_t u = u_begin; u < u_end;) {
      int rti, t0, t1;
      ua_segment(u, u_end, ntiles, rti, t0, t1);
      const int rb = rti * UA_ROWS;
      int row[2];
      bool act[2];
      float marg[2], nrm[2];
      int escale[2];
#pragma unroll
      for (int rt = 0; rt < 2; ++rt) {
        const int c = rb + rt * 128 + r;
        act[rt] = c < ncand;
        row[rt] = act[rt] ? __ldcg(a.cand + c) : 0;
        float fn[M];
        ua_load_fn<M>(a, row[rt], fn);
        float nn = 0.0f, mx = 0.0f;
        bool fin = true;
#pragma unroll
        for (int k = 0; k < M; ++k) {
          fin = fin && isfinite(fn[k]);
          nn = fmaf(fn[k], fn[k], nn);
          mx = fmaxf(mx, fabsf(fn[k]));
        }
        const float norm = sqrtf(nn);
        const bool ok = fin && mx > 0.0f && isfinite(norm);
        if (act[rt] && !ok) {
          if (t0 == 0 && cgp == rt && grp == 0) {   // once per row: the segment with tile 0
            a.fb_cand[atomicAdd(a.fb_ctl, 1)] = row[rt];
            atomicAdd(const_cast<int*>(a.info) + MO_INFO_ASSOC_FALLBACK, 1);
          }
          act[rt] = false;
        }
        // the accumulators hold t~ / 2^e: the margin 2 eps = 2^-15 ||f|| / 2^e in the same units
        int e = 0;
        if (act[rt]) frexpf(mx, &e);
        marg[rt] = ldexpf(norm, -15 - e);
        escale[rt] = e;
        nrm[rt] = norm;
        if (cgp == rt && grp == 0) {   // row r of A tile rt: [h(f) | h(f) | l(f)] / 2^e, zero-padded
          __half hk[16 * KS];
#pragma unroll
          for (int kp = 0; kp < 16 * KS; ++kp) {
            __half v = __float2half_rn(0.0f);
            if (kp < 3 * M && act[rt]) {
              const int part = kp / M, kk = kp - part * M;
              const float x = ldexpf(fn[kk], -e);
              const __half h = __float2half_rn(x);
              v = part == 2 ? __float2half_rn(__fsub_rn(x, __half2float(h))) : h;
            }
            hk[kp] = v;
          }
          uint8_t* dst = sA + rt * ATILE;
#pragma unroll
          for (int k = 0; k < KS; ++k)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              uint32_t wv[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const __half2 h2 = __halves2half2(hk[k * 16 + hh * 8 + 2 * i], hk[k * 16 + hh * 8 + 2 * i + 1]);
                wv[i] = *reinterpret_cast<const uint32_t*>(&h2);
              }
              *reinterpret_cast<uint4*>(dst + k * UA_A_STEP + ua_off(r, hh * 8)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
            }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor core reads
      ua_arrive(&sAReady);
      float mxr[2] = {-__int_as_float(0x7f800000), -__int_as_float(0x7f800000)};
      if (a.ref_Ho > 0) {   // lattice seeds (see ua_guess): t_c >= g - 2^-18 |f|, t~ >= t_c / 2^e - eps
#pragma unroll
        for (int rt = 0; rt < 2; ++rt) {
          if (!act[rt]) continue;
          float fn[M];
          ua_load_fn<M>(a, row[rt], fn);
          const double g = ua_guess<M>(fn, a.ref_Ho, a.ref_Hi);
          if (g > 0.0) {
            // marg = 2 eps in filter units; the seed sits eps + 2^-18 |f| / 2^e below the point's key
            const double seed = g * (double)ldexpf(1.0f, -escale[rt]) - 0.5 * (double)marg[rt] -
                                (double)ldexpf(nrm[rt], -18 - escale[rt]);
            mxr[rt] = (float)seed - fabsf((float)seed) * 1e-6f;   // round down
          }
        }
      }
      int cnt[2] = {0, 0};
      unsigned long long best[2] = {0ull, 0ull};
      const int wu = a.ref_Ho > 0 ? 0 : min(UA_WARM, t1 - t0);
      for (int ti = 0; ti < wu + (t1 - t0); ++ti, ++gt) {
        if ((gt & (UA_GROUPS - 1)) != grp) continue;   // the other group's tile
        const bool warm = ti < wu || (dbg & 1);   // warm-up pass: running maxima only (dbg 1: always)
        const int t = warm ? t0 + ti : t0 + ti - wu;
        const int buf = gt & 1;
        const unsigned tph = (unsigned)(gt >> 1) & 1u;
        mbar_wait(&sTFull[buf], tph);
        tc_fence_after();
        // this thread's 64 columns of row tile 0, then of row tile 1 (two loads in flight each; 64 live
        // values); the buffer is released once both are in registers
#pragma unroll
        for (int rt = 0; rt < 2; ++rt) {
          uint32_t u[2][32];
#pragma unroll
          for (int h = 0; h < 2; ++h)
            ua_ld32(tmem + lane_addr + (uint32_t)(buf * 2 + rt) * UA_N + (uint32_t)(cgp * 64 + h * 32), u[h]);
          ua_ld_wait();
          if (rt == 1) {
            tc_fence_before();
            ua_arrive(&sTEmpty[buf]);
          }
          if (!act[rt]) continue;
          const float sm0 = max32(u[0]), sm1 = max32(u[1]);
          if (warm) {
            mxr[rt] = fmaxf(mxr[rt], fmaxf(sm0, sm1));
            continue;
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float s = h ? sm1 : sm0;
            if (s >= mxr[rt] - marg[rt]) {   // a column within 2 eps of the best seen: remember the chunk
              const float mn = fmaxf(mxr[rt], s), th = mn - marg[rt];
              uint32_t qm = 0;
#pragma unroll
              for (int i = 0; i < 32; ++i) qm |= (__uint_as_float(u[h][i]) >= th ? 1u : 0u) << i;
              if (cnt[rt] == UA_NB) {   // full: drop the chunks the new maximum excludes, evaluate the rest
                int kept = 0;
                for (int b2 = 0; b2 < UA_NB; ++b2) {
                  const int idx = (rt * UA_NB + b2) * UA_EPI + et;
                  if (sCV[idx] >= th) {
                    const int to = (rt * UA_NB + kept) * UA_EPI + et;
                    sCV[to] = sCV[idx];
                    sCC[to] = sCC[idx];
                    sCM[to] = sCM[idx];
                    ++kept;
                  }
                }
                if (kept == UA_NB) {
                  for (int b2 = 0; b2 < UA_NB; ++b2) {
                    const int idx = (rt * UA_NB + b2) * UA_EPI + et;
                    ua_exact_cols<M>(a, colref, row[rt], sCC[idx], sCM[idx], best[rt]);
                  }
                  kept = 0;
                }
                cnt[rt] = kept;
              }
              const int to = (rt * UA_NB + cnt[rt]) * UA_EPI + et;
              sCV[to] = s;
              sCC[to] = t * UA_N + cgp * 64 + h * 32;
              sCM[to] = qm;
              ++cnt[rt];
              mxr[rt] = mn;
            }
          }
        }
      }
#pragma unroll
      for (int rt = 0; rt < 2; ++rt) {
        if (!act[rt]) continue;
        const float th = mxr[rt] - marg[rt];
        for (int b = 0; b < cnt[rt]; ++b) {
          const int idx = (rt * UA_NB + b) * UA_EPI + et;
          if (sCV[idx] >= th) ua_exact_cols<M>(a, colref, row[rt], sCC[idx], sCM[idx], best[rt]);
        }
        if (best[rt]) atomicMax(&a.akey[row[rt]], best[rt]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(UA_TMEM_COLS) : "memory");
  }
}

int launch_assoc_umma(const AssocArgs& a, int m, int64_t R, cudaStream_t s) {
  if (R <= 0) return MO_OK;
  if (!a.zumma || m < 2 || m > 16 || a.zbeg != 0 || a.zend != a.w) return MO_ERR_PARAM;
  if (!a.in_step) {
    if (cudaMemsetAsync(a.fb_ctl, 0, sizeof(int), s) != cudaSuccess) return MO_ERR_CUDA;
    if (cudaMemsetAsync(const_cast<int*>(a.info) + MO_INFO_ASSOC_FALLBACK, 0, sizeof(int), s) != cudaSuccess)
      return MO_ERR_CUDA;
  }
  static int sms = 0;
  static bool attr[17] = {};
  static int dbg = -1;   // MO_UMMA_DEBUG (timing experiments only; results invalid when set)
  if (dbg < 0) {
    const char* e = getenv("MO_UMMA_DEBUG");
    dbg = e ? atoi(e) : 0;
  }
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const dim3 grid((unsigned)sms), blk(UA_THREADS);
  switch (m) {
#define MO_UA_CASE(MM)                                                                                      \
  case MM:                                                                                                  \
    if (!attr[MM]) {                                                                                        \
      if (cudaFuncSetAttribute(k_assoc_umma<MM>, cudaFuncAttributeMaxDynamicSharedMemorySize,              \
                               (int)ua_smem(ua_ks(MM))) != cudaSuccess)                                     \
        return MO_ERR_CUDA;                                                                                 \
      attr[MM] = true;                                                                                      \
    }                                                                                                       \
    MO_TRY(launch_ex(k_assoc_umma<MM>, grid, blk, ua_smem(ua_ks(MM)), s, false, g_mo_pdl, a, dbg));          \
    break;
    MO_UA_CASE(2) MO_UA_CASE(3) MO_UA_CASE(4) MO_UA_CASE(5) MO_UA_CASE(6) MO_UA_CASE(7) MO_UA_CASE(8)
    MO_UA_CASE(9) MO_UA_CASE(10) MO_UA_CASE(11) MO_UA_CASE(12) MO_UA_CASE(13) MO_UA_CASE(14)
    MO_UA_CASE(15) MO_UA_CASE(16)
#undef MO_UA_CASE
    default: return MO_ERR_PARAM;
  }
  return launch_assoc_fallback(a, m, s);
}

}  // namespace mo
