// Shared device/host helpers for the manyobj B200 engine (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/manyobj_b200.h"

#ifndef __CUDACC__
#error "mo_common.cuh is CUDA-only"
#endif

#define MO_WARP 32
#define MO_FULL 0xffffffffu
#define MO_RANK_UNRANKED (-2)
#define MO_RANK_DROPPED 0x7fffffff
#define MO_INF 0x7fffffff

// Launch-error check used by every entry point: converts a CUDA error to MO_ERR_CUDA.
#define MO_CHECK_LAUNCH()                                  \
  do {                                                     \
    cudaError_t e__ = cudaGetLastError();                  \
    if (e__ != cudaSuccess) return MO_ERR_CUDA;            \
  } while (0)

#define MO_TRY(expr)                                       \
  do {                                                     \
    int s__ = (expr);                                      \
    if (s__ != MO_OK) return s__;                          \
  } while (0)

namespace mo {

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Order-preserving map FP32 -> uint32 (total order for non-NaN values, -0 < +0 is fine here).
__device__ __forceinline__ uint32_t f2ord(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MO_FULL, v, o);
  return v;
}
// float min through integer atomics (non-negative floats order as ints, negative ones reversed as uints)
__device__ __forceinline__ void atomic_min_float(float* addr, float v) {
  if (v >= 0.0f)
    atomicMin(reinterpret_cast<int*>(addr), __float_as_int(v));
  else
    atomicMax(reinterpret_cast<unsigned*>(addr), __float_as_uint(v));
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t t = __shfl_xor_sync(MO_FULL, v, o);
    v = t < v ? t : v;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t t = __shfl_xor_sync(MO_FULL, v, o);
    v = t > v ? t : v;
  }
  return v;
}
__device__ __forceinline__ uint32_t warp_min_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(MO_FULL, v, o));
  return v;
}
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(MO_FULL, v, o));
  return v;
}

// Warp-aggregated histogram increment: lanes with equal `bin` elect one leader
// (__match_any_sync) that adds the group's population with a single atomic.
__device__ __forceinline__ void warp_agg_add(int* hist, int bin, bool active) {
  unsigned act = __ballot_sync(MO_FULL, active);
  if (!active) return;
  unsigned peers = __match_any_sync(act, bin);
  int leader = __ffs(peers) - 1;
  if ((int)lane_id() == leader) atomicAdd(hist + bin, __popc(peers));
}

// Warp-aggregated allocation from a global counter: every lane of the (full) warp
// calls it with its count (0 allowed); one atomic per warp; returns the lane's
// offset (only meaningful when cnt > 0).  Slot order within the counter is
// scheduling-dependent, so callers must not depend on it.
__device__ __forceinline__ int warp_alloc(int* ctr, int cnt) {
  const int lane = (int)lane_id();
  int x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(MO_FULL, x, o);
    if (lane >= o) x += t;
  }
  const int total = __shfl_sync(MO_FULL, x, 31);
  int base = 0;
  if (lane == 31 && total > 0) base = atomicAdd(ctr, total);
  base = __shfl_sync(MO_FULL, base, 31);
  return base + x - cnt;
}

// Block-wide exclusive scan of one int per thread (blockDim.x multiple of 32, <= 1024).
// `sh` must hold >= 33 ints.  Returns the exclusive prefix; *total gets the block sum.
__device__ __forceinline__ int block_excl_scan(int v, int* sh, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(MO_FULL, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < nw ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(MO_FULL, s, o);
      if (lane >= o) s += t;
    }
    if (lane < nw) sh[lane] = s;
    if (lane == 31) sh[32] = s;
  }
  __syncthreads();
  int res = x - v + (wid > 0 ? sh[wid - 1] : 0);
  *total = sh[32];
  __syncthreads();
  return res;
}

// Sense-reversing software grid barrier for persistent kernels launched with
// cudaLaunchAttributeCooperative (all CTAs co-resident).  `bar` = {count, gen}.
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid barrier for co-resident (cooperative) grids, self-resetting: bar[0] counts arrivals, bar[1] is
// the generation.  Arrival is one acq_rel atomic (it releases this CTA's writes -- ordered before it by
// the __syncthreads -- and acquires those of the earlier arrivals); the last arriver restores the count
// and bumps the generation with a release atomic; the others spin on an acquire load of the generation.
// (The previous fence + relaxed-atomic form paid two full MEMBAR.GPU on the critical path.)
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (gridDim.x == 1) return;
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire_gpu(bar + 1);
    unsigned arrived;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(bar) : "memory");
    if (arrived + 1u == gridDim.x) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
    } else {
      while (ld_acquire_gpu(bar + 1) == gen) __nanosleep(20);
    }
  }
  __syncthreads();
}

// "Last block out": true in exactly one block, the last to arrive; every other block's writes before
// its arrival are visible to it.  Nobody waits, so a final single-block phase starts as soon as the
// grid's work is done (no barrier release round trip) and the other blocks retire.  Shares the
// self-resetting count of grid_sync's slot (the last block restores 0).
// CONTRACT: grid_last must be the LAST use of `bar` in a launch.  The reset is a plain relaxed store
// and non-last blocks do not wait for it, so a later grid_sync / grid_last on the same slot in the
// same launch could count a stale arrival and release early.  Call sites (k_front_peel, k_prep) use
// it as their final synchronisation only.
__device__ __forceinline__ bool grid_last(unsigned* bar) {
  __shared__ int sLast;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned arrived;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(bar) : "memory");
    sLast = arrived + 1u == gridDim.x;
    if (sLast) asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
  }
  __syncthreads();
  return sLast != 0;
}

// Programmatic dependent launch (PDL): kernels of a generation are launched
// with cudaLaunchAttributeProgrammaticStreamSerialization, so the next
// kernel's CTAs are scheduled while the previous one drains.  pdl_wait()
// (griddepcontrol.wait) blocks until the previous grid has completed and its
// writes are visible -- every such kernel calls it before touching inputs;
// it is a no-op when the kernel was launched without the attribute.
// pdl_trigger() lets the dependent grid launch early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Set by mo_step / mo_step_phases / mo_niche_phases while they enqueue a
// generation (per host thread): the launchers then add the PDL attribute.
extern thread_local bool g_mo_pdl;

// Launch with optional cooperative / PDL attributes (cudaLaunchKernelEx).
template <typename... KArgs, typename... Args>
inline int launch_ex(void (*fn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool coop, bool pdl,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (coop) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (cudaLaunchKernelEx(&cfg, fn, static_cast<KArgs>(args)...) != cudaSuccess) return MO_ERR_CUDA;
  if (cudaGetLastError() != cudaSuccess) return MO_ERR_CUDA;
  return MO_OK;
}

// Phase trace for the persistent kernels: block 0 / thread 0 stamps the
// global nanosecond timer into tr[slot] (tr == nullptr: no-op).  Read back by
// the host (engine.Engine.trace()) to time phases inside one launch.
__device__ __forceinline__ void trace_mark_any(unsigned long long* tr, int slot) {   // any block
  if (tr != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[slot] = t;
  }
}

__device__ __forceinline__ void trace_mark(unsigned long long* tr, int slot) {
  if (tr != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[slot] = t;
  }
}

}  // namespace mo
