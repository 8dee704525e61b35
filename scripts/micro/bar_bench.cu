// Grid barrier (global atomics, as mo_common.cuh grid_sync) vs hardware cluster barrier cost.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
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
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__global__ void k_grid(unsigned* bar, int iters, int* data) {
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) data[blockIdx.x] += 1;
    grid_sync(bar);
  }
}
__global__ void k_cluster(int iters, int* data) {
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) data[blockIdx.x] += 1;
    cluster_sync();
  }
}
int main() {
  unsigned* bar; int* data;
  cudaMalloc(&bar, 8); cudaMalloc(&data, 4096 * 4);
  cudaMemset(bar, 0, 8); cudaMemset(data, 0, 4096 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000;
  for (int blocks : {8, 16, 32, 74, 148, 296}) for (int thr : {256, 512, 1024}) {
    void* args[] = {&bar, (void*)&iters, &data};
    cudaLaunchCooperativeKernel((void*)k_grid, blocks, thr, args, 0, 0);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_grid, blocks, thr, args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("grid    blocks %4d threads %4d : %7.3f us per barrier %s\n", blocks, thr, ms * 1e3 / iters, err ? cudaGetErrorString(err) : "");
  }
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) for (int thr : {256, 512, 1024}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs); cfg.blockDim = dim3(thr);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_cluster, iters, data);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k_cluster, iters, data);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("cluster size   %4d threads %4d : %7.3f us per barrier %s\n", cs, thr, ms * 1e3 / iters, err ? cudaGetErrorString(err) : "");
  }
  return 0;
}
